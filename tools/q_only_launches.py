import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2602_01613_b200 import qwen_stack as Q
lay = Q._tn("tucker2-256", Q.QDIM, Q.HIDDEN, seed=5)
p = lay.plan(torch.bfloat16)
x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
for _ in range(2): y = p.forward(x)
torch.cuda.synchronize(); print("ok")
