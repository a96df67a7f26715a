"""ncu driver: cfg1 TT (64,64,64,64) r32, M=16, fp32 generic chain, two forwards."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
lay = S.make_layer("tt", (64, 64, 64, 64), 2, (32, 32, 32), seed=1)
p = lay.plan(torch.float32)
x = torch.randn(16, 4096, device="cuda")
for _ in range(2):
    y = p.forward(x)
torch.cuda.synchronize()
print("ok", p.info["plan_small_name"])
