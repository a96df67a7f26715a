"""ncu driver: one cfg3 gate TT r64 forward at M=8192 (cut plan), after a warm-up call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
fam, ms, rm, ranks = S.CFG3_GATE
layer = S.make_layer(fam, ms, rm, ranks, seed=30_064)
p = layer.plan(torch.bfloat16, flags=int(os.environ.get("FLAGS", "0")))
x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
y = p.forward(x)
y = p.forward(x)
torch.cuda.synchronize()
print("ok", p.info["plan_large_name"])
