"""ncu driver: Tucker-2 R256 gate/up/down MLP block (dual path) at M=8192, two forwards."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
g = S.make_layer("tucker", (25600, 5120), 1, (256, 256), seed=1)
u = S.make_layer("tucker", (25600, 5120), 1, (256, 256), seed=2)
d = S.make_layer("tucker", (5120, 25600), 1, (256, 256), seed=3)
mlp = TNMLP(g, u, d)
x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = mlp(x)
torch.cuda.synchronize()
print("ok", mlp.fused)
