"""ncu driver: cfg3 fused MLP block at M=8192 (two forwards)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
layers = [S.make_layer(*S.CFG3_GATE, seed=1), S.make_layer(*S.CFG3_GATE, seed=2), S.make_layer(*S.CFG3_DOWN, seed=3)]
mlp = TNMLP(*layers)
x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = mlp(x)
torch.cuda.synchronize()
print("ok", mlp.fused)
