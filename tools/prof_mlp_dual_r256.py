"""cfg4 edge-layer MLP (Tucker-2 R256 gate/up/down, dual path) at M=8192: timing + launch list driver."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
M = 8192
lays = [S.make_layer("tucker", sh, 1, (256, 256), seed=61_000 + i) for i, sh in
        enumerate([(25600, 5120), (25600, 5120), (5120, 25600)])]
mlp = TNMLP(*lays)
x = torch.randn(M, 5120, device="cuda").to(torch.bfloat16)
y = torch.empty(M, 5120, device="cuda", dtype=torch.bfloat16)
ws = mlp.workspace(M)
for _ in range(3):
    mlp.forward(x, out=y, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    mlp.forward(x, out=y, ws=ws)
e1.record(); torch.cuda.synchronize()
print("dual MLP R256 us:", e0.elapsed_time(e1) / 10 * 1e3, "fused", mlp.fused)
