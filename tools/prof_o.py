"""cfg4 o projection (Tucker-2 R256, 8192 -> 5120) at M=8192: first-step strategy A/B."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
lay = S.make_layer("tucker", (5120, 8192), 1, (256, 256), seed=2)
pl = lay.plan(torch.bfloat16)
x = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
y = torch.empty(8192, 5120, device="cuda", dtype=torch.bfloat16)
ws = pl.workspace(8192)
for _ in range(3): pl.forward(x, out=y, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): pl.forward(x, out=y, ws=ws)
e1.record(); torch.cuda.synchronize()
print("o us:", e0.elapsed_time(e1) / 20 * 1e3)
