"""ncu driver: one decode pass (M=32) through a 7-layer cfg2 chain via tnl_stack_forward."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack
layers = [S.make_layer(f, ms, rm, rk, seed=20_000 + 100 * i) for i, (_, f, ms, rm, rk) in enumerate(S.CFG2_VARIANTS)]
st = TNStack(layers, torch.bfloat16)
x = torch.randn(int(os.environ.get("M", "32")), 5120, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = st.forward(x)
torch.cuda.synchronize()
print("ok", y.shape)
