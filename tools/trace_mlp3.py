"""MMA-warp cycle breakdown of the pair MLP kernel (CTA pair 0)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_01613_b200 import _native as N, synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
layers = [S.make_layer(*S.CFG3_GATE, seed=1), S.make_layer(*S.CFG3_GATE, seed=2), S.make_layer(*S.CFG3_DOWN, seed=3)]
mlp = TNMLP(*layers)
buf = torch.zeros(32 * 1024, dtype=torch.int64, device="cuda")
N.check(N.load().tnl_plan_set_trace(mlp.plans[0].handle, ctypes.c_void_p(buf.data_ptr())))
x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = mlp(x)
torch.cuda.synchronize()
a = buf[4096:4104].cpu().numpy()
names = ["wait full", "wait gu_empty", "issue G/U+commit", "wait h_full", "issue D+commits", "loop/other"]
tot = a[:6].sum()
for n, v in zip(names, a[:6]):
    print(f"{n:18s} {v:9d} cyc  {100*v/tot:5.1f}%")
print("total", tot, "cycles")
