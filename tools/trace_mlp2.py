"""Epilogue phase timeline of the pair MLP kernel (CTA 0): gu_full wait -> TMEM loads -> math+st issue -> st wait -> arrive."""
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
t = buf.view(-1, 4).cpu().numpy().astype(np.int64)
e = t[256:512]
t0 = t[0, 0]
n = int((t[:256, 2] > 0).sum())
f = lambda v: round((v - t0) / 1e3, 3)
for i in list(range(0, 6)) + list(range(30, 40)):
    print(i, "mma", f(t[i, 0]), f(t[i, 1]), "| epi gu_full", f(t[i, 2]), "ld", f(e[i, 0]), "st_issued", f(e[i, 1]), "st_done", f(e[i, 2]), "arrived", f(t[i, 3]))
d = buf[2048:2048 + 8 * 128].view(-1, 8).cpu().numpy().astype(np.int64)
print("MMA loop: [pre-full, post-full, post-gu_empty | mma_d(j): pre-h, post-h, issued | producer load(j) issued]")
for i in list(range(0, 6)) + list(range(30, 40)):
    print(i, f(d[i, 0]), f(t[i, 0]), f(d[i, 1]), "|", f(d[i, 2]), f(d[i, 3]), f(d[i, 4]), "| load", f(d[i, 5]))
