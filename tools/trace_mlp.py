"""Per-chunk timeline of CTA (0,0) of the fused MLP middle kernel (cfg3, M=8192)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_01613_b200 import _native as N, synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
M = int(os.environ.get("M", "8192"))
layers = [S.make_layer(*S.CFG3_GATE, seed=1), S.make_layer(*S.CFG3_GATE, seed=2), S.make_layer(*S.CFG3_DOWN, seed=3)]
mlp = TNMLP(*layers)
buf = torch.zeros(32 * 1024, dtype=torch.int64, device="cuda")
N.check(N.load().tnl_plan_set_trace(mlp.plans[0].handle, ctypes.c_void_p(buf.data_ptr())))
x = torch.randn(M, 5120, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = mlp(x)
torch.cuda.synchronize()
t = buf.view(-1, 4).cpu().numpy().astype(np.int64)
n = int((t[:, 0] > 0).sum())
t0 = t[0, 0]
print("chunks", n)
for i in list(range(0, min(n, 8))) + list(range(max(8, n - 4), n)):
    print(i, [(t[i, k] - t0) / 1e3 for k in range(4)])
e = buf.view(-1, 4).cpu().numpy().astype(np.int64)[256:256 + n]
for i in (1, 2, 3, n - 2):
    print("epi", i, "gu_full", (t[i, 2] - t0) / 1e3, "h_empty_ok", (e[i, 2] - t0) / 1e3, "tmem_done", (e[i, 0] - t0) / 1e3,
          "sts_done", (e[i, 1] - t0) / 1e3, "h_full", (t[i, 3] - t0) / 1e3)
d = np.diff(t[:n, 0]) / 1e3
print("mean us per chunk (mma start)", d.mean(), "epi span", ((t[:n, 3] - t[:n, 2]) / 1e3).mean())
# MMA-warp detail (pair kernel): [before full wait, after full+gu_empty waits, mma_d: before h wait, after h wait, after D issue]
d = buf[2048:2048 + 8 * 128].view(-1, 8).cpu().numpy().astype(np.int64)
for i in list(range(0, 6)) + list(range(38, 44)):
    print("mma", i, [round((d[i, k] - t0) / 1e3, 3) for k in range(5)])
