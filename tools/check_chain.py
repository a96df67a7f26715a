"""Cluster-resident decode chain (tnl_chain_forward) vs the kernel-per-boundary stack path and
the float64 oracle chain; timing of both on the cfg2 bank."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack

torch.manual_seed(0)
layers = [S.make_layer(f, ms, rm, rk, seed=20_000 + 100 * i) for i, (_, f, ms, rm, rk) in enumerate(S.CFG2_VARIANTS)]
a = TNStack(layers, torch.bfloat16, cluster=True)
b = TNStack(layers, torch.bfloat16, cluster=False)
print("chain handle:", a.chain, flush=True)
assert a.chain is not None
for m in (1, 5, 16, 17, 32):
    x = torch.randn(m, 5120, device="cuda").to(torch.bfloat16)
    ya = a.forward(x)
    yb = b.forward(x)
    torch.cuda.synchronize()
    d = float((ya.float() - yb.float()).norm() / yb.float().norm())
    rep = all(torch.equal(a.forward(x), ya) for _ in range(20))
    print(f"M={m}: rel diff chain vs stack {d:.3e}; finite {bool(torch.isfinite(ya).all())}; bitwise repeatable {rep}", flush=True)

bank = S.cfg2_bank(int(os.environ.get("COPIES", "10")))
bl = [l for _, l in bank]
for cl in (False, True):
    st = TNStack(bl, torch.bfloat16, cluster=cl)
    st.capture(64, host_io=False, microbatches=2)
    for _ in range(5):
        st.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 100
    print(f"cluster={cl}: {ms * 1e3:.1f} us/step, {64 * len(bl) / ms / 1e3 / 1e6:.2f} M tokens/s", flush=True)

# timeline of one pass (M=32) through the bank: clock64 stamps per layer, CTA 0
import ctypes
from paper_2602_01613_b200 import _native as N
st = TNStack(bl, torch.bfloat16, cluster=True)
buf = torch.zeros(16 * 256 * 16, dtype=torch.int64, device="cuda")
N.check(N.load().tnl_chain_set_trace(st.chain, ctypes.c_void_p(buf.data_ptr())))
x = torch.randn(32, 5120, device="cuda").to(torch.bfloat16)
for _ in range(3):
    st.forward(x)
torch.cuda.synchronize()
tr = buf.view(16, 256, 16).cpu().numpy()
EVN = ["mma:xready", "mma:A_issued", "mma:tready", "mma:B_issued", "epi:adone", "own:rsfull", "epi:bdone", "epi:x_done",
       "mma:fence_done", "epi:x_stored", "epi:x_fenced", "epi:rs_sent", "own:ag_sent", "prod:B_first_push",
       "prod:B_last_push", "mma:B_first_landed"]
for c in (0, 15):
    print(f"CTA {c}: cycles per layer (mean of layers 2..{len(bl)-2}) between events")
    t = tr[c, :len(bl)]
    per = np.diff(t[:, 0])
    print("  layer period (xready->xready):", np.round(per[:14]).astype(int).tolist())
    for l in range(0, 8):
        print("  L%d " % l + " ".join(f"{EVN[e]}={t[l, e] - t[l, 0]}" for e in range(16)))
