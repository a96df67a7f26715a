"""Timeline of the decode kernels (per-CTA %globaltimer stamps) in a graph-replayed chain."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_01613_b200 import _native as N
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--variants", default="2,2,2,0,0,0")
ap.add_argument("--cycles", action="store_true", help="library built with -DTNL_TRACE_CLOCK: stamps are SM cycles, "
                "reported relative to each CTA's pdl_passed")
a = ap.parse_args()
vs = [int(t) for t in a.variants.split(",")]
layers = []
for i, v in enumerate(vs):
    name, fam, ms, rm, ranks = S.CFG2_VARIANTS[v]
    layers.append(S.make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * i))
st = TNStack(layers, torch.bfloat16)
bufs = []
lib = N.load()
for p in st.plans:
    b = torch.zeros(2 * 1024 * 16, dtype=torch.int64, device="cuda")
    N.check(lib.tnl_plan_set_trace(p.handle, ctypes.c_void_p(b.data_ptr())))
    bufs.append(b)
st.capture(a.m, host_io=False)
for _ in range(3):
    st.replay()
torch.cuda.synchronize()
for b in bufs:
    b.zero_()
st.replay()
torch.cuda.synchronize()
EV = ["start", "setup", "w_issued", "pdl_passed", "mma_first", "mma_issued", "epi_pdl", "act_ready", "done", "stored", "end"]
EVF = ["start", "setup", "w_issued", "pdl_passed", "T_landed", "T_converted", "B_done", "x_ready", "A_done", "reds_issued", "end",
       "epi_pdl", "stg0", "stg_last", "conv0_done", "mma_has_last"]
t0 = None
for li, (v, b) in enumerate(zip(vs, bufs)):
    arr = b.view(2, 1024, 16).cpu().numpy()
    for ph in range(2):
        blk = arr[ph]
        used = blk[:, 0] > 0
        if not used.any():
            continue
        blk = blk[used].astype(np.int64)
        if a.cycles and ph == 1 and li + 1 < len(vs):
            ref = blk[:, 3].copy()
            for e in range(blk.shape[1]):
                blk[:, e] = np.where(blk[:, e] > 0, blk[:, e] - ref + 10**9, 0)
            row = []
            for e, nm in enumerate(EVF):
                col = blk[:, e]
                col = col[col > 0] - 10**9
                if len(col):
                    row.append(f"{nm}={int(col.min())}/{int(np.median(col))}/{int(col.max())}")
            print(f"L{li} v{v} fused-cycles ctas={used.sum()}: " + " ".join(row))
            continue
        if a.cycles:
            continue
        if t0 is None:
            t0 = blk[:, 0].min()
        row = []
        names = EVF if (ph == 1 and li + 1 < len(vs)) else EV
        for e, nm in enumerate(names):
            col = blk[:, e]
            col = col[col > 0]
            if len(col) == 0:
                continue
            if nm.endswith("cycles"):
                row.append(f"{nm}={int(col.min())}/{int(np.median(col))}/{int(col.max())}")
                continue
            row.append(f"{nm}={(col.min()-t0)/1e3:.2f}/{(np.median(col)-t0)/1e3:.2f}/{(col.max()-t0)/1e3:.2f}")
        kind = "fused" if (ph == 1 and li + 1 < len(vs)) else "phase" + "AB"[ph]
        print(f"L{li} v{v} {kind} ctas={used.sum()}: " + " ".join(row))
