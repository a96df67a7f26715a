"""cfg4: Qwen3-32B-shaped 64-layer mixed-TN stack — decode (M=1, 64) and prefill (M=8192).

Prints JSON lines: tokens/s through the whole stack, params, chain flops, roofline time.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_01613_b200.qwen_stack import QwenTNStack

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=64)
ap.add_argument("--ms", default="1,64,8192")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--unfused-mlp", action="store_true")
ap.add_argument("--serial-kv", action="store_true", help="k/v on the main stream (no fork)")
ap.add_argument("--no-fuse-qo", action="store_true", help="decode: q and o as two tnl_forward calls")
ap.add_argument("--no-fold", action="store_true", help="prefill: separate residual-add + RMSNorm passes")
ap.add_argument("--microbatches", type=int, default=2, help="decode: concurrent token groups (M <= 64)")
a = ap.parse_args()
HBM, TC = 6554.6e9, 1635e12

t0 = time.time()
st = QwenTNStack(a.layers, fused_mlp=not a.unfused_mlp)
st.concurrent_kv = not a.serial_kv
st.fuse_qo = not a.no_fuse_qo
st.fold_prefill = not a.no_fold
build_s = time.time() - t0
P = st.param_count()
F = st.chain_flops_per_token()
print(json.dumps({"layers": a.layers, "projections": 7 * a.layers, "params": P, "chain_flops_per_token": F,
                  "build_s": build_s, "fused_mlp_blocks": st.fused_mlp_count()}), flush=True)
for m in [int(t) for t in a.ms.split(",")]:
    g = st.capture(m, microbatches=a.microbatches)
    st.x.normal_()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    byts = 2 * (P + m * sum(r + c for _, lay, _ in st.projections() for r, c in [lay.matrix_shape]))
    t_roof = max(byts / HBM, m * F / TC)
    print(json.dumps({"M": m, "ms_per_pass": ms, "tokens_per_s": m / (ms / 1e3), "t_roofline_ms": 1e3 * t_roof,
                      "frac_roofline": 1e3 * t_roof / ms, "finite": bool(torch.isfinite(st.x).all())}), flush=True)
    del g
    torch.cuda.empty_cache()
