"""cfg3 prefill: Qwen3-32B MLP TT projections at M=8192 (bf16), vs dense cuBLAS.

Prints one JSON object per layer/plan: time, tokens/s, algorithmic GB/s, % of HBM peak,
chain TFLOP/s. Inputs (M x 5120 or M x 25600 bf16) exceed... no: 84 MB < L2; each
timed iteration rotates through 4 distinct input buffers (336 MB > 126 MB L2).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_01613_b200 as tnl
from paper_2602_01613_b200 import synthetic as S

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=8192)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--ranks", default="64")
ap.add_argument("--plans", default="0")
a = ap.parse_args()
HBM, TC = 6554.6, 1635.0


def timeit(fn, iters):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


M = a.m
for r in [int(t) for t in a.ranks.split(",")]:
    for which, (fam, ms, rm, _) in (("gate", S.CFG3_GATE), ("down", S.CFG3_DOWN)):
        layer = S.make_layer(fam, ms, rm, (r, r, r), seed=30_000 + r)
        rows, cols = layer.matrix_shape
        xs = [torch.randn(M, cols, device="cuda").to(torch.bfloat16) for _ in range(4)]
        for flags in [int(t) for t in a.plans.split(",")]:
            p = layer.plan(torch.bfloat16, flags=flags)
            y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
            ws = p.workspace(M)
            ms_ = timeit(lambda i: p.forward(xs[i % 4], out=y, ws=ws), a.iters)
            byts = 2 * (tnl.param_count(layer) + M * (rows + cols))
            fl = M * layer.chain_flops_per_token()
            print(json.dumps({"layer": f"{which} TT r{r}", "plan": p.info["plan_large_name"], "flags": flags,
                              "M": M, "ms": ms_, "tokens_per_s": M / (ms_ / 1e3),
                              "alg_GBps": byts / (ms_ / 1e3) / 1e9, "frac_hbm": byts / (ms_ / 1e3) / 1e9 / HBM,
                              "chain_TFLOPs": fl / (ms_ / 1e3) / 1e12,
                              "t_roof_us": 1e6 * max(byts / (HBM * 1e9), fl / (TC * 1e12))}), flush=True)
        # dense cuBLAS of the uncompressed weight
        w = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
        yd = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
        msd = timeit(lambda i: torch.matmul(xs[i % 4], w.t(), out=yd), a.iters)
        print(json.dumps({"layer": f"{which} dense cuBLAS", "M": M, "ms": msd, "tokens_per_s": M / (msd / 1e3),
                          "TFLOPs": 2 * M * rows * cols / (msd / 1e3) / 1e12}), flush=True)
        del xs, w, yd
