"""cfg2 decode sweep: M in {1..64} through the 70-layer bank, per-layer path vs fused stack path,
vs dense cuBLAS; CUDA-graph replays timed with events. Prints one JSON line per (M, path)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_01613_b200 as tnl
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack

ap = argparse.ArgumentParser()
ap.add_argument("--ms", default="1,2,4,8,16,32,64")
ap.add_argument("--copies", type=int, default=10)
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
bank = S.cfg2_bank(a.copies)
layers = [l for _, l in bank]
L = len(layers)


def graph_time(fn, iters):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


stack = TNStack(layers, torch.bfloat16)
plans = stack.plans
ws_dense = [torch.randn(5120, 5120, device="cuda").to(torch.bfloat16) for _ in range(L)]
for m in [int(t) for t in a.ms.split(",")]:
    x = torch.randn(m, 5120, device="cuda").to(torch.bfloat16)
    bufs = [torch.empty(m, 5120, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    ws = torch.zeros(max(p.workspace_bytes(m) for p in plans), dtype=torch.uint8, device="cuda")

    def per_layer():
        cur = x
        for i, p in enumerate(plans):
            p.forward(cur, out=bufs[i % 2], ws=ws)
            cur = bufs[i % 2]

    def fused():
        stack.forward(x, out=bufs[0])

    def dense():
        cur = x
        for i, w in enumerate(ws_dense):
            torch.matmul(cur, w.t(), out=bufs[i % 2])
            cur = bufs[i % 2]

    res = {}
    plans_gemv = [l.plan(torch.bfloat16, flags=tnl.PLAN_GEMV) for l in layers] if m <= 8 else None

    def gemv():
        cur = x
        for i, p in enumerate(plans_gemv):
            p.forward(cur, out=bufs[i % 2], ws=ws)
            cur = bufs[i % 2]

    paths = (("per_layer", per_layer), ("fused_stack", fused), ("dense_cublas", dense))
    if plans_gemv:
        paths = paths + (("gemv_per_layer", gemv),)
    for name, fn in paths:
        ms_ = graph_time(fn, a.iters)
        res[name] = ms_
        print(json.dumps({"M": m, "path": name, "ms_per_step": ms_, "us_per_layer": 1e3 * ms_ / L,
                          "tokens_per_s": m * L / (ms_ / 1e3)}), flush=True)
    print(json.dumps({"M": m, "speedup_fused_vs_dense": res["dense_cublas"] / res["fused_stack"]}), flush=True)
