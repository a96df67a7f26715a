"""cfg3 at r in {32, 64, 128}: gate / down projections and the MLP block at
M = 8192 (bf16), each with its HBM / chain-flop roofline, and whether the block ran fused."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_01613_b200 as tnl  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402
from paper_2602_01613_b200.mlp import TNMLP  # noqa: E402

HBM, TC = 6549.1e9, 1624e12
M = 8192
xs = [torch.randn(M, 5120, device="cuda").to(torch.bfloat16) for _ in range(2)]


def timeit(fn, iters=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for r in (32, 64, 128):
    g = S.make_layer("tt", (160, 160, 64, 80), 2, (r, r, r), seed=33_000 + r)
    u = S.make_layer("tt", (160, 160, 64, 80), 2, (r, r, r), seed=33_100 + r)
    d = S.make_layer("tt", (64, 80, 160, 160), 2, (r, r, r), seed=33_200 + r)
    line = {"r": r, "M": M}
    for name, lay in (("gate", g), ("down", d)):
        rows, cols = lay.matrix_shape
        p = lay.plan(torch.bfloat16)
        y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
        xin = [torch.randn(M, cols, device="cuda").to(torch.bfloat16) for _ in range(2)]
        ws = p.workspace(M)
        ms = timeit(lambda i: p.forward(xin[i % 2], out=y, ws=ws))
        byts = 2 * (tnl.param_count(lay) + M * (rows + cols))
        flops = M * lay.chain_flops_per_token()
        t_roof = max(byts / HBM, flops / TC)
        line[name] = {"ms": round(ms, 4), "frac_roofline": round(t_roof / (ms / 1e3), 3), "plan": p.info["plan_large_name"]}
    mlp = TNMLP(g, u, d)
    y = torch.empty(M, 5120, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda i: mlp.forward(xs[i % 2], out=y))
    P = sum(tnl.param_count(l) for l in (g, u, d))
    F = M * sum(l.chain_flops_per_token() for l in (g, u, d))
    t_roof = max(2 * (P + M * 2 * 5120) / HBM, F / TC)
    line["mlp_block"] = {"ms": round(ms, 4), "fused": mlp.fused, "t_roofline_ms": round(1e3 * t_roof, 4),
                         "frac_roofline": round(t_roof / (ms / 1e3), 3)}
    print(json.dumps(line), flush=True)
