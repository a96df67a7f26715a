"""bf16 core-by-core chain (TNL_PLAN_CHAIN: fused chain kernels where they exist, tcgen05 strided
contraction steps elsewhere) vs the default merged-cut plan, at the BASELINE layer shapes and
M in {1, 64, 8192}. One JSON line per (layer, M): ms per forward of each plan, kernel launches per
forward, and the weight bytes each plan streams (cores vs pre-contracted panels)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_01613_b200 as tnl  # noqa: E402
from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

LAYERS = [(n, S.make_layer(f, ms, rm, rk, seed=72_000 + i)) for i, (n, f, ms, rm, rk) in enumerate(S.CFG2_VARIANTS)]
LAYERS += [("cfg3 gate tt r64", S.make_layer(*S.CFG3_GATE, seed=72_100)),
           ("cfg3 down tt r64", S.make_layer(*S.CFG3_DOWN, seed=72_101))]
LAYERS += [(f"cfg4 gate {k}", Q._tn(k, Q.FFN, Q.HIDDEN, seed=72_200 + i)) for i, k in enumerate(("tr4", "tucker4"))]


def time_plan(p, x, y, ws, iters=20):
    for _ in range(3):
        p.forward(x, out=y, ws=ws)
    torch.cuda.synchronize()
    tnl.launch_count(reset=True)
    p.forward(x, out=y, ws=ws)
    launches = tnl.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        p.forward(x, out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters, launches


for name, lay in LAYERS:
    rows, cols = lay.matrix_shape
    for m in (1, 64, 8192):
        x = torch.randn(m, cols, device="cuda").to(torch.bfloat16)
        y = torch.empty(m, rows, device="cuda", dtype=torch.bfloat16)
        line = {"layer": name, "rows": rows, "cols": cols, "M": m, "core_bytes_bf16": 2 * tnl.param_count(lay)}
        for flags, key in ((tnl.PLAN_AUTO, "cut"), (tnl.PLAN_CHAIN, "chain")):
            p = lay.plan(torch.bfloat16, flags=flags)
            ms, n = time_plan(p, x, y, p.workspace(m))
            line[key] = {"ms": round(ms, 4), "launches": n, "plan": p.info["plan_large_name"]}
        line["chain_over_cut"] = round(line["chain"]["ms"] / line["cut"]["ms"], 2)
        print(json.dumps(line), flush=True)
