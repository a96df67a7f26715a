"""Tucker-2 prefill: the fused on-chip chain (tnl_plan CHAIN -> tucker2_chain_kernel) vs the
merged-cut plan (two GEMM steps, T through HBM) vs the three-launch chain (TNL_TUCKER_FUSED=0 in
a subprocess), at the BASELINE Tucker-2 shapes, M = 8192. One JSON line per shape."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_01613_b200 as tnl  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

HBM = 6554.6e9
SHAPES = [("q", 8192, 5120, 256), ("o", 5120, 8192, 256), ("k/v", 1024, 5120, 128), ("cfg2 R64", 5120, 5120, 64),
          ("cfg2 R128", 5120, 5120, 128), ("cfg2 R256", 5120, 5120, 256), ("edge gate", 25600, 5120, 256),
          ("edge down", 5120, 25600, 256)]
only = os.environ.get("ONLY_FLAGS")
M = 8192


def time_plan(p, xs, y, ws, iters=20):
    for i in range(3):
        p.forward(xs[i % len(xs)], out=y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        p.forward(xs[i % len(xs)], out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, rows, cols, R in SHAPES:
    lay = S.make_layer("tucker", (rows, cols), 1, (R, R), seed=71_000 + rows + cols + R)
    xs = [torch.randn(M, cols, device="cuda").to(torch.bfloat16) for _ in range(2)]
    y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
    line = {"layer": name, "rows": rows, "cols": cols, "R": R, "M": M}
    byts = 2 * (tnl.param_count(lay) + M * (rows + cols))
    for flags, key in ((tnl.PLAN_CUT, "cut"), (tnl.PLAN_CHAIN, "chain")):
        if only and key not in only.split(","):
            continue
        p = lay.plan(torch.bfloat16, flags=flags)
        ms = time_plan(p, xs, y, p.workspace(M))
        line[key] = {"ms": ms, "GBps": byts / (ms / 1e3) / 1e9, "frac_hbm": byts / (ms / 1e3) / HBM}
    if not only:
        env = dict(os.environ, TNL_TUCKER_FUSED="0", ONLY_FLAGS="chain")
        out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
        for ln in out.stdout.splitlines():
            d = json.loads(ln)
            if d["layer"] == name:
                line["chain_3launch"] = d.get("chain")
    print(json.dumps(line), flush=True)
    if only:
        continue
