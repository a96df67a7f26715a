"""Plan-build time of the cfg4 stack, split by stage (TNL_BUILD_PROFILE=1 lines from libtnl) and by
projection kind. Usage: TNL_BUILD_PROFILE=1 python tools/build_profile.py [n_layers] 2> build.log"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200.mlp import TNMLP  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6
torch.cuda.init()
tot = {}
for l in range(n):
    kinds = Q.layer_kinds(l, 64) if n == 64 else Q.layer_kinds(l if l < 2 else 2 + l, 64)
    blk = {}
    for j, name in enumerate(("q", "k", "v", "o", "gate", "up", "down")):
        rows, cols = Q.SHAPES[name]
        t0 = time.perf_counter()
        lay = Q._tn(kinds[name], rows, cols, seed=40_000 + 100 * l + 10 * j)
        t1 = time.perf_counter()
        lay.plan(torch.bfloat16)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        k = f"{name}:{kinds[name]}"
        a = tot.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t1 - t0
        a[2] += t2 - t1
        blk[name] = lay
    t0 = time.perf_counter()
    TNMLP(blk["gate"], blk["up"], blk["down"])
    torch.cuda.synchronize()
    a = tot.setdefault("mlp_block", [0, 0.0, 0.0])
    a[0] += 1
    a[2] += time.perf_counter() - t0
for k, (c, h, d) in sorted(tot.items()):
    print(f"{k:24s} n={c:3d} host_gen={1e3 * h / c:8.1f} ms  plan={1e3 * d / c:8.1f} ms", flush=True)
