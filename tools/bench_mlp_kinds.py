"""cfg4 MLP blocks by kind at M = 8192 (graph-timed): TT r64 / TR4 (the on-chip middle kernel) and
Tucker-4 / Tucker-2 R256 (the dual SiLU kernel). One JSON line per kind."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200.mlp import TNMLP  # noqa: E402

M = 8192
xs = [torch.randn(M, Q.HIDDEN, device="cuda").to(torch.bfloat16) for _ in range(4)]
for kind in ("tt64", "tr4", "tucker4", "tucker2-256"):
    g = Q._tn(kind, Q.FFN, Q.HIDDEN, seed=1)
    u = Q._tn(kind, Q.FFN, Q.HIDDEN, seed=2)
    d = Q._tn(kind, Q.HIDDEN, Q.FFN, seed=3)
    mlp = TNMLP(g, u, d)
    y = torch.empty(M, Q.HIDDEN, device="cuda", dtype=torch.bfloat16)
    ws = mlp.workspace(M)
    it = [0]

    def step():
        mlp.forward(xs[it[0] % 4], out=y, ws=ws)
        it[0] += 1

    step()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(4):
            step()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"kind": kind, "fused": bool(mlp.fused), "ms": round(e0.elapsed_time(e1) / 20, 4),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("TNL_")}}), flush=True)
    mlp.close()
