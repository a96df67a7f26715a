"""A/B timing of prefill projections at M=8192 (CUDA events, 20 iterations, two input buffers >
L2): the cfg4 q / o / k / Tucker-4 gate / down and the cfg3 TT r64 gate. Prints one JSON line;
TNL_LIB_AB selects an alternative in-tree build."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

M = 8192
specs = {"q": ("tucker2-256", Q.QDIM, Q.HIDDEN), "o": ("tucker2-256", Q.HIDDEN, Q.QDIM),
         "k": ("tucker2-128", Q.KVDIM, Q.HIDDEN), "gate_t4": ("tucker4", Q.FFN, Q.HIDDEN),
         "down_t4": ("tucker4", Q.HIDDEN, Q.FFN), "gate_edge": ("tucker2-256", Q.FFN, Q.HIDDEN)}
out = {"lib": os.environ.get("TNL_LIB_AB", "default")}
for name, (kind, rows, cols) in list(specs.items()) + [("cfg3_gate", (None, None, None))]:
    lay = S.make_layer(*S.CFG3_GATE, seed=5) if kind is None else Q._tn(kind, rows, cols, seed=5)
    rows, cols = lay.matrix_shape
    p = lay.plan(torch.bfloat16)
    xs = [torch.randn(M, cols, device="cuda").to(torch.bfloat16) for _ in range(2)]
    y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
    ws = p.workspace(M)
    for i in range(3):
        p.forward(xs[i % 2], out=y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        p.forward(xs[i % 2], out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    del xs, y
print(json.dumps(out), flush=True)
