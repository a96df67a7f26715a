"""Order effect probe: the ab_prefill layer sequence, then cfg3 gate timed 10 x 20 iterations with
the SM clock / throttle reasons sampled (bench.ClockSampler) — is the occasional 2.5x slow cfg3 gate
a clock / power effect or a placement effect?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

M = 8192
keep = []
for kind, rows, cols in (("tucker2-256", Q.QDIM, Q.HIDDEN), ("tucker2-256", Q.HIDDEN, Q.QDIM), ("tucker4", Q.FFN, Q.HIDDEN),
                         ("tucker4", Q.HIDDEN, Q.FFN)):
    lay = Q._tn(kind, rows, cols, seed=5)
    p = lay.plan(torch.bfloat16)
    x = torch.randn(M, cols, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
    for _ in range(20):
        p.forward(x, out=y)
    torch.cuda.synchronize()
    if os.environ.get("KEEP"):
        keep.append((lay, p, x, y))
    del x, y
lay = S.make_layer(*S.CFG3_GATE, seed=5)
p = lay.plan(torch.bfloat16)
xs = [torch.randn(M, 5120, device="cuda").to(torch.bfloat16) for _ in range(2)]
y = torch.empty(M, 25600, device="cuda", dtype=torch.bfloat16)
ws = p.workspace(M)
cs = bench.ClockSampler(0)
cs.start()
res = []
for rep in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        p.forward(xs[i % 2], out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1) / 20 * 1e3, 1))
clk = cs.stop()
print(json.dumps({"keep": bool(os.environ.get("KEEP")), "us": res, "clocks": clk, "y_ptr": hex(y.data_ptr()),
                  "x_ptr": [hex(t.data_ptr()) for t in xs], "ws_ptr": hex(ws.data_ptr())}))
