"""The occasional 2.5x slow cfg3 gate prefill (~240 vs 96 us) seen when the gate runs after the cfg4
layers in one process (tools/ab_prefill.py): replicate that order, time the gate, and break it down
per kernel with torch.profiler (CUPTI activity records: no kernel serialisation)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

M = 8192
specs = [("tucker2-256", Q.QDIM, Q.HIDDEN), ("tucker2-256", Q.HIDDEN, Q.QDIM), ("tucker2-128", Q.KVDIM, Q.HIDDEN),
         ("tucker4", Q.FFN, Q.HIDDEN), ("tucker4", Q.HIDDEN, Q.FFN), ("tucker2-256", Q.FFN, Q.HIDDEN)]
for kind, rows, cols in specs:  # same allocations as ab_prefill
    lay = Q._tn(kind, rows, cols, seed=5)
    p = lay.plan(torch.bfloat16)
    xs = [torch.randn(M, cols, device="cuda").to(torch.bfloat16) for _ in range(2)]
    y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
    ws = p.workspace(M)
    for i in range(23):
        p.forward(xs[i % 2], out=y, ws=ws)
    torch.cuda.synchronize()
    del xs, y
lay = S.make_layer(*S.CFG3_GATE, seed=5)
p = lay.plan(torch.bfloat16)
xs = [torch.randn(M, 5120, device="cuda").to(torch.bfloat16) for _ in range(2)]
y = torch.empty(M, 25600, device="cuda", dtype=torch.bfloat16)
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
us = e0.elapsed_time(e1) / 20 * 1e3
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(10):
        p.forward(xs[i % 2], out=y, ws=ws)
    torch.cuda.synchronize()
kern = {}
for ev in prof.key_averages():
    if ev.device_time_total > 0:
        kern[ev.key[:60]] = round(ev.device_time_total / max(ev.count, 1), 1)
print(json.dumps({"gate_us": round(us, 1), "kernels_us": kern, "y": hex(y.data_ptr()), "ws": hex(ws.data_ptr()),
                  "x": [hex(t.data_ptr()) for t in xs]}), flush=True)
