"""cfg3 gate TT r64 prefill (M = 8192) timed repeatedly under different buffer placements: after a
large dummy allocation of `pad` GB (shifts every later buffer), per step (launch list of one
forward) — to find the source of the occasional 2.5x slower runs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import synthetic as S  # noqa: E402

pad_gb = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
pad = torch.empty(int(pad_gb * 2**30), dtype=torch.uint8, device="cuda") if pad_gb > 0 else None
lay = S.make_layer(*S.CFG3_GATE, seed=5)
p = lay.plan(torch.bfloat16)
M = 8192
xs = [torch.randn(M, 5120, device="cuda").to(torch.bfloat16) for _ in range(2)]
y = torch.empty(M, 25600, device="cuda", dtype=torch.bfloat16)
ws = p.workspace(M)
res = []
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(20):
        p.forward(xs[i % 2], out=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1) / 20 * 1e3, 1))
print(json.dumps({"pad_gb": pad_gb, "us": res, "y_ptr_mod_2M": y.data_ptr() % (2 << 20), "y_ptr": hex(y.data_ptr()),
                  "x_ptr": [hex(t.data_ptr()) for t in xs], "ws_ptr": hex(ws.data_ptr())}))
