"""One bf16 chain-plan forward (TNL_PLAN_CHAIN) per layer at M=8192, for an ncu launch list of its
steps: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python
tools/prof_chain_steps.py`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_01613_b200 as tnl  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

M = int(os.environ.get("M", "8192"))
for name, lay in (("cfg3 gate", S.make_layer(*S.CFG3_GATE, seed=1)),
                  ("tr4 r16", S.make_layer("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16), seed=2))):
    rows, cols = lay.matrix_shape
    p = lay.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN)
    x = torch.randn(M, cols, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, rows, device="cuda", dtype=torch.bfloat16)
    ws = p.workspace(M)
    p.forward(x, out=y, ws=ws)
    torch.cuda.synchronize()
    print(name, "done", flush=True)
