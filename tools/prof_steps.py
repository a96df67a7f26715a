"""One cfg4 q projection (Tucker-2 R256, 8192x5120) forward at M=8192 after a warm-up — the target of
an ncu launch list (per-step durations of the cut plan). KIND=o / kv / gate_t4 selects others."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import qwen_stack as Q  # noqa: E402

kind = os.environ.get("KIND", "q")
spec = {"q": ("tucker2-256", Q.QDIM, Q.HIDDEN), "o": ("tucker2-256", Q.HIDDEN, Q.QDIM), "kv": ("tucker2-128", Q.KVDIM, Q.HIDDEN),
        "gate_t4": ("tucker4", Q.FFN, Q.HIDDEN), "down_t4": ("tucker4", Q.HIDDEN, Q.FFN)}[kind]
lay = Q._tn(spec[0], spec[1], spec[2], seed=5)
p = lay.plan(torch.bfloat16)
x = torch.randn(8192, spec[2], device="cuda").to(torch.bfloat16)
y = torch.empty(8192, spec[1], device="cuda", dtype=torch.bfloat16)
ws = p.workspace(8192)
for _ in range(3):
    p.forward(x, out=y, ws=ws)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("fwd")
p.forward(x, out=y, ws=ws)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", kind)
