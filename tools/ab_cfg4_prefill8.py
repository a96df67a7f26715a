"""cfg4 8-layer prefill (M = 8192, CUDA graph) timing for A/B of stack-level switches (env vars are
read by the library once per process: run one process per setting)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200.qwen_stack import QwenTNStack  # noqa: E402

st = QwenTNStack(8, mlp_kinds=["tt64", "tr4", "tucker4", "tt64", "tr4", "tucker4", "tt64", "tr4"])
g = st.capture(8192)
st.x.normal_()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
res = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1) / 5, 4))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TNL_")}, "ms": res,
                  "finite": bool(torch.isfinite(st.x).all())}))
