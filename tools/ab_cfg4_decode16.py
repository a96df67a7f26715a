"""cfg4 16-layer decode (CUDA graph) for A/B of the stack's decode switches: argv = m microbatches
concurrent_kv fuse_qo (env TNL_* read once per process)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200.qwen_stack import QwenTNStack  # noqa: E402

m, mb, kv, qo = (int(a) for a in sys.argv[1:5])
st = QwenTNStack(16)
st.concurrent_kv, st.fuse_qo = bool(kv), bool(qo)
g = st.capture(m, microbatches=mb)
st.x.normal_()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"m": m, "microbatches": mb, "concurrent_kv": kv, "fuse_qo": qo,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("TNL_")},
                  "ms": round(e0.elapsed_time(e1) / 20, 4)}))
