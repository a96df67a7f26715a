"""cfg2 decode bank (70 layers, M tokens, CUDA graph) timed for A/B of compile-time variants
(TNL_LIB_AB=exp/libtnl_<name>.so). argv: m microbatches [iters]. Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import synthetic as S  # noqa: E402
from paper_2602_01613_b200.stack import TNStack  # noqa: E402

m, mb = int(sys.argv[1]), int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 50
layers = [l for _, l in S.cfg2_bank(10)]
st = TNStack(layers, torch.bfloat16)
st.capture(m, host_io=False, microbatches=mb)
for _ in range(5):
    st.replay()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / iters)
print(json.dumps({"lib": os.path.basename(os.environ.get("TNL_LIB_AB", "libtnl.so")), "m": m, "microbatches": mb,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("TNL_") and k != "TNL_LIB_AB"},
                  "ms": [round(t, 4) for t in ts]}))
