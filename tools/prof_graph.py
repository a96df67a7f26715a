"""Replays the bench's cfg2 decode graph (70 layers, M=64, two token groups) a few times — the
target of `ncu --graph-profiling graph` (one profiled workload per graph replay: DRAM bytes and
duration of the whole step, not serialised cold launches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_01613_b200 import synthetic as S  # noqa: E402
from paper_2602_01613_b200.stack import TNStack  # noqa: E402

copies = int(os.environ.get("COPIES", "10"))
bank = S.cfg2_bank(copies)
st = TNStack([l for _, l in bank], torch.bfloat16)
st.capture(64, host_io=False, microbatches=2)
st.x_dev.copy_(torch.tensor(S.make_x(64, 5120, seed=29_999), dtype=torch.bfloat16, device="cuda"))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("replay")
for _ in range(int(os.environ.get("REPLAYS", "5"))):
    st.replay()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok", st.launches_per_pass)
