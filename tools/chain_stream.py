"""Pure weight-stream time of the cluster chain kernel (TNL_CHAIN_DEBUG=1: no dependencies)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack
bl = [l for _, l in S.cfg2_bank(10)]
st = TNStack(bl, torch.bfloat16, cluster=True)
for mb in (1, 2, 4):
    st.capture(32 * mb, host_io=False, microbatches=mb)
    for _ in range(3):
        st.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    per_cta = 223e6 / 16
    print(f"debug={os.environ.get('TNL_CHAIN_DEBUG')} clusters={mb}: {ms*1e3:.1f} us/pass -> per-SM {per_cta/ms/1e6:.1f} GB/s", flush=True)
