"""Single launches of the round-2 kernels for `ncu --set full` captures (one process, one kernel
each, after a warm-up): KERNEL=tucker2 -> tucker2_chain_kernel (q: 8192x5120 R256, M=8192);
KERNEL=jacobi -> jacobi_parallel_kernel (one 5120x640 unfolding, 2 sweeps); KERNEL=svd_finish."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_01613_b200 as tnl  # noqa: E402
from paper_2602_01613_b200 import _native as N  # noqa: E402
from paper_2602_01613_b200 import synthetic as S  # noqa: E402

k = os.environ.get("KERNEL", "tucker2")
if k == "tucker2":
    lay = S.make_layer("tucker", (8192, 5120), 1, (256, 256), seed=71_000)
    p = lay.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN)
    x = torch.randn(8192, 5120, device="cuda").to(torch.bfloat16)
    y = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
    ws = p.workspace(8192)
    for _ in range(3):
        p.forward(x, out=y, ws=ws)
elif k == "jacobi":
    rng = np.random.default_rng(1)
    a = rng.standard_normal((5120, 640))
    w = torch.tensor(np.ascontiguousarray(a.T), device="cuda")
    r = torch.eye(640, dtype=torch.float64, device="cuda")
    N.check(N.load().tnl_jacobi_sweeps_parallel(ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(r.data_ptr()), 640, 5120,
                                                640, 1e-12, 2, None, None))
else:
    from paper_2602_01613_b200 import jacobi as J

    J.svd_batched(np.random.default_rng(2).standard_normal((64, 256, 128)))
torch.cuda.synchronize()
print("ok", k)
