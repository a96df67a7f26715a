"""Batched one-sided Jacobi sweeps: GPU vs the reference's compiled kernel.

Problems are the Jacobi inputs `_jacobi_svd` builds (`tensor_core.py:210-212`: work = a.T,
rot = I), a of shape (m, n) standard normal, B independent problems per launch (e.g. the
unfoldings of a batch of layers being decomposed). Prints one JSON line per shape:
GPU problems/s and rotations/s (CUDA events around one launch of the whole batch) and the
CPU reference (`oracle/_ref/_jacobi_cy`, built from the reference's own C, one core — it
holds the GIL, `_jacobi_cy.pyx:11`) on a bounded sample of the same problems.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import build_ref
from paper_2602_01613_b200 import jacobi as J

ref = build_ref.load()
for (b, m, n) in [(592, 64, 32), (592, 128, 64), (296, 256, 128)]:
    rng = np.random.default_rng(b * 1000 + m + n)
    a = rng.standard_normal((b, m, n))
    work0 = torch.tensor(np.ascontiguousarray(np.swapaxes(a, 1, 2)), device="cuda")
    rot0 = torch.eye(n, dtype=torch.float64, device="cuda").expand(b, n, n).contiguous()
    w, r = work0.clone(), rot0.clone()
    J.jacobi_sweeps_batched(w, r)  # warm-up
    torch.cuda.synchronize()
    w, r = work0.clone(), rot0.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sweeps = J.jacobi_sweeps_batched(w, r)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sw = sweeps.cpu().numpy()
    rot_per_problem = float(sw.mean()) * n * (n - 1) / 2
    line = {"batch": b, "m": m, "n": n, "gpu_ms": ms, "gpu_problems_per_s": b / (ms / 1e3),
            "mean_sweeps": float(sw.mean()), "gpu_pair_visits_per_s": b * rot_per_problem / (ms / 1e3)}
    if ref is not None:
        k = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 3.0 and k < b:
            wk, rk = np.ascontiguousarray(a[k].T), np.eye(n)
            ref.jacobi_sweeps(wk, rk, J.JACOBI_TOL, J.JACOBI_MAX_SWEEPS)
            k += 1
        dt = time.perf_counter() - t0
        line["cpu_reference"] = {"kind": "reference", "cores": 1, "sample_problems": k,
                                 "problems_per_s": k / dt, "what": "oracle/_ref/_jacobi_cy (reference C), 1 core"}
        line["speedup_vs_cpu_1core"] = line["gpu_problems_per_s"] / line["cpu_reference"]["problems_per_s"]
    print(json.dumps(line), flush=True)
