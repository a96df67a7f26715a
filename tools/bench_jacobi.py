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

# one large single problem (a Qwen-shaped unfolding): the round-robin parallel order on all SMs
# (tnl_jacobi_sweeps_parallel) vs the batched cyclic kernel (one warp) and the reference's cyclic
# C kernel (1 core, one sweep timed: a full run takes hours)
for (m, n) in [(5120, 640)]:
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n)) @ np.diag(np.linspace(1.0, 1e-3, n)) @ np.linalg.qr(rng.standard_normal((n, n)))[0]
    w0 = torch.tensor(np.ascontiguousarray(a.T), device="cuda")
    r0 = torch.eye(n, dtype=torch.float64, device="cuda")
    import ctypes

    from paper_2602_01613_b200 import _native as N

    lib = N.load()
    line = {"m": m, "n": n}
    for kind in ("parallel", "cyclic_warp"):
        w, r = w0.clone(), r0.clone()
        sw = torch.zeros(1, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if kind == "parallel":
            N.check(lib.tnl_jacobi_sweeps_parallel(ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(r.data_ptr()), n, m, n,
                                                   J.JACOBI_TOL, J.JACOBI_MAX_SWEEPS, ctypes.c_void_p(sw.data_ptr()),
                                                   None))
            e1.record()
        else:
            sw = J.jacobi_sweeps_batched(w[None].contiguous(), r[None].contiguous(), J.JACOBI_TOL, 2)
            e1.record()
        torch.cuda.synchronize()
        line[kind] = {"ms": e0.elapsed_time(e1), "sweeps": int(sw.cpu()[0])}
    line["cyclic_warp"]["note"] = "max_sweeps=2 (the one-warp cyclic kernel is serial over all n(n-1)/2 pairs)"
    line["parallel"]["ms_per_sweep"] = line["parallel"]["ms"] / line["parallel"]["sweeps"]
    line["cyclic_warp"]["ms_per_sweep"] = line["cyclic_warp"]["ms"] / max(1, line["cyclic_warp"]["sweeps"])
    res = J.full_svd(a, parallel=True)
    s = np.linalg.svd(a, compute_uv=False)
    line["max_rel_spectrum_err_vs_lapack"] = float(np.max(np.abs(res.values - s)) / s[0])
    if ref is not None:
        wk, rk = np.ascontiguousarray(a.T), np.eye(n)
        t0 = time.perf_counter()
        ref.jacobi_sweeps(wk, rk, J.JACOBI_TOL, 1)
        line["cpu_reference_one_sweep_s"] = time.perf_counter() - t0
        line["speedup_per_sweep_vs_cpu_1core"] = line["cpu_reference_one_sweep_s"] / (line["parallel"]["ms_per_sweep"] / 1e3)
    print(json.dumps(line), flush=True)
