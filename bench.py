"""Benchmark: TN-linear tokens/s + TFLOP/s (% roofline) vs dense cuBLAS, Qwen3-32B shapes.

Workload (BASELINE.json configs[1], "cfg2"): decode, M tokens (default 64)
through a chain of L = 7 x copies distinct 5120->5120 TN projections —
Tucker-2 R64/R128/R256, TR2 (8,8)/(16,16), TR4 (64,80|64,80) r8/r16 —
random-init cores (Philox seeds), synthetic activations.
A "step" is one pass of the M tokens through all L layers. The bank's weights
exceed the 126 MB L2, so every step streams them from HBM (L2-cold by
construction, no flush needed). value = M * L / t_step  [tokens/s per layer].

    python bench.py [--gpus N --steps K --warmup W --m 64 --copies 10]
    python bench.py --impl reference ...   # the reference's CPU algorithm (oracle port)

N > 1 (torchrun): every rank runs its own replica (independent decode streams,
no collective on the data path; "scaling": "weak"); value is the sum over
ranks, timed as the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TN-linear tokens/s + TFLOP/s (% roofline) vs dense cuBLAS, Qwen3-32B shapes"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# reference CPU algorithm (oracle port of layer_to_matrix(L) @ x, float64)
# ---------------------------------------------------------------------------


def cpu_reference_sample(m: int, steps: int, variants=None, chain: bool = False, budget_s: float = 0.0):
    """Time the reference algorithm on host cores; one cfg2 layer per step, cycling variants.

    The reference's only forward is ``layer_to_matrix(L) @ x`` (tn_decompositions.py:364-365,
    sensitivity.py:156) in float64; oracle/tn_oracle.py restates it (TR trace alpha-by-alpha).
    """
    import numpy as np

    from oracle import tn_oracle as O
    from paper_2602_01613_b200 import synthetic as S

    variants = variants or S.CFG2_VARIANTS
    layers = []
    for v, (name, fam, ms, rm, ranks) in enumerate(variants):
        L = S.make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * v)
        kw = dict(family=fam, mode_shape=ms, row_mode_count=rm)
        if fam == "tucker":
            kw.update(core=L.core.astype(np.float64), factors=[u.astype(np.float64) for u in L.factors])
        else:
            kw.update(cores=[c.astype(np.float64) for c in L.cores])
        layers.append((name, O.OracleLayer(**kw)))
    x = S.make_x(m, 5120, seed=29_999).astype(np.float64).T.copy()  # (cols, M) reference orientation
    times = []
    names = []
    t_start = time.perf_counter()
    for i in range(steps):
        # bounded sample: once every variant has been timed, stop at the time budget
        if budget_s > 0 and i >= len(layers) and time.perf_counter() - t_start > budget_s:
            break
        name, L = layers[i % len(layers)]
        t0 = time.perf_counter()
        y = O.apply_chain(L, x) if chain else O.apply_reference(L, x)
        times.append(time.perf_counter() - t0)
        names.append(name)
        assert y.shape == (5120, m)
    return times, names


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def import_reference():
    """The UNMODIFIED reference package (minima) installed into baseline/_ref (git-ignored, travels
    to the GPU box); None when it is not installed."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "minima")):
        return None
    if path not in sys.path:
        sys.path.append(path)
    try:
        from minima import tn_decompositions as T

        return T
    except Exception:
        return None


def reference_sample(m: int, steps: int, budget_s: float):
    """Time the reference's own forward, ``layer_to_matrix(L) @ x`` (tn_decompositions.py:364-365,
    sensitivity.py:156), with the UNMODIFIED minima package on the cfg2 layers, float64, all host
    threads; one layer per step cycling the 7 variants. A TR reconstruct materialises r0^2 * 26 M
    doubles (54 GB at r0 = 16): a variant whose transient does not fit in 60 % of the available host
    memory runs the oracle port instead (reported per variant)."""
    import numpy as np

    from paper_2602_01613_b200 import synthetic as S

    T = import_reference()
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    layers = []
    for v, (name, fam, ms, rm, ranks) in enumerate(S.CFG2_VARIANTS):
        L = S.make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * v)
        kw = dict(family=fam, mode_shape=ms, row_mode_count=rm)
        if fam == "tucker":
            kw.update(core=L.core.astype(np.float64), factors=[u.astype(np.float64) for u in L.factors])
        else:
            kw.update(cores=[c.astype(np.float64) for c in L.cores])
        transient = 8 * (ranks[0] ** 2 if fam == "tr" else 1) * math.prod(ms)
        if T is not None and transient < 0.6 * avail:
            layers.append((name, "reference", T.CompressedLayer(**kw), T.layer_to_matrix))
        else:
            from oracle import tn_oracle as O

            layers.append((name, "port", O.OracleLayer(**kw), O.layer_to_matrix))
    x = S.make_x(m, 5120, seed=29_999).astype(np.float64).T.copy()  # (cols, M) reference orientation
    times, names, kinds = [], [], {}
    t_start = time.perf_counter()
    for i in range(steps):
        if budget_s > 0 and i >= len(layers) and time.perf_counter() - t_start > budget_s:
            break
        name, kind, L, to_matrix = layers[i % len(layers)]
        t0 = time.perf_counter()
        y = to_matrix(L) @ x
        times.append(time.perf_counter() - t0)
        names.append(name)
        kinds[name] = kind
        assert y.shape == (5120, m)
        del y
    return times, names, kinds


def run_reference(args):
    """Reference arm: the reference's own CPU forward on host cores, rank 0 only.

    A step is one cfg2 layer through the unmodified minima package (variants cycled); at least
    one layer of each of the 7 variants is measured even when K < 7, and value = M / (mean over
    variants of the per-variant mean time), so the figure does not depend on which variants K
    covers.
    """
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nthreads = cpu_cores()
    steps = max(args.steps, 1)
    n = max(steps, 7)
    # each step is one layer; the sample stops after ~120 s of host work (at least one layer of
    # every variant) so the reference arm ends within a few minutes
    times, names, kinds = reference_sample(args.m, n, budget_s=120.0)
    n = len(times)
    per = {}
    for nm, t in zip(names, times):
        per.setdefault(nm, []).append(t)
    mean_layer_s = sum(sum(v) / len(v) for v in per.values()) / len(per)
    value = args.m / mean_layer_s
    kind = "reference" if all(k == "reference" for k in kinds.values()) else "port"
    sample = (f"{n} layers (one per step, cycling the {len(per)} cfg2 5120x5120 variants), M={args.m}, "
              "float64 layer_to_matrix(L) @ x through the unmodified reference package (minima, "
              "installed in baseline/_ref); value = M / mean per-variant layer time")
    line = {
        "metric": METRIC,
        "impl": "reference",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * mean_layer_s,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": nthreads, "kind": kind, "sample": sample,
                         "per_variant_s": {k: sum(v) / len(v) for k, v in per.items()},
                         "per_variant_impl": kinds},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args):
    return {
        "workload": f"cfg2 decode: M={args.m} tokens through a chain of {7 * args.copies} distinct "
                    "5120->5120 TN layers (Tucker-2 R64/R128/R256, TR2 (8,8)/(16,16), TR4 r8/r16; "
                    f"{args.copies} copies each)",
        "m": args.m,
        "layers": 7 * args.copies,
        "shape": "5120x5120 (Qwen3-32B attention projection)",
        "l2_policy": "bank weights > 126 MB L2: streamed from HBM every step",
        "parallelism": f"replicas x{args.gpus}" if args.gpus > 1 else "single",
        "microbatches": args.microbatches,
        "graph": "one CUDA graph per step; the M tokens run as `microbatches` concurrent groups on forked streams",
    }


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel (dec_fused_kernel) from the committed
    `ncu --set full` capture (profiles/r02/ncu_dec_fused.json, tools/ncu_dec_summary.py); (None, reason) if absent."""
    here = os.path.dirname(os.path.abspath(__file__))
    path = os.path.join(here, "profiles", "r02", "ncu_dec_fused.json")  # HEAD build (r01: the first capture)
    if not os.path.exists(path):
        path = os.path.join(here, "profiles", "r01", "ncu_dec_fused.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return (d["fused_mean_dram_bytes_per_launch"],
                "dram__bytes_read.sum + dram__bytes_write.sum per dec_fused_kernel launch (mean over the cfg2 "
                f"boundaries), ncu --set full capture {os.path.relpath(path)}; algorithmic weight bytes per launch "
                f"{d['fused_mean_weight_bytes_per_launch']:.0f}")
    except (OSError, KeyError, ValueError):
        return None, "no ncu capture committed"


def ncu_graph_step_bytes():
    """DRAM bytes of one replay of the decode graph (`ncu --graph-profiling graph`, the whole
    70-layer step as one workload: profiles/r02/ncu_graph_decode_step.csv, tools/prof_graph.py);
    median over the captured replays. (None, reason) if absent."""
    import csv

    path = os.path.join(ROOT, "profiles", "r02", "ncu_graph_decode_step.csv")
    try:
        lines = [ln for ln in open(path) if ln.startswith('"')]
        rows = list(csv.reader(lines))
        h = rows[0]
        per = {}
        for r in rows[1:]:
            per.setdefault(r[0], {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
        tot = sorted(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in per.values())
        return tot[len(tot) // 2], (f"ncu --graph-profiling graph, dram__bytes_read.sum + dram__bytes_write.sum per "
                                    f"replay of the whole step, median of {len(tot)} replays ({os.path.relpath(path, ROOT)})")
    except (OSError, ValueError, KeyError, IndexError):
        return None, "no graph-level ncu capture committed"


def capture_steps(step, n, torch):
    """n calls of `step` captured in one CUDA graph (after one eager warm call on the capture stream), so
    per-call timings of host-driven paths are free of host launch jitter."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            step()
    return g


def time_graph(replay, steps, warmup, torch, dist=None):
    for _ in range(warmup):
        replay()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        replay()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    return ms / steps


# ---------------------------------------------------------------------------
# cfg4: the 64-layer Qwen3-32B-shaped mixed-TN stack (secondary lines) vs a measured dense stack
# ---------------------------------------------------------------------------


class DenseQwenStack:
    """The same decoder step as QwenTNStack with UNCOMPRESSED bf16 weights and cuBLAS matmuls
    (torch.matmul), pre-norm RMSNorm and SiLU*mul as torch ops, attention core a pass-through:
        h = rms(x); q, k, v = h Wq^T, h Wk^T, h Wv^T; x += q Wo^T
        h = rms(x); x += (silu(h Wg^T) * (h Wu^T)) Wd^T
    64 layers x (8192x5120 + 2x1024x5120 + 5120x8192 + 2x25600x5120 + 5120x25600) = 31.2 G params
    (62.4 GB bf16, resident in HBM). Random-init weights, N(0, 1/cols)."""

    def __init__(self, n_layers, torch):
        from paper_2602_01613_b200 import qwen_stack as Q

        self.torch = torch
        self.w = []
        for _ in range(n_layers):
            blk = {}
            for name, (rows, cols) in Q.SHAPES.items():
                blk[name] = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda").normal_(0, cols ** -0.5)
            self.w.append(blk)
        self.params = sum(w.numel() for blk in self.w for w in blk.values())

    def forward(self, x):
        torch = self.torch
        F = torch.nn.functional

        def rms(t):
            tf = t.float()
            return (tf * torch.rsqrt(tf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(torch.bfloat16)

        for blk in self.w:
            h = rms(x)
            q = torch.matmul(h, blk["q"].t())
            torch.matmul(h, blk["k"].t())
            torch.matmul(h, blk["v"].t())
            x = x + torch.matmul(q, blk["o"].t())
            h = rms(x)
            x = x + torch.matmul(F.silu(torch.matmul(h, blk["gate"].t())) * torch.matmul(h, blk["up"].t()),
                                 blk["down"].t())
        return x


def capture_graph(fn, torch):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


def bench_cfg4(hbm, tc, torch, n_layers=64, ms=(1, 64, 8192), dense=True, reps=(5, 5, 2)):
    """BASELINE cfg4: the full 64-layer mixed-TN stack (sensitivity-mix layout) —
    decode M=1 and M=64 (CUDA graph, two token groups on forked streams) and prefill M=8192
    (folded residual/RMSNorm) — each against the same decoder with uncompressed weights on cuBLAS,
    measured in the same process. Roofline per pass: bytes = sum over the 448 projections of
    2*(P + M*(rows+cols)), flops = M * sum of chain flops; the RMSNorm/residual traffic of the
    decoder is not counted (it is the same for both stacks)."""
    from paper_2602_01613_b200.qwen_stack import HIDDEN, QwenTNStack

    t0 = time.perf_counter()
    st = QwenTNStack(n_layers)
    build = dict(st.build_s, total=time.perf_counter() - t0)
    P = st.param_count()
    F = st.chain_flops_per_token()
    rc = sum(r + c for _, lay, _ in st.projections() for r, c in [lay.matrix_shape])
    out = {"layers": n_layers, "projections": 7 * n_layers, "params": P, "chain_flops_per_token": F,
           "build_s": build, "fused_mlp_blocks": st.fused_mlp_count(), "lines": {}}
    for m, k in zip(ms, reps):
        g = st.capture(m, microbatches=2)
        st.x.normal_()
        ms_tn = time_graph(g.replay, k, 2, torch, None)
        finite = bool(torch.isfinite(st.x).all())
        byts = 2 * (P + m * rc)
        t_roof = max(byts / (hbm * 1e9), m * F / (tc * 1e12))
        bound = "hbm" if byts / (hbm * 1e9) >= m * F / (tc * 1e12) else "tensor"
        out["lines"][f"M={m}"] = {
            "phase": "decode" if m <= 64 else "prefill", "ms_per_pass": ms_tn, "tokens_per_s": m / (ms_tn / 1e3),
            "roofline": {"bound": bound, "t_roofline_ms": 1e3 * t_roof, "frac": 1e3 * t_roof / ms_tn,
                         "alg_bytes": byts, "alg_flops": m * F, "achieved_GBps": byts / (ms_tn / 1e3) / 1e9,
                         "achieved_chain_TFLOPs": m * F / (ms_tn / 1e3) / 1e12},
            "finite": finite}
        del g
        torch.cuda.empty_cache()
    del st
    torch.cuda.empty_cache()
    if dense:
        D = DenseQwenStack(n_layers, torch)
        out["dense_params"] = D.params
        for m, k in zip(ms, reps):
            x = torch.randn(m, HIDDEN, device="cuda").to(torch.bfloat16)
            g = capture_graph(lambda: D.forward(x), torch)
            ms_d = time_graph(g.replay, k, 1, torch, None)
            ln = out["lines"][f"M={m}"]
            ln["dense_cublas"] = {"ms_per_pass": ms_d, "tokens_per_s": m / (ms_d / 1e3),
                                  "weight_GB": 2 * D.params / 1e9}
            ln["speedup_vs_dense"] = ms_d / ln["ms_per_pass"]
            del g
            torch.cuda.empty_cache()
        del D
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="tnl", choices=["tnl", "reference"])
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--copies", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense cuBLAS comparison")
    ap.add_argument("--no-prefill", action="store_true", help="skip the secondary cfg3 prefill measurement")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the secondary cfg4 64-layer stack measurement")
    ap.add_argument("--cfg4-layers", type=int, default=64)
    ap.add_argument("--flags", type=int, default=0, help="TNL_PLAN_* preference for every layer")
    ap.add_argument("--microbatches", type=int, default=2,
                    help="concurrent token groups (streams) the M tokens are split into inside the graph")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import numpy as np
    import torch

    import paper_2602_01613_b200 as tnl
    from paper_2602_01613_b200 import synthetic as S
    from paper_2602_01613_b200.stack import TNStack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hbm, tc, peak_kind = peaks()

    bank = S.cfg2_bank(args.copies)
    layers = [l for _, l in bank]
    stack = TNStack(layers, torch.bfloat16, flags=args.flags)
    M, L = args.m, len(layers)
    x0 = torch.tensor(S.make_x(M, 5120, seed=29_999 + rank), dtype=torch.bfloat16, device="cuda")

    # device-resident throughput (value): graph of one pass, inputs already in HBM
    stack.capture(M, host_io=False, microbatches=args.microbatches)
    stack.x_dev.copy_(x0)
    launches_per_step = stack.launches_per_pass
    sampler = ClockSampler(local)
    sampler.start()
    t_end = time.time() + 1.0
    while time.time() < t_end:  # soak so the clock samples see a loaded GPU
        stack.replay()
        torch.cuda.synchronize()
    ms_step = time_graph(stack.replay, args.steps, args.warmup, torch, dist)
    clocks = sampler.stop()
    # SPEC micro-benchmark contract: per-replay median / IQR over >= 10 reps
    reps = []
    for _ in range(max(20, 10)):
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        stack.replay()
        b_.record()
        b_.synchronize()
        reps.append(a_.elapsed_time(b_))
    q = np.percentile(reps, [25, 50, 75])
    rep_stats = {"reps": len(reps), "median_ms": float(q[1]), "iqr_ms": float(q[2] - q[0]),
                 "note": "each replay timed alone (launch gap included), so median >= ms_per_step"}
    y_dev = stack.y_dev.clone()

    # end-to-end through the public API: pinned host x -> H2D -> L layers -> D2H y, one graph
    e2e_stack = TNStack(layers, torch.bfloat16, flags=args.flags)
    zero_copy = os.environ.get("TNL_E2E_ZERO_COPY", "1") != "0"  # A/B switch: SM-driven copies instead
    e2e_stack.capture(M, host_io=True, microbatches=args.microbatches, zero_copy=zero_copy)
    e2e_stack.x_host.copy_(x0.cpu())
    ms_e2e = time_graph(e2e_stack.replay, args.steps, args.warmup, torch, dist)
    torch.cuda.synchronize()
    d = (e2e_stack.y_host.float() - y_dev.cpu().float()).norm() / y_dev.cpu().float().norm()
    assert float(d) < 5e-2, f"e2e output differs from the device-resident pass ({float(d)})"

    # algorithmic accounting: bytes = 2*(P + M*(rows+cols)), flops = M * chain flops
    alg_bytes = sum(2 * (tnl.param_count(l) + M * (5120 + 5120)) for l in layers)
    alg_flops = sum(M * l.chain_flops_per_token() for l in layers)
    plan_bytes = sum(p.info["weight_bytes"] for p in stack.plans)
    t_s = ms_step / 1e3
    value = world * M * L / t_s
    achieved_gbs = alg_bytes / t_s / 1e9
    t_roof = max(alg_bytes / (hbm * 1e9), alg_flops / (tc * 1e12))

    # per-variant breakdown (chains of the same variant)
    breakdown = {}
    for v, (name, *_rest) in enumerate(S.CFG2_VARIANTS):
        sub = TNStack([l for n, l in bank if n == name], torch.bfloat16, flags=args.flags)
        sub.capture(M, host_io=False, microbatches=args.microbatches)
        ms_sub = time_graph(sub.replay, max(args.steps // 4, 10), 3, torch, None)
        breakdown[name] = {
            "l2": "hot (the 10 layers of one variant fit in the 126 MB L2)",
            "us_per_layer": 1e3 * ms_sub / len(sub.plans),
            "plan": sub.plans[0].info["plan_large_name"],
            "launches_per_layer": sub.launches_per_pass / len(sub.plans),
        }
        del sub

    # L2-hot vs L2-cold (SURVEY 8(d) GPU timing): the bank (223 MB of panels) streams from HBM every
    # step; the same layers grouped by variant run with their weights resident in L2
    rep_of = {}
    for n, l in bank:
        rep_of.setdefault(n, l)
    hot = TNStack([rep_of[n] for n, _ in bank], torch.bfloat16, flags=args.flags)  # 7 distinct layers, shared plans
    hot.capture(M, host_io=False, microbatches=args.microbatches)
    hot.x_dev.copy_(x0)
    hot_ms = time_graph(hot.replay, args.steps, args.warmup, torch, dist)
    hot_bytes = sum(p.info["weight_bytes"] for p in {id(p): p for p in hot.plans}.values())
    l2 = {"cold": {"ms_per_step": ms_step, "value": world * M * L / t_s},
          "hot": {"ms_per_step": hot_ms, "value": world * M * L / (hot_ms / 1e3),
                  "how": f"same 70-layer chain and order, but every layer of a variant shares one plan: "
                         f"{hot_bytes / 1e6:.0f} MB of panels stay L2-resident"}}
    del hot

    dense = None
    if not args.no_dense:
        ws = [torch.randn(5120, 5120, device="cuda").to(torch.bfloat16) for _ in range(L)]
        xd = x0.clone()
        bufs = [torch.empty(M, 5120, dtype=torch.bfloat16, device="cuda") for _ in range(2)]

        def dense_pass():
            cur = xd
            for i, w in enumerate(ws):
                torch.matmul(cur, w.t(), out=bufs[i % 2])
                cur = bufs[i % 2]

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            dense_pass()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            dense_pass()
        ms_dense = time_graph(g.replay, args.steps, args.warmup, torch, dist)
        dense = {"value": world * M * L / (ms_dense / 1e3), "unit": "tokens/s", "ms_per_step": ms_dense,
                 "what": "torch.matmul (cuBLAS) bf16 of the uncompressed 5120x5120 weights, same chain, CUDA graph"}
        del ws

    # secondary (not the headline): cfg3 prefill, Qwen3-32B MLP TT r64 projections at M=8192
    prefill = None
    if not args.no_prefill:
        prefill = {}
        for which, (fam, ms_, rm, rk) in (("gate", S.CFG3_GATE), ("down", S.CFG3_DOWN)):
            lay = S.make_layer(fam, ms_, rm, rk, seed=30_064)
            rows_, cols_ = lay.matrix_shape
            pl = lay.plan(torch.bfloat16)
            Mp = 8192
            xs = [torch.randn(Mp, cols_, device="cuda").to(torch.bfloat16) for _ in range(4)]  # 336+ MB > L2
            yp = torch.empty(Mp, rows_, device="cuda", dtype=torch.bfloat16)
            wsp = pl.workspace(Mp)
            it = [0]

            def pre_step():
                pl.forward(xs[it[0] % 4], out=yp, ws=wsp)
                it[0] += 1

            g_p = capture_steps(pre_step, 4, torch)  # one replay = 4 forwards over the 4 inputs
            ms_p = time_graph(g_p.replay, 5, 1, torch, None) / 4
            del g_p
            byts = 2 * (tnl.param_count(lay) + Mp * (rows_ + cols_))
            prefill[which] = {"layer": f"TT r64 {ms_}", "M": Mp, "ms": ms_p, "tokens_per_s": Mp / (ms_p / 1e3),
                              "alg_GBps": byts / (ms_p / 1e3) / 1e9, "frac_hbm": byts / (ms_p / 1e3) / 1e9 / hbm,
                              "plan": pl.info["plan_large_name"]}
            del xs, yp
        # the whole cfg3 MLP block (5120 -> 25600 -> 5120, TT r64 gate/up/down): fused path, h on chip
        from paper_2602_01613_b200.mlp import TNMLP

        g_, u_, d_ = (S.make_layer(f, ms_, rm, rk, seed=31_000 + i) for i, (f, ms_, rm, rk) in
                      enumerate((S.CFG3_GATE, S.CFG3_GATE, S.CFG3_DOWN)))
        blk = TNMLP(g_, u_, d_)
        Mp = 8192
        xs = [torch.randn(Mp, 5120, device="cuda").to(torch.bfloat16) for _ in range(4)]
        yp = torch.empty(Mp, 5120, device="cuda", dtype=torch.bfloat16)
        wsp = blk.workspace(Mp)
        it = [0]

        def mlp_step():
            blk.forward(xs[it[0] % 4], out=yp, ws=wsp)
            it[0] += 1

        g_b = capture_steps(mlp_step, 4, torch)
        ms_b = time_graph(g_b.replay, 5, 1, torch, None) / 4
        del g_b
        P3 = sum(tnl.param_count(l_) for l_ in (g_, u_, d_))
        b_bytes = 2 * (P3 + Mp * (5120 + 5120))
        b_flops = Mp * sum(l_.chain_flops_per_token() for l_ in (g_, u_, d_))
        t_roof_mlp = max(b_bytes / (hbm * 1e9), b_flops / (tc * 1e12))
        # what the kernels execute (merged cut: 2*r_cut*(rows+cols) per token and projection)
        x_flops = Mp * sum(l_.plan(torch.bfloat16).info["cut_flops_per_token"] for l_ in (g_, u_, d_))
        prefill["mlp_block"] = {"what": "Qwen3-32B MLP block y = down(silu(gate(x)) * up(x)), TT r64, one tnl_mlp_forward",
                                "M": Mp, "ms": ms_b, "tokens_per_s": Mp / (ms_b / 1e3), "fused": bool(blk.fused),
                                "t_roofline_ms": 1e3 * t_roof_mlp, "frac_roofline": t_roof_mlp / (ms_b / 1e3),
                                "chain_TFLOPs": b_flops / (ms_b / 1e3) / 1e12,
                                "executed_flops": x_flops, "executed_TFLOPs": x_flops / (ms_b / 1e3) / 1e12,
                                "frac_tensor_executed": x_flops / (tc * 1e12) / (ms_b / 1e3),
                                "note": "frac_roofline divides the chain-flop/byte roofline time by the block time; "
                                        "frac_tensor_executed is the flops the kernels execute (merged cut) over "
                                        "the tensor-core peak"}
        blk.close()
        del xs, yp

    # secondary (cfg5, N > 1 only): prefill of the cfg3 gate projection sharded over the ranks —
    # output-mode sharded (each rank owns 25600/N rows of the leading output mode and stores them into
    # every peer's symmetric-memory y over NVLink) and token-sharded (no collective); max over ranks
    sharded = None
    if world > 1 and not args.no_prefill:
        try:
            from paper_2602_01613_b200.sharded import OutputShardedLayer, TokenShardedLayer

            fam, ms_, rm, rk = S.CFG3_GATE
            lay = S.make_layer(fam, ms_, rm, rk, seed=30_064)
            Mp = 8192
            xs = torch.randn(Mp, 5120, device="cuda").to(torch.bfloat16)
            osl = OutputShardedLayer(lay, dtype=torch.bfloat16, device=torch.device("cuda", local))
            tsl = TokenShardedLayer(lay, dtype=torch.bfloat16, device=torch.device("cuda", local))
            yfull = torch.empty(Mp, 25600, device="cuda", dtype=torch.bfloat16)
            ms_o = time_graph(lambda: osl.forward(xs, out=yfull), 10, 3, torch, dist)
            ms_t = time_graph(lambda: tsl.forward(xs), 10, 3, torch, dist)
            sharded = {"layer": f"TT r64 {ms_}", "M": Mp, "world": world,
                       "output_sharded": {"ms": ms_o, "tokens_per_s": Mp / (ms_o / 1e3),
                                          "allgather_bytes_per_rank": 2 * Mp * 25600 // world,
                                          "how": "row-restricted plan per rank storing its slice of i0 straight into "
                                                 "its columns of y (strided TMA store); NCCL groups: y in symmetric "
                                                 "memory, P2P stores of the slice into every peer's y + one device "
                                                 "barrier (no gather buffer, no permute); max over ranks; eager "
                                                 "(host-driven exchange), not a graph replay"},
                       "token_sharded": {"ms": ms_t, "tokens_per_s": Mp / (ms_t / 1e3),
                                         "how": "M/N tokens per rank, full weights, no collective; max over ranks"}}
        except Exception as exc:  # report, never fail the headline run
            sharded = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # secondary: cfg1 (BASELINE configs[0]) TT (64,64|64,64) r32, M=16 — fp32 generic chain (the
    # reference-precision path, CUDA-core bound) and bf16 plans; 8 distinct layers (> L2? no: 2 MB)
    cfg1 = None
    if not args.no_prefill:
        cfg1 = {}
        lays = [S.make_layer("tt", (64, 64, 64, 64), 2, (32, 32, 32), seed=10_000 + 100 * i) for i in range(8)]
        x16 = torch.randn(16, 4096, device="cuda")
        props = torch.cuda.get_device_properties(0)
        clk_ghz = (clocks or {}).get("sm_max_mhz", 1965.0) / 1e3
        fp32_peak = props.multi_processor_count * 128 * 2 * clk_ghz / 1e3  # TFLOP/s (FFMA)
        for dt, name in ((torch.float32, "fp32"), (torch.bfloat16, "bf16")):
            pls = [l.plan(dt) for l in lays]
            xs = x16.to(dt)
            wss = [p.workspace(16) for p in pls]
            outs = [torch.empty(16, 4096, device="cuda", dtype=dt) for _ in pls]

            def c1():
                for p, w_, o_ in zip(pls, wss, outs):
                    p.forward(xs, out=o_, ws=w_)

            s1 = torch.cuda.Stream()
            s1.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s1):
                c1()
            torch.cuda.current_stream().wait_stream(s1)
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1, stream=s1):
                c1()
            ms1 = time_graph(g1.replay, 200, 10, torch, None) / len(lays)
            c1_bytes = (4 if dt == torch.float32 else 2) * (tnl.param_count(lays[0]) + 16 * 8192)
            c1_flops = 16 * lays[0].chain_flops_per_token()
            peak_t = fp32_peak if dt == torch.float32 else tc
            c1_troof = max(c1_bytes / (hbm * 1e9), c1_flops / (peak_t * 1e12))
            cfg1[name] = {"us_per_layer": 1e3 * ms1, "tokens_per_s": 16 / (ms1 / 1e3), "chain_TFLOPs": c1_flops / (ms1 / 1e3) / 1e12,
                          "frac_roofline": c1_troof / (ms1 / 1e3), "roofline_peak": (f"fp32 CUDA-core {fp32_peak:.1f} TFLOP/s"
                                                                                   if name == "fp32" else "bf16 tensor / HBM"),
                          "plan": pls[0].info["plan_small_name"]}

    stack_cfg4 = None
    if world == 1 and not args.no_cfg4:
        try:
            stack_cfg4 = bench_cfg4(hbm, tc, torch, n_layers=args.cfg4_layers, dense=not args.no_dense)
        except Exception as exc:  # report, never fail the headline run
            stack_cfg4 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        times, names = cpu_reference_sample(M, 7)
        ctimes, _ = cpu_reference_sample(M, 7, chain=True)
        cpu = {"value": M * len(times) / sum(times), "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
               "chain_path": {"value": M * len(ctimes) / sum(ctimes), "unit": "tokens/s",
                              "what": "reference-semantics core-by-core chain (SURVEY Appendix A) in float64, "
                                      "same layers and threads (SURVEY 8(d) CPU row ii)"},
               "sample": f"one layer of each of the 7 cfg2 variants at M={M}, reference algorithm "
                         "layer_to_matrix(L) @ x in float64 (oracle port), numpy/OpenBLAS threads",
               "per_variant_s": {n: t for n, t in zip(names, times)}}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": workload_config(args),
        "tflops": alg_flops * world / t_s / 1e12,
        "roofline": {
            "kernel": "TN-linear layer forward (all launches of one layer, averaged over the bank)",
            "bound": "hbm",
            "achieved": achieved_gbs,
            "peak": hbm,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": achieved_gbs / hbm,
            "traffic": ncu_traffic()[0],
            "traffic_note": ncu_traffic()[1],
            "dram_bytes_per_step_graph": ncu_graph_step_bytes()[0],
            "dram_bytes_per_step_graph_note": ncu_graph_step_bytes()[1] + "; the two token groups each stream "
                                              "the 223 MB of panels (latency-bound chain: L2-hot runs no faster)",
            "algorithmic_bytes_per_step": alg_bytes,
            "plan_weight_bytes_per_step": plan_bytes,
            "t_roofline_ms": 1e3 * t_roof,
            "frac_of_roofline_time": 1e3 * t_roof / ms_step,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": world * M * L / (ms_e2e / 1e3), "unit": "tokens/s",
                "h2d_bytes_per_step": e2e_stack.h2d_bytes, "d2h_bytes_per_step": e2e_stack.d2h_bytes,
                "ms_per_step": ms_e2e, "api": "TNStack CUDA graph: per token group, tnl_stack_forward_host — the first kernel reads the pinned host x over the bus, the 70-layer chain runs, the last kernel writes the pinned host y (zero-copy H2D/D2H)"},
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_step": launches_per_step,
        "clocks": clocks,
        "dense_cublas": dense,
        "speedup_vs_dense": (value / dense["value"]) if dense else None,
        "breakdown": breakdown,
        "l2_hot_vs_cold": l2,
        "replay_stats": rep_stats,
        "prefill_cfg3": prefill,
        "cfg1_m16": cfg1,
        "sharded_prefill_cfg5": sharded,
        "stack_cfg4": stack_cfg4,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
