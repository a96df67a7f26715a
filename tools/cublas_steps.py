"""cuBLAS (torch.matmul, bf16) on the exact GEMM shapes of the prefill cut steps, M = 8192 — the
reference point for the tcgen05 step kernels (tools/ab_prefill.py times the same layers)."""
import json

import torch

M = 8192
shapes = {  # name: (K, N) of  out (M x N) = X (M x K) . W^T
    "q_step1": (5120, 256), "q_step2": (256, 8192), "o_step1": (8192, 256), "o_step2": (256, 5120),
    "k_step1": (5120, 128), "k_step2": (128, 1024), "t4gate_step2": (256, 25600), "t4down_step1": (25600, 256),
    "cfg3gate_step1": (5120, 64), "cfg3gate_step2": (64, 25600),
}
out = {}
for name, (K, N) in shapes.items():
    xs = [torch.randn(M, K, device="cuda").to(torch.bfloat16) for _ in range(2)]
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for i in range(3):
        torch.matmul(xs[i % 2], w.t(), out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        torch.matmul(xs[i % 2], w.t(), out=y)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    out[name] = {"us": round(us, 1), "TFLOPs": round(2 * M * K * N / us / 1e6, 1),
                 "GBps": round(2 * (M * K + N * K + M * N) / us / 1e3, 1)}
print(json.dumps(out))
