"""cfg4 q projection (Tucker-2 R256, 5120 -> 8192) at M=8192: per-step launch list under ncu and
the step-2 GEMM shape (8192 x 8192 x 256) against cuBLAS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S

def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3

lay = S.make_layer("tucker", (8192, 5120), 1, (256, 256), seed=1)
pl = lay.plan(torch.bfloat16)
M = 8192
x = torch.randn(M, 5120, device="cuda").to(torch.bfloat16)
y = torch.empty(M, 8192, device="cuda", dtype=torch.bfloat16)
ws = pl.workspace(M)
print("q forward us:", round(t(lambda: pl.forward(x, out=y, ws=ws)), 1), "plan", pl.info["plan_large_name"])
T = torch.randn(M, 256, device="cuda").to(torch.bfloat16)
W = torch.randn(8192, 256, device="cuda").to(torch.bfloat16)
print("cuBLAS T.W^T (8192x8192x256) us:", round(t(lambda: torch.matmul(T, W.t(), out=y)), 1))
X = torch.randn(M, 5120, device="cuda").to(torch.bfloat16)
U = torch.randn(256, 5120, device="cuda").to(torch.bfloat16)
T2 = torch.empty(M, 256, device="cuda", dtype=torch.bfloat16)
print("cuBLAS X.U^T (8192x256x5120) us:", round(t(lambda: torch.matmul(X, U.t(), out=T2)), 1))
