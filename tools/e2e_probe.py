"""Decompose the e2e (host I/O) overhead of the decode bench: copies alone vs the graph with
and without per-group staggered copies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.stack import TNStack


def timeit(fn, steps=200, warm=10):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps * 1e3


M = 64
xh = torch.randn(M, 5120).to(torch.bfloat16).pin_memory()
yh = torch.empty(M, 5120, dtype=torch.bfloat16).pin_memory()
xd = torch.empty(M, 5120, dtype=torch.bfloat16, device="cuda")
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    xd.copy_(xh, non_blocking=True)
    yh.copy_(xd, non_blocking=True)
print(f"copies only (H2D+D2H 655 KB each, graph): {timeit(g.replay):.1f} us")
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2, stream=st):
    xd.copy_(xh, non_blocking=True)
print(f"H2D only: {timeit(g2.replay):.1f} us")
g3 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g3, stream=st):
    yh.copy_(xd, non_blocking=True)
print(f"D2H only: {timeit(g3.replay):.1f} us")
import ctypes
from paper_2602_01613_b200 import _native as N
lib = N.load()
for name, dst, src in (("H2D", xd, xh), ("D2H", yh, xd)):
    gk = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gk, stream=st):
        N.check(lib.tnl_copy_async(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()), dst.numel() * 2,
                                   ctypes.c_void_p(st.cuda_stream)))
    print(f"{name} tnl_copy_async: {timeit(gk.replay):.1f} us")
xd2 = torch.empty_like(xd)
lib.tnl_copy_async(ctypes.c_void_p(xd2.data_ptr()), ctypes.c_void_p(xh.data_ptr()), xd.numel() * 2, None)
torch.cuda.synchronize()
assert torch.equal(xd2.cpu(), xh), "H2D copy mismatch"
yh.zero_()
lib.tnl_copy_async(ctypes.c_void_p(yh.data_ptr()), ctypes.c_void_p(xd2.data_ptr()), xd.numel() * 2, None)
torch.cuda.synchronize()
assert torch.equal(yh, xh), "D2H copy mismatch"
print("copy checks ok")

bank = S.cfg2_bank(10)
layers = [l for _, l in bank]
for mb in (1, 2):
    s0 = TNStack(layers, torch.bfloat16)
    s0.capture(M, host_io=False, microbatches=mb)
    print(f"mb={mb} device-resident: {timeit(s0.replay):.1f} us/step")
    for zc in (False, True):
        s1 = TNStack(layers, torch.bfloat16)
        s1.capture(M, host_io=True, microbatches=mb, zero_copy=zc)
        s1.x_host.copy_(torch.randn(M, 5120).to(torch.bfloat16))
        s1.replay(); torch.cuda.synchronize()
        y0 = s1.y_host.clone()
        s0.x_dev.copy_(s1.x_host.cuda()); s0.replay(); torch.cuda.synchronize()
        err = float((y0.float() - s0.y_dev.cpu().float()).norm() / s0.y_dev.cpu().float().norm())
        print(f"mb={mb} e2e zero_copy={zc}: {timeit(s1.replay):.1f} us/step (rel diff vs device pass {err:.2e})")
