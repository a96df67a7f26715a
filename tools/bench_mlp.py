"""cfg3 MLP block (5120 -> 25600 -> 5120, TT r64), M=8192 bf16: fused vs unfused vs dense cuBLAS."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_01613_b200 import synthetic as S
from paper_2602_01613_b200.mlp import TNMLP
import paper_2602_01613_b200 as tnl

M = int(os.environ.get("M", "8192"))
layers = [S.make_layer(*S.CFG3_GATE, seed=30_100), S.make_layer(*S.CFG3_GATE, seed=30_200),
          S.make_layer(*S.CFG3_DOWN, seed=30_300)]
xs = [torch.randn(M, 5120, device="cuda").to(torch.bfloat16) for _ in range(4)]

def timeit(fn, iters=20):
    # CUDA-graph replays of 4 calls (eager Python loops pick up host launch jitter)
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(4): fn(i)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters // 4): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (4 * (iters // 4))

P = sum(tnl.param_count(l) for l in layers)
F = sum(l.chain_flops_per_token() for l in layers) * M
byts = 2 * (P + M * 2 * 5120)
for fused in (True, False):
    mlp = TNMLP(*layers, fused=fused)
    y = torch.empty(M, 5120, device="cuda", dtype=torch.bfloat16)
    ms = timeit(lambda i: mlp.forward(xs[i % 4], out=y))
    print(json.dumps({"M": M, "fused": mlp.fused, "ms": ms, "tokens_per_s": M / (ms / 1e3),
                      "frac_hbm_block": byts / (ms / 1e3) / 6554.6e9, "t_roof_us": 1e6 * max(byts / 6554.6e9, F / 1635e12)}), flush=True)
wg = torch.randn(25600, 5120, device="cuda").to(torch.bfloat16); wu = torch.randn(25600, 5120, device="cuda").to(torch.bfloat16)
wd = torch.randn(5120, 25600, device="cuda").to(torch.bfloat16)
def dense(i):
    x = xs[i % 4]
    h = torch.nn.functional.silu(x @ wg.t()) * (x @ wu.t())
    return h @ wd.t()
ms = timeit(dense, 5)
print(json.dumps({"M": M, "dense_cublas_ms": ms, "tokens_per_s": M / (ms / 1e3)}), flush=True)
