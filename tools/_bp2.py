import cProfile, pstats, sys, os, time
sys.path.insert(0, "/root/repo")
import torch
torch.cuda.init()
from paper_2602_01613_b200 import qwen_stack as Q
lays = [Q._tn(k, *Q.SHAPES[n], seed=40_000 + i) for i, (n, k) in enumerate([("q","tucker2-256")]*4 + [("down","tt64")]*2 + [("gate","tucker2-256")]*2)]
torch.zeros(1, device="cuda")
pr = cProfile.Profile(); pr.enable()
for l in lays:
    t = time.perf_counter(); l.plan(torch.bfloat16); torch.cuda.synchronize(); print("plan %.1f ms" % (1e3 * (time.perf_counter() - t)), flush=True)
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(15)
