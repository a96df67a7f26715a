"""Small driver for ncu: a few cfg2 layers at decode M, repeated (no timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2602_01613_b200 import synthetic as S

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variants", default="0,2,6")
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
layers = []
for v in [int(t) for t in a.variants.split(",")]:
    name, fam, ms, rm, ranks = S.CFG2_VARIANTS[v]
    layers.append(S.make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * v))
x = torch.tensor(S.make_x(a.m, 5120, seed=1), dtype=torch.bfloat16, device="cuda")
plans = [l.plan(torch.bfloat16, flags=a.flags) for l in layers]
for _ in range(a.reps):
    for p in plans:
        y = p.forward(x)
torch.cuda.synchronize()
print("ok", [p.info["plan_large_name"] for p in plans])
