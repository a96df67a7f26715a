"""Summarise an `ncu --set full --page raw --csv` capture of tools/prof_stack.py (one decode pass of
the 7-variant cfg2 chain) into the JSON bench.py reads for roofline.traffic: per launch the cold
duration, DRAM bytes and the algorithmic weight bytes (A_out of layer l + B_in of layer l+1, bf16,
r_pad = cut rank rounded up to 16). usage: ncu_dec_summary.py raw.csv out.json source-note"""
import csv
import json
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2602_01613_b200 import synthetic as S  # noqa: E402


def cut_rank(fam, ranks, rm):
    if fam == "tucker":
        return ranks[0]
    return ranks[0] * ranks[rm]  # TR: closure x cut bond


raw, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader([ln for ln in open(raw) if ln.startswith('"')]))
h = rows[0]
recs = rows[2:]  # row 1 holds the units
rp = [-(-cut_rank(f, rk, rm) // 16) * 16 for (_, f, ms, rm, rk) in S.CFG2_VARIANTS]
launches = []
fused = 0
for r in recs:
    d = dict(zip(h, r))
    name = d["Kernel Name"]
    us = float(d["gpu__time_duration.sum"].replace(",", "")) / 1e3
    rd = float(d["dram__bytes_read.sum"].replace(",", ""))
    wr = float(d["dram__bytes_write.sum"].replace(",", ""))
    if "dec_fused" in name:
        w = 2 * (5120 * rp[fused] + rp[fused + 1] * 5120)
        fused += 1
    elif "<1>" in name or ", 1>" in name:
        w = 2 * 5120 * rp[-1]
    else:
        w = 2 * rp[0] * 5120
    launches.append({"kernel": name.split("(")[0][-40:], "grid": d.get("launch__grid_size"), "us_cold": us,
                     "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6, "weight_bytes_MB": w / 1e6})
f = [l for l in launches if "dec_fused" in l["kernel"]]
summary = {"what": "ncu --set full --clock-control none of one decode pass (M=32 token group, BN=32) through the "
                   "7-variant cfg2 chain (tools/prof_stack.py): dec_kernel<...,0> = layer-0 phase A, dec_fused_kernel = "
                   "the 6 layer boundaries, dec_kernel<...,1> = last phase B. Cold and serialised: compare shares, "
                   "not absolute times.",
           "source": note, "launches": launches,
           "fused_mean_dram_bytes_per_launch": sum(1e6 * (l["dram_read_MB"] + l["dram_write_MB"]) for l in f) / len(f),
           "fused_mean_weight_bytes_per_launch": sum(1e6 * l["weight_bytes_MB"] for l in f) / len(f),
           "fused_mean_us_cold": sum(l["us_cold"] for l in f) / len(f)}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "launches"}))
