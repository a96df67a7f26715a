"""Summarise an `ncu --set full` capture of tools/prof_stack.py (one or more decode passes
through the 7-variant cfg2 chain) into profiles/<round>/ncu_dec_fused.json, the file bench.py
reads for roofline.traffic.

    python tools/ncu_summary.py gpurun_out/ncu_stack_v9.ncu-rep profiles/r01/ncu_dec_fused.json
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
metrics = "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
ix = {k: h.index(k) for k in h}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# weight bytes (bf16) per launch of the chain: phase A of layer 0 = B_in^0; boundary l = A_out^l + B_in^{l+1};
# last phase B = A_out^6. cfg2 variants in S.CFG2_VARIANTS order, cut ranks padded to 16: 64,128,256,64,256,64,256
cuts = [64, 128, 256, 64, 256, 64, 256]
wb = [2 * 5120 * cuts[0]] + [2 * 5120 * (cuts[l] + cuts[l + 1]) for l in range(6)] + [2 * 5120 * cuts[6]]
launches = []
for k, r in enumerate(rows[2:]):
    rd = float(r[ix["dram__bytes_read.sum"]]) * scale[units[ix["dram__bytes_read.sum"]]]
    wr = float(r[ix["dram__bytes_write.sum"]]) * scale[units[ix["dram__bytes_write.sum"]]]
    launches.append({"kernel": r[ix["Kernel Name"]].split("(")[0].replace("void ", ""), "grid": int(r[ix["launch__grid_size"]]),
                     "us_cold": float(r[ix["gpu__time_duration.sum"]]), "dram_read_MB": rd / 1e6,
                     "dram_write_MB": wr / 1e6, "weight_bytes_MB": wb[k % 8] / 1e6})
fused = [l for l in launches if "dec_fused_kernel" in l["kernel"]]
res = {
    "what": "ncu --set full --clock-control none of decode passes (M=32 token group, BN=32) through the 7-variant "
            "cfg2 chain (tools/prof_stack.py): dec_kernel<32,4,0> = layer-0 phase A, dec_fused_kernel<32> = the 6 "
            "layer boundaries, dec_kernel<32,4,1> = last phase B. Cold and serialised: compare shares, not absolute times.",
    "source": rep,
    "launches": launches,
    "fused_mean_dram_bytes_per_launch": sum((l["dram_read_MB"] + l["dram_write_MB"]) * 1e6 for l in fused) / len(fused),
    "fused_mean_weight_bytes_per_launch": sum(l["weight_bytes_MB"] * 1e6 for l in fused) / len(fused),
    "fused_mean_us_cold": sum(l["us_cold"] for l in fused) / len(fused),
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}, indent=1))
