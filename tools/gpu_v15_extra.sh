# v15: decode-chain launch list of the bench (dec_* kernels only) + repeat the gate r64 prefill timing across processes.
set -x
for r in 1 2 3 4 5; do python tools/bench_prefill.py --ranks 64 --iters 50 2>&1 | grep '"plan"' | cut -c1-120; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:dec -c 300 --csv \
  --log-file gpurun_out/launches_bench_dec_v15.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch_dec.log 2>&1; echo launches rc=$?
