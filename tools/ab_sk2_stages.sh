# A/B: split-K pair first prefill step with 7 (default build) vs 8 TMA stages (libtnl_sk8.so).
set -x
D=paper_2602_01613_b200
cp $D/libtnl.so /tmp/libtnl_base.so
for r in 1 2; do
  cp /tmp/libtnl_base.so $D/libtnl.so; python tools/bench_prefill.py --ranks 32,64,128 --iters 50 > gpurun_out/ab_base_$r.jsonl 2>&1
  cp $D/libtnl_sk8.so $D/libtnl.so;   python tools/bench_prefill.py --ranks 32,64,128 --iters 50 > gpurun_out/ab_sk8_$r.jsonl 2>&1
done
cp $D/libtnl_sk8.so $D/libtnl.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_sk8.log 2>&1; tail -2 gpurun_out/pytest_sk8.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_v15.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
for f in gpurun_out/ab_*.jsonl; do echo "== $f"; cut -c1-220 $f; done
