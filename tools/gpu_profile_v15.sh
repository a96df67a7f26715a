# Round-1 v15 profile pass: launch list of the bench command + ncu --set full of the cfg3 prefill kernels.
set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/b_noprof.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_v15.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/prof_prefill.py || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/prefill_v15 -f \
  python tools/prof_prefill.py > gpurun_out/ncu_prefill.log 2>&1; echo full rc=$?
ncu -i gpurun_out/prefill_v15.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/ncu_prefill_v15_summary.csv 2>&1
cat gpurun_out/ncu_prefill_v15_summary.csv | cut -c1-300
