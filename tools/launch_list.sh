#!/bin/bash
# ncu per-launch device times of one timed bench iteration (cold-cache,
# serialised: compare SHARES).  M=2 micro-batches keeps ncu's per-launch
# serialisation within minutes; kernels per (layer, micro-batch) are the
# same as at M=16.
out=gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 4200 -c 1700 --csv \
  --log-file $out/launches_m2.csv python bench.py --steps 1 --warmup 3 --microbatches 2 --no-cpu-baseline \
  > $out/ncu_bench_m2.log 2>&1
echo "rc=$?"; wc -l $out/launches_m2.csv; tail -3 $out/ncu_bench_m2.log
