#!/bin/bash
# ncu per-launch device times across one full M=16 bench iteration (after 3
# warm-up iterations of ~10.2k launches); compare the kernel-time sum with the
# measured iteration time to size the inter-kernel gaps.
out=gpurun_out
mkdir -p $out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 30700 -c 10300 --csv \
  --log-file $out/launches_m16.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > $out/ncu_bench_m16.log 2>&1
echo "rc=$?"
