#!/bin/bash
# ncu per-launch device time and DRAM bytes across one full M=16 bench
# iteration (after 3 warm-up iterations of ~10.2k launches): kernel-time
# shares, and per-launch DRAM traffic of the tcgen05 GEMM for bench.py's
# roofline.traffic.  Cold-cache and serialised: compare SHARES.
out=gpurun_out
mkdir -p $out
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -s 30700 -c 10300 --csv --log-file $out/launches_m16.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > $out/ncu_bench_m16.log 2>&1
echo "rc=$?"
