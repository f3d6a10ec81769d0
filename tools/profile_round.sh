#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU).
#  1. launch list of one bench step (after 3 warm-up iterations)
#  2. --set full capture of the top kernels (tcgen05 GEMM, flash attention)
set -x
out=gpurun_out
mkdir -p $out
export GS_BENCH_SMALL=1
# ~10.6k launches per 1.3B iteration; skip warm-up + timed value run, capture one iteration
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 42000 -c 11000 --csv \
  --log-file $out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 40 -c 3 \
  -o $out/prof_gemm python tools/gemm_probe.py > $out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fa_ -s 6 -c 4 \
  -o $out/prof_attn python tools/gemm_probe.py > $out/ncu_attn.log 2>&1
ls -la $out
