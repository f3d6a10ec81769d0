#!/bin/bash
# Standalone kernel timings + ncu --set full of the GEMM / attention kernels at
# GPT-1.3B shapes (tools/gemm_probe.py launch order).  Run under gpurun.
out=gpurun_out
mkdir -p $out
timeout 300 python tools/gemm_probe.py > $out/probe.jsonl 2> $out/probe.err
# gemm_probe order: 6 GEMM shapes x (3 warm + 20 timed) launches each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 0 -c 1 \
  -o $out/prof_qkv -f python tools/gemm_probe.py > $out/ncu_qkv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 92 -c 1 \
  -o $out/prof_wgrad -f python tools/gemm_probe.py > $out/ncu_wgrad.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_ -s 3 -c 1 \
  -o $out/prof_fafwd -f python tools/gemm_probe.py > $out/ncu_fafwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fa_bwd -s 3 -c 1 \
  -o $out/prof_fabwd -f python tools/gemm_probe.py > $out/ncu_fabwd.log 2>&1
for f in qkv wgrad fafwd fabwd; do
  ncu -i $out/prof_$f.ncu-rep --page raw --csv > $out/raw_$f.csv 2>/dev/null
done
ls -la $out
