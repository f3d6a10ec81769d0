#!/bin/bash
# full-set ncu of the CTA-pair GEMM variants at GPT-1.3B shapes (gemm_probe order)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel -s 30 -c 6 \
  -o gpurun_out/prof_gemm2 python tools/gemm_probe.py > gpurun_out/ncu_gemm2.log 2>&1
tail -3 gpurun_out/ncu_gemm2.log
