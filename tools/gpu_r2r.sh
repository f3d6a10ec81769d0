# attention backward dQ drain A/B: SMEM staging + TMA reduce-add (default) vs red.global from registers
mkdir -p gpurun_out
for v in 0 1; do
  GS_ATTN_DQ_RED=$v timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" > gpurun_out/r2r_attn_tests_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_attn_tests_$v.log
done
for rep in 1 2; do for v in 0 1; do
  GS_ATTN_DQ_RED=$v timeout 600 python tools/gemm_probe.py attn 2>/dev/null | grep -E '"attn_|layer_' > gpurun_out/r2r_probe_${v}_$rep.jsonl
done; done
# BASELINE configs[4] on a 2-layer slice of the GPT-175B geometry: params + optimizer state on NVMe
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "test_fp32_engine_matches_oracle" > gpurun_out/r2r_engine.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_engine.log
df -h /tmp > gpurun_out/r2r_df.txt
timeout 2700 python bench.py --config gpt175b-2layer --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r2r_bench175.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_bench175.log
