# LayerNorm forward bulk-staged vs register-staged A/B; ncu --set full at HEAD (GEMM, attention, LayerNorm)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/r2t_ln_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_ln_tests.log
for rep in 1 2; do for v in 0 1; do
  GS_LN_BULK=$v timeout 600 python tools/gemm_probe.py attn 2>/dev/null | grep -E '"ln_' > gpurun_out/r2t_probe_ln_${v}_$rep.jsonl
done; done
run() {  # tag, kernel regex, skip, args...
  tag=$1; k=$2; sk=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o gpurun_out/r2t_$tag -f python tools/ncu_targets.py "$@" > gpurun_out/r2t_ncu_$tag.log 2>&1
  ncu -i gpurun_out/r2t_$tag.ncu-rep --page raw --csv > gpurun_out/r2t_raw_$tag.csv 2>/dev/null
  gzip -f gpurun_out/r2t_raw_$tag.csv
}
run ln_fwd_2048 ln_fwd 2 ln_fwd 2048
run ln_bwd_2048 ln_bwd 2 ln_bwd 2048
run ln_fwd_8192 ln_fwd 2 ln_fwd 8192
run ln_bwd_8192 ln_bwd 2 ln_bwd 8192
export GS_LN_BULK=0; run ln_fwd_2048_regs ln_fwd 2 ln_fwd 2048; unset GS_LN_BULK
run qkv tc_gemm_kernel 2 qkv
run wgrad tc_gemm_kernel 2 wgrad
run attn_fwd fa_fwd 2 attn_fwd
run attn_bwd fa_bwd 2 attn_bwd
rm -f gpurun_out/r2t_*.ncu-rep
# the data-parallel path under the bench harness: two ranks (torchrun re-launch) sharing cuda:0 — a functional check
timeout 1200 python bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --no-cpu-baseline --calibrate 0 > gpurun_out/r2t_bench_dp2.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_bench_dp2.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2t_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2t_bench.log
