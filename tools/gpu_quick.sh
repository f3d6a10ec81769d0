mkdir -p gpurun_out
rm -f gpurun_out/bn_ab.txt
for r in 1 2 3; do for v in 1 0; do
  echo "bn192=$v $(GS_GEMM_BN192=$v timeout 120 python tools/gemm_probe.py 2>&1 | grep fwd_qkv)" >> gpurun_out/bn_ab.txt
done; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" > gpurun_out/t_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/t_gemm.log
for r in 1 2; do for v in 1 0; do
  GS_GEMM_BN192=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1
  echo "bench bn192=$v $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/bn_ab.txt
done; done
