mkdir -p gpurun_out
rm -f gpurun_out/attn_var.txt
for v in "GS_ATTN_FWD=2" "GS_ATTN_FWD=3" "GS_ATTN_FWD=2" "GS_ATTN_FWD=3"; do
  echo "$v $(env $v timeout 120 python tools/gemm_probe.py 2>&1 | head -1)" >> gpurun_out/attn_var.txt
done
timeout 120 python tools/attn_accuracy.py > gpurun_out/attn_acc.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do for v in 2 3; do
  GS_ATTN_FWD=$v timeout 600 python bench.py > gpurun_out/b.log 2>&1
  echo "fwd=$v $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/attn_var.txt
done; done
