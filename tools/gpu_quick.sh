mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/pdl_ab.txt
for r in 1 2; do for v in 1 0; do
  GS_PDL=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1
  echo "pdl=$v $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["losses"][-1] if d.get("losses") else None)')" >> gpurun_out/pdl_ab.txt
done; done
for v in 1 0; do echo "probe pdl=$v $(GS_PDL=$v timeout 120 python tools/gemm_probe.py 2>&1 | grep layer_ | tr '\n' ' ')" >> gpurun_out/pdl_ab.txt; done
