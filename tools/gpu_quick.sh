mkdir -p gpurun_out
L=paper_2512_17570_b200/libgreedysnake.so
cp $L /tmp/lib_new.so
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/pdl2_ab.txt
for r in 1 2; do
  cp /tmp/lib_new.so $L
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1
  echo "new $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/pdl2_ab.txt
  cp paper_2512_17570_b200/libgreedysnake_prev.so $L
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1
  echo "prev $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/pdl2_ab.txt
done
cp /tmp/lib_new.so $L
for v in new prev; do
  [ $v = prev ] && cp paper_2512_17570_b200/libgreedysnake_prev.so $L
  echo "probe $v $(timeout 120 python tools/gemm_probe.py 2>&1 | grep layer_ | tr '\n' ' ')" >> gpurun_out/pdl2_ab.txt
done
cp /tmp/lib_new.so $L
