mkdir -p gpurun_out
rm -f gpurun_out/prio_ab.txt
for r in 1 2; do for p in 0 1 2; do
  GS_STREAM_PRIO=$p timeout 600 python bench.py > gpurun_out/b.log 2>&1
  echo "prio=$p $(tail -1 gpurun_out/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/prio_ab.txt
done; done
