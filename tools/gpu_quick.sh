mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
for r in 1 2 3; do for v in new old; do
  if [ $v = old ]; then export GS_AB_KEEP_U=1; else unset GS_AB_KEEP_U; fi
  timeout 600 python bench.py > gpurun_out/b.log 2>&1
  echo "$v $(grep '^{' gpurun_out/b.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"])')" >> gpurun_out/ab.txt
done; done
