#!/bin/bash
# End-of-round evidence on one B200 (run under gpurun): GPU tests, smoke,
# both bench arms, kernel probe, executor trace summary, attention grid
# schedules, ncu --set full captures of the top kernels (raw pages exported to
# CSV) and the ncu launch list of one M=16 bench iteration.
out=gpurun_out
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/final_pytest.log 2>&1; echo "rc=$?" >> $out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/final_smoke.log 2>&1; echo "rc=$?" >> $out/final_smoke.log
timeout 900 python bench.py > $out/final_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/final_bench_ref.log 2>&1
timeout 300 python tools/gemm_probe.py > $out/final_probe.jsonl 2>&1
timeout 600 python tools/trace_gaps.py 16 6 > $out/final_trace_gaps.txt 2>&1
timeout 300 python tools/attn_grid_trace.py > $out/final_attn_grid.txt 2>&1
for k in "tc_gemm_kernel:qkv" "tc_gemm_kernel:fc1" "tc_gemm_kernel:wgrad" "fa_fwd_tc3:attn_fwd" "fa_bwd_tc4:attn_bwd"; do
  IFS=: read -r name tag <<< "$k"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -s 2 -c 1 \
    -o $out/final_prof_$tag -f python tools/ncu_targets.py $tag > $out/final_ncu_$tag.log 2>&1
  ncu -i $out/final_prof_$tag.ncu-rep --page raw --csv > $out/final_raw_$tag.csv 2>/dev/null
  ncu -i $out/final_prof_$tag.ncu-rep --page source --csv --print-source sass > $out/final_sass_$tag.csv 2>/dev/null
  gzip -f $out/final_sass_$tag.csv
  rm -f $out/final_prof_$tag.ncu-rep   # keep gpurun_out under the 64 MiB copy-back limit
done
bash tools/launch_list_m16.sh > $out/final_launch_list.log 2>&1
gzip -f $out/launches_m16.csv
ls -la $out
