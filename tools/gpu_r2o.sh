# LayerNorm rewrite (C <= 2 vectors per lane) + host-worker scheduling A/B + GPT-65B slice
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/r2o_ln_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_ln_tests.log
timeout 900 python tools/gemm_probe.py > gpurun_out/r2o_probe.jsonl 2> gpurun_out/r2o_probe.err; echo "rc=$?" >> gpurun_out/r2o_probe.err
timeout 600 python tools/trace_phase.py 16 3 > gpurun_out/r2o_trace_nice.log 2>&1
GS_HOST_SCHED=idle timeout 600 python tools/trace_phase.py 16 3 > gpurun_out/r2o_trace_idle.log 2>&1
timeout 1500 python bench.py --config gpt65b-8layer --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r2o_bench_65b.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_bench_65b.log
df -h /tmp > gpurun_out/r2o_df.txt; free -g >> gpurun_out/r2o_df.txt
# one full M=16 iteration's launch list (skip the 3 warm-up iterations, 10146 launches each)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 30438 -c 10146 --csv --log-file gpurun_out/r2o_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --calibrate 0 > gpurun_out/r2o_ncu_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2o_ncu_bench.log
gzip -f gpurun_out/r2o_launches.csv
