# per-slice SSD placement: oracle parity, per-task physical bytes, GPT-65B / 175B slices
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_dp.py tests/test_cli.py -q -x -rs -m gpu > gpurun_out/r3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_tests.log
GS_TRACE_SSD_LIST=1 timeout 1200 python tools/trace_phase.py --config gpt65b-8layer --ring 4 > gpurun_out/r3b_trace65.log 2>&1
timeout 1500 python bench.py --config gpt65b-8layer --ssd-ring 4 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3b_bench65_m32.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_bench65_m32.log
timeout 1500 python bench.py --config gpt65b-8layer --microbatches 64 --ssd-ring 4 --opt-tier 3 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3b_bench65_m64_host.log 2>&1; echo "rc=$?" >> gpurun_out/r3b_bench65_m64_host.log
