# NVMe queue behaviour inside the GPT-65B slice (per-task GB/s, gaps); world-2 tests with the capped reduce grid
mkdir -p gpurun_out
timeout 1200 python tools/trace_phase.py --config gpt65b-8layer --ring 4 > gpurun_out/r2z_trace65.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/r2z_dp.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_dp.log
