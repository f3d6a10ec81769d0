# AVX-512 host Adam on the GPU box: bit-exactness there, host-tier engine / parity tests, bench, trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_host_adam.py -q > gpurun_out/r3g_host_adam.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_host_adam.log
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_production_parity.py -q -x -m gpu -k "3 or OPT_HOST or host or fp32_mode" > gpurun_out/r3g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3g_bench.log
timeout 600 python tools/trace_phase.py > gpurun_out/r3g_trace.log 2>&1
python -c "import paper_2512_17570_b200 as gs; print(gs.host_probe())" > gpurun_out/r3g_host_probe.log 2>&1
