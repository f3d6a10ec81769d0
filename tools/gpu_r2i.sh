mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -rs > gpurun_out/r2i_engine.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_engine.log
timeout 900 python bench.py --config gpt1.3b-host-opt --no-cpu-baseline > gpurun_out/r2i_bench_host.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_bench_host.log
timeout 600 python tools/trace_phase.py 16 3 > gpurun_out/r2i_trace_host.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs -s -k "production_parity or test_cli" > gpurun_out/r2i_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_parity.log
