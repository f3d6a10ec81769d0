mkdir -p gpurun_out
grep -m1 "model name" /proc/cpuinfo > gpurun_out/r2h_cpu.txt; grep -m1 flags /proc/cpuinfo | tr ' ' '\n' | grep -E "avx512f|avx2|amx" >> gpurun_out/r2h_cpu.txt; lscpu >> gpurun_out/r2h_cpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -rs > gpurun_out/r2h_engine.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_engine.log
timeout 900 python bench.py --config gpt1.3b-host-opt --no-cpu-baseline > gpurun_out/r2h_bench_host.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_bench_host.log
timeout 600 python tools/trace_phase.py 16 3 > gpurun_out/r2h_trace_host.log 2>&1
timeout 900 python bench.py --config gpt1.3b-stream-opt --no-cpu-baseline > gpurun_out/r2h_bench_stream.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_bench_stream.log
