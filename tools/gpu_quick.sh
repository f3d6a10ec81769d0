mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q > gpurun_out/t_k.log 2>&1; echo "rc=$?" >> gpurun_out/t_k.log
timeout 300 python tools/gemm_probe.py > gpurun_out/probe8.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench8.log 2>&1
