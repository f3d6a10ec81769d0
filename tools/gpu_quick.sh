mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/t_k.log 2>&1; echo "rc=$?" >> gpurun_out/t_k.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench23.log 2>&1
