# horizontal schedule on the host-core tier (the ablation under the vertical run's resource model)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x -k "horizontal" > gpurun_out/r2w_horiz_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_horiz_tests.log
timeout 900 python bench.py --schedule horizontal --no-cpu-baseline --calibrate 0 > gpurun_out/r2w_bench_horizontal.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_bench_horizontal.log
