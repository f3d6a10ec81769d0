mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dp.py -q -x -rs > gpurun_out/r2x_dp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2x_dp_tests.log
