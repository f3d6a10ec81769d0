mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "repeatable" > gpurun_out/t_rep.log 2>&1; echo "rc=$?" >> gpurun_out/t_rep.log
