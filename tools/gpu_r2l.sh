mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -rs > gpurun_out/r2l_dp.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_dp.log
timeout 600 python -m pytest tests/test_gpu_engine.py -q -x -k "peer_comm" > gpurun_out/r2l_w1.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_w1.log
