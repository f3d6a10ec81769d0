mkdir -p gpurun_out
timeout 300 python tools/attn_grid_trace.py > gpurun_out/attn_grid.txt 2>&1
timeout 300 python tools/attn_accuracy.py > gpurun_out/attn_acc.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention or fused" > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
