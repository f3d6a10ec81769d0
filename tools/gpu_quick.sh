mkdir -p gpurun_out
timeout 120 python tools/attn_grid_trace.py > gpurun_out/attn_grid.txt 2>&1
