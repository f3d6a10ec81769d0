# GEMM event timing with non-PDL fence grids around the timed pair (span on the same launches), and fence alone
mkdir -p gpurun_out
GS_PROF_FENCE=1 GS_PROF_SPAN_ON_EVENTS=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 > gpurun_out/r4f_fence_span.log 2>&1
GS_PROF_FENCE=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 > gpurun_out/r4f_fence.log 2>&1
