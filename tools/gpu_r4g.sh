# per-sample event vs in-kernel span of the timed GEMM launches: default host tier, 4 host threads, HBM-resident optimizer (no host Adam)
mkdir -p gpurun_out
GS_PROF_SPAN_ON_EVENTS=1 GS_PROF_DUMP=gpurun_out/r4g_pairs_host12.csv GS_HOST_PROF=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 > gpurun_out/r4g_host12.log 2>&1
GS_PROF_SPAN_ON_EVENTS=1 GS_PROF_DUMP=gpurun_out/r4g_pairs_host4.csv GS_HOST_PROF=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 --host-threads 4 > gpurun_out/r4g_host4.log 2>&1
GS_PROF_SPAN_ON_EVENTS=1 GS_PROF_DUMP=gpurun_out/r4g_pairs_hbm.csv GS_HOST_PROF=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 --config gpt1.3b-hbm-opt > gpurun_out/r4g_hbm.log 2>&1
