mkdir -p gpurun_out
GS_TRACE_SSD_LIST=1 timeout 1200 python tools/trace_phase.py --config gpt65b-8layer --ring 4 > gpurun_out/r3a_trace65.log 2>&1
GS_TRACE_SSD_LIST=1 timeout 1200 python tools/trace_phase.py 32 3 --config gpt65b-8layer --ring 4 > gpurun_out/r3a_trace65_host.log 2>&1
