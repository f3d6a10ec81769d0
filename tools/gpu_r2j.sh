mkdir -p gpurun_out
for t in 4 8 12 16; do timeout 600 python tools/trace_phase.py 16 3 $t > gpurun_out/r2j_trace_t$t.log 2>&1; done
