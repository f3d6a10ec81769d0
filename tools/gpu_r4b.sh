# attribution runs: layer burst vs sustained (power cap), event-bracketed GEMM spans, host Adam thread count with the AVX-512 step
mkdir -p gpurun_out
timeout 300 python tools/layer_sustained.py > gpurun_out/r4b_layer_sustained.log 2>&1
GS_PROF_SPAN_ON_EVENTS=1 timeout 600 python bench.py --no-cpu-baseline --calibrate 0 > gpurun_out/r4b_bench_span_on_events.log 2>&1
for t in 6 8 16; do timeout 600 python tools/trace_phase.py 16 3 $t > gpurun_out/r4b_trace_t$t.log 2>&1; done
