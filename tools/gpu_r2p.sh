# LayerNorm forward single-pass, 1.3B bench with it, GPT-65B slice: staging-ring A/B and batch sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm" > gpurun_out/r2p_ln_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_ln_tests.log
timeout 900 python tools/gemm_probe.py 2>&1 | grep -E "ln_|layer_" > gpurun_out/r2p_probe_ln.jsonl
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2p_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_bench.log
timeout 900 python tools/trace_phase.py --config gpt65b-8layer --ring 2 > gpurun_out/r2p_trace65_ring2.log 2>&1
timeout 900 python tools/trace_phase.py --config gpt65b-8layer --ring 4 > gpurun_out/r2p_trace65_ring4.log 2>&1
for M in 64 96; do timeout 1500 python bench.py --config gpt65b-8layer --microbatches $M --ssd-ring 4 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r2p_bench65_m$M.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_bench65_m$M.log; done
