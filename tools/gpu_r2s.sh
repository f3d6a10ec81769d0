# round-2 ablations on the current code: 1.3B batch sweep / alpha 0 / horizontal / optimizer state on NVMe
# (host-core CpuStep), 13B configs[2] shape alpha on/off x M
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --tier 3 > gpurun_out/r2s_sweep13.jsonl 2> gpurun_out/r2s_sweep13.err
timeout 2700 python tools/sweep.py --model gpt13b --tier 3 > gpurun_out/r2s_sweep13b.jsonl 2> gpurun_out/r2s_sweep13b.err
