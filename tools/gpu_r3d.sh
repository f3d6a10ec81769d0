# configs[2] shape (GPT-13B, half the Adam state on NVMe) alpha on/off x M on the per-slice placement
mkdir -p gpurun_out
timeout 3000 python tools/sweep.py --model gpt13b --tier 3 > gpurun_out/r3d_sweep13b.jsonl 2> gpurun_out/r3d_sweep13b.err
