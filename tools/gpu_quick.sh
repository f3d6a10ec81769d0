mkdir -p gpurun_out
timeout 300 python tools/gemm_probe.py > gpurun_out/probe7.jsonl 2>&1
