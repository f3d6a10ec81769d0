mkdir -p gpurun_out
GS_ATTN_TRACE=1 timeout 300 python tools/gemm_probe.py > /dev/null 2> gpurun_out/attn_trace4.txt
timeout 300 python tools/gemm_probe.py > gpurun_out/probe16.jsonl 2>&1
