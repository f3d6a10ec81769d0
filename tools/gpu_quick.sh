mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/gemm_probe.py > gpurun_out/probe21_$i.jsonl 2>&1; done
