mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_all.log
timeout 300 python tools/gemm_probe.py > gpurun_out/probe12.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/bench12.log 2>&1
