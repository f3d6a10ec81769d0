mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
timeout 300 python tools/gemm_probe.py > gpurun_out/probe2.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench2.log 2>&1
