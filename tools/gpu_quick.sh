mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_engine.py -q -k "bf16" > gpurun_out/t_bf16.log 2>&1; echo "rc=$?" >> gpurun_out/t_bf16.log
