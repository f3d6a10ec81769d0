# round-2 first GPU pass: GPU tests, smoke, bench (configs[1] as written), reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
df -h /tmp . > gpurun_out/df.txt; free -g >> gpurun_out/df.txt; nproc >> gpurun_out/df.txt
timeout 1500 python -m pytest tests -m gpu -q -rs -s -k "production_parity" > gpurun_out/r2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r2_parity.log
timeout 1500 python -m pytest tests -m gpu -q -rs -k "not production_parity" > gpurun_out/r2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.log
timeout 900 python bench.py --config gpt1.3b-hbm-opt --no-cpu-baseline > gpurun_out/r2_bench_hbm.log 2>&1; echo "rc=$?" >> gpurun_out/r2_bench_hbm.log
