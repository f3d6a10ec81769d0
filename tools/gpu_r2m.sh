mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/r2m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_pytest.log
timeout 900 python bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench_dp2.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_bench_dp2.log
