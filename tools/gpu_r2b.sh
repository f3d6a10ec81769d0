mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs -s -k "production_parity or test_cli" > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2b_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_bench.log
