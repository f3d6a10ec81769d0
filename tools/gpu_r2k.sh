mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs -x > gpurun_out/r2k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_smoke.log
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_bench.log
