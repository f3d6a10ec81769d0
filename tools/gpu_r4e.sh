# final HEAD validation: full GPU suite (incl. the bench-workload parity test), smoke, bench + reference arm
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -rs > gpurun_out/r4e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4e_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4e_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r4e_smoke.log
timeout 900 python bench.py > gpurun_out/r4e_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4e_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r4e_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r4e_ref.log
