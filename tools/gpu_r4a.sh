# re-entry HEAD validation (AVX-512 host Adam): bit-exactness on the box CPU, full GPU suite, smoke, bench + reference arm, trace
mkdir -p gpurun_out
python -c "import paper_2512_17570_b200 as gs; print(gs.host_probe())" > gpurun_out/r4a_host_probe.log 2>&1
timeout 600 python -m pytest tests/test_host_adam.py -q > gpurun_out/r4a_host_adam.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_host_adam.log
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r4a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_smoke.log
timeout 900 python bench.py > gpurun_out/r4a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r4a_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_ref.log
timeout 600 python tools/trace_phase.py > gpurun_out/r4a_trace.log 2>&1
