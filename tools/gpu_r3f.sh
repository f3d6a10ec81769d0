# final HEAD validation: full GPU suite, smoke, driver bench + reference arm, 65B slice at the saturating batch
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r3f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_smoke.log
timeout 900 python bench.py > gpurun_out/r3f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r3f_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_ref.log
timeout 1800 python bench.py --config gpt65b-8layer --microbatches 96 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3f_bench65_m96.log 2>&1; echo "rc=$?" >> gpurun_out/r3f_bench65_m96.log
