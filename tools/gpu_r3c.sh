# per-slice SSD placement: the full GPU suite, then the 65B batch sweep on the host-core tier, 175B slice, 13B alpha on/off at M=32
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r3c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_pytest.log
for M in 32 96 128; do timeout 1800 python bench.py --config gpt65b-8layer --microbatches $M --ssd-ring 4 --opt-tier 3 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3c_bench65_m${M}_host.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_bench65_m${M}_host.log; done
timeout 2700 python bench.py --config gpt175b-2layer --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3c_bench175.log 2>&1; echo "rc=$?" >> gpurun_out/r3c_bench175.log
