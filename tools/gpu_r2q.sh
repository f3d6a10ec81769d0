# GEMM in-kernel span roofline, one-iteration launch list with the new LayerNorm, GPT-65B M=128 and the host-Adam tier
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2q_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_bench.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 21400 -c 7200 --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --calibrate 0 > gpurun_out/r2q_ncu_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_ncu_bench.log
gzip -f gpurun_out/r2q_launches.csv
timeout 1800 python bench.py --config gpt65b-8layer --microbatches 128 --ssd-ring 4 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r2q_bench65_m128.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_bench65_m128.log
timeout 1500 python bench.py --config gpt65b-8layer --microbatches 64 --ssd-ring 4 --opt-tier 3 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r2q_bench65_m64_host.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_bench65_m64_host.log
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pytest.log
