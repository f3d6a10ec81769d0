# bench workload (24 layers, M=16) vs torch fp32 parity test
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_production_parity.py -q -s -m gpu -k bench_configuration > gpurun_out/r4d_bench_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r4d_bench_parity.log
