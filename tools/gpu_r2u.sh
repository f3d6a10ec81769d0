# world-4 data-parallel functional run under the bench harness (4 ranks share cuda:0), HEAD bench + reference arm
mkdir -p gpurun_out
timeout 1500 python bench.py --gpus 4 --share-gpu --steps 2 --warmup 3 --no-cpu-baseline --calibrate 0 > gpurun_out/r2u_bench_dp4.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench_dp4.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/r2u_bench_dp4.log
timeout 900 python bench.py > gpurun_out/r2u_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r2u_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_ref.log
