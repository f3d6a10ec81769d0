mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/bench_k2.log 2>/dev/null; echo "rc=$?" >> gpurun_out/bench_k2.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/bench_ref_k2.log 2>/dev/null; echo "rc=$?" >> gpurun_out/bench_ref_k2.log
