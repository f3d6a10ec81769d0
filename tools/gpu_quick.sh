mkdir -p gpurun_out
timeout 1500 python bench.py --config gpt13b-nvme --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.log 2>&1; echo "rc=$?" >> gpurun_out/bench13.log
