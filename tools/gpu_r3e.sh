# GPT-65B slice: NVMe staging ring 4 vs 8 (slot-reuse hazards) at M=32 / 96, and an SSD task trace
mkdir -p gpurun_out
GS_TRACE_SSD_LIST=1 timeout 1200 python tools/trace_phase.py --config gpt65b-8layer > gpurun_out/r3e_trace65_m32.log 2>&1
for M in 32 96; do timeout 1800 python bench.py --config gpt65b-8layer --microbatches $M --ssd-ring 8 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r3e_bench65_m${M}_ring8.log 2>&1; echo "rc=$?" >> gpurun_out/r3e_bench65_m${M}_ring8.log; done
