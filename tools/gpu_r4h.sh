# GPT-65B 8-layer slice batch sweep at HEAD (AVX-512 host Adam), host-core tier, per-slice placement
mkdir -p gpurun_out
for M in 32 64 96 128; do timeout 1800 python bench.py --config gpt65b-8layer --microbatches $M --ssd-ring 4 --opt-tier 3 --steps 3 --warmup 3 --calibrate 0 --no-cpu-baseline > gpurun_out/r4h_bench65_m${M}.log 2>&1; echo "rc=$?" >> gpurun_out/r4h_bench65_m${M}.log; done
