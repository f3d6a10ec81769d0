# round-2 re-entry: full validation pass at HEAD (tests, smoke, bench, reference arm, launch list)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2n_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_smoke.log
timeout 900 python bench.py > gpurun_out/r2n_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/r2n_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_ref.log
timeout 900 python bench.py --config gpt1.3b-hbm-opt --no-cpu-baseline > gpurun_out/r2n_bench_hbm.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_bench_hbm.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2n_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --calibrate 0 > gpurun_out/r2n_ncu_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_ncu_bench.log
gzip -f gpurun_out/r2n_launches.csv
