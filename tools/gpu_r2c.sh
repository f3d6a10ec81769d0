mkdir -p gpurun_out
timeout 300 ./tools/probes/zc_probe > gpurun_out/r2c_zc.log 2>&1
timeout 600 python tools/trace_phase.py 16 2 > gpurun_out/r2c_trace.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs -s -k "production_parity and not fp32" > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
