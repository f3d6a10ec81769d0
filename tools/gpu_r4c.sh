# fused dQ cast A/B (attention backward), attention tests
mkdir -p gpurun_out
for m in 0 1 0 1; do GS_DQ_FUSED=$m timeout 300 python tools/attn_bwd_ab.py >> gpurun_out/r4c_ab.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "attention or attn" > gpurun_out/r4c_attn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4c_attn_tests.log
