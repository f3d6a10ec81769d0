mkdir -p gpurun_out
L=paper_2512_17570_b200/libgreedysnake.so
cp $L /tmp/lib_new.so
rm -f gpurun_out/attn_ab.txt
for r in 1 2 3; do
  cp /tmp/lib_new.so $L; echo "new $(timeout 120 python tools/gemm_probe.py 2>&1 | sed -n 1p)" >> gpurun_out/attn_ab.txt
  cp paper_2512_17570_b200/libgreedysnake_prev.so $L; echo "prev $(timeout 120 python tools/gemm_probe.py 2>&1 | sed -n 1p)" >> gpurun_out/attn_ab.txt
done
cp /tmp/lib_new.so $L
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "attention" > gpurun_out/t_attn.log 2>&1; echo "rc=$?" >> gpurun_out/t_attn.log
