mkdir -p gpurun_out
python - > gpurun_out/nvme_uring.txt 2>&1 <<'PY'
import ctypes as C, os, subprocess, sys
sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs
out = (C.c_double * 3)()
gs.check(gs.lib().gs_nvme_probe(b"/tmp", C.c_uint64(4 << 30), out)); print("uring", list(out))
PY
GS_NVME_URING=0 python - >> gpurun_out/nvme_uring.txt 2>&1 <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs
out = (C.c_double * 3)()
gs.check(gs.lib().gs_nvme_probe(b"/tmp", C.c_uint64(4 << 30), out)); print("threads", list(out))
PY
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q > gpurun_out/t_engine_uring.log 2>&1; echo "rc=$?" >> gpurun_out/t_engine_uring.log
timeout 2700 python tools/sweep.py --model gpt13b --steps 2 --warmup 1 > gpurun_out/sweep13b.jsonl 2> gpurun_out/sweep13b.err
