"""Does GPU compute slow the PCIe copies?  Bidirectional 16 MiB copies
(pinned <-> HBM) alone, then while a bf16 GEMM loop (tcgen05, GPT-1.3B FC1
shape) runs on another stream."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()
MB = 1 << 20
chunk, n = 16 * MB, 64
h_src = torch.empty(n * chunk, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n * chunk, dtype=torch.uint8, pin_memory=True)
d_buf = torch.empty(2 * n * chunk, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
M, N, K = 4096, 8192, 2048
A = torch.randn(M * K, device="cuda").bfloat16()
B = torch.randn(N * K, device="cuda").bfloat16()
Cc = torch.empty(M * N, device="cuda", dtype=torch.bfloat16)
G = torch.empty(M * N, device="cuda", dtype=torch.bfloat16)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def copies():
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s1)
    s2.wait_event(ev0)
    for i in range(n):
        with torch.cuda.stream(s1):
            d_buf[i * chunk:(i + 1) * chunk].copy_(h_src[i * chunk:(i + 1) * chunk], non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst[i * chunk:(i + 1) * chunk].copy_(d_buf[(n + i) * chunk:(n + i + 1) * chunk], non_blocking=True)
    s1.wait_stream(s2)
    ev1.record(s1)
    return ev0, ev1


for mode in ("alone", "with_gemm", "with_gemm_capped", "alone"):
    torch.cuda.synchronize()
    if mode.startswith("with_gemm"):
        with torch.cuda.stream(s3):
            # "capped": ~1 s of GEMMs queued, copies start behind 0.4 s of them
            # so the GPU is at its power cap while they run
            for _ in range(200 if mode == "with_gemm" else 6000):
                gs.check(lib.gs_gemm(1, M, N, K, p(A), 1, p(B), 1, p(Cc), None, p(G), 3, C.c_void_p(s3.cuda_stream)))
    if mode == "with_gemm_capped":

        import time; time.sleep(0.4)
    e0, e1 = copies()
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "gbs_per_direction": n * chunk / (e0.elapsed_time(e1) / 1e3) / 1e9}), flush=True)
