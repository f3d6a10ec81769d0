"""Pinned-memory flavour vs PCIe throughput: cudaHostAlloc default vs
write-combined vs portable|mapped, 16 MiB copies, each direction alone and
both at once (cudart through ctypes)."""
import ctypes as C
import json

import torch

rt = C.CDLL("libcudart.so")
MB = 1 << 20
chunk, n = 16 * MB, 64
dev = torch.empty(2 * n * chunk, dtype=torch.uint8, device="cuda")
d_dst, d_src = dev[: n * chunk], dev[n * chunk:]
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()


def host(flags):
    p = C.c_void_p()
    assert rt.cudaHostAlloc(C.byref(p), C.c_size_t(n * chunk), C.c_uint(flags)) == 0
    return p


def run(hsrc, hdst, h2d, d2h):
    kind_h2d, kind_d2h = 1, 2
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    s_h2d.wait_event(ev0)
    s_d2h.wait_event(ev0)
    for i in range(n):
        if h2d:
            rt.cudaMemcpyAsync(C.c_void_p(d_dst.data_ptr() + i * chunk), C.c_void_p(hsrc.value + i * chunk),
                               C.c_size_t(chunk), kind_h2d, C.c_void_p(s_h2d.cuda_stream))
        if d2h:
            rt.cudaMemcpyAsync(C.c_void_p(hdst.value + i * chunk), C.c_void_p(d_src.data_ptr() + i * chunk),
                               C.c_size_t(chunk), kind_d2h, C.c_void_p(s_d2h.cuda_stream))
    torch.cuda.current_stream().wait_stream(s_h2d)
    torch.cuda.current_stream().wait_stream(s_d2h)
    ev1.record()
    torch.cuda.synchronize()
    return n * chunk / (ev0.elapsed_time(ev1) / 1e3) / 1e9


for name, flags in [("default", 0), ("portable", 1), ("write_combined", 4), ("portable_wc", 5)]:
    a, b = host(flags), host(flags)
    res = {}
    for pat, (h, d) in {"h2d": (1, 0), "d2h": (0, 1), "bidir": (1, 1)}.items():
        run(a, b, h, d)
        res[pat] = max(run(a, b, h, d) for _ in range(3))
    print(json.dumps({"flags": name, **res}), flush=True)
    rt.cudaFreeHost(a)
    rt.cudaFreeHost(b)
