"""Does the size of the pinned host region matter?  Bidirectional 16 MiB
pinned <-> HBM copies cycling through a small (1 GiB) region vs walking a
large one (8 GiB per direction, every copy a fresh range) — the executor's
checkpoint / parameter images are several GB.  Also: the same over memory
from aligned_alloc + madvise(MADV_HUGEPAGE) + cudaHostRegister."""
import ctypes as C
import json
import mmap

import torch

MB, GB = 1 << 20, 1 << 30
chunk = 16 * MB
libc = C.CDLL("libc.so.6")
libc.aligned_alloc.restype = C.c_void_p
libc.aligned_alloc.argtypes = [C.c_size_t, C.c_size_t]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
libc.memset.argtypes = [C.c_void_p, C.c_int, C.c_size_t]
libc.memset.restype = C.c_void_p
cudart = C.CDLL("libcudart.so") if False else None
try:
    cudart = C.CDLL("libcudart.so.12")
except OSError:
    import glob
    import os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = C.CDLL(cands[0])
cudart.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]


def thp_buffer(nbytes, huge):
    p = libc.aligned_alloc(2 * MB, nbytes)
    if huge:
        libc.madvise(p, nbytes, 14)  # MADV_HUGEPAGE
    libc.memset(p, 1, nbytes)
    assert cudart.cudaHostRegister(C.c_void_p(p), C.c_size_t(nbytes), 0) == 0
    return p


def torch_buffer(nbytes):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    t.fill_(1)
    return t.data_ptr(), t


big = 8 * GB
d_a = torch.empty(GB, dtype=torch.uint8, device="cuda")
d_b = torch.empty(GB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
cudart.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]


def run(h_src, h_dst, region, n=128):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s1)
    s2.wait_event(e0)
    for i in range(n):
        off = (i * chunk) % region
        doff = (i * chunk) % GB
        cudart.cudaMemcpyAsync(C.c_void_p(d_a.data_ptr() + doff), C.c_void_p(h_src + off), chunk, 1, C.c_void_p(s1.cuda_stream))
        cudart.cudaMemcpyAsync(C.c_void_p(h_dst + off), C.c_void_p(d_b.data_ptr() + doff), chunk, 2, C.c_void_p(s2.cuda_stream))
    s1.wait_stream(s2)
    e1.record(s1)
    torch.cuda.synchronize()
    return n * chunk / (e0.elapsed_time(e1) / 1e3) / 1e9


keep = []
for name, mk in (("torch_pinned", lambda n: torch_buffer(n)), ("register_4k", lambda n: (thp_buffer(n, False), None)),
                 ("register_thp", lambda n: (thp_buffer(n, True), None))):
    src, a = mk(big)
    dst, b = mk(big)
    keep += [a, b]
    for region in (GB, big):
        run(src, dst, region, 16)
        r = max(run(src, dst, region) for _ in range(3))
        print(json.dumps({"alloc": name, "region_gb": region / GB, "bidir_gbs_per_direction": r}), flush=True)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
