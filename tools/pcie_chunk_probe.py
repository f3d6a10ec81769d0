"""PCIe copy-engine throughput vs copy size, one direction and both at once,
with and without a host-DRAM load running beside it (host threads streaming
memcpy, standing in for the host-core Adam): does the forward phase's 82 GB/s
bidirectional rate come from the plan's 6-17 MB copies, from DRAM contention,
or from the executor?  CUDA events on the copy streams; pinned host memory.

usage: python tools/pcie_chunk_probe.py > gpurun_out/pcie_chunks.jsonl"""
import json
import threading
import time

import numpy as np
import torch

TOTAL = 2 << 30  # bytes per direction per measurement


def run(chunk, bidir, host_load):
    n = TOTAL // chunk
    h_src = torch.empty(TOTAL, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(TOTAL, dtype=torch.uint8, pin_memory=True)
    d_dst = torch.empty(TOTAL, dtype=torch.uint8, device="cuda")
    d_src = torch.empty(TOTAL, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    stop = threading.Event()
    loaders = []
    if host_load:
        a = np.ones(256 << 20, np.uint8)
        b = np.empty_like(a)

        def spin():
            while not stop.is_set():
                np.copyto(b, a)
        loaders = [threading.Thread(target=spin, daemon=True) for _ in range(host_load)]
        for t in loaders:
            t.start()
        time.sleep(0.2)
    for it in range(2):  # warm-up pass, then the timed one
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(s1):
            e[0].record()
            for i in range(n):
                d_dst[i * chunk:(i + 1) * chunk].copy_(h_src[i * chunk:(i + 1) * chunk], non_blocking=True)
            e[1].record()
        if bidir:
            with torch.cuda.stream(s2):
                e[2].record()
                for i in range(n):
                    h_dst[i * chunk:(i + 1) * chunk].copy_(d_src[i * chunk:(i + 1) * chunk], non_blocking=True)
                e[3].record()
        torch.cuda.synchronize()
    stop.set()
    for t in loaders:
        t.join()
    h2d = TOTAL / (e[0].elapsed_time(e[1]) / 1e3) / 1e9
    d2h = TOTAL / (e[2].elapsed_time(e[3]) / 1e3) / 1e9 if bidir else None
    return h2d, d2h


for host_load in (0, 12):
    for bidir in (False, True):
        for chunk in (1 << 20, 4 << 20, 6_291_456, 16_777_216, 64 << 20, 256 << 20, 1 << 30):
            h2d, d2h = run(chunk, bidir, host_load)
            print(json.dumps({"chunk_bytes": chunk, "bidirectional": bidir, "host_memcpy_threads": host_load,
                              "h2d_gbs": round(h2d, 2), "d2h_gbs": round(d2h, 2) if d2h else None}), flush=True)
