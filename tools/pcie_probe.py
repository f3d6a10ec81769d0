"""PCIe copy-engine probe: pinned host <-> HBM bandwidth for 16 MiB copies
(the executor's checkpoint size class), one vs two CUDA streams per
direction, one direction alone vs both at once."""
import json

import torch

MB = 1 << 20
chunk, n = 16 * MB, 64  # 1 GiB per direction
h_src = torch.empty(n * chunk, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n * chunk, dtype=torch.uint8, pin_memory=True)
d_dst = torch.empty(n * chunk, dtype=torch.uint8, device="cuda")
d_src = torch.empty(n * chunk, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(h2d_streams, d2h_streams, split=1):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for s in streams:
        s.wait_event(ev0)
    for i in range(n):
        for k in range(split):
            lo, hi = i * chunk + k * chunk // split, i * chunk + (k + 1) * chunk // split
            if h2d_streams:
                with torch.cuda.stream(streams[(i * split + k) % h2d_streams]):
                    d_dst[lo:hi].copy_(h_src[lo:hi], non_blocking=True)
            if d2h_streams:
                with torch.cuda.stream(streams[2 + (i * split + k) % d2h_streams]):
                    h_dst[lo:hi].copy_(d_src[lo:hi], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    return (n * chunk) / (ms / 1e3) / 1e9


for name, args in [("h2d_1s", (1, 0)), ("h2d_2s", (2, 0)), ("h2d_2s_split", (2, 0, 2)), ("d2h_1s", (0, 1)),
                   ("d2h_2s", (0, 2)), ("bidir_1s", (1, 1)), ("bidir_2s", (2, 2)), ("bidir_2s_split", (2, 2, 2))]:
    run(*args)
    best = max(run(*args) for _ in range(3))
    print(json.dumps({"pattern": name, "gbs_per_direction": best}), flush=True)
