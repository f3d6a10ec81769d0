"""Layer FwdCompute / RecomputeAndBwd back to back (gs_layer_bench, no
executor, no offload) at the GPT-1.3B layer geometry, short burst vs sustained
(long enough for the board to reach its power cap), with the SM clock sampled
by nvidia-smi during each run: separates the in-step backward time into what
the power cap explains and what the executor adds."""
import ctypes as C
import json
import subprocess
import sys
import threading
import time

sys.path.insert(0, ".")
import paper_2512_17570_b200 as gs  # noqa: E402

lib = gs.lib()


def clocks_during(fn):
    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                      "-i", "0"], capture_output=True, text=True, timeout=5).stdout.strip()
                mhz, w = out.split(",")
                samples.append((float(mhz), float(w)))
            except Exception:
                pass
            time.sleep(0.05)

    t = threading.Thread(target=poll)
    t.start()
    r = fn()
    stop.set()
    t.join()
    samples.sort()
    med = samples[len(samples) // 2] if samples else (None, None)
    return r, med, len(samples)


for iters in (10, 100, 1000):
    out = (C.c_double * 4)()
    _, (mhz, w), n = clocks_during(lambda: gs.check(lib.gs_layer_bench(1, 2, 2048, 2048, 16, iters, out)))
    print(json.dumps(dict(iters=iters, fwd_ms=out[0], recompute_bwd_ms=out[2], sm_mhz_median=mhz, power_w=w,
                          clock_samples=n)), flush=True)
