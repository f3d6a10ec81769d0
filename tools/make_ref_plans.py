"""Freeze plans dumped by the REFERENCE's own builder as golden fixtures.

oracle/_ref/liboffsim_ref.so is the reference offsim library compiled from
/root/reference/proj/src (oracle/Makefile); its plan_to_json
(proj/src/json_io.cpp:142-180) is the `offsim simulate --emit-plan` format
(proj/tests/cli_end_to_end.cmake:64-72).  The GPU box has no /root/reference,
so the replay test (tests/test_cli.py) executes these committed dumps, and a
CPU test re-derives them from the reference wherever it is mounted.

Writes tests/golden/ref_plans/<name>.json (the plan) and <name>.ledger.json
(the reference's vertical_traffic / horizontal_traffic rows, traffic.cpp:44-94).
Run:  python tools/make_ref_plans.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bindings as ob  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "ref_plans")

# name: (variant, (N, h, heads, s, b, lp), M, split, alpha)
CASES = {
    "tiny_vertical_split1_1_05_a025": ("vertical", (4, 64, 4, 32, 2, 4), 4, (1.0, 1.0, 0.5), 0.25),
    "tiny_vertical_allssd_a0": ("vertical", (4, 64, 4, 32, 2, 4), 4, (0.0, 0.0, 0.0), 0.0),
    "tiny_horizontal_split1_1_05": ("horizontal", (4, 64, 4, 32, 2, 4), 4, (1.0, 1.0, 0.5), 0.0),
    "tiny_vertical_bf16_split1_1_1_a02": ("vertical", (2, 256, 2, 256, 2, 2), 2, (1.0, 1.0, 1.0), 0.2),
}


def dump(name):
    variant, (N, h, H, s, b, lp), M, split, alpha = CASES[name]
    model = ob.model_array(N, h, H, s, b, lp=lp)
    plan = ob.ref_plan_json(variant, model, M, split, alpha)
    led = ob.ref_ledger(variant, model, M, split, alpha)
    return plan, {"ledger": led.tolist(), "rows": "link (h2d, d2h, ssd_read, ssd_write) x data kind",
                  "variant": variant, "model": [N, h, H, s, b, lp], "microbatches": M, "split": list(split),
                  "alpha": alpha}


def main():
    os.makedirs(OUT, exist_ok=True)
    for name in CASES:
        plan, led = dump(name)
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            f.write(plan)
        with open(os.path.join(OUT, name + ".ledger.json"), "w") as f:
            json.dump(led, f, indent=1)
        print(name, len(json.loads(plan)["tasks"]), "tasks")


if __name__ == "__main__":
    main()
