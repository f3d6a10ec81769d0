"""ctypes bindings to the TEST-ONLY checkers under oracle/.

* liboracle.so        numeric CPU oracle (oracle/gs_oracle.c)
* _ref/liboffsim_ref  the reference's own offsim library + C shim (oracle/ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liboffsim_ref.so")

# task kinds, as offsim::TaskKind
FWD, BWD, STEP, XFER, FIXED = 0, 1, 2, 3, 4
KIND_OF = {"fwd": FWD, "bwd": BWD, "cpu_step": STEP, "xfer": XFER, "fixed_ops": FIXED}


class GsoCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("n_layers", "hidden", "heads", "seq", "mb_size", "vocab")]


class GsoAdam(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay")]


class GsoTask(C.Structure):
    _fields_ = [("kind", C.c_int), ("layer", C.c_int), ("mb", C.c_int), ("stage", C.c_int),
                ("elements", C.c_longlong)]


@dataclass
class Geometry:
    n_layers: int = 4
    hidden: int = 64
    heads: int = 4
    seq: int = 32
    mb_size: int = 2
    vocab: int = 128

    def cfg(self) -> GsoCfg:
        return GsoCfg(self.n_layers, self.hidden, self.heads, self.seq, self.mb_size, self.vocab)

    @property
    def P(self) -> int:
        return 12 * self.hidden * self.hidden

    @property
    def n_fixed(self) -> int:
        return (self.vocab + self.seq) * self.hidden


# the reference's only tiny GPT: proj/tests/helpers.hpp:10-19 (vocab is ours)
TINY = Geometry()


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


_oracle = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
        lib = C.CDLL(ORACLE_SO)
        lib.gso_normal.restype = C.c_double
        lib.gso_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.gso_splitmix64.restype = C.c_uint64
        lib.gso_splitmix64.argtypes = [C.c_uint64]
        lib.gso_head.restype = C.c_double
        _oracle = lib
    return _oracle


def init_params(g: Geometry, seed: int = 42):
    lib = oracle()
    cfg = g.cfg()
    layers = np.empty((g.n_layers, g.P), np.float32)
    for l in range(g.n_layers):
        lib.gso_init_layer(C.byref(cfg), C.c_uint64(seed), l, _f32p(layers[l]))
    fixed = np.empty(g.n_fixed, np.float32)
    lib.gso_init_fixed(C.byref(cfg), C.c_uint64(seed), _f32p(fixed),
                       _f32p(fixed[g.vocab * g.hidden:]))
    return layers, fixed


def make_tokens(g: Geometry, iters: int, M: int, seed: int = 1234):
    lib = oracle()
    cfg = g.cfg()
    out = np.empty((iters, M, g.mb_size, g.seq + 1), np.int32)
    for it in range(iters):
        lib.gso_make_tokens(C.byref(cfg), C.c_uint64(seed), it, M,
                            out[it].ctypes.data_as(C.POINTER(C.c_int32)))
    return out


def compute_tasks(plan_json: dict):
    """Compute tasks of a plan (JSON dict) in plan order, as GsoTask[]."""
    rows = [t for t in plan_json["tasks"] if t["kind"] != "xfer"]
    arr = (GsoTask * len(rows))()
    for i, t in enumerate(rows):
        arr[i] = GsoTask(KIND_OF[t["kind"]], t["layer"], t["microbatch"], t["stage"],
                         t.get("elements", 0))
    return arr


def train(g: Geometry, adam: dict, M: int, plan_json: dict | None, tokens, layers, fixed,
          flush: bool = True):
    """Run the oracle.  plan_json None -> plain loop.  Returns (losses, layers,
    fixed, (m, v), (fm, fv)) with the inputs left untouched."""
    lib = oracle()
    cfg = g.cfg()
    a = GsoAdam(adam["lr"], adam["beta1"], adam["beta2"], adam["eps"], adam["weight_decay"])
    iters = tokens.shape[0]
    p = np.ascontiguousarray(layers, np.float32).copy()
    f = np.ascontiguousarray(fixed, np.float32).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    fm, fv = np.zeros_like(f), np.zeros_like(f)
    losses = np.zeros(iters, np.float32)
    tok = np.ascontiguousarray(tokens, np.int32)
    tp = tok.ctypes.data_as(C.POINTER(C.c_int32))
    if plan_json is None:
        rc = lib.gso_train_plain(C.byref(cfg), C.byref(a), M, iters, tp, _f32p(losses), _f32p(p),
                                 _f32p(m), _f32p(v), _f32p(f), _f32p(fm), _f32p(fv))
    else:
        tasks = compute_tasks(plan_json)
        rc = lib.gso_train(C.byref(cfg), C.byref(a), M, tasks, len(tasks), iters, tp, _f32p(losses),
                           _f32p(p), _f32p(m), _f32p(v), _f32p(f), _f32p(fm), _f32p(fv), int(flush))
    if rc != 0:
        raise RuntimeError("oracle training failed")
    return losses, p, f, (m, v), (fm, fv)


# ------------------------------------------------------------ reference lib
_ref = None


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


def model_array(n_layers, hidden, heads, seq, mb, lp=2, fp=4, states=3, dp=1):
    return (C.c_int * 9)(n_layers, hidden, heads, seq, mb, lp, fp, states, dp)


VARIANTS = {"single-fb": 0, "horizontal": 1, "vertical": 2}


def ref_plan_json(variant: str, model, mbs: int, split, alpha=0.0, extra=False) -> str:
    lib = ref()
    out = C.c_char_p()
    rc = lib.ref_plan_json(VARIANTS[variant], model, mbs, int(extra), (C.c_double * 3)(*split),
                           C.c_double(alpha), C.byref(out))
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    s = C.string_at(out).decode()
    lib.ref_free(out)
    return s


def ref_ledger(variant: str, model, mbs: int, split, alpha=0.0, extra=False):
    lib = ref()
    out = (C.c_ulonglong * 20)()
    rc = lib.ref_ledger(VARIANTS[variant], model, mbs, int(extra), (C.c_double * 3)(*split),
                        C.c_double(alpha), out)
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    return np.array(list(out), np.uint64).reshape(4, 5)


def ref_simulate_json(plan_json: str, machine) -> str:
    lib = ref()
    out = C.c_char_p()
    rc = lib.ref_simulate_json(plan_json.encode(), (C.c_double * 13)(*machine), C.byref(out))
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    s = C.string_at(out).decode()
    lib.ref_free(out)
    return s


def ref_vertical_plan(g: Geometry, M: int, split=(0, 0, 0), alpha=0.0, lp=4, dp=1) -> dict:
    model = model_array(g.n_layers, g.hidden, g.heads, g.seq, g.mb_size, lp=lp, dp=dp)
    return json.loads(ref_plan_json("vertical", model, M, split, alpha))


def ref_planner(mode: str, model, machine, mbs=1, alpha=0.0, steps=100):
    """Reference planner (oracle/_ref): mode "solve" | "optimal" | "grid";
    returns (feasible, M, alpha, x_ckpt, x_param, x_opt, t_fwd, t_bwd,
    iteration, throughput)."""
    lib = ref()
    out = (C.c_double * 10)()
    rc = lib.ref_planner({"solve": 0, "optimal": 1, "grid": 2}[mode], model, (C.c_double * 13)(*machine), mbs,
                         C.c_double(alpha), steps, out)
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    return tuple(out)


def ref_rooflines(model, machine, batch, x_opt):
    """(io_roofline, compute_roofline) of the reference (oracle/_ref)."""
    lib = ref()
    out = (C.c_double * 2)()
    rc = lib.ref_rooflines(model, (C.c_double * 13)(*machine), C.c_ulonglong(batch), C.c_double(x_opt), out)
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    return out[0], out[1]


def ref_solve_lp(A, b, c):
    lib = ref()
    m, n = len(A), len(c)
    flat = (C.c_double * max(1, m * n))(*[v for row in A for v in row])
    out = (C.c_double * (3 + n))()
    rc = lib.ref_solve_lp(m, n, flat, (C.c_double * max(1, m))(*b), (C.c_double * n)(*c), out)
    if rc != 0:
        raise RuntimeError(f"reference rc={rc}: {lib.ref_last_error().decode()}")
    return bool(out[0]), bool(out[1]), out[2], list(out[3:])
