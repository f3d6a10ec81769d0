"""GreedySnake hot path on B200 — Python host binding over libgreedysnake.so.

The product is the C++/CUDA library built in-tree (csrc/Makefile): the
drop-in ``offsim`` scheduler API (build_vertical, ledgers, simulate) and the
real executor that runs a plan on sm_100a kernels, PCIe DMA and NVMe I/O.
This module binds its C-ABI (include/greedysnake.h) with ctypes and mirrors
the reference's names (proj/include/offsim/*.hpp): ModelSpec, StorageSplit,
build_vertical, build_horizontal, vertical_traffic, plan_traffic, simulate,
plus Engine (the executor).  There is no Python or CPU fallback: importing
fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgreedysnake.so")

LINKS = ("H2D", "D2H", "SSD_read", "SSD_write")
DATA = ("param", "ckpt", "grad_accum", "interlayer_grad", "opt_state")
TASK_KINDS = ("fwd", "bwd", "cpu_step", "xfer", "fixed_ops")
RESOURCES = ("compute", "cpu_step", "pcie_h2d", "pcie_d2h", "ssd_read", "ssd_write")
# Engine(opt_tier=...): where the CPU-resident optimizer fraction lives and
# what steps it (include/offsim/executor.hpp OptTier)
OPT_AUTO, OPT_HBM, OPT_STREAM, OPT_HOST = 0, 1, 2, 3

OK, ERR_PLAN_BUG, ERR_VALIDATION, ERR_INFEASIBLE, ERR_CUDA, ERR_RUNTIME = range(6)


class OffsimError(RuntimeError):
    code = ERR_RUNTIME


class ValidationError(OffsimError):
    """offsim::ValidationError (CLI exit 2)."""
    code = ERR_VALIDATION


class InfeasibleError(OffsimError):
    """offsim::InfeasibleError (CLI exit 3)."""
    code = ERR_INFEASIBLE


class PlanBugError(OffsimError):
    """offsim::PlanBugError (CLI exit 1)."""
    code = ERR_PLAN_BUG


class CudaError(OffsimError):
    code = ERR_CUDA


_ERRORS = {ERR_PLAN_BUG: PlanBugError, ERR_VALIDATION: ValidationError, ERR_INFEASIBLE: InfeasibleError,
           ERR_CUDA: CudaError, ERR_RUNTIME: OffsimError}


# ----------------------------------------------------------------- structs
class _ModelSpec(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "num_layers", "hidden_dim", "num_heads", "seq_len", "microbatch_size", "low_precision_bytes",
        "full_precision_bytes", "optimizer_states_per_element", "data_parallel_degree")]


class _Split(C.Structure):
    _fields_ = [("x_ckpt", C.c_double), ("x_param", C.c_double), ("x_opt", C.c_double)]


class _Machine(C.Structure):
    _fields_ = [("gpu_mem_bytes", C.c_uint64), ("cpu_usable_dram_bytes", C.c_uint64),
                ("pcie_h2d_bw", C.c_double), ("pcie_d2h_bw", C.c_double), ("ssd_read_bw", C.c_double),
                ("ssd_write_bw", C.c_double), ("fwd_compute_time_per_layer_per_mb", C.c_double),
                ("bwd_compute_time_per_layer_per_mb", C.c_double), ("cpu_step_throughput", C.c_double),
                ("fixed_overhead_time", C.c_double), ("num_gpus", C.c_int), ("gpu_working_set_bytes", C.c_uint64),
                ("ssd_duplex", C.c_int)]


class _Task(C.Structure):
    _fields_ = [("id", C.c_int), ("kind", C.c_int), ("layer", C.c_int), ("microbatch", C.c_int), ("stage", C.c_int),
                ("data", C.c_int), ("link", C.c_int), ("bytes", C.c_uint64), ("elements", C.c_uint64),
                ("cross_iter_dep", C.c_int), ("num_deps", C.c_int)]


class _EngineConfig(C.Structure):
    _fields_ = [("model", _ModelSpec), ("vocab_size", C.c_int), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float), ("seed", C.c_uint64),
                ("device", C.c_int), ("nvme_dir", C.c_char_p), ("odirect", C.c_int), ("opt_tier", C.c_int),
                ("record_trace", C.c_int), ("profile_kernels", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("comm_id", C.c_void_p), ("force_collectives", C.c_int), ("ssd_ring_layers", C.c_int),
                ("host_threads", C.c_int)]


class _RunReport(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("iterations", C.c_int), ("gpu_launches", C.c_int),
                ("ledger", C.c_uint64 * 20), ("extension", C.c_uint64 * 20), ("physical", C.c_uint64 * 20),
                ("gpu_bytes", C.c_uint64), ("host_pinned_bytes", C.c_uint64)]


class _TraceRecord(C.Structure):
    _fields_ = [("iteration", C.c_int), ("task", C.c_int), ("resource", C.c_int), ("t_start_ms", C.c_double),
                ("t_end_ms", C.c_double), ("bytes", C.c_uint64), ("physical_bytes", C.c_uint64),
                ("t_host_ms", C.c_double)]


# ------------------------------------------------------------------ loading
_lib = None


def lib() -> C.CDLL:
    """The loaded libgreedysnake.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (make -C paper_2512_17570_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.gs_last_error.restype = C.c_char_p
        L.gs_version.restype = C.c_char_p
        L.gs_plan_overlap_window.restype = C.c_int64
        L.gs_plan_overlap_window.argtypes = [C.c_void_p]
        L.gs_plan_num_tasks.argtypes = [C.c_void_p]
        L.gs_plan_free.argtypes = [C.c_void_p]
        L.gs_plan_free.restype = None
        L.gs_engine_destroy.argtypes = [C.c_void_p]
        L.gs_engine_destroy.restype = None
        L.gs_attention_bwd_workspace.restype = C.c_size_t
        L.gs_launch_count.restype = C.c_int64
        L.gs_vertical_traffic.argtypes = [C.POINTER(_ModelSpec), C.c_int, C.POINTER(_Split), C.c_double,
                                          C.POINTER(C.c_uint64)]
        L.gs_plan_build_vertical.argtypes = [C.POINTER(_ModelSpec), C.c_int, C.POINTER(_Split), C.c_double,
                                             C.POINTER(C.c_void_p)]
        L.gs_adam_step_packed.argtypes = [C.c_float] * 5 + [C.c_int, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p,
                                                            C.c_int, C.c_int64, C.c_void_p]
        L.gs_io_roofline.argtypes = [C.POINTER(_ModelSpec), C.POINTER(_Machine), C.c_ulonglong, C.c_double,
                                     C.POINTER(C.c_double)]
        L.gs_compute_roofline.argtypes = [C.POINTER(_ModelSpec), C.POINTER(_Machine), C.POINTER(C.c_double)]
        L.gs_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.gs_ctx_stream.argtypes = [C.c_void_p]
        L.gs_ctx_stream.restype = C.c_void_p
        L.gs_ctx_sync.argtypes = [C.c_void_p]
        L.gs_ctx_destroy.argtypes = [C.c_void_p]
        L.gs_ctx_destroy.restype = None
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().gs_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, OffsimError)(msg)


# --------------------------------------------------------- reference mirror
@dataclass
class ModelSpec:
    """offsim::ModelSpec (proj/include/offsim/model.hpp:11-23)."""
    num_layers: int = 1
    hidden_dim: int = 1
    num_heads: int = 1
    seq_len: int = 1
    microbatch_size: int = 1
    low_precision_bytes: int = 2
    full_precision_bytes: int = 4
    optimizer_states_per_element: int = 3
    data_parallel_degree: int = 1

    def _c(self) -> _ModelSpec:
        return _ModelSpec(self.num_layers, self.hidden_dim, self.num_heads, self.seq_len, self.microbatch_size,
                          self.low_precision_bytes, self.full_precision_bytes, self.optimizer_states_per_element,
                          self.data_parallel_degree)

    @property
    def params_per_layer(self) -> int:
        return 12 * self.hidden_dim * self.hidden_dim


@dataclass
class StorageSplit:
    """offsim::StorageSplit (schedule.hpp:22-29): CPU-resident fractions."""
    x_ckpt: float = 0.0
    x_param: float = 0.0
    x_opt: float = 0.0

    def _c(self) -> _Split:
        return _Split(self.x_ckpt, self.x_param, self.x_opt)


@dataclass
class MachineSpec:
    """offsim::MachineSpec (machine.hpp:12-33)."""
    gpu_mem_bytes: int = 0
    cpu_usable_dram_bytes: int = 0
    pcie_h2d_bw: float = 0.0
    pcie_d2h_bw: float = 0.0
    ssd_read_bw: float = 0.0
    ssd_write_bw: float = 0.0
    fwd_compute_time_per_layer_per_mb: float = 0.0
    bwd_compute_time_per_layer_per_mb: float = 0.0
    cpu_step_throughput: float = 0.0
    fixed_overhead_time: float = 0.0
    num_gpus: int = 1
    gpu_working_set_bytes: int = 0
    ssd_duplex: bool = True

    def _c(self) -> _Machine:
        return _Machine(self.gpu_mem_bytes, self.cpu_usable_dram_bytes, self.pcie_h2d_bw, self.pcie_d2h_bw,
                        self.ssd_read_bw, self.ssd_write_bw, self.fwd_compute_time_per_layer_per_mb,
                        self.bwd_compute_time_per_layer_per_mb, self.cpu_step_throughput, self.fixed_overhead_time,
                        self.num_gpus, self.gpu_working_set_bytes, int(self.ssd_duplex))


def _ledger(arr) -> np.ndarray:
    return np.array(list(arr), dtype=np.uint64).reshape(4, 5)


class SchedulePlan:
    """Owner of an offsim::SchedulePlan built by the library."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gs_plan_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def __len__(self) -> int:
        return lib().gs_plan_num_tasks(self._h)

    def info(self) -> dict:
        """Header fields: variant, alpha (delay ratio), microbatches, layers."""
        v, a, m, n = C.c_int(), C.c_double(), C.c_int(), C.c_int()
        check(lib().gs_plan_info(self._h, C.byref(v), C.byref(a), C.byref(m), C.byref(n)))
        return dict(variant=("single-fb", "horizontal", "vertical")[v.value], alpha=a.value, microbatches=m.value,
                    layers=n.value)

    def task(self, i: int) -> dict:
        t = _Task()
        check(lib().gs_plan_task(self._h, i, C.byref(t)))
        deps = (C.c_int * max(1, t.num_deps))()
        n = C.c_int()
        check(lib().gs_plan_task_deps(self._h, i, deps, t.num_deps, C.byref(n)))
        return dict(id=t.id, kind=TASK_KINDS[t.kind], layer=t.layer, microbatch=t.microbatch, stage=t.stage,
                    data=DATA[t.data], link=LINKS[t.link], bytes=t.bytes, elements=t.elements,
                    cross_iter_dep=t.cross_iter_dep, deps=list(deps)[:n.value])

    def to_json(self) -> str:
        n = C.c_size_t()
        check(lib().gs_plan_to_json(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().gs_plan_to_json(self._h, buf, n.value, C.byref(n)))
        return buf.value.decode()

    def as_dict(self) -> dict:
        return json.loads(self.to_json())

    @staticmethod
    def from_json(text: str) -> "SchedulePlan":
        h = C.c_void_p()
        check(lib().gs_plan_from_json(text.encode(), C.byref(h)))
        return SchedulePlan(h)


def build_vertical(model: ModelSpec, num_microbatches: int, split: StorageSplit, alpha: float) -> SchedulePlan:
    """offsim::build_vertical (schedule.hpp:79-80)."""
    h = C.c_void_p()
    m, s = model._c(), split._c()
    check(lib().gs_plan_build_vertical(C.byref(m), num_microbatches, C.byref(s), C.c_double(alpha), C.byref(h)))
    return SchedulePlan(h)


def build_horizontal(model: ModelSpec, num_microbatches: int, split: StorageSplit) -> SchedulePlan:
    """offsim::build_horizontal (schedule.hpp:73-74)."""
    h = C.c_void_p()
    m, s = model._c(), split._c()
    check(lib().gs_plan_build_horizontal(C.byref(m), num_microbatches, C.byref(s), C.byref(h)))
    return SchedulePlan(h)


def vertical_traffic(model: ModelSpec, num_microbatches: int, split: StorageSplit, alpha: float) -> np.ndarray:
    """offsim::vertical_traffic (traffic.hpp:44-46): [link][data] bytes."""
    out = (C.c_uint64 * 20)()
    m, s = model._c(), split._c()
    check(lib().gs_vertical_traffic(C.byref(m), num_microbatches, C.byref(s), C.c_double(alpha), out))
    return _ledger(out)


def horizontal_traffic(model: ModelSpec, num_microbatches: int, split: StorageSplit) -> np.ndarray:
    out = (C.c_uint64 * 20)()
    m, s = model._c(), split._c()
    check(lib().gs_horizontal_traffic(C.byref(m), num_microbatches, C.byref(s), out))
    return _ledger(out)


def plan_traffic(plan: SchedulePlan) -> np.ndarray:
    """offsim::plan_traffic (traffic.hpp:50)."""
    out = (C.c_uint64 * 20)()
    check(lib().gs_plan_traffic(plan.handle, out))
    return _ledger(out)


def overlap_window(plan: SchedulePlan) -> int:
    return int(lib().gs_plan_overlap_window(plan.handle))


def comm_unique_id() -> bytes:
    """128 random bytes naming a data-parallel job's peer-memory communicator
    (rank 0 draws them, every rank passes them as Engine(comm_id=...))."""
    buf = (C.c_uint8 * 128)()
    check(lib().gs_comm_unique_id(buf))
    return bytes(buf)


def shard_range(params_per_layer: int, world: int, rank: int) -> tuple:
    """[lo, hi) of a layer's elements owned by `rank` (ZeRO-3 shards of
    ceil(P / world) elements, the last one short) — the executor's layout."""
    ps = -(-params_per_layer // world)
    lo = min(params_per_layer, rank * ps)
    return lo, min(params_per_layer, lo + ps)


class _PlannerSolution(C.Structure):
    _fields_ = [("feasible", C.c_int), ("num_microbatches", C.c_int), ("alpha", C.c_double), ("split", _Split),
                ("t_fwd_stage", C.c_double), ("t_bwd_stage", C.c_double), ("iteration_estimate", C.c_double),
                ("throughput_estimate", C.c_double)]


@dataclass
class PlannerSolution:
    """offsim::PlannerSolution (planner.hpp:13-22)."""
    feasible: bool
    num_microbatches: int
    alpha: float
    split: "StorageSplit"
    t_fwd_stage: float
    t_bwd_stage: float
    iteration_estimate: float
    throughput_estimate: float


def _solution(o: _PlannerSolution) -> PlannerSolution:
    return PlannerSolution(bool(o.feasible), o.num_microbatches, o.alpha,
                           StorageSplit(o.split.x_ckpt, o.split.x_param, o.split.x_opt), o.t_fwd_stage,
                           o.t_bwd_stage, o.iteration_estimate, o.throughput_estimate)


def solve_config(model: ModelSpec, machine: MachineSpec, num_microbatches: int, alpha: float) -> PlannerSolution:
    """The storage-split LP for fixed (M, alpha) (planner.hpp:27-28)."""
    out = _PlannerSolution()
    check(lib().gs_solve_config(C.byref(model._c()), C.byref(machine._c()), num_microbatches, C.c_double(alpha),
                                C.byref(out)))
    return _solution(out)


def find_optimal_config(model: ModelSpec, machine: MachineSpec) -> PlannerSolution:
    """Algorithm 1's outer search over M and the alpha grid (planner.hpp:33)."""
    out = _PlannerSolution()
    check(lib().gs_find_optimal_config(C.byref(model._c()), C.byref(machine._c()), C.byref(out)))
    return _solution(out)


def grid_search_config(model: ModelSpec, machine: MachineSpec, num_microbatches: int, alpha: float,
                       steps: int = 100) -> PlannerSolution:
    """Exhaustive split grid, the LP's cross-check (planner.hpp:38-40)."""
    out = _PlannerSolution()
    check(lib().gs_grid_search_config(C.byref(model._c()), C.byref(machine._c()), num_microbatches,
                                      C.c_double(alpha), steps, C.byref(out)))
    return _solution(out)


def io_roofline(model: ModelSpec, machine: MachineSpec, batch_samples: int, x_opt: float = 0.0) -> float:
    """Samples/s bound from the SSD optimizer-state round trip (roofline.hpp:12-13); inf without SSD bytes."""
    out = C.c_double()
    check(lib().gs_io_roofline(C.byref(model._c()), C.byref(machine._c()), batch_samples, C.c_double(x_opt),
                               C.byref(out)))
    return out.value


def compute_roofline(model: ModelSpec, machine: MachineSpec) -> float:
    """Samples/s bound from the calibrated per-layer compute times (roofline.hpp:17)."""
    out = C.c_double()
    check(lib().gs_compute_roofline(C.byref(model._c()), C.byref(machine._c()), C.byref(out)))
    return out.value


class Context:
    """One per device (gs_ctx_create): selects the device, owns a non-blocking
    stream for the kernel entry points."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().gs_ctx_create(device, C.byref(h)))
        self.handle = h

    @property
    def stream(self) -> C.c_void_p:
        return C.c_void_p(lib().gs_ctx_stream(self.handle))

    def sync(self) -> None:
        check(lib().gs_ctx_sync(self.handle))

    def close(self) -> None:
        if self.handle:
            lib().gs_ctx_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_lp(A, b, c):
    """min c.x s.t. A x <= b, x >= 0 (simplex.hpp:17): (feasible, bounded, objective, x)."""
    m, n = len(A), len(c)
    flat = (C.c_double * max(1, m * n))(*[v for row in A for v in row])
    x = (C.c_double * n)()
    f, bd, obj = C.c_int(), C.c_int(), C.c_double()
    check(lib().gs_solve_lp(m, n, flat, (C.c_double * max(1, m))(*b), (C.c_double * n)(*c), C.byref(f), C.byref(bd),
                            C.byref(obj), x))
    return bool(f.value), bool(bd.value), obj.value, list(x)


def simulate(plan: SchedulePlan, machine: MachineSpec) -> dict:
    """report_to_json(offsim::simulate(plan, machine)) (simulator.hpp:34)."""
    n = C.c_size_t()
    mc = machine._c()
    check(lib().gs_simulate_json(plan.handle, C.byref(mc), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    check(lib().gs_simulate_json(plan.handle, C.byref(mc), buf, n.value, C.byref(n)))
    return json.loads(buf.value.decode())


# ------------------------------------------------------------------- engine
@dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0


@dataclass
class RunReport:
    total_ms: float
    iterations: int
    gpu_launches: int
    losses: list
    ledger: np.ndarray
    extension: np.ndarray
    physical: np.ndarray
    gpu_bytes: int
    host_pinned_bytes: int
    trace: list = field(default_factory=list)


class Engine:
    """offsim::Executor — runs a plan on the B200 (include/offsim/executor.hpp)."""

    def __init__(self, plan: SchedulePlan, model: ModelSpec, vocab_size: int, adam: AdamConfig = AdamConfig(),
                 seed: int = 42, device: int = 0, nvme_dir: str = "/tmp", odirect: bool = True, opt_tier: int = 0,
                 record_trace: bool = False, profile: bool = False, rank: int = 0, world: int = 1,
                 comm_id: bytes | None = None, force_collectives: bool = False, ssd_ring_layers: int = 0,
                 host_threads: int = 0):
        self.model = model
        self.vocab_size = vocab_size
        self.plan = plan
        self.microbatches = plan.info()["microbatches"]
        self._nvme = nvme_dir.encode()
        self._id = C.create_string_buffer(bytes(comm_id), 128) if comm_id is not None else None
        cfg = _EngineConfig(model._c(), vocab_size, adam.lr, adam.beta1, adam.beta2, adam.eps, adam.weight_decay,
                            seed, device, self._nvme, int(odirect), opt_tier, int(record_trace), int(profile),
                            rank, world, C.cast(self._id, C.c_void_p) if self._id is not None else None,
                            int(force_collectives), int(ssd_ring_layers), int(host_threads))
        h = C.c_void_p()
        check(lib().gs_engine_create(plan.handle, C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().gs_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        if _lib is not None:
            self.close()

    def run(self, tokens, iterations: int | None = None, tokens_on_device: bool = False,
            device_ptr: int | None = None) -> RunReport:
        """tokens: int32 array [iterations][M][b][s+1] (host); or pass
        device_ptr (an int address) with tokens_on_device=True."""
        m = self.model
        shape = (self.microbatches, m.microbatch_size, m.seq_len + 1)
        if device_ptr is None:
            tok = np.ascontiguousarray(tokens, dtype=np.int32)
            iterations = tok.shape[0] if iterations is None else iterations
            if tok.shape != (iterations,) + shape:
                raise ValidationError(f"tokens must have shape {(iterations,) + shape} "
                                      f"[iterations][M][b][s+1], got {tok.shape}")
            if tok.size and (int(tok.min()) < 0 or int(tok.max()) >= self.vocab_size):
                raise ValidationError(f"token ids must lie in [0, {self.vocab_size})")
            ptr = tok.ctypes.data_as(C.c_void_p)
        else:
            if iterations is None or iterations < 1:
                raise ValidationError("device tokens need iterations >= 1")
            ptr = C.c_void_p(device_ptr)
        losses = (C.c_double * iterations)()
        rep = _RunReport()
        check(lib().gs_engine_run(self._h, iterations, ptr, int(tokens_on_device), losses, C.byref(rep)))
        n = C.c_int()
        check(lib().gs_engine_trace(self._h, None, 0, C.byref(n)))
        trace = []
        if n.value:
            arr = (_TraceRecord * n.value)()
            check(lib().gs_engine_trace(self._h, arr, n.value, C.byref(n)))
            trace = [dict(iteration=r.iteration, task=r.task, resource=RESOURCES[r.resource], t_start_ms=r.t_start_ms,
                          t_end_ms=r.t_end_ms, bytes=r.bytes, physical_bytes=r.physical_bytes,
                          t_host_ms=r.t_host_ms) for r in arr]
        return RunReport(rep.total_ms, rep.iterations, rep.gpu_launches, list(losses), _ledger(rep.ledger),
                         _ledger(rep.extension), _ledger(rep.physical), rep.gpu_bytes, rep.host_pinned_bytes, trace)

    def kernel_profile(self) -> dict:
        """{class: (sampled flops, sampled ms, sampled launches, all launches)}
        of the last run (profiling on)."""
        f, m, n, t = (C.c_double * 5)(), (C.c_double * 5)(), (C.c_int * 5)(), (C.c_int64 * 5)()
        check(lib().gs_engine_kernel_profile(self._h, f, m, n, t))
        names = ("gemm", "attention_fwd", "attention_bwd", "layernorm", "other")
        out = {k: (f[i], m[i], n[i], t[i]) for i, k in enumerate(names) if n[i]}
        sf, sm, sn = C.c_double(), C.c_double(), C.c_int()
        check(lib().gs_engine_gemm_span_profile(self._h, C.byref(sf), C.byref(sm), C.byref(sn)))
        if sn.value:
            out["gemm_span"] = (sf.value, sm.value, sn.value, t[0])
        return out

    def set_profiling(self, stride: int) -> None:
        check(lib().gs_engine_set_profiling(self._h, int(stride)))

    def set_trace(self, on: bool) -> None:
        check(lib().gs_engine_set_trace(self._h, int(bool(on))))

    def flush(self) -> None:
        check(lib().gs_engine_flush(self._h))

    def read_params(self):
        P = self.model.params_per_layer
        layers = np.empty((self.model.num_layers, P), np.float32)
        fixed = np.empty((self.vocab_size + self.model.seq_len) * self.model.hidden_dim, np.float32)
        check(lib().gs_engine_read_params(self._h, layers.ctypes.data_as(C.c_void_p),
                                          fixed.ctypes.data_as(C.c_void_p)))
        return layers, fixed

    def read_moments(self):
        P = self.model.params_per_layer
        m = np.empty((self.model.num_layers, P), np.float32)
        v = np.empty_like(m)
        check(lib().gs_engine_read_moments(self._h, m.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
        return m, v

    def read_fixed_moments(self):
        n = (self.vocab_size + self.model.seq_len) * self.model.hidden_dim
        m, v = np.empty(n, np.float32), np.empty(n, np.float32)
        check(lib().gs_engine_read_fixed_moments(self._h, m.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
        return m, v


def host_probe(threads: int = 0, elements: int = 1 << 26) -> dict:
    """Host DRAM as the host-core optimizer step (OPT_HOST) sees it
    (gs_host_probe): multi-threaded copy GB/s (read + write bytes) and the
    host Adam's own rate on pinned memory."""
    out = (C.c_double * 3)()
    check(lib().gs_host_probe(int(threads), C.c_uint64(elements), out))
    return {"copy_gbs": out[0], "adam_gelem_s": out[1], "threads": int(out[2])}
