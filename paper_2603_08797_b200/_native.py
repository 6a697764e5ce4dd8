"""ctypes binding of libjsv.so (include/jsv.h).  Fails loudly: no CPU fallback."""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigError, NativeError

MAX_TASKS = 16
MAX_EDGES = 32
MAX_PATHS = 64
MAX_ITEMS = 16
MAX_MIX = 8

SPACE_A, SPACE_S, SPACE_T = 1, 2, 4
BINDING_NAMES = {0: "throughput", 1: "latency", 2: "resources", 3: "accuracy", 4: "coverage"}

_I32P = C.POINTER(C.c_int32)
_F64P = C.POINTER(C.c_double)
_U8P = C.POINTER(C.c_uint8)
_U32P = C.POINTER(C.c_uint32)


class ProblemDesc(C.Structure):
    _fields_ = [
        ("n_tasks", C.c_int32), ("n_edges", C.c_int32), ("n_paths", C.c_int32), ("entry", C.c_int32),
        ("topo", _I32P), ("decl", _I32P), ("succ_off", _I32P), ("edge_dst", _I32P),
        ("pred_off", _I32P), ("pred_edge", _I32P), ("path_off", _I32P), ("path_task", _I32P),
        ("path_frac", _F64P), ("var_off", _I32P), ("var_acc", _F64P), ("var_fac_off", _I32P),
        ("var_fac", _F64P), ("most_acc", _I32P), ("key_off", _I32P), ("key_var", _I32P),
        ("key_seg", _I32P), ("key_batch", _I32P), ("key_cost", _I32P), ("key_lat", _F64P),
        ("key_thr", _F64P), ("sub_off", _I32P), ("sub_key", _I32P), ("grp_off", _I32P),
        ("grp_rep", _I32P), ("a_max", C.c_double),
    ]


class Request(C.Structure):
    _fields_ = [
        ("budget", C.c_int32), ("space", C.c_uint32), ("slack", C.c_double),
        ("has_override", _U8P), ("override_val", _F64P), ("pareto_width", C.c_int32),
        ("exhaustive_limit", C.c_int32), ("eps", C.c_double), ("n_mix", C.c_int32),
        ("mix", C.c_double * MAX_MIX), ("feasible_only", C.c_int32),
    ]


class Probe(C.Structure):
    _fields_ = [
        ("demand", C.c_double), ("slo_eff", C.c_double), ("acc_slo", C.c_double),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("uni_lat_budget", C.c_double * MAX_TASKS), ("uni_floor", C.c_double * MAX_TASKS),
        ("uni_weight", C.c_double * MAX_TASKS), ("uni_best_hput", C.c_double * MAX_TASKS),
        ("uni_best_slices", C.c_int32 * MAX_TASKS), ("uni_min_cost", C.c_int32 * MAX_TASKS),
    ]


class PlanOut(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32), ("has_config", C.c_int32), ("binding", C.c_int32),
        ("dead", C.c_int32), ("objective", C.c_double), ("a_obj", C.c_double),
        ("nodes", C.c_int64), ("leaves", C.c_int64),
        ("pool_size", C.c_int32 * MAX_TASKS), ("pool_present", C.c_int32 * MAX_TASKS),
        ("truncated", C.c_int32 * MAX_TASKS),
        ("n_items", C.c_int32 * MAX_TASKS), ("items", (C.c_uint32 * MAX_ITEMS) * MAX_TASKS),
        ("hput", (C.c_double * MAX_ITEMS) * MAX_TASKS),
        ("latency", C.c_double * MAX_TASKS), ("capacity", C.c_double * MAX_TASKS),
        ("demand", C.c_double * MAX_TASKS), ("accuracy", C.c_double * MAX_TASKS),
        ("slices", C.c_int32 * MAX_TASKS), ("fanout", C.c_double * MAX_EDGES),
        ("path_acc", C.c_double * MAX_PATHS), ("total_slices", C.c_int32),
        ("uncovered_mask", C.c_uint32), ("lat_margin", C.c_double * MAX_PATHS),
        ("thr_margin", C.c_double * MAX_TASKS), ("res_margin", C.c_double),
        ("acc_margin", C.c_double),
    ]


class Geometry(C.Structure):
    _fields_ = [("n_profiles", C.c_int32), ("slices_per_gpu", C.c_int32), ("start_off", _I32P),
                ("start_pos", _I32P), ("start_width", _I32P), ("order_rank", _I32P)]


class DemandOut(C.Structure):
    _fields_ = [("demand", C.c_double), ("probes", C.c_int32), ("status", C.c_int32),
                ("gpu_probes", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("ms_stage1", C.c_float), ("ms_stage2", C.c_float), ("ms_total", C.c_float),
                ("candidates_generated", C.c_int64), ("leaves", C.c_int64), ("nodes", C.c_int64),
                ("kernel_launches", C.c_int32), ("dims", C.c_int32), ("pair_tests_a", C.c_int64),
                ("pair_tests_b", C.c_int64), ("leaf_work", C.c_int64),
                ("exh_candidates", C.c_int64), ("exh_probes", C.c_int32), ("exh_pad_", C.c_int32),
                ("swept", C.c_int64), ("live_prefixes", C.c_int64),
                ("s1_shadow_tests", C.c_int64), ("s1_exact_tests", C.c_int64)]


EXPORTS = {
    "jsv_last_error": (C.c_char_p, []),
    "jsv_version": (C.c_int, []),
    "jsv_device_count": (C.c_int, []),
    "jsv_context_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "jsv_context_destroy": (None, [C.c_void_p]),
    "jsv_problem_create": (C.c_int, [C.c_void_p, C.POINTER(ProblemDesc), C.POINTER(C.c_void_p)]),
    "jsv_problem_destroy": (None, [C.c_void_p]),
    "jsv_plan_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.c_int32,
                                 C.POINTER(Probe), C.POINTER(PlanOut)]),
    "jsv_plan_batch_shard": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.c_int32,
                                       C.POINTER(Probe), C.c_int32, C.c_int32, C.POINTER(PlanOut)]),
    "jsv_max_demand_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.c_int32,
                                       C.POINTER(Probe), C.c_double, C.POINTER(DemandOut),
                                       C.POINTER(PlanOut)]),
    "jsv_derive": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.POINTER(Probe),
                             _I32P, _U32P, C.POINTER(PlanOut)]),
    "jsv_validate": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.POINTER(Probe),
                               _F64P, _F64P, _F64P, C.c_int32, C.c_double, C.c_uint32,
                               C.POINTER(PlanOut)]),
    "jsv_brute_force": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.POINTER(Probe),
                                  C.c_int32, C.c_int64, C.POINTER(C.c_int64), _I32P,
                                  C.POINTER(PlanOut)]),
    "jsv_pool_dump": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(Request), C.POINTER(Probe),
                                C.c_int32, C.c_int32, _I32P, _I32P, _U32P, _F64P, _I32P]),
    "jsv_last_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "jsv_host_alloc": (C.c_void_p, [C.c_size_t]),
    "jsv_host_free": (None, [C.c_void_p]),
    "jsv_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "jsv_set_strategy": (C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    "jsv_set_shard": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
    "jsv_kernel_times": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int64)]),
    "jsv_pack": (C.c_int, [C.POINTER(Geometry), _I32P, C.c_int32, C.c_int32, C.c_int64, _I32P,
                           _I32P, _I32P, _I32P]),
    "jsv_min_gpus": (C.c_int, [C.POINTER(Geometry), _I32P, C.c_int32, C.c_int64, _I32P]),
}

KERNEL_NAMES = ("generate", "stats", "pairs_a", "compact", "pairs_b", "truncate", "mrank",
                "s2_prep", "s2_level", "s2_leaf", "s2_reduce", "finalize", "uninformed", "bucket",
                "s2_prefix", "s2_exh", "s2_xreduce", "s2_xsort", "fo_prep", "fo_enum",
                "fo_eval", "x_live")

STRATEGY_SEARCH, STRATEGY_EXHAUSTIVE, STRATEGY_AUTO = 0, 1, 2
STRATEGIES = {"search": STRATEGY_SEARCH, "exhaustive": STRATEGY_EXHAUSTIVE, "auto": STRATEGY_AUTO}


def set_strategy(ctx, strategy: str, max_candidates: int = 1 << 31) -> None:
    """Stage-2 strategy of a context (include/jsv.h jsv_set_strategy)."""
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; expected one of {sorted(STRATEGIES)}")
    check(load_library().jsv_set_strategy(ctx, STRATEGIES[strategy], int(max_candidates)))


def set_shard(ctx, rank: int, world: int) -> None:
    """Evaluate only shard `rank` of `world` of every exhaustive sweep (jsv_set_shard)."""
    check(load_library().jsv_set_shard(ctx, int(rank), int(world)))


def profile(ctx, on: bool, kernels=None) -> None:
    """Per-kernel CUDA events on/off; ``kernels`` (names of KERNEL_NAMES) limits them."""
    arg = 1 if on else 0
    if on and kernels is not None:
        arg = (1 << 30) | sum(1 << KERNEL_NAMES.index(k) for k in kernels)
    check(load_library().jsv_profile(ctx, arg))


def kernel_times(ctx) -> dict:
    n = len(KERNEL_NAMES)
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    load_library().jsv_kernel_times(ctx, n, ms, cnt)
    return {KERNEL_NAMES[i]: (ms[i], cnt[i]) for i in range(n)}

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libjsv.so")
_lib = None
_ctx = {}
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libjsv.so and declare every export; raises NativeError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the planner has no CPU fallback)"
        )
    lib = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = load_library().jsv_last_error().decode()
    if rc == 5:
        raise ConfigError(msg)
    raise NativeError(f"libjsv error {rc}: {msg}")


def context(device: int | None = None) -> C.c_void_p:
    """Process-wide context for one device (created lazily)."""
    lib = load_library()
    if device is None:
        device = int(os.environ.get("JSV_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _lock:
        if device not in _ctx:
            h = C.c_void_p()
            check(lib.jsv_context_create(device, C.byref(h)))
            _ctx[device] = h
        return _ctx[device]


def last_stats(ctx) -> Stats:
    s = Stats()
    check(load_library().jsv_last_stats(ctx, C.byref(s)))
    return s


class _PinnedOut(threading.local):
    """Per-thread page-locked array of PlanOut records for plan_batch's results (the
    device-to-host copy lands in it directly; plan_batch decodes before returning,
    so one buffer per thread is reused call after call)."""

    def __init__(self):
        self.ptr = None
        self.cap = 0

    def get(self, n: int):
        if n > self.cap:
            lib = load_library()
            cap = max(n, 2 * self.cap, 64)
            ptr = lib.jsv_host_alloc(C.sizeof(PlanOut) * cap)
            if not ptr:
                return None
            if self.ptr:
                lib.jsv_host_free(self.ptr)
            self.ptr, self.cap = ptr, cap
        return (PlanOut * n).from_address(self.ptr)

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.jsv_host_free(self.ptr)
            self.ptr = None


_pinned_out = _PinnedOut()


def pinned_outs(n: int):
    """A PlanOut[n] view of this thread's page-locked result buffer (or None)."""
    return _pinned_out.get(n)
