"""Loader and thin Python bindings for libdagsched_b200.so (the C-ABI).

The product path is the CUDA library; there is no CPU fallback. If the
library is missing or no CUDA device is visible, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi
from .batch import DagBatch, combine_status

HERE = os.path.dirname(os.path.abspath(__file__))
# DAGSCHED_LIB: another build of the library (A/B measurements only)
LIB_PATH = os.environ.get("DAGSCHED_LIB") or os.path.join(HERE, "_lib", "libdagsched_b200.so")

_lock = threading.Lock()
_lib = None


class DagschedError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_abi.STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _sig(lib):
    P = C.POINTER
    table = {
        "ds_last_error": (C.c_char_p, []),
        "ds_version": (C.c_char_p, []),
        "ds_device_count": (C.c_int, [P(C.c_int)]),
        "ds_analyze_batch": (C.c_int, [P(_abi.ds_dag_batch), P(_abi.ds_platform), C.c_uint32,
                                       P(_abi.ds_results), C.c_int, C.c_void_p, C.c_uint32]),
        "ds_analyze_batch16": (C.c_int, [P(_abi.ds_dag_batch16), P(_abi.ds_platform), C.c_uint32,
                                         P(_abi.ds_results), C.c_int]),
        "ds_analyze_batch_multi": (C.c_int, [P(_abi.ds_dag_batch), P(_abi.ds_platform), C.c_uint32,
                                             P(_abi.ds_results), P(C.c_int), C.c_int]),
        "ds_analyze_batch_tri": (C.c_int, [P(_abi.ds_dag_batch_tri), P(_abi.ds_platform), C.c_uint32,
                                           P(_abi.ds_results), C.c_int]),
        "ds_analyze_batch_tri_multi": (C.c_int, [P(_abi.ds_dag_batch_tri), P(_abi.ds_platform), C.c_uint32,
                                                 P(_abi.ds_results), P(C.c_int), C.c_int]),
        "ds_analyze_batch16_multi": (C.c_int, [P(_abi.ds_dag_batch16), P(_abi.ds_platform), C.c_uint32,
                                               P(_abi.ds_results), P(C.c_int), C.c_int]),
        "ds_shard_range": (C.c_int, [C.c_uint64, C.c_int, C.c_int, P(C.c_uint64), P(C.c_uint64)]),
        "ds_schedule_batch": (C.c_int, [P(_abi.ds_dag_batch), P(_abi.ds_platform),
                                        P(_abi.ds_scheme_out), C.c_int]),
        "ds_corpus_generate": (C.c_int, [P(_abi.ds_gen_config), C.c_int64, C.c_uint32, P(C.c_void_p)]),
        "ds_corpus_view": (C.c_int, [C.c_void_p, P(_abi.ds_dag_batch)]),
        "ds_corpus_free": (None, [C.c_void_p]),
        "ds_corpus_gen_ms": (C.c_float, [C.c_void_p]),
        "ds_simulate_greedy_batch": (C.c_int, [P(_abi.ds_dag_batch), P(_abi.ds_platform), P(_abi.ds_greedy_cfg),
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
        "ds_session_kernel_times": (C.c_int, [C.c_void_p, P(C.c_float), P(C.c_char_p), C.c_int]),
        "ds_session_create": (C.c_int, [P(_abi.ds_dag_batch), P(_abi.ds_platform), C.c_uint32,
                                        C.c_int, P(C.c_void_p)]),
        "ds_session_run": (C.c_int, [C.c_void_p, P(C.c_float)]),
        "ds_session_results": (C.c_int, [C.c_void_p, P(_abi.ds_results)]),
        "ds_session_free": (C.c_int, [C.c_void_p]),
    }
    for name, (res, args) in table.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def lib():
    """The loaded product library (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DagschedError(_abi.DS_ENODEV, f"{LIB_PATH} not built (run `make` or __graft_entry__.build())")
            _lib = _sig(C.CDLL(LIB_PATH))
        return _lib


def check(rc: int):
    if rc != _abi.DS_OK:
        raise DagschedError(rc, lib().ds_last_error().decode())


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().ds_device_count(C.byref(n))
    return n.value if rc == _abi.DS_OK else 0


def platform(sm_count: int, t_min=1, min_load=None) -> _abi.ds_platform:
    """ds_platform for M = sm_count SMs and t_min. min_load is DagTask::make's
    load floor on the device: None -> t_min (generate()'s tasks), 1 -> 1
    (make's default argument), "premade" -> tasks already validated."""
    from fractions import Fraction
    t = Fraction(t_min)
    flags = {None: 0, 1: _abi.DS_PF_MIN_LOAD_ONE, "premade": _abi.DS_PF_PREMADE}[min_load]
    return _abi.ds_platform(int(sm_count), flags, t.numerator, t.denominator)


def gen_config(depth_min=5, depth_max=8, max_width=8, avg_load=20, load_jitter=0.5,
               edge_density=0.2, seed=1, integer_loads=True, exact_mean=False, t_min=1):
    from fractions import Fraction
    a, t = Fraction(avg_load), Fraction(t_min)
    return _abi.ds_gen_config(depth_min, depth_max, max_width, int(integer_loads),
                              a.numerator, a.denominator, float(load_jitter), float(edge_density),
                              int(seed), t.numerator, t.denominator, int(exact_mean), 0)


def _results(n: int, with_groups=True):
    st = np.zeros(n, np.int32)
    b = np.zeros((n, 10), np.int64)
    ng = np.zeros(n, np.uint16) if with_groups else None
    r = _abi.ds_results(st.ctypes.data, b.ctypes.data, ng.ctypes.data if ng is not None else None)
    return st, b, ng, r


def _finish(batch: DagBatch, st, b, ng):
    """Merge packer (id-level) and device validation; failed DAGs carry no bounds."""
    status = combine_status(batch.pack_status, st)
    bad = status != _abi.DS_OK
    if bad.any():
        b[bad] = 0
        if ng is not None:
            ng[bad] = 0
    return status, b, ng


def analyze(batch: DagBatch, sm_count: int, t_min=1, mask: int = _abi.DS_M_ALL, device: int = 0, min_load=None):
    """Batched bound analysis on one GPU -> (status[n], bounds[n, 10], n_groups[n]).
    min_load: DagTask::make's load floor on the device (see platform())."""
    st, b, ng, r = _results(batch.n_dags)
    cb = batch.as_c()
    pl = platform(sm_count, t_min, min_load)
    check(lib().ds_analyze_batch(C.byref(cb), C.byref(pl), mask, C.byref(r), device, None, 0))
    return _finish(batch, st, b, ng)


def analyze16(batch: DagBatch, sm_count: int, t_min=1, mask: int = _abi.DS_M_ALL, device: int = 0,
              min_load=None):
    """analyze() over the compact 16-bit wire form (ds_analyze_batch16)."""
    st, b, ng, r = _results(batch.n_dags)
    load16, edges16 = batch.compact16()
    cb = batch.as_c16(load16, edges16)
    pl = platform(sm_count, t_min, min_load)
    check(lib().ds_analyze_batch16(C.byref(cb), C.byref(pl), mask, C.byref(r), device))
    return _finish(batch, st, b, ng)


def analyze_multi(batch: DagBatch, sm_count: int, devices, t_min=1, mask: int = _abi.DS_M_ALL, min_load=None):
    st, b, ng, r = _results(batch.n_dags)
    cb = batch.as_c()
    pl = platform(sm_count, t_min, min_load)
    devs = (C.c_int * len(devices))(*devices)
    check(lib().ds_analyze_batch_multi(C.byref(cb), C.byref(pl), mask, C.byref(r), devs, len(devices)))
    return _finish(batch, st, b, ng)


def analyze16_multi(batch: DagBatch, sm_count: int, devices, t_min=1, mask: int = _abi.DS_M_ALL, min_load=None):
    """analyze_multi() over the compact 16-bit wire form (ds_analyze_batch16_multi)."""
    st, b, ng, r = _results(batch.n_dags)
    load16, edges16 = batch.compact16()
    cb = batch.as_c16(load16, edges16)
    pl = platform(sm_count, t_min, min_load)
    devs = (C.c_int * len(devices))(*devices)
    check(lib().ds_analyze_batch16_multi(C.byref(cb), C.byref(pl), mask, C.byref(r), devs, len(devices)))
    return _finish(batch, st, b, ng)


def analyze_tri(batch: DagBatch, sm_count: int, t_min=1, mask: int = _abi.DS_M_ALL, device: int = 0,
                min_load=None, devices=None):
    """analyze() over the triangular wire form (ds_analyze_batch_tri, or
    ds_analyze_batch_tri_multi over `devices`)."""
    st, b, ng, r = _results(batch.n_dags)
    load16, adj_off, adj = batch.tri()
    cb = batch.as_ctri(load16, adj_off, adj)
    pl = platform(sm_count, t_min, min_load)
    if devices is None:
        check(lib().ds_analyze_batch_tri(C.byref(cb), C.byref(pl), mask, C.byref(r), device))
    else:
        devs = (C.c_int * len(devices))(*devices)
        check(lib().ds_analyze_batch_tri_multi(C.byref(cb), C.byref(pl), mask, C.byref(r), devs, len(devices)))
    return _finish(batch, st, b, ng)


def shard_range(n_dags: int, n_shards: int, shard: int) -> tuple[int, int]:
    """The library's contiguous split (ds_shard_range) — host-only."""
    lo, hi = C.c_uint64(), C.c_uint64()
    check(lib().ds_shard_range(n_dags, n_shards, shard, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


class Corpus:
    """Generated corpus (product generator, generator.cpp semantics): on the
    host, or on the current CUDA device with ``gpu=True`` (K5)."""

    def __init__(self, count: int, pinned: bool = False, gpu: bool = False, **cfg):
        self.h = C.c_void_p()
        g = gen_config(**cfg)
        flags = (_abi.DS_F_PINNED if pinned else 0) | (_abi.DS_F_GPU_GENERATE if gpu else 0)
        check(lib().ds_corpus_generate(C.byref(g), int(count), flags, C.byref(self.h)))
        self.gen_ms = float(lib().ds_corpus_gen_ms(self.h))
        self.view = _abi.ds_dag_batch()
        check(lib().ds_corpus_view(self.h, C.byref(self.view)))
        v = self.view
        n = v.n_dags
        self.n_dags = n

        def arr(ptr, count, ct, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(count,)).view(dt)

        self.node_off = arr(v.node_off, n + 1, C.c_uint32, np.uint32)
        self.edge_off = arr(v.edge_off, n + 1, C.c_uint32, np.uint32)
        nn, ne = int(self.node_off[-1]), int(self.edge_off[-1])
        self.load_num = arr(v.load_num, nn, C.c_int64, np.int64)
        self.load_den = arr(v.load_den, nn, C.c_int64, np.int64)
        self.edges = arr(v.edges, ne, C.c_uint32, np.uint32)

    def batch(self) -> DagBatch:
        """Zero-copy DagBatch view (valid while this object lives)."""
        b = DagBatch(self.node_off, self.edge_off, self.load_num, self.load_den, self.edges,
                     np.zeros(self.n_dags, np.int32))
        b._owner = self
        return b

    def close(self):
        if self.h:
            lib().ds_corpus_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """Device-resident batch; ``run()`` replays the analysis kernel(s)."""

    def __init__(self, batch: DagBatch, sm_count: int, t_min=1, mask: int = _abi.DS_M_ALL, device: int = 0):
        self.h = C.c_void_p()
        self.n = batch.n_dags
        cb = batch.as_c()
        pl = platform(sm_count, t_min)
        check(lib().ds_session_create(C.byref(cb), C.byref(pl), mask, device, C.byref(self.h)))

    def run(self) -> float:
        ms = C.c_float(0)
        check(lib().ds_session_run(self.h, C.byref(ms)))
        return ms.value

    def kernel_times(self) -> dict:
        """{kernel name: ms} of the last run (events between launches)."""
        ms = (C.c_float * 8)()
        names = (C.c_char_p * 8)()
        k = lib().ds_session_kernel_times(self.h, ms, names, 8)
        if k < 0:
            check(-k)
        return {names[i].decode(): float(ms[i]) for i in range(k)}

    def results(self):
        st, b, ng, r = _results(self.n)
        check(lib().ds_session_results(self.h, C.byref(r)))
        return st, b, ng

    def close(self):
        if self.h:
            lib().ds_session_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def validate(batch: DagBatch, sm_count: int, samples: int, scale_min, scale_max, seed: int, t_min=1,
             device: int = 0):
    """Batched Theorem-1 check (run_validation, experiment.cpp:163-240) on GPU.

    Returns (summary dict, per-DAG status, violations, tight_worst, tight_scaled).
    `seed` is the GenConfig seed the corpus came from (sample seeds are
    seed + 7919 * d + s as in the reference)."""
    from fractions import Fraction
    L = lib()
    f = L.ds_validate_batch
    P = C.POINTER
    f.restype = C.c_int
    f.argtypes = [P(_abi.ds_dag_batch), P(_abi.ds_platform), C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                  C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(_abi.ds_validation), C.c_int]
    n = batch.n_dags
    st = np.zeros(n, np.int32)
    viol = np.zeros(n, np.int32)
    tw = np.zeros(n, np.float64)
    ts = np.zeros(n, np.float64)
    summ = _abi.ds_validation()
    smin, smax = Fraction(scale_min), Fraction(scale_max)
    cb = batch.as_c()
    pl = platform(sm_count, t_min)
    check(f(C.byref(cb), C.byref(pl), int(samples), smin.numerator, smin.denominator, smax.numerator,
            smax.denominator, int(seed), st.ctypes.data, viol.ctypes.data, tw.ctypes.data, ts.ctypes.data,
            C.byref(summ), device))
    summary = {"tasks": summ.tasks, "runs": summ.runs, "violations": summ.violations,
               "mean_tightness_worst": summ.mean_tightness_worst,
               "mean_tightness_scaled": summ.mean_tightness_scaled}
    return summary, combine_status(batch.pack_status, st), viol, tw, ts
