"""TEST INFRASTRUCTURE — ctypes bindings for the two CPU checkers.

* ``Checker("ref")``    -> oracle/_ref/libdagsched_ref.so, the reference's own
  sources compiled against oracle/shim (see oracle/Makefile).
* ``Checker("oracle")`` -> oracle/_build/libdagsched_oracle.so, the independent
  restatement in oracle/src.

Both implement oracle/oracle_api.h over the packed batch format of
include/dagsched_b200.h. Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from fractions import Fraction

import numpy as np

from paper_2602_20826_b200 import _abi
from paper_2602_20826_b200.batch import DagBatch, from_arrays

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libdagsched_ref.so"),
    "oracle": os.path.join(HERE, "_build", "libdagsched_oracle.so"),
}
PREFIX = {"ref": "ref_", "oracle": "orc_"}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def platform(sm_count: int, t_min=1) -> _abi.ds_platform:
    t = Fraction(t_min)
    return _abi.ds_platform(int(sm_count), 0, t.numerator, t.denominator)


def gen_config(depth_min=5, depth_max=8, max_width=8, avg_load=20, load_jitter=0.5,
               edge_density=0.2, seed=1, integer_loads=True, exact_mean=False,
               t_min=1) -> _abi.ds_gen_config:
    a, t = Fraction(avg_load), Fraction(t_min)
    return _abi.ds_gen_config(depth_min, depth_max, max_width, int(integer_loads),
                              a.numerator, a.denominator, float(load_jitter),
                              float(edge_density), int(seed), t.numerator, t.denominator,
                              int(exact_mean), 0)


class Checker:
    def __init__(self, kind: str = "ref"):
        if not available(kind):
            raise FileNotFoundError(f"{LIBS[kind]} not built (make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(LIBS[kind])
        p = PREFIX[kind]
        self._f = {}
        sig = {
            "last_error": (C.c_char_p, []),
            "free": (None, [C.c_void_p]),
            "corpus_from_packed": (C.c_void_p, [C.POINTER(_abi.ds_dag_batch), C.c_int64, C.c_int64, C.c_void_p]),
            "corpus_generate": (C.c_void_p, [C.POINTER(_abi.ds_gen_config), C.c_int64]),
            "corpus_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
            "corpus_pack": (C.c_int, [C.c_void_p] + [C.c_void_p] * 5),
            "corpus_free": (None, [C.c_void_p]),
            "corpus_evaluate": (C.c_double, [C.c_void_p, C.POINTER(_abi.ds_platform), C.c_uint32, C.c_int, C.c_void_p, C.c_void_p]),
            "scheme_json": (C.c_void_p, [C.c_void_p, C.c_uint64, C.POINTER(_abi.ds_platform)]),
            "analyze_json": (C.c_void_p, [C.c_void_p, C.c_uint64, C.POINTER(_abi.ds_platform)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(self.lib, p + name)
            fn.restype = res
            fn.argtypes = args
            self._f[name] = fn

    def error(self) -> str:
        return (self._f["last_error"]() or b"").decode()

    # ---------------------------------------------------------------- corpora
    def corpus(self, batch: DagBatch, min_load=1) -> "Corpus":
        m = Fraction(min_load)
        st = np.zeros(batch.n_dags, np.int32)
        cb = batch.as_c(with_den=True)
        h = self._f["corpus_from_packed"](C.byref(cb), m.numerator, m.denominator, st.ctypes.data)
        return Corpus(self, h, batch.n_dags, st)

    def corpus_with_ids(self, batch: DagBatch, node_ids, min_load=1) -> "Corpus":
        """corpus() with the tasks' real node ids (flat, ascending per DAG):
        the reference's write_scheme then names entities by id (ref only)."""
        m = Fraction(min_load)
        st = np.zeros(batch.n_dags, np.int32)
        ids = np.ascontiguousarray(node_ids, np.int64)
        cb = batch.as_c(with_den=True)
        f = self.lib.ref_corpus_from_packed_ids
        f.restype = C.c_void_p
        f.argtypes = [C.POINTER(_abi.ds_dag_batch), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
        h = f(C.byref(cb), m.numerator, m.denominator, ids.ctypes.data, st.ctypes.data)
        return Corpus(self, h, batch.n_dags, st)

    def generate(self, count: int, **cfg) -> "Corpus":
        g = gen_config(**cfg)
        h = self._f["corpus_generate"](C.byref(g), int(count))
        if not h:
            raise ValueError(self.error())
        return Corpus(self, h, count, np.zeros(count, np.int32))


class Corpus:
    def __init__(self, chk: Checker, handle, n_dags: int, parse_status: np.ndarray):
        self.chk, self.h, self.n_dags, self.parse_status = chk, handle, n_dags, parse_status

    def __del__(self):
        if getattr(self, "h", None):
            self.chk._f["corpus_free"](self.h)
            self.h = None

    def pack(self) -> DagBatch:
        n, nn, ne = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.chk._f["corpus_size"](self.h, C.byref(n), C.byref(nn), C.byref(ne))
        node_off = np.zeros(n.value + 1, np.uint32)
        edge_off = np.zeros(n.value + 1, np.uint32)
        ln = np.zeros(nn.value, np.int64)
        ld = np.zeros(nn.value, np.int64)
        ed = np.zeros(ne.value, np.uint32)
        rc = self.chk._f["corpus_pack"](self.h, node_off.ctypes.data, edge_off.ctypes.data,
                                        ln.ctypes.data, ld.ctypes.data, ed.ctypes.data)
        if rc != 0:
            raise ValueError(self.chk.error())
        return from_arrays(node_off, edge_off, ln, ld, ed)

    def evaluate(self, sm_count: int, t_min=1, mask: int = _abi.DS_M_ALL, parallel=True):
        """-> (status int32[n], bounds int64[n, 10], seconds)."""
        st = self.parse_status.copy()
        b = np.zeros((self.n_dags, 10), np.int64)
        pl = platform(sm_count, t_min)
        secs = self.chk._f["corpus_evaluate"](self.h, C.byref(pl), mask, int(parallel),
                                              st.ctypes.data, b.ctypes.data)
        return st, b, secs

    def _json(self, fn: str, d: int, sm_count: int, t_min):
        pl = platform(sm_count, t_min)
        p = self.chk._f[fn](self.h, d, C.byref(pl))
        if not p:
            raise RuntimeError(self.chk.error())
        try:
            return json.loads(C.string_at(p).decode())
        finally:
            self.chk._f["free"](p)

    def scheme(self, d: int, sm_count: int, t_min=1) -> dict:
        """write_scheme() JSON of schedule(task d) (task_io.cpp:94-148)."""
        return self._json("scheme_json", d, sm_count, t_min)

    def analyze(self, d: int, sm_count: int, t_min=1) -> dict:
        return self._json("analyze_json", d, sm_count, t_min)


def ref_run_validation(corpus_size: int, sm_count: int, samples: int, scale_min, scale_max, t_min=1,
                       parallel=True, **cfg) -> dict:
    """The reference's run_validation on generate_corpus(cfg, corpus_size)."""
    chk = Checker("ref")
    f = chk.lib.ref_run_validation
    f.restype = C.c_int
    f.argtypes = [C.POINTER(_abi.ds_gen_config), C.c_int, C.POINTER(_abi.ds_platform), C.c_int, C.c_int64,
                  C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
    g = gen_config(t_min=t_min, **cfg)
    pl = platform(sm_count, t_min)
    smin, smax = Fraction(scale_min), Fraction(scale_max)
    out = np.zeros(3, np.int64)
    dbl = np.zeros(2, np.float64)
    rc = f(C.byref(g), corpus_size, C.byref(pl), samples, smin.numerator, smin.denominator, smax.numerator,
           smax.denominator, int(parallel), out.ctypes.data, dbl.ctypes.data)
    if rc != 0:
        raise RuntimeError(chk.error())
    return {"tasks": int(out[0]), "runs": int(out[1]), "violations": int(out[2]),
            "mean_tightness_worst": float(dbl[0]), "mean_tightness_scaled": float(dbl[1])}


def ref_run_experiment(sweep: str, values, sm_count: int, corpus_size: int,
                       methods=("proposed", "greedy", "greedy_unaware", "graham_para"),
                       normalize_to="greedy_unaware", t_min=1, **cfg) -> str:
    """The reference's run_experiment + write_csv -> CSV text."""
    names = ("proposed", "greedy", "greedy_unaware", "graham_para")
    chk = Checker("ref")
    f = chk.lib.ref_run_experiment
    f.restype = C.c_void_p
    f.argtypes = [C.c_char, C.c_void_p, C.c_int, C.POINTER(_abi.ds_gen_config), C.POINTER(_abi.ds_platform),
                  C.c_int, C.c_uint32, C.c_int]
    vals = np.asarray(list(values), np.int64)
    g = gen_config(t_min=t_min, **cfg)
    pl = platform(sm_count, t_min)
    mask = 0
    for m in methods:
        mask |= 1 << names.index(m)
    ptr = f(sweep.encode(), vals.ctypes.data, len(vals), C.byref(g), C.byref(pl), corpus_size, mask,
            names.index(normalize_to))
    if not ptr:
        raise RuntimeError(chk.error())
    try:
        return C.string_at(ptr).decode()
    finally:
        chk._f["free"](ptr)


def _text(chk, ptr) -> str:
    if not ptr:
        raise RuntimeError(chk.error())
    try:
        return C.string_at(ptr).decode()
    finally:
        chk._f["free"](ptr)


def _tm(scaled, smin, smax):
    smin, smax = Fraction(smin), Fraction(smax)
    return (int(bool(scaled)), smin.numerator, smin.denominator, smax.numerator, smax.denominator)


def ref_sim_greedy(corpus: Corpus, sm_count: int, runs: int, policy: str = "random", policy_seed: int = 0,
                   scaled: bool = False, time_seed: int = 0, scale_min=1, scale_max=1, t_min=1):
    """simulate_greedy per DAG x run (policy seed policy_seed + r) -> (status[n, runs], makespan[n, runs, 2])."""
    chk = corpus.chk
    f = chk.lib.ref_sim_greedy
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.POINTER(_abi.ds_platform), C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                  C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    st = np.zeros((corpus.n_dags, runs), np.int32)
    mk = np.zeros((corpus.n_dags, runs, 2), np.int64)
    sc, a, b, c, d = _tm(scaled, scale_min, scale_max)
    pl = platform(sm_count, t_min)
    f(corpus.h, C.byref(pl), int(policy == "random"), policy_seed, runs, sc, time_seed, a, b, c, d,
      st.ctypes.data, mk.ctypes.data)
    return st, mk


def ref_sim_greedy_trace(corpus: Corpus, d: int, sm_count: int, policy: str = "random", policy_seed: int = 0,
                         scaled: bool = False, time_seed: int = 0, scale_min=1, scale_max=1, t_min=1) -> str:
    chk = corpus.chk
    f = chk.lib.ref_sim_greedy_trace
    f.restype = C.c_void_p
    f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_abi.ds_platform), C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                  C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    sc, a, b, c, e = _tm(scaled, scale_min, scale_max)
    pl = platform(sm_count, t_min)
    return _text(chk, f(corpus.h, d, C.byref(pl), int(policy == "random"), policy_seed, sc, time_seed, a, b, c, e))


def ref_sim_scheme_trace(corpus: Corpus, d: int, sm_count: int, scaled: bool = False, time_seed: int = 0,
                         scale_min=1, scale_max=1, t_min=1) -> str:
    chk = corpus.chk
    f = chk.lib.ref_sim_scheme_trace
    f.restype = C.c_void_p
    f.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(_abi.ds_platform), C.c_int, C.c_uint64, C.c_int64, C.c_int64,
                  C.c_int64, C.c_int64]
    sc, a, b, c, e = _tm(scaled, scale_min, scale_max)
    pl = platform(sm_count, t_min)
    return _text(chk, f(corpus.h, d, C.byref(pl), sc, time_seed, a, b, c, e))


def ref_task_roundtrip(text: str, min_load=1, seed=None):
    """write_task(read_task(text, min_load)) -> (status, text or None)."""
    chk = Checker("ref")
    f = chk.lib.ref_task_roundtrip
    f.restype = C.c_void_p
    f.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.POINTER(C.c_int32)]
    m = Fraction(min_load)
    st = C.c_int32(0)
    p = f(text.encode(), m.numerator, m.denominator, int(seed is not None), int(seed or 0), C.byref(st))
    if not p:
        return int(st.value), None
    return int(st.value), _text(chk, p)


def ref_run_benchmarks(paths, sm_counts, avg_loads, greedy_runs: int, seed: int) -> str:
    """write_bench_table(run_benchmarks(...)) -> CSV text."""
    chk = Checker("ref")
    f = chk.lib.ref_run_benchmarks
    f.restype = C.c_void_p
    f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_uint64]
    arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
    sms = np.asarray(sm_counts, np.int32)
    avg = np.asarray(avg_loads, np.int64)
    return _text(chk, f(arr, len(paths), sms.ctypes.data, len(sms), avg.ctypes.data, len(avg), greedy_runs, seed))
