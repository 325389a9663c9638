"""Packed DAG batches — the host-side form of ``std::vector<DagTask>``.

Layout (include/dagsched_b200.h, ``ds_dag_batch``): DAG d owns the node range
``[node_off[d], node_off[d+1])`` in ascending-id order (a node's local index is
the rank of its id, so every "ties by id" rule of the reference becomes "ties
by index") and the edge range ``[edge_off[d], edge_off[d+1])`` of
``(from_local << 16) | to_local`` words. Loads are exact rationals
``load_num / load_den``.

Validation that needs node ids (duplicate ids, unknown edge endpoints;
dag.cpp:28-60) happens here, at packing time, exactly where the reference's
``DagTask::make`` does it; everything id-free (self loops, cycles, single
source/sink, loads) is checked by the device kernel.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, Sequence

import numpy as np

from . import _abi


@dataclass
class DagBatch:
    node_off: np.ndarray  # uint32 [n+1]
    edge_off: np.ndarray  # uint32 [n+1]
    load_num: np.ndarray  # int64 [N]
    load_den: np.ndarray  # int64 [N]
    edges: np.ndarray     # uint32 [E]
    pack_status: np.ndarray  # int32 [n]: DS_OK or an id-level validation code
    node_ids: list | None = None  # per DAG, sorted original ids (None: ids = indices)

    @property
    def n_dags(self) -> int:
        return int(self.node_off.shape[0] - 1)

    @property
    def n_nodes(self) -> int:
        return int(self.node_off[-1]) - int(self.node_off[0])  # indices are relative to node_off[0]

    @property
    def n_edges(self) -> int:
        return int(self.edge_off[-1]) - int(self.edge_off[0])

    def sizes(self) -> np.ndarray:
        return np.diff(self.node_off.astype(np.int64))

    def nbytes(self, with_den: bool = True) -> int:
        b = self.node_off.nbytes + self.edge_off.nbytes + self.load_num.nbytes + self.edges.nbytes
        return b + (self.load_den.nbytes if with_den else 0)

    def integer_loads(self) -> bool:
        return bool(np.all(self.load_den == 1))

    def as_c(self, with_den: bool | None = None) -> _abi.ds_dag_batch:
        if with_den is None:
            with_den = not self.integer_loads()
        for a in (self.node_off, self.edge_off, self.load_num, self.load_den, self.edges):
            assert a.flags["C_CONTIGUOUS"]
        return _abi.ds_dag_batch(
            self.n_dags, self.node_off.ctypes.data, self.edge_off.ctypes.data,
            self.load_num.ctypes.data, self.load_den.ctypes.data if with_den else None,
            self.edges.ctypes.data)

    def compact16_ok(self) -> bool:
        """Fits ds_dag_batch16: integer loads in [1, 65535], <= 256 nodes per DAG."""
        return (self.integer_loads() and self.load_num.size > 0 and int(self.load_num.min()) >= 1
                and int(self.load_num.max()) <= 0xFFFF and int(self.sizes().max(initial=0)) <= 256)

    def compact16(self, out=None):
        """(load u16 [N], edges u16 [E]: from << 8 | to) — the ds_dag_batch16
        wire form. `out` = preallocated (e.g. pinned) arrays to fill."""
        if not self.compact16_ok():
            raise ValueError("batch does not fit the 16-bit wire form")
        load = out[0] if out else np.empty(self.load_num.shape, np.uint16)
        edges = out[1] if out else np.empty(self.edges.shape, np.uint16)
        np.copyto(load, self.load_num, casting="unsafe")
        np.copyto(edges, ((self.edges >> 16) << 8) | (self.edges & 0xFF), casting="unsafe")
        return load, edges

    def as_c16(self, load16: np.ndarray, edges16: np.ndarray) -> _abi.ds_dag_batch16:
        for a in (self.node_off, self.edge_off, load16, edges16):
            assert a.flags["C_CONTIGUOUS"]
        return _abi.ds_dag_batch16(self.n_dags, self.node_off.ctypes.data, self.edge_off.ctypes.data,
                                   load16.ctypes.data, edges16.ctypes.data)

    def tri_ok(self) -> bool:
        """Fits ds_dag_batch_tri: integer loads in [0, 65535], <= 64 nodes per
        DAG, every edge u < v (local indices are a topological order)."""
        if not (self.integer_loads() and self.load_num.size > 0 and int(self.load_num.min()) >= 0
                and int(self.load_num.max()) <= 0xFFFF and int(self.sizes().max(initial=0)) <= 64):
            return False
        return bool(np.all((self.edges >> 16) < (self.edges & 0xFFFF)))

    def tri_words(self) -> np.ndarray:
        """adj_off (uint32 [n+1], in u32 words) of the triangular form."""
        n = self.sizes()
        words = (n * (n - 1) // 2 + 31) // 32
        off = np.zeros(self.n_dags + 1, np.uint32)
        np.cumsum(words, out=off[1:])
        return off

    def tri(self, out=None):
        """(load u16 [N], adj_off u32 [n+1], adj u32 [W]) — the ds_dag_batch_tri
        wire form: node v's predecessors are bits v(v-1)/2 + u of its DAG's
        words. `out` = preallocated (load, adj) arrays to fill (e.g. pinned;
        adj sized tri_words()[-1])."""
        if not self.tri_ok():
            raise ValueError("batch does not fit the triangular wire form")
        adj_off = self.tri_words()
        nw = int(adj_off[-1])
        load = out[0] if out else np.empty(self.load_num.shape, np.uint16)
        np.copyto(load, self.load_num, casting="unsafe")
        ecount = np.diff(self.edge_off.astype(np.int64))
        dag = np.repeat(np.arange(self.n_dags, dtype=np.int64), ecount)
        u = (self.edges >> 16).astype(np.int64)
        v = (self.edges & 0xFFFF).astype(np.int64)
        bit = adj_off[dag].astype(np.int64) * 32 + v * (v - 1) // 2 + u
        bits = np.zeros(nw * 32, np.bool_)
        bits[bit] = True  # duplicate edges collapse, as DagTask::make dedups them
        words = np.packbits(bits, bitorder="little").view(np.uint32)
        adj = out[1] if out else np.empty(nw, np.uint32)
        np.copyto(adj, words)
        return load, adj_off, adj

    def as_ctri(self, load16: np.ndarray, adj_off: np.ndarray, adj: np.ndarray) -> _abi.ds_dag_batch_tri:
        for a in (self.node_off, adj_off, load16, adj):
            assert a.flags["C_CONTIGUOUS"]
        return _abi.ds_dag_batch_tri(self.n_dags, self.node_off.ctypes.data, adj_off.ctypes.data,
                                     load16.ctypes.data, adj.ctypes.data)

    def slice(self, lo: int, hi: int) -> "DagBatch":
        """DAGs [lo, hi) as a new batch with rebased offsets."""
        n0, n1 = int(self.node_off[lo]), int(self.node_off[hi])
        e0, e1 = int(self.edge_off[lo]), int(self.edge_off[hi])
        return DagBatch(
            np.ascontiguousarray(self.node_off[lo:hi + 1] - n0, dtype=np.uint32),
            np.ascontiguousarray(self.edge_off[lo:hi + 1] - e0, dtype=np.uint32),
            np.ascontiguousarray(self.load_num[n0:n1]), np.ascontiguousarray(self.load_den[n0:n1]),
            np.ascontiguousarray(self.edges[e0:e1]),
            np.ascontiguousarray(self.pack_status[lo:hi]),
            None if self.node_ids is None else self.node_ids[lo:hi])


def _frac(x) -> Fraction:
    if isinstance(x, Fraction):
        return x
    if isinstance(x, str):
        return Fraction(x)
    if isinstance(x, int):
        return Fraction(x)
    if isinstance(x, tuple):
        return Fraction(x[0], x[1])
    return Fraction(str(x))  # shortest decimal, like task_io.cpp:29-35


def pack(dags: Iterable[tuple[Sequence, Sequence[tuple[int, int]]]]) -> DagBatch:
    """Pack ``[(nodes, edges), ...]``.

    ``nodes`` is a sequence of ``(id, load)`` pairs or a plain list of loads
    (ids 0..n-1); ``edges`` is a sequence of ``(from_id, to_id)``. Loads may be
    ints, Fractions, ``(num, den)`` tuples or strings such as ``"15/2"``.
    """
    node_off, edge_off, nums, dens, words, status, all_ids = [0], [0], [], [], [], [], []
    for nodes, edges in dags:
        nodes = list(nodes)
        if nodes and not isinstance(nodes[0], (tuple, list)):
            nodes = list(enumerate(nodes))
        nodes = sorted(((int(i), _frac(l)) for i, l in nodes), key=lambda t: t[0])
        ids = [i for i, _ in nodes]
        st = _abi.DS_OK
        if not nodes:
            st = _abi.DS_E_EMPTY
        elif len(set(ids)) != len(ids):
            st = _abi.DS_E_DUP_ID
        elif len(ids) > _abi.DS_MAX_NODES:
            st = _abi.DS_ETOOBIG
        index = {i: k for k, i in enumerate(ids)}
        local = []
        if st == _abi.DS_OK:
            # dag.cpp:49-66: edges sorted + deduplicated, then checked in that
            # order for an unknown endpoint or a self loop (first hit wins).
            for u, v in sorted(set((int(a), int(b)) for a, b in edges)):
                if u not in index or v not in index:
                    st = _abi.DS_E_EDGE
                    break
                if u == v:
                    st = _abi.DS_E_SELFLOOP
                    break
                local.append((index[u] << 16) | index[v])
            if st != _abi.DS_OK:
                local = []
        for _, l in nodes:
            nums.append(l.numerator)
            dens.append(l.denominator)
        words.extend(local)
        node_off.append(len(nums))
        edge_off.append(len(words))
        status.append(st)
        all_ids.append(ids)
    return DagBatch(np.asarray(node_off, np.uint32), np.asarray(edge_off, np.uint32),
                    np.asarray(nums, np.int64), np.asarray(dens, np.int64),
                    np.asarray(words, np.uint32), np.asarray(status, np.int32), all_ids)


def from_arrays(node_off, edge_off, load_num, load_den, edges) -> DagBatch:
    n = len(node_off) - 1
    return DagBatch(np.ascontiguousarray(node_off, np.uint32), np.ascontiguousarray(edge_off, np.uint32),
                    np.ascontiguousarray(load_num, np.int64), np.ascontiguousarray(load_den, np.int64),
                    np.ascontiguousarray(edges, np.uint32), np.zeros(n, np.int32))


def bounds_as_fractions(bounds: np.ndarray, d: int) -> dict:
    row = bounds[d * 10:(d + 1) * 10] if bounds.ndim == 1 else bounds[d]
    out = {}
    for k, name in enumerate(_abi.BOUND_NAMES):
        num, den = int(row[2 * k]), int(row[2 * k + 1])
        out[name] = None if den == 0 else Fraction(num, den)
    return out


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data_as(C.c_void_p).value


_PACK_FIRST = (_abi.DS_E_EMPTY, _abi.DS_E_DUP_ID, _abi.DS_ETOOBIG)


def combine_status(pack_status: np.ndarray, device_status: np.ndarray) -> np.ndarray:
    """Merge id-level (packer) and device validation in the reference's order.

    dag.cpp checks: empty, duplicate id (packer) -> load >= min (device) ->
    unknown endpoint / self loop (packer, first in sorted edge order) ->
    cycle, sources, sinks (device) -> scheduler's load >= t_min (device).
    """
    p = np.asarray(pack_status)
    d = np.asarray(device_status)
    out = np.where(p == _abi.DS_OK, d, p)
    out = np.where((p != _abi.DS_OK) & ~np.isin(p, _PACK_FIRST) & (d == _abi.DS_E_LOAD), d, out)
    return out.astype(np.int32)
