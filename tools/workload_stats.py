"""Shape of the K1 workload on the C5 corpus (GPU): nodes, edges, division
groups, executed groups, members / launches / unlaunched candidates per
group, splits. Guides where the per-DAG instruction budget goes.

  python tools/workload_stats.py [--dags 20000] [--M 148]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_20826_b200 import _abi, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dags", type=int, default=20000)
    ap.add_argument("--M", type=int, default=148)
    a = ap.parse_args()
    corp = _lib.Corpus(a.dags, seed=1)
    b = corp.batch()
    n, N = b.n_dags, b.n_nodes
    st = np.zeros(n, np.int32)
    ne = np.zeros(n, np.uint16)
    ng = np.zeros(n, np.uint16)
    nd = np.zeros(n, np.uint16)
    nb = np.zeros(N, np.int16)
    ndg = np.zeros(N, np.int16)
    ents = np.zeros(2 * N, dtype=np.dtype(_abi.ds_entity_rec))
    grps = np.zeros(N, dtype=np.dtype(_abi.ds_group_rec))
    bnd = np.zeros((n, 10), np.int64)
    sizes = np.diff(b.node_off.astype(np.int64))
    ubase = np.concatenate([[0], np.cumsum(sizes * ((sizes + 63) // 64))]).astype(np.int64)
    unl_w = np.zeros(max(int(ubase[-1]), 1), np.uint64)  # unlaunched-candidate masks (header layout)
    out = _abi.ds_scheme_out(st.ctypes.data, ne.ctypes.data, ng.ctypes.data, nd.ctypes.data, nb.ctypes.data,
                             ndg.ctypes.data, ents.ctypes.data, grps.ctypes.data, bnd.ctypes.data, unl_w.ctypes.data)
    _lib.check(_lib.lib().ds_schedule_batch(C.byref(b.as_c()), C.byref(_lib.platform(a.M)), C.byref(out), 0))
    nodes = np.diff(b.node_off.astype(np.int64))
    edges = np.diff(b.edge_off.astype(np.int64))
    g = grps[: int(ng.sum())] if False else None
    # group slots are per-DAG bases at node_off (one slot per node)
    mem, lau, unl, withl = [], [], [], 0
    for d in range(n):
        base = int(b.node_off[d])
        for j in range(int(ng[d])):
            r = grps[base + j]
            mem.append(int(r["n_members"]))
            lau.append(int(r["n_launches"]))
            w = (int(sizes[d]) + 63) // 64
            unl.append(sum(bin(int(x)).count("1") for x in unl_w[ubase[d] + j * w: ubase[d] + (j + 1) * w]))
            withl += r["n_launches"] > 0
    splits = int(sum(1 for d in range(n) for k in range(int(ne[d]))
                     if ents[2 * int(b.node_off[d]) + k]["part"] == 1))
    G = len(mem)
    print(f"dags {n}  ok {(st == 0).mean():.3f}  M {a.M}")
    print(f"nodes/dag {nodes.mean():.2f} (max {nodes.max()})  edges/dag {edges.mean():.2f}  "
          f"nodes>32: {(nodes > 32).mean():.3f}")
    print(f"division groups/dag {nd.mean():.2f}  executed groups/dag {ng.mean():.2f}  entities/dag {ne.mean():.2f}")
    print(f"members/group {np.mean(mem):.2f} (hist {np.bincount(mem)[:10].tolist()})")
    print(f"launches/group {np.mean(lau):.3f}  groups with launches {withl / G:.3f}  "
          f"unlaunched cands/group {np.mean(unl):.3f}  splits/dag {splits / n:.3f}")


if __name__ == "__main__":
    main()
