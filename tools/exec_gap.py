#!/usr/bin/env python
"""Where does an executor's makespan go? (diagnostic, one GPU)

For a few C2 DAGs and each engine variant, from the per-CTA %globaltimer
stamps of one replay:
  cp_us     longest path through the plan's edges using each entity's
            measured duration (first CTA start -> last CTA end), zero gaps
  gap_us    makespan - cp_us: dispatch/launch/dependency latency on the
            critical chain plus waiting for SMs
  sm_gbs    per-SM bandwidth of the critical chain's CTAs (bytes / CTA time)
  work_us   total bytes / measured HBM copy peak (the no-dependency floor)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench_executor import dag_from_batch  # noqa: E402
from paper_2602_20826_b200 import _lib, scheme  # noqa: E402
from paper_2602_20826_b200 import executor as X  # noqa: E402
from paper_2602_20826_b200.batch import pack  # noqa: E402


def analyse(plan, res, r, bpe):
    st = res.stamps[r]
    sl = X.plan_slots(plan)
    n = len(plan.entities)
    win = [(int(st[sl[i]:sl[i + 1], 0].min()), int(st[sl[i]:sl[i + 1], 1].max())) for i in range(n)]
    t0 = min(w[0] for w in win)
    dur = [(b - a) / 1e3 for a, b in win]
    # entities are in a topological order in every plan kind
    fin = [0.0] * n
    arg = [-1] * n
    for i, e in enumerate(plan.entities):
        best, bp = 0.0, -1
        for p in e.preds:
            if fin[p] > best:
                best, bp = fin[p], p
        fin[i] = best + dur[i]
        arg[i] = bp
    last = int(np.argmax(fin))
    chain = []
    while last >= 0:
        chain.append(last)
        last = arg[last]
    mk = (max(w[1] for w in win) - t0) / 1e3
    cta_gbs = []
    for i in chain:
        e = plan.entities[i]
        s = st[sl[i]:sl[i + 1]]
        for k in range(len(s)):
            el = (e.hi - e.lo) / e.parallelism
            cta_gbs.append(el * bpe / max(1, int(s[k, 1] - s[k, 0])))
    # gaps along the chain: start(i) - end(pred on chain)
    gaps = []
    for a, b in zip(chain[1:], chain[:-1]):
        gaps.append((win[b][0] - win[a][1]) / 1e3)
    return {"makespan_us": mk, "cp_us": max(fin), "gap_us": mk - max(fin), "chain_len": len(chain),
            "chain_gap_mean_us": float(np.mean(gaps)) if gaps else 0.0,
            "chain_sm_gbs_mean": float(np.mean(cta_gbs)),
            "chain_dur_us": [round(dur[i], 1) for i in reversed(chain)],
            "chain_m": [plan.entities[i].parallelism for i in reversed(chain)]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dags", type=int, default=6)
    ap.add_argument("--replays", type=int, default=30)
    ap.add_argument("--unit", type=int, default=1 << 17)
    ap.add_argument("--workload", type=int, default=X.WL_MIX32)
    ap.add_argument("--variants", default="proposed,proposed_deps,dynamic,dynamic_deps,dynamic_deps_tma,multistream,multistream_tma,dyn_multistream,multistream_free")
    ap.add_argument("--sm-limit", type=int, default=0)
    ap.add_argument("--avg-load", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "exec_gap.json"))
    args = ap.parse_args()
    M = args.sm_limit or 148
    peak = 6539.2
    corpus = _lib.Corpus(600, seed=1, avg_load=args.avg_load)
    b = corpus.batch()
    sizes = np.diff(b.node_off.astype(np.int64))
    picked = [d for d in range(b.n_dags) if 20 <= sizes[d] <= 50][:args.dags]
    dags = [dag_from_batch(b, d) for d in picked]
    schemes, st = scheme.schedule_batch(pack(dags), M)
    bpe = X.BYTES_PER_ELEM[args.workload]
    out = []
    for (loads, edges), sch in zip(dags, schemes):
        row = {"n": len(loads), "groups": len(sch.groups)}
        tot = sum(X.node_elements(loads, args.unit)) * bpe
        row["work_us"] = tot / (peak * 1e3) * 148 / M
        for kind in args.variants.split(","):
            engine = (X.ENGINE_STREAMS if kind.endswith("_host") else
                      X.ENGINE_DYNAMIC if kind.startswith("dyn") else
                      X.ENGINE_GRAPH_FREE if kind.endswith("_free") else X.ENGINE_GRAPH)
            chunk = 0
            if "_c" in kind and kind.startswith("dyn"):  # e.g. dynamic_deps_c32768: chunked ranks
                kind, chunk = kind.split("_c")[0], int(kind.split("_c")[1])
            wl = X.WL_MIX32_TMA if kind.endswith("_tma") else args.workload
            kind_ = kind.replace("_tma", "")
            if kind_.startswith(("proposed", "dynamic")):
                plan = X.plan_from_scheme(sch, loads, args.unit, barrier_groups=not kind_.endswith("_deps"))
            else:
                plan = X.plan_baseline(kind_.replace("_free", "").replace("dyn_", "").replace("_host", ""), loads, edges, M, args.unit)
            ex = X.Executor(plan, workload=wl, engine=engine, sm_limit=args.sm_limit, chunk_elems=chunk)
            res = ex.run(args.replays, warmup=3, stamps=True)
            if engine == X.ENGINE_GRAPH_FREE:
                plan._slots = ex.slots
                for e in plan.entities:
                    e.parallelism *= X.FREE_CTA_FACTOR
            a = [analyse(plan, res, r, bpe) for r in range(args.replays)]
            med = int(np.argsort([x["makespan_us"] for x in a])[len(a) // 2])
            row[kind + (f"_c{chunk}" if chunk else "")] = a[med]
            ex.close()
        out.append(row)
        print(json.dumps({k: (v if not isinstance(v, dict) else {kk: vv for kk, vv in v.items()
                                                                   if not kk.startswith("chain_")
                                                                   or kk in ("chain_gap_mean_us",
                                                                             "chain_sm_gbs_mean")})
                          for k, v in row.items()}), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
