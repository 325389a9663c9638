#!/usr/bin/env python
"""Executor study (diagnostic, one GPU): per DAG and variant the makespan
percentiles, the SM-busy fraction (sum of CTA busy time / (M x makespan)) and
the DAG's achieved bandwidth (bytes / makespan), plus, for chosen DAGs, the
per-entity windows of the median replay — where the schedule leaves SMs idle
next to naive multi-stream launch.

  python tools/exec_study.py --dags c1,c3,c4_0,c4_1,c4_2,c2:4 --replays 100 --windows c4_0
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench_executor import dag_from_batch, normalise  # noqa: E402
from paper_2602_20826_b200 import _lib, scheme, workloads  # noqa: E402
from paper_2602_20826_b200 import executor as X  # noqa: E402
from paper_2602_20826_b200.batch import pack  # noqa: E402


def make_dags(spec, M):
    out = []
    for tok in spec.split(","):
        if tok == "c1":
            out.append(("c1", normalise(*workloads.c1_fork_join())))
        elif tok == "c3":
            out.append(("c3", normalise(*workloads.inception_dag())))
        elif tok.startswith("c4_"):
            s = int(tok[3:])
            out.append((tok, normalise(*workloads.oversized_dag(s, M))))
        elif tok.startswith("c2:"):
            k = int(tok[3:])
            b = _lib.Corpus(400, seed=1).batch()
            sizes = np.diff(b.node_off.astype(np.int64))
            for d in [d for d in range(b.n_dags) if 20 <= sizes[d] <= 50][:k]:
                out.append((f"c2_seed{1 + d}", dag_from_batch(b, d)))
    return out


def plan_for(kind, sch, loads, edges, M, unit):
    if kind == "dynamic_ms":  # naive multi-stream's plan (original edges, m = min(m^max, M)) on the dynamic engine
        return X.plan_baseline("multistream", loads, edges, M, unit)
    if kind.endswith("_prio"):
        return X.plan_from_scheme(sch, loads, unit, mode=X.PLAN_PRIORITY)
    if kind.startswith(("proposed", "dynamic")):
        return X.plan_from_scheme(sch, loads, unit, barrier_groups=not kind.endswith("_deps"))
    return X.plan_baseline(kind.replace("_host", ""), loads, edges, M, unit)


def engine_for(kind):
    return (X.ENGINE_DYNAMIC if kind.startswith("dynamic") else
            X.ENGINE_STREAMS if kind.endswith("_host") else X.ENGINE_GRAPH)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dags", default="c1,c3,c4_0,c4_1,c4_2,c2:4")
    ap.add_argument("--variants", default="dynamic_prio,dynamic_deps,proposed_deps,multistream,multistream_host")
    ap.add_argument("--replays", type=int, default=100)
    ap.add_argument("--unit", type=int, default=1 << 17)
    ap.add_argument("--windows", default="c4_0")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "exec_study.json"))
    ap.add_argument("--sm-limit", type=int, default=0, help="green context of this many SMs (0: the whole GPU)")
    args = ap.parse_args()
    M = args.sm_limit or 148
    dags = make_dags(args.dags, M)
    schemes, st = scheme.schedule_batch(pack([d for _, d in dags]), M)
    res = []
    for (name, (loads, edges)), sch in zip(dags, schemes):
        row = {"dag": name, "n": len(loads), "groups": len(sch.groups), "bound_units": str(sch.bounds["proposed"])}
        tot_bytes = sum(X.node_elements(loads, args.unit)) * 8
        row["work_us_at_6539"] = tot_bytes / 6539.2e3
        for kind in args.variants.split(","):
            plan = plan_for(kind, sch, loads, edges, M, args.unit)
            ex = X.Executor(plan, workload=X.WL_MIX32_TMA, engine=engine_for(kind), sm_limit=args.sm_limit)
            r = ex.run(args.replays, warmup=3, stamps=True)
            ex.close()
            mk = r.makespan_us
            busy = []
            for k in range(args.replays):
                s = r.stamps[k]
                busy.append(float((s[:, 1] - s[:, 0]).astype(np.float64).sum() / 1e3 / (M * mk[k])))
            med = int(np.argsort(mk)[len(mk) // 2])
            v = {"p50": float(np.median(mk)), "p99": float(np.percentile(mk, 99)), "max": float(mk.max()),
                 "busy_frac_p50": float(np.median(busy)), "gbs_p50": tot_bytes / float(np.median(mk)) / 1e3}
            if name in args.windows.split(","):
                w = X.entity_windows(plan, r, med)
                t0 = min(a for a, _ in w)
                v["windows"] = [[e.name, e.group, e.parallelism, round((a - t0) / 1e3, 2), round((b - t0) / 1e3, 2)]
                                for e, (a, b) in zip(plan.entities, w)]
            row[kind] = v
        res.append(row)
        print(json.dumps({k: ({kk: vv for kk, vv in v.items() if kk != "windows"} if isinstance(v, dict) else v)
                          for k, v in row.items()}), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
