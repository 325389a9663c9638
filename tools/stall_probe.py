#!/usr/bin/env python
"""Sporadic ~ms stalls in executor replays: which configurations see them?
Runs one C2 DAG many times per (sm_limit, workload, engine) and reports the
replays whose makespan exceeds 1.5x the median, with their start times."""
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

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
b = _lib.Corpus(40, seed=1).batch()
loads, edges = dag_from_batch(b, 1)
for sm_limit in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8,0").split(",")]:
    M = sm_limit or 148
    sch = scheme.schedule_batch(pack([(loads, edges)]), M)[0][0]
    for wl, wname in ((X.WL_MIX32, "ldg"),) if len(sys.argv) > 3 else ((X.WL_MIX32, "ldg"), (X.WL_MIX32_TMA, "tma")):
        for engine, ename in ((X.ENGINE_GRAPH, "graph"),) if len(sys.argv) > 3 else ((X.ENGINE_GRAPH, "graph"), (X.ENGINE_DYNAMIC, "dynamic")):
            plan = X.plan_from_scheme(sch, loads, 1 << 17, barrier_groups=False)
            ex = X.Executor(plan, workload=wl, engine=engine, sm_limit=sm_limit)
            r = ex.run(reps, warmup=3, stamps=True)
            mk = r.makespan_us
            med = float(np.median(mk))
            bad = np.nonzero(mk > 1.5 * med)[0]
            starts = r.stamps[:, :, 0].min(axis=1).astype(np.float64) / 1e6  # ms
            print(json.dumps({"M": M, "wl": wname, "engine": ename, "median_us": round(med, 1),
                              "stalls": len(bad), "stall_extra_us": [round(float(mk[i] - med), 1) for i in bad[:8]],
                              "stall_at_ms": [round(float(starts[i] - starts[0]), 1) for i in bad[:8]],
                              "run_ms": round(float(starts[-1] - starts[0]), 1)}), flush=True)
            ex.close()
