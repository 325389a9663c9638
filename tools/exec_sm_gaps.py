#!/usr/bin/env python
"""Per-SM idle gaps between consecutive CTAs / ranks (diagnostic, one GPU):
for each variant, the median replay's stamps grouped by %smid, and the gaps
t0(next) - t1(prev) on each SM — where the dynamic engine and hardware CTA
dispatch differ under contention.

  python tools/exec_sm_gaps.py --sm-limit 32 --dags c2:6
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from exec_study import engine_for, make_dags, plan_for  # noqa: E402
from paper_2602_20826_b200 import executor as X  # noqa: E402
from paper_2602_20826_b200 import scheme  # noqa: E402
from paper_2602_20826_b200.batch import pack  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dags", default="c2:6")
    ap.add_argument("--variants", default="dynamic_prio,dynamic_ms,multistream")
    ap.add_argument("--replays", type=int, default=30)
    ap.add_argument("--unit", type=int, default=1 << 17)
    ap.add_argument("--sm-limit", type=int, default=32)
    args = ap.parse_args()
    M = args.sm_limit or 148
    dags = make_dags(args.dags, M)
    schemes, _ = scheme.schedule_batch(pack([d for _, d in dags]), M)
    out = {}
    for (name, (loads, edges)), sch in zip(dags, schemes):
        for kind in args.variants.split(","):
            plan = plan_for(kind, sch, loads, edges, M, args.unit)
            ex = X.Executor(plan, workload=X.WL_MIX32_TMA, engine=engine_for(kind), sm_limit=args.sm_limit)
            r = ex.run(args.replays, warmup=3, stamps=True)
            ex.close()
            med = int(np.argsort(r.makespan_us)[len(r.makespan_us) // 2])
            st = r.stamps[med].astype(np.int64)
            sm = r.smids[med]
            t0 = st[:, 0].min()
            gaps, busy, items = [], 0, 0
            for s in np.unique(sm):
                w = st[sm == s]
                w = w[np.argsort(w[:, 0])]
                busy += int((w[:, 1] - w[:, 0]).sum())
                items += len(w)
                gaps += list((w[1:, 0] - w[:-1, 1]) / 1e3)
            g = np.array(gaps) if gaps else np.zeros(1)
            rec = out.setdefault(kind, {"gap_us": [], "items_per_sm": [], "makespan_us": [], "item_us": []})
            rec["gap_us"] += g.tolist()
            rec["items_per_sm"].append(items / max(1, len(np.unique(sm))))
            rec["makespan_us"].append(float(r.makespan_us[med]))
            rec["item_us"].append(busy / 1e3 / max(1, items))
    for kind, rec in out.items():
        g = np.array(rec["gap_us"])
        print(f"{kind:>14}: makespan {np.mean(rec['makespan_us']):7.1f} us  items/SM {np.mean(rec['items_per_sm']):5.1f}"
              f"  item {np.mean(rec['item_us']):5.2f} us  gap p50 {np.median(g):5.2f} mean {g.mean():5.2f}"
              f" p90 {np.percentile(g, 90):6.2f} us  (n {len(g)})", flush=True)
    json.dump({k: {kk: (vv if kk != "gap_us" else None) for kk, vv in v.items()} for k, v in out.items()},
              open(os.path.join(ROOT, "gpurun_out", "exec_sm_gaps.json"), "w"))


if __name__ == "__main__":
    main()
