#!/usr/bin/env python
"""Where do the rare ~2 ms executor stalls come from? (diagnostic, one GPU)

1. tools/heartbeat on every SM for `--hb-secs` seconds with nothing else
   running: gaps in %globaltimer reads seen by all SMs at once mean the
   context was off the GPU (another context, a driver pause).
2. One C2 DAG on the dynamic engine (DS_PLAN_PRIORITY), `--replays` stamped
   replays: for every replay >= 1 ms above the median, the per-CTA stamps —
   is one rank slow (an SM stalled) or is every SM idle for the gap (the
   whole GPU paused)?
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hb-secs", type=float, default=30)
    ap.add_argument("--replays", type=int, default=40000)
    args = ap.parse_args()
    out = {}
    hb = os.path.join(ROOT, "tools", "heartbeat")
    if args.hb_secs > 0 and os.path.exists(hb):
        r = subprocess.run([hb, str(args.hb_secs), "296", "200"], capture_output=True, text=True)
        try:
            h = json.loads(r.stdout)
            out["heartbeat"] = {k: h[k] for k in ("secs", "ctas", "thresh_us", "n_gaps")}
            out["heartbeat"]["gaps_first"] = h["gaps"][:40]
        except Exception as e:  # noqa: BLE001
            out["heartbeat"] = {"error": str(e), "stdout": r.stdout[-500:], "stderr": r.stderr[-500:]}
        print(json.dumps(out["heartbeat"])[:2000], flush=True)
    from bench_executor import dag_from_batch
    from paper_2602_20826_b200 import _lib, scheme
    from paper_2602_20826_b200 import executor as X
    from paper_2602_20826_b200.batch import pack
    b = _lib.Corpus(40, seed=1).batch()
    loads, edges = dag_from_batch(b, 1)
    sch = scheme.schedule_batch(pack([(loads, edges)]), 148)[0][0]
    plan = X.plan_from_scheme(sch, loads, 1 << 17, mode=X.PLAN_PRIORITY)
    ex = X.Executor(plan, workload=X.WL_MIX32_TMA, engine=X.ENGINE_DYNAMIC)
    res = []
    chunk = 5000
    t_first = None
    for c in range(0, args.replays, chunk):
        r = ex.run(chunk, warmup=2, stamps=True)
        mk = r.makespan_us
        med = float(np.median(mk))
        for i in np.nonzero(mk > med + 1000.0)[0]:
            st = r.stamps[i].astype(np.int64)
            t0 = st[:, 0].min()
            dur = (st[:, 1] - st[:, 0]) / 1e3
            starts = np.sort(st[:, 0] - t0) / 1e3
            ends = np.sort(st[:, 1] - t0) / 1e3
            # largest interval with no CTA running
            ev = sorted([(s, 1) for s in (st[:, 0] - t0) / 1e3] + [(e, -1) for e in (st[:, 1] - t0) / 1e3])
            run, last, idle, idle_at = 0, 0.0, 0.0, 0.0
            for t, dlt in ev:
                if run == 0 and t - last > idle:
                    idle, idle_at = t - last, last
                run += dlt
                last = t
            slow = np.argsort(-dur)[:3]
            if t_first is None:
                t_first = int(r.stamps[0, :, 0].min())
            res.append({"replay": c + int(i), "makespan_us": round(float(mk[i]), 1), "median_us": round(med, 1),
                        "longest_cta_us": [round(float(dur[j]), 1) for j in slow],
                        "longest_cta_sm": [int(r.smids[i, j]) for j in slow],
                        "median_cta_us": round(float(np.median(dur)), 1),
                        "max_all_idle_gap_us": round(idle, 1), "gap_at_us": round(idle_at, 1),
                        "at_s": round((int(t0) - t_first) / 1e9, 3)})
            print(json.dumps(res[-1]), flush=True)
    ex.close()
    out["stalls"] = res
    out["replays"] = args.replays
    with open(os.path.join(ROOT, "gpurun_out", "stall_probe2.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
