"""A/B of the graph engine with per-node group priorities (graph_prio) against
the dynamic engine's group-priority claiming and the multi-stream baselines:
bench.makespan_summary at reduced replay counts, all variants on the same DAGs.
Usage: python tools/exec_graph_prio.py [replays] [n_c2] > out.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n_c2 = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = bench.makespan_summary(0, replays=reps, replays_other=reps, n_c2=n_c2, n_c2_other=n_c2)
print(json.dumps(out))
for cfg, c in sorted(out["configs"].items()):
    row = {k: round(v["p50_us"], 1) for k, v in c.items() if isinstance(v, dict)}
    print(cfg, row, file=sys.stderr)
print("over_bound_raw", out["replays_over_bound_raw"], file=sys.stderr)
print("measured_over_bound", {k: round(v["max"], 3) for k, v in out["measured_over_bound"].items()}, file=sys.stderr)
