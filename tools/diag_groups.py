"""Per-group timing diagnostic for one DAG under the executor (prints a table)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_20826_b200 import _lib, scheme, executor as X
from paper_2602_20826_b200.batch import pack

sm_limit = int(sys.argv[1]) if len(sys.argv) > 1 else 32
engine = int(sys.argv[3]) if len(sys.argv) > 3 else 0
avg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cal = X.calibrate(1 << 17, sm_limit=sm_limit)
M = cal["sm_count"]
print("cal", {k: round(v, 2) if isinstance(v, float) else v for k, v in cal.items()})
c = _lib.Corpus(60, seed=1, avg_load=avg)
b = c.batch()
sizes = np.diff(b.node_off.astype(np.int64))
d = [i for i in range(b.n_dags) if 20 <= sizes[i] <= 50][0]
n0, n1 = int(b.node_off[d]), int(b.node_off[d + 1])
loads = [int(x) for x in b.load_num[n0:n1]]
e0, e1 = int(b.edge_off[d]), int(b.edge_off[d + 1])
edges = [(int(w) >> 16, int(w) & 0xFFFF) for w in b.edges[e0:e1]]
sch = scheme.schedule_batch(pack([(loads, edges)]), M)[0][0]
plan = X.plan_from_scheme(sch, loads, 1 << 17)
ex = X.Executor(plan, sm_limit=sm_limit, engine=engine)
res = ex.run(20, warmup=3)
r = 5
win = X.entity_windows(plan, res, r)
t0 = min(w[0] for w in win)
print("bound_us", round(X.bound_us(sch, cal), 1), "measured", round(res.makespan_us[r], 1))
by = {}
for i, e in enumerate(plan.entities):
    by.setdefault(e.group, []).append(i)
prev_end = None
acc = 0.0
for j, g in enumerate(sch.groups):
    idx = by[j]
    s = min(win[i][0] for i in idx) - t0
    en = max(win[i][1] for i in idx) - t0
    stag = max(win[i][0] for i in idx) - min(win[i][0] for i in idx)
    k = len(idx)
    model = float(g.response) * cal["tau_us"]
    acc += model + (k - 1) * cal["eps_us"] + (cal["delta_us"] if j else 0)
    durs = [(win[i][1] - win[i][0]) / 1e3 for i in idx]
    ms = [plan.entities[i].parallelism for i in idx]
    ex_units = [float(plan.entities[i].exec_units) for i in idx]
    print(f"g{j:2d} k={k} R={str(g.response):6s} model={model:6.1f} dur={(en - s) / 1e3:6.1f} gap={(s - prev_end) / 1e3 if prev_end is not None else 0:5.1f} "
          f"stag={stag / 1e3:4.1f} end={en / 1e3:7.1f} bound_acc={acc:7.1f} m={ms} ent_dur={[round(x, 1) for x in durs]} units={ex_units}")
    prev_end = en
