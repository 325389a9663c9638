"""Regenerate DESIGN.md's executor tables (M = 148 C1-C4 and the contended
M = 32 / 8 table) from profiles/r02_bench_line.json, so the prose numbers and
the committed bench line cannot drift apart.  python tools/design_tables.py"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_line.json")))
m = d["makespan"]
order = ["graph_prio", "dynamic_prio", "multistream_host", "multistream", "proposed", "proposed_deps",
         "dynamic_deps", "serial"]
names = {"C1": "C1 fork-join", "C2": "C2 (100 DAGs)", "C3": "C3 Inception", "C4": "C4 oversized (3 DAGs)"}
rows = []
for c in ["C1", "C2", "C3", "C4"]:
    v = m["configs"][c]
    best = min(("graph_prio", "dynamic_prio"), key=lambda k: v[k]["p50_us"])
    cells = []
    for k in order:
        x = v[k]
        p50 = f"**{x['p50_us']:.1f}**" if k == best else f"{x['p50_us']:.1f}"
        cells.append(f"{p50} / {x['p99_us']:.1f} / {x['max_us']:.1f}")
    rows.append(f"  | {names[c]} | " + " | ".join(cells) + " |")
t1 = "\n".join(rows)
ct = m["contended"]
rows = []
for M in ("32", "8"):
    cells = []
    for c in ["C1", "C2", "C3", "C4"]:
        v = ct["M" + M]["configs"][c]
        ks = ["graph_prio", "dynamic_prio", "multistream_host", "multistream"]
        best = min(ks, key=lambda k: v[k]["p50_us"])
        cells.append(" / ".join((f"**{v[k]['p50_us']:.1f}**" if k == best else f"{v[k]['p50_us']:.1f}") for k in ks))
    rows.append(f"  | {M} | " + " | ".join(cells) + " |")
t2 = "\n".join(rows)
path = os.path.join(ROOT, "DESIGN.md")
s = open(path).read()
a = s.index("  | C1 fork-join | ", s.index("| config | graph_prio | dynamic_prio"))
b = s.index("\n\n", a)
s = s[:a] + t1 + s[b:]
a = s.index("  | 32 | ")
b = s.index("\n\n", a)
s = s[:a] + t2 + s[b:]
open(path, "w").write(s)
print(t1)
print(t2)
