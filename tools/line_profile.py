"""Per-source-line executed instructions / stall share of one kernel from an
ncu report (SourceCounters) and the matching cubin's `nvdisasm -g` listing.
  python tools/line_profile.py rep.ncu-rep k1_back /tmp/x.sass [top]"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles"))
import sass_hotspots as sh  # noqa: E402

rep, kname, sass = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name-base", os.environ.get("NCU_NAME_BASE", "function"), "-k",
                      f"regex:{kname}"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
for i, row in enumerate(r):
    if "Address" in row and "Source" in row:
        h, rows = row, r[i + 1:]
        break
mangled = {"k1_fast": "_ZN2ds7k1_fastILb0EEEvNS_6K1ArgsE", "k1_front": "_ZN2ds8k1_frontILb0EEEvNS_6K1ArgsE", "k1_mid": "_ZN2ds6k1_midILb0EEEvNS_6K1ArgsE",
           "k1_back": "_ZN2ds7k1_backILb0EEEvNS_6K1ArgsE",
           "k1_back_lane": "_ZN2ds12k1_back_laneILb0ELi8EEEvNS_6K1ArgsE"}.get(kname, kname)
ins = sh.load_sass(sass, mangled)
print("rows", len(rows), "sass", len(ins))
ie, tt = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
by = collections.defaultdict(lambda: [0.0, 0.0])
for (f, line), x in zip(ins, rows):
    by[line][0] += float(x[ie] or 0)
    by[line][1] += float(x[tt] or 0)
T = sum(v[0] for v in by.values())
S = sum(v[1] for v in by.values())
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_20826_b200", "csrc")
src = {}
for fn in ("k1_analysis.cuh", "rat.cuh"):
    src[fn] = open(os.path.join(root, fn)).read().split("\n")
print(f"total {T / 1e6:.1f}M warp instructions")
for line, (e, st) in sorted(by.items(), key=lambda t: -t[1][0])[:top]:
    if line is None:
        continue
    f, l = line.split(":")
    t = src[f][int(l) - 1].strip() if f in src else ""
    print(f"{e / 1e6:8.1f}M {e / T * 100:5.1f}% st {st / S * 100:5.1f}%  {line:22s} {t[:90]}")
