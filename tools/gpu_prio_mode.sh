# graph_prio priority-level mapping A/B (DS_GRAPH_PRIO_MODE 0/1/2) at M = 148 / 32 / 8.
mkdir -p gpurun_out
for m in 148 32 8; do
  for mode in 0 1 2; do
    lim=$m; [ $m = 148 ] && lim=0
    DS_GRAPH_PRIO_MODE=$mode timeout 600 python tools/exec_study.py --sm-limit $lim --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
      --variants graph_prio,multistream_host --out gpurun_out/pm_${m}_$mode.json > gpurun_out/pm_${m}_$mode.log 2>&1 || echo "M=$m mode=$mode failed"
  done
done
python - <<'PY'
import json, numpy as np
for m in (148, 32, 8):
    for mode in (0, 1, 2):
        rows = json.load(open(f"gpurun_out/pm_{m}_{mode}.json"))
        c2 = [r for r in rows if r["dag"].startswith("c2")]
        o = {r["dag"]: round(r["graph_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        print(f"M={m} mode={mode} C2 graph_prio {np.mean([r['graph_prio']['p50'] for r in c2]):.1f} naive {np.mean([r['multistream_host']['p50'] for r in c2]):.1f}", o)
PY
