mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/gp_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/gp_pytest.log
timeout 1200 python tools/exec_graph_prio.py 300 20 > gpurun_out/gp.json 2> gpurun_out/gp.err; echo "ab rc $?"
tail -8 gpurun_out/gp.err
for m in 32 8; do
  timeout 900 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants graph_prio,dynamic_prio,multistream,multistream_host --out gpurun_out/gp_m$m.json > gpurun_out/gp_m$m.log 2>&1; echo "M=$m rc $?"
done
python - <<'PY'
import json, numpy as np
for m in (32, 8):
    rows = json.load(open(f"gpurun_out/gp_m{m}.json"))
    vs = [k for k in rows[0] if isinstance(rows[0][k], dict)]
    c2 = [r for r in rows if r["dag"].startswith("c2")]
    print("M", m, "C2 mean p50", {v: round(float(np.mean([r[v]["p50"] for r in c2])), 1) for v in vs})
    for r in rows:
        if not r["dag"].startswith("c2"):
            print(f"{r['dag']:>12}", {v: round(r[v]["p50"], 1) for v in vs})
PY
