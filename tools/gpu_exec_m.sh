# Executor under contention: C1-C4 + 12 C2 DAGs at M = 32 and 8 (green contexts).
mkdir -p gpurun_out
for m in 32 8 148; do
  timeout 900 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,dynamic_ms,multistream,multistream_host --out gpurun_out/exec_m$m.json > gpurun_out/exec_m$m.log 2>&1; echo "M=$m rc $?"
done
python - <<'PY'
import json
for m in (32, 8, 148):
    rows = json.load(open(f"gpurun_out/exec_m{m}.json"))
    vs = [k for k in rows[0] if isinstance(rows[0][k], dict)]
    print("M", m, "  ".join(vs))
    for r in rows:
        print(f"{r['dag']:>12}", "  ".join(f"{r[v]['p50']:8.1f}" for v in vs))
PY
