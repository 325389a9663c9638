# Dynamic engine probe variants: two-pass probe (default) vs one-pass (DS_DYN_PROBE2=0), claim-ahead on.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/ahead2_pytest.log 2>&1; echo "executor pytest rc $?"; tail -2 gpurun_out/ahead2_pytest.log
for m in 32 148 8; do for p2 in 1 0; do
  DS_DYN_PROBE2=$p2 timeout 600 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,multistream,multistream_host --out gpurun_out/ahead2_m${m}_$p2.json > gpurun_out/ahead2_m${m}_$p2.log 2>&1; echo "M=$m probe2=$p2 rc $?"
done; done
python - <<'PY'
import json, numpy as np
for m in (32, 148, 8):
    for p2 in (1, 0):
        rows = json.load(open(f"gpurun_out/ahead2_m{m}_{p2}.json"))
        c2 = [r for r in rows if r["dag"].startswith("c2")]
        s = {v: np.mean([r[v]["p50"] for r in c2]) for v in ("dynamic_prio", "multistream", "multistream_host")}
        o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        oh = {r["dag"]: round(r["multistream_host"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        print(f"M={m} probe2={p2} C2 mean p50: " + "  ".join(f"{k} {v:.1f}" for k, v in s.items()), o, "host", oh)
PY
