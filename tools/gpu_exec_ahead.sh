# Dynamic engine: claim-ahead (default) vs claim-after (DS_DYN_AHEAD=0), executor tests first.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/ahead_pytest.log 2>&1; echo "executor pytest rc $?"; tail -3 gpurun_out/ahead_pytest.log
for m in 32 148 8; do for ah in 1 0; do
  DS_DYN_AHEAD=$ah timeout 600 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,multistream,multistream_host --out gpurun_out/ahead_m${m}_$ah.json > gpurun_out/ahead_m${m}_$ah.log 2>&1; echo "M=$m ahead=$ah rc $?"
done; done
python - <<'PY'
import json, numpy as np
for m in (32, 148, 8):
    for ah in (1, 0):
        rows = json.load(open(f"gpurun_out/ahead_m{m}_{ah}.json"))
        c2 = [r for r in rows if r["dag"].startswith("c2")]
        s = {v: np.mean([r[v]["p50"] for r in c2]) for v in ("dynamic_prio", "multistream", "multistream_host")}
        o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        oh = {r["dag"]: round(r["multistream_host"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        print(f"M={m} ahead={ah} C2 mean p50: " + "  ".join(f"{k} {v:.1f}" for k, v in s.items()), o, "host", oh)
PY
