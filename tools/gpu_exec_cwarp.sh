# Dynamic engine with the completion warp outside the main barrier: executor
# tests, per-SM gaps, then C2/C4 at M = 32, 8, 148.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/cw_pytest.log 2>&1; echo "executor pytest rc $?"; tail -2 gpurun_out/cw_pytest.log
for m in 32 148; do echo "== gaps M $m"; timeout 600 python tools/exec_sm_gaps.py --sm-limit $m --dags c2:6; done
run() {  # M tag
  timeout 600 python tools/exec_study.py --sm-limit $1 --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,multistream,multistream_host --out gpurun_out/cw_$2.json > gpurun_out/cw_$2.log 2>&1; echo "$2 rc $?"
}
run 32 m32; run 8 m8; run 0 m148
python - <<'PY'
import json, numpy as np
for tag in ("m32", "m8", "m148"):
    rows = json.load(open(f"gpurun_out/cw_{tag}.json"))
    c2 = [r for r in rows if r["dag"].startswith("c2")]
    s = {v: np.mean([r[v]["p50"] for r in c2]) for v in ("dynamic_prio", "multistream", "multistream_host")}
    o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
    oh = {r["dag"]: round(r["multistream_host"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
    print(f"{tag} C2 mean p50: " + "  ".join(f"{k} {v:.1f}" for k, v in s.items()), o, "host", oh)
PY
