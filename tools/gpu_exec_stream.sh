# Claim-ahead engine with the ring streaming across items: executor tests, then
# the contended study (M = 32, 8; claim-ahead on by default there) and M = 148
# with claim-ahead forced on/off.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/xs_pytest.log 2>&1; echo "executor pytest rc $?"; tail -2 gpurun_out/xs_pytest.log
DS_DYN_AHEAD=1 timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/xs_pytest_ahead.log 2>&1; echo "executor pytest (ahead forced) rc $?"; tail -2 gpurun_out/xs_pytest_ahead.log
run() {  # M tag env...
  m=$1; tag=$2; shift 2
  env "$@" timeout 600 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,multistream,multistream_host --out gpurun_out/xs_${tag}.json > gpurun_out/xs_${tag}.log 2>&1; echo "$tag rc $?"
}
run 32 m32
run 8 m8
run 32 m32_off DS_DYN_AHEAD=0
run 0 m148_on DS_DYN_AHEAD=1
run 0 m148
python - <<'PY'
import json, numpy as np
for tag in ("m32", "m32_off", "m8", "m148_on", "m148"):
    rows = json.load(open(f"gpurun_out/xs_{tag}.json"))
    c2 = [r for r in rows if r["dag"].startswith("c2")]
    s = {v: np.mean([r[v]["p50"] for r in c2]) for v in ("dynamic_prio", "multistream", "multistream_host")}
    o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
    oh = {r["dag"]: round(r["multistream_host"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
    print(f"{tag} C2 mean p50: " + "  ".join(f"{k} {v:.1f}" for k, v in s.items()), o, "host", oh)
PY
