# Dynamic engine: reservations on (default) vs off (DS_DYN_RESERVE=0) at M = 32, 8, 148.
mkdir -p gpurun_out
run() {  # M tag env...
  m=$1; tag=$2; shift 2
  env "$@" timeout 600 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 --windows none \
    --variants dynamic_prio,multistream,multistream_host --out gpurun_out/xr_${tag}.json > gpurun_out/xr_${tag}.log 2>&1; echo "$tag rc $?"
}
run 32 m32_res1; run 32 m32_res0 DS_DYN_RESERVE=0
run 8 m8_res1; run 8 m8_res0 DS_DYN_RESERVE=0
run 0 m148_res1; run 0 m148_res0 DS_DYN_RESERVE=0
python - <<'PY'
import json, numpy as np
for tag in ("m32_res1", "m32_res0", "m8_res1", "m8_res0", "m148_res1", "m148_res0"):
    rows = json.load(open(f"gpurun_out/xr_{tag}.json"))
    c2 = [r for r in rows if r["dag"].startswith("c2")]
    s = {v: np.mean([r[v]["p50"] for r in c2]) for v in ("dynamic_prio", "multistream", "multistream_host")}
    o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
    print(f"{tag} C2 mean p50: " + "  ".join(f"{k} {v:.1f}" for k, v in s.items()), o)
PY
