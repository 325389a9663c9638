# Same-session A/B: claim-ahead (default inside partitions) vs DS_DYN_AHEAD=0, M = 32 and 8.
mkdir -p gpurun_out
run() {  # M tag env
  m=$1; tag=$2; shift 2
  env "$@" timeout 600 python tools/exec_study.py --sm-limit $m --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 \
    --windows none --variants dynamic_prio,multistream_host --out gpurun_out/ab2_$tag.json > gpurun_out/ab2_$tag.log 2>&1
  echo "$tag rc $?"
}
for r in 1 2; do
  run 32 m32_on$r; run 32 m32_off$r DS_DYN_AHEAD=0
  run 8 m8_on$r; run 8 m8_off$r DS_DYN_AHEAD=0
done
python - <<'PY'
import json, numpy as np
for m in ("m32", "m8"):
    for v in ("on1", "off1", "on2", "off2"):
        rows = json.load(open(f"gpurun_out/ab2_{m}_{v}.json"))
        c2 = [r for r in rows if r["dag"].startswith("c2")]
        s = np.mean([r["dynamic_prio"]["p50"] for r in c2])
        o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        print(f"{m} {v}: C2 dynamic_prio {s:.1f}", o)
PY
