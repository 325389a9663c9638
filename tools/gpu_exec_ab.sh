# Executor A/B in one session: the HEAD library (build_ab/old) vs the working
# tree's, alternating, C1-C4 at M = 148 and 32.
mkdir -p gpurun_out
run() {  # M tag lib
  DAGSCHED_LIB=$3 timeout 600 python tools/exec_study.py --sm-limit $1 --dags c1,c3,c4_0,c4_1,c4_2,c2:12 --replays 100 \
    --windows none --variants dynamic_prio,multistream,multistream_host --out gpurun_out/ab_$2.json > gpurun_out/ab_$2.log 2>&1
  echo "$2 rc $?"
}
OLD=$PWD/build_ab/old/libdagsched_b200.so
NEW=$PWD/paper_2602_20826_b200/_lib/libdagsched_b200.so
for r in 1 2; do
  run 0 m148_old$r $OLD; run 0 m148_new$r $NEW
  run 32 m32_old$r $OLD; run 32 m32_new$r $NEW
done
python - <<'PY'
import json, numpy as np
for m in ("m148", "m32"):
    for v in ("old1", "new1", "old2", "new2"):
        rows = json.load(open(f"gpurun_out/ab_{m}_{v}.json"))
        c2 = [r for r in rows if r["dag"].startswith("c2")]
        s = np.mean([r["dynamic_prio"]["p50"] for r in c2])
        h = np.mean([r["multistream_host"]["p50"] for r in c2])
        o = {r["dag"]: round(r["dynamic_prio"]["p50"], 1) for r in rows if not r["dag"].startswith("c2")}
        print(f"{m} {v}: C2 dynamic_prio {s:.1f} (host {h:.1f})", o)
PY
