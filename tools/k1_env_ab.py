"""A/B of K1 environment knobs on the 1M C5 corpus (Session, device-resident):
per setting the median pass time, per-kernel times and a checksum of every
result (settings must agree bit for bit).
  python tools/k1_env_ab.py DS_LANE_STAGE=0 DS_LANE_STAGE=1"""
import os
import subprocess
import sys

CODE = r'''
import sys, statistics, hashlib; sys.path.insert(0, ".")
from paper_2602_20826_b200 import _lib
b = _lib.Corpus(1000000, pinned=True, seed=1, gpu=True).batch()
for n in (1000000, 125000):
    s = _lib.Session(b.slice(0, n), 148)
    for _ in range(3): s.run()
    ms = statistics.median(s.run() for _ in range(15))
    st, bo, ng = s.results()
    h = hashlib.sha1(st.tobytes() + bo.tobytes() + ng.tobytes()).hexdigest()[:12]
    kt = s.kernel_times()
    print(f"n {n} {ms:.3f} ms sha {h} " + " ".join(f"{k} {v:.3f}" for k, v in kt.items()), flush=True)
'''
for setting in sys.argv[1:]:
    env = dict(os.environ)
    for kv in setting.split(","):
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print("==", setting)
    print(out.stdout.strip(), out.stderr.strip()[-500:])
