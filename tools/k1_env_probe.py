"""K1 session time (1M C5 DAGs, M=148) under environment settings, one
process per setting:  python tools/k1_env_probe.py DS_K1_SPLIT=0 DS_K1_SPLIT=1"""
import os
import subprocess
import sys

CODE = r'''
import sys; sys.path.insert(0, ".")
from paper_2602_20826_b200 import _lib
c = _lib.Corpus(1000000, seed=1, gpu=True)
s = _lib.Session(c.batch(), 148)
for _ in range(3): s.run()
t = sorted(s.run() for _ in range(5))
st, b, ng = s.results()
kt = {k: round(v, 3) for k, v in s.kernel_times().items()}
print(f"{t[2]:.3f} ms  ok={(st == 0).mean():.4f} bsum={int(b[:, 0].sum())} {kt}")
'''
for setting in sys.argv[1:]:
    env = dict(os.environ)
    for kv in setting.split(","):
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(setting, out.stdout.strip(), out.stderr.strip()[-300:])
