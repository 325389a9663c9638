"""K1 time vs resident CTAs per SM (DS_K1_CTAS_PER_SM), one process per setting."""
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
print(t[2])
'''
for k in sys.argv[1:] or ["1", "2", "3", "4", "5", "6", "7", "8"]:
    env = dict(os.environ, DS_K1_CTAS_PER_SM=k)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(k, out.stdout.strip(), out.stderr.strip()[-200:])
