"""End-to-end ds_analyze_batch time (1M C5 DAGs, pinned host buffers) under
environment settings:  python tools/e2e_probe.py DS_CHUNKS=4 DS_CHUNKS=8"""
import os
import subprocess
import sys

CODE = r'''
import sys, time, ctypes as C; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2602_20826_b200 import _abi, _lib
n = 1000000
corpus = _lib.Corpus(n, pinned=True, seed=1, gpu=True)
b = corpus.batch()
st = torch.zeros(n, dtype=torch.int32, pin_memory=True).numpy()
bo = torch.zeros((n, 10), dtype=torch.int64, pin_memory=True).numpy()
ng = torch.zeros(n, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
r = _abi.ds_results(st.ctypes.data, bo.ctypes.data, ng.ctypes.data)
cb, pl, L = b.as_c(), _lib.platform(148), _lib.lib()
for _ in range(3): _lib.check(L.ds_analyze_batch(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), 0, None, 0))
ts = []
for _ in range(7):
    t0 = time.perf_counter(); _lib.check(L.ds_analyze_batch(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), 0, None, 0)); ts.append(time.perf_counter() - t0)
ts.sort(); print(f"e2e median {1e3 * ts[3]:.2f} ms  min {1e3 * ts[0]:.2f}  ok={(st == 0).mean():.4f} bsum={int(bo[:, 0].sum())}")
'''
for setting in sys.argv[1:]:
    env = dict(os.environ)
    for kv in setting.split(","):
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print(setting, out.stdout.strip(), out.stderr.strip()[-300:])
