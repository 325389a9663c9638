#!/usr/bin/env python
"""Launch each K2 node kernel at full grid (148 CTAs x 4 Mi elements, > L2)
a few times — the command `ncu` wraps for the node-kernel HBM roofline
(profiles/r01_k2_ncu.csv)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20826_b200 import executor as X  # noqa: E402

for wl in (X.WL_MIX32_TMA, X.WL_MIX32, X.WL_MIX32_LDG8, X.WL_AXPY32):
    ms, _ = X.node_kernel_bench(wl, 148, 1 << 22, reps=2)
    print(wl, ms)
