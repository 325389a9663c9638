#!/usr/bin/env python
"""Per-SM bandwidth of the K2 node kernels vs how many SMs are busy.

A DAG's critical path is a chain of nodes each holding a few SMs (m <= load),
so what bounds the makespan there is how fast ONE SM streams its slice when
the rest of the chip is idle, not the full-chip HBM roofline. Consecutive
launches rotate over >= 512 MB (ds_node_kernel_bench) so every launch streams
from HBM.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20826_b200 import executor as X  # noqa: E402

WLS = {"ldg4": X.WL_MIX32, "ldg8": X.WL_MIX32_LDG8, "tma6x32k": X.WL_MIX32_TMA}


def placement():
    import ctypes as C
    L = X._sig()
    L.ds_node_placement_bench.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.c_int, C.POINTER(C.c_double), C.c_int]
    out = []
    for elems in (1 << 17, 1 << 20):
        for k in (2, 8, 16, 32, 64, 74):
            row = {"elems": elems, "k": k}
            pats = {"contig": list(range(k)), "contig_hi": list(range(148 - k, 148)),
                    "even": list(range(0, 2 * k, 2)), "spread": [i * 148 // k for i in range(k)]}
            for name, sms in pats.items():
                m = (C.c_uint32 * 8)()
                for v in sms:
                    m[v >> 5] |= 1 << (v & 31)
                span = C.c_double()
                assert L.ds_node_placement_bench(m, elems, 20, C.byref(span), 0) == 0
                row[name] = {"us": round(span.value / 1e3, 2),
                             "GBs_per_sm": round(elems * 8 / span.value, 1)}
            print(json.dumps(row), flush=True)
            out.append(row)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "placement.json"), "w"), indent=1)


def main():
    if "--placement" in sys.argv:
        return placement()
    out = []
    for elems in (1 << 17, 1 << 20):
        for ctas in (1, 8, 20, 40, 74, 148):
            row = {"elems_per_cta": elems, "ctas": ctas}
            for name, wl in WLS.items():
                ms, span = X.node_kernel_bench(wl, ctas, elems, reps=30)
                byts = ctas * elems * 8
                row[name] = {"us": round(ms * 1e3, 2), "span_us": round(span / 1e3, 2),
                             "GBs": round(byts / (ms * 1e-3) / 1e9, 1),
                             "GBs_per_sm": round(byts / (ms * 1e-3) / 1e9 / ctas, 1)}
            print(json.dumps(row), flush=True)
            out.append(row)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "node_bw_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
