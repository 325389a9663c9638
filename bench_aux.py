#!/usr/bin/env python
"""Benchmark of the widened rows: each GPU path next to the
reference's own CPU path (oracle/_ref, the reference sources; OpenMP on all
host cores where the reference parallelises) on the same inputs, with the
results compared in the same run.

  K5  generate_corpus (generator.cpp:98-108): device generation (ms from
      CUDA events) vs the host generator and the reference's generate_corpus
  K4  run_validation (experiment.cpp:163-240, SPEC AC2's 1000 DAGs x 10
      samples and a 100k-DAG version): ds_validate_batch vs ref run_validation
  K6  simulate_greedy (simulator.cpp:96-190): 10k DAGs x 10 random-policy
      runs, ds_simulate_greedy_batch vs the reference per (DAG, run)
  run_experiment (experiment.cpp:81-161, the Fig. 4 M sweep, 1000 DAGs per
      point): the GPU sweep vs the reference's

GPU times are wall clock around the public call (host buffers in, results
out). Writes profiles/r01_aux_bench.json.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402  (the checker / reference CPU path)
from paper_2602_20826_b200 import _lib, experiment, simulator  # noqa: E402


def timed(f):
    t0 = time.perf_counter()
    r = f()
    return r, time.perf_counter() - t0


def main():
    out = {"host_cores": os.cpu_count()}
    ref = bindings.Checker("ref" if bindings.available("ref") else "oracle")
    out["reference"] = "oracle/_ref" if ref.kind == "ref" else "oracle (restatement)"
    _lib.Corpus(1000, gpu=True).close()  # warm-up: context, modules

    # ---------------------------------------------------------------- K5
    n = 1_000_000
    g, wall_g = timed(lambda: _lib.Corpus(n, gpu=True))
    h, wall_h = timed(lambda: _lib.Corpus(n))
    r, wall_r = timed(lambda: ref.generate(n // 10))  # 100k: the reference path is single-threaded
    bg, bh = g.batch(), h.batch()
    same = all(np.array_equal(getattr(bg, k), getattr(bh, k)) for k in ("node_off", "edge_off", "load_num", "edges"))
    br = r.pack()
    same_ref = all(np.array_equal(getattr(br, k), getattr(bh.slice(0, n // 10), k))
                   for k in ("node_off", "edge_off", "load_num", "edges"))
    out["k5_generate"] = {"dags": n, "gpu_device_ms": g.gen_ms, "gpu_wall_s": wall_g, "host_openmp_wall_s": wall_h,
                          "reference_wall_s_per_100k": wall_r, "reference_dags_per_s": (n // 10) / wall_r,
                          "gpu_dags_per_s_device": n / (g.gen_ms / 1e3), "bit_identical_gpu_vs_host": same,
                          "bit_identical_host_vs_reference_100k": same_ref}
    g.close()
    h.close()

    # ---------------------------------------------------------------- K4
    k4 = []
    for count in (1000, 100_000):
        c = _lib.Corpus(count, seed=1)
        b = c.batch()
        (summ, *_), wall = timed(lambda: _lib.validate(b, 148, 10, "1/2", 1, seed=1))
        row = {"dags": count, "samples": 10, "gpu_wall_s": wall, "gpu_summary": summ}
        if count <= 1000 or ref.kind == "ref":
            rs, rwall = timed(lambda: bindings.ref_run_validation(count, 148, 10, "1/2", 1, seed=1))
            row.update({"reference_wall_s": rwall, "reference_summary": rs,
                        "identical": rs == {k: summ[k] for k in rs}})
        k4.append(row)
        c.close()
    out["k4_run_validation"] = k4

    # ---------------------------------------------------------------- K6
    c = _lib.Corpus(10_000, seed=3)
    b = c.batch()
    runs = 10
    (st, num, den, _), wall = timed(lambda: simulator.simulate_greedy_batch(b, 148, runs=runs, policy="random",
                                                                            policy_seed=5))
    rc = ref.corpus(b)
    (rst, rmk), rwall = timed(lambda: bindings.ref_sim_greedy(rc, 148, runs, policy="random", policy_seed=5))
    same = bool(np.array_equal(st, rst) and np.array_equal(num, rmk[:, :, 0]) and np.array_equal(den, rmk[:, :, 1]))
    out["k6_simulate_greedy"] = {"dags": 10_000, "runs": runs, "gpu_wall_s": wall, "reference_wall_s": rwall,
                                 "identical": same}
    c.close()

    # ---------------------------------------------------------------- run_experiment (Fig. 4: M sweep)
    # 50 DAGs per point: at >= 100 the reference's exact 128-bit mean
    # overflows; the GPU sweep also runs the paper's 1000
    values = [8, 16, 32, 64, 128, 256]
    rows, wall = timed(lambda: experiment.run_experiment("M", values, {"seed": 1}, 148, 50))
    csv_gpu = experiment.write_csv(rows)
    row = {"sweep": "M", "values": values, "corpus_size": 50, "gpu_wall_s": wall}
    if ref.kind == "ref":
        csv_ref, rwall = timed(lambda: bindings.ref_run_experiment("M", values, 148, 50, seed=1))
        row.update({"reference_wall_s": rwall, "identical_csv": csv_ref == csv_gpu})
    _, wall1k = timed(lambda: experiment.run_experiment("M", values, {"seed": 1}, 148, 1000))
    row["gpu_wall_s_1000_per_point"] = wall1k
    out["run_experiment"] = row

    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out" if len(sys.argv) < 2 else sys.argv[1], "r01_aux_bench.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
