"""Sweep driver over the GPU batch boundary — the reference's run_experiment /
write_csv (experiment.cpp:81-161) with evaluate_corpus on the device.

Per sweep value a fresh corpus is generated on the host (bit-identical to
generate_corpus), all bounds come from one K1 launch, and the per-task
normalised bounds are averaged exactly. The reference accumulates that mean
in 128-bit rationals (and throws std::overflow_error when the sum's
denominator outgrows them); here Python's unbounded Fractions hold it, so the
CSV equals the reference's wherever the reference completes, and still
exists where it would not.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from . import _abi, _lib

METHODS = ("proposed", "greedy", "greedy_unaware", "graham_para")


def format_fixed(q: Fraction, digits: int) -> str:
    """rational.cpp:93-112: fixed point, half away from zero."""
    scale = 10 ** digits
    s = q * scale
    num, den = s.numerator, s.denominator
    whole = abs(num) // den * (1 if num >= 0 else -1)
    rem = abs(num - whole * den)
    if rem * 2 >= den:
        whole += -1 if num < 0 else 1
    neg = whole < 0
    whole = abs(whole)
    units, frac = str(whole // scale), str(whole % scale)
    if digits == 0:
        return ("-" if neg else "") + units
    return ("-" if neg else "") + units + "." + frac.rjust(digits, "0")


def run_experiment(sweep: str, values, base: dict, sm_count: int, corpus_size: int,
                   methods=METHODS, normalize_to: str = "greedy_unaware", t_min=1, device: int = 0):
    """-> list of row dicts (ResultRow fields, experiment.hpp:35-44)."""
    if not values:
        raise ValueError("no sweep values")
    if corpus_size < 1:
        raise ValueError("corpus_size must be >= 1")
    cols = list(methods) + ([normalize_to] if normalize_to not in methods else [])
    mask = 0
    for m in cols:
        mask |= 1 << METHODS.index(m)
    rows = []
    for value in values:
        cfg = dict(base)
        M = sm_count
        if sweep == "M":
            M = int(value)
        elif sweep == "P":
            cfg["max_width"] = int(value)
        elif sweep == "V":
            cfg["depth_min"] = cfg["depth_max"] = int(value)
        else:
            raise ValueError(sweep)
        corpus = _lib.Corpus(corpus_size, t_min=t_min, **cfg)
        st, b, _ = _lib.analyze(corpus.batch(), M, t_min, mask, device)
        if (st != _abi.DS_OK).any():
            raise RuntimeError(f"analysis failed for {int((st != 0).sum())} DAGs "
                               f"(first status {_abi.STATUS_NAMES[int(st[st != 0][0])]})")
        bound = {m: [Fraction(int(b[i, 2 * METHODS.index(m)]), int(b[i, 2 * METHODS.index(m) + 1]))
                     for i in range(corpus_size)] for m in cols}
        ref = bound[normalize_to]
        for m in methods:
            norms = [x / r for x, r in zip(bound[m], ref)]
            mean = sum(norms, Fraction(0)) / corpus_size
            mean_d = float(mean)  # to_double
            var = 0.0
            for q in norms:  # the reference's order of double accumulation
                d = float(q) - mean_d
                var += d * d
            var /= corpus_size
            rows.append({"sweep_var": sweep, "sweep_value": int(value), "method": m, "mean_norm": mean,
                         "std_norm": math.sqrt(var), "mean_abs": sum(bound[m], Fraction(0)) / corpus_size,
                         "n": corpus_size, "seed": int(cfg.get("seed", 1))})
    return rows


def write_csv(rows) -> str:
    """experiment.cpp:152-161 byte for byte."""
    out = ["sweep_var,sweep_value,method,mean_norm,std_norm,mean_abs,n,seed\n"]
    for r in rows:
        out.append(f"{r['sweep_var']},{r['sweep_value']},{r['method']},{format_fixed(r['mean_norm'], 6)},"
                   f"{r['std_norm']:.6f},{format_fixed(r['mean_abs'], 6)},{r['n']},{r['seed']}\n")
    return "".join(out)


# ------------------------------------------------------------ run_benchmarks
def run_benchmarks(fixture_paths, sm_counts, avg_loads, greedy_runs: int, seed: int, device: int = 0):
    """run_benchmarks (experiment.cpp:242-291) -> list of BenchCell dicts.

    Per fixture (unit loads scaled to each average) and M: the proposed bound
    and schedule (K1, schedule-detail mode), the greedy bound (K1), the
    simulated schedule makespan (simulate_scheme, worst case), and
    `greedy_runs` random-policy greedy simulations (K6, policy seeds seed + r)
    summarised in the reference's accumulation order."""
    import os

    from . import scheme as S
    from . import simulator as SIM
    from . import task_io
    from .batch import pack

    if greedy_runs < 1:
        raise ValueError("greedy_runs must be >= 1")
    variants = []  # (fixture name, avg, Task)
    for path in fixture_paths:
        base = task_io.read_task_file(path)
        name = os.path.splitext(os.path.basename(path))[0]
        for avg in avg_loads:
            nodes = [(i, l * Fraction(int(avg))) for i, l in base.nodes]
            variants.append((name, int(avg), task_io.make_task(nodes, base.edges)))
    batch = pack([t.as_pack() for _, _, t in variants])
    per_m = {}
    for M in sm_counts:
        M = int(M)
        st, bounds, _ = _lib.analyze(batch, M, 1, _abi.DS_M_PROPOSED | _abi.DS_M_GREEDY, device)
        schemes, sst = S.schedule_batch(batch, M, 1, device)
        gst, gnum, gden, _ = SIM.simulate_greedy_batch(batch, M, greedy_runs, "random", seed, None, 1,
                                                      device=device)
        per_m[M] = (st, bounds, schemes, sst, gst, gnum, gden)
    cells = []
    for k, (name, avg, task) in enumerate(variants):
        for M in sm_counts:
            M = int(M)
            st, bounds, schemes, sst, gst, gnum, gden = per_m[M]
            for code in (int(st[k]), int(sst[k]), *(int(x) for x in gst[k])):
                if code != _abi.DS_OK:
                    raise _lib.DagschedError(code, f"benchmark {name} avg {avg} M {M} failed")
            pb = Fraction(int(bounds[k, 0]), int(bounds[k, 1]))
            gb = Fraction(int(bounds[k, 2]), int(bounds[k, 3]))
            ps = SIM.simulate_scheme(schemes[k], ids=task.ids).makespan
            s = sq = mx = 0.0
            for r in range(greedy_runs):
                mk = SIM.to_double(Fraction(int(gnum[k, r]), int(gden[k, r])))
                s += mk
                sq += mk * mk
                mx = max(mx, mk)
            avg_v = s / greedy_runs
            cells.append({"fixture": name, "sm_count": M, "avg_load": avg, "proposed_bound": pb,
                          "greedy_bound": gb, "proposed_sim": ps, "greedy_sim_max": mx,
                          "greedy_sim_avg": avg_v,
                          "greedy_sim_std": math.sqrt(max(0.0, sq / greedy_runs - avg_v * avg_v))})
    return cells


def write_bench_table(cells) -> str:
    """write_bench_table (experiment.cpp:293-307) byte for byte."""
    out = ["fixture,M,avg_load,proposed_bound,greedy_bound,proposed_sim,greedy_sim_max,greedy_sim_avg,"
           "greedy_sim_std\n"]
    for c in cells:
        out.append(f"{c['fixture']},{c['sm_count']},{c['avg_load']},{format_fixed(c['proposed_bound'], 4)},"
                   f"{format_fixed(c['greedy_bound'], 4)},{format_fixed(c['proposed_sim'], 4)},"
                   f"{c['greedy_sim_max']:.4f},{c['greedy_sim_avg']:.4f},{c['greedy_sim_std']:.4f}\n")
    return "".join(out)
