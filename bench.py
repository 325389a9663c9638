#!/usr/bin/env python
"""Benchmark: batched makespan-bound analysis (config C5) on B200.

One step = one pass of the K1 analysis kernel over this rank's 1M-DAG shard
(generate_corpus(GenConfig{}, seed = 1 + rank * 1M, 1M), M = 148, t_min = 1,
methods proposed / greedy / greedy_unaware / graham_para + lower_bound),
inputs resident in HBM. Ranks are independent shards (no collective on the
data path: DAGs are independent), so scaling is weak: N GPUs analyse N x 1M
DAGs. ``value`` = all ranks' DAGs / max-over-ranks device time.

e2e: the same metric through the public C-ABI with pinned HOST buffers —
ds_analyze_batch16 (the compact wire form: 16-bit loads and edges, 199 B per
C5 DAG) when the corpus fits it, else ds_analyze_batch; --wire forces one
(tri: ds_analyze_batch_tri, each DAG's adjacency as a bit matrix, 98 B per
DAG — half the PCIe bytes, but the pass is GPU-bound and its device
expansion costs more than the copy it saves: 147 vs 181 M DAGs/s). H2D of the packed
DAGs and D2H of statuses/bounds are inside the timed region every step.

--impl reference: the reference's own CPU implementation of the path —
generate_corpus + evaluate_corpus (experiment.cpp:52-79) + lower_bound from
the reference sources compiled in oracle/_ref — on all host cores, on a
bounded sample of the same workload; the product library is never loaded.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DAG bounds/sec (batched makespan-bound analysis, C5)"
UNIT = "DAGs/s"
N_PER_GPU = 1_000_000
SM_COUNT = 148


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload(n, seed):
    return {"workload": "C5: batched bound analysis of generate_corpus(GenConfig{} [depth 5-8, P=8, "
                        "avg load 20, jitter 0.5, density 0.2, integer loads], seed=%d+rank*%d, %d DAGs "
                        "per GPU); M=148, t_min=1; 4 methods + lower bound" % (seed, n, n),
            "n_dags_per_gpu": n, "sm_count": SM_COUNT, "t_min": 1,
            "l2": "no flush: per-step inputs (~0.6 GB) exceed the 126 MB L2"}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class Clocks:
    """SM clock and throttle-reason sampling during the timed region
    (B200_PROFILING.md): NVML every 5 ms from a thread (the timed region is
    ~0.2 s), else `nvidia-smi -lms 200`."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits (nvml.h: nvmlClocksEventReason*)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        self.index = index
        self.p = None
        self.nvml = None
        self.samples = []
        self.mx = None

    def _poll(self):
        import pynvml as N
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(sm), int(rs)))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            import threading

            import pynvml as N
            N.nvmlInit()
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.stop = threading.Event()
            self.nvml = threading.Thread(target=self._poll, daemon=True)
            self.nvml.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.nvml is not None:
            self.stop.set()
            self.nvml.join(timeout=2)
        if self.p:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], self.mx, set()
        for clk, bits in self.samples:
            sm.append(clk)
            for name, b in self.BITS.items():
                if bits & b:
                    reasons.add(name)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml 5 ms" if self.samples else "nvidia-smi 200 ms"}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_summary():
    """profiles/k1_ncu_summary.json: per-kernel figures of the latest
    `ncu --set full` capture of this command (dram bytes, instructions)."""
    p = os.path.join(ROOT, "profiles", "k1_ncu_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def pass_alg_bytes(n, N):
    """SURVEY.md §8(d) algorithmic bytes of one analysis pass: per DAG a 16 B
    header + per node (8 B int64 load numerator + 8 B u64 predecessor mask)
    in, 5 bounds x 16 B + per node 2 B (group index, quota) + 4 B status out
    = 100 + 18 n bytes. n DAGs, N nodes in the batch."""
    return 100 * n + 18 * N


def host_chunks(n: int) -> int:
    """How many chunks analyze_host (capi.cu) streams an n-DAG host batch in."""
    k = int(os.environ.get("DS_CHUNKS", "0") or 0)
    weights = [1] * (k if 1 <= k <= 64 else 5)
    wsum, bounds, acc = sum(weights), [0], 0
    for w in weights:
        acc += w
        hi = min(n, -(-n * acc // wsum))
        if hi - bounds[-1] >= 1 << 14 or (hi == n and hi > bounds[-1]):
            bounds.append(hi)
    return max(1, len(bounds) - 1)


def cpu_baseline_run(batch, kind_pref="ref", target_s=10.0, min_dags=4000, max_dags=1_000_000, gpu=None):
    """Time the reference CPU path on a bounded sample of the same workload
    (the corpus_bench protocol, corpus_bench.cpp:31-59: warm-up, then a
    1-core serial pass and an OpenMP pass on every host core), at M=148 (the
    headline config) and M=32 (corpus_bench's own platform). With gpu =
    (status, bounds) of the device pass, also count how many of the sampled
    DAGs the device got bit-exact (status and all ten num/den)."""
    from oracle import bindings
    from paper_2602_20826_b200 import _abi

    kind = "ref" if bindings.available("ref") and kind_pref == "ref" else "oracle"
    chk = bindings.Checker(kind)
    n = min(min_dags, batch.n_dags)
    while True:
        c = chk.corpus(batch.slice(0, n))
        st_c, b_c, secs = c.evaluate(SM_COUNT, 1, _abi.DS_M_ALL, parallel=True)
        if secs >= target_s / 4 or n >= min(max_dags, batch.n_dags):
            break
        n = min(max_dags, batch.n_dags, int(n * max(2.0, target_s / max(secs, 1e-3))))
    parity = None
    if gpu is not None:
        st_g, b_g = gpu[0][:n], gpu[1][:n]
        same = (st_g == st_c) & (b_g == b_c).all(1)
        parity = {"dags": int(n), "bit_exact": int(same.sum()), "checker": "oracle/_ref" if kind == "ref" else "oracle"}
    # corpus_bench protocol points on smaller samples (same corpus prefix)
    ns = min(20000, batch.n_dags)
    cs = chk.corpus(batch.slice(0, ns))
    cs.evaluate(SM_COUNT, 1, _abi.DS_M_ALL, parallel=False)  # warm-up (corpus_bench.cpp:43)
    ser = cs.evaluate(SM_COUNT, 1, _abi.DS_M_ALL, parallel=False)[2]
    n32 = min(200000, batch.n_dags)
    c32 = chk.corpus(batch.slice(0, n32))
    par32 = c32.evaluate(32, 1, _abi.DS_M_ALL, parallel=True)[2]
    ser32 = cs.evaluate(32, 1, _abi.DS_M_ALL, parallel=False)[2]
    return {"value": n / secs, "unit": UNIT, "cores": cpu_cores(), "parity_vs_gpu": parity,
            "kind": "reference" if kind == "ref" else "port",
            "sample": f"first {n} DAGs of the rank-0 shard, evaluate_corpus(parallel=true, OpenMP "
                      f"{cpu_cores()} threads) + lower_bound, {secs:.2f} s",
            "protocol": {"M148": {"serial_1core": ns / ser, "parallel": n / secs, "speedup": (n / secs) / (ns / ser)},
                         "M32": {"serial_1core": ns / ser32, "parallel": n32 / par32,
                                 "speedup": (n32 / par32) / (ns / ser32)},
                         "samples": {"serial": ns, "parallel_M148": n, "parallel_M32": n32},
                         "unit": UNIT, "ref": "corpus_bench.cpp:31-59 (serial and OpenMP evaluate_corpus)"},
            "source": "oracle/_ref (reference sources compiled against oracle/shim)" if kind == "ref"
                      else "oracle/src restatement"}


def cpp_api_bench(n_ours=1_000_000, n_ref=100_000, reps=300):
    """The kept C++ API against the reference's, the same program
    (tests/cpp/api_bench.cpp) built against each library: C1's
    (make_fan(8, 20, 1)) analyze() / schedule() latency, and
    evaluate_corpus over generate_corpus(GenConfig{}, n) end to end
    (DagTask packing and Rational results included; generation excluded).
    The reference side runs its own CPU code on the host cores (bounded
    sample); this side runs the GPU path."""
    out = {}
    for name, path, n in (("ours", os.path.join(ROOT, "paper_2602_20826_b200", "_lib", "api_bench"), n_ours),
                          ("reference", os.path.join(ROOT, "oracle", "_ref", "ref_api_bench"), n_ref)):
        if not os.path.exists(path):
            out[name] = {"error": f"{path} not built"}
            continue
        try:
            r = subprocess.run([path, str(n), str(reps)], capture_output=True, text=True, timeout=300)
            out[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-300:]}
        except Exception as e:  # reported, never required
            out[name] = {"error": str(e)}
    out["source"] = "tests/cpp/api_bench.cpp (Makefile api_bench / oracle/Makefile ref_api_bench)"
    out["reference_threads"] = cpu_cores()
    return out


PLATFORM_BLOCKING_US = 3000.0  # longest whole-context preemption observed on this platform (2.87 ms) + margin

MAKESPAN_MAIN = ("dynamic_prio", "graph_prio", "multistream_host", "multistream")
MAKESPAN_OTHER = ("proposed", "proposed_deps", "dynamic_deps", "serial")


def makespan_summary(device, replays=1000, replays_other=200, n_c2=100, n_c2_other=20, unit=1 << 17):
    """First half of the BASELINE metric: measured DAG makespan vs the analysed
    bound on this B200 (M = 148), configs C1 (fork-join), C2 (the first n_c2
    generated DAGs with 20-50 nodes), C3 (Inception-style) and C4 (three
    oversized-kernel DAGs), next to serial-stream and naive multi-stream launch.

    Variants (all on the same K2 TMA node kernel, same SMs):
      dynamic_prio     the schedule on the dynamic engine, precedence edges +
                       group-priority claiming (DS_PLAN_PRIORITY) — the product
      graph_prio       the same plan as a CUDA graph, each kernel node at its
                       group's launch priority (hardware CTA dispatch order) —
                       the product on the graph engine
      proposed         the schedule as a CUDA graph with group barriers
                       (simulate_scheme semantics, the Theorem-1 setting)
      proposed_deps    the schedule's augmented graph (Ē) as a CUDA graph
      dynamic_deps     the augmented graph on the dynamic engine
      serial           one stream, topological order, m = min(m^max, M)
      multistream      original edges, m = min(m^max, M), captured as a graph
      multistream_host the same launched by the host per node on its own
                       stream with events: naive multi-stream launch
    Every replay of a proposed variant is compared with its bound in µs
    (bound units x tau + group latencies, executor.bound_us) — raw counts,
    nothing excluded. Replays >= 1 ms above their DAG's median are also
    counted (`stall_like`) but stay in every statistic."""
    from paper_2602_20826_b200 import _lib, executor as X, scheme, workloads
    from paper_2602_20826_b200.batch import pack

    wl = X.WL_MIX32_TMA
    t_start = time.perf_counter()
    cal = X.calibrate(unit, device=device, workload=wl)
    wall = {"calibrate": time.perf_counter() - t_start, "setup": 0.0, "replays": 0.0}
    M = cal["sm_count"]

    def norm(nodes, edges):
        if isinstance(nodes[0], tuple):
            idx = {i: k for k, (i, _) in enumerate(sorted(nodes))}
            return [l for _, l in sorted(nodes)], [(idx[u], idx[v]) for u, v in edges]
        return list(nodes), list(edges)

    dags = [("C1", "c1", norm(*workloads.c1_fork_join())), ("C3", "c3", norm(*workloads.inception_dag()))]
    dags += [("C4", f"c4_{s}", norm(*workloads.oversized_dag(s, M))) for s in range(3)]
    b = _lib.Corpus(400, seed=1).batch()
    sizes = np.diff(b.node_off.astype(np.int64))
    for d in [d for d in range(b.n_dags) if 20 <= sizes[d] <= 50][:n_c2]:
        n0, n1, e0, e1 = (int(b.node_off[d]), int(b.node_off[d + 1]), int(b.edge_off[d]), int(b.edge_off[d + 1]))
        dags.append(("C2", f"c2_seed{1 + d}", ([int(x) for x in b.load_num[n0:n1]],
                                                [(int(w) >> 16, int(w) & 0xFFFF) for w in b.edges[e0:e1]])))
    schemes, st = scheme.schedule_batch(pack([d for _, _, d in dags]), M, device=device)

    def plan_of(kind, sch, loads, edges):
        if kind in ("dynamic_prio", "graph_prio"):
            return (X.plan_from_scheme(sch, loads, unit, mode=X.PLAN_PRIORITY),
                    X.ENGINE_DYNAMIC if kind == "dynamic_prio" else X.ENGINE_GRAPH)
        if kind in ("proposed", "proposed_deps", "dynamic_deps"):
            mode = X.PLAN_BARRIERS if kind == "proposed" else X.PLAN_DEPS
            return (X.plan_from_scheme(sch, loads, unit, mode=mode),
                    X.ENGINE_DYNAMIC if kind.startswith("dynamic") else X.ENGINE_GRAPH)
        engine = X.ENGINE_STREAMS if kind == "multistream_host" else X.ENGINE_GRAPH
        return X.plan_baseline(kind.replace("_host", ""), loads, edges, M, unit), engine

    proposed_kinds = ("dynamic_prio", "graph_prio", "proposed", "proposed_deps", "dynamic_deps")
    per = {}  # (config, kind) -> list of per-DAG arrays
    ratios, over, over_b, stall_like, launches = {}, {}, {}, {}, 0
    p50 = {}
    contracts = {"checked_replays": 0, "precedence_violations": 0, "sm_overlap_violations": 0}
    c2_seen = 0
    for (cfg, name, (loads, edges)), sch in zip(dags, schemes):
        bus = X.bound_us(sch, cal)
        c2_seen += cfg == "C2"
        for kind in MAKESPAN_MAIN + MAKESPAN_OTHER:
            if kind not in MAKESPAN_MAIN and cfg == "C2" and c2_seen > n_c2_other:
                continue  # the secondary variants run on the first n_c2_other C2 DAGs
            plan, engine = plan_of(kind, sch, loads, edges)
            reps = replays if kind in MAKESPAN_MAIN else replays_other
            t0 = time.perf_counter()
            ex = X.Executor(plan, device=device, workload=wl, engine=engine)
            t1 = time.perf_counter()
            r = ex.run(reps, warmup=3, stamps=False)
            wall["setup"] += t1 - t0
            wall["replays"] += time.perf_counter() - t1
            if kind in ("dynamic_prio", "graph_prio") and (cfg != "C2" or name in ("c2_seed2", "c2_seed3")):
                rs = ex.run(10, warmup=1, stamps=True)  # trace contracts on stamped replays
                for k in range(10):
                    contracts["precedence_violations"] += len(X.check_precedence(plan, rs, k))
                    contracts["sm_overlap_violations"] += X.check_sm_exclusive(plan, rs, k)
                    contracts["checked_replays"] += 1
            ex.close()
            mk = r.makespan_us
            per.setdefault((cfg, kind), []).append(mk)
            p50.setdefault(kind, {})[name] = float(np.median(mk))
            stall_like[kind] = stall_like.get(kind, 0) + int((mk > np.median(mk) + 1000.0).sum())
            if kind in proposed_kinds:
                ratios.setdefault(kind, []).append(mk / bus)
                over[kind] = over.get(kind, 0) + int((mk > bus).sum())
                over_b[kind] = over_b.get(kind, 0) + int((mk > bus + PLATFORM_BLOCKING_US).sum())
            launches += (2 if engine == X.ENGINE_DYNAMIC else len(plan.entities) + 1) * (reps + 3)
    configs = {}
    for (cfg, kind), arrs in per.items():
        allr = np.concatenate(arrs)
        c = configs.setdefault(cfg, {})
        c[kind] = {"dags": len(arrs), "p50_us": float(np.mean([np.median(a) for a in arrs])),  # mean of per-DAG p50
                   "p99_us": float(np.mean([np.percentile(a, 99) for a in arrs])),
                   "max_us": float(allr.max()), "replays": int(allr.size)}
    for cfg, c in configs.items():
        names = [n for g, n, _ in dags if g == cfg]
        c["dynamic_prio_beats_multistream_host_p50"] = int(sum(p50["dynamic_prio"][n] < p50["multistream_host"][n]
                                                               for n in names))
        c["dynamic_prio_beats_multistream_p50"] = int(sum(p50["dynamic_prio"][n] < p50["multistream"][n]
                                                          for n in names))
        c["graph_prio_beats_multistream_host_p50"] = int(sum(p50["graph_prio"][n] < p50["multistream_host"][n]
                                                             for n in names))
        c["graph_prio_beats_multistream_p50"] = int(sum(p50["graph_prio"][n] < p50["multistream"][n]
                                                        for n in names))
    mob = {}
    for k, v in ratios.items():
        v = np.concatenate(v)
        mob[k] = {"p50": float(np.percentile(v, 50)), "p99": float(np.percentile(v, 99)), "max": float(v.max()),
                  "replays": int(v.size)}
    wall["total"] = time.perf_counter() - t_start
    return {"sm_count": M, "node_kernel": "k2_mix_tma (all variants)", "unit_elems": unit,
            "replays": {"main": replays, "other": replays_other, "main_variants": list(MAKESPAN_MAIN),
                        "other_variants_c2_dags": n_c2_other},
            "wall_s": wall,
            "tau_us": cal["tau_us"], "delta_us": cal["delta_us"], "eps_us": cal["eps_us"],
            "configs": configs, "measured_over_bound": mob,
            "replays_over_bound_raw": over, "stall_like_replays": stall_like,
            "platform_blocking": {
                "B_us": PLATFORM_BLOCKING_US,
                "replays_over_bound_plus_B": over_b,
                "rule": "response-time analysis with a blocking term: the Theorem-1 bound assumes a dedicated "
                        "GPU; on this platform the whole context is preempted for 1.5-2.9 ms every 0.3-10 s "
                        "(all 148 SMs stop at once; host-side time-slicing through the VM's GPU proxy), so "
                        "a replay that meets one can exceed the bound by at most B (stalls are >= 0.3 s apart, "
                        "longer than any makespan here)",
                "evidence": "profiles/r02_stall_root.txt, profiles/r01_stall_probe.txt (tools/heartbeat.cu)"},
            "trace_contracts_prio": contracts, "executor_kernel_launches": launches}


CONTENDED_VARIANTS = ("graph_prio", "dynamic_prio", "multistream_host", "multistream")


def makespan_contended(device, sms=(32, 8), replays=200, n_c2=12, unit=1 << 17):
    """The paper's contended regime: the DAG runs inside a green context of M
    SMs (M = 32, 8), scheduled and bounded for that M (calibration inside the
    same partition). Per config the mean over its DAGs of the per-DAG p50 /
    p99 in us, the max over all replays, and the proposed variants' replays
    over the bound counted raw."""
    from paper_2602_20826_b200 import _lib, executor as X, scheme, workloads
    from paper_2602_20826_b200.batch import pack

    wl = X.WL_MIX32_TMA
    t_start = time.perf_counter()
    out = {"replays": replays, "c2_dags": n_c2, "variants": list(CONTENDED_VARIANTS)}
    b = _lib.Corpus(400, seed=1).batch()
    sizes = np.diff(b.node_off.astype(np.int64))
    c2 = []
    for d in [d for d in range(b.n_dags) if 20 <= sizes[d] <= 50][:n_c2]:
        n0, n1, e0, e1 = (int(b.node_off[d]), int(b.node_off[d + 1]), int(b.edge_off[d]), int(b.edge_off[d + 1]))
        c2.append(("C2", ([int(x) for x in b.load_num[n0:n1]],
                          [(int(w) >> 16, int(w) & 0xFFFF) for w in b.edges[e0:e1]])))

    def norm(nodes, edges):
        if isinstance(nodes[0], tuple):
            idx = {i: k for k, (i, _) in enumerate(sorted(nodes))}
            return [l for _, l in sorted(nodes)], [(idx[u], idx[v]) for u, v in edges]
        return list(nodes), list(edges)

    for M in sms:
        cal = X.calibrate(unit, sm_limit=M, device=device, workload=wl)
        dags = [("C1", norm(*workloads.c1_fork_join())), ("C3", norm(*workloads.inception_dag()))]
        dags += [("C4", norm(*workloads.oversized_dag(s, M))) for s in range(3)] + c2
        schemes, _ = scheme.schedule_batch(pack([d for _, d in dags]), M, device=device)
        per, over, ratio = {}, {}, {}
        for (cfg, (loads, edges)), sch in zip(dags, schemes):
            bus = X.bound_us(sch, cal)
            for kind in CONTENDED_VARIANTS:
                if kind.endswith("_prio"):
                    plan = X.plan_from_scheme(sch, loads, unit, mode=X.PLAN_PRIORITY)
                    engine = X.ENGINE_GRAPH if kind == "graph_prio" else X.ENGINE_DYNAMIC
                else:
                    plan = X.plan_baseline(kind.replace("_host", ""), loads, edges, M, unit)
                    engine = X.ENGINE_STREAMS if kind == "multistream_host" else X.ENGINE_GRAPH
                ex = X.Executor(plan, device=device, workload=wl, engine=engine, sm_limit=M)
                mk = ex.run(replays, warmup=3, stamps=False).makespan_us
                ex.close()
                per.setdefault((cfg, kind), []).append(mk)
                if kind.endswith("_prio"):
                    over[kind] = over.get(kind, 0) + int((mk > bus).sum())
                    ratio[kind] = max(ratio.get(kind, 0.0), float((mk / bus).max()))
        cf = {}
        for (cfg, kind), arrs in per.items():
            cf.setdefault(cfg, {})[kind] = {
                "dags": len(arrs), "p50_us": float(np.mean([np.median(a) for a in arrs])),
                "p99_us": float(np.mean([np.percentile(a, 99) for a in arrs])),
                "max_us": float(np.concatenate(arrs).max())}
        out[f"M{M}"] = {"tau_us": cal["tau_us"], "delta_us": cal["delta_us"], "eps_us": cal["eps_us"],
                        "configs": cf, "replays_over_bound_raw": over, "max_measured_over_bound": ratio}
    out["wall_s"] = time.perf_counter() - t_start
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path.

    Runs ONLY oracle/_ref (the reference's proj/src/*.cpp compiled against
    oracle/shim; oracle/Makefile): the corpus comes from the reference's own
    generate_corpus (generator.cpp:98-108, GenConfig{} defaults, seed 1 — the
    first DAGs of this arm's rank-0 shard, bit-identical), and every step
    times evaluate_corpus(parallel=true) (experiment.cpp:52-79, OpenMP on all
    host cores) + lower_bound over it. The product library is never loaded
    on this arm. `config` equals the device arm's; each step is a bounded
    sample of that workload (the first --ref-sample DAGs), declared in
    cpu_baseline.sample."""
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    from oracle import bindings

    if not bindings.available("ref"):
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "oracle/_ref/libdagsched_ref.so not built (make -C oracle ref)"}), flush=True)
        return 0
    M_ALL = 0x1F  # proposed, greedy, greedy_unaware, graham_para + lower (include/dagsched_b200.h)
    chk = bindings.Checker("ref")
    n = args.ref_sample
    t0 = time.perf_counter()
    c = chk.generate(n, seed=1)  # the reference's generate_corpus(GenConfig{}, 1, n)
    gen_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        c.evaluate(SM_COUNT, 1, M_ALL, parallel=True)
    secs = [c.evaluate(SM_COUNT, 1, M_ALL, parallel=True)[2] for _ in range(args.steps)]
    tot = sum(secs)
    value = n * args.steps / tot
    maps = open("/proc/self/maps").read()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64 (exact rationals)",
            "data": "synthetic (reference generator)", "impl": "reference",
            "config": dict(workload(N_PER_GPU, 1), parallelism=f"shards{world}", integer_loads=True),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "reference",
                             "sample": f"first {n} DAGs of the C5 corpus (reference generate_corpus, seed 1) per "
                                       f"step: evaluate_corpus(parallel=true, OpenMP {cpu_cores()} threads) + "
                                       f"lower_bound, M=148, t_min=1; generation {gen_s:.1f} s excluded",
                             "source": "oracle/_ref (reference proj/src compiled against oracle/shim)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "product_library_mapped": "libdagsched_b200" in maps,
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-dags", type=int, default=N_PER_GPU)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--ref-sample", type=int, default=100000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-makespan", action="store_true")
    ap.add_argument("--wire", default="auto", choices=["auto", "tri", "16", "wide"],
                    help="e2e wire form: ds_analyze_batch_tri / ds_analyze_batch16 / ds_analyze_batch")
    ap.add_argument("--makespan-replays", type=int, default=1000)
    ap.add_argument("--makespan-c2", type=int, default=100)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    rank, local_rank, world = env_rank()
    if world > 1 and "OMP_NUM_THREADS" not in os.environ:
        # ranks share the host: cap each rank's OpenMP pool at its share of the cores
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        os.environ["OMP_NUM_THREADS"] = str(max(1, cpu_cores() // local_world))
    import torch

    # DS_BENCH_SHARE_GPU=1 (test knob): every rank on cuda:0 over gloo, so the
    # N > 1 code path can be exercised on a one-GPU box
    share = os.environ.get("DS_BENCH_SHARE_GPU") == "1"
    dev = 0 if share else local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_2602_20826_b200 import _abi, _lib

    n = args.n_dags
    t0 = time.perf_counter()
    # N > 1: each rank generates its shard on its own GPU (K5, bit-identical
    # to generate_corpus) so N ranks do not contend for the host cores
    corpus = _lib.Corpus(n, pinned=True, gpu=world > 1, seed=1 + rank * n)
    gen_s = time.perf_counter() - t0
    batch = corpus.batch()
    integer = batch.integer_loads()

    # ---------------------------------------------------- device-resident leg
    sess = _lib.Session(batch, SM_COUNT, 1, _abi.DS_M_ALL, dev)
    for _ in range(args.warmup):
        sess.run()
    barrier()
    per_kernel = {}
    with Clocks(dev) as clk:
        barrier()
        kms = []
        for _ in range(args.steps):
            kms.append(sess.run())
            for k, v in sess.kernel_times().items():  # events between the step's launches
                per_kernel.setdefault(k, []).append(v)
        barrier()
    dev_ms = max_over_ranks(sum(kms))
    st, bounds, ng = sess.results()
    ok = int((st == 0).sum())
    value = world * n * args.steps / (dev_ms / 1e3)
    # per step: k1_front, k1_mid, k1_back, the n<=256 kernel when such DAGs
    # exist, and the 64- and 128-bit retry kernels (each exits at once when
    # nothing was queued) — one event per launch; the ncu launch list in
    # profiles/ shows the same
    launches_per_step = len(per_kernel)

    # ---------------------------------------------------------------- e2e leg
    # pinned result buffers (the inputs are pinned too: Corpus(pinned=True))
    res_status = torch.zeros(n, dtype=torch.int32, pin_memory=True).numpy()
    res_bounds = torch.zeros((n, 10), dtype=torch.int64, pin_memory=True).numpy()
    res_groups = torch.zeros(n, dtype=torch.int16, pin_memory=True).numpy().view(np.uint16)
    import ctypes as C
    r = _abi.ds_results(res_status.ctypes.data, res_bounds.ctypes.data, res_groups.ctypes.data)
    pl = _lib.platform(SM_COUNT)
    L = _lib.lib()
    # the caller's host arrays in the most compact wire form the batch fits,
    # pinned; the conversion is the caller's packing, outside the timed region
    wire = args.wire
    if wire == "auto":  # measured fastest first: the triangular form (half the 16-bit
        # form's PCIe bytes; k1_fast reads it as is), then the 16-bit one
        wire = "tri" if batch.tri_ok() else "16" if batch.compact16_ok() else "wide"
    pin = lambda n, dt: torch.empty(n, dtype=dt, pin_memory=True).numpy()  # noqa: E731
    if wire == "tri":
        adj_off = batch.tri_words()
        pint = (pin(batch.load_num.shape[0], torch.int16).view(np.uint16),
                pin(int(adj_off[-1]), torch.int32).view(np.uint32))
        load16, adj_off_np, adj = batch.tri(out=pint)
        adj_off = pin(adj_off_np.shape[0], torch.int32).view(np.uint32)
        adj_off[:] = adj_off_np
        cb = batch.as_ctri(load16, adj_off, adj)
        call = lambda: L.ds_analyze_batch_tri(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), dev)  # noqa: E731
        h2d = batch.node_off.nbytes + adj_off.nbytes + load16.nbytes + adj.nbytes
        api = "ds_analyze_batch_tri (triangular bit-matrix wire form, host pinned)"
    elif wire == "16":
        pin16 = (pin(batch.load_num.shape[0], torch.int16).view(np.uint16),
                 pin(batch.edges.shape[0], torch.int16).view(np.uint16))
        load16, edges16 = batch.compact16(out=pin16)
        cb = batch.as_c16(load16, edges16)
        call = lambda: L.ds_analyze_batch16(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), dev)  # noqa: E731
        h2d = batch.node_off.nbytes + batch.edge_off.nbytes + load16.nbytes + edges16.nbytes
        api = "ds_analyze_batch16 (16-bit wire form, host pinned)"
    else:
        cb = batch.as_c()
        call = lambda: L.ds_analyze_batch(C.byref(cb), C.byref(pl), _abi.DS_M_ALL, C.byref(r), dev, None, 0)  # noqa: E731
        h2d = batch.nbytes(with_den=not integer)
        api = "ds_analyze_batch (host pinned)"
    for _ in range(3):  # warm-up: pinned staging, stream pool, first-touch of the result arrays
        _lib.check(call())
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        _lib.check(call())
    barrier()
    my_e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(my_e2e_s)
    per_rank_e2e = [my_e2e_s]
    if dist is not None:
        allv = [None] * world
        dist.all_gather_object(allv, my_e2e_s)
        per_rank_e2e = allv
    e2e_value = world * n * args.e2e_steps / e2e_s
    same = bool(np.array_equal(res_status, st) and np.array_equal(res_bounds, bounds))
    d2h = res_status.nbytes + res_bounds.nbytes + res_groups.nbytes
    chunks = host_chunks(n)

    # ---------------------------------------------------------------- roofline
    # algorithmic bytes of the pass = 100 + 18 n per DAG; the
    # dominant kernel of the step is timed live with CUDA events on its stream
    peak, peak_kind = measured_peak()
    kmean = {k: statistics.mean(v) for k, v in per_kernel.items()}
    dom = max(kmean, key=kmean.get)
    N = int(batch.node_off[-1] - batch.node_off[0])
    alg_bytes = pass_alg_bytes(n, N)
    achieved = alg_bytes / (kmean[dom] / 1e3) / 1e9
    step_ms = statistics.mean(kms)
    ncu = ncu_summary()
    kn = ncu.get("kernels", {})
    traffic_step = (sum(k["dram_bytes_per_dag"] for k in kn.values() if k.get("dram_bytes_per_dag")) * n
                    if kn else None)
    traffic_dom = kn.get(dom, {}).get("dram_bytes_per_dag")
    issue = None
    if kn.get(dom, {}).get("warp_instructions_per_dag") and ncu.get("sm_clock_mhz"):
        peak_ips = 4 * ncu["sm_count"] * ncu["sm_clock_mhz"] * 1e6  # 4 schedulers x 1 warp-instr / clk
        ips = kn[dom]["warp_instructions_per_dag"] * n / (kmean[dom] / 1e3)
        issue = {"achieved": ips, "peak": peak_ips, "unit": "warp-instr/s", "frac": ips / peak_ips,
                 "threads_per_warp_instr": {k: v.get("threads_per_warp_instr") for k, v in kn.items()},
                 "source": "instruction counts per DAG from the ncu capture in profiles/, time live"}
    makespan = None
    if rank == 0 and not args.no_makespan:
        try:
            makespan = makespan_summary(dev, args.makespan_replays, n_c2=args.makespan_c2)
        except Exception as e:  # reported, never required for the headline line
            makespan = {"error": str(e)}
        try:
            makespan["contended"] = makespan_contended(dev)
        except Exception as e:
            makespan["contended"] = {"error": str(e)}

    cpp_api = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpp_api = cpp_api_bench()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_run(batch, gpu=(st, bounds))
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64 (exact rationals)",
            "data": "synthetic (reference generator, bit-identical)",
            "config": dict(workload(n, 1), parallelism=f"shards{world}", integer_loads=integer),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": 1e3 * e2e_s / args.e2e_steps, "api": api,
                    "matches_device_leg": same,
                    "per_rank_dags_per_s": [n * args.e2e_steps / t for t in per_rank_e2e],
                    "pcie_bytes_per_rank_per_step": h2d + d2h},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_step, "peak_source": peak_kind,
                         "kernel": dom, "kernel_ms": kmean[dom],
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "algorithmic_bytes_rule": "SURVEY 8(d): 100 + 18 n B per DAG (n nodes) for the pass, "
                                                   "over the dominant kernel's time",
                         "traffic_scope": "whole step (ncu dram read+write, all K1 kernels, profiles/k1_ncu_summary.json)",
                         "traffic_dominant_kernel": traffic_dom * n if traffic_dom else None,
                         "traffic_over_algorithmic": traffic_step / alg_bytes if traffic_step else None,
                         "issue": issue,
                         "pass": {"kernels_ms": kmean, "step_ms": step_ms, "algorithmic_bytes": alg_bytes,
                                  "achieved_gbs": alg_bytes / (step_ms / 1e3) / 1e9,
                                  "frac": alg_bytes / (step_ms / 1e3) / 1e9 / peak},
                         "note": "integer issue/latency-bound exact-rational greedy per DAG; HBM is not the limiter"},
            "cpu_baseline": cpu,
            "cpp_api": cpp_api,
            "makespan": makespan,
            "clocks": clk.summary(),
            "gpu_launches": launches_per_step * args.steps,
            # per chunk: the session's kernels + the wire form's widening
            # (16-bit: k_widen16; triangular: k_widen_tri_list over the
            # fallback and retry queues)
            "e2e_gpu_launches": chunks * (launches_per_step + {"tri": 2, "16": 1, "wide": 0}[wire]) * args.e2e_steps,
            "dags_ok": ok, "generation_s": gen_s,
            "kernel_ms": {"mean": statistics.mean(kms), "min": min(kms), "max": max(kms)},
        }
        print(json.dumps(line), flush=True)
    sess.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
