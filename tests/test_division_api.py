"""build_blocks / local_paths / build_groups / scale_parallelism /
parallel_candidates (division.cpp:10-126, scheduler.cpp:99-146) against the
reference.

tests/cpp/division_dump.cpp is compiled twice from one source: against the
reference's own headers and library (oracle/_ref/ref_division_dump, which
made tests/golden/division.json.gz — tests/golden/make_golden.py) and against
this repo's kept API (api_division_dump). 353 cases: the SPEC's known answers
(Fig. 2 at M = 3..148, chain, diamond, fans, the 4,2,2 apportion) and
generated corpora (default, wide, heavy) at M in {3, 4, 8, 32, 148}.

CPU: the host-side functions (build_blocks, local_paths, scale_parallelism,
parallel_candidates over the reference's groups) equal the reference's.
GPU: build_groups (the device's division phase) equals the reference's, and
so do the device's per-node outputs of ds_schedule_batch (node_block,
node_div_group) on the same DAGs.
"""
import gzip
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2602_20826_b200.batch import pack

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_20826_b200", "_lib")
DUMP = os.path.join(LIB, "api_division_dump")
GOLDEN = os.path.join(ROOT, "tests", "golden", "division.json.gz")


@pytest.fixture(scope="module")
def golden():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)["cases"]


def _groups_file(golden, path):
    with open(path, "w") as f:
        for c, case in enumerate(golden):
            for g, grp in enumerate(case["groups"]):
                f.write(f"G {c} {g} " + " ".join(map(str, grp)) + "\n")


def test_spec_known_answers(golden):
    """SPEC.md:198-218, 270-279 as the reference computed them."""
    by = {(c["name"], c["sm_count"]): c for c in golden}
    f6 = by[("fig2", 6)]
    assert [b["members"] for b in f6["blocks"]] == [[1, 3, 4], [2, 5, 6], [7]]
    assert [b["paths"] for b in f6["blocks"][:2]] == [[[1, 3], [1, 4]], [[2], [5], [6]]]
    assert f6["groups"] == [[1], [3, 4], [2, 5, 6], [7]]
    assert f6["scale"][2] == [[2, 3], [5, 2], [6, 1]]           # loads 4,2,2 on M=6 -> 3,2,1
    assert f6["cands"][1][0] == [2]                              # para(pi_2) = {v2}
    assert by[("chain3", 4)]["groups"] == [[10], [11], [12]]
    d = by[("diamond_1_5_2_1", 4)]
    assert [b["members"] for b in d["blocks"]] == [[0, 1, 2], [3]]
    assert d["groups"] == [[0], [1], [2], [3]]                   # Rule 2 collapse on a (m^max 5 >= 4)


@pytest.mark.skipif(not os.path.exists(DUMP), reason="api_division_dump not built (make cppapi)")
def test_host_division_helpers_match_reference(golden, tmp_path):
    gf = tmp_path / "groups.txt"
    _groups_file(golden, gf)
    r = subprocess.run([DUMP, "--host-only", str(gf)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)["cases"]
    assert len(got) == len(golden)
    for g, want in zip(got, golden):
        want = {k: v for k, v in want.items() if k != "groups"}
        assert g == want, (g["name"], g["sm_count"])


@pytest.mark.gpu
def test_build_groups_on_device_matches_reference(golden):
    r = subprocess.run([DUMP], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)["cases"]
    assert len(got) == len(golden)
    for g, want in zip(got, golden):
        assert g == want, (g["name"], g["sm_count"])


@pytest.mark.gpu
def test_device_node_block_and_div_group_match_reference(golden):
    """ds_schedule_batch's node_block / node_div_group per node (rank space)
    against the reference's build_blocks / build_groups."""
    from oracle import bindings
    from paper_2602_20826_b200 import scheme

    corpora = {"default_seed": dict(seed=1, count=60), "wide_seed": dict(seed=300, count=20, max_width=24,
                                                                          depth_min=6, depth_max=10, avg_load=40),
               "heavy_seed": dict(seed=100, count=20, avg_load=200)}
    ref = bindings.Checker("ref")
    by = {(c["name"], c["sm_count"]): c for c in golden}
    checked = 0
    for prefix, cfg in corpora.items():
        cfg = dict(cfg)
        count, seed = cfg.pop("count"), cfg["seed"]
        b = ref.generate(count, **cfg).pack()
        for M in sorted({m for (n, m) in by if n.startswith(prefix)}):
            schemes, st = scheme.schedule_batch(b, M)
            for d in range(count):
                want = by[(f"{prefix}{seed + d}", M)]
                s = schemes[d]
                assert s is not None and st[d] == 0
                nb = np.full(len(s.node_block), -1)
                for k, blk in enumerate(want["blocks"]):
                    nb[blk["members"]] = k  # generated tasks: node id = local index
                assert list(nb) == s.node_block, (prefix, d, M)
                ndg = np.full(len(s.node_div_group), -1)
                for k, grp in enumerate(want["groups"]):
                    ndg[grp] = k
                assert list(ndg) == s.node_div_group, (prefix, d, M)
                assert s.n_div_groups == len(want["groups"])
                checked += 1
    assert checked == 60 * 4 + 20 * 3 + 20 * 2


REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_division_dump")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_DUMP), reason="oracle/_ref not built (make ref)")
def test_big_dags_division_match_reference():
    """DAGs of ~190-940 nodes (the device's k1_big size classes behind
    build_groups): blocks, local paths, groups, scaling and candidates from
    the kept API equal the reference's own build of the same program."""
    got = subprocess.run([DUMP, "--big"], capture_output=True, text=True, timeout=600)
    want = subprocess.run([REF_DUMP, "--big"], capture_output=True, text=True, timeout=600)
    assert got.returncode == 0, got.stderr[-2000:]
    assert want.returncode == 0, want.stderr[-2000:]
    g, w = json.loads(got.stdout)["cases"], json.loads(want.stdout)["cases"]
    assert len(g) == len(w) == 24
    assert max(len(sum(c["groups"], [])) for c in w) > 512  # the W = 16 class is covered
    for a, b in zip(g, w):
        assert a == b, (a["name"], a["sm_count"])
