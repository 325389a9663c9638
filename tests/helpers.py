"""Shared test helpers: golden-fixture loading and comparisons."""
from __future__ import annotations

import gzip
import json
import os
from fractions import Fraction

import numpy as np

from paper_2602_20826_b200.batch import from_arrays, pack

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixtures():
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        return json.load(f)["cases"]


def fixture_raw_batch(case):
    """Pack a fixture exactly as tests/golden/make_golden.py fed the reference."""
    nodes = sorted(((int(i), Fraction(l)) for i, l in case["nodes"]), key=lambda t: t[0])
    ids = [i for i, _ in nodes]
    idx = {i: k for k, i in enumerate(ids)}
    words = [(idx.get(u, len(ids)) << 16) | idx.get(v, len(ids)) for u, v in case["edges"]]
    return from_arrays([0, len(nodes)], [0, len(words)], [l.numerator for _, l in nodes],
                       [l.denominator for _, l in nodes], words)


def rename_scheme(j, mapping):
    """write_scheme JSON with every entity's origin mapped through `mapping`
    (e.g. node id -> local index, to compare with a checker that names
    entities by index)."""
    def name(s):
        o, sep, rest = s.partition(":")
        return str(mapping[int(o)]) + sep + rest
    j = json.loads(json.dumps(j))
    for g in j["groups"]:
        g["bottleneck"] = name(g["bottleneck"])
        for m in g["members"] + g["launches"]:
            m["entity"] = name(m["entity"])
    for s in j["segmentations"]:
        for k in ("source", "parallel", "residual"):
            s[k] = name(s[k])
    j["extra_deps"] = [[name(a), name(b)] for a, b in j["extra_deps"]]
    for e in j["entities"]:
        e["id"] = name(e["id"])
        e["preds"] = [name(p) for p in e["preds"]]
    return j


def id_to_rank(case):
    ids = sorted(int(i) for i, _ in case["nodes"])
    return {i: k for k, i in enumerate(ids)}


def min_load_arg(case):
    """The device's DagTask::make floor for a fixture: its min_load when the
    golden was made with one other than t_min (None = t_min)."""
    return 1 if case.get("min_load") == "1" else None


def fixture_batch(case):
    """Pack a fixture through the product packer (id-level validation included)."""
    return pack([([(int(i), Fraction(l)) for i, l in case["nodes"]], [tuple(e) for e in case["edges"]])])


def corpus(name="corpus_default.npz", tag="default"):
    z = np.load(os.path.join(GOLDEN, name))
    b = from_arrays(z[f"{tag}__node_off"], z[f"{tag}__edge_off"], z[f"{tag}__load_num"],
                    z[f"{tag}__load_den"], z[f"{tag}__edges"])
    res = {}
    for k in z.files:
        if k.startswith(f"{tag}__status_M"):
            M = int(k.split("_M")[1])
            res[M] = (z[k], z[f"{tag}__bounds_M{M}"])
    cfg = json.loads(bytes(z[f"{tag}__config"]).decode())
    return b, res, cfg


def schemes():
    with gzip.open(os.path.join(GOLDEN, "schemes.jsonl.gz"), "rt") as f:
        for line in f:
            yield json.loads(line)


def normalise_scheme(j):
    """Order-insensitive view of write_scheme JSON (nlohmann sorts keys)."""
    return json.loads(json.dumps(j, sort_keys=True))
