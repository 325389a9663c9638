"""GPU run_validation (K4) against the reference's own run_validation
(tests/golden/validation.json, made by oracle/_ref): same violation counts
and bit-identical mean tightness doubles (same RNG streams, exact rational
makespans, the reference's summation order)."""
import json
import os

import pytest

from paper_2602_20826_b200 import _lib
from tests import helpers

pytestmark = pytest.mark.gpu


def _cases():
    with open(os.path.join(helpers.GOLDEN, "validation.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"M{c['sm_count']}_S{c['samples']}")
def test_validation_matches_reference(case):
    cfg = case["config"]
    corpus = _lib.Corpus(case["corpus_size"], **cfg)
    summary, st, viol, tw, ts = _lib.validate(corpus.batch(), case["sm_count"], case["samples"],
                                              case["scale_min"], case["scale_max"], seed=cfg.get("seed", 1))
    want = case["summary"]
    assert (st == 0).all()
    assert summary["tasks"] == want["tasks"] and summary["runs"] == want["runs"]
    assert summary["violations"] == want["violations"] == 0  # Theorem 1 holds
    assert summary["mean_tightness_worst"].hex() == want["mean_tightness_worst"]
    assert summary["mean_tightness_scaled"].hex() == want["mean_tightness_scaled"]
    assert (tw == 1.0).all() and (ts <= 1.0).all()


def test_validation_rejects_bad_scales():
    corpus = _lib.Corpus(4, seed=1)
    with pytest.raises(_lib.DagschedError):
        _lib.validate(corpus.batch(), 8, 3, "3/4", "1/2", seed=1)
    with pytest.raises(_lib.DagschedError):
        _lib.validate(corpus.batch(), 8, 3, 0, 1, seed=1)


@pytest.mark.parametrize("cfg", [dict(depth_min=16, depth_max=26, max_width=32, seed=900),
                                 dict(depth_min=26, depth_max=34, max_width=48, seed=901)],
                         ids=["p32", "p48"])
def test_validation_big_dags_match_reference_live(cfg):
    """run_validation over DAGs of ~190-940 nodes (K1's k1_big classes in
    detail mode, then K4) against the reference's run_validation on the same
    generated corpus, computed live by oracle/_ref."""
    from oracle import bindings
    n, M, S = 12, 32, 4
    want = bindings.ref_run_validation(n, M, S, "1/2", 1, **cfg)
    corpus = _lib.Corpus(n, **cfg)
    assert int(corpus.batch().sizes().max()) > (256 if cfg["max_width"] == 32 else 512)
    summary, st, viol, tw, ts = _lib.validate(corpus.batch(), M, S, "1/2", 1, seed=cfg["seed"])
    assert summary["tasks"] == want["tasks"] and summary["runs"] == want["runs"]
    assert summary["violations"] == want["violations"] == 0
    assert summary["mean_tightness_worst"] == want["mean_tightness_worst"]
    assert summary["mean_tightness_scaled"] == want["mean_tightness_scaled"]
