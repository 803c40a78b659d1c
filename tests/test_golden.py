"""Oracle against the cited fixtures in tests/golden/ (no GPU).

Every expected value in tests/golden/*.json was typed in from the passage it cites
(PAPER.md, SPEC.md worked examples, or the Random123 known-answer vectors); none comes
from the CUDA path or from the oracle.  This file only turns the fixture into oracle
calls and compares.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).parent / "golden"


def load(name):
    with open(GOLDEN / name) as f:
        doc = json.load(f)
    assert doc.get("citation"), f"{name} has no citation"
    return doc


def _ray(r):
    return np.array([np.inf if v == "inf" else v for v in r], np.float32)


def _logit(p):
    return math.log(p / (1 - p))


def test_golden_fixtures_all_cited():
    files = sorted(GOLDEN.glob("*.json"))
    assert len(files) >= 8
    for f in files:
        load(f.name)


def test_golden_hash_index(orc):          # P1
    for c in load("hash_index.json")["cases"]:
        assert orc.corner_index(1024, 0, c["log2T"], *c["cell"]) == c["index"], c


def test_golden_level_resolutions(orc):   # P2
    for c in load("level_resolutions.json")["cases"]:
        g = orc.Grid(c["L"], c["log2T"])
        assert list(g.res) == c["res"]
        assert g.n_entries == c["entries"]
        if "dense" in c:
            assert list(g.dense) == c["dense"]


def test_golden_network_size(orc):        # P4
    d = load("network_size.json")
    g = orc.Grid(d["L"], d["log2T"], F=d["F"])
    assert round(g.n_entries * d["F"] * d["bytes_per_feature"] / 1e6, 1) == d["printed_MB"]


def test_golden_slab_interval(orc):       # P6
    d = load("slab_interval.json")
    lo, hi = np.array(d["box"]["lo"], np.float32), np.array(d["box"]["hi"], np.float32)
    for c in d["cases"]:
        h, te, tx, *_ = orc.slab(_ray(c["ray"]), lo, hi)
        assert bool(h) == c["hit"], c
        if c["hit"]:
            assert (te, tx) == tuple(c["interval"]), c


def test_golden_segment_sampling(orc):    # P9
    for c in load("segment_sampling.json")["cases"]:
        pts = orc.segment_points(_ray(c["ray"]), c["t0"], c["t1"], c["n"], np.array(c["dom_min"], np.float32),
                                 c["dom_inv"])
        np.testing.assert_array_equal(pts, np.array(c["points"], np.float32))


def test_golden_losses(orc):              # P12
    cases = {c["name"]: c for c in load("losses.json")["cases"]}
    big = 1e3                                        # sigmoid(1e3) == 1 in double
    c = cases["BCE(0.5, 1) = ln 2"]
    _, terms, _ = orc.sample_loss(np.array([_logit(c["pred_vis"]), 0, 0, 0, 0, 0, 0, 0]),
                                  np.array([c["gt_vis"], 0, 0, 0, 0, 0, 0, 0, 0], float))
    assert abs(terms[0] - c["value"]) < 1e-15
    c = cases["L1(0.25, 0.75) = 0.5"]
    _, terms, _ = orc.sample_loss(np.array([-30, _logit(c["pred_t"]), 0, 0, 1, 0, 0, 0]),
                                  np.array([0, c["gt_t"], 0, 0, 1, 0.5, 0.5, 0.5, 0], float))
    assert abs(terms[1] - c["value"]) < 1e-12
    c = cases["relL2((1,1,1),(0,0,0)) = 1/1.01"]
    _, terms, _ = orc.sample_loss(np.array([-30, 0, 0, 0, 1, big, big, big]),
                                  np.array([0, 0.5, 0, 0, 1] + [c["gt_albedo"]] * 3 + [0], float))
    assert abs(terms[3] - c["value"]) < 1e-12
    c = cases["weighted sum of (0.1, 0.2, 0.3, 0.4) = 1.3"]
    v, dd, nn, aa = c["terms"]
    a = 0.6
    y = a - math.sqrt(aa * (a * a + 0.01))                   # (a - y)^2 / (a^2 + 0.01) = aa
    z = np.array([math.log(math.expm1(v)), 0.0, nn, nn, nn, _logit(a), _logit(a), _logit(a)])
    gt = np.array([0, 0.5 - dd, 0, 0, 0, y, y, y, 0], float)
    L, terms, _ = orc.sample_loss(z, gt)
    np.testing.assert_allclose(terms, c["terms"], atol=1e-12)
    assert abs(L - c["total"]) < 1e-12
    c = cases["gating: miss -> only 2 * BCE"]
    L, terms, _ = orc.sample_loss(np.array([_logit(c["pred_vis"]), 7, -3, 2, 9, -4, 5, 1]),
                                  np.array([c["gt_vis"], 0.1, 1, 0, 0, 0.3, 0.3, 0.3, 0], float))
    assert abs(L - c["total"]) < 1e-15 and terms[1] == terms[2] == terms[3] == 0.0


def test_golden_triangle(orc):            # P16
    for c in load("triangle.json")["cases"]:
        h, t, *_ = orc.triangle_hit(c["o"], c["d"], *c["tri"])
        assert h == c["hit"], c
        if c["hit"]:
            assert t == pytest.approx(c["t"], abs=1e-15)


def test_golden_philox_kat(orc):          # P18
    for c in load("philox_kat.json")["cases"]:
        out = orc.philox4x32_10([int(x, 16) for x in c["ctr"]], [int(x, 16) for x in c["key"]])
        assert [int(x) for x in out] == [int(x, 16) for x in c["out"]]
