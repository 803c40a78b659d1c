"""Pins of the oracle's logic replay (`orc_replay`) and of its (t_enter, id) leaf order.

`orc_replay` is the checker of the exact tier (hit mask, winning leaf, t bits, query count
of the GPU's own z trace; SURVEY §8(c) tier iv), and `leaf_list`'s sort is what every
traversal comparison rests on.  Neither may be trusted because it agrees with itself, so:

* the replay is tied to the double-precision query oracle `orc_query` (a separate
  implementation of P:103/P:161 in double): fed `orc_query`'s own z trace rounded to fp32,
  it must reproduce hit, leaf and query count on every ray whose decisions are not within
  fp32 rounding of a tie;
* hand-built z traces on a hand-built cut, whose answers are derived here from the stop
  rule of C5 (front-to-back walk, query iff t_enter <= t_best: strict `>` terminates; best
  = argmin (t, t_enter, id)) and C13 (z_vis = 0 is a miss), pin termination on equal keys
  and the tie rule;
* the (t_enter, id) order is checked against numpy's lexsort of brute-force slab results,
  on cuts built to produce equal t_enter values.
"""
import numpy as np
import pytest

import synth

INF = np.float32(np.inf)


# ------------------------------------------------------------------ replay vs double query
@pytest.fixture(scope="module")
def tiny_cut():
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny()
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    ctx.build_cut(64)
    return sc, ctx.cut(0)


@pytest.mark.parametrize("mode", [0, 1])
def test_replay_reproduces_double_query_on_its_own_trace(orc, tiny_cut, mode):
    """P:103, P:161 (C5): orc_replay on orc_query's z (cast to fp32) gives orc_query's hit,
    leaf and query count wherever no decision sits within fp32 rounding of a tie."""
    sc, cut = tiny_cut
    g = orc.Grid(8, 14)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=7).reshape(-1, 2)
    layers = synth.random_mlp(64, 2, 64, seed=2)
    rays = np.concatenate([synth.camera_rays(64, 64, (0.0, 0.0, 3.5), vfov_deg=40.0),
                           synth.random_rays(3000, seed=11)], 0)
    cap = 64
    o = orc.query(g, 4, tab, layers, cut["leaf_lo"], cut["leaf_hi"], rays, mode=mode, trace_cap=cap,
                  dom_box=orc.scene_box(sc))
    leaf, te, tx, cnt = orc.leaf_lists(rays, cut["leaf_lo"], cut["leaf_hi"], cap)
    assert cnt.max() < cap                                     # the trace holds every queried leaf
    decided = (o["margin"] >= 1e-5) & (o["tmargin"] >= 1e-4)
    assert decided.mean() > 0.99
    zt = o["z_trace"].astype(np.float32)
    rep = orc.replay(cut["leaf_lo"], cut["leaf_hi"], rays[decided], zt[decided], mode=mode)
    assert rep["missing"] == 0
    assert np.array_equal(rep["hit"], o["hit"][decided])
    assert np.array_equal(rep["leaf"], o["leaf"][decided])
    assert np.array_equal(rep["nq"], o["nq"][decided])
    h = o["hit"][decided] == 1
    assert h.sum() > 300
    # fp32 decode vs double decode of the same z: a few ulp of t (C27)
    assert np.all(np.abs(rep["t"][h] - o["t"][decided][h]) <= 4e-6 * np.abs(o["t"][decided][h]))
    assert np.abs(rep["albedo"][h] - o["albedo"][decided][h]).max() <= 1e-6
    assert np.abs(rep["normal"][h] - o["normal"][decided][h]).max() <= 1e-6
    assert np.all(np.isinf(rep["t"][~h])) and np.all(rep["leaf"][~h] == -1)
    # and every ray not hit queried every leaf it intersects (nothing to terminate on) in R2
    if mode == 0:
        assert np.array_equal(rep["nq"][~h], cnt[decided][~h])


# ------------------------------------------------------------------ hand-built cut and traces
# A ray along +z from the origin; leaf boxes are slabs in z (|x|,|y| <= 1), so every
# t_enter / t_exit is an exact small integer:
#   leaf 0: z in [1, 2]   leaf 1: z in [2, 3]   leaf 2: z in [1, 4]   leaf 3: z in [5, 6]
# (t_enter, id) order: leaf 0 (1), leaf 2 (1), leaf 1 (2), leaf 3 (5).
LO = np.array([[-1, -1, 1], [-1, -1, 2], [-1, -1, 1], [-1, -1, 5]], np.float32)
HI = np.array([[1, 1, 2], [1, 1, 3], [1, 1, 4], [1, 1, 6]], np.float32)
RAY = np.array([[0, 0, 0, 0, 0, 0, 1, np.inf]], np.float32)
ORDER = [0, 2, 1, 3]
HIT, MISS = -5.0, 5.0
FAR, NEAR = 100.0, -100.0      # sigma_f32(+100) = 1 exactly -> t = t_exit; sigma(-100) -> t = t_enter


def _trace(per_leaf):
    """per_leaf: {leaf id: (z_vis, z_t)} -> z trace [1][4][8] in list order (NaN = absent)."""
    zt = np.full((1, 4, 8), np.nan, np.float32)
    for k, lf in enumerate(ORDER):
        if lf in per_leaf:
            zt[0, k, :] = 0.0
            zt[0, k, 0], zt[0, k, 1] = per_leaf[lf]
            zt[0, k, 4] = 1.0
    return zt


def test_hand_cut_list_order(orc):
    leaf, te, tx, cnt = orc.leaf_lists(RAY, LO, HI, 4)
    assert leaf[0].tolist() == ORDER and cnt[0] == 4
    assert te[0].tolist() == [1, 1, 2, 5] and tx[0].tolist() == [2, 4, 3, 6]


def test_sigmoid_saturation_used_by_hand_cases(orc):
    assert orc.sigmoid_f32(FAR) == 1.0
    assert 0.0 < orc.sigmoid_f32(NEAR) < 1e-37     # t = t0 + tiny*(t1-t0) rounds to t0 for t0 >= 1


@pytest.mark.parametrize("case", [
    # 1. leaf 0 hits at its exit t = 2 = t_best; leaf 2 (t_enter 1 <= 2) is queried and misses;
    #    leaf 1 has t_enter == t_best = 2: strict `>` termination -> it IS queried; it hits at
    #    its entry t = 2 (a t tie) with t_enter 2 > 1 -> leaf 0 stays best; leaf 3 (5 > 2) is not.
    ({0: (HIT, FAR), 2: (MISS, 0.0), 1: (HIT, NEAR), 3: (HIT, NEAR)}, 0, (1, 0, 2.0, 3)),
    # 2. ties in t AND t_enter: leaves 0 and 2 both hit at t = 1 = their t_enter -> lower id (0);
    #    leaf 1's t_enter 2 > 1 terminates.
    ({0: (HIT, NEAR), 2: (HIT, NEAR), 1: (HIT, NEAR), 3: (HIT, NEAR)}, 0, (1, 0, 1.0, 2)),
    # 3. the later-queried leaf is nearer: leaf 0 hits at 2, leaf 2 at 1 -> leaf 2 wins; then
    #    leaf 1 (t_enter 2 > 1) terminates.
    ({0: (HIT, FAR), 2: (HIT, NEAR), 1: (HIT, NEAR), 3: (HIT, NEAR)}, 0, (1, 2, 1.0, 2)),
    # 4. z_vis == 0 is sigma = 0.5: a miss (C13); nothing hits -> every leaf queried.
    ({0: (0.0, 0.0), 2: (0.0, 0.0), 1: (0.0, 0.0), 3: (0.0, 0.0)}, 0, (0, -1, np.inf, 4)),
    # 5. only the last leaf hits: t = its exit 6.
    ({0: (MISS, 0.0), 2: (MISS, 0.0), 1: (MISS, 0.0), 3: (HIT, FAR)}, 0, (1, 3, 6.0, 4)),
    # 6. R1 (first confident hit): stops at leaf 0 although leaf 2 is nearer.
    ({0: (HIT, FAR), 2: (HIT, NEAR), 1: (HIT, NEAR), 3: (HIT, NEAR)}, 1, (1, 0, 2.0, 1)),
    # 7. R1 with leading misses.
    ({0: (MISS, 0.0), 2: (MISS, 0.0), 1: (HIT, FAR), 3: (HIT, NEAR)}, 1, (1, 1, 3.0, 3)),
    # 8. leaf 2 hits at its exit 4; leaf 1 (t_enter 2 <= 4) queried, hits at its exit 3 < 4 ->
    #    leaf 1 wins; leaf 3 (t_enter 5 > 3) terminates.
    ({0: (MISS, 0.0), 2: (HIT, FAR), 1: (HIT, FAR), 3: (HIT, NEAR)}, 0, (1, 1, 3.0, 3)),
])
def test_replay_hand_built_traces(orc, case):
    per_leaf, mode, (hit, leaf, t, nq) = case
    rep = orc.replay(LO, HI, RAY, _trace(per_leaf), mode=mode)
    assert rep["missing"] == 0
    assert (int(rep["hit"][0]), int(rep["leaf"][0]), int(rep["nq"][0])) == (hit, leaf, nq)
    assert rep["t"][0] == np.float32(t)


def test_replay_reports_missing_trace_entries(orc):
    # leaf 1 is needed (t_enter 2 <= t_best 2) but absent from the trace -> one missing ray
    rep = orc.replay(LO, HI, RAY, _trace({0: (HIT, FAR), 2: (MISS, 0.0)}))
    assert rep["missing"] == 1


def test_double_query_hand_built_ties(orc):
    """The same stop/tie rules in the double oracle: a zero model (every z = bias) on the
    hand-built cut.  Always-hit at t_enter: leaves 0 and 2 tie in (t, t_enter) -> leaf 0,
    leaf 1 (t_enter 2 > 1) terminates -> 2 queries.  Always-hit at t_exit: leaf 0 at 2,
    leaf 2 at 4, leaf 1 (t_enter 2 == t_best) queried, exit 3 > 2 -> leaf 0, 3 queries."""
    g = orc.Grid(2, 6)
    tab = np.zeros((g.n_entries, 2), np.float16)

    def model(vis, tb):
        b = np.zeros(8, np.float32)
        b[0], b[1], b[4] = vis, tb, 1.0
        return [(np.zeros((4, 12), np.float16), np.zeros(4, np.float32)), (np.zeros((8, 4), np.float16), b)]

    o = orc.query(g, 3, tab, model(-5.0, -200.0), LO, HI, RAY)
    assert (o["hit"][0], o["leaf"][0], o["nq"][0]) == (1, 0, 2) and o["t"][0] == 1.0
    o = orc.query(g, 3, tab, model(-5.0, 200.0), LO, HI, RAY)
    assert (o["hit"][0], o["leaf"][0], o["nq"][0]) == (1, 0, 3) and o["t"][0] == 2.0
    o = orc.query(g, 3, tab, model(0.0, 0.0), LO, HI, RAY)                # tie -> miss everywhere
    assert (o["hit"][0], o["leaf"][0], o["nq"][0]) == (0, -1, 4)


# ------------------------------------------------------------------ (t_enter, id) order vs lexsort
def _tie_heavy_cut(rng, n=40):
    """Boxes whose z faces sit on a coarse lattice (many exactly equal t_enter for rays along
    +-z), plus nested boxes sharing faces, plus random boxes."""
    lo, hi = [], []
    for i in range(n):
        if i % 3 == 0:
            z0 = float(rng.integers(-3, 3)) * 0.25
            lo.append([rng.uniform(-1, 0), rng.uniform(-1, 0), z0])
            hi.append([rng.uniform(0, 1), rng.uniform(0, 1), z0 + 0.25 * float(rng.integers(1, 4))])
        elif i % 3 == 1:
            j = len(lo) - 1
            lo.append([lo[j][0] * 0.5, lo[j][1] * 0.5, lo[j][2]])          # same z face as box j
            hi.append([hi[j][0] * 0.5, hi[j][1] * 0.5, hi[j][2] + 0.25])
        else:
            a = rng.uniform(-1, 0.6, 3)
            lo.append(list(a))
            hi.append(list(a + rng.uniform(0.1, 0.6, 3)))
    return np.asarray(lo, np.float32), np.asarray(hi, np.float32)


def _brute_order(orc, ray, lo, hi):
    ids, te, tx = [], [], []
    for i in range(lo.shape[0]):
        h, _, _, a, b = orc.slab(ray, lo[i], hi[i])
        if h:
            ids.append(i); te.append(a); tx.append(b)
    ids = np.asarray(ids, np.int32)
    te = np.asarray(te, np.float32)
    tx = np.asarray(tx, np.float32)
    o = np.lexsort((ids, te))                                  # primary t_enter, then id
    return ids[o], te[o], tx[o]


def test_leaf_list_order_is_lexsort_of_brute_force_slabs(orc):
    rng = np.random.default_rng(31)
    lo, hi = _tie_heavy_cut(rng)
    rays = []
    for _ in range(150):                                       # along +-z: lattice ties in t_enter
        s = 1.0 if rng.random() < 0.5 else -1.0
        rays.append([rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4), -2.0 * s, 0.0, 0, 0, s, np.inf])
    for _ in range(60):                                        # origin inside boxes: t_enter = tmin ties
        rays.append([*rng.uniform(-0.3, 0.3, 3), 0.0, *synth.random_rays(1, seed=int(rng.integers(1e6)))[0, 4:7],
                     np.inf])
    rays = np.concatenate([np.asarray(rays, np.float32), synth.random_rays(200, seed=4)], 0)
    cap = lo.shape[0]
    leaf, te, tx, cnt = orc.leaf_lists(rays, lo, hi, cap)
    n_ties = 0
    for r in range(rays.shape[0]):
        ids, bte, btx = _brute_order(orc, rays[r], lo, hi)
        assert cnt[r] == ids.size
        assert leaf[r, :cnt[r]].tolist() == ids.tolist()
        assert np.array_equal(te[r, :cnt[r]], bte) and np.array_equal(tx[r, :cnt[r]], btx)
        assert np.all(leaf[r, cnt[r]:] == -1)
        n_ties += int(np.sum(np.diff(bte) == 0)) if bte.size > 1 else 0
    assert n_ties > 100                                        # the equal-t_enter case is exercised
