"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the pin it implements and the passage it
follows.  None of these re-types the oracle's formula and compares it with itself:
they use printed values, closed forms, special cases, invariants and brute force.
"""
import math

import numpy as np
import pytest

import synth

PRIMES = (1, 2654435761, 805459861)


# ------------------------------------------------------------------ P1 hash (P:101 -> [Mueller22])
def test_p1_hash_regression_constants(orc):
    assert orc.corner_index(1024, 0, 14, 0, 0, 0) == 0
    assert orc.corner_index(1024, 0, 14, 1, 0, 0) == 1
    assert orc.corner_index(1024, 0, 10, 1, 2, 3) == 476
    assert orc.corner_index(1024, 0, 14, 1, 2, 3) == 13788
    assert orc.corner_index(1024, 0, 19, 1, 2, 3) == 128476
    assert orc.corner_index(1024, 0, 19, 7, 11, 13) == 280589


def test_p1_hash_x_neighbour_invariant(orc):
    # pi_1 = 1 => for even x, the x-neighbour's index is idx ^ 1 (adjacent table entry).
    rng = np.random.default_rng(0)
    for _ in range(200):
        x = int(rng.integers(0, 512)) * 2
        y, z = (int(v) for v in rng.integers(0, 1025, size=2))
        a = orc.corner_index(1024, 0, 19, x, y, z)
        b = orc.corner_index(1024, 0, 19, x + 1, y, z)
        assert b == a ^ 1


# ------------------------------------------------------------------ P2/P3/P4 levels, dense index, sizing
def test_p2_level_resolutions(orc):
    g = orc.Grid(8, 14)  # 8 levels, 8^3 .. 1024^3 -> b = 2 exactly
    assert list(g.res) == [8 * 2 ** l for l in range(8)]
    assert list(g.dense) == [1, 1, 0, 0, 0, 0, 0, 0]            # (N+1)^3 <= 2^14 only for N=8,16
    assert g.n_entries == 729 + 4913 + 6 * 2 ** 14
    g16 = orc.Grid(16, 19)
    assert g16.res[0] == 8 and g16.res[-1] == 1024
    assert list(g16.res) == [8, 11, 15, 21, 29, 40, 55, 76, 106, 147, 203, 280, 388, 536, 741, 1024]
    assert np.all(np.diff(g16.res) > 0)
    assert g16.n_entries == 4_939_575


def test_p3_dense_index_bijective(orc):
    for N in (1, 2, 3, 8):
        seen = set()
        for z in range(N + 1):
            for y in range(N + 1):
                for x in range(N + 1):
                    seen.add(orc.corner_index(N, 1, 14, x, y, z))
        assert seen == set(range((N + 1) ** 3))


def test_p4_network_size_matches_paper(orc):
    # P:393/P:419/P:423 print a 10.8 MB network at T=2^18, L=8, F=4, fp16.
    g = orc.Grid(8, 18, F=4)
    mb = g.n_entries * 4 * 2 / 1e6
    assert round(mb, 1) == 10.8
    all_hash = 8 * 2 ** 18 * 4 * 2 / 1e6                         # the reading C2 rejects
    assert round(all_hash, 1) != 10.8


# ------------------------------------------------------------------ P5 trilinear encode
def _table_for(g, fn):
    """fp16 table whose dense-level entries hold fn(x,y,z) at each grid vertex."""
    tab = np.zeros((g.n_entries, g.F), np.float16)
    for l in range(g.L):
        N = int(g.res[l])
        if not g.dense[l]:
            continue
        z, y, x = np.meshgrid(np.arange(N + 1), np.arange(N + 1), np.arange(N + 1), indexing="ij")
        vals = fn(x.ravel(), y.ravel(), z.ravel())
        idx = x.ravel() + (N + 1) * (y.ravel() + (N + 1) * z.ravel())
        for j in range(g.F):
            tab[g.offset[l] + idx, j] = vals * (j + 1)
    return tab


def test_p5_weights_sum_to_one(orc):
    g = orc.Grid(8, 14)
    tab = np.ones((g.n_entries, 2), np.float16)
    pts = np.random.default_rng(1).random((500, 3), dtype=np.float32)
    feat, _ = orc.encode_points(g, tab, pts)
    assert np.max(np.abs(feat - 1.0)) < 1e-14


def test_p5_reproduces_linear_functions_on_dense_levels(orc):
    # Trilinear interpolation is exact on affine functions: with T[v] = vx + 2vy + 3vz
    # at every dense vertex, feature = s_x + 2 s_y + 3 s_z where s = x*N.
    g = orc.Grid(8, 14)
    tab = _table_for(g, lambda x, y, z: x + 2 * y + 3 * z)
    pts = np.random.default_rng(2).random((300, 3), dtype=np.float32)
    feat, _ = orc.encode_points(g, tab, pts)
    for l in range(2):
        N = np.float32(g.res[l])
        s = (pts * N).astype(np.float64)
        want = s[:, 0] + 2 * s[:, 1] + 3 * s[:, 2]
        np.testing.assert_allclose(feat[:, l * 2 + 0], want, atol=1e-12)
        np.testing.assert_allclose(feat[:, l * 2 + 1], 2 * want, atol=1e-12)


def test_p5_corner_one_hot_and_edge_midpoint(orc):
    g = orc.Grid(8, 14)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=3).reshape(-1, 2)
    rng = np.random.default_rng(4)
    # grid vertices of the coarsest level are vertices of every level (8 | N_l)
    v = rng.integers(0, 8, size=(50, 3))
    pts = (v / 8.0).astype(np.float32)
    feat, idx = orc.encode_points(g, tab, pts)
    for l in range(g.L):
        want = tab[g.offset[l] + idx[:, l, 0]].astype(np.float64)
        np.testing.assert_array_equal(feat[:, 2 * l:2 * l + 2], want)
    # edge midpoint at level 0 (N=8): mean of the two x-adjacent corners
    c = rng.integers(0, 8, size=(50, 3))
    p = np.stack([(c[:, 0] + 0.5) / 8.0, c[:, 1] / 8.0, c[:, 2] / 8.0], 1).astype(np.float32)
    feat, idx = orc.encode_points(g, tab, p)
    want = 0.5 * (tab[idx[:, 0, 0]].astype(np.float64) + tab[idx[:, 0, 1]].astype(np.float64))
    np.testing.assert_allclose(feat[:, 0:2], want, atol=1e-15)
    # corner 0 of level 0 is the dense vertex c (closed form)
    np.testing.assert_array_equal(idx[:, 0, 0], c[:, 0] + 9 * (c[:, 1] + 9 * c[:, 2]))


def test_p5_continuity_across_cell_faces(orc):
    g = orc.Grid(8, 14)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=5).reshape(-1, 2)
    rng = np.random.default_rng(6)
    base = rng.random((200, 3), dtype=np.float32)
    face = (np.floor(base[:, 0] * 1024) / 1024).astype(np.float32)
    eps = np.float32(2.0 ** -20)
    a = base.copy(); a[:, 0] = face - eps
    b = base.copy(); b[:, 0] = face + eps
    fa, _ = orc.encode_points(g, tab, np.clip(a, 0, 1))
    fb, _ = orc.encode_points(g, tab, np.clip(b, 0, 1))
    # Lipschitz bound: |d feat/dx| <= 2 N max|T| -> |diff| <= 2*2^-20*1024*2 ~ 0.004
    assert np.max(np.abs(fa - fb)) < 0.01


# ------------------------------------------------------------------ P6 slab
def test_p6_slab_worked_examples(orc):
    lo, hi = np.array([-1, -1, -1], np.float32), np.array([1, 1, 1], np.float32)
    h, te, tx, *_ = orc.slab([0, 0, -2, 0, 0, 0, 1, np.inf], lo, hi)
    assert h and te == 1.0 and tx == 3.0
    h, te, tx, *_ = orc.slab([0, 0, 0, 0, 0, 0, 1, np.inf], lo, hi)      # starts inside (C7)
    assert h and te == 0.0 and tx == 1.0
    h, *_ = orc.slab([0, 0, -2, 0, 0, 0, -1, np.inf], lo, hi)           # pointing away
    assert not h
    h, *_ = orc.slab([3, 0, -2, 0, 0, 0, 1, np.inf], lo, hi)            # parallel, outside
    assert not h


def test_p6_slab_vs_point_sampling(orc):
    rng = np.random.default_rng(7)
    for _ in range(300):
        lo = rng.uniform(-1, 0.5, 3).astype(np.float32)
        hi = (lo + rng.uniform(0.01, 1.0, 3)).astype(np.float32)
        o = rng.uniform(-2, 2, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        ray = np.array([*o, 0, *d, np.inf], np.float32)
        h, te, tx, *_ = orc.slab(ray, lo, hi)
        ts = np.linspace(0, 8, 2001)
        P = ray[None, 0:3].astype(np.float64) + ts[:, None] * ray[None, 4:7].astype(np.float64)
        inside = np.all((P >= lo - 1e-6) & (P <= hi + 1e-6), axis=1)
        strict = np.all((P > lo + 1e-4) & (P < hi - 1e-4), axis=1)
        if strict.any():
            assert h
        if h:
            mid = np.linspace(te, tx, 9)[1:-1]
            Pm = ray[None, 0:3] + mid[:, None] * ray[None, 4:7]
            assert np.all((Pm >= lo - 1e-5) & (Pm <= hi + 1e-5))
            assert ts[inside].min() >= te - 0.01 and ts[inside].max() <= tx + 0.01
        else:
            assert not strict.any()


# ------------------------------------------------------------------ P9 sampling
def test_p9_midpoint_samples(orc):
    pts = orc.segment_points([0, 0, 0, 0, 0, 0, 1, np.inf], 0.0, 3.0, 3, np.zeros(3, np.float32), 0.25)
    np.testing.assert_array_equal(pts[:, 2], np.array([0.5, 1.5, 2.5], np.float32) * 0.25)
    np.testing.assert_array_equal(pts[:, :2], 0)


def test_p9_reversed_ray_reverses_points(orc):
    fwd = orc.segment_points([0, 0, 0, 0, 0, 0, 1, np.inf], 0.0, 3.0, 4, np.zeros(3, np.float32), 0.25)
    bwd = orc.segment_points([0, 0, 3, 0, 0, 0, -1, np.inf], 0.0, 3.0, 4, np.zeros(3, np.float32), 0.25)
    np.testing.assert_array_equal(fwd, bwd[::-1])
    rng = np.random.default_rng(8)
    for _ in range(50):
        o = rng.uniform(-1, 1, 3)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        e = o + 1.7 * d
        f = orc.segment_points([*o, 0, *d, np.inf], 0.0, 1.7, 4, np.full(3, -2, np.float32), 0.25)
        b = orc.segment_points([*e, 0, *(-d), np.inf], 0.0, 1.7, 4, np.full(3, -2, np.float32), 0.25)
        np.testing.assert_allclose(f, b[::-1], atol=1e-6)


def test_p9_jittered_samples_stay_in_strata(orc):
    rng = np.random.default_rng(9)
    xi = rng.random(4, dtype=np.float32)
    pts = orc.segment_points([0, 0, 0, 0, 0, 0, 1, np.inf], 0.0, 4.0, 4, np.zeros(3, np.float32), 0.125, xi=xi)
    z = pts[:, 2] / 0.125
    np.testing.assert_allclose(z, np.arange(4) + xi, atol=1e-6)


# ------------------------------------------------------------------ P10 MLP
def test_p10_mlp_zero_weights_and_numpy_matmul(orc):
    layers = [(np.zeros((8, 12), np.float16), np.zeros(8, np.float32)),
              (np.zeros((8, 8), np.float16), np.zeros(8, np.float32))]
    z = orc.mlp_forward(layers, np.random.default_rng(0).normal(size=(5, 12)))
    assert np.all(z == 0)                                   # sigmoid channels -> 0.5, linear -> 0
    layers = synth.random_mlp(64, 2, 64, seed=11)
    x = np.random.default_rng(1).normal(size=(40, 64))
    h = x
    for k, (W, b) in enumerate(layers):
        h = h @ W.astype(np.float64).T + b.astype(np.float64)
        if k + 1 < len(layers):
            h = np.maximum(h, 0)
    np.testing.assert_allclose(orc.mlp_forward(layers, x), h, rtol=1e-12, atol=1e-12)


def test_p10_mlp_hand_computed_unit(orc):
    W1 = np.zeros((2, 2), np.float16); W1[0, 0] = 2.0; W1[0, 1] = -1.0
    b1 = np.array([0.5, -1.0], np.float32)
    W2 = np.zeros((8, 2), np.float16); W2[0, 0] = 3.0; W2[1, 1] = 1.0
    b2 = np.zeros(8, np.float32); b2[2] = 0.25
    z = orc.mlp_forward([(W1, b1), (W2, b2)], np.array([[1.0, 0.5]]))
    # h0 = relu(2*1 - 0.5 + 0.5) = 2 ; h1 = relu(-1) = 0 ; z0 = 6, z1 = 0, z2 = 0.25
    assert z[0, 0] == 6.0 and z[0, 1] == 0.0 and z[0, 2] == 0.25


# ------------------------------------------------------------------ P8/P11 query semantics
def _one_layer_mlp(d_in, vis_bias, t_bias, nz=(0.0, 0.0, 1.0)):
    W = np.zeros((8, d_in), np.float16)
    b = np.zeros(8, np.float32)
    b[0] = vis_bias; b[1] = t_bias; b[2:5] = nz
    return [(np.zeros((4, d_in), np.float16), np.zeros(4, np.float32)), (np.zeros((8, 4), np.float16), b)]


def test_p8_p11_query_semantics(orc):
    g = orc.Grid(2, 6)
    tab = np.zeros((g.n_entries, 2), np.float16)
    lo = np.array([[-1, -1, -1], [-1, -1, 2]], np.float32)
    hi = np.array([[1, 1, 1], [1, 1, 4]], np.float32)
    rays = np.array([[0, 0, -3, 0, 0, 0, 1, np.inf],     # crosses both leaves
                     [5, 5, -3, 0, 0, 0, 1, np.inf]], np.float32)  # misses everything
    # always-hit model with t_local = sigmoid(-40) ~ 0 -> t = t_enter of the near leaf
    out = orc.query(g, 3, tab, _one_layer_mlp(12, -5.0, -40.0), lo, hi, rays)
    assert out["hit"].tolist() == [1, 0]
    assert out["nq"].tolist() == [1, 0]                  # near hit prunes far, miss -> 0
    assert abs(out["t"][0] - 2.0) < 1e-12 and out["leaf"][0] == 0 and np.isinf(out["t"][1])
    np.testing.assert_allclose(out["normal"][0], [0, 0, 1])
    # t_local -> 1: t = t_exit of the near leaf
    out = orc.query(g, 3, tab, _one_layer_mlp(12, -5.0, 40.0), lo, hi, rays)
    assert abs(out["t"][0] - 4.0) < 1e-12
    # tie sigma(z_vis) = 0.5 -> miss (C13): every intersected leaf queried
    out = orc.query(g, 3, tab, _one_layer_mlp(12, 0.0, 0.0), lo, hi, rays)
    assert out["hit"].tolist() == [0, 0] and out["nq"].tolist() == [2, 0]


def test_p8_single_leaf_cut_is_one_query(orc):
    g = orc.Grid(2, 6)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=1).reshape(-1, 2)
    rays = synth.random_rays(200, seed=3)
    lo = np.array([[-1, -1, -1]], np.float32)
    hi = np.array([[1, 1, 1]], np.float32)
    out = orc.query(g, 3, tab, synth.random_mlp(12, 1, 8, seed=4), lo, hi, rays)
    leaf, te, tx, cnt = orc.leaf_lists(rays, lo, hi, 1)
    assert np.array_equal(out["nq"], cnt)


def test_p8_order_independence_R2_vs_R1(orc):
    # R2 result = argmin over ALL intersected leaves (proof in DESIGN.md C5); R1 stops at
    # the first reported hit.  Overlapping leaves make them differ.
    g = orc.Grid(4, 8)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=6).reshape(-1, 2)
    layers = synth.random_mlp(24, 1, 16, seed=7)
    rng = np.random.default_rng(8)
    lo = rng.uniform(-0.8, 0.2, (12, 3)).astype(np.float32)
    hi = (lo + rng.uniform(0.3, 0.8, (12, 3))).astype(np.float32)
    rays = synth.random_rays(1500, seed=9, lo=(-0.5,) * 3, hi=(0.5,) * 3)
    r2 = orc.query(g, 3, tab, layers, lo, hi, rays, mode=0)
    r1 = orc.query(g, 3, tab, layers, lo, hi, rays, mode=1)
    # Brute force: evaluate EVERY intersected leaf from the primitives (sample, encode,
    # MLP) and take argmin (t, t_enter, id); R2 must return it although it skips leaves.
    # The walk order for R1 comes from brute-force slabs + numpy's lexsort on (t_enter, id),
    # not from the oracle's own leaf_list.
    dmin, dinv = orc.domain(lo, hi)
    n_first_hit_differs = 0
    cnt = np.zeros(len(rays), np.int32)
    for r in range(len(rays)):
        slabs = [orc.slab(rays[r], lo[i], hi[i]) for i in range(lo.shape[0])]
        ids = [i for i in range(lo.shape[0]) if slabs[i][0]]
        te = np.asarray([slabs[i][3] for i in ids], np.float32)
        tx = np.asarray([slabs[i][4] for i in ids], np.float32)
        order = np.lexsort((np.asarray(ids), te)) if ids else []
        cnt[r] = len(ids)
        cands = []
        first = None
        for k in order:
            pts = orc.segment_points(rays[r], te[k], tx[k], 3, dmin, dinv)
            feat, _ = orc.encode_points(g, tab, pts)
            z = orc.mlp_forward(layers, feat.reshape(1, -1))[0]
            if z[0] < 0:
                t = float(te[k]) + 1 / (1 + math.exp(-z[1])) * (float(tx[k]) - float(te[k]))
                cands.append((t, float(te[k]), int(ids[k])))
                if first is None:
                    first = cands[-1]
        if cands:
            best = min(cands)
            assert r2["hit"][r] == 1 and r2["leaf"][r] == best[2] and abs(r2["t"][r] - best[0]) < 1e-6
            assert r1["hit"][r] == 1 and r1["leaf"][r] == first[2]
            n_first_hit_differs += first != best
        else:
            assert r2["hit"][r] == 0 and r1["hit"][r] == 0
            assert r2["nq"][r] == cnt[r]
    assert np.all(r1["nq"] <= r2["nq"])
    assert n_first_hit_differs > 0                                # overlap makes R1 != R2 somewhere


# ------------------------------------------------------------------ P12 losses
def _logit(p):
    return math.log(p / (1 - p))


def test_p12_loss_examples(orc):
    gt_miss = np.array([1, 0, 0, 0, 0, 0, 0, 0, 0], float)
    L, terms, _ = orc.sample_loss(np.array([0, 5, 9, 9, 9, 9, 9, 9]), gt_miss)
    assert abs(terms[0] - math.log(2)) < 1e-15                 # BCE(0.5, 1) = ln 2
    assert terms[1] == terms[2] == terms[3] == 0.0              # gating: miss -> only BCE
    assert abs(L - 2 * math.log(2)) < 1e-15
    gt = np.array([0, 0.75, 0, 0, 1, 0, 0, 0, 0], float)
    _, terms, _ = orc.sample_loss(np.array([-30, _logit(0.25), 0, 0, 1, 1e3, 1e3, 1e3]), gt)
    assert abs(terms[1] - 0.5) < 1e-12                          # L1(0.25, 0.75)
    assert abs(terms[3] - 1 / 1.01) < 1e-12                     # relL2((1,1,1),(0,0,0))
    # combined: terms (0.1, 0.2, 0.3, 0.4) -> 2*0.1 + 2*0.2 + 0.3 + 0.4 = 1.3
    a = 0.6
    y = a - math.sqrt(0.4 * (a * a + 0.01))
    zvis = math.log(math.exp(0.1) - 1)                           # softplus(z) = 0.1, gt_vis = 0
    gt = np.array([0, 0.3, 0.1, 0.2, 0.3, y, y, y, 0], float)
    z = np.array([zvis, _logit(0.5), 0.4, 0.5, 0.6, _logit(a), _logit(a), _logit(a)])
    L, terms, _ = orc.sample_loss(z, gt)
    np.testing.assert_allclose(terms, [0.1, 0.2, 0.3, 0.4], atol=1e-12)
    assert abs(L - 1.3) < 1e-12


def test_p12_loss_gradient_vs_finite_differences(orc):
    rng = np.random.default_rng(10)
    for trial in range(20):
        z = rng.normal(size=8) * 2
        gt = np.concatenate([[trial % 2], rng.random(1), rng.normal(size=3), rng.random(3), [0]])
        _, _, dz = orc.sample_loss(z, gt)
        h = 1e-6
        for k in range(8):
            zp, zm = z.copy(), z.copy()
            zp[k] += h; zm[k] -= h
            fd = (orc.sample_loss(zp, gt)[0] - orc.sample_loss(zm, gt)[0]) / (2 * h)
            if k >= 5 and gt[0] == 0:
                # relative L2 stops the gradient through its denominator (C19): the
                # full derivative adds -(a-y)^2 2a/(a^2+0.01)^2 /3 * a(1-a)
                a = 1 / (1 + math.exp(-z[k]))
                fd += (a - gt[k]) ** 2 * 2 * a / (a * a + 0.01) ** 2 / 3 * a * (1 - a)
            assert abs(fd - dz[k]) < 1e-6 * max(1, abs(fd))


# ------------------------------------------------------------------ P14 Adam
def test_p14_adam_closed_form_constant_gradient(orc):
    g = 0.37
    p = np.array([1.5]); m = np.zeros(1); v = np.zeros(1)
    for t in range(1, 51):
        orc.adam(p, np.array([g]), m, v, t)
        # m_hat = g and v_hat = g^2 exactly in exact arithmetic -> step = lr*g/(|g|+eps)
        assert abs(p[0] - (1.5 - t * 0.01 * g / (abs(g) + 1e-8))) < 1e-12
    p = np.array([2.0]); m = np.zeros(1); v = np.zeros(1)
    orc.adam(p, np.zeros(1), m, v, 1)
    assert p[0] == 2.0 and m[0] == 0 and v[0] == 0


# ------------------------------------------------------------------ P16 triangle GT
def test_p16_triangle_examples(orc):
    v0, v1, v2 = [-1, -1, 0], [1, -1, 0], [0, 1, 0]
    h, t, *_ = orc.triangle_hit([0, 0, -1], [0, 0, 1], v0, v1, v2)
    assert h and t == 1.0
    h, *_ = orc.triangle_hit([0, 0, -1], [0, 0, 1], [-1, -1, -2], [1, -1, -2], [0, 1, -2])
    assert not h                                                 # behind the origin


def test_p16_triangle_vs_plane_and_inside_test(orc):
    rng = np.random.default_rng(12)
    agree = 0
    for _ in range(3000):
        V = rng.uniform(-1, 1, (3, 3))
        o = rng.uniform(-2, 2, 3)
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        h, t, *_ = orc.triangle_hit(o, d, V[0], V[1], V[2])
        n = np.cross(V[1] - V[0], V[2] - V[0])
        den = d @ n
        if abs(den) < 1e-9:
            continue
        tp = ((V[0] - o) @ n) / den
        P = o + tp * d
        s = [np.cross(V[(i + 1) % 3] - V[i], P - V[i]) @ n for i in range(3)]
        inside = all(x > 0 for x in s) or all(x < 0 for x in s)
        margin = min(abs(x) for x in s) / (np.linalg.norm(n) ** 2)
        if margin < 1e-9 or abs(tp) < 1e-9:
            continue
        expect = inside and tp >= 0
        assert h == expect
        if h:
            assert abs(t - tp) < 1e-9 * max(1, abs(tp))
        agree += 1
    assert agree > 2500


def _test_cut(scene, k=4):
    """A hand-made cut for the oracle tests: k slabs of triangles by centroid x."""
    V = scene.verts.astype(np.float64)
    cen = V[scene.tris].mean(axis=1)
    edges = np.quantile(cen[:, 0], np.linspace(0, 1, k + 1))
    part = np.clip(np.searchsorted(edges, cen[:, 0], side="right") - 1, 0, k - 1)
    diag = float(np.linalg.norm(V.max(0) - V.min(0)))
    off, tris, blo, bhi, llo, lhi = [0], [], [], [], [], []
    for i in range(k):
        ids = np.nonzero(part == i)[0].astype(np.int32)
        tris.append(ids)
        off.append(off[-1] + len(ids))
        P = scene.verts[scene.tris[ids]].reshape(-1, 3)
        lo, hi = P.min(0), P.max(0)
        pad = max(1e-3 * float(np.linalg.norm(hi.astype(np.float64) - lo)), 1e-6 * diag)
        blo.append(lo); bhi.append(hi)
        llo.append((lo - np.float32(pad)).astype(np.float32)); lhi.append((hi + np.float32(pad)).astype(np.float32))
    return (np.array(off, np.int64), np.concatenate(tris), np.array(blo, np.float32), np.array(bhi, np.float32),
            np.array(llo, np.float32), np.array(lhi, np.float32), diag)


def test_p7_cut_checker(orc):
    sc = synth.scene_tiny(nu=6)
    off, lt, blo, bhi, llo, lhi, diag = _test_cut(sc)
    assert orc.check_cut(sc.verts, sc.tris, off, lt, blo, bhi, llo, lhi, diag) == 0
    lt2 = lt.copy(); lt2[0] = lt2[1]                              # a triangle twice, one missing
    assert orc.check_cut(sc.verts, sc.tris, off, lt2, blo, bhi, llo, lhi, diag) & 1
    lhi2 = lhi.copy(); lhi2[0] += 0.01                           # wrong inflation
    assert orc.check_cut(sc.verts, sc.tris, off, lt, blo, bhi, llo, lhi2, diag) & 8


def test_p16_label_is_subset_monotone(orc):
    sc = synth.scene_tiny(nu=6)
    off, lt, blo, bhi, llo, lhi, diag = _test_cut(sc, k=1)
    rays = synth.random_rays(300, seed=13)
    leaf, te, tx, cnt = orc.leaf_lists(rays, llo, lhi, 1)
    ok = cnt > 0
    rays, te, tx = rays[ok], te[ok, 0], tx[ok, 0]
    whole = orc.label(sc, off, lt, rays, np.zeros(len(rays), np.int32), te, tx)
    half = orc.label(sc, np.array([0, len(lt) // 2], np.int64), lt[: len(lt) // 2], rays,
                     np.zeros(len(rays), np.int32), te, tx)
    both = (whole[:, 0] == 0) & (half[:, 0] == 0)
    assert np.all(whole[both, 8] <= half[both, 8])                # parent t <= child t
    assert np.all(whole[half[:, 0] == 0, 0] == 0)                 # subset hit -> superset hit
    assert (whole[:, 0] == 0).sum() > 50
    nrm = np.linalg.norm(whole[whole[:, 0] == 0, 2:5], axis=1)
    np.testing.assert_allclose(nrm, 1.0, atol=1e-12)
    # brute force over every triangle equals the list-based label for the full list
    for r in range(0, len(rays), 37):
        best = None
        for ti in range(sc.n_tris):
            V = sc.verts[sc.tris[ti]].astype(np.float64)
            h, t, *_ = orc.triangle_hit(rays[r, :3], rays[r, 4:7], V[0], V[1], V[2], float(te[r]), float(tx[r]))
            if h and (best is None or t < best):
                best = t
        assert (best is None) == (whole[r, 0] == 1)
        if best is not None:
            assert best == whole[r, 8]


# ------------------------------------------------------------------ P13 gradients, P15 acceptance
def _small_train_setup(orc, n_rays=300, seed=20):
    sc = synth.scene_tiny(nu=4)
    off, lt, blo, bhi, llo, lhi, diag = _test_cut(sc, k=2)
    g = orc.Grid(2, 6, F=2)
    tab = synth.random_params_fp16(g.n_entries * 2, seed=seed, lo=-0.5, hi=0.5).reshape(-1, 2)
    layers = synth.random_mlp(12, 1, 8, seed=seed + 1, out_scale=1.0)   # widths [12, 8, 8]
    rays = synth.random_rays(n_rays, seed=seed + 2)
    u = synth.random_uniform(n_rays, seed=seed + 3)
    xi = synth.random_uniform(n_rays * 3, seed=seed + 4).reshape(n_rays, 3)
    return sc, off, lt, llo, lhi, g, tab, layers, rays, u, xi


def test_p13_gradients_vs_central_differences(orc):
    sc, off, lt, llo, lhi, g, tab, layers, rays, u, xi = _small_train_setup(orc)
    rank = np.zeros(2, np.float32)
    out = orc.train_grad(g, 3, tab, layers, llo, lhi, rank, off, lt, sc, rays, u, xi)
    assert out["n_acc"] > 50
    leaf, te, tx, cnt = orc.leaf_lists(rays, llo, lhi, 1)
    acc = out["accepted"]
    dims = np.array([12, 8, 8], np.int32)
    W_all = np.concatenate([W.astype(np.float64).ravel() for W, _ in layers])
    b_all = np.concatenate([b.astype(np.float64) for _, b in layers])
    T = tab.astype(np.float64).ravel()

    den = np.zeros((len(rays), 3))
    L0 = orc.batch_loss_double(g, 3, T, dims, W_all, b_all, llo, lhi, rays, xi, acc, te[:, 0], tx[:, 0],
                               out["gt"], den, 0)

    def loss(T_, W_, b_):   # relative-L2 denominators frozen at theta_0: the stop-gradient (C19)
        return orc.batch_loss_double(g, 3, T_, dims, W_, b_, llo, lhi, rays, xi, acc, te[:, 0], tx[:, 0],
                                     out["gt"], den, 1)

    assert abs(L0 - out["loss_sum"][0] / out["n_acc"]) < 1e-12
    h = 1e-6
    rng = np.random.default_rng(0)
    checks = [("T", i) for i in np.nonzero(out["g_table"])[0][rng.permutation(np.count_nonzero(out["g_table"]))[:40]]]
    checks += [("W", i) for i in rng.permutation(W_all.size)[:40]] + [("b", i) for i in range(b_all.size)]
    for kind, i in checks:
        arrs = {"T": T.copy(), "W": W_all.copy(), "b": b_all.copy()}
        arrs[kind][i] += h
        lp = loss(arrs["T"], arrs["W"], arrs["b"])
        arrs[kind][i] -= 2 * h
        lm = loss(arrs["T"], arrs["W"], arrs["b"])
        fd = (lp - lm) / (2 * h)
        an = {"T": out["g_table"], "W": out["g_W"], "b": out["g_b"]}[kind][i]
        assert abs(fd - an) <= 1e-4 * max(abs(fd), 1e-3), (kind, i, fd, an)
    # touched rows: nonzero table gradients only at corners of accepted samples' points
    touched = np.count_nonzero(out["g_table"].reshape(-1, 2).any(axis=1))
    assert 0 < touched <= g.n_entries


def test_p15_acceptance_floor_and_single_leaf(orc):
    sc, off, lt, llo, lhi, g, tab, layers, rays, u, xi = _small_train_setup(orc)
    # single-leaf rank vector with all ranks equal -> probability 1
    out = orc.train_grad(g, 3, tab, layers, llo, lhi, np.zeros(2, np.float32), off, lt, sc, rays, u, xi)
    assert np.all(out["accepted"][out["first_leaf"] >= 0] == 1)
    # lowest-rank leaf is accepted with probability 0.005 (P:197 floor)
    n = 400_000
    rays = np.tile(np.array([[-3, 0.01, 0.02, 0, 1, 0, 0, np.inf]], np.float32), (n, 1))
    u = synth.random_uniform(n, seed=99)
    xi = synth.random_uniform(n * 3, seed=98).reshape(n, 3)
    lo = np.array([[-1, -1, -1], [0.5, -1, -1]], np.float32)
    hi = np.array([[0, 1, 1], [1, 1, 1]], np.float32)
    rank = np.array([-100.0, 0.0], np.float32)                    # leaf 0 is the first hit
    out = orc.train_grad(g, 3, tab, layers, lo, hi, rank, off, lt, sc, rays, u, xi)
    rate = out["accepted"].mean()
    assert 0.0045 <= rate <= 0.0055


# ------------------------------------------------------------------ C27 decode sigmoid
def test_c27_sigmoid_f32_vs_exact(orc):
    """The fp32 decode sigmoid against the exact logistic function (closed form, evaluated
    in double by numpy): a few fp32 ulp everywhere, the exact special values at 0 and in
    the saturated tails, monotone, and the symmetry s(-z) = 1 - s(z) to fp32 rounding."""
    zs = np.concatenate([np.linspace(-30, 30, 6001), [-100.0, -87.5, -20.0, -1e-6, 0.0, 1e-6, 20.0, 87.5, 100.0]])
    zs = zs.astype(np.float32)
    got = np.array([orc.sigmoid_f32(float(z)) for z in zs], np.float64)
    exact = 1.0 / (1.0 + np.exp(-zs.astype(np.float64)))
    assert np.all(np.abs(got - exact) <= 4 * np.spacing(np.float32(exact)).astype(np.float64) + 1e-37)
    assert orc.sigmoid_f32(0.0) == 0.5
    assert orc.sigmoid_f32(100.0) == 1.0 and orc.sigmoid_f32(-100.0) < 1e-37
    inner = np.argsort(zs)
    assert np.all(np.diff(got[inner]) >= 0)
    for z in (0.25, 1.0, 3.5, 9.0):
        assert abs(orc.sigmoid_f32(-z) - (1.0 - orc.sigmoid_f32(z))) <= 2 ** -23


# ------------------------------------------------------------------ T0 Philox-4x32-10 (C28')
def test_t0_philox_known_answer_vectors(orc):
    """Philox-4x32-10 against the published known-answer vectors (Random123 kat_vectors)."""
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        assert tuple(int(x) for x in orc.philox4x32_10(ctr, key)) == want


def test_t0_training_rays_distribution(orc):
    """The T0 recipe: origins inside the box, unit directions, U in [0,1); moments of a large
    batch match the uniform / isotropic closed forms (mean 1/2, E[d] = 0, E[d_z^2] = 1/3);
    shards (i0) reproduce the whole batch; the step changes every draw."""
    box = (-1.5, -1.5, -1.5, 1.5, 1.5, 1.5)
    rays, u, xi = orc.gen_train_rays(7, 3, 0, 200000, box, 4)
    assert np.all(rays[:, :3] >= -1.5) and np.all(rays[:, :3] < 1.5)
    assert np.allclose(np.linalg.norm(rays[:, 4:7], axis=1), 1.0, atol=1e-6)
    assert np.all((u >= 0) & (u < 1)) and np.all((xi >= 0) & (xi < 1))
    assert abs(u.mean() - 0.5) < 5e-3 and abs(xi.mean() - 0.5) < 5e-3
    assert np.all(np.abs(rays[:, 4:7].mean(0)) < 1e-2) and abs((rays[:, 6] ** 2).mean() - 1 / 3) < 5e-3
    assert abs(rays[:, :3].mean()) < 1e-2
    r2, u2, x2 = orc.gen_train_rays(7, 3, 1000, 500, box, 4)
    assert np.array_equal(r2, rays[1000:1500]) and np.array_equal(u2, u[1000:1500]) and np.array_equal(x2, xi[1000:1500])
    r3, u3, _ = orc.gen_train_rays(7, 4, 0, 1000, box, 4)
    assert np.mean(u3 == u[:1000]) < 0.01


def test_p13_backward_given_equals_train_grad_and_bounds(orc):
    """orc_train_backward_given (T6/T7 from given features and dL/dz, used to compare the
    GPU's chain stage by stage) fed the oracle's OWN per-sample features and dL/dz (from the
    pinned encode, MLP and loss) reproduces orc_train_grad's gradients (pinned by central
    differences above) times the accepted count; its magnitude sums bound |g|; its hidden
    deltas give dW by an independent numpy contraction; z equals the numpy float64 MLP."""
    sc, off, lt, llo, lhi, g, tab, layers, rays, u, xi = _small_train_setup(orc, n_rays=400, seed=23)
    rank = np.zeros(2, np.float32)
    full = orc.train_grad(g, 3, tab, layers, llo, lhi, rank, off, lt, sc, rays, u, xi)
    acc = np.nonzero(full["accepted"])[0]
    assert acc.size > 60
    leaf, te, tx, cnt = orc.leaf_lists(rays, llo, lhi, 1)
    box = np.concatenate([llo.min(0), lhi.max(0)]).astype(np.float32)      # = the union-of-leaves domain
    dmin, dinv = orc.domain(llo, lhi)
    x = np.stack([orc.encode_points(g, tab, orc.segment_points(rays[r], te[r, 0], tx[r, 0], 3, dmin, dinv,
                                                              xi[r]))[0].reshape(-1) for r in acc])
    z = orc.mlp_forward(layers, x)
    dz = np.stack([orc.sample_loss(z[i], full["gt"][r])[2] for i, r in enumerate(acc)])
    o = orc.train_backward_given(g, 3, tab, layers, box, rays[acc], te[acc, 0], tx[acc, 0], xi[acc], x, dz,
                                 want_deltas=True)
    m = acc.size
    for k in ("g_table", "g_W", "g_b"):
        np.testing.assert_allclose(o[k], full[k] * m, rtol=1e-12, atol=1e-14)
        assert np.all(o[k + "_abs"] >= np.abs(o[k]) - 1e-15)
    np.testing.assert_allclose(o["z"], z, rtol=1e-13, atol=1e-14)
    assert np.all(o["z_abs"] >= np.abs(o["z"]) - 1e-15)
    # dW of the output layer = sum dz (x) h_1 and of layer 0 = sum delta_0 (x) x (numpy einsum
    # over the hidden deltas / activations)
    W0, b0 = layers[0]
    h1 = np.maximum(x @ W0.astype(np.float64).T + b0, 0.0)
    d0 = o["hidden_delta"][:, 0, :8]
    np.testing.assert_allclose(o["g_W"][:8 * 12], np.einsum("so,si->oi", d0, x).ravel(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(o["g_W"][8 * 12:], np.einsum("so,si->oi", dz, h1).ravel(), rtol=1e-11, atol=1e-13)
    # ReLU margin: 0 for a unit whose pre-activation is exactly 0 with non-zero operands
    # (w = +1 on feature 0, -1 on feature 1, and the given x has x_0 == x_1)
    assert np.all(o["relu_margin"] > 0)
    lay = [(W.copy(), b.copy()) for W, b in layers]
    lay[0][0][:] = 0
    lay[0][1][:] = 0.0
    lay[0][0][0, 0], lay[0][0][0, 1] = 1.0, -1.0
    x2 = x[:3].copy()
    x2[:, 1] = x2[:, 0]
    assert np.all(x2[:, 0] != 0)
    o2 = orc.train_backward_given(g, 3, tab, lay, box, rays[acc[:3]], te[acc[:3], 0], tx[acc[:3], 0], xi[acc[:3]],
                                  x2, dz[:3])
    assert np.all(o2["relu_margin"] == 0.0)


# ------------------------------------------------------------------ NEXT-1 construction
def test_next1_expand_cut_pins(orc):
    """orc_expand_cut on a hand-built base BVH: root 0 -> (1, 2); 1 -> (3, 4); 2 -> (5, 6);
    3..6 leaves.  Cut {1, 2}: the leaf of larger r = 2 ln q + ln p is split (a larger p can
    outweigh a smaller q only by the log ratio); a tie goes to the lower leaf index; a
    base leaf is passed over; asking for more splits than possible stops at the leaves."""
    ca = np.array([1, 3, 5, 0, 1, 2, 3], np.int32)
    cb = np.array([2, 4, 6, -1, -1, -1, -1], np.int32)
    cut = np.array([1, 2], np.int32)
    # r(1) = 2 ln 0.5 + ln 0.5 = -2.08 ; r(2) = 2 ln 0.2 + ln 0.8 = -3.44 -> split node 1
    assert orc.expand_cut(ca, cb, cut, [0.5, 0.2], [0.5, 0.8], 1).tolist() == [2, 3, 4]
    # the factor 2 on the loss: r(1) = 2 ln 0.3 + ln 0.1 = -4.71 > r(2) = 2 ln 0.1 + ln 0.5 =
    # -5.30, although the raw product q p ranks node 2 first (0.03 < 0.05)
    assert orc.expand_cut(ca, cb, cut, [0.3, 0.1], [0.1, 0.5], 1).tolist() == [2, 3, 4]
    assert orc.expand_cut(ca, cb, cut, [0.4, 0.4], [0.5, 0.5], 1).tolist() == [2, 3, 4]      # tie: lower index
    assert orc.expand_cut(ca, cb, cut, [0.4, 0.4], [0.5, 0.5], 2).tolist() == [3, 4, 5, 6]
    leafy = np.array([3, 4, 2], np.int32)                  # 3, 4 are base leaves
    assert orc.expand_cut(ca, cb, leafy, [0.9, 0.9, 0.1], [0.9, 0.9, 0.1], 1).tolist() == [3, 4, 5, 6]
    assert orc.expand_cut(ca, cb, leafy, [0.9, 0.9, 0.1], [0.9, 0.9, 0.1], 5).tolist() == [3, 4, 5, 6]


def test_next1_leaf_error_stats_from_records(orc):
    """q = mean loss of a leaf's accepted samples, p = fraction of rays whose first leaf it
    is (C38), computed from per-ray records by hand."""
    first = np.array([0, 0, 1, -1, 2, 0, 1, 1])
    acc = np.array([1, 0, 1, 0, 1, 1, 0, 1])
    loss = np.array([1.0, 9.0, 2.0, 9.0, 5.0, 3.0, 9.0, 4.0])
    q, p, samples, ls = orc.leaf_error_stats(first, acc, loss, 4)
    assert q.tolist() == [2.0, 3.0, 5.0, 0.0]
    assert p.tolist() == [3 / 8, 3 / 8, 1 / 8, 0.0]
    assert samples.tolist() == [2, 2, 1, 0] and ls.tolist() == [4.0, 6.0, 5.0, 0.0]
