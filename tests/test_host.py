"""Host-side logic and the C-ABI boundary, without a GPU (device = -1 contexts)."""
import re
import os
import ctypes as C

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_16237_b200 import build
    build.build()
    from paper_2405_16237_b200 import nbvh
    return nbvh.load_library()


def test_library_exports_every_declared_symbol(lib):
    from paper_2405_16237_b200 import nbvh
    hdr = open(os.path.join(ROOT, "include", "nbvh.h")).read()
    declared = set(re.findall(r"\b(nbvh_[a-z_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    assert declared == set(nbvh.SIGNATURES), declared ^ set(nbvh.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name


@pytest.fixture(scope="module")
def tiny_host(lib):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny()
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    n, st = ctx.build_cut(64)
    assert n == 64 and st == 0
    return ctx, sc


def test_level_table_matches_oracle(orc, lib):
    from paper_2405_16237_b200 import Context
    for L, log2_T, F in [(8, 14, 2), (16, 19, 2), (8, 18, 4)]:
        npts = 96 // (L * F) if L * F <= 96 and 96 % (L * F) == 0 else 128 // (L * F)
        ctx = Context(device=-1, L=L, log2_T=log2_T, F=F, n_points=npts)
        res, dense, off, n = ctx.level_table()
        g = orc.Grid(L, log2_T, F)
        assert np.array_equal(res, g.res) and np.array_equal(dense, g.dense)
        assert np.array_equal(off, g.offset) and n == g.n_entries
        assert ctx.param_count(0) == g.n_entries * F
        ctx.close()


def test_cut_structure_checked_by_oracle(orc, tiny_host):
    ctx, sc = tiny_host
    cut = ctx.cut(0)
    diag = float(np.linalg.norm(sc.verts.astype(np.float64).max(0) - sc.verts.astype(np.float64).min(0)))
    bad = orc.check_cut(sc.verts, sc.tris, cut["tri_off"], cut["tris"], cut["base_lo"], cut["base_hi"],
                        cut["leaf_lo"], cut["leaf_hi"], diag)
    assert bad == 0, bad
    assert cut["n_inner"] == cut["n_leaves"] - 1             # binary snapshot


def test_domain_matches_oracle(orc, tiny_host):
    """C4 (amended): the grid domain is the cube around the scene's inflated root box, the
    same for every cut; bit-exact against the oracle's own computation from the mesh."""
    ctx, sc = tiny_host
    cut = ctx.cut(0)
    dmin, dinv = orc.domain(*np.split(orc.scene_box(sc).reshape(1, 6), 2, axis=1))
    assert np.array_equal(dmin, cut["dom_min"]) and dinv == cut["dom_inv"][0]
    # and it contains every inflated leaf box of the cut
    side = 1.0 / dinv
    assert np.all(cut["leaf_lo"] >= dmin) and np.all(cut["leaf_hi"] <= dmin + side)


@pytest.mark.parametrize("target", [1, 9, 64, 500])
def test_domain_is_cut_independent(orc, lib, target):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=10)
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    ctx.build_cut(target)
    cut = ctx.cut(0)
    dmin, dinv = orc.domain(*np.split(orc.scene_box(sc).reshape(1, 6), 2, axis=1))
    assert np.array_equal(dmin, cut["dom_min"]) and dinv == cut["dom_inv"][0]
    if target == 1:                 # single-leaf cut: the root box itself (union of leaf boxes)
        d1, i1 = orc.domain(cut["leaf_lo"], cut["leaf_hi"])
        assert np.array_equal(d1, dmin) and i1 == dinv


@pytest.mark.parametrize("target", [1, 2, 7, 300])
def test_cut_sizes_and_partition(orc, lib, target):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=8)
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    n, st = ctx.build_cut(target)
    assert n == target
    cut = ctx.cut(0)
    diag = float(np.linalg.norm(sc.verts.astype(np.float64).max(0) - sc.verts.astype(np.float64).min(0)))
    assert orc.check_cut(sc.verts, sc.tris, cut["tri_off"], cut["tris"], cut["base_lo"], cut["base_hi"],
                         cut["leaf_lo"], cut["leaf_hi"], diag) == 0


def test_cut_clamped_to_base_leaves(lib):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=2)                               # 80 triangles
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    n, st = ctx.build_cut(10_000)
    assert st == 1 and n < 80                                 # NBVH_WARN_CLAMPED


def test_error_driven_expansion(orc, lib):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=8)
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    ctx.build_cut(8)
    q = np.ones(8, np.float32); p = np.full(8, 0.1, np.float32)
    q[3] = 10.0                                              # leaf 3 has the largest rank 2 ln q + ln p
    before = ctx.cut(0)
    n, _ = ctx.build_cut(9, q=q, p=p)
    after = ctx.cut(0)
    assert n == 9
    # leaf 3's triangles are now split over two leaves; the others are unchanged
    t3 = set(before["tris"][before["tri_off"][3]:before["tri_off"][4]].tolist())
    groups = [set(after["tris"][after["tri_off"][i]:after["tri_off"][i + 1]].tolist()) for i in range(9)]
    inside = [g for g in groups if g <= t3]
    assert len(inside) == 2 and set().union(*inside) == t3


def test_sah_bvh_traversal_equals_brute_force(orc, lib):
    """Leaf lists over a 1-leaf-per-base-leaf cut = brute force over all base leaves."""
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=4)
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    n, st = ctx.build_cut(10_000)
    cut = ctx.cut(0)
    sizes = np.diff(cut["tri_off"])
    assert sizes.max() <= 4 and sizes.min() >= 1           # SAH leaves hold <= 4 triangles


def test_bad_arguments_rejected(lib):
    from paper_2405_16237_b200 import Context, NbvhError
    with pytest.raises(NbvhError):
        Context(device=-1, L=3, F=2, n_points=4)              # L*F not a multiple of 8
    ctx = Context(device=-1)
    with pytest.raises(NbvhError):
        ctx.build_cut(16)                                    # no mesh yet (ESTATE)
    with pytest.raises(NbvhError):
        ctx.query(np.zeros((1, 8), np.float32))              # host-only context


@pytest.mark.parametrize("mesh_nu,start,splits", [(22, 16, 5), (22, 64, 40), (2, 24, 30)])
def test_error_driven_expansion_matches_oracle(orc, lib, mesh_nu, start, splits):
    """NEXT-1: nbvh_build_cut with per-leaf (q, p) expands the cut exactly as the
    oracle's expansion step does -- the `splits` highest-ranked splittable leaves replaced by
    their children (a small mesh makes some cut leaves base-BVH leaves, which are skipped)."""
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny(nu=mesh_nu)
    ctx = Context(device=-1)
    ctx.set_mesh(sc)
    n0, _ = ctx.build_cut(start)
    nodes0 = ctx.cut_nodes()
    ca, cb = ctx.base_bvh()
    rng = np.random.default_rng(start + splits)
    q = rng.uniform(0.05, 2.0, n0).astype(np.float32)
    p = rng.uniform(0.001, 0.2, n0).astype(np.float32)
    n1, _ = ctx.build_cut(n0 + splits, q=q, p=p)
    want = orc.expand_cut(ca, cb, nodes0, q.astype(np.float64), p.astype(np.float64), splits)
    assert np.array_equal(np.sort(ctx.cut_nodes()), want)
    assert n1 == want.size
    if mesh_nu == 2:
        assert np.any(cb[nodes0] < 0) and n1 < n0 + splits            # base leaves passed over


def test_construct_ranks_follow_the_oracle_statistics(orc):
    """construct.ranks_from_stats (the host side of NEXT-1) on the per-leaf sums the gradient
    buffer tail carries gives r = 2 ln q + ln p with the oracle's q, p from per-ray records."""
    from paper_2405_16237_b200.construct import ranks_from_stats
    rng = np.random.default_rng(9)
    n_rays, n_leaves = 5000, 37
    first = rng.integers(-1, n_leaves, n_rays)
    acc = (rng.random(n_rays) < 0.6) & (first >= 0)
    loss = rng.uniform(0.01, 3.0, n_rays)
    q, p, samples, ls = orc.leaf_error_stats(first, acc, loss, n_leaves)
    firsts = np.bincount(first[first >= 0], minlength=n_leaves)
    r, q2, p2 = ranks_from_stats(ls, samples, firsts, n_rays)
    ok = samples > 0
    assert ok.all()
    np.testing.assert_allclose(q2, q, rtol=1e-12)
    np.testing.assert_allclose(p2, p, rtol=1e-12)
    np.testing.assert_allclose(r, (2 * np.log(q) + np.log(p)).astype(np.float32), rtol=1e-6)
