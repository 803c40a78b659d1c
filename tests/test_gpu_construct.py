"""Error-driven construction and multi-cut LoD on the GPU.

NEXT-1 / NEXT-2 of SURVEY §8(f).  The construction trains the model through the library's
training step while splitting the leaves of largest rank r = 2 ln q + ln p; the checks are
structural (the cut is a valid cover of the mesh, LoD slots are nested coarse-to-fine and
share the grid), statistical (training reduces the loss) and a self-consistency quality
check against the exact geometry (P17 is "parity unpinned": no paper weights exist).
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _batch_fn(n, n_points, seed0):
    def f(step):
        rays = synth.random_rays(n, seed=seed0 + step)          # 50%-inflated box, uniform dirs
        u = synth.random_uniform(n, seed=seed0 + 100000 + step)
        xi = synth.random_uniform(n * n_points, seed=seed0 + 200000 + step).reshape(n, n_points)
        return tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (rays, u, xi))
    return f


@pytest.fixture(scope="module")
def built():
    from paper_2405_16237_b200 import Context
    from paper_2405_16237_b200.construct import construct, Schedule
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2, seed=5)
    ctx.set_mesh(sc)
    ctx.build_cut(1)
    ctx.reserve(1 << 14)
    hist = construct(ctx, 64, _batch_fn(1 << 13, 4, 1000),
                     Schedule(iters0=10, splits0=2, growth=1.6, final_iters=400, lod_every=40, max_lods=3))
    return ctx, sc, hist


def test_construction_reaches_target_and_valid_cut(orc, built):
    ctx, sc, hist = built
    cut = ctx.cut(0)
    assert cut["n_leaves"] == 64
    diag = float(np.linalg.norm(sc.verts.astype(np.float64).max(0) - sc.verts.astype(np.float64).min(0)))
    assert orc.check_cut(sc.verts, sc.tris, cut["tri_off"], cut["tris"], cut["base_lo"], cut["base_hi"],
                         cut["leaf_lo"], cut["leaf_hi"], diag) == 0
    # the leaf count grows round by round and the loss falls with training
    ns = [h.n_leaves for h in hist]
    assert ns[0] == 1 and all(b >= a for a, b in zip(ns, ns[1:])) and ns[-1] == 64
    assert hist[-1].loss < 0.8 * hist[0].loss, [h.loss for h in hist]


def test_lod_slots_nested_and_share_the_grid(orc, built):
    ctx, sc, hist = built
    lods = hist[-1].lods
    assert len(lods) >= 2
    counts = [ctx.cut(s)["n_leaves"] for s in lods] + [ctx.cut(0)["n_leaves"]]
    assert all(b >= a for a, b in zip(counts, counts[1:])) and counts[0] < counts[-1]
    d0 = ctx.cut(0)
    for s in lods:
        c = ctx.cut(s)
        assert np.array_equal(c["dom_min"], d0["dom_min"]) and c["dom_inv"][0] == d0["dom_inv"][0]   # C4'
        # every registered cut is a valid cover and is coarser than (an ancestor cut of) slot 0
        owner = np.empty(int(c["tri_off"][-1]), np.int64)
        for i in range(c["n_leaves"]):
            owner[c["tris"][c["tri_off"][i]:c["tri_off"][i + 1]]] = i
        for i in range(d0["n_leaves"]):
            tris = d0["tris"][d0["tri_off"][i]:d0["tri_off"][i + 1]]
            assert np.unique(owner[tris]).size == 1                 # fine leaf inside one coarse leaf


def test_trained_model_sees_the_geometry(orc, built):
    """Self-consistency (P17 unpinned): after construction + training, the neural hit mask of
    the tiny camera agrees with exact ray/triangle intersection on most rays, and LoD queries
    run on every registered cut."""
    ctx, sc, hist = built
    rays = synth.camera_rays(64, 64, (0.0, 0.0, 3.5), vfov_deg=40.0)
    out = ctx.query(torch.from_numpy(rays).cuda())
    torch.cuda.synchronize()
    hit = out["hit"].cpu().numpy()
    n = rays.shape[0]
    gt = orc.label(sc, np.array([0, sc.tris.shape[0]], np.int64), np.arange(sc.tris.shape[0], dtype=np.int32),
                   rays, np.zeros(n, np.int32), rays[:, 3].copy(), np.full(n, 1e30, np.float32))
    gt_hit = (gt[:, 0] == 0).astype(np.uint8)
    agree = (hit == gt_hit).mean()
    assert agree >= 0.85, agree
    for s in hist[-1].lods:
        o = ctx.query(torch.from_numpy(rays).cuda(), lod=s)
        torch.cuda.synchronize()
        assert (o["hit"].cpu().numpy() == gt_hit).mean() >= 0.7
