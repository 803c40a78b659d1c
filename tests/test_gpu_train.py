"""GPU parity of the companion training step against the oracle (double precision).

Exact: first-leaf selection and acceptance decisions (fp32 on both sides), ground-truth
visibility and hit distance (double Moller-Trumbore with the same op order).
Tolerances: labels' normal/albedo 1e-6; loss sums 5e-3 relative;
gradients (fp16 forward/backward operands, fp32 accumulation) 3e-2 relative L2 error per
parameter block and cosine >= 0.999; Adam 1e-5 relative.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _setup(n_rays=6000, seed=30, leaves=64, rank=None, hidden=2):
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    import oracle as orc
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=hidden)
    ctx.set_mesh(sc)
    ctx.build_cut(leaves)
    ctx.reserve(n_rays)
    tab = synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=seed, lo=-0.5, hi=0.5)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(64, hidden, 64, seed=seed + 1, out_scale=1.0)
    ctx.set_mlp(layers)
    cut = ctx.cut(0)
    if rank is None:
        rank = np.zeros(cut["n_leaves"], np.float32)
    ctx.set_leaf_rank(rank)
    rays = synth.random_rays(n_rays, seed=seed + 2)                     # 50%-inflated box (C16)
    u = synth.random_uniform(n_rays, seed=seed + 3)
    xi = synth.random_uniform(n_rays * 4, seed=seed + 4).reshape(n_rays, 4)
    o = orc.train_grad(orc.Grid(8, 14, 2), 4, tab.reshape(-1, 2), layers, cut["leaf_lo"], cut["leaf_hi"], rank,
                       cut["tri_off"], cut["tris"], sc, rays, u, xi, dom_box=orc.scene_box(sc))
    return ctx, sc, cut, tab, layers, rays, u, xi, o


def _to(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.fixture(scope="module")
def batch():
    rank = np.random.default_rng(5).normal(size=64).astype(np.float32) * 3     # varied acceptance
    return _setup(rank=rank)


def test_selection_and_labels_exact(batch):
    ctx, sc, cut, tab, layers, rays, u, xi, o = batch
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    gt, acc, leaf, loss = ctx.debug_train_samples(rays.shape[0])
    torch.cuda.synchronize()
    gt, acc, leaf = gt.cpu().numpy(), acc.cpu().numpy(), leaf.cpu().numpy()
    assert np.array_equal(leaf, o["first_leaf"])
    assert np.array_equal(acc, o["accepted"])
    a = acc == 1
    assert 0.1 < a.mean() < 0.9
    assert np.array_equal(gt[a, 0], o["gt"][a, 0].astype(np.float32))
    hit = a & (o["gt"][:, 0] == 0)
    assert hit.sum() > 100
    assert np.array_equal(gt[hit, 8], o["gt"][hit, 8].astype(np.float32))       # t_hit bits
    assert np.abs(gt[hit, 1] - o["gt"][hit, 1]).max() <= 1e-6
    assert np.abs(gt[hit, 2:8] - o["gt"][hit, 2:8]).max() <= 1e-6
    st = ctx.train_stats()
    assert st["n_accepted"] == o["n_acc"] and st["n_first_hit"] == int((o["first_leaf"] >= 0).sum())


def test_loss_and_gradients_vs_oracle(batch):
    from paper_2405_16237_b200 import dp
    ctx, sc, cut, tab, layers, rays, u, xi, o = batch
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    st = ctx.train_stats()
    assert abs(st["loss_sum"] - o["loss_sum"][0]) <= 5e-3 * abs(o["loss_sum"][0])
    g = dp.grad_tensor(ctx).cpu().numpy().astype(np.float64)
    n_t, n_w = tab.size, o["g_W"].size
    m = o["n_acc"]
    blocks = {"tables": (g[:n_t], o["g_table"] * m), "weights": (g[n_t:n_t + n_w], o["g_W"] * m),
              "biases": (g[n_t + n_w:n_t + n_w + o["g_b"].size], o["g_b"] * m)}
    for name, (gg, oo) in blocks.items():
        rel = np.linalg.norm(gg - oo) / np.linalg.norm(oo)
        cos = gg @ oo / (np.linalg.norm(gg) * np.linalg.norm(oo))
        assert rel <= 3e-2 and cos >= 0.999, (name, rel, cos)
    tail = g[n_t + n_w + o["g_b"].size:]
    assert tail[0] == m                                                        # accepted count
    per_leaf = tail[1:1 + 3 * cut["n_leaves"]].reshape(-1, 3)
    assert per_leaf[:, 1].sum() == m
    assert per_leaf[:, 2].sum() == (o["first_leaf"] >= 0).sum()
    assert abs(per_leaf[:, 0].sum() - o["loss_sum"][0]) <= 5e-3 * o["loss_sum"][0]


def test_table_gradient_support_matches_oracle(batch):
    """S:249 (gradient sparsity): the table entries with a non-zero gradient are exactly the
    corners the accepted samples touched (the oracle's support); an index error anywhere in
    the scatter (wrong level offset, corner, hash term) changes the set."""
    from paper_2405_16237_b200 import dp
    ctx, sc, cut, tab, layers, rays, u, xi, o = batch
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    g = dp.grad_tensor(ctx).cpu().numpy()[:tab.size].reshape(-1, 2)
    gs = np.any(g != 0, axis=1)
    os_ = np.any(o["g_table"].reshape(-1, 2) != 0, axis=1)
    assert os_.sum() > 1000
    assert (gs & ~os_).sum() == 0                                   # nothing outside the support
    assert (os_ & ~gs).sum() <= max(3, int(1e-3 * os_.sum()))       # fp cancellation to exactly 0 only


def test_query_bitwise_deterministic():
    """S:299 / S:670: the query path is bitwise reproducible run to run (no value depends on
    atomics order or scheduling)."""
    from paper_2405_16237_b200 import Context
    ctx, sc, cut, tab, layers, rays, u, xi, o = _setup(n_rays=20000, seed=60)
    d_rays = _to(rays)
    a = {k: v.clone() for k, v in ctx.query(d_rays).items()}
    for _ in range(3):
        b = ctx.query(d_rays)
        for k in a:
            assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("hidden", [2, 3])
@pytest.mark.parametrize("path", ["tcgen05", "mma_sync"])
def test_weight_gradients_per_layer(hidden, path, monkeypatch):
    """Per-layer weight and bias gradients vs the oracle, on both weight-gradient kernels:
    the tcgen05/TMEM contraction (k_train_dw_tc) and the mma.sync fallback (k_train_dw)."""
    from paper_2405_16237_b200 import dp
    if path == "mma_sync":
        monkeypatch.setenv("NBVH_DW_MMA_SYNC", "1")
    else:
        monkeypatch.delenv("NBVH_DW_MMA_SYNC", raising=False)
    ctx, sc, cut, tab, layers, rays, u, xi, o = _setup(n_rays=5000, seed=40 + hidden, hidden=hidden)
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    torch.cuda.synchronize()
    g = dp.grad_tensor(ctx).cpu().numpy().astype(np.float64)
    m = o["n_acc"]
    n_t = tab.size
    dims = [64] + [64] * hidden + [8]
    wo = n_t
    go = 0
    for k in range(len(dims) - 1):
        n = dims[k] * dims[k + 1]
        gg, oo = g[wo:wo + n], o["g_W"][go:go + n] * m
        rel = np.linalg.norm(gg - oo) / np.linalg.norm(oo)
        assert rel <= 3e-2, (path, hidden, k, rel)
        wo += n
        go += n
    nb = o["g_b"].size
    gb, ob = g[wo:wo + nb], o["g_b"] * m
    assert np.linalg.norm(gb - ob) / np.linalg.norm(ob) <= 3e-2


def test_gradients_paper_default_variant():
    """NEXT-4: F=4 (8-byte entries), n=3 points, 4 hidden layers (D_in = 96: the weight
    gradients fall back to the mma.sync kernel, Mtot = 288 > 256)."""
    from paper_2405_16237_b200 import Context, PARAM_TABLES, dp
    import oracle as orc
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=4, log2_T=18, n_points=3, hidden_layers=4)
    ctx.set_mesh(sc)
    ctx.build_cut(64)
    n = 4000
    ctx.reserve(n)
    tab = synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=50, lo=-0.5, hi=0.5)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(96, 4, 64, seed=51, out_scale=1.0)
    ctx.set_mlp(layers)
    cut = ctx.cut(0)
    rank = np.zeros(cut["n_leaves"], np.float32)
    ctx.set_leaf_rank(rank)
    rays = synth.random_rays(n, seed=52)
    u = synth.random_uniform(n, seed=53)
    xi = synth.random_uniform(n * 3, seed=54).reshape(n, 3)
    o = orc.train_grad(orc.Grid(8, 18, 4), 3, tab.reshape(-1, 4), layers, cut["leaf_lo"], cut["leaf_hi"], rank,
                       cut["tri_off"], cut["tris"], sc, rays, u, xi, dom_box=orc.scene_box(sc))
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    st = ctx.train_stats()
    assert st["n_accepted"] == o["n_acc"] and o["n_acc"] > 300
    assert abs(st["loss_sum"] - o["loss_sum"][0]) <= 5e-3 * abs(o["loss_sum"][0])
    g = dp.grad_tensor(ctx).cpu().numpy().astype(np.float64)
    m = o["n_acc"]
    n_t, n_w, n_b = tab.size, o["g_W"].size, o["g_b"].size
    for name, gg, oo in (("tables", g[:n_t], o["g_table"] * m), ("weights", g[n_t:n_t + n_w], o["g_W"] * m),
                         ("biases", g[n_t + n_w:n_t + n_w + n_b], o["g_b"] * m)):
        rel = np.linalg.norm(gg - oo) / np.linalg.norm(oo)
        assert rel <= 3e-2, (name, rel)


def test_adam_step_vs_oracle(batch):
    from paper_2405_16237_b200 import dp, PARAM_ALL
    import oracle as orc
    ctx, sc, cut, tab, layers, rays, u, xi, o = batch
    p0 = ctx.get_params(PARAM_ALL).astype(np.float64)
    ctx.set_params(PARAM_ALL, p0.astype(np.float32))                # also restarts Adam (step 1)
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    g = dp.grad_tensor(ctx).cpu().numpy().astype(np.float64)
    n_p = p0.size
    grad = g[:n_p] / max(1.0, g[n_p])
    ctx.apply_update(0.01)
    p1 = ctx.get_params(PARAM_ALL).astype(np.float64)
    ref = p0.copy()
    m = np.zeros_like(ref)
    v = np.zeros_like(ref)
    orc.adam(ref, grad, m, v, 1, lr=0.01)
    assert np.abs(p1 - ref).max() <= 1e-5 * (1 + np.abs(ref).max())


def test_two_half_batches_sum_to_full_batch():
    """DP decomposition on one GPU without cross-waiting kernels: the gradient buffers
    of two contexts over the two halves sum to the full-batch buffer (fp32 atomics)."""
    from paper_2405_16237_b200 import dp
    full = _setup(n_rays=4000, seed=40)
    ctx, sc, cut, tab, layers, rays, u, xi, o = full
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    g_full = dp.grad_tensor(ctx).clone()
    parts = []
    for r in range(2):
        sl = dp.shard(rays.shape[0], r, 2)
        ctx.train_backward(_to(rays[sl]), _to(u[sl]), _to(xi[sl]))
        parts.append(dp.grad_tensor(ctx).clone())
    s = (parts[0] + parts[1]).double()
    rel = (s - g_full.double()).norm() / g_full.double().norm()
    assert rel <= 1e-5, rel


def test_training_reduces_loss():
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2, seed=3)
    ctx.set_mesh(sc)
    ctx.build_cut(64)
    n = 1 << 15
    ctx.reserve(n)
    losses = []
    for step in range(150):
        rays = _to(synth.random_rays(n, seed=1000 + step))
        u = _to(synth.random_uniform(n, seed=2000 + step))
        xi = _to(synth.random_uniform(n * 4, seed=3000 + step).reshape(n, 4))
        ctx.train_step(rays, u, xi, lr=0.01)
        st = ctx.train_stats()
        losses.append(st["loss_sum"] / max(1, st["n_accepted"]))
    assert np.mean(losses[-10:]) < 0.6 * np.mean(losses[:5]), (losses[:5], losses[-10:])


def test_t0_generated_rays_match_oracle():
    """nbvh_gen_train_rays (T0, Philox-4x32-10 on the device) against the oracle's own Philox
    and recipe (C28'): origins, z, u, xi, tmin, tmax bit-exact; the direction's x, y within a
    few ulp (cos / sin); a data-parallel shard equals the slice of the whole batch; the
    default box is the scene box with every axis extent x1.5 (C16)."""
    import oracle as orc
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    ctx.set_mesh(sc)
    ctx.build_cut(16)
    n = 100000
    box = (-1.5, -1.25, -1.0, 1.5, 1.25, 1.0)
    rays, u, xi = (t.cpu().numpy() for t in ctx.gen_train_rays(seed=7, step=5, n=n, box=box))
    wr, wu, wxi = orc.gen_train_rays(7, 5, 0, n, box, 4)
    assert np.array_equal(rays[:, [0, 1, 2, 3, 6, 7]].view(np.uint32), wr[:, [0, 1, 2, 3, 6, 7]].view(np.uint32))
    assert np.array_equal(u.view(np.uint32), wu.view(np.uint32)) and np.array_equal(xi.view(np.uint32), wxi.view(np.uint32))
    assert np.abs(rays[:, 4:6] - wr[:, 4:6]).max() <= 4e-7
    r2, u2, x2 = (t.cpu().numpy() for t in ctx.gen_train_rays(seed=7, step=5, n=777, i0=4321, box=box))
    assert np.array_equal(r2, rays[4321:4321 + 777]) and np.array_equal(u2, u[4321:4321 + 777])
    # default box (C16): the scene's bounding box (no C15 padding), each axis extent x1.5
    rd, _, _ = (t.cpu().numpy() for t in ctx.gen_train_rays(seed=7, step=5, n=20000))
    b = orc.scene_box(sc, rel=0.0, abs_=0.0).astype(np.float64)
    ext = b[3:] - b[:3]
    mid = (b[:3] + b[3:]) / 2
    lo, hi = mid - 0.75 * ext, mid + 0.75 * ext
    assert np.all(rd[:, :3] >= lo - 1e-5) and np.all(rd[:, :3] <= hi + 1e-5)
    assert np.all(rd[:, :3].min(0) < lo + 0.05 * ext) and np.all(rd[:, :3].max(0) > hi - 0.05 * ext)


def test_tcgen05_weight_gradients_at_bench_size(monkeypatch):
    """k_train_dw_tc at the bench's size (2^20 rays on the 1080p scene: many K-chunks per CTA,
    ring-buffer reuse) against the mma.sync weight-gradient kernel on the same batch."""
    from paper_2405_16237_b200 import Context, PARAM_TABLES, dp
    c = synth.CONFIGS["1080p"]
    h = c["hash"]
    ctx = Context(device=0, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers)
    sc = synth.scene_1080p(c["seeds"]["mesh"])
    ctx.set_mesh(sc)
    ctx.build_cut(c["leaves"])
    n = 1 << 20
    ctx.reserve(n)
    ctx.set_params(PARAM_TABLES, synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=5).astype(np.float32))
    ctx.set_mlp(synth.random_mlp(ctx.d_in, h.hidden_layers, 64, seed=6, out_scale=1.0))
    ctx.set_leaf_rank(np.zeros(ctx.cut(0)["n_leaves"], np.float32))
    rays, u, xi = ctx.gen_train_rays(seed=7, step=1, n=n, box=None)      # C16 box, as bench.py
    n_t = ctx.param_count(PARAM_TABLES)
    n_w = ctx.param_count(1)                                        # PARAM_WEIGHTS
    grads = {}
    for path in ("tc", "mma"):
        if path == "mma":
            monkeypatch.setenv("NBVH_DW_MMA_SYNC", "1")
        else:
            monkeypatch.delenv("NBVH_DW_MMA_SYNC", raising=False)
        ctx.train_backward(rays, u, xi)
        grads[path] = dp.grad_tensor(ctx).cpu().numpy()[n_t:n_t + n_w].astype(np.float64)
    assert ctx.train_stats()["n_accepted"] > 100000
    a, b = grads["tc"], grads["mma"]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-3


def test_scatter_variants_at_bench_size(monkeypatch):
    """The hash-grid gradient scatter at the bench's size, three ways: the default
    warp-aggregated kernel (levels 0-5 grouped by cell), k_train_scatter with the coarse dense
    levels 0-2 in shared-memory fixed point (NBVH_SCATTER_AGG=0), and k_train_scatter with
    every level on global reductions (also NBVH_PRIV_BYTES=0): equal up to fp32 summation
    order, entry by entry (|a - b| <= 1e-4 |b| + 1e-6 max |b|)."""
    from paper_2405_16237_b200 import Context, PARAM_TABLES, dp
    c = synth.CONFIGS["1080p"]
    h = c["hash"]
    ctx = Context(device=0, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers)
    ctx.set_mesh(synth.scene_1080p(c["seeds"]["mesh"]))
    ctx.build_cut(c["leaves"])
    n = 1 << 19
    ctx.reserve(n)
    ctx.set_params(PARAM_TABLES, synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=5).astype(np.float32))
    ctx.set_mlp(synth.random_mlp(ctx.d_in, h.hidden_layers, 64, seed=6, out_scale=1.0))
    ctx.set_leaf_rank(np.zeros(ctx.cut(0)["n_leaves"], np.float32))
    rays, u, xi = ctx.gen_train_rays(seed=9, step=2, n=n, box=None)      # C16 box, as bench.py
    n_t = ctx.param_count(PARAM_TABLES)
    g = {}
    for name, env in (("agg", {}), ("priv", {"NBVH_SCATTER_AGG": "0"}),
                      ("global", {"NBVH_SCATTER_AGG": "0", "NBVH_PRIV_BYTES": "0"})):
        for k in ("NBVH_SCATTER_AGG", "NBVH_PRIV_BYTES"):
            if k in env:
                monkeypatch.setenv(k, env[k])
            else:
                monkeypatch.delenv(k, raising=False)
        ctx.train_backward(rays, u, xi)
        g[name] = dp.grad_tensor(ctx).cpu().numpy()[:n_t].astype(np.float64)
    b = g["global"]
    for name in ("agg", "priv"):
        a = g[name]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-4
        assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b) + 1e-6 * np.abs(b).max()), name


def test_training_step_at_bench_size_sampled_vs_oracle():
    """The training forward path at the bench's size (2^19 device-generated rays on the 1080p
    scene: grid-stride tiles in every kernel) against the oracle on a strided subset of the
    same rays: first leaf, acceptance and ground truth exact, per-sample loss within the
    fp16-network tolerance."""
    import oracle as orc
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    c = synth.CONFIGS["1080p"]
    h = c["hash"]
    sc = synth.scene_1080p(c["seeds"]["mesh"])
    ctx = Context(device=0, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers)
    ctx.set_mesh(sc)
    ctx.build_cut(c["leaves"])
    n = 1 << 19
    ctx.reserve(n)
    tab = synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=5, lo=-0.5, hi=0.5)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(ctx.d_in, h.hidden_layers, 64, seed=6, out_scale=1.0)
    ctx.set_mlp(layers)
    cut = ctx.cut(0)
    rank = np.random.default_rng(3).normal(size=cut["n_leaves"]).astype(np.float32)
    ctx.set_leaf_rank(rank)
    rays, u, xi = ctx.gen_train_rays(seed=11, step=4, n=n, box=None)      # C16 box, as bench.py
    ctx.train_backward(rays, u, xi)
    gt, acc, leaf, loss = (t.cpu().numpy() for t in ctx.debug_train_samples(n))
    sub = np.arange(0, n, 257)
    r_np, u_np, xi_np = rays.cpu().numpy()[sub], u.cpu().numpy()[sub], xi.cpu().numpy()[sub]
    o = orc.train_grad(orc.Grid(h.L, h.log2_T, h.F), h.n_points, tab.reshape(-1, h.F), layers, cut["leaf_lo"],
                       cut["leaf_hi"], rank, cut["tri_off"], cut["tris"], sc, r_np, u_np, xi_np,
                       dom_box=orc.scene_box(sc))
    assert np.array_equal(leaf[sub], o["first_leaf"]) and np.array_equal(acc[sub], o["accepted"])
    a = acc[sub] == 1
    assert a.sum() > 100
    assert np.array_equal(gt[sub][a, 0], o["gt"][a, 0].astype(np.float32))
    lg, lo_ = loss[sub][a].astype(np.float64), o["loss"][a]
    close = np.abs(lg - lo_) <= 5e-2 * np.abs(lo_) + 1e-3
    assert close.mean() >= 0.99, close.mean()


def test_nonfinite_gradient_skips_the_update():
    """S:254 / S:480 (SURVEY §5 failure detection): a non-finite value anywhere in the
    gradient buffer makes nbvh_apply_update skip the step -- parameters (and so the fp16
    inference copy) unchanged and NBVH_ENONFINITE reported by the stats call -- and the
    skipped steps do not advance Adam's step count: the next finite update is Adam step 1,
    equal to a fresh context's first update on the same batch."""
    from paper_2405_16237_b200 import Context, PARAM_ALL, dp
    from paper_2405_16237_b200.nbvh import NbvhError
    ctx, sc, cut, tab, layers, rays, u, xi, o = _setup(n_rays=3000, seed=80)
    p0 = ctx.get_params(PARAM_ALL)
    ctx.set_params(PARAM_ALL, p0)                                   # restarts Adam
    q0 = ctx.query(_to(rays[:500]))
    q0 = {k: v.clone() for k, v in q0.items()}
    for bad in (float("nan"), float("inf"), float("-inf")):
        ctx.train_backward(_to(rays), _to(u), _to(xi))
        g = dp.grad_tensor(ctx)
        g[len(p0) // 3] = bad
        ctx.apply_update(0.01)
        with pytest.raises(NbvhError) as ei:
            ctx.train_stats()
        assert ei.value.status == -4                                # NBVH_ENONFINITE
        assert np.array_equal(ctx.get_params(PARAM_ALL), p0)
    q1 = ctx.query(_to(rays[:500]))
    for k in q0:
        assert torch.equal(q0[k], q1[k]), k                         # inference copy untouched
    ctx.train_backward(_to(rays), _to(u), _to(xi))
    ctx.apply_update(0.01)
    assert ctx.train_stats()["skipped"] == 0
    p1 = ctx.get_params(PARAM_ALL)
    fresh = _setup(n_rays=3000, seed=80)[0]
    fresh.set_params(PARAM_ALL, p0)
    fresh.train_backward(_to(rays), _to(u), _to(xi))
    fresh.apply_update(0.01)
    p2 = fresh.get_params(PARAM_ALL)
    assert np.abs(p1 - p2).max() <= 1e-4                           # step 1, not step 4 (|diff| ~ 4e-3)
    assert np.abs(p1 - p0).max() > 5e-3


def test_dp_two_contexts_stay_byte_identical():
    """SURVEY §8(e) data parallelism on one GPU without cross-waiting kernels: two contexts,
    each holding half of every batch, sum their gradient buffers (the all-reduce), and both
    apply the update.  After several steps their parameters are byte-identical, and equal
    (to fp32 summation order) to one context trained on the whole batches."""
    from paper_2405_16237_b200 import PARAM_ALL, dp
    ranks = [_setup(n_rays=4000, seed=90)[0] for _ in range(2)]
    single = _setup(n_rays=4000, seed=90)[0]
    assert dp.param_checksum(ranks[0]) == dp.param_checksum(ranks[1]) == dp.param_checksum(single)
    for step in range(6):
        rays = synth.random_rays(4000, seed=500 + step)
        u = synth.random_uniform(4000, seed=600 + step)
        xi = synth.random_uniform(4000 * 4, seed=700 + step).reshape(4000, 4)
        bufs = []
        for r, ctx in enumerate(ranks):
            sl = dp.shard(4000, r, 2)
            ctx.train_backward(_to(rays[sl]), _to(u[sl]), _to(xi[sl]))
            bufs.append(dp.grad_tensor(ctx))
        total = bufs[0] + bufs[1]                                    # the all-reduce (sum)
        for b in bufs:
            b.copy_(total)
        for ctx in ranks:
            ctx.apply_update(0.01)
        single.train_backward(_to(rays), _to(u), _to(xi))
        single.apply_update(0.01)
        assert dp.param_checksum(ranks[0]) == dp.param_checksum(ranks[1]), step
    pa, ps = ranks[0].get_params(PARAM_ALL), single.get_params(PARAM_ALL)
    # summation order only: Adam's normalised steps move a parameter by ~lr, so an fp32-order
    # difference can flip a step only where the gradient is ~0 (a handful of entries)
    d = np.abs(pa - ps)
    assert np.median(d) <= 1e-6 and np.quantile(d, 0.99) <= 1e-2 * 0.01 and d.max() <= 6 * 2 * 0.01


def test_train_step_draws_its_own_rays():
    """nbvh_train_step with no rays: the library draws T0 itself -- Philox with
    key = the config's seed and step = its own batch counter, the C16 box -- so two self-drawn
    steps train on exactly the batches nbvh_gen_train_rays(seed, 0) and (seed, 1) give."""
    from paper_2405_16237_b200 import Context, PARAM_ALL
    sc = synth.scene_tiny()

    def mk():
        ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2, seed=5)
        ctx.set_mesh(sc)
        ctx.build_cut(64)
        ctx.reserve(1 << 14)
        return ctx

    a, b = mk(), mk()
    assert np.array_equal(a.get_params(PARAM_ALL), b.get_params(PARAM_ALL))
    n = 1 << 14
    for step in range(2):
        a.train_step(n=n, lr=0.01)
        sa = a.train_stats()
        rays, u, xi = b.gen_train_rays(seed=5, step=step, n=n)
        b.train_step(rays, u, xi, lr=0.01)
        sb = b.train_stats()
        assert sa["n_accepted"] == sb["n_accepted"] > 1000 and sa["n_first_hit"] == sb["n_first_hit"]
        assert abs(sa["loss_sum"] - sb["loss_sum"]) <= 1e-6 * abs(sb["loss_sum"])
    assert np.abs(a.get_params(PARAM_ALL) - b.get_params(PARAM_ALL)).max() <= 1e-4   # fp32 atomics order
