"""GPU parity of the query path (encode, MLP, traversal, full query) against the oracle.

All calls go through the C-ABI (libnbvh.so) via the thin binding; the oracle is the
plain CPU implementation in oracle/.  Tolerances:
  * indices, leaf lists, t_enter/t_exit, hit masks, winning leaves, query counts: exact
  * encode features (fp16 out, U[-1,1] tables): 2e-3 absolute
  * MLP: decoded outputs (sigmoid channels, unit normal) 1e-2 absolute; raw z 2e-2*(1+|z|)
  * end-to-end hit mask vs the double oracle: identical on rays whose decisive
    visibilities satisfy |sigmoid(z_vis)-0.5| >= 1e-2 and whose t comparisons are >= 5e-3
    apart (C30); band rays counted (< 1%; 2.5% for the paper-default variant, C35)
"""
import math

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _mk_ctx(cfg_name="tiny", scene=None, leaves=None, seed=2, list_cap=16, mode=0, table_seed=7, **over):
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    c = synth.CONFIGS[cfg_name]
    h = c["hash"]
    kw = dict(L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers,
              list_cap=list_cap, mode=mode)
    kw.update(over)
    ctx = Context(device=0, **kw)
    sc = scene if scene is not None else (synth.scene_tiny() if cfg_name == "tiny" else synth.scene_1080p())
    ctx.set_mesh(sc)
    ctx.build_cut(leaves or c["leaves"])
    ctx.reserve(20000)
    n_tab = ctx.param_count(PARAM_TABLES)
    tab = synth.random_params_fp16(n_tab, seed=table_seed)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(ctx.d_in, kw["hidden_layers"], 64, seed=seed)
    ctx.set_mlp(layers)
    return ctx, sc, tab.reshape(-1, kw["F"]), layers


@pytest.fixture(scope="module")
def tiny():
    return _mk_ctx("tiny")


def _grid(orc, ctx):
    return orc.Grid(ctx.cfg.L, ctx.cfg.log2_T, ctx.cfg.F)


# ------------------------------------------------------------------ encode
def test_encode_indices_exact_features_close(orc, tiny):
    ctx, sc, tab, layers = tiny
    rng = np.random.default_rng(0)
    pts = rng.random((20000, 3), dtype=np.float32)
    pts[:50] = 0.0
    pts[50:100] = 1.0
    pts[100:400] = (rng.integers(0, 1025, (300, 3)) / 1024.0).astype(np.float32)   # on cell faces
    feat, idx = ctx.debug_encode(torch.from_numpy(pts).cuda())
    want, widx = orc.encode_points(_grid(orc, ctx), tab, pts)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), widx)
    err = np.abs(feat.float().cpu().numpy() - want)
    assert err.max() <= 2e-3, err.max()


@pytest.mark.parametrize("L,F,npts,log2_T", [(16, 2, 4, 19), (8, 4, 3, 18), (4, 2, 4, 12)])
def test_encode_other_configs(orc, L, F, npts, log2_T):
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    ctx = Context(device=0, L=L, F=F, n_points=npts, log2_T=log2_T, hidden_layers=2)
    n = ctx.param_count(PARAM_TABLES)
    tab = synth.random_params_fp16(n, seed=3)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    pts = np.random.default_rng(1).random((5000, 3), dtype=np.float32)
    feat, idx = ctx.debug_encode(torch.from_numpy(pts).cuda())
    want, widx = orc.encode_points(orc.Grid(L, log2_T, F), tab.reshape(-1, F), pts)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32), widx)
    assert np.abs(feat.float().cpu().numpy() - want).max() <= 2e-3


# ------------------------------------------------------------------ MLP
def _sig(z):
    return 1 / (1 + np.exp(-z))


def _z_abs(layers, x):
    """Magnitude of the MLP's forward (|W| |h| + |b| per layer, ReLU masks of the true
    forward): the scale of the rounding error of each fp16 activation."""
    h, ha = x.astype(np.float64), np.abs(x.astype(np.float64))
    for k, (W, b) in enumerate(layers):
        W = W.astype(np.float64)
        pre, pa = h @ W.T + b, ha @ np.abs(W).T + np.abs(b)
        if k + 1 < len(layers):
            h, ha = np.maximum(pre, 0.0), np.where(pre > 0, pa, 0.0)
        else:
            h, ha = pre, pa
    return ha


@pytest.mark.parametrize("d_in,hidden", [(64, 2), (128, 3), (96, 4), (32, 1)])
def test_mlp_tensor_core_vs_oracle(orc, d_in, hidden):
    """nbvh_debug_mlp runs k_query's own per-warp MLP (query_mlp_rows16: fp16 operands, fp32
    accumulation, hidden activations rounded to fp16).  Raw z vs the double oracle on the
    same fp16 inputs: within the rounding bound H 2^-11 z_abs, and within north_star's 1e-2
    absolute tier on every row."""
    from paper_2405_16237_b200 import Context
    L, F, npts = {64: (8, 2, 4), 128: (16, 2, 4), 96: (8, 4, 3), 32: (4, 2, 4)}[d_in]
    ctx = Context(device=0, L=L, F=F, n_points=npts, hidden_layers=hidden)
    layers = synth.random_mlp(d_in, hidden, 64, seed=5)
    ctx.set_mlp(layers)
    m = 1000 + 77                                              # ragged tail over 128-row tiles
    x = (np.random.default_rng(2).random((m, d_in)) * 0.8 - 0.4).astype(np.float16)
    z = ctx.debug_mlp(torch.from_numpy(x).cuda()).cpu().numpy()
    want = orc.mlp_forward(layers, x.astype(np.float64))
    err = np.abs(z - want)
    assert np.all(err <= hidden * 2.0 ** -11 * _z_abs(layers, x) + 1e-5), err.max()
    assert err.max() <= 1e-2, err.max()
    for ch in (1, 5, 6, 7):
        assert np.abs(_sig(z[:, ch]) - _sig(want[:, ch])).max() <= 1e-2
    agree = np.sign(z[:, 0]) == np.sign(want[:, 0])
    band = np.abs(_sig(want[:, 0]) - 0.5) < 1e-2
    assert np.all(agree | band)


@pytest.mark.parametrize("d_in,hidden", [(64, 2), (128, 3), (96, 4), (32, 1), (128, 1)])
def test_mlp_tcgen05_vs_oracle(orc, d_in, hidden):
    """The tcgen05/TMEM/TMA batched MLP (nbvh_mlp_forward) vs the double-precision oracle, on a
    ragged batch (the last 128-row tile is partly out of range: TMA zero-fills it)."""
    from paper_2405_16237_b200 import Context
    L, F, npts = {64: (8, 2, 4), 128: (16, 2, 4), 96: (8, 4, 3), 32: (4, 2, 4)}[d_in]
    ctx = Context(device=0, L=L, F=F, n_points=npts, hidden_layers=hidden)
    layers = synth.random_mlp(d_in, hidden, 64, seed=6)
    ctx.set_mlp(layers)
    m = 3 * 1024 + 77
    x = (np.random.default_rng(3).random((m, d_in)) * 0.8 - 0.4).astype(np.float16)
    z = ctx.mlp_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    want = orc.mlp_forward(layers, x.astype(np.float64))
    assert np.all(np.abs(z - want) <= 2e-2 * (1 + np.abs(want))), np.abs(z - want).max()
    zs = ctx.debug_mlp(torch.from_numpy(x).cuda()).cpu().numpy()            # the mma.sync path
    assert np.all(np.abs(z - zs) <= 2e-2 * (1 + np.abs(zs)))


# ------------------------------------------------------------------ traversal
def _rays_tiny(n_random=3000):
    cam = synth.camera_rays(64, 64, (0.0, 0.0, 3.5), vfov_deg=40.0)
    rnd = synth.random_rays(n_random, seed=11)
    return np.concatenate([cam, rnd], 0)


@pytest.mark.parametrize("cap", [24])
def test_traversal_lists_bit_exact(orc, tiny, cap):
    ctx, sc, tab, layers = tiny
    rays = _rays_tiny()
    cut = ctx.cut(0)
    leaf, te, tx, cnt = ctx.debug_traverse(torch.from_numpy(rays).cuda(), cap)
    wl, wte, wtx, wcnt = orc.leaf_lists(rays, cut["leaf_lo"], cut["leaf_hi"], cap)
    assert np.array_equal(cnt.cpu().numpy(), wcnt)
    assert np.array_equal(leaf.cpu().numpy(), wl)
    m = wl >= 0
    assert np.array_equal(te.cpu().numpy()[m], wte[m]) and np.array_equal(tx.cpu().numpy()[m], wtx[m])
    assert wcnt.max() >= 8                # depth of the tiny 64-leaf cut on these rays (oracle: 8);
                                          # resumption past K: test_traversal_small_capacity


def test_traversal_small_capacity(orc):
    ctx, sc, tab, layers = _mk_ctx("tiny", list_cap=3)
    rays = _rays_tiny(1000)
    cut = ctx.cut(0)
    leaf, te, tx, cnt = ctx.debug_traverse(torch.from_numpy(rays).cuda(), 12)
    wl, wte, wtx, wcnt = orc.leaf_lists(rays, cut["leaf_lo"], cut["leaf_hi"], 12)
    assert np.array_equal(leaf.cpu().numpy(), wl) and np.array_equal(cnt.cpu().numpy(), wcnt)
    m = wl >= 0
    assert np.array_equal(te.cpu().numpy()[m], wte[m]) and np.array_equal(tx.cpu().numpy()[m], wtx[m])
    assert wcnt.max() > 3                                      # resumption past the capacity (C6)


@pytest.mark.parametrize("cfg_name,list_cap,packet", [("tiny", 3, False), ("tiny", 12, False), ("tiny", 16, False),
                                                      ("tiny", 12, True), ("1080p", 12, False)])
def test_product_traversal_lists_exact(orc, monkeypatch, cfg_name, list_cap, packet):
    """The PRODUCT traversal (k_traverse, as nbvh_query launches it) against the oracle's
    brute-force (t_enter, id)-ordered lists: the first K = list_cap entries bit-exact (ids,
    t_enter, t_exit), fill = min(count, K), and the resume flag set wherever the ray
    intersects more than K leaves (C6; it may also be set conservatively when a pruned
    subtree's box is hit but none of its leaves are)."""
    if packet:
        monkeypatch.setenv("NBVH_TRAVERSE", "packet")
    else:
        monkeypatch.delenv("NBVH_TRAVERSE", raising=False)
    ctx, sc, tab, layers = _mk_ctx(cfg_name, list_cap=list_cap, table_seed=9, seed=6)
    if cfg_name == "tiny":
        rays = _rays_tiny(4000)
        sample = np.arange(rays.shape[0])
    else:
        c = synth.CONFIGS["1080p"]
        rays = synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"])
        sample = np.arange(0, rays.shape[0], 1031)
    ctx.reserve(rays.shape[0])
    leaf, te, tx, fill, more = (t.cpu().numpy() for t in ctx.debug_traverse_product(torch.from_numpy(rays).cuda()))
    cut = ctx.cut(0)
    wl, wte, wtx, wcnt = orc.leaf_lists(rays[sample], cut["leaf_lo"], cut["leaf_hi"], list_cap)
    leaf, te, tx, fill, more = leaf[sample], te[sample], tx[sample], fill[sample], more[sample]
    assert np.array_equal(fill, np.minimum(wcnt, list_cap))
    assert np.array_equal(leaf, wl)
    m = wl >= 0
    assert np.array_equal(te[m], wte[m]) and np.array_equal(tx[m], wtx[m])
    assert np.all(more[wcnt > list_cap] == 1)
    assert np.all(more[fill < list_cap] == 0)                   # nothing can be pruned below K
    if list_cap == 3:
        assert (wcnt > list_cap).sum() > 100                      # overflow exercised
    assert fill.max() >= min(list_cap, 4)


# ------------------------------------------------------------------ end-to-end query
def _check_query(orc, ctx, tab, layers, rays, mode=0, cap=64, lod=0, band_max=0.01, tband=5e-3, ztol=2e-2,
                 dec_tol=1e-2):
    cut = ctx.cut(lod)
    out, zt = ctx.debug_query_trace(torch.from_numpy(rays).cuda(), cap, lod=lod)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    zt = zt.cpu().numpy()
    # (1) logic replay of the GPU's own z values: exact
    rep = orc.replay(cut["leaf_lo"], cut["leaf_hi"], rays, zt, mode=mode)
    assert rep["missing"] == 0
    assert np.array_equal(g["hit"], rep["hit"])
    assert np.array_equal(g["leaf"], rep["leaf"])
    assert np.array_equal(g["n_queries"], rep["nq"])
    assert np.array_equal(g["t"].view(np.uint32), rep["t"].view(np.uint32))
    assert np.abs(g["normal"] - rep["normal"]).max() <= 1e-6
    assert np.abs(g["albedo"] - rep["albedo"]).max() <= 1e-6
    # (2) the double-precision oracle
    o = orc.query(_grid(orc, ctx), ctx.cfg.n_points, tab, layers, cut["leaf_lo"], cut["leaf_hi"], rays, mode=mode,
                  trace_cap=cap, dom_box=orc.scene_box(ctx.scene))
    clear = (o["margin"] >= 1e-2) & (o["tmargin"] >= tband)
    assert np.array_equal(g["hit"][clear], o["hit"][clear])
    assert np.array_equal(g["leaf"][clear], o["leaf"][clear])
    assert np.array_equal(g["n_queries"][clear], o["nq"][clear])
    assert (~clear).mean() < band_max, (~clear).mean()             # C30 band (< 1%)
    h = clear & (o["hit"] == 1)
    assert np.abs(g["t"][h] - o["t"][h]).max() <= 2e-3 * 3.5     # C23: t / scene diagonal
    assert np.abs(g["albedo"][h] - o["albedo"][h]).max() <= dec_tol
    assert np.abs(g["normal"][h] - o["normal"][h]).max() <= dec_tol
    # traced z vs oracle z for every query both made
    both = ~np.isnan(zt[..., 0]) & ~np.isnan(o["z_trace"][..., 0])
    zg, zo = zt[both], o["z_trace"][both]
    assert np.all(np.abs(zg - zo) <= ztol * (1 + np.abs(zo))), (np.abs(zg - zo) / (1 + np.abs(zo))).max()
    return g, o


def test_query_tiny_end_to_end(orc, tiny):
    ctx, sc, tab, layers = tiny
    g, o = _check_query(orc, ctx, tab, layers, _rays_tiny())
    assert g["hit"].sum() > 500 and g["n_queries"].max() >= 2


@pytest.mark.parametrize("over", [dict(n_points=2), dict(n_points=1, L=16)])
def test_query_other_point_counts(orc, over):
    """k_query_warp derives each row's sample points from its slot (no point tile; the two
    half-warps take points of opposite parity): n = 2 (one point per half-warp) and n = 1 (the
    second half-warp idle in the encode), end to end against the oracle.  What this test
    targets is the exact part (replay, and hit / leaf / query count on every ray outside the
    ambiguity band); the band's size is a property of the random decoder, and at D_in = 32
    it is larger than the main configurations' 1% (1.4% measured), so it is bounded at 3%."""
    ctx, sc, tab, layers = _mk_ctx("tiny", **over)
    g, o = _check_query(orc, ctx, tab, layers, _rays_tiny(), band_max=0.03)
    assert g["hit"].sum() > 100 and g["n_queries"].max() >= 2


def test_query_first_hit_mode(orc):
    ctx, sc, tab, layers = _mk_ctx("tiny", mode=1)
    _check_query(orc, ctx, tab, layers, _rays_tiny(), mode=1)


def test_query_refill_path(orc):
    ctx, sc, tab, layers = _mk_ctx("tiny", list_cap=2)
    g, _ = _check_query(orc, ctx, tab, layers, _rays_tiny())
    assert ctx.query_stats()["n_refills"] > 0


def test_query_single_leaf_and_empty(orc):
    ctx, sc, tab, layers = _mk_ctx("tiny", leaves=1)
    rays = _rays_tiny(500)
    g, o = _check_query(orc, ctx, tab, layers, rays)
    assert np.all(g["n_queries"] <= 1)
    out = ctx.query(torch.zeros(0, 8, device="cuda"))            # n = 0 is a no-op
    assert out["hit"].numel() == 0


def test_query_lod_slots(orc):
    """Multi-cut LoD: three cuts of one hash grid in slots 0-2; every slot's query is
    checked against the oracle on that slot's leaf boxes (grid domain shared, C4')."""
    ctx, sc, tab, layers = _mk_ctx("tiny", leaves=64)
    ctx.build_cut(8, lod=1)
    ctx.build_cut(24, lod=2)
    rays = _rays_tiny(1500)
    for lod in (2, 1, 0):
        g, o = _check_query(orc, ctx, tab, layers, rays, lod=lod)
        assert g["n_queries"].max() >= 1
    assert ctx.cut(1)["n_leaves"] == 8 and ctx.cut(2)["n_leaves"] == 24


def test_query_paper_default_variant(orc):
    """NEXT-4: the paper's own model shape (L=8, F=4, T=2^18, n=3, 4x64 MLP; D_in = 96)."""
    ctx, sc, tab, layers = _mk_ctx("paper")
    assert ctx.d_in == 96
    # C35: this 4-hidden-layer model's logits spread less under the same He x10 recipe
    # (std 2.7 vs 3.8): 2.2% of its rays are in the band, computed by the oracle alone.
    g, o = _check_query(orc, ctx, tab, layers, _rays_tiny(1500), band_max=0.025)
    assert g["hit"].sum() > 200


def test_query_host_path_equals_device_path(tiny):
    ctx, sc, tab, layers = tiny
    rays = _rays_tiny()
    d = {k: v.cpu().numpy() for k, v in ctx.query(torch.from_numpy(rays).cuda()).items()}
    h = ctx.query_host(rays)
    for k in d:
        assert np.array_equal(d[k].reshape(h[k].shape), h[k]), k


def test_query_host_path_chunked_interleaved(tiny):
    """Multi-chunk host path (n >= 2^18: block-interleaved chunks, strided 2-D copies, a ragged
    partial block) returns exactly what the device path returns."""
    ctx, sc, tab, layers = tiny
    cam = synth.camera_rays(600, 512, (0.0, 0.0, 3.5), vfov_deg=40.0)
    rays = np.concatenate([cam, synth.random_rays(1237, seed=21)], 0)       # 308,437 rays
    ctx.reserve(rays.shape[0])
    d = {k: v.cpu().numpy() for k, v in ctx.query(torch.from_numpy(rays).cuda()).items()}
    h = ctx.query_host(rays)
    for k in d:
        assert np.array_equal(d[k].reshape(h[k].shape), h[k]), k
    assert d["hit"].sum() > 1000


def test_query_1080p_sampled_full_size(orc):
    """cfg 2 at full size in the bench's launch configuration; sampled rays vs oracle."""
    ctx, sc, tab, layers = _mk_ctx("1080p", table_seed=9, seed=6)
    c = synth.CONFIGS["1080p"]
    rays = synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"])
    ctx.reserve(rays.shape[0])
    out = ctx.query(torch.from_numpy(rays).cuda())
    torch.cuda.synchronize()
    st = ctx.query_stats()
    assert st["n_rays"] == rays.shape[0] and st["n_queries"] > rays.shape[0] // 2
    sample = np.arange(0, rays.shape[0], 4099)
    cut = ctx.cut(0)
    o = orc.query(_grid(orc, ctx), 4, tab, layers, cut["leaf_lo"], cut["leaf_hi"], rays[sample],
                  dom_box=orc.scene_box(sc))
    g = {k: v.cpu().numpy()[sample] for k, v in out.items()}
    clear = (o["margin"] >= 1e-2) & (o["tmargin"] >= 5e-3)
    assert np.array_equal(g["hit"][clear], o["hit"][clear])
    assert np.array_equal(g["leaf"][clear], o["leaf"][clear])
    assert np.array_equal(g["n_queries"][clear], o["nq"][clear])
    h = clear & (o["hit"] == 1)
    assert h.sum() > 50
    assert np.abs(g["t"][h] - o["t"][h]).max() <= 2e-3 * 2.9


def test_gather_probe_runs_and_validates():
    """nbvh_gather_probe (the §8(d) random-gather roofline): issues at least the requested
    gathers, touches only the table (the XOR sink is reproducible for a fixed seed), and
    rejects bad arguments."""
    from paper_2405_16237_b200.nbvh import gather_probe, NbvhError
    tab = torch.arange(1 << 16, dtype=torch.int32, device="cuda")
    sink = torch.empty(148 * 8 * 256 * 2, dtype=torch.int32, device="cuda")
    for eb in (4, 32):
        n = gather_probe(tab, eb, 1 << 20, sink, seed=3)
        assert n >= 1 << 20
        a = sink.clone()
        gather_probe(tab, eb, 1 << 20, sink, seed=3)
        assert torch.equal(a, sink)
    with pytest.raises(NbvhError):
        gather_probe(tab, 8, 1 << 20, sink)
    with pytest.raises(NbvhError):
        gather_probe(tab[:3 * 4096], 4, 1 << 20, sink)          # not a power of two
    # the texture-pipe probe reads the same entries: with the same seed, the TEX-only run's
    # XOR sink equals the load-pipe run's (same chains, same addresses)
    from paper_2405_16237_b200.nbvh import gather_probe_tex
    gather_probe(tab, 4, 1 << 20, sink, seed=5)
    ldg = sink.clone()
    assert gather_probe_tex(tab, 1 << 20, sink, seed=5) >= 1 << 20
    assert torch.equal(ldg, sink)
    assert gather_probe_tex(tab, 1 << 20, sink, mixed=True, seed=5) >= 1 << 20
    assert torch.equal(ldg, sink)
    with pytest.raises(NbvhError):
        gather_probe_tex(tab[:3 * 4096], 1 << 20, sink)


def test_query_host_path_full_frame():
    """The host path at the bench's full size (6 block-interleaved chunks on two query streams,
    strided copies) returns exactly what the device path returns, twice in a row."""
    ctx, sc, tab, layers = _mk_ctx("1080p", table_seed=9, seed=6, list_cap=12)
    c = synth.CONFIGS["1080p"]
    rays = synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"])
    ctx.reserve(rays.shape[0])
    d = {k: v.cpu().numpy() for k, v in ctx.query(torch.from_numpy(rays).cuda()).items()}
    for _ in range(2):
        h = ctx.query_host(rays)
        for k in d:
            assert np.array_equal(d[k].reshape(h[k].shape), h[k]), k
    assert ctx.query_stats()["n_queries"] > rays.shape[0] // 2


def test_atomic_probe_counts_every_reduction():
    """nbvh_atomic_probe (the §8(d) scatter roofline): the table's sum equals the number of
    reductions issued (each adds 1 per component), and bad arguments are rejected."""
    from paper_2405_16237_b200.nbvh import atomic_probe, NbvhError
    for vec in (1, 2, 4):
        tab = torch.zeros(1 << 16, dtype=torch.float32, device="cuda")
        n = atomic_probe(tab, vec, 1 << 20)
        torch.cuda.synchronize()
        assert n >= 1 << 20 and int(tab.double().sum().item()) == n * vec
    with pytest.raises(NbvhError):
        atomic_probe(torch.zeros(3 << 10, device="cuda"), 1, 1 << 10)


def _degenerate_rays():
    """Axis-aligned directions (zero components: 1/d = inf in the slab test), origins inside
    and outside the geometry, rays starting on a box plane, finite [tmin, tmax] windows that
    clip the scene, an empty window (tmin > tmax) and a zero-length window."""
    rng = np.random.default_rng(5)
    rays = []
    axes = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1), (0.6, 0.8, 0), (0, -0.6, 0.8)]
    for d in axes:
        for _ in range(40):
            o = rng.uniform(-1.6, 1.6, 3)
            o[np.nonzero(d)[0][0]] = -2.5 * np.sign(d[np.nonzero(d)[0][0]])      # start outside, facing in
            rays.append([*o, 0.0, *d, np.inf])
    for _ in range(60):                                                        # inside the sphere shell
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        rays.append([*rng.uniform(-0.3, 0.3, 3), 0.0, *d, np.inf])
    for _ in range(60):                                                        # clipped windows
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        o = -3.0 * d + rng.uniform(-0.2, 0.2, 3)
        t0 = rng.uniform(0.0, 2.5)
        rays.append([*o, t0, *d, t0 + rng.uniform(0.05, 1.5)])
    rays.append([0.0, 0.0, 3.0, 2.0, 0.0, 0.0, -1.0, 1.0])                    # tmin > tmax
    rays.append([0.0, 0.0, 3.0, 2.0, 0.0, 0.0, -1.0, 2.0])                    # zero-length window
    rays.append([1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0, np.inf])                  # grazing along a plane
    return np.asarray(rays, np.float32)


@pytest.mark.parametrize("list_cap", [1, 16])
def test_query_degenerate_rays_and_list_extremes(orc, list_cap):
    """Edge cases of the query path against the oracle (logic replay exact, double oracle
    within tolerance): zero direction components, clipped / empty ray windows, origins
    inside the geometry, at the smallest (1) and largest (16) per-ray list capacity."""
    ctx, sc, tab, layers = _mk_ctx("tiny", list_cap=list_cap)
    rays = _degenerate_rays()
    g, o = _check_query(orc, ctx, tab, layers, rays)
    assert g["hit"][-3] == 0 and g["hit"][-2] == 0                           # empty / zero windows
    assert g["hit"].sum() > 10 and g["n_queries"].sum() > 300


def test_query_kernel_variants(orc, monkeypatch):
    """The two query kernels: the default per-warp one (mma.sync MLP of each warp's 16 rows)
    and NBVH_QUERY_MLP=tc, the warp-specialised one (the decoder MLP of 128-row tiles on
    tcgen05 in an MLP warpgroup, worker warps with two slot sets).  Each passes the parity
    checks (logic replay exact, double oracle within tolerance) on the tiny scene; on the 1080p
    frame at full size they agree on every decision except rays whose z differs by fp32
    summation order."""
    for variant in ("tc", "warp"):
        monkeypatch.setenv("NBVH_QUERY_MLP", variant)
        ctx, sc, tab, layers = _mk_ctx("tiny")
        _check_query(orc, ctx, tab, layers, _rays_tiny())
    # per-warp kernel A/B hook: fewer warps per CTA
    for env in (dict(NBVH_QUERY_WARPS="5"),):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        ctx, sc, tab, layers = _mk_ctx("tiny")
        _check_query(orc, ctx, tab, layers, _rays_tiny())
        for k in env:
            monkeypatch.delenv(k)
    ctx2, sc2, tab2, layers2 = _mk_ctx("1080p", table_seed=9, seed=6, list_cap=12)
    c = synth.CONFIGS["1080p"]
    rays = torch.from_numpy(synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"])).cuda()
    ctx2.reserve(rays.shape[0])
    monkeypatch.setenv("NBVH_QUERY_MLP", "tc")
    t = {k: v.cpu().numpy() for k, v in ctx2.query(rays).items()}
    st = ctx2.query_stats()
    assert st["n_mlp_tiles"] > 0 and st["n_mlp_rows"] == st["n_queries"]        # every query on tcgen05
    monkeypatch.setenv("NBVH_QUERY_MLP", "warp")
    m = {k: v.cpu().numpy() for k, v in ctx2.query(rays).items()}
    assert ctx2.query_stats()["n_mlp_tiles"] == 0
    assert (t["hit"] != m["hit"]).mean() < 1e-3 and (t["leaf"] != m["leaf"]).mean() < 2e-3
    same = (t["hit"] == 1) & (m["hit"] == 1) & (t["leaf"] == m["leaf"])
    assert np.abs(t["t"][same] - m["t"][same]).max() < 1e-2


def test_query_ws_drain_and_partial_tiles(orc, monkeypatch):
    """The warp-specialised kernel's drain path: ray counts that leave partly claimed feature
    tiles (1, 7, 17, 129, 1000 rays, fewer rays than worker slots) finish and match the
    replay of their own z trace exactly."""
    monkeypatch.setenv("NBVH_QUERY_MLP", "tc")
    ctx, sc, tab, layers = _mk_ctx("tiny")
    base = _rays_tiny(1000)
    for n in (1, 7, 17, 129, 1000):
        rays = base[:n]
        cut = ctx.cut(0)
        out, zt = ctx.debug_query_trace(torch.from_numpy(rays).cuda(), 32)
        torch.cuda.synchronize()
        g = {k: v.cpu().numpy() for k, v in out.items()}
        rep = orc.replay(cut["leaf_lo"], cut["leaf_hi"], rays, zt.cpu().numpy())
        assert rep["missing"] == 0
        assert np.array_equal(g["hit"], rep["hit"]) and np.array_equal(g["leaf"], rep["leaf"])
        assert np.array_equal(g["n_queries"], rep["nq"])
        assert ctx.query_stats()["n_mlp_rows"] == int(g["n_queries"].sum())


def test_query_small_batches_tail_rows(orc):
    """The default kernel with fewer rays than a warp's slots from the start: every iteration
    runs with <= 8 occupied rows, where each row's chunks are spread over 4-32 lanes (the
    tail encode path), and rays whose lists need refills.  Ray counts 1, 2, 3, 5, 9, 17, 33;
    every hit record and query count equals the replay of the kernel's own z trace, and the
    decided rays agree with the double oracle."""
    ctx, sc, tab, layers = _mk_ctx("tiny", list_cap=2)
    base = _rays_tiny(2000)
    cut = ctx.cut(0)
    _, _, _, cnt = orc.leaf_lists(base, cut["leaf_lo"], cut["leaf_hi"], 1)
    live = base[cnt >= 2][:200]                      # rays with >= 2 leaves (refills at K = 2)
    assert live.shape[0] >= 33
    for n in (1, 2, 3, 5, 9, 17, 33):
        rays = np.ascontiguousarray(live[:n])
        out, zt = ctx.debug_query_trace(torch.from_numpy(rays).cuda(), 32)
        torch.cuda.synchronize()
        g = {k: v.cpu().numpy() for k, v in out.items()}
        rep = orc.replay(cut["leaf_lo"], cut["leaf_hi"], rays, zt.cpu().numpy())
        assert rep["missing"] == 0
        assert np.array_equal(g["hit"], rep["hit"]) and np.array_equal(g["leaf"], rep["leaf"])
        assert np.array_equal(g["n_queries"], rep["nq"])
        assert np.array_equal(g["t"].view(np.uint32), rep["t"].view(np.uint32))
    _check_query(orc, ctx, tab, layers, np.ascontiguousarray(live[:33]), band_max=0.1)


def test_query_host_path_first_hit_mode_and_lod(monkeypatch):
    """The host path with R1 (first confident hit, C5) and with a non-zero LoD slot returns
    exactly the device path's records."""
    ctx, sc, tab, layers = _mk_ctx("tiny", mode=1)
    ctx.copy_cut(0, 2)
    cam = synth.camera_rays(600, 512, (0.0, 0.0, 3.5), vfov_deg=40.0)
    ctx.reserve(cam.shape[0])
    for lod in (0, 2):
        d = {k: v.cpu().numpy() for k, v in ctx.query(torch.from_numpy(cam).cuda(), lod=lod).items()}
        h = ctx.query_host(cam, lod=lod)
        for k in d:
            assert np.array_equal(d[k].reshape(h[k].shape), h[k]), (lod, k)
        assert d["hit"].sum() > 1000


@pytest.mark.parametrize("d_in,hidden", [(128, 3), (96, 4), (32, 2)])
def test_mlp_tcgen05_many_tiles_per_slot(orc, d_in, hidden):
    """The persistent tcgen05 MLP when every CTA runs several tiles through each slot (stage
    reuse, mbarrier phase flips, aliased X/H buffers): all rows vs the mma.sync path, a strided
    sample vs the double oracle."""
    from paper_2405_16237_b200 import Context
    L, F, npts = {64: (8, 2, 4), 128: (16, 2, 4), 96: (8, 4, 3), 32: (4, 2, 4)}[d_in]
    ctx = Context(device=0, L=L, F=F, n_points=npts, hidden_layers=hidden)
    layers = synth.random_mlp(d_in, hidden, 64, seed=8)
    ctx.set_mlp(layers)
    m = 148 * 5 * 4 * 128 + 77                                   # ~4 uses of each of 5 slots per CTA
    x = torch.rand(m, d_in, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4))
    x = (x * 0.8 - 0.4).half()
    z = ctx.mlp_forward(x).cpu().numpy()
    zs = ctx.debug_mlp(x).cpu().numpy()
    assert np.all(np.abs(z - zs) <= 2e-2 * (1 + np.abs(zs)))
    idx = np.arange(0, m, 97)
    want = orc.mlp_forward(layers, x.cpu().numpy()[idx].astype(np.float64))
    assert np.all(np.abs(z[idx] - want) <= 2e-2 * (1 + np.abs(want)))


@pytest.mark.parametrize("cfg_name,list_cap", [("tiny", 3), ("tiny", 12), ("1080p", 12)])
def test_packet_traversal_identical(monkeypatch, cfg_name, list_cap):
    """NBVH_TRAVERSE=packet (one node stack per warp, per-lane lists and votes) produces the
    same per-ray lists as the per-thread traversal: the whole query output is bit-identical,
    on coherent camera rays and on incoherent random rays."""
    ctx, sc, tab, layers = _mk_ctx(cfg_name, list_cap=list_cap, table_seed=9, seed=6)
    if cfg_name == "tiny":
        rays = _rays_tiny(5000)
    else:
        c = synth.CONFIGS["1080p"]
        rays = np.concatenate([synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"]),
                               synth.random_rays(100000, seed=3)])
    ctx.reserve(rays.shape[0])
    d_rays = torch.from_numpy(rays).cuda()
    monkeypatch.delenv("NBVH_TRAVERSE", raising=False)
    a = {k: v.clone() for k, v in ctx.query(d_rays).items()}
    monkeypatch.setenv("NBVH_TRAVERSE", "packet")
    b = ctx.query(d_rays)
    for k in a:
        assert torch.equal(a[k], b[k]), k


# ------------------------------------------------------------------ bf16 query path (mlp_dtype = 1)
@pytest.mark.parametrize("d_in,hidden", [(64, 2), (128, 3)])
def test_mlp_bf16_vs_oracle(orc, d_in, hidden):
    """C39: with mlp_dtype = 1 the query kernel's MLP (what nbvh_debug_mlp runs) takes bf16
    features and weights (fp32 accumulation, hidden activations rounded to bf16).  Against
    the double oracle on the same bf16 inputs and the fp16 weights: within the bf16 rounding
    bound (2H + 3) 2^-9 z_abs (weights of H + 1 layers, H activation roundings, 2^-9 the bf16
    unit roundoff), and within north_star's 1e-2 tier for unit-scale output layers."""
    from paper_2405_16237_b200 import Context
    L, F, npts = {64: (8, 2, 4), 128: (16, 2, 4)}[d_in]
    for out_scale, check_abs in ((10.0, False), (1.0, True)):
        ctx = Context(device=0, L=L, F=F, n_points=npts, hidden_layers=hidden, mlp_dtype=1)
        layers = synth.random_mlp(d_in, hidden, 64, seed=5, out_scale=out_scale)
        ctx.set_mlp(layers)
        m = 1000 + 77
        x = torch.from_numpy((np.random.default_rng(2).random((m, d_in)) * 0.8 - 0.4).astype(np.float32))
        xb = x.to(torch.bfloat16)
        z = ctx.debug_mlp(xb.cuda()).cpu().numpy()
        xd = xb.float().numpy().astype(np.float64)
        want = orc.mlp_forward(layers, xd)
        err = np.abs(z - want)
        assert np.all(err <= (2 * hidden + 3) * 2.0 ** -9 * _z_abs(layers, xd) + 1e-5), err.max()
        if check_abs:
            assert err.max() <= 1e-2, err.max()


def test_query_bf16_end_to_end(orc):
    """The bf16 query path end to end on the tiny scene: the logic replay of its own z trace
    exact, the double oracle identical on decided rays (north_star's bf16 tier: visibility
    margin 1e-2; t comparisons 2e-2 apart for the coarser bf16 t) with the band < 2%;
    decoded albedo / normal within 2.5e-2 (a quarter of the bf16 logit error)."""
    ctx, sc, tab, layers = _mk_ctx("tiny", mlp_dtype=1)
    # decoded channels: |d sigmoid| <= |dz| / 4 with the bf16 z error (~0.08 at |z| ~ 5)
    # raw z of the whole chain (features and weights rounded to bf16, 2^-9) vs the double oracle:
    # 8x the fp16 path's 2e-2 (1 + |z|), bf16 having 3 fewer mantissa bits
    g, o = _check_query(orc, ctx, tab, layers, _rays_tiny(), band_max=0.02, tband=2e-2, ztol=0.16, dec_tol=2.5e-2)
    assert g["hit"].sum() > 500


def test_deep_cut_traversal_full_base_bvh(orc):
    """The deepest cut the scenes give: every base-BVH leaf of the 988,928-triangle 1080p scene
    (532,435 SAH leaves of <= 4 triangles, depth 24).  Product lists (k_traverse, K = 16) vs
    the oracle's brute force, and the query's exact replay.  (k_traverse's shared memory is
    (depth + 2 + 3K) x 512 B; the launcher opts in past 48 KB, i.e. depth > 46 at K = 16,
    which no SAH tree of these scenes reaches.)"""
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    sc = synth.scene_1080p()
    c = synth.CONFIGS["1080p"]["hash"]
    ctx = Context(device=0, L=c.L, F=c.F, log2_T=c.log2_T, n_points=c.n_points, hidden_layers=c.hidden_layers,
                  list_cap=16)
    ctx.set_mesh(sc)
    n_leaves, clamped = ctx.build_cut(10 ** 7)
    ca, cb = ctx.base_bvh()
    n_base = int((cb < 0).sum())
    assert n_leaves == n_base
    depth, st = 0, [(0, 1)]
    while st:
        j, k = st.pop()
        depth = max(depth, k)
        if cb[j] >= 0:
            st += [(int(ca[j]), k + 1), (int(cb[j]), k + 1)]
    print(f"full cut: {n_leaves} leaves, depth {depth}, traversal smem {(depth + 2 + 48) * 512} B")
    tab = synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=3)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(ctx.d_in, c.hidden_layers, 64, seed=4)
    ctx.set_mlp(layers)
    cc = synth.CONFIGS["1080p"]
    rays = synth.camera_rays(*cc["res"], cc["eye"], vfov_deg=cc["vfov"])
    rays = np.ascontiguousarray(rays[np.linspace(0, rays.shape[0] - 1, 2000).astype(np.int64)])
    ctx.reserve(rays.shape[0])
    cut = ctx.cut(0)
    leaf, te, tx, fill, more = (v.cpu().numpy() for v in ctx.debug_traverse_product(torch.from_numpy(rays).cuda()))
    wl, wte, wtx, wcnt = orc.leaf_lists(rays, cut["leaf_lo"], cut["leaf_hi"], 16)
    assert np.array_equal(fill, np.minimum(wcnt, 16))
    for i in range(rays.shape[0]):
        k = fill[i]
        assert np.array_equal(leaf[i, :k], wl[i, :k])
    assert wcnt.max() > 16 and np.all(more[wcnt > 16] == 1)
    # the query's logic on this cut: exact replay of its own z trace (the double-oracle band
    # does not apply: half a million leaves put many t comparisons within 5e-3)
    out, zt = ctx.debug_query_trace(torch.from_numpy(rays).cuda(), 64)
    g = {k: v.cpu().numpy() for k, v in out.items()}
    rep = orc.replay(cut["leaf_lo"], cut["leaf_hi"], rays, zt.cpu().numpy(), mode=0)
    assert rep["missing"] == 0
    assert np.array_equal(g["hit"], rep["hit"]) and np.array_equal(g["leaf"], rep["leaf"])
    assert np.array_equal(g["n_queries"], rep["nq"])
    assert np.array_equal(g["t"].view(np.uint32), rep["t"].view(np.uint32))
