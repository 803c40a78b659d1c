"""Element-by-element parity of the training step's stages (T3-T7) against the oracle.

Every stage of the GPU's chain is compared with the oracle on the GPU's own inputs to that
stage, so each comparison isolates one kernel step, with a tolerance derived from the
floating-point operations of that step ("training tolerances"):

* T3 features x (fp32 trilinear blend of fp16 entries, rounded to fp16) vs the oracle's
  double encode of the same fp32 sample points: |dx| <= 2^-11 |x| + 1e-6 (the fp32 blend).
* T4 raw z (fp16 x, fp16 weights, fp32 accumulation, hidden activations rounded to fp16)
  vs the oracle's double MLP on the GPU's x: |dz| <= H 2^-11 z_abs + 1e-6, where z_abs is
  the same forward on absolute values (|W| |h| + |b|): each of the H fp16 roundings of a
  hidden activation perturbs it by <= 2^-11 of its magnitude.
* T5 per-sample loss and dL/dz, for every accepted sample, vs the oracle's double loss of
  the GPU's z and labels: fp32 evaluation of the same formulas.
* T6 hidden deltas (fp16) and the weight / bias gradients, T7 the hash-table gradient (fp32
  atomics), vs the oracle's double reverse mode from the GPU's x and dL/dz
  (orc_train_backward_given): per element |dg| <= ((H + 2) 2^-11 + m 2^-24) g_abs + 1e-7,
  g_abs = the same reverse mode on absolute values.  (H + 2) fp16 roundings: dL/dz, the H
  deltas; m 2^-24: fp32 summation over the m samples; weights and biases also carry the
  absolute rounding of fp16 subnormal deltas ((H + 1) 2^-25 |input| per sample).

ReLU decisions are floating-point decisions (C36): the oracle takes the kernel's own (the
exported activations' act > 0) and every decision where the two disagree must lie within
the rounding bound of its threshold: |pre| <= (H + 1) 2^-11 x magnitude.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

U = 2.0 ** -11          # fp16 unit roundoff
U32 = 2.0 ** -24

CONFIGS = {
    # name: (L, F, log2_T, n_points, hidden)
    "tiny_h2": (8, 2, 14, 4, 2),
    "tiny_h3": (8, 2, 14, 4, 3),
    "cfg2_grid": (16, 2, 19, 4, 3),        # the bench's grid/MLP shape (D_in 128) on the tiny scene
    "paper": (8, 4, 18, 3, 4),             # NEXT-4 (D_in 96; dW on the mma.sync fallback)
}


def _to(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _run(name, dw_path, monkeypatch, n_rays=6000, seed=70, scatter="agg"):
    import oracle as orc
    from paper_2405_16237_b200 import Context, PARAM_TABLES, dp
    if dw_path == "mma_sync":
        monkeypatch.setenv("NBVH_DW_MMA_SYNC", "1")
    else:
        monkeypatch.delenv("NBVH_DW_MMA_SYNC", raising=False)
    # T7 kernel: "agg" = the default warp-aggregated scatter, "priv" = k_train_scatter with the
    # shared-memory fixed-point levels (NBVH_SCATTER_AGG=0)
    if scatter == "priv":
        monkeypatch.setenv("NBVH_SCATTER_AGG", "0")
    else:
        monkeypatch.delenv("NBVH_SCATTER_AGG", raising=False)
    L, F, log2_T, npts, H = CONFIGS[name]
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=L, F=F, log2_T=log2_T, n_points=npts, hidden_layers=H)
    ctx.set_mesh(sc)
    ctx.build_cut(64)
    ctx.reserve(n_rays)
    tab = synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=seed, lo=-0.5, hi=0.5)
    ctx.set_params(PARAM_TABLES, tab.astype(np.float32))
    layers = synth.random_mlp(ctx.d_in, H, 64, seed=seed + 1, out_scale=1.0)
    ctx.set_mlp(layers)
    cut = ctx.cut(0)
    rank = np.random.default_rng(seed).normal(size=cut["n_leaves"]).astype(np.float32)
    ctx.set_leaf_rank(rank)
    rays = synth.random_rays(n_rays, seed=seed + 2)
    u = synth.random_uniform(n_rays, seed=seed + 3)
    xi = synth.random_uniform(n_rays * npts, seed=seed + 4).reshape(n_rays, npts)
    g = orc.Grid(L, log2_T, F)
    box = orc.scene_box(sc)
    leaf, te, tx, cnt = orc.leaf_lists(rays, cut["leaf_lo"], cut["leaf_hi"], 1)
    tabF = tab.reshape(-1, F)
    ctx.debug_train_capture(True)

    def gpu_pass(uu):
        ctx.train_backward(_to(rays), _to(uu), _to(xi))
        a = ctx.debug_train_activations(n_rays)
        torch.cuda.synchronize()
        out = {k: (None if v is None else v.cpu().numpy()) for k, v in a.items()}
        gt, acc, lf, loss = (t.cpu().numpy() for t in ctx.debug_train_samples(n_rays))
        out.update(gt=gt, acc=acc, loss=loss, grad=dp.grad_tensor(ctx).cpu().numpy().astype(np.float64))
        return out

    p = gpu_pass(u)
    masks = np.transpose(p["act"] > 0, (1, 0, 2)).astype(np.uint8)             # [m][H][64]
    r = p["ray"]
    o = orc.train_backward_given(g, npts, tabF, layers, box, rays[r], te[r, 0], tx[r, 0], xi[r],
                                 p["x"].astype(np.float64), p["dz"].astype(np.float64), masks=masks,
                                 want_deltas=True)
    return dict(ctx=ctx, sc=sc, cut=cut, g=g, tab=tabF, layers=layers, rays=rays, xi=xi, te=te, tx=tx, box=box,
                p=p, o=o, H=H, npts=npts, F=F, u=u, rank=rank)


@pytest.mark.parametrize("name,dw_path,scatter", [("tiny_h2", "tcgen05", "agg"), ("tiny_h3", "tcgen05", "agg"),
                                                  ("cfg2_grid", "tcgen05", "agg"), ("cfg2_grid", "mma_sync", "priv"),
                                                  ("paper", "tcgen05", "agg"), ("paper", "tcgen05", "priv")])
def test_training_stages_elementwise(name, dw_path, scatter, monkeypatch):
    import oracle as orc
    from paper_2405_16237_b200 import PARAM_TABLES
    R = _run(name, dw_path, monkeypatch, scatter=scatter)
    p, o, H, g = R["p"], R["o"], R["H"], R["g"]
    m = p["ray"].size
    assert m > 500, m
    # the kernel's ReLU decisions: disagreements with the double sign only within rounding
    assert np.all(o["flip_margin"] <= (H + 1) * U), o["flip_margin"].max()
    assert (o["mask_flips"] > 0).mean() < 0.05, (o["mask_flips"] > 0).mean()
    r = p["ray"]
    # ---- T3 features: the oracle's own double encode of the same fp32 sample points
    dmin, dinv = orc.domain(*np.split(R["box"].reshape(1, 6), 2, axis=1))
    pts = np.stack([orc.segment_points(R["rays"][i], R["te"][i, 0], R["tx"][i, 0], R["npts"], dmin, dinv, R["xi"][i])
                    for i in r])
    feat, _ = orc.encode_points(g, R["tab"], pts.reshape(-1, 3))
    x_orc = feat.reshape(m, -1)
    x_gpu = p["x"].astype(np.float64)
    assert np.all(np.abs(x_gpu - x_orc) <= U * np.abs(x_orc) + 1e-6), np.abs(x_gpu - x_orc).max()
    # ---- T4 raw z: double MLP on the GPU's own features
    z = p["z"].astype(np.float64)
    tol_z = H * U * o["z_abs"] + 1e-6
    assert np.all(np.abs(z - o["z"]) <= tol_z), (np.abs(z - o["z"]) / tol_z).max()
    # ---- T5 loss and dL/dz of every accepted sample, from the GPU's z and labels
    gt = p["gt"][r].astype(np.float64)
    Ls = np.zeros(m)
    dzs = np.zeros((m, 8))
    for i in range(m):
        Ls[i], _, dzs[i] = orc.sample_loss(z[i], gt[i])
    assert np.all(np.abs(p["loss"][r] - Ls) <= 2e-5 * (1 + np.abs(Ls))), np.abs(p["loss"][r] - Ls).max()
    dz = p["dz"].astype(np.float64)
    ok = np.all(np.abs(dz - dzs) <= 2e-5 * (1 + np.abs(dzs)), axis=1)
    assert ok.mean() >= 0.999, ok.mean()            # an L1 subgradient at an exact fp32 tie may differ
    # ---- T6 hidden deltas (fp16), per layer
    for j in range(H):
        dg = p["delta"][j].astype(np.float64)
        do, da = o["hidden_delta"][:, j, :], o["hidden_delta_abs"][:, j, :]
        tol = (H - j + 2) * U * da + 6e-8
        assert np.all(np.abs(dg - do) <= tol), (j, (np.abs(dg - do) / tol).max())
    # ---- T6 weight/bias gradients and T7 table gradients: every element
    grad = p["grad"]
    n_t = R["ctx"].param_count(PARAM_TABLES)
    n_w, n_b = o["g_W"].size, o["g_b"].size
    rt = (H + 2) * U + m * U32
    # fp16 subnormals: a delta (or dL/dz cast) below 2^-14 is rounded with ABSOLUTE error
    # <= 2^-25, so each sample adds up to (H + 1) 2^-25 |input| to a weight gradient
    # (|input| = 1 for biases) on top of the relative bound
    ins = [p["x"].astype(np.float64)] + [p["act"][k].astype(np.float64) for k in range(H)]
    dims = [ins[0].shape[1]] + [64] * H + [8]
    under_w, under_b = [], []
    for k in range(H + 1):
        col = np.abs(ins[k]).sum(0)                                     # sum over samples, per input unit
        under_w.append(np.tile(col, dims[k + 1]))
        under_b.append(np.full(dims[k + 1], float(m)))
    under_w = (H + 1) * 2.0 ** -25 * np.concatenate(under_w)
    under_b = (H + 1) * 2.0 ** -25 * np.concatenate(under_b)
    for blk, gg, oo, aa, un in (("tables", grad[:n_t], o["g_table"], o["g_table_abs"], 0.0),
                                ("weights", grad[n_t:n_t + n_w], o["g_W"], o["g_W_abs"], under_w),
                                ("biases", grad[n_t + n_w:n_t + n_w + n_b], o["g_b"], o["g_b_abs"], under_b)):
        tol = rt * aa + un + 1e-7
        bad = np.abs(gg - oo) > tol
        assert not bad.any(), (blk, int(bad.sum()), (np.abs(gg - oo) / tol).max(), np.nonzero(bad)[0][:8],
                               aa[bad][:8], oo[bad][:8], gg[bad][:8])
        assert np.count_nonzero(oo) > 0.5 * min(oo.size, 1000) or blk == "tables"
    # ---- tail: accepted count, per-leaf sample and first-hit counts exact, loss sums (fp32 atomics)
    tail = grad[n_t + n_w + n_b:]
    assert tail[0] == m
    per_leaf = tail[1:1 + 3 * R["cut"]["n_leaves"]].reshape(-1, 3)
    lf = R["ctx"].debug_train_samples(R["rays"].shape[0])[2].cpu().numpy()
    assert np.array_equal(per_leaf[:, 1], np.bincount(lf[r], minlength=per_leaf.shape[0]))
    first = lf[lf >= 0]
    assert np.array_equal(per_leaf[:, 2], np.bincount(first, minlength=per_leaf.shape[0]))
    want_leaf_loss = np.bincount(lf[r], weights=Ls, minlength=per_leaf.shape[0])
    assert np.all(np.abs(per_leaf[:, 0] - want_leaf_loss) <= 1e-4 * (1 + want_leaf_loss))


def test_training_forward_vs_full_double_chain(monkeypatch):
    """The whole forward (T3-T5) against the oracle's own double chain (orc_train_grad, its
    double features and MLP, its own ReLU decisions): per-sample z within the fp16 chain's
    bound (H + 1) 2^-11 z_abs on samples without a flipped ReLU decision (x is rounded once
    more than in the staged check), and every such sample's loss within the loss's Lipschitz
    bound of that z error."""
    import oracle as orc
    R = _run("tiny_h2", "tcgen05", monkeypatch)
    p, H = R["p"], R["H"]
    r = p["ray"]
    full = orc.train_grad(R["g"], R["npts"], R["tab"], R["layers"], R["cut"]["leaf_lo"], R["cut"]["leaf_hi"],
                          R["rank"], R["cut"]["tri_off"], R["cut"]["tris"], R["sc"], R["rays"], R["u"], R["xi"],
                          dom_box=R["box"])
    assert np.array_equal(np.nonzero(full["accepted"])[0], np.sort(r))
    dmin, dinv = orc.domain(*np.split(R["box"].reshape(1, 6), 2, axis=1))
    pts = np.stack([orc.segment_points(R["rays"][i], R["te"][i, 0], R["tx"][i, 0], R["npts"], dmin, dinv, R["xi"][i])
                    for i in r])
    x_orc = orc.encode_points(R["g"], R["tab"], pts.reshape(-1, 3))[0].reshape(r.size, -1)
    z_orc = orc.mlp_forward(R["layers"], x_orc)
    z = p["z"].astype(np.float64)
    ok = R["o"]["mask_flips"] == 0
    assert ok.mean() > 0.95
    tol = (H + 1) * U * R["o"]["z_abs"] + 1e-6
    assert np.all(np.abs(z - z_orc)[ok] <= tol[ok]), (np.abs(z - z_orc)[ok] / tol[ok]).max()
    # loss: |dL| <= sum_c Lip_c |dz_c| with Lip = max |dL/dz_c|: 2 (2 BCE: 2|sigma - y|),
    # 1/2 (2 L1 of sigma), 1/3 per normal component, <= 3.1 per albedo channel (relative L2)
    lip = np.array([2.0, 0.5, 1 / 3, 1 / 3, 1 / 3, 3.1, 3.1, 3.1])
    bound = (np.abs(z - z_orc) * lip).sum(1) + 1e-5
    dl = np.abs(p["loss"][r] - full["loss"][r])
    assert np.all((dl <= bound + 2e-5 * np.abs(full["loss"][r]))[ok])
