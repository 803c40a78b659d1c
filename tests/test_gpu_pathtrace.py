"""NEXT-3: hybrid path tracing pieces (PAPER §7) on the GPU.

* the classical BLAS query (nbvh_intersect_mesh) against the oracle's exact ray/triangle
  ground truth over the whole mesh: hit mask and hit t bit-exact (double Moller-Trumbore with
  the same operation order), normal/albedo to 1e-6;
* the wavefront shading step against a plain numpy float32 re-implementation of the same
  formula and the same counter-based hash;
* a hybrid render (classical terrain + neural spheres) is finite, non-negative, bounded by
  the sky radiance, and its alive-ray counts never grow.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_intersect_mesh_vs_oracle(orc):
    from paper_2405_16237_b200 import Context
    sc = synth.scene_tiny()
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    ctx.set_mesh(sc)
    rays = np.concatenate([synth.camera_rays(64, 64, (0.0, 0.0, 3.5), vfov_deg=40.0),
                           synth.random_rays(3000, seed=77)], 0)
    out = ctx.intersect_mesh(torch.from_numpy(rays).cuda())
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    n, nt = rays.shape[0], sc.tris.shape[0]
    gt = orc.label(sc, np.array([0, nt], np.int64), np.arange(nt, dtype=np.int32), rays, np.zeros(n, np.int32),
                   rays[:, 3].copy(), rays[:, 7].copy())
    hit = (gt[:, 0] == 0).astype(np.uint8)
    assert np.array_equal(g["hit"], hit) and hit.sum() > 1000
    h = hit == 1
    assert np.array_equal(g["t"][h], gt[h, 8].astype(np.float32))
    assert np.abs(g["normal"][h] - gt[h, 2:5]).max() <= 1e-6
    assert np.abs(g["albedo"][h] - gt[h, 5:8]).max() <= 1e-6
    assert np.all(np.isinf(g["t"][~h])) and np.all(g["leaf"][~h] == -1)


def _pcg(v):
    v = v.astype(np.uint64) & 0xFFFFFFFF
    state = (v * 747796405 + 2891336453) & 0xFFFFFFFF
    word = (((state >> ((state >> 28) + 4)) ^ state) * 277803737) & 0xFFFFFFFF
    return ((word >> 22) ^ word) & 0xFFFFFFFF


def _uniform(seed, ray, bounce, k):
    h = _pcg(np.uint64(seed & 0xFFFFFFFF) ^ _pcg(np.uint64((seed >> 32) + 0x9E3779B9)))
    h = _pcg(h ^ (ray.astype(np.uint64) & 0xFFFFFFFF))
    h = _pcg(h ^ (ray.astype(np.uint64) >> 32) ^ np.uint64(bounce << 8) ^ np.uint64(k))
    return (h >> 8).astype(np.float32) * np.float32(1.0 / 16777216.0)


def test_pt_shade_vs_numpy():
    from paper_2405_16237_b200 import Context
    from paper_2405_16237_b200.pathtrace import SKY
    rng = np.random.default_rng(3)
    n = 5000
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    rays = synth.random_rays(n, seed=5)
    rays[::7, 3], rays[::7, 7] = 1.0, 0.0                             # some dead rays
    def rec(p_hit):
        nrm = rng.normal(size=(n, 3)).astype(np.float32)
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        return dict(hit=(rng.random(n) < p_hit).astype(np.uint8), t=rng.uniform(0.1, 2, n).astype(np.float32),
                    normal=nrm, albedo=rng.uniform(0.2, 0.9, (n, 3)).astype(np.float32),
                    leaf=np.zeros(n, np.int32), n_queries=np.zeros(n, np.int32))
    A, B = rec(0.5), rec(0.5)
    thr = rng.uniform(0.3, 1, (n, 3)).astype(np.float32)
    rad = rng.uniform(0, 0.1, (n, 3)).astype(np.float32)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dA, dB = {k: dev(v) for k, v in A.items()}, {k: dev(v) for k, v in B.items()}
    dthr, drad, dnext = dev(thr), dev(rad), torch.empty(n, 8, device="cuda")
    alive = torch.zeros(1, dtype=torch.int32, device="cuda")
    seed, bounce, eps = 0x1234567890, 2, 1e-4
    ctx.pt_shade(dev(rays), dA, dB, dthr, drad, dnext, seed, bounce, SKY, eps, alive)
    torch.cuda.synchronize()
    # reference (numpy float32, same formula)
    f = np.float32
    live = rays[:, 3] <= rays[:, 7]
    ta = np.where(A["hit"] == 1, A["t"], np.inf).astype(f)
    tb = np.where(B["hit"] == 1, B["t"], np.inf).astype(f)
    use_b = (B["hit"] == 1) & (tb < ta)
    anyhit = (A["hit"] == 1) | (B["hit"] == 1)
    d = rays[:, 4:7]
    e = np.maximum(f(0), d[:, 1] / np.maximum(np.linalg.norm(d, axis=1), f(1e-20)))
    sky = SKY[:3] + (SKY[3:] - SKY[:3]) * e[:, None]
    want_rad = rad + np.where((live & ~anyhit)[:, None], thr * sky, 0)
    nrm = np.where(use_b[:, None], B["normal"], A["normal"])
    nrm = np.where((np.sum(nrm * d, 1) > 0)[:, None], -nrm, nrm)
    alb = np.where(use_b[:, None], B["albedo"], A["albedo"])
    want_thr = np.where((live & anyhit)[:, None], thr * alb, thr)
    assert np.allclose(drad.cpu().numpy(), want_rad, atol=1e-6)
    assert np.allclose(dthr.cpu().numpy(), want_thr, atol=1e-6)
    nx = dnext.cpu().numpy()
    cont = live & anyhit
    assert int(alive.item()) == int(cont.sum())
    assert np.all(nx[~cont, 3] > nx[~cont, 7])                      # ended rays are empty intervals
    t = np.where(use_b, tb, ta)
    p = rays[:, :3] + t[:, None] * d
    assert np.allclose(nx[cont, :3], (p + eps * nrm)[cont], atol=1e-5)
    r = np.arange(n, dtype=np.int64)
    u1, u2 = _uniform(seed, r, bounce, 0), _uniform(seed, r, bounce, 1)
    lz = np.sqrt(np.maximum(0, 1 - u1))
    cos_t = np.sum(nx[:, 4:7] * nrm, 1)
    assert np.allclose(cos_t[cont], lz[cont], atol=1e-5)             # cosine-weighted: cos(theta) = sqrt(1-u1)
    assert np.allclose(np.linalg.norm(nx[cont, 4:7], axis=1), 1, atol=1e-5)


def _hybrid_scene(cut_leaves=64, lod_leaves=None):
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    terrain, spheres = synth.scene_1080p_parts(grid=48, nu=6)
    neural = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    neural.set_mesh(spheres)
    neural.build_cut(cut_leaves)
    if lod_leaves:
        neural.build_cut(lod_leaves, lod=1)                       # a coarser LoD of the same grid
    neural.set_params(PARAM_TABLES, synth.random_params_fp16(neural.param_count(PARAM_TABLES), seed=4)
                      .astype(np.float32))
    neural.set_mlp(synth.random_mlp(neural.d_in, 2, 64, seed=5))
    classical = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    classical.set_mesh(terrain)
    return neural, classical, terrain, spheres


IDENTITY = np.concatenate([np.eye(3), np.zeros((3, 1))], 1)


def test_hybrid_render_bounded():
    """The TLAS renderer (compacted wavefront): finite, non-negative radiance bounded by the
    sky, alive path counts that never grow, most pixels lit."""
    from paper_2405_16237_b200.pathtrace import PathTracer, SKY
    neural, classical, _, _ = _hybrid_scene()
    rays = torch.from_numpy(synth.camera_rays(96, 64, (0.0, 0.6, 1.6), vfov_deg=50.0)).cuda()
    pt = PathTracer([(neural, "neural"), (classical, "mesh")], [(0, IDENTITY), (1, IDENTITY)], rays.shape[0])
    rad, alive = pt.render(rays, bounces=4, seed=9)
    rad = rad.cpu().numpy()
    assert np.all(np.isfinite(rad)) and rad.min() >= 0 and rad.max() <= SKY.max() + 1e-6
    assert alive[0] == rays.shape[0] and np.all(np.diff(alive) <= 0) and alive[1] < alive[0]
    assert (rad.sum(1) > 0).mean() > 0.5


@pytest.mark.parametrize("lod_secondary", [0, 1])
def test_tlas_renderer_equals_flat_renderer(lod_secondary):
    """With identity instances [neural, mesh], the compacted TLAS renderer must give the
    radiance of the round-1 flat renderer (every ray to both BLAS, no compaction): the
    random streams are keyed by pixel, the merge's tie rule (lower BLAS number) is
    nbvh_pt_shade's (neural first), and compaction changes no per-ray computation.  With
    lod_secondary = 1 both switch the neural BLAS to a coarser cut after the primary hit
    (P:342)."""
    from paper_2405_16237_b200.pathtrace import PathTracer, PathTracerFlat
    neural, classical, _, _ = _hybrid_scene(lod_leaves=8)
    rays = torch.from_numpy(synth.camera_rays(128, 96, (0.0, 0.6, 1.6), vfov_deg=50.0)).cuda()
    n = rays.shape[0]
    pt = PathTracer([(neural, "neural"), (classical, "mesh")], [(0, IDENTITY), (1, IDENTITY)], n,
                    lod_secondary=lod_secondary)
    a, alive = pt.render(rays, bounces=3, seed=5)
    a = a.cpu().numpy().copy()
    flat = PathTracerFlat(neural, classical, n)
    b, alive_b = flat.render(rays, bounces=3, seed=5, lod_secondary=lod_secondary)
    b = b.cpu().numpy()
    # equal up to the merge's renormalisation of the (already unit) normal: a few ulp
    assert np.abs(a - b).max() <= 1e-5, np.abs(a - b).max()
    assert list(alive[1:]) == alive_b.cpu().numpy()[:2].tolist()        # continuing paths per bounce
    if lod_secondary:
        c, _ = PathTracer([(neural, "neural"), (classical, "mesh")], [(0, IDENTITY), (1, IDENTITY)], n,
                          lod_secondary=0).render(rays, bounces=3, seed=5)
        assert not np.array_equal(a, c.cpu().numpy())                   # the switch is live


def _rot(axis, ang):
    c, s_ = np.cos(ang), np.sin(ang)
    i, j = [k for k in range(3) if k != axis]
    r = np.eye(3)
    r[i, i], r[i, j], r[j, i], r[j, j] = c, -s_, s_, c
    return r


def test_tlas_instances_vs_oracle(orc):
    """TLAS with affine instances of two classical BLAS (three instances of the icosphere --
    identity, rotated + translated + uniformly scaled, anisotropically scaled -- and one of a
    second mesh) against the oracle's brute-force closest hit over all the instances' triangles
    transformed to world space: identical hit masks away from grazing rays, t within fp32
    transform rounding, the winning instance, and world normals (A^T n, normalised) and albedo."""
    from paper_2405_16237_b200 import Context
    from paper_2405_16237_b200.pathtrace import Tlas
    from synth.scenes import Scene
    a_sc = synth.scene_tiny(nu=8)
    b_sc = synth.scene_tiny(seed=3, nu=6)
    ca = Context(device=0)
    ca.set_mesh(a_sc)
    cb = Context(device=0)
    cb.set_mesh(b_sc)
    M = [IDENTITY,
         np.concatenate([0.7 * _rot(1, 0.6) @ _rot(0, 0.3), np.array([[2.6], [0.2], [-0.5]])], 1),
         np.concatenate([np.diag([1.4, 0.6, 0.9]), np.array([[-2.5], [0.0], [0.3]])], 1),
         np.concatenate([_rot(2, 1.1), np.array([[0.1], [2.4], [0.0]])], 1)]
    blas_of = [0, 0, 0, 1]
    scenes = [a_sc, b_sc]
    inst = []
    for k, m in enumerate(M):
        v = scenes[blas_of[k]].verts.astype(np.float64)
        inst.append((blas_of[k], m, v.min(0), v.max(0)))
    tl = Tlas(ca, inst)
    rng = np.random.default_rng(11)
    n = 6000
    o = rng.uniform(-5, 5, (n, 3))
    tgt = rng.uniform(-3, 3, (n, 3)) + np.array([0, 0.5, 0])
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.zeros((n, 8), np.float32)
    rays[:, :3], rays[:, 4:7], rays[:, 7] = o, d, np.inf
    cap = n * 3
    lr = torch.empty(2 * cap, 8, device="cuda")
    src = torch.empty(2 * cap, dtype=torch.int32, device="cuda")
    ins = torch.empty(2 * cap, dtype=torch.int32, device="cuda")
    counts = torch.zeros(2, dtype=torch.int32, device="cuda")
    d_rays = torch.from_numpy(rays).cuda()
    tl.dispatch(d_rays, n, lr, src, ins, counts, cap)
    cnt = counts.cpu().numpy()
    lists = [ca.alloc_hits(cap), ca.alloc_hits(cap)]
    for k, ctx in enumerate((ca, cb)):
        if cnt[k]:
            ctx.intersect_mesh(lr[k * cap:k * cap + int(cnt[k])], out={key: v[:int(cnt[k])] for key, v in lists[k].items()})
    out = ca.alloc_hits(n)
    tl.merge(n, counts, cap, src, ins, lists, out)
    torch.cuda.synchronize()
    assert tl.overflow() == 0
    g = {k: v.cpu().numpy() for k, v in out.items()}
    # oracle: every instance's triangles in world space (vertices and normals transformed in
    # double), one brute-force closest hit
    V, T, N, A, owner = [], [], [], [], []
    off = 0
    for k, m in enumerate(M):
        sc = scenes[blas_of[k]]
        mm = np.asarray(m, np.float64)
        V.append(sc.verts.astype(np.float64) @ mm[:, :3].T + mm[:, 3])
        # M^-T n per vertex, not renormalised: the shading normal (barycentric blend, then
        # normalised) is then the transform of the object-space one, as A^T n is
        N.append(sc.vnormals.astype(np.float64) @ np.linalg.inv(mm[:, :3]))
        T.append(sc.tris.astype(np.int64) + off)
        A.append(sc.albedo)
        owner.append(np.full(sc.tris.shape[0], k))
        off += sc.verts.shape[0]
    world = Scene(verts=np.concatenate(V).astype(np.float32), tris=np.concatenate(T).astype(np.uint32),
                  vnormals=np.concatenate(N).astype(np.float32), albedo=np.concatenate(A).astype(np.float32))
    owner = np.concatenate(owner)
    nt = world.tris.shape[0]
    gt = orc.label(world, np.array([0, nt], np.int64), np.arange(nt, dtype=np.int32), rays, np.zeros(n, np.int32),
                   rays[:, 3].copy(), rays[:, 7].copy())
    hit = gt[:, 0] == 0
    assert hit.sum() > 1000
    agree = (g["hit"] == 1) == hit
    assert agree.mean() >= 0.999, agree.mean()                             # grazing rays only
    both = hit & (g["hit"] == 1)
    assert np.all(np.abs(g["t"][both] - gt[both, 8]) <= 1e-4 * (1 + gt[both, 8]))
    assert np.abs(g["normal"][both] - gt[both, 2:5]).max() <= 2e-3
    assert np.abs(g["albedo"][both] - gt[both, 5:8]).max() <= 1e-6
    assert set(np.unique(g["leaf"][both])) == {0, 1, 2, 3}


def test_intersect_mesh_deep_bvh_vs_oracle(orc):
    """A chain-shaped base BVH (plates at exponentially growing spacing, so SAH peels one
    off per level): the closest-hit stack is sized by the measured depth, not a fixed 64."""
    from paper_2405_16237_b200 import Context
    from synth.scenes import Scene
    n_plates = 40
    xs = np.cumsum(1.25 ** np.arange(n_plates)).astype(np.float32)
    V, T = [], []
    for i, x in enumerate(xs):
        V += [(x, -1.0, -1.0), (x, 1.0, -1.0), (x, 0.0, 1.5)]
        T.append((3 * i, 3 * i + 1, 3 * i + 2))
    V = np.array(V, np.float32)
    nrm = np.tile(np.array([[-1.0, 0.0, 0.0]], np.float32), (V.shape[0], 1))
    sc = Scene(verts=V, tris=np.array(T, np.uint32), vnormals=nrm,
               albedo=np.full((n_plates, 3), 0.5, np.float32))
    ctx = Context(device=0, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    ctx.set_mesh(sc)
    rng = np.random.default_rng(5)
    n = 4000
    rays = np.zeros((n, 8), np.float32)
    start = rng.integers(0, n_plates, n)
    rays[:, 0] = xs[start] - rng.uniform(0.01, 0.5, n).astype(np.float32)
    rays[:, 1:3] = rng.uniform(-0.6, 0.6, (n, 2))
    d = np.stack([np.ones(n), rng.uniform(-0.02, 0.02, n), rng.uniform(-0.02, 0.02, n)], 1)
    rays[:, 4:7] = d / np.linalg.norm(d, axis=1, keepdims=True)
    rays[:, 3] = 0.0
    rays[:, 7] = 1e30
    out = ctx.intersect_mesh(torch.from_numpy(rays).cuda())
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in out.items()}
    gt = orc.label(sc, np.array([0, n_plates], np.int64), np.arange(n_plates, dtype=np.int32), rays,
                   np.zeros(n, np.int32), rays[:, 3].copy(), rays[:, 7].copy())
    hit = (gt[:, 0] == 0).astype(np.uint8)
    assert np.array_equal(g["hit"], hit) and hit.sum() > n // 2
    h = hit == 1
    assert np.array_equal(g["t"][h], gt[h, 8].astype(np.float32))
