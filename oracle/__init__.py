"""CPU oracle for the N-BVH neural ray-query hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
leg may import this package.  The product package (paper_2405_16237_b200) never
imports it.  The arithmetic lives in nbvh_oracle.cpp (C++17, double for continuous
quantities, binary32 for the discrete decisions); this module only builds it and
marshals numpy arrays.  Functions with no independent pin: none except the
end-to-end reconstruction *quality* of a trained model (P17, "parity unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nbvh_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-fno-fast-math", "-ffp-contract=off", "-msse2", "-mfpmath=sse",
               "-fopenmp", "-shared", "-fPIC", _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_half_to_double.restype = C.c_double
        _lib.orc_level_table.restype = C.c_int64
        _lib.orc_corner_index.restype = C.c_uint32
        _lib.orc_slab.restype = C.c_int
        _lib.orc_replay.restype = C.c_int64
        _lib.orc_check_cut.restype = C.c_int32
        _lib.orc_triangle_hit.restype = C.c_int
        _lib.orc_sample_loss.restype = C.c_double
        _lib.orc_train_grad.restype = C.c_int64
        _lib.orc_batch_loss_double.restype = C.c_double
        _lib.orc_num_threads.restype = C.c_int32
        _lib.orc_sigmoid_f32.restype = C.c_float
        _lib.orc_sigmoid_f32.argtypes = [C.c_float]
        _lib.orc_expand_cut.restype = C.c_int32
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(C.c_int32(n))


# ---------------------------------------------------------------- grid
class Grid:
    """Level table computed by the oracle itself (C1, C2)."""

    def __init__(self, L, log2_T, F=2, base_res=8, max_res=1024):
        self.L, self.log2_T, self.F, self.base_res, self.max_res = L, log2_T, F, base_res, max_res
        self.res = np.zeros(L, np.int32)
        self.dense = np.zeros(L, np.int32)
        self.offset = np.zeros(L, np.int64)
        self.n_entries = int(lib().orc_level_table(L, log2_T, base_res, max_res, _p(self.res), _p(self.dense),
                                                   _p(self.offset)))


def half_to_double(h: int) -> float:
    return float(lib().orc_half_to_double(C.c_uint16(h)))


def corner_index(N, dense, log2_T, x, y, z) -> int:
    return int(lib().orc_corner_index(C.c_int32(N), C.c_int32(dense), C.c_int(log2_T), C.c_uint32(x),
                                      C.c_uint32(y), C.c_uint32(z)))


def encode_points(grid: Grid, table_fp16: np.ndarray, pts: np.ndarray):
    """pts float32 [m,3] in [0,1] -> (features float64 [m, L*F], indices uint32 [m, L, 8])."""
    pts = _c(pts, np.float32)
    tab = _c(table_fp16, np.float16).view(np.uint16)
    m = pts.shape[0]
    feat = np.zeros((m, grid.L * grid.F), np.float64)
    idx = np.zeros((m, grid.L, 8), np.uint32)
    lib().orc_encode_points(grid.L, grid.F, grid.log2_T, _p(grid.res), _p(grid.dense), _p(grid.offset), _p(tab),
                            _p(pts), C.c_int64(m), _p(feat), _p(idx))
    return feat, idx


# ---------------------------------------------------------------- geometry
def slab(ray, lo, hi):
    ray = _c(ray, np.float32)
    lo = _c(lo, np.float32)
    hi = _c(hi, np.float32)
    te = np.zeros(1, np.float32)
    tx = np.zeros(1, np.float32)
    h = lib().orc_slab(_p(ray), _p(lo), _p(hi), _p(te), _p(tx))
    return bool(h), float(te[0]), float(tx[0]), te[0], tx[0]


def leaf_lists(rays, leaf_lo, leaf_hi, cap):
    rays = _c(rays, np.float32)
    lo = _c(leaf_lo, np.float32)
    hi = _c(leaf_hi, np.float32)
    n = rays.shape[0]
    leaf = np.zeros((n, cap), np.int32)
    te = np.zeros((n, cap), np.float32)
    tx = np.zeros((n, cap), np.float32)
    cnt = np.zeros(n, np.int32)
    lib().orc_leaf_lists(_p(rays), C.c_int64(n), _p(lo), _p(hi), C.c_int32(lo.shape[0]), C.c_int32(cap),
                         _p(leaf), _p(te), _p(tx), _p(cnt))
    return leaf, te, tx, cnt


def scene_box(scene, rel=1e-3, abs_=1e-6):
    """Inflated root box of the scene (C4 as amended for shared-grid LoD cuts, C15)."""
    box = np.zeros(6, np.float32)
    tris = _c(scene.tris, np.uint32)
    lib().orc_scene_box(_p(_c(scene.verts, np.float32)), _p(tris), C.c_int64(tris.shape[0]), C.c_float(rel),
                        C.c_float(abs_), _p(box))
    return box


def _box(dom_box):
    return None if dom_box is None else _p(_c(dom_box, np.float32))


def domain(leaf_lo, leaf_hi):
    lo = _c(leaf_lo, np.float32)
    hi = _c(leaf_hi, np.float32)
    dmin = np.zeros(3, np.float32)
    dinv = np.zeros(1, np.float32)
    lib().orc_domain(_p(lo), _p(hi), C.c_int32(lo.shape[0]), _p(dmin), _p(dinv))
    return dmin, dinv[0]


def segment_points(ray, t0, t1, n, dom_min, dom_inv, xi=None):
    ray = _c(ray, np.float32)
    dmin = _c(dom_min, np.float32)
    pts = np.zeros((n, 3), np.float32)
    xi_a = _c(xi, np.float32) if xi is not None else None
    lib().orc_segment_points(_p(ray), C.c_float(t0), C.c_float(t1), C.c_int(n), _p(xi_a), _p(dmin),
                             C.c_float(dom_inv), _p(pts))
    return pts


# ---------------------------------------------------------------- MLP
def _mlp_arrays(layers):
    dims = [layers[0][0].shape[1]] + [W.shape[0] for W, _ in layers]
    W_all = np.concatenate([_c(W, np.float16).reshape(-1) for W, _ in layers]).view(np.uint16)
    b_all = np.concatenate([_c(b, np.float32).reshape(-1) for _, b in layers])
    return np.asarray(dims, np.int32), W_all, b_all


def mlp_forward(layers, x):
    dims, W_all, b_all = _mlp_arrays(layers)
    x = _c(x, np.float64)
    m = x.shape[0]
    z = np.zeros((m, dims[-1]), np.float64)
    lib().orc_mlp_forward(C.c_int(len(layers)), _p(dims), _p(W_all), _p(b_all), _p(x), C.c_int64(m), _p(z))
    return z


# ---------------------------------------------------------------- query
def query(grid: Grid, n_points, table_fp16, layers, leaf_lo, leaf_hi, rays, mode=0, trace_cap=0, dom_box=None):
    """dom_box (6 floats, nullable): the grid-domain box (scene_box); None = union of the leaf boxes."""
    dims, W_all, b_all = _mlp_arrays(layers)
    tab = _c(table_fp16, np.float16).view(np.uint16)
    rays = _c(rays, np.float32)
    lo = _c(leaf_lo, np.float32)
    hi = _c(leaf_hi, np.float32)
    n = rays.shape[0]
    out = dict(hit=np.zeros(n, np.uint8), t=np.zeros(n, np.float32), normal=np.zeros((n, 3), np.float32),
               albedo=np.zeros((n, 3), np.float32), leaf=np.zeros(n, np.int32), nq=np.zeros(n, np.int32),
               margin=np.zeros(n, np.float64), tmargin=np.zeros(n, np.float64))
    zt = np.zeros((n, trace_cap, 8), np.float64) if trace_cap else None
    lib().orc_query(grid.L, grid.F, grid.log2_T, n_points, len(layers), _p(grid.res), _p(grid.dense),
                    _p(grid.offset), _p(tab), _p(dims), _p(W_all), _p(b_all), _p(lo), _p(hi),
                    C.c_int32(lo.shape[0]), _p(rays), C.c_int64(n), C.c_int32(mode), _p(out["hit"]),
                    _p(out["t"]), _p(out["normal"]), _p(out["albedo"]), _p(out["leaf"]), _p(out["nq"]),
                    _p(out["margin"]), _p(zt), C.c_int32(trace_cap), _p(out["tmargin"]), _box(dom_box))
    if zt is not None:
        out["z_trace"] = zt
    return out


def philox4x32_10(ctr, key):
    """Philox-4x32-10 block (the T0 generator, C28')."""
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def gen_train_rays(seed, step, i0, n, box, n_points):
    """T0 training rays + draws (rays [n, 8], u [n], xi [n, n_points]) per C28'."""
    rays = np.zeros((n, 8), np.float32)
    u = np.zeros(n, np.float32)
    xi = np.zeros((n, max(n_points, 1)), np.float32)
    bx = np.ascontiguousarray(np.asarray(box, np.float32).reshape(6))
    lib().orc_gen_train_rays(C.c_uint64(seed), C.c_uint64(step), C.c_int64(i0), C.c_int64(n), _p(bx),
                             C.c_int32(n_points), _p(rays), _p(u), _p(xi))
    return rays, u, xi[:, :n_points]


def sigmoid_f32(z: float) -> float:
    """The decode's fp32 sigmoid (C27), as the logic replay evaluates it."""
    return float(lib().orc_sigmoid_f32(C.c_float(z)))


def replay(leaf_lo, leaf_hi, rays, z_trace, mode=0):
    lo = _c(leaf_lo, np.float32)
    hi = _c(leaf_hi, np.float32)
    rays = _c(rays, np.float32)
    zt = _c(z_trace, np.float32)
    n, cap = zt.shape[0], zt.shape[1]
    out = dict(hit=np.zeros(n, np.uint8), t=np.zeros(n, np.float32), normal=np.zeros((n, 3), np.float32),
               albedo=np.zeros((n, 3), np.float32), leaf=np.zeros(n, np.int32), nq=np.zeros(n, np.int32))
    miss = lib().orc_replay(_p(lo), _p(hi), C.c_int32(lo.shape[0]), _p(rays), C.c_int64(n), C.c_int32(mode),
                            _p(zt), C.c_int32(cap), _p(out["hit"]), _p(out["t"]), _p(out["normal"]),
                            _p(out["albedo"]), _p(out["leaf"]), _p(out["nq"]))
    out["missing"] = int(miss)
    return out


# ---------------------------------------------------------------- cut / GT / training
def check_cut(verts, tris, leaf_tri_off, leaf_tris, base_lo, base_hi, leaf_lo, leaf_hi, scene_diag):
    v = _c(verts, np.float32)
    t = _c(tris, np.uint32)
    off = _c(leaf_tri_off, np.int64)
    lt = _c(leaf_tris, np.int32)
    return int(lib().orc_check_cut(_p(v), _p(t), C.c_int64(t.shape[0]), C.c_int32(off.shape[0] - 1), _p(off),
                                   _p(lt), _p(_c(base_lo, np.float32)), _p(_c(base_hi, np.float32)),
                                   _p(_c(leaf_lo, np.float32)), _p(_c(leaf_hi, np.float32)),
                                   C.c_double(scene_diag)))


def triangle_hit(o, d, v0, v1, v2, t0=0.0, t1=np.inf):
    arrs = [_c(a, np.float64) for a in (o, d, v0, v1, v2)]
    t = np.zeros(1)
    b1 = np.zeros(1)
    b2 = np.zeros(1)
    h = lib().orc_triangle_hit(*[_p(a) for a in arrs], C.c_double(t0), C.c_double(t1), _p(t), _p(b1), _p(b2))
    return bool(h), float(t[0]), float(b1[0]), float(b2[0])


def label(scene, leaf_tri_off, leaf_tris, rays, leaf, t0, t1):
    n = rays.shape[0]
    gt = np.zeros((n, 9), np.float64)
    lib().orc_label(_p(_c(scene.verts, np.float32)), _p(_c(scene.tris, np.uint32)),
                    _p(_c(scene.vnormals, np.float32)), _p(_c(scene.albedo, np.float32)),
                    _p(_c(leaf_tri_off, np.int64)), _p(_c(leaf_tris, np.int32)), _p(_c(rays, np.float32)),
                    _p(_c(leaf, np.int32)), _p(_c(t0, np.float32)), _p(_c(t1, np.float32)), C.c_int64(n), _p(gt))
    return gt


def sample_loss(z, gt):
    z = _c(z, np.float64)
    gt = _c(gt, np.float64)
    terms = np.zeros(4)
    dz = np.zeros(8)
    L = lib().orc_sample_loss(_p(z), _p(gt), _p(terms), _p(dz))
    return float(L), terms, dz


def train_grad(grid: Grid, n_points, table_fp16, layers, leaf_lo, leaf_hi, leaf_rank, leaf_tri_off, leaf_tris,
               scene, rays, u, xi, dom_box=None):
    dims, W_all, b_all = _mlp_arrays(layers)
    tab = _c(table_fp16, np.float16).view(np.uint16)
    rays = _c(rays, np.float32)
    n = rays.shape[0]
    nW = int(sum(int(dims[k]) * int(dims[k + 1]) for k in range(len(layers))))
    nb = int(sum(int(dims[k + 1]) for k in range(len(layers))))
    out = dict(g_table=np.zeros(grid.n_entries * grid.F), g_W=np.zeros(nW), g_b=np.zeros(nb),
               accepted=np.zeros(n, np.uint8), first_leaf=np.zeros(n, np.int32), loss=np.zeros(n),
               gt=np.zeros((n, 9)), loss_sum=np.zeros(1))
    lo = _c(leaf_lo, np.float32)
    n_acc = lib().orc_train_grad(
        grid.L, grid.F, grid.log2_T, n_points, len(layers), _p(grid.res), _p(grid.dense), _p(grid.offset), _p(tab),
        C.c_int64(grid.n_entries), _p(dims), _p(W_all), _p(b_all), _p(lo), _p(_c(leaf_hi, np.float32)),
        C.c_int32(lo.shape[0]), _p(_c(leaf_rank, np.float32)), _p(_c(leaf_tri_off, np.int64)),
        _p(_c(leaf_tris, np.int32)), _p(_c(scene.verts, np.float32)), _p(_c(scene.tris, np.uint32)),
        _p(_c(scene.vnormals, np.float32)), _p(_c(scene.albedo, np.float32)), _p(rays), C.c_int64(n),
        _p(_c(u, np.float32)), _p(_c(xi, np.float32)), _p(out["g_table"]), _p(out["g_W"]), _p(out["g_b"]),
        _p(out["accepted"]), _p(out["first_leaf"]), _p(out["loss"]), _p(out["gt"]), _p(out["loss_sum"]),
        _box(dom_box))
    out["n_acc"] = int(n_acc)
    return out


def train_backward_given(grid: Grid, n_points, table_fp16, layers, dom_box, rays, t0, t1, xi, x, dz,
                         masks=None, want_deltas=False):
    """T6/T7 in double from GIVEN per-sample features x [m, D] and dL/dz [m, 8] (e.g. the
    GPU's own); samples are segments [t0, t1] of rays with jitter xi.  masks (optional uint8
    [m, H, 64]): ReLU decisions taken by the caller (the GPU's own, C36) instead of
    the double pre-activation's sign.  Returns sums (not means) g_table/g_W/g_b, their
    magnitude sums *_abs, z / z_abs of the MLP on x, the ReLU margin per sample (min over
    hidden units of |pre| / magnitude), per sample the number of given masks that disagree
    with the double sign and the largest margin among them, optionally hidden deltas."""
    dims, W_all, b_all = _mlp_arrays(layers)
    tab = _c(table_fp16, np.float16).view(np.uint16)
    rays = _c(rays, np.float32)
    m = rays.shape[0]
    nW = int(sum(int(dims[k]) * int(dims[k + 1]) for k in range(len(layers))))
    nb = int(sum(int(dims[k + 1]) for k in range(len(layers))))
    H = len(layers) - 1
    ne = grid.n_entries * grid.F
    out = dict(g_table=np.zeros(ne), g_W=np.zeros(nW), g_b=np.zeros(nb), g_table_abs=np.zeros(ne),
               g_W_abs=np.zeros(nW), g_b_abs=np.zeros(nb), z=np.zeros((m, 8)), z_abs=np.zeros((m, 8)),
               relu_margin=np.zeros(m), mask_flips=np.zeros(m, np.int32), flip_margin=np.zeros(m))
    hd = np.zeros((m, H, 64)) if want_deltas else None
    hda = np.zeros((m, H, 64)) if want_deltas else None
    mk = None if masks is None else _c(masks, np.uint8).reshape(m, H, 64)
    lib().orc_train_backward_given(
        grid.L, grid.F, grid.log2_T, n_points, len(layers), _p(grid.res), _p(grid.dense), _p(grid.offset), _p(tab),
        C.c_int64(grid.n_entries), _p(dims), _p(W_all), _p(b_all), _p(_c(dom_box, np.float32)), C.c_int64(m),
        _p(rays), _p(_c(t0, np.float32)), _p(_c(t1, np.float32)), _p(_c(xi, np.float32)), _p(_c(x, np.float64)),
        _p(_c(dz, np.float64)), _p(mk), _p(out["g_table"]), _p(out["g_W"]), _p(out["g_b"]), _p(out["g_table_abs"]),
        _p(out["g_W_abs"]), _p(out["g_b_abs"]), _p(out["z"]), _p(out["z_abs"]), _p(out["relu_margin"]),
        _p(out["mask_flips"]), _p(out["flip_margin"]), _p(hd), _p(hda))
    if want_deltas:
        out["hidden_delta"], out["hidden_delta_abs"] = hd, hda
    return out


def batch_loss_double(grid: Grid, n_points, table, dims, W_all, b_all, leaf_lo, leaf_hi, rays, xi, accepted,
                      t0, t1, gt, den=None, den_mode=0, dom_box=None):
    lo = _c(leaf_lo, np.float32)
    if den is None:
        den = np.zeros((rays.shape[0], 3))
    return float(lib().orc_batch_loss_double(
        grid.L, grid.F, grid.log2_T, n_points, len(dims) - 1, _p(grid.res), _p(grid.dense), _p(grid.offset),
        _p(_c(table, np.float64)), _p(_c(dims, np.int32)), _p(_c(W_all, np.float64)), _p(_c(b_all, np.float64)),
        _p(lo), _p(_c(leaf_hi, np.float32)), C.c_int32(lo.shape[0]), _p(_c(rays, np.float32)),
        C.c_int64(rays.shape[0]), _p(_c(xi, np.float32)), _p(_c(accepted, np.uint8)), _p(_c(t0, np.float32)),
        _p(_c(t1, np.float32)), _p(_c(gt, np.float64)), _p(den), C.c_int32(den_mode), _box(dom_box)))


def leaf_error_stats(first_leaf, accepted, sample_loss, n_leaves):
    """Per-leaf node-error statistics of one training batch: q = the leaf's training
    loss (mean of its accepted samples' losses), p = the fraction of the batch's rays whose
    first intersected leaf it is (C38).  Returns (q [n], p [n], samples [n], loss sum [n])."""
    fl = np.asarray(first_leaf)
    acc = np.asarray(accepted).astype(bool)
    n_rays = fl.shape[0]
    samples = np.bincount(fl[acc], minlength=n_leaves).astype(np.float64)
    loss_sum = np.bincount(fl[acc], weights=np.asarray(sample_loss, np.float64)[acc], minlength=n_leaves)
    first = np.bincount(fl[fl >= 0], minlength=n_leaves).astype(np.float64)
    q = np.divide(loss_sum, samples, out=np.zeros(n_leaves), where=samples > 0)
    return q, first / max(n_rays, 1), samples, loss_sum


def expand_cut(child_a, child_b, leaf_base, q, p, n_splits):
    """One cut-expansion step: the n_splits highest-ranked splittable leaves
    (r = 2 ln q + ln p) replaced by their two children; returns the sorted new node set."""
    lb = _c(leaf_base, np.int32)
    out = np.zeros(lb.size + n_splits, np.int32)
    n = lib().orc_expand_cut(_p(_c(child_a, np.int32)), _p(_c(child_b, np.int32)), C.c_int32(lb.size), _p(lb),
                             _p(_c(q, np.float64)), _p(_c(p, np.float64)), C.c_int32(n_splits), _p(out))
    return out[:n]


def adam(param, grad, m, v, step, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
    for a in (param, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = _c(grad, np.float64)
    lib().orc_adam(_p(param), _p(g), _p(m), _p(v), C.c_int64(param.size), C.c_int64(step), C.c_double(lr),
                   C.c_double(beta1), C.c_double(beta2), C.c_double(eps))
