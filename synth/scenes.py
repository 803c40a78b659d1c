"""Seeded procedural scenes, rays and random parameter values.

Scene recipe follows SURVEY.md §8(d) "Synthetic inputs":
  * cfg 1 (tiny): class-I geodesic icosphere, frequency 22 -> 9,680 triangles,
    radially displaced by a 4-octave sine sum, 3D-checker albedo, area-weighted
    vertex normals; 64x64 pinhole camera at (0,0,3.5), vfov 40 deg.
  * cfg 2 (1080p): 512x512-quad fBm value-noise heightfield (524,288 tris) plus
    48 displaced icospheres on a jittered 8x6 grid (464,640 tris) -> 988,928
    triangles; 1920x1080 pinhole camera at (0,0.6,1.6) looking at the origin,
    vfov 50 deg.
The paper's own scenes are proprietary (Table 2); these
stand-ins reproduce the workload's shape (triangle count, depth complexity,
coherent primary rays), not its content.

Nothing here implements the N-BVH method: no slab test, hashing, encoding,
MLP or decode.  Both the oracle and the CUDA path consume these arrays.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Scene:
    verts: np.ndarray     # float32 [nv, 3]
    tris: np.ndarray      # uint32 [nt, 3]
    vnormals: np.ndarray  # float32 [nv, 3] unit
    albedo: np.ndarray    # float32 [nt, 3] in [0, 1]

    @property
    def n_tris(self) -> int:
        return int(self.tris.shape[0])


@dataclasses.dataclass(frozen=True)
class HashCfg:
    L: int            # levels
    log2_T: int       # table size exponent
    F: int            # features per level
    n_points: int     # samples per segment
    hidden_layers: int
    width: int = 64
    base_res: int = 8
    max_res: int = 1024


# BASELINE.json "configs" (cfg 1 and cfg 2 are the query workloads).
CONFIGS = {
    "tiny": dict(hash=HashCfg(L=8, log2_T=14, F=2, n_points=4, hidden_layers=2),
                 leaves=64, res=(64, 64), eye=(0.0, 0.0, 3.5), vfov=40.0,
                 seeds=dict(mesh=1, weights=2, train=3)),
    "1080p": dict(hash=HashCfg(L=16, log2_T=19, F=2, n_points=4, hidden_layers=3),
                  leaves=2048, res=(1920, 1080), eye=(0.0, 0.6, 1.6), vfov=50.0,
                  seeds=dict(mesh=4, weights=5, train=6)),
    # the paper's own setting (8 levels, 4 features, 4x64 MLP;
    # 2^18 hash map; three points per segment) on the tiny scene.
    "paper": dict(hash=HashCfg(L=8, log2_T=18, F=4, n_points=3, hidden_layers=4),
                  leaves=64, res=(64, 64), eye=(0.0, 0.0, 3.5), vfov=40.0,
                  seeds=dict(mesh=1, weights=12, train=13)),
}


# ---------------------------------------------------------------- meshes
def _icosahedron():
    p = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
                  [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
                  [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]], dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    return v, f


def icosphere(nu: int) -> tuple[np.ndarray, np.ndarray]:
    """Class-I geodesic sphere of frequency nu: 20*nu^2 triangles, 10*nu^2+2 vertices (float64 unit)."""
    v, f = _icosahedron()
    pts, tris = [], []
    base = 0
    for a, b, c in f:
        A, B, C = v[a], v[b], v[c]
        idx = {}
        local = []
        for i in range(nu + 1):
            for j in range(nu + 1 - i):
                idx[(i, j)] = len(local)
                local.append(A + (B - A) * (i / nu) + (C - A) * (j / nu))
        for i in range(nu):
            for j in range(nu - i):
                tris.append((base + idx[(i, j)], base + idx[(i + 1, j)], base + idx[(i, j + 1)]))
                if i + j < nu - 1:
                    tris.append((base + idx[(i + 1, j)], base + idx[(i + 1, j + 1)], base + idx[(i, j + 1)]))
        pts.extend(local)
        base += len(local)
    P = np.asarray(pts)
    P /= np.linalg.norm(P, axis=1, keepdims=True)
    key = np.round(P * 1e9).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    V = P[first]
    T = inv.reshape(-1)[np.asarray(tris, dtype=np.int64)]
    # outward orientation
    e = np.cross(V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]])
    flip = (e * V[T].mean(axis=1)).sum(axis=1) < 0
    T[flip] = T[flip][:, ::-1]
    return V, T


def _displace_sphere(V: np.ndarray, rng: np.random.Generator, amp: float = 0.1) -> np.ndarray:
    r = np.ones(len(V))
    for k in range(1, 5):
        a = rng.normal(size=3)
        a /= np.linalg.norm(a)
        phi = rng.uniform(0, 2 * math.pi)
        r += amp * 2.0 ** (-k) * np.sin(2.0 ** (k + 1) * (V @ a) + phi)
    return V * r[:, None]


def _vertex_normals(V: np.ndarray, T: np.ndarray) -> np.ndarray:
    e = np.cross(V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]])  # 2*area*n
    N = np.zeros_like(V)
    for k in range(3):
        np.add.at(N, T[:, k], e)
    N /= np.maximum(np.linalg.norm(N, axis=1, keepdims=True), 1e-30)
    return N


def _checker_albedo(V: np.ndarray, T: np.ndarray, cells: int = 8) -> np.ndarray:
    c = V[T].mean(axis=1)
    k = np.floor((c + 1.0) * 0.5 * cells).astype(np.int64)
    par = (k.sum(axis=1) & 1).astype(bool)
    col = np.where(par[:, None], np.array([0.8, 0.3, 0.2]), np.array([0.2, 0.6, 0.9]))
    return col


def _finish(V, T, A) -> Scene:
    N = _vertex_normals(V, T)
    return Scene(verts=V.astype(np.float32), tris=T.astype(np.uint32),
                 vnormals=N.astype(np.float32), albedo=A.astype(np.float32))


def scene_tiny(seed: int = 1, nu: int = 22) -> Scene:
    """cfg 1: displaced icosphere, 20*nu^2 = 9,680 triangles, fitted to [-1,1]^3."""
    rng = np.random.default_rng(seed)
    V, T = icosphere(nu)
    V = _displace_sphere(V, rng)
    V /= np.abs(V).max()
    return _finish(V, T, _checker_albedo(V, T))


def _value_noise(x: np.ndarray, z: np.ndarray, freq: int, rng: np.random.Generator) -> np.ndarray:
    lat = rng.uniform(-1, 1, size=(freq + 2, freq + 2))
    u = (x + 1) * 0.5 * freq
    w = (z + 1) * 0.5 * freq
    i = np.clip(np.floor(u).astype(np.int64), 0, freq)
    j = np.clip(np.floor(w).astype(np.int64), 0, freq)
    fu, fw = u - i, w - j
    su, sw = fu * fu * (3 - 2 * fu), fw * fw * (3 - 2 * fw)
    a = lat[i, j] * (1 - su) + lat[i + 1, j] * su
    b = lat[i, j + 1] * (1 - su) + lat[i + 1, j + 1] * su
    return a * (1 - sw) + b * sw


def _fbm_fn(rng: np.random.Generator, octaves: int = 5, amp: float = 0.15):
    seeds = rng.integers(0, 2**31, size=octaves)

    def h(x, z):
        tot = np.zeros_like(x, dtype=np.float64)
        norm = 0.0
        for o in range(octaves):
            r = np.random.default_rng(int(seeds[o]))
            tot += 0.5 ** o * _value_noise(x, z, 4 * 2 ** o, r)
            norm += 0.5 ** o
        return amp * tot / norm
    return h


def scene_1080p_parts(seed: int = 4, grid: int = 512, nu: int = 22) -> tuple[Scene, Scene]:
    """cfg 3 (hybrid scene): the cfg-2 scene split into its two instances -- the heightfield
    (classical BLAS) and the 48 icospheres (neural BLAS) -- same geometry and albedo."""
    full = scene_1080p(seed, grid, nu)
    nt = 2 * grid * grid
    nv = (grid + 1) * (grid + 1)
    terrain = Scene(full.verts[:nv], full.tris[:nt], full.vnormals[:nv], full.albedo[:nt])
    spheres = Scene(full.verts[nv:], (full.tris[nt:] - nv).astype(full.tris.dtype), full.vnormals[nv:],
                    full.albedo[nt:])
    return terrain, spheres


def scene_1080p(seed: int = 4, grid: int = 512, nu: int = 22) -> Scene:
    """cfg 2: fBm heightfield (grid^2*2 tris) + 48 displaced icospheres -> 988,928 tris."""
    rng = np.random.default_rng(seed)
    h = _fbm_fn(rng)
    g = np.linspace(-1.0, 1.0, grid + 1)
    X, Z = np.meshgrid(g, g, indexing="ij")
    Y = h(X, Z)
    Vt = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
    ii, jj = np.meshgrid(np.arange(grid), np.arange(grid), indexing="ij")
    v00 = (ii * (grid + 1) + jj).reshape(-1)
    v10 = v00 + (grid + 1)
    v01 = v00 + 1
    v11 = v10 + 1
    Tt = np.concatenate([np.stack([v00, v01, v10], 1), np.stack([v10, v01, v11], 1)], axis=0)
    # orient up (+y)
    e = np.cross(Vt[Tt[:, 1]] - Vt[Tt[:, 0]], Vt[Tt[:, 2]] - Vt[Tt[:, 0]])
    flip = e[:, 1] < 0
    Tt[flip] = Tt[flip][:, ::-1]
    Vs0, Ts0 = icosphere(nu)
    Vparts, Tparts = [Vt], [Tt]
    base = len(Vt)
    for gx in range(8):
        for gz in range(6):
            cx = -0.9 + 1.8 * (gx + 0.5) / 8 + rng.uniform(-0.3, 0.3) * 1.8 / 8
            cz = -0.9 + 1.8 * (gz + 0.5) / 6 + rng.uniform(-0.3, 0.3) * 1.8 / 6
            rad = rng.uniform(0.04, 0.12)
            cy = float(h(np.array([cx]), np.array([cz]))[0]) + 0.8 * rad
            Vs = _displace_sphere(Vs0, rng) * rad + np.array([cx, cy, cz])
            Vparts.append(Vs)
            Tparts.append(Ts0 + base)
            base += len(Vs)
    V = np.concatenate(Vparts, 0)
    T = np.concatenate(Tparts, 0)
    return _finish(V, T, _checker_albedo(V, T))


# ---------------------------------------------------------------- rays
def camera_rays(width: int, height: int, eye, target=(0.0, 0.0, 0.0), vfov_deg: float = 40.0,
                up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """Pinhole primary rays through pixel centres, AoS float32 [H*W, 8] =
    (ox,oy,oz,tmin, dx,dy,dz,tmax), row-major pixels, tmin=0, tmax=+inf."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right /= np.linalg.norm(right)
    upv = np.cross(right, fwd)
    th = math.tan(math.radians(vfov_deg) * 0.5)
    aspect = width / height
    xs = (2.0 * (np.arange(width) + 0.5) / width - 1.0) * th * aspect
    ys = (1.0 - 2.0 * (np.arange(height) + 0.5) / height) * th
    Xs, Ys = np.meshgrid(xs, ys)  # [H, W]
    d = fwd[None, None, :] + Xs[..., None] * right + Ys[..., None] * upv
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    d = d.reshape(-1, 3)
    out = np.empty((d.shape[0], 8), np.float32)
    out[:, 0:3] = eye
    out[:, 3] = 0.0
    out[:, 4:7] = d
    out[:, 7] = np.inf
    return out


def random_rays(n: int, seed: int, lo=(-1.5, -1.5, -1.5), hi=(1.5, 1.5, 1.5)) -> np.ndarray:
    """Origins uniform in the box [lo,hi], directions uniform on the sphere; AoS float32 [n, 8]."""
    rng = np.random.default_rng(seed)
    o = rng.uniform(lo, hi, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    out = np.empty((n, 8), np.float32)
    out[:, 0:3] = o
    out[:, 3] = 0.0
    out[:, 4:7] = d
    out[:, 7] = np.inf
    return out


# ---------------------------------------------------------------- parameters / random draws
def random_params_fp16(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """n values U[lo,hi] rounded to fp16; returned as float16 array."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=n).astype(np.float16)


def random_mlp(d_in: int, hidden_layers: int, width: int, seed: int, n_out: int = 8,
               out_scale: float = 10.0, bias_scale: float = 0.1):
    """He-uniform weights (fp16, [out][in] row-major) and small random fp32 biases.
    The output layer is scaled by out_scale so that logits spread (SURVEY.md §8(c) parity weights (a))."""
    rng = np.random.default_rng(seed)
    dims = [d_in] + [width] * hidden_layers + [n_out]
    layers = []
    for k in range(len(dims) - 1):
        fan_in, fan_out = dims[k], dims[k + 1]
        lim = math.sqrt(6.0 / fan_in)
        W = rng.uniform(-lim, lim, size=(fan_out, fan_in))
        if k == len(dims) - 2:
            W *= out_scale
        b = rng.uniform(-bias_scale, bias_scale, size=fan_out)
        layers.append((W.astype(np.float16), b.astype(np.float32)))
    return layers


def random_uniform(n: int, seed: int) -> np.ndarray:
    """n draws U[0,1) as float32 (acceptance u, stratification jitter xi)."""
    rng = np.random.default_rng(seed)
    return rng.random(n, dtype=np.float32)
