"""Hybrid wavefront path tracer over a two-level hierarchy (NEXT-3, BASELINE cfg 3; PAPER §7,
P:267).

A TLAS (nbvh_tlas_build: a BVH over instance boxes) places BLAS in the world through affine
transforms; a BLAS is neural (an N-BVH context answered by nbvh_query) or classical (a context
whose own triangle mesh is intersected through its base BVH, nbvh_intersect_mesh), and both
yield the same hit record.  Every bounce, on the COMPACTED alive paths only:

  nbvh_tlas_dispatch   TLAS traversal; each crossed instance gets the path's ray in its object
                       space, appended to its BLAS's list
  query / intersect    one call per BLAS on its list; the neural BLAS uses LoD slot
                       `lod_primary` for camera rays and `lod_secondary` after the first hit
                       ("switch to a coarser LoD after the primary hit")
  nbvh_tlas_merge      closest hit per path, normal back to world space
  nbvh_pt_shade_compact  sky radiance for escaped paths, diffuse continuation for hits, the
                       continuing paths appended to the next bounce's compacted list

This module only sequences C-ABI calls; every per-ray step runs in the library's kernels.
The list sizes of each bounce are read back to the host (one small copy per bounce) because
the BLAS calls take their ray count on the host.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .nbvh import Hits, Instance, MAX_BLAS, _ptr, _stream_ptr, load_library

SKY = np.array([0.9, 0.95, 1.0, 0.35, 0.55, 1.0], np.float32)   # horizon rgb, zenith rgb


def affine_inverse(m34: np.ndarray) -> np.ndarray:
    """Inverse of the 3x4 affine map x -> M x + t (object -> world): world -> object [A | b]."""
    m = np.asarray(m34, np.float64).reshape(3, 4)
    a = np.linalg.inv(m[:, :3])
    return np.concatenate([a, -(a @ m[:, 3])[:, None]], axis=1)


def world_box(m34, lo, hi):
    """World box of an object box under x -> M x + t (the 8 corners)."""
    m = np.asarray(m34, np.float64).reshape(3, 4)
    c = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])], np.float64)
    w = c @ m[:, :3].T + m[:, 3]
    return w.min(0), w.max(0)


class Tlas:
    """nbvh_tlas: instances = [(blas index, object->world 3x4, object box lo, hi)]."""

    def __init__(self, ctx, instances):
        self.lib = load_library()
        self.ctx = ctx
        arr = (Instance * len(instances))()
        self.n_inst = len(instances)
        self.inst_blas = []
        self.w2o = []
        for i, (b, m34, lo, hi) in enumerate(instances):
            a = affine_inverse(m34)
            wlo, whi = world_box(m34, lo, hi)
            # the box must contain everything the BLAS can report: an N-BVH's leaf boxes are
            # inflated by up to max(1e-3 diag, 1e-6 scene diag) per side (C15)
            pad = 4e-3 * float(np.linalg.norm(whi - wlo)) + 1e-6
            arr[i].world_to_object[:] = [float(v) for v in a.reshape(-1)]
            arr[i].lo[:] = [float(v - pad) for v in wlo]
            arr[i].hi[:] = [float(v + pad) for v in whi]
            arr[i].blas = int(b)
            self.inst_blas.append(int(b))
            self.w2o.append(a)
        self.n_blas = max(self.inst_blas) + 1
        assert self.n_blas <= MAX_BLAS
        h = C.c_void_p()
        ctx._ck(self.lib.nbvh_tlas_build(ctx.h, C.cast(arr, C.c_void_p), self.n_inst, C.byref(h)), "tlas_build")
        self.h = h

    def close(self):
        if self.h:
            self.lib.nbvh_tlas_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dispatch(self, rays, m, out_rays, out_src, out_inst, counts, cap, stream=None):
        self.ctx._ck(self.lib.nbvh_tlas_dispatch(self.ctx.h, self.h, _ptr(rays), int(m), _ptr(out_rays), _ptr(out_src),
                                                 _ptr(out_inst), _ptr(counts), int(cap), _stream_ptr(stream)),
                     "tlas_dispatch")

    def merge(self, m, counts, cap, src, inst, lists, out, stream=None):
        arr = (Hits * self.n_blas)(*[self.ctx._hits(h) for h in lists])
        self.ctx._ck(self.lib.nbvh_tlas_merge(self.ctx.h, self.h, int(m), _ptr(counts), int(cap), _ptr(src),
                                              _ptr(inst), C.cast(arr, C.c_void_p), self.ctx._hits(out),
                                              _stream_ptr(stream)), "tlas_merge")

    def overflow(self) -> int:
        f = np.zeros(1, np.int32)
        self.ctx._ck(self.lib.nbvh_tlas_overflow(self.ctx.h, self.h, _ptr(f)), "tlas_overflow")
        return int(f[0])


class PathTracer:
    """blas = [(context, "neural" | "mesh")]; instances = [(blas index, object->world 3x4)].
    Object boxes: a neural BLAS's scene box (its mesh bounds), a classical BLAS's mesh bounds."""

    def __init__(self, blas, instances, n_max: int, device="cuda", lod_primary: int = 0, lod_secondary=None):
        import torch
        self.blas = blas
        self.device = device
        self.lod_primary = lod_primary
        self.lod_secondary = lod_primary if lod_secondary is None else lod_secondary
        boxes = []
        for ctx, kind in blas:
            v = np.asarray(ctx.scene.verts, np.float64)
            boxes.append((v.min(0), v.max(0)))
        self.tlas = Tlas(blas[0][0], [(b, m, *boxes[b]) for b, m in instances])
        per_blas = np.bincount(self.tlas.inst_blas, minlength=len(blas))
        self.cap = int(n_max * max(1, int(per_blas.max())))
        for ctx, kind in blas:
            if kind == "neural":
                ctx.reserve(self.cap)
        self.n_max = n_max
        f32 = dict(dtype=torch.float32, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        nb = len(blas)
        self.lrays = torch.empty(nb * self.cap, 8, **f32)
        self.lsrc = torch.empty(nb * self.cap, **i32)
        self.linst = torch.empty(nb * self.cap, **i32)
        self.counts = torch.zeros(nb, **i32)
        self.lhits = [blas[0][0].alloc_hits(self.cap, device) for _ in range(nb)]
        self.hits = blas[0][0].alloc_hits(n_max, device)
        self.rays = [torch.empty(n_max, 8, **f32), torch.empty(n_max, 8, **f32)]
        self.pix = [torch.empty(n_max, **i32), torch.empty(n_max, **i32)]
        self.thr = [torch.empty(n_max, 3, **f32), torch.empty(n_max, 3, **f32)]
        self.radiance = torch.empty(n_max, 3, **f32)
        self.next_count = torch.zeros(1, **i32)

    def render(self, rays, bounces: int = 4, seed: int = 0, sky=SKY, eps: float = 1e-4, stream=None):
        """rays: device float32 [n, 8] primary (camera) rays, n <= n_max.  Returns (radiance
        [n, 3], alive path counts entering each bounce [bounces] (host ints))."""
        import torch
        n = rays.shape[0]
        assert n <= self.n_max
        cur, nxt = 0, 1
        self.rays[cur][:n].copy_(rays)
        self.pix[cur][:n].copy_(torch.arange(n, dtype=torch.int32, device=self.device))
        self.thr[cur][:n].fill_(1.0)
        self.radiance[:n].zero_()
        sky_a = np.ascontiguousarray(sky, np.float32)
        ctx0 = self.blas[0][0]
        m = n
        alive = []
        for b in range(bounces):
            alive.append(m)
            if m == 0:
                continue
            self.tlas.dispatch(self.rays[cur], m, self.lrays, self.lsrc, self.linst, self.counts, self.cap, stream)
            counts = self.counts.cpu().numpy()                         # the BLAS calls take n on the host
            lists = []
            for k, (ctx, kind) in enumerate(self.blas):
                cnt = int(min(counts[k], self.cap))
                sub_rays = self.lrays[k * self.cap:k * self.cap + cnt]
                out = {key: v for key, v in self.lhits[k].items()}
                if cnt:
                    oc = {key: v[:cnt] for key, v in out.items()}
                    if kind == "neural":
                        ctx.query(sub_rays, lod=self.lod_primary if b == 0 else self.lod_secondary, out=oc,
                                  stream=stream)
                    else:
                        ctx.intersect_mesh(sub_rays, out=oc, stream=stream)
                lists.append(out)
            self.tlas.merge(m, self.counts, self.cap, self.lsrc.view(-1), self.linst.view(-1),
                            [{key: v for key, v in h.items()} for h in lists], self.hits, stream)
            self.next_count.zero_()
            ctx0._ck(ctx0.lib.nbvh_pt_shade_compact(
                ctx0.h, _ptr(self.rays[cur]), int(m), ctx0._hits(self.hits), _ptr(self.pix[cur]), _ptr(self.thr[cur]),
                _ptr(self.radiance), _ptr(self.rays[nxt]), _ptr(self.pix[nxt]), _ptr(self.thr[nxt]),
                _ptr(self.next_count), int(seed), int(b), _ptr(sky_a), float(eps), _stream_ptr(stream)),
                "pt_shade_compact")
            m = int(self.next_count.item())
            cur, nxt = nxt, cur
        if self.tlas.overflow():
            raise RuntimeError("TLAS dispatch list or stack overflow")
        return self.radiance[:n], alive


class PathTracerFlat:
    """Round-1 reference renderer without a TLAS: both BLAS answer EVERY ray (identity
    transforms), dead rays stay in the arrays (tmin > tmax), nbvh_pt_shade picks the closer
    hit (ties: neural).  Kept to A/B the compacted TLAS renderer: with identity instances
    [neural, mesh] both give the same radiance (the random streams are keyed by pixel)."""

    def __init__(self, neural_ctx, classical_ctx=None, n_max: int = 0, device="cuda"):
        import torch
        self.neural, self.classical = neural_ctx, classical_ctx
        self.device = device
        self.n_max = n_max
        self.ha = self.neural.alloc_hits(n_max, device)
        self.hb = self.neural.alloc_hits(n_max, device) if classical_ctx is not None else None
        self.rays = [torch.empty(n_max, 8, device=device), torch.empty(n_max, 8, device=device)]
        self.thr = torch.empty(n_max, 3, device=device)
        self.rad = torch.empty(n_max, 3, device=device)
        self.alive = torch.zeros(8, dtype=torch.int32, device=device)

    def render(self, rays, bounces: int = 4, seed: int = 0, lod_primary: int = 0, lod_secondary=None, sky=SKY,
               eps: float = 1e-4, stream=None):
        n = rays.shape[0]
        lod2 = lod_primary if lod_secondary is None else lod_secondary
        cur, nxt = self.rays
        cur[:n].copy_(rays)
        self.thr[:n].fill_(1.0)
        self.rad[:n].zero_()
        self.alive.zero_()
        sub = lambda h: None if h is None else {k: v[:n] for k, v in h.items()}
        ha, hb = sub(self.ha), sub(self.hb)
        for b in range(bounces):
            self.neural.query(cur[:n], lod=lod_primary if b == 0 else lod2, out=ha, stream=stream)
            if self.classical is not None:
                self.classical.intersect_mesh(cur[:n], out=hb, stream=stream)
            self.neural.pt_shade(cur[:n], ha, hb, self.thr[:n], self.rad[:n], nxt[:n], seed, b, sky, eps,
                                 self.alive[b:b + 1], stream=stream)
            cur, nxt = nxt, cur
        return self.rad[:n], self.alive[:bounces]
