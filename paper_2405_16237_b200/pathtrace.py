"""Hybrid wavefront path tracer (NEXT-3, BASELINE cfg 3; PAPER §7).

Two BLAS share one ray stream: a neural one (an N-BVH context queried with nbvh_query) and a
classical one (a context whose own triangle mesh is intersected through its base BVH,
nbvh_intersect_mesh).  Every bounce: both BLAS answer the same rays with the same hit record,
nbvh_pt_shade keeps the closer hit, adds sky radiance for escaped rays and continues hits
diffusely.  This module only sequences the C-ABI calls on one stream; every per-ray step
runs in the library's kernels.  Multi-GPU: frames (or ray batches) are split over ranks with
no collective (replicas, like the query).
"""
from __future__ import annotations

import numpy as np

SKY = np.array([0.9, 0.95, 1.0, 0.35, 0.55, 1.0], np.float32)   # horizon rgb, zenith rgb


class PathTracer:
    def __init__(self, neural_ctx, classical_ctx=None, n_max: int = 0, device="cuda"):
        import torch
        self.neural, self.classical = neural_ctx, classical_ctx
        self.device = device
        self.n_max = 0
        self._alloc(n_max, torch)

    def _alloc(self, n, torch):
        if n <= self.n_max:
            return
        self.n_max = n
        self.ha = self.neural.alloc_hits(n, self.device)
        self.hb = self.neural.alloc_hits(n, self.device) if self.classical is not None else None
        self.rays = [torch.empty(n, 8, device=self.device), torch.empty(n, 8, device=self.device)]
        self.thr = torch.empty(n, 3, device=self.device)
        self.rad = torch.empty(n, 3, device=self.device)
        self.alive = torch.zeros(8, dtype=torch.int32, device=self.device)

    def render(self, rays, bounces: int = 4, seed: int = 0, lod: int = 0, sky=SKY, eps: float = 1e-4, stream=None):
        """rays: device float32 [n, 8] primary rays.  Returns (radiance [n, 3] view, alive
        counts per bounce as a device tensor: rays that continued after each bounce)."""
        import torch
        n = rays.shape[0]
        self._alloc(n, torch)
        cur, nxt = self.rays
        cur[:n].copy_(rays)
        self.thr[:n].fill_(1.0)
        self.rad[:n].zero_()
        self.alive.zero_()
        sub = lambda h: None if h is None else {k: v[:n] for k, v in h.items()}
        ha, hb = sub(self.ha), sub(self.hb)
        for b in range(bounces):
            self.neural.query(cur[:n], lod=lod, out=ha, stream=stream)
            if self.classical is not None:
                self.classical.intersect_mesh(cur[:n], out=hb, stream=stream)
            self.neural.pt_shade(cur[:n], ha, hb, self.thr[:n], self.rad[:n], nxt[:n], seed, b, sky, eps,
                                 self.alive[b:b + 1], stream=stream)
            cur, nxt = nxt, cur
        return self.rad[:n], self.alive[:bounces]
