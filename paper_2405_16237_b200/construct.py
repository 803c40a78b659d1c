"""Error-driven N-BVH construction (BASELINE cfg 4's "error-driven cuts").

PAPER §5.1: start from the root of the base BVH; alternate training the model on the
current cut with splitting the leaves of largest error into their two children; the number
of training iterations between expansions and the number of splits both grow by a user
factor; stop at the target leaf count and run one final, longer training round.
Node error: rank r = 2 log q + log p, q = the leaf's training loss (mean over its
samples), p = the fraction of training rays that hit it first.  Acceptance: a ray's
first leaf is trained with probability max(r_hat/r_hat_max, 0.005) (C18) -- ranks are
handed to the library with nbvh_set_leaf_rank after every round.  Level of detail:
every `lod_every` iterations the current cut is registered in the next LoD slot
(nbvh_copy_cut); during training a registered cut (or the working cut) is picked uniformly
at random, and only steps on the working cut feed its statistics.

This module only orchestrates C-ABI calls (every step runs in the library's kernels); the
per-leaf statistics are accumulated on the device from the gradient-buffer tail.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Schedule:
    """P:180 schedule.  Defaults follow fig. train_time_ablation's budget shape: a
    cut-optimisation phase followed by a longer training-only phase."""
    iters0: int = 20            # training iterations before the first expansion
    splits0: int = 1            # leaves split at the first expansion
    growth: float = 1.5         # factor applied to both after every expansion
    final_iters: int = 200      # final training round on the finished cut
    lod_every: int = 0          # register an LoD every this many iterations; 0 = off
    lod_at_leaves: tuple = ()   # alternatively: register when the cut first reaches these sizes
    max_lods: int = 3
    lr: float = 0.01            # Adam


@dataclass
class RoundLog:
    n_leaves: int
    iters: int
    loss: float                 # mean per-sample loss over the round (working cut)
    lods: list = field(default_factory=list)


def _leaf_of_triangle(cut) -> np.ndarray:
    owner = np.empty(int(cut["tri_off"][-1]), np.int64)
    for i in range(cut["n_leaves"]):
        owner[cut["tris"][cut["tri_off"][i]:cut["tri_off"][i + 1]]] = i
    return owner


def ranks_from_stats(loss_sum, samples, first_hits, n_rays):
    """r = 2 ln q + ln p.  Leaves without samples keep the lowest rank of the cut."""
    q = np.where(samples > 0, loss_sum / np.maximum(samples, 1), np.nan)
    p = first_hits / max(n_rays, 1)
    r = 2.0 * np.log(np.maximum(q, 1e-12)) + np.log(np.maximum(p, 1e-12))
    r = np.where(np.isfinite(r), r, np.nan)
    fill = np.nanmin(r) if np.any(np.isfinite(r)) else 0.0
    return np.where(np.isnan(r), fill, r).astype(np.float32), q, p


def construct(ctx, target_leaves: int, batch_fn, schedule: Schedule | None = None, stream=None, log=None,
              distributed: bool = True, group=None):
    """Build an error-driven cut of `target_leaves` leaves in LoD slot 0 while training the
    context's model.  batch_fn(step) -> (rays, u, xi) device tensors of one training batch
    (under data parallelism: this rank's shard).  Returns the per-round log; registered LoD
    cuts are in slots 1.. (coarsest first).

    distributed=True: every step all-reduces the gradient buffer over `group` (when a process
    group is initialised), and the per-leaf statistics are read from the REDUCED buffer, with
    the ray count summed over ranks, so every rank computes the same ranks and builds the same
    cut.  Pass distributed=False when only one rank runs the construction."""
    import torch
    from . import dp
    sch = schedule or Schedule()
    world = dp.world_size(group) if distributed else 1
    ctx.build_cut(1)                                            # the root
    ctx.set_leaf_rank(np.zeros(1, np.float32))
    n_params = ctx.param_count(3)
    iters, splits = sch.iters0, sch.splits0
    step = 0
    lods = []                                                   # registered slots
    rng = np.random.default_rng(12345)
    history = []

    def train_round(n_iters, collect):
        nonlocal step
        n_leaves = ctx.cut(0)["n_leaves"]
        acc = torch.zeros(1 + 3 * n_leaves, dtype=torch.float64, device="cuda")
        n_rays = 0
        for _ in range(n_iters):
            rays, u, xi = batch_fn(step)
            pool = [0] + lods
            lod = pool[int(rng.integers(len(pool)))] if lods else 0     # P:252 random cut
            ctx.train_backward(rays, u, xi, lod, stream=stream)
            g = dp.grad_tensor(ctx)
            if world > 1:
                dp.allreduce_grads(g, group)
            if collect and lod == 0:                            # global statistics (after the reduce)
                acc += g[n_params:n_params + 1 + 3 * n_leaves].double()
                n_rays += rays.shape[0]
            ctx.apply_update(sch.lr, stream=stream)
            step += 1
            if sch.lod_every and step % sch.lod_every == 0 and len(lods) < sch.max_lods:
                slot = len(lods) + 1
                ctx.copy_cut(0, slot)                           # register an LoD
                lods.append(slot)
        if world > 1:                                           # rays of every rank's shard
            nr = torch.tensor([n_rays], dtype=torch.float64, device=acc.device)
            dp.allreduce_grads(nr, group)
            n_rays = int(nr.item())
        a = acc.cpu().numpy()
        per = a[1:].reshape(-1, 3) if n_leaves else np.zeros((0, 3))
        return per[:, 0], per[:, 1], per[:, 2], n_rays, (a[0] and per[:, 0].sum() / max(a[0], 1))

    pending = sorted(sch.lod_at_leaves)
    while True:
        cut = ctx.cut(0)
        n = cut["n_leaves"]
        while pending and n >= pending[0] and len(lods) < sch.max_lods:
            pending.pop(0)
            slot = len(lods) + 1
            ctx.copy_cut(0, slot)                                # register an LoD
            lods.append(slot)
        loss_sum, samples, first, n_rays, mean_loss = train_round(iters, True)
        history.append(RoundLog(n, iters, float(mean_loss), list(lods)))
        if log:
            log(history[-1])
        if n >= target_leaves:
            break
        r, q, p = ranks_from_stats(loss_sum, samples, first, n_rays)
        owner = _leaf_of_triangle(cut)
        new_n, _ = ctx.build_cut(min(target_leaves, n + splits), q=np.nan_to_num(q, nan=1e-12).astype(np.float32),
                                 p=p.astype(np.float32))
        if new_n == n:                                          # nothing left to split
            break
        new = ctx.cut(0)
        parent = owner[new["tris"][new["tri_off"][:-1]]]       # each new leaf lies inside one old leaf
        ctx.set_leaf_rank(r[parent])                            # children inherit the rank (C18)
        iters = int(math.ceil(iters * sch.growth))
        splits = int(math.ceil(splits * sch.growth))
    # final, longer training round on the finished cut
    loss_sum, samples, first, n_rays, mean_loss = train_round(sch.final_iters, True)
    r, _, _ = ranks_from_stats(loss_sum, samples, first, n_rays)
    ctx.set_leaf_rank(r)
    history.append(RoundLog(ctx.cut(0)["n_leaves"], sch.final_iters, float(mean_loss), list(lods)))
    if log:
        log(history[-1])
    return history
