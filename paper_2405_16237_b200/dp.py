"""Multi-GPU plumbing: one process per GPU, torch.distributed for the process
group, NCCL on the GPU box (gloo in the CPU tests).

Training (BASELINE cfg 5): the global batch is split over ranks; each rank runs
nbvh_train_backward on its shard, the flat fp32 gradient buffer (nbvh_grad_buffer) is
all-reduced (sum) once per step and every rank applies the same Adam step.  The buffer holds
the parameter gradients of the SUM of per-sample losses, then the accepted-sample count, then
per-leaf (loss sum, samples, first hits); summed over ranks it is exactly the single-process
buffer of the whole batch, and nbvh_apply_update divides by the summed count (C29).

Query (BASELINE cfgs 2/3): the model is replicated -- built once on rank 0 and broadcast at
init (`broadcast_model`) -- and one frame's rays are partitioned over ranks by interleaved
16x16 pixel tiles (`tile_partition`) for load balance (depth complexity varies across the
screen).  There is no collective on the query's data path.
"""
from __future__ import annotations

import hashlib

import numpy as np


class _CudaArray:
    """Zero-copy view of a library-owned device buffer (CUDA array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def grad_tensor(ctx):
    """The context's gradient buffer as a torch tensor (no copy)."""
    import torch
    ptr, n = ctx.grad_buffer()
    return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{ctx.device}")


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def world_size(group=None) -> int:
    d = _dist()
    return d.get_world_size(group) if d else 1


def rank_of(group=None) -> int:
    d = _dist()
    return d.get_rank(group) if d else 0


def shard(n_global: int, rank: int, world: int) -> slice:
    """Contiguous, balanced split of a global batch of n_global rays."""
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return slice(start, start + base + (1 if rank < rem else 0))


def _morton_order(n: int) -> np.ndarray:
    """(y, x) of an n x n block (n a power of two) in Z order."""
    k = np.arange(n * n)
    x = np.zeros_like(k)
    y = np.zeros_like(k)
    for b in range(int(np.log2(n))):
        x |= ((k >> (2 * b)) & 1) << b
        y |= ((k >> (2 * b + 1)) & 1) << b
    return y, x


def tile_partition(width: int, height: int, rank: int, world: int, tile: int = 16, inner: str = "morton") -> np.ndarray:
    """Row-major pixel indices owned by `rank` when a width x height frame is cut into
    tile x tile tiles dealt round-robin along diagonals ((tx + ty) mod world), so every rank
    gets tiles from every part of the screen.  Pixels are listed tile by tile; inside a tile in
    Z (Morton) order (inner="morton": any 16 consecutive rays form a 4x4 block -- the rays a
    query-kernel warp takes together) or row-major (inner="rows").  Ragged edge tiles are
    clipped to the frame."""
    ntx, nty = (width + tile - 1) // tile, (height + tile - 1) // tile
    my, mx = _morton_order(tile) if inner == "morton" else np.divmod(np.arange(tile * tile), tile)
    out = []
    for ty in range(nty):
        for tx in range(ntx):
            if (tx + ty) % world != rank:
                continue
            ys, xs = ty * tile + my, tx * tile + mx
            keep = (ys < height) & (xs < width)
            out.append((ys[keep] * width + xs[keep]).astype(np.int64))
    return np.concatenate(out).astype(np.int64) if out else np.zeros(0, np.int64)


def allreduce_grads(buf, group=None):
    d = _dist()
    if d and d.get_world_size(group) > 1:
        d.all_reduce(buf, op=d.ReduceOp.SUM, group=group)
    return buf


def broadcast_model(ctx, src: int = 0, group=None, device=None):
    """Replicate the model (every parameter block: tables, weights, biases) from rank `src`
    to all ranks -- the query path's one collective, at init."""
    import torch
    from .nbvh import PARAM_ALL
    d = _dist()
    if not d or d.get_world_size(group) == 1:
        return
    p = ctx.get_params(PARAM_ALL)
    t = torch.from_numpy(p)
    if device is not None:
        t = t.to(device)
    d.broadcast(t, src=src, group=group)
    ctx.set_params(PARAM_ALL, t.cpu().numpy())


def param_checksum(ctx) -> str:
    """SHA-256 of the fp32 master parameters (host copy)."""
    from .nbvh import PARAM_ALL
    return hashlib.sha256(ctx.get_params(PARAM_ALL).tobytes()).hexdigest()


def params_identical_across_ranks(ctx, group=None) -> bool:
    """True iff every rank holds byte-identical parameters (gathered checksums)."""
    d = _dist()
    mine = param_checksum(ctx)
    if not d or d.get_world_size(group) == 1:
        return True
    allsums = [None] * d.get_world_size(group)
    d.all_gather_object(allsums, mine, group=group)
    return all(s == mine for s in allsums)


def leaf_stats(buf, n_params: int, n_leaves: int):
    """(accepted count, per-leaf [n_leaves, 3] (loss sum, samples, first hits)) from a gradient
    buffer -- read it AFTER allreduce_grads so every rank sees the global statistics and
    builds the same cut."""
    tail = buf[n_params:n_params + 1 + 3 * n_leaves]
    return tail[0], tail[1:].reshape(n_leaves, 3)


def train_step_dp(ctx, rays, u, xi, lod: int = 0, lr: float = 0.01, group=None):
    """One data-parallel step on this rank's shard (rays/u/xi are the local slices)."""
    ctx.train_backward(rays, u, xi, lod)
    allreduce_grads(grad_tensor(ctx), group)
    ctx.apply_update(lr)
