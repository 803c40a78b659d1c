"""Data-parallel training step (BASELINE cfg 5): one process per GPU, the global batch
split over ranks, one all-reduce (sum) of the flat fp32 gradient buffer per step.

The buffer (nbvh_grad_buffer) holds the parameter gradients of the SUM of per-sample
losses, then the accepted-sample count, then per-leaf (loss sum, samples, first hits);
summing it over ranks gives exactly the single-process buffer of the whole batch, and
nbvh_apply_update divides by the summed count, so every rank applies the same Adam
step to identical parameters.
"""
from __future__ import annotations


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


def shard(n_global: int, rank: int, world: int) -> slice:
    """Contiguous, balanced split of a global batch of n_global rays."""
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return slice(start, start + base + (1 if rank < rem else 0))


def allreduce_grads(buf, group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def train_step_dp(ctx, rays, u, xi, lod: int = 0, lr: float = 0.01, group=None):
    """One data-parallel step on this rank's shard (rays/u/xi are the local slices)."""
    ctx.train_backward(rays, u, xi, lod)
    allreduce_grads(grad_tensor(ctx), group)
    ctx.apply_update(lr)
