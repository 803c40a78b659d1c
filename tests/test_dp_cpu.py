"""World-size-2 gloo test (CPU) of the data-parallel decomposition used by
paper_2405_16237_b200.dp: each rank produces the SUM-of-losses gradient of its shard plus
the accepted count in the buffer tail; one all-reduce (sum) then division by the summed
count must equal the full-batch mean gradient.  Gradients come from the oracle here
(injected by the test; the product never imports it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as orc
    import synth
    from paper_2405_16237_b200 import dp
    from tests.test_oracle_pins import _small_train_setup
    sc, off, lt, llo, lhi, g, tab, layers, rays, u, xi = _small_train_setup(orc, n_rays=400, seed=50)
    sl = dp.shard(rays.shape[0], rank, world)
    o = orc.train_grad(g, 3, tab, layers, llo, lhi, np.zeros(2, np.float32), off, lt, sc, rays[sl], u[sl], xi[sl])
    m = o["n_acc"]
    buf = torch.from_numpy(np.concatenate([o["g_table"] * m, o["g_W"] * m, o["g_b"] * m, [m]]))
    dp.allreduce_grads(buf)
    mean = (buf[:-1] / buf[-1]).numpy()
    full = orc.train_grad(g, 3, tab, layers, llo, lhi, np.zeros(2, np.float32), off, lt, sc, rays, u, xi)
    want = np.concatenate([full["g_table"], full["g_W"], full["g_b"]])
    out_q.put((rank, float(np.abs(mean - want).max()), float(np.abs(want).max()), int(buf[-1])))
    dist.destroy_process_group()


def test_dp_allreduce_equals_full_batch():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, scale, count in res:
        assert err <= 1e-12 * max(1.0, scale), (rank, err)
        assert count > 20


def test_shard_is_a_partition():
    from paper_2405_16237_b200 import dp
    for n in (1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            idx = np.concatenate([np.arange(n)[dp.shard(n, r, world)] for r in range(world)])
            assert np.array_equal(idx, np.arange(n))


# ------------------------------------------------------------------ query partition
@pytest.mark.parametrize("w,h,world", [(1920, 1080, 1), (1920, 1080, 2), (1920, 1080, 8), (64, 64, 3), (37, 21, 4)])
def test_tile_partition_covers_frame_once_and_balances(w, h, world):
    from paper_2405_16237_b200 import dp
    parts = [dp.tile_partition(w, h, r, world) for r in range(world)]
    allidx = np.concatenate(parts)
    assert allidx.size == w * h and np.array_equal(np.sort(allidx), np.arange(w * h))
    sizes = np.array([p.size for p in parts])
    assert sizes.max() - sizes.min() <= 2 * 16 * 16 * max(1, (h + 15) // 16 // 8)   # within a few tiles
    if w * h >= 1920 * 1080 and world > 1:
        # every rank owns tiles in every 1/8th band of rows (interleaved, not contiguous)
        for p in parts:
            bands = np.unique((p // w) * 8 // h)
            assert bands.size == 8
    # tile-major, Z order inside a tile: the first 16 pixels of a rank form a 4x4 block
    p0 = parts[0]
    if w >= 16 and h >= 16:
        ys, xs = np.divmod(p0[:16], w)
        assert ys.max() - ys.min() == 3 and xs.max() - xs.min() == 3
    rows = dp.tile_partition(w, h, 0, world, inner="rows")
    assert np.array_equal(np.sort(rows), np.sort(p0))
    if w >= 16:
        assert np.all(np.diff(rows[:16]) == 1)


def _bcast_worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2405_16237_b200 import Context, dp, PARAM_ALL
    ctx = Context(device=-1, L=8, F=2, log2_T=14, n_points=4, hidden_layers=2)
    n = ctx.param_count(PARAM_ALL)
    ctx.set_params(PARAM_ALL, np.random.default_rng(100 + rank).standard_normal(n).astype(np.float32))
    before = dp.params_identical_across_ranks(ctx)
    dp.broadcast_model(ctx, src=0)
    after = dp.params_identical_across_ranks(ctx)
    want = np.random.default_rng(100).standard_normal(n).astype(np.float32)
    same_as_rank0 = bool(np.array_equal(ctx.get_params(PARAM_ALL), want))
    # per-leaf statistics read after the reduce (construct()): every rank sees the
    # same global tail of a product-shaped buffer (params | count | n_leaves x 3)
    import torch
    n_leaves = 64
    rng = np.random.default_rng(7 + rank)
    buf = torch.from_numpy(np.concatenate([rng.standard_normal(n), [rng.integers(10, 50)],
                                           rng.integers(0, 9, 3 * n_leaves)]).astype(np.float32))
    local_count = float(buf[n])
    dp.allreduce_grads(buf)
    count, per_leaf = dp.leaf_stats(buf, n, n_leaves)
    digest = __import__("hashlib").sha256(buf.numpy().tobytes()).hexdigest()
    out_q.put((rank, before, after, same_as_rank0, float(count), local_count, per_leaf.shape, digest))
    dist.destroy_process_group()


def test_model_broadcast_and_reduced_stats_identical_across_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, before, after, same0, count, local, shape, digest in res:
        assert not before and after and same0
        assert shape == (64, 3)
    assert res[0][4] == res[0][5] + res[1][5] == res[1][4]          # global accepted count on both
    assert res[0][7] == res[1][7]                                    # byte-identical reduced buffers
