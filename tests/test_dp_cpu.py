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
