"""Run the tiny query / host path / training step / tcgen05 MLP with the library named by
NBVH_LIB (the debug-checks build): any failed device-side bounds check aborts with an error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import synth
from paper_2405_16237_b200 import Context, PARAM_TABLES, LIB_PATH

assert LIB_PATH == os.environ["NBVH_LIB"], LIB_PATH
h = synth.CONFIGS["tiny"]["hash"]
ctx = Context(device=0, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers, list_cap=3)
sc = synth.scene_tiny()
ctx.set_mesh(sc)
ctx.build_cut(64)
ctx.set_params(PARAM_TABLES, synth.random_params_fp16(ctx.param_count(PARAM_TABLES), seed=7).astype(np.float32))
ctx.set_mlp(synth.random_mlp(ctx.d_in, h.hidden_layers, 64, seed=2))
rays = np.concatenate([synth.camera_rays(64, 64, (0.0, 0.0, 3.5), vfov_deg=40.0), synth.random_rays(3000, seed=11)])
ctx.reserve(20000)
d = ctx.query(torch.from_numpy(rays).cuda())
hh = ctx.query_host(rays)
torch.cuda.synchronize()
assert np.array_equal(d["hit"].cpu().numpy(), hh["hit"])
ctx.set_leaf_rank(np.zeros(ctx.cut(0)["n_leaves"], np.float32))
for step in range(3):
    r, u, xi = ctx.gen_train_rays(seed=5, step=step, n=8192, box=(-1.5, -1.5, -1.5, 1.5, 1.5, 1.5))
    ctx.train_step(r, u, xi)
# the other T7 kernel (privatised fixed-point levels) and the warp-specialised query kernel
os.environ["NBVH_SCATTER_AGG"] = "0"
ctx.train_step(*ctx.gen_train_rays(seed=5, step=3, n=8192, box=(-1.5, -1.5, -1.5, 1.5, 1.5, 1.5)))
del os.environ["NBVH_SCATTER_AGG"]
os.environ["NBVH_QUERY_MLP"] = "tc"
dw = ctx.query(torch.from_numpy(rays).cuda())
del os.environ["NBVH_QUERY_MLP"]
torch.cuda.synchronize()
assert dw["hit"].numel() == rays.shape[0]
# classical closest-hit traversal (bvh_closest: farther-child stack sized by the BVH depth)
mh = ctx.intersect_mesh(torch.from_numpy(rays).cuda())
x = (torch.rand(1000, ctx.d_in, device="cuda") - 0.5).half()
ctx.mlp_forward(x)
torch.cuda.synchronize()
st = ctx.query_stats()
print("debug checks ok", int(d["hit"].sum().item()), st["n_refills"], ctx.train_stats()["n_accepted"],
      int(mh["hit"].sum().item()))
