"""Print the chunk timeline of nbvh_query_host (NBVH_HOST_TIMELINE=1) for the 1080p frame,
plus the e2e time of a few calls."""
import os, sys, time
os.environ["NBVH_HOST_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
ctx, sc, rays_np, c = bench.build_model("1080p", 0, 0, 12)
n = rays_np.shape[0]
ctx.reserve(n)
pin = torch.from_numpy(rays_np).pin_memory()
hb = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory(), "t": torch.empty(n).pin_memory(),
      "normal": torch.empty(n, 3).pin_memory(), "albedo": torch.empty(n, 3).pin_memory()}
hbn = {k: v.numpy() for k, v in hb.items()}
for i in range(4):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    ctx.query_host(pin.numpy(), out=hbn)
    print(f"wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
