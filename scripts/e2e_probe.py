"""Diagnose the end-to-end (host buffers) query pipeline: nbvh_query_host vs a torch-stream
re-implementation of the same chunked upload / query / download schedule."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
ctx, sc, rays_np, c = bench.build_model("1080p", 0, 0, 12)
n = rays_np.shape[0]
ctx.reserve(n)
pin = torch.from_numpy(rays_np).pin_memory()
hb = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory(), "t": torch.empty(n).pin_memory(),
      "normal": torch.empty(n, 3).pin_memory(), "albedo": torch.empty(n, 3).pin_memory()}
hbn = {k: v.numpy() for k, v in hb.items()}
for _ in range(3):
    ctx.query_host(pin.numpy(), out=hbn)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ctx.query_host(pin.numpy(), out=hbn)
t_c = (time.perf_counter() - t0) / 10
# torch re-implementation
d_rays = torch.empty(n, 8, device="cuda")
dout = ctx.alloc_hits(n)
sH, sD = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()
def pipeline(chunks):
    step = (n + chunks - 1) // chunks
    evs_h, evs_q = [], []
    for k in range(chunks):
        o, m = k * step, min(step, n - k * step)
        with torch.cuda.stream(sH):
            d_rays[o:o + m].copy_(pin[o:o + m], non_blocking=True)
            e = torch.cuda.Event(); e.record(sH); evs_h.append(e)
    for k in range(chunks):
        o, m = k * step, min(step, n - k * step)
        main.wait_event(evs_h[k])
        sub = {kk: v[o:o + m] for kk, v in dout.items()}
        ctx.query(d_rays[o:o + m], out=sub)
        e = torch.cuda.Event(); e.record(main)
        sD.wait_event(e)
        with torch.cuda.stream(sD):
            for kk in hb:
                hb[kk][o:o + m].copy_(dout[kk][o:o + m], non_blocking=True)
    torch.cuda.synchronize()
for ch in (1, 4, 8, 16):
    pipeline(ch)
    t0 = time.perf_counter()
    for _ in range(10):
        pipeline(ch)
    print(f"torch pipeline chunks={ch}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
# pieces
def tm(fn, reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
print(f"nbvh_query_host: {t_c * 1e3:.3f} ms")
print(f"H2D rays only: {tm(lambda: d_rays.copy_(pin, non_blocking=True)):.3f} ms")
print(f"query only: {tm(lambda: ctx.query(d_rays, out=dout)):.3f} ms")
print(f"D2H hits only: {tm(lambda: [hb[k].copy_(dout[k], non_blocking=True) for k in hb]):.3f} ms")
# overlap capability: a full-frame query while unrelated H2D / D2H copies run on other streams
d_rays2 = torch.empty_like(d_rays)
dout2 = ctx.alloc_hits(n)
def concurrent():
    with torch.cuda.stream(sH):
        d_rays2.copy_(pin, non_blocking=True)
    with torch.cuda.stream(sD):
        for k in hb:
            hb[k].copy_(dout2[k], non_blocking=True)
    ctx.query(d_rays, out=dout)
print(f"query || H2D || D2H (independent): {tm(concurrent):.3f} ms")
def copies_only():
    with torch.cuda.stream(sH):
        d_rays2.copy_(pin, non_blocking=True)
    with torch.cuda.stream(sD):
        for k in hb:
            hb[k].copy_(dout2[k], non_blocking=True)
print(f"H2D || D2H: {tm(copies_only):.3f} ms")
def q_h2d():
    with torch.cuda.stream(sH):
        d_rays2.copy_(pin, non_blocking=True)
    ctx.query(d_rays, out=dout)
print(f"query || H2D: {tm(q_h2d):.3f} ms")
# per-call fixed cost: query time vs ray count
for frac in (1, 2, 4, 8):
    m = n // frac
    sub = {k: v[:m] for k, v in dout.items()}
    print(f"query of n/{frac} ({m} rays): {tm(lambda: ctx.query(d_rays[:m], out=sub)):.3f} ms")
