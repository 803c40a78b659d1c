"""Cost of chunking the device-resident query: the 1080p frame as 1 launch vs k contiguous
or block-interleaved chunks, on one stream and alternating two streams."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
ctx, sc, rays_np, c = bench.build_model("1080p", 0, 0, 12)
n = rays_np.shape[0]
ctx.reserve(n)
rays = torch.from_numpy(rays_np).cuda()
out = ctx.alloc_hits(n)
main = torch.cuda.current_stream()
s2 = torch.cuda.Stream()
# block-interleaved permutation (blocks of 1024, weights 1,2,3,3,2,1 like nbvh_query_host)
W = [1, 2, 3, 3, 2, 1]
B = 1024
per = n // (B * sum(W))
idx = []
first = 0
for w in W:
    ch = []
    for r in range(per):
        s0 = (r * sum(W) + first) * B
        ch.append(torch.arange(s0, s0 + w * B))
    first += w
    idx.append(torch.cat(ch))
idx[-1] = torch.cat([idx[-1], torch.arange(per * sum(W) * B, n)])
perm = torch.cat(idx).cuda()
rays_i = rays[perm].contiguous()
sizes = [len(i) for i in idx]

def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(reps):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

print("1 launch", timed(lambda: ctx.query(rays, out=out)))
def chunks(src, two):
    o = 0
    for k, m in enumerate(sizes):
        sub = {kk: v[o:o + m] for kk, v in out.items()}
        if two and k % 2:
            s2.wait_stream(main)
            with torch.cuda.stream(s2):
                ctx.query(src[o:o + m], out=sub, stream=s2)
        else:
            ctx.query(src[o:o + m], out=sub)
        o += m
    main.wait_stream(s2)
print("6 interleaved chunks, one stream", timed(lambda: chunks(rays_i, False)))
print("6 contiguous chunks, one stream", timed(lambda: chunks(rays, False)))
