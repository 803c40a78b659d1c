#!/usr/bin/env python
"""N-BVH neural ray-query benchmark (BASELINE.json metric: neural ray queries Mrays/s).

Default workload = BASELINE configs[1] ("1080p"): 988,928-triangle procedural scene,
2,048-leaf cut, hash grid L=16 T=2^19 F=2, n=4 samples, MLP 3x64; one step = one full
1920x1080 frame of primary rays through nbvh_query (traversal + the persistent query kernel).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1080p|tiny] [--impl ours|reference]

Multi-GPU (torchrun): the model is built on rank 0 and broadcast at init; every step's ONE
1080p frame is split over the ranks by interleaved 16x16 pixel tiles; no collective on the
data path; value = the frame's rays / max rank time ("scaling": "strong").  A weak-scaling
line (every rank queries the whole frame) is reported beside it for N > 1.  `--impl reference` times the CPU oracle (oracle/) on a
bounded sample of the same workload (there is no reference implementation to install:
the paper ships no code).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "neural ray queries Mrays/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def stop(self):
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_model(cfg_name: str, device: int, rank: int = 0, list_cap: int = 12, mlp_dtype: int = 0):
    """Synthetic scene + cut + random-init model of the named BASELINE config."""
    from paper_2405_16237_b200 import Context, PARAM_TABLES
    c = synth.CONFIGS[cfg_name]
    h = c["hash"]
    sc = synth.scene_tiny(c["seeds"]["mesh"]) if cfg_name == "tiny" else synth.scene_1080p(c["seeds"]["mesh"])
    ctx = Context(device=device, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers,
                  list_cap=list_cap, mlp_dtype=mlp_dtype)
    ctx.set_mesh(sc)
    ctx.build_cut(c["leaves"])
    n_tab = ctx.param_count(PARAM_TABLES)
    ctx.set_params(PARAM_TABLES, synth.random_params_fp16(n_tab, seed=c["seeds"]["weights"]).astype(np.float32))
    ctx.set_mlp(synth.random_mlp(ctx.d_in, h.hidden_layers, 64, seed=c["seeds"]["weights"] + 1))
    eye = np.asarray(c["eye"], np.float64)
    if rank:
        eye = eye + np.array([0.05 * np.sin(rank), 0.0, 0.05 * np.cos(rank)])
    rays = synth.camera_rays(*c["res"], eye, vfov_deg=c["vfov"])
    return ctx, sc, rays, c


def _profiled_traffic(kernel: str = "k_query"):
    """DRAM bytes per launch of `kernel` from the newest committed ncu --set full summary
    (profiles/r*_ncu_full_query.txt, written by scripts/ncu_summary.py)."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_query.txt")))
    if not files:
        return None, None
    txt = open(files[-1]).read()
    m = re.search(r"== void " + kernel + r"(?:_warp)?<[^\n]*\n(.*?)(?:\n==|\Z)", txt, re.S)
    if not m:
        return None, None
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for key in ("DRAM read", "DRAM write"):
        mm = re.search(key + r"\s+([0-9.]+)\s+(\w+)", m.group(1))
        if not mm:
            return None, None
        tot += float(mm.group(1)) * units.get(mm.group(2), 1)
    return tot, os.path.basename(files[-1])


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_model(ctx, c):
    """The context's model as the oracle takes it (fp16 tables, (W, b) layers)."""
    h = c["hash"]
    from paper_2405_16237_b200 import PARAM_TABLES, PARAM_WEIGHTS, PARAM_BIASES
    tab = ctx.get_params(PARAM_TABLES).astype(np.float16).reshape(-1, h.F)
    W = ctx.get_params(PARAM_WEIGHTS)
    b = ctx.get_params(PARAM_BIASES)
    dims = [ctx.d_in] + [64] * h.hidden_layers + [8]
    layers, wo, bo = [], 0, 0
    for k in range(len(dims) - 1):
        layers.append((W[wo:wo + dims[k] * dims[k + 1]].reshape(dims[k + 1], dims[k]).astype(np.float16),
                       b[bo:bo + dims[k + 1]]))
        wo += dims[k] * dims[k + 1]
        bo += dims[k + 1]
    return tab, layers


def cpu_oracle_rate(ctx, c, rays, target_s: float = 12.0, one_thread_s: float = 4.0):
    """Time the oracle (as it stands) on an evenly spaced sample of the frame's rays
    (np.linspace over the whole frame, so sky and geometry are represented in proportion),
    on all host cores and on one thread."""
    import oracle
    h = c["hash"]
    g = oracle.Grid(h.L, h.log2_T, h.F)
    tab, layers = _oracle_model(ctx, c)
    cut = ctx.cut(0)
    box = oracle.scene_box(ctx.scene)
    N = rays.shape[0]

    def timed(n):
        idx = np.unique(np.linspace(0, N - 1, max(1, min(n, N))).astype(np.int64))
        t0 = time.perf_counter()
        oracle.query(g, h.n_points, tab, layers, cut["leaf_lo"], cut["leaf_hi"], rays[idx], dom_box=box)
        return idx.size, time.perf_counter() - t0

    def rate(budget):
        n, dt = timed(512)                                 # calibrate, then size the sample to the budget
        for _ in range(3):
            if dt >= budget / 3 or n >= N:
                break
            n, dt = timed(int(n * budget / max(dt, 1e-9)))
        return n, dt

    cores = oracle.num_threads()
    n, dt = rate(target_s)
    oracle.set_num_threads(1)
    try:
        n1, dt1 = rate(one_thread_s)
    finally:
        oracle.set_num_threads(cores)
    return {"value": n / dt / 1e6, "unit": "Mrays/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} rays evenly spaced over the {N}-ray frame (np.linspace), C++ double oracle, "
                      f"brute-force leaf scan, OpenMP on {cores} threads", "seconds": dt,
            "one_thread": {"value": n1 / dt1 / 1e6, "unit": "Mrays/s", "rays": n1, "seconds": dt1},
            "cpu_model": _cpu_model(), "host_cpus": os.cpu_count()}


def _workload(cfg: str) -> str:
    return f"{cfg}: " + ("988,928-tri procedural terrain+spheres, 2048-leaf cut, L=16 T=2^19 F=2 n=4, MLP 3x64, "
                         "1920x1080 primary rays" if cfg == "1080p" else
                         "9,680-tri displaced icosphere, 64-leaf cut, L=8 T=2^14 F=2 n=4, MLP 2x64, 64x64 primary rays")


def _time_frames(ctx, rays, out, steps, flush, stream):
    """CUDA-event time (ms) of each of `steps` nbvh_query calls; L2 flushed between calls
    (outside the events)."""
    import torch
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(float(i))                                  # evict L2 between timed steps
        starts[i].record(stream)
        ctx.query(rays, out=out)                               # async: counter reset + 2 kernels
        ends[i].record(stream)
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def _max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2405_16237_b200 import dp
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    ctx, sc, frame_np, c = build_model(args.config, local, 0, args.list_cap, 1 if args.mlp_dtype == "bf16" else 0)
    # the model is built on rank 0 and replicated by one broadcast at init
    t0 = time.perf_counter()
    dp.broadcast_model(ctx, src=0, device="cuda")
    bcast_s = time.perf_counter() - t0
    identical = dp.params_identical_across_ranks(ctx)
    assert identical, "model broadcast left ranks with different parameters"
    # strong scaling: ONE 1080p frame per step, its 16x16 tiles dealt round-robin to the ranks
    if args.order in ("tiles", "tiles_rows"):
        idx = dp.tile_partition(*c["res"], rank, world, inner="morton" if args.order == "tiles" else "rows")
    else:
        idx = np.arange(frame_np.shape[0])[dp.shard(frame_np.shape[0], rank, world)]
    rays_np = np.ascontiguousarray(frame_np[idx])
    n = rays_np.shape[0]
    n_frame = frame_np.shape[0]
    ctx.reserve(max(n, n_frame))
    rays = torch.from_numpy(rays_np).cuda()
    out = ctx.alloc_hits(max(n, n_frame))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2

    ctx.set_profiling(False)
    for _ in range(args.warmup):
        ctx.query(rays, out=out)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    step_ms = _time_frames(ctx, rays, out, args.steps, flush, stream)
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clocks.stop()
    # host cost of one nbvh_query call (enqueue only, no synchronisation)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(5):
        ctx.query(rays, out=out)
    host_ms = (time.perf_counter() - h0) / 5 * 1e3
    torch.cuda.synchronize()
    st = ctx.query_stats()                                     # counters of the last step
    launches = st["n_launches"] * args.steps
    iters = st["n_iters"]
    t_ms = _max_over_ranks(sum(step_ms), world)
    total_rays = n_frame * args.steps                          # every rank's tiles of the frame
    value = total_rays / (t_ms / 1e3) / 1e6
    q_all = torch.tensor([st["n_queries"]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(q_all)
    queries_per_ray = float(q_all.item()) / n_frame

    # weak-scaling line (N > 1 only): every rank queries the whole frame
    weak = None
    if world > 1:
        full = torch.from_numpy(frame_np).cuda()
        for _ in range(args.warmup):
            ctx.query(full, out=out)
        dist.barrier()
        torch.cuda.synchronize()
        wms = _max_over_ranks(sum(_time_frames(ctx, full, out, args.steps, flush, stream)), world)
        dist.barrier()
        weak = {"scaling": "weak", "value": n_frame * args.steps * world / (wms / 1e3) / 1e6, "unit": "Mrays/s",
                "ms_per_step": wms / args.steps, "rays_per_step_per_gpu": n_frame}
        del full

    # live per-kernel timing of the dominant kernel (persistent fused query), one profiled
    # pass per step (separate from the timed region; events on the launching stream)
    ctx.set_profiling(True)
    wave_ms, trav_ms, prof_q = [], [], []
    for i in range(max(3, args.steps)):
        flush.fill_(float(i))
        ctx.query(rays, out=out)
        st2 = ctx.query_stats()
        wave_ms.append(st2["ms_query"])
        trav_ms.append(st2["ms_traverse"])
        prof_q.append(st2["n_queries"])
    ctx.set_profiling(False)
    h = c["hash"]
    useful_gather = h.n_points * h.L * 8 * h.F * 2                # fp16 corner bytes per query (§8(d))
    mean_q = statistics.mean(prof_q)
    wave_s = statistics.mean(wave_ms) / 1e3
    achieved = mean_q * useful_gather / wave_s / 1e9
    hbm, tflops, peak_src = _peaks()
    traffic, traffic_src = _profiled_traffic("k_query")
    mlp_flops = 2 * (ctx.d_in * 64 + (h.hidden_layers - 1) * 64 * 64 + 64 * 8)

    # end-to-end through the public host API: pinned host rays in, host results out
    pin = torch.from_numpy(rays_np).pin_memory()
    hb = {"hit": torch.empty(n, dtype=torch.uint8).pin_memory(), "t": torch.empty(n).pin_memory(),
          "normal": torch.empty(n, 3).pin_memory(), "albedo": torch.empty(n, 3).pin_memory()}
    hbn = {k: v.numpy() for k, v in hb.items()}
    pin_np = pin.numpy()
    ctx.query_host(pin_np, out=hbn)
    torch.cuda.synchronize()
    e2e_s = []
    if world > 1:
        dist.barrier()
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.query_host(pin_np, out=hbn)                       # synchronous: H2D + query + D2H
        e2e_s.append(time.perf_counter() - t0)
    e2e_t = _max_over_ranks(sum(e2e_s), world)
    d2h = n * (1 + 4 + 12 + 12)                                   # hit, t, normal, albedo
    e2e = {"value": n_frame * args.steps / e2e_t / 1e6, "unit": "Mrays/s",
           "h2d_bytes_per_step": n * 32, "d2h_bytes_per_step": d2h,
           "note": "per rank; value = the frame's rays / max-over-ranks time"}

    gather = bench_gather(args)
    # the best random 4-byte gather rate the probe reaches on the load pipe, the texture pipe
    # or both (k_query_warp gathers its hashed levels through the texture pipe)
    l2_peak = max(v for v in (gather.get("l2_random_4B_GBps"), gather.get("l2_random_4B_tex_GBps"),
                              gather.get("l2_random_4B_lsu_tex_GBps")) if v)
    mlp = bench_mlp(ctx, args)
    train = bench_train(ctx, args, world, rank) if args.train else None
    lod = bench_lod(args, local) if (args.lod and rank == 0) else None
    pt = bench_pathtrace(args, local) if (args.pt and rank == 0) else None

    roof = {"bound": "l2_gather", "kernel": "k_query (persistent: sample+encode+MLP+decode+terminate, slot refill)",
            "achieved": achieved, "peak": l2_peak, "unit": "GB/s", "frac": achieved / l2_peak if l2_peak else None,
            "peak_source": "measured live (nbvh_gather_probe / nbvh_gather_probe_tex): random 4-byte gathers "
                           "from a 16 MB L2-resident table counted as 32-byte sectors/s, the best of the load "
                           "pipe, the texture pipe and both together",
            "achieved_definition": "queries x 2,048 useful fp16 corner bytes (n*L*8*F*2, SURVEY §8(d)) / the "
                                   "kernel's CUDA-event time",
            "traffic": traffic,
            "traffic_source": f"profiles/{traffic_src}: dram__bytes_read.sum + dram__bytes_write.sum of one "
                              "launch (tables are L2-resident)" if traffic else None,
            "useful_gather_bytes_per_query": useful_gather, "queries_per_launch_sum": mean_q,
            "kernel_ms_per_step": statistics.mean(wave_ms), "traverse_ms_per_step": statistics.mean(trav_ms),
            "frac_of_hbm_useful": achieved / hbm, "hbm_peak": hbm, "hbm_peak_source": peak_src,
            "mlp_tflops": mean_q * mlp_flops / wave_s / 1e12,
            "mlp_frac_of_bf16_peak": mean_q * mlp_flops / wave_s / 1e12 / tflops}
    prof = _profiled_l2_reads("k_query")
    if prof and l2_peak:
        sec, dur, src = prof
        roof["l2_sector_frac"] = sec * 32 / wave_s / 1e9 / l2_peak
        roof["l2_sector_frac_definition"] = (f"SURVEY §8(d) graded metric: ncu lts__t_sectors_op_read (profiles/{src}: "
                                             f"{sec:.4g} sectors per launch) x 32 B / the live kernel time / peak")

    line = None
    if rank == 0:
        cpu = cpu_oracle_rate(ctx, c, frame_np, target_s=args.cpu_seconds) if args.cpu_seconds > 0 else None
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.mlp_dtype, "data": "synthetic",
            "config": {"workload": _workload(args.config),
                       "rays_per_step": n_frame, "rays_per_step_rank0": n,
                       "model": "random-init tables U[-1,1], He MLP (x10 output)",
                       "l2_flush": "256 MB write between timed steps, outside the per-step CUDA events",
                       "parallelism": f"one frame per step split over {world} rank(s) by interleaved 16x16 tiles "
                                      "(strong); model replicated by broadcast at init",
                       "ray_order": args.order},
            "gpu_launches": launches,
            "queries_per_ray": queries_per_ray, "slot_iterations_per_step": iters,
            "wall_s_timed_region": wall, "host_enqueue_ms_per_query": host_ms, "list_cap": args.list_cap,
            "list_refills_per_step": st["n_refills"],
            "mlp_tiles_per_step": st.get("n_mlp_tiles"), "mlp_rows_per_tile": (st["n_mlp_rows"] / st["n_mlp_tiles"]
                                                                               if st.get("n_mlp_tiles") else None),
            "ws_wait_frac": ([c / st["ws_cycles"][2] for c in st["ws_cycles"][:2]] if st.get("n_mlp_tiles") else None),
            "model_broadcast": {"bytes": 4 * ctx.param_count(3), "seconds": bcast_s, "params_identical": identical},
            "roofline": roof, "weak_scaling": weak,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(), "mlp": mlp, "gather_roofline": gather,
            "train": train, "lod": lod, "pathtrace": pt,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_train(ctx, args, world, rank):
    """BASELINE cfg 5: training-step throughput on the cfg-2 scene and grid.  Global batch
    2^20 rays split over the ranks (strong scaling); per step every rank draws its shard's
    rays and random draws on the device (T0, nbvh_gen_train_rays, C28'), runs
    nbvh_train_backward, all-reduces the flat gradient buffer (NCCL, N>1) and applies Adam.
    Rays: origins uniform in the 50%-inflated box, uniform directions."""
    import torch
    import torch.distributed as dist
    from paper_2405_16237_b200 import dp
    n_global = 1 << 20
    sl = dp.shard(n_global, rank, world)
    cut = ctx.cut(0)
    ctx.set_leaf_rank(np.zeros(cut["n_leaves"], np.float32))
    h = synth.CONFIGS["1080p"]["hash"]
    # T0 on the device (nbvh_gen_train_rays, Philox-4x32-10, key 7, counter = step): every
    # step draws fresh rays, acceptance draws and jitter for this rank's shard of the global
    # batch, inside the timed region.  Origins in the C16 box: the scene's bounding box with
    # every axis extent x1.5 about its centre, the library's default (box=None).
    box = None
    n_local = sl.stop - sl.start
    buf = ctx.gen_train_rays(seed=7, step=0, n=n_local, i0=sl.start, box=box)

    def step(k):
        ctx.gen_train_rays(seed=7, step=k, n=n_local, i0=sl.start, box=box, out=buf)
        dp.train_step_dp(ctx, *buf)

    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms = float(tm.item())
    st = ctx.train_stats()
    acc = torch.tensor([st["n_accepted"], st["n_first_hit"]], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(acc)
    n_acc_global, n_first_global = (float(v) for v in acc.cpu().numpy())
    ctx.set_profiling(True)
    step(0)
    torch.cuda.synchronize()
    ph = ctx.train_stats()["ms_phase"]
    ctx.set_profiling(False)
    _, n_grad = ctx.grad_buffer()
    h = ctx.cfg
    # T7 in algorithmic units: one gradient term per (sample, point, level, corner); the
    # scatter groups them into far fewer reductions (warp aggregation, 16-byte reductions)
    terms = st["n_accepted"] * h.n_points * h.L * 8
    term_rate = terms / (ph["bwd"] / 1e3) / 1e9 if ph.get("bwd") else None
    return {"metric": "training rays/s (BASELINE cfg 5)", "value": n_global / (ms / 1e3) / 1e6, "unit": "Mrays/s",
            "accepted_samples_per_s": n_acc_global / (ms / 1e3) / 1e6, "accepted_unit": "M samples/s",
            "ray_box": "C16: scene bounding box, every axis extent x1.5 about its centre (P:142)",
            "global_batch": n_global, "scaling": "strong", "ms_per_step": ms,
            "accepted_per_step": n_acc_global, "first_hit_per_step": n_first_global,
            "accepted_per_step_rank0": st["n_accepted"], "first_hit_per_step_rank0": st["n_first_hit"],
            "phase_ms_rank0": ph, "allreduce_bytes": 4 * n_grad if world > 1 else 0,
            "gpu_launches_per_step": st["n_launches"] + 1,          # + the T0 generator
            "bwd_T7_terms_per_step": terms, "bwd_T7_Gterms_per_s": term_rate,
            "bwd_bound": "L1 data-pipe wavefronts of the scatter (82% of peak; 63.6 M reduction sectors per "
                         "step after warp aggregation), profiles/NOTES.md r2d"}


def bench_lod(args, device):
    """BASELINE cfg 4: multi-cut LoD query.  Three error-driven cuts of the cfg-2 scene
    (~128, ~512 and 2048 leaves, registered during one construction run) share
    one hash grid; 1080p frames from three camera distances (1.6, 6.4, 25.6) are queried at
    the fine, middle and coarse LoD.  Also reports the far frame at the finest cut, i.e. the
    speed-up an LoD switch buys (P:342 reports 1.5-2x after the primary hit)."""
    import torch
    from paper_2405_16237_b200 import Context
    from paper_2405_16237_b200.construct import construct, Schedule
    c = synth.CONFIGS["1080p"]
    h = c["hash"]
    sc = synth.scene_1080p(c["seeds"]["mesh"])
    ctx = Context(device=device, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points, hidden_layers=h.hidden_layers,
                  list_cap=args.list_cap, seed=11)
    ctx.set_mesh(sc)
    ctx.build_cut(1)
    n_train = 1 << 16
    ctx.reserve(max(n_train, c["res"][0] * c["res"][1]))

    def batch(step):
        rays = synth.random_rays(n_train, seed=9000 + step % 8)
        u = synth.random_uniform(n_train, seed=9100 + step % 8)
        xi = synth.random_uniform(n_train * h.n_points, seed=9200 + step % 8).reshape(n_train, h.n_points)
        return tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (rays, u, xi))

    batches = [batch(i) for i in range(8)]
    t0 = time.perf_counter()
    hist = construct(ctx, 2048, lambda s: batches[s % 8],
                     Schedule(iters0=2, splits0=8, growth=2.0, final_iters=100, lod_at_leaves=(128, 512)),
                     distributed=False)                          # rank 0 alone runs this section
    build_s = time.perf_counter() - t0
    slots = {"fine": 0, "middle": 2, "coarse": 1}
    out = ctx.alloc_hits(c["res"][0] * c["res"][1])
    res = {}
    stream = torch.cuda.current_stream()
    for name, dist, lod in (("near", 1.6, 0), ("mid", 6.4, 2), ("far", 25.6, 1), ("far@fine", 25.6, 0)):
        # same view direction; the field of view narrows with distance so the scene covers
        # the same part of the frame (a zoomed camera: same screen-space work, coarser LoD)
        eye = np.array([0.0, 0.6, 1.6]) * (dist / 1.6)
        vfov = float(np.degrees(2.0 * np.arctan(np.tan(np.radians(c["vfov"]) / 2.0) * 1.6 / dist)))
        rays = torch.from_numpy(synth.camera_rays(*c["res"], eye, vfov_deg=vfov)).cuda()
        for _ in range(3):
            ctx.query(rays, lod=lod, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ctx.query(rays, lod=lod, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        st = ctx.query_stats()
        res[name] = {"lod_slot": lod, "leaves": ctx.cut(lod)["n_leaves"], "camera_distance": dist,
                     "ms_per_frame": ms, "Mrays_per_s": rays.shape[0] / ms / 1e3,
                     "queries_per_ray": st["n_queries"] / rays.shape[0]}
    return {"metric": "multi-cut LoD query Mrays/s (BASELINE cfg 4)", "unit": "Mrays/s",
            "construction": {"rounds": len(hist), "seconds": build_s, "rays_per_step": n_train,
                             "leaves_per_round": [hlog.n_leaves for hlog in hist],
                             "final_mean_loss": hist[-1].loss},
            "frames": res,
            "lod_speedup_far": res["far"]["Mrays_per_s"] / res["far@fine"]["Mrays_per_s"]}


def bench_pathtrace(args, device):
    """BASELINE cfg 3: hybrid path tracing at 1080p, 4 bounces, 1 sample per pixel, through a
    TLAS (PAPER §7): the cfg-2 terrain as a classical BLAS (524,288 triangles, base-BVH
    traversal) and the 48 icospheres as a neural BLAS (464,640 triangles, an error-driven
    1,024-leaf N-BVH trained for a short schedule, with a 256-leaf LoD registered on the way),
    instanced twice (identity, and a rotated, scaled copy lifted above the terrain).  Every
    bounce runs on the compacted alive paths; the neural BLAS switches to the coarse LoD after
    the primary hit -- reported with and without the switch."""
    import torch
    from paper_2405_16237_b200 import Context
    from paper_2405_16237_b200.construct import construct, Schedule
    from paper_2405_16237_b200.pathtrace import PathTracer
    c = synth.CONFIGS["1080p"]
    h = c["hash"]
    terrain, spheres = synth.scene_1080p_parts(c["seeds"]["mesh"])
    neural = Context(device=device, L=h.L, F=h.F, log2_T=h.log2_T, n_points=h.n_points,
                     hidden_layers=h.hidden_layers, list_cap=args.list_cap, seed=21)
    neural.set_mesh(spheres)
    classical = Context(device=device, L=8, F=2, log2_T=14, n_points=4, hidden_layers=1)
    classical.set_mesh(terrain)
    n_train = 1 << 16
    n_px = c["res"][0] * c["res"][1]
    neural.build_cut(1)
    neural.reserve(max(n_train, n_px))
    batches = []
    for b in range(8):
        r = synth.random_rays(n_train, seed=9500 + b)
        u = synth.random_uniform(n_train, seed=9600 + b)
        xi = synth.random_uniform(n_train * h.n_points, seed=9700 + b).reshape(n_train, h.n_points)
        batches.append(tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (r, u, xi)))
    t0 = time.perf_counter()
    construct(neural, 1024, lambda s: batches[s % 8],
              Schedule(iters0=2, splits0=8, growth=2.0, final_iters=300, lod_at_leaves=(256,)),
              distributed=False)                                 # rank 0 alone runs this section
    build_s = time.perf_counter() - t0
    ang = 0.5
    rot = np.array([[np.cos(ang), 0.0, np.sin(ang)], [0.0, 1.0, 0.0], [-np.sin(ang), 0.0, np.cos(ang)]])
    inst = [(0, np.concatenate([np.eye(3), np.zeros((3, 1))], 1)),
            (0, np.concatenate([0.8 * rot, np.array([[0.0], [0.35], [-0.3]])], 1)),
            (1, np.concatenate([np.eye(3), np.zeros((3, 1))], 1))]
    rays = torch.from_numpy(synth.camera_rays(*c["res"], c["eye"], vfov_deg=c["vfov"])).cuda()
    stream = torch.cuda.current_stream()
    res = {}
    for name, lod2 in (("lod_switch", 1), ("fine_only", 0)):
        pt = PathTracer([(neural, "neural"), (classical, "mesh")], inst, n_px, lod_secondary=lod2)
        for i in range(3):
            pt.render(rays, bounces=4, seed=i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        traced = 0
        e0.record(stream)
        for i in range(args.steps):
            _, alive = pt.render(rays, bounces=4, seed=100 + i)
            traced += sum(alive)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        res[name] = {"ms_per_frame": ms, "Mrays_per_s": traced / args.steps / ms / 1e3,
                     "paths_entering_bounce": alive, "lod_after_primary_hit": lod2}
    return {"metric": "hybrid path tracing (BASELINE cfg 3)", "unit": "Mrays/s",
            "value": res["lod_switch"]["Mrays_per_s"], "ms_per_frame": res["lod_switch"]["ms_per_frame"],
            "resolution": list(c["res"]), "spp": 1, "bounces": 4, "instances": len(inst),
            "tlas": "BVH over 3 instance boxes (2 instances of the neural BLAS, 1 of the classical BLAS)",
            "variants": res, "lod_switch_speedup": res["fine_only"]["ms_per_frame"] / res["lod_switch"]["ms_per_frame"],
            "neural_blas": {"tris": spheres.n_tris, "leaves": neural.cut(0)["n_leaves"],
                            "lod1_leaves": neural.cut(1)["n_leaves"], "train_s": build_s},
            "classical_blas": {"tris": terrain.n_tris}}


def bench_mlp(ctx, args):
    """The decoder MLP alone on tcgen05 (nbvh_mlp_forward): one frame's worth of queries
    (2,377,813 rows of D_in = 128 fp16 features -> 8 outputs) streamed from HBM; tensor-pipe
    throughput against the measured dense bf16 peak (fp16 runs at the same rate)."""
    import torch
    m = 2377813
    g = torch.Generator(device="cuda").manual_seed(17)
    x = (torch.rand(m, ctx.d_in, device="cuda", generator=g) * 0.8 - 0.4).half()
    z = torch.empty(m, 8, device="cuda")
    for _ in range(3):
        ctx.mlp_forward(x, z)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ctx.mlp_forward(x, z)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    h = ctx.cfg.hidden_layers
    flop_mma = 2 * 128 * (ctx.d_in * 64 + (h - 1) * 64 * 64 + 64 * 16) * ((m + 127) // 128)   # issued MMA work
    flop_alg = 2 * m * (ctx.d_in * 64 + (h - 1) * 64 * 64 + 64 * 8)                             # 8 real outputs
    hbm, tflops, src = _peaks()
    bytes_io = m * (ctx.d_in * 2 + 32)
    return {"kernel": "k_mlp_tc (tcgen05 + TMEM + TMA)", "rows": m, "ms": ms,
            "tflops_algorithmic": flop_alg / ms / 1e9, "tflops_issued": flop_mma / ms / 1e9,
            "frac_of_bf16_peak": flop_mma / ms / 1e9 / tflops, "peak_tflops": tflops, "peak_source": src,
            "io_GBps": bytes_io / ms / 1e6, "io_frac_of_hbm": bytes_io / ms / 1e6 / hbm}


def _profiled_l2_reads(kernel: str = "k_query"):
    """(L2 read sectors from L1/TEX, duration s) of `kernel` from the newest committed ncu
    summary (profiles/r*_ncu_full_query.txt)."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_query.txt")))
    if not files:
        return None
    txt = open(files[-1]).read()
    m = re.search(r"== void " + kernel + r"(?:_warp)?<[^\n]*\n(.*?)(?:\n==|\Z)", txt, re.S)
    if not m:
        return None
    sec = re.search(r"L2 read sectors from L1/TEX\s+([0-9.]+)", m.group(1))
    dur = re.search(r"duration\s+([0-9.]+)\s+(\w+)", m.group(1))
    if not sec or not dur:
        return None
    scale = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9}.get(dur.group(2), 1e-3)
    return float(sec.group(1)), float(dur.group(1)) * scale, os.path.basename(files[-1])


def bench_gather(args):
    """SURVEY §8(d) encode roofline: the measured random-sector read peak of an L2-resident
    table (nbvh_gather_probe: 4-byte gathers = hashed levels, 32-byte = dense corner records)
    and of an HBM-resident one, and the query kernel's L2 read-sector rate (its committed ncu
    profile) as a fraction of the L2 peak."""
    import torch
    from paper_2405_16237_b200.nbvh import gather_probe
    sink = torch.empty(148 * 8 * 256 * 2, dtype=torch.int32, device="cuda")
    out = {}
    cases = (("l2_random_4B", 16 << 20, 4, 1 << 28), ("l2_random_32B", 16 << 20, 32, 1 << 27),
             ("hbm_random_4B", 1 << 30, 4, 1 << 27))
    stream = torch.cuda.current_stream()
    for name, nbytes, eb, n in cases:
        tab = torch.randint(0, 1 << 30, (nbytes // 4,), dtype=torch.int32, device="cuda")
        gather_probe(tab, eb, n, sink)                                   # warm (L2 fill)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = 0
        for i in range(3):
            done += gather_probe(tab, eb, n, sink, seed=i + 2)
        e1.record(stream)
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        out[name + "_Gsectors_per_s"] = done / s / 1e9                  # one 32-byte sector per gather
        out[name + "_GBps"] = done * 32 / s / 1e9
        del tab
    # the same 4-byte gathers through the texture pipe (k_query_warp's hashed levels), and with
    # half of them on each pipe: the peak of a kernel that uses both L1 input pipes
    from paper_2405_16237_b200.nbvh import gather_probe_tex
    tab = torch.randint(0, 1 << 30, ((16 << 20) // 4,), dtype=torch.int32, device="cuda")
    for name, mixed in (("l2_random_4B_tex", False), ("l2_random_4B_lsu_tex", True)):
        gather_probe_tex(tab, 1 << 26, sink, mixed=mixed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = gather_probe_tex(tab, 1 << 28, sink, mixed=mixed, seed=7)
        e1.record(stream)
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        out[name + "_Gsectors_per_s"] = done / s / 1e9
        out[name + "_GBps"] = done * 32 / s / 1e9
    del tab
    from paper_2405_16237_b200.nbvh import atomic_probe
    for vec in (1, 2, 4):                                                # T7 scatter roofline
        tab = torch.zeros((32 << 20) // 4, dtype=torch.float32, device="cuda")   # ~ the cfg-2 gradient buffer
        atomic_probe(tab, vec, 1 << 26)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        done = sum(atomic_probe(tab, vec, 1 << 27, seed=i + 2) for i in range(2))
        e1.record(stream)
        torch.cuda.synchronize()
        out[f"l2_red_{'' if vec == 1 else f'v{vec}_'}f32_Gops"] = done / (e0.elapsed_time(e1) / 1e3) / 1e9
        del tab
    prof = _profiled_l2_reads("k_query")
    if prof:
        sec, dur, src = prof
        out["k_query_l2_read_GBps"] = sec * 32 / dur / 1e9
        out["k_query_frac_of_l2_random_peak"] = out["k_query_l2_read_GBps"] / out["l2_random_4B_GBps"]
        out["k_query_profile"] = src
    return out


def run_reference(args):
    """The CPU oracle timed as it stands on bounded samples of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_2405_16237_b200 import Context  # host-only context: scene/cut/params, no GPU
    ctx, sc, rays, c = build_model(args.config, -1)
    per_step = max(256, rays.shape[0] // 256) if args.config == "1080p" else rays.shape[0]
    stride = max(1, rays.shape[0] // per_step)
    h = c["hash"]
    g = oracle.Grid(h.L, h.log2_T, h.F)
    tab, layers = _oracle_model(ctx, c)
    cut = ctx.cut(0)
    box = oracle.scene_box(sc)

    def step(i):
        sample = rays[(i % stride)::stride][:per_step]
        oracle.query(g, h.n_points, tab, layers, cut["leaf_lo"], cut["leaf_hi"], sample, dom_box=box)
        return sample.shape[0]

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    done = sum(step(args.warmup + i) for i in range(args.steps))
    dt = time.perf_counter() - t0
    v = done / dt / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "Mrays/s", "n_gpus": args.gpus,
            "device": "cpu (the oracle runs on the host cores; no GPU is used)", "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload(args.config), "rays_per_step": per_step},
            "cpu_baseline": {"value": v, "unit": "Mrays/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"{per_step} rays per step (every {stride}th primary ray, offset by step)",
                             "cpu_model": _cpu_model(), "host_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="1080p", choices=["1080p", "tiny"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle timing budget (0 = skip)")
    ap.add_argument("--list-cap", type=int, default=12, help="per-ray ordered leaf-list capacity K (C6)")
    ap.add_argument("--train", type=int, default=1, help="also time the cfg-5 training step (1/0)")
    ap.add_argument("--lod", type=int, default=1, help="also run the cfg-4 multi-cut LoD query (1/0)")
    ap.add_argument("--pt", type=int, default=1, help="also run the cfg-3 hybrid path tracer (1/0)")
    ap.add_argument("--mlp-dtype", default="f16", choices=["f16", "bf16"],
                    help="query-path MLP operands (nbvh_config.mlp_dtype, C39)")
    ap.add_argument("--order", default="tiles", choices=["tiles", "tiles_rows", "rows"],
                    help="ray order / rank partition: 16x16 tiles dealt round-robin, Z order inside a tile "
                         "(default) or row-major inside (tiles_rows); or row-major shards (rows)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
