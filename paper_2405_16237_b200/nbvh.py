"""Thin ctypes binding of libnbvh.so (include/nbvh.h).  Argument marshalling only:
every step of the query and training path runs in the library's CUDA kernels.

Device buffers are torch tensors (PyTorch supplies device memory, streams and process
groups); host buffers are numpy arrays.  There is no fallback: if libnbvh.so is missing
or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NBVH_LIB") or os.path.join(_HERE, "libnbvh.so")   # NBVH_LIB: e.g. the debug-checks build

STATUS = {0: "OK", 1: "WARN_CLAMPED", -1: "EINVAL", -2: "ERANGE", -3: "ESTATE", -4: "ENONFINITE", -5: "ECUDA",
          -6: "ENOMEM"}
PARAM_TABLES, PARAM_WEIGHTS, PARAM_BIASES, PARAM_ALL = 0, 1, 2, 3


class NbvhError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"nbvh {STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("L", C.c_int32), ("F", C.c_int32), ("log2_T", C.c_int32), ("base_res", C.c_int32),
                ("max_res", C.c_int32), ("n_points", C.c_int32), ("hidden_layers", C.c_int32),
                ("width", C.c_int32), ("list_cap", C.c_int32), ("mode", C.c_int32), ("inflate_rel", C.c_float),
                ("inflate_abs", C.c_float), ("seed", C.c_uint64), ("mlp_dtype", C.c_int32), ("reserved0", C.c_int32)]


class Hits(C.Structure):
    _fields_ = [("hit", C.c_void_p), ("t", C.c_void_p), ("normal", C.c_void_p), ("albedo", C.c_void_p),
                ("leaf", C.c_void_p), ("n_queries", C.c_void_p)]


class Instance(C.Structure):
    """nbvh_instance: world_to_object row-major 3x4, world box, BLAS number."""
    _fields_ = [("world_to_object", C.c_float * 12), ("lo", C.c_float * 3), ("hi", C.c_float * 3),
                ("blas", C.c_int32), ("pad", C.c_int32)]


MAX_BLAS = 8


class QueryStats(C.Structure):
    _fields_ = [("n_rays", C.c_int64), ("n_queries", C.c_int64), ("n_iters", C.c_int32),
                ("n_launches", C.c_int32), ("n_refills", C.c_int32), ("ms_traverse", C.c_float),
                ("ms_query", C.c_float), ("n_mlp_tiles", C.c_int32), ("n_mlp_rows", C.c_int32),
                ("ws_cycles", C.c_int64 * 3)]


class TrainStats(C.Structure):
    _fields_ = [("n_rays", C.c_int64), ("n_first_hit", C.c_int64), ("n_accepted", C.c_int64),
                ("loss_sum", C.c_double), ("loss_terms", C.c_double * 4), ("n_launches", C.c_int32),
                ("skipped", C.c_int32), ("ms_phase", C.c_float * 6)]


_lib = None

# (name, argtypes) — every entry point declared in include/nbvh.h
_P, _I32, _I64, _F = C.c_void_p, C.c_int32, C.c_int64, C.c_float
SIGNATURES = {
    "nbvh_config_default": (None, [_P]),
    "nbvh_create": (C.c_int, [_P, C.c_int, _P]),
    "nbvh_destroy": (None, [_P]),
    "nbvh_last_error": (C.c_char_p, [_P]),
    "nbvh_level_table": (C.c_int, [_P, _P, _P, _P, _P]),
    "nbvh_param_count": (C.c_int, [_P, _I32, _P]),
    "nbvh_get_params": (C.c_int, [_P, _I32, _P, _I64]),
    "nbvh_set_params": (C.c_int, [_P, _I32, _P, _I64]),
    "nbvh_reserve": (C.c_int, [_P, _I64]),
    "nbvh_set_mesh": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _P]),
    "nbvh_build_cut": (C.c_int, [_P, _I32, _P, _P, _I32, _P]),
    "nbvh_copy_cut": (C.c_int, [_P, _I32, _I32]),
    "nbvh_cut_info": (C.c_int, [_P, _I32, _P, _P]),
    "nbvh_get_cut": (C.c_int, [_P, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "nbvh_query": (C.c_int, [_P, _P, _I64, _I32, Hits, _P]),
    "nbvh_query_host": (C.c_int, [_P, _P, _I64, _I32, Hits, _P]),
    "nbvh_get_query_stats": (C.c_int, [_P, _P]),
    "nbvh_set_profiling": (C.c_int, [_P, _I32]),
    "nbvh_train_backward": (C.c_int, [_P, _P, _I64, _P, _P, _I32, _P]),
    "nbvh_grad_buffer": (C.c_int, [_P, _P, _P]),
    "nbvh_apply_update": (C.c_int, [_P, _F, _P]),
    "nbvh_train_step": (C.c_int, [_P, _P, _I64, _P, _P, _I32, _F, _P]),
    "nbvh_get_train_stats": (C.c_int, [_P, _P]),
    "nbvh_set_leaf_rank": (C.c_int, [_P, _I32, _P]),
    "nbvh_mlp_forward": (C.c_int, [_P, _P, _I64, _P, _P]),
    "nbvh_gen_train_rays": (C.c_int, [_P, C.c_uint64, C.c_uint64, _I64, _I64, _P, _P, _P, _P, _P]),
    "nbvh_intersect_mesh": (C.c_int, [_P, _P, _I64, Hits, _P]),
    "nbvh_gather_probe": (C.c_int, [_P, _I64, _I32, _I64, C.c_uint32, _P, _I64, _P, _P]),
    "nbvh_gather_probe_tex": (C.c_int, [_P, _I64, _I32, _I64, C.c_uint32, _P, _I64, _P, _P]),
    "nbvh_atomic_probe": (C.c_int, [_P, _I64, _I32, _I64, C.c_uint32, _P, _P]),
    "nbvh_pt_shade": (C.c_int, [_P, _P, _I64, Hits, Hits, _P, _P, _P, C.c_uint64, _I32, _P, _F, _P, _P]),
    "nbvh_tlas_build": (C.c_int, [_P, _P, _I32, _P]),
    "nbvh_get_base_bvh": (C.c_int, [_P, _P, _P, _P]),
    "nbvh_get_cut_nodes": (C.c_int, [_P, _I32, _P]),
    "nbvh_tlas_destroy": (None, [_P]),
    "nbvh_tlas_dispatch": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P, _P, _I64, _P]),
    "nbvh_tlas_merge": (C.c_int, [_P, _P, _I64, _P, _I64, _P, _P, _P, Hits, _P]),
    "nbvh_tlas_overflow": (C.c_int, [_P, _P, _P]),
    "nbvh_pt_shade_compact": (C.c_int, [_P, _P, _I64, Hits, _P, _P, _P, _P, _P, _P, _P, C.c_uint64, _I32, _P, _F,
                                        _P]),
    "nbvh_debug_traverse": (C.c_int, [_P, _P, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "nbvh_debug_traverse_product": (C.c_int, [_P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P]),
    "nbvh_debug_encode": (C.c_int, [_P, _P, _I64, _P, _P, _P]),
    "nbvh_debug_mlp": (C.c_int, [_P, _P, _I64, _P, _P]),
    "nbvh_debug_query_trace": (C.c_int, [_P, _P, _I64, _I32, Hits, _P, _I32, _P]),
    "nbvh_debug_train_samples": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "nbvh_debug_train_capture": (C.c_int, [_P, _I32]),
    "nbvh_debug_train_activations": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
}


def load_library(path: str = LIB_PATH):
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(x):
    """Device pointer of a torch tensor / host pointer of a numpy array / None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else None
    return getattr(stream, "cuda_stream", stream)


def gather_probe(table, entry_bytes: int, n_gathers: int, sink, seed: int = 1, stream=None) -> int:
    """nbvh_gather_probe: n_gathers random entry_bytes-wide reads of the device tensor `table`
    (asynchronous); returns the number of gathers issued."""
    done = C.c_int64(0)
    st = load_library().nbvh_gather_probe(_ptr(table), table.numel() * table.element_size(), int(entry_bytes),
                                          int(n_gathers), int(seed) & 0xFFFFFFFF, _ptr(sink), sink.numel(),
                                          C.byref(done), _stream_ptr(stream))
    if st != 0:
        raise NbvhError(st, "gather_probe: bad arguments")
    return int(done.value)


def gather_probe_tex(table, n_gathers: int, sink, mixed: bool = False, seed: int = 1, stream=None) -> int:
    """nbvh_gather_probe_tex: n_gathers random 4-byte reads of `table` through the texture pipe
    (mixed: half of them through the load pipe); synchronises the stream; returns the count."""
    done = C.c_int64(0)
    st = load_library().nbvh_gather_probe_tex(_ptr(table), table.numel() * table.element_size(), 1 if mixed else 0,
                                              int(n_gathers), int(seed) & 0xFFFFFFFF, _ptr(sink), sink.numel(),
                                              C.byref(done), _stream_ptr(stream))
    if st != 0:
        raise NbvhError(st, "gather_probe_tex: bad arguments")
    return int(done.value)


def atomic_probe(table, vec: int, n_ops: int, seed: int = 1, stream=None) -> int:
    """nbvh_atomic_probe: n_ops random fp32 (vec 1) or fp32x2 (vec 2) reductions into the device
    float tensor `table` (asynchronous); returns the number issued."""
    done = C.c_int64(0)
    st = load_library().nbvh_atomic_probe(_ptr(table), table.numel() * table.element_size(), int(vec), int(n_ops),
                                           int(seed) & 0xFFFFFFFF, C.byref(done), _stream_ptr(stream))
    if st != 0:
        raise NbvhError(st, "atomic_probe: bad arguments")
    return int(done.value)


def default_config(**kw) -> Config:
    cfg = Config()
    load_library().nbvh_config_default(C.byref(cfg))
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


class Context:
    """One nbvh_ctx (one device per process).  device=-1 gives a host-only context."""

    def __init__(self, device: int = 0, **cfg):
        self.lib = load_library()
        self.cfg = default_config(**cfg)
        h = C.c_void_p()
        st = self.lib.nbvh_create(C.byref(self.cfg), device, C.byref(h))
        if st != 0:
            raise NbvhError(st, "nbvh_create failed")
        self.h = h
        self.device = device
        self.d_in = self.cfg.n_points * self.cfg.L * self.cfg.F

    def close(self):
        if self.h:
            self.lib.nbvh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, st, what):
        if st < 0:
            raise NbvhError(st, f"{what}: {self.lib.nbvh_last_error(self.h).decode()}")
        return st

    # ---------------------------------------------------------------- model
    def level_table(self):
        L = self.cfg.L
        res = np.zeros(L, np.int32)
        dense = np.zeros(L, np.int32)
        off = np.zeros(L, np.int64)
        n = np.zeros(1, np.int64)
        self._ck(self.lib.nbvh_level_table(self.h, _ptr(res), _ptr(dense), _ptr(off), _ptr(n)), "level_table")
        return res, dense, off, int(n[0])

    def param_count(self, block):
        n = np.zeros(1, np.int64)
        self._ck(self.lib.nbvh_param_count(self.h, block, _ptr(n)), "param_count")
        return int(n[0])

    def get_params(self, block=PARAM_ALL):
        a = np.zeros(self.param_count(block), np.float32)
        self._ck(self.lib.nbvh_get_params(self.h, block, _ptr(a), a.size), "get_params")
        return a

    def set_params(self, block, values):
        a = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
        self._ck(self.lib.nbvh_set_params(self.h, block, _ptr(a), a.size), "set_params")

    def set_mlp(self, layers):
        """layers: [(W [out][in], b [out])] in forward order."""
        self.set_params(PARAM_WEIGHTS, np.concatenate([np.asarray(W, np.float32).ravel() for W, _ in layers]))
        self.set_params(PARAM_BIASES, np.concatenate([np.asarray(b, np.float32).ravel() for _, b in layers]))

    def reserve(self, n):
        self._ck(self.lib.nbvh_reserve(self.h, int(n)), "reserve")

    # ---------------------------------------------------------------- scene
    def set_mesh(self, scene):
        self.scene = scene
        v = np.ascontiguousarray(scene.verts, np.float32)
        t = np.ascontiguousarray(scene.tris, np.uint32)
        n = np.ascontiguousarray(scene.vnormals, np.float32) if scene.vnormals is not None else None
        a = np.ascontiguousarray(scene.albedo, np.float32) if scene.albedo is not None else None
        self._ck(self.lib.nbvh_set_mesh(self.h, _ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(n), _ptr(a)),
                 "set_mesh")

    def build_cut(self, target, lod=0, q=None, p=None):
        out = np.zeros(1, np.int32)
        qa = None if q is None else np.ascontiguousarray(q, np.float32)
        pa = None if p is None else np.ascontiguousarray(p, np.float32)
        st = self._ck(self.lib.nbvh_build_cut(self.h, int(target), _ptr(qa), _ptr(pa), lod, _ptr(out)), "build_cut")
        return int(out[0]), st

    def copy_cut(self, src_lod, dst_lod):
        self._ck(self.lib.nbvh_copy_cut(self.h, int(src_lod), int(dst_lod)), "copy_cut")

    def cut(self, lod=0):
        nl = np.zeros(1, np.int32)
        ni = np.zeros(1, np.int32)
        self._ck(self.lib.nbvh_cut_info(self.h, lod, _ptr(nl), _ptr(ni)), "cut_info")
        n = int(nl[0])
        d = dict(leaf_lo=np.zeros((n, 3), np.float32), leaf_hi=np.zeros((n, 3), np.float32),
                 base_lo=np.zeros((n, 3), np.float32), base_hi=np.zeros((n, 3), np.float32),
                 tri_off=np.zeros(n + 1, np.int64), dom_min=np.zeros(3, np.float32), dom_inv=np.zeros(1, np.float32))
        self._ck(self.lib.nbvh_get_cut(self.h, lod, _ptr(d["leaf_lo"]), _ptr(d["leaf_hi"]), _ptr(d["base_lo"]),
                                       _ptr(d["base_hi"]), _ptr(d["tri_off"]), None, None, None), "get_cut")
        d["tris"] = np.zeros(int(d["tri_off"][-1]), np.int32)
        self._ck(self.lib.nbvh_get_cut(self.h, lod, None, None, None, None, _ptr(d["tri_off"]), _ptr(d["tris"]),
                                       _ptr(d["dom_min"]), _ptr(d["dom_inv"])), "get_cut")
        d["n_leaves"] = n
        d["n_inner"] = int(ni[0])
        return d

    def base_bvh(self):
        """(child_a, child_b) int32 arrays of the base BVH (leaf: child_b < 0)."""
        n = np.zeros(1, np.int64)
        self._ck(self.lib.nbvh_get_base_bvh(self.h, None, None, _ptr(n)), "get_base_bvh")
        a = np.zeros(int(n[0]), np.int32)
        b = np.zeros(int(n[0]), np.int32)
        self._ck(self.lib.nbvh_get_base_bvh(self.h, _ptr(a), _ptr(b), _ptr(n)), "get_base_bvh")
        return a, b

    def cut_nodes(self, lod=0):
        """Base-BVH node of every leaf of the cut in slot lod."""
        out = np.zeros(self.cut(lod)["n_leaves"], np.int32)
        self._ck(self.lib.nbvh_get_cut_nodes(self.h, lod, _ptr(out)), "get_cut_nodes")
        return out

    def set_leaf_rank(self, rank, lod=0):
        r = np.ascontiguousarray(rank, np.float32)
        self._ck(self.lib.nbvh_set_leaf_rank(self.h, lod, _ptr(r)), "set_leaf_rank")

    # ---------------------------------------------------------------- query
    @staticmethod
    def alloc_hits(n, device="cuda"):
        import torch
        return dict(hit=torch.empty(n, dtype=torch.uint8, device=device),
                    t=torch.empty(n, dtype=torch.float32, device=device),
                    normal=torch.empty(n, 3, dtype=torch.float32, device=device),
                    albedo=torch.empty(n, 3, dtype=torch.float32, device=device),
                    leaf=torch.empty(n, dtype=torch.int32, device=device),
                    n_queries=torch.empty(n, dtype=torch.int32, device=device))

    @staticmethod
    def _hits(out):
        return Hits(_ptr(out["hit"]), _ptr(out["t"]), _ptr(out["normal"]), _ptr(out["albedo"]), _ptr(out.get("leaf")),
                    _ptr(out.get("n_queries")))

    def query(self, rays, lod=0, out=None, stream=None):
        """rays: cuda float32 tensor [n, 8]."""
        n = rays.shape[0]
        if out is None:
            out = self.alloc_hits(n, rays.device)
        self._ck(self.lib.nbvh_query(self.h, _ptr(rays), n, lod, self._hits(out), _stream_ptr(stream)), "query")
        return out

    def gen_train_rays(self, seed: int, step: int, n: int, i0: int = 0, box=None, out=None, stream=None):
        """nbvh_gen_train_rays: (rays [n, 8], u [n], xi [n, n_points]) device tensors for rays
        [i0, i0 + n) of training step `step` (Philox-4x32-10, key = seed)."""
        import torch
        if out is None:
            out = (torch.empty(n, 8, device=f"cuda:{self.device}"), torch.empty(n, device=f"cuda:{self.device}"),
                   torch.empty(n, self.cfg.n_points, device=f"cuda:{self.device}"))
        bx = None if box is None else np.ascontiguousarray(np.asarray(box, np.float32).reshape(6))
        self._ck(self.lib.nbvh_gen_train_rays(self.h, int(seed), int(step), int(i0), int(n), _ptr(bx),
                                              _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), _stream_ptr(stream)),
                 "gen_train_rays")
        return out

    def mlp_forward(self, x, z=None, stream=None):
        """tcgen05 batched MLP: x cuda fp16 [m, D_in] -> z cuda fp32 [m, 8]."""
        import torch
        m = x.shape[0]
        if z is None:
            z = torch.empty(m, 8, dtype=torch.float32, device=x.device)
        self._ck(self.lib.nbvh_mlp_forward(self.h, _ptr(x), m, _ptr(z), _stream_ptr(stream)), "mlp_forward")
        return z

    def intersect_mesh(self, rays, out=None, stream=None):
        """Classical closest hit against this context's own mesh (the classical BLAS)."""
        n = rays.shape[0]
        if out is None:
            out = self.alloc_hits(n, rays.device)
        self._ck(self.lib.nbvh_intersect_mesh(self.h, _ptr(rays), n, self._hits(out), _stream_ptr(stream)),
                 "intersect_mesh")
        return out

    def pt_shade(self, rays, neural, classical, throughput, radiance, next_rays, seed, bounce, sky, eps, alive,
                 stream=None):
        sky_a = np.ascontiguousarray(sky, np.float32)
        empty = Hits(None, None, None, None, None, None)
        self._ck(self.lib.nbvh_pt_shade(self.h, _ptr(rays), rays.shape[0], self._hits(neural),
                                        self._hits(classical) if classical is not None else empty,
                                        _ptr(throughput), _ptr(radiance), _ptr(next_rays), int(seed), int(bounce),
                                        _ptr(sky_a), float(eps), _ptr(alive), _stream_ptr(stream)), "pt_shade")

    def query_host(self, rays_np, out=None, lod=0, stream=None):
        """End-to-end path: host (ideally pinned) numpy rays -> host numpy results."""
        n = rays_np.shape[0]
        if out is None:
            out = dict(hit=np.zeros(n, np.uint8), t=np.zeros(n, np.float32), normal=np.zeros((n, 3), np.float32),
                       albedo=np.zeros((n, 3), np.float32), leaf=np.zeros(n, np.int32),
                       n_queries=np.zeros(n, np.int32))
        self._ck(self.lib.nbvh_query_host(self.h, _ptr(rays_np), n, lod, self._hits(out), _stream_ptr(stream)),
                 "query_host")
        return out

    def query_stats(self):
        s = QueryStats()
        self._ck(self.lib.nbvh_get_query_stats(self.h, C.byref(s)), "query_stats")
        return dict(n_rays=s.n_rays, n_queries=s.n_queries, n_iters=s.n_iters, n_launches=s.n_launches,
                    n_refills=s.n_refills, ms_traverse=s.ms_traverse, ms_query=s.ms_query,
                    n_mlp_tiles=s.n_mlp_tiles, n_mlp_rows=s.n_mlp_rows, ws_cycles=list(s.ws_cycles))

    def set_profiling(self, on=True):
        self._ck(self.lib.nbvh_set_profiling(self.h, int(bool(on))), "set_profiling")

    # ---------------------------------------------------------------- training
    def train_backward(self, rays, u, xi, lod=0, stream=None):
        self._ck(self.lib.nbvh_train_backward(self.h, _ptr(rays), rays.shape[0], _ptr(u), _ptr(xi), lod,
                                              _stream_ptr(stream)), "train_backward")

    def grad_buffer(self):
        import torch
        p = C.c_void_p()
        n = np.zeros(1, np.int64)
        self._ck(self.lib.nbvh_grad_buffer(self.h, C.byref(p), _ptr(n)), "grad_buffer")
        return p.value, int(n[0])

    def apply_update(self, lr=0.01, stream=None):
        self._ck(self.lib.nbvh_apply_update(self.h, float(lr), _stream_ptr(stream)), "apply_update")

    def train_step(self, rays=None, u=None, xi=None, lod=0, lr=0.01, stream=None, n=None):
        """One training step; rays/u/xi None: the library draws n rays itself (T0)."""
        count = rays.shape[0] if rays is not None else int(n)
        self._ck(self.lib.nbvh_train_step(self.h, _ptr(rays), count, _ptr(u), _ptr(xi), lod, float(lr),
                                          _stream_ptr(stream)), "train_step")

    def train_stats(self):
        s = TrainStats()
        self._ck(self.lib.nbvh_get_train_stats(self.h, C.byref(s)), "train_stats")
        return dict(n_rays=s.n_rays, n_first_hit=s.n_first_hit, n_accepted=s.n_accepted, loss_sum=s.loss_sum,
                    loss_terms=list(s.loss_terms), n_launches=s.n_launches, skipped=s.skipped,
                    ms_phase=dict(zip(("select", "label", "fwd", "bwd", "dw", "adam"), list(s.ms_phase))))

    # ---------------------------------------------------------------- parity hooks
    def debug_traverse(self, rays, cap, lod=0, stream=None):
        import torch
        n = rays.shape[0]
        leaf = torch.empty(n, cap, dtype=torch.int32, device=rays.device)
        te = torch.empty(n, cap, dtype=torch.float32, device=rays.device)
        tx = torch.empty(n, cap, dtype=torch.float32, device=rays.device)
        cnt = torch.empty(n, dtype=torch.int32, device=rays.device)
        self._ck(self.lib.nbvh_debug_traverse(self.h, _ptr(rays), n, lod, cap, _ptr(leaf), _ptr(te), _ptr(tx),
                                              _ptr(cnt), _stream_ptr(stream)), "debug_traverse")
        return leaf, te, tx, cnt

    def debug_encode(self, pts, want_index=True, stream=None):
        import torch
        m = pts.shape[0]
        L, F = self.cfg.L, self.cfg.F
        feat = torch.empty(m, L * F, dtype=torch.float16, device=pts.device)
        idx = torch.empty(m, L, 8, dtype=torch.int32, device=pts.device) if want_index else None
        self._ck(self.lib.nbvh_debug_encode(self.h, _ptr(pts), m, _ptr(feat), _ptr(idx), _stream_ptr(stream)),
                 "debug_encode")
        return feat, idx

    def debug_mlp(self, x16, stream=None):
        import torch
        m = x16.shape[0]
        z = torch.empty(m, 8, dtype=torch.float32, device=x16.device)
        self._ck(self.lib.nbvh_debug_mlp(self.h, _ptr(x16), m, _ptr(z), _stream_ptr(stream)), "debug_mlp")
        return z

    def debug_query_trace(self, rays, cap, lod=0, stream=None):
        import torch
        n = rays.shape[0]
        out = self.alloc_hits(n, rays.device)
        zt = torch.empty(n, cap, 8, dtype=torch.float32, device=rays.device)
        self._ck(self.lib.nbvh_debug_query_trace(self.h, _ptr(rays), n, lod, self._hits(out), _ptr(zt), cap,
                                                 _stream_ptr(stream)), "debug_query_trace")
        return out, zt

    def debug_train_samples(self, n, stream=None):
        import torch
        gt = torch.empty(n, 9, dtype=torch.float32, device="cuda")
        acc = torch.empty(n, dtype=torch.uint8, device="cuda")
        leaf = torch.empty(n, dtype=torch.int32, device="cuda")
        loss = torch.empty(n, dtype=torch.float32, device="cuda")
        self._ck(self.lib.nbvh_debug_train_samples(self.h, _ptr(gt), _ptr(acc), _ptr(leaf), _ptr(loss),
                                                   _stream_ptr(stream)), "debug_train_samples")
        return gt, acc, leaf, loss

    def debug_train_capture(self, enable: bool):
        self._ck(self.lib.nbvh_debug_train_capture(self.h, 1 if enable else 0), "debug_train_capture")

    def debug_train_activations(self, n_rays, stream=None):
        """Per-sample intermediates of the last training batch (compacted sample order):
        dict(ray [m] int32, x [m, D_in] fp16, z [m, 8] (capture on, else None), dz [m, 8],
        act / delta [hidden, m, 64] fp16)."""
        import torch
        dev = f"cuda:{self.device}"
        H = self.cfg.hidden_layers
        ray = torch.empty(n_rays, dtype=torch.int32, device=dev)
        x = torch.empty(n_rays * self.d_in, dtype=torch.float16, device=dev)
        z = torch.empty(n_rays * 8, dtype=torch.float32, device=dev)
        dz = torch.empty(n_rays * 8, dtype=torch.float32, device=dev)
        act = torch.empty(H * n_rays * 64, dtype=torch.float16, device=dev)
        dl = torch.empty(H * n_rays * 64, dtype=torch.float16, device=dev)
        m = np.zeros(1, np.int64)

        def call(zp):
            return self.lib.nbvh_debug_train_activations(self.h, _ptr(ray), _ptr(x), zp, _ptr(dz), _ptr(act),
                                                         _ptr(dl), _ptr(m), _stream_ptr(stream))
        st = call(_ptr(z))
        zt = z
        if st == -3:                                  # NBVH_ESTATE: capture off -> no z
            self._ck(call(None), "debug_train_activations")
            zt = None
        else:
            self._ck(st, "debug_train_activations")
        mm = int(m[0])
        return dict(ray=ray[:mm], x=x[:mm * self.d_in].view(mm, self.d_in),
                    z=None if zt is None else zt[:mm * 8].view(mm, 8), dz=dz[:mm * 8].view(mm, 8),
                    act=act[:H * mm * 64].view(H, mm, 64), delta=dl[:H * mm * 64].view(H, mm, 64))

    def debug_traverse_product(self, rays, lod=0, stream=None):
        """The product k_traverse's lists: (leaf [n, K], te, tx, fill [n], more [n])."""
        import torch
        n, K = rays.shape[0], self.cfg.list_cap
        dev = rays.device
        leaf = torch.empty(n, K, dtype=torch.int32, device=dev)
        te = torch.empty(n, K, dtype=torch.float32, device=dev)
        tx = torch.empty(n, K, dtype=torch.float32, device=dev)
        fill = torch.empty(n, dtype=torch.int32, device=dev)
        more = torch.empty(n, dtype=torch.int32, device=dev)
        self._ck(self.lib.nbvh_debug_traverse_product(self.h, _ptr(rays), n, lod, _ptr(leaf), _ptr(te), _ptr(tx),
                                                      _ptr(fill), _ptr(more), _stream_ptr(stream)),
                 "debug_traverse_product")
        return leaf, te, tx, fill, more
