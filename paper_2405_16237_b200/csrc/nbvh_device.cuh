// nbvh_device.cuh — device building blocks of the N-BVH query/training kernels (sm_100a).
//
//  * slab():            ray/AABB interval, binary32 with a fixed op order (C7, C25)
//  * collect_leaves():  shallow N-BVH traversal emitting the (t_enter, id)-ordered leaf
//                       list, capacity K in registers, resumable from a key (C5, C6)
//  * segment_point():   stratified sample positions, normalised to the grid domain (P:133,
//                       P:146; C4, C8)
//  * encode_chunk():    multires hash-grid gather + trilinear blend of 8/F levels -> 16 B
//                       of fp16 features (C1-C3)
//  * mlp_rows16():      D_in -> 64 (ReLU) x hidden -> 8 MLP for 16 rows on tensor cores,
//                       activations kept in registers between layers
//  * decode helpers:    hit = z_vis < 0, local distance, normal, albedo
//
// Bit-exactness: every operation that decides a discrete result the oracle must match
// (intervals, sample positions, grid cells) uses explicit round-to-nearest intrinsics
// so nvcc cannot contract it into an FMA.  Continuous blends use FMA freely.
#pragma once

// Device-side bounds checks, compiled in only by the debug-checks build (build.py debug=True,
// -DNBVH_DEBUG_CHECKS): a failed check stops the kernel with a device assert (file / line).
#ifdef NBVH_DEBUG_CHECKS
#include <cassert>
#define NBVH_DCHECK(cond) assert(cond)
#else
#define NBVH_DCHECK(cond) ((void)0)
#endif

#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

#include "nbvh_internal.h"

namespace nbvh {

constexpr uint32_t kPrime1 = 2654435761u;   // [Mueller22] spatial-hash primes
constexpr uint32_t kPrime2 = 805459861u;

struct GridDev {
    int32_t L, F, n_points, log2_T;
    int32_t res[kMaxLevels];
    int32_t dense[kMaxLevels];
    uint32_t offset[kMaxLevels];     // canonical entry offset of each level (parameter layout)
    uint32_t inf_offset[kMaxLevels]; // entry offset of each level in the inference table
    const __half* table;             // fp16 inference table (layout: see LevelSm)
    float dom_min[3];
    float dom_inv;
    unsigned long long tex;          // texture object over `table` (0: none -> LDG gathers)
};

struct MlpDev {
    int32_t d_in, hidden;
    const __half* W;                 // layers concatenated, [out][in] row-major (bf16 bits if bf16)
    const float* b;
    int32_t bf16;                    // query path: operands in bf16 (nbvh_config.mlp_dtype = 1)
};

struct CutDev {
    const InnerNode* inner;
    const float4* leaf_box;          // [n_leaves][2]: (lo.xyz, 0), (hi.xyz, 0)
    int32_t n_leaves;
    int32_t depth;                   // inner levels of the snapshot (host-computed)
};

// ------------------------------------------------------------------ slab test
// tl=(lo-o)*inv, th=(hi-o)*inv, tn=fminf(tl,th), tf=fmaxf(tl,th), te = left-fold fmaxf over
// (tn.x, tn.y, tn.z, tmin), tx = left-fold fminf over (tf.x, tf.y, tf.z, tmax); hit iff te <= tx.
struct RayDev {
    float o[3], inv[3], d[3], tmin, tmax;
};

__device__ __forceinline__ RayDev load_ray(const float4* rays, int64_t r) {
    float4 a = __ldg(rays + 2 * r), b = __ldg(rays + 2 * r + 1);
    RayDev R;
    R.o[0] = a.x; R.o[1] = a.y; R.o[2] = a.z; R.tmin = a.w;
    R.d[0] = b.x; R.d[1] = b.y; R.d[2] = b.z; R.tmax = b.w;
#pragma unroll
    for (int k = 0; k < 3; ++k) R.inv[k] = __fdiv_rn(1.0f, R.d[k]);
    return R;
}

__device__ __forceinline__ bool slab(const RayDev& R, const float* lo, const float* hi, float& te, float& tx) {
    float tn[3], tf[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float tl = __fmul_rn(__fsub_rn(lo[k], R.o[k]), R.inv[k]);
        float th = __fmul_rn(__fsub_rn(hi[k], R.o[k]), R.inv[k]);
        tn[k] = fminf(tl, th);
        tf[k] = fmaxf(tl, th);
    }
    te = fmaxf(fmaxf(fmaxf(tn[0], tn[1]), tn[2]), R.tmin);
    tx = fminf(fminf(fminf(tf[0], tf[1]), tf[2]), R.tmax);
    return te <= tx;
}

__device__ __forceinline__ bool key_less(float a_te, int a_id, float b_te, int b_id) {
    return a_te < b_te || (a_te == b_te && a_id < b_id);
}

// ------------------------------------------------------------------ ordered leaf list
// Collects the intersected cut leaves whose key (t_enter, id) is greater than `after`
// (when has_after), keeping the `cap` (<= K) smallest keys sorted in registers; returns
// how many leaves qualified in total (so the caller knows whether more remain, C6).
// Inner boxes are exact unions of their children, so by monotone rounding a pruned
// subtree contains no intersected leaf: the result equals a brute-force scan (C5).
// With `prune`, once the list is full a subtree whose entry exceeds the cap-th key is
// skipped (none of its leaves can enter the list); the return value is then only a lower
// bound and *more (nullable) reports whether leaves beyond the list may exist.
// Traversal stacks: per-thread local array (rare paths) or a shared-memory column
// [row][blockDim.x] sized by the cut's depth (the per-ray query path).
struct LocalStack {
    int s[64];
    int sp = 0;
    static constexpr int cap = 64;
    __device__ __forceinline__ void push(int v) { s[sp++] = v; }
    __device__ __forceinline__ int pop() { return s[--sp]; }
};
struct SmemStack {
    int* col;            // &stack[0][threadIdx.x]
    int stride;          // blockDim.x
    int cap;             // rows
    int sp = 0;
    __device__ __forceinline__ void push(int v) { col[(sp++) * stride] = v; }
    __device__ __forceinline__ int pop() { return col[(--sp) * stride]; }
};

//
// t_bound: leaves (and subtrees) entering strictly after t_bound are ignored.  The query
// passes the ray's current best hit t: front-to-back termination never queries such a leaf
// (C5), and the bound only decreases, so dropping them is exact.
template <int K, class Stack>
__device__ int collect_leaves(const CutDev& cut, const RayDev& R, bool has_after, float after_te, int after_id,
                              int cap, float (&lte)[K], float (&ltx)[K], int (&lid)[K], int& n_out,
                              int* err_flag, Stack& stack, bool prune = false, bool* more = nullptr,
                              float t_bound = __builtin_huge_valf()) {
    int n = 0, total = 0;
    bool pruned = false;
    auto full_and_beyond = [&](float te) {
        if (!prune || n < cap) return false;
        float last = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j == cap - 1) last = lte[j];
        return te > last;
    };
    auto consider = [&](int leaf, float te, float tx) {
        if (has_after && !key_less(after_te, after_id, te, leaf)) return;
        ++total;
        float cte = te, ctx = tx;
        int cid = leaf;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (j < n && key_less(cte, cid, lte[j], lid[j])) {
                float t0 = lte[j], t1 = ltx[j];
                int i0 = lid[j];
                lte[j] = cte; ltx[j] = ctx; lid[j] = cid;
                cte = t0; ctx = t1; cid = i0;
            }
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j == n && n < cap) { lte[j] = cte; ltx[j] = ctx; lid[j] = cid; }
        if (n < cap) ++n;
    };
    if (cut.n_leaves == 1) {
        float4 a = __ldg(cut.leaf_box), b = __ldg(cut.leaf_box + 1);
        float lo[3] = {a.x, a.y, a.z}, hi[3] = {b.x, b.y, b.z}, te, tx;
        if (slab(R, lo, hi, te, tx)) consider(0, te, tx);
    } else {
        // the next node lives in a register; only the farther of two wanted children is
        // pushed (same visiting order as push-both-then-pop)
        stack.sp = 0;
        int node = 0;
        while (true) {
            const float4* p = reinterpret_cast<const float4*>(cut.inner + node);
            float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3);
            float llo[3] = {q0.x, q0.y, q0.z}, lhi[3] = {q0.w, q1.x, q1.y};
            float rlo[3] = {q1.z, q1.w, q2.x}, rhi[3] = {q2.y, q2.z, q2.w};
            int cl = __float_as_int(q3.x), cr = __float_as_int(q3.y);
            float lte_, ltx_, rte_, rtx_;
            bool hl = slab(R, llo, lhi, lte_, ltx_) && !(lte_ > t_bound);
            bool hr = slab(R, rlo, rhi, rte_, rtx_) && !(rte_ > t_bound);
            if (hl && cl < 0) consider(-1 - cl, lte_, ltx_);
            if (hr && cr < 0) consider(-1 - cr, rte_, rtx_);
            bool pl = hl && cl >= 0, pr = hr && cr >= 0;
            if (pl && full_and_beyond(lte_)) { pl = false; pruned = true; }
            if (pr && full_and_beyond(rte_)) { pr = false; pruned = true; }
            // the nearer child is visited next, the farther one later
            if (pl && pr) {
                if (stack.sp + 1 > stack.cap) { if (err_flag) atomicOr(err_flag, 1); break; }
                const bool l_first = lte_ <= rte_;
                stack.push(l_first ? cr : cl);
                node = l_first ? cl : cr;
            } else if (pl) {
                node = cl;
            } else if (pr) {
                node = cr;
            } else {
                if (stack.sp == 0) break;
                node = stack.pop();
            }
        }
    }
    n_out = n;
    if (more) *more = pruned || total > n;
    return total;
}

// Convenience overload with a per-thread local stack.
template <int K>
__device__ int collect_leaves(const CutDev& cut, const RayDev& R, bool has_after, float after_te, int after_id,
                              int cap, float (&lte)[K], float (&ltx)[K], int (&lid)[K], int& n_out,
                              int* err_flag, bool prune = false, bool* more = nullptr,
                              float t_bound = __builtin_huge_valf()) {
    LocalStack st;
    return collect_leaves<K, LocalStack>(cut, R, has_after, after_te, after_id, cap, lte, ltx, lid, n_out, err_flag,
                                         st, prune, more, t_bound);
}

// ------------------------------------------------------------------ segment sampling
// u = (2i+1)/(2n) (inference) or (i+xi)/n (training); dt = t1-t0; t = t0+u*dt;
// p = o + t*d; x = clamp((p-dom_min)*dom_inv, 0, 1); every op rounded (no FMA).
__device__ __forceinline__ void segment_point_u(const GridDev& g, const float o[3], const float d[3], float t0,
                                                float t1, float u, float x[3]) {
    float dt = __fsub_rn(t1, t0);
    float t = __fadd_rn(t0, __fmul_rn(u, dt));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float p = __fadd_rn(o[k], __fmul_rn(t, d[k]));
        float v = __fmul_rn(__fsub_rn(p, g.dom_min[k]), g.dom_inv);
        x[k] = fminf(fmaxf(v, 0.0f), 1.0f);
    }
}
__device__ __forceinline__ float segment_u(int i, int n, const float* xi) {
    return xi ? __fdiv_rn(__fadd_rn((float)i, xi[i]), (float)n) : __fdiv_rn((float)(2 * i + 1), (float)(2 * n));
}
__device__ __forceinline__ void segment_point(const GridDev& g, const float o[3], const float d[3], float t0, float t1,
                                              int i, int n, const float* xi, float x[3]) {
    segment_point_u(g, o, d, t0, t1, segment_u(i, n, xi), x);
}

// ------------------------------------------------------------------ grid cell of a level
struct Cell {
    uint32_t idx[8];    // corner entry index within the level (corner bit0=x, bit1=y, bit2=z)
    float w[8];         // trilinear weights
};

__device__ __forceinline__ void level_cell(const GridDev& g, int l, const float x[3], Cell& c) {
    const int N = g.res[l];
    int ci[3];
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float s = __fmul_rn(x[k], (float)N);
        int v = (int)floorf(s);
        v = min(v, N - 1);
        v = max(v, 0);
        ci[k] = v;
        f[k] = __fsub_rn(s, (float)v);
    }
    const float wx[2] = {1.0f - f[0], f[0]}, wy[2] = {1.0f - f[1], f[1]}, wz[2] = {1.0f - f[2], f[2]};
    if (g.dense[l]) {
        const uint32_t n1 = (uint32_t)N + 1u;
        const uint32_t bx = (uint32_t)ci[0], by = (uint32_t)ci[1] * n1, bz = (uint32_t)ci[2] * n1 * n1;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            c.idx[k] = bx + (k & 1) + by + ((k >> 1) & 1) * n1 + bz + ((k >> 2) & 1) * n1 * n1;
    } else {
        const uint32_t mask = (1u << g.log2_T) - 1u;
        const uint32_t hx[2] = {(uint32_t)ci[0], (uint32_t)ci[0] + 1u};
        const uint32_t hy[2] = {(uint32_t)ci[1] * kPrime1, ((uint32_t)ci[1] + 1u) * kPrime1};
        const uint32_t hz[2] = {(uint32_t)ci[2] * kPrime2, ((uint32_t)ci[2] + 1u) * kPrime2};
#pragma unroll
        for (int k = 0; k < 8; ++k) c.idx[k] = (hx[k & 1] ^ hy[(k >> 1) & 1] ^ hz[(k >> 2) & 1]) & mask;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) c.w[k] = wx[k & 1] * wy[(k >> 1) & 1] * wz[(k >> 2) & 1];
}

// ------------------------------------------------------------------ encode 8 halves
// One 16-byte chunk of the concatenated feature vector: NL = 8/F consecutive levels of
// one sample point.  All 8*NL corner loads are issued before any is consumed.
template <int F>
__device__ __forceinline__ uint4 encode_chunk(const GridDev& g, const float x[3], int l0, uint32_t* idx_out) {
    constexpr int NL = 8 / F;
    Cell cell[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) level_cell(g, l0 + j, x, cell[j]);
    if (idx_out) {
#pragma unroll
        for (int j = 0; j < NL; ++j)
#pragma unroll
            for (int k = 0; k < 8; ++k) idx_out[j * 8 + k] = cell[j].idx[k];
    }
    uint4 out;
    uint32_t* o32 = reinterpret_cast<uint32_t*>(&out);
    if constexpr (F == 2) {
        uint32_t v[NL][8];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const uint32_t* base = reinterpret_cast<const uint32_t*>(g.table) + g.offset[l0 + j];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[j][k] = __ldg(base + cell[j].idx[k]);
        }
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float2 f = __half22float2(*reinterpret_cast<const __half2*>(&v[j][k]));
                a0 = fmaf(cell[j].w[k], f.x, a0);
                a1 = fmaf(cell[j].w[k], f.y, a1);
            }
            __half2 h = __floats2half2_rn(a0, a1);
            o32[j] = *reinterpret_cast<uint32_t*>(&h);
        }
    } else {  // F == 4
        uint2 v[NL][8];
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const uint2* base = reinterpret_cast<const uint2*>(g.table) + g.offset[l0 + j];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[j][k] = __ldg(base + cell[j].idx[k]);
        }
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][k].x));
                float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v[j][k].y));
                a[0] = fmaf(cell[j].w[k], f0.x, a[0]);
                a[1] = fmaf(cell[j].w[k], f0.y, a[1]);
                a[2] = fmaf(cell[j].w[k], f1.x, a[2]);
                a[3] = fmaf(cell[j].w[k], f1.y, a[3]);
            }
            __half2 h0 = __floats2half2_rn(a[0], a[1]), h1 = __floats2half2_rn(a[2], a[3]);
            o32[2 * j] = *reinterpret_cast<uint32_t*>(&h0);
            o32[2 * j + 1] = *reinterpret_cast<uint32_t*>(&h1);
        }
    }
    return out;
}

// ------------------------------------------------------------------ packed fp32x2 helpers
// sm_100 executes `fma.rn.f32x2` / `mul.rn.f32x2` as one FFMA2 / FMUL2 instruction on a
// register pair; each lane of the pair is rounded exactly like the scalar op.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
// c + w * v, w broadcast to both lanes
__device__ __forceinline__ unsigned long long fma2s(float w, unsigned long long v, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(w, w)), "l"(v), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long h2_to_f2(uint32_t h) {
    const __half2 v = *reinterpret_cast<const __half2*>(&h);
    return pk2(__low2float(v), __high2float(v));
}

// Mixed-precision blend step (FHFMA): a0 += w * v.lo, a1 += w * v.hi with w the low (SEL = 0)
// or high (SEL = 1) fp16 of w2, fp32 accumulation; no half -> float conversions.
template <int SEL>
__device__ __forceinline__ void fhfma2(uint32_t w2, uint32_t v, float& a0, float& a1) {
    if constexpr (SEL == 0)
        asm("{.reg .f16 w, x, vl, vh; mov.b32 {w, x}, %2; mov.b32 {vl, vh}, %3;\n"
            "fma.rn.f32.f16 %0, w, vl, %0; fma.rn.f32.f16 %1, w, vh, %1;}"
            : "+f"(a0), "+f"(a1) : "r"(w2), "r"(v));
    else
        asm("{.reg .f16 w, x, vl, vh; mov.b32 {x, w}, %2; mov.b32 {vl, vh}, %3;\n"
            "fma.rn.f32.f16 %0, w, vl, %0; fma.rn.f32.f16 %1, w, vh, %1;}"
            : "+f"(a0), "+f"(a1) : "r"(w2), "r"(v));
}
// (lo, hi) fp32 -> fp16x2, round to nearest
__device__ __forceinline__ uint32_t f2_to_h2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t f2_to_bf2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// the MLP operand type of the query path: fp16 (default) or bf16 (nbvh_config.mlp_dtype = 1)
template <bool kBf>
__device__ __forceinline__ uint32_t f2_to_x2(float lo, float hi) {
    if constexpr (kBf) return f2_to_bf2(lo, hi);
    else return f2_to_h2(lo, hi);
}

// ------------------------------------------------------------------ level table in shared memory
// The fp16 *inference* table keeps hashed levels in the parameter layout (T entries of F
// halves) but stores every dense level corner-packed: cell c = x + N*y + N^2*z holds its 8
// corner entries (corner bit0 = x, bit1 = y, bit2 = z) contiguously, 16*F bytes, so one
// dense (point, level) lookup is ONE 32-byte sector (F=2: one 256-bit load) instead of 8
// scattered 4-byte gathers.  It is a re-layout of the same parameters (rebuilt from the
// fp32 master after every update, k_refresh_table), not a different model.
// One 32-byte record per level: the first 16 bytes are what the encode reads (one
// broadcast LDS.128 per level: all lanes of a warp encode the same level at once), the
// second 16 bytes the canonical layout (training scatter, parity hooks).
struct LevelSm {
    float resf;          // N_l as float (exact: N_l < 2^24)
    uint32_t off;        // entry offset of the level in the inference table
    uint32_t nx, nxy;    // dense: N, N^2 (packed-cell index); hashed: 0, 0
    uint32_t coff;       // canonical entry offset (gradient / parameter layout)
    uint32_t n1, n1sq;   // dense: N+1, (N+1)^2 (canonical vertex index, C2); hashed: 0, 0
    float tops;          // 2^23 + N - 1 (exact): the cell clamp of cell_coord
};

// Stage the level table from the kernel parameter block with compile-time indices only
// (a runtime index into a by-value parameter array makes ptxas copy the whole block to
// local memory).
__device__ __forceinline__ void stage_levels(const GridDev& g, LevelSm* lv, int tid) {
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) {
        if (tid == l && l < g.L) {
            const uint32_t N = (uint32_t)g.res[l], n1 = N + 1u;
            const bool dn = g.dense[l] != 0;
            lv[l].resf = (float)g.res[l];
            lv[l].off = g.inf_offset[l];
            lv[l].nx = dn ? N : 0u;
            lv[l].nxy = dn ? N * N : 0u;
            lv[l].coff = g.offset[l];
            lv[l].n1 = dn ? n1 : 0u;
            lv[l].n1sq = dn ? n1 * n1 : 0u;
            lv[l].tops = __fadd_rn((float)g.res[l], 8388607.0f);
        }
    }
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256)
// Table gathers carry L1::evict_last: the tables are the data worth keeping in L1 (the
// read-once streams are loaded evict-first).  Without L1 allocation the hashed gathers lose
// their L1 hits (1522 vs 1686 Mrays/s, profiles/NOTES.md).
template <typename E>
__device__ __forceinline__ E ldg_el(const E* p);
template <>
__device__ __forceinline__ uint32_t ldg_el<uint32_t>(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::evict_last.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <>
__device__ __forceinline__ uint2 ldg_el<uint2>(const uint2* p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::evict_last.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.L1::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}

// Cell coordinate c = min(floor(s), N-1) of s in [0, 2^23) and its integer value without
// the XU pipe: adding 2^23 with round-toward-minus-infinity leaves floor(s) in the low
// mantissa bits (exact); the clamp to N-1 is applied in that shifted domain (tops =
// 2^23 + N-1, exact), so the cell costs FADD.RM + FMNMX + FADD + one integer subtract
// instead of FRND + F2I + clamps.
__device__ __forceinline__ float cell_coord(float s, float tops, uint32_t& i) {
    const float t = fminf(__fadd_rd(s, 8388608.0f), tops);
    i = (uint32_t)(__float_as_int(t) - 0x4B000000);
    return __fsub_rn(t, 8388608.0f);
}

// Cell of one level from the shared-memory level record: corner indices within the level
// and trilinear weights (same arithmetic as encode_chunk_sm).  Used by the training
// backward scatter.
// (i0, i1, i2) receives the cell's integer coordinates.
__device__ __forceinline__ void level_cell_sm(const LevelSm& P, uint32_t hmask, float x0, float x1, float x2,
                                              Cell& c, uint32_t& i0, uint32_t& i1, uint32_t& i2) {
    const float s0 = __fmul_rn(x0, P.resf), s1 = __fmul_rn(x1, P.resf), s2 = __fmul_rn(x2, P.resf);
    const float tops = P.tops;                              // 2^23 + N - 1 (exact)
    const float c0 = cell_coord(s0, tops, i0), c1 = cell_coord(s1, tops, i1), c2 = cell_coord(s2, tops, i2);
    const float f0 = __fsub_rn(s0, c0), f1 = __fsub_rn(s1, c1), f2 = __fsub_rn(s2, c2);
    if (P.n1) {   // canonical dense vertex index (C2)
        const uint32_t b = i0 + i1 * P.n1 + i2 * P.n1sq;
#pragma unroll
        for (int k = 0; k < 8; ++k) c.idx[k] = b + (k & 1) + ((k >> 1) & 1) * P.n1 + ((k >> 2) & 1) * P.n1sq;
    } else {
        const uint32_t hx[2] = {i0 & hmask, (i0 + 1u) & hmask};
        const uint32_t hy[2] = {(i1 * kPrime1) & hmask, ((i1 + 1u) * kPrime1) & hmask};
        const uint32_t hz[2] = {(i2 * kPrime2) & hmask, ((i2 + 1u) * kPrime2) & hmask};
#pragma unroll
        for (int k = 0; k < 8; ++k) c.idx[k] = hx[k & 1] ^ hy[(k >> 1) & 1] ^ hz[(k >> 2) & 1];
    }
    const float wx[2] = {1.0f - f0, f0}, wy[2] = {1.0f - f1, f1}, wz[2] = {1.0f - f2, f2};
#pragma unroll
    for (int k = 0; k < 8; ++k) c.w[k] = wx[k & 1] * wy[(k >> 1) & 1] * wz[(k >> 2) & 1];
}
__device__ __forceinline__ void level_cell_sm(const LevelSm& P, uint32_t hmask, float x0, float x1, float x2,
                                              Cell& c) {
    uint32_t i0, i1, i2;
    level_cell_sm(P, hmask, x0, x1, x2, c, i0, i1, i2);
}

// In-flight state of one 16-byte chunk: the gathered corner entries and the cell fractions.
template <int F>
struct ChunkGather {
    using Entry = typename std::conditional<F == 2, uint32_t, uint2>::type;
    Entry v[8 / F][8];
    float fr[8 / F][3];
};

// Step 1 of encode_chunk_sm: cell, corner indices and all 8*NL gathers issued (the index
// registers die as soon as the loads are issued; only the fractions are kept).  Splitting
// issue from finish lets the caller keep two chunks' gathers in flight.
template <int F, bool kTex = false>
__device__ __forceinline__ void encode_issue(const LevelSm* lv, const void* tab, uint32_t hmask, float x0, float x1,
                                             float x2, int l0, uint32_t* idx_out, ChunkGather<F>& G,
                                             unsigned long long tex = 0) {
    constexpr int NL = 8 / F;
    static_assert(F == 2 || F == 4, "F must be 2 or 4");
    using Entry = typename ChunkGather<F>::Entry;
    const Entry* T = reinterpret_cast<const Entry*>(tab);
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        const LevelSm P = lv[l0 + j];
        const float s0 = __fmul_rn(x0, P.resf), s1 = __fmul_rn(x1, P.resf), s2 = __fmul_rn(x2, P.resf);
        const float tops = P.tops;                          // 2^23 + N - 1 (exact)
        uint32_t i0, i1, i2;
        const float c0 = cell_coord(s0, tops, i0), c1 = cell_coord(s1, tops, i1), c2 = cell_coord(s2, tops, i2);
        G.fr[j][0] = __fsub_rn(s0, c0);
        G.fr[j][1] = __fsub_rn(s1, c1);
        G.fr[j][2] = __fsub_rn(s2, c2);
        if (idx_out) {   // parity hook: canonical corner indices within the level
            if (P.nx) {
                const uint32_t b = i0 + i1 * P.n1 + i2 * P.n1sq;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    idx_out[j * 8 + k] = b + (k & 1) + ((k >> 1) & 1) * P.n1 + ((k >> 2) & 1) * P.n1sq;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    idx_out[j * 8 + k] = ((i0 + (k & 1)) ^ ((i1 + ((k >> 1) & 1)) * kPrime1) ^
                                          ((i2 + ((k >> 2) & 1)) * kPrime2)) & hmask;
            }
        }
        // the level's base pointer once per level: per corner one IMAD.WIDE.U32 (index * entry +
        // base), no 32-bit offset add
        const Entry* Tl = T + P.off;
        if (P.nx) {
            // dense level: the cell's 8 corners are one contiguous 16*F-byte record
            NBVH_DCHECK(i0 < P.nx && i1 < P.nx && i2 < P.nx);
            const uint32_t cell = i0 + i1 * P.nx + i2 * P.nxy;
            if constexpr (F == 2) {
                ldg256(Tl + 8u * cell, G.v[j]);
            } else {
                uint32_t lo[8], hi[8];
                ldg256(Tl + 8u * cell, lo);
                ldg256(Tl + 8u * cell + 4u, hi);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    G.v[j][k] = make_uint2(lo[2 * k], lo[2 * k + 1]);
                    G.v[j][4 + k] = make_uint2(hi[2 * k], hi[2 * k + 1]);
                }
            }
        } else {
            // hashed level (C3): (x*1 ^ y*pi2 ^ z*pi3) mod T, masks distributed; the
            // x term needs no mask: x+1 <= N < T on every hashed level (checked at creation)
            NBVH_DCHECK(i0 + 1u <= hmask);     // unmasked x term stays inside the level
            const uint32_t hx[2] = {i0, i0 + 1u};
            const uint32_t hy[2] = {(i1 * kPrime1) & hmask, ((i1 + 1u) * kPrime1) & hmask};
            const uint32_t hz[2] = {(i2 * kPrime2) & hmask, ((i2 + 1u) * kPrime2) & hmask};
            // 32-bit entry index (n_entries < 2^32), one IMAD.WIDE.U32 per gather address
            if constexpr (kTex && F == 2) {
                // through the TEX pipe (a texture object over the same fp16 table, element
                // reads): the query kernel's limit is the LSU data pipe, which the TEX pipe
                // does not share -- the dense levels' 32-byte records stay on LDG.256
                // hashed levels are T-aligned in the inference layout (off + h = off | h), so
                // the offset folds into the z term: one 3-input XOR per corner address
                NBVH_DCHECK((P.off & hmask) == 0u);
                const uint32_t hzo[2] = {hz[0] | P.off, hz[1] | P.off};
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    G.v[j][k] = tex1Dfetch<unsigned int>(
                        (cudaTextureObject_t)tex, (int)(hx[k & 1] ^ hy[(k >> 1) & 1] ^ hzo[(k >> 2) & 1]));
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    G.v[j][k] = ldg_el(Tl + (hx[k & 1] ^ hy[(k >> 1) & 1] ^ hz[(k >> 2) & 1]));
            }
        }
    }
}

// Step 2: trilinear weights (wx*wy)*wz and the blend with fp32 accumulation, level by level
// -> 8 halves.  kHalfW (inference): weights rounded once to fp16 (relative error <= 2^-12,
// DESIGN.md reading R-blend) so each corner is two mixed-precision FMAs (FHFMA) with no
// half -> float conversions; otherwise (training forward, whose features feed the
// gradients) fp32 weights and converted entries.
template <int F, bool kHalfW, bool kBf = false>
__device__ __forceinline__ uint4 encode_finish(const ChunkGather<F>& G) {
    constexpr int NL = 8 / F;
    uint4 out;
    uint32_t* o32 = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        const float f0 = G.fr[j][0], f1 = G.fr[j][1], f2 = G.fr[j][2];
        const unsigned long long wx = pk2(1.0f - f0, f0);
        const unsigned long long wxy0 = mul2(wx, pk2(1.0f - f1, 1.0f - f1));
        const unsigned long long wxy1 = mul2(wx, pk2(f1, f1));
        const unsigned long long wz0 = pk2(1.0f - f2, 1.0f - f2), wz1 = pk2(f2, f2);
        const unsigned long long wp[4] = {mul2(wxy0, wz0), mul2(wxy1, wz0), mul2(wxy0, wz1), mul2(wxy1, wz1)};
        if constexpr (kHalfW) {
            uint32_t wh[4];   // corner weights k = 2i, 2i+1 as fp16x2
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 t = upk2(wp[i]);
                wh[i] = f2_to_h2(t.x, t.y);
            }
            if constexpr (F == 2) {
                float a0 = 0.f, a1 = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    fhfma2<0>(wh[i], G.v[j][2 * i], a0, a1);
                    fhfma2<1>(wh[i], G.v[j][2 * i + 1], a0, a1);
                }
                o32[j] = f2_to_x2<kBf>(a0, a1);
            } else {
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    fhfma2<0>(wh[i], G.v[j][2 * i].x, a0, a1);
                    fhfma2<0>(wh[i], G.v[j][2 * i].y, a2, a3);
                    fhfma2<1>(wh[i], G.v[j][2 * i + 1].x, a0, a1);
                    fhfma2<1>(wh[i], G.v[j][2 * i + 1].y, a2, a3);
                }
                o32[2 * j] = f2_to_x2<kBf>(a0, a1);
                o32[2 * j + 1] = f2_to_x2<kBf>(a2, a3);
            }
        } else {
            float w[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 t = upk2(wp[i]);
                w[2 * i] = t.x;
                w[2 * i + 1] = t.y;
            }
            if constexpr (F == 2) {
                unsigned long long acc = 0ull;   // (+0, +0)
#pragma unroll
                for (int k = 0; k < 8; ++k) acc = fma2s(w[k], h2_to_f2(G.v[j][k]), acc);
                const float2 a = upk2(acc);
                o32[j] = f2_to_h2(a.x, a.y);
            } else {
                unsigned long long a01 = 0ull, a23 = 0ull;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a01 = fma2s(w[k], h2_to_f2(G.v[j][k].x), a01);
                    a23 = fma2s(w[k], h2_to_f2(G.v[j][k].y), a23);
                }
                const float2 p = upk2(a01), q = upk2(a23);
                o32[2 * j] = f2_to_h2(p.x, p.y);
                o32[2 * j + 1] = f2_to_h2(q.x, q.y);
            }
        }
    }
    return out;
}

// Encode NL = 8/F consecutive levels l0.. of one point x (normalised, in [0,1]^3) into
// 16 bytes of fp16 features: s = x*N, c = min(floor(s), N-1), f = s - c (exact), corner
// entries (dense: corner-packed cell record; hashed: 8 gathers, C2, C3), trilinear weights
// (wx*wy)*wz, blend in fp32.  idx_out (nullable) receives the 8*NL
// canonical corner indices within their levels (parity hook).
template <int F, bool kHalfW = true, bool kBf = false, bool kTex = false>
__device__ __forceinline__ uint4 encode_chunk_sm(const LevelSm* lv, const void* tab, uint32_t hmask, float x0,
                                                 float x1, float x2, int l0, uint32_t* idx_out,
                                                 unsigned long long tex = 0) {
    ChunkGather<F> G;
    encode_issue<F, kTex>(lv, tab, hmask, x0, x1, x2, l0, idx_out, G, tex);
    return encode_finish<F, kHalfW, kBf>(G);
}

// ------------------------------------------------------------------ tensor-core MLP
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_relu_half2(float a, float b) {
    __half2 h = __floats2half2_rn(fmaxf(a, 0.f), fmaxf(b, 0.f));
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma16816_bf(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <bool kBf>
__device__ __forceinline__ void mma16816x(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    if constexpr (kBf) mma16816_bf(c, a, b0, b1);
    else mma16816(c, a, b0, b1);
}
template <bool kBf>
__device__ __forceinline__ uint32_t pack_relu_x2(float a, float b) {
    // ReLU fused into the conversion (cvt .relu: one instruction instead of two max + cvt);
    // identical values -- max(x, 0) commutes with round-to-nearest
    uint32_t r;
    if constexpr (kBf) asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    else asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

// Shared-memory layout of the staged MLP (row strides padded by 8 halves so that the
// 8-row ldmatrix phases hit 8 distinct 16-byte bank groups).
struct MlpSmem {
    __half* w0;      // [64][d_in + 8]
    __half* wh;      // [hidden-1][64][72]
    __half* wo;      // [8][72]
    float* b;        // [64*hidden + 8]
};

__host__ __device__ constexpr int mlp_smem_halves(int d_in, int hidden) {
    return 64 * (d_in + 8) + (hidden - 1) * 64 * 72 + 8 * 72;
}

// Stage weights and biases from global memory (16-byte copies by all threads).
__device__ __forceinline__ void stage_mlp(const MlpDev& m, const MlpSmem& s, int tid, int nthreads) {
    const int D = m.d_in, cpr0 = D / 8;
    const uint4* W = reinterpret_cast<const uint4*>(m.W);
    for (int i = tid; i < 64 * cpr0; i += nthreads) {
        int row = i / cpr0, c = i % cpr0;
        *reinterpret_cast<uint4*>(s.w0 + row * (D + 8) + c * 8) = __ldg(W + i);
    }
    const uint4* Wh = W + 64 * cpr0;
    for (int i = tid; i < (m.hidden - 1) * 64 * 8; i += nthreads) {
        int row = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(s.wh + row * 72 + c * 8) = __ldg(Wh + i);
    }
    const uint4* Wo = Wh + (m.hidden - 1) * 64 * 8;
    for (int i = tid; i < 8 * 8; i += nthreads) {
        int row = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(s.wo + row * 72 + c * 8) = __ldg(Wo + i);
    }
    for (int i = tid; i < 64 * m.hidden + 8; i += nthreads) s.b[i] = __ldg(m.b + i);
}

// MLP of the 16 rows [r0, r0+16) of a feature tile x (row stride d_in+8 halves) on
// mma.sync m16n8k16 (fp16 in, fp32 accumulate).  Layer outputs stay in registers: the
// m16n8 accumulator layout of two adjacent n-tiles is exactly the m16k16 A-operand
// layout of the next layer.  Writes the 8 raw outputs of each row to z[row*8 + c].
template <int D, bool kBf = false>
__device__ __forceinline__ void mlp_rows16(const MlpSmem& s, int hidden, const __half* x, int r0, float* z, int lane) {
    const int g = lane >> 2, t = lane & 3;
    float acc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        float b0 = s.b[nt * 8 + 2 * t], b1 = s.b[nt * 8 + 2 * t + 1];
        acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
    }
    const uint32_t xa = (uint32_t)__cvta_generic_to_shared(x + (r0 + (lane & 15)) * (D + 8) + (lane >> 4) * 8);
    const uint32_t wa = (uint32_t)__cvta_generic_to_shared(s.w0 + ((lane & 7) + ((lane >> 4) << 3)) * (D + 8) +
                                                           ((lane >> 3) & 1) * 8);
#pragma unroll
    for (int kb = 0; kb < D / 16; ++kb) {
        uint32_t a[4];
        ldsm_x4(xa + kb * 32, a[0], a[1], a[2], a[3]);
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(wa + np * 16 * (D + 8) * 2 + kb * 32, b0, b1, b2, b3);
            mma16816x<kBf>(acc[2 * np], a, b0, b1);
            mma16816x<kBf>(acc[2 * np + 1], a, b2, b3);
        }
    }
    uint32_t h[4][4];   // next-layer A fragments, k-block kb = hidden units 16kb..16kb+15
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
        h[kb][0] = pack_relu_x2<kBf>(acc[2 * kb][0], acc[2 * kb][1]);
        h[kb][1] = pack_relu_x2<kBf>(acc[2 * kb][2], acc[2 * kb][3]);
        h[kb][2] = pack_relu_x2<kBf>(acc[2 * kb + 1][0], acc[2 * kb + 1][1]);
        h[kb][3] = pack_relu_x2<kBf>(acc[2 * kb + 1][2], acc[2 * kb + 1][3]);
    }
    for (int layer = 1; layer < hidden; ++layer) {
        const __half* W = s.wh + (layer - 1) * 64 * 72;
        const float* bb = s.b + layer * 64;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            float b0 = bb[nt * 8 + 2 * t], b1 = bb[nt * 8 + 2 * t + 1];
            acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
        }
        const uint32_t wb = (uint32_t)__cvta_generic_to_shared(W + ((lane & 7) + ((lane >> 4) << 3)) * 72 +
                                                               ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(wb + np * 16 * 72 * 2 + kb * 32, b0, b1, b2, b3);
                mma16816x<kBf>(acc[2 * np], h[kb], b0, b1);
                mma16816x<kBf>(acc[2 * np + 1], h[kb], b2, b3);
            }
        }
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
            h[kb][0] = pack_relu_x2<kBf>(acc[2 * kb][0], acc[2 * kb][1]);
            h[kb][1] = pack_relu_x2<kBf>(acc[2 * kb][2], acc[2 * kb][3]);
            h[kb][2] = pack_relu_x2<kBf>(acc[2 * kb + 1][0], acc[2 * kb + 1][1]);
            h[kb][3] = pack_relu_x2<kBf>(acc[2 * kb + 1][2], acc[2 * kb + 1][3]);
        }
    }
    // output layer: 64 -> 8, linear
    float o[4];
    {
        // read here (volatile) rather than hoisted above the hidden layers, where the pair
        // would be held -- or spilled -- across them
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                     : "=f"(o[0]), "=f"(o[1])
                     : "r"((uint32_t)__cvta_generic_to_shared(s.b + hidden * 64 + 2 * t)));
        o[2] = o[0];
        o[3] = o[1];
    }
    const uint32_t wo = (uint32_t)__cvta_generic_to_shared(s.wo + (lane & 7) * 72 + ((lane >> 3) & 1) * 8);
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
        uint32_t b0, b1;
        ldsm_x2(wo + kb * 32, b0, b1);
        mma16816x<kBf>(o, h[kb], b0, b1);
    }
    z[(r0 + g) * 8 + 2 * t] = o[0];
    z[(r0 + g) * 8 + 2 * t + 1] = o[1];
    z[(r0 + g + 8) * 8 + 2 * t] = o[2];
    z[(r0 + g + 8) * 8 + 2 * t + 1] = o[3];
}

// fp16-accumulating m16n8k16 (the accumulator is two f16x2 registers: rows g and g+8,
// columns 2t, 2t+1) -- the precision tiny-cuda-nn's fully fused MLP uses (C34)
__device__ __forceinline__ void mma16816h(uint32_t (&c)[2], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};\n"
        : "+r"(c[0]), "+r"(c[1])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ uint32_t relu_h2(uint32_t v) {
    return h2_bits(__hmax2(*reinterpret_cast<__half2*>(&v), __float2half2_rn(0.f)));
}

// mlp_rows16 with fp16 accumulation: half the accumulator registers, the next layer's A
// fragment is the accumulator itself after ReLU.
template <int D>
__device__ __forceinline__ void mlp_rows16h(const MlpSmem& s, int hidden, const __half* x, int r0, float* z, int lane) {
    const int g = lane >> 2, t = lane & 3;
    uint32_t acc[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        const uint32_t b = h2_bits(__floats2half2_rn(s.b[nt * 8 + 2 * t], s.b[nt * 8 + 2 * t + 1]));
        acc[nt][0] = b;
        acc[nt][1] = b;
    }
    const uint32_t xa = (uint32_t)__cvta_generic_to_shared(x + (r0 + (lane & 15)) * (D + 8) + (lane >> 4) * 8);
    const uint32_t wa = (uint32_t)__cvta_generic_to_shared(s.w0 + ((lane & 7) + ((lane >> 4) << 3)) * (D + 8) +
                                                           ((lane >> 3) & 1) * 8);
#pragma unroll
    for (int kb = 0; kb < D / 16; ++kb) {
        uint32_t a[4];
        ldsm_x4(xa + kb * 32, a[0], a[1], a[2], a[3]);
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t b0, b1, b2, b3;
            ldsm_x4(wa + np * 16 * (D + 8) * 2 + kb * 32, b0, b1, b2, b3);
            mma16816h(acc[2 * np], a, b0, b1);
            mma16816h(acc[2 * np + 1], a, b2, b3);
        }
    }
    uint32_t h[4][4];
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
        h[kb][0] = relu_h2(acc[2 * kb][0]);
        h[kb][1] = relu_h2(acc[2 * kb][1]);
        h[kb][2] = relu_h2(acc[2 * kb + 1][0]);
        h[kb][3] = relu_h2(acc[2 * kb + 1][1]);
    }
    for (int layer = 1; layer < hidden; ++layer) {
        const __half* W = s.wh + (layer - 1) * 64 * 72;
        const float* bb = s.b + layer * 64;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const uint32_t b = h2_bits(__floats2half2_rn(bb[nt * 8 + 2 * t], bb[nt * 8 + 2 * t + 1]));
            acc[nt][0] = b;
            acc[nt][1] = b;
        }
        const uint32_t wb = (uint32_t)__cvta_generic_to_shared(W + ((lane & 7) + ((lane >> 4) << 3)) * 72 +
                                                               ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
            for (int np = 0; np < 4; ++np) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(wb + np * 16 * 72 * 2 + kb * 32, b0, b1, b2, b3);
                mma16816h(acc[2 * np], h[kb], b0, b1);
                mma16816h(acc[2 * np + 1], h[kb], b2, b3);
            }
        }
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
            h[kb][0] = relu_h2(acc[2 * kb][0]);
            h[kb][1] = relu_h2(acc[2 * kb][1]);
            h[kb][2] = relu_h2(acc[2 * kb + 1][0]);
            h[kb][3] = relu_h2(acc[2 * kb + 1][1]);
        }
    }
    // output layer: 64 -> 8, linear; fp32 accumulation for the outputs
    float o[4];
    {
        const float* bb = s.b + hidden * 64;
        o[0] = bb[2 * t]; o[1] = bb[2 * t + 1]; o[2] = o[0]; o[3] = o[1];
    }
    const uint32_t wo = (uint32_t)__cvta_generic_to_shared(s.wo + (lane & 7) * 72 + ((lane >> 3) & 1) * 8);
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
        uint32_t b0, b1;
        ldsm_x2(wo + kb * 32, b0, b1);
        mma16816(o, h[kb], b0, b1);
    }
    z[(r0 + g) * 8 + 2 * t] = o[0];
    z[(r0 + g) * 8 + 2 * t + 1] = o[1];
    z[(r0 + g + 8) * 8 + 2 * t] = o[2];
    z[(r0 + g + 8) * 8 + 2 * t + 1] = o[3];
}

// ------------------------------------------------------------------ decode
// sigmoid in fp32 from correctly rounded operations only (C27), so the host's
// logic replay reproduces it bit for bit: e^x by x = n ln2 + r (two fmas), a degree-7
// Taylor polynomial of e^r (|r| <= 0.35), exact scaling by 2^n, then 1 / (1 + e^-z).
__device__ __forceinline__ float sigmoid_f(float z) {
    const float x = fminf(fmaxf(-z, -87.0f), 87.0f);
    const float n = rintf(__fmul_rn(x, 1.44269504f));
    float r = __fmaf_rn(-n, 0.693145751953125f, x);
    r = __fmaf_rn(-n, 1.42860677e-6f, r);
    float p = 1.98412698e-4f;
    p = __fmaf_rn(p, r, 1.38888889e-3f);
    p = __fmaf_rn(p, r, 8.33333333e-3f);
    p = __fmaf_rn(p, r, 4.16666667e-2f);
    p = __fmaf_rn(p, r, 1.66666667e-1f);
    p = __fmaf_rn(p, r, 0.5f);
    p = __fmaf_rn(p, r, 1.0f);
    p = __fmaf_rn(p, r, 1.0f);
    const float e = __fmul_rn(p, __int_as_float(((int)n + 127) << 23));
    return __fdiv_rn(1.0f, __fadd_rn(1.0f, e));
}

}  // namespace nbvh
