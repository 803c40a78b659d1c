// nbvh_train_kernels.cuh — device code of the companion training step (P:142, P:193-247,
// P:275):
//   k_train_select   T1  first intersected cut leaf + stochastic acceptance (C18)
//   k_train_label    T2  ground truth by intersecting the leaf's own triangles (C17)
//   k_train_fwd      T3-T5 jittered encode, MLP forward (activations kept), gated loss + dL/dz
//   k_train_bwd      T6/T7 delta chain through the MLP on tensor cores, dL/dx, hash-grid
//                    gradient scatter with warp-aggregated atomics
//   k_train_dw       T6  weight gradients dW = delta^T x as split-K tensor-core GEMMs
//   k_adam           T9  Adam (C20) + fp16 inference-copy refresh
#pragma once

#include <cuda_fp16.h>

#include "nbvh_device.cuh"
#include "nbvh_internal.h"
#include "nbvh_tcgen05.cuh"
#include "nbvh_bvh.cuh"

namespace nbvh {

struct TrainArgs {
    GridDev g;
    MlpDev m;
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    const float* u;          // [n] acceptance draws
    const float* xi;         // [n][n_points] jitter
    const float* rank;       // [n_leaves]
    float rank_min, rank_hmax;   // fp32: min rank, (max-min)+eps (C18)
    const int32_t* leaf_base;
    const BvhNode* nodes;
    int32_t bvh_rows;        // closest-hit stack rows (>= base-BVH depth)
    const float* tri_v;
    const float* tri_n;
    const float* tri_a;
    const int32_t* tri_id;
    // per ray (debug / stats)
    uint8_t* r_acc;
    int32_t* r_leaf;
    float* r_gt;             // [n][9]
    float* r_loss;
    // per sample (compact)
    int32_t* n_samples;      // device counter
    int32_t* n_first;        // device counter
    int32_t* s_ray;
    int32_t* s_leaf;
    float* s_t0;
    float* s_t1;
    float* s_gt;             // [M][9]
    __half* X;               // [M][D]
    __half* A;               // [hidden][M][64] post-ReLU activations
    __half* Dl;              // [hidden][M][64] deltas dL/d(pre-activation)
    float* dZ;               // [M][8]
    float* Z;                // [M][8] raw MLP outputs (nullable: parity capture only)
    // outputs
    float* grad;             // flat fp32: tables, weights, biases, tail
    float* tail;             // [0] accepted count, [1 + 3*leaf + {0,1,2}] loss sum, samples, first hits
    double* loss_acc;        // [5]: total, vis, dist, normal, albedo (weights applied)
    int64_t cap;             // capacity of the per-sample arrays
    int32_t priv_levels;     // coarse levels accumulated in shared memory by k_train_scatter
    int32_t priv_floats;     // their gradient floats (levels 0..priv_levels-1 are a prefix)
    float* gx;               // [cap][D] fp32 dL/dx per sample (k_train_bwd -> k_train_scatter)
    unsigned long long tex_gx;   // texture object over gx (float2 texels; 0: read with loads)
    float* sc_dense;         // T7 scratch of the global dense levels: cell-packed, 8 corners x F
    float* sc_hash;          // T7 scratch of the hashed levels: [T][F], 16-byte aligned per level
    int32_t* sc_priv;        // [scatter CTAs][priv_floats] fixed-point partial sums
    int64_t sc_off[kMaxLevels];   // float offset of a level's scratch (dense: in sc_dense; hashed: in sc_hash)
    int64_t sc_dense_n, sc_hash_n;   // scratch sizes (floats)
    int64_t hash_coff0;              // canonical entry offset of the first hashed level when the hashed
                                     // levels are one contiguous range in both layouts (else -1)
    int64_t hash_floats;             // floats of that range (a multiple of 4)
    int32_t scatter_ctas;
    int32_t agg_levels;      // k_train_scatter_agg: levels 0..agg_levels-1 warp-aggregated (0: k_train_scatter)
    int32_t* leaf_hist;      // k_train_select: accepted samples per leaf (nullable; the sort's counts)
    int32_t use_tc_dw;       // weight GEMMs on tcgen05 (k_train_dw_tc) when the shape allows
};

// ------------------------------------------------------------------ T1 select
__global__ void __launch_bounds__(128) k_train_select(TrainArgs a) {
    extern __shared__ int stk_raw[];        // traversal stack [depth+2][128]
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool acc = false;
    int leaf = -1;
    float te = 0.f, tx = 0.f;
    if (r < a.n_rays) {
        RayDev R = load_ray(a.rays, r);
        float lte[1], ltx[1];
        int lid[1], n = 0;
        SmemStack st{stk_raw + threadIdx.x, (int)blockDim.x, a.cut.depth + 2};
        // first leaf in (t_enter, id) order; the list of 1 prunes every subtree entering later
        int total = collect_leaves<1, SmemStack>(a.cut, R, false, 0.f, 0, 1, lte, ltx, lid, n, nullptr, st, true);
        if (total > 0) {
            leaf = lid[0];
            te = lte[0];
            tx = ltx[0];
            atomicAdd(a.n_first, 1);
            atomicAdd(a.tail + 1 + 3 * leaf + 2, 1.0f);
            // trained with probability max(r/r_max, 0.005) on shifted ranks (C18)
            const float rh = __fadd_rn(__fsub_rn(a.rank[leaf], a.rank_min), 1e-6f);
            const float p = fmaxf(__fdiv_rn(rh, a.rank_hmax), 0.005f);
            acc = a.u[r] < p;
            if (acc && a.leaf_hist) atomicAdd(a.leaf_hist + leaf, 1);
        }
        a.r_acc[r] = acc ? 1 : 0;
        a.r_leaf[r] = leaf;
        a.r_loss[r] = 0.f;
#pragma unroll
        for (int k = 0; k < 9; ++k) a.r_gt[9 * r + k] = 0.f;
    }
    const unsigned m = __ballot_sync(0xffffffffu, acc);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(a.n_samples, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (acc) {
        const int i = base + __popc(m & ((1u << lane) - 1u));
        a.s_ray[i] = (int)r;
        a.s_leaf[i] = leaf;
        a.s_t0[i] = te;
        a.s_t1[i] = tx;
    }
}

// ------------------------------------------------------------------ T2 label
// Ground truth by intersecting the first leaf's own triangles (C17): closest
// hit below the leaf's base-BVH node within the leaf segment [t0, t1] (bvh_closest, double
// Moller-Trumbore with the oracle's operation order).
__global__ void __launch_bounds__(128) k_train_label(TrainArgs a) {
    const int M = *a.n_samples;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int r = a.s_ray[i];
    RayDev R = load_ray(a.rays, r);
    const float t0 = a.s_t0[i], t1 = a.s_t1[i];
    extern __shared__ int stk_raw[];                     // stack column [bvh_rows][128]
    const BvhHit h = bvh_closest(a.nodes, a.tri_v, a.tri_id, a.leaf_base[a.s_leaf[i]], R, t0, t1,
                                 stk_raw + threadIdx.x, 128, a.bvh_rows);
    float gt[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) gt[k] = 0.f;
    gt[0] = h.found ? 0.f : 1.f;
    if (h.found) {
        const double dt = (double)t1 - (double)t0;
        gt[1] = dt > 0.0 ? (float)((h.t - (double)t0) / dt) : 0.f;
        float n[3];
        shading_normal(a.tri_n, h, n);
        for (int k = 0; k < 3; ++k) gt[2 + k] = n[k];
        for (int k = 0; k < 3; ++k) gt[5 + k] = a.tri_a[3 * (int64_t)h.slot + k];
        gt[8] = (float)h.t;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        a.s_gt[9 * (int64_t)i + k] = gt[k];
        a.r_gt[9 * (int64_t)r + k] = gt[k];
    }
}

// ------------------------------------------------------------------ shared tile helpers
struct SampleDesc {
    float o[3], d[3], t0, t1;
    float xi[4];
    int ray, leaf, valid, pad;
};

__device__ __forceinline__ void load_sample_desc(const TrainArgs& a, int i, int M, SampleDesc& q) {
    q.valid = i < M;
    if (!q.valid) return;
    const int r = a.s_ray[i];
    q.ray = r;
    q.leaf = a.s_leaf[i];
    q.t0 = a.s_t0[i];
    q.t1 = a.s_t1[i];
    float4 r0 = __ldg(a.rays + 2 * (int64_t)r), r1 = __ldg(a.rays + 2 * (int64_t)r + 1);
    q.o[0] = r0.x; q.o[1] = r0.y; q.o[2] = r0.z;
    q.d[0] = r1.x; q.d[1] = r1.y; q.d[2] = r1.z;
    for (int k = 0; k < a.g.n_points && k < 4; ++k) q.xi[k] = a.xi[(int64_t)r * a.g.n_points + k];
}

__device__ __forceinline__ float sigm(float z) { return 1.0f / (1.0f + __expf(-z)); }
__device__ __forceinline__ float sgnf(float v) { return v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f); }

// Gated weighted loss of one sample and dL/dz (C19).
__device__ __forceinline__ float sample_loss(const float* z, const float* gt, float* terms, float* dz) {
    const float y = gt[0];
    const float lvis = fmaxf(z[0], 0.f) - z[0] * y + log1pf(__expf(-fabsf(z[0])));
    const float g = y == 0.f ? 1.f : 0.f;
    const float st = sigm(z[1]);
    const float ldist = fabsf(st - gt[1]);
    float lnorm = 0.f, lalb = 0.f;
    dz[0] = 2.f * (sigm(z[0]) - y);
    dz[1] = g * 2.f * sgnf(st - gt[1]) * st * (1.f - st);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float dn = z[2 + k] - gt[2 + k];
        lnorm += fabsf(dn) * (1.f / 3.f);
        dz[2 + k] = g * sgnf(dn) * (1.f / 3.f);
        const float av = sigm(z[5 + k]);
        const float den = av * av + 0.01f;
        const float da = av - gt[5 + k];
        lalb += da * da / den * (1.f / 3.f);
        dz[5 + k] = g * 2.f * da / den * (1.f / 3.f) * av * (1.f - av);
    }
    terms[0] = 2.f * lvis;
    terms[1] = g * 2.f * ldist;
    terms[2] = g * lnorm;
    terms[3] = g * lalb;
    return terms[0] + terms[1] + terms[2] + terms[3];
}

}  // namespace nbvh

namespace nbvh {

// ------------------------------------------------------------------ samples grouped by leaf
// A counting sort of the accepted samples by leaf (a permutation of the batch: every sum over
// samples is unchanged): k_train_select counts them per leaf (TrainArgs::leaf_hist), a scan
// turns the counts into offsets, k_sort_place scatters.  A leaf's samples are spatially close,
// so the warps of the label, forward and backward kernels read coherent lines -- random
// training rays otherwise touch ~3x the L1 sectors per encoded point of a coherent query --
// and the default T7 scatter groups a warp's items by grid cell (k_train_scatter_agg);
// k_train_scatter (NBVH_SCATTER_AGG=0) walks them in a scrambled order instead.

// in-place exclusive scan of hist[n] by one CTA of 1024 threads (chunks of 1024 with a carry)
__global__ void __launch_bounds__(1024) k_sort_scan(int32_t* hist, int n) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + tid;
        const int v = i < n ? hist[i] : 0;
        int x = v;                                             // inclusive scan within the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int w = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;                                    // inclusive over warps
        }
        __syncthreads();
        const int excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
        if (i < n) hist[i] = excl;
        __syncthreads();
        if (tid == 0) carry += wsum[31];
        __syncthreads();
    }
}

struct SortedSamples {
    int32_t* ray;
    int32_t* leaf;
    float* t0;
    float* t1;
};

__global__ void k_sort_place(TrainArgs a, int32_t* offs, SortedSamples o) {
    const int M = *a.n_samples;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
        const int leaf = a.s_leaf[i];
        const int pos = atomicAdd(offs + leaf, 1);
        o.ray[pos] = a.s_ray[i];
        o.leaf[pos] = leaf;
        o.t0[pos] = a.s_t0[i];
        o.t1[pos] = a.s_t1[i];
    }
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void red_add_v2(float* p, float x, float y) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};\n" ::"l"(p), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_half2(uint32_t v) {
    return __half22float2(*reinterpret_cast<const __half2*>(&v));
}

// ------------------------------------------------------------------ T3-T5 forward + loss
// Warp-owned 16-sample blocks, no block-wide barrier after the staging (the query kernel's
// structure): lanes 0-15 fetch the block's segments and jittered points (C8), the two
// half-warps encode neighbouring points of the same 16 samples at the same levels into the
// warp's feature rows (fp32 trilinear weights: the training features feed the gradients),
// the rows go out for the weight gradient of layer 0, the MLP runs on mma.sync with the
// hidden activations written out for the backward pass, then the gated loss and dL/dz per
// sample.
constexpr int kFwdWarps = 16;

struct FwdSmemPlan {
    size_t w, bias, lv, warp0, feat, z, xs, per_warp, total;
    __host__ __device__ FwdSmemPlan(int d_in, int hidden, int n_points) {
        w = 0;
        bias = w + (((size_t)mlp_smem_halves(d_in, hidden) * 2 + 15) & ~(size_t)15);
        lv = bias + (((size_t)(64 * hidden + 8) * 4 + 15) & ~(size_t)15);
        warp0 = lv + ((sizeof(LevelSm) * kMaxLevels + 15) & ~(size_t)15);
        feat = 0;
        z = feat + (((size_t)16 * (d_in + 8) * 2 + 15) & ~(size_t)15);
        xs = z + 16 * 8 * 4;
        per_warp = xs + (((size_t)16 * n_points * 3 * 4 + 15) & ~(size_t)15);
        total = warp0 + per_warp * kFwdWarps;
    }
};

template <int F, int D, bool kTex = false>
__global__ void __launch_bounds__(kFwdWarps * 32, 1) k_train_fwd(TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int M = *a.n_samples;
    const int n_pts = a.g.n_points, L = a.g.L, H = a.m.hidden;
    if ((int64_t)blockIdx.x * kFwdWarps * 16 >= M) return;
    const FwdSmemPlan plan(D, H, n_pts);
    MlpSmem ms;
    ms.w0 = reinterpret_cast<__half*>(smem_raw + plan.w);
    ms.wh = ms.w0 + 64 * (D + 8);
    ms.wo = ms.wh + (H - 1) * 64 * 72;
    ms.b = reinterpret_cast<float*>(smem_raw + plan.bias);
    LevelSm* lv = reinterpret_cast<LevelSm*>(smem_raw + plan.lv);
    unsigned char* wbase = smem_raw + plan.warp0 + plan.per_warp * warp;
    __half* feat = reinterpret_cast<__half*>(wbase + plan.feat);              // [16][D+8]
    float* zt = reinterpret_cast<float*>(wbase + plan.z);                     // [16][8]
    float* xs = reinterpret_cast<float*>(wbase + plan.xs);                    // [n_pts*3][16]
    stage_mlp(a.m, ms, tid, blockDim.x);
    stage_levels(a.g, lv, tid);
    __syncthreads();
    const int cpp = (L * F) / 8;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t hmask = (1u << a.g.log2_T) - 1u;
    for (int64_t blk = (int64_t)blockIdx.x * kFwdWarps + warp; blk * 16 < M; blk += (int64_t)gridDim.x * kFwdWarps) {
        const int64_t i0 = blk * 16;
        const int nv = (int)min((int64_t)16, (int64_t)M - i0);
        SampleDesc q;
        q.valid = 0;
        if (lane < 16) {
            load_sample_desc(a, (int)(i0 + lane), M, q);
            if (q.valid)
#pragma unroll
                for (int p = 0; p < 4; ++p) {       // jittered stratified points (C8)
                    if (p >= n_pts) break;          // n_points <= 4 (checked by the host)
                    float x[3];
                    segment_point(a.g, q.o, q.d, q.t0, q.t1, p, n_pts, q.xi, x);
                    xs[(p * 3 + 0) * 16 + lane] = x[0];
                    xs[(p * 3 + 1) * 16 + lane] = x[1];
                    xs[(p * 3 + 2) * 16 + lane] = x[2];
                }
        }
        __syncwarp();
        {   // encode: lane -> row lane % 16, the half-warps take points of opposite parity
            const int r = lane & 15, h = lane >> 4;
            if (r < nv) {
                for (int p = h; p < n_pts; p += 2) {
                    const float x0 = xs[(p * 3 + 0) * 16 + r], x1 = xs[(p * 3 + 1) * 16 + r],
                                x2 = xs[(p * 3 + 2) * 16 + r];
                    for (int lc = 0; lc < cpp; ++lc)
                        *reinterpret_cast<uint4*>(feat + r * (D + 8) + (p * cpp + lc) * 8) =
                            encode_chunk_sm<F, false, false, kTex>(lv, a.g.table, hmask, x0, x1, x2, lc * (8 / F),
                                                                   nullptr, a.g.tex);
                }
            }
        }
        __syncwarp();
        // features out (for the weight gradient of layer 0)
        for (int e = lane; e < 16 * (D / 8); e += 32) {
            const int row = e / (D / 8), c = e % (D / 8);
            if (row < nv)
                reinterpret_cast<uint4*>(a.X + (i0 + row) * D)[c] = *reinterpret_cast<const uint4*>(feat + row * (D + 8) + c * 8);
        }
        // MLP forward: 16 rows; hidden activations to global
        {
            float acc[8][4];
            for (int nt = 0; nt < 8; ++nt) {
                float b0 = ms.b[nt * 8 + 2 * t], b1 = ms.b[nt * 8 + 2 * t + 1];
                acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
            }
            const uint32_t xa = (uint32_t)__cvta_generic_to_shared(feat + (lane & 15) * (D + 8) + (lane >> 4) * 8);
            const uint32_t wa = (uint32_t)__cvta_generic_to_shared(ms.w0 + ((lane & 7) + ((lane >> 4) << 3)) * (D + 8) +
                                                                   ((lane >> 3) & 1) * 8);
#pragma unroll
            for (int kb = 0; kb < D / 16; ++kb) {
                uint32_t af[4];
                ldsm_x4(xa + kb * 32, af[0], af[1], af[2], af[3]);
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(wa + np * 16 * (D + 8) * 2 + kb * 32, b0, b1, b2, b3);
                    mma16816(acc[2 * np], af, b0, b1);
                    mma16816(acc[2 * np + 1], af, b2, b3);
                }
            }
            uint32_t h[4][4];
            for (int layer = 0; layer < H; ++layer) {
                if (layer > 0) {
                    const __half* W = ms.wh + (layer - 1) * 64 * 72;
                    const float* bb = ms.b + layer * 64;
                    for (int nt = 0; nt < 8; ++nt) {
                        float b0 = bb[nt * 8 + 2 * t], b1 = bb[nt * 8 + 2 * t + 1];
                        acc[nt][0] = b0; acc[nt][1] = b1; acc[nt][2] = b0; acc[nt][3] = b1;
                    }
                    const uint32_t wb = (uint32_t)__cvta_generic_to_shared(W + ((lane & 7) + ((lane >> 4) << 3)) * 72 +
                                                                           ((lane >> 3) & 1) * 8);
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                        for (int np = 0; np < 4; ++np) {
                            uint32_t b0, b1, b2, b3;
                            ldsm_x4(wb + np * 16 * 72 * 2 + kb * 32, b0, b1, b2, b3);
                            mma16816(acc[2 * np], h[kb], b0, b1);
                            mma16816(acc[2 * np + 1], h[kb], b2, b3);
                        }
                }
#pragma unroll
                for (int kb = 0; kb < 4; ++kb) {
                    h[kb][0] = pack_relu_half2(acc[2 * kb][0], acc[2 * kb][1]);
                    h[kb][1] = pack_relu_half2(acc[2 * kb][2], acc[2 * kb][3]);
                    h[kb][2] = pack_relu_half2(acc[2 * kb + 1][0], acc[2 * kb + 1][1]);
                    h[kb][3] = pack_relu_half2(acc[2 * kb + 1][2], acc[2 * kb + 1][3]);
                }
                // activations out through the (consumed) feature rows: fragment layout -> [16][64]
                // rows in shared memory, then 16-byte row-contiguous stores (a 4-byte fragment
                // store per lane would touch 16 rows' lines per instruction)
                __half* Al = a.A + (int64_t)layer * a.cap * 64;
                __syncwarp();                     // every lane's ldmatrix of the previous contents done
#pragma unroll
                for (int kb = 0; kb < 4; ++kb) {
                    *reinterpret_cast<uint32_t*>(feat + g * (D + 8) + kb * 16 + 2 * t) = h[kb][0];
                    *reinterpret_cast<uint32_t*>(feat + g * (D + 8) + kb * 16 + 8 + 2 * t) = h[kb][2];
                    *reinterpret_cast<uint32_t*>(feat + (g + 8) * (D + 8) + kb * 16 + 2 * t) = h[kb][1];
                    *reinterpret_cast<uint32_t*>(feat + (g + 8) * (D + 8) + kb * 16 + 8 + 2 * t) = h[kb][3];
                }
                __syncwarp();
#pragma unroll
                for (int c = lane; c < 16 * 8; c += 32) {
                    const int row = c >> 3, c8 = c & 7;
                    if (row < nv)
                        *reinterpret_cast<uint4*>(Al + (i0 + row) * 64 + c8 * 8) =
                            *reinterpret_cast<const uint4*>(feat + row * (D + 8) + c8 * 8);
                }
            }
            float o[4];
            {
                const float* bb = ms.b + H * 64;
                o[0] = bb[2 * t]; o[1] = bb[2 * t + 1]; o[2] = o[0]; o[3] = o[1];
            }
            const uint32_t wo = (uint32_t)__cvta_generic_to_shared(ms.wo + (lane & 7) * 72 + ((lane >> 3) & 1) * 8);
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
                uint32_t b0, b1;
                ldsm_x2(wo + kb * 32, b0, b1);
                mma16816(o, h[kb], b0, b1);
            }
            zt[g * 8 + 2 * t] = o[0];
            zt[g * 8 + 2 * t + 1] = o[1];
            zt[(g + 8) * 8 + 2 * t] = o[2];
            zt[(g + 8) * 8 + 2 * t + 1] = o[3];
        }
        __syncwarp();
        // gated loss and dL/dz (lanes 0-15 own the rows)
        float terms[4] = {0.f, 0.f, 0.f, 0.f}, Ls = 0.f;
        if (lane < 16 && q.valid) {
            const int64_t i = i0 + lane;
            float gt[9], dz[8];
#pragma unroll
            for (int k = 0; k < 9; ++k) gt[k] = a.s_gt[9 * i + k];
            Ls = sample_loss(zt + lane * 8, gt, terms, dz);
            float4* dst = reinterpret_cast<float4*>(a.dZ + i * 8);
            dst[0] = make_float4(dz[0], dz[1], dz[2], dz[3]);
            dst[1] = make_float4(dz[4], dz[5], dz[6], dz[7]);
            if (a.Z) {
                float4* zd = reinterpret_cast<float4*>(a.Z + i * 8);
                const float* zz = zt + lane * 8;
                zd[0] = make_float4(zz[0], zz[1], zz[2], zz[3]);
                zd[1] = make_float4(zz[4], zz[5], zz[6], zz[7]);
            }
            a.r_loss[q.ray] = Ls;
            atomicAdd(a.tail + 1 + 3 * q.leaf, Ls);
            atomicAdd(a.tail + 1 + 3 * q.leaf + 1, 1.0f);
        }
        float v[5] = {Ls, terms[0], terms[1], terms[2], terms[3]};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
            if (lane == 0) atomicAdd(a.loss_acc + k, (double)v[k]);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ T6 backward (delta chain)
// Per warp (16 samples): delta_H = dL/dz; delta_k = (delta_{k+1} W_{k+1}) * relu'(h_k)
// on tensor cores (B operands via ldmatrix.trans of the [out][in] weights), deltas of the
// hidden layers written out for the weight gradients; dL/dx = delta_0 W_0 written out (fp32)
// for the hash-grid scatter (k_train_scatter, T7).
struct BwdSmem {
    __half* w0;   // [64][D+8]
    __half* wh;   // [H-1][64][72]
    __half* wo;   // [16][72], rows 8..15 zero
};
// bytes of k_train_bwd's shared memory: the weights, then per warp one staging tile that
// turns the fragment-layout row accesses into row-contiguous 16-byte global accesses:
// [16][D+4] fp32 for dL/dx, aliased by [16][72] fp16 for the activation masks and deltas
__host__ __device__ constexpr size_t bwd_weights_bytes(int D, int H) {
    return ((size_t)64 * (D + 8) + (size_t)(H - 1) * 64 * 72 + 16 * 72) * 2;
}
__host__ __device__ constexpr size_t bwd_tile_bytes(int D) { return (size_t)16 * (D + 4) * 4; }
constexpr int kBwdWarps = 8;

template <int F, int D>
__global__ void __launch_bounds__(256, 2) k_train_bwd(TrainArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int M = *a.n_samples;
    const int n_tiles = (M + kTileQ - 1) / kTileQ;
    if ((int)blockIdx.x >= n_tiles) return;
    const int H = a.m.hidden;
    BwdSmem s;
    s.w0 = reinterpret_cast<__half*>(smem_raw);
    s.wh = s.w0 + 64 * (D + 8);
    s.wo = s.wh + (H - 1) * 64 * 72;
    {   // stage weights (fp16 inference copy == forward operands)
        const uint4* W = reinterpret_cast<const uint4*>(a.m.W);
        const int cpr0 = D / 8;
        for (int i = tid; i < 64 * cpr0; i += blockDim.x)
            *reinterpret_cast<uint4*>(s.w0 + (i / cpr0) * (D + 8) + (i % cpr0) * 8) = __ldg(W + i);
        const uint4* Wh = W + 64 * cpr0;
        for (int i = tid; i < (H - 1) * 64 * 8; i += blockDim.x)
            *reinterpret_cast<uint4*>(s.wh + (i / 8) * 72 + (i % 8) * 8) = __ldg(Wh + i);
        const uint4* Wo = Wh + (H - 1) * 64 * 8;
        for (int i = tid; i < 16 * 8; i += blockDim.x)
            *reinterpret_cast<uint4*>(s.wo + (i / 8) * 72 + (i % 8) * 8) = i < 64 ? __ldg(Wo + i) : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    const int g = lane >> 2, t = lane & 3;
    float* gxs = reinterpret_cast<float*>(smem_raw + ((bwd_weights_bytes(D, H) + 15) & ~(size_t)15) +
                                          (size_t)warp * bwd_tile_bytes(D));      // [16][D+4]
    __half* ts = reinterpret_cast<__half*>(gxs);                                  // [16][72] (aliases)
    // warp item = 16 samples; no block-wide barrier after the staging
    for (int blk = blockIdx.x * kBwdWarps + warp; blk * 16 < M; blk += gridDim.x * kBwdWarps) {
        const int64_t gr0 = (int64_t)blk * 16 + g, gr1 = gr0 + 8;
        const bool v0 = gr0 < M, v1 = gr1 < M;
        const int nv = min(16, M - blk * 16);
        // delta_H = dL/dz as an m16k16 A fragment (k 8..15 zero)
        uint32_t af[4][4];
        {
            float2 d0 = v0 ? *reinterpret_cast<const float2*>(a.dZ + gr0 * 8 + 2 * t) : make_float2(0.f, 0.f);
            float2 d1 = v1 ? *reinterpret_cast<const float2*>(a.dZ + gr1 * 8 + 2 * t) : make_float2(0.f, 0.f);
            af[0][0] = pack_half2(d0.x, d0.y);
            af[0][1] = pack_half2(d1.x, d1.y);
            af[0][2] = 0u;
            af[0][3] = 0u;
        }
        for (int k = H - 1; k >= 0; --k) {
            float acc[8][4];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
            const bool from_out = (k == H - 1);
            const __half* W = from_out ? s.wo : s.wh + k * 64 * 72;   // W_{k+1}: [K][64], row stride 72
            const int ksteps = from_out ? 1 : 4;
            const uint32_t wb = (uint32_t)__cvta_generic_to_shared(W + (lane & 15) * 72 + (lane >> 4) * 8);
            for (int kb = 0; kb < ksteps; ++kb) {
#pragma unroll
                for (int np = 0; np < 4; ++np) {
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(wb + kb * 16 * 72 * 2 + np * 32, b0, b1, b2, b3);
                    mma16816(acc[2 * np], af[kb], b0, b1);
                    mma16816(acc[2 * np + 1], af[kb], b2, b3);
                }
            }
            // relu'(h_k) mask and store delta_k (rows staged through ts: 16-byte row-contiguous
            // global loads / stores instead of 4-byte fragment accesses spread over 16 rows)
            const __half* Ak = a.A + (int64_t)k * a.cap * 64;
            __half* Dk = a.Dl + (int64_t)k * a.cap * 64;
            const int64_t r0 = (int64_t)blk * 16;
#pragma unroll
            for (int c = lane; c < 16 * 8; c += 32) {
                const int row = c >> 3, c8 = c & 7;
                *reinterpret_cast<uint4*>(ts + row * 72 + c8 * 8) =
                    row < nv ? *reinterpret_cast<const uint4*>(Ak + (r0 + row) * 64 + c8 * 8) : make_uint4(0, 0, 0, 0);
            }
            __syncwarp();
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int col = nt * 8 + 2 * t;
                const float2 h0 = unpack_half2(*reinterpret_cast<const uint32_t*>(ts + g * 72 + col));
                const float2 h1 = unpack_half2(*reinterpret_cast<const uint32_t*>(ts + (g + 8) * 72 + col));
                acc[nt][0] = h0.x > 0.f ? acc[nt][0] : 0.f;
                acc[nt][1] = h0.y > 0.f ? acc[nt][1] : 0.f;
                acc[nt][2] = h1.x > 0.f ? acc[nt][2] : 0.f;
                acc[nt][3] = h1.y > 0.f ? acc[nt][3] : 0.f;
            }
            __syncwarp();                     // masks read before the deltas overwrite the tile
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int col = nt * 8 + 2 * t;
                *reinterpret_cast<uint32_t*>(ts + g * 72 + col) = pack_half2(acc[nt][0], acc[nt][1]);
                *reinterpret_cast<uint32_t*>(ts + (g + 8) * 72 + col) = pack_half2(acc[nt][2], acc[nt][3]);
            }
            __syncwarp();
#pragma unroll
            for (int c = lane; c < 16 * 8; c += 32) {
                const int row = c >> 3, c8 = c & 7;
                if (row < nv)
                    *reinterpret_cast<uint4*>(Dk + (r0 + row) * 64 + c8 * 8) = *reinterpret_cast<const uint4*>(ts + row * 72 + c8 * 8);
            }
            __syncwarp();                     // tile free for the next layer
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
                af[kb][0] = pack_half2(acc[2 * kb][0], acc[2 * kb][1]);
                af[kb][1] = pack_half2(acc[2 * kb][2], acc[2 * kb][3]);
                af[kb][2] = pack_half2(acc[2 * kb + 1][0], acc[2 * kb + 1][1]);
                af[kb][3] = pack_half2(acc[2 * kb + 1][2], acc[2 * kb + 1][3]);
            }
        }
        // dL/dx = delta_0 W_0  ([16 x 64] x [64 x D]) -> fp32 rows of a.gx
        const uint32_t w0b = (uint32_t)__cvta_generic_to_shared(s.w0 + (lane & 15) * (D + 8) + (lane >> 4) * 8);
#pragma unroll 1
        for (int np = 0; np < D / 16; ++np) {
            float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(w0b + kb * 16 * (D + 8) * 2 + np * 32, b0, b1, b2, b3);
                mma16816(acc[0], af[kb], b0, b1);
                mma16816(acc[1], af[kb], b2, b3);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int c = (2 * np + j) * 8 + 2 * t;
                *reinterpret_cast<float2*>(gxs + g * (D + 4) + c) = make_float2(acc[j][0], acc[j][1]);
                *reinterpret_cast<float2*>(gxs + (g + 8) * (D + 4) + c) = make_float2(acc[j][2], acc[j][3]);
            }
        }
        __syncwarp();
        // dL/dx rows out, 16 bytes per lane, row-contiguous
        for (int c = lane; c < 16 * (D / 4); c += 32) {
            const int row = c / (D / 4), c4 = c - row * (D / 4);
            if (row < nv)
                *reinterpret_cast<float4*>(a.gx + ((int64_t)blk * 16 + row) * D + c4 * 4) =
                    *reinterpret_cast<const float4*>(gxs + row * (D + 4) + c4 * 4);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ T7 hash-grid gradient scatter
// P:61 (hash-grid backprop): dL/dT[entry] += w_corner * dL/dfeat for every corner of every
// (sample, point, level).  One thread per (sample, point): the point is recomputed from the
// sample descriptor (same op order as the forward), dL/dx of its L levels read from a.gx.
// Three destinations, so that no two lanes race on a hot address and the L2 sees fewer,
// wider reductions (T7 is bound by L2 reduction throughput):
//   * coarse dense levels l < priv_levels: a CTA-private shared-memory accumulator in fixed
//     point (native 32-bit ATOMS.ADD; fp32 shared atomics are CAS loops on sm_100): each
//     contribution v = hi + lo with hi = rint(v 2^10) 2^-10 and |lo| <= 2^-11 added to two
//     int32 sums at scales 2^10 and 2^28 (resolution 2^-28), written per CTA to a.sc_priv and
//     summed over CTAs in 64-bit integers by k_train_scatter_finish (C37);
//   * other dense levels: a cell-packed scratch (the 8 corners of a cell contiguous, like the
//     inference table): four 16-byte red.global.add.v4.f32 per point-level instead of eight
//     8-byte ones; k_train_scatter_finish gathers each vertex's 8 cells;
//   * hashed levels: an aligned [T][F] scratch: the x-neighbour corners of an even cell
//     coordinate are entries e, e^1 of one 16-byte pair (pi_1 = 1) -> one red.v4 (F = 2).
constexpr float kFixHi = 1024.0f;              // 2^10: scale of the high part
constexpr float kFixLo = 268435456.0f;         // 2^28: scale of the low part (|lo| <= 2^-11: 2^14
                                               // worst-case same-sign contributions per entry and CTA)
constexpr float kFixLimit = 1048576.0f;        // 2^20: larger contributions go to a global fp32 atomic

template <int F>
__device__ __forceinline__ void red_entry(float* p, const float* v) {
    if constexpr (F == 2) red_add_v2(p, v[0], v[1]);
    else asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                      "f"(v[3]) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float x, float y, float z, float w) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x), "f"(y), "f"(z), "f"(w)
                 : "memory");
}

template <int F>
__global__ void __launch_bounds__(256) k_train_scatter(TrainArgs a) {
    extern __shared__ __align__(16) int32_t priv[];          // [2][priv_floats]: high, low parts
    __shared__ LevelSm lv[kMaxLevels];
    const int tid = threadIdx.x;
    stage_levels(a.g, lv, tid);
    for (int i = tid; i < 2 * a.priv_floats; i += blockDim.x) priv[i] = 0;
    __syncthreads();
    const int M = *a.n_samples, NP = a.g.n_points, L = a.g.L, D = NP * L * F;
    const uint32_t hmask = (1u << a.g.log2_T) - 1u;
    const int64_t items = (int64_t)M * NP;
    // the samples arrive grouped by leaf (k_sort_place): walk them in a scrambled order, i ->
    // i * scr mod M with scr prime to M, so a warp's reductions land on unrelated entries
    const uint64_t scr = (M % 1000003) ? 1000003ull : 998244353ull;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + tid; it < items; it += (int64_t)gridDim.x * blockDim.x) {
        const int iq = (int)(it / NP), p = (int)(it - (int64_t)iq * NP);
        const int i = (int)(((uint64_t)iq * scr) % (uint64_t)M);   // scrambled sample order (a bijection)
        // the sample's segment and jitter straight from global memory (a SampleDesc with a
        // runtime-indexed xi would live in local memory)
        const int r = a.s_ray[i];
        const float4 r0 = __ldg(a.rays + 2 * (int64_t)r), r1 = __ldg(a.rays + 2 * (int64_t)r + 1);
        const float o[3] = {r0.x, r0.y, r0.z}, d[3] = {r1.x, r1.y, r1.z};
        float x[3];
        segment_point(a.g, o, d, a.s_t0[i], a.s_t1[i], p, NP, a.xi + (int64_t)r * NP, x);   // the forward's point (C8)
        const float* gq = a.gx + (int64_t)i * D + p * L * F;
        for (int l = 0; l < L; ++l) {
            const LevelSm P = lv[l];
            float gv[F];
#pragma unroll
            for (int f = 0; f < F; ++f) gv[f] = gq[l * F + f];
            Cell cell;
            uint32_t i0, i1, i2;
            level_cell_sm(P, hmask, x[0], x[1], x[2], cell, i0, i1, i2);
            if (l < a.priv_levels) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int f = 0; f < F; ++f) {
                        const float v = cell.w[k] * gv[f];
                        const int64_t e = (int64_t)(P.coff + cell.idx[k]) * F + f;
                        NBVH_DCHECK(e < a.priv_floats);
                        if (fabsf(v) < kFixLimit) {
                            const float hi = rintf(v * kFixHi);                 // exact: |v 2^10| < 2^30
                            const float lo = __fmaf_rn(-hi, 1.0f / kFixHi, v);  // exact remainder
                            atomicAdd(priv + e, (int)hi);
                            atomicAdd(priv + a.priv_floats + e, __float2int_rn(lo * kFixLo));
                        } else {
                            atomicAdd(a.grad + e, v);
                        }
                    }
            } else if (P.n1) {
                // cell-packed scratch: cell = i0 + N i1 + N^2 i2, 8 corners x F floats
                float* base = a.sc_dense + a.sc_off[l] + (int64_t)(i0 + P.nx * i1 + P.nxy * i2) * 8 * F;
#pragma unroll
                for (int j = 0; j < 4; ++j) {              // corners 2j (x) and 2j+1 (x+1)
                    if constexpr (F == 2) {
                        red_add_v4(base + 4 * j, cell.w[2 * j] * gv[0], cell.w[2 * j] * gv[1],
                                   cell.w[2 * j + 1] * gv[0], cell.w[2 * j + 1] * gv[1]);
                    } else {
                        float u[F], w2[F];
#pragma unroll
                        for (int f = 0; f < F; ++f) { u[f] = cell.w[2 * j] * gv[f]; w2[f] = cell.w[2 * j + 1] * gv[f]; }
                        red_entry<F>(base + (2 * j) * F, u);
                        red_entry<F>(base + (2 * j + 1) * F, w2);
                    }
                }
            } else {
                float* base = a.sc_hash + a.sc_off[l];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t e0 = cell.idx[2 * j], e1 = cell.idx[2 * j + 1];
                    float u[F], w2[F];
#pragma unroll
                    for (int f = 0; f < F; ++f) { u[f] = cell.w[2 * j] * gv[f]; w2[f] = cell.w[2 * j + 1] * gv[f]; }
                    if (F == 2 && (e0 ^ e1) == 1u) {       // one aligned 16-byte pair {e, e^1}
                        const bool lo0 = e0 < e1;
                        red_add_v4(base + (int64_t)(e0 & ~1u) * 2, lo0 ? u[0] : w2[0], lo0 ? u[1] : w2[1],
                                   lo0 ? w2[0] : u[0], lo0 ? w2[1] : u[1]);
                    } else {
                        red_entry<F>(base + (int64_t)e0 * F, u);
                        red_entry<F>(base + (int64_t)e1 * F, w2);
                    }
                }
            }
        }
    }
    __syncthreads();
    int32_t* out = a.sc_priv + (int64_t)blockIdx.x * 2 * a.priv_floats;
    for (int i = tid; i < 2 * a.priv_floats; i += blockDim.x) out[i] = priv[i];
}

// T7 with warp aggregation (the default; the samples in leaf order, k_sort_place): a warp's 32
// items are 8 samples x 4 points of (mostly) one leaf, so on the coarse levels many of them
// fall into the same grid cell.  On levels l < agg_levels the lanes are grouped by cell
// (__match_any_sync on the cell coordinates); the group's 8F sums sum_j w_j[k] g_j[f]
// (ascending lane order, fp32) are spread over its lanes -- the lane of rank q computes values
// q, q + cnt, ... from the members' weights and dL/dx staged in shared memory -- and the
// group's lowest lane makes the one set of reductions for the cell (the destinations of
// k_train_scatter; on privatised levels the group sum is split into the fixed-point parts).
// Finer levels: one set per item.  Measured on the cfg-5 step (profiles/NOTES.md r2d): L1
// data-pipe wavefronts are what bound the scatter (a red sector or a shared atomic is one
// each); aggregating levels 0-5 instead of privatising 0-2 removes the shared atomics and
// ~1/6 of the red sectors for ~1/4 more shared loads/stores: 0.720 vs 0.749 ms backward.
// (Tried: a register butterfly for whole-warp groups, 0.765; redux.sync fixed-point group
// sums, 0.784.)
template <int F>
__global__ void __launch_bounds__(256) k_train_scatter_agg(TrainArgs a) {
    extern __shared__ __align__(16) int32_t priv[];          // [2][priv_floats], then per warp [32][8F]
    __shared__ LevelSm lv[kMaxLevels];
    constexpr int S = 8 * F;                                  // floats per lane slot (>= 8 + F)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* abuf = reinterpret_cast<float*>(priv + ((2 * a.priv_floats + 3) & ~3)) + warp * 32 * S;
    stage_levels(a.g, lv, tid);
    for (int i = tid; i < 2 * a.priv_floats; i += blockDim.x) priv[i] = 0;
    __syncthreads();
    const int M = *a.n_samples, NP = a.g.n_points, L = a.g.L, D = NP * L * F;
    const uint32_t hmask = (1u << a.g.log2_T) - 1u;
    const int64_t items = (int64_t)M * NP;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (tid & ~31); base < items;
         base += (int64_t)gridDim.x * blockDim.x) {              // warp-uniform trip count
        const int64_t it = base + lane;
        const bool valid = it < items;
        const int i = valid ? (int)(it / NP) : 0, p = valid ? (int)(it - (int64_t)i * NP) : 0;
        const int r = a.s_ray[i];
        const float4 r0 = __ldg(a.rays + 2 * (int64_t)r), r1 = __ldg(a.rays + 2 * (int64_t)r + 1);
        const float o[3] = {r0.x, r0.y, r0.z}, d[3] = {r1.x, r1.y, r1.z};
        float x[3];
        segment_point(a.g, o, d, a.s_t0[i], a.s_t1[i], p, NP, a.xi + (int64_t)r * NP, x);   // the forward's point (C8)
        const float* gq = a.gx + (int64_t)i * D + p * L * F;
        for (int l = 0; l < L; ++l) {
            const LevelSm P = lv[l];
            float gv[F];
            if (F == 2 && a.tex_gx) {      // through the texture pipe: the load pipe is this kernel's limit
                const float2 v = valid ? tex1Dfetch<float2>((cudaTextureObject_t)a.tex_gx, (int)(it * L + l))
                                       : make_float2(0.f, 0.f);
                gv[0] = v.x;
                gv[F - 1] = v.y;
            } else {
#pragma unroll
                for (int f = 0; f < F; ++f) gv[f] = valid ? gq[l * F + f] : 0.f;
            }
            Cell cell;
            uint32_t i0, i1, i2;
            level_cell_sm(P, hmask, x[0], x[1], x[2], cell, i0, i1, i2);
            float u[8][F];
            bool emit = valid;
            int cnt = 1;
            if (l < a.agg_levels) {
                const uint32_t N = (uint32_t)P.resf;
                const uint32_t key = valid ? i0 + N * (i1 + N * i2) : (0x80000000u | (uint32_t)lane);   // N^3 < 2^31
                const unsigned peers = __match_any_sync(0xffffffffu, key);
                cnt = __popc(peers);
                if (cnt > 1) {
                    float* my = abuf + lane * S;
#pragma unroll
                    for (int k = 0; k < 8; ++k) my[k] = cell.w[k];
#pragma unroll
                    for (int f = 0; f < F; ++f) my[8 + f] = gv[f];
                }
                __syncwarp();
                const int leader = __ffs(peers) - 1, rank = __popc(peers & lt);
                float res[S];
                if (cnt > 1) {
#pragma unroll
                    for (int t = 0; t < S; ++t) {
                        const int v = rank + t * cnt;
                        res[t] = 0.f;
                        if (v < S) {
                            const int k = v / F, f = v - k * F;
                            float acc = 0.f;
                            for (unsigned m = peers; m; m &= m - 1u) {
                                const float* js = abuf + (__ffs(m) - 1) * S;
                                acc = __fadd_rn(acc, __fmul_rn(js[k], js[8 + f]));
                            }
                            res[t] = acc;
                        }
                    }
                }
                __syncwarp();
                if (cnt > 1) {
#pragma unroll
                    for (int t = 0; t < S; ++t) {
                        const int v = rank + t * cnt;
                        if (v < S) abuf[leader * S + v] = res[t];
                    }
                }
                __syncwarp();
                if (cnt > 1) {
                    NBVH_DCHECK(leader >= 0 && leader < 32 && rank < cnt);
                    emit = valid && lane == leader;
                    if (emit) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
#pragma unroll
                            for (int f = 0; f < F; ++f) u[k][f] = abuf[lane * S + k * F + f];
                    }
                }
            }
            if (cnt == 1) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int f = 0; f < F; ++f) u[k][f] = __fmul_rn(cell.w[k], gv[f]);
            }
            if (!emit) continue;
            if (l < a.priv_levels) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int f = 0; f < F; ++f) {
                        const float v = u[k][f];
                        const int64_t e = (int64_t)(P.coff + cell.idx[k]) * F + f;
                        NBVH_DCHECK(e < a.priv_floats);
                        if (fabsf(v) < kFixLimit) {
                            const float hi = rintf(v * kFixHi);
                            const float lo = __fmaf_rn(-hi, 1.0f / kFixHi, v);
                            atomicAdd(priv + e, (int)hi);
                            atomicAdd(priv + a.priv_floats + e, __float2int_rn(lo * kFixLo));
                        } else {
                            atomicAdd(a.grad + e, v);
                        }
                    }
            } else if (P.n1) {
                NBVH_DCHECK(i0 < P.nx && i1 < P.nx && i2 < P.nx);
                float* dst = a.sc_dense + a.sc_off[l] + (int64_t)(i0 + P.nx * i1 + P.nxy * i2) * 8 * F;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if constexpr (F == 2) {
                        red_add_v4(dst + 4 * j, u[2 * j][0], u[2 * j][1], u[2 * j + 1][0], u[2 * j + 1][1]);
                    } else {
                        red_entry<F>(dst + (2 * j) * F, u[2 * j]);
                        red_entry<F>(dst + (2 * j + 1) * F, u[2 * j + 1]);
                    }
                }
            } else {
                float* dst = a.sc_hash + a.sc_off[l];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t e0 = cell.idx[2 * j], e1 = cell.idx[2 * j + 1];
                    NBVH_DCHECK(e0 <= hmask && e1 <= hmask);
                    if (F == 2 && (e0 ^ e1) == 1u) {
                        const bool lo0 = e0 < e1;
                        const float a0 = u[2 * j][0], a1 = u[2 * j][F - 1], b0 = u[2 * j + 1][0], b1 = u[2 * j + 1][F - 1];
                        red_add_v4(dst + (int64_t)(e0 & ~1u) * 2, lo0 ? a0 : b0, lo0 ? a1 : b1, lo0 ? b0 : a0,
                                   lo0 ? b1 : a1);
                    } else {
                        red_entry<F>(dst + (int64_t)e0 * F, u[2 * j]);
                        red_entry<F>(dst + (int64_t)e1 * F, u[2 * j + 1]);
                    }
                }
            }
        }
    }
    __syncthreads();
    int32_t* out = a.sc_priv + (int64_t)blockIdx.x * 2 * a.priv_floats;
    for (int i = tid; i < 2 * a.priv_floats; i += blockDim.x) out[i] = priv[i];
}

// Scratch -> canonical gradient buffer (every table entry written exactly once):
//   coarse dense levels: the CTAs' fixed-point partials summed in 64-bit integers (exact,
//   order-independent) and scaled once; other dense levels: each vertex gathers its corner
//   of the up to 8 cells that contain it; hashed levels: a copy.
template <int F>
__global__ void __launch_bounds__(256) k_train_scatter_finish(TrainArgs a) {
    __shared__ LevelSm lv[kMaxLevels];
    stage_levels(a.g, lv, threadIdx.x);
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t e = t0; e < a.priv_floats; e += stride) {
        long long hi = 0, lo = 0;                    // integer sums: exact, any order
        const int32_t* part = a.sc_priv + e;
        const int64_t cs = 2 * (int64_t)a.priv_floats;
        int c = 0;
        for (; c + 8 <= a.scatter_ctas; c += 8) {    // 16 independent loads in flight
            int32_t h[8], l[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                h[u] = __ldcs(part + (c + u) * cs);
                l[u] = __ldcs(part + (c + u) * cs + a.priv_floats);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                hi += h[u];
                lo += l[u];
            }
        }
        for (; c < a.scatter_ctas; ++c) {
            hi += part[c * cs];
            lo += part[c * cs + a.priv_floats];
        }
        // += : keeps the rare overflow-path atomics
        a.grad[e] += (float)((double)hi * (1.0 / (double)kFixHi) + (double)lo * (1.0 / (double)kFixLo));
    }
    for (int l = a.priv_levels; l < a.g.L; ++l) {
        const LevelSm P = lv[l];
        if (P.n1) {
            const uint32_t n1 = P.n1, N = n1 - 1u, nv = P.n1sq * n1;
            const float* sc = a.sc_dense + a.sc_off[l];
            for (int64_t v = t0; v < nv; v += stride) {
                const uint32_t z = (uint32_t)v / P.n1sq, rem = (uint32_t)v - z * P.n1sq, y = rem / n1, x = rem - y * n1;
                float acc[F];
#pragma unroll
                for (int f = 0; f < F; ++f) acc[f] = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {              // cell (x - dx, y - dy, z - dz), corner k = (dx, dy, dz)
                    const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
                    const int cx = (int)x - dx, cy = (int)y - dy, cz = (int)z - dz;
                    if (cx < 0 || cy < 0 || cz < 0 || cx >= (int)N || cy >= (int)N || cz >= (int)N) continue;
                    const float* src = sc + ((int64_t)cx + N * ((int64_t)cy + N * cz)) * 8 * F + k * F;
#pragma unroll
                    for (int f = 0; f < F; ++f) acc[f] += src[f];
                }
#pragma unroll
                for (int f = 0; f < F; ++f) a.grad[((int64_t)P.coff + v) * F + f] = acc[f];
            }
        } else if (a.hash_coff0 < 0) {
            const int64_t n = (int64_t)(1u << a.g.log2_T) * F;
            const float* sc = a.sc_hash + a.sc_off[l];
            for (int64_t i = t0; i < n; i += stride) a.grad[(int64_t)P.coff * F + i] = sc[i];
        }
    }
    if (a.hash_coff0 >= 0) {
        // the hashed levels as one flat copy: 16-byte loads of the (16-byte aligned) scratch,
        // 8-byte stores into the canonical buffer (aligned to 8 bytes only), four loads in
        // flight per thread -- a per-level 4-byte loop was latency-bound (63 us, r2k)
        const int64_t n4 = a.hash_floats / 4;
        const float4* src = reinterpret_cast<const float4*>(a.sc_hash);
        float2* dst = reinterpret_cast<float2*>(a.grad + a.hash_coff0 * F);
        for (int64_t i = t0; i < n4; i += 4 * stride) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < n4) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < n4) {
                    const int64_t j = 2 * (i + u * stride);
                    __stcs(dst + j, make_float2(v[u].x, v[u].y));
                    __stcs(dst + j + 1, make_float2(v[u].z, v[u].w));
                }
        }
    }
}

// ------------------------------------------------------------------ T6 weight gradients
// dW_k = delta_k^T x_k over the batch as split-K tensor-core GEMMs: each CTA reduces a
// chunk of samples in registers and adds its partial once (red.global.add.v2.f32).
// Hidden layers on mma.sync (fp16 operands, fp32 accumulate); the 8-output layer on
// CUDA cores from the fp32 dL/dz.
constexpr int kDwChunk = 2048;

// The mma.sync fallback used when the tcgen05 contraction does not fit (Mtot > 256).
template <int D>
__global__ void __launch_bounds__(256, 1) k_train_dw(TrainArgs a, int64_t w_off, int64_t b_off) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int M = *a.n_samples;
    const int64_t c0 = (int64_t)blockIdx.x * kDwChunk;
    if (c0 >= M) return;
    const int64_t c1 = min((int64_t)M, c0 + kDwChunk);
    const int H = a.m.hidden;
    __half* sd = reinterpret_cast<__half*>(smem_raw);          // delta tile [128][72]
    __half* sx = sd + kTileQ * 72;                             // input tile [128][D+8]
    float* sz = reinterpret_cast<float*>(sx + kTileQ * (D + 8));   // dZ tile [128][8]
    const int g = lane >> 2, t = lane & 3;
    int64_t woff = w_off, boff = b_off;
    for (int k = 0; k < H; ++k) {
        const int in = k == 0 ? D : 64;
        const int NT = in / 8;               // n-tiles of 8
        const int mt = warp & 3;             // 16 output units per warp
        const int nt0 = (warp >> 2) * (NT / 2);
        float acc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        float dbias = 0.f;
        const __half* Dk = a.Dl + (int64_t)k * a.cap * 64;
        const __half* Xk = k == 0 ? a.X : a.A + (int64_t)(k - 1) * a.cap * 64;
        for (int64_t r = c0; r < c1; r += kTileQ) {
            for (int i = tid; i < kTileQ * 8; i += blockDim.x) {
                const int row = i / 8, c = i % 8;
                uint4 v = r + row < c1 ? reinterpret_cast<const uint4*>(Dk + (r + row) * 64)[c] : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(sd + row * 72 + c * 8) = v;
            }
            for (int i = tid; i < kTileQ * (in / 8); i += blockDim.x) {
                const int row = i / (in / 8), c = i % (in / 8);
                uint4 v = r + row < c1 ? reinterpret_cast<const uint4*>(Xk + (r + row) * in)[c] : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(sx + row * (D + 8) + c * 8) = v;
            }
            __syncthreads();
            if (tid < 64) {
                float sacc = 0.f;
                for (int row = 0; row < kTileQ; ++row) sacc += __half2float(sd[row * 72 + tid]);
                dbias += sacc;
            }
            const uint32_t aa = (uint32_t)__cvta_generic_to_shared(
                sd + ((lane & 7) + ((lane >> 4) << 3)) * 72 + mt * 16 + ((lane >> 3) & 1) * 8);
            const uint32_t ba = (uint32_t)__cvta_generic_to_shared(sx + (lane & 15) * (D + 8) + (lane >> 4) * 8);
#pragma unroll
            for (int ks = 0; ks < kTileQ / 16; ++ks) {
                uint32_t af[4];
                ldsm_x4_t(aa + ks * 16 * 72 * 2, af[0], af[1], af[2], af[3]);
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                    if (2 * jp < NT / 2) {
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4_t(ba + ks * 16 * (D + 8) * 2 + (nt0 + 2 * jp) * 16, b0, b1, b2, b3);
                        mma16816(acc[2 * jp], af, b0, b1);
                        mma16816(acc[2 * jp + 1], af, b2, b3);
                    }
                }
            }
            __syncthreads();
        }
        // flush partial sums
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j < NT / 2) {
                const int col = (nt0 + j) * 8 + 2 * t;
                const int u0 = mt * 16 + g, u1 = u0 + 8;
                red_add_v2(a.grad + woff + (int64_t)u0 * in + col, acc[j][0], acc[j][1]);
                red_add_v2(a.grad + woff + (int64_t)u1 * in + col, acc[j][2], acc[j][3]);
            }
        }
        if (tid < 64) atomicAdd(a.grad + boff + tid, dbias);
        woff += (int64_t)64 * in;
        boff += 64;
    }
    // output layer (64 -> 8): dW = dZ^T h_{H-1}, db = sum dZ, fp32 on CUDA cores
    {
        const __half* Ah = a.A + (int64_t)(H - 1) * a.cap * 64;
        float accw[2] = {0.f, 0.f}, accb = 0.f;
        const int o = tid / 32, i0 = (tid % 32) * 2;            // 8 outputs x 64 inputs, 2 per thread
        for (int64_t r = c0; r < c1; r += kTileQ) {
            for (int i = tid; i < kTileQ * 8; i += blockDim.x) {
                const int row = i / 8, c = i % 8;
                uint4 v = r + row < c1 ? reinterpret_cast<const uint4*>(Ah + (r + row) * 64)[c] : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(sx + row * (D + 8) + c * 8) = v;
            }
            for (int i = tid; i < kTileQ * 8; i += blockDim.x) {
                const int row = i / 8;
                sz[i] = r + row < c1 ? a.dZ[(r + row) * 8 + (i % 8)] : 0.f;
            }
            __syncthreads();
            for (int row = 0; row < kTileQ; ++row) {
                const float dz = sz[row * 8 + o];
                float2 h = __half22float2(*reinterpret_cast<const __half2*>(sx + row * (D + 8) + i0));
                accw[0] = fmaf(dz, h.x, accw[0]);
                accw[1] = fmaf(dz, h.y, accw[1]);
                if (i0 == 0) accb += dz;
            }
            __syncthreads();
        }
        red_add_v2(a.grad + woff + (int64_t)o * 64 + i0, accw[0], accw[1]);
        if (i0 == 0) atomicAdd(a.grad + boff + o, accb);
    }
}

// ------------------------------------------------------------------ T6 biases + output layer
// Companion of k_train_dw_tc: every bias gradient (column sums of the deltas, and of dL/dz
// for the output layer) and the 8-output layer's weight gradient dW_out = dZ^T h_{H-1}, in
// fp32 on CUDA cores.  Memory-bound streaming pass over the samples: each thread owns a
// 16-byte column group (8 deltas of one row) or an (output, 8-input) pair; per-CTA partial
// sums meet in shared memory and are flushed with one atomic per parameter per CTA.
constexpr int kBatch = 4;                        // rows in flight per thread (k_train_bias_out)
__global__ void __launch_bounds__(256, 2) k_train_bias_out(TrainArgs a, int64_t w_out_off, int64_t b_off) {
    // per-thread / per-warp partial sums, reduced over the row slots after one barrier (no
    // shared-memory atomics: they are CAS loops on sm_100)
    __shared__ float p1[256 * 8];                // (1): [slot * groups + g][8]
    __shared__ float p2[8 * 576];                // (2): [warp][8 x 64 weights, 8 biases, pad]
    const int tid = threadIdx.x;
    const int H = a.m.hidden;
    const int groups = H * 8;                    // 8 groups of 8 columns per hidden layer
    const int rows1 = blockDim.x / groups;
    const int M = *a.n_samples;
    // (1) hidden-layer biases: thread -> (row slot, layer, 8-column group)
    {
        const int rows_per_pass = rows1;
        const int slot = tid / groups, g = tid - slot * groups;
        const int layer = g >> 3, c0 = (g & 7) * 8;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (slot < rows_per_pass) {
            const __half* Dk = a.Dl + (int64_t)layer * a.cap * 64 + c0;
            const int64_t step = (int64_t)gridDim.x * rows_per_pass;
            // kBatch independent row loads in flight per thread (a streaming pass needs
            // ~40 KB in flight per SM to cover HBM latency)
            for (int64_t r = (int64_t)blockIdx.x * rows_per_pass + slot; r < M; r += kBatch * step) {
                uint4 v[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    v[u] = r + u * step < M ? __ldcs(reinterpret_cast<const uint4*>(Dk + (r + u * step) * 64))
                                            : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const __half2* h = reinterpret_cast<const __half2*>(&v[u]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float2 f = __half22float2(h[j]);
                        acc[2 * j] += f.x;
                        acc[2 * j + 1] += f.y;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) p1[tid * 8 + j] = acc[j];
        }
    }
    // (2) output layer: thread -> (row slot, 8-input group); each row's activations (16 B per
    //     thread) and its 8 output deltas are read once, 8 x 8 products accumulated
    {
        const int rows_per_pass = blockDim.x / 8;
        const int slot = tid >> 3, i0 = (tid & 7) * 8;
        float accw[8][8], accb[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            accb[o] = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) accw[o][j] = 0.f;
        }
        const __half* Ah = a.A + (int64_t)(H - 1) * a.cap * 64 + i0;
        const int64_t step = (int64_t)gridDim.x * rows_per_pass;
        for (int64_t r = (int64_t)blockIdx.x * rows_per_pass + slot; r < M; r += kBatch * step) {
            float4 d0[kBatch], d1[kBatch];
            uint4 v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int64_t ru = r + u * step;
                const bool ok = ru < M;   // rows past M add zeros
                d0[u] = ok ? *reinterpret_cast<const float4*>(a.dZ + ru * 8) : make_float4(0.f, 0.f, 0.f, 0.f);
                d1[u] = ok ? *reinterpret_cast<const float4*>(a.dZ + ru * 8 + 4) : make_float4(0.f, 0.f, 0.f, 0.f);
                v[u] = ok ? __ldcs(reinterpret_cast<const uint4*>(Ah + ru * 64)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const float dz[8] = {d0[u].x, d0[u].y, d0[u].z, d0[u].w, d1[u].x, d1[u].y, d1[u].z, d1[u].w};
                const __half2* hh = reinterpret_cast<const __half2*>(&v[u]);
                float f[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 t = __half22float2(hh[j]);
                    f[2 * j] = t.x;
                    f[2 * j + 1] = t.y;
                }
#pragma unroll
                for (int o = 0; o < 8; ++o) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) accw[o][j] = fmaf(dz[o], f[j], accw[o][j]);
                    accb[o] += dz[o];
                }
            }
        }
        // the 4 row slots of a warp that share i0 (lane bits 3-4) are summed with shuffles
#pragma unroll
        for (int o = 0; o < 8; ++o) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                accw[o][j] += __shfl_xor_sync(0xffffffffu, accw[o][j], 8);
                accw[o][j] += __shfl_xor_sync(0xffffffffu, accw[o][j], 16);
            }
            accb[o] += __shfl_xor_sync(0xffffffffu, accb[o], 8);
            accb[o] += __shfl_xor_sync(0xffffffffu, accb[o], 16);
        }
        if ((tid & 31) < 8) {
            float* pw = p2 + (tid >> 5) * 576;
#pragma unroll
            for (int o = 0; o < 8; ++o) {
#pragma unroll
                for (int j = 0; j < 8; ++j) pw[o * 64 + i0 + j] = accw[o][j];
                if (i0 == 0) pw[512 + o] = accb[o];
            }
        }
    }
    __syncthreads();
    // one global atomic per parameter per CTA
    for (int i = tid; i < H * 64; i += blockDim.x) {
        const int g = (i >> 6) * 8 + ((i & 63) >> 3), j = i & 7;
        float v = 0.f;
        for (int sl = 0; sl < rows1; ++sl) v += p1[(sl * groups + g) * 8 + j];
        atomicAdd(a.grad + b_off + i, v);
    }
    const int nw = blockDim.x >> 5;
    for (int i = tid; i < 520; i += blockDim.x) {             // 512 weights + 8 biases
        float v = 0.f;
        for (int w = 0; w < nw; ++w) v += p2[w * 576 + i];
        if (i < 512) atomicAdd(a.grad + w_out_off + i, v);
        else atomicAdd(a.grad + b_off + H * 64 + (i - 512), v);
    }
}

// ------------------------------------------------------------------ T6 weight gradients on tcgen05
// Every weight GEMM of the input and hidden layers as ONE tensor-core contraction over the
// samples: D[Mtot x Ntot] += Ain[Mtot x K] * Bd[Ntot x K]^T with K = samples,
//   Ain rows [0, D)                 : input features X,                 layer 0 inputs
//   Ain rows [D+64(k-1), D+64k)     : post-ReLU activations A_{k-1},     layer k inputs
//   Bd  rows [64k, 64k+64)          : deltas Dl_k (dL/d pre-activation)
// The diagonal blocks D[rows of layer k][cols 64k..] are dW_k^T; the off-diagonal blocks
// are discarded (3x the useful flops, free on the tensor pipe; one operand pass over HBM).
// One CTA of 4 warps per SM, split-K over 64-sample chunks: 128 threads stage chunks with
// cp.async into the MN-major no-swizzle canonical layout (4-stage ring, loads issued two
// chunks ahead so the operand stream is not latency-bound), thread 0 issues
// tcgen05.mma (M=128 halves, N=Ntot, K=16) into a TMEM accumulator and commits each stage
// to an mbarrier; the epilogue reads TMEM (tcgen05.ld) and adds the useful blocks into the
// gradient buffer once per CTA.
constexpr int kDwK = 64;            // samples per chunk (4 MMA K-steps)
constexpr int kDwGB = kDwK * 16;    // bytes of one 8-row group of a stage (kDwK/8 core matrices of 128 B)
constexpr int kDwStages = 4;
constexpr int kDwAhead = 2;         // chunks whose loads are in flight while one is multiplied

__host__ __device__ constexpr int dw_tc_mtot(int D, int H) { return D + 64 * (H - 1); }
__host__ __device__ constexpr size_t dw_tc_smem(int D, int H) {
    return (size_t)kDwStages * ((size_t)((dw_tc_mtot(D, H) + 127) / 128) * 16 + (size_t)H * 8) * kDwGB + 64;
}
__host__ __device__ constexpr bool dw_tc_ok(int D, int H) {
    return dw_tc_mtot(D, H) <= 256 && 64 * H <= 256 && dw_tc_smem(D, H) <= 227 * 1024;
}

constexpr int kDwThreads = 128;     // 4 warps stage operands and read back (one per TMEM lane quadrant)
template <int D, int H>
__global__ void __launch_bounds__(kDwThreads, 1) k_train_dw_tc(TrainArgs a, int64_t w_off) {
    constexpr int Mtot = dw_tc_mtot(D, H), Mh = (Mtot + 127) / 128, Ntot = 64 * H;
    constexpr int MG = Mh * 16, NG = Ntot / 8;                // 8-row groups of A, B
    constexpr uint32_t kAB = MG * kDwGB, kBB = NG * kDwGB;    // bytes per stage
    constexpr uint32_t kIdesc = tc::idesc_f16(128, Ntot, true, true);
    extern __shared__ __align__(16) unsigned char smem_dw[];
    unsigned char* stA = smem_dw;
    unsigned char* stB = smem_dw + kDwStages * kAB;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(stB + kDwStages * kBB);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + kDwStages);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int M = *a.n_samples;
    const int n_chunks = (M + kDwK - 1) / kDwK;
    if (tid == 0) {
        for (int i = 0; i < kDwStages; ++i) tc::mbar_init(mbar + i, 1);
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;

    // one 16-byte unit = 8 consecutive MN elements of one sample; thread -> (sample, group parity)
    auto stage = [&](int chunk, int st) {
        const int64_t s0 = (int64_t)chunk * kDwK;
        unsigned char* A = stA + st * kAB;
        unsigned char* B = stB + st * kBB;
        constexpr int kPar = kDwThreads / kDwK;              // threads per sample
        const int k = tid / kPar, par = tid % kPar;          // kDwK samples x kPar groups per pass
        const int64_t sm = s0 + k;
        const bool ok = sm < M;
        const int64_t sr = ok ? sm : 0;
        const uint32_t koff = (uint32_t)((k >> 3) * 128 + (k & 7) * 16);
        for (int g = par; g < MG; g += kPar) {                // A: features / activations
            const int row = g * 8;
            const __half* src;
            if (row < D) src = a.X + sr * D + row;
            else if (row < Mtot) src = a.A + (int64_t)((row - D) / 64) * a.cap * 64 + sr * 64 + ((row - D) & 63);
            else src = a.X;                                   // padding rows: never read back
            tc::cp16_zfill(A + g * kDwGB + koff, src, ok && row < Mtot);
        }
        for (int g = par; g < NG; g += kPar) {                // B: deltas
            const int col = g * 8;
            const __half* src = a.Dl + (int64_t)(col / 64) * a.cap * 64 + sr * 64 + (col & 63);
            tc::cp16_zfill(B + g * kDwGB + koff, src, ok);
        }
    };

    // prologue: the first kDwAhead chunks' loads
#pragma unroll
    for (int p = 0; p < kDwAhead; ++p) {
        const int c = blockIdx.x + p * gridDim.x;
        if (c < n_chunks) stage(c, p);
        tc::cp_commit();
    }
    int it = 0;
    for (int c = blockIdx.x; c < n_chunks; c += gridDim.x, ++it) {
        const int st = it % kDwStages;
        {   // loads of chunk it + kDwAhead into the stage last multiplied at it + kDwAhead - kDwStages
            const int cn = c + kDwAhead * gridDim.x, jn = it + kDwAhead, stn = jn % kDwStages;
            if (jn >= kDwStages) tc::mbar_wait(mbar + stn, ((jn / kDwStages) - 1) & 1);
            if (cn < n_chunks) stage(cn, stn);
            tc::cp_commit();                  // (an empty group past the end keeps the count uniform)
        }
        tc::cp_wait<kDwAhead>();              // this chunk's group has landed
        tc::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t a0 = tc::smem_u32(stA + st * kAB), b0 = tc::smem_u32(stB + st * kBB);
#pragma unroll
            for (int kk = 0; kk < kDwK / 16; ++kk) {
                const uint64_t bd = tc::smem_desc(b0 + kk * 256, 128, kDwGB);
#pragma unroll
                for (int h = 0; h < Mh; ++h) {
                    const uint64_t ad = tc::smem_desc(a0 + h * 16 * kDwGB + kk * 256, 128, kDwGB);
                    tc::mma_f16(tmem + h * 256, ad, bd, kIdesc, (it > 0 || kk > 0) ? 1u : 0u);
                }
            }
            tc::commit(mbar + st);
        }
    }
    // drain: wait for the last committed stage, then read the accumulator
    if (it > 0) {
        const int last = it - 1;
        tc::mbar_wait(mbar + (last % kDwStages), (last / kDwStages) & 1);
    }
    tc::fence_after();
    if (it > 0 && tid < 128) {
        // thread tid <-> TMEM lane tid <-> A row (h*128 + tid); useful columns = its layer's deltas
#pragma unroll 1
        for (int h = 0; h < Mh; ++h) {
            const int row = h * 128 + tid;
            int layer = -1, in = 0, i = 0;
            if (row < D) { layer = 0; in = D; i = row; }
            else if (row < Mtot) { layer = 1 + (row - D) / 64; in = 64; i = (row - D) & 63; }
            int64_t base = w_off;
            for (int l = 0; l < layer; ++l) base += (int64_t)64 * (l == 0 ? D : 64);
#pragma unroll 1
            for (int cb = 0; cb < Ntot; cb += 32) {
                float v[32];
                tc::ld32(tmem, (uint32_t)(warp * 32), (uint32_t)(h * 256 + cb), v);   // warp-collective
                if (layer >= 0 && cb >= 64 * layer && cb < 64 * layer + 64) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int o = cb - 64 * layer + j;                 // output unit
                        atomicAdd(a.grad + base + (int64_t)o * in + i, v[j]);
                    }
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

// ------------------------------------------------------------------ T9 Adam
__global__ void k_check_finite(const float* __restrict__ g, int64_t n, int32_t* flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) bad |= !isfinite(g[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

struct AdamArgs {
    float* param;
    const float* grad;
    float* m;
    float* v;
    int64_t n;
    const float* count;   // accepted-sample count (after the all-reduce)
    const int32_t* bad;
    int32_t* step;        // device Adam step count: advanced only by an applied update
    float lr, beta1, beta2, eps;
    __half* table16;
    int64_t n_table;
    __half* W16;
    int64_t n_W;
};

// P:275 Adam with default hyper-parameters (C20): dense, bias-corrected; the gradient is
// the batch mean (sum / accepted count).  The fp16 MLP weights are refreshed in place; the
// fp16 inference table is rebuilt afterwards by k_refresh_table (corner-packed layout).
// ic1 / ic2 = 1 / (1 - beta^t): the bias corrections of step t = (device step count) + 1,
// so an update skipped for a non-finite gradient does not advance t.
__device__ __forceinline__ float adam_one(const AdamArgs& a, float g, float& m, float& v, float p, float scale,
                                          float ic1, float ic2) {
    const float gr = g * scale;
    m = a.beta1 * m + (1.0f - a.beta1) * gr;
    v = a.beta2 * v + (1.0f - a.beta2) * gr * gr;
    return p - a.lr * (m * ic1) / (sqrtf(v * ic2) + a.eps);
}

// Vectorised (float4) over the flat parameter buffer; the fp16 MLP-weight copy is written for
// the elements inside the weight block.
__global__ void k_adam(AdamArgs a) {
    if (*a.bad) return;
    const float scale = 1.0f / fmaxf(1.0f, *a.count);
    const double t = (double)(*a.step + 1);
    const float ic1 = (float)(1.0 / (1.0 - pow((double)a.beta1, t)));
    const float ic2 = (float)(1.0 / (1.0 - pow((double)a.beta2, t)));
    const int64_t n4 = a.n / 4;
    const int64_t w0 = a.n_table, w1 = a.n_table + a.n_W;
    float4* P = reinterpret_cast<float4*>(a.param);
    const float4* G = reinterpret_cast<const float4*>(a.grad);
    float4* Mv = reinterpret_cast<float4*>(a.m);
    float4* Vv = reinterpret_cast<float4*>(a.v);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
        const float4 g = G[q];
        float4 m = Mv[q], v = Vv[q], p = P[q];
        p.x = adam_one(a, g.x, m.x, v.x, p.x, scale, ic1, ic2);
        p.y = adam_one(a, g.y, m.y, v.y, p.y, scale, ic1, ic2);
        p.z = adam_one(a, g.z, m.z, v.z, p.z, scale, ic1, ic2);
        p.w = adam_one(a, g.w, m.w, v.w, p.w, scale, ic1, ic2);
        Mv[q] = m;
        Vv[q] = v;
        P[q] = p;
        const int64_t i = 4 * q;
        if (i + 3 >= w0 && i < w1) {
            const float pv[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (i + k >= w0 && i + k < w1) a.W16[i + k - w0] = __float2half_rn(pv[k]);
        }
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
        float m = a.m[i], v = a.v[i];
        const float p = adam_one(a, a.grad[i], m, v, a.param[i], scale, ic1, ic2);
        a.m[i] = m;
        a.v[i] = v;
        a.param[i] = p;
        if (i >= w0 && i < w1) a.W16[i - w0] = __float2half_rn(p);
    }
}

// Advances the device step count after an applied update (one thread; stream-ordered after
// k_adam, which read it).
__global__ void k_adam_commit(const int32_t* bad, int32_t* step) {
    if (!*bad) *step += 1;
}

}  // namespace nbvh
