// nbvh_kernels.cu — the N-BVH neural ray-query hot path on sm_100a.
//
//   k_traverse    Q0+Q1: load rays, traverse the shallow N-BVH of the chosen cut, write
//                 the (t_enter, id)-ordered leaf list (capacity K) and seed the wave.
//   k_query_wave  Q2-Q6, fused: for a 128-query tile of active rays, sample the
//                 current leaf segment, hash-grid encode into shared memory, run the
//                 MLP on tensor cores, decode, update the per-ray best hit, decide
//                 front-to-back termination and compact the survivors into the next
//                 wave's active list with warp-aggregated atomics.
//   k_debug_*     the same device functions with intermediate results exposed.
//
// Paper passages: P:103 (front-to-back probing, early termination)
// (segment sampling, feature concatenation, MLP decode), P:161 (queries per ray =
// leaves met before a hit), P:201/P:237/P:243 (visibility threshold, local distance,
// normal, albedo).  Readings C1-C26: DESIGN.md §3.
#include <cuda_runtime.h>

#include "nbvh_device.cuh"
#include "nbvh_launch.h"

namespace nbvh {

// ------------------------------------------------------------------ traversal
__global__ void __launch_bounds__(128) k_traverse(TraverseArgs a) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r < a.n_rays;
    bool active = false;
    if (valid) {
        RayDev R = load_ray(a.rays, r);
        float lte[kListK], ltx[kListK];
        int lid[kListK], n = 0;
        bool more = false;
        collect_leaves<kListK>(a.cut, R, false, 0.f, 0, a.cap, lte, ltx, lid, n, a.err, true, &more);
        const int total = n;
#pragma unroll
        for (int j = 0; j < kListK; ++j)
            if (j < n) {
                a.lst_leaf[(int64_t)j * a.n_rays + r] = lid[j];
                a.lst_te[(int64_t)j * a.n_rays + r] = lte[j];
                a.lst_tx[(int64_t)j * a.n_rays + r] = ltx[j];
            }
        a.st.pos[r] = 0;
        a.st.base[r] = 0;
        a.st.nbuf[r] = n;
        a.st.more[r] = more ? 1 : 0;
        a.st.bt[r] = __int_as_float(0x7f800000);
        a.st.bte[r] = 0.f;
        a.st.bleaf[r] = -1;
        a.st.nq[r] = 0;
        // initial miss record (visibility 1 = no intersection)
        a.out.hit[r] = 0;
        a.out.t[r] = __int_as_float(0x7f800000);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a.out.normal[3 * r + k] = 0.f;
            a.out.albedo[3 * r + k] = 0.f;
        }
        if (a.out.leaf) a.out.leaf[r] = -1;
        if (total == 0 && a.out.n_queries) a.out.n_queries[r] = 0;
        active = total > 0;
    }
    // warp-aggregated append to the wave-0 active list
    const unsigned m = __ballot_sync(0xffffffffu, active);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(a.cnt_out, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (active) a.act_out[base + __popc(m & ((1u << lane) - 1u))] = (int)r;
}

// Debug traversal: full lists up to `cap` (may exceed K) by repeated resumption.
__global__ void __launch_bounds__(128) k_debug_traverse(DebugTraverseArgs a) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.n_rays) return;
    RayDev R = load_ray(a.rays, r);
    float lte[kListK], ltx[kListK];
    int lid[kListK];
    int written = 0, n = 0;
    bool has_after = false;
    float after_te = 0.f;
    int after_id = 0;
    int total = -1;
    while (true) {
        int rem = collect_leaves<kListK>(a.cut, R, has_after, after_te, after_id, a.k, lte, ltx, lid, n, a.err);
        if (total < 0) total = rem;
#pragma unroll
        for (int j = 0; j < kListK; ++j)
            if (j < n && written + j < a.cap) {
                a.leaf[r * a.cap + written + j] = lid[j];
                a.te[r * a.cap + written + j] = lte[j];
                a.tx[r * a.cap + written + j] = ltx[j];
            }
        if (n == 0) break;
#pragma unroll
        for (int j = 0; j < kListK; ++j)
            if (j == n - 1) { after_te = lte[j]; after_id = lid[j]; }
        written += n;
        has_after = true;
        if (written >= a.cap || rem <= n) break;
    }
    for (int j = written; j < a.cap; ++j) {
        a.leaf[r * a.cap + j] = -1;
        a.te[r * a.cap + j] = 0.f;
        a.tx[r * a.cap + j] = 0.f;
    }
    a.count[r] = total;
}

// ------------------------------------------------------------------ fused query wave
// Rare path, kept out of line so the wave kernel's register allocation is not sized for
// a second traversal: refill ray r's list with the leaves after its last key (C6).
__device__ __noinline__ int refill_list(const WaveArgs& a, int r, int nbuf) {
    const int64_t last = (int64_t)(nbuf - 1) * a.n_rays + r;
    const float kte = a.lst_te[last];
    const int kid = a.lst_leaf[last];
    RayDev R = load_ray(a.rays, r);
    float lte[kListK], ltx[kListK];
    int lid[kListK], n = 0;
    bool more = false;
    collect_leaves<kListK>(a.cut, R, true, kte, kid, a.cap, lte, ltx, lid, n, a.err, true, &more);
#pragma unroll
    for (int j = 0; j < kListK; ++j)
        if (j < n) {
            a.lst_leaf[(int64_t)j * a.n_rays + r] = lid[j];
            a.lst_te[(int64_t)j * a.n_rays + r] = lte[j];
            a.lst_tx[(int64_t)j * a.n_rays + r] = ltx[j];
        }
    a.st.nbuf[r] = n;
    a.st.more[r] = more ? 1 : 0;
    atomicAdd(a.n_refills, 1);
    return n;
}

struct QueryDesc {
    float o[3], d[3], te, tx;
    int ray, leaf, pos, valid;
};

template <int F, int D>
__global__ void __launch_bounds__(256, 2) k_query_wave(WaveArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_act = *a.cnt_in;
    // Tile size: 128 queries (one M=128 MMA tile) when the wave is large; sparse tail
    // waves spread their queries over every resident CTA instead (latency-bound).
    int qpt = (n_act + gridDim.x - 1) / gridDim.x;
    qpt = qpt > kTileQ ? kTileQ : (qpt < 8 ? 8 : qpt);
    const int n_tiles = (n_act + qpt - 1) / qpt;
    if ((int)blockIdx.x >= n_tiles) return;

    // shared-memory carve-up
    MlpSmem ms;
    __half* feat = reinterpret_cast<__half*>(smem_raw);                 // [128][D+8]
    ms.w0 = feat + kTileQ * (D + 8);
    ms.wh = ms.w0 + 64 * (D + 8);
    ms.wo = ms.wh + (a.m.hidden - 1) * 64 * 72;
    float* zt = reinterpret_cast<float*>(ms.wo + 8 * 72);              // [128][8]
    ms.b = zt + kTileQ * 8;
    QueryDesc* qd = reinterpret_cast<QueryDesc*>(ms.b + 64 * a.m.hidden + 8);

    stage_mlp(a.m, ms, tid, blockDim.x);

    const int L = a.g.L, n_pts = a.g.n_points;
    constexpr int kChunks = D / 8;
    const int chunks_per_point = (L * F) / 8;

    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int first = tile * qpt;
        const int nv = min(qpt, n_act - first);                       // valid queries in this tile
        // 1. query descriptors: ray, current list entry
        if (tid < nv) {
            const int r = a.act_in[first + tid];
            const int pos = a.st.pos[r];
            const int slot = pos - a.st.base[r];
            const int64_t li = (int64_t)slot * a.n_rays + r;
            QueryDesc q;
            q.valid = 1;
            q.ray = r;
            q.pos = pos;
            q.leaf = a.lst_leaf[li];
            q.te = a.lst_te[li];
            q.tx = a.lst_tx[li];
            float4 r0 = __ldg(a.rays + 2 * (int64_t)r), r1 = __ldg(a.rays + 2 * (int64_t)r + 1);
            q.o[0] = r0.x; q.o[1] = r0.y; q.o[2] = r0.z;
            q.d[0] = r1.x; q.d[1] = r1.y; q.d[2] = r1.z;
            qd[tid] = q;
        }
        __syncthreads();

        // 2. sample + encode: items (query, 16-byte chunk), query-minor so that a warp's
        //    lanes gather for neighbouring rays at the same level (coherent lines)
        for (int i = tid; i < nv * kChunks; i += blockDim.x) {
            const int q = i % nv, c = i / nv;
            const QueryDesc& Q = qd[q];
            const int p = c / chunks_per_point;
            const int l0 = ((c % chunks_per_point) * 8) / F;
            float x[3];
            segment_point(a.g, Q.o, Q.d, Q.te, Q.tx, p, n_pts, nullptr, x);
            *reinterpret_cast<uint4*>(feat + q * (D + 8) + c * 8) = encode_chunk<F>(a.g, x, l0, nullptr);
        }
        __syncthreads();

        // 3. MLP on tensor cores: warp w -> rows 16w..16w+15 (rows >= nv are ignored)
        if (warp * 16 < nv) mlp_rows16<D>(ms, a.m.hidden, feat, warp * 16, zt, lane);
        __syncthreads();

        // 4. decode, best-hit update, termination, compaction (one thread per query)
        if (warp * 32 < nv) {
            bool survive = false;
            int ray = -1;
            if (tid < nv) {
                const QueryDesc& Q = qd[tid];
                const int r = Q.ray;
                ray = r;
                const float* z = zt + tid * 8;
                int pos = Q.pos;
                if (a.z_trace && pos < a.trace_cap) {
                    float4* dst = reinterpret_cast<float4*>(a.z_trace + ((int64_t)r * a.trace_cap + pos) * 8);
                    dst[0] = make_float4(z[0], z[1], z[2], z[3]);
                    dst[1] = make_float4(z[4], z[5], z[6], z[7]);
                }
                const int nq = a.st.nq[r] + 1;
                float bt = a.st.bt[r], bte = a.st.bte[r];
                int bleaf = a.st.bleaf[r];
                const bool hit = z[0] < 0.0f;                          // sigmoid(z) < 0.5 (C13)
                if (hit) {
                    const float tl = sigmoid_f(z[1]);                  // local distance
                    const float t = __fadd_rn(Q.te, __fmul_rn(tl, __fsub_rn(Q.tx, Q.te)));
                    const bool better = bleaf < 0 || t < bt ||
                                        (t == bt && (Q.te < bte || (Q.te == bte && Q.leaf < bleaf)));
                    if (better) {
                        bt = t; bte = Q.te; bleaf = Q.leaf;
                        float nn = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(z[2], z[2]), __fmul_rn(z[3], z[3])),
                                                        __fmul_rn(z[4], z[4])));
                        nn = fmaxf(nn, 1e-6f);
                        a.out.hit[r] = 1;
                        a.out.t[r] = t;
#pragma unroll
                        for (int k = 0; k < 3; ++k) {
                            a.out.normal[3 * r + k] = __fdiv_rn(z[2 + k], nn);
                            a.out.albedo[3 * r + k] = sigmoid_f(z[5 + k]);
                        }
                        if (a.out.leaf) a.out.leaf[r] = Q.leaf;
                        a.st.bt[r] = bt;
                        a.st.bte[r] = bte;
                        a.st.bleaf[r] = bleaf;
                    }
                }
                ++pos;
                bool done = a.mode == 1 && hit;                         // R1: first confident hit (C5)
                if (!done) {
                    int base = a.st.base[r], nbuf = a.st.nbuf[r];
                    if (pos - base >= nbuf) {
                        if (!a.st.more[r]) {
                            done = true;                                 // every intersected leaf visited
                        } else {
                            // list exhausted, more leaves may remain: resume after the last key (C6)
                            nbuf = refill_list(a, r, nbuf);
                            base = pos;
                            a.st.base[r] = base;
                            done = nbuf == 0;
                        }
                    }
                    if (!done) {
                        const float next_te = a.lst_te[(int64_t)(pos - base) * a.n_rays + r];
                        done = bleaf >= 0 && next_te > bt;             // front-to-back termination
                    }
                }
                a.st.pos[r] = pos;
                a.st.nq[r] = nq;
                if (done && a.out.n_queries) a.out.n_queries[r] = nq;
                survive = !done;
            }
            const unsigned m = __ballot_sync(0xffffffffu, survive);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(a.cnt_out, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (survive) a.act_out[base + __popc(m & ((1u << lane) - 1u))] = ray;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ debug: encode points
template <int F>
__global__ void __launch_bounds__(128) k_debug_encode(DebugEncodeArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.m) return;
    const float x[3] = {a.pts[3 * i], a.pts[3 * i + 1], a.pts[3 * i + 2]};
    const int L = a.g.L;
    const int chunks = (L * F) / 8;
    uint32_t idx[64];
    for (int c = 0; c < chunks; ++c) {
        const int l0 = c * 8 / F;
        uint4 v = encode_chunk<F>(a.g, x, l0, a.index ? idx : nullptr);
        reinterpret_cast<uint4*>(a.feat + i * (int64_t)L * F)[c] = v;
        if (a.index)
            for (int j = 0; j < 8 / F * 8; ++j) a.index[(i * L + l0) * 8 + j] = idx[j];
    }
}

// ------------------------------------------------------------------ debug: MLP rows
template <int D>
__global__ void __launch_bounds__(256, 2) k_debug_mlp(DebugMlpArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    MlpSmem ms;
    __half* feat = reinterpret_cast<__half*>(smem_raw);
    ms.w0 = feat + kTileQ * (D + 8);
    ms.wh = ms.w0 + 64 * (D + 8);
    ms.wo = ms.wh + (a.m.hidden - 1) * 64 * 72;
    float* zt = reinterpret_cast<float*>(ms.wo + 8 * 72);
    ms.b = zt + kTileQ * 8;
    stage_mlp(a.m, ms, tid, blockDim.x);
    const int64_t n_tiles = (a.rows + kTileQ - 1) / kTileQ;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int i = tid; i < kTileQ * (D / 8); i += blockDim.x) {
            const int row = i / (D / 8), c = i % (D / 8);
            const int64_t gr = tile * kTileQ + row;
            uint4 v = gr < a.rows ? reinterpret_cast<const uint4*>(a.x + gr * D)[c] : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(feat + row * (D + 8) + c * 8) = v;
        }
        __syncthreads();
        mlp_rows16<D>(ms, a.m.hidden, feat, warp * 16, zt, lane);
        __syncthreads();
        for (int i = tid; i < kTileQ * 8; i += blockDim.x) {
            const int64_t gr = tile * kTileQ + i / 8;
            if (gr < a.rows) a.z[gr * 8 + (i % 8)] = zt[i];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ launchers
size_t wave_smem_bytes(int d_in, int hidden) {
    return (size_t)kTileQ * (d_in + 8) * 2 + (size_t)mlp_smem_halves(d_in, hidden) * 2 + kTileQ * 8 * 4 +
           (64 * hidden + 8) * 4 + kTileQ * sizeof(QueryDesc);
}
size_t mlp_smem_bytes(int d_in, int hidden) {
    return (size_t)kTileQ * (d_in + 8) * 2 + (size_t)mlp_smem_halves(d_in, hidden) * 2 + kTileQ * 8 * 4 +
           (64 * hidden + 8) * 4;
}

template <typename Kern>
static int resident_blocks(Kern k, int threads, size_t smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (per_sm > 0 ? per_sm : 1) * sms;
}

template <int F, int D>
static cudaError_t launch_wave_t(const WaveArgs& a, cudaStream_t s) {
    const size_t smem = wave_smem_bytes(D, a.m.hidden);
    static int grid_by_hidden[kMaxHidden + 1] = {0};
    int& grid = grid_by_hidden[a.m.hidden];
    if (!grid) grid = resident_blocks(k_query_wave<F, D>, 256, smem);
    k_query_wave<F, D><<<grid, 256, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_query_wave(const WaveArgs& a, cudaStream_t s) {
    const int F = a.g.F, D = a.m.d_in;
    if (F == 2 && D == 32) return launch_wave_t<2, 32>(a, s);
    if (F == 2 && D == 64) return launch_wave_t<2, 64>(a, s);
    if (F == 2 && D == 96) return launch_wave_t<2, 96>(a, s);
    if (F == 2 && D == 128) return launch_wave_t<2, 128>(a, s);
    if (F == 4 && D == 64) return launch_wave_t<4, 64>(a, s);
    if (F == 4 && D == 96) return launch_wave_t<4, 96>(a, s);
    if (F == 4 && D == 128) return launch_wave_t<4, 128>(a, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.n_rays + 127) / 128;
    k_traverse<<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_debug_traverse(const DebugTraverseArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.n_rays + 127) / 128;
    k_debug_traverse<<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_debug_encode(const DebugEncodeArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.m + 127) / 128;
    if (a.g.F == 2) k_debug_encode<2><<<(unsigned)blocks, 128, 0, s>>>(a);
    else k_debug_encode<4><<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

template <int D>
static cudaError_t launch_mlp_t(const DebugMlpArgs& a, cudaStream_t s) {
    const size_t smem = mlp_smem_bytes(D, a.m.hidden);
    int grid = resident_blocks(k_debug_mlp<D>, 256, smem);
    const int64_t tiles = (a.rows + kTileQ - 1) / kTileQ;
    if (tiles < grid) grid = (int)tiles;
    if (grid < 1) grid = 1;
    k_debug_mlp<D><<<grid, 256, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_debug_mlp(const DebugMlpArgs& a, cudaStream_t s) {
    switch (a.m.d_in) {
        case 32: return launch_mlp_t<32>(a, s);
        case 64: return launch_mlp_t<64>(a, s);
        case 96: return launch_mlp_t<96>(a, s);
        case 128: return launch_mlp_t<128>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace nbvh
