// nbvh_probe.cu — the random-gather roofline of SURVEY §8(d) ("Q2+Q3 encode: L2 gather;
// roofline denominator: measured L2 random-sector read peak, §7 step 0").  A persistent grid
// reads uniformly random entries of an L2-resident table (4-byte entries: one sector per load,
// the hashed-level gathers; 32-byte entries: the corner-packed dense records) with 8
// independent address chains per thread, so the number is bounded by the memory system, not
// by latency.  The bench turns it into sectors/s and reports the query kernel's L2 read-sector
// rate (from its ncu profile) as a fraction of it.
#include <cuda_runtime.h>

#include "nbvh_capi_internal.h"

namespace nbvh {

template <int kBytes>
__global__ void __launch_bounds__(256) k_gather_probe(const uint32_t* __restrict__ tab, uint32_t mask,
                                                      int64_t per_thread, uint32_t seed, uint32_t* sink) {
    constexpr int kChains = 8;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) st[c] = (tid * 0x9E3779B9u) ^ (seed + 0x85EBCA6Bu * (uint32_t)(c + 1));
    uint32_t acc = 0;
    for (int64_t i = 0; i < per_thread; i += kChains) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            st[c] = st[c] * 1664525u + 1013904223u;              // LCG; address independent of data
            const uint32_t e = (st[c] >> 7) & mask;
            if constexpr (kBytes == 4) {
                acc ^= __ldg(tab + e);
            } else {
                uint32_t r[8];
                asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                               "=r"(r[7])
                             : "l"(tab + 8ull * e));
                acc ^= r[0] ^ r[1] ^ r[2] ^ r[3] ^ r[4] ^ r[5] ^ r[6] ^ r[7];
            }
        }
    }
    sink[tid] = acc;
}

// The same 4-byte random gathers through the TEX pipe (tex1Dfetch on a texture object over the
// table, as k_query_warp's hashed levels), or half of the chains on each pipe (kMixed).
template <bool kMixed>
__global__ void __launch_bounds__(256) k_gather_probe_tex(cudaTextureObject_t tex, const uint32_t* __restrict__ tab,
                                                          uint32_t mask, int64_t per_thread, uint32_t seed,
                                                          uint32_t* sink) {
    constexpr int kChains = 8;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) st[c] = (tid * 0x9E3779B9u) ^ (seed + 0x85EBCA6Bu * (uint32_t)(c + 1));
    uint32_t acc = 0;
    for (int64_t i = 0; i < per_thread; i += kChains) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            st[c] = st[c] * 1664525u + 1013904223u;
            const uint32_t e = (st[c] >> 7) & mask;
            if (kMixed && (c & 1)) acc ^= __ldg(tab + e);
            else acc ^= tex1Dfetch<unsigned int>(tex, (int)e);
        }
    }
    sink[tid] = acc;
}

// Random fp32 reductions into an L2-resident table (the T7 hash-grid scatter's roofline,
// "measured L2 atomic peak"): kVec = 1 -> red.global.add.f32, 2 ->
// red.global.add.v2.f32 (8-byte aligned pairs, what k_train_bwd issues for F = 2), 4 ->
// red.global.add.v4.f32 (16-byte aligned quads: two F = 2 entries).
template <int kVec>
__global__ void __launch_bounds__(256) k_atomic_probe(float* __restrict__ tab, uint32_t mask, int64_t per_thread,
                                                      uint32_t seed) {
    constexpr int kChains = 8;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t st[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) st[c] = (tid * 0x9E3779B9u) ^ (seed + 0x85EBCA6Bu * (uint32_t)(c + 1));
    for (int64_t i = 0; i < per_thread; i += kChains) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            st[c] = st[c] * 1664525u + 1013904223u;
            const uint32_t e = (st[c] >> 7) & mask;
            if constexpr (kVec == 1)
                asm volatile("red.global.add.f32 [%0], %1;" ::"l"(tab + e), "f"(1.0f) : "memory");
            else if constexpr (kVec == 2)
                asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(tab + 2ull * e), "f"(1.0f), "f"(1.0f)
                             : "memory");
            else
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(tab + 4ull * e), "f"(1.0f),
                             "f"(1.0f), "f"(1.0f), "f"(1.0f)
                             : "memory");
        }
    }
}

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_atomic_probe(float* d_table, int64_t table_bytes, int32_t vec, int64_t n_ops,
                                         uint32_t seed, int64_t* n_done, void* stream) {
    if (!d_table || (vec != 1 && vec != 2 && vec != 4) || n_ops <= 0 || (reinterpret_cast<uintptr_t>(d_table) & 15))
        return NBVH_EINVAL;
    const int64_t n_entries = table_bytes / (4 * vec);
    if (n_entries < 1 || (n_entries & (n_entries - 1))) return NBVH_EINVAL;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t threads = (int64_t)sms * 8 * 256;
    int64_t per_thread = (n_ops + threads - 1) / threads;
    per_thread = (per_thread + 7) / 8 * 8;
    const uint32_t mask = (uint32_t)(n_entries - 1);
    cudaStream_t s = (cudaStream_t)stream;
    if (vec == 1)
        k_atomic_probe<1><<<sms * 8, 256, 0, s>>>(d_table, mask, per_thread, seed);
    else if (vec == 2)
        k_atomic_probe<2><<<sms * 8, 256, 0, s>>>(d_table, mask, per_thread, seed);
    else
        k_atomic_probe<4><<<sms * 8, 256, 0, s>>>(d_table, mask, per_thread, seed);
    if (n_done) *n_done = per_thread * threads;
    return cudaGetLastError() == cudaSuccess ? NBVH_OK : NBVH_ECUDA;
}

extern "C" nbvh_status nbvh_gather_probe(const void* d_table, int64_t table_bytes, int32_t entry_bytes,
                                         int64_t n_gathers, uint32_t seed, uint32_t* d_sink, int64_t sink_len,
                                         int64_t* n_done, void* stream) {
    if (!d_table || !d_sink || (entry_bytes != 4 && entry_bytes != 32) || table_bytes < entry_bytes ||
        n_gathers <= 0 || (reinterpret_cast<uintptr_t>(d_table) & 31))
        return NBVH_EINVAL;
    const int64_t n_entries = table_bytes / entry_bytes;
    if (n_entries & (n_entries - 1)) return NBVH_EINVAL;        // power of two (mask addressing)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t threads = (int64_t)sms * 8 * 256;
    if (sink_len < threads) return NBVH_EINVAL;
    int64_t per_thread = (n_gathers + threads - 1) / threads;
    per_thread = (per_thread + 7) / 8 * 8;
    const uint32_t mask = (uint32_t)(n_entries - 1);
    cudaStream_t s = (cudaStream_t)stream;
    if (entry_bytes == 4)
        k_gather_probe<4><<<sms * 8, 256, 0, s>>>(static_cast<const uint32_t*>(d_table), mask, per_thread, seed, d_sink);
    else
        k_gather_probe<32><<<sms * 8, 256, 0, s>>>(static_cast<const uint32_t*>(d_table), mask, per_thread, seed, d_sink);
    if (n_done) *n_done = per_thread * threads;
    return cudaGetLastError() == cudaSuccess ? NBVH_OK : NBVH_ECUDA;
}

extern "C" nbvh_status nbvh_gather_probe_tex(const void* d_table, int64_t table_bytes, int32_t mixed,
                                             int64_t n_gathers, uint32_t seed, uint32_t* d_sink, int64_t sink_len,
                                             int64_t* n_done, void* stream) {
    if (!d_table || !d_sink || table_bytes < 4 || n_gathers <= 0 || (reinterpret_cast<uintptr_t>(d_table) & 31) ||
        (mixed != 0 && mixed != 1))
        return NBVH_EINVAL;
    const int64_t n_entries = table_bytes / 4;
    if ((n_entries & (n_entries - 1)) || n_entries > ((int64_t)1 << 27)) return NBVH_EINVAL;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t threads = (int64_t)sms * 8 * 256;
    if (sink_len < threads) return NBVH_EINVAL;
    int64_t per_thread = (n_gathers + threads - 1) / threads;
    per_thread = (per_thread + 7) / 8 * 8;
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<void*>(d_table);
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned int>();
    rd.res.linear.sizeInBytes = (size_t)table_bytes;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    td.filterMode = cudaFilterModePoint;
    td.addressMode[0] = cudaAddressModeClamp;
    cudaTextureObject_t tex = 0;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) {
        cudaGetLastError();
        return NBVH_ECUDA;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t mask = (uint32_t)(n_entries - 1);
    const uint32_t* tab = static_cast<const uint32_t*>(d_table);
    if (mixed) k_gather_probe_tex<true><<<sms * 8, 256, 0, s>>>(tex, tab, mask, per_thread, seed, d_sink);
    else k_gather_probe_tex<false><<<sms * 8, 256, 0, s>>>(tex, tab, mask, per_thread, seed, d_sink);
    cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(s);               // the texture object must outlive the launch
    cudaDestroyTextureObject(tex);
    if (n_done) *n_done = per_thread * threads;
    return e == cudaSuccess ? NBVH_OK : NBVH_ECUDA;
}
