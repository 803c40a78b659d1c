// nbvh_mlp_tc.cu — the decoder MLP (D_in -> 64 (ReLU) x H -> 8) as a batched
// tcgen05 / TMEM / TMA kernel: the "MLP on tensor cores" of the north star measured on its own
// (nbvh_mlp_forward).  Streaming X (m x D_in fp16) is most of its bytes, so the design goal is
// to keep enough X loads in flight to run at HBM speed while the tensor core works:
// one persistent CTA per SM runs kSlots independent 128-row tiles at once; each slot owns a
// 64-column TMEM accumulator, a hidden-activation buffer and (stage j % nst, nst a multiple of
// kSlots) the X stages its tiles land in; a stage is refilled by TMA as soon as layer 0 of its
// tile has read it, so the load hides under that tile's hidden layers and the other slots' work.
//   warp 4*kSlots (one lane)    TMA producer.  D_in % 64 == 0: two 64-column boxes per tile
//                               in the 128-byte-swizzle layout (8-row x 128-byte atoms, the
//                               MMA reads it through SWIZZLE_128B descriptors); otherwise one
//                               {8 halves, 128 rows} box per 16-byte K-group (no-swizzle
//                               canonical core matrices).  Rows past m are zero-filled by TMA.
//   warp 4*kSlots+1+g           MMA issuer of slot g: whole warp converged, one elected lane
//                               issues (operands stay in uniform registers); one issuer per
//                               slot, since one warp issuing every slot's ~24 MMAs per tile was
//                               the limit.  tcgen05.mma.cta_group::1.kind::f16, M = 128, N = 64
//                               (16 for the output layer), fp32 accumulator in TMEM, commits to
//                               mbarriers.
//   warps 4g..4g+3              epilogue of slot g: tcgen05.ld of the row's accumulator
//                               (warp <-> TMEM lanes 32(w%4)..+31 <-> rows), ReLU + fp16 pack
//                               in one instruction per pair (cvt.rn.relu.f16x2.f32), 16-byte
//                               stores into the slot's H buffer (generic -> async proxy fence);
//                               z stored for the output layer
// Biases ride on the tensor core: every A tile carries one extra K=16 step whose first two
// columns are 1 and whose B columns hold the bias split as hi + lo fp16 (b = hi + lo to ~2^-22
// relative), so the accumulator already holds W x + b.
// The CTA's j-th tile is blockIdx.x + j * gridDim.x and runs in slot j % kSlots.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "nbvh_capi_internal.h"
#include "nbvh_tcgen05.cuh"

namespace nbvh {

constexpr int kSlots = 3;
constexpr int kMaxStages = 2 * kSlots;
constexpr uint32_t kTmemCols = 256;     // power of two >= 64 * kSlots

struct MlpTcArgs {
    const __half* W;     // layers concatenated [out][in] fp16 (inference copy)
    const float* b;      // biases fp32
    float* z;            // [m][8] out
    int64_t m;
    int32_t hidden;
    int32_t nst;         // X stages, a multiple of kSlots
};

constexpr int kKgH = 64 / 8 + 2;   // K-groups (16 B = 8 halves) of an H buffer / hidden W: data + bias step

__host__ __device__ constexpr uint32_t mlp_tc_stage_smem(int D) { return (uint32_t)(128 * (D / 8 + 2) * 16); }
__host__ __device__ constexpr uint32_t mlp_tc_fixed_smem(int D, int H) {
    return (uint32_t)(kSlots * 128 * kKgH * 16          // H buffers
                      + 64 * (D / 8 + 2) * 16            // W0 (+ bias columns)
                      + (H - 1) * 64 * kKgH * 16
                      + 16 * kKgH * 16                   // W_out padded to 16 rows
                      + 8 * (2 * kMaxStages + 2 * kSlots) + 16);   // barriers + TMEM slot
}

__device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

constexpr int kMlpWarps = 5 * kSlots + 1;

template <int D, int H>
__global__ void __launch_bounds__(kMlpWarps * 32, 1) k_mlp_tc(const __grid_constant__ CUtensorMap tmx, MlpTcArgs a) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    // 128-byte-swizzled X stages need 1024-byte alignment (the launch requests 1 KB extra)
    unsigned char* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
    constexpr bool kSw = D % 64 == 0;                         // X in 128-byte-swizzled 64-column boxes
    constexpr int KX = D / 8 + 2;                             // K-groups of an X stage; bias step at D/8
    const int nst = a.nst;
    unsigned char* sX = sm;                                   // nst x [KX][128 rows][16 B]
    unsigned char* sH = sX + nst * 128 * KX * 16;             // kSlots x [kKgH][128][16 B]
    unsigned char* sW0 = sH + kSlots * 128 * kKgH * 16;       // [KX][64][16 B]
    unsigned char* sWh = sW0 + 64 * KX * 16;                  // [H-1][kKgH][64][16 B]
    unsigned char* sWo = sWh + (H - 1) * 64 * kKgH * 16;      // [kKgH][16][16 B]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sWo + 16 * kKgH * 16);
    uint64_t* x_full = bar;                                   // [nst] X landed
    uint64_t* x_empty = bar + kMaxStages;                     // [nst] layer 0 done with it
    uint64_t* acc_full = bar + 2 * kMaxStages;                // [kSlots] a layer's MMAs done
    uint64_t* h_ready = acc_full + kSlots;                    // [kSlots] epilogue done with a layer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_ready + kSlots);
    const int tid = threadIdx.x, warp = tid >> 5;

    // Stage W [N][K] (+ bias as two extra K columns: hi, lo) in the K-major canonical layout:
    // element (n, k) at (k/8) * (Npad*16) + n*16 + (k%8)*2 bytes.
    auto stage_w = [&](unsigned char* dst, const __half* src, const float* bias, int N, int K, int Npad) {
        const int kg = K / 8 + 2;
        for (int i = tid; i < Npad * kg; i += blockDim.x) {
            const int n = i / kg, g = i % kg;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (n < N) {
                if (g < K / 8) {
                    v = *reinterpret_cast<const uint4*>(src + (int64_t)n * K + g * 8);
                } else if (g == K / 8) {
                    const __half hi = __float2half_rn(bias[n]);
                    const __half lo = __float2half_rn(bias[n] - __half2float(hi));
                    v.x = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
                }
            }
            *reinterpret_cast<uint4*>(dst + g * (Npad * 16) + n * 16) = v;
        }
    };
    stage_w(sW0, a.W, a.b, 64, D, 64);
    for (int l = 0; l < H - 1; ++l)
        stage_w(sWh + l * 64 * kKgH * 16, a.W + 64 * D + (int64_t)l * 64 * 64, a.b + 64 * (l + 1), 64, 64, 64);
    stage_w(sWo, a.W + 64 * D + (int64_t)(H - 1) * 64 * 64, a.b + 64 * H, 8, 64, 16);
    // the bias step of every A buffer: columns (1, 1, 0, ...), then a zero K-group
    const uint4 ones = make_uint4(0x3C003C00u, 0u, 0u, 0u);     // fp16 1.0, 1.0
    for (int i = tid; i < (nst + kSlots) * 128; i += blockDim.x) {
        const int buf = i / 128, r = i % 128;
        unsigned char* A = buf < nst ? sX + buf * 128 * KX * 16 + (D / 8) * 2048
                                     : sH + (buf - nst) * 128 * kKgH * 16 + 8 * 2048;
        *reinterpret_cast<uint4*>(A + r * 16) = ones;
        *reinterpret_cast<uint4*>(A + 2048 + r * 16) = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        for (int i = 0; i < nst; ++i) {
            tc::mbar_init(x_full + i, 1);
            tc::mbar_init(x_empty + i, 1);
        }
        for (int g = 0; g < kSlots; ++g) {
            tc::mbar_init(acc_full + g, 1);
            tc::mbar_init(h_ready + g, 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 0) tc::tmem_alloc<kTmemCols>(tmem_slot);
    tc::fence_proxy_async();                                  // staged weights / bias steps -> tensor core
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t n_tiles = (a.m + 127) / 128;
    const int n_mine = n_tiles > blockIdx.x ? (int)((n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;

    if (warp == 4 * kSlots) {
        // ---------------- TMA producer: tile j into ring stage j % nst once layer 0 of tile
        // j - nst has read it
        if ((tid & 31) == 0) {
            tc::prefetch_tmap(&tmx);
            int st = 0;
            uint32_t use = 0;
            for (int j = 0; j < n_mine; ++j) {
                if (use > 0) tc::mbar_wait(x_empty + st, (use - 1) & 1);
                tc::mbar_arrive_expect_tx(x_full + st, 128 * D * 2);
                unsigned char* dst = sX + st * 128 * KX * 16;
                const int row0 = (int)((blockIdx.x + (int64_t)j * gridDim.x) * 128);
                if constexpr (kSw) {                       // 64-column swizzled boxes
                    for (int c = 0; c < D / 64; ++c) tc::tma_load_2d(dst + c * 16384, &tmx, c * 64, row0, x_full + st);
                } else {                                   // one box per 16-byte K-group
                    for (int kg = 0; kg < D / 8; ++kg)
                        tc::tma_load_2d(dst + kg * 2048, &tmx, kg * 8, row0, x_full + st);
                }
                if (++st == nst) {
                    st = 0;
                    ++use;
                }
            }
        }
    } else if (warp > 4 * kSlots) {
        // ---------------- MMA issuer of slot g: its tiles, layer by layer.  Descriptors are
        // built once and stepped by constant adds (the 14-bit start-address field never
        // carries: smem < 256 KB).
        const int g = warp - 4 * kSlots - 1;
        constexpr uint32_t id64 = tc::idesc_f16(128, 64, false, false);
        constexpr uint32_t id16 = tc::idesc_f16(128, 16, false, false);
        const uint64_t dW0 = tc::smem_desc(tc::smem_u32(sW0), 1024, 128);
        const uint64_t dWh = tc::smem_desc(tc::smem_u32(sWh), 1024, 128);
        const uint64_t dWo = tc::smem_desc(tc::smem_u32(sWo), 256, 128);
        const uint64_t dX = tc::smem_desc(tc::smem_u32(sX), 2048, 128);
        const uint64_t dXsw = tc::smem_desc_sw128(tc::smem_u32(sX), 1024);
        const uint64_t dH = tc::smem_desc(tc::smem_u32(sH + g * 128 * kKgH * 16), 2048, 128);
        const uint32_t acc = tmem + (uint32_t)(g * 64);
        uint32_t use = 0;
        for (int j = g; j < n_mine; j += kSlots, ++use) {
            // h_ready completes H + 1 times per tile; wait for the previous tile's last one
            if (use > 0) tc::mbar_wait(h_ready + g, (use * (H + 1) - 1) & 1);
            const int st = j % nst;
            tc::mbar_wait(x_full + st, (uint32_t)(j / nst) & 1);
            tc::fence_after();
            const uint64_t dXs = dX + (uint64_t)(st * 128 * KX);   // 16-byte units
            if constexpr (kSw) {
                const uint64_t dXw = dXsw + (uint64_t)(st * 128 * KX);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)                // atom kk/4, 32 bytes per K step
                    tc::mma_f16_elect(acc, dXw + (kk / 4) * 1024 + (kk % 4) * 2, dW0 + kk * 128, id64, kk > 0);
                tc::mma_f16_elect(acc, dXs + (D / 16) * 256, dW0 + (D / 16) * 128, id64, 1);   // bias
            } else {
#pragma unroll
                for (int kk = 0; kk < D / 16 + 1; ++kk)            // last step: bias
                    tc::mma_f16_elect(acc, dXs + kk * 256, dW0 + kk * 128, id64, kk > 0);
            }
            tc::commit_elect(x_empty + st);                        // X stage free
            tc::commit_elect(acc_full + g);
#pragma unroll
            for (int l = 1; l <= H; ++l) {
                tc::mbar_wait(h_ready + g, (uint32_t)((use * (H + 1) + l - 1) & 1));
                tc::fence_after();
                if (l < H) {
#pragma unroll
                    for (int kk = 0; kk < 5; ++kk)                 // last step: bias
                        tc::mma_f16_elect(acc, dH + kk * 256, dWh + (l - 1) * 64 * kKgH + kk * 128, id64, kk > 0);
                } else {
#pragma unroll
                    for (int kk = 0; kk < 5; ++kk)
                        tc::mma_f16_elect(acc, dH + kk * 256, dWo + kk * 32, id16, kk > 0);
                }
                tc::commit_elect(acc_full + g);
            }
        }
    } else {
        // ---------------- epilogue of slot g = warp / 4: row 32*(warp%4) + lane
        const int g = warp >> 2, q = warp & 3;
        const int row = q * 32 + (tid & 31);
        unsigned char* hb = sH + g * 128 * kKgH * 16;
        const uint32_t acc = tmem + (uint32_t)(g * 64);
        uint32_t acc_n = 0;
        for (int j = g; j < n_mine; j += kSlots) {
            const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
            for (int l = 0; l <= H; ++l) {
                tc::mbar_wait(acc_full + g, (acc_n++) & 1);
                tc::fence_after();
                if (l < H) {
                    float v[32], w[32];
                    tc::ld32(acc, (uint32_t)(q * 32), 0u, v);
                    tc::ld32(acc, (uint32_t)(q * 32), 32u, w);
                    tc::fence_before();
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        *reinterpret_cast<uint4*>(hb + k * 2048 + row * 16) =
                            make_uint4(relu_pack(v[8 * k], v[8 * k + 1]), relu_pack(v[8 * k + 2], v[8 * k + 3]),
                                       relu_pack(v[8 * k + 4], v[8 * k + 5]), relu_pack(v[8 * k + 6], v[8 * k + 7]));
                        *reinterpret_cast<uint4*>(hb + (k + 4) * 2048 + row * 16) =
                            make_uint4(relu_pack(w[8 * k], w[8 * k + 1]), relu_pack(w[8 * k + 2], w[8 * k + 3]),
                                       relu_pack(w[8 * k + 4], w[8 * k + 5]), relu_pack(w[8 * k + 6], w[8 * k + 7]));
                    }
                    tc::fence_proxy_async();
                    tc::mbar_arrive(h_ready + g);
                } else {
                    float v[16];
                    tc::ld16(acc, (uint32_t)(q * 32), 0u, v);
                    tc::fence_before();
                    tc::mbar_arrive(h_ready + g);                    // accumulator free for the next tile
                    const int64_t r = t * 128 + row;
                    if (r < a.m) {
                        float4* dst = reinterpret_cast<float4*>(a.z + r * 8);
                        dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                        dst[1] = make_float4(v[4], v[5], v[6], v[7]);
                    }
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<kTmemCols>(tmem);
}

// ---- tensor map for X [m][D] fp16: box {8 halves (one K-group), 128 rows}
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

template <int D, int H>
static cudaError_t launch_mlp_tc_t(const __half* x, int64_t m, const MlpTcArgs& a, cudaStream_t s) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)m};
    const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    constexpr bool kSw = D % 64 == 0;
    const cuuint32_t box[2] = {kSw ? 64u : 8u, 128};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, kSw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    // as many X stages as fit next to the H buffers and weights
    static int budget = 0;                                    // opt-in dynamic smem minus static
    if (!budget) {
        int dev = 0, optin = 0;
        cudaFuncAttributes fa{};
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (cudaFuncGetAttributes(&fa, k_mlp_tc<D, H>) != cudaSuccess) return cudaErrorInvalidDeviceFunction;
        budget = optin - (int)fa.sharedSizeBytes;
        cudaFuncSetAttribute(k_mlp_tc<D, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, budget);
    }
    const uint32_t fixed = mlp_tc_fixed_smem(D, H), stage = mlp_tc_stage_smem(D);
    int nst = (int)(((uint32_t)budget - 1024u - fixed) / stage);
    // a multiple of kSlots, so each stage only ever serves one slot and no barrier waiter can
    // run more than one phase ahead (parity waits are ambiguous beyond that)
    nst = nst > kMaxStages ? kMaxStages : nst;
    nst -= nst % kSlots;
    if (nst < kSlots) return cudaErrorInvalidConfiguration;
    MlpTcArgs b = a;
    b.nst = nst;
    const uint32_t smem = fixed + (uint32_t)nst * stage + 1024u;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (m + 127) / 128;
    const int grid = (int)(tiles < sms ? tiles : sms);
    k_mlp_tc<D, H><<<grid, kMlpWarps * 32, smem, s>>>(tm, b);
    return cudaGetLastError();
}

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_mlp_forward(nbvh_ctx* c, const uint16_t* x, int64_t m, float* z, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (m < 0 || (m > 0 && (!x || !z))) return fail(c, NBVH_EINVAL, "mlp_forward: bad args");
    if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(z) & 15))
        return fail(c, NBVH_EINVAL, "mlp_forward: x and z must be 16-byte aligned");
    if (m == 0) return NBVH_OK;
    MlpTcArgs a{};
    a.W = c->d_W16;
    a.b = c->d_params + c->n_table + c->n_W;
    a.z = z;
    a.m = m;
    a.hidden = c->cfg.hidden_layers;
    const __half* xh = reinterpret_cast<const __half*>(x);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e;
    switch (c->d_in * 8 + a.hidden) {
#define NBVH_MLP_CASE(D, H) \
    case D * 8 + H: e = launch_mlp_tc_t<D, H>(xh, m, a, s); break;
#define NBVH_MLP_CASES(D) NBVH_MLP_CASE(D, 1) NBVH_MLP_CASE(D, 2) NBVH_MLP_CASE(D, 3) NBVH_MLP_CASE(D, 4)
        NBVH_MLP_CASES(32)
        NBVH_MLP_CASES(64)
        NBVH_MLP_CASES(96)
        NBVH_MLP_CASES(128)
#undef NBVH_MLP_CASES
#undef NBVH_MLP_CASE
        default: return fail(c, NBVH_EINVAL, "mlp_forward: unsupported D_in / hidden layers");
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "mlp_forward");
    return NBVH_OK;
}
