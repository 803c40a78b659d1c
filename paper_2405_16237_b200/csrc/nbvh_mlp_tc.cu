// nbvh_mlp_tc.cu — the decoder MLP (D_in -> 64 (ReLU) x H -> 8) as a batched
// tcgen05 / TMEM / TMA kernel: the "MLP on tensor cores" of the north star measured on its own
// (nbvh_mlp_forward).  Streaming X (m x D_in fp16) is most of its bytes, so the design goal is
// to keep enough X loads in flight to run at HBM speed while the tensor core works:
// one persistent CTA per SM runs NS independent 128-row tiles at once (NS = 5 for D_in >= 64,
// 3 below); each slot owns a 64-column TMEM accumulator, an X stage (stage j % nst) and a
// hidden-activation buffer — for D_in >= 64 the hidden activations overwrite the slot's X
// stage once layer 0 has read it (see mlp_alias), which is what makes room for five slots.
//   warp 4*NS (one lane)    TMA producer.  D_in % 64 == 0: two 64-column boxes per tile in the
//                           128-byte-swizzle layout (8-row x 128-byte atoms, read by the MMA
//                           through SWIZZLE_128B descriptors); otherwise one {8 halves, 128
//                           rows} box per 16-byte K-group (no-swizzle canonical core
//                           matrices).  Rows past m are zero-filled by TMA.
//   warp 4*NS+1+g           MMA issuer of slot g: whole warp converged, one elected lane issues
//                           (operands stay in uniform registers); one issuer per slot, since
//                           one warp issuing every slot's ~24 MMAs per tile was the limit.
//                           tcgen05.mma.cta_group::1.kind::f16, M = 128, N = 64 (16 for the
//                           output layer), fp32 accumulator in TMEM, commits to mbarriers.
//   warps 4g..4g+3          epilogue of slot g: tcgen05.ld of the row's accumulator (warp <->
//                           TMEM lanes 32(w%4)..+31 <-> rows), ReLU + fp16 pack in one
//                           instruction per pair (cvt.rn.relu.f16x2.f32), 16-byte stores into
//                           the slot's H buffer (generic -> async proxy fence); z stored for
//                           the output layer.
// Biases ride on the tensor core: every layer has one extra K=16 step whose A columns are
// (1, 1, 0, ...) and whose B columns hold the bias split as hi + lo fp16 (b = hi + lo to
// ~2^-22 relative), so the accumulator already holds W x + b.
// The CTA's j-th tile is blockIdx.x + j * gridDim.x and runs in slot j % NS.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "nbvh_capi_internal.h"
#include "nbvh_tcgen05.cuh"

namespace nbvh {

struct MlpTcArgs {
    const __half* W;     // layers concatenated [out][in] fp16 (inference copy)
    const float* b;      // biases fp32
    float* z;            // [m][8] out
    int64_t m;
    int32_t hidden;
    int32_t nst;         // X stages (a multiple of the slot count; = slots when aliased)
};

constexpr int kKgH = 64 / 8 + 2;   // K-groups (16 B = 8 halves) of an H buffer / hidden W: data + bias step

// Two buffer schemes (template kAlias):
//  * separate (D_in < 64): per slot an X stage with its own bias K-step columns and an H
//    buffer; the next X tile of a slot lands while its hidden layers run;
//  * aliased (D_in >= 64): the hidden activations overwrite the slot's X stage once layer 0
//    has consumed it (one ones-tile serves every bias step), so the same shared memory holds
//    more slots; a slot's next X tile is fetched after its output layer.
__host__ __device__ constexpr int mlp_slots(int D) { return D >= 64 ? 5 : 3; }
__host__ __device__ constexpr bool mlp_alias(int D) { return D >= 64; }
__host__ __device__ constexpr uint32_t mlp_tmem_cols(int ns) { return ns * 64 <= 128 ? 128 : (ns * 64 <= 256 ? 256 : 512); }
__host__ __device__ constexpr uint32_t mlp_tc_stage_smem(int D) {
    return (uint32_t)(128 * (D / 8 + (mlp_alias(D) ? 0 : 2)) * 16);
}
__host__ __device__ constexpr uint32_t mlp_tc_fixed_smem(int D, int H) {
    return (uint32_t)((mlp_alias(D) ? 128 * 2 * 16 : mlp_slots(D) * 128 * kKgH * 16)   // ones tile | H buffers
                      + 64 * (D / 8 + 2) * 16            // W0 (+ bias columns)
                      + (H - 1) * 64 * kKgH * 16
                      + 16 * kKgH * 16                   // W_out padded to 16 rows
                      + 8 * (2 * 2 * mlp_slots(D) + 2 * mlp_slots(D)) + 16);   // barriers + TMEM slot
}

__device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int D, int H>
__global__ void __launch_bounds__((5 * mlp_slots(D) + 1) * 32, 1)
    k_mlp_tc(const __grid_constant__ CUtensorMap tmx, MlpTcArgs a) {
    constexpr int NS = mlp_slots(D);
    constexpr bool kAlias = mlp_alias(D);
    constexpr int kMaxStages = 2 * NS;
    constexpr uint32_t kTmemCols = mlp_tmem_cols(NS);
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    // 128-byte-swizzled X stages need 1024-byte alignment (the launch requests 1 KB extra)
    unsigned char* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
    constexpr bool kSw = D % 64 == 0;                         // X in 128-byte-swizzled 64-column boxes
    constexpr int KX = D / 8 + (kAlias ? 0 : 2);              // K-groups of an X stage (+ bias step)
    constexpr int KW0 = D / 8 + 2;                            // K-groups of W0 (+ bias columns)
    const int nst = a.nst;
    unsigned char* sX = sm;                                   // nst x [KX][128 rows][16 B]
    unsigned char* sAux = sX + nst * 128 * KX * 16;           // aliased: ones tile [2][128][16 B];
                                                              // separate: NS x H [kKgH][128][16 B]
    unsigned char* sW0 = sAux + (kAlias ? 128 * 2 * 16 : NS * 128 * kKgH * 16);   // [KW0][64][16 B]
    unsigned char* sWh = sW0 + 64 * KW0 * 16;                 // [H-1][kKgH][64][16 B]
    unsigned char* sWo = sWh + (H - 1) * 64 * kKgH * 16;      // [kKgH][16][16 B]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sWo + 16 * kKgH * 16);
    uint64_t* x_full = bar;                                   // [nst] X landed
    uint64_t* x_empty = bar + kMaxStages;                     // [nst] X stage free again
    uint64_t* acc_full = bar + 2 * kMaxStages;                // [NS] a layer's MMAs done
    uint64_t* h_ready = acc_full + NS;                        // [NS] epilogue done with a layer
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(h_ready + NS);
    const int tid = threadIdx.x, warp = tid >> 5;
    auto h_buf = [&](int g) { return kAlias ? sX + g * 128 * KX * 16 : sAux + g * 128 * kKgH * 16; };

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
    // bias K-step A columns: (1, 1, 0, ...) then a zero K-group -- one shared tile (aliased) or
    // after the data groups of every X stage and H buffer (separate)
    const uint4 ones = make_uint4(0x3C003C00u, 0u, 0u, 0u);     // fp16 1.0, 1.0
    const int n_bias_tiles = kAlias ? 1 : nst + NS;
    for (int i = tid; i < n_bias_tiles * 128; i += blockDim.x) {
        const int buf = i / 128, r = i % 128;
        unsigned char* A = kAlias ? sAux
                                  : (buf < nst ? sX + buf * 128 * KX * 16 + (D / 8) * 2048
                                               : sAux + (buf - nst) * 128 * kKgH * 16 + 8 * 2048);
        *reinterpret_cast<uint4*>(A + r * 16) = ones;
        *reinterpret_cast<uint4*>(A + 2048 + r * 16) = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        for (int i = 0; i < nst; ++i) {
            tc::mbar_init(x_full + i, 1);
            tc::mbar_init(x_empty + i, 1);
        }
        for (int g = 0; g < NS; ++g) {
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

    if (warp == 4 * NS) {
        // ---------------- TMA producer: tile j into stage j % nst once that stage is free
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
    } else if (warp > 4 * NS) {
        // ---------------- MMA issuer of slot g: its tiles, layer by layer.  Descriptors are
        // built once and stepped by constant adds (the 14-bit start-address field never
        // carries: smem < 256 KB).
        const int g = warp - 4 * NS - 1;
        constexpr uint32_t id64 = tc::idesc_f16(128, 64, false, false);
        constexpr uint32_t id16 = tc::idesc_f16(128, 16, false, false);
        const uint64_t dW0 = tc::smem_desc(tc::smem_u32(sW0), 1024, 128);
        const uint64_t dWh = tc::smem_desc(tc::smem_u32(sWh), 1024, 128);
        const uint64_t dWo = tc::smem_desc(tc::smem_u32(sWo), 256, 128);
        const uint64_t dX = tc::smem_desc(tc::smem_u32(sX), 2048, 128);
        const uint64_t dXsw = tc::smem_desc_sw128(tc::smem_u32(sX), 1024);
        const uint64_t dH = tc::smem_desc(tc::smem_u32(h_buf(g)), 2048, 128);
        // bias K-step A operand of the hidden / output layers
        const uint64_t dHb = kAlias ? tc::smem_desc(tc::smem_u32(sAux), 2048, 128) : dH + 4 * 256;
        const uint32_t acc = tmem + (uint32_t)(g * 64);
        uint32_t use = 0;
        for (int j = g; j < n_mine; j += NS, ++use) {
            // h_ready completes H + 1 times per tile; wait for the previous tile's last one
            if (use > 0) tc::mbar_wait(h_ready + g, (use * (H + 1) - 1) & 1);
            const int st = j % nst;
            tc::mbar_wait(x_full + st, (uint32_t)(j / nst) & 1);
            tc::fence_after();
            const uint64_t dXs = dX + (uint64_t)(st * 128 * KX);   // 16-byte units
            const uint64_t dXb = kAlias ? dHb : dXs + (D / 16) * 256;   // bias step A operand
            if constexpr (kSw) {
                const uint64_t dXw = dXsw + (uint64_t)(st * 128 * KX);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)                // atom kk/4, 32 bytes per K step
                    tc::mma_f16_elect(acc, dXw + (kk / 4) * 1024 + (kk % 4) * 2, dW0 + kk * 128, id64, kk > 0);
            } else {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    tc::mma_f16_elect(acc, dXs + kk * 256, dW0 + kk * 128, id64, kk > 0);
            }
            tc::mma_f16_elect(acc, dXb, dW0 + (D / 16) * 128, id64, 1);   // bias
            if constexpr (!kAlias) tc::commit_elect(x_empty + st);    // X stage free (H is separate)
            tc::commit_elect(acc_full + g);
#pragma unroll
            for (int l = 1; l <= H; ++l) {
                tc::mbar_wait(h_ready + g, (uint32_t)((use * (H + 1) + l - 1) & 1));
                tc::fence_after();
                if (l < H) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc::mma_f16_elect(acc, dH + kk * 256, dWh + (l - 1) * 64 * kKgH + kk * 128, id64, kk > 0);
                    tc::mma_f16_elect(acc, dHb, dWh + (l - 1) * 64 * kKgH + 4 * 128, id64, 1);   // bias
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc::mma_f16_elect(acc, dH + kk * 256, dWo + kk * 32, id16, kk > 0);
                    tc::mma_f16_elect(acc, dHb, dWo + 4 * 32, id16, 1);   // bias
                    if constexpr (kAlias) tc::commit_elect(x_empty + st);   // stage (X, then H) free
                }
                tc::commit_elect(acc_full + g);
            }
        }
    } else {
        // ---------------- epilogue of slot g = warp / 4: row 32*(warp%4) + lane
        const int g = warp >> 2, q = warp & 3;
        const int row = q * 32 + (tid & 31);
        unsigned char* hb = h_buf(g);
        const uint32_t acc = tmem + (uint32_t)(g * 64);
        uint32_t acc_n = 0;
        for (int j = g; j < n_mine; j += NS) {
            const int64_t t = blockIdx.x + (int64_t)j * gridDim.x;
            for (int l = 0; l <= H; ++l) {
                tc::mbar_wait(acc_full + g, (acc_n++) & 1);
                tc::fence_after();
                if (l < H) {
#pragma unroll
                    for (int half = 0; half < 2; ++half) {          // 32 accumulator columns at a time
                        float v[32];
                        tc::ld32(acc, (uint32_t)(q * 32), (uint32_t)(32 * half), v);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            *reinterpret_cast<uint4*>(hb + (k + 4 * half) * 2048 + row * 16) =
                                make_uint4(relu_pack(v[8 * k], v[8 * k + 1]), relu_pack(v[8 * k + 2], v[8 * k + 3]),
                                           relu_pack(v[8 * k + 4], v[8 * k + 5]),
                                           relu_pack(v[8 * k + 6], v[8 * k + 7]));
                    }
                    tc::fence_before();
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
    constexpr int NS = mlp_slots(D);
    const uint32_t fixed = mlp_tc_fixed_smem(D, H), stage = mlp_tc_stage_smem(D);
    int nst = (int)(((uint32_t)budget - 1024u - fixed) / stage);
    // a multiple of the slot count, so each stage only ever serves one slot and no barrier
    // waiter can run more than one phase ahead (parity waits are ambiguous beyond that);
    // exactly one stage per slot when the hidden activations alias it
    nst = nst > (mlp_alias(D) ? NS : 2 * NS) ? (mlp_alias(D) ? NS : 2 * NS) : nst;
    nst -= nst % NS;
    if (nst < NS) return cudaErrorInvalidConfiguration;
    MlpTcArgs b = a;
    b.nst = nst;
    const uint32_t smem = fixed + (uint32_t)nst * stage + 1024u;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (m + 127) / 128;
    const int grid = (int)(tiles < sms ? tiles : sms);
    k_mlp_tc<D, H><<<grid, (5 * NS + 1) * 32, smem, s>>>(tm, b);
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
