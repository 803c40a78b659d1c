// nbvh_capi.cu — implementation of the C ABI in include/nbvh.h: context and parameter
// management, scene/cut upload, the query driver (device and chunked host paths) and the
// parity hooks.
// The training entry points live in nbvh_train.cu.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/nbvh.h"
#include "nbvh_capi_internal.h"

using namespace nbvh;

// ------------------------------------------------------------------ helpers
namespace nbvh {

nbvh_status fail(nbvh_ctx* c, nbvh_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

nbvh_status cuda_fail(nbvh_ctx* c, cudaError_t e, const char* where) {
    if (c) {
        c->poisoned = true;
        c->err = std::string(where) + ": " + cudaGetErrorString(e);
    }
    return NBVH_ECUDA;
}

nbvh_status check_device(nbvh_ctx* c) {
    if (!c) return NBVH_EINVAL;
    if (c->poisoned) return NBVH_ECUDA;
    if (c->device < 0) return fail(c, NBVH_ESTATE, "host-only context (created with cuda_device = -1)");
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
    return NBVH_OK;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) return cudaSuccess;
    return cudaMalloc((void**)p, count * sizeof(T));
}

template <typename T>
static void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

GridDev make_grid(const nbvh_ctx* c, int lod) {
    GridDev g{};
    g.L = c->cfg.L;
    g.F = c->cfg.F;
    g.n_points = c->cfg.n_points;
    g.log2_T = c->cfg.log2_T;
    for (int l = 0; l < c->cfg.L; ++l) {
        g.res[l] = c->res[l];
        g.dense[l] = c->dense[l];
        g.offset[l] = (uint32_t)c->offset[l];
        g.inf_offset[l] = (uint32_t)c->inf_offset[l];
    }
    g.table = c->d_table16;
    g.tex = c->tex_table;
    if (lod >= 0) {
        const HostCut& hc = c->cuts[lod];
        for (int k = 0; k < 3; ++k) g.dom_min[k] = hc.dom_min[k];
        g.dom_inv = hc.dom_inv;
    }
    return g;
}

MlpDev make_mlp(const nbvh_ctx* c) {
    MlpDev m{};
    m.d_in = c->d_in;
    m.hidden = c->cfg.hidden_layers;
    m.W = c->d_W16;
    m.b = c->d_params + c->n_table + c->n_W;
    return m;
}

CutDev make_cut(const nbvh_ctx* c, int lod) {
    CutDev d{};
    d.inner = c->dcut[lod].inner;
    d.leaf_box = c->dcut[lod].leaf_box;
    d.n_leaves = c->cuts[lod].n_leaves;
    d.depth = c->dcut[lod].depth;
    return d;
}

// fp32 master -> fp16 inference copy (MLP weights; biases stay fp32).
__global__ void k_refresh_fp16(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) dst[i] = __float2half_rn(src[i]);
}
__global__ void k_refresh_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) dst[i] = __float2bfloat16_rn(src[i]);
}

// fp32 master tables -> fp16 inference table: hashed levels copied, dense levels
// corner-packed (LevelSm in nbvh_device.cuh).  blockIdx.y = level; one thread per dense
// cell (gathers its 8 corners, writes one 16*F-byte record) or per 4 hashed entries.
// F is a template parameter so the record stays in registers (no local memory).
template <int F>
__global__ void k_refresh_table(const float* __restrict__ src, __half* __restrict__ dst, GridDev g) {
    __shared__ LevelSm lv[kMaxLevels];
    stage_levels(g, lv, threadIdx.x);
    __syncthreads();
    const LevelSm P = lv[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (P.nx) {
        // dense level: cell c's record = its 8 corner vertices' features (corner-packed)
        const uint32_t n_cells = P.nxy * P.nx;
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells; c += stride) {
            const uint32_t cell = (uint32_t)c;
            const uint32_t cz = cell / P.nxy, rem = cell - cz * P.nxy;
            const uint32_t cy = rem / P.nx, cx = rem - cy * P.nx;
            const uint32_t b = cx + cy * P.n1 + cz * P.n1sq;
            uint32_t rec[4 * F];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t idx = b + (k & 1) + ((k >> 1) & 1) * P.n1 + ((k >> 2) & 1) * P.n1sq;
                const float* sp = src + ((int64_t)P.coff + idx) * F;
                if constexpr (F == 2) {
                    const __half2 h = __float22half2_rn(__ldg(reinterpret_cast<const float2*>(sp)));
                    rec[k] = *reinterpret_cast<const uint32_t*>(&h);
                } else {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(sp));
                    const __half2 h0 = __floats2half2_rn(v.x, v.y), h1 = __floats2half2_rn(v.z, v.w);
                    rec[2 * k] = *reinterpret_cast<const uint32_t*>(&h0);
                    rec[2 * k + 1] = *reinterpret_cast<const uint32_t*>(&h1);
                }
            }
            uint4* d = reinterpret_cast<uint4*>(dst + ((int64_t)P.off + 8ll * cell) * F);
#pragma unroll
            for (int v = 0; v < F; ++v)                          // 16*F bytes
                d[v] = make_uint4(rec[4 * v], rec[4 * v + 1], rec[4 * v + 2], rec[4 * v + 3]);
        }
    } else {
        // hashed level: the canonical layout, 4 entries per thread: 8- or 16-byte loads (the
        // level's master offset can be odd), one 16-byte store per 8 halves
        const int64_t n4 = ((int64_t)1 << g.log2_T) / 4;
        uint4* dp = reinterpret_cast<uint4*>(dst + (int64_t)P.off * F);
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += stride) {
            const float* sp = src + ((int64_t)P.coff + 4 * e) * F;
            if constexpr (F == 2) {
                const float2 v0 = __ldg(reinterpret_cast<const float2*>(sp)),
                             v1 = __ldg(reinterpret_cast<const float2*>(sp + 2)),
                             v2 = __ldg(reinterpret_cast<const float2*>(sp + 4)),
                             v3 = __ldg(reinterpret_cast<const float2*>(sp + 6));
                const __half2 o[4] = {__float22half2_rn(v0), __float22half2_rn(v1), __float22half2_rn(v2),
                                      __float22half2_rn(v3)};
                dp[e] = *reinterpret_cast<const uint4*>(o);
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(sp) + 2 * h),
                                 b = __ldg(reinterpret_cast<const float4*>(sp) + 2 * h + 1);
                    const __half2 o[4] = {__floats2half2_rn(a.x, a.y), __floats2half2_rn(a.z, a.w),
                                          __floats2half2_rn(b.x, b.y), __floats2half2_rn(b.z, b.w)};
                    dp[2 * e + h] = *reinterpret_cast<const uint4*>(o);
                }
            }
        }
    }
}

static void launch_refresh_table(nbvh_ctx* c, cudaStream_t s) {
    const GridDev g = make_grid(c, -1);
    if (g.F == 2) k_refresh_table<2><<<dim3(148, c->cfg.L), 256, 0, s>>>(c->d_params, c->d_table16, g);
    else k_refresh_table<4><<<dim3(148, c->cfg.L), 256, 0, s>>>(c->d_params, c->d_table16, g);
}

nbvh_status refresh_fp16(nbvh_ctx* c, cudaStream_t s) {
    const int64_t nt = c->n_table, nw = c->n_W;
    launch_refresh_table(c, s);
    k_refresh_fp16<<<148, 256, 0, s>>>(c->d_params + nt, c->d_W16, nw);
    if (c->d_Wb16) k_refresh_bf16<<<148, 256, 0, s>>>(c->d_params + nt, c->d_Wb16, nw);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "refresh_fp16");
    return NBVH_OK;
}

nbvh_status refresh_table(nbvh_ctx* c, cudaStream_t s) {
    launch_refresh_table(c, s);
    if (c->d_Wb16) k_refresh_bf16<<<148, 256, 0, s>>>(c->d_params + c->n_table, c->d_Wb16, c->n_W);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "refresh_table");
    return NBVH_OK;
}

}  // namespace nbvh

// ------------------------------------------------------------------ lifecycle
extern "C" void nbvh_config_default(nbvh_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->L = 8;
    cfg->F = 2;
    cfg->log2_T = 14;
    cfg->base_res = 8;
    cfg->max_res = 1024;
    cfg->n_points = 4;
    cfg->hidden_layers = 2;
    cfg->width = 64;
    cfg->list_cap = 12;
    cfg->mode = 0;
    cfg->inflate_rel = 1e-3f;
    cfg->inflate_abs = 1e-6f;
    cfg->seed = 1;
}

namespace {

uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
double unit(uint64_t& s) { return (double)(splitmix64(s) >> 11) * (1.0 / 9007199254740992.0); }

}  // namespace

extern "C" nbvh_status nbvh_create(const nbvh_config* cfg, int cuda_device, nbvh_ctx** out) {
    if (!cfg || !out) return NBVH_EINVAL;
    *out = nullptr;
    const nbvh_config& c = *cfg;
    if (c.L < 1 || c.L > kMaxLevels || (c.F != 2 && c.F != 4) || c.log2_T < 4 || c.log2_T > 24 || c.base_res < 1 ||
        c.max_res < c.base_res || c.n_points < 1 || c.hidden_layers < 1 || c.hidden_layers > kMaxHidden ||
        c.width != kWidth || c.list_cap < 1 || c.list_cap > kListK || (c.mode != 0 && c.mode != 1) ||
        (c.mlp_dtype != 0 && c.mlp_dtype != 1))
        return NBVH_EINVAL;
    const int d_in = c.n_points * c.L * c.F;
    if ((c.L * c.F) % 8 != 0 || !(d_in == 32 || d_in == 64 || d_in == 96 || d_in == 128)) return NBVH_EINVAL;
    nbvh_ctx* x = new (std::nothrow) nbvh_ctx();
    if (!x) return NBVH_ENOMEM;
    x->cfg = c;
    x->device = cuda_device;
    x->d_in = d_in;
    level_table(c.L, c.log2_T, c.base_res, c.max_res, x->res, x->dense, x->offset, &x->n_entries);
    x->n_table = x->n_entries * c.F;
    for (int l = 0; l < c.L; ++l)           // hashed levels: the encode's x term is unmasked (x+1 <= N < T)
        if (!x->dense[l] && x->res[l] >= (1 << c.log2_T)) {
            delete x;
            return NBVH_EINVAL;
        }
    {   // inference layout: dense levels corner-packed (8 entries per cell), 8-entry aligned;
        // hashed levels T-aligned, so that offset + hash = offset | hash (the TEX encode folds
        // the offset into its XOR)
        int64_t o = 0;
        const int64_t T = (int64_t)1 << c.log2_T;
        for (int l = 0; l < c.L; ++l) {
            if (!x->dense[l]) o = (o + T - 1) & ~(T - 1);
            x->inf_offset[l] = o;
            const int64_t N = x->res[l];
            o += x->dense[l] ? 8 * N * N * N : (int64_t)1 << c.log2_T;
            o = (o + 7) & ~(int64_t)7;
        }
        x->n_inf = o;
        if (o >= ((int64_t)1 << 32)) {
            delete x;
            return NBVH_EINVAL;
        }
    }
    x->n_W = (int64_t)64 * d_in + (int64_t)(c.hidden_layers - 1) * 64 * 64 + 8 * 64;
    x->n_b = (int64_t)64 * c.hidden_layers + 8;
    // C21 initialisation
    x->h_params.resize(x->n_table + x->n_W + x->n_b);
    uint64_t s = c.seed * 0x2545F4914F6CDD1Dull + 12345;
    for (int64_t i = 0; i < x->n_table; ++i) x->h_params[i] = (float)((unit(s) * 2.0 - 1.0) * 1e-4);
    int64_t o = x->n_table;
    for (int k = 0; k <= c.hidden_layers; ++k) {
        const int fan_in = k == 0 ? d_in : 64, fan_out = k == c.hidden_layers ? 8 : 64;
        const double lim = std::sqrt(6.0 / fan_in);
        for (int64_t i = 0; i < (int64_t)fan_in * fan_out; ++i) x->h_params[o++] = (float)((unit(s) * 2.0 - 1.0) * lim);
    }
    for (int64_t i = 0; i < x->n_b; ++i) x->h_params[o++] = 0.0f;
    if (cuda_device >= 0) {
        cudaError_t e = cudaSetDevice(cuda_device);
        if (e == cudaSuccess) e = dalloc(&x->d_params, x->h_params.size());
        if (e == cudaSuccess) e = dalloc(&x->d_table16, x->n_inf * c.F);
        if (e == cudaSuccess) {
            // a linear texture over the fp16 inference table: one texel = one entry (F halves),
            // element reads through the TEX pipe (the query kernel's hashed-level gathers)
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = x->d_table16;
            rd.res.linear.desc = c.F == 2 ? cudaCreateChannelDesc<unsigned int>() : cudaCreateChannelDesc<uint2>();
            rd.res.linear.sizeInBytes = (size_t)x->n_inf * c.F * 2;
            cudaTextureDesc td{};
            td.readMode = cudaReadModeElementType;
            td.filterMode = cudaFilterModePoint;
            td.addressMode[0] = cudaAddressModeClamp;
            td.normalizedCoords = 0;
            cudaTextureObject_t t = 0;
            if (cudaCreateTextureObject(&t, &rd, &td, nullptr) == cudaSuccess) x->tex_table = t;
            else { cudaGetLastError(); x->tex_table = 0; }
        }
        if (e == cudaSuccess) e = dalloc(&x->d_W16, x->n_W);
        if (e == cudaSuccess && c.mlp_dtype == 1) e = cudaMalloc((void**)&x->d_Wb16, (size_t)x->n_W * 2);
        if (e == cudaSuccess) e = dalloc(&x->d_misc, kCounterBlocks * kCounterStride);
        if (e == cudaSuccess) e = cudaMallocHost((void**)&x->h_misc, kCounterBlocks * kCounterStride * sizeof(int32_t));
        if (e == cudaSuccess)
            e = cudaMemcpy(x->d_params, x->h_params.data(), x->h_params.size() * 4, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemset(x->d_misc, 0, kCounterBlocks * kCounterStride * sizeof(int32_t));
        if (e != cudaSuccess) {
            x->err = std::string("nbvh_create: ") + cudaGetErrorString(e);
            nbvh_destroy(x);
            cudaGetLastError();
            return e == cudaErrorMemoryAllocation ? NBVH_ENOMEM : NBVH_ECUDA;
        }
        nbvh_status st = refresh_fp16(x, 0);
        if (st == NBVH_OK) {
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) st = cuda_fail(x, e, "nbvh_create");
        }
        if (st != NBVH_OK) {
            nbvh_destroy(x);
            return st;
        }
    }
    *out = x;
    return NBVH_OK;
}

static void free_workspace(nbvh_ctx* c) {
    dfree(c->d_lst);
    dfree(c->d_state);
    dfree(c->d_act);
    dfree(c->d_act_long);
    dfree(c->d_stage_rays);
    dfree(c->d_stage_hits);
    c->reserved = 0;
}

extern "C" void nbvh_destroy(nbvh_ctx* c) {
    if (!c) return;
    if (c->device >= 0) {
        cudaSetDevice(c->device);
        free_workspace(c);
        for (int l = 0; l < kMaxLod; ++l) {
            dfree(c->dcut[l].inner);
            dfree(c->dcut[l].leaf_box);
            dfree(c->dcut[l].leaf_base);
            dfree(c->dcut[l].rank);
        }
        dfree(c->d_params);
        if (c->tex_table) cudaDestroyTextureObject((cudaTextureObject_t)c->tex_table);
        c->tex_table = 0;
        dfree(c->d_table16);
        dfree(c->d_W16);
        if (c->d_Wb16) cudaFree(c->d_Wb16);
        c->d_Wb16 = nullptr;
        dfree(c->d_misc);
        if (c->h_misc) cudaFreeHost(c->h_misc);
        for (cudaEvent_t x : c->events) cudaEventDestroy(x);
        for (cudaStream_t x : c->aux_stream)
            if (x) cudaStreamDestroy(x);
        free_scene_device(c);
        free_train_device(c);
    }
    delete c;
}

extern "C" const char* nbvh_last_error(const nbvh_ctx* c) { return c ? c->err.c_str() : "null context"; }

extern "C" nbvh_status nbvh_level_table(const nbvh_ctx* c, int32_t* res, int32_t* dense, int64_t* offset,
                                        int64_t* n_entries) {
    if (!c) return NBVH_EINVAL;
    for (int l = 0; l < c->cfg.L; ++l) {
        if (res) res[l] = c->res[l];
        if (dense) dense[l] = c->dense[l];
        if (offset) offset[l] = c->offset[l];
    }
    if (n_entries) *n_entries = c->n_entries;
    return NBVH_OK;
}

static bool block_range(const nbvh_ctx* c, int32_t block, int64_t* off, int64_t* n) {
    switch (block) {
        case NBVH_PARAM_TABLES: *off = 0; *n = c->n_table; return true;
        case NBVH_PARAM_WEIGHTS: *off = c->n_table; *n = c->n_W; return true;
        case NBVH_PARAM_BIASES: *off = c->n_table + c->n_W; *n = c->n_b; return true;
        case NBVH_PARAM_ALL: *off = 0; *n = c->n_table + c->n_W + c->n_b; return true;
    }
    return false;
}

extern "C" nbvh_status nbvh_param_count(const nbvh_ctx* c, int32_t block, int64_t* n) {
    int64_t off;
    if (!c || !n || !block_range(c, block, &off, n)) return NBVH_EINVAL;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_get_params(nbvh_ctx* c, int32_t block, float* dst, int64_t n) {
    int64_t off, cnt;
    if (!c || !dst || !block_range(c, block, &off, &cnt) || n != cnt) return fail(c, NBVH_EINVAL, "get_params: bad block/size");
    if (c->device < 0) {
        std::memcpy(dst, c->h_params.data() + off, cnt * 4);
        return NBVH_OK;
    }
    nbvh_status st = check_device(c);
    if (st) return st;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(dst, c->d_params + off, cnt * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "get_params");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_set_params(nbvh_ctx* c, int32_t block, const float* src, int64_t n) {
    int64_t off, cnt;
    if (!c || !src || !block_range(c, block, &off, &cnt) || n != cnt) return fail(c, NBVH_EINVAL, "set_params: bad block/size");
    std::memcpy(c->h_params.data() + off, src, cnt * 4);
    if (c->device < 0) return NBVH_OK;
    nbvh_status st = check_device(c);
    if (st) return st;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(c->d_params + off, src, cnt * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(c, e, "set_params");
    st = refresh_fp16(c, 0);
    if (st) return st;
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "set_params");
    // Adam state restarts for externally set parameters
    reset_adam(c);
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_reserve(nbvh_ctx* c, int64_t max_rays) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (max_rays < 1 || max_rays > (int64_t)1 << 30) return fail(c, NBVH_EINVAL, "reserve: max_rays out of range");
    if (max_rays <= c->reserved) return NBVH_OK;
    cudaDeviceSynchronize();
    free_workspace(c);
    const size_t n = (size_t)max_rays;
    cudaError_t e = dalloc(&c->d_lst, kListK * n);
    if (e == cudaSuccess) e = dalloc(&c->d_state, 2 * n);
    if (e == cudaSuccess) e = dalloc(&c->d_act, n);
    if (e == cudaSuccess) e = dalloc(&c->d_act_long, n);
    if (e == cudaSuccess) e = dalloc(&c->d_stage_rays, 8 * n);
    if (e == cudaSuccess) e = dalloc(&c->d_stage_hits, 10 * n);
    if (e != cudaSuccess) {
        free_workspace(c);
        cudaGetLastError();
        return fail(c, NBVH_ENOMEM, std::string("reserve: ") + cudaGetErrorString(e));
    }
    c->reserved = max_rays;
    return reserve_train(c, max_rays);
}

// ------------------------------------------------------------------ scene + cut
extern "C" nbvh_status nbvh_set_mesh(nbvh_ctx* c, const float* xyz, int64_t nv, const uint32_t* tri, int64_t nt,
                                     const float* vnormal, const float* tri_albedo) {
    if (c) c->base_depth = -1;
    if (!c) return NBVH_EINVAL;
    if (c->poisoned) return NBVH_ECUDA;
    if (!xyz || !tri || nv < 3 || nt < 1 || nt > (int64_t)1 << 30) return fail(c, NBVH_EINVAL, "set_mesh: bad mesh");
    for (int64_t i = 0; i < 3 * nt; ++i)
        if (tri[i] >= (uint64_t)nv) return fail(c, NBVH_EINVAL, "set_mesh: vertex index out of range");
    for (int64_t i = 0; i < 3 * nv; ++i)
        if (!std::isfinite(xyz[i])) return fail(c, NBVH_EINVAL, "set_mesh: non-finite vertex");
    HostScene& sc = c->sc;
    sc = HostScene{};
    sc.xyz.assign(xyz, xyz + 3 * nv);
    sc.tri.assign(tri, tri + 3 * nt);
    if (vnormal) {
        sc.vnormal.assign(vnormal, vnormal + 3 * nv);
    } else {
        std::vector<double> acc(3 * nv, 0.0);
        for (int64_t t = 0; t < nt; ++t) {
            const float* a = xyz + 3 * tri[3 * t];
            const float* b = xyz + 3 * tri[3 * t + 1];
            const float* d = xyz + 3 * tri[3 * t + 2];
            double e1[3], e2[3];
            for (int k = 0; k < 3; ++k) { e1[k] = (double)b[k] - a[k]; e2[k] = (double)d[k] - a[k]; }
            double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
            for (int v = 0; v < 3; ++v)
                for (int k = 0; k < 3; ++k) acc[3 * tri[3 * t + v] + k] += n[k];
        }
        sc.vnormal.resize(3 * nv);
        for (int64_t v = 0; v < nv; ++v) {
            double l = std::sqrt(acc[3 * v] * acc[3 * v] + acc[3 * v + 1] * acc[3 * v + 1] + acc[3 * v + 2] * acc[3 * v + 2]);
            for (int k = 0; k < 3; ++k) sc.vnormal[3 * v + k] = l > 0 ? (float)(acc[3 * v + k] / l) : 0.f;
        }
    }
    if (tri_albedo) sc.albedo.assign(tri_albedo, tri_albedo + 3 * nt);
    else sc.albedo.assign(3 * nt, 0.5f);
    build_sah_bvh(sc);
    c->has_mesh = true;
    for (int l = 0; l < kMaxLod; ++l) c->has_cut[l] = false;
    if (c->device >= 0) return upload_scene(c);
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_build_cut(nbvh_ctx* c, int32_t target, const float* leaf_q, const float* leaf_p,
                                      int32_t lod, int32_t* out_n) {
    if (!c) return NBVH_EINVAL;
    if (c->poisoned) return NBVH_ECUDA;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "build_cut: lod slot out of range");
    if (!c->has_mesh) return fail(c, NBVH_ESTATE, "build_cut: no mesh");
    if (target < 1) return fail(c, NBVH_EINVAL, "build_cut: target < 1");
    if ((leaf_q == nullptr) != (leaf_p == nullptr)) return fail(c, NBVH_EINVAL, "build_cut: give both q and p or neither");
    if (leaf_q && !c->has_cut[lod]) return fail(c, NBVH_ESTATE, "build_cut: q/p expansion needs an existing cut");
    HostCut nc;
    int clamped = build_cut(c->sc, target, leaf_q ? &c->cuts[lod] : nullptr, leaf_q, leaf_p, c->cfg.inflate_rel,
                            c->cfg.inflate_abs, nc);
    c->cuts[lod] = std::move(nc);
    c->has_cut[lod] = true;
    if (out_n) *out_n = c->cuts[lod].n_leaves;
    if (c->device >= 0) {
        nbvh_status st = upload_cut(c, lod);
        if (st) return st;
    }
    return clamped ? NBVH_WARN_CLAMPED : NBVH_OK;
}

extern "C" nbvh_status nbvh_copy_cut(nbvh_ctx* c, int32_t src_lod, int32_t dst_lod) {
    if (!c) return NBVH_EINVAL;
    if (c->poisoned) return NBVH_ECUDA;
    if (src_lod < 0 || src_lod >= kMaxLod || dst_lod < 0 || dst_lod >= kMaxLod)
        return fail(c, NBVH_ERANGE, "copy_cut: lod slot out of range");
    if (!c->has_cut[src_lod]) return fail(c, NBVH_ESTATE, "copy_cut: empty source slot");
    if (src_lod == dst_lod) return NBVH_OK;
    c->cuts[dst_lod] = c->cuts[src_lod];
    c->has_cut[dst_lod] = true;
    if (c->device >= 0) {
        nbvh_status st = upload_cut(c, dst_lod);
        if (st) return st;
    }
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_cut_info(const nbvh_ctx* c, int32_t lod, int32_t* n_leaves, int32_t* n_inner) {
    if (!c) return NBVH_EINVAL;
    if (lod < 0 || lod >= kMaxLod) return NBVH_ERANGE;
    if (!c->has_cut[lod]) return NBVH_ESTATE;
    if (n_leaves) *n_leaves = c->cuts[lod].n_leaves;
    if (n_inner) *n_inner = (int32_t)c->cuts[lod].inner.size();
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_get_base_bvh(const nbvh_ctx* c, int32_t* child_a, int32_t* child_b, int64_t* n_nodes) {
    if (!c) return NBVH_EINVAL;
    if (!c->has_mesh) return NBVH_ESTATE;
    const int64_t n = (int64_t)c->sc.nodes.size();
    if (n_nodes) *n_nodes = n;
    for (int64_t i = 0; i < n; ++i) {
        if (child_a) child_a[i] = c->sc.nodes[i].a;
        if (child_b) child_b[i] = c->sc.nodes[i].b;
    }
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_get_cut_nodes(const nbvh_ctx* c, int32_t lod, int32_t* leaf_base) {
    if (!c || !leaf_base) return NBVH_EINVAL;
    if (lod < 0 || lod >= kMaxLod) return NBVH_ERANGE;
    if (!c->has_cut[lod]) return NBVH_ESTATE;
    const HostCut& hc = c->cuts[lod];
    std::memcpy(leaf_base, hc.leaf_base.data(), sizeof(int32_t) * (size_t)hc.n_leaves);
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_get_cut(const nbvh_ctx* c, int32_t lod, float* leaf_lo, float* leaf_hi, float* base_lo,
                                    float* base_hi, int64_t* tri_off, int32_t* tris, float* dom_min, float* dom_inv) {
    if (!c) return NBVH_EINVAL;
    if (lod < 0 || lod >= kMaxLod) return NBVH_ERANGE;
    if (!c->has_cut[lod]) return NBVH_ESTATE;
    const HostCut& hc = c->cuts[lod];
    const int32_t n = hc.n_leaves;
    if (leaf_lo) std::memcpy(leaf_lo, hc.leaf_lo.data(), 12 * (size_t)n);
    if (leaf_hi) std::memcpy(leaf_hi, hc.leaf_hi.data(), 12 * (size_t)n);
    int64_t acc = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t node = hc.leaf_base[i];
        const BvhNode& bn = c->sc.nodes[node];
        for (int k = 0; k < 3; ++k) {
            if (base_lo) base_lo[3 * i + k] = bn.lo[k];
            if (base_hi) base_hi[3 * i + k] = bn.hi[k];
        }
        // triangles of the subtree = contiguous prim range [first, last)
        int32_t lo = node, hi = node;
        while (c->sc.nodes[lo].b >= 0) lo = c->sc.nodes[lo].a;
        while (c->sc.nodes[hi].b >= 0) hi = c->sc.nodes[hi].b;
        const int32_t first = c->sc.nodes[lo].a, last = c->sc.nodes[hi].a - c->sc.nodes[hi].b;
        if (tri_off) tri_off[i] = acc;
        if (tris)
            for (int32_t j = first; j < last; ++j) tris[acc + (j - first)] = c->sc.prim[j];
        acc += last - first;
    }
    if (tri_off) tri_off[n] = acc;
    if (dom_min)
        for (int k = 0; k < 3; ++k) dom_min[k] = hc.dom_min[k];
    if (dom_inv) *dom_inv = hc.dom_inv;
    return NBVH_OK;
}

// ------------------------------------------------------------------ query
namespace nbvh {

__global__ void k_reset_counters(QueryCounters* ctr, int all) {
    int32_t* w = reinterpret_cast<int32_t*>(ctr);
    const int n = (int)(sizeof(QueryCounters) / sizeof(int32_t));
    const int t = threadIdx.x;    // per-launch words: cnt (2), next (3), cnt_long (5)
    if (t < n && (all || t == 2 || t == 3 || t == 5)) w[t] = 0;
}

QueryCounters* counter_block(nbvh_ctx* c, int block) {
    return reinterpret_cast<QueryCounters*>(c->d_misc + (size_t)block * kCounterStride);
}

cudaEvent_t ctx_event(nbvh_ctx* c, int i) {
    while ((int)c->events.size() <= i) {
        cudaEvent_t x;
        cudaEventCreate(&x);
        c->events.push_back(x);
    }
    return c->events[i];
}

// One query = memset of the counters + k_traverse + one persistent k_query launch, all
// stream-ordered on `s` with no host synchronisation.  `reset_stats` zeroes the whole
// counter block (statistics of a public call); otherwise only the per-launch work-list
// counters are reset and the statistics accumulate (chunked host path).
nbvh_status run_query(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, int32_t lod, const HitsDev& out, float* z_trace,
                      int32_t trace_cap, cudaStream_t s, bool reset_stats, int64_t work_off, int block) {
    // workspace slice [work_off, work_off + n) of every per-ray buffer and counter block
    // `block`: disjoint slices let the host path run two chunks' queries concurrently
    QueryCounters* ctr = counter_block(c, block);
    // counter reset by a one-thread kernel, not cudaMemsetAsync: a memset may queue on a copy
    // engine behind the host path's bulk uploads and serialise the pipeline
    k_reset_counters<<<1, 32, 0, s>>>(ctr, reset_stats ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "query: counter reset");
    RayState st = c->state();
    st.nbuf += work_off;
    st.more += work_off;
    float4* lst = c->d_lst + kListK * work_off;
    WorkRec* act = c->d_act + work_off;
    WorkRec* act_long = c->d_act_long + work_off;
    TraverseArgs ta{};
    ta.cut = make_cut(c, lod);
    ta.rays = reinterpret_cast<const float4*>(rays);
    ta.n_rays = n;
    ta.cap = c->cfg.list_cap;
    ta.lst = lst;
    ta.st = st;
    ta.out = out;
    ta.act_out = act;
    ta.act_long = act_long;
    ta.ctr = ctr;
    if (c->profiling) cudaEventRecord(ctx_event(c, 0), s);
    e = launch_traverse(ta, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "query: traverse");
    if (c->profiling) cudaEventRecord(ctx_event(c, 1), s);
    QueryArgs qa{};
    qa.g = make_grid(c, lod);
    {
        const char* ev = std::getenv("NBVH_QUERY_TEX");       // A/B hook: 0 = hashed gathers on LDG
        if (ev && ev[0] == '0') qa.g.tex = 0;
    }
    qa.m = make_mlp(c);
    if (c->d_Wb16) {                      // bf16 query path (mlp_dtype = 1, C39)
        qa.m.W = reinterpret_cast<const __half*>(c->d_Wb16);
        qa.m.bf16 = 1;
    }
    qa.cut = make_cut(c, lod);
    qa.rays = reinterpret_cast<const float4*>(rays);
    qa.n_rays = n;
    qa.cap = c->cfg.list_cap;
    qa.mode = c->cfg.mode;
    qa.lst = lst;
    qa.nbuf = st.nbuf;
    qa.more = st.more;
    qa.out = out;
    qa.act = act;
    qa.cnt = &ctr->cnt;
    qa.act_long = act_long;
    qa.cnt_long = &ctr->cnt_long;
    qa.next = &ctr->next;
    qa.z_trace = z_trace;
    qa.trace_cap = trace_cap;
    qa.ctr = ctr;
    e = launch_query(qa, n, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "query: persistent query kernel");
    if (c->profiling) cudaEventRecord(ctx_event(c, 2), s);
    if (reset_stats && block == 0) {
        c->qstats = nbvh_query_stats{};
        c->qstats_launches = 0;
        c->qstats_blocks = 1;
    }
    c->qstats_blocks = std::max(c->qstats_blocks, block + 1);
    c->qstats.n_rays += n;
    c->qstats_launches += 3;
    c->qstats_pending = true;
    c->qstats_stream = s;
    return NBVH_OK;
}

// Resolve the device counters of the last query call (synchronises the device: the host
// path's chunks run on two streams).
nbvh_status resolve_query_stats(nbvh_ctx* c) {
    if (!c->qstats_pending) return NBVH_OK;
    const int nb = std::max(1, c->qstats_blocks);
    cudaError_t e = cudaStreamSynchronize(c->qstats_stream);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(c->h_misc, c->d_misc, (size_t)nb * kCounterStride * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "query stats");
    c->qstats_pending = false;
    int64_t nq = 0;
    int32_t iters = 0, refills = 0, err = 0, tiles = 0, rows = 0;
    int64_t wsc[3] = {0, 0, 0};
    for (int b = 0; b < nb; ++b) {
        const QueryCounters* q = reinterpret_cast<const QueryCounters*>(c->h_misc + (size_t)b * kCounterStride);
        nq += (int64_t)q->n_queries;
        iters = std::max(iters, q->max_iter);
        refills += q->refills;
        err |= q->err;
        tiles += q->mlp_tiles;
        rows += q->mlp_rows;
        for (int k = 0; k < 3; ++k) wsc[k] += (int64_t)q->ws_cycles[k];
    }
    for (int k = 0; k < 3; ++k) c->qstats.ws_cycles[k] = wsc[k];
    c->qstats.n_mlp_tiles = tiles;
    c->qstats.n_mlp_rows = rows;
    c->qstats.n_queries = nq;
    c->qstats.n_iters = iters;
    c->qstats.n_launches = c->qstats_launches;
    c->qstats.n_refills = refills;
    c->qstats.ms_traverse = 0.f;
    c->qstats.ms_query = 0.f;
    if (c->profiling && c->events.size() >= 3) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->events[0], c->events[1]) == cudaSuccess) c->qstats.ms_traverse = ms;
        if (cudaEventElapsedTime(&ms, c->events[1], c->events[2]) == cudaSuccess) c->qstats.ms_query = ms;
        cudaGetLastError();
    }
    if (err) return fail(c, NBVH_ECUDA, "query: traversal stack overflow (N-BVH deeper than 64)");
    return NBVH_OK;
}

nbvh_status check_query(nbvh_ctx* c, const void* rays, int64_t n, int32_t lod, const nbvh_hits& out) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "query: lod out of range");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "query: no cut in this LoD slot");
    if (n < 0 || (n > 0 && (!rays || !out.hit || !out.t || !out.normal || !out.albedo)))
        return fail(c, NBVH_EINVAL, "query: null pointer or negative n");
    if (n > c->reserved) return fail(c, NBVH_ESTATE, "query: n exceeds nbvh_reserve");
    return NBVH_OK;
}

}  // namespace nbvh

static HitsDev to_dev(const nbvh_hits& h) {
    return HitsDev{h.hit, h.t, h.normal, h.albedo, h.leaf, h.n_queries};
}

extern "C" nbvh_status nbvh_query(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, int32_t lod, nbvh_hits out,
                                  void* stream) {
    nbvh_status st = check_query(c, rays, n, lod, out);
    if (st) return st;
    if (n == 0) return NBVH_OK;
    return run_query(c, rays, n, lod, to_dev(out), nullptr, 0, (cudaStream_t)stream, true, 0, 0);
}

// Block-interleaved chunking of the host path.  The ray array is cut into blocks of
// kHostBlock rays grouped in periods of W = sum(w_k) blocks; chunk k takes w_k consecutive
// blocks of every period (one strided 2-D copy per direction and field), so every chunk
// samples the whole frame and carries work in proportion to w_k (contiguous chunks of an
// image are sky at the top and terrain at the bottom).  The first and last chunks are
// lighter so the pipeline's head (first upload) and tail (last download) are short.
// Blocks after the last full period go to the last chunk.
namespace nbvh {
constexpr int64_t kHostBlock = 1024;
constexpr int kMaxChunks = 8;

struct ChunkPlan {
    int64_t w = 0;             // blocks per period
    int64_t first = 0;         // first block of the chunk within a period
    int64_t rows = 0;          // full periods
    int64_t tail = 0;          // rays of the trailing region (last chunk only)
    int64_t dev_off = 0;       // first ray of the chunk in the device staging buffers
    int64_t blk = kHostBlock;  // rays per block
    int64_t size() const { return rows * w * blk + tail; }
};

static int plan_chunks(int64_t n, ChunkPlan* plan) {
    int wts[kMaxChunks] = {1, 2, 3, 3, 2, 1};                     // measured best of a sweep (1080p)
    int chunks = n >= (1 << 20) ? 6 : (n >= (1 << 18) ? 2 : 1);
    if (chunks == 2) wts[0] = wts[1] = 1;
    if (chunks == 1) wts[0] = 1;
    if (const char* ev = std::getenv("NBVH_HOST_WEIGHTS")) {     // tuning hook, e.g. "1,2,2,2,1"
        chunks = 0;
        for (const char* p = ev; *p && chunks < kMaxChunks;) {
            wts[chunks++] = std::max(1, std::atoi(p));
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
        if (chunks == 0) { chunks = 1; wts[0] = 1; }
    }
    int64_t W = 0;
    for (int k = 0; k < chunks; ++k) W += wts[k];
    // NBVH_HOST_CONTIG=1: one period, i.e. contiguous chunks (tuning hook)
    const char* cev = std::getenv("NBVH_HOST_CONTIG");
    int64_t blk = kHostBlock;
    if (const char* bev = std::getenv("NBVH_HOST_BLOCK")) blk = std::max<int64_t>(1, std::atoll(bev));   // tuning hook
    if (cev && cev[0] == '1') blk = std::max<int64_t>(1, n / W);
    const int64_t periods = n / (blk * W);
    int64_t off = 0, first = 0;
    for (int k = 0; k < chunks; ++k) {
        ChunkPlan& p = plan[k];
        p.w = wts[k];
        p.first = first;
        first += wts[k];
        p.rows = periods;
        p.blk = blk;
        p.tail = k == chunks - 1 ? n - periods * W * blk : 0;
        p.dev_off = off;
        off += p.size();
    }
    return chunks;
}

// strided host <-> contiguous device copy of one field of a chunk (elem bytes per ray)
static cudaError_t copy_chunk(void* host, void* dev, size_t elem, int64_t n, int64_t W, const ChunkPlan& p,
                              cudaMemcpyKind kind, cudaStream_t s) {
    char* h = static_cast<char*>(host);
    char* d = static_cast<char*>(dev) + p.dev_off * elem;
    const size_t bw = (size_t)p.blk * elem;
    cudaError_t e = cudaSuccess;
    if (p.rows) {
        char* hb = h + (size_t)p.first * bw;
        const size_t width = (size_t)p.w * bw, hpitch = (size_t)W * bw;
        if (kind == cudaMemcpyHostToDevice)
            e = cudaMemcpy2DAsync(d, width, hb, hpitch, width, (size_t)p.rows, kind, s);
        else
            e = cudaMemcpy2DAsync(hb, hpitch, d, width, width, (size_t)p.rows, kind, s);
    }
    if (e == cudaSuccess && p.tail) {
        char* ht = h + (size_t)(n - p.tail) * elem;
        char* dt = d + (size_t)(p.rows * p.w) * bw;
        e = kind == cudaMemcpyHostToDevice ? cudaMemcpyAsync(dt, ht, (size_t)p.tail * elem, kind, s)
                                           : cudaMemcpyAsync(ht, dt, (size_t)p.tail * elem, kind, s);
    }
    return e;
}
}  // namespace nbvh

extern "C" nbvh_status nbvh_query_host(nbvh_ctx* c, const nbvh_ray* h_rays, int64_t n, int32_t lod, nbvh_hits h_out,
                                       void* stream) {
    nbvh_status st = check_query(c, h_rays, n, lod, h_out);
    if (st) return st;
    if (n == 0) return NBVH_OK;
    // Pipeline over chunks: host->device copies on one auxiliary stream, the queries in order
    // on the caller's stream (they share the query workspace), device->host copies on a
    // second auxiliary stream; events order chunk k's query after its upload and its
    // download after its query, so copies of chunks k+1 / k-1 overlap the query of chunk k.
    cudaStream_t S = (cudaStream_t)stream;
    for (int i = 0; i < 3; ++i)
        if (!c->aux_stream[i]) {
            cudaError_t e0 = cudaStreamCreateWithFlags(&c->aux_stream[i], cudaStreamNonBlocking);
            if (e0 != cudaSuccess) return cuda_fail(c, e0, "query_host: stream");
        }
    cudaStream_t H = c->aux_stream[0], Dn = c->aux_stream[1];
    // chunks alternate between the caller's stream and a second query stream; each chunk uses
    // its own workspace slice and counter block, so consecutive chunks' kernels overlap (one
    // chunk's tail CTAs next to the next chunk's first CTAs)
    cudaStream_t Q[2] = {S, c->aux_stream[2]};
    cudaError_t e0 = cudaEventRecord(ctx_event(c, 31), S);            // Q[1] starts after prior work on S
    if (e0 == cudaSuccess) e0 = cudaStreamWaitEvent(Q[1], ctx_event(c, 31), 0);
    if (e0 != cudaSuccess) return cuda_fail(c, e0, "query_host: stream order");
    ChunkPlan plan[kMaxChunks];
    const int chunks = plan_chunks(n, plan);
    int64_t W = 0;
    for (int k = 0; k < chunks; ++k) W += plan[k].w;
    // staging layout: t[n], normal[3n], albedo[3n], leaf[n], nq[n], hit bytes
    float* base = c->d_stage_hits;
    HitsDev d{};
    d.t = base;
    d.normal = base + n;
    d.albedo = base + 4 * n;
    d.leaf = reinterpret_cast<int32_t*>(base + 7 * n);
    d.n_queries = reinterpret_cast<int32_t*>(base + 8 * n);
    d.hit = reinterpret_cast<uint8_t*>(base + 9 * n);
    nbvh_ray* d_rays = reinterpret_cast<nbvh_ray*>(c->d_stage_rays);
    cudaError_t e = cudaSuccess;
    // events 32.. : [32+2k] upload k done, [33+2k] query k done (0-2 query profiling, 16-23 training);
    // 64 + 4k + {0 upload start, 1 query start, 2 download start, 3 download done}: the
    // NBVH_HOST_TIMELINE=1 diagnostic (chunk timeline printed to stderr, scripts/e2e_timeline.py)
    static const bool timeline = std::getenv("NBVH_HOST_TIMELINE") != nullptr;
    for (int k = 0; k < chunks && e == cudaSuccess; ++k) {
        if (timeline) cudaEventRecord(ctx_event(c, 64 + 4 * k), H);
        e = copy_chunk(const_cast<nbvh_ray*>(h_rays), d_rays, sizeof(nbvh_ray), n, W, plan[k],
                       cudaMemcpyHostToDevice, H);
        if (e == cudaSuccess) e = cudaEventRecord(ctx_event(c, 32 + 2 * k), H);
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "query_host: H2D");
    for (int k = 0; k < chunks; ++k) {
        const int64_t o = plan[k].dev_off, m = plan[k].size();
        if (m == 0) continue;
        HitsDev dk{d.hit + o, d.t + o, d.normal + 3 * o, d.albedo + 3 * o, d.leaf + o, d.n_queries + o};
        cudaStream_t Sq = Q[k & 1];
        e = cudaStreamWaitEvent(Sq, ctx_event(c, 32 + 2 * k), 0);
        if (e != cudaSuccess) return cuda_fail(c, e, "query_host: wait");
        if (timeline) cudaEventRecord(ctx_event(c, 65 + 4 * k), Sq);
        st = run_query(c, d_rays + o, m, lod, dk, nullptr, 0, Sq, true, o, k);
        if (st) return st;
        e = cudaEventRecord(ctx_event(c, 33 + 2 * k), Sq);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(Dn, ctx_event(c, 33 + 2 * k), 0);
        if (timeline) cudaEventRecord(ctx_event(c, 66 + 4 * k), Dn);
        if (e == cudaSuccess) e = copy_chunk(h_out.hit, d.hit, 1, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e == cudaSuccess) e = copy_chunk(h_out.t, d.t, 4, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e == cudaSuccess)
            e = copy_chunk(h_out.normal, d.normal, 12, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e == cudaSuccess)
            e = copy_chunk(h_out.albedo, d.albedo, 12, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e == cudaSuccess && h_out.leaf)
            e = copy_chunk(h_out.leaf, d.leaf, 4, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e == cudaSuccess && h_out.n_queries)
            e = copy_chunk(h_out.n_queries, d.n_queries, 4, n, W, plan[k], cudaMemcpyDeviceToHost, Dn);
        if (e != cudaSuccess) return cuda_fail(c, e, "query_host: copies");
        if (timeline) cudaEventRecord(ctx_event(c, 67 + 4 * k), Dn);
    }
    e = cudaStreamSynchronize(Dn);
    if (e == cudaSuccess) e = cudaStreamSynchronize(Q[1]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(S);
    if (e != cudaSuccess) return cuda_fail(c, e, "query_host: D2H");
    if (timeline) {
        auto at = [&](int i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx_event(c, 64), ctx_event(c, i));
            return ms;
        };
        for (int k = 0; k < chunks; ++k)
            std::fprintf(stderr, "chunk %d (%lld rays): up %.3f-%.3f  query %.3f-%.3f  down %.3f-%.3f ms\n", k,
                         (long long)plan[k].size(), at(64 + 4 * k), at(32 + 2 * k), at(65 + 4 * k), at(33 + 2 * k),
                         at(66 + 4 * k), at(67 + 4 * k));
    }
    c->qstats.n_rays = n;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_set_profiling(nbvh_ctx* c, int32_t on) {
    if (!c) return NBVH_EINVAL;
    c->profiling = on != 0;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_get_query_stats(nbvh_ctx* c, nbvh_query_stats* out) {
    if (!c || !out) return NBVH_EINVAL;
    nbvh_status st = resolve_query_stats(c);
    *out = c->qstats;
    return st;
}

// ------------------------------------------------------------------ parity hooks
extern "C" nbvh_status nbvh_debug_traverse(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, int32_t lod, int32_t cap,
                                           int32_t* leaf, float* te, float* tx, int32_t* count, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "debug_traverse: lod");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "debug_traverse: no cut");
    if (n < 0 || cap < 1 || (n > 0 && (!rays || !leaf || !te || !tx || !count)))
        return fail(c, NBVH_EINVAL, "debug_traverse: bad args");
    if (n == 0) return NBVH_OK;
    DebugTraverseArgs a{};
    a.cut = make_cut(c, lod);
    a.rays = reinterpret_cast<const float4*>(rays);
    a.n_rays = n;
    a.cap = cap;
    a.k = c->cfg.list_cap;
    a.leaf = leaf;
    a.te = te;
    a.tx = tx;
    a.count = count;
    a.err = c->d_misc;
    cudaError_t e = launch_debug_traverse(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_traverse");
    return NBVH_OK;
}

// The product traversal's per-ray lists, unpacked from k_traverse's own outputs (the work
// records hold entry 0, the fill count and the more-flag; the list buffer the rest).
__global__ void k_unpack_product_lists(const WorkRec* act_long, const WorkRec* act, const QueryCounters* ctr,
                                       const float4* lst, int64_t n_rays, int32_t K, int32_t* leaf, float* te,
                                       float* tx, int32_t* fill, int32_t* more) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_long = ctr->cnt_long, total = n_long + ctr->cnt;
    if (i >= total) return;
    const WorkRec w = i < n_long ? act_long[i] : act[i - n_long];
    const int64_t r = __float_as_int(w.o.w);
    const int st = __float_as_int(w.d.w), nn = st & 0xffff;
    fill[r] = nn;
    more[r] = st >> 16;
    for (int j = 0; j < nn && j < K; ++j) {
        const float4 e = j == 0 ? w.e0 : lst[(int64_t)j * n_rays + r];
        leaf[r * K + j] = __float_as_int(e.z);
        te[r * K + j] = e.x;
        tx[r * K + j] = e.y;
    }
}

extern "C" nbvh_status nbvh_debug_traverse_product(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, int32_t lod,
                                                   int32_t* leaf, float* te, float* tx, int32_t* fill, int32_t* more,
                                                   void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "debug_traverse_product: lod");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "debug_traverse_product: no cut");
    if (n < 0 || (n > 0 && (!rays || !leaf || !te || !tx || !fill || !more)))
        return fail(c, NBVH_EINVAL, "debug_traverse_product: bad args");
    if (n > c->reserved) return fail(c, NBVH_ESTATE, "debug_traverse_product: n exceeds nbvh_reserve");
    if (n == 0) return NBVH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int K = c->cfg.list_cap;
    QueryCounters* ctr = counter_block(c, 0);
    k_reset_counters<<<1, 32, 0, s>>>(ctr, 1);
    HitsDev out{};
    unsigned char* scratch = nullptr;                      // miss records of k_traverse (not compared)
    cudaError_t e = cudaMallocAsync((void**)&scratch, (size_t)n * 37, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(leaf, 0xff, (size_t)n * K * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(te, 0, (size_t)n * K * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(tx, 0, (size_t)n * K * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(fill, 0, (size_t)n * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(more, 0, (size_t)n * 4, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_traverse_product");
    out.hit = scratch;
    out.t = reinterpret_cast<float*>(scratch + n);
    out.normal = out.t + n;
    out.albedo = out.normal + 3 * n;
    out.leaf = reinterpret_cast<int32_t*>(out.albedo + 3 * n);
    out.n_queries = out.leaf + n;
    TraverseArgs ta{};
    ta.cut = make_cut(c, lod);
    ta.rays = reinterpret_cast<const float4*>(rays);
    ta.n_rays = n;
    ta.cap = K;
    ta.lst = c->d_lst;
    ta.st = c->state();
    ta.out = out;
    ta.act_out = c->d_act;
    ta.act_long = c->d_act_long;
    ta.ctr = ctr;
    e = launch_traverse(ta, s);                            // the product kernel (k_traverse)
    if (e == cudaSuccess) {
        k_unpack_product_lists<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->d_act_long, c->d_act, ctr, c->d_lst, n,
                                                                         K, leaf, te, tx, fill, more);
        e = cudaGetLastError();
    }
    cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_traverse_product");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_encode(nbvh_ctx* c, const float* pts, int64_t m, uint16_t* feat, uint32_t* index,
                                         void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (m < 0 || (m > 0 && (!pts || !feat))) return fail(c, NBVH_EINVAL, "debug_encode: bad args");
    if (m == 0) return NBVH_OK;
    DebugEncodeArgs a{};
    a.g = make_grid(c, -1);
    a.pts = pts;
    a.m = m;
    a.feat = reinterpret_cast<__half*>(feat);
    a.index = index;
    cudaError_t e = launch_debug_encode(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_encode");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_mlp(nbvh_ctx* c, const uint16_t* x, int64_t m, float* z, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (m < 0 || (m > 0 && (!x || !z))) return fail(c, NBVH_EINVAL, "debug_mlp: bad args");
    if (m == 0) return NBVH_OK;
    DebugMlpArgs a{};
    a.m = make_mlp(c);
    if (c->d_Wb16) {                      // the query path's own MLP: bf16 operands (C39)
        a.m.W = reinterpret_cast<const __half*>(c->d_Wb16);
        a.m.bf16 = 1;
    }
    a.x = reinterpret_cast<const __half*>(x);
    a.rows = m;
    a.z = z;
    cudaError_t e = launch_debug_mlp(a, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_mlp");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_query_trace(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, int32_t lod,
                                              nbvh_hits out, float* z_trace, int32_t cap, void* stream) {
    nbvh_status st = check_query(c, rays, n, lod, out);
    if (st) return st;
    if (!z_trace || cap < 1) return fail(c, NBVH_EINVAL, "debug_query_trace: bad trace");
    if (n == 0) return NBVH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(z_trace, 0xff, (size_t)n * cap * 8 * sizeof(float), s);   // NaN
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_query_trace: memset");
    return run_query(c, rays, n, lod, to_dev(out), z_trace, cap, s, true, 0, 0);
}
