// nbvh_train.cu — scene/cut upload and the companion training step (T0-T9).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include <cmath>
#include <string>

#include "nbvh_capi_internal.h"
#include "nbvh_train_kernels.cuh"

namespace nbvh {

struct TrainWork {
    int64_t cap = 0;                 // rays (and samples) per call
    uint8_t* r_acc = nullptr;
    int32_t* r_leaf = nullptr;
    float* r_gt = nullptr;
    float* r_loss = nullptr;
    int32_t* s_ray = nullptr;
    int32_t* s_leaf = nullptr;
    float* s_t0 = nullptr;
    float* s_t1 = nullptr;
    float* s_gt = nullptr;
    __half* X = nullptr;
    __half* A = nullptr;
    __half* Dl = nullptr;
    float* dZ = nullptr;
    float* Z = nullptr;              // [cap][8] raw z, allocated only while parity capture is on
    float* gx = nullptr;             // [cap][D] dL/dx (bwd -> scatter)
    unsigned long long tex_gx = 0;   // texture object over gx (float2 texels; the scatter's reads, F = 2)
    int32_t* ss_ray = nullptr;       // samples grouped by leaf (k_sort_place): ray, leaf, t0, t1
    int32_t* ss_leaf = nullptr;
    float* ss_t0 = nullptr;
    float* ss_t1 = nullptr;
    int32_t* leaf_hist = nullptr;    // [hist_cap] per-leaf counts -> offsets
    int64_t hist_cap = 0;
    float* sc_dense = nullptr;       // T7 scratch: cell-packed dense levels
    float* sc_hash = nullptr;        // T7 scratch: aligned hashed levels
    int32_t* sc_priv = nullptr;      // T7 fixed-point partials of the coarse levels, per scatter CTA
    int64_t sc_dense_floats = 0, sc_hash_floats = 0, sc_priv_ints = 0;
    bool capture = false;
    float* grad = nullptr;           // params + 1 + 3 * tail_leaves
    int64_t tail_leaves = 0;
    float* m = nullptr;
    float* v = nullptr;
    int32_t* counters = nullptr;     // [0] samples, [1] first hits, [2] non-finite flag
    double* loss_acc = nullptr;      // [5]
    int32_t* adam_step = nullptr;    // device: Adam updates applied (skipped updates excluded)
    float* draw = nullptr;           // nbvh_train_step's own T0 draws: rays [n][8], u [n], xi [n][n_points]
    int64_t draw_cap = 0;
    uint64_t draw_step = 0;          // Philox counter of the next self-drawn batch
    int32_t lod = 0;
    int32_t launches = 0;
    cudaStream_t stream = nullptr;
    bool profiled = false, adam_profiled = false;
};

template <typename T>
static cudaError_t upload(T** dst, const T* src, size_t count) {
    if (*dst) cudaFree(*dst);
    *dst = nullptr;
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc((void**)dst, count * sizeof(T));
    if (e == cudaSuccess) e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

nbvh_status upload_scene(nbvh_ctx* c) {
    nbvh_status st = check_device(c);
    if (st) return st;
    const HostScene& sc = c->sc;
    const int64_t nt = (int64_t)sc.tri.size() / 3;
    std::vector<float> v(9 * nt), n(9 * nt), a(3 * nt);
    std::vector<int32_t> id(nt);
    for (int64_t i = 0; i < nt; ++i) {
        const int32_t t = sc.prim[i];
        id[i] = t;
        for (int j = 0; j < 3; ++j) {
            const uint32_t vi = sc.tri[3 * t + j];
            for (int k = 0; k < 3; ++k) {
                v[9 * i + 3 * j + k] = sc.xyz[3 * vi + k];
                n[9 * i + 3 * j + k] = sc.vnormal[3 * vi + k];
            }
        }
        for (int k = 0; k < 3; ++k) a[3 * i + k] = sc.albedo[3 * t + k];
    }
    cudaError_t e = upload(&c->dscene.nodes, sc.nodes.data(), sc.nodes.size());
    if (e == cudaSuccess) e = upload(&c->dscene.tri_v, v.data(), v.size());
    if (e == cudaSuccess) e = upload(&c->dscene.tri_n, n.data(), n.size());
    if (e == cudaSuccess) e = upload(&c->dscene.tri_a, a.data(), a.size());
    if (e == cudaSuccess) e = upload(&c->dscene.tri_id, id.data(), id.size());
    if (e != cudaSuccess) return cuda_fail(c, e, "upload_scene");
    c->dscene.n_tris = nt;
    return NBVH_OK;
}

nbvh_status upload_cut(nbvh_ctx* c, int lod) {
    nbvh_status st = check_device(c);
    if (st) return st;
    const HostCut& hc = c->cuts[lod];
    // the device traversal stack holds 64 entries: at most depth+1 are live (P:163 shallow hierarchy)
    int32_t cut_depth = 0;
    if (hc.n_leaves > 1) {
        std::vector<std::pair<int32_t, int32_t>> todo{{0, 1}};
        int32_t depth = 0;
        while (!todo.empty()) {
            auto [i0, dpt] = todo.back();
            todo.pop_back();
            depth = std::max(depth, dpt);
            for (int32_t ch : {hc.inner[i0].l, hc.inner[i0].r})
                if (ch >= 0) todo.push_back({ch, dpt + 1});
        }
        if (depth > 62) return fail(c, NBVH_EINVAL, "cut hierarchy deeper than the 62 levels the traversal stack holds");
        cut_depth = depth;
    }
    std::vector<float4> box(2 * (size_t)hc.n_leaves);
    for (int32_t i = 0; i < hc.n_leaves; ++i) {
        box[2 * i] = make_float4(hc.leaf_lo[3 * i], hc.leaf_lo[3 * i + 1], hc.leaf_lo[3 * i + 2], 0.f);
        box[2 * i + 1] = make_float4(hc.leaf_hi[3 * i], hc.leaf_hi[3 * i + 1], hc.leaf_hi[3 * i + 2], 0.f);
    }
    cudaDeviceSynchronize();
    DeviceCut& d = c->dcut[lod];
    cudaError_t e = upload(&d.inner, hc.inner.data(), hc.inner.size());
    if (e == cudaSuccess) e = upload(&d.leaf_box, box.data(), box.size());
    if (e == cudaSuccess) e = upload(&d.leaf_base, hc.leaf_base.data(), hc.leaf_base.size());
    if (e == cudaSuccess) e = upload(&d.rank, hc.rank.data(), hc.rank.size());
    if (e != cudaSuccess) return cuda_fail(c, e, "upload_cut");
    d.depth = cut_depth;
    return NBVH_OK;
}

void free_scene_device(nbvh_ctx* c) {
    DeviceScene& d = c->dscene;
    for (void* p : {(void*)d.nodes, (void*)d.tri_v, (void*)d.tri_n, (void*)d.tri_a, (void*)d.tri_id})
        if (p) cudaFree(p);
    d = DeviceScene{};
}

template <typename T>
static void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

static void free_work(TrainWork* w) {
    dfree(w->r_acc); dfree(w->r_leaf); dfree(w->r_gt); dfree(w->r_loss);
    dfree(w->s_ray); dfree(w->s_leaf); dfree(w->s_t0); dfree(w->s_t1); dfree(w->s_gt);
    if (w->tex_gx) cudaDestroyTextureObject((cudaTextureObject_t)w->tex_gx);
    w->tex_gx = 0;
    dfree(w->X); dfree(w->A); dfree(w->Dl); dfree(w->dZ); dfree(w->Z); dfree(w->gx);
    dfree(w->ss_ray); dfree(w->ss_leaf); dfree(w->ss_t0); dfree(w->ss_t1);
}

void free_train_device(nbvh_ctx* c) {
    if (!c->train) return;
    free_work(c->train);
    dfree(c->train->grad);
    dfree(c->train->m);
    dfree(c->train->v);
    dfree(c->train->counters);
    dfree(c->train->loss_acc);
    dfree(c->train->adam_step);
    dfree(c->train->sc_dense);
    dfree(c->train->sc_hash);
    dfree(c->train->sc_priv);
    dfree(c->train->draw);
    dfree(c->train->leaf_hist);
    delete c->train;
    c->train = nullptr;
}

static int64_t n_params(const nbvh_ctx* c) { return c->n_table + c->n_W + c->n_b; }

// Gradient buffer, Adam moments and counters (independent of the batch size).
static nbvh_status ensure_train_state(nbvh_ctx* c, int64_t tail_leaves) {
    if (!c->train) c->train = new TrainWork();
    TrainWork* w = c->train;
    cudaError_t e = cudaSuccess;
    if (!w->m) {
        const size_t np = (size_t)n_params(c);
        e = cudaMalloc((void**)&w->m, np * 4);
        if (e == cudaSuccess) e = cudaMalloc((void**)&w->v, np * 4);
        if (e == cudaSuccess) e = cudaMemset(w->m, 0, np * 4);
        if (e == cudaSuccess) e = cudaMemset(w->v, 0, np * 4);
        if (e == cudaSuccess) e = cudaMalloc((void**)&w->counters, 16 * sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMalloc((void**)&w->loss_acc, 8 * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc((void**)&w->adam_step, sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMemset(w->adam_step, 0, sizeof(int32_t));
    }
    if (e == cudaSuccess && (!w->grad || tail_leaves > w->tail_leaves)) {
        dfree(w->grad);
        const size_t ng = (size_t)(n_params(c) + 1 + 3 * tail_leaves);
        e = cudaMalloc((void**)&w->grad, ng * 4);
        if (e == cudaSuccess) e = cudaMemset(w->grad, 0, ng * 4);
        w->tail_leaves = tail_leaves;
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "train state");
    return NBVH_OK;
}

nbvh_status reserve_train(nbvh_ctx* c, int64_t max_rays) {
    nbvh_status st = ensure_train_state(c, 1);
    if (st) return st;
    TrainWork* w = c->train;
    if (w->cap >= max_rays) return NBVH_OK;
    free_work(w);
    const size_t n = (size_t)max_rays, H = (size_t)c->cfg.hidden_layers, D = (size_t)c->d_in;
    cudaError_t e = cudaMalloc((void**)&w->r_acc, n);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->r_leaf, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->r_gt, n * 9 * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->r_loss, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->s_ray, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->s_leaf, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->s_t0, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->s_t1, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->s_gt, n * 9 * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->X, n * D * 2);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->A, H * n * 64 * 2);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->Dl, H * n * 64 * 2);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->dZ, n * 8 * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->gx, n * D * 4);
    if (e == cudaSuccess && c->cfg.F == 2 && (int64_t)n * D / 2 <= ((int64_t)1 << 27)) {
        // the T7 scatter reads dL/dx through the texture pipe (its load pipe is the limit)
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = w->gx;
        rd.res.linear.desc = cudaCreateChannelDesc<float2>();
        rd.res.linear.sizeInBytes = (size_t)n * D * 4;
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        td.filterMode = cudaFilterModePoint;
        td.addressMode[0] = cudaAddressModeClamp;
        cudaTextureObject_t t = 0;
        if (cudaCreateTextureObject(&t, &rd, &td, nullptr) == cudaSuccess) w->tex_gx = t;
        else cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->ss_ray, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->ss_leaf, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->ss_t0, n * 4);
    if (e == cudaSuccess) e = cudaMalloc((void**)&w->ss_t1, n * 4);
    if (e != cudaSuccess) {
        free_work(w);
        cudaGetLastError();
        return fail(c, NBVH_ENOMEM, std::string("reserve (training): ") + cudaGetErrorString(e));
    }
    w->cap = max_rays;
    return NBVH_OK;
}

void reset_adam(nbvh_ctx* c) {
    if (!c->train || !c->train->m) return;
    const size_t np = (size_t)n_params(c);
    cudaMemset(c->train->m, 0, np * 4);
    cudaMemset(c->train->v, 0, np * 4);
    cudaMemset(c->train->adam_step, 0, sizeof(int32_t));
}

// launchers (templated on F, D)
// Shared memory of k_train_bwd: the weights and one staging tile per warp
static size_t bwd_smem(int D, int H) {
    return ((bwd_weights_bytes(D, H) + 15) & ~(size_t)15) + (size_t)kBwdWarps * bwd_tile_bytes(D);
}
// Gradient floats of coarse levels k_train_scatter accumulates in shared memory (8 bytes
// each: two int32 fixed-point parts), budgeted for two CTAs per SM.
constexpr int64_t kScatterPrivBudget = 52 * 1024;
// Levels the default scatter warp-aggregates (k_train_scatter_agg; profiles/NOTES.md r2d)
constexpr int kScatterAggLevels = 6;
// Dynamic shared memory of the T7 scatter: the fixed-point accumulator, and with warp
// aggregation one [32][8F]-float slot array per warp (8 warps)
static size_t scatter_smem(const TrainArgs& a) {
    const size_t priv = (size_t)((2 * (int64_t)a.priv_floats + 3) & ~(int64_t)3) * 4;
    return priv + (a.agg_levels > 0 ? (size_t)8 * 32 * 8 * a.g.F * 4 : 0);
}
// CTAs of the scatter per SM: as many as its shared memory allows (<= 6)
static int scatter_ctas_per_sm(const TrainArgs& a) {
    const int64_t per_cta = (int64_t)scatter_smem(a) + 2048;
    int64_t cap = 6;
    if (const char* ev = std::getenv("NBVH_SCATTER_CTAS")) cap = std::max(1, std::atoi(ev));   // A/B hook
    return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (int64_t)(228 * 1024) / per_cta));
}

// T7 scratch layout (k_train_scatter): every dense level cell-packed (N^3 cells x 8 corners x
// F floats) in sc_dense, every hashed level [T][F] in sc_hash; offsets 16-byte aligned.
static nbvh_status ensure_scatter_scratch(nbvh_ctx* c, TrainArgs& a, int sms) {
    TrainWork* w = c->train;
    const int F = c->cfg.F;
    int64_t nd = 0, nh = 0;
    for (int l = 0; l < c->cfg.L; ++l) {
        if (c->dense[l]) {
            a.sc_off[l] = nd;
            nd += (int64_t)c->res[l] * c->res[l] * c->res[l] * 8 * F;
        } else {
            a.sc_off[l] = nh;
            nh += ((int64_t)1 << c->cfg.log2_T) * F;
        }
        nd = (nd + 3) & ~(int64_t)3;
        nh = (nh + 3) & ~(int64_t)3;
    }
    const int64_t np = (int64_t)sms * scatter_ctas_per_sm(a) * 2 * a.priv_floats;
    cudaError_t e = cudaSuccess;
    if (nd > w->sc_dense_floats) {
        dfree(w->sc_dense);
        e = cudaMalloc((void**)&w->sc_dense, (size_t)std::max<int64_t>(nd, 4) * 4);
        w->sc_dense_floats = nd;
    }
    if (e == cudaSuccess && nh > w->sc_hash_floats) {
        dfree(w->sc_hash);
        e = cudaMalloc((void**)&w->sc_hash, (size_t)std::max<int64_t>(nh, 4) * 4);
        w->sc_hash_floats = nh;
    }
    if (e == cudaSuccess && np > w->sc_priv_ints) {
        dfree(w->sc_priv);
        e = cudaMalloc((void**)&w->sc_priv, (size_t)std::max<int64_t>(np, 4) * 4);
        w->sc_priv_ints = np;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, NBVH_ENOMEM, "train: T7 scratch");
    }
    // the hashed levels (coarse-to-fine, after the dense ones) are contiguous in the scratch
    // (T*F floats each, a multiple of 4) and, if also in the canonical layout, copied flat
    a.hash_coff0 = -1;
    a.hash_floats = nh;
    {
        int64_t first = -1, expect = 0;
        bool contiguous = true;
        for (int l = 0; l < c->cfg.L; ++l) {
            if (c->dense[l]) {
                if (first >= 0) contiguous = false;          // a dense level after a hashed one
                continue;
            }
            if (first < 0) first = expect = c->offset[l];
            if (c->offset[l] != expect || a.sc_off[l] != (expect - first) * F) contiguous = false;
            expect += (int64_t)1 << c->cfg.log2_T;
        }
        if (first >= 0 && contiguous) a.hash_coff0 = first;
    }
    a.sc_dense = w->sc_dense;
    a.sc_hash = w->sc_hash;
    a.sc_priv = w->sc_priv;
    a.scatter_ctas = sms * scatter_ctas_per_sm(a);
    w->sc_dense_floats = std::max(w->sc_dense_floats, nd);
    return NBVH_OK;
}

// ev (nullable): 6 events recorded before select and after select, label, fwd, bwd, dW
// a0: the arguments with the select kernel's (unsorted) sample arrays; a: the same with the
// leaf-sorted arrays, which every kernel after the sort reads; hist: n_leaves ints.
template <int F, int D>
static cudaError_t launch_train_fd(const TrainArgs& a0, const TrainArgs& a, int32_t* hist, int64_t n, int64_t w_off,
                                   int64_t b_off, cudaStream_t s, int* launches, cudaEvent_t* ev) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int H = a.m.hidden;
    const size_t smem_fwd = FwdSmemPlan(D, H, a.g.n_points).total;
    const size_t smem_bwd = bwd_smem(D, H);
    const size_t smem_sc = scatter_smem(a);
    const size_t smem_dw = (size_t)kTileQ * 72 * 2 + (size_t)kTileQ * (D + 8) * 2 + kTileQ * 8 * 4;
    // T3 gathers of the hashed levels through the TEX pipe when the texture object exists (F = 2)
    const bool tex = a.g.tex != 0 && F == 2 && !(std::getenv("NBVH_TRAIN_TEX") && std::getenv("NBVH_TRAIN_TEX")[0] == '0');
    auto fwd = tex ? k_train_fwd<F, D, true> : k_train_fwd<F, D, false>;
    cudaError_t e = cudaFuncSetAttribute(fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fwd);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_train_bwd<F, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bwd);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_train_dw<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dw);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(a.agg_levels > 0 ? (const void*)k_train_scatter_agg<F> : (const void*)k_train_scatter<F>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_sc);
    if (e != cudaSuccess) return e;
    const unsigned blocks_n = (unsigned)((n + 127) / 128);
    // every launch is checked at once: a failed launch must not leave a step that silently
    // skipped a phase
    if ((e = cudaMemsetAsync(hist, 0, sizeof(int32_t) * (size_t)a.cut.n_leaves, s)) != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[0], s);
    TrainArgs asel = a0;
    asel.leaf_hist = hist;                    // T1 counts the accepted samples per leaf
    k_train_select<<<blocks_n, 128, (size_t)(a.cut.depth + 2) * 128 * sizeof(int), s>>>(asel);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // group the samples by leaf (the later kernels read a's sorted arrays)
    k_sort_scan<<<1, 1024, 0, s>>>(hist, a.cut.n_leaves);
    k_sort_place<<<2 * sms, 256, 0, s>>>(a0, hist, SortedSamples{a.s_ray, a.s_leaf, a.s_t0, a.s_t1});
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 2;
    if (ev) cudaEventRecord(ev[1], s);
    k_train_label<<<blocks_n, 128, (size_t)a.bvh_rows * 128 * sizeof(int), s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[2], s);
    const int grid_fwd = sms;                 // persistent: one CTA of kFwdWarps warps per SM
    fwd<<<grid_fwd, kFwdWarps * 32, smem_fwd, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[3], s);
    k_train_bwd<F, D><<<2 * sms, 256, smem_bwd, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // T7: scatter into the scratch (dense / hashed regions zeroed first), then the canonical
    // gradient buffer
    e = cudaMemsetAsync(a.sc_dense, 0, sizeof(float) * (size_t)a.sc_dense_n, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.sc_hash, 0, sizeof(float) * (size_t)a.sc_hash_n, s);
    if (e != cudaSuccess) return e;
    if (a.agg_levels > 0) k_train_scatter_agg<F><<<a.scatter_ctas, 256, smem_sc, s>>>(a);
    else k_train_scatter<F><<<a.scatter_ctas, 256, smem_sc, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_train_scatter_finish<F><<<4 * sms, 256, 0, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *launches += 2;
    if (ev) cudaEventRecord(ev[4], s);
    const unsigned dw_grid = (unsigned)((n + kDwChunk - 1) / kDwChunk);
    bool tc_done = false;
    if (a.use_tc_dw) {
        // weight GEMMs of the input + hidden layers on tcgen05; biases and the 8-output layer
        // on the CUDA-core kernel
        auto run_tc = [&](auto kern, int Hc) {
            const size_t sm = dw_tc_smem(D, Hc);
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (e != cudaSuccess) return;
            kern<<<sms, kDwThreads, sm, s>>>(a, w_off);
            e = cudaGetLastError();
            tc_done = e == cudaSuccess;
        };
        if (H == 1 && dw_tc_ok(D, 1)) run_tc(k_train_dw_tc<D, 1>, 1);
        else if (H == 2 && dw_tc_ok(D, 2)) run_tc(k_train_dw_tc<D, 2>, 2);
        else if (H == 3 && dw_tc_ok(D, 3)) run_tc(k_train_dw_tc<D, 3>, 3);
        else if (H == 4 && dw_tc_ok(D, 4)) run_tc(k_train_dw_tc<D, 4>, 4);
        if (e != cudaSuccess) return e;
    }
    if (tc_done) {
        // output-layer weights follow the input and hidden layers in the weight block
        int64_t w_out = w_off + (int64_t)64 * D + (int64_t)(H - 1) * 64 * 64;
        k_train_bias_out<<<2 * sms, 256, 0, s>>>(a, w_out, b_off);
        ++*launches;
    } else {
        k_train_dw<D><<<dw_grid > 0 ? dw_grid : 1, 256, smem_dw, s>>>(a, w_off, b_off);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (ev) cudaEventRecord(ev[5], s);
    *launches += 5;
    return cudaGetLastError();
}

__global__ void k_store_count(const int32_t* n, float* dst) { *dst = (float)*n; }

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_set_leaf_rank(nbvh_ctx* c, int32_t lod, const float* h_rank) {
    if (!c || !h_rank) return NBVH_EINVAL;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "set_leaf_rank: lod");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "set_leaf_rank: no cut");
    HostCut& hc = c->cuts[lod];
    for (int32_t i = 0; i < hc.n_leaves; ++i)
        if (!std::isfinite(h_rank[i])) return fail(c, NBVH_EINVAL, "set_leaf_rank: non-finite rank");
    std::memcpy(hc.rank.data(), h_rank, sizeof(float) * hc.n_leaves);
    if (c->device >= 0) {
        nbvh_status st = check_device(c);
        if (st) return st;
        cudaError_t e = cudaMemcpy(c->dcut[lod].rank, h_rank, sizeof(float) * hc.n_leaves, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(c, e, "set_leaf_rank");
    }
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_train_backward(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, const float* u,
                                           const float* xi, int32_t lod, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "train_backward: lod");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "train_backward: no cut");
    if (n < 0 || (n > 0 && (!rays || !u || !xi))) return fail(c, NBVH_EINVAL, "train_backward: null pointer");
    if (n > c->reserved) return fail(c, NBVH_ESTATE, "train_backward: n exceeds nbvh_reserve");
    if (c->cfg.n_points > 4) return fail(c, NBVH_EINVAL, "train_backward: n_points > 4 not supported");
    const HostCut& hc = c->cuts[lod];
    st = ensure_train_state(c, hc.n_leaves);
    if (st) return st;
    st = reserve_train(c, c->reserved);
    if (st) return st;
    TrainWork* w = c->train;
    cudaStream_t s = (cudaStream_t)stream;
    w->stream = s;
    w->lod = lod;
    w->launches = 0;
    const int64_t ng = n_params(c) + 1 + 3 * (int64_t)hc.n_leaves;
    cudaError_t e = cudaMemsetAsync(w->grad, 0, (size_t)ng * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(w->counters, 0, 16 * sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(w->loss_acc, 0, 8 * sizeof(double), s);
    if (e != cudaSuccess) return cuda_fail(c, e, "train_backward: memset");
    c->tstats = nbvh_train_stats{};
    c->tstats.n_rays = n;
    if (n == 0) return NBVH_OK;
    // C18 rank normalisation in fp32 (the oracle does the same operations)
    float rmin = hc.rank[0], rmax = hc.rank[0];
    for (int32_t i = 1; i < hc.n_leaves; ++i) {
        rmin = std::fmin(rmin, hc.rank[i]);
        rmax = std::fmax(rmax, hc.rank[i]);
    }
    TrainArgs a{};
    a.g = make_grid(c, lod);
    a.m = make_mlp(c);
    a.cut = make_cut(c, lod);
    a.rays = reinterpret_cast<const float4*>(rays);
    a.n_rays = n;
    a.u = u;
    a.xi = xi;
    a.rank = c->dcut[lod].rank;
    a.rank_min = rmin;
    a.rank_hmax = (rmax - rmin) + 1e-6f;
    a.leaf_base = c->dcut[lod].leaf_base;
    a.nodes = c->dscene.nodes;
    if (c->base_depth < 0) c->base_depth = base_bvh_depth(c->sc);
    if (c->base_depth > kBvhStack) return fail(c, NBVH_EINVAL, "train: base BVH deeper than the stack");
    a.bvh_rows = c->base_depth > 0 ? c->base_depth : 1;
    a.tri_v = c->dscene.tri_v;
    a.tri_n = c->dscene.tri_n;
    a.tri_a = c->dscene.tri_a;
    a.tri_id = c->dscene.tri_id;
    a.r_acc = w->r_acc;
    a.r_leaf = w->r_leaf;
    a.r_gt = w->r_gt;
    a.r_loss = w->r_loss;
    a.n_samples = w->counters;
    a.n_first = w->counters + 1;
    a.s_ray = w->s_ray;
    a.s_leaf = w->s_leaf;
    a.s_t0 = w->s_t0;
    a.s_t1 = w->s_t1;
    a.s_gt = w->s_gt;
    a.X = w->X;
    a.A = w->A;
    a.Dl = w->Dl;
    a.dZ = w->dZ;
    if (w->capture && !w->Z) {
        e = cudaMalloc((void**)&w->Z, (size_t)w->cap * 8 * 4);
        if (e != cudaSuccess) return cuda_fail(c, e, "train_backward: capture buffer");
    }
    a.Z = w->capture ? w->Z : nullptr;
    a.grad = w->grad;
    a.tail = w->grad + n_params(c);
    a.loss_acc = w->loss_acc;
    a.cap = w->cap;
    // coarse dense levels whose gradients fit a CTA-private shared-memory accumulator (the
    // longest prefix that fits next to k_train_bwd's other shared memory, or NBVH_PRIV_BYTES)
    a.priv_levels = 0;
    a.priv_floats = 0;
    // NBVH_DW_MMA_SYNC=1 forces the mma.sync weight-gradient kernel (A/B parity tests)
    {
        const char* ev = std::getenv("NBVH_DW_MMA_SYNC");
        a.use_tc_dw = (ev && ev[0] == '1') ? 0 : 1;
    }
    {
        // T7: warp aggregation on the coarse levels (kScatterAggLevels; NBVH_SCATTER_AGG=n
        // overrides, 0 selects k_train_scatter with the privatised levels)
        const char* ev = std::getenv("NBVH_SCATTER_AGG");
        a.agg_levels = std::max(0, std::min(ev ? std::atoi(ev) : kScatterAggLevels, (int)c->cfg.L));
        // the grouping key is the cell's linear index N^3 < 2^31 (bit 31 marks idle lanes)
        while (a.agg_levels > 0 &&
               (int64_t)c->res[a.agg_levels - 1] * c->res[a.agg_levels - 1] * c->res[a.agg_levels - 1] >= (1ll << 31))
            --a.agg_levels;
    }
    // shared-memory privatisation: only without aggregation by default (NBVH_PRIV_BYTES
    // overrides; 0 disables)
    const char* pev = std::getenv("NBVH_PRIV_BYTES");
    const int64_t priv_budget = pev ? std::min<int64_t>(std::atoll(pev), kScatterPrivBudget)
                                    : (a.agg_levels > 0 ? 0 : kScatterPrivBudget);
    for (int l = 0; l < c->cfg.L && c->dense[l]; ++l) {
        const int64_t end = (c->offset[l] + (int64_t)(c->res[l] + 1) * (c->res[l] + 1) * (c->res[l] + 1)) * c->cfg.F;
        if (end * 4 > priv_budget) break;
        a.priv_levels = l + 1;
        a.priv_floats = (int32_t)end;
    }
    a.gx = w->gx;
    {
        const char* ev = std::getenv("NBVH_SCATTER_TEX");      // A/B hook: 0 = dL/dx on the load pipe
        a.tex_gx = (ev && ev[0] == '0') ? 0ull : w->tex_gx;
    }
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        st = ensure_scatter_scratch(c, a, sms);
        if (st) return st;
        a.sc_dense_n = w->sc_dense_floats;
        a.sc_hash_n = w->sc_hash_floats;
    }
    if (hc.n_leaves > w->hist_cap) {
        dfree(w->leaf_hist);
        e = cudaMalloc((void**)&w->leaf_hist, sizeof(int32_t) * (size_t)hc.n_leaves);
        if (e != cudaSuccess) return cuda_fail(c, e, "train_backward: leaf histogram");
        w->hist_cap = hc.n_leaves;
    }
    TrainArgs as = a;                         // the leaf-sorted sample arrays (k_sort_place)
    as.s_ray = w->ss_ray;
    as.s_leaf = w->ss_leaf;
    as.s_t0 = w->ss_t0;
    as.s_t1 = w->ss_t1;
    const int64_t w_off = c->n_table, b_off = c->n_table + c->n_W;
    const int F = c->cfg.F, D = c->d_in;
    int launches = 0;
    cudaEvent_t evs[6];
    cudaEvent_t* ev = nullptr;
    if (c->profiling) {
        for (int i = 0; i < 6; ++i) evs[i] = ctx_event(c, 16 + i);
        ev = evs;
    }
    w->profiled = c->profiling;
    if (F == 2 && D == 32) e = launch_train_fd<2, 32>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 2 && D == 64) e = launch_train_fd<2, 64>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 2 && D == 96) e = launch_train_fd<2, 96>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 2 && D == 128) e = launch_train_fd<2, 128>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 4 && D == 64) e = launch_train_fd<4, 64>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 4 && D == 96) e = launch_train_fd<4, 96>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else if (F == 4 && D == 128) e = launch_train_fd<4, 128>(a, as, w->leaf_hist, n, w_off, b_off, s, &launches, ev);
    else return fail(c, NBVH_EINVAL, "train_backward: unsupported (F, D_in)");
    if (e != cudaSuccess) return cuda_fail(c, e, "train_backward: launch");
    k_store_count<<<1, 1, 0, s>>>(w->counters, a.tail);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "train_backward: count");
    w->launches = launches + 1;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_grad_buffer(nbvh_ctx* c, float** d_grad, int64_t* n_floats) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!d_grad || !n_floats) return fail(c, NBVH_EINVAL, "grad_buffer: null pointer");
    if (!c->train || !c->train->grad) return fail(c, NBVH_ESTATE, "grad_buffer: no training batch yet");
    *d_grad = c->train->grad;
    *n_floats = n_params(c) + 1 + 3 * (int64_t)c->cuts[c->train->lod].n_leaves;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_apply_update(nbvh_ctx* c, float lr, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!c->train || !c->train->grad) return fail(c, NBVH_ESTATE, "apply_update: no gradient");
    if (!(lr >= 0.f) || !std::isfinite(lr)) return fail(c, NBVH_EINVAL, "apply_update: bad lr");
    TrainWork* w = c->train;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t np = n_params(c);
    cudaError_t e = cudaMemsetAsync(w->counters + 2, 0, 4, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "apply_update");
    if (c->profiling) cudaEventRecord(ctx_event(c, 22), s);
    k_check_finite<<<592, 256, 0, s>>>(w->grad, np, w->counters + 2);
    AdamArgs a{};
    a.param = c->d_params;
    a.grad = w->grad;
    a.m = w->m;
    a.v = w->v;
    a.n = np;
    a.count = w->grad + np;
    a.bad = w->counters + 2;
    a.lr = lr;
    a.beta1 = 0.9f;
    a.beta2 = 0.999f;
    a.eps = 1e-8f;
    a.step = w->adam_step;
    a.table16 = c->d_table16;
    a.n_table = c->n_table;
    a.W16 = c->d_W16;
    a.n_W = c->n_W;
    k_adam<<<4 * 148, 256, 0, s>>>(a);
    k_adam_commit<<<1, 1, 0, s>>>(w->counters + 2, w->adam_step);
    st = refresh_table(c, s);
    if (st) return st;
    if (c->profiling) cudaEventRecord(ctx_event(c, 23), s);
    w->adam_profiled = c->profiling;
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "apply_update: adam");
    w->launches += 4;
    w->stream = s;
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_train_step(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, const float* u, const float* xi,
                                       int32_t lod, float lr, void* stream) {
    if (!rays && !u && !xi && n > 0) {
        // T0 in the library (C16, C28'): Philox-4x32-10 draws of training step
        // `draw_step` (key = the context's seed) into context-owned buffers
        nbvh_status st = check_device(c);
        if (st) return st;
        st = ensure_train_state(c, 1);
        if (st) return st;
        TrainWork* w = c->train;
        const int np = c->cfg.n_points;
        if (n > w->draw_cap) {
            dfree(w->draw);
            cudaError_t e = cudaMalloc((void**)&w->draw, (size_t)n * (8 + 1 + np) * sizeof(float));
            if (e != cudaSuccess) return cuda_fail(c, e, "train_step: ray buffers");
            w->draw_cap = n;
        }
        float* d_rays = w->draw;
        float* d_u = d_rays + 8 * n;
        float* d_xi = d_u + n;
        st = nbvh_gen_train_rays(c, c->cfg.seed, w->draw_step++, 0, n, nullptr, reinterpret_cast<nbvh_ray*>(d_rays),
                                 d_u, d_xi, stream);
        if (st) return st;
        rays = reinterpret_cast<const nbvh_ray*>(d_rays);
        u = d_u;
        xi = d_xi;
    }
    nbvh_status st = nbvh_train_backward(c, rays, n, u, xi, lod, stream);
    if (st) return st;
    return nbvh_apply_update(c, lr, stream);
}

extern "C" nbvh_status nbvh_get_train_stats(nbvh_ctx* c, nbvh_train_stats* out) {
    if (!c || !out) return NBVH_EINVAL;
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!c->train || !c->train->counters) return fail(c, NBVH_ESTATE, "train_stats: no training call yet");
    TrainWork* w = c->train;
    cudaError_t e = cudaStreamSynchronize(w->stream);
    int32_t cnt[3];
    double la[5];
    if (e == cudaSuccess) e = cudaMemcpy(cnt, w->counters, sizeof(cnt), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(la, w->loss_acc, sizeof(la), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "train_stats");
    c->tstats.n_accepted = cnt[0];
    c->tstats.n_first_hit = cnt[1];
    c->tstats.loss_sum = la[0];
    for (int k = 0; k < 4; ++k) c->tstats.loss_terms[k] = la[1 + k];
    c->tstats.n_launches = w->launches;
    c->tstats.skipped = cnt[2] != 0;
    for (int k = 0; k < 6; ++k) c->tstats.ms_phase[k] = 0.f;
    if (w->profiled)
        for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&c->tstats.ms_phase[k], c->events[16 + k], c->events[17 + k]);
    if (w->adam_profiled) cudaEventElapsedTime(&c->tstats.ms_phase[5], c->events[22], c->events[23]);
    cudaGetLastError();
    *out = c->tstats;
    return cnt[2] ? NBVH_ENONFINITE : NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_train_samples(nbvh_ctx* c, float* gt, uint8_t* acc, int32_t* leaf, float* loss,
                                                void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!c->train || !c->train->r_acc) return fail(c, NBVH_ESTATE, "debug_train_samples: no training batch yet");
    const int64_t n = c->tstats.n_rays;
    cudaStream_t s = (cudaStream_t)stream;
    TrainWork* w = c->train;
    cudaError_t e = cudaSuccess;
    if (gt) e = cudaMemcpyAsync(gt, w->r_gt, (size_t)n * 9 * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && acc) e = cudaMemcpyAsync(acc, w->r_acc, (size_t)n, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && leaf) e = cudaMemcpyAsync(leaf, w->r_leaf, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && loss) e = cudaMemcpyAsync(loss, w->r_loss, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_train_samples");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_train_capture(nbvh_ctx* c, int32_t enable) {
    nbvh_status st = check_device(c);
    if (st) return st;
    st = ensure_train_state(c, 1);
    if (st) return st;
    c->train->capture = enable != 0;
    if (!enable) dfree(c->train->Z);
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_debug_train_activations(nbvh_ctx* c, int32_t* d_sample_ray, uint16_t* d_x, float* d_z,
                                                    float* d_dz, uint16_t* d_act, uint16_t* d_delta, int64_t* h_m,
                                                    void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!h_m) return fail(c, NBVH_EINVAL, "debug_train_activations: null count pointer");
    if (!c->train || !c->train->X) return fail(c, NBVH_ESTATE, "debug_train_activations: no training batch yet");
    TrainWork* w = c->train;
    if (d_z && !(w->capture && w->Z)) return fail(c, NBVH_ESTATE, "debug_train_activations: z needs capture on");
    cudaStream_t s = (cudaStream_t)stream;
    int32_t m32 = 0;
    cudaError_t e = cudaMemcpyAsync(&m32, w->counters, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_train_activations");
    const size_t m = (size_t)m32, D = (size_t)c->d_in, H = (size_t)c->cfg.hidden_layers;
    *h_m = (int64_t)m;
    // the kernels after the select run on the leaf-sorted sample order (k_sort_place)
    if (d_sample_ray) e = cudaMemcpyAsync(d_sample_ray, w->ss_ray, m * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && d_x) e = cudaMemcpyAsync(d_x, w->X, m * D * 2, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && d_z) e = cudaMemcpyAsync(d_z, w->Z, m * 8 * 4, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && d_dz) e = cudaMemcpyAsync(d_dz, w->dZ, m * 8 * 4, cudaMemcpyDeviceToDevice, s);
    for (size_t k = 0; e == cudaSuccess && d_act && k < H; ++k)       // [H][cap][64] -> [H][m][64]
        e = cudaMemcpyAsync(d_act + k * m * 64, w->A + k * (size_t)w->cap * 64, m * 64 * 2,
                            cudaMemcpyDeviceToDevice, s);
    for (size_t k = 0; e == cudaSuccess && d_delta && k < H; ++k)
        e = cudaMemcpyAsync(d_delta + k * m * 64, w->Dl + k * (size_t)w->cap * 64, m * 64 * 2,
                            cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "debug_train_activations");
    return NBVH_OK;
}
