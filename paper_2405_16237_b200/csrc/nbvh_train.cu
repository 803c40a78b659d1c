// nbvh_train.cu — scene/cut upload and the companion training step (T0-T9).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "nbvh_capi_internal.h"

namespace nbvh {

struct TrainWork {
    int64_t cap = 0;
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
    return NBVH_OK;
}

void free_scene_device(nbvh_ctx* c) {
    DeviceScene& d = c->dscene;
    for (void* p : {(void*)d.nodes, (void*)d.tri_v, (void*)d.tri_n, (void*)d.tri_a, (void*)d.tri_id})
        if (p) cudaFree(p);
    d = DeviceScene{};
}

void free_train_device(nbvh_ctx* c) {
    delete c->train;
    c->train = nullptr;
}

nbvh_status reserve_train(nbvh_ctx* c, int64_t max_rays) {
    (void)c;
    (void)max_rays;
    return NBVH_OK;
}

void reset_adam(nbvh_ctx* c) { (void)c; }

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_set_leaf_rank(nbvh_ctx* c, int32_t lod, const float* h_rank) {
    if (!c || !h_rank) return NBVH_EINVAL;
    if (lod < 0 || lod >= kMaxLod) return fail(c, NBVH_ERANGE, "set_leaf_rank: lod");
    if (!c->has_cut[lod]) return fail(c, NBVH_ESTATE, "set_leaf_rank: no cut");
    HostCut& hc = c->cuts[lod];
    std::memcpy(hc.rank.data(), h_rank, sizeof(float) * hc.n_leaves);
    if (c->device >= 0) {
        nbvh_status st = check_device(c);
        if (st) return st;
        cudaError_t e = cudaMemcpy(c->dcut[lod].rank, h_rank, sizeof(float) * hc.n_leaves, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_fail(c, e, "set_leaf_rank");
    }
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_train_backward(nbvh_ctx* c, const nbvh_ray*, int64_t, const float*, const float*, int32_t,
                                           void*) {
    return fail(c, NBVH_ESTATE, "train_backward: not implemented yet");
}
extern "C" nbvh_status nbvh_grad_buffer(nbvh_ctx* c, float**, int64_t*) {
    return fail(c, NBVH_ESTATE, "grad_buffer: not implemented yet");
}
extern "C" nbvh_status nbvh_apply_update(nbvh_ctx* c, float, void*) {
    return fail(c, NBVH_ESTATE, "apply_update: not implemented yet");
}
extern "C" nbvh_status nbvh_train_step(nbvh_ctx* c, const nbvh_ray*, int64_t, const float*, const float*, int32_t,
                                       float, void*) {
    return fail(c, NBVH_ESTATE, "train_step: not implemented yet");
}
extern "C" nbvh_status nbvh_get_train_stats(nbvh_ctx* c, nbvh_train_stats* out) {
    if (!c || !out) return NBVH_EINVAL;
    *out = c->tstats;
    return NBVH_OK;
}
extern "C" nbvh_status nbvh_debug_train_samples(nbvh_ctx* c, float*, uint8_t*, int32_t*, float*, void*) {
    return fail(c, NBVH_ESTATE, "debug_train_samples: not implemented yet");
}
