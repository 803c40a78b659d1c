// nbvh_tlas.cu — NEXT-3 (BASELINE cfg 3): the two-level hierarchy of the hybrid
// path tracer (PAPER §7: "a TLAS holds several BLAS; a BLAS is classical or N-BVH, and
// both query types yield the same type of intersection data"; wavefront design).
//
//   nbvh_tlas_build      host: a binary BVH over the world-space boxes of the instances
//                        (median split on the longest axis), uploaded to the device
//   k_tlas_dispatch      per alive ray: traverse the TLAS, and for every instance whose box
//                        the ray crosses append the ray, transformed into the instance's
//                        object space (o' = A o + b, d' = A d: the same t parameterises both),
//                        to that instance's BLAS ray list
//   k_tlas_merge_*       closest hit over all (instance, BLAS) answers of a ray: atomicMin of
//                        a 64-bit key (t bits, list, entry), then the winner's record with the
//                        normal brought back to world space (A^T n, normalised)
//   k_pt_shade_compact   one wavefront step over the compacted alive paths: sky radiance for
//                        escaped paths, diffuse continuation for hits, appended to the next
//                        bounce's compacted path list (ray, pixel, throughput)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "nbvh_capi_internal.h"
#include "nbvh_device.cuh"

namespace nbvh {

constexpr int kMaxBlas = NBVH_MAX_BLAS;

struct TlasNode {              // 32 bytes: box + children (child < 0: instance -1 - c)
    float lo[3];
    int32_t l;
    float hi[3];
    int32_t r;
};

struct TlasDev {
    const TlasNode* nodes;
    const nbvh_instance* inst;
    int32_t n_nodes, n_inst;
};

// ---- counter-based random numbers (the same PCG hash as k_pt_shade)
__device__ __forceinline__ uint32_t pcg32(uint32_t v) {
    const uint32_t state = v * 747796405u + 2891336453u;
    const uint32_t word = ((state >> ((state >> 28u) + 4u)) ^ state) * 277803737u;
    return (word >> 22u) ^ word;
}
__device__ __forceinline__ float pt_uniform(uint64_t seed, int64_t key, int bounce, int k) {
    uint32_t h = pcg32((uint32_t)seed ^ pcg32((uint32_t)(seed >> 32) + 0x9E3779B9u));
    h = pcg32(h ^ (uint32_t)key);
    h = pcg32(h ^ (uint32_t)(key >> 32) ^ ((uint32_t)bounce << 8) ^ (uint32_t)k);
    return (float)(h >> 8) * (1.0f / 16777216.0f);
}

struct DispatchArgs {
    TlasDev t;
    const float4* rays;            // [m] world rays (compacted)
    int64_t m;
    float4* out_rays;              // [n_blas][cap] object-space rays
    int32_t* out_src;              // [n_blas][cap] source ray (index into rays)
    int32_t* out_inst;             // [n_blas][cap] instance
    int32_t* counts;               // [n_blas]
    int64_t cap;
    int32_t* overflow;             // set if a list overflowed
};

// Packet traversal: the warp walks the (small) TLAS together -- a node is entered if any lane
// crosses its box -- so the node loads are broadcasts, the stack is warp-uniform (shared
// memory) and each leaf costs ONE atomic per warp for all the lanes that append to its BLAS
// list (a per-lane atomic on the few list counters serialises the whole frame).
__global__ void __launch_bounds__(128) k_tlas_dispatch(DispatchArgs a) {
    __shared__ int stack_sm[4][32];
    const int lane = threadIdx.x & 31;
    int* stack = stack_sm[threadIdx.x >> 5];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    RayDev R{};
    bool valid = i < a.m;
    if (valid) {
        R = load_ray(a.rays, i);
        valid = R.tmin <= R.tmax;
    }
    if (!__any_sync(0xffffffffu, valid)) return;
    int sp = 0, node = 0;
    while (true) {
        const TlasNode nd = a.t.nodes[node];
        float te, tx;
        const bool hit = valid && slab(R, nd.lo, nd.hi, te, tx);
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        if (hm && nd.l < 0) {                                     // leaf: one instance
            const int ins = -1 - nd.l;
            const nbvh_instance I = a.t.inst[ins];
            const int b = I.blas;
            int base = 0;
            if (lane == 0) base = atomicAdd(a.counts + b, __popc(hm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (hit) {
                const int slot = base + __popc(hm & ((1u << lane) - 1u));
                if (slot < a.cap) {
                    const float* A = I.world_to_object;
                    float o[3], d[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        o[k] = A[4 * k] * R.o[0] + A[4 * k + 1] * R.o[1] + A[4 * k + 2] * R.o[2] + A[4 * k + 3];
                        d[k] = A[4 * k] * R.d[0] + A[4 * k + 1] * R.d[1] + A[4 * k + 2] * R.d[2];
                    }
                    const int64_t e = (int64_t)b * a.cap + slot;
                    a.out_rays[2 * e] = make_float4(o[0], o[1], o[2], R.tmin);
                    a.out_rays[2 * e + 1] = make_float4(d[0], d[1], d[2], R.tmax);
                    a.out_src[e] = (int32_t)i;
                    a.out_inst[e] = ins;
                } else {
                    atomicOr(a.overflow, 1);
                }
            }
        } else if (hm) {
            if (sp < 32) {
                if (lane == 0) stack[sp] = nd.r;
                ++sp;
            } else if (lane == 0) {
                atomicOr(a.overflow, 2);
            }
            __syncwarp();
            node = nd.l;
            continue;
        }
        if (sp == 0) break;
        --sp;
        __syncwarp();
        node = stack[sp];
    }
}

struct MergeArgs {
    int64_t m;
    unsigned long long* key;       // [m]
    const int32_t* counts;         // [n_blas]
    int64_t cap;
    const int32_t* src;            // [n_blas][cap]
    const int32_t* inst;           // [n_blas][cap]
    HitsDev lists[kMaxBlas];       // per BLAS: its answers, entry j = ray list entry j
    int32_t n_blas;
    const nbvh_instance* instances;
    HitsDev out;                   // [m] world hits; leaf = instance (or -1)
};

__global__ void k_tlas_merge_init(MergeArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.m) a.key[i] = ~0ull;
}

// key = t bits (t >= 0: unsigned order = float order) | list << 24 | entry -> the nearest
// hit, ties by list then entry (deterministic)
__global__ void k_tlas_merge_min(MergeArgs a, int b) {
    const int64_t n = min((int64_t)a.counts[b], a.cap);
    const HitsDev& H = a.lists[b];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (!H.hit[j]) continue;
        const float t = fmaxf(H.t[j], 0.f);
        const unsigned long long k =
            ((unsigned long long)__float_as_uint(t) << 32) | ((unsigned long long)b << 24) | (unsigned long long)j;
        atomicMin(a.key + a.src[(int64_t)b * a.cap + j], k);
    }
}

__global__ void k_tlas_merge_out(MergeArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.m) return;
    const unsigned long long k = a.key[i];
    if (k == ~0ull) {
        a.out.hit[i] = 0;
        a.out.t[i] = __int_as_float(0x7f800000);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            a.out.normal[3 * i + c] = 0.f;
            a.out.albedo[3 * i + c] = 0.f;
        }
        if (a.out.leaf) a.out.leaf[i] = -1;
        return;
    }
    const int b = (int)((k >> 24) & 0xff);
    const int64_t j = (int64_t)(k & 0xffffff);
    const HitsDev& H = a.lists[b];
    const int ins = a.inst[(int64_t)b * a.cap + j];
    const float* A = a.instances[ins].world_to_object;
    float n[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)                                   // A^T n_object (inverse transpose)
        n[c] = A[c] * H.normal[3 * j] + A[4 + c] * H.normal[3 * j + 1] + A[8 + c] * H.normal[3 * j + 2];
    const float nl = fmaxf(sqrtf(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]), 1e-20f);
    a.out.hit[i] = 1;
    a.out.t[i] = H.t[j];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        a.out.normal[3 * i + c] = n[c] / nl;
        a.out.albedo[3 * i + c] = H.albedo[3 * j + c];
    }
    if (a.out.leaf) a.out.leaf[i] = ins;
}

struct ShadeCArgs {
    const float4* rays;            // [m] world rays of the alive paths
    int64_t m;
    HitsDev hits;                  // [m]
    const int32_t* pixel;          // [m]
    const float* thr;              // [m][3]
    float* radiance;               // [n_px][3] (accumulated)
    float4* next_rays;             // [m] compacted continuing paths
    int32_t* next_pixel;
    float* next_thr;
    int32_t* next_count;
    uint64_t seed;
    int32_t bounce;
    float sky_h[3], sky_z[3];
    float eps;
};

__global__ void __launch_bounds__(256) k_pt_shade_compact(ShadeCArgs s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool cont = false;
    float4 n0 = make_float4(0.f, 0.f, 0.f, 0.f), n1 = n0;
    float th[3] = {0.f, 0.f, 0.f};
    int px = 0;
    if (i < s.m) {
        const float4 r0 = s.rays[2 * i], r1 = s.rays[2 * i + 1];
        px = s.pixel[i];
#pragma unroll
        for (int k = 0; k < 3; ++k) th[k] = s.thr[3 * i + k];
        const float d[3] = {r1.x, r1.y, r1.z};
        if (!s.hits.hit[i]) {
            // escaped: sky radiance, horizon-to-zenith gradient over the direction's elevation
            const float len = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            const float e = fmaxf(0.f, d[1] / fmaxf(len, 1e-20f));
#pragma unroll
            for (int k = 0; k < 3; ++k)
                atomicAdd(s.radiance + 3 * (int64_t)px + k, th[k] * (s.sky_h[k] + (s.sky_z[k] - s.sky_h[k]) * e));
        } else {
            const float t = s.hits.t[i];
            float nrm[3] = {s.hits.normal[3 * i], s.hits.normal[3 * i + 1], s.hits.normal[3 * i + 2]};
            if (nrm[0] * d[0] + nrm[1] * d[1] + nrm[2] * d[2] > 0.f)   // face the incoming ray
                for (int k = 0; k < 3; ++k) nrm[k] = -nrm[k];
            const float nl = sqrtf(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
            if (nl > 1e-12f) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    nrm[k] /= nl;
                    th[k] *= s.hits.albedo[3 * i + k];                    // diffuse: f cos / pdf = albedo
                }
                // cosine-weighted direction around nrm (orthonormal basis of Duff et al.); the
                // random stream is keyed by the pixel, so compaction does not change it
                const float u1 = pt_uniform(s.seed, px, s.bounce, 0), u2 = pt_uniform(s.seed, px, s.bounce, 1);
                const float rr = sqrtf(u1), phi = 6.283185307f * u2;
                const float lx = rr * cosf(phi), ly = rr * sinf(phi), lz = sqrtf(fmaxf(0.f, 1.f - u1));
                const float sg = copysignf(1.f, nrm[2]);
                const float aa = -1.f / (sg + nrm[2]), bb = nrm[0] * nrm[1] * aa;
                const float tx[3] = {1.f + sg * nrm[0] * nrm[0] * aa, sg * bb, -sg * nrm[0]};
                const float ty[3] = {bb, sg + nrm[1] * nrm[1] * aa, -nrm[1]};
                float nd[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) nd[k] = lx * tx[k] + ly * ty[k] + lz * nrm[k];
                const float p[3] = {r0.x + t * d[0], r0.y + t * d[1], r0.z + t * d[2]};
                n0 = make_float4(p[0] + s.eps * nrm[0], p[1] + s.eps * nrm[1], p[2] + s.eps * nrm[2], 0.f);
                n1 = make_float4(nd[0], nd[1], nd[2], __int_as_float(0x7f800000));
                cont = true;
            }
        }
    }
    // warp-aggregated append of the continuing paths
    const unsigned m = __ballot_sync(0xffffffffu, cont);
    int base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(s.next_count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (cont) {
        const int slot = base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
        s.next_rays[2 * (int64_t)slot] = n0;
        s.next_rays[2 * (int64_t)slot + 1] = n1;
        s.next_pixel[slot] = px;
#pragma unroll
        for (int k = 0; k < 3; ++k) s.next_thr[3 * (int64_t)slot + k] = th[k];
    }
}

}  // namespace nbvh

using namespace nbvh;

struct nbvh_tlas {
    TlasNode* d_nodes = nullptr;
    nbvh_instance* d_inst = nullptr;
    int32_t n_nodes = 0, n_inst = 0, n_blas = 0;
    int32_t* d_overflow = nullptr;
    unsigned long long* d_key = nullptr;
    int64_t key_cap = 0;
};

namespace {
// Binary BVH over instance boxes: median split of the box centres on the longest axis.
int32_t build_tlas_node(std::vector<TlasNode>& out, const nbvh_instance* inst, std::vector<int32_t>& ids, int lo,
                        int hi) {
    const int32_t me = (int32_t)out.size();
    out.push_back(TlasNode{});
    float blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = lo; i < hi; ++i)
        for (int k = 0; k < 3; ++k) {
            blo[k] = std::min(blo[k], inst[ids[i]].lo[k]);
            bhi[k] = std::max(bhi[k], inst[ids[i]].hi[k]);
        }
    TlasNode nd{};
    for (int k = 0; k < 3; ++k) {
        nd.lo[k] = blo[k];
        nd.hi[k] = bhi[k];
    }
    if (hi - lo == 1) {
        nd.l = -1 - ids[lo];
        nd.r = -1 - ids[lo];
    } else {
        int ax = 0;
        for (int k = 1; k < 3; ++k)
            if (bhi[k] - blo[k] > bhi[ax] - blo[ax]) ax = k;
        const int mid = (lo + hi) / 2;
        std::nth_element(ids.begin() + lo, ids.begin() + mid, ids.begin() + hi, [&](int32_t a, int32_t b) {
            const float ca = inst[a].lo[ax] + inst[a].hi[ax], cb = inst[b].lo[ax] + inst[b].hi[ax];
            return ca < cb || (ca == cb && a < b);
        });
        nd.l = build_tlas_node(out, inst, ids, lo, mid);
        nd.r = build_tlas_node(out, inst, ids, mid, hi);
    }
    out[me] = nd;
    return me;
}
}  // namespace

extern "C" nbvh_status nbvh_tlas_build(nbvh_ctx* c, const nbvh_instance* h_inst, int32_t n_inst, nbvh_tlas** out) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!h_inst || !out || n_inst < 1 || n_inst > 4096) return fail(c, NBVH_EINVAL, "tlas_build: bad arguments");
    int32_t n_blas = 0;
    for (int32_t i = 0; i < n_inst; ++i) {
        if (h_inst[i].blas < 0 || h_inst[i].blas >= kMaxBlas) return fail(c, NBVH_ERANGE, "tlas_build: blas index");
        for (int k = 0; k < 3; ++k)
            if (!(h_inst[i].hi[k] >= h_inst[i].lo[k])) return fail(c, NBVH_EINVAL, "tlas_build: instance box");
        n_blas = std::max(n_blas, h_inst[i].blas + 1);
    }
    std::vector<TlasNode> nodes;
    std::vector<int32_t> ids(n_inst);
    std::iota(ids.begin(), ids.end(), 0);
    build_tlas_node(nodes, h_inst, ids, 0, n_inst);
    nbvh_tlas* t = new nbvh_tlas();
    cudaError_t e = cudaMalloc((void**)&t->d_nodes, nodes.size() * sizeof(TlasNode));
    if (e == cudaSuccess) e = cudaMalloc((void**)&t->d_inst, (size_t)n_inst * sizeof(nbvh_instance));
    if (e == cudaSuccess) e = cudaMalloc((void**)&t->d_overflow, sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemcpy(t->d_nodes, nodes.data(), nodes.size() * sizeof(TlasNode), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(t->d_inst, h_inst, (size_t)n_inst * sizeof(nbvh_instance), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(t->d_overflow, 0, sizeof(int32_t));
    if (e != cudaSuccess) {
        cudaFree(t->d_nodes);
        cudaFree(t->d_inst);
        cudaFree(t->d_overflow);
        delete t;
        return cuda_fail(c, e, "tlas_build");
    }
    t->n_nodes = (int32_t)nodes.size();
    t->n_inst = n_inst;
    t->n_blas = n_blas;
    *out = t;
    return NBVH_OK;
}

extern "C" void nbvh_tlas_destroy(nbvh_tlas* t) {
    if (!t) return;
    cudaFree(t->d_nodes);
    cudaFree(t->d_inst);
    cudaFree(t->d_overflow);
    cudaFree(t->d_key);
    delete t;
}

extern "C" nbvh_status nbvh_tlas_dispatch(nbvh_ctx* c, nbvh_tlas* t, const nbvh_ray* d_rays, int64_t m,
                                          nbvh_ray* d_out_rays, int32_t* d_out_src, int32_t* d_out_inst,
                                          int32_t* d_counts, int64_t cap, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!t || m < 0 || cap < 0 || (m > 0 && (!d_rays || !d_out_rays || !d_out_src || !d_out_inst || !d_counts)))
        return fail(c, NBVH_EINVAL, "tlas_dispatch: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * (size_t)t->n_blas, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "tlas_dispatch");
    if (m == 0) return NBVH_OK;
    DispatchArgs a{};
    a.t = TlasDev{t->d_nodes, t->d_inst, t->n_nodes, t->n_inst};
    a.rays = reinterpret_cast<const float4*>(d_rays);
    a.m = m;
    a.out_rays = reinterpret_cast<float4*>(d_out_rays);
    a.out_src = d_out_src;
    a.out_inst = d_out_inst;
    a.counts = d_counts;
    a.cap = cap;
    a.overflow = t->d_overflow;
    k_tlas_dispatch<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "tlas_dispatch");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_tlas_merge(nbvh_ctx* c, nbvh_tlas* t, int64_t m, const int32_t* d_counts, int64_t cap,
                                       const int32_t* d_src, const int32_t* d_inst, const nbvh_hits* h_lists,
                                       nbvh_hits d_out, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!t || m < 0 || (m > 0 && (!d_counts || !d_src || !d_inst || !h_lists || !d_out.hit || !d_out.t ||
                                  !d_out.normal || !d_out.albedo)))
        return fail(c, NBVH_EINVAL, "tlas_merge: bad arguments");
    if (cap >= (1 << 24)) return fail(c, NBVH_EINVAL, "tlas_merge: list capacity >= 2^24");
    if (m == 0) return NBVH_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (m > t->key_cap) {
        cudaFree(t->d_key);
        t->d_key = nullptr;
        cudaError_t e = cudaMalloc((void**)&t->d_key, (size_t)m * sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_fail(c, e, "tlas_merge");
        t->key_cap = m;
    }
    MergeArgs a{};
    a.m = m;
    a.key = t->d_key;
    a.counts = d_counts;
    a.cap = cap;
    a.src = d_src;
    a.inst = d_inst;
    a.n_blas = t->n_blas;
    for (int b = 0; b < t->n_blas; ++b) {
        const nbvh_hits& h = h_lists[b];
        if (!h.hit || !h.t || !h.normal || !h.albedo) return fail(c, NBVH_EINVAL, "tlas_merge: BLAS hit record");
        a.lists[b] = HitsDev{h.hit, h.t, h.normal, h.albedo, h.leaf, h.n_queries};
    }
    a.instances = t->d_inst;
    a.out = HitsDev{d_out.hit, d_out.t, d_out.normal, d_out.albedo, d_out.leaf, d_out.n_queries};
    const unsigned g = (unsigned)((m + 255) / 256);
    k_tlas_merge_init<<<g, 256, 0, s>>>(a);
    for (int b = 0; b < t->n_blas; ++b) k_tlas_merge_min<<<(unsigned)std::min<int64_t>(4 * 148, (cap + 255) / 256 + 1), 256, 0, s>>>(a, b);
    k_tlas_merge_out<<<g, 256, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "tlas_merge");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_tlas_overflow(nbvh_ctx* c, nbvh_tlas* t, int32_t* h_flag) {
    if (!c || !t || !h_flag) return NBVH_EINVAL;
    cudaError_t e = cudaMemcpy(h_flag, t->d_overflow, sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "tlas_overflow");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_pt_shade_compact(nbvh_ctx* c, const nbvh_ray* d_rays, int64_t m, nbvh_hits d_hits,
                                             const int32_t* d_pixel, const float* d_thr, float* d_radiance,
                                             nbvh_ray* d_next_rays, int32_t* d_next_pixel, float* d_next_thr,
                                             int32_t* d_next_count, uint64_t seed, int32_t bounce, const float* sky,
                                             float eps, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (m < 0 || !sky || (m > 0 && (!d_rays || !d_hits.hit || !d_hits.t || !d_hits.normal || !d_hits.albedo ||
                                    !d_pixel || !d_thr || !d_radiance || !d_next_rays || !d_next_pixel ||
                                    !d_next_thr || !d_next_count)))
        return fail(c, NBVH_EINVAL, "pt_shade_compact: bad arguments");
    if (m == 0) return NBVH_OK;
    ShadeCArgs s{};
    s.rays = reinterpret_cast<const float4*>(d_rays);
    s.m = m;
    s.hits = HitsDev{d_hits.hit, d_hits.t, d_hits.normal, d_hits.albedo, nullptr, nullptr};
    s.pixel = d_pixel;
    s.thr = d_thr;
    s.radiance = d_radiance;
    s.next_rays = reinterpret_cast<float4*>(d_next_rays);
    s.next_pixel = d_next_pixel;
    s.next_thr = d_next_thr;
    s.next_count = d_next_count;
    s.seed = seed;
    s.bounce = bounce;
    for (int k = 0; k < 3; ++k) {
        s.sky_h[k] = sky[k];
        s.sky_z[k] = sky[3 + k];
    }
    s.eps = eps;
    k_pt_shade_compact<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "pt_shade_compact");
    return NBVH_OK;
}
