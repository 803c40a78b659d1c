// nbvh_pathtrace.cu — NEXT-3 (BASELINE cfg 3): the pieces of a wavefront hybrid
// path tracer (PAPER §7: "a BLAS is classical or N-BVH; both query types yield the
// same type of intersection data"; a software CUDA wavefront path tracer).
//
//   k_mesh_intersect  classical BLAS: closest hit of each ray against the context's own
//                     triangle mesh (its SAH base BVH), written as an nbvh_hits record
//   k_pt_shade        one wavefront step: the closer of the neural and the classical hit,
//                     sky radiance for escaped rays, diffuse (cosine-weighted) continuation
//                     with throughput *= albedo, counter-based random numbers
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "nbvh_bvh.cuh"
#include "nbvh_capi_internal.h"

namespace nbvh {

struct MeshArgs {
    const BvhNode* nodes;
    int32_t bvh_rows;        // closest-hit stack rows (>= base-BVH depth)
    const float* tri_v;
    const float* tri_n;
    const float* tri_a;
    const int32_t* tri_id;
    const float4* rays;
    int64_t n;
    HitsDev out;
};

__global__ void __launch_bounds__(128) k_mesh_intersect(MeshArgs a) {
    extern __shared__ int stk_raw[];                      // stack column [bvh_rows][128]
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.n) return;
    const RayDev R = load_ray(a.rays, r);
    const BvhHit h = R.tmin <= R.tmax
                         ? bvh_closest(a.nodes, a.tri_v, a.tri_id, 0, R, R.tmin, R.tmax, stk_raw + threadIdx.x, 128, a.bvh_rows)
                         : BvhHit{false, 0.0, 0.0, 0.0, -1, -1};
    a.out.hit[r] = h.found ? 1 : 0;
    a.out.t[r] = h.found ? (float)h.t : __int_as_float(0x7f800000);
    float n[3] = {0.f, 0.f, 0.f};
    if (h.found) shading_normal(a.tri_n, h, n);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a.out.normal[3 * r + k] = n[k];
        a.out.albedo[3 * r + k] = h.found ? a.tri_a[3 * (int64_t)h.slot + k] : 0.f;
    }
    if (a.out.leaf) a.out.leaf[r] = h.found ? h.tri : -1;      // classical: the triangle id
    if (a.out.n_queries) a.out.n_queries[r] = 0;
}

// ---- counter-based random numbers: PCG output hash of (seed, ray, bounce, k)
__device__ __forceinline__ uint32_t pcg_hash(uint32_t v) {
    const uint32_t state = v * 747796405u + 2891336453u;
    const uint32_t word = ((state >> ((state >> 28u) + 4u)) ^ state) * 277803737u;
    return (word >> 22u) ^ word;
}
__device__ __forceinline__ float rng_uniform(uint64_t seed, int64_t ray, int bounce, int k) {
    uint32_t h = pcg_hash((uint32_t)seed ^ pcg_hash((uint32_t)(seed >> 32) + 0x9E3779B9u));
    h = pcg_hash(h ^ (uint32_t)ray);
    h = pcg_hash(h ^ (uint32_t)(ray >> 32) ^ ((uint32_t)bounce << 8) ^ (uint32_t)k);
    return (float)(h >> 8) * (1.0f / 16777216.0f);               // [0, 1)
}

struct ShadeArgs {
    const float4* rays;
    int64_t n;
    HitsDev a;           // neural hit record
    HitsDev b;           // classical hit record (b.hit == nullptr: absent)
    float* throughput;   // [n][3]
    float* radiance;     // [n][3]
    float4* next;        // [n][2] next rays (dead rays: tmin = 1 > tmax = 0)
    uint64_t seed;
    int32_t bounce;
    float sky_h[3], sky_z[3];
    float eps;           // origin offset along the normal
    int32_t* alive;      // count of continuing rays (device, accumulated)
};

__global__ void __launch_bounds__(256) k_pt_shade(ShadeArgs s) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool cont = false;
    if (r < s.n) {
        const float4 r0 = s.rays[2 * r], r1 = s.rays[2 * r + 1];
        float4 n0 = make_float4(0.f, 0.f, 0.f, 1.f), n1 = make_float4(0.f, 0.f, 1.f, 0.f);   // dead ray
        if (r0.w <= r1.w) {                                              // alive: tmin <= tmax
            const bool ha = s.a.hit[r] != 0, hb = s.b.hit ? s.b.hit[r] != 0 : false;
            const float ta = ha ? s.a.t[r] : __int_as_float(0x7f800000);
            const float tb = hb ? s.b.t[r] : __int_as_float(0x7f800000);
            const bool use_b = hb && tb < ta;
            float thr[3] = {s.throughput[3 * r], s.throughput[3 * r + 1], s.throughput[3 * r + 2]};
            const float d[3] = {r1.x, r1.y, r1.z};
            if (!ha && !hb) {
                // escaped: sky radiance, horizon-to-zenith gradient over the direction's elevation
                const float len = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
                const float e = fmaxf(0.f, d[1] / fmaxf(len, 1e-20f));
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    s.radiance[3 * r + k] += thr[k] * (s.sky_h[k] + (s.sky_z[k] - s.sky_h[k]) * e);
            } else {
                const HitsDev& H = use_b ? s.b : s.a;
                const float t = use_b ? tb : ta;
                float nrm[3] = {H.normal[3 * r], H.normal[3 * r + 1], H.normal[3 * r + 2]};
                if (nrm[0] * d[0] + nrm[1] * d[1] + nrm[2] * d[2] > 0.f)       // face the incoming ray
                    for (int k = 0; k < 3; ++k) nrm[k] = -nrm[k];
                const float nl = sqrtf(nrm[0] * nrm[0] + nrm[1] * nrm[1] + nrm[2] * nrm[2]);
                if (nl > 1e-12f) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) nrm[k] /= nl;
#pragma unroll
                    for (int k = 0; k < 3; ++k) thr[k] *= H.albedo[3 * r + k];   // diffuse BSDF: f cos / pdf = albedo
                    // cosine-weighted direction around nrm (orthonormal basis of Duff et al.)
                    const float u1 = rng_uniform(s.seed, r, s.bounce, 0), u2 = rng_uniform(s.seed, r, s.bounce, 1);
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
#pragma unroll
            for (int k = 0; k < 3; ++k) s.throughput[3 * r + k] = thr[k];
        }
        s.next[2 * r] = n0;
        s.next[2 * r + 1] = n1;
    }
    const unsigned m = __ballot_sync(0xffffffffu, cont);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(s.alive, __popc(m));
}

int32_t base_bvh_depth(const HostScene& sc) {
    if (sc.nodes.empty()) return 0;
    std::vector<std::pair<int32_t, int32_t>> todo{{0, 1}};
    int32_t depth = 0;
    while (!todo.empty()) {
        auto [i, dp] = todo.back();
        todo.pop_back();
        depth = std::max(depth, dp);
        if (sc.nodes[i].b >= 0) {
            todo.push_back({sc.nodes[i].a, dp + 1});
            todo.push_back({sc.nodes[i].b, dp + 1});
        }
    }
    return depth;
}

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_intersect_mesh(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, nbvh_hits out, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (!c->has_mesh) return fail(c, NBVH_ESTATE, "intersect_mesh: no mesh");
    if (n < 0 || (n > 0 && (!rays || !out.hit || !out.t || !out.normal || !out.albedo)))
        return fail(c, NBVH_EINVAL, "intersect_mesh: null pointer or negative n");
    if (n == 0) return NBVH_OK;
    if (c->base_depth < 0) c->base_depth = base_bvh_depth(c->sc);
    if (c->base_depth > kBvhStack) return fail(c, NBVH_EINVAL, "intersect_mesh: base BVH deeper than the stack");
    MeshArgs a{};
    a.nodes = c->dscene.nodes;
    a.bvh_rows = c->base_depth > 0 ? c->base_depth : 1;
    a.tri_v = c->dscene.tri_v;
    a.tri_n = c->dscene.tri_n;
    a.tri_a = c->dscene.tri_a;
    a.tri_id = c->dscene.tri_id;
    a.rays = reinterpret_cast<const float4*>(rays);
    a.n = n;
    a.out = HitsDev{out.hit, out.t, out.normal, out.albedo, out.leaf, out.n_queries};
    const int64_t blocks = (n + 127) / 128;
    k_mesh_intersect<<<(unsigned)blocks, 128, (size_t)a.bvh_rows * 128 * sizeof(int), (cudaStream_t)stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "intersect_mesh");
    return NBVH_OK;
}

extern "C" nbvh_status nbvh_pt_shade(nbvh_ctx* c, const nbvh_ray* rays, int64_t n, nbvh_hits hits_neural,
                                     nbvh_hits hits_classical, float* throughput, float* radiance, nbvh_ray* next,
                                     uint64_t seed, int32_t bounce, const float* sky, float eps, int32_t* alive,
                                     void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (n < 0 || (n > 0 && (!rays || !hits_neural.hit || !hits_neural.t || !hits_neural.normal ||
                            !hits_neural.albedo || !throughput || !radiance || !next || !sky || !alive)))
        return fail(c, NBVH_EINVAL, "pt_shade: null pointer or negative n");
    if (hits_classical.hit && (!hits_classical.t || !hits_classical.normal || !hits_classical.albedo))
        return fail(c, NBVH_EINVAL, "pt_shade: incomplete classical hit record");
    if (n == 0) return NBVH_OK;
    ShadeArgs s{};
    s.rays = reinterpret_cast<const float4*>(rays);
    s.n = n;
    s.a = HitsDev{hits_neural.hit, hits_neural.t, hits_neural.normal, hits_neural.albedo, nullptr, nullptr};
    s.b = HitsDev{hits_classical.hit, hits_classical.t, hits_classical.normal, hits_classical.albedo, nullptr, nullptr};
    s.throughput = throughput;
    s.radiance = radiance;
    s.next = reinterpret_cast<float4*>(next);
    s.seed = seed;
    s.bounce = bounce;
    for (int k = 0; k < 3; ++k) {
        s.sky_h[k] = sky[k];
        s.sky_z[k] = sky[3 + k];
    }
    s.eps = eps;
    s.alive = alive;
    k_pt_shade<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "pt_shade");
    return NBVH_OK;
}
