// nbvh_raygen.cu — T0 of the training step ("rays ... randomly generated",
// P:193): the training rays and the method's random draws, on the device, from the
// counter-based generator Philox-4x32-10 (Salmon et al., SC'11; the oracle implements the same
// generator independently).  Ray i of step s (global index i, so data-parallel ranks that
// generate their shards reproduce the single-process batch) uses counter (i, draw, s_lo, s_hi)
// and key (seed_lo, seed_hi):
//   draw 0: origin x, y, z ~ U[box] and the acceptance draw u (T1, C18)
//   draw 1: direction: z = 1 - 2 U, phi = 2 pi U, d = (sqrt(1 - z^2) cos phi, .. sin phi, z)
//   draw 2: stratification jitter xi[0..n_points) (C8, n_points <= 4)
// U = (x >> 8) * 2^-24 in [0, 1); tmin = 0, tmax = +inf.
#include <cuda_runtime.h>

#include "nbvh_capi_internal.h"

namespace nbvh {

struct Philox4 {
    uint32_t v[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                                 uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return Philox4{{c0, c1, c2, c3}};
}

__device__ __forceinline__ float u01(uint32_t x) { return __uint2float_rn(x >> 8) * 5.9604644775390625e-8f; }

struct RayGenArgs {
    uint32_t k0, k1, s0, s1;
    int64_t i0, n;
    float lo[3], hi[3];
    int32_t n_points;
    float4* rays;
    float* u;
    float* xi;
};

__global__ void __launch_bounds__(256) k_gen_train_rays(RayGenArgs a) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= a.n) return;
    const uint32_t i = (uint32_t)(a.i0 + j);
    const Philox4 p0 = philox4x32_10(i, 0u, a.s0, a.s1, a.k0, a.k1);
    const Philox4 p1 = philox4x32_10(i, 1u, a.s0, a.s1, a.k0, a.k1);
    float o[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) o[k] = __fadd_rn(a.lo[k], __fmul_rn(__fsub_rn(a.hi[k], a.lo[k]), u01(p0.v[k])));
    const float z = __fsub_rn(1.0f, __fmul_rn(2.0f, u01(p1.v[0])));
    const float rr = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, __fmul_rn(z, z))));
    float sp, cp;
    sincosf(__fmul_rn(6.28318530717958647692f, u01(p1.v[1])), &sp, &cp);
    a.rays[2 * j] = make_float4(o[0], o[1], o[2], 0.0f);
    a.rays[2 * j + 1] = make_float4(__fmul_rn(rr, cp), __fmul_rn(rr, sp), z, __int_as_float(0x7f800000));
    a.u[j] = u01(p0.v[3]);
    if (a.n_points > 0) {
        const Philox4 p2 = philox4x32_10(i, 2u, a.s0, a.s1, a.k0, a.k1);
        for (int k = 0; k < a.n_points; ++k) a.xi[j * a.n_points + k] = u01(p2.v[k]);
    }
}

}  // namespace nbvh

using namespace nbvh;

extern "C" nbvh_status nbvh_gen_train_rays(nbvh_ctx* c, uint64_t seed, uint64_t step, int64_t i0, int64_t n,
                                           const float* box, nbvh_ray* d_rays, float* d_u, float* d_xi, void* stream) {
    nbvh_status st = check_device(c);
    if (st) return st;
    if (n < 0 || i0 < 0 || i0 + n > (int64_t)UINT32_MAX || (n > 0 && (!d_rays || !d_u || !d_xi)))
        return fail(c, NBVH_EINVAL, "gen_train_rays: bad args");
    if (c->cfg.n_points > 4) return fail(c, NBVH_EINVAL, "gen_train_rays: n_points > 4");
    if (n == 0) return NBVH_OK;
    RayGenArgs a{};
    a.k0 = (uint32_t)seed;
    a.k1 = (uint32_t)(seed >> 32);
    a.s0 = (uint32_t)step;
    a.s1 = (uint32_t)(step >> 32);
    a.i0 = i0;
    a.n = n;
    if (box) {
        for (int k = 0; k < 3; ++k) {
            a.lo[k] = box[k];
            a.hi[k] = box[3 + k];
            if (!(a.hi[k] >= a.lo[k])) return fail(c, NBVH_EINVAL, "gen_train_rays: box");
        }
    } else {
        // C16 ("the 50%-inflated scene bounding box"): the scene's root box (min/max
        // over all triangle vertices), each axis extent x1.5 about its centre.
        if (!c->has_mesh || c->sc.nodes.empty()) return fail(c, NBVH_ESTATE, "gen_train_rays: no mesh");
        const nbvh::BvhNode& r = c->sc.nodes[0];
        for (int k = 0; k < 3; ++k) {
            const float mid = (r.lo[k] + r.hi[k]) * 0.5f;
            const float half = (r.hi[k] - r.lo[k]) * 0.75f;
            a.lo[k] = mid - half;
            a.hi[k] = mid + half;
        }
    }
    a.n_points = c->cfg.n_points;
    a.rays = reinterpret_cast<float4*>(d_rays);
    a.u = d_u;
    a.xi = d_xi;
    k_gen_train_rays<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "gen_train_rays");
    return NBVH_OK;
}
