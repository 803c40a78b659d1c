// nbvh_bvh.cuh — classical closest-hit traversal of the base BVH (the BVH is the
// "probing machine" for ground truth; the classical BLAS of the hybrid renderer).
// Double-precision Moller-Trumbore with the oracle's operation order (no FMA), conservative
// fp32 node boxes, nearer child first, pruning beyond the best hit.
#pragma once

#include "nbvh_device.cuh"
#include "nbvh_internal.h"

namespace nbvh {

constexpr int kBvhStack = 64;          // traversal stack rows (base-BVH depth checked at set_mesh)

// Moller-Trumbore in double with the oracle's operation order (no FMA), so the hit
// decisions and t are bit-identical to the double-precision ground truth.
__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
    c[0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    c[1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    c[2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
}

__device__ __forceinline__ bool tri_hit(const double* o, const double* d, const float* tv, double t0, double t1,
                                        double& t, double& b1, double& b2) {
    double v0[3], e1[3], e2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        v0[k] = tv[k];
        e1[k] = __dsub_rn((double)tv[3 + k], v0[k]);
        e2[k] = __dsub_rn((double)tv[6 + k], v0[k]);
    }
    double p[3];
    cross3(d, e2, p);
    const double det = dot3(e1, p);
    if (fabs(det) < 1e-20) return false;
    const double inv = __ddiv_rn(1.0, det);
    double s[3] = {__dsub_rn(o[0], v0[0]), __dsub_rn(o[1], v0[1]), __dsub_rn(o[2], v0[2])};
    const double uu = __dmul_rn(dot3(s, p), inv);
    if (uu < 0.0 || uu > 1.0) return false;
    double q[3];
    cross3(s, e1, q);
    const double vv = __dmul_rn(dot3(d, q), inv);
    if (vv < 0.0 || __dadd_rn(uu, vv) > 1.0) return false;
    const double tt = __dmul_rn(dot3(e2, q), inv);
    if (tt < t0 || tt > t1) return false;
    t = tt;
    b1 = uu;
    b2 = vv;
    return true;
}


struct BvhHit {
    bool found;
    double t, b1, b2;
    int tri, slot;
};

// Conservative fp32 box of a base-BVH node: a relative slack, so the fp32 slab test never
// rejects a box that the double-precision triangle test could hit.
__device__ __forceinline__ bool bvh_box(const BvhNode& nd, const RayDev& R, float& te, float& tx) {
    float lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float e = 1e-5f * (fabsf(nd.lo[k]) + fabsf(nd.hi[k]) + 1e-3f);
        lo[k] = nd.lo[k] - e;
        hi[k] = nd.hi[k] + e;
    }
    return slab(R, lo, hi, te, tx);
}

// Closest hit below node `root` within [t0, t1]; ties by lowest original triangle id (C32).
// stack_col: this thread's column of a shared-memory stack [stack_rows][stride]; the host
// sizes stack_rows >= base-BVH depth, which the farther-child-only stack never exceeds.
// Both children are tested where their parent is visited (their boxes are loaded there
// anyway, for the near-first order); the nearer one is visited next from registers and only
// the farther one is pushed, then re-tested when popped because the best hit may have
// tightened t_cut meanwhile.  Nodes are visited in the same order and under the same test
// as a push-both / test-on-pop traversal, so the result is the same.
__device__ __forceinline__ BvhHit bvh_closest(const BvhNode* nodes, const float* tri_v, const int32_t* tri_id,
                                              int root, const RayDev& R, float t0, float t1, int* stack_col,
                                              int stride, int stack_rows) {
    const double o[3] = {R.o[0], R.o[1], R.o[2]}, d[3] = {R.d[0], R.d[1], R.d[2]};
    BvhHit h{false, 0.0, 0.0, 0.0, -1, -1};
    float t_cut = t1 * 1.00001f + 1e-6f;        // conservative upper bound: segment end, then best hit
    const float t_lo = t0 * 0.99999f - 1e-6f;
    // a node entering beyond the best hit so far holds no closer (or tying) hit: the
    // conservative boxes and the relative slack keep this exact w.r.t. the double test
    auto admit = [&](const BvhNode& nd) {
        float te, tx;
        return bvh_box(nd, R, te, tx) && !(te > t_cut) && !(tx < t_lo);
    };
    int sp = 0;
    BvhNode nd = nodes[root];
    bool have = admit(nd);
    while (have) {
        if (nd.b < 0) {
            for (int j = nd.a; j < nd.a - nd.b; ++j) {
                double th, b1, b2;
                if (tri_hit(o, d, tri_v + 9 * (int64_t)j, (double)t0, (double)t1, th, b1, b2)) {
                    const int id = tri_id[j];
                    if (!h.found || th < h.t || (th == h.t && id < h.tri)) {
                        h = BvhHit{true, th, b1, b2, id, j};
                        t_cut = fminf(t_cut, (float)th * 1.00001f + 1e-6f);
                    }
                }
            }
        } else {
            const BvhNode ca = nodes[nd.a];
            const BvhNode cb = nodes[nd.b];
            const bool ha = admit(ca), hb = admit(cb);
            if (ha && hb) {
                // nearer child first (box centre along the ray) so the best hit tightens t_cut early
                float da = 0.f, db = 0.f;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    da = fmaf(ca.lo[k] + ca.hi[k], R.d[k], da);
                    db = fmaf(cb.lo[k] + cb.hi[k], R.d[k], db);
                }
                const bool a_first = da <= db;
                NBVH_DCHECK(sp < stack_rows);
                if (sp < stack_rows) stack_col[(sp++) * stride] = a_first ? nd.b : nd.a;
                nd = a_first ? ca : cb;
                continue;
            }
            if (ha || hb) {
                nd = ha ? ca : cb;
                continue;
            }
        }
        have = false;
        while (sp > 0 && !have) {
            nd = nodes[stack_col[(--sp) * stride]];
            have = admit(nd);
        }
    }
    return h;
}

// barycentric-interpolated vertex normal of the hit, normalised (C22)
__device__ __forceinline__ void shading_normal(const float* tri_n, const BvhHit& h, float n_out[3]) {
    const float* tn = tri_n + 9 * (int64_t)h.slot;
    double n[3];
    for (int k = 0; k < 3; ++k)
        n[k] = (1.0 - h.b1 - h.b2) * (double)tn[k] + h.b1 * (double)tn[3 + k] + h.b2 * (double)tn[6 + k];
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    for (int k = 0; k < 3; ++k) n_out[k] = nn > 0 ? (float)(n[k] / nn) : 0.f;
}

}  // namespace nbvh
