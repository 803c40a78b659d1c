// nbvh_internal.h — product-internal types shared by the host core (nbvh_host.cpp),
// the C ABI (nbvh_capi.cu) and the kernels (nbvh_kernels.cu, nbvh_train.cu).
// Not part of the public ABI (include/nbvh.h).  Shares nothing with oracle/.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace nbvh {

constexpr int kMaxLevels = 32;
constexpr int kMaxLod = 8;
constexpr int kListK = 16;          // register capacity of the per-ray ordered leaf list (C6)
constexpr int kWidth = 64;          // hidden width
constexpr int kOut = 8;             // [vis, t, n.xyz, albedo.rgb] (C12)
constexpr int kMaxHidden = 4;       // P:275 uses 4 hidden layers
constexpr int kTileQ = 128;         // queries per CTA tile (one MMA M=128 tile)

// Base-BVH node (host + device, 32 B).  Inner: a = left child, b = right child (> 0).
// Leaf: a = first primitive (in prim order), b = -count.
struct BvhNode {
    float lo[3];
    int32_t a;
    float hi[3];
    int32_t b;
};

// Inner node of the shallow N-BVH snapshot: both child boxes stored in the
// parent so one fetch tests both.  Child c >= 0: inner node; c < 0: leaf id -1-c.
struct InnerNode {
    float l_lo[3], l_hi[3];
    float r_lo[3], r_hi[3];
    int32_t l, r;
    int32_t pad[2];
};
static_assert(sizeof(InnerNode) == 64, "InnerNode must be 64 B");

struct HostCut {
    int32_t n_leaves = 0;
    std::vector<int32_t> leaf_base;            // base-BVH node of each leaf (DFS order)
    std::vector<float> leaf_lo, leaf_hi;       // inflated leaf boxes [n][3]
    std::vector<InnerNode> inner;              // snapshot; root = inner[0] unless n_leaves == 1
    std::vector<float> rank;                   // acceptance rank per leaf (C18)
    float dom_min[3] = {0, 0, 0};
    float dom_inv = 1.0f;
};

struct HostScene {
    std::vector<float> xyz;        // [nv][3]
    std::vector<uint32_t> tri;     // [nt][3]
    std::vector<float> vnormal;    // [nv][3]
    std::vector<float> albedo;     // [nt][3]
    std::vector<BvhNode> nodes;    // base BVH, root = 0
    std::vector<int32_t> prim;     // prim order: prim[i] = original triangle id
    std::vector<int32_t> parent;   // parent per node (-1 for root)
    double scene_diag = 0.0;
    int64_t n_base_leaves = 0;
};

// Host core (nbvh_host.cpp)
void build_sah_bvh(HostScene& sc);
// Returns NBVH status code semantics: 0 ok, 1 clamped.
int build_cut(const HostScene& sc, int32_t target, const HostCut* prev, const float* leaf_q, const float* leaf_p,
              float inflate_rel, float inflate_abs, HostCut& out);
void level_table(int L, int log2_T, int base_res, int max_res, int32_t* res, int32_t* dense, int64_t* offset,
                 int64_t* total);

}  // namespace nbvh
