// nbvh_host.cpp — host core: base-BVH construction (full-sweep SAH), error-/area-driven
// cut selection with node inflation, the shallow N-BVH snapshot, and the hash-grid
// level table.  CPU only; the result is uploaded by nbvh_capi.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <queue>
#include <vector>

#include "nbvh_internal.h"

namespace nbvh {

// ---------------------------------------------------------------- level table
// L levels from base_res^3 to max_res^3, geometric spacing; N_l = floor(base*b^l
// + 1e-9) (C1).  Dense index iff (N+1)^3 <= T, else spatial hash of size T (C2).
void level_table(int L, int log2_T, int base_res, int max_res, int32_t* res, int32_t* dense, int64_t* offset,
                 int64_t* total) {
    const double growth = L > 1 ? std::exp(std::log((double)max_res / (double)base_res) / (double)(L - 1)) : 1.0;
    const int64_t T = int64_t(1) << log2_T;
    int64_t acc = 0;
    for (int l = 0; l < L; ++l) {
        const int64_t N = (int64_t)std::floor((double)base_res * std::pow(growth, (double)l) + 1e-9);
        const int64_t n1 = N + 1, vol = n1 * n1 * n1;
        res[l] = (int32_t)N;
        dense[l] = vol <= T;
        offset[l] = acc;
        acc += vol <= T ? vol : T;
    }
    *total = acc;
}

// ---------------------------------------------------------------- SAH builder
namespace {

struct PrimBox {
    float lo[3], hi[3], c[3];
};

struct Box {
    float lo[3] = {std::numeric_limits<float>::infinity(), std::numeric_limits<float>::infinity(),
                   std::numeric_limits<float>::infinity()};
    float hi[3] = {-std::numeric_limits<float>::infinity(), -std::numeric_limits<float>::infinity(),
                   -std::numeric_limits<float>::infinity()};
    void grow(const float* l, const float* h) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], l[k]);
            hi[k] = std::max(hi[k], h[k]);
        }
    }
    double area() const {
        double e[3];
        for (int k = 0; k < 3; ++k) e[k] = std::max(0.0, (double)hi[k] - (double)lo[k]);
        return 2.0 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]);
    }
};

struct TmpNode {
    Box box;
    int32_t left = -1, right = -1;   // TmpNode indices; -1 for leaves
    int32_t begin = 0, end = 0;
};

struct Builder {
    const std::vector<PrimBox>& pb;
    std::vector<int32_t>& idx;
    std::vector<TmpNode> nodes;
    std::atomic<int32_t> next{1};

    Builder(const std::vector<PrimBox>& p, std::vector<int32_t>& i) : pb(p), idx(i), nodes(2 * p.size() + 1) {}

    void sort_axis(int32_t b, int32_t e, int axis) {
        std::sort(idx.begin() + b, idx.begin() + e, [&](int32_t x, int32_t y) {
            float cx = pb[x].c[axis], cy = pb[y].c[axis];
            return cx < cy || (cx == cy && x < y);
        });
    }

    // Full-sweep SAH ("sweeping SAH builder"): for every axis sort centroids and
    // evaluate every split position; C_trav = C_isect = 1; leaf of <= 4 prims when no
    // split is cheaper.  Ties: lowest axis, then lowest position (deterministic).
    void build(int32_t ni, int32_t b, int32_t e) {
        TmpNode& nd = nodes[ni];
        nd.begin = b;
        nd.end = e;
        for (int32_t i = b; i < e; ++i) nd.box.grow(pb[idx[i]].lo, pb[idx[i]].hi);
        const int32_t n = e - b;
        if (n == 1) return;
        const double sa = nd.box.area();
        double best = std::numeric_limits<double>::infinity();
        int best_axis = -1;
        int32_t best_pos = -1;
        std::vector<double> left_area(n);
        if (sa > 0.0) {
            for (int axis = 0; axis < 3; ++axis) {
                sort_axis(b, e, axis);
                Box acc;
                for (int32_t i = 0; i < n - 1; ++i) {
                    acc.grow(pb[idx[b + i]].lo, pb[idx[b + i]].hi);
                    left_area[i + 1] = acc.area();
                }
                Box racc;
                for (int32_t i = n - 1; i >= 1; --i) {
                    racc.grow(pb[idx[b + i]].lo, pb[idx[b + i]].hi);
                    double cost = 1.0 + (left_area[i] * i + racc.area() * (n - i)) / sa;
                    if (cost < best || (cost == best && (axis < best_axis || (axis == best_axis && i < best_pos)))) {
                        best = cost;
                        best_axis = axis;
                        best_pos = i;
                    }
                }
            }
        }
        if (n <= 4 && !(best < (double)n)) return;   // leaf
        if (best_axis < 0) {                           // degenerate: median split on x
            best_axis = 0;
            best_pos = n / 2;
        }
        if (best_axis != 2) sort_axis(b, e, best_axis);
        int32_t l = next.fetch_add(2);
        nd.left = l;
        nd.right = l + 1;
        const int32_t mid = b + best_pos;
        if (n > 8192) {
#pragma omp task default(shared) firstprivate(l, b, mid)
            build(l, b, mid);
#pragma omp task default(shared) firstprivate(l, mid, e)
            build(l + 1, mid, e);
#pragma omp taskwait
        } else {
            build(l, b, mid);
            build(l + 1, mid, e);
        }
    }
};

}  // namespace

void build_sah_bvh(HostScene& sc) {
    const int64_t nt = (int64_t)sc.tri.size() / 3;
    std::vector<PrimBox> pb(nt);
    for (int64_t t = 0; t < nt; ++t) {
        PrimBox& p = pb[t];
        for (int k = 0; k < 3; ++k) {
            p.lo[k] = std::numeric_limits<float>::infinity();
            p.hi[k] = -std::numeric_limits<float>::infinity();
        }
        for (int v = 0; v < 3; ++v)
            for (int k = 0; k < 3; ++k) {
                float x = sc.xyz[3 * sc.tri[3 * t + v] + k];
                p.lo[k] = std::min(p.lo[k], x);
                p.hi[k] = std::max(p.hi[k], x);
            }
        for (int k = 0; k < 3; ++k) p.c[k] = 0.5f * (p.lo[k] + p.hi[k]);
    }
    std::vector<int32_t> idx(nt);
    std::iota(idx.begin(), idx.end(), 0);
    Builder B(pb, idx);
#pragma omp parallel
#pragma omp single
    B.build(0, 0, (int32_t)nt);

    // Flatten depth-first (left first): root = 0, deterministic regardless of threads.
    sc.nodes.clear();
    sc.parent.clear();
    sc.prim.assign(idx.begin(), idx.end());
    sc.n_base_leaves = 0;
    struct Item { int32_t tmp, parent, is_right; };
    std::vector<Item> stack{{0, -1, 0}};
    while (!stack.empty()) {
        Item it = stack.back();
        stack.pop_back();
        const TmpNode& t = B.nodes[it.tmp];
        const int32_t me = (int32_t)sc.nodes.size();
        BvhNode n{};
        for (int k = 0; k < 3; ++k) {
            n.lo[k] = t.box.lo[k];
            n.hi[k] = t.box.hi[k];
        }
        if (t.left < 0) {
            n.a = t.begin;
            n.b = -(t.end - t.begin);
            ++sc.n_base_leaves;
        }
        sc.nodes.push_back(n);
        sc.parent.push_back(it.parent);
        if (it.parent >= 0) {
            if (it.is_right) sc.nodes[it.parent].b = me;
            else sc.nodes[it.parent].a = me;
        }
        if (t.left >= 0) {
            stack.push_back({t.right, me, 1});
            stack.push_back({t.left, me, 0});
        }
    }
    Box root;
    root.grow(sc.nodes[0].lo, sc.nodes[0].hi);
    double d2 = 0;
    for (int k = 0; k < 3; ++k) {
        double e = (double)root.hi[k] - (double)root.lo[k];
        d2 += e * e;
    }
    sc.scene_diag = std::sqrt(d2);
}

// ---------------------------------------------------------------- cut + snapshot
namespace {

bool is_leaf(const BvhNode& n) { return n.b < 0; }

double node_area(const BvhNode& n) {
    double e[3];
    for (int k = 0; k < 3; ++k) e[k] = std::max(0.0, (double)n.hi[k] - (double)n.lo[k]);
    return 2.0 * (e[0] * e[1] + e[1] * e[2] + e[2] * e[0]);
}

// C15: each side grows by max(rel * node diagonal, abs * scene diagonal); rounding to the
// nearest float of (lo - pad) keeps the inflated box a superset of the base box.
void inflate(const BvhNode& n, double scene_diag, float rel, float abs_, float* lo, float* hi) {
    double d2 = 0;
    for (int k = 0; k < 3; ++k) {
        double e = (double)n.hi[k] - (double)n.lo[k];
        d2 += e * e;
    }
    double pad = std::max((double)rel * std::sqrt(d2), (double)abs_ * scene_diag);
    for (int k = 0; k < 3; ++k) {
        lo[k] = (float)((double)n.lo[k] - pad);
        hi[k] = (float)((double)n.hi[k] + pad);
    }
}

struct SnapBuilder {
    const HostScene& sc;
    const std::vector<char>& in_cut;
    HostCut& out;
    float rel, abs_;

    // returns child code (>= 0 inner index, < 0 leaf -1-id) and its box
    int32_t visit(int32_t node, float* lo, float* hi) {
        if (in_cut[node]) {
            int32_t id = (int32_t)out.leaf_base.size();
            out.leaf_base.push_back(node);
            float l[3], h[3];
            inflate(sc.nodes[node], sc.scene_diag, rel, abs_, l, h);
            for (int k = 0; k < 3; ++k) {
                out.leaf_lo.push_back(l[k]);
                out.leaf_hi.push_back(h[k]);
                lo[k] = l[k];
                hi[k] = h[k];
            }
            return -1 - id;
        }
        int32_t me = (int32_t)out.inner.size();
        out.inner.push_back(InnerNode{});
        float llo[3], lhi[3], rlo[3], rhi[3];
        int32_t l = visit(sc.nodes[node].a, llo, lhi);
        int32_t r = visit(sc.nodes[node].b, rlo, rhi);
        InnerNode& in = out.inner[me];
        in.l = l;
        in.r = r;
        for (int k = 0; k < 3; ++k) {
            in.l_lo[k] = llo[k];
            in.l_hi[k] = lhi[k];
            in.r_lo[k] = rlo[k];
            in.r_hi[k] = rhi[k];
            lo[k] = std::min(llo[k], rlo[k]);   // exact union
            hi[k] = std::max(lhi[k], rhi[k]);
        }
        return me;
    }
};

}  // namespace

int build_cut(const HostScene& sc, int32_t target, const HostCut* prev, const float* leaf_q, const float* leaf_p,
              float inflate_rel, float inflate_abs, HostCut& out) {
    const int32_t n_nodes = (int32_t)sc.nodes.size();
    int clamped = 0;
    if (target > sc.n_base_leaves) {
        target = (int32_t)sc.n_base_leaves;
        clamped = 1;
    }
    if (target < 1) target = 1;
    std::vector<char> in_cut(n_nodes, 0);
    if (prev && leaf_q && leaf_p && prev->n_leaves > 0) {
        // Error-driven expansion: rank r = 2 ln q + ln p; split the
        // highest-ranked splittable leaves, each at most once, up to the target count.
        const int32_t n = prev->n_leaves;
        std::vector<int32_t> order(n);
        std::iota(order.begin(), order.end(), 0);
        std::vector<double> r(n);
        for (int32_t i = 0; i < n; ++i)
            r[i] = 2.0 * std::log(std::max((double)leaf_q[i], 1e-9)) + std::log(std::max((double)leaf_p[i], 1e-9));
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return r[a] > r[b]; });
        for (int32_t i = 0; i < n; ++i) in_cut[prev->leaf_base[i]] = 1;
        int32_t count = n;
        for (int32_t k = 0; k < n && count < target; ++k) {
            int32_t node = prev->leaf_base[order[k]];
            if (is_leaf(sc.nodes[node])) continue;
            in_cut[node] = 0;
            in_cut[sc.nodes[node].a] = 1;
            in_cut[sc.nodes[node].b] = 1;
            ++count;
        }
    } else {
        // Static score: split the cut node of largest surface area (p is
        // proportional to surface area), ties by lowest node index.
        using Item = std::pair<double, int32_t>;
        auto cmp = [](const Item& a, const Item& b) { return a.first < b.first || (a.first == b.first && a.second > b.second); };
        std::priority_queue<Item, std::vector<Item>, decltype(cmp)> pq(cmp);
        std::vector<int32_t> fixed;
        pq.push({node_area(sc.nodes[0]), 0});
        while (!pq.empty() && (int32_t)(pq.size() + fixed.size()) < target) {
            Item it = pq.top();
            pq.pop();
            const BvhNode& nd = sc.nodes[it.second];
            if (is_leaf(nd)) {
                fixed.push_back(it.second);
                continue;
            }
            pq.push({node_area(sc.nodes[nd.a]), nd.a});
            pq.push({node_area(sc.nodes[nd.b]), nd.b});
        }
        for (int32_t f : fixed) in_cut[f] = 1;
        while (!pq.empty()) {
            in_cut[pq.top().second] = 1;
            pq.pop();
        }
    }
    out = HostCut{};
    SnapBuilder sb{sc, in_cut, out, inflate_rel, inflate_abs};
    float lo[3], hi[3];
    int32_t root = sb.visit(0, lo, hi);
    (void)root;
    out.n_leaves = (int32_t)out.leaf_base.size();
    out.rank.assign(out.n_leaves, 0.0f);
    // Grid domain (C4 as amended for shared-grid LoD cuts), fp32: cube of
    // side max extent around the scene's root box inflated per C15 -- the same for every
    // cut, so all LoD slots (and every stage of the error-driven construction) index the
    // one hash grid identically.
    float dlo[3], dhi[3];
    inflate(sc.nodes[0], sc.scene_diag, inflate_rel, inflate_abs, dlo, dhi);
    const float ex = dhi[0] - dlo[0], ey = dhi[1] - dlo[1], ez = dhi[2] - dlo[2];
    const float side = std::fmax(std::fmax(ex, ey), ez);
    for (int k = 0; k < 3; ++k) {
        const float mid = (dlo[k] + dhi[k]) * 0.5f;
        out.dom_min[k] = mid - side * 0.5f;
    }
    out.dom_inv = 1.0f / side;
    return clamped;
}

}  // namespace nbvh
