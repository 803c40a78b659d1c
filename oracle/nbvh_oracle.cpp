// nbvh_oracle.cpp — CPU ORACLE FOR N-BVH NEURAL RAY QUERIES.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// leg may load this library.  The product (paper_2405_16237_b200/) never links,
// imports or calls it, and this file shares no code, header or table with it.
//
// Citation key: "P:n" = /root/reference/PAPER.md line n (section named alongside);
// "C<k>" = the reading register in DESIGN.md §3 (= SURVEY.md §8(c) ambiguity register).
//
// Precision: continuous quantities (interpolation, MLP, losses, gradients, Adam,
// triangle ground truth) are computed in double.  Discrete decisions that the GPU
// must reproduce bit-for-bit (slab intervals, sample positions, grid cells) are
// computed in IEEE binary32 with the operation order stated next to each, compiled
// with -ffp-contract=off (no FMA) on SSE.
//
// Parity status per function is listed in DESIGN.md §4; every function here is
// pinned by a `-m "not gpu"` test in tests/test_oracle_pins.py except
// orc_query's end-to-end *quality* (P17: "parity unpinned" — the paper ships no
// weights or per-query numbers).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// ------------------------------------------------------------------ fp16 decode
// IEEE 754 binary16 -> double, written from the format definition
// (1 sign bit, 5 exponent bits, bias 15, 10 fraction bits).
double orc_half_to_double(uint16_t h) {
    int s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023;
    double v;
    if (e == 0) v = std::ldexp((double)m, -24);                       // subnormal
    else if (e == 31) v = m ? std::numeric_limits<double>::quiet_NaN()
                            : std::numeric_limits<double>::infinity();
    else v = std::ldexp((double)(1024 + m), e - 25);                  // normal
    return s ? -v : v;
}

// ------------------------------------------------------------------ level table
// P:275 (§6 "Neural model & training"): "The hash grid contains 8 levels, starting from
// a base resolution of 8^3 to a maximum resolution of 1024^3".  Geometric spacing
// b = (max/base)^(1/(L-1)), N_l = floor(base*b^l + 1e-9)        (C1)
// Level l is dense iff (N_l+1)^3 <= T and then holds (N_l+1)^3 entries, else T (C2).
// Returns the total number of entries; offsets are cumulative entry counts.
int64_t orc_level_table(int L, int log2_T, int base_res, int max_res,
                        int32_t* res, int32_t* dense, int64_t* offset) {
    const int64_t T = (int64_t)1 << log2_T;
    const double b = (L > 1) ? std::exp((std::log((double)max_res) - std::log((double)base_res)) / (L - 1)) : 1.0;
    int64_t off = 0;
    for (int l = 0; l < L; ++l) {
        int64_t N = (int64_t)std::floor((double)base_res * std::pow(b, (double)l) + 1e-9);
        int64_t full = (N + 1) * (N + 1) * (N + 1);
        res[l] = (int32_t)N;
        dense[l] = full <= T ? 1 : 0;
        offset[l] = off;
        off += dense[l] ? full : T;
    }
    return off;
}

// ------------------------------------------------------------------ corner index
// Dense level: x + (N+1)(y + (N+1) z).  Hashed level, [Mueller22] as cited at P:101
// (§3): (x*1 XOR y*2654435761 XOR z*805459861) mod T, in uint32 arithmetic (C3).
uint32_t orc_corner_index(int32_t N, int32_t dense, int log2_T, uint32_t x, uint32_t y, uint32_t z) {
    if (dense) {
        uint32_t n1 = (uint32_t)N + 1u;
        return x + n1 * (y + n1 * z);
    }
    uint32_t h = (x * 1u) ^ (y * 2654435761u) ^ (z * 805459861u);
    return h & ((1u << log2_T) - 1u);
}

// ------------------------------------------------------------------ grid features
// Fig. node_encoding: "at each point collect features from a multi-resolution
// hash grid".  Per level: s = x*N (fp32), c = min(floor(s), N-1), f = s - c (fp32, exact);
// the 8 corners c+delta (delta bit0=x, bit1=y, bit2=z) are fetched and trilinearly
// weighted, w = prod_k (delta_k ? f_k : 1-f_k) (double).  Output [L][F], coarse -> fine.
static void encode_point(int L, int F, int log2_T, const int32_t* res, const int32_t* dense,
                         const int64_t* offset, const uint16_t* table, const float x[3],
                         double* feat /*L*F*/, uint32_t* idx_out /*L*8, nullable*/) {
    for (int l = 0; l < L; ++l) {
        const int32_t N = res[l];
        int32_t c[3];
        float f[3];
        for (int k = 0; k < 3; ++k) {
            float s = x[k] * (float)N;
            int32_t ci = (int32_t)std::floor(s);
            if (ci > N - 1) ci = N - 1;
            if (ci < 0) ci = 0;
            c[k] = ci;
            f[k] = s - (float)ci;
        }
        for (int j = 0; j < F; ++j) feat[l * F + j] = 0.0;
        for (int corner = 0; corner < 8; ++corner) {
            int d0 = corner & 1, d1 = (corner >> 1) & 1, d2 = (corner >> 2) & 1;
            uint32_t idx = orc_corner_index(N, dense[l], log2_T, (uint32_t)(c[0] + d0),
                                            (uint32_t)(c[1] + d1), (uint32_t)(c[2] + d2));
            if (idx_out) idx_out[l * 8 + corner] = idx;
            double w = (d0 ? (double)f[0] : 1.0 - (double)f[0]) *
                       (d1 ? (double)f[1] : 1.0 - (double)f[1]) *
                       (d2 ? (double)f[2] : 1.0 - (double)f[2]);
            const uint16_t* row = table + (offset[l] + (int64_t)idx) * F;
            for (int j = 0; j < F; ++j) feat[l * F + j] += w * orc_half_to_double(row[j]);
        }
    }
}

void orc_encode_points(int L, int F, int log2_T, const int32_t* res, const int32_t* dense,
                       const int64_t* offset, const uint16_t* table, const float* pts, int64_t m,
                       double* feat /*[m][L*F]*/, uint32_t* idx /*[m][L][8], nullable*/) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        encode_point(L, F, log2_T, res, dense, offset, table, pts + 3 * i, feat + i * (int64_t)L * F,
                     idx ? idx + i * (int64_t)L * 8 : nullptr);
}

// ------------------------------------------------------------------ ray / box slab test
// P:103 (§3), P:116 (§4 "Motivation"): the query is parameterised by the ray-box
// entry/exit interval.  fp32, op order: inv=1/d; tl=(lo-o)*inv; th=(hi-o)*inv;
// tn=fminf(tl,th); tf=fmaxf(tl,th); te=max(tn.x,tn.y,tn.z,tmin) (left fold);
// tx=min(tf.x,tf.y,tf.z,tmax); hit iff te <= tx.  A ray starting inside -> te = tmin (C7).
int orc_slab(const float* ray /*ox,oy,oz,tmin,dx,dy,dz,tmax*/, const float* lo, const float* hi,
             float* t_enter, float* t_exit) {
    float tn[3], tf[3];
    for (int k = 0; k < 3; ++k) {
        float inv = 1.0f / ray[4 + k];
        float tl = (lo[k] - ray[k]) * inv;
        float th = (hi[k] - ray[k]) * inv;
        tn[k] = std::fmin(tl, th);
        tf[k] = std::fmax(tl, th);
    }
    float te = std::fmax(std::fmax(std::fmax(tn[0], tn[1]), tn[2]), ray[3]);
    float tx = std::fmin(std::fmin(std::fmin(tf[0], tf[1]), tf[2]), ray[7]);
    *t_enter = te;
    *t_exit = tx;
    return te <= tx ? 1 : 0;
}

// ------------------------------------------------------------------ ordered leaf list
// P:161 (§5): queries happen "upon reaching a leaf node"; "front-to-back probing".
// Brute force over every cut leaf (no hierarchy), sorted by (t_enter, leaf id) (C5).
struct Entry { float te, tx; int32_t leaf; };

static void leaf_list(const float* ray, const float* leaf_lo, const float* leaf_hi, int32_t n_leaves,
                      std::vector<Entry>& out) {
    out.clear();
    for (int32_t i = 0; i < n_leaves; ++i) {
        float te, tx;
        if (orc_slab(ray, leaf_lo + 3 * i, leaf_hi + 3 * i, &te, &tx)) out.push_back({te, tx, i});
    }
    std::sort(out.begin(), out.end(), [](const Entry& a, const Entry& b) {
        return a.te < b.te || (a.te == b.te && a.leaf < b.leaf);
    });
}

// Writes up to `cap` entries per ray ([n][cap] row-major); count[i] = total number of
// intersected leaves (may exceed cap).
void orc_leaf_lists(const float* rays, int64_t n, const float* leaf_lo, const float* leaf_hi,
                    int32_t n_leaves, int32_t cap, int32_t* leaf, float* t_enter, float* t_exit,
                    int32_t* count) {
#pragma omp parallel
    {
        std::vector<Entry> L;
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < n; ++r) {
            leaf_list(rays + 8 * r, leaf_lo, leaf_hi, n_leaves, L);
            count[r] = (int32_t)L.size();
            for (int32_t k = 0; k < cap; ++k) {
                bool ok = k < (int32_t)L.size();
                leaf[r * cap + k] = ok ? L[k].leaf : -1;
                t_enter[r * cap + k] = ok ? L[k].te : 0.0f;
                t_exit[r * cap + k] = ok ? L[k].tx : 0.0f;
            }
        }
    }
}

// ------------------------------------------------------------------ grid domain
// P:105 (§3): "a single global neural model encompassing the entire geometry".  The grid
// covers the cube around the root box (union of the inflated cut-leaf boxes), side =
// largest extent, centred (C4).  fp32 op order: lo/hi = min/max over leaves;
// side = max(hi.x-lo.x, hi.y-lo.y, hi.z-lo.z); c = (lo+hi)*0.5; dom_min = c - side*0.5;
// dom_inv = 1/side.
// C4 (as amended for multi-cut LoD: one hash grid shared by every cut): the
// domain box is the scene's root box inflated per C15, identical for every cut; callers
// pass that single box (orc_scene_box) as a 1-"leaf" list.
// Root box = min/max over the vertices of all triangles (exact in fp32); pad =
// max(rel * diag, abs * diag) in double (diag of the root = the scene diagonal);
// lo = fp32(lo - pad), hi = fp32(hi + pad) ("slightly" inflated, C15).
void orc_scene_box(const float* verts, const uint32_t* tris, int64_t nt, float rel, float abs_, float* box) {
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t t = 0; t < nt; ++t)
        for (int c = 0; c < 3; ++c) {
            const float* v = verts + 3 * (int64_t)tris[3 * t + c];
            for (int k = 0; k < 3; ++k) {
                lo[k] = std::fmin(lo[k], v[k]);
                hi[k] = std::fmax(hi[k], v[k]);
            }
        }
    double d2 = 0;
    for (int k = 0; k < 3; ++k) {
        const double e = (double)hi[k] - (double)lo[k];
        d2 += e * e;
    }
    const double diag = std::sqrt(d2);
    const double pad = std::max((double)rel * diag, (double)abs_ * diag);
    for (int k = 0; k < 3; ++k) {
        box[k] = (float)((double)lo[k] - pad);
        box[3 + k] = (float)((double)hi[k] + pad);
    }
}

void orc_domain(const float* leaf_lo, const float* leaf_hi, int32_t n_leaves, float* dom_min, float* dom_inv) {
    float lo[3], hi[3];
    for (int k = 0; k < 3; ++k) { lo[k] = leaf_lo[k]; hi[k] = leaf_hi[k]; }
    for (int32_t i = 1; i < n_leaves; ++i)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::fmin(lo[k], leaf_lo[3 * i + k]);
            hi[k] = std::fmax(hi[k], leaf_hi[3 * i + k]);
        }
    float side = std::fmax(std::fmax(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
    for (int k = 0; k < 3; ++k) {
        float c = (lo[k] + hi[k]) * 0.5f;
        dom_min[k] = c - side * 0.5f;
    }
    *dom_inv = 1.0f / side;
}

// ------------------------------------------------------------------ segment sampling
// P:133 ("We sample uniformly along a given ray-box intersection interval")
// ("stratified point-sampling along the ray").  u_i = (2i+1)/(2n) at inference, or
// (i + xi_i)/n when jitter xi is given (training) (C8).  fp32, op order:
// dt = t1-t0; t = t0 + u*dt; p = o + t*d; x = clamp((p - dom_min)*dom_inv, 0, 1).
// Points are ordered entry -> exit: the concatenation order encodes the direction.
void orc_segment_points(const float* ray, float t0, float t1, int n, const float* xi /*nullable, n*/,
                        const float* dom_min, float dom_inv, float* pts /*[n][3]*/) {
    float dt = t1 - t0;
    for (int i = 0; i < n; ++i) {
        float u = xi ? ((float)i + xi[i]) / (float)n : (float)(2 * i + 1) / (float)(2 * n);
        float t = t0 + u * dt;
        for (int k = 0; k < 3; ++k) {
            float p = ray[k] + t * ray[4 + k];
            float x = (p - dom_min[k]) * dom_inv;
            pts[3 * i + k] = std::fmin(std::fmax(x, 0.0f), 1.0f);
        }
    }
}

// ------------------------------------------------------------------ MLP
// hidden layers of 64 neurons with ReLU; the output layer is linear here and the
// sigmoid / linear output activations are applied by the decode (C10-C12).
// Weights are fp16 [out][in] row-major (converted exactly to double), biases fp32.
// Layer k has dims[k] inputs and dims[k+1] outputs; n_layers = hidden + 1.
static void mlp_forward_one(int n_layers, const int32_t* dims, const uint16_t* const* W,
                            const float* const* b, const double* x, double* z,
                            std::vector<double>* acts /*nullable: post-activation per layer*/) {
    std::vector<double> h(x, x + dims[0]), nxt;
    if (acts) acts[0] = h;
    for (int k = 0; k < n_layers; ++k) {
        nxt.assign(dims[k + 1], 0.0);
        for (int o = 0; o < dims[k + 1]; ++o) {
            double s = (double)b[k][o];
            for (int i = 0; i < dims[k]; ++i) s += orc_half_to_double(W[k][(int64_t)o * dims[k] + i]) * h[i];
            nxt[o] = (k + 1 < n_layers) ? (s > 0.0 ? s : 0.0) : s;
        }
        h.swap(nxt);
        if (acts) acts[k + 1] = h;
    }
    for (int o = 0; o < dims[n_layers]; ++o) z[o] = h[o];
}

// W_all / b_all: layers concatenated in order.
static void split_layers(int n_layers, const int32_t* dims, const uint16_t* W_all, const float* b_all,
                         std::vector<const uint16_t*>& W, std::vector<const float*>& b) {
    W.resize(n_layers);
    b.resize(n_layers);
    int64_t wo = 0, bo = 0;
    for (int k = 0; k < n_layers; ++k) {
        W[k] = W_all + wo;
        b[k] = b_all + bo;
        wo += (int64_t)dims[k] * dims[k + 1];
        bo += dims[k + 1];
    }
}

void orc_mlp_forward(int n_layers, const int32_t* dims, const uint16_t* W_all, const float* b_all,
                     const double* x, int64_t m, double* z) {
    std::vector<const uint16_t*> W;
    std::vector<const float*> b;
    split_layers(n_layers, dims, W_all, b_all, W, b);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        mlp_forward_one(n_layers, dims, W.data(), b.data(), x + i * dims[0], z + i * dims[n_layers], nullptr);
}

// ------------------------------------------------------------------ decode
static double sigmoid(double v) { return 1.0 / (1.0 + std::exp(-v)); }

// ------------------------------------------------------------------ full neural ray query
// Model description passed to the query / training oracles.
struct OrcModel {
    int32_t L, F, log2_T, n_points, n_layers;
    const int32_t* res; const int32_t* dense; const int64_t* offset;
    const uint16_t* table;          // fp16 [entries][F]
    const int32_t* dims;            // n_layers+1
    const uint16_t* W_all; const float* b_all;
    const float* dom_min; float dom_inv;
};

// One (ray, leaf) neural query (Fig. node_encoding): sample the
// interval, encode every point, concatenate [point][level][F], decode with the MLP.
static void neural_query(const OrcModel& M, const std::vector<const uint16_t*>& W,
                         const std::vector<const float*>& b, const float* ray, float t0, float t1,
                         const float* xi, double* z, double* x_in /*nullable D_in*/,
                         uint32_t* idx /*nullable n*L*8*/, float* pts_out /*nullable n*3*/,
                         std::vector<double>* acts) {
    const int n = M.n_points, LF = M.L * M.F;
    std::vector<float> pts(3 * n);
    orc_segment_points(ray, t0, t1, n, xi, M.dom_min, M.dom_inv, pts.data());
    std::vector<double> x(n * LF);
    for (int i = 0; i < n; ++i)
        encode_point(M.L, M.F, M.log2_T, M.res, M.dense, M.offset, M.table, &pts[3 * i], &x[i * LF],
                     idx ? idx + i * M.L * 8 : nullptr);
    if (x_in) std::copy(x.begin(), x.end(), x_in);
    if (pts_out) std::copy(pts.begin(), pts.end(), pts_out);
    mlp_forward_one(M.n_layers, M.dims, W.data(), b.data(), x.data(), z, acts);
}

// P:161 (§5) traversal semantics, P:201 (§5.2 "Visibility": hit iff sigmoid < 0.5, C13),
// P:237 ("locally learning the distance": t = t0 + sigmoid(z_t)(t1-t0)), P:243 (normal,
// albedo).  mode 0 = R2 nearest hit: walk the (t_enter, id)-ordered list, query a leaf
// iff t_enter <= t_best, keep argmin (t, t_enter, id).  mode 1 = R1: stop at the first
// leaf whose query reports a hit (C5).
// Outputs per ray: hit, t, normal[3], albedo[3], leaf, n_queries, and margin = min over
// its queries of |sigmoid(z_vis) - 0.5| (for the ambiguity band), z_trace [n][cap][8]
// (NaN where not queried, nullable), tmargin (nullable) = min distance between the best
// t and any t it was compared with (termination entries, competing hits): decisions
// closer than the MLP's precision are ambiguous too.
void orc_query(int32_t L, int32_t F, int32_t log2_T, int32_t n_points, int32_t n_layers,
               const int32_t* res, const int32_t* dense, const int64_t* offset, const uint16_t* table,
               const int32_t* dims, const uint16_t* W_all, const float* b_all,
               const float* leaf_lo, const float* leaf_hi, int32_t n_leaves,
               const float* rays, int64_t n, int32_t mode,
               uint8_t* hit, float* t_out, float* normal, float* albedo, int32_t* leaf_out,
               int32_t* nq_out, double* margin, double* z_trace, int32_t cap, double* tmargin,
               const float* dom_box) {
    float dom_min[3], dom_inv;
    if (dom_box) orc_domain(dom_box, dom_box + 3, 1, dom_min, &dom_inv);
    else orc_domain(leaf_lo, leaf_hi, n_leaves, dom_min, &dom_inv);
    OrcModel M{L, F, log2_T, n_points, n_layers, res, dense, offset, table, dims, W_all, b_all, dom_min, dom_inv};
    std::vector<const uint16_t*> W;
    std::vector<const float*> b;
    split_layers(n_layers, dims, W_all, b_all, W, b);
    const int n_out = dims[n_layers];
#pragma omp parallel
    {
        std::vector<Entry> lst;
        std::vector<double> z(n_out);
#pragma omp for schedule(dynamic, 16)
        for (int64_t r = 0; r < n; ++r) {
            const float* ray = rays + 8 * r;
            leaf_list(ray, leaf_lo, leaf_hi, n_leaves, lst);
            if (z_trace)
                for (int64_t k = 0; k < (int64_t)cap * 8; ++k) z_trace[r * cap * 8 + k] = std::nan("");
            bool found = false;
            double bt = 0, bte = 0, bn[3] = {0, 0, 0}, ba[3] = {0, 0, 0};
            int32_t bleaf = -1, nq = 0;
            double marg = std::numeric_limits<double>::infinity();
            double tmarg = std::numeric_limits<double>::infinity();
            for (size_t k = 0; k < lst.size(); ++k) {
                const Entry& e = lst[k];
                if (found) tmarg = std::min(tmarg, std::fabs((double)e.te - bt));
                if (found && (double)e.te > bt) break;              // front-to-back termination
                neural_query(M, W, b, ray, e.te, e.tx, nullptr, z.data(), nullptr, nullptr, nullptr, nullptr);
                ++nq;
                if (z_trace && (int32_t)k < cap)
                    for (int c = 0; c < 8; ++c) z_trace[(r * cap + k) * 8 + c] = z[c];
                marg = std::min(marg, std::fabs(sigmoid(z[0]) - 0.5));
                if (z[0] < 0.0) {                                    // sigmoid(z_vis) < 0.5: hit
                    double tl = sigmoid(z[1]);
                    double t = (double)e.te + tl * ((double)e.tx - (double)e.te);
                    if (found) tmarg = std::min(tmarg, std::fabs(t - bt));
                    bool better = !found || t < bt || (t == bt && ((double)e.te < bte ||
                                  ((double)e.te == bte && e.leaf < bleaf)));
                    if (better) {
                        found = true; bt = t; bte = e.te; bleaf = e.leaf;
                        double nn = std::sqrt(z[2] * z[2] + z[3] * z[3] + z[4] * z[4]);
                        nn = std::max(nn, 1e-6);
                        for (int c = 0; c < 3; ++c) { bn[c] = z[2 + c] / nn; ba[c] = sigmoid(z[5 + c]); }
                    }
                    if (mode == 1) break;                            // R1: first confident hit
                }
            }
            hit[r] = found ? 1 : 0;
            t_out[r] = found ? (float)bt : std::numeric_limits<float>::infinity();
            for (int c = 0; c < 3; ++c) {
                normal[3 * r + c] = (float)bn[c];
                albedo[3 * r + c] = (float)ba[c];
            }
            leaf_out[r] = bleaf;
            nq_out[r] = nq;
            margin[r] = marg;
            if (tmargin) tmargin[r] = tmarg;
        }
    }
}

// ------------------------------------------------------------------ fp32 decode sigmoid (C27)
// The decode's sigmoid as DESIGN.md C27 defines it: correctly rounded fp32 operations only
// (mul, fma, rint, add, div), so every IEEE-754 implementation produces the same bits.
//   x = clamp(-z, -87, 87); n = rint(x * log2 e); r = x - n ln2 (hi/lo, two fmas);
//   p = degree-7 Taylor polynomial of e^r (Horner, fmas); e = p * 2^n; s = 1 / (1 + e).
// |r| <= 0.35 so the truncation error is < 6e-9 relative; s agrees with the exact sigmoid
// to a few fp32 ulp (pinned in tests/test_oracle.py).
static float sigmoid_f32(float z) {
    const float x = std::fmin(std::fmax(-z, -87.0f), 87.0f);
    const float n = std::nearbyint(x * 1.44269504f);
    float r = std::fma(-n, 0.693145751953125f, x);
    r = std::fma(-n, 1.42860677e-6f, r);
    float p = 1.98412698e-4f;
    p = std::fma(p, r, 1.38888889e-3f);
    p = std::fma(p, r, 8.33333333e-3f);
    p = std::fma(p, r, 4.16666667e-2f);
    p = std::fma(p, r, 1.66666667e-1f);
    p = std::fma(p, r, 0.5f);
    p = std::fma(p, r, 1.0f);
    p = std::fma(p, r, 1.0f);
    const int32_t bits = ((int32_t)n + 127) << 23;
    float scale;
    std::memcpy(&scale, &bits, 4);
    const float e = p * scale;
    return 1.0f / (1.0f + e);
}
extern "C" float orc_sigmoid_f32(float z) { return sigmoid_f32(z); }

// ------------------------------------------------------------------ logic replay (fp32)
// The decisions of the query (termination, hit, best-hit selection) replayed in fp32 on
// a given z per (ray, list position) — e.g. the z the GPU recorded — so that hit mask,
// winning leaf, t bits and query count can be compared exactly (SURVEY §8(c) tier iv).
// fp32 op order: tl = sigmoid_f32(z_t) (C27); t = t0 + tl*(t1-t0);
// normal: nn = sqrtf(nx*nx + ny*ny + nz*nz) (left fold), n/fmaxf(nn, 1e-6f);
// albedo = sigmoid_f32(z).  Returns the number of rays where a needed z was
// missing (NaN) from the trace.
int64_t orc_replay(const float* leaf_lo, const float* leaf_hi, int32_t n_leaves, const float* rays,
                   int64_t n, int32_t mode, const float* z_trace /*[n][cap][8]*/, int32_t cap,
                   uint8_t* hit, float* t_out, float* normal, float* albedo, int32_t* leaf_out,
                   int32_t* nq_out) {
    int64_t missing = 0;
#pragma omp parallel
    {
        std::vector<Entry> lst;
#pragma omp for schedule(dynamic, 64) reduction(+ : missing)
        for (int64_t r = 0; r < n; ++r) {
            const float* ray = rays + 8 * r;
            leaf_list(ray, leaf_lo, leaf_hi, n_leaves, lst);
            bool found = false;
            float bt = 0, bte = 0, bn[3] = {0, 0, 0}, ba[3] = {0, 0, 0};
            int32_t bleaf = -1, nq = 0;
            for (size_t k = 0; k < lst.size(); ++k) {
                const Entry& e = lst[k];
                if (found && e.te > bt) break;
                if ((int32_t)k >= cap || std::isnan(z_trace[(r * cap + k) * 8])) { ++missing; break; }
                const float* z = z_trace + (r * cap + k) * 8;
                ++nq;
                if (z[0] < 0.0f) {
                    float tl = sigmoid_f32(z[1]);
                    float t = e.te + tl * (e.tx - e.te);
                    bool better = !found || t < bt || (t == bt && (e.te < bte || (e.te == bte && e.leaf < bleaf)));
                    if (better) {
                        found = true; bt = t; bte = e.te; bleaf = e.leaf;
                        float nn = std::sqrt(z[2] * z[2] + z[3] * z[3] + z[4] * z[4]);
                        nn = std::fmax(nn, 1e-6f);
                        for (int c = 0; c < 3; ++c) { bn[c] = z[2 + c] / nn; ba[c] = sigmoid_f32(z[5 + c]); }
                    }
                    if (mode == 1) break;
                }
            }
            hit[r] = found ? 1 : 0;
            t_out[r] = found ? bt : std::numeric_limits<float>::infinity();
            for (int c = 0; c < 3; ++c) { normal[3 * r + c] = bn[c]; albedo[3 * r + c] = ba[c]; }
            leaf_out[r] = bleaf;
            nq_out[r] = nq;
        }
    }
    return missing;
}

// ------------------------------------------------------------------ cut structure check
// P:180 (§5.1): the N-BVH leaves are "a cut in this BVH": every triangle lies in exactly
// one leaf's subtree.  P:275: nodes are inflated "slightly" (C15: each side grown by
// max(1e-3*diag(node), 1e-6*diag(scene))).  Inputs: mesh, per-leaf triangle lists (CSR),
// per-leaf uninflated base boxes and inflated leaf boxes.  Returns a bitmask:
// 1 = a triangle is in zero or several leaves; 2 = a triangle AABB escapes its base box;
// 4 = a base box escapes its leaf box; 8 = inflation differs from C15 by > 1e-5 relative.
int32_t orc_check_cut(const float* verts, const uint32_t* tris, int64_t nt, int32_t n_leaves,
                      const int64_t* leaf_tri_off, const int32_t* leaf_tris,
                      const float* base_lo, const float* base_hi, const float* leaf_lo,
                      const float* leaf_hi, double scene_diag) {
    int32_t bad = 0;
    std::vector<int32_t> seen(nt, 0);
    for (int32_t l = 0; l < n_leaves; ++l) {
        for (int64_t j = leaf_tri_off[l]; j < leaf_tri_off[l + 1]; ++j) {
            int32_t t = leaf_tris[j];
            if (t < 0 || t >= nt) { bad |= 1; continue; }
            seen[t] += 1;
            for (int v = 0; v < 3; ++v)
                for (int k = 0; k < 3; ++k) {
                    float p = verts[3 * tris[3 * t + v] + k];
                    if (p < base_lo[3 * l + k] || p > base_hi[3 * l + k]) bad |= 2;
                }
        }
        double d2 = 0;
        for (int k = 0; k < 3; ++k) {
            if (base_lo[3 * l + k] < leaf_lo[3 * l + k] || base_hi[3 * l + k] > leaf_hi[3 * l + k]) bad |= 4;
            double e = (double)base_hi[3 * l + k] - (double)base_lo[3 * l + k];
            d2 += e * e;
        }
        double pad = std::max(1e-3 * std::sqrt(d2), 1e-6 * scene_diag);
        for (int k = 0; k < 3; ++k) {
            double plo = (double)base_lo[3 * l + k] - (double)leaf_lo[3 * l + k];
            double phi = (double)leaf_hi[3 * l + k] - (double)base_hi[3 * l + k];
            double tol = 1e-5 * pad + 4.0 * std::ldexp(1.0, -23) * (std::fabs((double)base_lo[3 * l + k]) + std::fabs((double)base_hi[3 * l + k]));
            if (std::fabs(plo - pad) > tol || std::fabs(phi - pad) > tol) bad |= 8;
        }
    }
    for (int64_t t = 0; t < nt; ++t)
        if (seen[t] != 1) bad |= 1;
    return bad;
}

// ------------------------------------------------------------------ triangle ground truth
// ground truth is "obtained by intersecting the actual geometry".  Moller-Trumbore
// in double (inputs fp32, converted exactly), op order as written; accepts t in [t0,t1].
// Returns 1 and (t, b1, b2) on a hit.  Degenerate (|det| < 1e-20) -> no hit.
int orc_triangle_hit(const double o[3], const double d[3], const double v0[3], const double v1[3],
                     const double v2[3], double t0, double t1, double* t_out, double* b1, double* b2) {
    double e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
    double e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
    double p[3] = {d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2], d[0] * e2[1] - d[1] * e2[0]};
    double det = e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2];
    if (std::fabs(det) < 1e-20) return 0;
    double inv = 1.0 / det;
    double s[3] = {o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]};
    double u = (s[0] * p[0] + s[1] * p[1] + s[2] * p[2]) * inv;
    if (u < 0.0 || u > 1.0) return 0;
    double q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2], s[0] * e1[1] - s[1] * e1[0]};
    double v = (d[0] * q[0] + d[1] * q[1] + d[2] * q[2]) * inv;
    if (v < 0.0 || u + v > 1.0) return 0;
    double t = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
    if (t < t0 || t > t1) return 0;
    *t_out = t; *b1 = u; *b2 = v;
    return 1;
}

// Nearest hit among a triangle list within [t0,t1]; ties -> lowest triangle id.
// gt: [vis, t_local, nx, ny, nz, ar, ag, ab, t_hit]; vis = 1 means NO intersection.
// Shading normal = barycentric blend of vertex normals, normalised (C22).
static void label_segment(const float* verts, const uint32_t* tris, const float* vnormals,
                          const float* tri_albedo, const int32_t* tri_list, int64_t n_list,
                          const float* ray, float t0, float t1, double* gt) {
    double o[3] = {ray[0], ray[1], ray[2]}, d[3] = {ray[4], ray[5], ray[6]};
    bool found = false;
    double bt = 0, bb1 = 0, bb2 = 0;
    int32_t btri = -1;
    for (int64_t j = 0; j < n_list; ++j) {
        int32_t t = tri_list[j];
        double v[3][3];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 3; ++k) v[a][k] = verts[3 * tris[3 * t + a] + k];
        double th, b1, b2;
        if (orc_triangle_hit(o, d, v[0], v[1], v[2], (double)t0, (double)t1, &th, &b1, &b2)) {
            if (!found || th < bt || (th == bt && t < btri)) { found = true; bt = th; bb1 = b1; bb2 = b2; btri = t; }
        }
    }
    for (int c = 0; c < 9; ++c) gt[c] = 0.0;
    gt[0] = found ? 0.0 : 1.0;
    if (!found) return;
    double dt = (double)t1 - (double)t0;
    gt[1] = dt > 0.0 ? (bt - (double)t0) / dt : 0.0;
    double n[3];
    for (int k = 0; k < 3; ++k)
        n[k] = (1.0 - bb1 - bb2) * vnormals[3 * tris[3 * btri + 0] + k] + bb1 * vnormals[3 * tris[3 * btri + 1] + k] +
               bb2 * vnormals[3 * tris[3 * btri + 2] + k];
    double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    for (int k = 0; k < 3; ++k) gt[2 + k] = nn > 0 ? n[k] / nn : 0.0;
    for (int k = 0; k < 3; ++k) gt[5 + k] = tri_albedo[3 * btri + k];
    gt[8] = bt;
}

// Batch labelling of (ray, leaf, [t0,t1]) segments against each leaf's triangle list.
void orc_label(const float* verts, const uint32_t* tris, const float* vnormals, const float* tri_albedo,
               const int64_t* leaf_tri_off, const int32_t* leaf_tris, const float* rays, const int32_t* leaf,
               const float* t0, const float* t1, int64_t n, double* gt /*[n][9]*/) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        int32_t l = leaf[i];
        label_segment(verts, tris, vnormals, tri_albedo, leaf_tris + leaf_tri_off[l],
                      leaf_tri_off[l + 1] - leaf_tri_off[l], rays + 8 * i, t0[i], t1[i], gt + 9 * i);
    }
}

// ------------------------------------------------------------------ losses
// Per-sample combined loss: L = 2 L_vis + g (2 L_dist + L_normal + L_albedo),
// g = [gt_vis == 0] ("If the ground-truth visibility is 1 ... we set the losses for
// all other data to zero").  L_vis = BCE(sigmoid(z0), gt_vis); L_dist =
// |sigmoid(z1) - gt_t|; L_normal = mean_3 |z2..4 - gt_n| (P:243, L1 on the
// linear output); L_albedo = mean_3 (a-y)^2/(sg(a)^2 + 0.01), a = sigmoid(z5..7)
// (P:243 relative L2, C19).  Writes the four terms and dL/dz[8]; returns L.
// den (nullable, 3): if den_mode == 1 the albedo denominators are taken from den (frozen,
// the value-level meaning of the stop-gradient), if den_mode == 0 they are written to it.
static double sample_loss_impl(const double* z, const double* gt, double* terms, double* dz, double* den,
                               int den_mode);
double orc_sample_loss(const double* z, const double* gt, double* terms /*4, nullable*/, double* dz /*8, nullable*/) {
    return sample_loss_impl(z, gt, terms, dz, nullptr, 0);
}
static double sample_loss_impl(const double* z, const double* gt, double* terms, double* dz, double* den,
                               int den_mode) {
    const double y = gt[0];
    // BCE(sigmoid(z), y) = softplus(z) - y z, written stably.
    double lvis = std::max(z[0], 0.0) - z[0] * y + std::log1p(std::exp(-std::fabs(z[0])));
    double g = (y == 0.0) ? 1.0 : 0.0;
    double st = sigmoid(z[1]);
    double ldist = std::fabs(st - gt[1]);
    double lnorm = 0, lalb = 0;
    for (int k = 0; k < 3; ++k) lnorm += std::fabs(z[2 + k] - gt[2 + k]) / 3.0;
    double a[3];
    for (int k = 0; k < 3; ++k) {
        a[k] = sigmoid(z[5 + k]);
        double dk = a[k] * a[k] + 0.01;
        if (den && den_mode == 1) dk = den[k];
        else if (den) den[k] = dk;
        lalb += (a[k] - gt[5 + k]) * (a[k] - gt[5 + k]) / dk / 3.0;
    }
    if (terms) { terms[0] = lvis; terms[1] = g * ldist; terms[2] = g * lnorm; terms[3] = g * lalb; }
    if (dz) {
        auto sgn = [](double v) { return v > 0 ? 1.0 : (v < 0 ? -1.0 : 0.0); };
        dz[0] = 2.0 * (sigmoid(z[0]) - y);
        dz[1] = g * 2.0 * sgn(st - gt[1]) * st * (1.0 - st);
        for (int k = 0; k < 3; ++k) dz[2 + k] = g * sgn(z[2 + k] - gt[2 + k]) / 3.0;
        for (int k = 0; k < 3; ++k)
            dz[5 + k] = g * 2.0 * (a[k] - gt[5 + k]) / (a[k] * a[k] + 0.01) / 3.0 * a[k] * (1.0 - a[k]);
    }
    return 2.0 * lvis + g * (2.0 * ldist + lnorm + lalb);
}

// ------------------------------------------------------------------ reverse mode of one sample
// P:142 ("the measured loss is back-propagated to the model's learnable parameters"),
// P:61 (hash-grid backprop).  acts[k] = input of layer k (acts[0] = the features x, then
// post-ReLU hidden activations); delta = dL/dz (already scaled).  Layer k (dims[k] ->
// dims[k+1]): g_b += delta, g_W += delta (x) acts[k], delta <- W_k^T delta masked by
// ReLU'(acts[k] > 0) for k > 0; the final delta = dL/dx is scattered into the tables
// through the trilinear weights of the sample's points (idx = corner indices).
// absolute = true runs the same recursion on |delta|, |W|, |acts| with the same masks:
// the magnitude sums that bound floating-point error (tests only; no step of the method).
// hidden_delta (nullable, [n_layers-1][64]): the masked delta of each hidden layer.
// mask (nullable, [n_layers-1][64]): ReLU decisions taken by someone else (the GPU kernel's
// own, C36) instead of acts > 0.  acts_abs (nullable): in absolute mode, the magnitudes of
// the layer inputs (|W| |h| + |b| of the forward) used instead of |acts|, so the sums also
// bound the error of inputs that were themselves rounded.
static void backward_sample(const OrcModel& M, const std::vector<const uint16_t*>& W,
                            const std::vector<double>* acts, std::vector<double> delta, const float* pts,
                            const uint32_t* idx, int64_t nW, int64_t nb, double* g_table, double* g_W, double* g_b,
                            bool absolute, double* hidden_delta, const uint8_t* mask = nullptr,
                            const std::vector<double>* acts_abs = nullptr) {
    const int n_layers = M.n_layers, L = M.L, F = M.F, LF = L * F;
    const int32_t* dims = M.dims;
    if (absolute)
        for (double& v : delta) v = std::fabs(v);
    int64_t wo = nW, bo = nb;
    for (int k = n_layers - 1; k >= 0; --k) {
        wo -= (int64_t)dims[k] * dims[k + 1];
        bo -= dims[k + 1];
        const std::vector<double>& hin = acts[k];
        const std::vector<double>& hmag = (absolute && acts_abs) ? acts_abs[k] : acts[k];
        std::vector<double> dprev(dims[k], 0.0);
        for (int o = 0; o < dims[k + 1]; ++o) {
            g_b[bo + o] += delta[o];
            for (int i = 0; i < dims[k]; ++i) {
                const double w = orc_half_to_double(W[k][(int64_t)o * dims[k] + i]);
                g_W[wo + (int64_t)o * dims[k] + i] += delta[o] * (absolute ? std::fabs(hmag[i]) : hin[i]);
                dprev[i] += delta[o] * (absolute ? std::fabs(w) : w);
            }
        }
        if (k > 0) {
            for (int i = 0; i < dims[k]; ++i) {                                          // ReLU'
                const bool on = mask ? mask[(k - 1) * 64 + i] != 0 : hin[i] > 0.0;
                dprev[i] = on ? dprev[i] : 0.0;
            }
            if (hidden_delta)
                for (int i = 0; i < dims[k]; ++i) hidden_delta[(k - 1) * 64 + i] = dprev[i];
        }
        delta.swap(dprev);
    }
    // delta = dL/dx (concatenated features) -> scatter into the tables through the
    // trilinear weights (hash-grid backprop).
    for (int p = 0; p < M.n_points; ++p)
        for (int l = 0; l < L; ++l) {
            const int32_t N = M.res[l];
            float f[3];
            for (int k = 0; k < 3; ++k) {
                float s = pts[3 * p + k] * (float)N;
                int32_t ci = (int32_t)std::floor(s);
                if (ci > N - 1) ci = N - 1;
                if (ci < 0) ci = 0;
                f[k] = s - (float)ci;
            }
            for (int corner = 0; corner < 8; ++corner) {
                int d0 = corner & 1, d1 = (corner >> 1) & 1, d2 = (corner >> 2) & 1;
                double w = (d0 ? (double)f[0] : 1.0 - (double)f[0]) * (d1 ? (double)f[1] : 1.0 - (double)f[1]) *
                           (d2 ? (double)f[2] : 1.0 - (double)f[2]);
                int64_t row = M.offset[l] + (int64_t)idx[(p * L + l) * 8 + corner];
                for (int j = 0; j < F; ++j) g_table[row * F + j] += w * delta[p * LF + l * F + j];
            }
        }
}

// ------------------------------------------------------------------ training gradient
// One training step's forward + backward in double ("the measured loss is
// back-propagated to the model's learnable parameters"; P:197 first-leaf-only training
// with acceptance probability max(r/r_max, 0.005), C18; P:193 rays against the cut).
// Inputs: rays [n][8]; u [n] acceptance draws; xi [n][n_points] stratification jitter;
// leaf_rank [n_leaves] (rank r; acceptance p = max((r - min r + 1e-6)/max(...), 0.005)
// in fp32, op order as written, so both sides take the decision in fp32).
// Outputs: gradients of the mean loss over accepted samples w.r.t. the fp16-valued
// parameters: g_table [entries*F], g_W (concatenated, [out][in]), g_b; per-sample
// records (accepted flag, leaf, loss) and the loss sum; returns #accepted.
int64_t orc_train_grad(int32_t L, int32_t F, int32_t log2_T, int32_t n_points, int32_t n_layers,
                       const int32_t* res, const int32_t* dense, const int64_t* offset, const uint16_t* table,
                       int64_t n_entries, const int32_t* dims, const uint16_t* W_all, const float* b_all,
                       const float* leaf_lo, const float* leaf_hi, int32_t n_leaves,
                       const float* leaf_rank, const int64_t* leaf_tri_off, const int32_t* leaf_tris,
                       const float* verts, const uint32_t* tris, const float* vnormals, const float* tri_albedo,
                       const float* rays, int64_t n, const float* u, const float* xi,
                       double* g_table, double* g_W, double* g_b,
                       uint8_t* accepted, int32_t* first_leaf, double* sample_loss, double* gt_out /*[n][9]*/,
                       double* loss_sum, const float* dom_box) {
    float dom_min[3], dom_inv;
    if (dom_box) orc_domain(dom_box, dom_box + 3, 1, dom_min, &dom_inv);
    else orc_domain(leaf_lo, leaf_hi, n_leaves, dom_min, &dom_inv);
    OrcModel M{L, F, log2_T, n_points, n_layers, res, dense, offset, table, dims, W_all, b_all, dom_min, dom_inv};
    std::vector<const uint16_t*> W;
    std::vector<const float*> b;
    split_layers(n_layers, dims, W_all, b_all, W, b);
    // acceptance probabilities (fp32, C18)
    float rmin = leaf_rank[0], rmax = leaf_rank[0];
    for (int32_t i = 1; i < n_leaves; ++i) { rmin = std::fmin(rmin, leaf_rank[i]); rmax = std::fmax(rmax, leaf_rank[i]); }
    const float eps = 1e-6f;
    float rhmax = (rmax - rmin) + eps;
    std::vector<float> pacc(n_leaves);
    for (int32_t i = 0; i < n_leaves; ++i) pacc[i] = std::fmax(((leaf_rank[i] - rmin) + eps) / rhmax, 0.005f);

    int64_t nW = 0, nb = 0;
    for (int k = 0; k < n_layers; ++k) { nW += (int64_t)dims[k] * dims[k + 1]; nb += dims[k + 1]; }
    std::fill(g_table, g_table + n_entries * F, 0.0);
    std::fill(g_W, g_W + nW, 0.0);
    std::fill(g_b, g_b + nb, 0.0);

    // pass 1: select + label (independent per ray)
    std::vector<float> s_t0(n), s_t1(n);
    int64_t n_acc = 0;
    std::vector<Entry> lst;
    for (int64_t r = 0; r < n; ++r) {
        accepted[r] = 0; first_leaf[r] = -1; sample_loss[r] = 0.0;
        for (int c = 0; c < 9; ++c) gt_out[9 * r + c] = 0.0;
        leaf_list(rays + 8 * r, leaf_lo, leaf_hi, n_leaves, lst);
        if (lst.empty()) continue;
        const Entry& e = lst[0];                                   // first leaf only
        first_leaf[r] = e.leaf;
        if (!(u[r] < pacc[e.leaf])) continue;                      // stochastic acceptance
        accepted[r] = 1;
        s_t0[r] = e.te; s_t1[r] = e.tx;
        ++n_acc;
        int32_t l = e.leaf;
        label_segment(verts, tris, vnormals, tri_albedo, leaf_tris + leaf_tri_off[l],
                      leaf_tri_off[l + 1] - leaf_tri_off[l], rays + 8 * r, e.te, e.tx, gt_out + 9 * r);
    }
    *loss_sum = 0.0;
    if (n_acc == 0) return 0;
    const double inv_m = 1.0 / (double)n_acc;                      // mean over accepted samples (C19)
    const int D = dims[0];
    // pass 2: forward, loss, backward (serial accumulation: deterministic)
    std::vector<double> z(8), dz(8), x(D);
    std::vector<uint32_t> idx(n_points * L * 8);
    std::vector<float> pts(3 * n_points);
    std::vector<std::vector<double>> acts(n_layers + 1);
    for (int64_t r = 0; r < n; ++r) {
        if (!accepted[r]) continue;
        neural_query(M, W, b, rays + 8 * r, s_t0[r], s_t1[r], xi + r * n_points, z.data(), x.data(),
                     idx.data(), pts.data(), acts.data());
        double lr = orc_sample_loss(z.data(), gt_out + 9 * r, nullptr, dz.data());
        sample_loss[r] = lr;
        *loss_sum += lr;
        // backward through the MLP and the hash grid (mean over accepted samples)
        std::vector<double> delta(dz.begin(), dz.end());
        for (int i = 0; i < dims[n_layers]; ++i) delta[i] *= inv_m;
        backward_sample(M, W, acts.data(), delta, pts.data(), idx.data(), nW, nb, g_table, g_W, g_b, false, nullptr);
    }
    return n_acc;
}

// Loss of the same batch for given (double) parameter values — used by the finite
// difference pin (P13).  With den_mode = 1 the relative-L2 denominators are frozen at the
// values recorded by a den_mode = 0 call, which is what the stop-gradient means (C19).  Parameters are passed as double arrays (not fp16) so that
// central differences can perturb them; selection/labels come from a previous
// orc_train_grad call (accepted, first_leaf, gt) so the loss is a smooth function.
double orc_batch_loss_double(int32_t L, int32_t F, int32_t log2_T, int32_t n_points, int32_t n_layers,
                             const int32_t* res, const int32_t* dense, const int64_t* offset,
                             const double* table, const int32_t* dims, const double* W_all, const double* b_all,
                             const float* leaf_lo, const float* leaf_hi, int32_t n_leaves,
                             const float* rays, int64_t n, const float* xi, const uint8_t* accepted,
                             const float* t0, const float* t1, const double* gt,
                             double* den /*[n][3]*/, int32_t den_mode, const float* dom_box) {
    float dom_min[3], dom_inv;
    if (dom_box) orc_domain(dom_box, dom_box + 3, 1, dom_min, &dom_inv);
    else orc_domain(leaf_lo, leaf_hi, n_leaves, dom_min, &dom_inv);
    const int LF = L * F;
    int64_t n_acc = 0;
    double tot = 0;
    std::vector<float> pts(3 * n_points);
    std::vector<double> h, nxt;
    for (int64_t r = 0; r < n; ++r) {
        if (!accepted[r]) continue;
        ++n_acc;
        orc_segment_points(rays + 8 * r, t0[r], t1[r], n_points, xi + r * n_points, dom_min, dom_inv, pts.data());
        h.assign(n_points * LF, 0.0);
        for (int p = 0; p < n_points; ++p)
            for (int l = 0; l < L; ++l) {
                const int32_t N = res[l];
                int32_t c[3];
                float f[3];
                for (int k = 0; k < 3; ++k) {
                    float s = pts[3 * p + k] * (float)N;
                    int32_t ci = (int32_t)std::floor(s);
                    if (ci > N - 1) ci = N - 1;
                    if (ci < 0) ci = 0;
                    c[k] = ci;
                    f[k] = s - (float)ci;
                }
                for (int corner = 0; corner < 8; ++corner) {
                    int d0 = corner & 1, d1 = (corner >> 1) & 1, d2 = (corner >> 2) & 1;
                    uint32_t ix = orc_corner_index(N, dense[l], log2_T, c[0] + d0, c[1] + d1, c[2] + d2);
                    double w = (d0 ? (double)f[0] : 1.0 - (double)f[0]) * (d1 ? (double)f[1] : 1.0 - (double)f[1]) *
                               (d2 ? (double)f[2] : 1.0 - (double)f[2]);
                    for (int j = 0; j < F; ++j) h[p * LF + l * F + j] += w * table[(offset[l] + ix) * F + j];
                }
            }
        int64_t wo = 0, bo = 0;
        for (int k = 0; k < n_layers; ++k) {
            nxt.assign(dims[k + 1], 0.0);
            for (int o = 0; o < dims[k + 1]; ++o) {
                double s = b_all[bo + o];
                for (int i = 0; i < dims[k]; ++i) s += W_all[wo + (int64_t)o * dims[k] + i] * h[i];
                nxt[o] = (k + 1 < n_layers) ? (s > 0 ? s : 0) : s;
            }
            wo += (int64_t)dims[k] * dims[k + 1];
            bo += dims[k + 1];
            h.swap(nxt);
        }
        tot += sample_loss_impl(h.data(), gt + 9 * r, nullptr, nullptr, den ? den + 3 * r : nullptr, den_mode);
    }
    return n_acc ? tot / (double)n_acc : 0.0;
}

// ------------------------------------------------------------------ backward from given (x, dL/dz)
// The training backward (T6 MLP reverse mode, T7 hash-grid scatter) of m
// samples from GIVEN features x[m][D] and output gradients dz[m][8] -- e.g. the GPU's own
// fp16 features and fp32 dL/dz -- so each stage of the GPU's chain can be compared with
// the oracle element by element.  Sample s is the segment [t0[s], t1[s]] of ray rays[s]
// with jitter xi[s] (points and corners as in orc_segment_points / encode_point).
// Outputs (sums over the samples, not means): g_table, g_W, g_b; their magnitude sums
// (the same recursion on absolute values, masks unchanged) g_*_abs; the forward z[m][8]
// (double MLP on the given x) and its magnitude z_abs (|W| |h| + |b| per layer); per
// sample the ReLU margin min over hidden units |h_pre| / (|W| |h_in| + |b|) -- how close
// a ReLU decision is to its threshold relative to the operand magnitudes; and (nullable)
// hidden-layer deltas [m][n_layers-1][64] with magnitudes.
void orc_train_backward_given(int32_t L, int32_t F, int32_t log2_T, int32_t n_points, int32_t n_layers,
                              const int32_t* res, const int32_t* dense, const int64_t* offset,
                              const uint16_t* table, int64_t n_entries, const int32_t* dims,
                              const uint16_t* W_all, const float* b_all, const float* dom_box, int64_t m,
                              const float* rays, const float* t0, const float* t1, const float* xi,
                              const double* x_in, const double* dz_in, const uint8_t* masks /*nullable*/,
                              double* g_table, double* g_W, double* g_b,
                              double* g_table_abs, double* g_W_abs, double* g_b_abs,
                              double* z_out, double* z_abs, double* relu_margin,
                              int32_t* mask_flips /*nullable [m]*/, double* flip_margin /*nullable [m]*/,
                              double* hidden_delta /*nullable*/, double* hidden_delta_abs /*nullable*/) {
    float dom_min[3], dom_inv;
    orc_domain(dom_box, dom_box + 3, 1, dom_min, &dom_inv);
    OrcModel M{L, F, log2_T, n_points, n_layers, res, dense, offset, table, dims, W_all, b_all, dom_min, dom_inv};
    std::vector<const uint16_t*> W;
    std::vector<const float*> b;
    split_layers(n_layers, dims, W_all, b_all, W, b);
    int64_t nW = 0, nb = 0;
    for (int k = 0; k < n_layers; ++k) { nW += (int64_t)dims[k] * dims[k + 1]; nb += dims[k + 1]; }
    std::fill(g_table, g_table + n_entries * F, 0.0);
    std::fill(g_table_abs, g_table_abs + n_entries * F, 0.0);
    std::fill(g_W, g_W + nW, 0.0);
    std::fill(g_W_abs, g_W_abs + nW, 0.0);
    std::fill(g_b, g_b + nb, 0.0);
    std::fill(g_b_abs, g_b_abs + nb, 0.0);
    const int D = dims[0], n_out = dims[n_layers], H = n_layers - 1;
    std::vector<float> pts(3 * n_points);
    std::vector<uint32_t> idx(n_points * L * 8);
    std::vector<double> feat(L * F);
    std::vector<std::vector<double>> acts(n_layers + 1), mags(n_layers + 1);
    std::vector<double> habs, nabs;
    for (int64_t s = 0; s < m; ++s) {
        orc_segment_points(rays + 8 * s, t0[s], t1[s], n_points, xi + s * n_points, dom_min, dom_inv, pts.data());
        for (int p = 0; p < n_points; ++p)
            encode_point(L, F, log2_T, res, dense, offset, table, &pts[3 * p], feat.data(), idx.data() + p * L * 8);
        const double* x = x_in + s * D;
        const uint8_t* mk = masks ? masks + s * H * 64 : nullptr;
        // forward in double on the given x: pre = b + W h (same order as mlp_forward_one);
        // hidden output = ReLU(pre), or, with given masks, pre where the mask is on, else 0;
        // magnitudes |W| |h| + |b| alongside; ReLU margin = min |pre| / magnitude
        double marg = std::numeric_limits<double>::infinity(), fmarg = 0.0;
        int32_t flips = 0;
        acts[0].assign(x, x + D);
        habs.assign(x, x + D);
        for (double& v : habs) v = std::fabs(v);
        for (int k = 0; k < n_layers; ++k) {
            mags[k] = habs;
            acts[k + 1].assign(dims[k + 1], 0.0);
            nabs.assign(dims[k + 1], 0.0);
            for (int o = 0; o < dims[k + 1]; ++o) {
                double sv = (double)b[k][o], sa = std::fabs((double)b[k][o]);
                for (int i = 0; i < dims[k]; ++i) {
                    const double w = orc_half_to_double(W[k][(int64_t)o * dims[k] + i]);
                    sv += w * acts[k][i];
                    sa += std::fabs(w) * habs[i];
                }
                if (k + 1 < n_layers) {
                    const double rm = sa > 0.0 ? std::fabs(sv) / sa : std::numeric_limits<double>::infinity();
                    marg = std::min(marg, rm);
                    const bool own = sv > 0.0;
                    const bool on = mk ? mk[k * 64 + o] != 0 : own;
                    if (on != own) { ++flips; fmarg = std::max(fmarg, rm); }
                    acts[k + 1][o] = on ? sv : 0.0;
                    nabs[o] = on ? sa : 0.0;
                } else {
                    acts[k + 1][o] = sv;
                    nabs[o] = sa;
                }
            }
            habs.swap(nabs);
        }
        for (int o = 0; o < n_out; ++o) {
            z_out[s * n_out + o] = acts[n_layers][o];
            z_abs[s * n_out + o] = habs[o];
        }
        relu_margin[s] = marg;
        if (mask_flips) mask_flips[s] = flips;
        if (flip_margin) flip_margin[s] = fmarg;
        std::vector<uint8_t> own_mask;
        if (!mk) {                                   // masks of the double forward itself
            own_mask.assign(H * 64, 0);
            for (int k = 0; k < H; ++k)
                for (int o = 0; o < dims[k + 1]; ++o) own_mask[k * 64 + o] = acts[k + 1][o] > 0.0;
            mk = own_mask.data();
        }
        std::vector<double> delta(dz_in + s * n_out, dz_in + (s + 1) * n_out);
        backward_sample(M, W, acts.data(), delta, pts.data(), idx.data(), nW, nb, g_table, g_W, g_b, false,
                        hidden_delta ? hidden_delta + s * H * 64 : nullptr, mk);
        backward_sample(M, W, acts.data(), delta, pts.data(), idx.data(), nW, nb, g_table_abs, g_W_abs, g_b_abs,
                        true, hidden_delta_abs ? hidden_delta_abs + s * H * 64 : nullptr, mk, mags.data());
    }
}

// ------------------------------------------------------------------ cut expansion (NEXT-1)
// P:180 ("Base-BVH cut optimization"): "we then expand the cut by splitting the nodes with
// largest error, replacing each with its two children"; P:185 ("Node error"): rank
// r = 2 log q + log p.  One expansion step of n_splits splits over the cut leaf_base[n]
// (base-BVH node ids; base BVH given by child_a / child_b, leaf iff child_b < 0):
// leaves in decreasing r (ties: lower leaf index first, C38); a base-BVH leaf cannot be
// split and is passed over; stop after n_splits splits or when the leaves run out.
// q, p > 0 (zero statistics are a caller's reading: C38).  out_nodes receives the new cut's
// nodes in increasing node id; returns their count.
int32_t orc_expand_cut(const int32_t* child_a, const int32_t* child_b, int32_t n_leaves, const int32_t* leaf_base,
                       const double* q, const double* p, int32_t n_splits, int32_t* out_nodes) {
    std::vector<double> r(n_leaves);
    for (int32_t i = 0; i < n_leaves; ++i) r[i] = 2.0 * std::log(q[i]) + std::log(p[i]);
    std::vector<int32_t> order(n_leaves);
    for (int32_t i = 0; i < n_leaves; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return r[a] > r[b]; });
    std::vector<int32_t> nodes;
    std::vector<char> split(n_leaves, 0);
    int32_t done = 0;
    for (int32_t k = 0; k < n_leaves && done < n_splits; ++k) {
        const int32_t nd = leaf_base[order[k]];
        if (child_b[nd] < 0) continue;                     // a base-BVH leaf: nothing to split
        split[order[k]] = 1;
        ++done;
    }
    for (int32_t i = 0; i < n_leaves; ++i) {
        const int32_t nd = leaf_base[i];
        if (split[i]) {
            nodes.push_back(child_a[nd]);
            nodes.push_back(child_b[nd]);
        } else {
            nodes.push_back(nd);
        }
    }
    std::sort(nodes.begin(), nodes.end());
    std::copy(nodes.begin(), nodes.end(), out_nodes);
    return (int32_t)nodes.size();
}

// ------------------------------------------------------------------ Adam
// "Adam optimizer [kingma2014adam] with default hyper-parameters and a learning
// rate of 0.01" (C20: beta1 0.9, beta2 0.999, eps 1e-8, bias-corrected, dense).
// step is the 1-based step number of this update.
void orc_adam(double* param, const double* grad, double* m, double* v, int64_t n, int64_t step,
              double lr, double beta1, double beta2, double eps) {
    const double c1 = 1.0 - std::pow(beta1, (double)step), c2 = 1.0 - std::pow(beta2, (double)step);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * grad[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * grad[i] * grad[i];
        double mh = m[i] / c1, vh = v[i] / c2;
        param[i] -= lr * mh / (std::sqrt(vh) + eps);
    }
}

int32_t orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

// Thread count for the following oracle calls (bench.py's 1-thread baseline figure).
void orc_set_num_threads(int32_t n) {
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

}  // extern "C"

// ------------------------------------------------------------------ T0 training rays (C28')
// Philox-4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
// SC'11): 10 rounds of (hi, lo) = M * c on words 0 and 2 with the key added by xor, the key
// bumped by the Weyl constants between rounds.  Pinned by the published known-answer vectors.
extern "C" void orc_philox4x32_10(const uint32_t* ctr_in, const uint32_t* key_in, uint32_t* out) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k[2] = {key_in[0], key_in[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n[4] = {hi1 ^ c[1] ^ k[0], lo1, hi0 ^ c[3] ^ k[1], lo0};
        for (int j = 0; j < 4; ++j) c[j] = n[j];
    }
    for (int j = 0; j < 4; ++j) out[j] = c[j];
}

// The training-ray recipe of DESIGN.md C28' (the device generator nbvh_gen_train_rays follows
// the same recipe; the two share no code): ray i of step s draws Philox(i, d, s_lo, s_hi; seed)
// for d = 0 (origin xyz, acceptance u), 1 (direction), 2 (jitter); U = (x >> 8) * 2^-24;
// origin = lo + (hi - lo) U; z = 1 - 2U, r = sqrt(max(0, 1 - z^2)), phi = 2 pi U,
// d = (r cos phi, r sin phi, z); tmin 0, tmax inf.  cos / sin are not correctly rounded on
// either side, so the GPU's direction x, y agree to a few ulp (everything else bit-exact).
extern "C" void orc_gen_train_rays(uint64_t seed, uint64_t step, int64_t i0, int64_t n, const float* box,
                                   int32_t n_points, float* rays, float* u, float* xi) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    auto U = [](uint32_t x) { return (float)(x >> 8) * 5.9604644775390625e-8f; };
    for (int64_t j = 0; j < n; ++j) {
        const uint32_t i = (uint32_t)(i0 + j);
        uint32_t p0[4], p1[4], p2[4];
        const uint32_t c0[4] = {i, 0u, (uint32_t)step, (uint32_t)(step >> 32)};
        const uint32_t c1[4] = {i, 1u, (uint32_t)step, (uint32_t)(step >> 32)};
        const uint32_t c2[4] = {i, 2u, (uint32_t)step, (uint32_t)(step >> 32)};
        orc_philox4x32_10(c0, key, p0);
        orc_philox4x32_10(c1, key, p1);
        orc_philox4x32_10(c2, key, p2);
        float* r = rays + 8 * j;
        for (int k = 0; k < 3; ++k) r[k] = box[k] + (box[3 + k] - box[k]) * U(p0[k]);
        r[3] = 0.0f;
        const float z = 1.0f - 2.0f * U(p1[0]);
        const float rr = std::sqrt(std::fmax(0.0f, 1.0f - z * z));
        const float phi = 6.28318530717958647692f * U(p1[1]);
        r[4] = rr * std::cos(phi);
        r[5] = rr * std::sin(phi);
        r[6] = z;
        r[7] = std::numeric_limits<float>::infinity();
        u[j] = U(p0[3]);
        for (int k = 0; k < n_points; ++k) xi[j * n_points + k] = U(p2[k]);
    }
}
