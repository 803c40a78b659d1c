// nbvh_kernels.cu — the N-BVH neural ray-query hot path on sm_100a.
//
//   k_traverse    Q0+Q1: load rays, traverse the shallow N-BVH of the chosen cut, write each
//                 ray's (t_enter, id)-ordered leaf list (capacity K) and append the ray
//                 (32-byte work record) to the long- or short-ray work list.
//   k_query_warp  Q2-Q7, one persistent launch per frame (the default): every warp owns 16
//                 ray slots and loops -- refill, sample, encode, MLP on mma.sync, decode.
//   k_query_ws    the same steps warp-specialised (NBVH_QUERY_MLP=tc): 16 worker warps own
//                 two sets of 16 ray slots each and loop -- refill empty slots from the work
//                 lists, sample the current leaf segment, hash-grid encode into a 16-row
//                 block of a 128-row feature tile, decode, update the best hit, decide
//                 front-to-back termination, write finished rays' hit records -- while one
//                 MLP warpgroup runs the decoder MLP of full tiles on tcgen05 (TMEM
//                 accumulators, weights read by the tensor core from shared memory).
//   k_debug_*     the same device functions with intermediate results exposed.
//
// Paper passages: P:103 (front-to-back probing, early termination)
// (segment sampling, feature concatenation, MLP decode), P:161 (queries per ray =
// leaves met before a hit), P:201/P:237/P:243 (visibility threshold, local distance,
// normal, albedo).  Readings C1-C36: DESIGN.md §3.
#include <cuda_runtime.h>

#include <cstdlib>

#include "nbvh_device.cuh"
#include "nbvh_launch.h"
#include "nbvh_tcgen05.cuh"

namespace nbvh {

// ------------------------------------------------------------------ traversal
// Q1 traversal of one ray with the ordered list held in shared memory (column layout
// [3][cap][blockDim]: t_enter, t_exit, leaf id), so inserting a leaf is a short shift loop
// instead of a K-wide predicated compare-swap in registers.  Leaves arrive roughly in
// front-to-back order (nearer child first), so the shift is usually empty.  Same result as
// collect_leaves<K>(..., prune = true): the `cap` smallest (t_enter, id) keys, sorted;
// `more` reports whether further intersected leaves may exist (C6).
__device__ __forceinline__ int traverse_smem_list(const CutDev& cut, const RayDev& R, int cap, float* lte, float* ltx,
                                                  int* lid, int S, SmemStack& stack, bool& more, int* err) {
    int n = 0;
    bool dropped = false;
    float last_te = 0.f;                         // key of entry cap-1 once the list is full
    int last_id = 0;
    auto consider = [&](int leaf, float te, float tx) {
        int pos;
        if (n == cap) {
            if (!key_less(te, leaf, last_te, last_id)) {
                dropped = true;
                return;
            }
            dropped = true;                      // the current last entry falls off
            pos = cap - 1;
        } else {
            pos = n++;
        }
        while (pos > 0) {
            const float pte = lte[(pos - 1) * S];
            const int pid = lid[(pos - 1) * S];
            if (!key_less(te, leaf, pte, pid)) break;
            lte[pos * S] = pte;
            ltx[pos * S] = ltx[(pos - 1) * S];
            lid[pos * S] = pid;
            --pos;
        }
        lte[pos * S] = te;
        ltx[pos * S] = tx;
        lid[pos * S] = leaf;
        if (n == cap) {
            last_te = lte[(cap - 1) * S];
            last_id = lid[(cap - 1) * S];
        }
    };
    if (cut.n_leaves == 1) {
        float4 a = __ldg(cut.leaf_box), b = __ldg(cut.leaf_box + 1);
        float lo[3] = {a.x, a.y, a.z}, hi[3] = {b.x, b.y, b.z}, te, tx;
        if (slab(R, lo, hi, te, tx)) consider(0, te, tx);
    } else {
        // the node to visit next lives in a register; only the farther child of a node with
        // two wanted children is pushed (same visiting order as push-both-then-pop)
        stack.sp = 0;
        int node = 0;
        while (true) {
            const float4* p = reinterpret_cast<const float4*>(cut.inner + node);
            float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3);
            float llo[3] = {q0.x, q0.y, q0.z}, lhi[3] = {q0.w, q1.x, q1.y};
            float rlo[3] = {q1.z, q1.w, q2.x}, rhi[3] = {q2.y, q2.z, q2.w};
            int cl = __float_as_int(q3.x), cr = __float_as_int(q3.y);
            float lte_, ltx_, rte_, rtx_;
            bool hl = slab(R, llo, lhi, lte_, ltx_);
            bool hr = slab(R, rlo, rhi, rte_, rtx_);
            if (hl && cl < 0) consider(-1 - cl, lte_, ltx_);
            if (hr && cr < 0) consider(-1 - cr, rte_, rtx_);
            bool pl = hl && cl >= 0, pr = hr && cr >= 0;
            if (n == cap) {                       // subtrees entering after the cap-th key
                if (pl && lte_ > last_te) { pl = false; dropped = true; }
                if (pr && rte_ > last_te) { pr = false; dropped = true; }
            }
            if (pl && pr) {
                if (stack.sp + 1 > stack.cap) { atomicOr(err, 1); break; }
                const bool l_first = lte_ <= rte_;
                stack.push(l_first ? cr : cl);
                node = l_first ? cl : cr;
            } else if (pl) {
                node = cl;
            } else if (pr) {
                node = cr;
            } else {
                if (stack.sp == 0) break;
                node = stack.pop();
            }
        }
    }
    more = dropped;
    return n;
}

// Packet variant for coherent rays (e.g. primary camera rays, 32 neighbouring pixels per
// warp): the warp walks ONE shared node stack; every lane tests both children against its
// own ray, inserts the leaves it hits into its own list and votes for the subtrees it still
// needs (a subtree is skipped only when no lane needs it).  Node loads become one broadcast
// per warp and the loop is divergence-free.  Child boxes lie inside their parent's (exact
// unions, monotone rounding), so a lane that misses a node misses its whole subtree, and a
// lane that pruned a subtree rejects its leaves in `consider` with the same `dropped`
// effect: every lane's list and `more` flag equal the per-thread traversal's.
__device__ __forceinline__ int traverse_packet(const CutDev& cut, const RayDev& R, bool valid, int cap, float* lte,
                                               float* ltx, int* lid, int S, int* wstack, int stack_cap, bool& more,
                                               int* err) {
    int n = 0;
    bool dropped = false;
    auto consider = [&](int leaf, float te, float tx) {
        int pos;
        if (n == cap) {
            if (!key_less(te, leaf, lte[(cap - 1) * S], lid[(cap - 1) * S])) {
                dropped = true;
                return;
            }
            dropped = true;
            pos = cap - 1;
        } else {
            pos = n++;
        }
        while (pos > 0) {
            const float pte = lte[(pos - 1) * S];
            const int pid = lid[(pos - 1) * S];
            if (!key_less(te, leaf, pte, pid)) break;
            lte[pos * S] = pte;
            ltx[pos * S] = ltx[(pos - 1) * S];
            lid[pos * S] = pid;
            --pos;
        }
        lte[pos * S] = te;
        ltx[pos * S] = tx;
        lid[pos * S] = leaf;
    };
    const int lane = threadIdx.x & 31;
    if (cut.n_leaves == 1) {
        float4 a = __ldg(cut.leaf_box), b = __ldg(cut.leaf_box + 1);
        float lo[3] = {a.x, a.y, a.z}, hi[3] = {b.x, b.y, b.z}, te, tx;
        if (valid && slab(R, lo, hi, te, tx)) consider(0, te, tx);
    } else {
        int sp = 1;                                     // warp-uniform
        if (lane == 0) wstack[0] = 0;
        __syncwarp();
        while (sp > 0) {
            const int node = wstack[--sp];
            __syncwarp();                               // everyone read the top before it is reused
            const float4* p = reinterpret_cast<const float4*>(cut.inner + node);
            const float4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2), q3 = __ldg(p + 3);
            const float llo[3] = {q0.x, q0.y, q0.z}, lhi[3] = {q0.w, q1.x, q1.y};
            const float rlo[3] = {q1.z, q1.w, q2.x}, rhi[3] = {q2.y, q2.z, q2.w};
            const int cl = __float_as_int(q3.x), cr = __float_as_int(q3.y);
            float lte_ = 0.f, ltx_ = 0.f, rte_ = 0.f, rtx_ = 0.f;
            bool hl = false, hr = false;
            if (valid) {
                hl = slab(R, llo, lhi, lte_, ltx_);
                hr = slab(R, rlo, rhi, rte_, rtx_);
                if (hl && cl < 0) consider(-1 - cl, lte_, ltx_);
                if (hr && cr < 0) consider(-1 - cr, rte_, rtx_);
            }
            bool pl = hl && cl >= 0, pr = hr && cr >= 0;
            if (n == cap) {                             // this lane's subtrees entering after its cap-th key
                const float last = lte[(cap - 1) * S];
                if (pl && lte_ > last) { pl = false; dropped = true; }
                if (pr && rte_ > last) { pr = false; dropped = true; }
            }
            const unsigned vl = __ballot_sync(0xffffffffu, pl), vr = __ballot_sync(0xffffffffu, pr);
            if (sp + 2 > stack_cap) {
                if (lane == 0) atomicOr(err, 1);
                break;
            }
            if (vl && vr) {
                // nearer child first for most lanes that want both
                const unsigned both = __ballot_sync(0xffffffffu, pl && pr);
                const unsigned lfirst = __ballot_sync(0xffffffffu, pl && pr && lte_ <= rte_);
                const bool l_first = 2 * __popc(lfirst) >= __popc(both);
                if (lane == 0) {
                    wstack[sp] = l_first ? cr : cl;
                    wstack[sp + 1] = l_first ? cl : cr;
                }
                sp += 2;
            } else if (vl || vr) {
                if (lane == 0) wstack[sp] = vl ? cl : cr;
                sp += 1;
            }
            __syncwarp();
        }
    }
    more = dropped;
    return n;
}

// One thread per ray: traversal stack and ordered list in shared memory (stack rows =
// cut depth + 2, list rows = 3 * cap).
template <bool kPacket>
__global__ void __launch_bounds__(128, 8) k_traverse(TraverseArgs a) {
    extern __shared__ int sm_raw[];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = r < a.n_rays;
    bool active = false;
    const int S = blockDim.x;
    float* lte = reinterpret_cast<float*>(sm_raw) + threadIdx.x;
    float* ltx = lte + a.cap * S;
    int* lid = sm_raw + 2 * a.cap * S + threadIdx.x;
    bool more_long = false, more = false;
    int n = 0;
    RayDev R;
    if (valid) {   // the ray is read once: evict-first, so the hierarchy's lines stay in L1
        const float4 ra = __ldcs(a.rays + 2 * r), rb = __ldcs(a.rays + 2 * r + 1);
        R.o[0] = ra.x; R.o[1] = ra.y; R.o[2] = ra.z; R.tmin = ra.w;
        R.d[0] = rb.x; R.d[1] = rb.y; R.d[2] = rb.z; R.tmax = rb.w;
#pragma unroll
        for (int k = 0; k < 3; ++k) R.inv[k] = __fdiv_rn(1.0f, R.d[k]);
    }
    if constexpr (kPacket) {      // every lane of the warp walks the shared stack
        int* wstack = sm_raw + 3 * a.cap * S + (threadIdx.x >> 5) * (a.cut.depth + 2);
        n = traverse_packet(a.cut, R, valid, a.cap, lte, ltx, lid, S, wstack, a.cut.depth + 2, more, &a.ctr->err);
    }
    if (valid) {
        if constexpr (!kPacket) {
            SmemStack st{sm_raw + 3 * a.cap * S + threadIdx.x, S, a.cut.depth + 2};
            n = traverse_smem_list(a.cut, R, a.cap, lte, ltx, lid, S, st, more, &a.ctr->err);
        }
        NBVH_DCHECK(n >= 0 && n <= a.cap && a.cap <= kListK);
        more_long = more || n >= 3;
        // entry 0 travels in the work record; the list keeps it only where a refill will read
        // it back (C6: the refill resumes after the last entry of a one-entry list)
        for (int j = (n == 1 && more) ? 0 : 1; j < n; ++j) {
            a.lst[(int64_t)j * a.n_rays + r] = make_float4(lte[j * S], ltx[j * S], __int_as_float(lid[j * S]), 0.f);
        }
        active = n > 0;
        if (!active) {
            // no intersected leaf: final miss record (visibility 1 = no intersection)
            a.out.hit[r] = 0;
            a.out.t[r] = __int_as_float(0x7f800000);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                a.out.normal[3 * r + k] = 0.f;
                a.out.albedo[3 * r + k] = 0.f;
            }
            if (a.out.leaf) a.out.leaf[r] = -1;
            if (a.out.n_queries) a.out.n_queries[r] = 0;
        }
    }
    // warp-aggregated append to the work lists of the query kernel: rays whose list is long
    // (or overflows) go to the "long" list, which the query kernel consumes first, so the
    // kernel's tail is made of short rays (longest-job-first)
    const bool is_long = active && (more_long);
    const unsigned ml = __ballot_sync(0xffffffffu, is_long);
    const unsigned ms = __ballot_sync(0xffffffffu, active && !is_long);
    const int lane = threadIdx.x & 31;
    int bl = 0, bs = 0;
    if (lane == 0 && ml) bl = atomicAdd(&a.ctr->cnt_long, __popc(ml));
    if (lane == 0 && ms) bs = atomicAdd(&a.ctr->cnt, __popc(ms));
    bl = __shfl_sync(0xffffffffu, bl, 0);
    bs = __shfl_sync(0xffffffffu, bs, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (active) {
        WorkRec w;
        w.o = make_float4(R.o[0], R.o[1], R.o[2], __int_as_float((int)r));
        w.d = make_float4(R.d[0], R.d[1], R.d[2], __int_as_float(n | (more ? 1 << 16 : 0)));
        w.e0 = make_float4(lte[0], ltx[0], __int_as_float(lid[0]), 0.f);   // list entry 0
        if (is_long) a.act_long[bl + __popc(ml & lt)] = w;
        else a.act_out[bs + __popc(ms & lt)] = w;
    }
}

// Debug traversal: full lists up to `cap` (may exceed K) by repeated resumption.
__global__ void __launch_bounds__(128) k_debug_traverse(DebugTraverseArgs a) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.n_rays) return;
    RayDev R = load_ray(a.rays, r);
    float lte[kListK], ltx[kListK];
    int lid[kListK];
    int written = 0, n = 0;
    bool has_after = false;
    float after_te = 0.f;
    int after_id = 0;
    int total = -1;
    while (true) {
        int rem = collect_leaves<kListK>(a.cut, R, has_after, after_te, after_id, a.k, lte, ltx, lid, n, a.err);
        if (total < 0) total = rem;
#pragma unroll
        for (int j = 0; j < kListK; ++j)
            if (j < n && written + j < a.cap) {
                a.leaf[r * a.cap + written + j] = lid[j];
                a.te[r * a.cap + written + j] = lte[j];
                a.tx[r * a.cap + written + j] = ltx[j];
            }
        if (n == 0) break;
#pragma unroll
        for (int j = 0; j < kListK; ++j)
            if (j == n - 1) { after_te = lte[j]; after_id = lid[j]; }
        written += n;
        has_after = true;
        if (written >= a.cap || rem <= n) break;
    }
    for (int j = written; j < a.cap; ++j) {
        a.leaf[r * a.cap + j] = -1;
        a.te[r * a.cap + j] = 0.f;
        a.tx[r * a.cap + j] = 0.f;
    }
    a.count[r] = total;
}

// ------------------------------------------------------------------ persistent fused query
// Rare path, kept out of line so the query kernel's register allocation is not sized for a
// second traversal: refill ray r's list with the leaves after its last key (C6).
__device__ __noinline__ int refill_list(CutDev cut, const float4* rays, int64_t n_rays, int cap, float4* lst,
                                        QueryCounters* ctr, int r, int nbuf, float t_bound, int* more_out) {
    const int64_t last = (int64_t)(nbuf - 1) * n_rays + r;
    const float4 ke = lst[last];
    const float kte = ke.x;
    const int kid = __float_as_int(ke.z);
    RayDev R = load_ray(rays, r);
    float lte[kListK], ltx[kListK];
    int lid[kListK], n = 0;
    bool more = false;
    collect_leaves<kListK>(cut, R, true, kte, kid, cap, lte, ltx, lid, n, &ctr->err, true, &more, t_bound);
#pragma unroll
    for (int j = 0; j < kListK; ++j)
        if (j < n) {
            lst[(int64_t)j * n_rays + r] = make_float4(lte[j], ltx[j], __int_as_float(lid[j]), 0.f);
        }
    *more_out = more ? 1 : 0;
    atomicAdd(&ctr->refills, 1);
    return n;
}

// The per-warp decoder MLP of k_query, and of nbvh_debug_mlp (which must run exactly the
// product's function).  fp32 accumulation (mlp_rows16): the raw z stays within the 1e-2
// tier of north_star against the double oracle.  The fp16-accumulating variant
// (mlp_rows16h, C34) was 1.4% faster in round 1 but its error grows with the layer width
// (K fp16 roundings per accumulator); kept for A/B only.
constexpr bool kQueryMlpF16Acc = false;
template <int D, bool kBf = false>
__device__ __forceinline__ void query_mlp_rows16(const MlpSmem& s, int hidden, const __half* x, int r0, float* z,
                                                 int lane) {
    if constexpr (kQueryMlpF16Acc && !kBf) mlp_rows16h<D>(s, hidden, x, r0, z, lane);
    else mlp_rows16<D, kBf>(s, hidden, x, r0, z, lane);
}

// Ray slots of one warp (structure of arrays in shared memory).  Lane s < kWarpQ owns slot
// s for the refill and decode steps; the encode and MLP steps work on the compacted rows.
constexpr int kWarpQ = 16;          // queries per slot set (one m16 / one 16-row tile block)
constexpr int kQueryWarps = 16;     // warps per CTA (one CTA per SM; bounded by shared memory)
constexpr int kQueryWarpsTex = 24;  // ... with TEX gathers: 24 at 80 registers (6 per SM sub-partition,
                                    // the most the 196 KB shared-memory carveout step holds): 0.800 ms vs
                                    // 0.816 at 22, 0.836 at 20 (profiles/NOTES.md r2l)
__host__ __device__ constexpr int query_warps(bool tex) { return tex ? kQueryWarpsTex : kQueryWarps; }

struct WarpSlots {
    int32_t ray[kWarpQ], pos[kWarpQ], base[kWarpQ], nbuf[kWarpQ], more[kWarpQ], bleaf[kWarpQ], nq[kWarpQ],
        leaf[kWarpQ], act[kWarpQ], fresh[kWarpQ],   // fresh: the current entry is in the slot (entry 0
                                                    // from the work record, later ones from the decode)
        pend[kWarpQ];                               // the list ran out with leaves remaining (C6):
                                                    // refilled at the top of the next iteration
    float o[3][kWarpQ], d[3][kWarpQ];
    float bt[kWarpQ], bte[kWarpQ], te[kWarpQ], tx[kWarpQ];
    float nrm[3][kWarpQ], alb[3][kWarpQ];
    float4 nxt[kWarpQ];      // the next list entry, prefetched (cp.async) while the row is encoded
};

__host__ __device__ constexpr size_t align16(size_t b) { return (b + 15) & ~(size_t)15; }
__host__ __device__ constexpr size_t align128(size_t b) { return (b + 127) & ~(size_t)127; }

// Lanes below this one (a special register: nothing kept live across the query loop).
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ---- the steps of a slot set, shared by both query kernels (Q2-Q7)

// (A) refill the set's empty slots with the next rays of the global work list (one atomic per
// warp; long rays first).  `exhausted` (shared, per warp) is set once the list is drained.
__device__ __forceinline__ void slots_refill(const QueryArgs& a, WarpSlots& S, int lane, int total, int n_long,
                                             int* exhausted) {
    const bool empty = lane < kWarpQ && S.ray[lane] < 0;
    const unsigned em = __ballot_sync(0xffffffffu, empty);
    if (em && !*exhausted) {
        const int ne = __popc(em);
        int base = 0;
        if (lane == 0) base = atomicAdd(a.next, ne);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (lane == 0) *exhausted = base + ne >= total;
        const int i = base + __popc(em & lanemask_lt());
        if (empty && i < total) {
            const WorkRec* wr = i < n_long ? a.act_long + i : a.act + (i - n_long);
            // read-once streams (work records, lists) are loaded evict-first so they do not
            // push the hash-table lines out of L1
            const float4 w0 = __ldcs(&wr->o), w1 = __ldcs(&wr->d), w2 = __ldcs(&wr->e0);
            const int r = __float_as_int(w0.w), st = __float_as_int(w1.w);
            S.te[lane] = w2.x;
            S.tx[lane] = w2.y;
            S.leaf[lane] = __float_as_int(w2.z);
            S.fresh[lane] = 1;
            NBVH_DCHECK(r >= 0 && r < a.n_rays && (st & 0xffff) >= 1 && (st & 0xffff) <= a.cap);
            S.ray[lane] = r;
            S.o[0][lane] = w0.x; S.o[1][lane] = w0.y; S.o[2][lane] = w0.z;
            S.d[0][lane] = w1.x; S.d[1][lane] = w1.y; S.d[2][lane] = w1.z;
            S.pos[lane] = 0;
            S.base[lane] = 0;
            S.nbuf[lane] = st & 0xffff;
            S.more[lane] = st >> 16;
            S.bt[lane] = __int_as_float(0x7f800000);
            S.bte[lane] = 0.f;
            S.bleaf[lane] = -1;
            S.nq[lane] = 0;
            S.pend[lane] = 0;
        }
    }
    __syncwarp();
}

// Q7: slot s's ray r is finished -- its hit record (a miss keeps t = +inf and zero
// vectors) and the slot freed.
__device__ __forceinline__ void slot_finish(const QueryArgs& a, WarpSlots& S, int s, int r) {
    const int bleaf = S.bleaf[s];
    const bool h = bleaf >= 0;
    a.out.hit[r] = h ? 1 : 0;
    a.out.t[r] = h ? S.bt[s] : __int_as_float(0x7f800000);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a.out.normal[3 * (int64_t)r + k] = h ? S.nrm[k][s] : 0.f;
        a.out.albedo[3 * (int64_t)r + k] = h ? S.alb[k][s] : 0.f;
    }
    if (a.out.leaf) a.out.leaf[r] = bleaf;
    if (a.out.n_queries) a.out.n_queries[r] = S.nq[s];
    S.ray[s] = -1;
}

// (A0) the slots whose list ran out with leaves remaining (marked by the decode) resume after
// their last key, bounded by the best hit (C6).  The traversal is an out-of-line call; made
// from here, where only the loop's invariants are live, instead of from inside the decode,
// it no longer makes every decode save and reload its live values around the call site.
__device__ __forceinline__ void slots_list_refill(const QueryArgs& a, WarpSlots& S, int lane) {
    const bool pend = lane < kWarpQ && S.ray[lane] >= 0 && S.pend[lane];
    if (__ballot_sync(0xffffffffu, pend) == 0u) return;   // warp-uniform: rare
    if (pend) {
        S.pend[lane] = 0;
        const int r = S.ray[lane];
        const int bleaf = S.bleaf[lane];
        const float bt = S.bt[lane];
        int more = 0;
        const int nbuf = refill_list(a.cut, a.rays, a.n_rays, a.cap, a.lst, a.ctr, r, S.nbuf[lane],
                                     bleaf >= 0 ? bt : __int_as_float(0x7f800000), &more);
        S.base[lane] = S.pos[lane];
        S.nbuf[lane] = nbuf;
        S.more[lane] = more;
        bool done = nbuf == 0;
        if (!done) {
            const float4 e = __ldcs(a.lst + r);                   // the new list's first entry
            done = bleaf >= 0 && e.x > bt;                         // front-to-back termination
            if (!done) {
                S.te[lane] = e.x;
                S.tx[lane] = e.y;
                S.leaf[lane] = __float_as_int(e.z);
                S.fresh[lane] = 1;
            }
        }
        if (done) slot_finish(a, S, lane, r);
    }
    __syncwarp();
}

// (B) compact the occupied slots into rows 0..nv-1 (S.act[row] = slot) and (C) fetch each
// ray's current leaf segment and its n stratified sample points (C8) into
// xs [NP*3][kWarpQ].  Returns nv (warp-uniform).
template <bool kXs = true>
__device__ __forceinline__ int slots_segment(const QueryArgs& a, WarpSlots& S, float* xs, int lane, int NP,
                                             const float* u_tab) {
    const bool occ = lane < kWarpQ && S.ray[lane] >= 0;
    const unsigned om = __ballot_sync(0xffffffffu, occ);
    const int nv = __popc(om);
    if (occ) {
        const int row = __popc(om & lanemask_lt());
        S.act[row] = lane;
        const int r = S.ray[lane];
        NBVH_DCHECK(S.pos[lane] - S.base[lane] >= 0 && S.pos[lane] - S.base[lane] < S.nbuf[lane] &&
                    S.nbuf[lane] <= kListK);
        const int64_t li = (int64_t)(S.pos[lane] - S.base[lane]) * a.n_rays + r;
        float te, tx;
        if (S.fresh[lane]) {              // the entry is already in the slot (work record / decode)
            S.fresh[lane] = 0;
            te = S.te[lane];
            tx = S.tx[lane];
        } else {
            const float4 e = __ldcs(a.lst + li);
            te = e.x;
            tx = e.y;
            S.leaf[lane] = __float_as_int(e.z);
            S.te[lane] = te;
            S.tx[lane] = tx;
        }
        // the entry after this one, for the decode's termination test: fetched into the slot
        // asynchronously (no registers held across the encode and the MLP)
        if (S.pos[lane] + 1 - S.base[lane] < S.nbuf[lane])
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(&S.nxt[lane])),
                         "l"(a.lst + li + a.n_rays)
                         : "memory");
        if constexpr (kXs) {   // else the encode derives the points from the slot (row_point)
            const float o[3] = {S.o[0][lane], S.o[1][lane], S.o[2][lane]};
            const float d[3] = {S.d[0][lane], S.d[1][lane], S.d[2][lane]};
            for (int p = 0; p < NP; ++p) {
                float x[3];
                segment_point_u(a.g, o, d, te, tx, u_tab[p], x);   // u_p = (2p+1)/(2NP), per CTA
                xs[(p * 3 + 0) * kWarpQ + row] = x[0];
                xs[(p * 3 + 1) * kWarpQ + row] = x[1];
                xs[(p * 3 + 2) * kWarpQ + row] = x[2];
            }
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    __syncwarp();
    return nv;
}

// (D) hash-grid encode of the nv rows: lane -> row q = lane % 16; the two half-warps take
// sample points of opposite parity at the same levels (neighbouring points of the same rays:
// coherent lines).  Chunk c (8 halves) of row q is stored at dst + c * cstride + q * rstride.
// Without xs (kXs = false, k_query_warp) each lane derives its row's point from the slot.
__device__ __forceinline__ void row_point(const QueryArgs& a, const WarpSlots& S, const float* u_tab, int q, int p,
                                          float x[3]) {
    const int s = S.act[q];
    const float o[3] = {S.o[0][s], S.o[1][s], S.o[2][s]};
    const float d[3] = {S.d[0][s], S.d[1][s], S.d[2][s]};
    segment_point_u(a.g, o, d, S.te[s], S.tx[s], u_tab[p], x);   // the same op sequence as (C)
}

template <int F, bool kBf = false, bool kSpread = false, bool kTex = false, bool kXs = true>
__device__ __forceinline__ void rows_encode(const QueryArgs& a, const LevelSm* lv, const float* xs, int nv, int lane,
                                            int NP, unsigned char* dst, int cstride, int rstride,
                                            const WarpSlots* S = nullptr, const float* u_tab = nullptr) {
    const int cpp = (a.g.L * F) / 8;      // 16-byte chunks per sample point
    const uint32_t hmask = (1u << a.g.log2_T) - 1u;
    if (kSpread && nv <= kWarpQ / 2) {
        // few rows (a launch's tail, where a warp's iteration time is the latency of its
        // sequential chunk rounds): spread each row's NP * cpp chunks over 32 / rp lanes
        // (rp = rows rounded up to a power of two), so the rounds per lane shrink with the row
        // count.  Every chunk is computed exactly as below, only by another lane.
        const int rp = nv > 4 ? 8 : (nv > 2 ? 4 : (nv > 1 ? 2 : 1));
        const int lpr = 32 / rp, q = lane & (rp - 1), h = lane / rp;
        if (q < nv) {
            for (int j = h; j < NP * cpp; j += lpr) {
                const int p = j / cpp, lc = j - p * cpp;
                float x[3];
                if constexpr (kXs) {
                    const float* xp = xs + p * 3 * kWarpQ;
                    x[0] = xp[q];
                    x[1] = xp[kWarpQ + q];
                    x[2] = xp[2 * kWarpQ + q];
                } else {
                    row_point(a, *S, u_tab, q, p, x);
                }
                const uint4 f = encode_chunk_sm<F, true, kBf, kTex>(lv, a.g.table, hmask, x[0], x[1], x[2],
                                                                    lc * (8 / F), nullptr, a.g.tex);
                *reinterpret_cast<uint4*>(dst + j * cstride + q * rstride) = f;
            }
        }
        __syncwarp();
        return;
    }
    const int q = lane & (kWarpQ - 1), h = lane / kWarpQ;
    if (q < nv) {
        for (int p = h; p < NP; p += 2) {
            float x[3];
            if constexpr (kXs) {
                const float* xp = xs + p * 3 * kWarpQ;
                x[0] = xp[q];
                x[1] = xp[kWarpQ + q];
                x[2] = xp[2 * kWarpQ + q];
            } else {
                row_point(a, *S, u_tab, q, p, x);
            }
            const float x0 = x[0], x1 = x[1], x2 = x[2];
            for (int lc = 0; lc < cpp; ++lc) {
                const int c = p * cpp + lc;
                const uint4 f = encode_chunk_sm<F, true, kBf, kTex>(lv, a.g.table, hmask, x0, x1, x2, lc * (8 / F),
                                                                    nullptr, a.g.tex);
                *reinterpret_cast<uint4*>(dst + c * cstride + q * rstride) = f;
            }
        }
    }
    __syncwarp();
}

// (F) decode the nv rows' raw outputs z [row][8], update each ray's
// best hit, decide front-to-back termination (C5, C6) and write the finished
// rays' hit records (Q7).  Returns the number of queries decoded.
__device__ __forceinline__ void rows_decode(const QueryArgs& a, WarpSlots& S, const float* zt, int nv, int lane) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");   // this lane's prefetched next entries
    __syncwarp();
    if (lane < nv) {
        const int s = S.act[lane];
        const int r = S.ray[s];
        const float* z = zt + lane * 8;
        int pos = S.pos[s];
        if (a.z_trace && pos < a.trace_cap) {
            float4* dst = reinterpret_cast<float4*>(a.z_trace + ((int64_t)r * a.trace_cap + pos) * 8);
            dst[0] = make_float4(z[0], z[1], z[2], z[3]);
            dst[1] = make_float4(z[4], z[5], z[6], z[7]);
        }
        const int nq = S.nq[s] + 1;
        const float te = S.te[s], tx = S.tx[s];
        const int leaf = S.leaf[s];
        float bt = S.bt[s];
        int bleaf = S.bleaf[s];
        const bool hit = z[0] < 0.0f;                                  // sigmoid(z) < 0.5 (C13)
        if (hit) {
            const float tl = sigmoid_f(z[1]);                          // local distance
            const float t = __fadd_rn(te, __fmul_rn(tl, __fsub_rn(tx, te)));
            const float bte = S.bte[s];
            const bool better = bleaf < 0 || t < bt || (t == bt && (te < bte || (te == bte && leaf < bleaf)));
            if (better) {
                bt = t;
                bleaf = leaf;
                S.bt[s] = t;
                S.bte[s] = te;
                S.bleaf[s] = leaf;
                float nn = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(z[2], z[2]), __fmul_rn(z[3], z[3])),
                                                __fmul_rn(z[4], z[4])));
                nn = fmaxf(nn, 1e-6f);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    S.nrm[k][s] = __fdiv_rn(z[2 + k], nn);
                    S.alb[k][s] = sigmoid_f(z[5 + k]);
                }
            }
        }
        ++pos;
        bool done = a.mode == 1 && hit;                                 // R1: first confident hit (C5)
        S.nq[s] = nq;
        if (!done) {
            if (pos - S.base[s] >= S.nbuf[s]) {
                if (!S.more[s]) done = true;                             // every intersected leaf visited
                else S.pend[s] = 1;                                      // refilled by (A0)
            } else {
                const float4 e = S.nxt[s];                               // the entry prefetched by (C)
                done = bleaf >= 0 && e.x > bt;                         // front-to-back termination
                if (!done) {            // the next entry stays in the slot: no reload in (C)
                    S.te[s] = e.x;
                    S.tx[s] = e.y;
                    S.leaf[s] = __float_as_int(e.z);
                    S.fresh[s] = 1;
                }
            }
        }
        S.pos[s] = pos;
        if (done) slot_finish(a, S, s, r);
    }
    __syncwarp();
}

// ------------------------------------------------------------------ query kernel, per-warp MLP
// Shared-memory plan of k_query_warp (bytes), shared by the kernel and its launcher: the MLP
// weights ([out][in] padded for ldmatrix) and level table once per CTA, then one private
// region per warp (feature rows [16][D+8], which the z tile aliases, and the slots).
struct QuerySmemPlan {
    size_t w, bias, lv, warp0, feat, z, xs, slots, per_warp, total;
    int warps;
    __host__ __device__ QuerySmemPlan(int d_in, int hidden, int n_points, int max_warps = kQueryWarps) {
        w = 0;
        bias = w + align16((size_t)mlp_smem_halves(d_in, hidden) * 2);
        lv = bias + align16((size_t)(64 * hidden + 8) * 4);
        warp0 = lv + align16(sizeof(LevelSm) * kMaxLevels);
        // z aliases the feature rows (the MLP's output layer writes it after its last read of
        // them) and there is no sample-point tile (the encode derives the points from the
        // slots): 6.3 KB per warp, so that 24 warps fit the 196 KB shared-memory carveout step
        // (the next step leaves the table gathers ~28 KB of L1, profiles/NOTES.md r2l)
        feat = 0;
        z = feat;
        xs = feat;
        slots = feat + align16((size_t)kWarpQ * (d_in + 8) * 2);
        (void)n_points;
        per_warp = slots + align16(sizeof(WarpSlots));
        // as many warps (<= max_warps) as fit the 227 KB per-CTA limit
        const size_t cap = 227 * 1024;
        warps = warp0 + per_warp > cap ? 0 : (int)((cap - warp0) / per_warp);
        if (warps > max_warps) warps = max_warps;
        total = warp0 + per_warp * warps;
    }
};

// One launch processes every ray that intersects the cut.  Each warp owns kWarpQ ray slots
// and runs its own loop with no block-wide barrier: (A) refill, (B/C) compact + segment,
// (D) encode into the warp's feature rows, (E) the MLP on mma.sync (one m16 row block,
// activations in registers), (F) decode.  Warps drift freely, so one warp's MLP or list
// refill overlaps other warps' gathers.  Selected with NBVH_QUERY_MLP=warp (A/B reference of
// the warp-specialised kernel below).
// A warp's private shared-memory region of k_query_warp, derived from a volatile read of
// %tid.x so that every use re-derives it (a few integer instructions) instead of keeping the
// addresses live across the encode and the MLP.
struct WarpPtrs {
    int lane, warp;
    __half* feat;      // [kWarpQ][D+8]
    float* zt;         // [kWarpQ][8]
    float* xs;         // [NP*3][kWarpQ]
    WarpSlots* S;
};
__device__ __forceinline__ WarpPtrs warp_ptrs(unsigned char* smem_raw, const QuerySmemPlan& plan) {
    int tid;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
    WarpPtrs P;
    P.lane = tid & 31;
    P.warp = tid >> 5;
    unsigned char* wbase = smem_raw + plan.warp0 + plan.per_warp * P.warp;
    P.feat = reinterpret_cast<__half*>(wbase + plan.feat);
    P.zt = reinterpret_cast<float*>(wbase + plan.z);
    P.xs = reinterpret_cast<float*>(wbase + plan.xs);
    P.S = reinterpret_cast<WarpSlots*>(wbase + plan.slots);
    return P;
}

template <int F, int D, bool kBf, bool kTex = false>
__global__ void __launch_bounds__(query_warps(kTex) * 32, 1) k_query_warp(QueryArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NP = a.g.n_points;
    const QuerySmemPlan plan(D, a.m.hidden, NP);
    MlpSmem ms;
    ms.w0 = reinterpret_cast<__half*>(smem_raw + plan.w);
    ms.wh = ms.w0 + 64 * (D + 8);
    ms.wo = ms.wh + (a.m.hidden - 1) * 64 * 72;
    ms.b = reinterpret_cast<float*>(smem_raw + plan.bias);
    LevelSm* lv = reinterpret_cast<LevelSm*>(smem_raw + plan.lv);
    WarpPtrs P = warp_ptrs(smem_raw, plan);
    stage_mlp(a.m, ms, tid, blockDim.x);
    stage_levels(a.g, lv, tid);
    __shared__ float s_u[16];                 // the segment's stratified offsets (NP <= 16: d_in <= 128)
    if (tid < NP) s_u[tid] = segment_u(tid, NP, nullptr);
    if (lane < kWarpQ) P.S->ray[lane] = -1;
    __syncthreads();                          // the only block-wide barrier
    // work-list sizes and per-warp statistics live in shared memory (read on refills / written
    // by one lane): kept out of the loop's registers
    __shared__ int s_work[2];                 // n_long, total
    __shared__ int s_stat[2 * 32];            // per warp: [0] queries evaluated, [1] loop iterations
    __shared__ int s_exh[32];                 // per warp: work list exhausted
    __shared__ int s_nv[32];                  // per warp: rows of the current iteration
    if (lane == 0) {
        s_work[0] = *a.cnt_long;              // long rays first (k_traverse), then the rest
        s_work[1] = s_work[0] + *a.cnt;       // rays with >= 1 intersected leaf
        s_stat[2 * warp] = s_stat[2 * warp + 1] = 0;
        s_exh[warp] = 0;
    }
    __syncwarp();
    while (true) {
        // the per-lane shared-memory addresses and the row count are re-derived after the
        // encode and the MLP instead of being held across them (ptxas spilled them to the stack)
        P = warp_ptrs(smem_raw, plan);
        WarpSlots& S = *P.S;
        slots_list_refill(a, S, P.lane);
        slots_refill(a, S, P.lane, s_work[1], s_work[0], s_exh + P.warp);
        const int nv = slots_segment<false>(a, S, nullptr, P.lane, NP, s_u);
        if (nv == 0) break;                   // work list drained and every slot finished
        if (P.lane == 0) {
            s_stat[2 * P.warp] += nv;
            s_stat[2 * P.warp + 1] += 1;
            s_nv[P.warp] = nv;
        }
        rows_encode<F, kBf, true, kTex, false>(a, lv, nullptr, nv, P.lane, NP, reinterpret_cast<unsigned char*>(P.feat),
                                               16, (D + 8) * 2, &S, s_u);
        const WarpPtrs Pm = warp_ptrs(smem_raw, plan);
        query_mlp_rows16<D, kBf>(ms, a.m.hidden, Pm.feat, 0, Pm.zt, Pm.lane);         // (E)
        __syncwarp();
        const WarpPtrs Pd = warp_ptrs(smem_raw, plan);
        rows_decode(a, *Pd.S, Pd.zt, *reinterpret_cast<volatile int*>(s_nv + Pd.warp), Pd.lane);
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->n_queries, (unsigned long long)s_stat[2 * warp]);
        atomicMax(&a.ctr->max_iter, s_stat[2 * warp + 1]);
    }
}

// ------------------------------------------------------------------ query kernel, tcgen05 MLP
// Warp-specialised persistent query kernel (NBVH_QUERY_MLP=tc): kWsWorkers worker warps own
// the ray slots -- two slot sets each -- and run refill / segment / encode / decode; one MLP
// warpgroup (4 warps, one per TMEM lane quarter) runs the decoder MLP of 128-row tiles on
// the 5th-generation tensor cores (tcgen05.mma, M = 128, fp32 accumulators in TMEM), so the
// weights never pass through the LSU: they are read once per 128 rows by the tensor core
// instead of once per 16 rows by ldmatrix.
//
// A worker encodes a set's (<= 16) rows into a 16-row block of the current feature tile
// (blocks are claimed in sequence; tile = claim / 8 over a ring of kWsTiles tiles) and
// arrives on the tile's `full` barrier, then turns to its other set; the MLP warpgroup
// processes tiles in claim order: layer 0 from the feature tile (its commit also frees the
// tile for the next generation), hidden layers through one activation tile (TMEM ->
// ReLU + fp16 -> shared memory), the 8 outputs written straight into the owning set's z rows,
// then one arrive on that set's `zr` barrier.  A worker decodes a set only after it has
// encoded its other set, so the MLP latency is hidden behind the other set's gathers.
// Drain: when every worker is idle (waiting for z or finished) and the current tile is only
// partly claimed, the MLP warpgroup closes it (claims jump to the next tile, the missing
// arrivals are made up) and processes it as is.
// Registers: 20 warps share the CTA's 640 x 96 registers; setmaxnreg moves them from the MLP
// warpgroup (32: its epilogue works 16 columns at a time) to the workers (112).  The MLP
// warpgroup waits with mbarrier.try_wait (suspended, no issue slots taken from the workers).
// Measured on the 1080p frame (profiles/NOTES.md r2a/r2b): 1.094 ms vs 0.983 ms for
// k_query_warp -- the LSU data pipe drops from 81% to 60% busy (no weight fragments) and the
// workers wait < 3% of their time for MLP results or tiles, but the workers' encode loop runs
// slower at 112 registers (spills) than the per-warp kernel's at 128.
constexpr int kWsWorkers = 16;                            // 4 warpgroups
constexpr int kWsWorkerRegs = 112, kWsMlpRegs = 32;        // setmaxnreg split of the CTA's 640 x 96 registers
constexpr int kWsTiles = 3;                                // at most; WsPlan::nt fits the smem limit
constexpr int kWsBlk = 8;                                  // 16-row blocks per 128-row tile
constexpr int kKgHid = 64 / 8 + 2;                         // K-groups of a hidden W (+ bias)

struct WsCtl {
    uint64_t full[kWsTiles];           // kWsBlk arrivals per tile generation (workers)
    uint64_t freeb[kWsTiles];          // layer-0 MMAs of the generation complete (tcgen05.commit)
    uint64_t mma;                      // MMA chain steps of the MLP warpgroup
    uint64_t zr[2 * kWsWorkers];       // z of a set's block written (one arrive per block)
    int seq;                           // block claims so far
    int idle;                          // workers waiting for z or finished
    int exited;                        // workers finished
    int cmd;                           // MLP warpgroup: 1 process the tile, 2 exit
    int owner[kWsTiles][kWsBlk];       // 2 * worker + set of each block; -1: none
    int nrows[kWsTiles][kWsBlk];       // valid rows of each block
    int work[2];                       // n_long, total
    int exh[kWsWorkers];               // per worker: work list exhausted
    int stat[kWsWorkers][2];           // per worker: queries, slot-set iterations
    uint32_t tmem;
};

struct WsPlan {
    size_t w0, wh, wo, ones, lv, ctl, tiles, htile, xs, sets, per_set, z, total;
    int tile_bytes, nt;
    __host__ __device__ WsPlan(int d_in, int hidden, int n_points) {
        w0 = 0;
        wh = w0 + (size_t)64 * (d_in / 8 + 2) * 16;
        wo = wh + (size_t)(hidden - 1) * 64 * kKgHid * 16;
        ones = wo + (size_t)16 * kKgHid * 16;
        lv = ones + 2 * 128 * 16;
        ctl = lv + align16(sizeof(LevelSm) * kMaxLevels);
        tiles = align128(ctl + sizeof(WsCtl));
        tile_bytes = (d_in / 8) * 2048;                        // [D/8 K-groups][128 rows][16 B]
        const size_t xs_bytes = align16((size_t)kWarpQ * n_points * 3 * 4);   // per worker (sets take turns)
        z = align16(sizeof(WarpSlots));                         // offset within a set region
        per_set = z + align16((size_t)kWarpQ * 8 * 4);
        const size_t rest = 8 * 2048 + xs_bytes * kWsWorkers + per_set * 2 * kWsWorkers;
        nt = kWsTiles;                                          // as many tiles as fit (>= 2)
        while (nt > 2 && tiles + (size_t)nt * tile_bytes + rest > 227 * 1024) --nt;
        htile = tiles + (size_t)nt * tile_bytes;                // hidden activations [8][128][16 B]
        xs = htile + 8 * 2048;
        sets = xs + xs_bytes * kWsWorkers;
        total = sets + per_set * 2 * kWsWorkers;
    }
};

template <int F, int D>
__global__ void __launch_bounds__((kWsWorkers + 4) * 32, 1) k_query_ws(QueryArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NP = a.g.n_points, H = a.m.hidden;
    const WsPlan plan(D, H, NP);
    LevelSm* lv = reinterpret_cast<LevelSm*>(smem_raw + plan.lv);
    WsCtl& C = *reinterpret_cast<WsCtl*>(smem_raw + plan.ctl);
    unsigned char* tiles = smem_raw + plan.tiles;
    unsigned char* htile = smem_raw + plan.htile;
    auto set_base = [&](int owner) { return smem_raw + plan.sets + plan.per_set * (size_t)owner; };

    // ---- staging: weights in the K-major canonical (core-matrix) layout, element (n, k) of
    // W [N][K] at (k/8) * (Npad*16) + n*16 + (k%8)*2, the bias as two extra K columns (hi + lo
    // fp16) multiplied by a ones tile in an extra K step
    auto stage_w = [&](unsigned char* dst, const __half* src, const float* bias, int N, int K, int Npad) {
        const int kg = K / 8 + 2;
        for (int i = tid; i < Npad * kg; i += blockDim.x) {
            const int n = i / kg, gk = i % kg;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (n < N) {
                if (gk < K / 8) {
                    v = *reinterpret_cast<const uint4*>(src + (int64_t)n * K + gk * 8);
                } else if (gk == K / 8) {
                    const __half hi = __float2half_rn(bias[n]);
                    const __half lo = __float2half_rn(bias[n] - __half2float(hi));
                    v.x = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
                }
            }
            *reinterpret_cast<uint4*>(dst + gk * (Npad * 16) + n * 16) = v;
        }
    };
    stage_w(smem_raw + plan.w0, a.m.W, a.m.b, 64, D, 64);
    for (int l = 0; l < H - 1; ++l)
        stage_w(smem_raw + plan.wh + (size_t)l * 64 * kKgHid * 16, a.m.W + 64 * D + (int64_t)l * 64 * 64,
                a.m.b + 64 * (l + 1), 64, 64, 64);
    stage_w(smem_raw + plan.wo, a.m.W + 64 * D + (int64_t)(H - 1) * 64 * 64, a.m.b + 64 * H, 8, 64, 16);
    for (int i = tid; i < 128; i += blockDim.x) {                           // bias K-step A columns
        *reinterpret_cast<uint4*>(smem_raw + plan.ones + i * 16) = make_uint4(0x3C003C00u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(smem_raw + plan.ones + 2048 + i * 16) = make_uint4(0u, 0u, 0u, 0u);
    }
    stage_levels(a.g, lv, tid);
    __shared__ float s_u[16];                 // the segment's stratified offsets (NP <= 16: d_in <= 128)
    if (tid < NP) s_u[tid] = segment_u(tid, NP, nullptr);
    if (warp < kWsWorkers && lane < kWarpQ) {
        reinterpret_cast<WarpSlots*>(set_base(2 * warp))->ray[lane] = -1;
        reinterpret_cast<WarpSlots*>(set_base(2 * warp + 1))->ray[lane] = -1;
    }
    if (tid == 0) {
        for (int t = 0; t < plan.nt; ++t) {
            tc::mbar_init(&C.full[t], kWsBlk);
            tc::mbar_init(&C.freeb[t], 1);
        }
        tc::mbar_init(&C.mma, 1);
        for (int i = 0; i < 2 * kWsWorkers; ++i) tc::mbar_init(&C.zr[i], 1);
        C.seq = 0;
        C.idle = 0;
        C.exited = 0;
        C.cmd = 0;
        C.work[0] = *a.cnt_long;              // long rays first (k_traverse), then the rest
        C.work[1] = C.work[0] + *a.cnt;       // rays with >= 1 intersected leaf
        tc::fence_barrier_init();
    }
    if (tid < kWsWorkers) {
        C.exh[tid] = 0;
        C.stat[tid][0] = C.stat[tid][1] = 0;
    }
    if (warp == kWsWorkers) tc::tmem_alloc<64>(&C.tmem);
    tc::fence_proxy_async();                  // staged weights -> tensor core (async proxy)
    tc::fence_before();
    __syncthreads();                          // the only block-wide barrier before the teardown
    tc::fence_after();

    if (warp < kWsWorkers) {
        // ================================================================ worker warps
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsWorkerRegs));
        // loop state in scalars (a runtime-indexed array would live in local memory): bit s of
        // zph = parity of set s's next z wait, of pend = set s has a block in flight; nv_pk =
        // rows of set 0 | rows of set 1 << 8
        uint32_t zph = 0, pend = 0, nv_pk = 0;
        int s = 0;
        long long t_z = 0, t_free = 0;                    // cycles waiting (lane 0's clock)
        const long long t_start = clock64();
        float* xs = reinterpret_cast<float*>(smem_raw + plan.xs + (size_t)warp * (plan.sets - plan.xs) / kWsWorkers);
        while (true) {
            unsigned char* sb = set_base(2 * warp + s);
            WarpSlots& S = *reinterpret_cast<WarpSlots*>(sb);
            float* zt = reinterpret_cast<float*>(sb + plan.z);
            if (pend & (1u << s)) {           // (F) this set's z: wait, then decode
                if (lane == 0) atomicAdd(&C.idle, 1);
                const long long t0 = clock64();
                tc::mbar_wait(&C.zr[2 * warp + s], (zph >> s) & 1u);
                t_z += clock64() - t0;
                if (lane == 0) atomicSub(&C.idle, 1);
                zph ^= 1u << s;
                pend &= ~(1u << s);
                rows_decode(a, S, zt, (int)((nv_pk >> (8 * s)) & 0xffu), lane);
            }
            slots_list_refill(a, S, lane);
            slots_refill(a, S, lane, C.work[1], C.work[0], &C.exh[warp]);
            const int nv = slots_segment(a, S, xs, lane, NP, s_u);
            nv_pk = (nv_pk & ~(0xffu << (8 * s))) | ((uint32_t)nv << (8 * s));
            if (nv == 0) {
                if (!(pend & (1u << (s ^ 1)))) break;   // both sets drained: done
                s ^= 1;
                continue;
            }
            if (lane == 0) {
                C.stat[warp][0] += nv;
                C.stat[warp][1] += 1;
            }
            // claim a 16-row block of the current tile; wait until the tile's previous
            // generation has been read by its layer-0 MMAs
            int q = 0;
            if (lane == 0) q = atomicAdd(&C.seq, 1);
            q = __shfl_sync(0xffffffffu, q, 0);
            const int tl = (q / kWsBlk) % plan.nt, gen = q / (kWsBlk * plan.nt), blk = q % kWsBlk;
            if (gen > 0) {
                const long long t0 = clock64();
                tc::mbar_wait(&C.freeb[tl], (uint32_t)(gen - 1) & 1u);
                t_free += clock64() - t0;
            }
            // (D) encode straight into the tile: row blk*16 + q, K-major canonical layout
            rows_encode<F, false, false, true>(a, lv, xs, nv, lane, NP, tiles + (size_t)tl * plan.tile_bytes + blk * 16 * 16, 2048, 16);
            if (lane == 0) {
                C.owner[tl][blk] = 2 * warp + s;
                C.nrows[tl][blk] = nv;
            }
            tc::fence_proxy_async();          // feature rows (generic) -> tensor core (async proxy)
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&C.full[tl]);
            pend |= 1u << s;
            s ^= 1;
        }
        if (lane == 0) {
            atomicAdd(&a.ctr->ws_cycles[0], (unsigned long long)t_z);
            atomicAdd(&a.ctr->ws_cycles[1], (unsigned long long)t_free);
            atomicAdd(&a.ctr->ws_cycles[2], (unsigned long long)(clock64() - t_start));
            atomicAdd(&C.exited, 1);
            atomicAdd(&C.idle, 1);
            atomicAdd(&a.ctr->n_queries, (unsigned long long)C.stat[warp][0]);
            atomicMax(&a.ctr->max_iter, C.stat[warp][1]);
        }
    } else {
        // ================================================================ MLP warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsMlpRegs));
        const int mw = warp - kWsWorkers;     // == warp % 4: the TMEM lane quarter it may access
        const uint32_t acc = C.tmem;
        constexpr uint32_t id64 = tc::idesc_f16(128, 64, false, false);
        constexpr uint32_t id16 = tc::idesc_f16(128, 16, false, false);
        const uint64_t dOnes = tc::smem_desc(tc::smem_u32(smem_raw + plan.ones), 2048, 128);
        const uint64_t dW0 = tc::smem_desc(tc::smem_u32(smem_raw + plan.w0), 1024, 128);
        const uint64_t dWh = tc::smem_desc(tc::smem_u32(smem_raw + plan.wh), 1024, 128);
        const uint64_t dWo = tc::smem_desc(tc::smem_u32(smem_raw + plan.wo), 256, 128);
        const uint64_t dH = tc::smem_desc(tc::smem_u32(htile), 2048, 128);
        const int row = 32 * mw + lane;
        uint32_t mph = 0;
        int n_tiles = 0, n_rows = 0;          // statistics (warp 0, lane 0)
        for (int T = 0;; ++T) {
            const int tl = T % plan.nt, gen = T / plan.nt;
            if (mw == 0) {
                int cmd = 1;
                if (lane == 0) {
                    const int base = T * kWsBlk;
                    // mbarrier.try_wait suspends the thread for a while before it gives up, so the
                    // waiting MLP warp takes no issue slots from the workers on its SMSP
                    while (!tc::mbar_try(&C.full[tl], (uint32_t)gen & 1u)) {
                        if (*(volatile int*)&C.idle < kWsWorkers) continue;
                        const int sq = *(volatile int*)&C.seq;
                        if (sq <= base) {
                            if (*(volatile int*)&C.exited == kWsWorkers) { cmd = 2; break; }
                        } else if (sq < base + kWsBlk && atomicCAS(&C.seq, sq, base + kWsBlk) == sq) {
                            // close the partly claimed tile: no block after sq - base is used
                            for (int b = sq - base; b < kWsBlk; ++b) C.owner[tl][b] = -1;
                            __threadfence_block();
                            for (int b = sq - base; b < kWsBlk; ++b) tc::mbar_arrive(&C.full[tl]);
                        }
                    }
                    C.cmd = cmd;
                }
                __syncwarp();
            }
            named_bar(1, 128);
            if (*(volatile int*)&C.cmd == 2) break;
            // layer 0 from the feature tile; its completion also frees the tile
            if (mw == 0) {
                tc::fence_after();
                const uint64_t dA = tc::smem_desc(tc::smem_u32(tiles + (size_t)tl * plan.tile_bytes), 2048, 128);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) tc::mma_f16_elect(acc, dA + kk * 256, dW0 + kk * 128, id64, kk > 0);
                tc::mma_f16_elect(acc, dOnes, dW0 + (D / 16) * 128, id64, 1);                 // bias
                tc::commit_elect(&C.freeb[tl]);
                tc::commit_elect(&C.mma);
            }
            for (int l = 0; l < H; ++l) {
                tc::mbar_wait(&C.mma, mph);
                mph ^= 1u;
                tc::fence_after();
#pragma unroll
#pragma unroll 1
                for (int q16 = 0; q16 < 4; ++q16) {                   // 64 columns, 16 at a time (few
                    float v[16];                                       // registers): ReLU + fp16 -> H tile
                    tc::ld16(acc, (uint32_t)(32 * mw), (uint32_t)(16 * q16), v);
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        uint4 o;
                        o.x = pack_relu_half2(v[8 * k], v[8 * k + 1]);
                        o.y = pack_relu_half2(v[8 * k + 2], v[8 * k + 3]);
                        o.z = pack_relu_half2(v[8 * k + 4], v[8 * k + 5]);
                        o.w = pack_relu_half2(v[8 * k + 6], v[8 * k + 7]);
                        *reinterpret_cast<uint4*>(htile + (2 * q16 + k) * 2048 + row * 16) = o;
                    }
                }
                tc::fence_proxy_async();
                tc::fence_before();
                named_bar(1, 128);
                if (mw == 0) {
                    tc::fence_after();
                    const bool out = l + 1 == H;
                    const uint64_t dW = out ? dWo : dWh + (uint64_t)(l * 64 * kKgHid);
                    const uint32_t kgu = out ? 16 : 64, id = out ? id16 : id64;   // K-group stride / 16 B
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) tc::mma_f16_elect(acc, dH + kk * 256, dW + kk * 2 * kgu, id, kk > 0);
                    tc::mma_f16_elect(acc, dOnes, dW + 8 * kgu, id, 1);                            // bias
                    tc::commit_elect(&C.mma);
                }
            }
            tc::mbar_wait(&C.mma, mph);
            mph ^= 1u;
            tc::fence_after();
            {   // the 8 outputs of row `row` -> the owning set's z rows
                float v[16];
                tc::ld16(acc, (uint32_t)(32 * mw), 0u, v);
                const int own = C.owner[tl][row >> 4];
                if (own >= 0) {
                    float4* z = reinterpret_cast<float4*>(set_base(own) + plan.z) + (row & 15) * 2;
                    z[0] = make_float4(v[0], v[1], v[2], v[3]);
                    z[1] = make_float4(v[4], v[5], v[6], v[7]);
                }
            }
            tc::fence_before();               // accumulator reads done before the next tile's MMAs
            named_bar(1, 128);
            if (mw == 0 && lane < kWsBlk) {
                const int own = C.owner[tl][lane];
                int nr = own >= 0 ? C.nrows[tl][lane] : 0;
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) nr += __shfl_xor_sync(0xffu, nr, o);
                if (lane == 0) {
                    ++n_tiles;
                    n_rows += nr;
                }
                if (own >= 0) tc::mbar_arrive(&C.zr[own]);
            }
        }
        if (mw == 0 && lane == 0) {
            atomicAdd(&a.ctr->mlp_tiles, n_tiles);
            atomicAdd(&a.ctr->mlp_rows, n_rows);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == kWsWorkers) tc::tmem_free<64>(C.tmem);
}

// ------------------------------------------------------------------ debug: encode points
// The product encode (encode_chunk_sm) on caller-supplied points, indices exposed.
template <int F>
__global__ void __launch_bounds__(128) k_debug_encode(DebugEncodeArgs a) {
    __shared__ LevelSm lv[kMaxLevels];
    stage_levels(a.g, lv, threadIdx.x);
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.m) return;
    const float x0 = a.pts[3 * i], x1 = a.pts[3 * i + 1], x2 = a.pts[3 * i + 2];
    const int L = a.g.L;
    const int chunks = (L * F) / 8;
    const uint32_t hmask = (1u << a.g.log2_T) - 1u;
    uint32_t idx[64];
    for (int c = 0; c < chunks; ++c) {
        const int l0 = c * 8 / F;
        uint4 v = encode_chunk_sm<F>(lv, a.g.table, hmask, x0, x1, x2, l0, a.index ? idx : nullptr);
        reinterpret_cast<uint4*>(a.feat + i * (int64_t)L * F)[c] = v;
        if (a.index)
            for (int j = 0; j < 8 / F * 8; ++j) a.index[(i * L + l0) * 8 + j] = idx[j];
    }
}

// ------------------------------------------------------------------ debug: MLP rows
template <int D, bool kBf>
__global__ void __launch_bounds__(256, 2) k_debug_mlp(DebugMlpArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    MlpSmem ms;
    __half* feat = reinterpret_cast<__half*>(smem_raw);
    ms.w0 = feat + kTileQ * (D + 8);
    ms.wh = ms.w0 + 64 * (D + 8);
    ms.wo = ms.wh + (a.m.hidden - 1) * 64 * 72;
    float* zt = reinterpret_cast<float*>(ms.wo + 8 * 72);
    ms.b = zt + kTileQ * 8;
    stage_mlp(a.m, ms, tid, blockDim.x);
    const int64_t n_tiles = (a.rows + kTileQ - 1) / kTileQ;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int i = tid; i < kTileQ * (D / 8); i += blockDim.x) {
            const int row = i / (D / 8), c = i % (D / 8);
            const int64_t gr = tile * kTileQ + row;
            uint4 v = gr < a.rows ? reinterpret_cast<const uint4*>(a.x + gr * D)[c] : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(feat + row * (D + 8) + c * 8) = v;
        }
        __syncthreads();
        query_mlp_rows16<D, kBf>(ms, a.m.hidden, feat, warp * 16, zt, lane);   // k_query's own MLP
        __syncthreads();
        for (int i = tid; i < kTileQ * 8; i += blockDim.x) {
            const int64_t gr = tile * kTileQ + i / 8;
            if (gr < a.rows) a.z[gr * 8 + (i % 8)] = zt[i];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ launchers
size_t mlp_smem_bytes(int d_in, int hidden) {
    return (size_t)kTileQ * (d_in + 8) * 2 + (size_t)mlp_smem_halves(d_in, hidden) * 2 + kTileQ * 8 * 4 +
           (64 * hidden + 8) * 4;
}

template <typename Kern>
static int resident_blocks(Kern k, int threads, size_t smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (per_sm > 0 ? per_sm : 1) * sms;
}

// Default: the per-warp mma.sync kernel (k_query_warp, 0.983 ms on the 1080p frame);
// NBVH_QUERY_MLP=tc selects the warp-specialised tcgen05 kernel (k_query_ws, 1.094 ms:
// profiles/NOTES.md r2).  Read per launch so tests can switch it.
static bool query_mlp_warp() {
    const char* ev = std::getenv("NBVH_QUERY_MLP");
    return !(ev && ev[0] == 't');
}
// NBVH_QUERY_WARPS=n caps k_query_warp's warps per CTA (A/B hook: fewer warps, less shared
// memory, a larger L1).  Measured on the 1080p frame (profiles/NOTES.md r2d): 16 / 14 / 13 /
// 12 warps -> 0.980 / 1.053 / 1.095 / 1.140 ms -- the gathers want warps, not L1 capacity.
// (Also tried there: 32 slots per warp, two m16 blocks sharing each weight fragment -- half
// the ldmatrix traffic, but only 12-15 warps fit: 1.033-1.041 ms.)
static int query_warps_cap(int plan_warps) {
    const char* ew = std::getenv("NBVH_QUERY_WARPS");
    const int w = ew ? std::atoi(ew) : 0;
    return w >= 1 && w < plan_warps ? w : plan_warps;
}

template <int kKind, typename Kern>             // kKind: one occupancy cache per kernel family
static cudaError_t launch_persistent(Kern k, int threads, size_t smem, int64_t max_work, int rows_per_cta,
                                     const QueryArgs& a, cudaStream_t s, int hidden, int n_points) {
    // The dynamic shared-memory opt-in is per function, not per shape: set it before every
    // launch (cheap), so a smaller shape launched in between cannot leave it too low.  The
    // occupancy query is cached per (device, hidden, n_points).
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    constexpr int kDevs = 16;
    static int cached[kDevs][kMaxHidden + 1][9][2] = {};     // [.][.][.][F == 4]: per instantiation
    int fallback = 0;
    int& grid_c = dev < kDevs ? cached[dev][hidden][n_points < 9 ? n_points : 8][a.g.F == 4] : fallback;
    if (!grid_c) grid_c = resident_blocks(k, threads, smem);
    int grid = grid_c;
    const int64_t need = (max_work + rows_per_cta - 1) / rows_per_cta;
    if (need < grid) grid = (int)(need > 0 ? need : 1);
    k<<<grid, threads, smem, s>>>(a);
    return cudaGetLastError();
}

template <int F, int D>
static cudaError_t launch_query_t(const QueryArgs& a, int64_t max_work, cudaStream_t s) {
    if (!query_mlp_warp() && !a.m.bf16 && a.g.tex != 0 && F == 2) {   // the tcgen05 variant: fp16, TEX gathers
        const WsPlan plan(D, a.m.hidden, a.g.n_points);
        if (plan.total <= 227 * 1024)
            return launch_persistent<0>(k_query_ws<F, D>, (kWsWorkers + 4) * 32, plan.total, max_work,
                                     2 * kWsWorkers * kWarpQ, a, s, a.m.hidden, a.g.n_points);
    }
    // hashed-level gathers through the TEX pipe when the context has its texture object (F = 2)
    const bool tex = a.g.tex != 0 && F == 2;
    QuerySmemPlan plan(D, a.m.hidden, a.g.n_points, query_warps(tex));
    if (plan.warps < 1) return cudaErrorInvalidValue;
    plan.warps = query_warps_cap(plan.warps);
    plan.total = plan.warp0 + plan.per_warp * plan.warps;
    if (const char* pe = std::getenv("NBVH_QUERY_SMEM_PAD"))   // A/B hook: unused shared memory (L1 carveout)
        plan.total += (size_t)std::atol(pe);
    if (a.m.bf16)
        return tex ? launch_persistent<5>(k_query_warp<F, D, true, true>, plan.warps * 32, plan.total, max_work,
                                          plan.warps * kWarpQ, a, s, a.m.hidden, a.g.n_points)
                   : launch_persistent<2>(k_query_warp<F, D, true>, plan.warps * 32, plan.total, max_work,
                                          plan.warps * kWarpQ, a, s, a.m.hidden, a.g.n_points);
    return tex ? launch_persistent<6>(k_query_warp<F, D, false, true>, plan.warps * 32, plan.total, max_work,
                                      plan.warps * kWarpQ, a, s, a.m.hidden, a.g.n_points)
               : launch_persistent<1>(k_query_warp<F, D, false>, plan.warps * 32, plan.total, max_work,
                                      plan.warps * kWarpQ, a, s, a.m.hidden, a.g.n_points);
}

cudaError_t launch_query(const QueryArgs& a, int64_t max_work, cudaStream_t s) {
    const int F = a.g.F, D = a.m.d_in;
    if (F == 2 && D == 32) return launch_query_t<2, 32>(a, max_work, s);
    if (F == 2 && D == 64) return launch_query_t<2, 64>(a, max_work, s);
    if (F == 2 && D == 96) return launch_query_t<2, 96>(a, max_work, s);
    if (F == 2 && D == 128) return launch_query_t<2, 128>(a, max_work, s);
    if (F == 4 && D == 64) return launch_query_t<4, 64>(a, max_work, s);
    if (F == 4 && D == 96) return launch_query_t<4, 96>(a, max_work, s);
    if (F == 4 && D == 128) return launch_query_t<4, 128>(a, max_work, s);
    return cudaErrorInvalidValue;
}

// NBVH_TRAVERSE=packet selects the warp-packet traversal (A/B hook; see traverse_packet).
cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.n_rays + 127) / 128;
    const char* ev = std::getenv("NBVH_TRAVERSE");
    if (ev && ev[0] == 'p') {
        const size_t smem = (size_t)(3 * a.cap * 128 + 4 * (a.cut.depth + 2)) * sizeof(int);
        k_traverse<true><<<(unsigned)blocks, 128, smem, s>>>(a);
    } else {
        // (depth + 2 + 3K) words per thread: past 48 KB for deep cuts / large K, so opt in
        const size_t smem = (size_t)(a.cut.depth + 2 + 3 * a.cap) * 128 * sizeof(int);
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(k_traverse<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        k_traverse<false><<<(unsigned)blocks, 128, smem, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_debug_traverse(const DebugTraverseArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.n_rays + 127) / 128;
    k_debug_traverse<<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_debug_encode(const DebugEncodeArgs& a, cudaStream_t s) {
    const int64_t blocks = (a.m + 127) / 128;
    if (a.g.F == 2) k_debug_encode<2><<<(unsigned)blocks, 128, 0, s>>>(a);
    else k_debug_encode<4><<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

template <int D, bool kBf>
static cudaError_t launch_mlp_tb(const DebugMlpArgs& a, cudaStream_t s) {
    const size_t smem = mlp_smem_bytes(D, a.m.hidden);
    int grid = resident_blocks(k_debug_mlp<D, kBf>, 256, smem);
    const int64_t tiles = (a.rows + kTileQ - 1) / kTileQ;
    if (tiles < grid) grid = (int)tiles;
    if (grid < 1) grid = 1;
    k_debug_mlp<D, kBf><<<grid, 256, smem, s>>>(a);
    return cudaGetLastError();
}
template <int D>
static cudaError_t launch_mlp_t(const DebugMlpArgs& a, cudaStream_t s) {
    return a.m.bf16 ? launch_mlp_tb<D, true>(a, s) : launch_mlp_tb<D, false>(a, s);
}

cudaError_t launch_debug_mlp(const DebugMlpArgs& a, cudaStream_t s) {
    switch (a.m.d_in) {
        case 32: return launch_mlp_t<32>(a, s);
        case 64: return launch_mlp_t<64>(a, s);
        case 96: return launch_mlp_t<96>(a, s);
        case 128: return launch_mlp_t<128>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace nbvh
