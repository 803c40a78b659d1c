// nbvh_launch.h — kernel argument blocks and launchers (product-internal).
#pragma once

#include <cuda_runtime.h>

#include "nbvh_device.cuh"

namespace nbvh {

struct HitsDev {
    uint8_t* hit;
    float* t;
    float* normal;
    float* albedo;
    int32_t* leaf;
    int32_t* n_queries;
};

// Per-ray list bookkeeping written by k_traverse and read when a ray enters a query slot.
struct RayState {
    int32_t* nbuf;    // entries held in the list buffer
    int32_t* more;    // 1 if intersected leaves beyond the buffer may exist (C6)
};

// Device counters of one nbvh_query call (zeroed by one memset per call).
struct QueryCounters {
    int32_t err;                  // bit 0: traversal stack overflow
    int32_t refills;              // list re-traversals (C6)
    int32_t cnt;                  // rays with >= 1 intersected leaf (k_traverse append count)
    int32_t next;                 // work-list cursor of the persistent query kernel
    int32_t max_iter;             // slot iterations of the busiest CTA
    int32_t cnt_long;             // rays queued on the "long" work list (many leaves: scheduled first)
    int32_t mlp_tiles;            // k_query_ws: MLP tiles processed
    int32_t mlp_rows;             // k_query_ws: valid rows in them
    unsigned long long n_queries; // neural queries (ray, leaf) evaluated
    unsigned long long ws_cycles[3];  // k_query_ws, summed over worker warps: waiting for z, waiting
                                      // for a free tile, total
};

// One work-list entry of the persistent query kernel, written by k_traverse: the ray itself
// and its list state, so a slot refill is one level of (coalesced, 3 x 16 B) loads instead of
// an index load followed by dependent ray / list-state loads.  (tmin / tmax are not needed
// past the traversal: the leaf intervals already respect them.)
struct WorkRec {
    float4 o;        // origin xyz, .w = ray index (int bits)
    float4 d;        // direction xyz, .w = nbuf | more << 16 (int bits)
    float4 e0;       // the first list entry: t_enter, t_exit, leaf id bits, 0
};

struct TraverseArgs {
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    int32_t cap;
    float4* lst;             // leaf lists [K][n_rays]: (t_enter, t_exit, leaf id bits, 0)
    RayState st;
    HitsDev out;
    WorkRec* act_out;
    WorkRec* act_long;       // rays with many intersected leaves (queued first, shorter tail)
    QueryCounters* ctr;
};

struct DebugTraverseArgs {
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    int32_t cap, k;
    int32_t* leaf;
    float* te;
    float* tx;
    int32_t* count;
    int32_t* err;
};

struct QueryArgs {
    GridDev g;
    MlpDev m;
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    int32_t cap;
    int32_t mode;
    float4* lst;             // leaf lists [K][n_rays]: (t_enter, t_exit, leaf id bits, 0)
    const int32_t* nbuf;
    const int32_t* more;
    HitsDev out;
    const WorkRec* act;      // work list: rays with >= 1 leaf (k_traverse)
    const int32_t* cnt;      // its length (device)
    const WorkRec* act_long; // long-ray work list, consumed before `act`
    const int32_t* cnt_long;
    int32_t* next;           // work-list cursor
    float* z_trace;
    int32_t trace_cap;
    QueryCounters* ctr;
};

struct DebugEncodeArgs {
    GridDev g;
    const float* pts;
    int64_t m;
    __half* feat;
    uint32_t* index;
};

struct DebugMlpArgs {
    MlpDev m;
    const __half* x;
    int64_t rows;
    float* z;
};

cudaError_t launch_traverse(const TraverseArgs& a, cudaStream_t s);
cudaError_t launch_debug_traverse(const DebugTraverseArgs& a, cudaStream_t s);
cudaError_t launch_query(const QueryArgs& a, int64_t max_work, cudaStream_t s);
cudaError_t launch_debug_encode(const DebugEncodeArgs& a, cudaStream_t s);
cudaError_t launch_debug_mlp(const DebugMlpArgs& a, cudaStream_t s);

}  // namespace nbvh
