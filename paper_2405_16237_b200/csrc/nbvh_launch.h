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

// Per-ray wave state, structure of arrays.
struct RayState {
    int32_t* pos;     // global index of the current list entry
    int32_t* base;    // global index of list slot 0
    int32_t* nbuf;    // entries held in the list buffer
    int32_t* more;    // 1 if intersected leaves beyond the buffer may exist (C6)
    float* bt;        // best hit t
    float* bte;       // its t_enter
    int32_t* bleaf;   // its leaf (-1: none)
    int32_t* nq;      // queries so far
};

struct TraverseArgs {
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    int32_t cap;
    int32_t* lst_leaf;
    float* lst_te;
    float* lst_tx;
    RayState st;
    HitsDev out;
    int32_t* act_out;
    int32_t* cnt_out;
    int32_t* err;
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

struct WaveArgs {
    GridDev g;
    MlpDev m;
    CutDev cut;
    const float4* rays;
    int64_t n_rays;
    int32_t cap;
    int32_t mode;
    int32_t* lst_leaf;
    float* lst_te;
    float* lst_tx;
    RayState st;
    HitsDev out;
    const int32_t* act_in;
    int32_t* act_out;
    const int32_t* cnt_in;
    int32_t* cnt_out;
    float* z_trace;
    int32_t trace_cap;
    int32_t* n_refills;
    int32_t* err;
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
cudaError_t launch_query_wave(const WaveArgs& a, cudaStream_t s);
cudaError_t launch_debug_encode(const DebugEncodeArgs& a, cudaStream_t s);
cudaError_t launch_debug_mlp(const DebugMlpArgs& a, cudaStream_t s);

}  // namespace nbvh
