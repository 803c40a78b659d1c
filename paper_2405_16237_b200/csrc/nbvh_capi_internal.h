// nbvh_capi_internal.h — the context object behind the opaque nbvh_ctx handle.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/nbvh.h"
#include "nbvh_internal.h"
#include "nbvh_launch.h"

namespace nbvh {

struct DeviceCut {
    InnerNode* inner = nullptr;
    float4* leaf_box = nullptr;   // [n][2]
    int32_t* leaf_base = nullptr;
    float* rank = nullptr;
    int32_t depth = 0;            // inner levels of the snapshot (sizes the traversal stack)
};

struct DeviceScene {
    BvhNode* nodes = nullptr;     // base BVH
    float* tri_v = nullptr;       // [nt][9] vertices in prim order
    float* tri_n = nullptr;       // [nt][9] vertex normals in prim order
    float* tri_a = nullptr;       // [nt][3] albedo in prim order
    int32_t* tri_id = nullptr;    // [nt] original triangle id
    int64_t n_tris = 0;
};

struct TrainWork;   // nbvh_train.cu
constexpr int kCounterStride = 16;  // int32 words per QueryCounters block (64 B)
constexpr int kCounterBlocks = 16;
}  // namespace nbvh

struct nbvh_ctx {
    nbvh_config cfg{};
    int device = -1;
    bool poisoned = false;
    std::string err;

    // hash grid / MLP geometry
    int32_t res[nbvh::kMaxLevels] = {0};
    int32_t dense[nbvh::kMaxLevels] = {0};
    int64_t offset[nbvh::kMaxLevels] = {0};
    int64_t n_entries = 0;
    int64_t inf_offset[nbvh::kMaxLevels] = {0};   // inference-table entry offsets (dense levels corner-packed)
    int64_t n_inf = 0;                             // inference-table entries
    int32_t d_in = 0;
    int64_t n_table = 0, n_W = 0, n_b = 0;

    // parameters: fp32 master (flat: tables, weights, biases) + fp16 inference copy
    std::vector<float> h_params;
    float* d_params = nullptr;
    __half* d_table16 = nullptr;
    unsigned long long tex_table = 0;  // texture object over d_table16 (TEX-pipe gathers, see LevelSm::pad)
    __half* d_W16 = nullptr;
    __nv_bfloat16* d_Wb16 = nullptr;   // bf16 copy of the MLP weights (mlp_dtype = 1: query path)

    // scene and cuts
    nbvh::HostScene sc;
    bool has_mesh = false;
    int32_t base_depth = -1;           // base-BVH depth (computed on first classical query)
    nbvh::HostCut cuts[nbvh::kMaxLod];
    bool has_cut[nbvh::kMaxLod] = {false};
    nbvh::DeviceCut dcut[nbvh::kMaxLod];
    nbvh::DeviceScene dscene;

    // query workspaces
    int64_t reserved = 0;
    float4* d_lst = nullptr;           // per-ray leaf lists [K][n]: (t_enter, t_exit, leaf bits, 0)
    int32_t* d_state = nullptr;        // 2 arrays of n int32: list fill, "more leaves" flag
    nbvh::WorkRec* d_act = nullptr;      // work list of the persistent query kernel
    nbvh::WorkRec* d_act_long = nullptr; // its long-ray part (consumed first)
    int32_t* d_misc = nullptr;         // kCounterBlocks QueryCounters blocks, kCounterStride int32 apart
    int32_t* h_misc = nullptr;         // pinned mirror
    float* d_stage_rays = nullptr;     // host-path staging
    float* d_stage_hits = nullptr;
    nbvh_query_stats qstats{};
    int32_t qstats_launches = 0;
    bool qstats_pending = false;       // device counters not yet read back
    int qstats_blocks = 1;             // counter blocks used by the last call
    cudaStream_t qstats_stream = nullptr;
    bool profiling = false;
    cudaStream_t aux_stream[3] = {nullptr, nullptr, nullptr};  // upload / download / 2nd query stream (host path)
    std::vector<cudaEvent_t> events;   // [0..2] query profiling, [16..23] training phases, [32..] host-path chunk order

    // training
    nbvh::TrainWork* train = nullptr;
    nbvh_train_stats tstats{};

    nbvh::RayState state() const {
        nbvh::RayState s;
        s.nbuf = d_state;
        s.more = d_state + reserved;
        return s;
    }
};

namespace nbvh {
nbvh_status fail(nbvh_ctx* c, nbvh_status s, const std::string& msg);
nbvh_status cuda_fail(nbvh_ctx* c, cudaError_t e, const char* where);
nbvh_status check_device(nbvh_ctx* c);
int32_t base_bvh_depth(const HostScene& sc);   // levels of the base BVH (root = 1)
GridDev make_grid(const nbvh_ctx* c, int lod);
MlpDev make_mlp(const nbvh_ctx* c);
CutDev make_cut(const nbvh_ctx* c, int lod);
nbvh_status refresh_fp16(nbvh_ctx* c, cudaStream_t s);
nbvh_status refresh_table(nbvh_ctx* c, cudaStream_t s);
cudaEvent_t ctx_event(nbvh_ctx* c, int i);
QueryCounters* counter_block(nbvh_ctx* c, int block);
nbvh_status resolve_query_stats(nbvh_ctx* c);
// nbvh_train.cu
nbvh_status upload_scene(nbvh_ctx* c);
nbvh_status upload_cut(nbvh_ctx* c, int lod);
void free_scene_device(nbvh_ctx* c);
void free_train_device(nbvh_ctx* c);
nbvh_status reserve_train(nbvh_ctx* c, int64_t max_rays);
void reset_adam(nbvh_ctx* c);
}  // namespace nbvh
