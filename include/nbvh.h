/* nbvh.h — C ABI of the B200-native N-BVH neural ray-query library (libnbvh.so).
 *
 * N-BVH (Weier et al., SIGGRAPH 2024, arXiv 2405.16237).  Citations "P:n" are lines of
 * the paper's text (/root/reference/PAPER.md, read-only at build time); the readings
 * "C<k>" are listed in DESIGN.md §3.
 *
 * Problem statement: a ray goes in; a hit record of visibility,
 * depth, normal and albedo comes out, computed by traversing a cut of the scene's BVH
 * (the N-BVH) and querying a multi-resolution hash grid + MLP at the leaves
 * the ray crosses (Fig. node_encoding).  The companion training step
 * learns the grid and MLP from BVH-probed ray/response pairs.
 *
 * Conventions (all entry points):
 *  - Every call returns nbvh_status; no C++ exception crosses the ABI.  Arguments are
 *    validated before any launch; on error the call has no effect and
 *    nbvh_last_error(ctx) describes it.  After a CUDA error the context is poisoned and
 *    every later call returns NBVH_ECUDA.
 *  - "host" pointers are CPU memory, copied during the call; "device" pointers are CUDA
 *    global memory of the context's device, owned by the caller, and must stay valid
 *    until the stream work completes.  Stream arguments are cudaStream_t passed as
 *    void*; NULL is the legacy default stream.  Calls taking a stream are asynchronous
 *    and stream-ordered unless stated otherwise; calls without one are synchronous.
 *  - One context per device; a context is not thread-safe.  Multi-GPU runs use one
 *    context per process (torch.distributed launches), see DESIGN.md §7.
 */
#ifndef NBVH_H
#define NBVH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NBVH_OK = 0,
    NBVH_WARN_CLAMPED = 1,   /* request clamped (e.g. target leaves > base-BVH leaves)      */
    NBVH_EINVAL = -1,        /* bad config, size, or NULL required pointer                  */
    NBVH_ERANGE = -2,        /* LoD slot / index out of range                               */
    NBVH_ESTATE = -3,        /* call order: no mesh / no cut / no device / not reserved     */
    NBVH_ENONFINITE = -4,    /* non-finite loss or gradient: update skipped, params intact  */
    NBVH_ECUDA = -5,         /* CUDA runtime error (context poisoned)                       */
    NBVH_ENOMEM = -6         /* allocation failed                                           */
} nbvh_status;

typedef struct nbvh_ctx nbvh_ctx;

/* One ray, 32 B, array-of-structs.  d need not be unit length.  The query considers
 * t in [tmin, tmax]; tmax may be +inf. */
typedef struct {
    float ox, oy, oz, tmin;
    float dx, dy, dz, tmax;
} nbvh_ray;

/* Per-ray results, structure-of-arrays, all device pointers of n elements (normal and
 * albedo n*3).  hit: 1 if the N-BVH reports an intersection (visibility < 0.5).
 * t: world distance along the ray, +inf on a miss.  normal: unit,
 * albedo in (0,1); zeros on a miss.  leaf (nullable): winning cut-leaf id or -1.
 * n_queries (nullable): neural queries performed for the ray. */
typedef struct {
    uint8_t* hit;
    float* t;
    float* normal;
    float* albedo;
    int32_t* leaf;
    int32_t* n_queries;
} nbvh_hits;

/* Model and query configuration.  Defaults (nbvh_config_default) = BASELINE cfg 1. */
typedef struct {
    int32_t L;              /* hash-grid levels (8)                                  */
    int32_t F;              /* features per level, 2 or 4 (4)                        */
    int32_t log2_T;         /* table size T = 2^log2_T per hashed level ("hash-map size") */
    int32_t base_res;       /* coarsest resolution (8)                               */
    int32_t max_res;        /* finest resolution (1024)                              */
    int32_t n_points;       /* samples per ray segment (three; BASELINE: 4)          */
    int32_t hidden_layers;  /* hidden layers of width 64 (4; BASELINE: 2 or 3)       */
    int32_t width;          /* hidden width; must be 64                                     */
    int32_t list_cap;       /* per-ray ordered leaf-list capacity K, 1..16, default 12 (C6) */
    int32_t mode;           /* 0 = nearest confident hit (R2), 1 = first confident hit (R1) (C5) */
    float inflate_rel;      /* node inflation, fraction of node diagonal (C15: 1e-3)        */
    float inflate_abs;      /* node inflation floor, fraction of scene diagonal (C15: 1e-6) */
    uint64_t seed;          /* parameter-initialisation seed (C21)                          */
    int32_t mlp_dtype;      /* query-path MLP operands: 0 = fp16 (default), 1 = bf16 (features and
                               weights rounded to bf16, fp32 accumulation; "half precision",
                               C39); training keeps fp16 operands                          */
    int32_t reserved0;
} nbvh_config;

/* Parameter blocks for nbvh_get_params / nbvh_set_params.  All are fp32 master values;
 * the fp16 inference copy is their round-to-nearest-even conversion (C14). */
typedef enum {
    NBVH_PARAM_TABLES = 0,  /* [n_entries][F], levels concatenated, offsets from nbvh_level_table */
    NBVH_PARAM_WEIGHTS = 1, /* layer k: [out][in] row-major, layers concatenated (in: D_in, 64..; out: 64.., 8) */
    NBVH_PARAM_BIASES = 2,  /* layer k: [out], concatenated                                  */
    NBVH_PARAM_ALL = 3      /* flat: tables, weights, biases — the gradient-buffer layout    */
} nbvh_param_block;

/* Counters of the last nbvh_query / nbvh_query_host / nbvh_debug_query_trace call.  They
 * live on the device until nbvh_get_query_stats reads them back. */
typedef struct {
    int64_t n_rays;
    int64_t n_queries;       /* sum over rays of neural queries (ray, leaf) evaluated       */
    int32_t n_iters;         /* slot iterations of the busiest CTA of the persistent kernel */
    int32_t n_launches;      /* kernels launched by the call                                */
    int32_t n_refills;       /* re-traversals after a leaf-list overflow (C6)               */
    float ms_traverse;       /* device time of the traversal kernel (profiling on, else 0)  */
    float ms_query;          /* device time of the persistent query kernel (profiling on)   */
    int32_t n_mlp_tiles;     /* 128-row MLP tiles run on tcgen05 (warp-specialised kernel)  */
    int32_t n_mlp_rows;      /* rows in them (<= 128 per tile; the rest is padding)         */
    int64_t ws_cycles[3];    /* warp-specialised kernel, SM cycles summed over worker warps:
                                waiting for MLP results, waiting for a free tile, total      */
} nbvh_query_stats;

/* Training counters of the last nbvh_train_backward / nbvh_train_step. */
typedef struct {
    int64_t n_rays;          /* rays offered                                                */
    int64_t n_first_hit;     /* rays that intersect at least one cut leaf                   */
    int64_t n_accepted;      /* samples trained (P:197 acceptance)                          */
    double loss_sum;         /* sum of per-sample combined losses                   */
    double loss_terms[4];    /* sums of vis, dist, normal, albedo terms (weights 2,2,1,1 applied) */
    int32_t n_launches;
    int32_t skipped;         /* 1 if the update was rejected (non-finite)                   */
    float ms_phase[6];       /* profiling on: device time of select (T1), label (T2),
                                fwd+loss (T3-T5), bwd+scatter (T6/T7), dW (T6), Adam (T9)  */
} nbvh_train_stats;

/* ---------------------------------------------------------------- lifecycle */
void nbvh_config_default(nbvh_config* cfg);
/* cuda_device >= 0: device context; -1: host-only context (mesh, BVH and cut building
 * only — every call that needs the GPU returns NBVH_ESTATE).  Parameters are
 * initialised per C21 from cfg->seed (tables U[-1e-4,1e-4], He-uniform weights, zero biases). */
nbvh_status nbvh_create(const nbvh_config* cfg, int cuda_device, nbvh_ctx** out);
void nbvh_destroy(nbvh_ctx* ctx);
/* Context-owned message of the last failing call; valid until the next call. */
const char* nbvh_last_error(const nbvh_ctx* ctx);
/* Hash-grid level table (C1, C2): res[L], dense[L] (0/1), offset[L] (entries); host outputs. */
nbvh_status nbvh_level_table(const nbvh_ctx* ctx, int32_t* res, int32_t* dense, int64_t* offset,
                             int64_t* n_entries);
/* Number of fp32 values in a parameter block. */
nbvh_status nbvh_param_count(const nbvh_ctx* ctx, int32_t block, int64_t* n);
nbvh_status nbvh_get_params(nbvh_ctx* ctx, int32_t block, float* host_dst, int64_t n);
nbvh_status nbvh_set_params(nbvh_ctx* ctx, int32_t block, const float* host_src, int64_t n);
/* Preallocate workspaces for up to max_rays rays per nbvh_query / nbvh_train_* call. */
nbvh_status nbvh_reserve(nbvh_ctx* ctx, int64_t max_rays);

/* ---------------------------------------------------------------- scene and cut (host) */
/* Copies the mesh (host pointers): xyz [nv][3], tri [nt][3] (vertex indices), vnormal
 * [nv][3] (nullable -> area-weighted normals are generated), tri_albedo [nt][3]
 * (nullable -> 0.5 grey).  Builds the base BVH on the CPU with a full-sweep SAH builder
 * (P:271), leaves of <= 4 triangles, and uploads it for ground-truth labelling. */
nbvh_status nbvh_set_mesh(nbvh_ctx* ctx, const float* xyz, int64_t nv, const uint32_t* tri, int64_t nt,
                          const float* vnormal, const float* tri_albedo);
/* Builds a cut through the base BVH with target_leaves leaves into LoD slot
 * lod_slot (0..7).  Nodes are split greedily by rank: with leaf_q/leaf_p
 * (nullable, per current leaf of that slot) r = 2 ln q + ln p; otherwise by
 * surface area (static score).  Leaves are inflated per C15; inner boxes of the
 * shallow N-BVH hierarchy are exact unions of their children.  Returns
 * NBVH_WARN_CLAMPED if target_leaves exceeds the number of base leaves. */
nbvh_status nbvh_build_cut(nbvh_ctx* ctx, int32_t target_leaves, const float* leaf_q, const float* leaf_p,
                           int32_t lod_slot, int32_t* out_n_leaves);
/* Registers a copy of the cut in LoD slot src_lod into slot dst_lod ("we register a
 * new LoD at regular training iteration intervals"); every slot indexes the same hash grid
 * and MLP (C4').  Host + device copy; NBVH_ESTATE if the source slot is empty. */
nbvh_status nbvh_copy_cut(nbvh_ctx* ctx, int32_t src_lod, int32_t dst_lod);
/* Cut inspection (host outputs, any pointer nullable): leaf boxes (inflated) [n][3],
 * base boxes (uninflated) [n][3], leaf triangle lists in CSR form (tri_off [n+1],
 * tris [n_tris], original triangle ids), grid domain (C4). */
nbvh_status nbvh_cut_info(const nbvh_ctx* ctx, int32_t lod, int32_t* n_leaves, int32_t* n_inner);
/* The base BVH the cuts are drawn from ("base-BVH cut"; SAH), host outputs,
 * nullable: n_nodes; per node child_a / child_b (inner node: the two child indices; leaf:
 * child_b < 0, child_a = its first primitive).  Node 0 is the root.  NBVH_ESTATE without a
 * mesh. */
nbvh_status nbvh_get_base_bvh(const nbvh_ctx* ctx, int32_t* child_a, int32_t* child_b, int64_t* n_nodes);
/* The base-BVH node of every leaf of LoD slot lod, in the cut's leaf order (host int32
 * [n_leaves]).  NBVH_ERANGE / NBVH_ESTATE on a bad or empty slot. */
nbvh_status nbvh_get_cut_nodes(const nbvh_ctx* ctx, int32_t lod, int32_t* leaf_base);
nbvh_status nbvh_get_cut(const nbvh_ctx* ctx, int32_t lod, float* leaf_lo, float* leaf_hi, float* base_lo,
                         float* base_hi, int64_t* tri_off, int32_t* tris, float* dom_min, float* dom_inv);

/* ---------------------------------------------------------------- query (device) */
/* Neural ray query of n rays (device nbvh_ray[n]) against LoD slot lod: cut
 * traversal with an ordered per-ray leaf list, per-leaf segment sampling + hash-grid
 * encode + MLP, decode and front-to-back termination with ray compaction.  Results in
 * caller-owned device arrays.  Requires nbvh_reserve(n).  Asynchronous: enqueues one
 * counter reset and two kernels on `stream` and returns without synchronising; the
 * context's query workspace is reused by the next call on any stream, so concurrent
 * queries on one context must be ordered by the caller. */
nbvh_status nbvh_query(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, int32_t lod, nbvh_hits d_out,
                       void* stream);
/* Same computation from HOST rays into HOST results (the end-to-end path): the rays are
 * cut into block-interleaved chunks (6 for n >= 2^20; NBVH_HOST_WEIGHTS / NBVH_HOST_CONTIG
 * are tuning hooks) whose uploads, queries (alternating two streams with disjoint workspace
 * slices) and downloads overlap; returns after the last download (synchronous).  Host
 * buffers should be pinned for full copy bandwidth.  NBVH_HOST_TIMELINE=1 prints the chunk
 * timeline to stderr. */
nbvh_status nbvh_query_host(nbvh_ctx* ctx, const nbvh_ray* h_rays, int64_t n, int32_t lod, nbvh_hits h_out,
                            void* stream);
/* Counters of the last query call; synchronises that call's stream to read them.  Also
 * reports a traversal stack overflow (NBVH_ECUDA) detected on the device. */
nbvh_status nbvh_get_query_stats(nbvh_ctx* ctx, nbvh_query_stats* out);
/* on != 0: record CUDA events around every kernel the query launches (on the query's
 * stream) and report their durations in nbvh_query_stats. */
nbvh_status nbvh_set_profiling(nbvh_ctx* ctx, int32_t on);

/* ---------------------------------------------------------------- MLP on tcgen05 (device) */
/* The decoder MLP alone (D_in -> 64 ReLU x hidden -> 8, linear outputs) on a batch
 * of m fp16 feature rows d_x [m][D_in] (bits as uint16, 16-byte aligned) -> raw outputs d_z
 * [m][8] fp32 (16-byte aligned), with the context's fp16 weights and fp32 biases.  tcgen05
 * tensor cores (M = 128-row tiles, fp32 accumulators in TMEM, X tiles loaded by TMA); the same
 * network the fused query kernel evaluates with mma.sync.  Asynchronous on `stream`. */
nbvh_status nbvh_mlp_forward(nbvh_ctx* ctx, const uint16_t* d_x, int64_t m, float* d_z, void* stream);

/* ---------------------------------------------------------------- measurement probe (device) */
/* The random-gather roofline of SURVEY §8(d) (encode is bound by L2 random-sector reads):
 * reads n_gathers uniformly random entries (entry_bytes 4 = one sector per load, like a hashed
 * level; 32 = a corner-packed dense record) of the device table d_table (table_bytes / entry_bytes
 * must be a power of two; 32-byte aligned), 8 independent address chains per thread on a grid
 * of SMs x 8 CTAs x 256 threads, and XORs the data into d_sink (>= SMs*2048 uint32, device).
 * *n_done (host) receives the number of gathers actually issued (rounded up).  No context;
 * the caller times it (CUDA events on `stream`).  NBVH_EINVAL on bad arguments. */
nbvh_status nbvh_gather_probe(const void* d_table, int64_t table_bytes, int32_t entry_bytes, int64_t n_gathers,
                              uint32_t seed, uint32_t* d_sink, int64_t sink_len, int64_t* n_done, void* stream);
/* The same 4-byte random gathers through the texture pipe (tex1Dfetch on a texture object the
 * call creates over d_table, as the query kernel's hashed levels read the table), or with half of
 * the address chains on each pipe (mixed = 1): the gather peak of a kernel that uses both L1
 * input pipes.  table_bytes / 4 a power of two <= 2^27; 32-byte aligned.  Synchronises `stream`
 * before it destroys the texture object.  NBVH_EINVAL on bad arguments, NBVH_ECUDA when the
 * texture object cannot be created. */
nbvh_status nbvh_gather_probe_tex(const void* d_table, int64_t table_bytes, int32_t mixed, int64_t n_gathers,
                                  uint32_t seed, uint32_t* d_sink, int64_t sink_len, int64_t* n_done, void* stream);
/* The scatter roofline of SURVEY §8(d) (T7 is bound by L2 atomics): n_ops uniformly random
 * fp32 reductions (vec 1: red.global.add.f32; vec 2: red.global.add.v2.f32 on 8-byte pairs,
 * as the training backward issues for F = 2; vec 4: red.global.add.v4.f32 on 16-byte quads)
 * of +1 into the device table d_table (table_bytes / (4 vec) a power of two; 16-byte
 * aligned; its contents are modified).  *n_done
 * (host) = reductions issued.  No context; the caller times it.  NBVH_EINVAL on bad arguments. */
nbvh_status nbvh_atomic_probe(float* d_table, int64_t table_bytes, int32_t vec, int64_t n_ops, uint32_t seed,
                              int64_t* n_done, void* stream);

/* ---------------------------------------------------------------- hybrid path tracing (device) */
/* NEXT-3 (BASELINE cfg 3; PAPER §7: "a BLAS is classical or N-BVH; both
 * query types yield the same type of intersection data").
 * Classical closest-hit query of n rays (device nbvh_ray[n], interval [tmin, tmax]) against
 * the context's own triangle mesh through its SAH base BVH, with double-precision
 * Moller-Trumbore (ties: lowest triangle id, C32).  Writes the nbvh_query hit record (normal:
 * interpolated vertex normal; albedo: the triangle's; leaf: the triangle id or -1;
 * n_queries: 0).  Requires nbvh_set_mesh; NBVH_EINVAL if the base BVH is deeper than 63
 * levels.  Asynchronous on `stream`. */
nbvh_status nbvh_intersect_mesh(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, nbvh_hits d_out, void* stream);
/* One wavefront step of the hybrid path tracer: for every ray with tmin <= tmax, take the
 * closer of the neural record d_neural and the classical record d_classical (d_classical.hit
 * may be NULL: no classical BLAS); an escaped ray adds throughput * sky(direction) to
 * d_radiance [n][3] (sky = host float[6]: horizon rgb, zenith rgb, blended by elevation) and
 * ends; a hit multiplies d_throughput [n][3] by the albedo (diffuse BSDF) and continues from
 * p + eps * n along a cosine-weighted direction drawn from a counter-based hash of
 * (seed, ray index, bounce).  d_next [n] receives the next rays (ended rays: tmin 1 > tmax 0);
 * *d_alive (device int32) is incremented by the number of continuing rays.  Asynchronous. */
nbvh_status nbvh_pt_shade(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, nbvh_hits d_neural, nbvh_hits d_classical,
                          float* d_throughput, float* d_radiance, nbvh_ray* d_next, uint64_t seed, int32_t bounce,
                          const float* sky, float eps, int32_t* d_alive, void* stream);

/* ---------------------------------------------------------------- two-level hierarchy (device) */
/* NEXT-3, PAPER §7: "a TLAS holds several BLAS; a BLAS is classical or N-BVH; both
 * query types yield the same type of intersection data".  An instance places one BLAS in the
 * world: world_to_object = row-major 3x4 [A | b] (x_object = A x_world + b; the same ray
 * parameter t in both spaces, d_object = A d_world, so hit distances need no conversion),
 * lo/hi = its world-space box, blas = the caller's BLAS number (< NBVH_MAX_BLAS). */
#define NBVH_MAX_BLAS 8
typedef struct {
    float world_to_object[12];
    float lo[3], hi[3];
    int32_t blas;
    int32_t pad;
} nbvh_instance;                                                    /* 80 bytes */
typedef struct nbvh_tlas nbvh_tlas;                                 /* opaque, device-resident */
/* Builds the TLAS: a binary BVH over the instances' world boxes (median split of the box
 * centres on the longest axis), uploaded to the context's device.  h_inst: host array of
 * n_inst (1..4096) instances, copied.  NBVH_EINVAL / NBVH_ERANGE on bad boxes / blas index. */
nbvh_status nbvh_tlas_build(nbvh_ctx* ctx, const nbvh_instance* h_inst, int32_t n_inst, nbvh_tlas** out);
void nbvh_tlas_destroy(nbvh_tlas* tlas);
/* TLAS traversal of m world rays d_rays [m]: for every instance whose box a ray crosses
 * within [tmin, tmax], the ray transformed into the instance's object space is appended to
 * that instance's BLAS list: d_out_rays [n_blas][cap] (object-space rays, same tmin/tmax),
 * d_out_src [n_blas][cap] (index of the world ray), d_out_inst [n_blas][cap] (instance),
 * d_counts [n_blas] (entries appended; zeroed first; a list overflowing cap raises the flag
 * read by nbvh_tlas_overflow).  Device pointers; asynchronous. */
nbvh_status nbvh_tlas_dispatch(nbvh_ctx* ctx, nbvh_tlas* tlas, const nbvh_ray* d_rays, int64_t m,
                               nbvh_ray* d_out_rays, int32_t* d_out_src, int32_t* d_out_inst, int32_t* d_counts,
                               int64_t cap, void* stream);
/* Closest hit per world ray over the BLAS answers: h_lists (host array, n_blas entries) holds
 * each BLAS's hit record for its dispatched list (entry j answers list entry j); the nearest
 * hit t wins (ties: lower BLAS number, then lower entry), its normal is brought back to world
 * space (A^T n, normalised); d_out [m] world hit record, leaf = the winning instance (or -1).
 * cap < 2^24.  Asynchronous. */
nbvh_status nbvh_tlas_merge(nbvh_ctx* ctx, nbvh_tlas* tlas, int64_t m, const int32_t* d_counts, int64_t cap,
                            const int32_t* d_src, const int32_t* d_inst, const nbvh_hits* h_lists,
                            nbvh_hits d_out, void* stream);
/* Host flag: 1 = a dispatch list overflowed its capacity, 2 = TLAS stack overflow (since
 * the build).  Synchronous. */
nbvh_status nbvh_tlas_overflow(nbvh_ctx* ctx, nbvh_tlas* tlas, int32_t* h_flag);
/* One wavefront step over COMPACTED alive paths: path i has world ray d_rays[i],
 * hit record d_hits[i], pixel d_pixel[i] and throughput d_thr[i][3].  Escaped paths add
 * throughput x sky (horizon-to-zenith gradient, sky[6]) to d_radiance[pixel][3] (atomic);
 * hits continue diffusely (throughput *= albedo, cosine-weighted direction from a
 * counter-based hash of (seed, pixel, bounce)) and are appended to d_next_rays / d_next_pixel /
 * d_next_thr at slots counted by *d_next_count (device, not reset).  Asynchronous. */
nbvh_status nbvh_pt_shade_compact(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t m, nbvh_hits d_hits,
                                  const int32_t* d_pixel, const float* d_thr, float* d_radiance,
                                  nbvh_ray* d_next_rays, int32_t* d_next_pixel, float* d_next_thr,
                                  int32_t* d_next_count, uint64_t seed, int32_t bounce, const float* sky,
                                  float eps, void* stream);

/* ---------------------------------------------------------------- training (device) */
/* T0: n training rays and the method's random draws for rays
 * [i0, i0 + n) of training step `step`, from the counter-based generator Philox-4x32-10
 * (counter = (global ray index, draw, step lo, step hi), key = seed): origins uniform in the
 * box (host float[6] lo xyz, hi xyz; NULL: the scene's bounding box with each axis extent
 * x1.5 about its centre, "50%-inflated scene bounding box", C16), directions uniform on the sphere (z = 1 - 2U, phi = 2 pi U), tmin 0,
 * tmax +inf -> d_rays [n]; acceptance draws -> d_u [n]; stratification jitter ->
 * d_xi [n][n_points] (U = (x >> 8) * 2^-24).  Global indexing makes data-parallel shards
 * (i0 = shard start) reproduce the single-process batch.  Device pointers; asynchronous.
 * NBVH_EINVAL on bad arguments or n_points > 4, NBVH_ESTATE if box is NULL and no mesh is set. */
nbvh_status nbvh_gen_train_rays(nbvh_ctx* ctx, uint64_t seed, uint64_t step, int64_t i0, int64_t n,
                                const float* box, nbvh_ray* d_rays, float* d_u, float* d_xi, void* stream);
/* Forward + backward of one training batch into the context's
 * fp32 gradient buffer (overwritten): for each ray the first intersected cut leaf of
 * LoD `lod` is accepted with probability max(r_hat/r_hat_max, 0.005) (C18)
 * using the caller's draws d_u[n] in [0,1); accepted segments are labelled by
 * intersecting that leaf's triangles (C17), sampled with jitter d_xi[n][n_points]
 * (C8), encoded, decoded, and the gated weighted loss (C19) is
 * back-propagated into the MLP and hash tables.  The gradient is of the SUM of
 * per-sample losses; nbvh_apply_update divides by the accepted-sample count.
 * d_rays/d_u/d_xi are device pointers. */
nbvh_status nbvh_train_backward(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, const float* d_u,
                                const float* d_xi, int32_t lod, void* stream);
/* The flat fp32 gradient buffer (device, context-owned, NBVH_PARAM_ALL layout) followed
 * by one float holding the accepted-sample count and n_leaves*3 per-leaf statistics
 * (loss sum, sample count, first-hit count) of the cut the batch was drawn on.  Data-parallel training all-reduces (sum) n_floats values
 * in place between nbvh_train_backward and nbvh_apply_update. */
nbvh_status nbvh_grad_buffer(nbvh_ctx* ctx, float** d_grad, int64_t* n_floats);
/* Adam step (C20) on every parameter with gradient g / max(1, accepted count
 * read from the buffer tail); refreshes the fp16 inference copy.  A non-finite
 * gradient skips the update (NBVH_ENONFINITE reported by nbvh_get_train_stats). */
nbvh_status nbvh_apply_update(nbvh_ctx* ctx, float lr, void* stream);
/* backward + apply_update on one rank.  d_rays, d_u and d_xi all NULL: the library draws
 * the n training rays and random numbers itself (T0: nbvh_gen_train_rays with key = the
 * config's seed, step = the context's self-drawn batch count, the C16 box), into
 * context-owned buffers. */
nbvh_status nbvh_train_step(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, const float* d_u,
                            const float* d_xi, int32_t lod, float lr, void* stream);
/* Counters of the last training call; synchronises the stream first. */
nbvh_status nbvh_get_train_stats(nbvh_ctx* ctx, nbvh_train_stats* out);
/* Per-leaf acceptance ranks r (C18) used by nbvh_train_backward (host, n_leaves floats). */
nbvh_status nbvh_set_leaf_rank(nbvh_ctx* ctx, int32_t lod, const float* h_rank);

/* ---------------------------------------------------------------- parity hooks (device) */
/* The same kernels with intermediate results exposed. */
/* Ordered leaf lists: leaf/t_enter/t_exit [n][cap] (row-major, -1 / 0 past the end),
 * count[n] = total intersected leaves (may exceed cap). */
nbvh_status nbvh_debug_traverse(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, int32_t lod, int32_t cap,
                                int32_t* d_leaf, float* d_t_enter, float* d_t_exit, int32_t* d_count,
                                void* stream);
/* The PRODUCT traversal (k_traverse, the kernel nbvh_query launches)
 * with the context's list capacity K = list_cap, unpacked per ray: leaf/te/tx [n][K]
 * (device; the first fill[r] entries of ray r in (t_enter, id) order, the rest -1 / 0),
 * fill [n] (entries kept, <= K) and more [n] (1 if further intersected leaves may exist
 * beyond the K-th key: the query kernel then resumes the traversal, C6).  Uses the
 * context's query workspace (n <= nbvh_reserve).  Asynchronous on `stream`. */
nbvh_status nbvh_debug_traverse_product(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, int32_t lod,
                                        int32_t* d_leaf, float* d_te, float* d_tx, int32_t* d_fill,
                                        int32_t* d_more, void* stream);
/* Encode m points already normalised to [0,1]^3 (float [m][3]): fp16 features
 * [m][L*F] (bits as uint16) and corner indices [m][L][8] (nullable). */
nbvh_status nbvh_debug_encode(nbvh_ctx* ctx, const float* d_points, int64_t m, uint16_t* d_feat,
                              uint32_t* d_index, void* stream);
/* The query kernel's own per-warp MLP on m input rows [m][D_in] (fp16 bits; bf16 bits
 * when mlp_dtype = 1) -> raw outputs z [m][8] (fp32). */
nbvh_status nbvh_debug_mlp(nbvh_ctx* ctx, const uint16_t* d_in, int64_t m, float* d_z, void* stream);
/* nbvh_query that also records the raw MLP output of every query: z_trace [n][cap][8]
 * (fp32, NaN where not queried, positions >= cap not recorded). */
nbvh_status nbvh_debug_query_trace(nbvh_ctx* ctx, const nbvh_ray* d_rays, int64_t n, int32_t lod,
                                   nbvh_hits d_out, float* d_z_trace, int32_t cap, void* stream);
/* Ground-truth labels of the last training batch: gt [n][9] = vis, t_local, normal,
 * albedo, t_hit (vis=1: no hit) with accepted[n] and first-leaf ids (device). */
nbvh_status nbvh_debug_train_samples(nbvh_ctx* ctx, float* d_gt, uint8_t* d_accepted, int32_t* d_leaf,
                                     float* d_loss, void* stream);
/* Parity capture of the training forward (T4): enable != 0 makes the following
 * nbvh_train_backward calls also store every sample's raw MLP output z (fp32, a
 * context-owned [max_rays][8] buffer allocated on the next call); enable = 0 frees it.
 * Off by default: the product path does not write z. */
nbvh_status nbvh_debug_train_capture(nbvh_ctx* ctx, int32_t enable);
/* Per-sample intermediates of the last training batch (P:142 forward/backward; T3-T6), in
 * the kernel's compacted sample order; *h_m (host) receives the sample count m (the call
 * synchronises `stream` to read it).  Device outputs, each nullable: d_sample_ray [m] ray
 * index of each sample; d_x [m][D_in] fp16 features (T3, bits as uint16); d_z [m][8] raw
 * MLP outputs (T4; needs nbvh_debug_train_capture on, else NBVH_ESTATE); d_dz [m][8] dL/dz
 * (T5); d_act [hidden][m][64] fp16 post-ReLU hidden activations (T4: the kernel's ReLU
 * decisions are act > 0); d_delta [hidden][m][64] fp16 deltas dL/d(pre-activation) of each
 * hidden layer (T6).  Buffers must hold the capacity implied by m (callers size them from
 * the ray count, an upper bound). */
nbvh_status nbvh_debug_train_activations(nbvh_ctx* ctx, int32_t* d_sample_ray, uint16_t* d_x, float* d_z,
                                         float* d_dz, uint16_t* d_act, uint16_t* d_delta, int64_t* h_m,
                                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NBVH_H */
