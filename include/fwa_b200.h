/*
 * fwa_b200.h — C ABI of the B200-native FlatFormer backbone (flattened window
 * attention) hot path.  Plain pointers and sizes only; no torch types.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *
 *   fwa_b200_backbone_forward        fwa::backbone::run_backbone(PillarSet, FwaConfig,
 *                                    BackboneParams, n_threads)   include/fwa/backbone.hpp:159-325
 *   fwa_b200_backbone_forward_device the same, inputs/outputs already in HBM
 *   fwa_b200_backbone_forward_batch  the same over F independent frames (one model), frame-
 *                                    parallel inside one GPU (BASELINE config 3)
 *   fwa_b200_backbone_forward_frames a stream of frames (one run_backbone each), PCIe copies
 *                                    pipelined with compute; = run_backbone per frame
 *                                    include/fwa/backbone.hpp:159-325
 *   fwa_b200_sort_plan               fwa::flatten::sort(coords, WindowSpec)  include/fwa/flatten.hpp:97-120
 *   fwa_b200_block_forward           fwa::kernels::fwa_block_forward(f, pe, params, n_groups)
 *                                    include/fwa/kernels.hpp:636-650
 *   fwa_b200_positional_embedding    fwa::kernels::positional_embedding  include/fwa/kernels.hpp:364-393
 *   fwa_b200_load_params             fwa::kernels::load_params (FWAP records)  include/fwa/kernels.hpp:177-206
 *                                    + fwa::kernels::validate  kernels.hpp:75-90
 *   fwa_b200_load_input_proj         BackboneParams::input_proj  include/fwa/backbone.hpp:74-81, 179-190
 *   fwa_b200_pillarize[_device]      fwa::geometry::pillarize on the GPU  include/fwa/geometry.hpp:246-300
 *   fwa_b200_row_checksums           `fwa attend` row_checksums  tools/fwa_cli.cpp:214-218
 *   fwa_b200_block_backward          fwa::kernels::fwa_block_backward  include/fwa/kernels.hpp:660-765
 *   fwa_b200_equal_window_forward    fwa::bench::bench_equal_window (padded SST-style baseline)
 *                                    include/fwa/bench.hpp:266-326
 *   fwa_b200_generate_points         fwa::geometry::generate_synthetic  include/fwa/geometry.hpp:355-386
 *   fwa_b200_pillar_params           fwa::geometry::random_pillar_params  include/fwa/geometry.hpp:71-79
 *   fwa_b200_generate_pillars        fwa::geometry::generate_synthetic + pillarize +
 *                                    random_pillar_params  include/fwa/geometry.hpp:355-386, 246-300, 71-79
 *   fwa_b200_init_params             fwa::backbone::init_backbone_params  include/fwa/backbone.hpp:83-102
 *
 * Status codes mirror the reference exception taxonomy (include/fwa/error.hpp:11-33),
 * which the reference CLI maps to exit codes 2 (config/parse/schema/shape) and
 * 3 (numeric/contract/other) (tools/fwa_cli.cpp:514-529).
 */
#ifndef FWA_B200_H
#define FWA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fwa_status {
    FWA_OK = 0,
    FWA_ERR_CONFIG = 1,   /* fwa::config_error   */
    FWA_ERR_PARSE = 2,    /* fwa::parse_error    */
    FWA_ERR_SCHEMA = 3,   /* fwa::schema_error   */
    FWA_ERR_SHAPE = 4,    /* fwa::shape_error    */
    FWA_ERR_NUMERIC = 5,  /* fwa::numeric_error  */
    FWA_ERR_CONTRACT = 6, /* fwa::contract_error */
    FWA_ERR_INTERNAL = 7,
    FWA_ERR_CUDA = 8      /* CUDA runtime / launch failure (no reference analogue) */
};

/* Arithmetic mode of the feature path.  Integer outputs (sort, groups, drops,
 * kept set, cache stats) are bit-exact in both modes. */
enum fwa_precision {
    FWA_PREC_BF16 = 0, /* tcgen05/TMEM GEMMs + mma.sync attention, bf16 operands, fp32
                          accumulate / LN / softmax / residual (default) */
    FWA_PREC_FP32 = 1, /* fp32 FFMA check mode (tolerance 1e-4) */
    FWA_PREC_BF16_3K = 2 /* bf16 numerics as FWA_PREC_BF16, but the three-kernel block pipeline
                            instead of the fused CTA-pair block kernel (A/B and regression) */
};

/* fwa::backbone::FwaConfig (backbone.hpp:22-34).  Window metres are
 * window_p{x,y} * resolution computed in fp64, exactly as window_x_m(). */
typedef struct fwa_config {
    double resolution;
    int32_t window_px, window_py;
    int32_t group_size;
    int32_t n_blocks;
    int32_t d_model, n_heads, d_ff;
} fwa_config_t;

/* fwa::backbone::BackboneOutput (backbone.hpp:128-135); caller-allocated.
 * features: capacity N*d_model (rows in ascending-id "active" order);
 * kept_indices: capacity N; dropped_ids: capacity N (per block, in sorted
 * tail order, blocks concatenated); dropped_per_block: n_blocks;
 * block_perms (optional, may be NULL; single-frame calls only): n_blocks x N,
 * row b holds block b's permutation as local indices into that block's
 * active list (the parity hook for flatten::sort/group).
 * stage_ms: StageTimes (backbone.hpp:109-126) of this call, device time measured with
 * CUDA events on the context stream, in FWA_STAGE_* order.  sort = the window sorts
 * (keys, bins, per-bin exact sort), group = groups / drops / kept set (compaction);
 * the fused block kernel does gather .. scatter in ONE launch, so its event time is
 * apportioned to gather / attention / ffn / scatter by the kernel's own per-phase
 * SM-clock counters.  Written by the host-buffer entry points. */
enum fwa_stage {
    FWA_STAGE_SORT = 0,
    FWA_STAGE_GROUP = 1,
    FWA_STAGE_GATHER = 2,
    FWA_STAGE_ATTENTION = 3,
    FWA_STAGE_FFN = 4,
    FWA_STAGE_SCATTER = 5,
    FWA_STAGES = 6
};
typedef struct fwa_output {
    float* features;
    int32_t* kept_indices;
    int32_t* dropped_ids;
    int32_t* dropped_per_block;
    int32_t* block_perms;
    int64_t n_kept;
    int32_t cache_computed; /* SortStats::sorts_computed (flatten.hpp:82-86) */
    int32_t cache_hits;     /* SortStats::cache_hits */
    double stage_ms[FWA_STAGES];
} fwa_output_t;

/* Per-frame results of a batch call: each frame is its own run_backbone, so each has
 * its own kept count, block-0 drop count (N mod G; later blocks drop nothing: K is a
 * multiple of G) and sort-cache statistics (the reference rule, backbone.hpp:224-234,
 * 285-316, evaluated on that frame's N). */
typedef struct fwa_frame_stats {
    int64_t n_kept;
    int32_t n_dropped;
    int32_t cache_computed, cache_hits;
} fwa_frame_stats_t;

typedef struct fwa_b200_ctx fwa_b200_ctx;

/* One context per device; all work is enqueued on `cuda_stream` (a
 * cudaStream_t; NULL = the context creates its own).  Calls on one context are
 * serialised on that stream; contexts on different devices run concurrently. */
int fwa_b200_ctx_create(int device, void* cuda_stream, fwa_b200_ctx** out);
/* The calling thread's current CUDA device (cudaGetDevice; 0 if none is set). */
int fwa_b200_current_device(void);
void fwa_b200_ctx_destroy(fwa_b200_ctx* ctx);
const char* fwa_b200_last_error(const fwa_b200_ctx* ctx);
int fwa_b200_set_precision(fwa_b200_ctx* ctx, int precision);
/* Number of CUDA kernels this context has launched so far (telemetry). */
int64_t fwa_b200_kernel_launches(const fwa_b200_ctx* ctx);
/* Synchronise the context stream and report deferred device-side conditions of the
 * last device-resident forward (fwa_b200_backbone_forward_device enqueues without a
 * host round trip): FWA_ERR_NUMERIC for non-finite inputs (kernels.hpp:460-461),
 * FWA_ERR_INTERNAL if the frame set's window range exceeded the fixed-capacity bin
 * histogram (re-run through fwa_b200_backbone_forward, which falls back automatically). */
int fwa_b200_sync_check(fwa_b200_ctx* ctx);

/* Stage timers on the context stream (CUDA events), the analogue of the
 * reference's StageTimer/StageTimes (backbone.hpp:109-151).  Enabling resets the
 * accumulators; fwa_b200_get_profile synchronises the stream and returns the
 * accumulated milliseconds and call counts per slot (arrays of FWA_PROF_SLOTS). */
enum fwa_prof_slot {
    FWA_PROF_SCHEDULE = 0,     /* window sorts + groups + drops + kept set (sort/group stages) */
    FWA_PROF_PE = 1,           /* positional embedding */
    FWA_PROF_LN_QKV = 2,       /* gather + LN1 + PE + packed QKV */
    FWA_PROF_ATTENTION = 3,    /* per-group MHSA */
    FWA_PROF_OUTPROJ_FFN = 4,  /* out-proj + residual + LN2 + FFN + residual + scatter */
    FWA_PROF_H2D = 5,
    FWA_PROF_D2H = 6,
    FWA_PROF_BLOCK = 7,        /* the fused one-launch block kernel (gather .. scatter) */
    FWA_PROF_SLOTS = 8
};
int fwa_b200_set_profiling(fwa_b200_ctx* ctx, int enable);
int fwa_b200_get_profile(fwa_b200_ctx* ctx, double* ms, int64_t* counts);

/* 1 if the tcgen05 bf16 path serves `cfg`, 0 if the fp32 SIMT kernels do. */
int fwa_b200_fast_path(const fwa_b200_ctx* ctx, const fwa_config_t* cfg);

/* Parse n_blocks back-to-back FWAP records (kernels.hpp:149-206), validate
 * shapes against cfg (config_error / shape_error / parse_error as the
 * reference), upload fp32 + bf16 copies to HBM.  Params stay resident. */
int fwa_b200_load_params(fwa_b200_ctx* ctx, const fwa_config_t* cfg, const void* fwap_blob,
                         size_t blob_len);

/* BackboneParams::input_proj (backbone.hpp:74-81, 179-190): weight d_model x f_in
 * (row-major fp32), bias d_model (NULL = zeros).  Resident like the block params;
 * f_in == 0 removes it.  The group-range split API (fwa_b200_split_*) takes d_model rows
 * and refuses to run while a projection is loaded (FWA_ERR_CONTRACT).  While one is loaded, the feats of every backbone_forward*
 * call are N x f_in (f64 or f32; the device-resident entry point: f32) and are projected
 * to d_model on the device, bit-exact with the reference's fp32 loop (acc = bias[j];
 * acc += w[j][c] * (float)x[c] in c order, no FMA contraction). */
int fwa_b200_load_input_proj(fwa_b200_ctx* ctx, int32_t d_model, int32_t f_in, const float* weight,
                             const float* bias);

/* run_backbone with HOST buffers: coords N x 2 f64 (pillar centres),
 * feats N x d_model, f64 if feats_is_f64 (cast to f32 on device exactly as
 * backbone.hpp:195-196) else f32.  Blocks until `out` is filled. */
int fwa_b200_backbone_forward(fwa_b200_ctx* ctx, const double* coords, const void* feats,
                              int feats_is_f64, int64_t n, const fwa_config_t* cfg,
                              fwa_output_t* out);

/* Same over F frames concatenated along rows: frame f owns rows
 * [frame_offsets[f], frame_offsets[f+1]).  Each frame is an independent
 * run_backbone (own sort, groups, drops); outputs are concatenated per frame
 * (kept ids and dropped ids are global row ids, dropped ids frame by frame);
 * out->n_kept is the total, out->dropped_per_block the sums over frames,
 * out->cache_* are frame 0's; per_frame (optional, capacity F) receives every
 * frame's own counts and cache statistics. */
int fwa_b200_backbone_forward_batch(fwa_b200_ctx* ctx, const double* coords, const void* feats,
                                    int feats_is_f64, const int64_t* frame_offsets, int n_frames,
                                    const fwa_config_t* cfg, fwa_output_t* out,
                                    fwa_frame_stats_t* per_frame);

/* A stream of F independent frames in separate host buffers, each exactly one
 * fwa_b200_backbone_forward (same outputs, same errors), pipelined: frame f+1's inputs
 * cross PCIe and frame f-1's outputs come back while frame f computes.  outs[f] as for
 * fwa_b200_backbone_forward (block_perms must be NULL): a caller's loop of
 * fwa::backbone::run_backbone over a frame sequence (include/fwa/backbone.hpp:159-325). */
int fwa_b200_backbone_forward_frames(fwa_b200_ctx* ctx, int n_frames, const double* const* coords,
                                     const void* const* feats, int feats_is_f64, const int64_t* n,
                                     const fwa_config_t* cfg, fwa_output_t* outs);

/* Device-resident variant (inputs already in HBM, outputs written to HBM,
 * enqueued on the context stream without a trailing host sync).  d_feats is
 * f32.  d_out_features: capacity N*d_model; d_out_kept: capacity N (may be
 * NULL).  *n_kept_out is known on the host before the call returns (it depends
 * only on N and group_size).  Single frame, or batch when frame_offsets != NULL. */
int fwa_b200_backbone_forward_device(fwa_b200_ctx* ctx, const double* d_coords,
                                     const float* d_feats, const int64_t* frame_offsets,
                                     int n_frames, const fwa_config_t* cfg,
                                     float* d_out_features, int32_t* d_out_kept,
                                     int64_t* n_kept_out);

/* Group-range split of ONE scene across ranks (BASELINE config 4), device buffers:
 *  split_begin:   build the full index schedule + PE from replicated coordinates (every
 *                 rank gets the identical schedule); *k_out = kept rows K.
 *  split_block:   block b over groups [group_begin, group_end) of its window-sort order:
 *                 reads d_x (pillar-id rows; block 0: the caller's f32 input), writes the
 *                 (group_end - group_begin)*G sorted-order output rows to d_y (local rows;
 *                 the all-gather of the ranks' d_y in rank order is the block's K x D output).
 *  split_scatter: after the caller's all-gather of d_y (NCCL), write the K rows back to
 *                 pillar-id order in d_dst (the next block's d_x), or -- for the last
 *                 block -- to active (ascending-id) order, the backbone output.
 * Block b's rows depend on every row of block b-1 (each block re-sorts), hence the
 * exchange between blocks (flatten.hpp:150-161, backbone.hpp:215-317). */
int fwa_b200_split_begin(fwa_b200_ctx* ctx, const double* d_coords, int64_t n, const fwa_config_t* cfg,
                         int64_t* k_out);
int fwa_b200_split_block(fwa_b200_ctx* ctx, int block, int64_t group_begin, int64_t group_end,
                         const float* d_x, float* d_y);
int fwa_b200_split_scatter(fwa_b200_ctx* ctx, int block, const float* d_y, float* d_dst);
/* block's window-sort order (K pillar ids, host buffer): lets the ranks derive, from the
 * replicated schedule, exactly which rows each peer needs for the next block (the
 * all-to-all exchange of split.py) */
int fwa_b200_split_plan(fwa_b200_ctx* ctx, int block, int32_t* ids_out);
/* the same into a device buffer (K int32), enqueued on the context stream */
int fwa_b200_split_plan_device(fwa_b200_ctx* ctx, int block, int32_t* d_ids_out);

/* Peer-memory variant of the split (the exchange fused into the block kernel): instead of a
 * collective between blocks, rank r's block-b kernel writes every output row straight into
 * the x buffer (N x d_model f32, pillar-id order) of the rank whose block-(b+1) group range
 * holds that pillar -- NVLink peer memory (x_peers from fwa_b200_ipc_open), so the transfer
 * overlaps the block's compute row by row; the last block writes every row into rank 0's
 * output buffer (out_peers[0], K x d_model, active order).  Between blocks the caller only
 * orders the ranks (e.g. a 1-element NCCL all-reduce on the context stream).
 *  p2p_setup: after split_begin; world <= 8; x_peers / out_peers: `world` device pointers
 *             valid in this process (this rank's own at [rank]); builds the per-block
 *             rank-tagged scatter rows of this rank's group range (split.py partition_groups).
 *  block_p2p: block b over this rank's range; d_x = block 0: the input rows (N x d_model f32,
 *             pillar-id order), later blocks: this rank's x buffer (x_peers[rank]).
 * bf16 fused path only (FWA_ERR_CONTRACT otherwise); < 2^28 pillars. */
int fwa_b200_split_p2p_setup(fwa_b200_ctx* ctx, int world, int rank, float* const* x_peers,
                             float* const* out_peers);
int fwa_b200_split_block_p2p(fwa_b200_ctx* ctx, int block, const float* d_x);

/* Device memory that can be shared across processes (cudaMalloc'd, so IPC handles refer to
 * the allocation base) and its CUDA IPC handles: export with fwa_b200_ipc_handle
 * (FWA_IPC_HANDLE_BYTES), open in a peer process with fwa_b200_ipc_open. */
#define FWA_IPC_HANDLE_BYTES 64
void* fwa_b200_alloc(fwa_b200_ctx* ctx, size_t bytes);
void fwa_b200_free(fwa_b200_ctx* ctx, void* d_ptr);
int fwa_b200_ipc_handle(fwa_b200_ctx* ctx, void* d_ptr, void* handle_out);
int fwa_b200_ipc_open(fwa_b200_ctx* ctx, const void* handle, void** d_ptr_out);
int fwa_b200_ipc_close(fwa_b200_ctx* ctx, void* d_ptr);

/* flatten::sort (minimum slice): host coords in, host permutation out. */
int fwa_b200_sort_plan(fwa_b200_ctx* ctx, const double* coords, int64_t n, double w_x,
                       double w_y, int shift, int major_axis_y, int32_t* perm_out);

/* fwa_block_forward on pre-grouped host rows f, pe (rows x D f32; rows =
 * n_groups * G) with ONE FWAP record.  Uses the context precision. */
int fwa_b200_block_forward(fwa_b200_ctx* ctx, const float* f, const float* pe, int64_t rows,
                           int32_t n_groups, const void* fwap_record, size_t record_len,
                           float* out);

/* positional_embedding: host coords N x 2 f64 -> host N x d f32. */
int fwa_b200_positional_embedding(fwa_b200_ctx* ctx, const double* coords, int64_t n,
                                  int32_t d_model, float* out);
/* the bf16 fast path's fp16 PE rows (IEEE binary16 bits, N x d), for parity tests */
int fwa_b200_positional_embedding_f16(fwa_b200_ctx* ctx, const double* coords, int64_t n,
                                      int32_t d_model, uint16_t* out);

/* geometry::pillarize (geometry.hpp:246-300) on the GPU: points x,y (n x 2 f64) +
 * features (n x f_in f64) -> pillars in ascending lexicographic (x-cell, y-cell) order,
 * members mean-pooled with the reference's pairwise summation in ingestion order, then
 * gelu(bias + W pooled) (W: d_out x f_in, bias may be NULL = zeros).  Cell order and
 * coordinates are bit-exact; features use the reference's fp64 operation order (CUDA erf
 * for libm erf).  coords_out == NULL only counts.  Host buffers; *n_pillars = P. */
int fwa_b200_pillarize(fwa_b200_ctx* ctx, const double* xy, const double* feats, int64_t n, int32_t f_in,
                       double resolution, const double* weight, const double* bias, int32_t d_out,
                       double* coords_out, double* feats_out, int64_t* n_pillars);
/* The same with device buffers (capacity = rows available in the outputs; n is always
 * enough), so the pillars can feed fwa_b200_backbone_forward_device directly. */
int fwa_b200_pillarize_device(fwa_b200_ctx* ctx, const double* d_xy, const double* d_feats, int64_t n,
                              int32_t f_in, double resolution, const double* d_weight, const double* d_bias,
                              int32_t d_out, double* d_coords_out, double* d_feats_out, int64_t capacity,
                              int64_t* n_pillars);

/* fwa_block_forward (cached) + fwa_block_backward (kernels.hpp:636-765) on the GPU, fp32,
 * deterministic: f, pe, grad_out are rows x d (n_groups blocks of G consecutive rows);
 * grad_f (rows x d) and grad_record (one FWAP record of the parameter gradients, the
 * record's size, may be NULL) are host buffers. */
int fwa_b200_block_backward(fwa_b200_ctx* ctx, const float* f, const float* pe, int64_t rows, int32_t n_groups,
                            const void* record, size_t record_len, const float* grad_out, float* grad_f,
                            void* grad_record);

/* Equal-window (SST-style) padded baseline (bench.hpp:266-326, workload.hpp:44-142):
 * partition by window (X axis, no shift), bucket windows by occupancy (bucket_edges,
 * strictly increasing, <= 8), pad each window to its bucket's largest occupancy with zero
 * rows, run block 0 of the loaded params per bucket with G = pad (the same kernels as
 * the equal-size path).  Device buffers; d_out = N x d_model features of the real rows
 * (input order).  The report mirrors WorkloadReport. */
typedef struct fwa_ew_report {
    int64_t n_windows;
    int32_t max_occ, min_nonzero_occ;
    double padding_factor; /* padded / actual attention MACs (workload.hpp:24-30, 92-142) */
    int64_t rows_padded;   /* rows pushed through the block kernel (sum of windows x pad) */
    int32_t n_buckets;
    int32_t bucket_edge[8], bucket_pad[8];
    int64_t bucket_windows[8];
} fwa_ew_report_t;
int fwa_b200_equal_window_forward(fwa_b200_ctx* ctx, const double* d_coords, const float* d_feats, int64_t n,
                                  const fwa_config_t* cfg, const int32_t* bucket_edges, int32_t n_edges,
                                  float* d_out, fwa_ew_report_t* report);

/* FNV-1a-64 of a byte string (bench.hpp:62-72): the `fwa attend` feature_hash over the
 * f32 feature bytes and the config_digest over the config JSON (host). */
uint64_t fwa_b200_fnv1a64(const void* bytes, size_t n);
/* `fwa attend` row checksums (tools/fwa_cli.cpp:214-218) of device features (n x d f32)
 * into device doubles: sum = 0.0; sum += (double)f[c] in column order -- bit-exact. */
int fwa_b200_row_checksums(fwa_b200_ctx* ctx, const float* d_features, int64_t n, int32_t d, double* d_out);

/* ---- host-side input generators (bit-identical to the reference's) ---- */

/* geometry::SceneSpec (geometry.hpp:310-319). */
typedef struct fwa_scene_spec {
    int32_t n_clusters, points_per_cluster_min, points_per_cluster_max;
    double cluster_sigma, extent_x, extent_y;
    int32_t n_background, f_in;
} fwa_scene_spec_t;

/* generate_synthetic(spec, seed) -> pillarize(cloud, resolution,
 * random_pillar_params(f_in, d_out, param_seed)).  Two-phase: call with
 * coords == NULL to get the pillar count, then again with buffers
 * (coords N x 2 f64, feats N x d_out f64).  Returns N or -status. */
int64_t fwa_b200_generate_pillars(const fwa_scene_spec_t* spec, uint64_t seed, double resolution,
                                  int32_t d_out, uint64_t param_seed, double* coords,
                                  double* feats);

/* generate_synthetic(spec, seed) raw point cloud: returns n; xy (n x 2) and feats
 * (n x f_in) filled when xy != NULL. */
int64_t fwa_b200_generate_points(const fwa_scene_spec_t* spec, uint64_t seed, double* xy, double* feats);
/* random_pillar_params(f_in, d_out, seed) weight (d_out x f_in, N(0, 0.5^2)); bias is 0.
 * Returns d_out * f_in or -status. */
int64_t fwa_b200_pillar_params(int32_t f_in, int32_t d_out, uint64_t seed, double* weight);

/* init_backbone_params(cfg, f_in == d_model, seed) as FWAP records.  Returns
 * the blob length (out may be NULL to size) or -status. */
int64_t fwa_b200_init_params(const fwa_config_t* cfg, uint64_t seed, void* out, size_t cap);
/* init_backbone_params(cfg, f_in, seed) for any input width: when f_in != d_model the
 * input projection weight (d_model x f_in, N(0, 0.1^2); its bias is 0) is drawn first into
 * proj_weight, as the reference does, then the FWAP records. */
int64_t fwa_b200_init_params_fin(const fwa_config_t* cfg, int32_t f_in, uint64_t seed, void* out, size_t cap,
                                 float* proj_weight);

#ifdef __cplusplus
}
#endif
#endif /* FWA_B200_H */
