/*
 * ec3r_b200.h — C ABI of the B200-native (sm_100a) dense data-parallel path
 * of EC3R-SLAM (arxiv 2510.02080).
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless its name ends in _h;
 *   - the caller owns every buffer; the library never frees or reallocates
 *     caller memory (the voxel hash is the one opaque, library-owned handle);
 *   - every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream) and returns 0 on success or a
 *     negative EC3R_E* code; per-item outcomes of batched calls are written
 *     to device status arrays (EC3R_ST_*), never returned;
 *   - no hidden global state: calls are reentrant and safe from several host
 *     threads on distinct streams;
 *   - Sim(3) / SE(3) values are 8 doubles {s, qw, qx, qy, qz, tx, ty, tz}
 *     (x -> s * R(q) x + t, s = 1 for poses), the value type of
 *     submap_slam.liegroups.Sim3Transform / Pose3 (liegroups.py:132-272);
 *   - intrinsics are 4 doubles {fx, fy, cx, cy} (geometry.py:28-37).
 *
 * Reference interfaces each entry point replaces are cited as
 * file:line into /root/reference/pkg/src/submap_slam.
 */
#ifndef EC3R_B200_H
#define EC3R_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EC3R_ABI_VERSION 1

#if defined(__GNUC__)
#define EC3R_API __attribute__((visibility("default")))
#else
#define EC3R_API
#endif

/* return codes */
#define EC3R_OK 0
#define EC3R_ECUDA (-1)      /* CUDA launch / runtime error */
#define EC3R_EARG (-2)       /* invalid argument (sizes, alignment, NULL) */
#define EC3R_EWORKSPACE (-3) /* workspace too small */
#define EC3R_ENOMEM (-4)

/* per-item status (batched registration); the Python layer maps these to
 * the reference exception types in the reference's precedence
 * (registration.py:59-93, mapping.py:174-187). */
#define EC3R_ST_OK 0
#define EC3R_ST_SKIP 1          /* < min_correspondences: edge skipped, not an error */
#define EC3R_ST_TOO_FEW 2       /* n < 3 -> TooFewCorrespondences */
#define EC3R_ST_ALL_ZERO 3      /* sum w <= 0 -> AllZeroConfidence */
#define EC3R_ST_DEGENERATE 4    /* collinear / coincident source -> DegenerateConfiguration */
#define EC3R_ST_NONPOS_SCALE 5  /* s <= 0 -> DegenerateConfiguration */

EC3R_API int ec3r_abi_version(void);
/* Process-wide count of kernels this library has launched (diagnostic; the
 * benchmark reports the delta over its timed region as gpu_launches). */
EC3R_API uint64_t ec3r_kernel_launches(void);
/* Kernel timing diagnostics: when enabled, CUDA events are recorded on the
 * launching stream around the tensor-core matcher pass (kernel 0), the pool
 * registration (1) and the frame fusion (2); ec3r_timing_get sums and clears
 * them (synchronizing on the events). */
EC3R_API void ec3r_timing_enable(int on);
EC3R_API int ec3r_timing_get(int kernel, double* ms_total, int64_t* n_launches);
/* Last CUDA error string of the calling thread's most recent failing call. */
EC3R_API const char* ec3r_last_error(void);

/* ---------------------------------------------------------------------
 * K1  inverse projection with compaction
 * replaces backend.inverse_project (backend.py:78-101)
 *
 * depth/conf: (F, H, W) float32, row-major; poses: F x 8 (anchor_from_cam);
 * frame_ids_h: host array of F ids.  Writes one row per pixel with
 * depth > 0, frames in order then row-major (v, u): points (N,3) float64
 * (bit-identical to the reference's float64 arithmetic on the float32
 * inputs), conf (N) float64, frame ids (N) int64, pixels (N,2) int64 (u,v).
 * Outputs must hold F*H*W rows; *n_out (device int64) receives N.
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_inverse_project_workspace(int F, int H, int W);
EC3R_API int ec3r_inverse_project(const float* depth, const float* conf, int F, int H, int W,
                         const double* K4_h, const double* poses_h, const int64_t* frame_ids_h,
                         double* out_points, double* out_conf, int64_t* out_fids,
                         int64_t* out_pixels, int64_t* n_out, void* workspace,
                         size_t workspace_bytes, void* stream);
/* As ec3r_inverse_project on float64 depth / confidence planes (a reference
 * ReconstructionOutput as decoded, backend.py:51-58): bit-identical float64
 * points for any input, not only float32-representable ones. */
EC3R_API int ec3r_inverse_project_f64(const double* depth, const double* conf, int F, int H, int W,
                                      const double* K4_h, const double* poses_h, const int64_t* frame_ids_h,
                                      double* out_points, double* out_conf, int64_t* out_fids, int64_t* out_pixels,
                                      int64_t* n_out, void* workspace, size_t workspace_bytes, void* stream);

/* Sim3Transform.apply (liegroups.py:259-260) on (n,3) float64 points,
 * bit-identical to the reference; the world-point transform of
 * Submap.world_points / Mapping.fused_cloud (mapping.py:56-57, 332-338). */
EC3R_API int ec3r_sim3_apply(const double* points, int64_t n, const double* sim3_h, double* out,
                             void* stream);

/* ---------------------------------------------------------------------
 * K2+K3  batched submap registration over pixel-identity correspondences
 * replaces Mapping._shared_correspondences + the gate/floor/align loop of
 * Mapping._registration_edges (mapping.py:138-183) and align_point_sets
 * (registration.py:38-102) for B edges in one launch.
 *
 * Frames live in a resident pool: depth_pool/conf_pool (n_slots, H, W)
 * float32; slot_poses (n_slots x 8, device) are anchor_from_cam of the frame
 * in its submap.  An edge (sm -> other) is the concatenation of its
 * segments seg_slots[2*k] (frame slot in sm), seg_slots[2*k+1] (same
 * keyframe's slot in other) for k in [edge_seg[e], edge_seg[e+1]).
 * Per edge: pairs valid where both depths > 0, w = min(conf_a, conf_b),
 * floor = floor_frac * max(w), keep = w >= floor; SKIP when fewer than
 * min_corr pairs / kept pairs, else Umeyama q ~ s R p + t.  Outputs per
 * edge: out_sim3 (B x 8), out_rms, out_count (kept), out_npairs (valid),
 * out_status.  keep_masks (optional, n_seg x H x W uint8) receives the
 * inlier mask (bit-exact contract).
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_register_edges_workspace(int n_edges);
EC3R_API int ec3r_register_edges(const float* depth_pool, const float* conf_pool, int H, int W,
                        const double* K4_h, const double* slot_poses, const int32_t* seg_slots,
                        const int32_t* edge_seg, int n_edges, double floor_frac, int min_corr,
                        int with_scale, double* out_sim3, double* out_rms, int64_t* out_count,
                        int64_t* out_npairs, int32_t* out_status, uint8_t* keep_masks,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Pose chaining of register_submap (mapping.py:190-211) on the device:
 * submaps 0..n_sub-1 in registration order; submap 0 is the fixed root (the
 * first submap, or a sharded window's halo stub) and keeps the caller's
 * sub_globals[0].  Submap j's edges are [sub_edge_off[j], sub_edge_off[j+1])
 * with edge_partner[e] < j the partner submap index.  Edges to partners that
 * were not committed (sub_status != OK) are ignored, SKIP edges are dropped,
 * the first error edge status aborts the submap (sub_status[j] = that status,
 * as align_point_sets raises out of the reference loop), and no surviving edge
 * gives sub_status[j] = EC3R_ST_SKIP (NoSharedKeyframes); such submaps keep
 * the caller's sub_globals entry.  Otherwise the OK edge with the largest
 * count (first on ties) sets sub_globals[j] = sub_globals[partner] o
 * edge_sim3[e].  slot_globals[s] for s in [sub_slot_off[j], sub_slot_off[j+1])
 * receives sub_globals[j].  sub_status (DEVICE, n_sub) is required.
 * Env EC3R_CHAIN_SMEM_CAP (bytes) caps the shared-memory staging (tests use
 * it to force the sequential walk). */
EC3R_API int ec3r_chain_poses(const double* edge_sim3, const int64_t* edge_count,
                              const int32_t* edge_status, const int32_t* edge_partner,
                              const int32_t* sub_edge_off, int n_sub, const int32_t* sub_slot_off,
                              double* sub_globals, double* slot_globals, int32_t* sub_status,
                              void* stream);

/* Sharded chain (SURVEY §8(e), row (a)+(b)): rank `rank` of `world` chained
 * its window relative to the predecessor's halo submap; window_last (DEVICE,
 * world x 8, all-gathered) holds every window's last-submap pose in its own
 * frame.  Left-composes O = W_0 o ... o W_{rank-1} into sub_globals (n_sub x 8)
 * and slot_globals (n_slots x 8) in place; offset_out (nullable, 8) gets O. */
EC3R_API int ec3r_apply_window_offset(const double* window_last, int world, int rank, double* sub_globals,
                                      int n_sub, double* slot_globals, int64_t n_slots, double* offset_out,
                                      void* stream);

/* ---------------------------------------------------------------------
 * K2+K3  batched weighted Umeyama on explicit correspondences
 * replaces align_point_sets (registration.py:38-102) / weighted_umeyama
 * (:105-112).  p, q: (sum n_b, 3) float64; w: (sum n_b) float64 or NULL
 * (uniform); offsets: B+1 int64 (device).  Reduction grouping is anchored
 * to element index (zero-weight tail elements leave results bit-identical).
 * Outputs: out_sim3 (B x 8), out_rms (B), out_status (B).
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_umeyama_workspace(int n_problems);
EC3R_API int ec3r_umeyama_batched(const double* p, const double* q, const double* w,
                         const int64_t* offsets, int n_problems, int with_scale,
                         double* out_sim3, double* out_rms, int32_t* out_status,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------
 * K1+K4  transform + voxel-hash fusion + downsampling
 * replaces Submap.world_points / Mapping.fused_cloud (mapping.py:56-57,
 * 332-338) with the declared fusion rule of oracle/fuse.py; keys are
 * _pack(floor(x / cell)) (_kernels/_numpy.py:50-55), bit-exact against the
 * reference's float64 transform.  Voxel-block hash: an open-addressing
 * table of 4x4x4 block keys over a pool of dense blocks holding float32
 * sums of conf * (x - voxel corner), sum of conf and a uint32 count.
 * capacity (create) = expected voxels; the pool holds capacity / 4 blocks
 * and overflow is reported in n_overflow (grow and re-run).
 * ------------------------------------------------------------------- */
typedef struct ec3r_vhash ec3r_vhash;

typedef struct {
    int64_t n_points_in;     /* points offered (depth > 0, conf > 0) */
    int64_t n_out_of_range;  /* cell outside the 21-bit key range: dropped */
    int64_t n_overflow;      /* table full: dropped (grow and re-run) */
    int64_t n_slow_path;     /* points resolved by the exact float64 path */
    int64_t n_blocks;        /* 4x4x4 voxel blocks allocated in the pool */
} ec3r_vhash_stats;

EC3R_API int ec3r_vhash_create(ec3r_vhash** out, int64_t capacity, double cell_size, void* stream);
/* As ec3r_vhash_create with the pool's block count and the block table's
 * entry count chosen explicitly (table_entries 0: 2x the pool, rounded up to
 * a power of two).  A map sized from a previous fill's stats (n_blocks,
 * voxels) with a sparse table keeps the per-fill clear and emit small while
 * inserting as fast as an oversized map. */
EC3R_API int ec3r_vhash_create_sized(ec3r_vhash** out, int64_t max_voxels, int64_t max_blocks,
                                     int64_t table_entries, double cell_size, void* stream);
EC3R_API int ec3r_vhash_destroy(ec3r_vhash* h);
EC3R_API int64_t ec3r_vhash_capacity(const ec3r_vhash* h);
EC3R_API int ec3r_vhash_clear(ec3r_vhash* h, void* stream);
/* Fuse whole frames of the pool: for each listed slot, every pixel with
 * depth > 0 and conf > 0 is inverse-projected with slot_poses[slot]
 * (anchor_from_cam) and mapped to the world by slot_globals[slot] (the
 * owning submap's global Sim(3)); slots is a device list of n slot ids. */
EC3R_API int ec3r_vhash_insert_frames(ec3r_vhash* h, const float* depth_pool, const float* conf_pool,
                             int H, int W, const double* K4_h, const double* slot_poses,
                             const double* slot_globals, const int32_t* slots, int n,
                             void* stream);
/* Reduction-floor diagnostic (no reference counterpart; bench.py extras).
 * ec3r_vhash_diag_log arms the NEXT ec3r_vhash_insert_frames call on h to
 * log its runs instead of reducing them: (pool voxel, count) uint32 pairs in
 * issue order into runs[0..cap), *n_dev (device, zeroed by the caller)
 * counting them; the map is left unchanged.  ec3r_vhash_diag_replay issues
 * exactly the logged reductions into h's pool (a float4 add per run, plus
 * the u32 count add when with_count != 0): the cost of the insert's own
 * reduction stream without its loads, keys and lookups.  Block-hash engine
 * only (EC3R_EARG on a map created for the binned engine). */
EC3R_API int ec3r_vhash_diag_log(ec3r_vhash* h, void* runs, int64_t cap, unsigned long long* n_dev);
EC3R_API int ec3r_vhash_diag_replay(ec3r_vhash* h, const void* runs, const unsigned long long* n_dev, int64_t cap,
                                    int with_count, void* stream);
/* Fuse explicit points (N,3) float64 with conf (N) float64 under sim3_h. */
EC3R_API int ec3r_vhash_insert_points(ec3r_vhash* h, const double* points, const double* conf, int64_t n,
                             const double* sim3_h, void* stream);
/* Copy the running counters to a host struct (synchronizes the stream). */
EC3R_API int ec3r_vhash_stats_get(ec3r_vhash* h, ec3r_vhash_stats* out_h, void* stream);
/* Emit the fused voxels: keys (U) int64 ascending (sorted when sort != 0),
 * centroid (U,3) float32, wsum (U) float32, count (U) int32; *n_out (device
 * int64) = U.  Outputs must hold U rows: query ec3r_vhash_count (device
 * int64) first, or size them for ec3r_vhash_capacity. */
EC3R_API size_t ec3r_vhash_extract_workspace(const ec3r_vhash* h);
EC3R_API int ec3r_vhash_count(ec3r_vhash* h, int64_t* n_out, void* stream);
EC3R_API int ec3r_vhash_extract(ec3r_vhash* h, int64_t* keys, float* centroid, float* wsum,
                       int32_t* count, int64_t* n_out, int sort, void* workspace,
                       size_t workspace_bytes, void* stream);
/* sort: 0 = block order, 1 = key order (U read back to the host, see
 * ec3r_vhash_extract_count), 2 = key order without the host read (U only in
 * *n_out on the device).  The block sort uses 32-bit relative keys once a
 * sort = 1 extract found the map's block extent fits them; sort = 2 checks
 * that fit on the device and, if the map has outgrown it, counts an emit
 * overflow (ec3r_vhash_stats_get n_overflow) instead of re-running: check the
 * stats after a sort = 2 extract and repeat it with sort = 1 on overflow. */
/* Voxel count of the last sorted extract on this handle (already known on
 * the host), or -1: lets a caller size its outputs without a device read. */
EC3R_API int64_t ec3r_vhash_extract_count(const ec3r_vhash* h);
/* Multi-GPU: emit raw partial sums (key, sum w*dx, sum w, count) bucketed
 * by owner rank = hash(key) mod n_ranks (1 <= n_ranks <= 64) for the
 * all-to-all (outputs hold U rows; workspace = ec3r_vhash_extract_workspace
 * + 1 KB), and merge received partials into a table. */
EC3R_API int ec3r_vhash_extract_partials(ec3r_vhash* h, int n_ranks, int64_t* keys, float* sums4,
                                int32_t* count, int64_t* rank_counts, void* workspace,
                                size_t workspace_bytes, void* stream);
EC3R_API int ec3r_vhash_merge_partials(ec3r_vhash* h, const int64_t* keys, const float* sums4,
                              const int32_t* count, int64_t n, void* stream);
/* Host-sync-free form of the exchange (replaces the per-step host reads of
 * the bucket sizes): owner r's partials go to the fixed slab
 * [r*cap, r*cap + slab_counts[r]) of the outputs (n_ranks*cap rows; rows
 * past a full slab are counted in *overflow, both device int64), so the
 * all-to-all uses equal splits; the receiver merges n_slabs slabs of cap rows
 * with their device counts.  Workspace = ec3r_vhash_extract_workspace + 17 KB.
 * Reference boundary: the owner-partitioned voxel map of SURVEY §8(e) over
 * mapping.py:332-338 + the declared fusion rule. */
EC3R_API int ec3r_vhash_extract_partials_fixed(ec3r_vhash* h, int n_ranks, int64_t cap, int64_t* keys,
                                               float* sums4, int32_t* count, int64_t* slab_counts,
                                               int64_t* overflow, void* workspace, size_t workspace_bytes,
                                               void* stream);
EC3R_API int ec3r_vhash_merge_partials_slabs(ec3r_vhash* h, const int64_t* keys, const float* sums4,
                                             const int32_t* count, int n_slabs, int64_t cap,
                                             const int64_t* slab_counts, void* stream);
/* ec3r_vhash_stats_get into a device buffer of 5 int64 (no host round trip;
 * block-hash maps). */
EC3R_API int ec3r_vhash_stats_device(ec3r_vhash* h, int64_t* out5, void* stream);

/* ---------------------------------------------------------------------
 * K5  brute-force mutual-NN + Lowe-ratio descriptor matching
 * replaces match_descriptors (tracking.py:143-170) for a batch of frame
 * pairs.  A: (sum N_p, D) and B: (sum M_p, D) bf16 rows (ld = D, D % 8 == 0
 * after zero padding); a_off_h/b_off_h: n_pairs+1 int64 row offsets (HOST).
 * The approximate similarity pass runs on tcgen05 tensor cores (fp32 TMEM
 * accumulators); every decision is certified against an error bound and
 * re-scored in float64 from the exact rows (A_x/B_x, dtype exact_dtype:
 * 0 = the bf16 rows are exact, 1 = float32, 2 = float64), so the result is
 * identical to the float64 reference.  norm_bound = max|a| * max|b| over the
 * rows (<= 0: computed on the device) scales the error bound.
 * Output: match_b (sum N_p) int32 =
 * matched B row within the pair or -1; n_match (n_pairs) int32.
 * ------------------------------------------------------------------- */
/* Workspace bytes for ec3r_match_batched on these row offsets (host
 * int64, n_pairs + 1 each): grows with sum_p ceil(N_p / 256) * M_p. */
EC3R_API size_t ec3r_match_workspace(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs);
EC3R_API int ec3r_match_batched(const uint16_t* A, const uint16_t* B, const void* A_x, const void* B_x,
                       int exact_dtype, const int64_t* a_off_h, const int64_t* b_off_h,
                       int n_pairs, int D, double ratio, double norm_bound, int32_t* match_b,
                       int32_t* n_match, void* workspace, size_t workspace_bytes, void* stream);
/* Shared maps: pair p's M_p = b_off_h[p+1] - b_off_h[p] columns are rows
 * [b_row_h[p], b_row_h[p] + M_p) of B (host int64 per pair; n_b_rows rows
 * in B), so consecutive frames tracked against one local map
 * (tracking.py:173-194) share its rows.  b_off_h stays the per-pair column
 * prefix (column state and outputs).  b_row_h = NULL: ec3r_match_batched. */
EC3R_API int ec3r_match_batched_rows(const uint16_t* A, const uint16_t* B, const void* A_x, const void* B_x,
                                     int exact_dtype, const int64_t* a_off_h, const int64_t* b_off_h,
                                     const int64_t* b_row_h, int64_t n_b_rows, int n_pairs, int D, double ratio,
                                     double norm_bound, int32_t* match_b, int32_t* n_match, void* workspace,
                                     size_t workspace_bytes, void* stream);
/* Diagnostics of the last ec3r_match_batched on this workspace (device
 * counters copied to host; synchronizes): rows / columns that needed the
 * float64 full rescan. */
EC3R_API int ec3r_match_stats(const void* workspace, int64_t total_a, int64_t total_b, int n_pairs,
                     int64_t* rows_rescanned_h, int64_t* cols_rescanned_h, void* stream);

/* ---------------------------------------------------------------------
 * K6  strided global loop retrieval
 * replaces the scoring of update_similarity (loops.py:184-243).
 * pooled: (K, D) float64 unit vectors in database insertion order.
 * Coarse pass: every stride-th keyframe vs every later one with
 * |dI| >= exclusion; hits s > tau_g refine over +-(stride-1) on both sides.
 * Outputs (device): coarse_pairs (n_coarse x 2 int32 order indices),
 * coarse_scores; cand_* = refined pairs with score > tau_l in the
 * reference emission order (duplicates kept; the host applies the
 * admitted-once rule); evaluated_* = every refined pair scored (for the
 * similarity-matrix cache).  Counts go to counts (4 int64: coarse,
 * candidates, evaluated, coarse hits).  Capacities: coarse =
 * (k_end - k_begin) * ceil(K/stride), cand/evaluated = cap_refine, coarse
 * hits = cap_refine / (2*stride-1)^2 + 1 (a count above a capacity means
 * the list was truncated: grow and call again).
 * ------------------------------------------------------------------- */
EC3R_API int ec3r_retrieval(const double* pooled, int K, int D, int stride, int exclusion, double tau_g,
                   double tau_l, int32_t* coarse_pairs, double* coarse_scores,
                   int32_t* cand_pairs, double* cand_scores, int32_t* eval_pairs,
                   double* eval_scores, int64_t cap_refine, int64_t* counts, int k_begin,
                   int k_end, void* workspace, size_t workspace_bytes, void* stream);
EC3R_API size_t ec3r_retrieval_workspace(int K, int stride, int64_t cap_refine);

/* ---------------------------------------------------------------------
 * K7  the reference's native-kernel plugin slot (_kernels/__init__.py:
 *     12-33: raycast, nn_query, nn_dists with the semantics of
 *     _kernels/_numpy.py), results bit-identical to it.
 * ec3r_nn_query replaces nn_query / nn_dists (_numpy.py:66-137): directed
 * nearest neighbours query -> ref through the grid hash of cell size
 * `cell`; query (n_query x 3) and ref (n_ref x 3) float64 row-major.
 * Output out_dist (n_query) float64 and out_idx (n_query) int64 (index into
 * ref; inf / -1 when ref is empty).  n_ref <= 2^31 - 1.
 * ec3r_raycast replaces raycast (_numpy.py:29-47): first-hit parameter of
 * each ray (origins, dirs: n x 3 float64) against the room shell and solid
 * boxes solids_h (HOST, n_solids x 6 float64 {min xyz, max xyz}, room
 * first); 0 where nothing is hit.  n_solids <= 64.
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_nn_workspace(int64_t n_ref, int64_t n_query);
EC3R_API int ec3r_nn_query(const double* query, int64_t n_query, const double* ref, int64_t n_ref,
                           double cell, double* out_dist, int64_t* out_idx, void* workspace,
                           size_t workspace_bytes, void* stream);
EC3R_API int ec3r_raycast(const double* origins, const double* dirs, int64_t n, const double* solids_h,
                          int n_solids, double* out_t, void* stream);
/* §8(f) rank 3: SyntheticBackend.decode (backend.py:228-281) over
 * render_depth (scenesim.py:145-163) on the device.  solids_h (HOST):
 * n_solids x {lo xyz, hi xyz} (room shell first, then the interior boxes);
 * frames (DEVICE): n_frames x 12 float64 {R_wc row-major, t_wc}; K4_h (HOST)
 * {fx, fy, cx, cy}.  Writes depth = first_hit * scale (x exp(sigma xi) when
 * sigma > 0) and conf = 1/(1+|xi|) (1 without noise, 0 where depth <= 0) as
 * float32 (n_frames, H, W) planes.  xi: Philox normals keyed by `key`
 * (same distribution as the reference's, not the same stream); with
 * sigma = 0 the output is the reference decode rounded to float32. */
EC3R_API int ec3r_synthetic_decode(const double* solids_h, int n_solids, const double* frames, int n_frames, int H,
                                   int W, const double* K4_h, double scale, double sigma, uint64_t key,
                                   float* out_depth, float* out_conf, void* stream);

/* ---------------------------------------------------------------------
 * K8  local loop candidates: replaces the projection count of
 * detect_local_candidates (loops.py:114-133 -> project_points,
 * geometry.py:87-109) for a whole window of keyframes in one launch.
 * positions (n_points x 3 float64), world_from_cam (n_keyframes x 8 float64
 * {s, q, t}), intrinsics_h (HOST, 6 doubles {fx, fy, cx, cy, width,
 * height}).  out_counts (n_keyframes int64, optional): points projecting
 * inside the image in front of the camera; out_cand (n_keyframes int32):
 * count / n_points > tau_p.
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_local_candidates_workspace(int n_keyframes);
EC3R_API int ec3r_local_candidates(const double* positions, int64_t n_points, const double* world_from_cam,
                                   int n_keyframes, const double* intrinsics_h, double tau_p,
                                   int64_t* out_counts, int32_t* out_cand, void* workspace,
                                   size_t workspace_bytes, void* stream);
/* As ec3r_local_candidates, plus the margin guard: every (keyframe, point)
 * whose visibility lies within 1e-6 px of the image border or 1e-12 of
 * Z_MIN is listed in amb_out (DEVICE, amb_cap x 3 int32: keyframe, point,
 * device decision); amb_count (DEVICE u64) receives the total (may exceed
 * amb_cap: re-run larger).  The host re-decides those points with the
 * reference's numpy expression (pts @ R.T + t, geometry.py:96-108) and
 * corrects the counts. */
EC3R_API int ec3r_local_candidates_ex(const double* positions, int64_t n_points, const double* world_from_cam,
                                      int n_keyframes, const double* intrinsics_h, double tau_p,
                                      int64_t* out_counts, int32_t* out_cand, int32_t* amb_out, int64_t amb_cap,
                                      unsigned long long* amb_count, void* workspace, size_t workspace_bytes,
                                      void* stream);

/* ---------------------------------------------------------------------
 * K9 (§8f rank 4): batched homography RANSAC (loop verification).
 * Replaces estimate_homography_ransac (geometry.py:594-640), called per
 * candidate by verify_candidate (loops.py:136-153).
 *
 * P problems; problem p owns matches [offsets[p], offsets[p+1]) of src / dst
 * ((total, 2) float64 pixels, DEVICE; offsets DEVICE int64).  rng_state
 * (DEVICE, P x 6 uint64): numpy PCG64 state of default_rng(seed) as
 * (state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger).
 *
 * ec3r_homography_ransac_score replays rng.choice(n, 4, replace=False) for
 * `iters` (= cfg.max_iterations) iterations and writes out_counts (P x iters
 * int32): the inlier count of each iteration's hypothesis, -1 where the
 * reference skips it (degenerate sample or failed DLT).  out_samples
 * (nullable, P x iters x 4 int32) receives the drawn indices.  The caller
 * walks the counts with the reference's acceptance / adaptive-stop rule and
 * passes each problem's chosen iteration (or -1) in `best` to
 * ec3r_homography_ransac_refit, with the SAME workspace: it writes the final
 * model (P x 9 float64, row-major, h22 = 1), the inlier mask (total uint8)
 * and the inlier count (P int32).
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_homography_workspace(int n_problems, int iters);
EC3R_API int ec3r_homography_ransac_score(const double* src, const double* dst, const int64_t* offsets,
                                          int n_problems, const uint64_t* rng_state, int iters,
                                          double pixel_threshold, int32_t* out_counts, int32_t* out_samples,
                                          void* workspace, size_t workspace_bytes, void* stream);
EC3R_API int ec3r_homography_ransac_refit(const double* src, const double* dst, const int64_t* offsets,
                                          int n_problems, const int32_t* best, int iters,
                                          double pixel_threshold, double* out_model, uint8_t* out_mask,
                                          int32_t* out_count, void* workspace, size_t workspace_bytes,
                                          void* stream);

/* -------------------------------------------------------------------
 * §8f rank 4, the tracking half: PnP RANSAC scoring.  Replaces the
 * per-hypothesis _reprojection_errors pass of solve_pnp_ransac
 * (geometry.py:414-474, called by tracking.py:208); the minimal EPnP
 * hypotheses stay in the reference's host solver (LAPACK null-space bases,
 * geometry.py:134-210).
 *
 * ec3r_ransac_draws: the replay of rng.choice(n, 4, replace=False) for
 * `iters` iterations of each problem (as ec3r_homography_ransac_score) into
 * out_samples (P x iters x 4 int32, DEVICE); workspace
 * ec3r_ransac_draws_workspace(P).
 *
 * ec3r_pnp_score: n_hyp hypotheses (hyp: n_hyp x 12 float64, R row-major
 * then t; hyp_problem: problem of each) scored over their problem's
 * correspondences (pts (total,3), pix (total,2) float64, offsets P+1,
 * K4 P x 4 {fx, fy, cx, cy}; all DEVICE): inlier count, sum of the inlier
 * errors, and an ambiguity flag (an error within guard * threshold of the
 * threshold, or a depth within 1e-12 of Z_MIN) the host resolves with the
 * reference expression.
 * ------------------------------------------------------------------- */
EC3R_API size_t ec3r_ransac_draws_workspace(int n_problems);
EC3R_API int ec3r_ransac_draws(const int64_t* offsets, int n_problems, const uint64_t* rng_state, int iters,
                               int32_t* out_samples, void* workspace, size_t workspace_bytes, void* stream);
EC3R_API int ec3r_pnp_score(const double* pts, const double* pix, const int64_t* offsets, const double* K4,
                            const double* hyp, const int32_t* hyp_problem, int n_hyp, double pixel_threshold,
                            double guard, int32_t* out_count, double* out_errsum, int32_t* out_ambiguous,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EC3R_B200_H */
