// Binned super-block fusion engine behind ec3r_vhash (see vbin.cu).
#pragma once

#include "common.cuh"
#include "fuse_common.cuh"

namespace ec3r {

struct BinFuse;

BinFuse* bf_create(int64_t max_voxels, int64_t max_bins, double cell, cudaStream_t st, int* rc);
void bf_destroy(BinFuse* b);
int bf_clear(BinFuse* b, cudaStream_t st);
// frame insertion: g.ftab must already hold the frame tables of g's slots
int bf_insert_frames(BinFuse* b, const FrameGeom& g, cudaStream_t st);
int bf_insert_points(BinFuse* b, const double* pts, const double* conf, int64_t n, const double* sim3_h,
                     cudaStream_t st);
// counters: n_in, n_out_of_range, n_overflow (dropped points + voxels), n_slow, n_bins
int bf_stats(BinFuse* b, int64_t out[5], cudaStream_t st);
// voxel count U (aggregates if needed; synchronises)
int bf_count(BinFuse* b, int64_t* U, cudaStream_t st);
// sorted emit into caller buffers (>= U rows); *n_out (device) = U, *U_host too
int bf_extract(BinFuse* b, int64_t* keys, float* centroid, float* wsum, int32_t* count, int64_t* n_out,
               int64_t* U_host, cudaStream_t st);
// owner-bucketed partials (key, sum c*(x - corner), sum c, count) as ec3r_vhash_extract_partials
int bf_extract_partials(BinFuse* b, int n_ranks, int64_t* keys, float* sums4, int32_t* count, int64_t* rank_counts,
                        cudaStream_t st);

}  // namespace ec3r
