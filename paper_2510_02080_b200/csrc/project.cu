// K1: inverse projection with stream compaction (backend.inverse_project,
// backend.py:78-101).  Points are bit-identical to the reference's float64
// arithmetic (exact __d*_rn sequences, common.cuh) on float32 pool planes or,
// through ec3r_inverse_project_f64, on a reference output's float64 depths.
//
// Three launches: per-tile valid counts -> single-CTA exclusive scan of the
// tile counts -> per-tile block scan + ordered write.  Output order is the
// reference's: frames in order, then row-major (v, u) within a frame.

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace ec3r {

constexpr int IP_NT = 256;
constexpr int IP_PER = 4;                   // pixels per thread (contiguous)
constexpr int IP_TILE = IP_NT * IP_PER;     // pixels per CTA

// T = float (the pool's planes) or double (a reference ReconstructionOutput:
// float64 depths, backend.py:51-58)
template <typename T>
__global__ void __launch_bounds__(IP_NT) ip_count_kernel(const T* __restrict__ depth, int64_t total,
                                                         int32_t* __restrict__ tile_counts) {
    const int64_t base = (int64_t)blockIdx.x * IP_TILE + (int64_t)threadIdx.x * IP_PER;
    int c = 0;
#pragma unroll
    for (int k = 0; k < IP_PER; ++k) c += (base + k < total && depth[base + k] > T(0)) ? 1 : 0;
    typedef cub::BlockReduce<int, IP_NT> BR;
    __shared__ typename BR::TempStorage tmp;
    const int s = BR(tmp).Sum(c);
    if (threadIdx.x == 0) tile_counts[blockIdx.x] = s;
}

// Exclusive scan of n tile counts in one CTA (sequential over chunks).
__global__ void __launch_bounds__(1024) ip_scan_kernel(const int32_t* __restrict__ counts, int64_t n,
                                                       int64_t* __restrict__ offsets, int64_t* __restrict__ total) {
    typedef cub::BlockScan<int64_t, 1024> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < n; b += 1024) {
        const int64_t i = b + threadIdx.x;
        int64_t v = i < n ? counts[i] : 0, ex, agg;
        BS(tmp).ExclusiveSum(v, ex, agg);
        if (i < n) offsets[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

template <typename T>
__global__ void __launch_bounds__(IP_NT) ip_write_kernel(const T* __restrict__ depth, const T* __restrict__ conf,
                                                         int H, int W, int64_t total, double fx, double fy, double cx,
                                                         double cy, const double* __restrict__ poses,
                                                         const int64_t* __restrict__ frame_ids,
                                                         const int64_t* __restrict__ offsets, double* __restrict__ pts,
                                                         double* __restrict__ oconf, int64_t* __restrict__ ofid,
                                                         int64_t* __restrict__ opix) {
    const int64_t base = (int64_t)blockIdx.x * IP_TILE + (int64_t)threadIdx.x * IP_PER;
    const int64_t HW = (int64_t)H * W;
    int flags = 0, c = 0;
#pragma unroll
    for (int k = 0; k < IP_PER; ++k) {
        const bool v = base + k < total && depth[base + k] > T(0);
        flags |= (v ? 1 : 0) << k;
        c += v;
    }
    typedef cub::BlockScan<int, IP_NT> BS;
    __shared__ typename BS::TempStorage tmp;
    int ex;
    BS(tmp).ExclusiveSum(c, ex);
    int64_t o = offsets[blockIdx.x] + ex;
#pragma unroll
    for (int k = 0; k < IP_PER; ++k) {
        if (!((flags >> k) & 1)) continue;
        const int64_t g = base + k;
        const int f = (int)(g / HW);
        const int64_t r = g - (int64_t)f * HW;
        const int v = (int)(r / W), u = (int)(r - (int64_t)v * W);
        const double z = (double)depth[g];
        const double ray[3] = {xm(ray_coef(u, cx, fx), z), xm(ray_coef(v, cy, fy), z), z};
        double out[3];
        pose_apply_exact(poses + 8 * f, ray, out);
        pts[3 * o + 0] = out[0];
        pts[3 * o + 1] = out[1];
        pts[3 * o + 2] = out[2];
        oconf[o] = (double)conf[g];
        ofid[o] = frame_ids[f];
        opix[2 * o] = u;
        opix[2 * o + 1] = v;
        ++o;
    }
}

// Sim3Transform.apply on explicit float64 points (liegroups.py:259-260),
// bit-identical to the reference (Submap.world_points, mapping.py:56-57).
__global__ void sim3_apply_kernel(const double* __restrict__ pts, int64_t n, Sim3Arg g, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double o[3];
    sim3_apply_exact(g.v, p, o);
    out[3 * i] = o[0];
    out[3 * i + 1] = o[1];
    out[3 * i + 2] = o[2];
}

}  // namespace ec3r

using namespace ec3r;

extern "C" int ec3r_sim3_apply(const double* points, int64_t n, const double* sim3_h, double* out, void* stream) {
    if (n < 0 || !sim3_h) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    Sim3Arg g;
    for (int k = 0; k < 8; ++k) g.v[k] = sim3_h[k];
    sim3_apply_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(points, n, g, out);
    EC3R_CHECK_LAUNCH("sim3_apply_kernel");
    return EC3R_OK;
}

extern "C" size_t ec3r_inverse_project_workspace(int F, int H, int W) {
    const int64_t total = (int64_t)F * H * W;
    const int64_t tiles = (total + IP_TILE - 1) / IP_TILE;
    // tile counts (int32) + tile offsets (int64) + poses (F*8 doubles) + frame ids (F int64)
    return align256(tiles * 4) + align256(tiles * 8) + align256((size_t)F * 64) + align256((size_t)F * 8);
}

template <typename T>
static int inverse_project_impl(const T* depth, const T* conf, int F, int H, int W, const double* K4_h,
                                const double* poses_h, const int64_t* frame_ids_h, double* out_points,
                                double* out_conf, int64_t* out_fids, int64_t* out_pixels, int64_t* n_out,
                                void* workspace, size_t workspace_bytes, void* stream) {
    if (F < 0 || H <= 0 || W <= 0 || !K4_h || !n_out) return EC3R_EARG;
    if (workspace_bytes < ec3r_inverse_project_workspace(F, H, W) || !workspace) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    const int64_t total = (int64_t)F * H * W;
    if (total == 0) {
        EC3R_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int64_t), st));
        return EC3R_OK;
    }
    const int64_t tiles = (total + IP_TILE - 1) / IP_TILE;
    Carver cv{(char*)workspace, 0};
    int32_t* counts = cv.take<int32_t>(tiles);
    int64_t* offs = cv.take<int64_t>(tiles);
    double* poses = cv.take<double>((size_t)F * 8);
    int64_t* fids = cv.take<int64_t>(F);
    EC3R_CUDA_TRY(cudaMemcpyAsync(poses, poses_h, sizeof(double) * 8 * F, cudaMemcpyHostToDevice, st));
    EC3R_CUDA_TRY(cudaMemcpyAsync(fids, frame_ids_h, sizeof(int64_t) * F, cudaMemcpyHostToDevice, st));
    ip_count_kernel<T><<<(unsigned)tiles, IP_NT, 0, st>>>(depth, total, counts);
    EC3R_CHECK_LAUNCH("ip_count_kernel");
    ip_scan_kernel<<<1, 1024, 0, st>>>(counts, tiles, offs, n_out);
    EC3R_CHECK_LAUNCH("ip_scan_kernel");
    ip_write_kernel<T><<<(unsigned)tiles, IP_NT, 0, st>>>(depth, conf, H, W, total, K4_h[0], K4_h[1], K4_h[2], K4_h[3],
                                                          poses, fids, offs, out_points, out_conf, out_fids, out_pixels);
    EC3R_CHECK_LAUNCH("ip_write_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_inverse_project(const float* depth, const float* conf, int F, int H, int W, const double* K4_h,
                                    const double* poses_h, const int64_t* frame_ids_h, double* out_points,
                                    double* out_conf, int64_t* out_fids, int64_t* out_pixels, int64_t* n_out,
                                    void* workspace, size_t workspace_bytes, void* stream) {
    return inverse_project_impl<float>(depth, conf, F, H, W, K4_h, poses_h, frame_ids_h, out_points, out_conf,
                                       out_fids, out_pixels, n_out, workspace, workspace_bytes, stream);
}

extern "C" int ec3r_inverse_project_f64(const double* depth, const double* conf, int F, int H, int W,
                                        const double* K4_h, const double* poses_h, const int64_t* frame_ids_h,
                                        double* out_points, double* out_conf, int64_t* out_fids, int64_t* out_pixels,
                                        int64_t* n_out, void* workspace, size_t workspace_bytes, void* stream) {
    return inverse_project_impl<double>(depth, conf, F, H, W, K4_h, poses_h, frame_ids_h, out_points, out_conf,
                                        out_fids, out_pixels, n_out, workspace, workspace_bytes, stream);
}
