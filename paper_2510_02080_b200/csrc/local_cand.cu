// K8: local loop candidate detection — the projection
// count of detect_local_candidates (loops.py:114-133) for a whole window of
// keyframes in one launch: for every (keyframe, map point) the visibility
// test of project_points (geometry.py:87-109) under world_from_cam.inverse()
// (liegroups.py:217-219), a warp-aggregated count per keyframe, and the
// decision count / N > tau_p.
//
// Operation order follows numpy: the inverse pose is rinv = conj(q),
// t' = -quat_rotate(rinv, t) (liegroups.py:90-95, 168-169); R = quat_to_matrix
// (:56-65); pc = ((p0 R_i0 + p1 R_i1) + p2 R_i2) + t'_i; u = fx * pc0 /
// safe_z + cx (geometry.py:99-102), all with _rn intrinsics (no FMA).  The
// matmul pts @ R.T runs in BLAS on the reference side, whose summation order
// is not pinned: a visibility decision can differ only for a point whose
// projection lies within an ulp of the image border or of z = Z_MIN.  Such
// points are listed (margin guard: a band of 1e-6 px around the border and
// 1e-12 around Z_MIN, far above the ~1e-12 px disagreement of the two
// summation orders) with the device's decision, and the host re-decides
// them with the reference's own numpy expression.

#include "common.cuh"

namespace ec3r {

constexpr double LC_Z_MIN = 1e-6;  // geometry.py:23

struct LcCam {
    double R[3][3];
    double t[3];
};

__device__ __forceinline__ void lc_camera(const double* wfc, LcCam& c) {
    // Pose3.inverse: rinv = (w, -x, -y, -z), t' = -rinv.apply(t)
    const double qi[4] = {wfc[1], -wfc[2], -wfc[3], -wfc[4]};
    const double t[3] = {wfc[5], wfc[6], wfc[7]};
    double r[3];
    quat_rotate_exact(qi, t, r);
    for (int i = 0; i < 3; ++i) c.t[i] = -r[i];
    const double w = qi[0], x = qi[1], y = qi[2], z = qi[3];
    c.R[0][0] = xs(1.0, xm(2.0, xa(xm(y, y), xm(z, z))));
    c.R[0][1] = xm(2.0, xs(xm(x, y), xm(w, z)));
    c.R[0][2] = xm(2.0, xa(xm(x, z), xm(w, y)));
    c.R[1][0] = xm(2.0, xa(xm(x, y), xm(w, z)));
    c.R[1][1] = xs(1.0, xm(2.0, xa(xm(x, x), xm(z, z))));
    c.R[1][2] = xm(2.0, xs(xm(y, z), xm(w, x)));
    c.R[2][0] = xm(2.0, xs(xm(x, z), xm(w, y)));
    c.R[2][1] = xm(2.0, xa(xm(y, z), xm(w, x)));
    c.R[2][2] = xs(1.0, xm(2.0, xa(xm(x, x), xm(y, y))));
}

__global__ void lc_count_kernel(const double* __restrict__ pts, int64_t n, const double* __restrict__ poses,
                                double fx, double fy, double cx, double cy, double wmax, double hmax,
                                unsigned long long* __restrict__ counts, int32_t* __restrict__ amb,
                                int64_t amb_cap, unsigned long long* __restrict__ amb_count) {
    __shared__ LcCam cam;
    const int k = blockIdx.y;
    if (threadIdx.x == 0) lc_camera(poses + 8 * (size_t)k, cam);
    __syncthreads();
    unsigned int local = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double p0 = pts[3 * i], p1 = pts[3 * i + 1], p2 = pts[3 * i + 2];
        double pc[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
            pc[r] = xa(xa(xa(xm(p0, cam.R[r][0]), xm(p1, cam.R[r][1])), xm(p2, cam.R[r][2])), cam.t[r]);
        const double z = pc[2];
        const double sz = fabs(z) > LC_Z_MIN ? z : 1.0;
        const double u = xa(__ddiv_rn(xm(fx, pc[0]), sz), cx);
        const double v = xa(__ddiv_rn(xm(fy, pc[1]), sz), cy);
        const bool vis = z > LC_Z_MIN && u >= 0.0 && u <= wmax && v >= 0.0 && v <= hmax;
        local += vis ? 1u : 0u;
        if (amb) {
            const double bp = 1e-6;
            const bool near_z = fabs(z - LC_Z_MIN) < 1e-12;
            const bool in_z = z > LC_Z_MIN - 1e-12;
            const bool near_uv = fabs(u) < bp || fabs(u - wmax) < bp || fabs(v) < bp || fabs(v - hmax) < bp;
            const bool in_uv = u > -bp && u < wmax + bp && v > -bp && v < hmax + bp;
            if ((near_z && in_uv) || (near_uv && in_z && in_uv)) {
                const unsigned long long o = atomicAdd(amb_count, 1ull);
                if ((int64_t)o < amb_cap) {
                    amb[3 * o] = k;
                    amb[3 * o + 1] = (int32_t)i;
                    amb[3 * o + 2] = vis ? 1 : 0;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    // one global atomic per CTA: warps add into shared memory first
    __shared__ unsigned int cta;
    if (threadIdx.x == 0) cta = 0u;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&cta, local);
    __syncthreads();
    if (threadIdx.x == 0 && cta) atomicAdd(counts + k, (unsigned long long)cta);
}

__global__ void lc_decide_kernel(const unsigned long long* __restrict__ counts, int K, int64_t n, double tau_p,
                                 int64_t* __restrict__ out_counts, int32_t* __restrict__ out_cand) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const unsigned long long c = counts[k];
    if (out_counts) out_counts[k] = (int64_t)c;
    out_cand[k] = (n > 0 && __ddiv_rn((double)c, (double)n) > tau_p) ? 1 : 0;  // loops.py:131
}

}  // namespace ec3r

using namespace ec3r;

extern "C" size_t ec3r_local_candidates_workspace(int n_keyframes) {
    return align256(sizeof(unsigned long long) * (size_t)(n_keyframes > 0 ? n_keyframes : 1));
}

extern "C" int ec3r_local_candidates_ex(const double* positions, int64_t n_points, const double* world_from_cam,
                                        int n_keyframes, const double* intrinsics_h, double tau_p, int64_t* out_counts,
                                        int32_t* out_cand, int32_t* amb_out, int64_t amb_cap,
                                        unsigned long long* amb_count, void* workspace, size_t workspace_bytes,
                                        void* stream) {
    if (n_points < 0 || n_keyframes < 0 || !intrinsics_h) return EC3R_EARG;
    if (n_keyframes == 0) return EC3R_OK;
    if (!world_from_cam || !out_cand || (n_points && !positions)) return EC3R_EARG;
    if (!workspace || workspace_bytes < ec3r_local_candidates_workspace(n_keyframes)) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    unsigned long long* counts = (unsigned long long*)workspace;
    EC3R_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (size_t)n_keyframes, st));
    if (amb_out && !amb_count) return EC3R_EARG;
    if (amb_count) EC3R_CUDA_TRY(cudaMemsetAsync(amb_count, 0, sizeof(unsigned long long), st));
    if (n_points > 0) {
        int64_t gx = (n_points + 255) / 256;
        if (gx > 4 * kNumSMs) gx = 4 * kNumSMs;
        const dim3 grid((unsigned)gx, (unsigned)n_keyframes);
        // width - 1, height - 1 as the reference compares against ints
        lc_count_kernel<<<grid, 256, 0, st>>>(positions, n_points, world_from_cam, intrinsics_h[0], intrinsics_h[1],
                                              intrinsics_h[2], intrinsics_h[3], intrinsics_h[4] - 1.0,
                                              intrinsics_h[5] - 1.0, counts, amb_out, amb_cap, amb_count);
        EC3R_CHECK_LAUNCH("lc_count_kernel");
    }
    lc_decide_kernel<<<(n_keyframes + 127) / 128, 128, 0, st>>>(counts, n_keyframes, n_points, tau_p, out_counts,
                                                               out_cand);
    EC3R_CHECK_LAUNCH("lc_decide_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_local_candidates(const double* positions, int64_t n_points, const double* world_from_cam,
                                     int n_keyframes, const double* intrinsics_h, double tau_p, int64_t* out_counts,
                                     int32_t* out_cand, void* workspace, size_t workspace_bytes, void* stream) {
    return ec3r_local_candidates_ex(positions, n_points, world_from_cam, n_keyframes, intrinsics_h, tau_p, out_counts,
                                    out_cand, nullptr, 0, nullptr, workspace, workspace_bytes, stream);
}
