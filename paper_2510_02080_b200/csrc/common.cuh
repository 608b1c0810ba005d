// Shared device helpers for the EC3R-SLAM B200 path (sm_100a).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/ec3r_b200.h"

namespace cg = cooperative_groups;

namespace ec3r {

// ---------------------------------------------------------------------------
// error plumbing (thread-local last error string, see ec3r_last_error)
void set_last_error(const char* where, cudaError_t e);
void set_last_error_msg(const char* msg);
void count_launch();  // diagnostic counter behind ec3r_kernel_launches()

// Optional kernel timing (ec3r_timing_enable): CUDA events recorded on the
// launching stream around the hot kernels, summed by ec3r_timing_get.
enum TimedKernel { TK_MATCH_TC = 0, TK_REGISTER = 1, TK_FUSE_INSERT = 2, TK_COUNT = 3 };
struct KernelTimer {
    cudaEvent_t e0 = nullptr;
    int k = -1;
    cudaStream_t st = nullptr;
    KernelTimer(int kernel, cudaStream_t stream);  // records the start event when timing is on
    void stop();                                  // records the end event
};

// Every kernel launch of the library is followed by this check (it also
// feeds the launch counter the benchmark reports as gpu_launches).
#define EC3R_CHECK_LAUNCH(where)                          \
    do {                                                  \
        ::ec3r::count_launch();                           \
        cudaError_t _e = cudaGetLastError();              \
        if (_e != cudaSuccess) {                          \
            ::ec3r::set_last_error(where, _e);            \
            return EC3R_ECUDA;                            \
        }                                                 \
    } while (0)

#define EC3R_CUDA_TRY(call)                               \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) {                          \
            ::ec3r::set_last_error(#call, _e);            \
            return EC3R_ECUDA;                            \
        }                                                 \
    } while (0)

struct Sim3Arg {
    double v[8];
};

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

// Workspace carving: consecutive 256-byte aligned regions.
static inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
struct Carver {
    char* base;
    size_t used;
    template <typename T>
    T* take(size_t count) {
        T* p = reinterpret_cast<T*>(base + used);
        used += align256(sizeof(T) * count);
        return p;
    }
};

// ---------------------------------------------------------------------------
// Exact float64 arithmetic: the reference is numpy float64 with one rounding
// per ufunc (no FMA contraction).  __d*_rn intrinsics are never contracted,
// so the sequences below reproduce numpy's results bit-for-bit.
__device__ __forceinline__ double xm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xs(double a, double b) { return __dsub_rn(a, b); }

// quat_rotate (liegroups.py:90-95): uv = 2 cross(v, p); p + w*uv + cross(v, uv),
// numpy.cross component order cp0 = a1*b2 - a2*b1, cp1 = a2*b0 - a0*b2,
// cp2 = a0*b1 - a1*b0, each product rounded separately.
__device__ __forceinline__ void quat_rotate_exact(const double* q, const double p[3], double o[3]) {
    const double w = q[0], vx = q[1], vy = q[2], vz = q[3];
    double u0 = xm(2.0, xs(xm(vy, p[2]), xm(vz, p[1])));
    double u1 = xm(2.0, xs(xm(vz, p[0]), xm(vx, p[2])));
    double u2 = xm(2.0, xs(xm(vx, p[1]), xm(vy, p[0])));
    double c0 = xs(xm(vy, u2), xm(vz, u1));
    double c1 = xs(xm(vz, u0), xm(vx, u2));
    double c2 = xs(xm(vx, u1), xm(vy, u0));
    o[0] = xa(xa(p[0], xm(w, u0)), c0);
    o[1] = xa(xa(p[1], xm(w, u1)), c1);
    o[2] = xa(xa(p[2], xm(w, u2)), c2);
}

// Pose3.apply (liegroups.py:208-209) and Sim3Transform.apply (:259-260);
// x8 = {s, qw, qx, qy, qz, tx, ty, tz}.
__device__ __forceinline__ void pose_apply_exact(const double* x8, const double p[3], double o[3]) {
    double r[3];
    quat_rotate_exact(x8 + 1, p, r);
    o[0] = xa(r[0], x8[5]);
    o[1] = xa(r[1], x8[6]);
    o[2] = xa(r[2], x8[7]);
}
__device__ __forceinline__ void sim3_apply_exact(const double* x8, const double p[3], double o[3]) {
    double r[3];
    quat_rotate_exact(x8 + 1, p, r);
    o[0] = xa(xm(x8[0], r[0]), x8[5]);
    o[1] = xa(xm(x8[0], r[1]), x8[6]);
    o[2] = xa(xm(x8[0], r[2]), x8[7]);
}

// Ray of pixel (u, v) at depth z (backend.py:89): ((u-cx)/fx*z, (v-cy)/fy*z, z).
// xcoef = (u - cx) / fx rounded exactly as numpy does.
__device__ __forceinline__ double ray_coef(int u, double c, double f) {
    return __ddiv_rn(xs((double)u, c), f);
}

// quaternion (w,x,y,z) -> rotation matrix (liegroups.py:55-64), float64
__host__ __device__ inline void quat_to_mat(const double* q, double m[3][3]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    m[0][0] = 1 - 2 * (y * y + z * z); m[0][1] = 2 * (x * y - w * z); m[0][2] = 2 * (x * z + w * y);
    m[1][0] = 2 * (x * y + w * z); m[1][1] = 1 - 2 * (x * x + z * z); m[1][2] = 2 * (y * z - w * x);
    m[2][0] = 2 * (x * z - w * y); m[2][1] = 2 * (y * z + w * x); m[2][2] = 1 - 2 * (x * x + y * y);
}

// ---------------------------------------------------------------------------
// 3x3 closed-form pieces of align_point_sets (registration.py:72-101)

// One-sided Jacobi SVD of A (3x3): A = U diag(sig) V^T with U = [u0 u1 u0xu1]
// (det U = +1) and sig[2] SIGNED; |sig| sorted descending.  High relative
// accuracy; converges in a handful of sweeps.
__device__ inline void svd3_jacobi(const double Ain[3][3], double U[3][3], double sig[3], double V[3][3]) {
    double A[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) { A[i][j] = Ain[i][j]; V[i][j] = (i == j) ? 1.0 : 0.0; }
    for (int sweep = 0; sweep < 40; ++sweep) {
        double off = 0.0;
        for (int pi = 0; pi < 3; ++pi) {
            const int i = (pi == 2) ? 1 : 0;
            const int j = (pi == 0) ? 1 : 2;
            double alpha = 0, beta = 0, gamma = 0;
            for (int k = 0; k < 3; ++k) {
                alpha += A[k][i] * A[k][i];
                beta += A[k][j] * A[k][j];
                gamma += A[k][i] * A[k][j];
            }
            if (gamma == 0.0) continue;
            const double nrm = sqrt(alpha * beta);
            if (nrm == 0.0) continue;
            const double rel = fabs(gamma) / nrm;
            if (rel <= 1e-17) continue;
            off = fmax(off, rel);
            const double zeta = (beta - alpha) / (2.0 * gamma);
            double t;
            if (fabs(zeta) > 1e150) t = 0.5 / zeta;
            else t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t);
            const double s = c * t;
            for (int k = 0; k < 3; ++k) {
                const double ai = A[k][i], aj = A[k][j];
                A[k][i] = c * ai - s * aj;
                A[k][j] = s * ai + c * aj;
                const double vi = V[k][i], vj = V[k][j];
                V[k][i] = c * vi - s * vj;
                V[k][j] = s * vi + c * vj;
            }
        }
        if (off <= 1e-16) break;
    }
    double nrm[3];
    for (int j = 0; j < 3; ++j) nrm[j] = sqrt(A[0][j] * A[0][j] + A[1][j] * A[1][j] + A[2][j] * A[2][j]);
    int ord[3] = {0, 1, 2};
    // sort descending by column norm (stable)
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 2 - a; ++b)
            if (nrm[ord[b]] < nrm[ord[b + 1]]) { int tmp = ord[b]; ord[b] = ord[b + 1]; ord[b + 1] = tmp; }
    double Vs[3][3], As[3][3];
    for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) { Vs[k][j] = V[k][ord[j]]; As[k][j] = A[k][ord[j]]; }
    for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k) V[k][j] = Vs[k][j];
    const double s0 = nrm[ord[0]], s1 = nrm[ord[1]];
    double u0[3], u1[3];
    if (s0 > 0) { for (int k = 0; k < 3; ++k) u0[k] = As[k][0] / s0; }
    else { u0[0] = 1; u0[1] = 0; u0[2] = 0; }
    if (s1 > 1e-300 && s1 > 1e-15 * s0) {
        for (int k = 0; k < 3; ++k) u1[k] = As[k][1] / s1;
        // re-orthogonalise against u0 (A's columns are orthogonal to ~1e-16)
        double d = u0[0] * u1[0] + u0[1] * u1[1] + u0[2] * u1[2];
        for (int k = 0; k < 3; ++k) u1[k] -= d * u0[k];
        double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
        for (int k = 0; k < 3; ++k) u1[k] /= n1;
    } else {
        // any unit vector orthogonal to u0
        double e[3] = {0, 0, 0};
        int m = (fabs(u0[0]) <= fabs(u0[1]) && fabs(u0[0]) <= fabs(u0[2])) ? 0 : (fabs(u0[1]) <= fabs(u0[2]) ? 1 : 2);
        e[m] = 1.0;
        double d = u0[m];
        for (int k = 0; k < 3; ++k) u1[k] = e[k] - d * u0[k];
        double n1 = sqrt(u1[0] * u1[0] + u1[1] * u1[1] + u1[2] * u1[2]);
        for (int k = 0; k < 3; ++k) u1[k] /= n1;
    }
    double u2[3] = {u0[1] * u1[2] - u0[2] * u1[1], u0[2] * u1[0] - u0[0] * u1[2], u0[0] * u1[1] - u0[1] * u1[0]};
    for (int k = 0; k < 3; ++k) { U[k][0] = u0[k]; U[k][1] = u1[k]; U[k][2] = u2[k]; }
    sig[0] = s0;
    sig[1] = s1;
    sig[2] = As[0][2] * u2[0] + As[1][2] * u2[1] + As[2][2] * u2[2];  // signed
}

__device__ inline double det3(const double m[3][3]) {
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

// Shepperd's method, liegroups.py:68-87, then normalised.
__device__ inline void mat_to_quat(const double m[3][3], double q[4]) {
    const double t = m[0][0] + m[1][1] + m[2][2];
    if (t > 0) {
        const double r = sqrt(1.0 + t), s = 0.5 / r;
        q[0] = 0.5 * r;
        q[1] = (m[2][1] - m[1][2]) * s;
        q[2] = (m[0][2] - m[2][0]) * s;
        q[3] = (m[1][0] - m[0][1]) * s;
    } else {
        int i = 0;
        if (m[1][1] > m[i][i]) i = 1;
        if (m[2][2] > m[i][i]) i = 2;
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        const double r = sqrt(1.0 + m[i][i] - m[j][j] - m[k][k]), s = 0.5 / r;
        q[0] = (m[k][j] - m[j][k]) * s;
        q[1 + i] = 0.5 * r;
        q[1 + j] = (m[j][i] + m[i][j]) * s;
        q[1 + k] = (m[k][i] + m[i][k]) * s;
    }
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int c = 0; c < 4; ++c) q[c] /= n;
}

// Centered, weight-normalised second moments of one alignment problem.
struct Moments {
    double W;             // sum of weights (raw)
    double pbar[3], qbar[3];
    double C[3][3];       // sum w dq dp^T / W   (rows: q, cols: p)  registration.py:77
    double M[3][3];       // sum w dp dp^T / W   (source scatter, degeneracy)
    double varq;          // sum w |dq|^2 / W    (closed-form residual)
};

struct Solution {
    int status;
    double s, quat[4], t[3];
    double R[3][3];
    double rms2_closed;
    double src_lambda[3];  // eigenvalues of M, descending
    double src_V[3][3];    // eigenvectors (columns)
};

// registration.py:78-98 from the moments.  Degeneracy is decided from the
// eigenvalues of M (sv of sqrt(w) dp squared); callers refine it with a
// rotated-basis pass when the ratio is suspicious (see umeyama.cu).
// The closed form after the two 3x3 decompositions (split out so that a
// caller can run the covariance SVD and the source eigen-decomposition in
// two threads at once).
__device__ inline void umeyama_finish(const Moments& mo, int with_scale, const double U[3][3], const double sig[3],
                                      const double V[3][3], const double lam[3], const double Vm[3][3],
                                      Solution& out);

__device__ inline void umeyama_solve(const Moments& mo, int with_scale, Solution& out) {
    double U[3][3], sig[3], V[3][3];
    svd3_jacobi(mo.C, U, sig, V);
    double Vm[3][3], Um[3][3], lam[3];
    svd3_jacobi(mo.M, Um, lam, Vm);  // symmetric PSD: singular values = eigenvalues
    umeyama_finish(mo, with_scale, U, sig, V, lam, Vm, out);
}

__device__ inline void umeyama_finish(const Moments& mo, int with_scale, const double U[3][3], const double sig[3],
                                      const double V[3][3], const double lam[3], const double Vm[3][3],
                                      Solution& out) {
    out.status = EC3R_ST_OK;
    for (int k = 0; k < 3; ++k) out.src_lambda[k] = fabs(lam[k]);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) out.src_V[i][j] = Vm[i][j];
    const double dV = det3(V) >= 0 ? 1.0 : -1.0;  // det U = +1 by construction
    // R = U diag(1, 1, dV) V^T  (reflection guard registration.py:85-87)
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            out.R[i][j] = U[i][0] * V[j][0] + U[i][1] * V[j][1] + dV * U[i][2] * V[j][2];
    const double var_p = mo.M[0][0] + mo.M[1][1] + mo.M[2][2];
    const double trRC = sig[0] + sig[1] + dV * sig[2];
    double s = 1.0;
    if (with_scale) {
        s = trRC / var_p;                       // registration.py:89-91
        if (!(s > 0)) out.status = EC3R_ST_NONPOS_SCALE;
    }
    out.s = s;
    for (int i = 0; i < 3; ++i)
        out.t[i] = mo.qbar[i] - s * (out.R[i][0] * mo.pbar[0] + out.R[i][1] * mo.pbar[1] + out.R[i][2] * mo.pbar[2]);
    mat_to_quat(out.R, out.quat);
    out.rms2_closed = mo.varq - 2.0 * s * trRC + s * s * var_p;
}

// Source-degeneracy rule registration.py:81-83 on singular values.
__device__ __forceinline__ bool src_degenerate(double sv0, double sv1) {
    return sv1 <= fmax(1e-12 * sv0, 1e-300);
}

// ---------------------------------------------------------------------------
// block reductions (deterministic: fixed butterfly + fixed warp order)
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch /* NT/32 */) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double r = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) r += scratch[k];
    return r;
}

}  // namespace ec3r
