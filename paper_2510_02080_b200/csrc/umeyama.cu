// K2+K3: batched confidence-weighted Umeyama Sim(3) on sm_100a.
//
// One thread-block CLUSTER (8 CTAs) per alignment problem.  Every phase
// streams the problem's data once with coalesced (128-bit where possible)
// loads, reduces per thread in float64, then per CTA (fixed shuffle tree) and
// across the cluster through distributed shared memory (fixed rank order), so
// results are deterministic and independent of scheduling.  The 3x3 closed
// form (one-sided Jacobi SVD, reflection guard, scale, translation,
// Shepperd quaternion) runs redundantly in every CTA from the identical
// cluster totals, so no extra broadcast round is needed; in the pool kernel
// the covariance SVD and the source eigen-decomposition run in two threads
// at once.
//
// Reference: registration.py:38-102 (align_point_sets), mapping.py:138-183
// (_shared_correspondences + gate/floor of _registration_edges).

#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace ec3r {

#ifndef EC3R_UM_CL
#define EC3R_UM_CL 8
#endif
constexpr int UM_CL = EC3R_UM_CL;  // CTAs per cluster (portable maximum 8)
constexpr int UM_NT = 256;  // threads per CTA

// Reduce K doubles across the CTA: result valid in out[0..K) for all threads
// after the trailing __syncthreads.  scratch: (UM_NT/32) * K doubles.
template <int K>
__device__ __forceinline__ void cta_sum(double (&v)[K], double* scratch, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        v[k] = x;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) scratch[warp * K + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double r = 0;
#pragma unroll
        for (int w = 0; w < UM_NT / 32; ++w) r += scratch[w * K + threadIdx.x];
        out[threadIdx.x] = r;
    }
    __syncthreads();
}

// Sum a K-vector published by every CTA of the cluster, in rank order.
template <int K>
__device__ __forceinline__ void cluster_sum(cg::cluster_group& cl, double* part, double* tot) {
    cl.sync();
    if (threadIdx.x < K) {
        double r = 0;
        for (int c = 0; c < UM_CL; ++c) r += cl.map_shared_rank(part, c)[threadIdx.x];
        tot[threadIdx.x] = r;
    }
    __syncthreads();
}

__device__ __forceinline__ void write_sim3(double* o, const Solution& s) {
    o[0] = s.s;
    o[1] = s.quat[0]; o[2] = s.quat[1]; o[3] = s.quat[2]; o[4] = s.quat[3];
    o[5] = s.t[0]; o[6] = s.t[1]; o[7] = s.t[2];
}

// ---------------------------------------------------------------------------
// Explicit correspondences (align_point_sets API).  Element e of a problem is
// owned by thread (e % UM_NT) of CTA ((e / UM_NT) % UM_CL): the grouping is a
// function of the element index only, so appending zero-weight elements adds
// exact +0.0 terms and leaves every result bit-identical
// (pkg/tests/test_registration.py:52-71).
template <bool HAS_W>
__global__ void __cluster_dims__(UM_CL, 1, 1) __launch_bounds__(UM_NT)
umeyama_explicit_kernel(const double* __restrict__ P, const double* __restrict__ Q,
                        const double* __restrict__ Wt, const int64_t* __restrict__ off,
                        int with_scale, double* __restrict__ out_sim3, double* __restrict__ out_rms,
                        int32_t* __restrict__ out_status) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int b = blockIdx.x / UM_CL;
    const int64_t i0 = off[b];
    const int64_t n = off[b + 1] - i0;
    __shared__ double scratch[(UM_NT / 32) * 16];
    __shared__ double part1[8], part2[16], part3[4];
    __shared__ double tot1[8], tot2[16], tot3[4];
    __shared__ Solution sol;
    if (n < 3) {  // registration.py:59-60 (uniform across the cluster)
        if (rank == 0 && threadIdx.x == 0) out_status[b] = EC3R_ST_TOO_FEW;
        return;
    }
    const double* p = P + 3 * i0;
    const double* q = Q + 3 * i0;
    const double* w = HAS_W ? Wt + i0 : nullptr;
    const int64_t stride = (int64_t)UM_CL * UM_NT;
    const int64_t first = (int64_t)rank * UM_NT + threadIdx.x;

    // phase 1: W, sum w p, sum w q  (registration.py:67-73)
    double a1[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int64_t e = first; e < n; e += stride) {
        const double wi = HAS_W ? w[e] : 1.0;
        a1[0] += wi;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            a1[1 + k] += wi * p[3 * e + k];
            a1[4 + k] += wi * q[3 * e + k];
        }
    }
    cta_sum<7>(a1, scratch, part1);
    cluster_sum<7>(cl, part1, tot1);
    const double Wsum = tot1[0];
    if (!(Wsum > 0)) {  // registration.py:68-69
        if (rank == 0 && threadIdx.x == 0) out_status[b] = EC3R_ST_ALL_ZERO;
        cl.sync();
        return;
    }
    double pbar[3], qbar[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) { pbar[k] = tot1[1 + k] / Wsum; qbar[k] = tot1[4 + k] / Wsum; }

    // phase 2: centred second moments (registration.py:74-77, 90)
    double a2[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a2[k] = 0;
    for (int64_t e = first; e < n; e += stride) {
        const double wi = HAS_W ? w[e] : 1.0;
        double dp[3], dq[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) { dp[k] = p[3 * e + k] - pbar[k]; dq[k] = q[3 * e + k] - qbar[k]; }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double wq = wi * dq[i];
#pragma unroll
            for (int j = 0; j < 3; ++j) a2[3 * i + j] += wq * dp[j];
        }
        const double wp0 = wi * dp[0], wp1 = wi * dp[1], wp2 = wi * dp[2];
        a2[9] += wp0 * dp[0]; a2[10] += wp0 * dp[1]; a2[11] += wp0 * dp[2];
        a2[12] += wp1 * dp[1]; a2[13] += wp1 * dp[2]; a2[14] += wp2 * dp[2];
        a2[15] += wi * (dq[0] * dq[0] + dq[1] * dq[1] + dq[2] * dq[2]);
    }
    cta_sum<16>(a2, scratch, part2);
    cluster_sum<16>(cl, part2, tot2);
    if (threadIdx.x == 0) {
        Moments mo;
        mo.W = Wsum;
        for (int k = 0; k < 3; ++k) { mo.pbar[k] = pbar[k]; mo.qbar[k] = qbar[k]; }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) mo.C[i][j] = tot2[3 * i + j] / Wsum;
        mo.M[0][0] = tot2[9] / Wsum; mo.M[0][1] = mo.M[1][0] = tot2[10] / Wsum;
        mo.M[0][2] = mo.M[2][0] = tot2[11] / Wsum; mo.M[1][1] = tot2[12] / Wsum;
        mo.M[1][2] = mo.M[2][1] = tot2[13] / Wsum; mo.M[2][2] = tot2[14] / Wsum;
        mo.varq = tot2[15] / Wsum;
        umeyama_solve(mo, with_scale, sol);
    }
    __syncthreads();

    // phase 3: residual (registration.py:100-101) and the source singular
    // values measured directly in the eigenbasis of the source scatter
    // (registration.py:81-83), accurate to ~1e-16 of sv0 like LAPACK's SVD.
    double a3[3] = {0, 0, 0};
    const double s = sol.s;
    double R[3][3], t[3], v0[3], v1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        t[i] = sol.t[i];
        v0[i] = sol.src_V[i][0];
        v1[i] = sol.src_V[i][1];
#pragma unroll
        for (int j = 0; j < 3; ++j) R[i][j] = sol.R[i][j];
    }
    for (int64_t e = first; e < n; e += stride) {
        const double wi = HAS_W ? w[e] : 1.0;
        const double px = p[3 * e], py = p[3 * e + 1], pz = p[3 * e + 2];
        double r2 = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double r = s * (R[i][0] * px + R[i][1] * py + R[i][2] * pz) + t[i] - q[3 * e + i];
            r2 += r * r;
        }
        a3[0] += wi * r2;
        const double dx = px - pbar[0], dy = py - pbar[1], dz = pz - pbar[2];
        const double y0 = v0[0] * dx + v0[1] * dy + v0[2] * dz;
        const double y1 = v1[0] * dx + v1[1] * dy + v1[2] * dz;
        a3[1] += wi * y0 * y0;
        a3[2] += wi * y1 * y1;
    }
    cta_sum<3>(a3, scratch, part3);
    cluster_sum<3>(cl, part3, tot3);
    if (rank == 0 && threadIdx.x == 0) {
        const double sv0 = sqrt(fmax(tot3[1] / Wsum, 0.0));
        const double sv1 = sqrt(fmax(tot3[2] / Wsum, 0.0));
        int st = sol.status;
        if (src_degenerate(fmax(sv0, sv1), fmin(sv0, sv1))) st = EC3R_ST_DEGENERATE;
        out_status[b] = st;
        write_sim3(out_sim3 + 8 * b, sol);
        out_rms[b] = sqrt(fmax(tot3[0] / Wsum, 0.0));
    }
    cl.sync();  // keep shared memory alive until every rank has read it
}

// ---------------------------------------------------------------------------
// Pixel-identity registration edges over the resident frame pool.

struct PoolArgs {
    const float* depth;
    const float* conf;
    const double* slot_poses;  // n_slots x 8
    const int32_t* seg_slots;  // n_seg x 2
    const int32_t* edge_seg;   // n_edges + 1
    int H, W;
    double fx, fy, cx, cy;
    double floor_frac;
    int min_corr, with_scale;
    float inv_w;  // 1/W for the division-free row split (images < 2^21 pixels)
    int use_tma;  // planes 16-byte aligned and H*W % 4 == 0: TMA-staged walk
    int ncl;      // CTAs per edge (the cluster size of the launch)
};

// Row / column of pixel px without an integer division: floor((px + 1/2) / W)
// through a float reciprocal is exact while px < 2^21 (relative error 2^-22
// against a fractional-part distance of at least 1/(2W)); larger images take
// the integer division.
// (scalars, not the PoolArgs reference: a reference to the kernel parameter
// makes ptxas copy the struct to local memory and reload it per pixel)
__device__ __forceinline__ void pix_uv(float inv_w, int W, int px, int& u, int& v) {
    if (inv_w > 0.f) v = __float2int_rd(__fmul_rn((float)px + 0.5f, inv_w));
    else v = px / W;
    u = px - v * W;
}

// Shared column tables are stored by (u mod 4, u / 4): the lanes of a warp
// visit pixels 4 apart in each of their four sub-steps, so this layout puts
// them on consecutive doubles (no bank conflicts) instead of 32 bytes apart.
__device__ __forceinline__ int col_ix(int u, int Wq) { return (u & 3) * Wq + (u >> 2); }

__device__ __forceinline__ void load_rot(const double* x8, double R[3][3], double t[3]) {
    quat_to_mat(x8 + 1, R);
    t[0] = x8[5]; t[1] = x8[6]; t[2] = x8[7];
}

// Visit every pixel of the edge's segments owned by this thread (4 pixels per
// visit: one 128-bit load from each of the four planes when aligned).
// seg_fn(sa, sb) runs on the whole CTA at the start of every segment,
// bracketed by CTA barriers, so it may rebuild shared tables.
template <class S, class F>
__device__ __forceinline__ void for_each_pixel4_seg(const PoolArgs& a, int s0, int s1, int rank, S&& seg_fn,
                                                    F&& f) {
    const int HW = a.H * a.W;
    const bool vec = (HW & 3) == 0;
    for (int sg = s0; sg < s1; ++sg) {
        const int sa = a.seg_slots[2 * sg], sb = a.seg_slots[2 * sg + 1];
        __syncthreads();
        seg_fn(sa, sb);
        __syncthreads();
        const float* da = a.depth + (size_t)sa * HW;
        const float* ca = a.conf + (size_t)sa * HW;
        const float* db = a.depth + (size_t)sb * HW;
        const float* cb = a.conf + (size_t)sb * HW;
        auto load = [&](int pix, float4& za, float4& wa, float4& zb, float4& wb) {
            if (vec) {
                za = __ldg(reinterpret_cast<const float4*>(da + pix));
                wa = __ldg(reinterpret_cast<const float4*>(ca + pix));
                zb = __ldg(reinterpret_cast<const float4*>(db + pix));
                wb = __ldg(reinterpret_cast<const float4*>(cb + pix));
            } else {
                float t0[4], t1[4], t2[4], t3[4];
                for (int k = 0; k < 4; ++k) {
                    const bool in = pix + k < HW;
                    t0[k] = in ? da[pix + k] : 0.f; t1[k] = in ? ca[pix + k] : 0.f;
                    t2[k] = in ? db[pix + k] : 0.f; t3[k] = in ? cb[pix + k] : 0.f;
                }
                za = make_float4(t0[0], t0[1], t0[2], t0[3]); wa = make_float4(t1[0], t1[1], t1[2], t1[3]);
                zb = make_float4(t2[0], t2[1], t2[2], t2[3]); wb = make_float4(t3[0], t3[1], t3[2], t3[3]);
            }
        };
        // the next visit's four 16-byte loads are in flight while this one
        // is reduced
        const int kStride = 4 * a.ncl * UM_NT;
        int pix = 4 * (rank * UM_NT + threadIdx.x);
        float4 za, wa, zb, wb;
        if (pix < HW) load(pix, za, wa, zb, wb);
        for (; pix < HW; pix += kStride) {
            float4 nza, nwa, nzb, nwb;
            if (pix + kStride < HW) load(pix + kStride, nza, nwa, nzb, nwb);
            f(sg, sa, sb, pix, za, wa, zb, wb);
            za = nza; wa = nwa; zb = nzb; wb = nwb;
        }
    }
}

// The same walk with the four planes staged in shared memory by TMA bulk
// copies: a ring of RE_NS stages of 4 x 4 KB (one visit of the CTA: 1,024
// pixels per plane), RE_NS - 1 visits in flight, one mbarrier per stage.
// Planes must be 16-byte aligned with H*W % 4 == 0 (checked by the caller).
#ifndef EC3R_RE_NS
#define EC3R_RE_NS 3
#endif
constexpr int RE_NS = EC3R_RE_NS;
constexpr int RE_CHUNK = 4 * UM_NT;  // pixels per plane per visit
struct Ring {
    float* buf;          // [RE_NS][4][RE_CHUNK]
    uint64_t* bar;       // [RE_NS]
    uint32_t parity;     // bit s: next wait parity of stage s
    int next;            // stage of the next visit
};

__device__ __forceinline__ uint32_t re_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class S, class F>
__device__ __forceinline__ void for_each_pixel4_seg_tma(const PoolArgs& a, int s0, int s1, int rank, Ring& rg,
                                                        S&& seg_fn, F&& f) {
    const int HW = a.H * a.W;
    const int kStride = 4 * a.ncl * UM_NT;
    const int base0 = 4 * rank * UM_NT;
    const int n_it = base0 < HW ? (HW - base0 + kStride - 1) / kStride : 0;
    for (int sg = s0; sg < s1; ++sg) {
        const int sa = a.seg_slots[2 * sg], sb = a.seg_slots[2 * sg + 1];
        __syncthreads();
        seg_fn(sa, sb);
        __syncthreads();
        const float* src[4] = {a.depth + (size_t)sa * HW, a.conf + (size_t)sa * HW, a.depth + (size_t)sb * HW,
                               a.conf + (size_t)sb * HW};
        auto issue = [&](int it, int st) {
            const int pb = base0 + it * kStride;
            const uint32_t bytes = 4u * (uint32_t)min(RE_CHUNK, HW - pb);
            const uint32_t bar = re_smem_u32(rg.bar + st);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4u * bytes)
                         : "memory");
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        re_smem_u32(rg.buf + (st * 4 + pl) * RE_CHUNK)),
                    "l"(src[pl] + pb), "r"(bytes), "r"(bar)
                    : "memory");
        };
        if (threadIdx.x == 0)
            for (int j = 0; j < min(RE_NS, n_it); ++j) issue(j, (rg.next + j) % RE_NS);
        for (int it = 0; it < n_it; ++it) {
            const int st = rg.next;
            rg.next = (st + 1 == RE_NS) ? 0 : st + 1;
            const uint32_t par = (rg.parity >> st) & 1u;
            rg.parity ^= 1u << st;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "RE_WAIT_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra RE_WAIT_%=;\n"
                "}\n" ::"r"(re_smem_u32(rg.bar + st)),
                "r"(par)
                : "memory");
            const int pix = base0 + it * kStride + 4 * threadIdx.x;
            if (pix < HW) {
                const float* b = rg.buf + st * 4 * RE_CHUNK + 4 * threadIdx.x;
                const float4 za = *reinterpret_cast<const float4*>(b);
                const float4 wa = *reinterpret_cast<const float4*>(b + RE_CHUNK);
                const float4 zb = *reinterpret_cast<const float4*>(b + 2 * RE_CHUNK);
                const float4 wb = *reinterpret_cast<const float4*>(b + 3 * RE_CHUNK);
                f(sg, sa, sb, pix, za, wa, zb, wb);
            }
            __syncthreads();  // stage st is free again
            if (threadIdx.x == 0 && it + RE_NS < n_it) issue(it + RE_NS, st);
        }
    }
}

template <typename F>
__device__ __forceinline__ void for_each_pixel4(const PoolArgs& a, int s0, int s1, int rank, F&& f) {
    for_each_pixel4_seg(a, s0, s1, rank, [](int, int) {}, f);
}

#ifndef EC3R_RE_MINB
#define EC3R_RE_MINB 2  // resident CTAs per SM the register budget is sized for
#endif
// Launched with a runtime cluster size a.ncl (<= 8, cudaLaunchKernelEx).
__global__ void __launch_bounds__(UM_NT, EC3R_RE_MINB)
register_edges_kernel(PoolArgs a, double* __restrict__ out_sim3, double* __restrict__ out_rms,
                      int64_t* __restrict__ out_count, int64_t* __restrict__ out_npairs,
                      int32_t* __restrict__ out_status, uint8_t* __restrict__ keep_masks) {
    extern __shared__ double tabs[];  // xc[4 Wq], yc[H]  (ray coefficients, backend.py:89)
    const int Wq = (a.W + 3) >> 2, Wp = 4 * Wq;
    double* xc = tabs;
    double* yc = tabs + Wp;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int e = blockIdx.x / a.ncl;
    const int s0 = a.edge_seg[e], s1 = a.edge_seg[e + 1];
    __shared__ double scratch[(UM_NT / 32) * 24];
    __shared__ double part2[24];
    __shared__ double tot2[24], tot3[4];
    __shared__ Solution sol;
    for (int u = threadIdx.x; u < a.W; u += UM_NT) xc[col_ix(u, Wq)] = (u - a.cx) / a.fx;
    for (int v = threadIdx.x; v < a.H; v += UM_NT) yc[v] = (v - a.cy) / a.fy;
    // TMA ring after the tables (xc, yc, 2 x (col, row) = 7 (H + Wp) doubles)
    __shared__ __align__(8) uint64_t ring_bar[RE_NS];
    Ring rg;
    rg.buf = reinterpret_cast<float*>(tabs + 7 * (a.H + Wp));
    rg.bar = ring_bar;
    rg.parity = 0;
    rg.next = 0;
    const bool use_tma = a.use_tma != 0;
    const float inv_w = a.inv_w;
    if (threadIdx.x == 0 && use_tma) {
        for (int st = 0; st < RE_NS; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(re_smem_u32(ring_bar + st)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int W = a.W;

    // ---- shift: fp64 mean of a fixed 8 x 8 sample of the first segment's
    // valid pixels (identical in every CTA of the cluster), so the raw
    // moments are centred before the single streaming pass; the sample's
    // max w seeds the running floor bound below.
    double shp[3], shq[3];
    float wsamp;
    {
        // scratch in the (not yet used) ring memory
        double (*smp)[7] = reinterpret_cast<double (*)[7]>(tabs + 7 * (a.H + Wp));
        float* smw = reinterpret_cast<float*>(tabs + 7 * (a.H + Wp) + 64 * 7);
        const int sa = a.seg_slots[2 * s0], sb = a.seg_slots[2 * s0 + 1];
        const size_t HW = (size_t)a.H * a.W;
        if (threadIdx.x < 64) {
            const int i = threadIdx.x >> 3, j = threadIdx.x & 7;
            const int v = ((2 * i + 1) * a.H) / 16, u = ((2 * j + 1) * W) / 16;
            const size_t px = (size_t)v * W + u;
            const float zA = a.depth[(size_t)sa * HW + px], zB = a.depth[(size_t)sb * HW + px];
            const float cA = a.conf[(size_t)sa * HW + px], cB = a.conf[(size_t)sb * HW + px];
            const bool ok = zA > 0.f && zB > 0.f;
            double R[3][3], t[3];
            const double x = xc[col_ix(u, Wq)], y = yc[v];
            load_rot(a.slot_poses + 8 * sa, R, t);
            for (int k = 0; k < 3; ++k) smp[threadIdx.x][k] = ok ? zA * (R[k][0] * x + R[k][1] * y + R[k][2]) + t[k] : 0.0;
            load_rot(a.slot_poses + 8 * sb, R, t);
            for (int k = 0; k < 3; ++k)
                smp[threadIdx.x][3 + k] = ok ? zB * (R[k][0] * x + R[k][1] * y + R[k][2]) + t[k] : 0.0;
            smp[threadIdx.x][6] = ok ? 1.0 : 0.0;
            smw[threadIdx.x] = ok ? fminf(cA, cB) : -1.0f;
        }
        __syncthreads();
        __shared__ double shift_sh[7];
        if (threadIdx.x < 7) {  // column sums in sample order
            double acc = 0;
            for (int k = 0; k < 64; ++k) acc += smp[k][threadIdx.x];
            shift_sh[threadIdx.x] = acc;
        } else if (threadIdx.x == 32) {
            float wm = -1.0f;
            for (int k = 0; k < 64; ++k) wm = fmaxf(wm, smw[k]);
            smw[64] = wm;
        }
        __syncthreads();
        const double cnt = shift_sh[6];
        if (cnt > 0) {
            for (int k = 0; k < 3; ++k) { shp[k] = shift_sh[k] / cnt; shq[k] = shift_sh[3 + k] / cnt; }
        } else {  // no valid sample pixel: the first segment's frame origins
            double R[3][3], t[3];
            load_rot(a.slot_poses + 8 * sa, R, t);
            for (int k = 0; k < 3; ++k) shp[k] = t[k];
            load_rot(a.slot_poses + 8 * sb, R, t);
            for (int k = 0; k < 3; ++k) shq[k] = t[k];
        }
        wsamp = smw[64];
    }

    // ---- single pass: validity count, max w, and the shifted float64 raw
    // moments of every pixel that is certainly kept.  keep = w >= floor with
    // floor = frac * max(w) (mapping.py:176-177) is only known after the
    // pass, but confidences lie in [0, 1] (backend.py:51-58, :262), so
    // max(w) <= 1 and every w >= tau = frac * 1 is kept; a w below
    // frac * (running max) is certainly dropped.  The few pixels in between
    // are listed per thread and settled once the floor is known.  Inputs
    // outside the contract (max(w) > 1) or a full list re-run the two-pass
    // form (uniform decision in the cluster), so the result never depends
    // on the bound.
    double* colA = yc + a.H;          // [3][4 Wq] (col_ix layout)
    double* rowA = colA + 3 * Wp;     // [3][H]
    double* colB = rowA + 3 * a.H;    // [3][4 Wq]
    double* rowB = colB + 3 * Wp;     // [3][H]
    __shared__ double tAB[6];
    auto build = [&](int sa, int sb) {
        double Ra[3][3], ta_[3], Rb[3][3], tb_[3];
        load_rot(a.slot_poses + 8 * sa, Ra, ta_);
        load_rot(a.slot_poses + 8 * sb, Rb, tb_);
        for (int u = threadIdx.x; u < W; u += UM_NT)
            for (int i = 0; i < 3; ++i) {
                colA[i * Wp + col_ix(u, Wq)] = Ra[i][0] * xc[col_ix(u, Wq)] + Ra[i][2];
                colB[i * Wp + col_ix(u, Wq)] = Rb[i][0] * xc[col_ix(u, Wq)] + Rb[i][2];
            }
        for (int v = threadIdx.x; v < a.H; v += UM_NT)
            for (int i = 0; i < 3; ++i) {
                rowA[i * a.H + v] = Ra[i][1] * yc[v];
                rowB[i * a.H + v] = Rb[i][1] * yc[v];
            }
        if (threadIdx.x < 3) {
            tAB[threadIdx.x] = ta_[threadIdx.x] - shp[threadIdx.x];
            tAB[3 + threadIdx.x] = tb_[threadIdx.x] - shq[threadIdx.x];
        }
    };
    double a2[24];
#pragma unroll
    for (int k = 0; k < 24; ++k) a2[k] = 0;
    auto add_moments = [&](double wi, const double (&pp)[3], const double (&qq)[3]) {
        a2[0] += wi;
        a2[1] += 1.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double wp = wi * pp[i];
            a2[2 + i] += wp;
            a2[5 + i] += wi * qq[i];
#pragma unroll
            for (int j = 0; j < 3; ++j) a2[8 + 3 * j + i] += wp * qq[j];  // sum w q_j p_i
        }
        const double wp0 = wi * pp[0], wp1 = wi * pp[1], wp2 = wi * pp[2];
        a2[17] += wp0 * pp[0]; a2[18] += wp0 * pp[1]; a2[19] += wp0 * pp[2];
        a2[20] += wp1 * pp[1]; a2[21] += wp1 * pp[2]; a2[22] += wp2 * pp[2];
        a2[23] += wi * (qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2]);
    };
    // one moment-pass body: keep(valid, wf) decides per pixel; 'unc' pixels
    // (single pass only) go to the thread's list
    constexpr int kUnc = 4;
    __shared__ int2 unc_list[UM_NT][kUnc];
    int n_unc = 0;
    bool unc_full = false;
    // float thresholds: (double)w >= d  <=>  w >= float_ru(d) for float w
    const float tau_f = __double2float_ru(__dmul_rn(a.floor_frac, 1.0));
    float m_run = wsamp;
    float lo_f = m_run > 0.f ? __double2float_ru(__dmul_rn(a.floor_frac, (double)m_run)) : 0.f;
    int nvalid_t = 0;
    auto pass = [&](auto single_c, float floor_f) {
        constexpr bool single = decltype(single_c)::value;
        auto body = [&](int sg, int sa, int sb, int pix, float4 za, float4 wa, float4 zb, float4 wb) {
            const float zA[4] = {za.x, za.y, za.z, za.w}, cA[4] = {wa.x, wa.y, wa.z, wa.w};
            const float zB[4] = {zb.x, zb.y, zb.z, zb.w}, cB[4] = {wb.x, wb.y, wb.z, wb.w};
            uint32_t kbits = 0;
            int u0, v0;
            pix_uv(inv_w, W, pix, u0, v0);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool valid = zA[k] > 0.f && zB[k] > 0.f;
                const float wf = fminf(cA[k], cB[k]);
                bool keep;
                if constexpr (single) {
                    nvalid_t += valid;
                    if (valid && wf > m_run) {
                        m_run = wf;
                        lo_f = __double2float_ru(__dmul_rn(a.floor_frac, (double)wf));
                    }
                    keep = valid && wf >= tau_f;
                    if (valid && !keep && !(wf < lo_f)) {
                        if (n_unc < kUnc) unc_list[threadIdx.x][n_unc++] = make_int2(sg, pix + k);
                        else unc_full = true;
                    }
                } else {
                    keep = valid && wf >= floor_f;  // mapping.py:177
                }
                if (keep) {
                    kbits |= 1u << (8 * k);
                    int u = u0 + k, v = v0;
                    if (u >= W) pix_uv(inv_w, W, pix + k, u, v);
                    const int cu = col_ix(u, Wq);
                    const double zaa = zA[k], zbb = zB[k];
                    double pp[3], qq[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        pp[i] = zaa * (colA[i * Wp + cu] + rowA[i * a.H + v]) + tAB[i];
                        qq[i] = zbb * (colB[i * Wp + cu] + rowB[i * a.H + v]) + tAB[3 + i];
                    }
                    add_moments((double)wf, pp, qq);
                }
            }
            if (keep_masks) {
                const int HW = a.H * a.W;
                uint8_t* km = keep_masks + (size_t)sg * HW + pix;
                if (((HW & 3) == 0)) *reinterpret_cast<uint32_t*>(km) = kbits;
                else for (int k = 0; k < 4 && pix + k < HW; ++k) km[k] = (kbits >> (8 * k)) & 1;
            }
        };
        if (use_tma) for_each_pixel4_seg_tma(a, s0, s1, rank, rg, build, body);
        else for_each_pixel4_seg(a, s0, s1, rank, build, body);
    };
    pass(std::true_type{}, 0.f);

    // cluster totals of the pass: valid count, max w, list overflow
    float wmax = m_run;
    unsigned full = unc_full ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        nvalid_t += __shfl_xor_sync(0xffffffffu, nvalid_t, o);
        full |= __shfl_xor_sync(0xffffffffu, full, o);
    }
    __shared__ float wmax_warp[UM_NT / 32];
    __shared__ int nv_warp[UM_NT / 32];
    __shared__ unsigned full_warp[UM_NT / 32];
    __shared__ double part1[3];
    __shared__ double tot1[3];
    if ((threadIdx.x & 31) == 0) {
        wmax_warp[threadIdx.x >> 5] = wmax;
        nv_warp[threadIdx.x >> 5] = nvalid_t;
        full_warp[threadIdx.x >> 5] = full;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = -1.0f;
        long long nv = 0;
        unsigned f = 0;
        for (int w = 0; w < UM_NT / 32; ++w) { m = fmaxf(m, wmax_warp[w]); nv += nv_warp[w]; f |= full_warp[w]; }
        part1[0] = (double)nv;
        part1[1] = (double)m;
        part1[2] = (double)f;
    }
    cl.sync();
    if (threadIdx.x == 0) {
        double nv = 0, m = -1.0, f = 0;
        for (int c = 0; c < a.ncl; ++c) {
            const double* pc = cl.map_shared_rank(part1, c);
            nv += pc[0];
            m = fmax(m, pc[1]);
            f = fmax(f, pc[2]);
        }
        tot1[0] = nv; tot1[1] = m; tot1[2] = f;
    }
    __syncthreads();
    const double nvalid = tot1[0];
    if (rank == 0 && threadIdx.x == 0) out_npairs[e] = (int64_t)nvalid;
    if (nvalid < a.min_corr) {  // mapping.py:174
        if (rank == 0 && threadIdx.x == 0) { out_status[e] = EC3R_ST_SKIP; out_count[e] = 0; }
        cl.sync();
        return;
    }
    // floor = frac * float(w.max())  (mapping.py:176), exact in float64
    const double floorv = __dmul_rn(a.floor_frac, tot1[1]);
    if (tot1[2] != 0.0 || !(tot1[1] <= 1.0)) {
        // outside the single-pass bound: the two-pass form (moments of every
        // w >= floor from scratch; rewrites the keep mask)
#pragma unroll
        for (int k = 0; k < 24; ++k) a2[k] = 0;
        pass(std::false_type{}, __double2float_ru(floorv));
    } else {
        // settle the thread's listed pixels (exact float64 chain, own order)
        const size_t HW = (size_t)a.H * a.W;
        for (int i = 0; i < n_unc; ++i) {
            const int2 ent = unc_list[threadIdx.x][i];
            const int sa = a.seg_slots[2 * ent.x], sb = a.seg_slots[2 * ent.x + 1];
            const float cA = a.conf[(size_t)sa * HW + ent.y], cB = a.conf[(size_t)sb * HW + ent.y];
            const float wf = fminf(cA, cB);
            if (!((double)wf >= floorv)) continue;
            const float zA = a.depth[(size_t)sa * HW + ent.y], zB = a.depth[(size_t)sb * HW + ent.y];
            int u, v;
            pix_uv(inv_w, W, ent.y, u, v);
            const double x = xc[col_ix(u, Wq)], y = yc[v];
            double R[3][3], t[3], pp[3], qq[3];
            load_rot(a.slot_poses + 8 * sa, R, t);
            for (int k = 0; k < 3; ++k) pp[k] = (double)zA * (R[k][0] * x + R[k][2] + R[k][1] * y) + (t[k] - shp[k]);
            load_rot(a.slot_poses + 8 * sb, R, t);
            for (int k = 0; k < 3; ++k) qq[k] = (double)zB * (R[k][0] * x + R[k][2] + R[k][1] * y) + (t[k] - shq[k]);
            add_moments((double)wf, pp, qq);
            if (keep_masks) keep_masks[(size_t)ent.x * HW + ent.y] = 1;
        }
    }
    cta_sum<24>(a2, scratch, part2);
    // only rank 0 finishes the edge: it sums the published partials in rank
    // order, and once it has read them the other CTAs leave (their SMs take
    // the next edges while rank 0 runs the serial closed form)
    cl.sync();
    if (rank == 0 && threadIdx.x < 24) {
        double r = 0;
        for (int c = 0; c < a.ncl; ++c) r += cl.map_shared_rank(part2, c)[threadIdx.x];
        tot2[threadIdx.x] = r;
    }
    cl.sync();
    if (rank != 0) return;
    __syncthreads();
    const double Wsum = tot2[0], nkeep = tot2[1];
    int early = 0;
    if (nkeep < a.min_corr) early = EC3R_ST_SKIP;       // mapping.py:178
    else if (nkeep < 3) early = EC3R_ST_TOO_FEW;         // registration.py:59
    else if (!(Wsum > 0)) early = EC3R_ST_ALL_ZERO;      // registration.py:68
    if (early) {
        if (threadIdx.x == 0) { out_status[e] = early; out_count[e] = (int64_t)nkeep; }
        return;
    }
    // the closed form: thread 32 decomposes the source moments while thread 0
    // decomposes the covariance (two serial 3x3 Jacobi runs in parallel)
    __shared__ double eig_sh[12];  // lam[3], Vm[3][3]
    Moments mo;
    double U[3][3], sig[3], V[3][3], mp[3];
    if (threadIdx.x == 0 || threadIdx.x == 32) {
        mo.W = Wsum;
        double mq[3];
        for (int k = 0; k < 3; ++k) { mp[k] = tot2[2 + k] / Wsum; mq[k] = tot2[5 + k] / Wsum; }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) mo.C[i][j] = tot2[8 + 3 * i + j] / Wsum - mq[i] * mp[j];
        const double m00 = tot2[17] / Wsum - mp[0] * mp[0], m01 = tot2[18] / Wsum - mp[0] * mp[1];
        const double m02 = tot2[19] / Wsum - mp[0] * mp[2], m11 = tot2[20] / Wsum - mp[1] * mp[1];
        const double m12 = tot2[21] / Wsum - mp[1] * mp[2], m22 = tot2[22] / Wsum - mp[2] * mp[2];
        mo.M[0][0] = m00; mo.M[0][1] = mo.M[1][0] = m01; mo.M[0][2] = mo.M[2][0] = m02;
        mo.M[1][1] = m11; mo.M[1][2] = mo.M[2][1] = m12; mo.M[2][2] = m22;
        mo.varq = tot2[23] / Wsum - (mq[0] * mq[0] + mq[1] * mq[1] + mq[2] * mq[2]);
        for (int k = 0; k < 3; ++k) { mo.pbar[k] = shp[k] + mp[k]; mo.qbar[k] = shq[k] + mq[k]; }
        if (threadIdx.x == 32) {
            double Um[3][3], Vm[3][3], lam[3];
            svd3_jacobi(mo.M, Um, lam, Vm);  // symmetric PSD: singular values = eigenvalues
            for (int k = 0; k < 3; ++k) eig_sh[k] = lam[k];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) eig_sh[3 + 3 * i + j] = Vm[i][j];
        } else {
            svd3_jacobi(mo.C, U, sig, V);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double lam[3], Vm[3][3];
        for (int k = 0; k < 3; ++k) lam[k] = eig_sh[k];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) Vm[i][j] = eig_sh[3 + 3 * i + j];
        umeyama_finish(mo, a.with_scale, U, sig, V, lam, Vm, sol);
        // stash the in-shift source centroid for the refinement pass
        sol.rms2_closed = fmax(sol.rms2_closed, 0.0);
        tot3[0] = mp[0]; tot3[1] = mp[1]; tot3[2] = mp[2];
    }
    __syncthreads();
    bool degenerate = src_degenerate(sqrt(sol.src_lambda[0]), sqrt(sol.src_lambda[1]));
    // Gram eigenvalues resolve sv1/sv0 only down to ~1e-8: near-degenerate
    // edges get the direct eigenbasis pass (uniform decision in the cluster).
    if (sol.src_lambda[1] <= 1e-10 * sol.src_lambda[0]) {
        const double mp0 = tot3[0], mp1 = tot3[1], mp2 = tot3[2];
        double v0[3], v1[3];
        for (int i = 0; i < 3; ++i) { v0[i] = sol.src_V[i][0]; v1[i] = sol.src_V[i][1]; }
        double a3[2] = {0, 0};
        auto eig_body = [&](int sg, int sa, int sb, int pix, float4 za, float4 wa, float4 zb, float4 wb) {
            const float zA[4] = {za.x, za.y, za.z, za.w}, cA[4] = {wa.x, wa.y, wa.z, wa.w};
            const float zB[4] = {zb.x, zb.y, zb.z, zb.w}, cB[4] = {wb.x, wb.y, wb.z, wb.w};
            for (int k = 0; k < 4; ++k) {
                const float wf = fminf(cA[k], cB[k]);
                if (zA[k] > 0.f && zB[k] > 0.f && (double)wf >= floorv) {
                    int u, v;
                    pix_uv(inv_w, W, pix + k, u, v);
                    const double z = zA[k];
                    double d[3];
                    for (int i = 0; i < 3; ++i) d[i] = z * (colA[i * Wp + col_ix(u, Wq)] + rowA[i * a.H + v]) + tAB[i];
                    d[0] -= mp0; d[1] -= mp1; d[2] -= mp2;
                    const double y0 = v0[0] * d[0] + v0[1] * d[1] + v0[2] * d[2];
                    const double y1 = v1[0] * d[0] + v1[1] * d[1] + v1[2] * d[2];
                    a3[0] += wf * y0 * y0;
                    a3[1] += wf * y1 * y1;
                }
            }
        };
        // rank 0 alone (the others have left): every rank's share in turn
        for (int r = 0; r < a.ncl; ++r) {
            if (use_tma) for_each_pixel4_seg_tma(a, s0, s1, r, rg, build, eig_body);
            else for_each_pixel4_seg(a, s0, s1, r, build, eig_body);
        }
        __syncthreads();
        cta_sum<2>(a3, scratch, tot3 + 2);  // tot3[2..3]; tot3[0..1] no longer needed
        const double sv0 = sqrt(fmax(tot3[2] / Wsum, 0.0)), sv1 = sqrt(fmax(tot3[3] / Wsum, 0.0));
        degenerate = src_degenerate(fmax(sv0, sv1), fmin(sv0, sv1));
    }
    if (threadIdx.x == 0) {
        int st = sol.status;
        if (degenerate) st = EC3R_ST_DEGENERATE;
        out_status[e] = st;
        out_count[e] = (int64_t)nkeep;
        write_sim3(out_sim3 + 8 * e, sol);
        out_rms[e] = sqrt(sol.rms2_closed);
    }
}

// ---------------------------------------------------------------------------
// Pose chaining of register_submap (mapping.py:200-204): the strongest edge
// (max count, first on ties — Python max()) sets
// global_j = global_partner o T (sim3_compose, liegroups.py:275-281).  The
// strongest edges are known before chaining, so the chain is pointer jumping
// over the partner tree (log2 rounds of parallel compositions); keeping it on
// the device removes the host round trip between registration and fusion.
__device__ void sim3_compose_dev(const double* a, const double* b, double* o) {
    const double aw = a[1], ax = a[2], ay = a[3], az = a[4];
    const double bw = b[1], bx = b[2], by = b[3], bz = b[4];
    double q[4] = {aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                   aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw};
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double r[3];
    const double tb[3] = {b[5], b[6], b[7]};
    quat_rotate_exact(a + 1, tb, r);
    o[0] = a[0] * b[0];
    for (int k = 0; k < 4; ++k) o[1 + k] = q[k] / n;
    for (int k = 0; k < 3; ++k) o[5 + k] = a[0] * r[k] + a[5 + k];
}

// The chain is sequential: thread 0 walks the submaps with every input and
// the globals staged in shared memory (the dependent global round trips of
// a direct walk cost ~1 us per submap); all threads then write back.
constexpr int CHAIN_NT = 256;

__host__ __device__ inline size_t chain_par_extra(int n_sub) {
    return 16 + sizeof(double) * 16 * (size_t)n_sub + sizeof(int) * 4 * (size_t)n_sub;
}
__host__ __device__ inline size_t chain_smem(int n_sub, int n_edges) {
    return sizeof(double) * 8 * ((size_t)n_sub + n_edges) + sizeof(int64_t) * n_edges +
           sizeof(int32_t) * (2 * (size_t)n_edges + 2 * n_sub + 1) + 16;
}

// Submap j's registration outcome (mapping.py:162-211): submap 0 is the
// chain's fixed root (the first submap, or a sharded window's halo stub).
// For j > 0 the partners are the earlier submaps that were committed
// (status OK); edges to them are walked in partner order: SKIP edges
// (< min_correspondences) are dropped, the first error status aborts the
// submap (align_point_sets raises out of the loop), and no surviving edge
// means NoSharedKeyframes (SKIP).  Returns the strongest edge (max count,
// first on ties) or -1.
__device__ inline int chain_select(int j, const int32_t* eo, const int32_t* est, const int64_t* ec,
                                   const int32_t* ep, const int32_t* sst, int* st_out) {
    *st_out = EC3R_ST_OK;
    if (j == 0) return -1;
    int best = -1;
    for (int e = eo[j]; e < eo[j + 1]; ++e) {
        if (sst[ep[e]] != EC3R_ST_OK) continue;
        if (est[e] == EC3R_ST_SKIP) continue;
        if (est[e] != EC3R_ST_OK) { *st_out = est[e]; return -1; }
        if (best < 0 || ec[e] > ec[best]) best = e;
    }
    if (best < 0) *st_out = EC3R_ST_SKIP;
    return best;
}

__global__ void __launch_bounds__(CHAIN_NT) chain_poses_kernel(
    const double* __restrict__ esim, const int64_t* __restrict__ ecount, const int32_t* __restrict__ estatus,
    const int32_t* __restrict__ epartner, const int32_t* __restrict__ sub_edge_off, int n_sub,
    const int32_t* __restrict__ sub_slot_off, double* __restrict__ sub_globals, double* __restrict__ slot_globals,
    int32_t* __restrict__ sub_status, size_t smem_cap) {
    extern __shared__ double csh[];
    const int n_edges = sub_edge_off[n_sub];
    const bool staged = chain_smem(n_sub, n_edges) <= smem_cap;
    // staged: everything in shared memory; else walk the global arrays
    double* g = staged ? csh : sub_globals;
    const double* es = esim;
    const int64_t* ec = ecount;
    const int32_t* est = estatus;
    const int32_t* ep = epartner;
    const int32_t* eo = sub_edge_off;
    int32_t* sst = sub_status;
    if (staged) {
        double* es_s = g + 8 * (size_t)n_sub;
        int64_t* ec_s = reinterpret_cast<int64_t*>(es_s + 8 * (size_t)n_edges);
        int32_t* est_s = reinterpret_cast<int32_t*>(ec_s + n_edges);
        int32_t* ep_s = est_s + n_edges;
        int32_t* eo_s = ep_s + n_edges;
        int32_t* sst_s = eo_s + n_sub + 1;
        for (int i = threadIdx.x; i < 8 * n_sub; i += CHAIN_NT) g[i] = sub_globals[i];
        for (int i = threadIdx.x; i < 8 * n_edges; i += CHAIN_NT) es_s[i] = esim[i];
        for (int i = threadIdx.x; i < n_edges; i += CHAIN_NT) {
            ec_s[i] = ecount[i];
            est_s[i] = estatus[i];
            ep_s[i] = epartner[i];
        }
        for (int i = threadIdx.x; i <= n_sub; i += CHAIN_NT) eo_s[i] = sub_edge_off[i];
        es = es_s; ec = ec_s; est = est_s; ep = ep_s; eo = eo_s; sst = sst_s;
    }
    __syncthreads();
    // parallel form (pointer jumping over the partner tree) when its extra
    // arrays fit next to the staged inputs: every submap's strongest edge is
    // known up front, so global_j = global_root o (T_a o ... o T_j) and the
    // chain takes log2(depth) rounds instead of n_sub dependent steps
    int32_t* sst_w = sst;
    const size_t base_b = chain_smem(n_sub, n_edges);
    const bool par = staged && base_b + chain_par_extra(n_sub) <= smem_cap;
    if (par) {
        double* T0 = (double*)((char*)csh + ((base_b + 15) & ~(size_t)15));
        double* T1 = T0 + 8 * (size_t)n_sub;
        int* an0 = (int*)(T1 + 8 * (size_t)n_sub);
        int* an1 = an0 + n_sub;
        int* rt0 = an1 + n_sub;
        int* rt1 = rt0 + n_sub;
        // statuses and strongest edges first.  A submap that is not
        // committed is not a partner of later submaps, so status j depends on
        // its partners' (all < j): rounds of parallel re-evaluation from
        // "all committed" reach the sequential walk's result (after round r
        // every submap r partner-levels deep is final) and stop when nothing
        // changes -- two rounds when every edge is usable
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) sst_w[j] = EC3R_ST_OK;
        __syncthreads();
        for (;;) {
            for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
                int st;
                rt1[j] = chain_select(j, eo, est, ec, ep, sst_w, &st);
                an1[j] = st;
            }
            __syncthreads();
            int changed = 0;
            for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
                changed |= an1[j] != sst_w[j];
                sst_w[j] = an1[j];
            }
            if (!__syncthreads_or(changed)) break;
        }
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
            const int best = rt1[j];
            an0[j] = best >= 0 ? ep[best] : -1;
            rt0[j] = best >= 0 ? -1 : j;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
            const int best = rt1[j];
            for (int k = 0; k < 8; ++k) T0[8 * j + k] = best >= 0 ? es[8 * best + k] : (k < 2 ? 1.0 : 0.0);
        }
        __syncthreads();
        for (int span = 1; span < n_sub; span <<= 1) {
            for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
                const int a = an0[j];
                if (a >= 0) {
                    sim3_compose_dev(T0 + 8 * a, T0 + 8 * j, T1 + 8 * j);
                    an1[j] = an0[a];
                    rt1[j] = an0[a] < 0 ? rt0[a] : -1;
                } else {
                    for (int k = 0; k < 8; ++k) T1[8 * j + k] = T0[8 * j + k];
                    an1[j] = -1;
                    rt1[j] = rt0[j];
                }
            }
            __syncthreads();
            double* tt = T0; T0 = T1; T1 = tt;
            int* ta = an0; an0 = an1; an1 = ta;
            int* tr = rt0; rt0 = rt1; rt1 = tr;
        }
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) {
            const int r = rt0[j];
            if (r != j) {  // roots keep their given global
                double o[8];
                sim3_compose_dev(g + 8 * r, T0 + 8 * j, o);
                for (int k = 0; k < 8; ++k) T1[8 * j + k] = o[k];
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT)
            if (rt0[j] != j)
                for (int k = 0; k < 8; ++k) g[8 * j + k] = T1[8 * j + k];
    } else if (threadIdx.x == 0) {
        for (int j = 0; j < n_sub; ++j) {
            int st;
            const int best = chain_select(j, eo, est, ec, ep, sst_w, &st);
            sst_w[j] = st;
            if (best >= 0) sim3_compose_dev(g + 8 * ep[best], es + 8 * best, g + 8 * j);
        }
    }
    __syncthreads();
    if (staged) {
        for (int i = threadIdx.x; i < 8 * n_sub; i += CHAIN_NT) sub_globals[i] = g[i];
        for (int j = threadIdx.x; j < n_sub; j += CHAIN_NT) sub_status[j] = sst[j];
    }
    // slot broadcast: a warp per submap, lane (slot, k) of its contiguous
    // slots (sub_slot_off) -- no per-slot search through global offsets
    const int lane = threadIdx.x & 31;
    for (int j = threadIdx.x >> 5; j < n_sub; j += CHAIN_NT / 32) {
        const int s0 = sub_slot_off[j], s1 = sub_slot_off[j + 1];
        for (int i = lane; i < 8 * (s1 - s0); i += 32) slot_globals[8 * (size_t)s0 + i] = g[8 * j + (i & 7)];
    }
}


}  // namespace ec3r

using namespace ec3r;

extern "C" int ec3r_chain_poses(const double* edge_sim3, const int64_t* edge_count, const int32_t* edge_status,
                                const int32_t* edge_partner, const int32_t* sub_edge_off, int n_sub,
                                const int32_t* sub_slot_off, double* sub_globals, double* slot_globals,
                                int32_t* sub_status, void* stream) {
    if (n_sub < 0 || !sub_edge_off || !sub_globals || !sub_status) return EC3R_EARG;
    if (n_sub == 0) return EC3R_OK;
    // the edge count lives on the device: reserve the full opt-in shared
    // memory; a chain that does not fit walks global memory instead
    const size_t smem = 227 * 1024;
    // test knob: a smaller cap forces the staged-sequential or the global walk
    size_t cap = smem;
    if (const char* e = getenv("EC3R_CHAIN_SMEM_CAP")) cap = std::min(smem, (size_t)strtoull(e, nullptr, 10));
    EC3R_CUDA_TRY(cudaFuncSetAttribute(chain_poses_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    chain_poses_kernel<<<1, CHAIN_NT, smem, as_stream(stream)>>>(edge_sim3, edge_count, edge_status, edge_partner,
                                                                sub_edge_off, n_sub, sub_slot_off, sub_globals,
                                                                slot_globals, sub_status, cap);
    EC3R_CHECK_LAUNCH("chain_poses_kernel");
    return EC3R_OK;
}

extern "C" size_t ec3r_umeyama_workspace(int) { return 0; }

extern "C" int ec3r_umeyama_batched(const double* p, const double* q, const double* w,
                                    const int64_t* offsets, int n_problems, int with_scale,
                                    double* out_sim3, double* out_rms, int32_t* out_status, void*,
                                    size_t, void* stream) {
    if (n_problems < 0 || !p || !q || !offsets || !out_sim3 || !out_rms || !out_status) return EC3R_EARG;
    if (n_problems == 0) return EC3R_OK;
    dim3 grid(n_problems * UM_CL), block(UM_NT);
    if (w)
        umeyama_explicit_kernel<true><<<grid, block, 0, as_stream(stream)>>>(p, q, w, offsets, with_scale,
                                                                            out_sim3, out_rms, out_status);
    else
        umeyama_explicit_kernel<false><<<grid, block, 0, as_stream(stream)>>>(p, q, w, offsets, with_scale,
                                                                             out_sim3, out_rms, out_status);
    EC3R_CHECK_LAUNCH("umeyama_explicit_kernel");
    return EC3R_OK;
}

extern "C" size_t ec3r_register_edges_workspace(int) { return 0; }

extern "C" int ec3r_register_edges(const float* depth_pool, const float* conf_pool, int H, int W,
                                   const double* K4_h, const double* slot_poses, const int32_t* seg_slots,
                                   const int32_t* edge_seg, int n_edges, double floor_frac, int min_corr,
                                   int with_scale, double* out_sim3, double* out_rms, int64_t* out_count,
                                   int64_t* out_npairs, int32_t* out_status, uint8_t* keep_masks, void*,
                                   size_t, void* stream) {
    if (n_edges < 0 || H <= 0 || W <= 0 || !depth_pool || !conf_pool || !K4_h || !slot_poses || !seg_slots ||
        !edge_seg)
        return EC3R_EARG;
    if (n_edges == 0) return EC3R_OK;
    PoolArgs a;
    a.depth = depth_pool; a.conf = conf_pool; a.slot_poses = slot_poses; a.seg_slots = seg_slots;
    a.edge_seg = edge_seg; a.H = H; a.W = W;
    a.fx = K4_h[0]; a.fy = K4_h[1]; a.cx = K4_h[2]; a.cy = K4_h[3];
    a.floor_frac = floor_frac; a.min_corr = min_corr; a.with_scale = with_scale;
    a.inv_w = (int64_t)H * W < (1 << 21) ? 1.0f / (float)W : 0.f;
    const size_t Wp = 4 * (size_t)((W + 3) / 4);
    a.use_tma = ((int64_t)H * W % 4 == 0) &&
                ((reinterpret_cast<uintptr_t>(depth_pool) | reinterpret_cast<uintptr_t>(conf_pool)) & 15) == 0 &&
                getenv("EC3R_RE_NOTMA") == nullptr;
    // xc, yc + two frames' col/row tables, then the TMA ring (which also holds
    // the 64-pixel shift sample: 64 x 7 doubles + 64 floats)
    const size_t ring = std::max(sizeof(float) * RE_NS * 4 * RE_CHUNK, sizeof(double) * 64 * 8 + 4);
    const size_t smem = sizeof(double) * 7 * (size_t)(H + Wp) + ring;
    if (smem > 48 * 1024) {
        EC3R_CUDA_TRY(cudaFuncSetAttribute(register_edges_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    }
    // Cluster size: one wave of clusters when the edges allow it.  With c
    // CTAs per edge the launch takes ceil(n / clusters_c) waves of 1/c of an
    // edge each plus a per-CTA fixed cost (tables, shift sample, closed form
    // on rank 0: ~3% of an edge's streaming, measured); pick the c in
    // {1, 2, 4, 8} minimising ceil(n / clusters_c) (1/c + 0.03), clusters_c
    // = the co-resident clusters of size c (cudaOccupancyMaxActiveClusters;
    // sizes 5-7 measured slower: they pack the GPCs worse).  EC3R_RE_CL
    // forces c.
    static std::atomic<int> max_clusters[4];  // per cluster size, computed once (benign duplicate queries)
    int ncl = 4;
    double best = 1e30;
    for (int i = 0; i < 4; ++i) {
        const int c = 1 << i;
        if (max_clusters[i].load() == 0) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)(c * 64));
            q.blockDim = dim3(UM_NT);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = (unsigned)c;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, register_edges_kernel, &q) != cudaSuccess || nc < 1) {
                cudaGetLastError();
                nc = std::max(1, 2 * kNumSMs / c);
            }
            max_clusters[i].store(nc);
        }
        const int mc = max_clusters[i].load();
        const double cost = (double)((n_edges + mc - 1) / mc) * (1.0 / c + 0.03);
        if (cost < best - 1e-12) { best = cost; ncl = c; }
    }
    if (const char* f = getenv("EC3R_RE_CL")) ncl = std::min(8, std::max(1, atoi(f)));
    a.ncl = ncl;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(n_edges * ncl));
    cfg.blockDim = dim3(UM_NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)ncl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    KernelTimer tk(TK_REGISTER, as_stream(stream));
    EC3R_CUDA_TRY(cudaLaunchKernelEx(&cfg, register_edges_kernel, a, out_sim3, out_rms, out_count, out_npairs,
                                     out_status, keep_masks));
    EC3R_CHECK_LAUNCH("register_edges_kernel");
    tk.stop();
    return EC3R_OK;
}

// ---------------------------------------------------------------------------
// Sharded chain (dist.WindowChain): rank r's chain is computed relative to
// its halo stub (the predecessor's last submap); the offset
// O_r = W_0 o W_1 o ... o W_{r-1} (W_q = window q's last-submap pose in its
// own frame, all-gathered) turns it into global poses.  Every thread
// recomputes the (<= world-long) prefix and left-composes its globals.
namespace ec3r {
__global__ void window_offset_kernel(const double* __restrict__ window_last, int rank, double* __restrict__ sub_globals,
                                     int n_sub, double* __restrict__ slot_globals, int64_t n_slots,
                                     double* __restrict__ offset_out) {
    double o[8] = {1.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < rank; ++q) {
        double t[8];
        sim3_compose_dev(o, window_last + 8 * q, t);
        for (int k = 0; k < 8; ++k) o[k] = t[k];
    }
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && offset_out)
        for (int k = 0; k < 8; ++k) offset_out[k] = o[k];
    double* g = i < n_sub ? sub_globals + 8 * i : (i - n_sub < n_slots ? slot_globals + 8 * (i - n_sub) : nullptr);
    if (!g) return;
    double in[8], out[8];
    for (int k = 0; k < 8; ++k) in[k] = g[k];
    sim3_compose_dev(o, in, out);
    for (int k = 0; k < 8; ++k) g[k] = out[k];
}
}  // namespace ec3r

extern "C" int ec3r_apply_window_offset(const double* window_last, int world, int rank, double* sub_globals,
                                        int n_sub, double* slot_globals, int64_t n_slots, double* offset_out,
                                        void* stream) {
    if (world < 1 || rank < 0 || rank >= world || n_sub < 0 || n_slots < 0) return EC3R_EARG;
    if ((rank > 0 && !window_last) || (n_sub && !sub_globals) || (n_slots && !slot_globals)) return EC3R_EARG;
    const int64_t n = (int64_t)n_sub + n_slots;
    if (n == 0 && !offset_out) return EC3R_OK;
    const int64_t blocks = (n + 127) / 128 > 0 ? (n + 127) / 128 : 1;
    window_offset_kernel<<<(unsigned)blocks, 128, 0, as_stream(stream)>>>(window_last, rank, sub_globals, n_sub,
                                                                        slot_globals, n_slots, offset_out);
    EC3R_CHECK_LAUNCH("window_offset_kernel");
    return EC3R_OK;
}
