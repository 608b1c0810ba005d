// K9: batched homography RANSAC for loop verification —
// estimate_homography_ransac (geometry.py:594-640) for many candidate pairs
// in three launches plus a host walk.
//
// The reference draws one 4-sample per iteration from
// np.random.default_rng(cfg.seed) (rng.choice(n, 4, replace=False),
// geometry.py:612), skips degenerate samples (:575-583) and failed DLTs, and
// stops adaptively (:620-625).  The draws do not depend on the outcomes, so
// every hypothesis of the max_iterations budget can be generated and scored
// at once:
//
//   hg_draw_kernel   one thread per problem replays numpy's PCG64 stream
//                    (128-bit LCG + XSL-RR, 32-bit halves buffered) through
//                    Generator.choice's path for size 4 (Floyd's sampling with
//                    Lemire-bounded integers, then a shuffle of the 4);
//   hg_hyp_kernel    one thread per (problem, iteration): the collinearity
//                    test (exact), Hartley normalisation (numpy op order) and
//                    the DLT null vector of the 8x9 system by Gaussian
//                    elimination with complete pivoting (LAPACK's SVD gives
//                    the same unit vector up to sign and rounding), det and
//                    h22 guards, H and H^-1;
//   hg_count_kernel  one warp per (problem, iteration): symmetric transfer
//                    errors (:558-572, numpy op order, _rn intrinsics) and the
//                    inlier count; -1 for skipped iterations;
//   host walk        the reference's sequential acceptance and adaptive
//                    max_iters in Python floats (math.log), over the counts;
//   hg_refit_kernel  one CTA per problem: the chosen hypothesis's mask, the
//                    all-inlier DLT (Hartley + 9x9 normal matrix + cyclic
//                    Jacobi, sv[-2] guard), its mask, and the keep rule
//                    (:633-639).
//
// Masks and counts equal the reference's unless an error lies within
// rounding (~1e-12 px) of the threshold; models agree to rounding.

#include <cub/block/block_reduce.cuh>

#include "common.cuh"

namespace ec3r {

constexpr int HG_REFIT_THREADS = 256;

// ---------------------------------------------------------------------------
// numpy PCG64 + Generator.choice(n, 4, replace=False)

struct Pcg64 {
    unsigned __int128 s, inc;
    int has32;
    uint32_t u32;
};

__device__ __forceinline__ uint64_t pcg_next64(Pcg64& g) {
    const unsigned __int128 mult = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    g.s = g.s * mult + g.inc;
    const uint64_t hi = (uint64_t)(g.s >> 64), lo = (uint64_t)g.s;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ uint32_t pcg_next32(Pcg64& g) {
    if (g.has32) {
        g.has32 = 0;
        return g.u32;
    }
    const uint64_t n = pcg_next64(g);
    g.has32 = 1;
    g.u32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
}

// random_bounded_uint64(off=0, rng=r, use_masked=false) for r < 2^32: Lemire.
// `extra` is set when a rejection drew another 32-bit word (probability
// < (r+1) / 2^32 per call).
__device__ __forceinline__ uint32_t pcg_bounded(Pcg64& g, uint32_t r, bool& extra) {
    if (r == 0) return 0;
    if (r == 0xFFFFFFFFu) return pcg_next32(g);
    const uint32_t ex = r + 1;
    uint64_t m = (uint64_t)pcg_next32(g) * ex;
    uint32_t left = (uint32_t)m;
    if (left < ex) {
        const uint32_t thr = (0xFFFFFFFFu - r) % ex;
        while (left < thr) {
            extra = true;
            m = (uint64_t)pcg_next32(g) * ex;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

// LCG jump-ahead (state after k steps) in O(log k) 128-bit multiplies
__device__ __forceinline__ unsigned __int128 pcg_advance(unsigned __int128 s, unsigned __int128 inc, uint64_t k) {
    unsigned __int128 cur_m = ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    unsigned __int128 cur_p = inc, acc_m = 1, acc_p = 0;
    while (k) {
        if (k & 1) {
            acc_m *= cur_m;
            acc_p = acc_p * cur_m + cur_p;
        }
        cur_p = (cur_m + 1) * cur_p;
        cur_m *= cur_m;
        k >>= 1;
    }
    return acc_m * s + acc_p;
}

// one Generator.choice(n, 4, replace=False) draw (Floyd + shuffle), in
// registers only
__device__ __forceinline__ int4 choice4(Pcg64& g, uint32_t j0, bool& extra) {
    uint32_t i0 = pcg_bounded(g, j0, extra);
    uint32_t i1 = pcg_bounded(g, j0 + 1, extra);
    i1 = (i1 == i0) ? j0 + 1 : i1;
    uint32_t i2 = pcg_bounded(g, j0 + 2, extra);
    i2 = (i2 == i0 || i2 == i1) ? j0 + 2 : i2;
    uint32_t i3 = pcg_bounded(g, j0 + 3, extra);
    i3 = (i3 == i0 || i3 == i1 || i3 == i2) ? j0 + 3 : i3;
    {  // _shuffle_int(4, 1, idx): i = 3, 2, 1 swaps idx[i] with idx[bounded(i)]
        const uint32_t r = pcg_bounded(g, 3u, extra), t = i3;
        i3 = r == 0 ? i0 : r == 1 ? i1 : r == 2 ? i2 : i3;
        i0 = r == 0 ? t : i0;
        i1 = r == 1 ? t : i1;
        i2 = r == 2 ? t : i2;
    }
    {
        const uint32_t r = pcg_bounded(g, 2u, extra), t = i2;
        i2 = r == 0 ? i0 : r == 1 ? i1 : i2;
        i0 = r == 0 ? t : i0;
        i1 = r == 1 ? t : i1;
    }
    {
        const uint32_t r = pcg_bounded(g, 1u, extra), t = i1;
        i1 = r == 0 ? i0 : i1;
        i0 = r == 0 ? t : i0;
    }
    return make_int4((int)i0, (int)i1, (int)i2, (int)i3);
}

__device__ __forceinline__ void load_pcg(const uint64_t* st, Pcg64& g) {
    g.s = ((unsigned __int128)st[0] << 64) | st[1];
    g.inc = ((unsigned __int128)st[2] << 64) | st[3];
    g.has32 = (int)st[4];
    g.u32 = (uint32_t)st[5];
}

// Parallel replay.  Without rejections every draw consumes exactly seven
// 32-bit words (4 Floyd + 3 shuffle; six when n == 4), so iteration `it`
// starts at word 7 it of the stream: thread t jumps the LCG to its first word and replays its
// iterations.  A thread that meets a rejection flags the problem, which the
// serial kernel below then redoes from the start.
constexpr int HG_DRAW_NT = 64;

__global__ void __launch_bounds__(HG_DRAW_NT) hg_draw_par_kernel(const int64_t* __restrict__ off, int iters,
                                                                 const uint64_t* __restrict__ state,
                                                                 int32_t* __restrict__ samples,
                                                                 int32_t* __restrict__ redo) {
    const int p = blockIdx.x;
    const int64_t n = off[p + 1] - off[p];
    if (threadIdx.x == 0) redo[p] = 0;
    if (n < 4) return;
    Pcg64 g;
    load_pcg(state + 6 * (size_t)p, g);
    __shared__ int flag;
    if (threadIdx.x == 0) flag = g.has32 ? 1 : 0;  // a buffered word shifts the stream: serial
    __syncthreads();
    if (flag) {
        if (threadIdx.x == 0) redo[p] = 1;
        return;
    }
    const int per = (iters + HG_DRAW_NT - 1) / HG_DRAW_NT;
    const int it0 = threadIdx.x * per, it1 = min(iters, it0 + per);
    bool extra = false;
    if (it0 < it1) {
        // bounded(0) draws nothing: with n == 4 a draw takes six words
        const uint64_t w = (n == 4 ? 6ull : 7ull) * (uint64_t)it0;  // first 32-bit word
        g.s = pcg_advance(g.s, g.inc, w >> 1);     // outputs before the word's
        g.has32 = 0;
        if (w & 1) (void)pcg_next32(g);            // odd word: the high half of the next output
        const uint32_t j0 = (uint32_t)(n - 4);
        int4* out = reinterpret_cast<int4*>(samples + (size_t)p * iters * 4);
        for (int it = it0; it < it1; ++it) out[it] = choice4(g, j0, extra);
    }
    if (extra) atomicOr(&flag, 1);
    __syncthreads();
    if (threadIdx.x == 0 && flag) redo[p] = 1;
}

// serial replay for flagged problems (rejections or a buffered word)
__global__ void hg_draw_serial_kernel(const int64_t* __restrict__ off, int P, const uint64_t* __restrict__ state,
                                      int iters, const int32_t* __restrict__ redo, int32_t* __restrict__ samples) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !redo[p]) return;
    const int64_t n = off[p + 1] - off[p];
    if (n < 4) return;
    Pcg64 g;
    load_pcg(state + 6 * (size_t)p, g);
    const uint32_t j0 = (uint32_t)(n - 4);
    bool extra = false;
    int4* out = reinterpret_cast<int4*>(samples + (size_t)p * iters * 4);
    for (int it = 0; it < iters; ++it) out[it] = choice4(g, j0, extra);
}

// ---------------------------------------------------------------------------
// hypotheses

__device__ __forceinline__ bool collinear3(const double (*p)[2], int drop) {
    int t[3], m = 0;
    for (int k = 0; k < 4; ++k)
        if (k != drop) t[m++] = k;
    const double d1x = xs(p[t[1]][0], p[t[0]][0]), d1y = xs(p[t[1]][1], p[t[0]][1]);
    const double d2x = xs(p[t[2]][0], p[t[0]][0]), d2y = xs(p[t[2]][1], p[t[0]][1]);
    return fabs(xs(xm(d1x, d2y), xm(d1y, d2x))) < 1e-9;
}

__device__ __forceinline__ bool sample_degenerate(const double (*p)[2]) {
    for (int d = 0; d < 4; ++d)
        if (collinear3(p, d)) return true;
    return false;
}

__device__ __forceinline__ double det3(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
           h[2] * (h[3] * h[7] - h[4] * h[6]);
}

__device__ __forceinline__ bool inv3(const double* h, double* o) {
    const double d = det3(h);
    if (d == 0.0) return false;
    const double r = 1.0 / d;
    o[0] = (h[4] * h[8] - h[5] * h[7]) * r;
    o[1] = (h[2] * h[7] - h[1] * h[8]) * r;
    o[2] = (h[1] * h[5] - h[2] * h[4]) * r;
    o[3] = (h[5] * h[6] - h[3] * h[8]) * r;
    o[4] = (h[0] * h[8] - h[2] * h[6]) * r;
    o[5] = (h[2] * h[3] - h[0] * h[5]) * r;
    o[6] = (h[3] * h[7] - h[4] * h[6]) * r;
    o[7] = (h[1] * h[6] - h[0] * h[7]) * r;
    o[8] = (h[0] * h[4] - h[1] * h[3]) * r;
    return true;
}

// Hartley normalisation of 4 points (geometry.py:534-543, numpy op order):
// returns s, c and writes the normalised points.
__device__ __forceinline__ void hartley4(const double (*p)[2], double (*q)[2], double& s, double& cx, double& cy) {
    cx = __ddiv_rn(xa(xa(xa(p[0][0], p[1][0]), p[2][0]), p[3][0]), 4.0);
    cy = __ddiv_rn(xa(xa(xa(p[0][1], p[1][1]), p[2][1]), p[3][1]), 4.0);
    double dn[4];
    for (int k = 0; k < 4; ++k) {
        const double dx = xs(p[k][0], cx), dy = xs(p[k][1], cy);
        dn[k] = __dsqrt_rn(xa(xm(dx, dx), xm(dy, dy)));
    }
    double d = __ddiv_rn(xa(xa(xa(dn[0], dn[1]), dn[2]), dn[3]), 4.0);
    if (d < 1e-12) d = 1.0;
    s = __ddiv_rn(1.4142135623730951, d);
    const double tx = xm(-s, cx), ty = xm(-s, cy);
    for (int k = 0; k < 4; ++k) {
        q[k][0] = xa(xm(p[k][0], s), tx);
        q[k][1] = xa(xm(p[k][1], s), ty);
    }
}

// Null vector of an 8x9 system by Gaussian elimination with complete
// pivoting; unit norm.  False when the system is rank deficient.
__device__ bool null_vector_8x9(double (*a)[9], double* x) {
    int col[9];
    for (int j = 0; j < 9; ++j) col[j] = j;
    for (int k = 0; k < 8; ++k) {
        int br = k, bc = k;
        double bv = -1.0;
        for (int r = k; r < 8; ++r)
            for (int c = k; c < 9; ++c) {
                const double v = fabs(a[r][col[c]]);
                if (v > bv) {
                    bv = v;
                    br = r;
                    bc = c;
                }
            }
        if (!(bv > 0.0)) return false;
        if (br != k)
            for (int j = 0; j < 9; ++j) {
                const double t = a[k][j];
                a[k][j] = a[br][j];
                a[br][j] = t;
            }
        const int tc = col[k];
        col[k] = col[bc];
        col[bc] = tc;
        const double piv = a[k][col[k]];
        for (int r = k + 1; r < 8; ++r) {
            const double f = a[r][col[k]] / piv;
            if (f == 0.0) continue;
            for (int c = k; c < 9; ++c) a[r][col[c]] -= f * a[k][col[c]];
        }
    }
    double v[9];
    v[col[8]] = 1.0;
    for (int k = 7; k >= 0; --k) {
        double acc = 0.0;
        for (int c = k + 1; c < 9; ++c) acc += a[k][col[c]] * v[col[c]];
        v[col[k]] = -acc / a[k][col[k]];
    }
    double nn = 0.0;
    for (int j = 0; j < 9; ++j) nn += v[j] * v[j];
    const double r = 1.0 / sqrt(nn);
    for (int j = 0; j < 9; ++j) x[j] = v[j] * r;
    return true;
}

// h (normalised coordinates, unit norm) -> inv(td) @ h @ ts / h22; false
// when the reference returns None (det or h22 guards, :554-556).
__device__ __forceinline__ bool denormalize(const double* hn, double ss, double scx, double scy, double sd, double dcx,
                                            double dcy, double* h) {
    if (fabs(det3(hn)) < 1e-12) return false;
    // m = hn @ ts, ts = [[ss, 0, -ss scx], [0, ss, -ss scy], [0, 0, 1]]
    double m[9];
    for (int r = 0; r < 3; ++r) {
        m[3 * r + 0] = hn[3 * r + 0] * ss;
        m[3 * r + 1] = hn[3 * r + 1] * ss;
        m[3 * r + 2] = hn[3 * r + 0] * (-ss * scx) + hn[3 * r + 1] * (-ss * scy) + hn[3 * r + 2];
    }
    // inv(td) = [[1/sd, 0, dcx], [0, 1/sd, dcy], [0, 0, 1]]
    const double is = 1.0 / sd;
    for (int c = 0; c < 3; ++c) {
        h[0 + c] = is * m[0 + c] + dcx * m[6 + c];
        h[3 + c] = is * m[3 + c] + dcy * m[6 + c];
        h[6 + c] = m[6 + c];
    }
    if (!(fabs(h[8]) > 1e-12)) return false;
    const double r22 = h[8];
    for (int j = 0; j < 9; ++j) h[j] = h[j] / r22;
    return true;
}

// hyps layout per (problem, iteration): [valid, h(9), hinv(9)] as 19 doubles
constexpr int HYP_STRIDE = 19;

__global__ void hg_hyp_kernel(const double* __restrict__ src, const double* __restrict__ dst,
                              const int64_t* __restrict__ off, int P, int iters, const int32_t* __restrict__ samples,
                              double* __restrict__ hyps) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (int64_t)P * iters) return;
    const int p = (int)(gid / iters);
    double* out = hyps + gid * HYP_STRIDE;
    const int64_t o = off[p], n = off[p + 1] - o;
    out[0] = 0.0;
    if (n < 4) return;
    const int32_t* smp = samples + gid * 4;
    double sp[4][2], dp[4][2];
    for (int k = 0; k < 4; ++k) {
        const int64_t i = o + smp[k];
        sp[k][0] = src[2 * i];
        sp[k][1] = src[2 * i + 1];
        dp[k][0] = dst[2 * i];
        dp[k][1] = dst[2 * i + 1];
    }
    if (sample_degenerate(sp) || sample_degenerate(dp)) return;
    double sn[4][2], dn[4][2], ss, scx, scy, sd, dcx, dcy;
    hartley4(sp, sn, ss, scx, scy);
    hartley4(dp, dn, sd, dcx, dcy);
    double a[8][9];
    for (int k = 0; k < 4; ++k) {
        const double x = sn[k][0], y = sn[k][1], u = dn[k][0], v = dn[k][1];
        double* r0 = a[2 * k];
        double* r1 = a[2 * k + 1];
        r0[0] = -x; r0[1] = -y; r0[2] = -1.0; r0[3] = 0.0; r0[4] = 0.0; r0[5] = 0.0;
        r0[6] = u * x; r0[7] = u * y; r0[8] = u;
        r1[0] = 0.0; r1[1] = 0.0; r1[2] = 0.0; r1[3] = -x; r1[4] = -y; r1[5] = -1.0;
        r1[6] = v * x; r1[7] = v * y; r1[8] = v;
    }
    double hn[9], h[9], hi[9];
    if (!null_vector_8x9(a, hn)) return;
    if (!denormalize(hn, ss, scx, scy, sd, dcx, dcy, h)) return;
    if (!inv3(h, hi)) return;
    out[0] = 1.0;
    for (int j = 0; j < 9; ++j) {
        out[1 + j] = h[j];
        out[10 + j] = hi[j];
    }
}

// symmetric transfer error (geometry.py:558-572) in numpy's op order
__device__ __forceinline__ void transfer(const double* m, double x, double y, double& ox, double& oy) {
    const double px = xa(xa(xm(x, m[0]), xm(y, m[1])), m[2]);
    const double py = xa(xa(xm(x, m[3]), xm(y, m[4])), m[5]);
    double w = xa(xa(xm(x, m[6]), xm(y, m[7])), m[8]);
    const bool bad = fabs(w) < 1e-12;
    if (bad) w = 1.0;
    ox = bad ? 1e9 : __ddiv_rn(px, w);
    oy = bad ? 1e9 : __ddiv_rn(py, w);
}

__device__ __forceinline__ bool is_inlier(const double* h, const double* hi, const double* s, const double* d,
                                          double thr) {
    double ax, ay, bx, by;
    transfer(h, s[0], s[1], ax, ay);
    transfer(hi, d[0], d[1], bx, by);
    const double e0 = xs(ax, d[0]), e1 = xs(ay, d[1]);
    const double f0 = xs(bx, s[0]), f1 = xs(by, s[1]);
    const double d1 = xa(xm(e0, e0), xm(e1, e1));
    const double d2 = xa(xm(f0, f0), xm(f1, f1));
    return __dsqrt_rn(xm(0.5, xa(d1, d2))) < thr;
}

// Fast path of is_inlier: one reciprocal per transfer instead of two
// divisions and no square root.  x = 0.5 (d1 + d2) is within
// 2e-14 M^2 of the exact value (M = the largest coordinate involved), and
// sqrt_rn(x) < thr is decided by x against thr^2 outside a band of
// 1e-13 M^2 + 1e-14 thr^2; inside the band the exact numpy-order test runs.
__device__ __forceinline__ void transfer_fast(const double* m, double x, double y, double& ox, double& oy) {
    const double px = xa(xa(xm(x, m[0]), xm(y, m[1])), m[2]);
    const double py = xa(xa(xm(x, m[3]), xm(y, m[4])), m[5]);
    const double w = xa(xa(xm(x, m[6]), xm(y, m[7])), m[8]);
    const bool bad = fabs(w) < 1e-12;
    const double r = __drcp_rn(bad ? 1.0 : w);
    ox = bad ? 1e9 : px * r;
    oy = bad ? 1e9 : py * r;
}

__device__ __forceinline__ bool is_inlier_fast(const double* h, const double* hi, const double* s, const double* d,
                                               double thr, double thr2, double cmax) {
    double ax, ay, bx, by;
    transfer_fast(h, s[0], s[1], ax, ay);
    transfer_fast(hi, d[0], d[1], bx, by);
    const double e0 = ax - d[0], e1 = ay - d[1], f0 = bx - s[0], f1 = by - s[1];
    const double x = 0.5 * ((e0 * e0 + e1 * e1) + (f0 * f0 + f1 * f1));
    const double m = fmax(fmax(fmax(fabs(ax), fabs(ay)), fmax(fabs(bx), fabs(by))), cmax);
    const double band = 1e-13 * m * m + 1e-14 * thr2;
    if (x < thr2 - band) return true;
    if (x > thr2 + band) return false;
    return is_inlier(h, hi, s, d, thr);
}

__global__ void hg_count_kernel(const double* __restrict__ src, const double* __restrict__ dst,
                                const int64_t* __restrict__ off, int P, int iters, const double* __restrict__ hyps,
                                const double* __restrict__ cmax_p, double thr, int32_t* __restrict__ counts) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= (int64_t)P * iters) return;
    const int p = (int)(w / iters);
    const double* hy = hyps + w * HYP_STRIDE;
    if (hy[0] == 0.0) {
        if (lane == 0) counts[w] = -1;
        return;
    }
    double h[9], hi[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        h[j] = hy[1 + j];
        hi[j] = hy[10 + j];
    }
    const int64_t o = off[p], n = off[p + 1] - o;
    const double cmax = cmax_p[p], thr2 = thr * thr;
    int c = 0;
    for (int64_t i = lane; i < n; i += 32)
        c += is_inlier_fast(h, hi, src + 2 * (o + i), dst + 2 * (o + i), thr, thr2, cmax) ? 1 : 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) counts[w] = c;
}

// ---------------------------------------------------------------------------
// refit (one CTA per problem)

// cyclic Jacobi eigen-decomposition of a symmetric 9x9 matrix (in place);
// eigenvectors in the columns of v
__device__ void jacobi9(double (*a)[9], double (*v)[9]) {
    for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) v[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int i = 0; i < 9; ++i) {
            diag += a[i][i] * a[i][i];
            for (int j = i + 1; j < 9; ++j) off += a[i][j] * a[i][j];
        }
        if (off <= 1e-300 || off <= 1e-34 * diag) break;
        for (int p = 0; p < 8; ++p)
            for (int q = p + 1; q < 9; ++q) {
                const double apq = a[p][q];
                if (apq == 0.0) continue;
                const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 9; ++k) {
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 9; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 9; ++k) {
                    const double vkp = v[k][p], vkq = v[k][q];
                    v[k][p] = c * vkp - s * vkq;
                    v[k][q] = s * vkp + c * vkq;
                }
            }
    }
}

template <int NT>
__device__ __forceinline__ double hg_sum(double x, double* red) {
    using BR = cub::BlockReduce<double, NT>;
    __shared__ typename BR::TempStorage tmp;
    const double r = BR(tmp).Sum(x);
    if (threadIdx.x == 0) *red = r;
    __syncthreads();
    const double out = *red;
    __syncthreads();
    return out;
}

__global__ void __launch_bounds__(HG_REFIT_THREADS)
hg_refit_kernel(const double* __restrict__ src, const double* __restrict__ dst, const int64_t* __restrict__ off,
                int iters, const double* __restrict__ hyps, const int32_t* __restrict__ best,
                const double* __restrict__ cmax, double thr,
                double* __restrict__ out_model, uint8_t* __restrict__ out_mask, int32_t* __restrict__ out_count) {
    const int p = blockIdx.x;
    const int64_t o = off[p], n = off[p + 1] - o;
    const int b = best[p];
    __shared__ double red;
    __shared__ double hsh[18];
    __shared__ int ok;
    double* model = out_model + 9 * (size_t)p;
    uint8_t* mask = out_mask + o;
    if (b < 0) {
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mask[i] = 0;
        if (threadIdx.x < 9) model[threadIdx.x] = (threadIdx.x % 4 == 0) ? 1.0 : 0.0;
        if (threadIdx.x == 0) out_count[p] = 0;
        return;
    }
    const double* hy = hyps + ((size_t)p * iters + b) * HYP_STRIDE;
    double h[9], hi[9];
    for (int j = 0; j < 9; ++j) {
        h[j] = hy[1 + j];
        hi[j] = hy[10 + j];
    }
    double c0 = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const bool in = is_inlier_fast(h, hi, src + 2 * (o + i), dst + 2 * (o + i), thr, thr * thr, cmax[p]);
        mask[i] = in ? 1 : 0;
        c0 += in ? 1.0 : 0.0;
    }
    __syncthreads();
    const int best_count = (int)hg_sum<HG_REFIT_THREADS>(c0, &red);
    if (threadIdx.x == 0) out_count[p] = best_count;
    if (threadIdx.x < 9) model[threadIdx.x] = h[threadIdx.x];
    if (best_count < 4) return;
    // Hartley normalisation over the inliers (geometry.py:534-543)
    double sx = 0, sy = 0, dx = 0, dy = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (mask[i]) {
            sx += src[2 * (o + i)];
            sy += src[2 * (o + i) + 1];
            dx += dst[2 * (o + i)];
            dy += dst[2 * (o + i) + 1];
        }
    const double m = (double)best_count;
    const double scx = hg_sum<HG_REFIT_THREADS>(sx, &red) / m, scy = hg_sum<HG_REFIT_THREADS>(sy, &red) / m;
    const double dcx = hg_sum<HG_REFIT_THREADS>(dx, &red) / m, dcy = hg_sum<HG_REFIT_THREADS>(dy, &red) / m;
    double ns = 0, nd = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (mask[i]) {
            const double* s = src + 2 * (o + i);
            const double* d = dst + 2 * (o + i);
            ns += sqrt((s[0] - scx) * (s[0] - scx) + (s[1] - scy) * (s[1] - scy));
            nd += sqrt((d[0] - dcx) * (d[0] - dcx) + (d[1] - dcy) * (d[1] - dcy));
        }
    double sdist = hg_sum<HG_REFIT_THREADS>(ns, &red) / m, ddist = hg_sum<HG_REFIT_THREADS>(nd, &red) / m;
    if (sdist < 1e-12) sdist = 1.0;
    if (ddist < 1e-12) ddist = 1.0;
    const double ss = 1.4142135623730951 / sdist, sd = 1.4142135623730951 / ddist;
    // normal matrix A^T A (45 unique entries), one thread-private copy each
    double g[45];
#pragma unroll
    for (int k = 0; k < 45; ++k) g[k] = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (mask[i]) {
            const double x = (src[2 * (o + i)] - scx) * ss, y = (src[2 * (o + i) + 1] - scy) * ss;
            const double u = (dst[2 * (o + i)] - dcx) * sd, v = (dst[2 * (o + i) + 1] - dcy) * sd;
            const double r0[9] = {-x, -y, -1.0, 0.0, 0.0, 0.0, u * x, u * y, u};
            const double r1[9] = {0.0, 0.0, 0.0, -x, -y, -1.0, v * x, v * y, v};
            int k = 0;
#pragma unroll
            for (int a = 0; a < 9; ++a)
#pragma unroll
                for (int c = a; c < 9; ++c) g[k++] += r0[a] * r0[c] + r1[a] * r1[c];
        }
    // the 45 sums: warp shuffles, then one pass over the warps' partials
    __shared__ double gw[HG_REFIT_THREADS / 32][45];
    __shared__ double gs[45];
#pragma unroll
    for (int k = 0; k < 45; ++k) {
        double t = g[k];
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o2);
        if ((threadIdx.x & 31) == 0) gw[threadIdx.x >> 5][k] = t;
    }
    __syncthreads();
    if (threadIdx.x < 45) {
        double t = 0.0;
        for (int w = 0; w < HG_REFIT_THREADS / 32; ++w) t += gw[w][threadIdx.x];
        gs[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double A[9][9], V[9][9];
        int k = 0;
        for (int a = 0; a < 9; ++a)
            for (int c = a; c < 9; ++c) {
                A[a][c] = gs[k];
                A[c][a] = gs[k];
                ++k;
            }
        jacobi9(A, V);
        int i0 = 0;
        for (int j = 1; j < 9; ++j)
            if (A[j][j] < A[i0][i0]) i0 = j;
        double l2 = INFINITY;  // second smallest eigenvalue -> sv[-2]^2
        for (int j = 0; j < 9; ++j)
            if (j != i0 && A[j][j] < l2) l2 = A[j][j];
        bool good = !(best_count > 4 && sqrt(fmax(l2, 0.0)) < 1e-12);
        double hn[9], h2[9], hi2[9];
        if (good) {
            for (int j = 0; j < 9; ++j) hn[j] = V[j][i0];
            good = denormalize(hn, ss, scx, scy, sd, dcx, dcy, h2) && inv3(h2, hi2);
        }
        ok = good ? 1 : 0;
        if (good)
            for (int j = 0; j < 9; ++j) {
                hsh[j] = h2[j];
                hsh[9 + j] = hi2[j];
            }
    }
    __syncthreads();
    if (!ok) return;
    double c2 = 0.0;
    for (int j = 0; j < 9; ++j) {
        h[j] = hsh[j];
        hi[j] = hsh[9 + j];
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        c2 += is_inlier_fast(h, hi, src + 2 * (o + i), dst + 2 * (o + i), thr, thr * thr, cmax[p]) ? 1.0 : 0.0;
    const int count2 = (int)hg_sum<HG_REFIT_THREADS>(c2, &red);
    if (count2 < best_count) return;  // keep the minimal hypothesis (:637)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        mask[i] = is_inlier_fast(h, hi, src + 2 * (o + i), dst + 2 * (o + i), thr, thr * thr, cmax[p]) ? 1 : 0;
    if (threadIdx.x < 9) model[threadIdx.x] = h[threadIdx.x];
    if (threadIdx.x == 0) out_count[p] = count2;
}

// per problem: the largest |coordinate| of its matches (the fast path's
// error scale)
__global__ void hg_cmax_kernel(const double* __restrict__ src, const double* __restrict__ dst,
                               const int64_t* __restrict__ off, double* __restrict__ cmax) {
    const int p = blockIdx.x;
    const int64_t o = off[p], n = off[p + 1] - o;
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < 2 * n; i += blockDim.x)
        m = fmax(m, fmax(fabs(src[2 * o + i]), fabs(dst[2 * o + i])));
    for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
    __shared__ double wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
        m = fmax(m, wm[0]);
        cmax[p] = m;
    }
}

static size_t hg_hyp_bytes(int P, int iters) { return align256(sizeof(double) * HYP_STRIDE * (size_t)P * iters); }
static size_t hg_sample_bytes(int P, int iters) { return align256(sizeof(int32_t) * 4 * (size_t)P * iters); }

}  // namespace ec3r

using namespace ec3r;

static size_t hg_cmax_bytes(int P) { return align256(sizeof(double) * (size_t)P); }

extern "C" size_t ec3r_homography_workspace(int n_problems, int iters) {
    if (n_problems <= 0 || iters <= 0) return 256;
    return hg_hyp_bytes(n_problems, iters) + hg_sample_bytes(n_problems, iters) + hg_cmax_bytes(n_problems) +
           align256(sizeof(int32_t) * (size_t)n_problems);
}

extern "C" int ec3r_homography_ransac_score(const double* src, const double* dst, const int64_t* offsets,
                                            int n_problems, const uint64_t* rng_state, int iters,
                                            double pixel_threshold, int32_t* out_counts, int32_t* out_samples,
                                            void* workspace, size_t workspace_bytes, void* stream) {
    if (n_problems < 0 || iters < 0) return EC3R_EARG;
    if (n_problems == 0 || iters == 0) return EC3R_OK;
    if (!src || !dst || !offsets || !rng_state || !out_counts) return EC3R_EARG;
    if (!workspace || workspace_bytes < ec3r_homography_workspace(n_problems, iters)) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    double* hyps = (double*)workspace;
    int32_t* samples = out_samples ? out_samples : (int32_t*)((char*)workspace + hg_hyp_bytes(n_problems, iters));
    int32_t* redo = (int32_t*)((char*)workspace + hg_hyp_bytes(n_problems, iters) +
                               hg_sample_bytes(n_problems, iters) + hg_cmax_bytes(n_problems));
    hg_draw_par_kernel<<<n_problems, HG_DRAW_NT, 0, st>>>(offsets, iters, rng_state, samples, redo);
    EC3R_CHECK_LAUNCH("hg_draw_par_kernel");
    hg_draw_serial_kernel<<<(n_problems + 63) / 64, 64, 0, st>>>(offsets, n_problems, rng_state, iters, redo,
                                                                 samples);
    EC3R_CHECK_LAUNCH("hg_draw_serial_kernel");
    const int64_t nh = (int64_t)n_problems * iters;
    hg_hyp_kernel<<<(unsigned)((nh + 127) / 128), 128, 0, st>>>(src, dst, offsets, n_problems, iters, samples, hyps);
    EC3R_CHECK_LAUNCH("hg_hyp_kernel");
    double* cmax = (double*)((char*)workspace + hg_hyp_bytes(n_problems, iters) + hg_sample_bytes(n_problems, iters));
    hg_cmax_kernel<<<n_problems, 256, 0, st>>>(src, dst, offsets, cmax);
    EC3R_CHECK_LAUNCH("hg_cmax_kernel");
    hg_count_kernel<<<(unsigned)((nh * 32 + 255) / 256), 256, 0, st>>>(src, dst, offsets, n_problems, iters, hyps,
                                                                       cmax, pixel_threshold, out_counts);
    EC3R_CHECK_LAUNCH("hg_count_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_homography_ransac_refit(const double* src, const double* dst, const int64_t* offsets,
                                            int n_problems, const int32_t* best, int iters, double pixel_threshold,
                                            double* out_model, uint8_t* out_mask, int32_t* out_count,
                                            void* workspace, size_t workspace_bytes, void* stream) {
    if (n_problems < 0 || iters < 0) return EC3R_EARG;
    if (n_problems == 0) return EC3R_OK;
    if (!src || !dst || !offsets || !best || !out_model || !out_mask || !out_count) return EC3R_EARG;
    if (!workspace || workspace_bytes < ec3r_homography_workspace(n_problems, iters)) return EC3R_EWORKSPACE;
    const double* cmax =
        (const double*)((const char*)workspace + hg_hyp_bytes(n_problems, iters) + hg_sample_bytes(n_problems, iters));
    hg_refit_kernel<<<n_problems, HG_REFIT_THREADS, 0, as_stream(stream)>>>(
        src, dst, offsets, iters, (const double*)workspace, best, cmax, pixel_threshold, out_model, out_mask,
        out_count);
    EC3R_CHECK_LAUNCH("hg_refit_kernel");
    return EC3R_OK;
}

// ---------------------------------------------------------------------------
// PnP RANSAC scoring (§8f rank 4, the tracking half: geometry.py:414-474,
// called by tracking.py:208).  The hypotheses (EPnP on each 4-point draw)
// come from the reference's host solver; the draws themselves are the
// device replay above.  One warp scores one hypothesis over all of its
// problem's correspondences with _reprojection_errors' operation order
// (geometry.py:117-126): pc = R p + t, z > Z_MIN, u = fx pc0 / z + cx,
// v = fy pc1 / z + cy, err = hypot(u - pix_u, v - pix_v), inlier = err < thr.
// A point whose error lies within `guard` (relative) of the threshold, or
// whose depth lies within 1e-12 of Z_MIN, flags the hypothesis ambiguous:
// the host re-scores it with the reference expression (BLAS summation order
// of pts @ R.T is not pinned).  The inlier error sum (fixed shuffle tree:
// deterministic) feeds the mean-error tie break, guarded the same way.

constexpr double kZMin = 1e-6;  // geometry.py:23

__global__ void pnp_score_kernel(const double* __restrict__ pts, const double* __restrict__ pix,
                                 const int64_t* __restrict__ off, const double* __restrict__ K4,
                                 const double* __restrict__ hyp, const int32_t* __restrict__ hyp_prob, int H,
                                 double thr, double guard, int32_t* __restrict__ out_count,
                                 double* __restrict__ out_errsum, int32_t* __restrict__ out_amb) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= H) return;
    const int p = hyp_prob[w];
    const double* h = hyp + 12 * w;
    double R[9], t[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) R[k] = h[k];
    t[0] = h[9]; t[1] = h[10]; t[2] = h[11];
    const double fx = K4[4 * p], fy = K4[4 * p + 1], cx = K4[4 * p + 2], cy = K4[4 * p + 3];
    const int64_t n0 = off[p], n1 = off[p + 1];
    int cnt = 0, amb = 0;
    double sum = 0.0;
    for (int64_t i = n0 + lane; i < n1; i += 32) {
        const double X = pts[3 * i], Y = pts[3 * i + 1], Z = pts[3 * i + 2];
        double pc[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            pc[k] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(X, R[3 * k]), __dmul_rn(Y, R[3 * k + 1])),
                                        __dmul_rn(Z, R[3 * k + 2])),
                              t[k]);
        const double z = pc[2];
        if (fabs(z - kZMin) <= 1e-12) amb = 1;
        if (z > kZMin) {
            const double u = __dadd_rn(__ddiv_rn(__dmul_rn(fx, pc[0]), z), cx);
            const double v = __dadd_rn(__ddiv_rn(__dmul_rn(fy, pc[1]), z), cy);
            const double err = hypot(__dsub_rn(u, pix[2 * i]), __dsub_rn(v, pix[2 * i + 1]));
            if (fabs(err - thr) <= guard * thr) amb = 1;
            if (err < thr) {
                ++cnt;
                sum += err;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        amb |= __shfl_xor_sync(0xffffffffu, amb, o);
    }
    if (lane == 0) {
        out_count[w] = cnt;
        out_errsum[w] = sum;
        out_amb[w] = amb;
    }
}

extern "C" size_t ec3r_ransac_draws_workspace(int n_problems) {
    return align256(sizeof(int32_t) * (size_t)(n_problems > 0 ? n_problems : 1));
}

extern "C" int ec3r_ransac_draws(const int64_t* offsets, int n_problems, const uint64_t* rng_state, int iters,
                                 int32_t* out_samples, void* workspace, size_t workspace_bytes, void* stream) {
    if (n_problems < 0 || iters < 0) return EC3R_EARG;
    if (n_problems == 0 || iters == 0) return EC3R_OK;
    if (!offsets || !rng_state || !out_samples) return EC3R_EARG;
    if (!workspace || workspace_bytes < ec3r_ransac_draws_workspace(n_problems)) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    int32_t* redo = (int32_t*)workspace;
    hg_draw_par_kernel<<<n_problems, HG_DRAW_NT, 0, st>>>(offsets, iters, rng_state, out_samples, redo);
    EC3R_CHECK_LAUNCH("hg_draw_par_kernel");
    hg_draw_serial_kernel<<<(n_problems + 63) / 64, 64, 0, st>>>(offsets, n_problems, rng_state, iters, redo,
                                                                 out_samples);
    EC3R_CHECK_LAUNCH("hg_draw_serial_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_pnp_score(const double* pts, const double* pix, const int64_t* offsets, const double* K4,
                              const double* hyp, const int32_t* hyp_problem, int n_hyp, double pixel_threshold,
                              double guard, int32_t* out_count, double* out_errsum, int32_t* out_ambiguous,
                              void* stream) {
    if (n_hyp < 0 || !(pixel_threshold > 0) || guard < 0) return EC3R_EARG;
    if (n_hyp == 0) return EC3R_OK;
    if (!pts || !pix || !offsets || !K4 || !hyp || !hyp_problem || !out_count || !out_errsum || !out_ambiguous)
        return EC3R_EARG;
    const int64_t threads = (int64_t)n_hyp * 32;
    pnp_score_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
        pts, pix, offsets, K4, hyp, hyp_problem, n_hyp, pixel_threshold, guard, out_count, out_errsum,
        out_ambiguous);
    EC3R_CHECK_LAUNCH("pnp_score_kernel");
    return EC3R_OK;
}
