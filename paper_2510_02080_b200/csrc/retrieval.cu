// K6: strided global loop retrieval scoring (update_similarity,
// loops.py:184-243) on sm_100a.
//
// Coarse pass: every stride-th keyframe against every later coarse keyframe
// outside the exclusion zone (one float64 dot per pair, D_e = 64 for the
// synthetic encoder).  Hits s > tau_g pull in the +-(stride-1) refinement
// window on both sides.  All outputs are emitted in the reference's
// emission order (coarse ai asc, bi asc, then da, db asc) through ordered
// block-scan compaction, so the host only applies the stateful
// admitted-once rule (loops.py:212-216,240-242).  Sharding: a rank scores
// the coarse rows ai in [k_begin, k_end); the per-rank lists concatenated in
// rank order equal the single-GPU lists.

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <algorithm>

#include "common.cuh"

namespace ec3r {

__device__ __forceinline__ double dotd(const double* __restrict__ a, const double* __restrict__ b, int D) {
    double s = 0.0;
    for (int k = 0; k < D; ++k) s = fma(a[k], b[k], s);
    return s;
}

// flags: 0 = not scored (bi <= ai or excluded), 1 = scored, 2 = scored + hit
__global__ void rt_coarse_kernel(const double* __restrict__ P, int K, int D, int stride, int excl, double tau_g,
                                 int Kc, int kb, double* __restrict__ dense_s, uint8_t* __restrict__ dense_f) {
    const int ai = kb + blockIdx.y;
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= Kc) return;
    const size_t o = (size_t)blockIdx.y * Kc + bi;
    uint8_t f = 0;
    double s = 0.0;
    const int ia = ai * stride, ib = bi * stride;
    if (bi > ai && abs(ia - ib) >= excl) {
        s = dotd(P + (size_t)ia * D, P + (size_t)ib * D, D);
        f = (s > tau_g) ? 2 : 1;
    }
    dense_s[o] = s;
    dense_f[o] = f;
}

// Refinement windows: hit h, offset r -> (da, db) = (r / (2s-1), r % (2s-1)) - (s-1)
// flags: 0 = skipped, 1 = scored, 2 = scored and sn > tau_l
__global__ void rt_refine_kernel(const double* __restrict__ P, int K, int D, int stride, int excl, double tau_l,
                                 int Kc, int kb, const int32_t* __restrict__ hits, const int64_t* __restrict__ counts,
                                 int64_t cap_h, double* __restrict__ rs, uint8_t* __restrict__ rf,
                                 int32_t* __restrict__ rpair) {
    const int64_t nh = min(counts[3], cap_h);
    const int w = 2 * stride - 1, R = w * w;
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int i = hits[h];
        const int ai = kb + i / Kc, bi = i % Kc;
        const int a0 = ai * stride, b0 = bi * stride;
        for (int r = threadIdx.x; r < R; r += blockDim.x) {
            const int da = r / w - (stride - 1), db = r % w - (stride - 1);
            const int ia = a0 + da, ib = b0 + db;
            const size_t o = (size_t)h * R + r;
            uint8_t f = 0;
            double s = 0.0;
            if (ia >= 0 && ia < K && ib >= 0 && ib < K && abs(ia - ib) >= excl) {
                s = dotd(P + (size_t)ia * D, P + (size_t)ib * D, D);
                f = (s > tau_l) ? 2 : 1;
            }
            rs[o] = s;
            rf[o] = f;
            rpair[2 * o] = ia;
            rpair[2 * o + 1] = ib;
        }
    }
}

// ---------------------------------------------------------------------------
// Multi-CTA ordered compaction of a flag array (0 / 1 / 2): per 4096-element
// chunk the counts of (f >= 1) and (f == 2), one exclusive scan over the
// chunks, then every chunk scatters its elements in order.  The single-CTA
// block-scan loops above it replaced cost ~6 ms at K = 4000.
constexpr int RC_NT = 256, RC_PER = 16, RC_CH = RC_NT * RC_PER;

__device__ __forceinline__ int64_t rc_len(int64_t n_static, const int64_t* n_dev, int64_t cap, int64_t mul) {
    return n_dev ? min(*n_dev, cap) * mul : n_static;
}

__global__ void __launch_bounds__(RC_NT) rt_chunk_count_kernel(const uint8_t* __restrict__ f, int64_t n_static,
                                                               const int64_t* __restrict__ n_dev, int64_t cap,
                                                               int64_t mul, int* __restrict__ c1,
                                                               int* __restrict__ c2) {
    typedef cub::BlockReduce<int, RC_NT> BR;
    __shared__ typename BR::TempStorage t1, t2;
    const int64_t n = rc_len(n_static, n_dev, cap, mul);
    const int64_t i0 = (int64_t)blockIdx.x * RC_CH + (int64_t)threadIdx.x * RC_PER;
    int a = 0, b = 0;
    for (int k = 0; k < RC_PER; ++k) {
        const int64_t i = i0 + k;
        const uint8_t v = i < n ? f[i] : 0;
        a += v >= 1;
        b += v == 2;
    }
    const int ta = BR(t1).Sum(a);
    const int tb = BR(t2).Sum(b);
    if (threadIdx.x == 0) { c1[blockIdx.x] = ta; c2[blockIdx.x] = tb; }
}

// in-place exclusive scan of both chunk-count arrays (one CTA); totals to
// out1 / out2
__global__ void __launch_bounds__(1024) rt_chunk_scan_kernel(int* __restrict__ c1, int* __restrict__ c2, int nchunks,
                                                             int64_t* __restrict__ out1, int64_t* __restrict__ out2) {
    typedef cub::BlockScan<int, 1024> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int carry1, carry2;
    if (threadIdx.x == 0) { carry1 = 0; carry2 = 0; }
    __syncthreads();
    for (int b = 0; b < nchunks; b += 1024) {
        const int i = b + threadIdx.x;
        const int v1 = i < nchunks ? c1[i] : 0, v2 = i < nchunks ? c2[i] : 0;
        int e1, e2, t1, t2;
        BS(tmp).ExclusiveSum(v1, e1, t1);
        __syncthreads();
        BS(tmp).ExclusiveSum(v2, e2, t2);
        if (i < nchunks) { c1[i] = carry1 + e1; c2[i] = carry2 + e2; }
        __syncthreads();
        if (threadIdx.x == 0) { carry1 += t1; carry2 += t2; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { *out1 = carry1; *out2 = carry2; }
}

// scatter: thread-local prefix over its 16 elements + block scan + chunk base
template <typename F>
__device__ __forceinline__ void rc_scatter(const uint8_t* __restrict__ f, int64_t n, const int* __restrict__ b1,
                                           const int* __restrict__ b2, F&& emit) {
    typedef cub::BlockScan<int, RC_NT> BS;
    __shared__ typename BS::TempStorage s1, s2;
    const int64_t i0 = (int64_t)blockIdx.x * RC_CH + (int64_t)threadIdx.x * RC_PER;
    uint8_t v[RC_PER];
    int a = 0, b = 0;
#pragma unroll
    for (int k = 0; k < RC_PER; ++k) {
        v[k] = i0 + k < n ? f[i0 + k] : 0;
        a += v[k] >= 1;
        b += v[k] == 2;
    }
    int ea, eb;
    BS(s1).ExclusiveSum(a, ea);
    BS(s2).ExclusiveSum(b, eb);
    int64_t o1 = (int64_t)b1[blockIdx.x] + ea, o2 = (int64_t)b2[blockIdx.x] + eb;
#pragma unroll
    for (int k = 0; k < RC_PER; ++k) {
        if (v[k] >= 1) emit(i0 + k, o1++, v[k] == 2 ? o2++ : (int64_t)-1);
    }
}

__global__ void __launch_bounds__(RC_NT) rt_coarse_scatter_kernel(const double* __restrict__ dense_s,
                                                                  const uint8_t* __restrict__ dense_f, int64_t n,
                                                                  int Kc, int kb, int stride, const int* __restrict__ b1,
                                                                  const int* __restrict__ b2,
                                                                  int32_t* __restrict__ cp, double* __restrict__ cs,
                                                                  int64_t cap_c, int32_t* __restrict__ hits,
                                                                  int64_t cap_h) {
    rc_scatter(dense_f, n, b1, b2, [&](int64_t i, int64_t o, int64_t oh) {
        if (o < cap_c) {
            cp[2 * o] = (int32_t)((kb + i / Kc) * stride);
            cp[2 * o + 1] = (int32_t)((i % Kc) * stride);
            cs[o] = dense_s[i];
        }
        if (oh >= 0 && oh < cap_h) hits[oh] = (int32_t)i;
    });
}

__global__ void __launch_bounds__(RC_NT) rt_refine_scatter_kernel(const double* __restrict__ rs,
                                                                  const uint8_t* __restrict__ rf,
                                                                  const int32_t* __restrict__ rpair,
                                                                  const int64_t* __restrict__ counts, int64_t cap_h,
                                                                  int64_t R, const int* __restrict__ b1,
                                                                  const int* __restrict__ b2,
                                                                  int32_t* __restrict__ candp,
                                                                  double* __restrict__ cands, int32_t* __restrict__ evp,
                                                                  double* __restrict__ evs, int64_t cap) {
    const int64_t n = min(counts[3], cap_h) * R;
    rc_scatter(rf, n, b1, b2, [&](int64_t i, int64_t o, int64_t oh) {
        if (o < cap) { evp[2 * o] = rpair[2 * i]; evp[2 * o + 1] = rpair[2 * i + 1]; evs[o] = rs[i]; }
        if (oh >= 0 && oh < cap) { candp[2 * oh] = rpair[2 * i]; candp[2 * oh + 1] = rpair[2 * i + 1]; cands[oh] = rs[i]; }
    });
}

}  // namespace ec3r

using namespace ec3r;

static int64_t coarse_rows(int K, int stride) { return (K + stride - 1) / stride; }

extern "C" size_t ec3r_retrieval_workspace(int K, int stride, int64_t cap_refine) {
    if (K <= 0 || stride <= 0) return 256;
    const int64_t Kc = coarse_rows(K, stride);
    const int64_t dense = Kc * Kc;
    const int64_t R = (int64_t)(2 * stride - 1) * (2 * stride - 1);
    const int64_t cap_h = cap_refine / R + 1;
    const int64_t nch = (std::max<int64_t>(dense, cap_h * R) + RC_CH - 1) / RC_CH + 1;
    return align256(8 * dense) + align256(dense) + align256(4 * (size_t)cap_h) + align256(8 * (size_t)(cap_h * R)) +
           align256((size_t)(cap_h * R)) + align256(8 * (size_t)(cap_h * R)) + align256(64) +
           2 * align256(4 * (size_t)nch);
}

extern "C" int ec3r_retrieval(const double* pooled, int K, int D, int stride, int exclusion, double tau_g,
                              double tau_l, int32_t* coarse_pairs, double* coarse_scores, int32_t* cand_pairs,
                              double* cand_scores, int32_t* eval_pairs, double* eval_scores, int64_t cap_refine,
                              int64_t* counts, int k_begin, int k_end, void* workspace, size_t workspace_bytes,
                              void* stream) {
    if (K < 0 || D <= 0 || stride <= 0 || !counts) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * 4, st));
    if (K == 0) return EC3R_OK;
    if (!workspace || workspace_bytes < ec3r_retrieval_workspace(K, stride, cap_refine)) return EC3R_EWORKSPACE;
    const int Kc = (int)coarse_rows(K, stride);
    if (k_end <= 0 || k_end > Kc) k_end = Kc;
    if (k_begin < 0) k_begin = 0;
    const int rows = k_end - k_begin;
    if (rows <= 0) return EC3R_OK;
    const int64_t R = (int64_t)(2 * stride - 1) * (2 * stride - 1);
    const int64_t cap_h = cap_refine / R + 1;
    Carver cv{(char*)workspace, 0};
    double* dense_s = cv.take<double>((size_t)Kc * Kc);
    uint8_t* dense_f = cv.take<uint8_t>((size_t)Kc * Kc);
    int32_t* hits = cv.take<int32_t>(cap_h);
    double* rs = cv.take<double>(cap_h * R);
    uint8_t* rf = cv.take<uint8_t>(cap_h * R);
    int32_t* rpair = cv.take<int32_t>(2 * cap_h * R);
    dim3 g1((Kc + 127) / 128, rows);
    rt_coarse_kernel<<<g1, 128, 0, st>>>(pooled, K, D, stride, exclusion, tau_g, Kc, k_begin, dense_s, dense_f);
    EC3R_CHECK_LAUNCH("rt_coarse_kernel");
    const int64_t cap_c = (int64_t)rows * Kc;
    const int64_t n_c = (int64_t)rows * Kc;
    const int64_t nch_max = (std::max<int64_t>((int64_t)Kc * Kc, cap_h * R) + RC_CH - 1) / RC_CH + 1;
    int* cb1 = cv.take<int>(nch_max);
    int* cb2 = cv.take<int>(nch_max);
    // coarse grid -> coarse pairs (scored) and hits, in row-major order
    const int nch_c = (int)((n_c + RC_CH - 1) / RC_CH);
    rt_chunk_count_kernel<<<nch_c, RC_NT, 0, st>>>(dense_f, n_c, nullptr, 0, 1, cb1, cb2);
    EC3R_CHECK_LAUNCH("rt_chunk_count_kernel");
    rt_chunk_scan_kernel<<<1, 1024, 0, st>>>(cb1, cb2, nch_c, counts + 0, counts + 3);
    EC3R_CHECK_LAUNCH("rt_chunk_scan_kernel");
    rt_coarse_scatter_kernel<<<nch_c, RC_NT, 0, st>>>(dense_s, dense_f, n_c, Kc, k_begin, stride, cb1, cb2,
                                                      coarse_pairs, coarse_scores, cap_c, hits, cap_h);
    EC3R_CHECK_LAUNCH("rt_coarse_scatter_kernel");
    rt_refine_kernel<<<kNumSMs * 4, 128, 0, st>>>(pooled, K, D, stride, exclusion, tau_l, Kc, k_begin, hits, counts,
                                                  cap_h, rs, rf, rpair);
    EC3R_CHECK_LAUNCH("rt_refine_kernel");
    // refinement windows -> evaluated pairs and admitted-candidate pairs
    const int nch_r = (int)((cap_h * R + RC_CH - 1) / RC_CH);
    rt_chunk_count_kernel<<<nch_r, RC_NT, 0, st>>>(rf, 0, counts + 3, cap_h, R, cb1, cb2);
    EC3R_CHECK_LAUNCH("rt_chunk_count_kernel");
    rt_chunk_scan_kernel<<<1, 1024, 0, st>>>(cb1, cb2, nch_r, counts + 2, counts + 1);
    EC3R_CHECK_LAUNCH("rt_chunk_scan_kernel");
    rt_refine_scatter_kernel<<<nch_r, RC_NT, 0, st>>>(rs, rf, rpair, counts, cap_h, R, cb1, cb2, cand_pairs,
                                                      cand_scores, eval_pairs, eval_scores, cap_refine);
    EC3R_CHECK_LAUNCH("rt_refine_scatter_kernel");
    return EC3R_OK;
}
