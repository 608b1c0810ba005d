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

#include <cub/block/block_scan.cuh>

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

// Ordered compaction of the dense coarse grid (one CTA, row-major order).
constexpr int RT_NT = 1024;
__global__ void __launch_bounds__(RT_NT) rt_coarse_compact_kernel(const double* __restrict__ dense_s,
                                                                  const uint8_t* __restrict__ dense_f, int64_t n,
                                                                  int Kc, int kb, int stride, int32_t* __restrict__ cp,
                                                                  double* __restrict__ cs, int64_t cap_c,
                                                                  int32_t* __restrict__ hits, int64_t cap_h,
                                                                  int64_t* __restrict__ counts) {
    typedef cub::BlockScan<int, RT_NT> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t carry_c, carry_h;
    if (threadIdx.x == 0) { carry_c = 0; carry_h = 0; }
    __syncthreads();
    for (int64_t b = 0; b < n; b += RT_NT) {
        const int64_t i = b + threadIdx.x;
        const uint8_t f = i < n ? dense_f[i] : 0;
        int ex_c, ex_h, ag_c, ag_h;
        BS(tmp).ExclusiveSum(f >= 1 ? 1 : 0, ex_c, ag_c);
        __syncthreads();
        BS(tmp).ExclusiveSum(f == 2 ? 1 : 0, ex_h, ag_h);
        if (f >= 1) {
            const int64_t o = carry_c + ex_c;
            if (o < cap_c) {
                cp[2 * o] = (int32_t)((kb + i / Kc) * stride);
                cp[2 * o + 1] = (int32_t)((i % Kc) * stride);
                cs[o] = dense_s[i];
            }
        }
        if (f == 2) {
            const int64_t o = carry_h + ex_h;
            if (o < cap_h) hits[o] = (int32_t)i;
        }
        __syncthreads();
        if (threadIdx.x == 0) { carry_c += ag_c; carry_h += ag_h; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counts[0] = carry_c;
        counts[3] = carry_h;  // scratch slot: number of coarse hits
    }
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

__global__ void __launch_bounds__(RT_NT) rt_refine_compact_kernel(const double* __restrict__ rs,
                                                                  const uint8_t* __restrict__ rf,
                                                                  const int32_t* __restrict__ rpair, int stride,
                                                                  int64_t cap_h, int32_t* __restrict__ candp,
                                                                  double* __restrict__ cands,
                                                                  int32_t* __restrict__ evp, double* __restrict__ evs,
                                                                  int64_t cap, int64_t* __restrict__ counts) {
    typedef cub::BlockScan<int, RT_NT> BS;
    __shared__ typename BS::TempStorage tmp;
    __shared__ int64_t carry_e, carry_c;
    const int w = 2 * stride - 1;
    const int64_t n = min(counts[3], cap_h) * (int64_t)(w * w);
    if (threadIdx.x == 0) { carry_e = 0; carry_c = 0; }
    __syncthreads();
    for (int64_t b = 0; b < n; b += RT_NT) {
        const int64_t i = b + threadIdx.x;
        const uint8_t f = i < n ? rf[i] : 0;
        int ex_e, ex_c, ag_e, ag_c;
        BS(tmp).ExclusiveSum(f >= 1 ? 1 : 0, ex_e, ag_e);
        __syncthreads();
        BS(tmp).ExclusiveSum(f == 2 ? 1 : 0, ex_c, ag_c);
        if (f >= 1) {
            const int64_t o = carry_e + ex_e;
            if (o < cap) { evp[2 * o] = rpair[2 * i]; evp[2 * o + 1] = rpair[2 * i + 1]; evs[o] = rs[i]; }
        }
        if (f == 2) {
            const int64_t o = carry_c + ex_c;
            if (o < cap) { candp[2 * o] = rpair[2 * i]; candp[2 * o + 1] = rpair[2 * i + 1]; cands[o] = rs[i]; }
        }
        __syncthreads();
        if (threadIdx.x == 0) { carry_e += ag_e; carry_c += ag_c; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counts[1] = carry_c;
        counts[2] = carry_e;
    }
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
    return align256(8 * dense) + align256(dense) + align256(4 * (size_t)cap_h) + align256(8 * (size_t)(cap_h * R)) +
           align256((size_t)(cap_h * R)) + align256(8 * (size_t)(cap_h * R)) + align256(64);
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
    rt_coarse_compact_kernel<<<1, RT_NT, 0, st>>>(dense_s, dense_f, (int64_t)rows * Kc, Kc, k_begin, stride,
                                                  coarse_pairs, coarse_scores, cap_c, hits, cap_h, counts);
    EC3R_CHECK_LAUNCH("rt_coarse_compact_kernel");
    rt_refine_kernel<<<kNumSMs * 4, 128, 0, st>>>(pooled, K, D, stride, exclusion, tau_l, Kc, k_begin, hits, counts,
                                                  cap_h, rs, rf, rpair);
    EC3R_CHECK_LAUNCH("rt_refine_kernel");
    rt_refine_compact_kernel<<<1, RT_NT, 0, st>>>(rs, rf, rpair, stride, cap_h, cand_pairs, cand_scores, eval_pairs,
                                                  eval_scores, cap_refine, counts);
    EC3R_CHECK_LAUNCH("rt_refine_compact_kernel");
    return EC3R_OK;
}
