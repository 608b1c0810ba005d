// K5 (exact side): float64 re-scoring kernels of the descriptor matcher and
// the final mutual-NN + Lowe-ratio decision (match_descriptors,
// tracking.py:143-170).
//
// The tensor-core pass (match_tc.cu) produces approximate float32
// similarities; every decision the reference makes (row argmin, column
// argmin, the second-smallest row value) is either certified from the
// approximate values plus an error bound, or recomputed here in float64
// from the exact rows:
//   d2 = max(2 - 2 * sim, 0)          tracking.py:153 (clamp included)
//   argmin with first-index ties      tracking.py:155-156 (np.argmin)
//   second = 2nd order statistic      tracking.py:166 (np.partition(row,1)[1])
//   reject if d_first > ratio^2 * second, skipped when M == 1   :165-168
// so the emitted matches are bit-identical to the float64 reference.

#include <cuda_bf16.h>

#include "common.cuh"
#include "match.cuh"

namespace ec3r {

template <typename T>
__device__ __forceinline__ double ldx(const T* p, int64_t i);
template <>
__device__ __forceinline__ double ldx<uint16_t>(const uint16_t* p, int64_t i) {
    return (double)__uint_as_float(((uint32_t)p[i]) << 16);
}
template <>
__device__ __forceinline__ double ldx<float>(const float* p, int64_t i) { return (double)p[i]; }
template <>
__device__ __forceinline__ double ldx<double>(const double* p, int64_t i) { return p[i]; }

__device__ __forceinline__ int find_pair(const int64_t* __restrict__ off, int n_pairs, int64_t r) {
    int lo = 0, hi = n_pairs;  // off[lo] <= r < off[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ double d2_of(double sim) {
    return fmax(__dsub_rn(2.0, __dmul_rn(2.0, sim)), 0.0);
}

// (d, idx) lexicographic "better": smaller d, then smaller index
__device__ __forceinline__ bool better(double d, int i, double db, int ib) { return d < db || (d == db && i < ib); }

// Exact row scan: for rows listed in `rows` (global A-row ids; or all rows
// when rows == nullptr), best column (first index on ties), d_first and the
// second order statistic of the row's d2 values.  One warp per row.
template <typename T>
__global__ void __launch_bounds__(256) mx_rows_kernel(const T* __restrict__ A, const T* __restrict__ B, int D,
                                                      const int64_t* __restrict__ a_off,
                                                      const int64_t* __restrict__ b_off, int n_pairs,
                                                      const int32_t* __restrict__ rows, const int64_t* __restrict__ n_rows_ptr,
                                                      int64_t n_rows_all, MatchRowState* __restrict__ rs) {
    extern __shared__ double arow_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* arow = arow_all + (size_t)warp * D;
    const int64_t n_rows = rows ? *n_rows_ptr : n_rows_all;
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < n_rows;
         t += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int64_t r = rows ? (int64_t)rows[t] : t;
        const int p = find_pair(a_off, n_pairs, r);
        const int64_t b0 = b_off[p], b1 = b_off[p + 1];
        __syncwarp();
        for (int k = lane; k < D; k += 32) arow[k] = ldx<T>(A, r * D + k);
        __syncwarp();
        double d1 = INFINITY, d2nd = INFINITY;
        int i1 = INT_MAX;
        for (int64_t j = b0 + lane; j < b1; j += 32) {
            double s = 0.0;
            const T* brow = B + j * D;
            for (int k = 0; k < D; ++k) s = fma(arow[k], ldx<T>(brow, k), s);
            const double d = d2_of(s);
            const int jj = (int)(j - b0);
            if (better(d, jj, d1, i1)) { d2nd = d1; d1 = d; i1 = jj; }
            else if (d < d2nd) d2nd = d;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od1 = __shfl_xor_sync(0xffffffffu, d1, o);
            const double od2 = __shfl_xor_sync(0xffffffffu, d2nd, o);
            const int oi1 = __shfl_xor_sync(0xffffffffu, i1, o);
            // merge two (best, second) summaries
            double nd1, nd2;
            int ni1;
            if (better(od1, oi1, d1, i1)) { nd1 = od1; ni1 = oi1; nd2 = fmin(d1, od2); }
            else { nd1 = d1; ni1 = i1; nd2 = fmin(od1, d2nd); }
            d1 = nd1; i1 = ni1; d2nd = nd2;
        }
        if (lane == 0) {
            rs[r].best = (b1 > b0) ? i1 : -1;
            rs[r].d1 = d1;
            rs[r].d2 = d2nd;
        }
    }
}

// Exact column scan: argmin over the pair's A rows of d2 (first index).
template <typename T>
__global__ void __launch_bounds__(256) mx_cols_kernel(const T* __restrict__ A, const T* __restrict__ B, int D,
                                                      const int64_t* __restrict__ a_off,
                                                      const int64_t* __restrict__ b_off, int n_pairs,
                                                      const int32_t* __restrict__ cols, const int64_t* __restrict__ n_cols_ptr,
                                                      int64_t n_cols_all, int32_t* __restrict__ col_best) {
    extern __shared__ double brow_all[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* brow = brow_all + (size_t)warp * D;
    const int64_t n_cols = cols ? *n_cols_ptr : n_cols_all;
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; t < n_cols;
         t += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int64_t c = cols ? (int64_t)cols[t] : t;
        const int p = find_pair(b_off, n_pairs, c);
        const int64_t a0 = a_off[p], a1 = a_off[p + 1];
        __syncwarp();
        for (int k = lane; k < D; k += 32) brow[k] = ldx<T>(B, c * D + k);
        __syncwarp();
        double d1 = INFINITY;
        int i1 = INT_MAX;
        for (int64_t i = a0 + lane; i < a1; i += 32) {
            double s = 0.0;
            const T* arow = A + i * D;
            for (int k = 0; k < D; ++k) s = fma(ldx<T>(arow, k), brow[k], s);
            const double d = d2_of(s);
            const int ii = (int)(i - a0);
            if (better(d, ii, d1, i1)) { d1 = d; i1 = ii; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, d1, o);
            const int oi = __shfl_xor_sync(0xffffffffu, i1, o);
            if (better(od, oi, d1, i1)) { d1 = od; i1 = oi; }
        }
        if (lane == 0) col_best[c] = (a1 > a0) ? i1 : -1;
    }
}

// Final decision per A row (tracking.py:159-169).
__global__ void mx_finalize_kernel(const MatchRowState* __restrict__ rs, const int32_t* __restrict__ col_best,
                                   const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                                   int64_t total_a, double ratio2, int32_t* __restrict__ match_b,
                                   int32_t* __restrict__ n_match) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= total_a) return;
    const int p = find_pair(a_off, n_pairs, r);
    const int64_t a0 = a_off[p], b0 = b_off[p], m = b_off[p + 1] - b0;
    int out = -1;
    const MatchRowState s = rs[r];
    if (m > 0 && s.best >= 0 && col_best[b0 + s.best] == (int)(r - a0)) {
        bool ok = true;
        if (m > 1 && s.d1 > ratio2 * s.d2) ok = false;
        if (ok) out = s.best;
    }
    match_b[r] = out;
    if (out >= 0) atomicAdd(&n_match[p], 1);
}

template <typename T>
int launch_exact(const T* A, const T* B, int D, const int64_t* a_off, const int64_t* b_off, int n_pairs,
                 const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all, const int32_t* cols,
                 const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs, int32_t* col_best,
                 cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)D * 8;
    if (smem > 48 * 1024) {
        EC3R_CUDA_TRY(cudaFuncSetAttribute(mx_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        EC3R_CUDA_TRY(cudaFuncSetAttribute(mx_cols_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    const unsigned grid = kNumSMs * 8;
    if (rows != nullptr || n_rows_all > 0) {
        mx_rows_kernel<T><<<grid, 256, smem, st>>>(A, B, D, a_off, b_off, n_pairs, rows, n_rows_ptr, n_rows_all, rs);
        EC3R_CHECK_LAUNCH("mx_rows_kernel");
    }
    if (cols != nullptr || n_cols_all > 0) {
        mx_cols_kernel<T><<<grid, 256, smem, st>>>(A, B, D, a_off, b_off, n_pairs, cols, n_cols_ptr, n_cols_all,
                                                    col_best);
        EC3R_CHECK_LAUNCH("mx_cols_kernel");
    }
    return EC3R_OK;
}

int match_exact_dispatch(const void* A, const void* B, int dtype, int D, const int64_t* a_off, const int64_t* b_off,
                         int n_pairs, const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all,
                         const int32_t* cols, const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs,
                         int32_t* col_best, cudaStream_t st) {
    switch (dtype) {
        case 0:
            return launch_exact<uint16_t>((const uint16_t*)A, (const uint16_t*)B, D, a_off, b_off, n_pairs, rows,
                                          n_rows_ptr, n_rows_all, cols, n_cols_ptr, n_cols_all, rs, col_best, st);
        case 1:
            return launch_exact<float>((const float*)A, (const float*)B, D, a_off, b_off, n_pairs, rows, n_rows_ptr,
                                       n_rows_all, cols, n_cols_ptr, n_cols_all, rs, col_best, st);
        case 2:
            return launch_exact<double>((const double*)A, (const double*)B, D, a_off, b_off, n_pairs, rows,
                                        n_rows_ptr, n_rows_all, cols, n_cols_ptr, n_cols_all, rs, col_best, st);
    }
    return EC3R_EARG;
}

int match_finalize(const MatchRowState* rs, const int32_t* col_best, const int64_t* a_off, const int64_t* b_off,
                   int n_pairs, int64_t total_a, double ratio, int32_t* match_b, int32_t* n_match, cudaStream_t st) {
    EC3R_CUDA_TRY(cudaMemsetAsync(n_match, 0, sizeof(int32_t) * n_pairs, st));
    if (total_a == 0) return EC3R_OK;
    mx_finalize_kernel<<<(unsigned)((total_a + 255) / 256), 256, 0, st>>>(rs, col_best, a_off, b_off, n_pairs,
                                                                         total_a, ratio * ratio, match_b, n_match);
    EC3R_CHECK_LAUNCH("mx_finalize_kernel");
    return EC3R_OK;
}

}  // namespace ec3r
