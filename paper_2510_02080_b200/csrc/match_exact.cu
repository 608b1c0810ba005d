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

// Four warp-cooperative float64 dots of one row x against rows y0..y0+3 of
// Y (16-byte chunks per lane, four independent loads in flight); every lane
// returns all four totals.  Rows past y_end contribute 0 (ignored).
template <typename T>
__device__ __forceinline__ void warp_dot4(const T* x, const T* Y, int64_t y0, int64_t y_end, int D, int lane,
                                          double (&s)[4]) {
    constexpr int N = Vec16<T>::N;
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = 0.0;
    for (int k = lane * N; k < D; k += 32 * N) {
        double a[N];
        Vec16<T>::load(x + k, a);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (y0 + u < y_end) {
                double b[N];
                Vec16<T>::load(Y + (y0 + u) * D + k, b);
#pragma unroll
                for (int i = 0; i < N; ++i) s[u] = fma(a[i], b[i], s[u]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
}

// Exact row scan: for rows listed in `rows` (global A-row ids; or all rows
// when rows == nullptr), best column (first index on ties), d_first and the
// second order statistic of the row's d2 values.  One CTA per row: its 8
// warps split the pair's B rows in 4-row strides (every warp-local running
// summary is warp-uniform), then warp 0 merges the 8 summaries.
constexpr int MX_NT = 256;
constexpr int MX_WARPS = MX_NT / 32;

template <typename T>
__global__ void __launch_bounds__(MX_NT) mx_rows_kernel(const T* __restrict__ A, const T* __restrict__ B, int D,
                                                        const int64_t* __restrict__ a_off,
                                                        const int64_t* __restrict__ b_off,
                                                        const int64_t* __restrict__ b_row, int n_pairs,
                                                        const int32_t* __restrict__ rows,
                                                        const int64_t* __restrict__ n_rows_ptr, int64_t n_rows_all,
                                                        MatchRowState* __restrict__ rs, MatchRowD* __restrict__ rsd) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sd1[MX_WARPS], sd2[MX_WARPS];
    __shared__ int si1[MX_WARPS];
    const int64_t n_rows = rows ? *n_rows_ptr : n_rows_all;
    for (int64_t t = blockIdx.x; t < n_rows; t += gridDim.x) {
        const int64_t r = rows ? (int64_t)rows[t] : t;
        const int p = find_pair(a_off, n_pairs, r);
        const int64_t b0 = b_off[p], b1 = b_off[p + 1];
        // the pair's B rows start at b_row[p] (shared maps) : shift the base
        const T* Bp = B + (b_row[p] - b0) * (int64_t)D;
        double d1 = INFINITY, d2nd = INFINITY;
        int i1 = INT_MAX;
        for (int64_t j = b0 + 4 * warp; j < b1; j += 4 * MX_WARPS) {
            double s[4];
            warp_dot4<T>(A + r * D, Bp, j, b1, D, lane, s);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (j + u >= b1) break;
                const double d = d2_of(s[u]);
                const int jj = (int)(j + u - b0);
                if (better(d, jj, d1, i1)) { d2nd = d1; d1 = d; i1 = jj; }
                else if (d < d2nd) d2nd = d;
            }
        }
        if (lane == 0) { sd1[warp] = d1; sd2[warp] = d2nd; si1[warp] = i1; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double m1 = sd1[0], m2 = sd2[0];
            int mi = si1[0];
            for (int w = 1; w < MX_WARPS; ++w) {  // merge (best, second) summaries
                if (better(sd1[w], si1[w], m1, mi)) { m2 = fmin(m1, sd2[w]); m1 = sd1[w]; mi = si1[w]; }
                else m2 = fmin(m2, sd1[w]);
            }
            MatchRowState h;
            h.best = (b1 > b0) ? mi : -1;
            h.ratio_ok = -1;
            h.mutual = -1;
            h.pad = 0;
            rs[r] = h;
            rsd[r] = MatchRowD{m1, m2};
        }
        __syncthreads();
    }
}

// Exact column scan: argmin over the pair's A rows of d2 (first index); one
// CTA per column.
template <typename T>
__global__ void __launch_bounds__(MX_NT) mx_cols_kernel(const T* __restrict__ A, const T* __restrict__ B, int D,
                                                        const int64_t* __restrict__ a_off,
                                                        const int64_t* __restrict__ b_off,
                                                        const int64_t* __restrict__ b_row, int n_pairs,
                                                        const int32_t* __restrict__ cols,
                                                        const int64_t* __restrict__ n_cols_ptr, int64_t n_cols_all,
                                                        int32_t* __restrict__ col_best) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double sd1[MX_WARPS];
    __shared__ int si1[MX_WARPS];
    const int64_t n_cols = cols ? *n_cols_ptr : n_cols_all;
    for (int64_t t = blockIdx.x; t < n_cols; t += gridDim.x) {
        const int64_t c = cols ? (int64_t)cols[t] : t;
        const int p = find_pair(b_off, n_pairs, c);
        const int64_t a0 = a_off[p], a1 = a_off[p + 1];
        double d1 = INFINITY;
        int i1 = INT_MAX;
        for (int64_t i = a0 + 4 * warp; i < a1; i += 4 * MX_WARPS) {
            double s[4];
            warp_dot4<T>(B + (b_row[p] + (c - b_off[p])) * D, A, i, a1, D, lane, s);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (i + u >= a1) break;
                const double d = d2_of(s[u]);
                const int ii = (int)(i + u - a0);
                if (better(d, ii, d1, i1)) { d1 = d; i1 = ii; }
            }
        }
        if (lane == 0) { sd1[warp] = d1; si1[warp] = i1; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double m1 = sd1[0];
            int mi = si1[0];
            for (int w = 1; w < MX_WARPS; ++w)
                if (better(sd1[w], si1[w], m1, mi)) { m1 = sd1[w]; mi = si1[w]; }
            col_best[c] = (a1 > a0) ? mi : -1;
        }
        __syncthreads();
    }
}

// Final decision per A row (tracking.py:159-169).
__global__ void mx_finalize_kernel(const MatchRowState* __restrict__ rs, const MatchRowD* __restrict__ rsd,
                                   const int32_t* __restrict__ col_best,
                                   const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                                   int64_t total_a, double ratio2, int32_t* __restrict__ match_b,
                                   int32_t* __restrict__ n_match) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // the CTA's first pair once (a proportional guess, exact for equal-sized
    // pairs, else the binary search), then each row steps forward: a CTA's
    // rows span few pairs
    __shared__ int p_cta;
    if (threadIdx.x == 0) {
        const int64_t r0 = (int64_t)blockIdx.x * blockDim.x < total_a ? (int64_t)blockIdx.x * blockDim.x : total_a - 1;
        const int64_t g = total_a > 0 ? r0 * n_pairs / total_a : 0;
        int q = (int)(g < (int64_t)n_pairs - 1 ? g : (int64_t)n_pairs - 1);
        int steps = 0;
        while (q > 0 && a_off[q] > r0 && steps < 4) { --q; ++steps; }
        while (q + 1 < n_pairs && a_off[q + 1] <= r0 && steps < 8) { ++q; ++steps; }
        const bool ok = a_off[q] <= r0 && (q + 1 >= n_pairs || a_off[q + 1] > r0);
        p_cta = ok ? q : find_pair(a_off, n_pairs, r0);
    }
    __syncthreads();
    if (r >= total_a) return;
    int p = p_cta;
    while (p + 1 < n_pairs && a_off[p + 1] <= r) ++p;
    const int64_t a0 = a_off[p], b0 = b_off[p], m = b_off[p + 1] - b0;
    int out = -1;
    const MatchRowState s = rs[r];
    if (m > 0 && s.best >= 0) {
        bool keep;
        if (s.ratio_ok >= 0) keep = s.ratio_ok != 0;  // certified from the tensor-core keys
        else {
            const MatchRowD d = rsd[r];
            keep = !(m > 1 && d.d1 > ratio2 * d.d2);
        }
        if (keep && (s.mutual == 1 || (s.mutual == -1 && col_best[b0 + s.best] == (int)(r - a0)))) out = s.best;
    }
    match_b[r] = out;
    // one atomic per (warp, pair) instead of one per match
    const unsigned same = __match_any_sync(__activemask(), p);
    const unsigned hits = __ballot_sync(__activemask(), out >= 0) & same;
    if (hits && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&n_match[p], __popc(hits));
}

template <typename T>
int launch_exact(const T* A, const T* B, int D, const int64_t* a_off, const int64_t* b_off, const int64_t* b_row,
                 int n_pairs,
                 const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all, const int32_t* cols,
                 const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs, MatchRowD* rsd, int32_t* col_best,
                 cudaStream_t st) {
    if (D % Vec16<T>::N != 0) return EC3R_EARG;  // rows must be 16-byte chunked
    const size_t smem = 0;
    const unsigned grid = kNumSMs * 8;
    if (rows != nullptr || n_rows_all > 0) {
        mx_rows_kernel<T><<<grid, 256, smem, st>>>(A, B, D, a_off, b_off, b_row, n_pairs, rows, n_rows_ptr, n_rows_all,
                                                    rs, rsd);
        EC3R_CHECK_LAUNCH("mx_rows_kernel");
    }
    if (cols != nullptr || n_cols_all > 0) {
        mx_cols_kernel<T><<<grid, 256, smem, st>>>(A, B, D, a_off, b_off, b_row, n_pairs, cols, n_cols_ptr, n_cols_all,
                                                    col_best);
        EC3R_CHECK_LAUNCH("mx_cols_kernel");
    }
    return EC3R_OK;
}

int match_exact_dispatch(const void* A, const void* B, int dtype, int D, const int64_t* a_off, const int64_t* b_off,
                         const int64_t* b_row, int n_pairs, const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all,
                         const int32_t* cols, const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs,
                         MatchRowD* rsd, int32_t* col_best, cudaStream_t st) {
    switch (dtype) {
        case 0:
            return launch_exact<uint16_t>((const uint16_t*)A, (const uint16_t*)B, D, a_off, b_off, b_row, n_pairs, rows,
                                          n_rows_ptr, n_rows_all, cols, n_cols_ptr, n_cols_all, rs, rsd, col_best, st);
        case 1:
            return launch_exact<float>((const float*)A, (const float*)B, D, a_off, b_off, b_row, n_pairs, rows, n_rows_ptr,
                                       n_rows_all, cols, n_cols_ptr, n_cols_all, rs, rsd, col_best, st);
        case 2:
            return launch_exact<double>((const double*)A, (const double*)B, D, a_off, b_off, b_row, n_pairs, rows,
                                        n_rows_ptr, n_rows_all, cols, n_cols_ptr, n_cols_all, rs, rsd, col_best, st);
    }
    return EC3R_EARG;
}

int match_finalize(const MatchRowState* rs, const MatchRowD* rsd, const int32_t* col_best, const int64_t* a_off,
                   const int64_t* b_off,
                   int n_pairs, int64_t total_a, double ratio, int32_t* match_b, int32_t* n_match, cudaStream_t st) {
    EC3R_CUDA_TRY(cudaMemsetAsync(n_match, 0, sizeof(int32_t) * n_pairs, st));
    if (total_a == 0) return EC3R_OK;
    mx_finalize_kernel<<<(unsigned)((total_a + 255) / 256), 256, 0, st>>>(rs, rsd, col_best, a_off, b_off, n_pairs,
                                                                         total_a, ratio * ratio, match_b, n_match);
    EC3R_CHECK_LAUNCH("mx_finalize_kernel");
    return EC3R_OK;
}

}  // namespace ec3r
