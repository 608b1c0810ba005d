// Shared declarations of the descriptor matcher (K5).
#pragma once

#include "common.cuh"

namespace ec3r {

// Per A-row outcome of the row side of match_descriptors (tracking.py:155,166).
// The hot part is 8 bytes (read by every certification pass); the float64
// (d1, d2) of a row live in a separate MatchRowD array, written only by the
// exact re-scan and read only when ratio_ok == -1.
struct MatchRowState {
    int32_t best;     // best column within the pair (first index on ties), -1 if none
    int8_t ratio_ok;  // -1: decide from (d1, d2); 0 / 1: ratio test already certified reject / pass
    int8_t mutual;    // -1: decide from col_best; 0 / 1: mutual check certified (tracking.py:160-162)
    int16_t pad;
};
struct MatchRowD {
    double d1;  // d2 value of the best column
    double d2;  // second order statistic of the row's d2 values
};

// 16-byte row chunks widened to float64 (rows are 16-byte aligned: D is
// padded to a multiple of 16 elements by the host layer).
template <typename T>
struct Vec16;
template <>
struct Vec16<uint16_t> {
    static constexpr int N = 8;
    __device__ __forceinline__ static void load(const uint16_t* p, double (&o)[8]) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            o[2 * i] = (double)__uint_as_float(w[i] << 16);
            o[2 * i + 1] = (double)__uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
};
template <>
struct Vec16<float> {
    static constexpr int N = 4;
    __device__ __forceinline__ static void load(const float* p, double (&o)[4]) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    }
};
template <>
struct Vec16<double> {
    static constexpr int N = 2;
    __device__ __forceinline__ static void load(const double* p, double (&o)[2]) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p));
        o[0] = v.x; o[1] = v.y;
    }
};

// Warp-cooperative float64 dot of two D-element rows (every lane returns
// the total).  Products of bf16 values are exact in float64 and the sums of
// <= 2^k such terms stay exact for descriptor-range exponents, so the result
// equals the reference's dgemm entry.
template <typename T>
__device__ __forceinline__ double warp_dot16(const T* a, const T* b, int D, int lane) {
    constexpr int N = Vec16<T>::N;
    double s = 0.0;
    for (int k = lane * N; k < D; k += 32 * N) {
        double x[N], y[N];
        Vec16<T>::load(a + k, x);
        Vec16<T>::load(b + k, y);
#pragma unroll
        for (int i = 0; i < N; ++i) s = fma(x[i], y[i], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

int match_exact_dispatch(const void* A, const void* B, int dtype, int D, const int64_t* a_off, const int64_t* b_off,
                         const int64_t* b_row, int n_pairs, const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all,
                         const int32_t* cols, const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs,
                         MatchRowD* rsd,
                         int32_t* col_best, cudaStream_t st);

int match_finalize(const MatchRowState* rs, const MatchRowD* rsd, const int32_t* col_best, const int64_t* a_off, const int64_t* b_off,
                   int n_pairs, int64_t total_a, double ratio, int32_t* match_b, int32_t* n_match, cudaStream_t st);

}  // namespace ec3r
