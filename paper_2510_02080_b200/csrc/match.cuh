// Shared declarations of the descriptor matcher (K5).
#pragma once

#include "common.cuh"

namespace ec3r {

// Per A-row outcome of the row side of match_descriptors (tracking.py:155,166).
struct MatchRowState {
    double d1;   // d2 value of the best column
    double d2;   // second order statistic of the row's d2 values
    int32_t best;  // best column within the pair (first index on ties), -1 if none
    int32_t pad;
};

int match_exact_dispatch(const void* A, const void* B, int dtype, int D, const int64_t* a_off, const int64_t* b_off,
                         int n_pairs, const int32_t* rows, const int64_t* n_rows_ptr, int64_t n_rows_all,
                         const int32_t* cols, const int64_t* n_cols_ptr, int64_t n_cols_all, MatchRowState* rs,
                         int32_t* col_best, cudaStream_t st);

int match_finalize(const MatchRowState* rs, const int32_t* col_best, const int64_t* a_off, const int64_t* b_off,
                   int n_pairs, int64_t total_a, double ratio, int32_t* match_b, int32_t* n_match, cudaStream_t st);

}  // namespace ec3r
