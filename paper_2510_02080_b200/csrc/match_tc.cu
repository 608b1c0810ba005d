// K5 (tensor-core side): approximate similarity pass.  Placeholder that
// lists every row and column for the exact float64 re-scan; replaced by the
// tcgen05 kernel.

#include "common.cuh"
#include "match.cuh"

namespace ec3r {

__global__ void mt_flag_all_kernel(int32_t* __restrict__ list, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) list[i] = (int32_t)i;
}

size_t match_tc_workspace(int64_t, int64_t, int) { return 256; }

int match_tc_run(const uint16_t* A, const uint16_t* B, const int64_t* a_off_d, const int64_t* b_off_d,
                 const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs, int D, int exact_dtype,
                 MatchRowState* rs, int32_t* col_best, int32_t* flag_rows, int32_t* flag_cols, int64_t* counters,
                 void* tc_ws, size_t tc_ws_bytes, cudaStream_t st) {
    (void)A; (void)B; (void)a_off_d; (void)b_off_d; (void)D; (void)exact_dtype; (void)rs; (void)col_best;
    (void)tc_ws; (void)tc_ws_bytes;
    const int64_t na = a_off_h[n_pairs], nb = b_off_h[n_pairs];
    mt_flag_all_kernel<<<(unsigned)((na + 255) / 256), 256, 0, st>>>(flag_rows, na);
    EC3R_CHECK_LAUNCH("mt_flag_all_kernel");
    mt_flag_all_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(flag_cols, nb);
    EC3R_CHECK_LAUNCH("mt_flag_all_kernel");
    int64_t c[2] = {na, nb};
    EC3R_CUDA_TRY(cudaMemcpyAsync(counters, c, sizeof(c), cudaMemcpyHostToDevice, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    return EC3R_OK;
}

}  // namespace ec3r
