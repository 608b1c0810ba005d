// C-ABI plumbing: version, thread-local error strings, and the matcher entry
// point that sequences the tensor-core pass and the exact re-scoring.

#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "match.cuh"

namespace ec3r {

static thread_local char g_last_error[512] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::atomic<int> g_timing{0};
static std::mutex g_timing_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timed[TK_COUNT];

KernelTimer::KernelTimer(int kernel, cudaStream_t stream) : k(kernel), st(stream) {
    if (!g_timing.load(std::memory_order_relaxed)) return;
    if (cudaEventCreate(&e0) != cudaSuccess) { e0 = nullptr; return; }
    cudaEventRecord(e0, st);
}

void KernelTimer::stop() {
    if (!e0) return;
    cudaEvent_t e1;
    if (cudaEventCreate(&e1) != cudaSuccess) { cudaEventDestroy(e0); e0 = nullptr; return; }
    cudaEventRecord(e1, st);
    std::lock_guard<std::mutex> g(g_timing_mu);
    g_timed[k].emplace_back(e0, e1);
    e0 = nullptr;
}

void set_last_error(const char* where, cudaError_t e) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}
void set_last_error_msg(const char* msg) { snprintf(g_last_error, sizeof(g_last_error), "%s", msg); }

// tensor-core approximate pass + certification (match_tc.cu)
int match_tc_run(const uint16_t* A, const uint16_t* B, const int64_t* a_off_d, const int64_t* b_off_d,
                 const int64_t* b_row_d, int64_t n_b_rows,
                 const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs, int D, int exact_dtype,
                 double norm_bound, double ratio, MatchRowState* rs, int32_t* flag_rows, int32_t* flag_cols,
                 int64_t* counters, void* tc_ws, size_t tc_ws_bytes, int* tc_used, cudaStream_t st);
int match_tc_need_cols(const int64_t* a_off_d, const int64_t* b_off_d, const int64_t* a_off_h,
                       const int64_t* b_off_h, int n_pairs, double ratio, MatchRowState* rs,
                       const MatchRowD* rsd, int32_t* col_best, int32_t* flag_cols, int64_t* counters, void* tc_ws,
                       cudaStream_t st);
size_t match_tc_workspace(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs);

}  // namespace ec3r

using namespace ec3r;

extern "C" int ec3r_abi_version(void) { return EC3R_ABI_VERSION; }
extern "C" uint64_t ec3r_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }
extern "C" const char* ec3r_last_error(void) { return g_last_error; }

extern "C" void ec3r_timing_enable(int on) { g_timing.store(on ? 1 : 0); }

// Sums the recorded launches of one timed kernel (0 match tensor-core pass,
// 1 pool registration, 2 frame fusion) and forgets them.  Synchronizes on the
// recorded events.
extern "C" int ec3r_timing_get(int kernel, double* ms_total, int64_t* n_launches) {
    if (kernel < 0 || kernel >= TK_COUNT || !ms_total || !n_launches) return EC3R_EARG;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    {
        std::lock_guard<std::mutex> g(g_timing_mu);
        ev.swap(g_timed[kernel]);
    }
    double tot = 0.0;
    for (auto& e : ev) {
        float ms = 0.f;
        EC3R_CUDA_TRY(cudaEventSynchronize(e.second));
        EC3R_CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
        tot += ms;
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    *ms_total = tot;
    *n_launches = (int64_t)ev.size();
    return EC3R_OK;
}

// Workspace of ec3r_match_batched:
//   a_off, b_off (n_pairs+1 int64 each), row state (total_a), col best
//   (total_b), flagged rows / cols lists (total_a / total_b int32),
//   counters (8 int64), then the tensor-core pass workspace.
extern "C" size_t ec3r_match_workspace(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs) {
    if (!a_off_h || !b_off_h || n_pairs < 0) return 0;
    const int64_t total_a = a_off_h[n_pairs], total_b = b_off_h[n_pairs];
    return 3 * align256(sizeof(int64_t) * (size_t)(n_pairs + 1)) + align256(sizeof(MatchRowState) * (size_t)total_a) +
           align256(sizeof(MatchRowD) * (size_t)total_a) +
           align256(sizeof(int32_t) * (size_t)total_b) + align256(sizeof(int32_t) * (size_t)total_a) +
           align256(sizeof(int32_t) * (size_t)total_b) + align256(sizeof(int64_t) * 8) +
           match_tc_workspace(a_off_h, b_off_h, n_pairs);
}

extern "C" int ec3r_match_batched(const uint16_t* A, const uint16_t* B, const void* A_x, const void* B_x,
                                  int exact_dtype, const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs, int D,
                                  double ratio, double norm_bound, int32_t* match_b, int32_t* n_match, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    return ec3r_match_batched_rows(A, B, A_x, B_x, exact_dtype, a_off_h, b_off_h, nullptr,
                                   (n_pairs > 0 && b_off_h) ? b_off_h[n_pairs] : 0, n_pairs, D, ratio, norm_bound,
                                   match_b, n_match, workspace, workspace_bytes, stream);
}

extern "C" int ec3r_match_batched_rows(const uint16_t* A, const uint16_t* B, const void* A_x, const void* B_x,
                                       int exact_dtype, const int64_t* a_off_h, const int64_t* b_off_h,
                                       const int64_t* b_row_h, int64_t n_b_rows, int n_pairs, int D, double ratio,
                                       double norm_bound, int32_t* match_b, int32_t* n_match, void* workspace,
                                       size_t workspace_bytes, void* stream) {
    if (n_pairs < 0 || D <= 0 || !a_off_h || !b_off_h || exact_dtype < 0 || exact_dtype > 2 || n_b_rows < 0)
        return EC3R_EARG;
    if (n_pairs == 0) return EC3R_OK;
    const int64_t total_a = a_off_h[n_pairs], total_b = b_off_h[n_pairs];
    if (b_row_h) {  // every pair's rows inside the map matrix B
        for (int p = 0; p < n_pairs; ++p)
            if (b_row_h[p] < 0 || b_row_h[p] + (b_off_h[p + 1] - b_off_h[p]) > n_b_rows) return EC3R_EARG;
    } else if (n_b_rows < total_b) {
        return EC3R_EARG;
    }
    if (!workspace || workspace_bytes < ec3r_match_workspace(a_off_h, b_off_h, n_pairs)) return EC3R_EWORKSPACE;
    if (exact_dtype == 0) { A_x = A; B_x = B; }
    if ((total_a && !A_x) || (total_b && !B_x)) return EC3R_EARG;
    if (!b_row_h) n_b_rows = total_b;
    cudaStream_t st = as_stream(stream);
    Carver cv{(char*)workspace, 0};
    int64_t* a_off = cv.take<int64_t>(n_pairs + 1);
    int64_t* b_off = cv.take<int64_t>(n_pairs + 1);
    int64_t* b_row = cv.take<int64_t>(n_pairs + 1);
    MatchRowState* rs = cv.take<MatchRowState>(total_a);
    MatchRowD* rsd = cv.take<MatchRowD>(total_a);
    int32_t* col_best = cv.take<int32_t>(total_b);
    int32_t* flag_rows = cv.take<int32_t>(total_a);
    int32_t* flag_cols = cv.take<int32_t>(total_b);
    int64_t* counters = cv.take<int64_t>(8);
    void* tc_ws = cv.base + cv.used;
    const size_t tc_bytes = workspace_bytes - cv.used;
    EC3R_CUDA_TRY(cudaMemcpyAsync(a_off, a_off_h, sizeof(int64_t) * (n_pairs + 1), cudaMemcpyHostToDevice, st));
    EC3R_CUDA_TRY(cudaMemcpyAsync(b_off, b_off_h, sizeof(int64_t) * (n_pairs + 1), cudaMemcpyHostToDevice, st));
    EC3R_CUDA_TRY(cudaMemcpyAsync(b_row, b_row_h ? b_row_h : b_off_h, sizeof(int64_t) * n_pairs,
                                  cudaMemcpyHostToDevice, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(int64_t) * 8, st));
    int rc;
    if (A != nullptr && B != nullptr && total_a > 0 && total_b > 0) {
        // tensor-core pass: certifies most rows and lists the rest; the
        // passing rows' mutual checks then list the columns they need
        int tc_used = 0;
        rc = match_tc_run(A, B, a_off, b_off, b_row, n_b_rows, a_off_h, b_off_h, n_pairs, D, exact_dtype, norm_bound,
                          ratio, rs, flag_rows, flag_cols, counters, tc_ws, tc_bytes, &tc_used, st);
        if (rc) return rc;
        if (tc_used) {
            rc = match_exact_dispatch(A_x, B_x, exact_dtype, D, a_off, b_off, b_row, n_pairs, flag_rows, counters + 0, 0,
                                      nullptr, nullptr, 0, rs, rsd, col_best, st);
            if (rc) return rc;
            rc = match_tc_need_cols(a_off, b_off, a_off_h, b_off_h, n_pairs, ratio, rs, rsd, col_best,
                                    flag_cols, counters, tc_ws, st);
            if (rc) return rc;
            rc = match_exact_dispatch(A_x, B_x, exact_dtype, D, a_off, b_off, b_row, n_pairs, nullptr, nullptr, 0,
                                      flag_cols, counters + 1, 0, rs, rsd, col_best, st);
        } else {
            rc = match_exact_dispatch(A_x, B_x, exact_dtype, D, a_off, b_off, b_row, n_pairs, flag_rows, counters + 0, 0,
                                      flag_cols, counters + 1, 0, rs, rsd, col_best, st);
        }
    } else {
        rc = match_exact_dispatch(A_x, B_x, exact_dtype, D, a_off, b_off, b_row, n_pairs, nullptr, nullptr, total_a, nullptr,
                                  nullptr, total_b, rs, rsd, col_best, st);
    }
    if (rc) return rc;
    return match_finalize(rs, rsd, col_best, a_off, b_off, n_pairs, total_a, ratio, match_b, n_match, st);
}

extern "C" int ec3r_match_stats(const void* workspace, int64_t total_a, int64_t total_b, int n_pairs,
                                int64_t* rows_h, int64_t* cols_h, void* stream) {
    if (!workspace || !rows_h || !cols_h || n_pairs < 1) return EC3R_EARG;
    Carver cv{(char*)workspace, 0};  // the layout of ec3r_match_batched_rows
    cv.take<int64_t>(n_pairs + 1);
    cv.take<int64_t>(n_pairs + 1);
    cv.take<int64_t>(n_pairs + 1);
    cv.take<MatchRowState>(total_a);
    cv.take<MatchRowD>(total_a);
    cv.take<int32_t>(total_b);
    cv.take<int32_t>(total_a);
    cv.take<int32_t>(total_b);
    int64_t* counters = cv.take<int64_t>(8);
    int64_t c[2];
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemcpyAsync(c, counters, sizeof(c), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    *rows_h = c[0];
    *cols_h = c[1];
    return EC3R_OK;
}
