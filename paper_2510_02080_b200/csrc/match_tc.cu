// K5 (tensor-core side): descriptor similarity on tcgen05 with a fused
// top-2 epilogue, sm_100a.
//
// Replaces the dgemm + argmin/partition of match_descriptors
// (tracking.py:152-166).  One persistent CTA per SM walks work units
// (pair, 256-row super-block, column range; the range is the whole pair
// unless the batch has too few row blocks to fill the GPU):
//   warp 0    TMA producer: the unit's two 128-row A blocks (K-major,
//             SWIZZLE_128B, resident for the unit) and a 4-stage ring of
//             128-column B k-blocks;
//   warp 1    TMEM allocator + single-thread tcgen05.mma issuer
//             (kind::f16, bf16 x bf16 -> fp32, M=128 N=128 K=16) into a
//             double-buffered 2 x 256-column TMEM accumulator;
//   warps 2-9 epilogue.  Each similarity becomes one 32-bit KEY: its fp32
//             bits with the 11 low mantissa bits replaced by a code — the
//             column within the 32-column chunk (row side) and the
//             (A block, lane) of its row (column side) — so a plain float
//             max/min returns the argmax with the value, and the epilogue is
//             ~6 ALU ops per similarity: 1 LOP3 key, per-row top-2 over
//             pairs (FMNMX / FMNMX3), per-column top-2 of the warp's 64 rows
//             with two CREDUX.MAX.F32 per column; the 4 lane quarters merge
//             in shared memory and each column's top-2 keys go to the
//             unit's own 8-byte slot with a plain store (no atomics).
// The N x M similarity matrix never exists in memory.  The key values are
// within eps_tc + 2^-12 |key| of the exact similarity, and certification
// (mt_decide_rows / mt_need_cols) proves every decision from them or lists
// it for the float64 re-scan of match_exact.cu, so the matches are
// bit-identical to the float64 reference.  A row is only re-scanned when its
// ratio test (tracking.py:167) is undecided, or it passes with an undecided
// argmax; a column only when a passing row needs its argmax and the keys do
// not settle it.

#include <atomic>
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "match.cuh"

namespace ec3r {

constexpr int TC_BM = 128;       // rows per A block (UMMA M)
constexpr int TC_NA = 2;         // A blocks resident per unit
constexpr int TC_BN = 128;       // columns per B tile (UMMA N)
constexpr int TC_BK = 64;        // bf16 per 128-byte swizzle row
constexpr int TC_STAGES = 4;     // B ring depth
#ifndef EC3R_MT_EPI16
#define EC3R_MT_EPI16 0  // 1: 16 epilogue warps on 16-column chunks (measured slower: 1.043 vs 0.937 ms,
                         // 96 registers by the per-SMSP register file, spills); 0: 8 warps on 32-column chunks
#endif
#if EC3R_MT_EPI16
constexpr int TC_EPI_WARPS = 16;  // 4 per TMEM lane quarter: one per 32-column quarter of the tile
constexpr int TC_CW = 16;         // columns per chunk (one tcgen05.ld.32x32b.x16 per A block)
#else
constexpr int TC_EPI_WARPS = 8;  // 2 per TMEM lane quarter: one per column half
constexpr int TC_CW = 32;
#endif
constexpr int TC_HP = TC_EPI_WARPS / 4;  // column parts per tile (warps per lane quarter)
constexpr int TC_EPI_THREADS = TC_EPI_WARPS * 32;
constexpr int TC_THREADS = 64 + TC_EPI_THREADS;  // producer + MMA + epilogue warps
constexpr int TC_BOX_BYTES = TC_BM * TC_BK * 2;  // 16 KB (A box and B box alike)
constexpr int TC_TMEM_COLS = 512;

// Similarity keys: fp32 bits, low 11 mantissa bits = code.
constexpr uint32_t KEY_MASK = 0xFFFFF800u;
constexpr float KEY_NEG = -3.0e38f;  // invalid row / column: below every real key, finite after coding

// Per A-row approximate top-2 keys and the best column (within the pair).
struct __align__(16) RowCand {
    float k1;
    float k2;
    int32_t c1;
    int32_t pad;
};

// One work unit: up to 256 rows of one pair against all its columns.  Its
// per-column top-2 keys go to col_slots[slot + column] (plain stores: each
// (unit, column) has its own slot; certification merges a pair's units).
struct __align__(16) TcUnit {
    int pair;
    int row0;        // first row of the unit within the packed A
    int col0;        // column range [col0, col1) within the pair (multiples of TC_BN)
    int col1;
    long long slot;  // column slot of the unit's first column
    int split;       // which column range (row candidates: cand[row * n_split + split])
    int pad;
};

struct TcParams {
    const int64_t* a_off;
    const int64_t* b_off;   // virtual column prefix (per-pair column state)
    const int64_t* b_row;   // first B row of each pair (pairs may share a map's rows)
    const TcUnit* units;
    int n_units;
    int kblocks;        // D / 64
    RowCand* cand;
    int n_split;
    unsigned long long* col_slots;  // per unit and column: (ordered best key << 32) | ordered second key
    // n_split == 1: the stage-1 row decision is made here (no decide kernel)
    MatchRowState* rs;
    int32_t* pending;
    int64_t* counters;
    const double* eps_d;  // tensor-core error bound eps_tc (device: no host round trip for the norm bound)
    double ratio2;
};

// ---------------------------------------------------------------------------
// PTX wrappers

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Same wait for the single-thread producer / MMA roles with a suspend-time
// hint, so their waits sleep instead of competing for issue slots with the
// epilogue warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// tcgen05.ld without the wait (the caller issues tcgen05.wait::ld before
// touching the registers, then pins them with reg_fence)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void reg_fence(uint32_t (&r)[16]) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]));
}
template <int N>
__device__ __forceinline__ void tmem_ld_async(uint32_t taddr, uint32_t (&r)[N]) {
    if constexpr (N == 16) tmem_ld16_async(taddr, r);
    else tmem_ld32_async(taddr, r);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void reg_fence(uint32_t (&r)[32]) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

__device__ __forceinline__ void sts_f2(uint32_t addr, float a, float b) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
    return v;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// not volatile: a pure function of the warp's values, so the compiler may
// overlap the column reductions of a chunk (volatile asm would serialise
// every CREDUX behind the previous column's dependent second reduction)
__device__ __forceinline__ float warp_max_f32(float x) {
    float r;
    asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
    return r;
}

// key = value bits above bit 11, code below: bimm = KEY_MASK | column code
// (an immediate), creg = KEY_MASK | row code; the two codes occupy disjoint
// bits, so (a & b & c) | (b ^ c) is the whole key in one LOP3.
// (inline PTX: left to itself the compiler splits it into two LOP3s)
template <uint32_t BIMM>
__device__ __forceinline__ float make_key(uint32_t v, uint32_t creg) {
    uint32_t k;
    asm("lop3.b32 %0, %1, %2, %3, 0xE6;" : "=r"(k) : "r"(v), "n"(BIMM), "r"(creg));
    return __uint_as_float(k);
}

// order-preserving float <-> uint32 (0 is below every finite key)
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t u = __float_as_uint(f);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o ^ 0x80000000u) : ~o);
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B
// apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO
    d |= (uint64_t)1 << 46;              // version
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, K-major, M=128, N=128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                            ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifndef EC3R_MT_COLFIRST
#define EC3R_MT_COLFIRST 0  // chunk epilogue: column side before the row side
#endif
#ifndef EC3R_MT_SPLITBAR
#define EC3R_MT_SPLITBAR 1  // per-tile colbuf handoff: only the merging warps wait
#endif

// d2 = max(2 - 2 s, 0) (tracking.py:153) on interval end points
__device__ __forceinline__ double d2c(double s) { return fmax(2.0 - 2.0 * s, 0.0); }

// Bound on |key - exact similarity|: the tensor-core error eps_tc plus the
// 2^11 ulps the code replaced (<= 2^-12 |key|).
__device__ __forceinline__ double key_eps(double k, double eps_tc) { return eps_tc + ldexp(fabs(k), -12) + 1e-30; }

// Relative slack on the ratio comparisons: covers the float64 rounding of
// d2 and ratio^2 * d2 in the reference (tracking.py:153,167).
constexpr double kRatioSlack = 1e-9;

// Stage-1 decision of one row from its merged candidate (see mt_decide_rows).
// Returns false when the row needs the float64 re-scan.
__device__ __forceinline__ bool row_decision(const RowCand& c, int64_t M, double eps_tc, double ratio2,
                                             MatchRowState& s) {
    s.best = -1; s.ratio_ok = 0; s.mutual = 0; s.pad = 0;
    if (M == 0) return true;  // no columns: no match
    if (M == 1) {             // one column: argmax certain, ratio test skipped (tracking.py:165)
        s.best = 0;
        s.ratio_ok = 1;
        return true;
    }
    const double a1 = c.k1, a2 = c.k2;
    const double e1 = key_eps(a1, eps_tc), e2 = key_eps(a2, eps_tc);
    if (d2c(a1 + e1) > ratio2 * d2c(a2 - e2) * (1.0 + kRatioSlack)) return true;  // certain reject
    if (a1 - e1 > a2 + e2 && a2 + e2 < 1.0 && d2c(a1 - e1) < ratio2 * d2c(a2 + e2) * (1.0 - kRatioSlack)) {
        s.best = c.c1;
        s.ratio_ok = 1;
        return true;
    }
    return false;
}

// Epilogue of one 32-column chunk of the thread's two rows (r0: A block 0,
// r1: A block 1).  Row side: the chunk's top-2 keys per row folded into the
// running (best, second, chunk base of best).  Column side: per column the
// top-2 keys over the warp's 64 rows, written to cb[j] by lane 0.
struct RowTop2 {
    float b, s;
    int cb;  // column base of the chunk holding b (b's code has the column within the chunk)
};

template <int J, int N>
__device__ __forceinline__ void make_keys(const uint32_t (&r0)[N], const uint32_t (&r1)[N], uint32_t creg0,
                                          uint32_t creg1, float (&k0)[N], float (&k1)[N]) {
    if constexpr (J < N) {
        k0[J] = make_key<KEY_MASK | ((uint32_t)J << 6)>(r0[J], creg0);
        k1[J] = make_key<KEY_MASK | ((uint32_t)J << 6)>(r1[J], creg1);
        make_keys<J + 1, N>(r0, r1, creg0, creg1, k0, k1);
    }
}

template <int N>
__device__ __forceinline__ void chunk_epilogue(uint32_t (&r0)[N], uint32_t (&r1)[N], int nv0, int nv1, int cbase,
                                               uint32_t creg0, uint32_t creg1, RowTop2& R0, RowTop2& R1,
                                               uint32_t cb, int lane) {
    // interior chunks (every row and column valid) skip the predicates
    if (!__all_sync(0xffffffffu, nv0 == N && nv1 == N)) {
        const uint32_t neg = __float_as_uint(KEY_NEG);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (j >= nv0) r0[j] = neg;
            if (j >= nv1) r1[j] = neg;
        }
    }
    float k0[N], k1[N];
    make_keys<0, N>(r0, r1, creg0, creg1, k0, k1);
#if EC3R_MT_COLFIRST
    // column side: fold the thread's two rows, then top-1 / top-2 over the
    // warp (keys are unique within a column: the code holds block and lane)
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const float hi = fmaxf(k0[j], k1[j]), lo = fminf(k0[j], k1[j]);
        const float m = warp_max_f32(hi);
        const float m2 = warp_max_f32(hi == m ? lo : hi);
        if (lane == 0) sts_f2(cb + 8u * j, m, m2);
    }
    // row side: top-2 over pairs (hi, lo) — 5 ops per 2 keys per row
    {
        float m0 = fmaxf(k0[0], k0[1]), s0 = fminf(k0[0], k0[1]);
        float m1 = fmaxf(k1[0], k1[1]), s1 = fminf(k1[0], k1[1]);
#pragma unroll
        for (int j = 2; j < N; j += 2) {
            const float h0 = fmaxf(k0[j], k0[j + 1]), l0 = fminf(k0[j], k0[j + 1]);
            const float t0 = fminf(m0, h0);
            m0 = fmaxf(m0, h0);
            s0 = fmax3f(s0, l0, t0);
            const float h1 = fmaxf(k1[j], k1[j + 1]), l1 = fminf(k1[j], k1[j + 1]);
            const float t1 = fminf(m1, h1);
            m1 = fmaxf(m1, h1);
            s1 = fmax3f(s1, l1, t1);
        }
        const float t0 = fminf(R0.b, m0);
        R0.cb = m0 > R0.b ? cbase : R0.cb;
        R0.b = fmaxf(R0.b, m0);
        R0.s = fmax3f(R0.s, s0, t0);
        const float t1 = fminf(R1.b, m1);
        R1.cb = m1 > R1.b ? cbase : R1.cb;
        R1.b = fmaxf(R1.b, m1);
        R1.s = fmax3f(R1.s, s1, t1);
    }
#else
    // row side: top-2 over pairs (hi, lo) — 5 ops per 2 keys per row
    {
        float m0 = fmaxf(k0[0], k0[1]), s0 = fminf(k0[0], k0[1]);
        float m1 = fmaxf(k1[0], k1[1]), s1 = fminf(k1[0], k1[1]);
#pragma unroll
        for (int j = 2; j < N; j += 2) {
            const float h0 = fmaxf(k0[j], k0[j + 1]), l0 = fminf(k0[j], k0[j + 1]);
            const float t0 = fminf(m0, h0);
            m0 = fmaxf(m0, h0);
            s0 = fmax3f(s0, l0, t0);
            const float h1 = fmaxf(k1[j], k1[j + 1]), l1 = fminf(k1[j], k1[j + 1]);
            const float t1 = fminf(m1, h1);
            m1 = fmaxf(m1, h1);
            s1 = fmax3f(s1, l1, t1);
        }
        const float t0 = fminf(R0.b, m0);
        R0.cb = m0 > R0.b ? cbase : R0.cb;
        R0.b = fmaxf(R0.b, m0);
        R0.s = fmax3f(R0.s, s0, t0);
        const float t1 = fminf(R1.b, m1);
        R1.cb = m1 > R1.b ? cbase : R1.cb;
        R1.b = fmaxf(R1.b, m1);
        R1.s = fmax3f(R1.s, s1, t1);
    }
    // column side: fold the thread's two rows, then top-1 / top-2 over the
    // warp (keys are unique within a column: the code holds block and lane)
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const float hi = fmaxf(k0[j], k1[j]), lo = fminf(k0[j], k1[j]);
        const float m = warp_max_f32(hi);
        const float m2 = warp_max_f32(hi == m ? lo : hi);
        if (lane == 0) sts_f2(cb + 8u * j, m, m2);
    }
#endif

}

__global__ void __launch_bounds__(TC_THREADS, 1)
mt_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the dynamic buffer (SWIZZLE_128B atoms)
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int KB = p.kblocks;
    unsigned char* sA = smem;                                   // TC_NA * KB boxes
    unsigned char* sB = sA + (size_t)TC_NA * KB * TC_BOX_BYTES;  // TC_STAGES boxes
    float2* colbuf = (float2*)(sB + (size_t)TC_STAGES * TC_BOX_BYTES);  // [2 tiles][4 quarters][TC_BN]
    float4* rsc = (float4*)(colbuf + 2 * 4 * TC_BN);  // [2 units][TC_HP - 1][TC_NA * TC_BM] part-row summaries
    uint64_t* bars = (uint64_t*)(rsc + 2 * (TC_HP - 1) * TC_NA * TC_BM);
    uint64_t* a_full = bars + 0;   // per k-block slice of the resident A (both blocks)
    uint64_t* a_empty = bars + 4;
    uint64_t* b_full = bars + 8;
    uint64_t* b_empty = b_full + TC_STAGES;
    uint64_t* t_full = b_empty + TC_STAGES;
    uint64_t* t_empty = t_full + 2;
    uint32_t* tmem_slot = (uint32_t*)(t_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) { mbar_init(a_full + s, 1); mbar_init(a_empty + s, 1); }
        for (int s = 0; s < TC_STAGES; ++s) { mbar_init(b_full + s, 1); mbar_init(b_empty + s, 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(t_full + s, 1); mbar_init(t_empty + s, TC_EPI_THREADS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TC_TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                const TcUnit un = p.units[u];
                const int64_t b0 = p.b_row[un.pair] + un.col0;
                const int n_tiles = (un.col1 - un.col0) / TC_BN;
                // A slices are refilled one k-block at a time as the previous
                // unit's last tile releases them, interleaved with the first
                // tile's B k-blocks, so the unit switch does not drain the MMA
                for (int t = 0; t < n_tiles; ++t) {
                    for (int kb = 0; kb < KB; ++kb) {
                        if (t == 0) {
                            mbar_wait_sleep(a_empty + kb, a_phase ^ 1);
                            mbar_expect_tx(a_full + kb, (uint32_t)(TC_NA * TC_BOX_BYTES));
                            for (int b = 0; b < TC_NA; ++b)
                                tma_load_2d(sA + (size_t)(b * KB + kb) * TC_BOX_BYTES, &tmA, a_full + kb, kb * TC_BK,
                                            un.row0 + b * TC_BM);
                        }
                        mbar_wait_sleep(b_empty + stage, phase ^ 1);
                        mbar_expect_tx(b_full + stage, TC_BOX_BYTES);
                        tma_load_2d(sB + (size_t)stage * TC_BOX_BYTES, &tmB, b_full + stage, kb * TC_BK,
                                    (int)(b0 + t * TC_BN));  // past the pair: rows of the next pair or TMA zero fill
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                a_phase ^= 1;
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, a_phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint32_t sA_addr = smem_u32(sA), sB_addr = smem_u32(sB);
            for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
                const TcUnit un = p.units[u];
                const int n_tiles = (un.col1 - un.col0) / TC_BN;
                for (int t = 0; t < n_tiles; ++t) {
                    mbar_wait_sleep(t_empty + acc, acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_base = tmem_base + (uint32_t)(acc * TC_NA * TC_BN);
                    for (int kb = 0; kb < KB; ++kb) {
                        if (t == 0) mbar_wait_sleep(a_full + kb, a_phase);
                        mbar_wait_sleep(b_full + stage, phase);
                        tc_fence_after();
                        const uint32_t bB = sB_addr + (uint32_t)(stage * TC_BOX_BYTES);
#pragma unroll
                        for (int k = 0; k < TC_BK / 16; ++k) {
                            const uint64_t bdesc = umma_desc_sw128(bB + k * 32);
#pragma unroll
                            for (int b = 0; b < TC_NA; ++b) {
                                const uint64_t adesc =
                                    umma_desc_sw128(sA_addr + (uint32_t)((b * KB + kb) * TC_BOX_BYTES) + k * 32);
                                tc_mma_bf16(d_base + b * TC_BN, adesc, bdesc, kIdesc, (kb | k) != 0);
                            }
                        }
                        tc_commit(b_empty + stage);
                        if (t == n_tiles - 1) tc_commit(a_empty + kb);  // slice kb free for the next unit
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc_commit(t_full + acc);
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                a_phase ^= 1;
            }
        }
    } else {
        // ===================== epilogue (warps 2..9) =====================
        // warp -> (TMEM lane quarter q, column half h).  Each thread owns two
        // rows — row q*32+lane of both A blocks — over the tile's 64 columns
        // [h*64, h*64+64), as two 32-column chunks (the second chunk's TMEM
        // load is in flight while the first is reduced).
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;  // column part of the tile: [h * 2 TC_CW, +2 TC_CW)
        const int et = threadIdx.x - 64;  // 0..255
        const uint32_t creg0 = KEY_MASK | (uint32_t)lane;         // A block 0
        const uint32_t creg1 = KEY_MASK | 32u | (uint32_t)lane;   // A block 1
        int acc = 0;
        uint32_t acc_phase = 0;
        int tb = 0;  // colbuf double buffer (alternates over all tiles of the CTA)
        // warps 2-5 merge the 4 quarter partials of the tile's columns; with
        // EC3R_MT_SPLITBAR the other warps only arrive at the tile's "full"
        // barrier (ids 2 + buffer) and wait on "merged" (ids 4 + buffer)
        // before reusing that buffer two tiles later
        const bool merger = et < TC_BN;
        int ttile = 0;
        int uiter = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x, ++uiter) {
            const TcUnit un = p.units[u];
            const int64_t a1 = p.a_off[un.pair + 1];
            const int64_t b0 = p.b_off[un.pair], b1 = p.b_off[un.pair + 1];
            const int M = (int)(b1 - b0);
            const int n_tiles = (un.col1 - un.col0) / TC_BN;
            RowTop2 R0{-INFINITY, -INFINITY, 0}, R1{-INFINITY, -INFINITY, 0};
            const int64_t row0 = (int64_t)un.row0 + q * 32 + lane, row1 = row0 + TC_BM;
            const bool rv0 = row0 < a1, rv1 = row1 < a1;
            for (int t = 0; t < n_tiles; ++t) {
#if EC3R_MT_SPLITBAR
                if (!merger && ttile >= 2) named_sync(4 + tb, TC_EPI_THREADS);  // tile ttile-2 merged
#endif
                mbar_wait(t_full + acc, acc_phase);
                tc_fence_after();
                const int col0 = un.col0 + t * TC_BN;
                const uint32_t ta =
                    tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * TC_NA * TC_BN + h * 2 * TC_CW);
                const uint32_t cbq = smem_u32(colbuf + (size_t)(tb * 4 + q) * TC_BN + h * 2 * TC_CW);
                uint32_t ra[TC_CW], rb[TC_CW], rc[TC_CW], rd[TC_CW];
                tmem_ld_async(ta, ra);
                tmem_ld_async(ta + TC_BN, rb);
                tmem_wait_ld();
                reg_fence(ra);
                reg_fence(rb);
                tmem_ld_async(ta + TC_CW, rc);
                tmem_ld_async(ta + TC_BN + TC_CW, rd);
                {
                    const int cbase = col0 + h * 2 * TC_CW;
                    const int ncol = min(TC_CW, M - cbase);
                    chunk_epilogue<TC_CW>(ra, rb, rv0 ? ncol : 0, rv1 ? ncol : 0, cbase, creg0, creg1, R0, R1, cbq,
                                          lane);
                }
                tmem_wait_ld();
                reg_fence(rc);
                reg_fence(rd);
                // accumulator drained: hand the TMEM buffer back to the MMA warp
                tc_fence_before();
                mbar_arrive(t_empty + acc);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                {
                    const int cbase = col0 + h * 2 * TC_CW + TC_CW;
                    const int ncol = min(TC_CW, M - cbase);
                    chunk_epilogue<TC_CW>(rc, rd, rv0 ? ncol : 0, rv1 ? ncol : 0, cbase, creg0, creg1, R0, R1,
                                          cbq + 8u * TC_CW, lane);
                }
#if EC3R_MT_SPLITBAR
                if (merger) named_sync(2 + tb, TC_EPI_THREADS);
                else named_arrive(2 + tb, TC_EPI_THREADS);
#else
                named_sync(1, TC_EPI_THREADS);
#endif
                // merge the 4 quarter partials of column et and fold into the
                // global state (colbuf is double-buffered: the next tile
                // writes the other half, so one barrier per tile suffices)
                if (merger && col0 + et < M) {
                    const uint32_t cb = smem_u32(colbuf + (size_t)tb * 4 * TC_BN + et);
                    const float2 v0 = lds_f2(cb), v1 = lds_f2(cb + 8u * TC_BN), v2 = lds_f2(cb + 16u * TC_BN),
                                 v3 = lds_f2(cb + 24u * TC_BN);
                    const float h01 = fmaxf(v0.x, v1.x), l01 = fminf(v0.x, v1.x);
                    const float h23 = fmaxf(v2.x, v3.x), l23 = fminf(v2.x, v3.x);
                    const float bk = fmaxf(h01, h23);
                    const float sk = fmax3f(fmax3f(l01, l23, fminf(h01, h23)), fmaxf(v0.y, v1.y), fmaxf(v2.y, v3.y));
                    const uint32_t qs = v0.x == bk ? 0u : v1.x == bk ? 1u : v2.x == bk ? 2u : 3u;
                    // bits 7..6 of the best key (column code, meaningless on
                    // this side) now hold the quarter: bits 7..0 = row in unit
                    const float bq = __uint_as_float((__float_as_uint(bk) & ~0xC0u) | (qs << 6));
                    __stcg(p.col_slots + un.slot + (col0 - un.col0) + et,
                           ((unsigned long long)f2ord(bq) << 32) | (unsigned long long)f2ord(sk));
                }
#if EC3R_MT_SPLITBAR
                if (merger) named_arrive(4 + tb, TC_EPI_THREADS);
#endif
                tb ^= 1;
                ++ttile;
            }
            // the two column-half warps of a quarter hold partial states of
            // the same rows: h = 1 hands its (best, second, column) over
            // rsc is double-buffered by unit parity: with split barriers the
            // h = 1 warps can finish a 1-2 tile unit and write its summaries
            // while the h = 0 warps still read the previous unit's; the buffer
            // they reuse two units later is ordered by the named_sync(1) in between
            // rsc[parity][part h - 1][A block][row]: parts 1.. hand their
            // (best, second, column) to part 0, which folds them in column
            // order (strictly greater wins: the first column on equal keys)
            const int ti = q * 32 + lane + (uiter & 1) * ((TC_HP - 1) * TC_NA * TC_BM);
            int c0 = R0.cb + (int)((__float_as_uint(R0.b) >> 6) & 31u);
            int c1 = R1.cb + (int)((__float_as_uint(R1.b) >> 6) & 31u);
            if (h >= 1) {
                float4* rp = rsc + (h - 1) * TC_NA * TC_BM;
                rp[ti] = make_float4(R0.b, R0.s, __int_as_float(c0), 0.f);
                rp[TC_BM + ti] = make_float4(R1.b, R1.s, __int_as_float(c1), 0.f);
            }
            named_sync(1, TC_EPI_THREADS);
            if (h == 0) {
#pragma unroll
                for (int hp = 0; hp < TC_HP - 1; ++hp) {
                    const float4* rp = rsc + hp * TC_NA * TC_BM;
                    const float4 o0 = rp[ti], o1 = rp[TC_BM + ti];
                    R0.s = fmax3f(R0.s, o0.y, fminf(R0.b, o0.x));
                    c0 = o0.x > R0.b ? __float_as_int(o0.z) : c0;
                    R0.b = fmaxf(R0.b, o0.x);
                    R1.s = fmax3f(R1.s, o1.y, fminf(R1.b, o1.x));
                    c1 = o1.x > R1.b ? __float_as_int(o1.z) : c1;
                    R1.b = fmaxf(R1.b, o1.x);
                }
                if (rv0) {
                    RowCand rc;
                    rc.k1 = R0.b;
                    rc.k2 = R0.s;
                    rc.c1 = c0;
                    rc.pad = 0;
                    p.cand[row0 * p.n_split + un.split] = rc;
                    if (p.n_split == 1) {
                        MatchRowState st;
                        if (row_decision(rc, M, __ldg(p.eps_d), p.ratio2, st)) p.rs[row0] = st;
                        else p.pending[atomicAdd((unsigned long long*)&p.counters[0], 1ull)] = (int32_t)row0;
                    }
                }
                if (rv1) {
                    RowCand rc;
                    rc.k1 = R1.b;
                    rc.k2 = R1.s;
                    rc.c1 = c1;
                    rc.pad = 0;
                    p.cand[row1 * p.n_split + un.split] = rc;
                    if (p.n_split == 1) {
                        MatchRowState st;
                        if (row_decision(rc, M, __ldg(p.eps_d), p.ratio2, st)) p.rs[row1] = st;
                        else p.pending[atomicAdd((unsigned long long*)&p.counters[0], 1ull)] = (int32_t)row1;
                    }
                }
            }
        }
#if EC3R_MT_SPLITBAR
        // consume the "merged" arrivals of the last two tiles
        if (!merger)
            for (int k = ttile >= 2 ? ttile - 2 : 0; k < ttile; ++k) named_sync(4 + (k & 1), TC_EPI_THREADS);
#endif
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TC_TMEM_COLS)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// certification

__device__ __forceinline__ int pair_of(const int64_t* __restrict__ off, int n_pairs, int64_t r) {
    int lo = 0, hi = n_pairs;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
}

// pair_of for one thread per row: thread 0 searches the CTA's first row and
// every thread steps forward from there (a CTA spans few pairs).  Call from
// all threads of the CTA (it contains a barrier).
__device__ __forceinline__ int pair_of_cta(const int64_t* __restrict__ off, int n_pairs, int64_t r, int64_t total) {
    __shared__ int p0;
    if (threadIdx.x == 0) {
        const int64_t r0 = (int64_t)blockIdx.x * blockDim.x < total ? (int64_t)blockIdx.x * blockDim.x : total - 1;
        // proportional guess (exact for equal-sized pairs, the batched
        // tracking case), a few steps either way, else the binary search
        const int64_t g = total > 0 ? r0 * n_pairs / total : 0;
        int q = (int)(g < (int64_t)n_pairs - 1 ? g : (int64_t)n_pairs - 1);
        int steps = 0;
        while (q > 0 && off[q] > r0 && steps < 4) { --q; ++steps; }
        while (q + 1 < n_pairs && off[q + 1] <= r0 && steps < 8) { ++q; ++steps; }
        const bool ok = off[q] <= r0 && (q + 1 >= n_pairs || off[q + 1] > r0);
        p0 = ok ? q : pair_of(off, n_pairs, r0);
    }
    __syncthreads();
    int p = p0;
    if (r < total)
        while (p + 1 < n_pairs && off[p + 1] <= r) ++p;
    return p;
}


// Stage 1 (one thread per row).  The exact top-2 similarities lie within the
// key bounds of the approximate ones, so
//   * the ratio test's reject (d_first > r^2 second, tracking.py:167) is
//     certain from the bounds alone — no argmax needed (most spurious rows);
//   * a pass is certain when the argmax is (a1 - a2 beyond both bounds, and
//     the runner-up cannot clamp to d2 = 0) and the bounds pass;
// everything else is listed for the float64 row re-scan.
__global__ void mt_decide_rows(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                               int64_t total_a, RowCand* __restrict__ cand, int n_split,
                               const double* __restrict__ eps_d, double ratio2,
                               MatchRowState* __restrict__ rs, int32_t* __restrict__ pending,
                               int64_t* __restrict__ counters, int only_empty) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int p = pair_of_cta(a_off, n_pairs, r, total_a);
    if (r >= total_a) return;
    const double eps_tc = *eps_d;
    const int64_t M = b_off[p + 1] - b_off[p];
    if (only_empty && M != 0) return;  // decided in the tensor-core epilogue
    MatchRowState s;
    if (M == 0) {  // no columns: no match (no unit wrote a candidate)
        row_decision(RowCand{}, 0, eps_tc, ratio2, s);
        rs[r] = s;
        return;
    }
    // merge the row's column-range candidates (top-2 keys, best column);
    // the merged candidate goes back to split 0 for the column stage
    RowCand c = cand[r * n_split];
    for (int sp = 1; sp < n_split; ++sp) {
        const RowCand o = cand[r * n_split + sp];
        if (o.c1 < 0) continue;  // range entirely past the pair's columns
        c.k2 = fmax3f(c.k2, o.k2, fminf(c.k1, o.k1));
        if (o.k1 > c.k1) { c.k1 = o.k1; c.c1 = o.c1; }
    }
    if (n_split > 1) cand[r * n_split] = c;
    if (row_decision(c, M, eps_tc, ratio2, s)) {
        rs[r] = s;
        return;
    }
    pending[atomicAdd((unsigned long long*)&counters[0], 1ull)] = (int32_t)r;
}

// Stage 2 (one thread per row, after the float64 row re-scan): rows that
// pass the ratio test need the mutual check best_a[best_b[i]] == i
// (tracking.py:160-162).  It is settled from the column's top-2 keys when
// they separate; otherwise the column is listed (once) for the float64
// column re-scan, which writes col_best.
__global__ void mt_need_cols(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                             int64_t total_a, const RowCand* __restrict__ cand, int n_split,
                             const unsigned long long* __restrict__ col_slots,
                             const long long* __restrict__ pair_slot, const double* __restrict__ eps_d, double ratio2,
                             MatchRowState* __restrict__ rs, const MatchRowD* __restrict__ rsd,
                             int32_t* __restrict__ col_best,
                             int32_t* __restrict__ pending, int64_t* __restrict__ counters) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int p = pair_of_cta(a_off, n_pairs, r, total_a);
    if (r >= total_a) return;
    const double eps_tc = *eps_d;
    const int64_t a0 = a_off[p], N = a_off[p + 1] - a0;
    const int64_t b0 = b_off[p], M = b_off[p + 1] - b0;
    const MatchRowState s = rs[r];
    if (M == 0 || s.best < 0) return;
    // (d1, d2) exist only for rows the exact re-scan decided (ratio_ok == -1)
    const MatchRowD sd = s.ratio_ok == -1 ? rsd[r] : MatchRowD{INFINITY, INFINITY};
    const bool keep = s.ratio_ok == 1 || (s.ratio_ok == -1 && (M <= 1 || !(sd.d1 > ratio2 * sd.d2)));
    if (!keep) return;
    const int64_t c = b0 + s.best, lr = r - a0;
    // merge the column's per-unit top-2 keys (units = 256-row blocks)
    uint32_t bo = 0, so = 0;
    int64_t rc = -1;
    const int n_rb = (int)((N + TC_NA * TC_BM - 1) / (TC_NA * TC_BM));
    const unsigned long long* sl = col_slots + pair_slot[p] + s.best;
    constexpr int kBatch = 4;  // independent slot loads in flight
    for (int rb0 = 0; rb0 < n_rb; rb0 += kBatch) {
        unsigned long long vv[kBatch];
#pragma unroll
        for (int q = 0; q < kBatch; ++q) vv[q] = rb0 + q < n_rb ? __ldcg(sl + (int64_t)(rb0 + q) * M) : 0ull;
#pragma unroll
        for (int q = 0; q < kBatch; ++q) {
            const int rb = rb0 + q;
            const uint32_t vb = (uint32_t)(vv[q] >> 32), vs = (uint32_t)vv[q];
            so = max(max(so, vs), min(bo, vb));
            if (vb > bo) {
                bo = vb;
                const uint32_t code = __float_as_uint(ord2f(vb));
                rc = (int64_t)rb * (TC_NA * TC_BM) + (int64_t)((code >> 5) & 1u) * TC_BM +
                     ((code >> 6) & 3u) * 32 + (code & 31u);
            }
        }
    }
    int mutual = -1;
    if (bo != 0) {
        const double cv = ord2f(bo);
        if (rc == lr) {
            const double sv = so ? (double)ord2f(so) : -INFINITY;
            if (N == 1 || sv < -1e30) mutual = 1;
            else if (cv - key_eps(cv, eps_tc) > sv + key_eps(sv, eps_tc) && sv + key_eps(sv, eps_tc) < 1.0)
                mutual = 1;
        } else if (rc >= 0 && rc < N) {
            // an approximate value of (r, c): the row's best key when it is
            // this element, else the exact similarity behind d1
            const RowCand rcand = cand[r * n_split];
            double kv = 0.0, ke = -1.0;
            if (rcand.c1 == s.best) { kv = rcand.k1; ke = key_eps(kv, eps_tc); }
            else if (s.ratio_ok == -1 && sd.d1 > 0.0) { kv = 1.0 - 0.5 * sd.d1; ke = 1e-12; }
            if (ke >= 0.0 && cv - key_eps(cv, eps_tc) > kv + ke) mutual = 0;
        }
    }
    rs[r].mutual = mutual;
    if (mutual == -1 && atomicCAS(col_best + c, -1, -2) == -1)
        pending[atomicAdd((unsigned long long*)&counters[1], 1ull)] = (int32_t)c;
}

// max squared row norm: one warp per row (grid-stride), the CTA's maximum in
// shared memory, one global atomic per CTA (a per-row atomic on one word
// serialises at L2)
__global__ void mt_norm_kernel(const uint16_t* __restrict__ X, int64_t rows, int D, unsigned int* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    __shared__ unsigned int smax;
    if (threadIdx.x == 0) smax = 0u;
    __syncthreads();
    unsigned int best = 0u;  // non-negative floats order like their bits
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        float s = 0.f;
        for (int k = lane * 8; k < D; k += 256) {
            double x[8];
            Vec16<uint16_t>::load(X + r * D + k, x);
#pragma unroll
            for (int i = 0; i < 8; ++i) s = fmaf((float)x[i], (float)x[i], s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        best = max(best, __float_as_uint(s));
    }
    if (lane == 0 && best) atomicMax(&smax, best);
    __syncthreads();
    if (threadIdx.x == 0 && smax) atomicMax(out, smax);
}

__global__ void mt_flag_all_kernel(int32_t* __restrict__ list, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) list[i] = (int32_t)i;
}

// Work units from the device row offsets.  mt_unit_scan (one CTA): per pair
// the unit and column-slot counts, exclusive-scanned in chunks of the CTA's
// threads; mt_units_kernel (one thread per unit): the unit's pair by binary
// search, then its (row block, column range).  A pair with `tiles` column
// tiles has min(tiles, n_split) ranges per row block; range j covers tiles
// [tiles * j / ns, tiles * (j + 1) / ns) (the host's count in match_tc_run).
__global__ void __launch_bounds__(1024) mt_unit_scan(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off,
                                                    int n_pairs, int n_split, long long* __restrict__ unit_base,
                                                    long long* __restrict__ pair_slot) {
    // each thread owns kPer consecutive pairs (serial prefix in registers),
    // one block scan of the per-thread totals per 1024 * kPer pairs: one
    // pass for batches up to 8,192 pairs (7,500 tracked frames: ~30 -> ~5 us)
    constexpr int kPer = 8;
    using BScan = cub::BlockScan<long long, 1024>;
    __shared__ typename BScan::TempStorage scan_tmp;
    __shared__ long long base_u, base_s;
    if (threadIdx.x == 0) { base_u = 0; base_s = 0; }
    __syncthreads();
    for (int p0 = 0; p0 < n_pairs; p0 += 1024 * kPer) {
        const int q0 = p0 + threadIdx.x * kPer;
        auto counts = [&](int p, long long& nu, long long& ns) {
            nu = 0; ns = 0;
            if (p < n_pairs) {
                const int64_t M = b_off[p + 1] - b_off[p], N = a_off[p + 1] - a_off[p];
                if (M > 0) {
                    const long long tiles = (M + TC_BN - 1) / TC_BN;
                    const long long rb = (N + TC_NA * TC_BM - 1) / (TC_NA * TC_BM);
                    nu = rb * (tiles < n_split ? tiles : n_split);
                    ns = rb * M;
                }
            }
        };
        long long su = 0, ss = 0;
        for (int k = 0; k < kPer; ++k) {  // totals, then the writes recompute (the offsets sit in L1)
            long long nu, ns;
            counts(q0 + k, nu, ns);
            su += nu;
            ss += ns;
        }
        long long eu, es, tu, ts;
        BScan(scan_tmp).ExclusiveSum(su, eu, tu);
        __syncthreads();
        BScan(scan_tmp).ExclusiveSum(ss, es, ts);
        long long cu = base_u + eu, cs = base_s + es;
        for (int k = 0; k < kPer; ++k) {
            const int p = q0 + k;
            long long nu, ns;
            counts(p, nu, ns);
            if (p < n_pairs) {
                unit_base[p] = cu;
                pair_slot[p] = cs;
            }
            cu += nu;
            cs += ns;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            base_u += tu;
            base_s += ts;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        unit_base[n_pairs] = base_u;
        pair_slot[n_pairs] = base_s;
    }
}

__global__ void mt_units_kernel(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                                int n_split, const long long* __restrict__ unit_base,
                                const long long* __restrict__ pair_slot, int64_t n_units, TcUnit* __restrict__ units) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_units) return;
    // proportional guess (exact for equal-sized pairs), else binary search
    const int64_t tot = unit_base[n_pairs];
    int lo = (int)min((int64_t)n_pairs - 1, tot > 0 ? u * n_pairs / tot : (int64_t)0);
    if (!(unit_base[lo] <= u && u < unit_base[lo + 1])) {
        lo = 0;
        int hi = n_pairs;  // unit_base[lo] <= u < unit_base[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (unit_base[mid] <= u) lo = mid; else hi = mid;
        }
    }
    while (lo + 1 < n_pairs && unit_base[lo + 1] <= u) ++lo;  // skip pairs without units
    const int p = lo;
    const int64_t M = b_off[p + 1] - b_off[p];
    const int tiles = (int)((M + TC_BN - 1) / TC_BN);
    const int ns = tiles < n_split ? tiles : n_split;
    const long long local = u - unit_base[p];
    const long long b = local / ns;
    const int j = (int)(local - b * ns);
    const int t0 = (int)((int64_t)tiles * j / ns), t1 = (int)((int64_t)tiles * (j + 1) / ns);
    units[u] = TcUnit{p, (int)(a_off[p] + b * TC_NA * TC_BM), t0 * TC_BN, t1 * TC_BN,
                      pair_slot[p] + b * M + t0 * TC_BN, j, 0};
}

// ---------------------------------------------------------------------------
// host side

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

static bool make_map(CUtensorMap* m, const uint16_t* base, int64_t rows, int D) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {TC_BK, TC_BM};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t tc_smem_bytes(int kblocks) {
    return 1024 + (size_t)TC_NA * kblocks * TC_BOX_BYTES + (size_t)TC_STAGES * TC_BOX_BYTES +
           sizeof(float2) * 2 * 4 * TC_BN + sizeof(float4) * 2 * (TC_HP - 1) * TC_NA * TC_BM +
           8 * (8 + 2 * TC_STAGES + 4) + 16;
}

// column slots: one per (unit, column) = sum over pairs of ceil(N/256) * M
static int64_t n_col_slots(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs) {
    int64_t n = 0;
    for (int p = 0; p < n_pairs; ++p)
        n += (a_off_h[p + 1] - a_off_h[p] + TC_NA * TC_BM - 1) / (TC_NA * TC_BM) * (b_off_h[p + 1] - b_off_h[p]);
    return n;
}

// Column ranges per row block: enough units for eight waves of CTAs when the
// batch has few row blocks (the configs[2] sweep's single pairs); 1 for
// batches of many pairs.  Row candidates are then merged across ranges.
static int choose_split(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs) {
    int64_t rb = 0, max_tiles = 1;
    for (int p = 0; p < n_pairs; ++p) {
        const int64_t N = a_off_h[p + 1] - a_off_h[p], M = b_off_h[p + 1] - b_off_h[p];
        if (M == 0 || N == 0) continue;
        rb += (N + TC_NA * TC_BM - 1) / (TC_NA * TC_BM);
        max_tiles = std::max<int64_t>(max_tiles, (M + TC_BN - 1) / TC_BN);
    }
    if (rb == 0) return 1;
    int64_t sp = (8 * kNumSMs + rb - 1) / rb;  // >= 8 waves: <= 1/8 wave quantization
    sp = std::min<int64_t>(std::min<int64_t>(sp, max_tiles), 64);
    return (int)std::max<int64_t>(sp, 1);
}

static int64_t max_units(int64_t ta, int n_pairs, int n_split) {
    return (ta / (TC_NA * TC_BM) + n_pairs + 1) * n_split;
}

size_t match_tc_workspace(const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs) {
    const int64_t ta = a_off_h[n_pairs];
    const int sp = choose_split(a_off_h, b_off_h, n_pairs);
    return align256(sizeof(RowCand) * (size_t)ta * sp) +
           align256(sizeof(unsigned long long) * (size_t)n_col_slots(a_off_h, b_off_h, n_pairs)) +
           2 * align256(sizeof(long long) * (size_t)(n_pairs + 1)) +
           align256(sizeof(TcUnit) * (size_t)max_units(ta, n_pairs, sp)) +
           align256(64);
}

struct TcWs {
    RowCand* cand;
    int n_split;
    unsigned long long* slots;
    long long* pair_slot;
    long long* unit_base;
    TcUnit* units;
    unsigned int* nb;
    size_t used;
};

static TcWs carve_tc(void* tc_ws, const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs) {
    const int64_t ta = a_off_h[n_pairs];
    Carver cv{(char*)tc_ws, 0};
    TcWs w;
    w.n_split = choose_split(a_off_h, b_off_h, n_pairs);
    w.cand = cv.take<RowCand>(ta * w.n_split);
    w.slots = cv.take<unsigned long long>(n_col_slots(a_off_h, b_off_h, n_pairs));
    w.pair_slot = cv.take<long long>(n_pairs + 1);
    w.unit_base = cv.take<long long>(n_pairs + 1);
    w.units = cv.take<TcUnit>(max_units(ta, n_pairs, w.n_split));
    w.nb = cv.take<unsigned int>(16);
    w.used = cv.used;
    return w;
}

// eps_tc, the tensor-core error bound (K5): fp32 accumulation of
// exact bf16 products, + bf16 rounding of the inputs when the exact rows are
// wider; the key quantisation is added per value (key_eps).  The norm bound
// is the caller's, or the device max row norms (mt_norm_kernel) rounded up.
__global__ void mt_eps_kernel(const unsigned int* __restrict__ nb, double norm_bound, int exact_dtype,
                              double* __restrict__ eps) {
    if (threadIdx.x != 0) return;
    if (!(norm_bound > 0)) {
        const float fa = __uint_as_float(nb[0]), fb = __uint_as_float(nb[1]);
        norm_bound = sqrt((double)fa * (1.0 + 1e-5)) * sqrt((double)fb * (1.0 + 1e-5)) + 1e-30;
    }
    double e = ldexp(norm_bound, -14);
    if (exact_dtype != 0) e += ldexp(norm_bound, -7);
    *eps = e;
}
// the device eps_tc lives in the workspace's norm words (nb[4..5])
static double* tc_eps(const TcWs& w) { return reinterpret_cast<double*>(w.nb + 4); }

// Tensor-core pass + stage-1 row decisions.  *tc_used = 0 when the shape or
// alignment rules out the tensor cores: every row and column is then listed
// for the float64 re-scan (counters[0] = rows, counters[1] = cols).
int match_tc_run(const uint16_t* A, const uint16_t* B, const int64_t* a_off_d, const int64_t* b_off_d,
                 const int64_t* b_row_d, int64_t n_b_rows,
                 const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs, int D, int exact_dtype,
                 double norm_bound, double ratio, MatchRowState* rs, int32_t* flag_rows, int32_t* flag_cols,
                 int64_t* counters, void* tc_ws, size_t tc_ws_bytes, int* tc_used, cudaStream_t st) {
    const int64_t ta = a_off_h[n_pairs], tb = b_off_h[n_pairs];
    *tc_used = 0;
    const bool tc_ok = (D % TC_BK == 0) && D <= 256 && (((uintptr_t)A | (uintptr_t)B) & 15) == 0 && ta > 0 &&
                       tb > 0 && get_encode() != nullptr;
    if (!tc_ok) {  // every decision goes to the float64 re-scan on the GPU
        mt_flag_all_kernel<<<(unsigned)((ta + 255) / 256), 256, 0, st>>>(flag_rows, ta);
        EC3R_CHECK_LAUNCH("mt_flag_all_kernel");
        mt_flag_all_kernel<<<(unsigned)((tb + 255) / 256), 256, 0, st>>>(flag_cols, tb);
        EC3R_CHECK_LAUNCH("mt_flag_all_kernel");
        int64_t c[2] = {ta, tb};
        EC3R_CUDA_TRY(cudaMemcpyAsync(counters, c, sizeof(c), cudaMemcpyHostToDevice, st));
        EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        return EC3R_OK;
    }
    const TcWs w = carve_tc(tc_ws, a_off_h, b_off_h, n_pairs);
    if (w.used > tc_ws_bytes) return EC3R_EWORKSPACE;
    // units and column-slot bases; units + pair bases travel in one copy
    // unit count on the host (grid size); the units themselves and the
    // pairs' column-slot bases are written on the device from the offsets
    int64_t n_units = 0;
    for (int pi = 0; pi < n_pairs; ++pi) {
        const int64_t M = b_off_h[pi + 1] - b_off_h[pi], N = a_off_h[pi + 1] - a_off_h[pi];
        if (M == 0) continue;
        const int64_t tiles = (M + TC_BN - 1) / TC_BN;
        n_units += (N + TC_NA * TC_BM - 1) / (TC_NA * TC_BM) * std::min<int64_t>(tiles, w.n_split);
    }
    mt_unit_scan<<<1, 1024, 0, st>>>(a_off_d, b_off_d, n_pairs, w.n_split, w.unit_base, w.pair_slot);
    EC3R_CHECK_LAUNCH("mt_unit_scan");
    if (n_units > 0) {
        mt_units_kernel<<<(unsigned)((n_units + 255) / 256), 256, 0, st>>>(a_off_d, b_off_d, n_pairs, w.n_split,
                                                                           w.unit_base, w.pair_slot, n_units,
                                                                           w.units);
        EC3R_CHECK_LAUNCH("mt_units_kernel");
    }
    if (!(norm_bound > 0)) {
        // max squared row norms of A and B (float32, rounded up in mt_eps_kernel)
        EC3R_CUDA_TRY(cudaMemsetAsync(w.nb, 0, 8, st));
        const auto norm_grid = [](int64_t rows) {
            return (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows * 32 + 255) / 256, (int64_t)kNumSMs * 8));
        };
        mt_norm_kernel<<<norm_grid(ta), 256, 0, st>>>(A, ta, D, w.nb);
        EC3R_CHECK_LAUNCH("mt_norm_kernel");
        mt_norm_kernel<<<norm_grid(n_b_rows), 256, 0, st>>>(B, n_b_rows, D, w.nb + 1);
        EC3R_CHECK_LAUNCH("mt_norm_kernel");
    }
    // eps_tc on the device (no host round trip: back-to-back calls queue)
    mt_eps_kernel<<<1, 32, 0, st>>>(w.nb, norm_bound, exact_dtype, tc_eps(w));
    EC3R_CHECK_LAUNCH("mt_eps_kernel");
    CUtensorMap tmA, tmB;
    if (!make_map(&tmA, A, ta, D) || !make_map(&tmB, B, n_b_rows, D)) {
        set_last_error_msg("cuTensorMapEncodeTiled failed");
        return EC3R_ECUDA;
    }
    TcParams prm;
    prm.a_off = a_off_d; prm.b_off = b_off_d; prm.b_row = b_row_d;
    prm.units = w.units; prm.n_units = (int)n_units; prm.kblocks = D / TC_BK;
    prm.cand = w.cand; prm.n_split = w.n_split; prm.col_slots = w.slots;
    prm.rs = rs; prm.pending = flag_rows; prm.counters = counters; prm.eps_d = tc_eps(w); prm.ratio2 = ratio * ratio;
    if (w.n_split > 1)  // ranges past a short pair's columns stay invalid (c1 = -1)
        EC3R_CUDA_TRY(cudaMemsetAsync(w.cand, 0xFF, sizeof(RowCand) * (size_t)ta * w.n_split, st));
    if (prm.n_units > 0) {
        const size_t smem = tc_smem_bytes(prm.kblocks);
        static std::atomic<size_t> smem_set{0};  // raise the opt-in limit once per size (benign duplicate sets)
        if (smem > smem_set.load()) {
            EC3R_CUDA_TRY(cudaFuncSetAttribute(mt_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            smem_set.store(smem);
        }
        int grid = prm.n_units < kNumSMs ? prm.n_units : kNumSMs;
        // EC3R_MT_GRID caps the persistent grid (SMs left free for concurrent
        // mapping kernels on another stream)
        if (const char* g = getenv("EC3R_MT_GRID")) grid = std::max(1, std::min(grid, atoi(g)));
        KernelTimer tk(TK_MATCH_TC, st);
        mt_tc_kernel<<<grid, TC_THREADS, smem, st>>>(tmA, tmB, prm);
        EC3R_CHECK_LAUNCH("mt_tc_kernel");
        tk.stop();
    }
    // with one column range the epilogue already decided every row of a pair
    // with columns; the kernel then only covers rows of column-less pairs
    bool any_empty = false;
    for (int pi = 0; pi < n_pairs && !any_empty; ++pi)
        any_empty = b_off_h[pi + 1] == b_off_h[pi] && a_off_h[pi + 1] > a_off_h[pi];
    if (w.n_split > 1 || any_empty) {
        mt_decide_rows<<<(unsigned)((ta + 255) / 256), 256, 0, st>>>(a_off_d, b_off_d, n_pairs, ta, w.cand,
                                                                     w.n_split, tc_eps(w), ratio * ratio, rs, flag_rows,
                                                                     counters, w.n_split == 1 ? 1 : 0);
        EC3R_CHECK_LAUNCH("mt_decide_rows");
    }
    *tc_used = 1;
    return EC3R_OK;
}

// Mutual checks of the passing rows (after the row re-scan); lists the
// columns that need the float64 column re-scan.  col_best is reset to -1.
int match_tc_need_cols(const int64_t* a_off_d, const int64_t* b_off_d, const int64_t* a_off_h,
                       const int64_t* b_off_h, int n_pairs, double ratio, MatchRowState* rs,
                       const MatchRowD* rsd, int32_t* col_best, int32_t* flag_cols, int64_t* counters, void* tc_ws,
                       cudaStream_t st) {
    const int64_t ta = a_off_h[n_pairs], tb = b_off_h[n_pairs];
    const TcWs w = carve_tc(tc_ws, a_off_h, b_off_h, n_pairs);
    EC3R_CUDA_TRY(cudaMemsetAsync(col_best, 0xFF, sizeof(int32_t) * (size_t)tb, st));
    mt_need_cols<<<(unsigned)((ta + 255) / 256), 256, 0, st>>>(a_off_d, b_off_d, n_pairs, ta, w.cand, w.n_split,
                                                               w.slots, w.pair_slot, tc_eps(w), ratio * ratio, rs,
                                                               rsd, col_best, flag_cols, counters);
    EC3R_CHECK_LAUNCH("mt_need_cols");
    return EC3R_OK;
}

}  // namespace ec3r
