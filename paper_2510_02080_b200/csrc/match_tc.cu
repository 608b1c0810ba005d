// K5 (tensor-core side): descriptor similarity on tcgen05 with a fused
// top-k epilogue, sm_100a.
//
// Replaces the dgemm + argmin/partition of match_descriptors
// (tracking.py:152-166).  One persistent CTA per SM walks work units
// (pair, 256-row super-block):
//   warp 0    TMA producer: the unit's two 128-row A blocks (K-major,
//             SWIZZLE_128B, resident for the unit) and a 4-stage ring of
//             128-column B k-blocks;
//   warp 1    TMEM allocator + single-thread tcgen05.mma issuer
//             (kind::f16, bf16 x bf16 -> fp32, M=128 N=128 K=16) into a
//             double-buffered 2 x 256-column TMEM accumulator;
//   warps 2-5 epilogue: tcgen05.ld 32x32b.x32 -> per-row running top-3
//             (registers) and per-column top-2 over the unit's rows
//             (REDUX.MAX on 32-bit keys that embed the lane), merged in
//             shared memory and folded into global per-column state with
//             two atomics per column.
// The N x M similarity matrix never exists in memory.  Approximate values
// then go through certification (mt_certify_*): every decision is either
// proven from the fp32 values plus an error bound or listed for the float64
// re-scan of match_exact.cu, so the matches are bit-identical to the float64
// reference.

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "match.cuh"

namespace ec3r {

constexpr int TC_BM = 128;       // rows per A block (UMMA M)
constexpr int TC_NA = 2;         // A blocks resident per unit
constexpr int TC_BN = 128;       // columns per B tile (UMMA N)
constexpr int TC_BK = 64;        // bf16 per 128-byte swizzle row
constexpr int TC_STAGES = 4;     // B ring depth
constexpr int TC_EPI_WARPS = 8;  // 2 per TMEM lane quarter: one per A block
constexpr int TC_EPI_THREADS = TC_EPI_WARPS * 32;
constexpr int TC_THREADS = 64 + TC_EPI_THREADS;  // producer + MMA + epilogue warps
constexpr int TC_BOX_BYTES = TC_BM * TC_BK * 2;  // 16 KB (A box and B box alike)
constexpr int TC_TMEM_COLS = 512;

// Per A-row approximate top-4 (value, column): the first three are re-scored
// in float64, the fourth bounds every other column.
constexpr int TC_TOPK = 4;
struct __align__(16) RowCand {
    float v[TC_TOPK];
    int32_t c[TC_TOPK];
};

struct TcParams {
    const int64_t* a_off;
    const int64_t* b_off;
    const int2* units;  // (pair, first row of the unit within the packed A)
    int n_units;
    int kblocks;        // D / 64
    float bias;         // makes every similarity + bias positive (ordered keys)
    RowCand* cand;
    unsigned long long* col_key;
    unsigned int* col_second;
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
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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

// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(TC_THREADS, 1)
mt_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-align the dynamic buffer (SWIZZLE_128B atoms)
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int KB = p.kblocks;
    unsigned char* sA = smem;                                   // TC_NA * KB boxes
    unsigned char* sB = sA + (size_t)TC_NA * KB * TC_BOX_BYTES;  // TC_STAGES boxes
    uint2* colbuf = (uint2*)(sB + (size_t)TC_STAGES * TC_BOX_BYTES);  // [TC_NA*4][TC_BN]
    uint64_t* bars = (uint64_t*)(colbuf + TC_NA * 4 * TC_BN);
    uint64_t* a_full = bars + 0;
    uint64_t* a_empty = bars + 1;
    uint64_t* b_full = bars + 2;
    uint64_t* b_empty = b_full + TC_STAGES;
    uint64_t* t_full = b_empty + TC_STAGES;
    uint64_t* t_empty = t_full + 2;
    uint32_t* tmem_slot = (uint32_t*)(t_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(a_full, 1);
        mbar_init(a_empty, 1);
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
                const int2 un = p.units[u];
                const int64_t b0 = p.b_off[un.x], b1 = p.b_off[un.x + 1];
                const int n_tiles = (int)((b1 - b0 + TC_BN - 1) / TC_BN);
                mbar_wait_sleep(a_empty, a_phase ^ 1);
                mbar_expect_tx(a_full, (uint32_t)(TC_NA * KB * TC_BOX_BYTES));
                for (int b = 0; b < TC_NA; ++b)
                    for (int kb = 0; kb < KB; ++kb)
                        tma_load_2d(sA + (size_t)(b * KB + kb) * TC_BOX_BYTES, &tmA, a_full, kb * TC_BK,
                                    un.y + b * TC_BM);
                a_phase ^= 1;
                for (int t = 0; t < n_tiles; ++t) {
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait_sleep(b_empty + stage, phase ^ 1);
                        mbar_expect_tx(b_full + stage, TC_BOX_BYTES);
                        tma_load_2d(sB + (size_t)stage * TC_BOX_BYTES, &tmB, b_full + stage, kb * TC_BK,
                                    (int)(b0 + t * TC_BN));
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
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
                const int2 un = p.units[u];
                const int64_t b0 = p.b_off[un.x], b1 = p.b_off[un.x + 1];
                const int n_tiles = (int)((b1 - b0 + TC_BN - 1) / TC_BN);
                mbar_wait_sleep(a_full, a_phase);
                a_phase ^= 1;
                tc_fence_after();
                for (int t = 0; t < n_tiles; ++t) {
                    mbar_wait_sleep(t_empty + acc, acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_base = tmem_base + (uint32_t)(acc * TC_NA * TC_BN);
                    for (int kb = 0; kb < KB; ++kb) {
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
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc_commit(t_full + acc);
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                tc_commit(a_empty);
            }
        }
    } else {
        // ===================== epilogue (warps 2..9) =====================
        // warp -> (TMEM lane quarter q, column half h).  Each thread owns two
        // rows — row q*32+lane of both A blocks — over the tile's 64 columns
        // [h*64, h*64+64): the two values of a column are folded in-thread
        // (max / min) before the warp reductions, halving the CREDUX count.
        // Column keys embed (block, lane) in their 6 low bits.
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int et = threadIdx.x - 64;  // 0..255
        const uint32_t code0 = 63u - (uint32_t)lane;        // block 0 (preferred on equal keys: smaller row)
        const uint32_t code1 = 31u - (uint32_t)lane;        // block 1
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
            const int2 un = p.units[u];
            const int64_t a1 = p.a_off[un.x + 1], a0 = p.a_off[un.x];
            const int64_t b0 = p.b_off[un.x], b1 = p.b_off[un.x + 1];
            const int M = (int)(b1 - b0);
            const int n_tiles = (M + TC_BN - 1) / TC_BN;
            // row state: best value / column and the second value (order
            // statistic, duplicates count) — all the decision stage needs
            float b0v = -INFINITY, s0v = -INFINITY, b1v = -INFINITY, s1v = -INFINITY;
            int b0c = -1, b1c = -1;
            const int64_t row0 = (int64_t)un.y + q * 32 + lane, row1 = row0 + TC_BM;
            const bool rv0 = row0 < a1, rv1 = row1 < a1;
            for (int t = 0; t < n_tiles; ++t) {
                mbar_wait(t_full + acc, acc_phase);
                tc_fence_after();
                const int col0 = t * TC_BN;
#pragma unroll 1
                for (int ch = 0; ch < 2; ++ch) {
                    const int cl = h * 64 + ch * 32;  // column offset within the tile
                    uint32_t r0[32], r1[32];
                    const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * TC_NA * TC_BN + cl);
                    tmem_ld32(ta, r0);
                    tmem_ld32(ta + TC_BN, r1);
                    const int cbase = col0 + cl;
                    const int ncol = min(32, M - cbase);  // valid columns (may be <= 0)
                    const int nv0 = rv0 ? ncol : 0, nv1 = rv1 ? ncol : 0;
                    // interior chunks (every row and column valid) skip all
                    // per-element predicates: warp-uniform fast path
                    const bool full = __all_sync(0xffffffffu, nv0 == 32 && nv1 == 32);
                    if (!full) {
                        // invalid entries become -bias: below every real value
                        // (|sim| <= bias / 2) and mapping to a zero-value key
                        const uint32_t sentinel = __float_as_uint(-p.bias);
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if (j >= nv0) r0[j] = sentinel;
                            if (j >= nv1) r1[j] = sentinel;
                        }
                    }
                    // row side, branch-free: second = max(second, min(v, best));
                    // strict > keeps the first column on equal values
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float v0 = __uint_as_float(r0[j]), v1 = __uint_as_float(r1[j]);
                        s0v = fmaxf(s0v, fminf(v0, b0v));
                        b0c = v0 > b0v ? cbase + j : b0c;
                        b0v = fmaxf(b0v, v0);
                        s1v = fmaxf(s1v, fminf(v1, b1v));
                        b1c = v1 > b1v ? cbase + j : b1c;
                        b1v = fmaxf(b1v, v1);
                    }
                    // column side: per column fold the thread's two rows, then
                    // top-1 and top-2 over the warp's 64 rows.  Invalid entries
                    // (-bias) map to zero-value keys.  All 32 first reductions
                    // are issued before the dependent second ones.
                    uint32_t hi[32], lo[32], m[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t k0 = (__float_as_uint(__uint_as_float(r0[j]) + p.bias) & 0xFFFFFFC0u) | code0;
                        const uint32_t k1 = (__float_as_uint(__uint_as_float(r1[j]) + p.bias) & 0xFFFFFFC0u) | code1;
                        hi[j] = max(k0, k1);
                        lo[j] = min(k0, k1);
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) m[j] = __reduce_max_sync(0xffffffffu, hi[j]);
                    uint32_t cm = 0, cm2 = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t m2 = __reduce_max_sync(0xffffffffu, hi[j] == m[j] ? lo[j] : hi[j]);
                        cm = (lane == j) ? m[j] : cm;
                        cm2 = (lane == j) ? m2 : cm2;
                    }
                    colbuf[q * TC_BN + cl + lane] = make_uint2(cm, cm2);
                }
                // accumulator drained: hand the TMEM buffer back to the MMA warp
                tc_fence_before();
                mbar_arrive(t_empty + acc);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                named_sync(1, TC_EPI_THREADS);
                // merge the 4 quarter partials of column et and fold into the global state
                if (et < TC_BN && col0 + et < M) {
                    unsigned long long best = 0;
                    uint32_t second = 0;
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                        const uint2 c = colbuf[qq * TC_BN + et];
                        if ((c.x & 0xFFFFFFC0u) == 0) continue;  // no valid row in this quarter
                        const uint32_t code = c.x & 63u;
                        const int bb = code >= 32 ? 0 : 1;
                        const int lanew = (bb == 0 ? 63 : 31) - (int)code;
                        const int64_t row = (int64_t)un.y - a0 + bb * TC_BM + qq * 32 + lanew;
                        const unsigned long long gk =
                            ((unsigned long long)(c.x & 0xFFFFFFC0u) << 32) | (0xFFFFFFFFull - (unsigned long long)row);
                        const uint32_t c2v = c.y & 0xFFFFFFC0u;  // zero-value keys contribute 0
                        if (gk > best) {
                            second = max(second, max(c2v, (uint32_t)(best >> 32)));
                            best = gk;
                        } else {
                            second = max(second, c.x & 0xFFFFFFC0u);
                        }
                    }
                    if (best) {
                        const int64_t gc = b0 + col0 + et;
                        const unsigned long long old = atomicMax(p.col_key + gc, best);
                        const uint32_t loser = (uint32_t)((old > best ? best : old) >> 32);
                        const uint32_t sec = max(second, loser);
                        if (sec) atomicMax(p.col_second + gc, sec);
                    }
                }
                named_sync(1, TC_EPI_THREADS);
            }
            // the two column-half warps of a quarter hold partial states of
            // the same rows: h = 1 hands its (best, column, second) over
            float4* rsc = reinterpret_cast<float4*>(colbuf);
            const int ti = q * 32 + lane;
            if (h == 1) {
                rsc[ti] = make_float4(b0v, __int_as_float(b0c), s0v, 0.f);
                rsc[TC_BM + ti] = make_float4(b1v, __int_as_float(b1c), s1v, 0.f);
            }
            named_sync(1, TC_EPI_THREADS);
            if (h == 0) {
                const float4 o0 = rsc[ti], o1 = rsc[TC_BM + ti];
                // merge two (best, column, second) summaries; h = 0 holds the
                // smaller columns of every tile only per tile, so ties go to
                // the smaller column explicitly
                auto merge = [](float& bv, int& bc, float& sv, float ov, int oc, float os) {
                    const bool take = ov > bv || (ov == bv && oc >= 0 && (bc < 0 || oc < bc));
                    sv = fmaxf(fminf(bv, ov), fmaxf(sv, os));
                    if (take) { bv = ov; bc = oc; }
                };
                merge(b0v, b0c, s0v, o0.x, __float_as_int(o0.y), o0.z);
                merge(b1v, b1c, s1v, o1.x, __float_as_int(o1.y), o1.z);
                if (rv0) {
                    RowCand rc;
                    rc.v[0] = b0v; rc.v[1] = s0v; rc.v[2] = rc.v[3] = -INFINITY;
                    rc.c[0] = b0c; rc.c[1] = rc.c[2] = rc.c[3] = -1;
                    p.cand[row0] = rc;
                }
                if (rv1) {
                    RowCand rc;
                    rc.v[0] = b1v; rc.v[1] = s1v; rc.v[2] = rc.v[3] = -INFINITY;
                    rc.c[0] = b1c; rc.c[1] = rc.c[2] = rc.c[3] = -1;
                    p.cand[row1] = rc;
                }
            }
            named_sync(1, TC_EPI_THREADS);
        }
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

__device__ __forceinline__ double d2x(double s) { return fmax(__dsub_rn(2.0, __dmul_rn(2.0, s)), 0.0); }

// Stage 1 (one thread per row): decide from the approximate values alone.
// Every true similarity is within eps of its tensor-core value, so the
// approximate order statistics bound the true ones: the argmax is certain
// when a1 - a2 > 2 eps (and the runner-up cannot clamp to d2 = 0), and the
// ratio test d1 > r^2 d2 (tracking.py:167) is certain when its interval
// bounds do not straddle.  Everything else goes to the float64 stages.
__device__ __forceinline__ double d2c(double s) { return fmax(2.0 - 2.0 * s, 0.0); }

__global__ void mt_decide_rows(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                               int64_t total_a, const RowCand* __restrict__ cand, double eps, double ratio2,
                               MatchRowState* __restrict__ rs, int32_t* __restrict__ pending,
                               int64_t* __restrict__ counters) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= total_a) return;
    const int p = pair_of(a_off, n_pairs, r);
    const int64_t M = b_off[p + 1] - b_off[p];
    MatchRowState s;
    s.d1 = INFINITY; s.d2 = INFINITY; s.best = -1; s.ratio_ok = -1;
    bool decided = false;
    if (M == 0) {
        decided = true;
    } else {
        const RowCand c = cand[r];
        const double a1 = c.v[0];
        if (M == 1) {
            decided = c.c[0] >= 0;
            s.best = c.c[0];
            s.ratio_ok = 1;  // ratio test skipped for a single column (tracking.py:165)
        } else {
            const double a2 = c.v[1];
            if (c.c[0] >= 0 && a1 - a2 > 2.0 * eps && a2 + eps < 1.0) {
                const double d1_lo = d2c(a1 + eps), d1_hi = d2c(a1 - eps);
                const double s_lo = d2c(a2 + eps), s_hi = d2c(a2 - eps);
                if (d1_lo > ratio2 * s_hi) { decided = true; s.ratio_ok = 0; }
                else if (d1_hi < ratio2 * s_lo) { decided = true; s.ratio_ok = 1; }
                s.best = c.c[0];
            }
        }
    }
    // undecided rows (~0.1-1%) go straight to the float64 full-row re-scan
    if (decided) rs[r] = s;
    else pending[atomicAdd((unsigned long long*)&counters[0], 1ull)] = (int32_t)r;
}

// Column side, stage 1: argmax certain when the best (quantised) key beats
// the second by more than the bound and the runner-up cannot clamp.
__global__ void mt_decide_cols(const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                               int64_t total_b, const unsigned long long* __restrict__ col_key,
                               const unsigned int* __restrict__ col_second, double bias, double eps,
                               int32_t* __restrict__ col_best, int32_t* __restrict__ pending,
                               int64_t* __restrict__ counters) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= total_b) return;
    const int p = pair_of(b_off, n_pairs, c);
    const int64_t N = a_off[p + 1] - a_off[p];
    if (N == 0) { col_best[c] = -1; return; }
    const unsigned long long k = col_key[c];
    const int64_t r1 = (int64_t)(0xFFFFFFFFull - (k & 0xFFFFFFFFull));
    bool ok = k != 0 && r1 >= 0 && r1 < N;
    if (ok && N >= 2) {
        const unsigned int s2 = col_second[c];
        if (s2 != 0) {
            const double a1 = (double)__uint_as_float((unsigned int)(k >> 32)) - bias;
            const double a2 = (double)__uint_as_float(s2) - bias;
            ok = (a1 - eps > a2 + eps) && (a2 + eps < 1.0);
        }
    }
    if (ok) col_best[c] = (int32_t)r1;
    else pending[atomicAdd((unsigned long long*)&counters[3], 1ull)] = (int32_t)c;
}

// Column side, stage 2 (one warp per pending column): the best row is
// re-scored; certified when the column's second value (plus the bound) is
// below it and below 1 (d2 clamp), else listed for the full re-scan.
template <typename T>
__global__ void mt_certify_cols(const T* __restrict__ A, const T* __restrict__ B, int D,
                                const int64_t* __restrict__ a_off, const int64_t* __restrict__ b_off, int n_pairs,
                                const int32_t* __restrict__ pending, const unsigned long long* __restrict__ col_key,
                                const unsigned int* __restrict__ col_second, double bias, double eps,
                                int32_t* __restrict__ col_best, int32_t* __restrict__ flag_cols,
                                int64_t* __restrict__ counters) {
    const int lane = threadIdx.x & 31;
    const int64_t n_pend = counters[3];
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_pend;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t c = pending[t];
    const int p = pair_of(b_off, n_pairs, c);
    const int64_t a0 = a_off[p], N = a_off[p + 1] - a0;
    const unsigned long long k = col_key[c];
    bool ok = k != 0;
    int64_t r1 = 0;
    double e1 = 0;
    if (ok) {
        r1 = (int64_t)(0xFFFFFFFFull - (k & 0xFFFFFFFFull));
        ok = r1 >= 0 && r1 < N;
        if (ok) e1 = warp_dot16<T>(A + (a0 + r1) * D, B + c * D, D, lane);
    }
    if (ok && N >= 2) {
        const unsigned int s2 = col_second[c];
        if (s2 != 0) {
            const double others = (double)__uint_as_float(s2) - bias + eps;
            ok = others < e1 && others < 1.0;
        }
    }
    if (lane == 0) {
        if (ok) col_best[c] = (int32_t)r1;
        else {
            const unsigned long long i = atomicAdd((unsigned long long*)&counters[1], 1ull);
            flag_cols[i] = (int32_t)c;
        }
    }
    }
}

__global__ void mt_norm_kernel(const uint16_t* __restrict__ X, int64_t rows, int D, unsigned int* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= rows) return;
    float s = 0.f;
    for (int k = lane * 8; k < D; k += 256) {
        double x[8];
        Vec16<uint16_t>::load(X + r * D + k, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) s = fmaf((float)x[i], (float)x[i], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) atomicMax(out, __float_as_uint(s));
}

__global__ void mt_flag_all_kernel(int32_t* __restrict__ list, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) list[i] = (int32_t)i;
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
           sizeof(uint2) * TC_NA * 4 * TC_BN + 8 * (2 + 2 * TC_STAGES + 4) + 16;
}

size_t match_tc_workspace(int64_t total_a, int64_t total_b, int n_pairs) {
    const int64_t max_units = total_a / TC_BM + n_pairs + 1;
    return align256(sizeof(RowCand) * (size_t)total_a) + align256(8 * (size_t)total_b) +
           align256(4 * (size_t)total_b) + align256(sizeof(int2) * (size_t)max_units) + align256(64) +
           align256(4 * (size_t)total_a) + align256(4 * (size_t)total_b);
}

// Stage 1 on every row / column, then stage-2 float64 certification of the
// pending ones.  The pending counts live on the device; stage 2 runs on a
// fixed persistent grid that strides over the lists, so no host
// synchronisation is needed.
template <typename T>
static int certify(const void* Ax, const void* Bx, int D, const int64_t* a_off, const int64_t* b_off, int n_pairs,
                   int64_t ta, int64_t tb, const RowCand* cand, const unsigned long long* ck, const unsigned int* cs,
                   double bias, double eps_row, double eps_col, double ratio2, MatchRowState* rs, int32_t* col_best,
                   int32_t* pend_rows, int32_t* pend_cols, int32_t* flag_rows, int32_t* flag_cols,
                   int64_t* counters, cudaStream_t st) {
    (void)pend_rows;
    mt_decide_rows<<<(unsigned)((ta + 255) / 256), 256, 0, st>>>(a_off, b_off, n_pairs, ta, cand, eps_row, ratio2, rs,
                                                                 flag_rows, counters);
    EC3R_CHECK_LAUNCH("mt_decide_rows");
    mt_decide_cols<<<(unsigned)((tb + 255) / 256), 256, 0, st>>>(a_off, b_off, n_pairs, tb, ck, cs, bias, eps_col,
                                                                 col_best, pend_cols, counters);
    EC3R_CHECK_LAUNCH("mt_decide_cols");
    mt_certify_cols<T><<<kNumSMs * 4, 256, 0, st>>>(
        (const T*)Ax, (const T*)Bx, D, a_off, b_off, n_pairs, pend_cols, ck, cs, bias, eps_col, col_best, flag_cols,
        counters);
    EC3R_CHECK_LAUNCH("mt_certify_cols");
    return EC3R_OK;
}

int match_tc_run(const uint16_t* A, const uint16_t* B, const void* A_x, const void* B_x, const int64_t* a_off_d,
                 const int64_t* b_off_d, const int64_t* a_off_h, const int64_t* b_off_h, int n_pairs, int D,
                 int exact_dtype, double norm_bound, double ratio, MatchRowState* rs, int32_t* col_best,
                 int32_t* flag_rows, int32_t* flag_cols, int64_t* counters, void* tc_ws, size_t tc_ws_bytes,
                 cudaStream_t st) {
    const int64_t ta = a_off_h[n_pairs], tb = b_off_h[n_pairs];
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
    Carver cv{(char*)tc_ws, 0};
    RowCand* cand = cv.take<RowCand>(ta);
    unsigned long long* ck = cv.take<unsigned long long>(tb);
    unsigned int* cs = cv.take<unsigned int>(tb);
    const int64_t max_units = ta / TC_BM + n_pairs + 1;
    int2* units = cv.take<int2>(max_units);
    unsigned int* nb = cv.take<unsigned int>(16);
    int32_t* pend_rows = cv.take<int32_t>(ta);
    int32_t* pend_cols = cv.take<int32_t>(tb);
    if (cv.used > tc_ws_bytes) return EC3R_EWORKSPACE;
    std::vector<int2> hu;
    hu.reserve(max_units);
    for (int pi = 0; pi < n_pairs; ++pi) {
        if (b_off_h[pi + 1] == b_off_h[pi]) continue;  // no columns: nothing to score
        for (int64_t r = a_off_h[pi]; r < a_off_h[pi + 1]; r += TC_NA * TC_BM) hu.push_back(make_int2(pi, (int)r));
    }
    EC3R_CUDA_TRY(cudaMemsetAsync(ck, 0, 8 * (size_t)tb, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(cs, 0, 4 * (size_t)tb, st));
    if (!hu.empty())
        EC3R_CUDA_TRY(cudaMemcpyAsync(units, hu.data(), sizeof(int2) * hu.size(), cudaMemcpyHostToDevice, st));
    if (!(norm_bound > 0)) {
        // max squared row norms of A and B (float32, rounded up below)
        EC3R_CUDA_TRY(cudaMemsetAsync(nb, 0, 8, st));
        mt_norm_kernel<<<(unsigned)((ta * 32 + 255) / 256), 256, 0, st>>>(A, ta, D, nb);
        EC3R_CHECK_LAUNCH("mt_norm_kernel");
        mt_norm_kernel<<<(unsigned)((tb * 32 + 255) / 256), 256, 0, st>>>(B, tb, D, nb + 1);
        EC3R_CHECK_LAUNCH("mt_norm_kernel");
        unsigned int h[2];
        EC3R_CUDA_TRY(cudaMemcpyAsync(h, nb, 8, cudaMemcpyDeviceToHost, st));
        EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        float fa, fb;
        memcpy(&fa, &h[0], 4);
        memcpy(&fb, &h[1], 4);
        norm_bound = sqrt((double)fa * (1.0 + 1e-5)) * sqrt((double)fb * (1.0 + 1e-5)) + 1e-30;
    }
    // error bounds (K5): fp32 tensor-core accumulation of exact
    // bf16 products, + key quantisation (5 low bits) on the column side,
    // + bf16 rounding of the inputs when the exact rows are wider.
    const double Bn = norm_bound;
    const float bias = (float)fmax(2.0, 2.0 * Bn);
    double eps_row = ldexp(Bn, -14);
    if (exact_dtype != 0) eps_row += ldexp(Bn, -7);
    // column keys drop 6 low mantissa bits (64 ulps of a value < 2 (bias + Bn))
    const double eps_col = eps_row + ldexp(2.0 * ((double)bias + Bn), -17);
    CUtensorMap tmA, tmB;
    if (!make_map(&tmA, A, ta, D) || !make_map(&tmB, B, tb, D)) {
        set_last_error_msg("cuTensorMapEncodeTiled failed");
        return EC3R_ECUDA;
    }
    TcParams prm;
    prm.a_off = a_off_d; prm.b_off = b_off_d;
    prm.units = units; prm.n_units = (int)hu.size(); prm.kblocks = D / TC_BK; prm.bias = bias;
    prm.cand = cand; prm.col_key = ck; prm.col_second = cs;
    if (prm.n_units > 0) {
        const size_t smem = tc_smem_bytes(prm.kblocks);
        EC3R_CUDA_TRY(cudaFuncSetAttribute(mt_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = prm.n_units < kNumSMs ? prm.n_units : kNumSMs;
        mt_tc_kernel<<<grid, TC_THREADS, smem, st>>>(tmA, tmB, prm);
        EC3R_CHECK_LAUNCH("mt_tc_kernel");
    }
    EC3R_CUDA_TRY(cudaMemsetAsync(counters, 0, 32, st));
    const double ratio2 = ratio * ratio;  // tracking.py:158
    switch (exact_dtype) {
        case 0:
            return certify<uint16_t>(A, B, D, a_off_d, b_off_d, n_pairs, ta, tb, cand, ck, cs, bias, eps_row, eps_col,
                                     ratio2, rs, col_best, pend_rows, pend_cols, flag_rows, flag_cols, counters, st);
        case 1:
            return certify<float>(A_x, B_x, D, a_off_d, b_off_d, n_pairs, ta, tb, cand, ck, cs, bias, eps_row,
                                  eps_col, ratio2, rs, col_best, pend_rows, pend_cols, flag_rows, flag_cols, counters,
                                  st);
        default:
            return certify<double>(A_x, B_x, D, a_off_d, b_off_d, n_pairs, ta, tb, cand, ck, cs, bias, eps_row,
                                   eps_col, ratio2, rs, col_best, pend_rows, pend_cols, flag_rows, flag_cols,
                                   counters, st);
    }
}

}  // namespace ec3r
