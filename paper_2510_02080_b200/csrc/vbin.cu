// K4: binned super-block voxel fusion (stage c) on sm_100a.
//
// Replaces Submap.world_points / Mapping.fused_cloud (mapping.py:56-57,
// 332-338) under the declared fusion rule of oracle/fuse.py: keys are
// _pack(floor(x / cell)) (_kernels/_numpy.py:50-55) of the exact float64
// chain (fuse_common.cuh), per key sum conf, conf-weighted centroid and
// count, output sorted by key.
//
// Why this shape.  The bench map has 18.7 points per voxel, almost all of it
// reuse ACROSS frames (1.37 points per voxel inside one frame), and on this
// part every atomic costs ~1.3 (L2 RED) to ~2 (shared ATOMS) cycles per lane
// on the SM while plain ALU work issues 128 lanes per cycle.  So no per-point
// atomic anywhere: points are grouped by 8x8x8-voxel super-block ("bin",
// 16 cm at 2 cm) with ballots and prefix counts, and every bin is reduced by
// a block radix sort + prefix sums.
//
//  1. bn_bin_frames_kernel (one pass over depth + confidence, 8 B/px): a warp
//     walks a contiguous 512-pixel span in 32-pixel slices.  Exact cells
//     (fuse_common.cuh), then the valid points of the span are compacted in
//     raster order into the span's payload region (one coalesced 8-byte
//     store per point: 9-bit voxel-in-bin index | 31-bit confidence | three
//     8-bit in-voxel offsets) and every raster run of equal bin becomes one
//     run record (start, length, bin id): ballots + shuffles, no atomics per
//     point.  Bin ids come from an open-addressing table of super-block keys
//     behind a per-warp cache (one lookup per run).
//  2. run records are counting-sorted by bin (one device scan + scatter).
//  3. bn_aggregate_kernel (persistent CTAs, dynamic bin fetch): a bin's runs
//     are flattened into chunks of AG_CH points, sorted by voxel index
//     (cub::BlockRadixSort on 9 key bits), and reduced with one block-wide
//     prefix sum of the fixed-point values: the head of a voxel's run
//     publishes its exclusive prefix, the tail adds (inclusive - exclusive)
//     into the bin's shared-memory accumulators with a plain store (the only
//     writer of that voxel in the chunk).  64-bit fixed-point integers make the
//     result independent of every ordering: run-to-run bit-for-bit
//     deterministic and independent of how the frames were split into calls.
//     The bin's occupied voxels are then written once, in in-bin (x, y, z)
//     order, with per-(bin, x, y) column counts.
//  4. ordered emit: bins are sorted by key; for bins grouped by x then y the
//     global key order of the voxel columns is a closed-form interleave of
//     (bin x, voxel x, bin y, voxel y, bin z); one exclusive scan of the column
//     counts in that order gives every column its output offset and
//     bn_permute_kernel writes the sorted map (no voxel sort).
//
// Precision of the declared rule: Σconf is exact to 2^-28 per point, the
// in-voxel offsets are quantised to cell/256 (centroid error <= cell/512 =
// 39 µm at 2 cm; the engine is selected for cells <= 2.56 cm, so always
// < 50 µm against the 1e-4 m tolerance).  Keys and counts are exact.

#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vbin.cuh"

namespace ec3r {

constexpr int BN_NT = 128;
constexpr int BN_WARPS = BN_NT / 32;
constexpr int BN_SPAN = 512;                 // entries (pixels / points) per warp span
constexpr int BN_CTA = BN_SPAN * BN_WARPS;   // entries per CTA region
constexpr int BN_WC = 128;                   // per-warp bin-id cache entries
constexpr int BN_SBV = 512;                  // voxels per bin (8^3)
constexpr int BN_LENB = 10;                  // run length bits (length <= 512)
constexpr uint32_t BN_DROP = 0xFFFFFFFFu;    // run record of a dropped run (bins full)
constexpr uint32_t BN_IDMASK = (1u << (32 - BN_LENB)) - 1u;  // 22-bit bin ids
constexpr int AG_NT = 256;
#ifndef EC3R_AG_IPT
#define EC3R_AG_IPT 8
#endif
constexpr int AG_IPT = EC3R_AG_IPT;
constexpr int AG_CH = AG_NT * AG_IPT;        // points per aggregation chunk
constexpr float kConfScale = 268435456.0f;   // 2^28: fixed-point confidence
constexpr double kConfInv = 1.0 / 268435456.0;

struct __align__(16) BinEntry {
    unsigned long long key;  // pack of super-block coordinates (cell >> 3)
    int id;                  // bin id; -1 while being published, -2 overflow
    int pad;
};

// counters
enum { C_IN = 0, C_OOR, C_OVF, C_SLOW, C_BINS, C_VOX, C_VOX_OVF, C_WORK, C_RUNS, C_N };

struct BinGroup {
    int start_x, n_x, off_xy, n_xy, r_z, pad;
};

// Aggregation / emit workspace (grown on demand, owned by the engine).
struct BfWs {
    uint32_t* run_off;      // max_bins + 1
    uint32_t* cursor;       // max_bins
    uint2* sorted;          // run records by bin
    unsigned long long* st_key;
    float4* st_sum;
    int32_t* st_cnt;
    uint32_t* st_tag;
    uint8_t* colcnt;        // n_bins * 64
    unsigned long long* skeys;   // n_bins (sorted)
    uint32_t* ids;
    uint32_t* sids;
    BinGroup* grp;
    uint32_t* scan_in;      // n_bins * 64
    uint32_t* col_base;     // n_bins * 64
    void* cub_tmp;
    size_t cub_bytes;
};

struct BinFuse {
    int64_t max_voxels = 0, max_bins = 0;
    double cell = 0.02;
    unsigned long long tmask = 0;
    BinEntry* table = nullptr;
    unsigned long long* bin_keys = nullptr;
    uint32_t* bin_slot = nullptr;
    uint32_t* bin_nrun = nullptr;
    unsigned long long* ctr = nullptr;
    // payload (u64 per entry) and run records (uint2 per entry) share one
    // index space of BN_SPAN-entry warp spans; span_nh = run records per span
    unsigned long long* pay = nullptr;
    uint2* runs = nullptr;
    uint32_t* span_nh = nullptr;
    int64_t cap = 0, used = 0;  // entries
    // aggregation / emit state
    bool dirty = true;
    int64_t n_bins = 0;
    char* ws = nullptr;
    size_t ws_cap = 0;
    BfWs view;
};

// ---------------------------------------------------------------------------
// bin table

__device__ __forceinline__ void bf_load_entry(const BinEntry* e, unsigned long long& key, int& id) {
    unsigned long long lo, hi;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(e) : "memory");
    key = lo;
    id = (int)(unsigned)(hi & 0xFFFFFFFFull);
}

__device__ __forceinline__ int bf_load_id(const BinEntry* e) {
    int id;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(id) : "l"(&e->id) : "memory");
    return id;
}

struct BinTab {
    BinEntry* table;
    unsigned long long tmask;
    unsigned long long* bin_keys;
    uint32_t* bin_slot;
    unsigned long long* ctr;
    int64_t max_bins;
};

// Find or allocate the bin of super-block key k (one thread).  Returns the
// bin id or -2 when the table or the bin arrays are full.
__device__ __noinline__ int bf_find_or_insert(const BinTab& t, unsigned long long k) {
    unsigned long long h = table_slot(k, t.tmask);
    for (unsigned long long probe = 0; probe <= t.tmask; ++probe) {
        BinEntry* e = t.table + h;
        unsigned long long ek;
        int id;
        bf_load_entry(e, ek, id);
        if (ek == k) {
            while (id == -1) id = bf_load_id(e);  // winner is publishing
            return id;
        }
        if (ek == kEmpty) {
            const unsigned long long prev = atomicCAS(&e->key, kEmpty, k);
            if (prev == kEmpty) {
                const unsigned long long slot = atomicAdd(&t.ctr[C_BINS], 1ull);
                int got = -2;
                if ((int64_t)slot < t.max_bins) {
                    got = (int)slot;
                    t.bin_keys[slot] = k;  // read by later kernels only
                    t.bin_slot[slot] = (uint32_t)h;
                }
                atomicExch(&e->id, got);
                return got;
            }
            if (prev == k) {
                int i2 = bf_load_id(e);
                while (i2 == -1) i2 = bf_load_id(e);
                return i2;
            }
        }
        h = (h + 1) & t.tmask;
    }
    return -2;
}

struct WarpCache {
    unsigned long long ckey[BN_WC];  // bin-id cache (key, id), one writer per entry
    int cid[BN_WC];
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Bin id of key through the warp's direct-mapped cache (entry from the low
// bits of the bin coordinates: neighbouring bins never share an entry).
// Lanes with act resolve; every lane of the warp must call.  Misses go to
// the global table; one lane per cache entry refills it.
__device__ __forceinline__ int bf_bin_id(const BinTab& t, WarpCache& w, bool act, unsigned long long key) {
    const int lane = threadIdx.x & 31;
    const int ce = (int)(((key >> 42) & 7u) | (((key >> 21) & 3u) << 3) | ((key & 3u) << 5));
    int id = -3;
    if (act && w.ckey[ce] == key) id = w.cid[ce];
    const bool miss = act && id == -3;
    if (__any_sync(0xffffffffu, miss)) {
        if (miss) id = bf_find_or_insert(t, key);
        const unsigned same = __match_any_sync(0xffffffffu, miss ? ce : -1);
        __syncwarp();
        if (miss && lane == __ffs(same) - 1 && id >= 0) {
            w.ckey[ce] = key;
            w.cid[ce] = id;
        }
        __syncwarp();
    }
    return id;
}

// ---------------------------------------------------------------------------
// 1. binning: warp spans of raster-ordered points

// payload: [63:55] voxel-in-bin index (x major), [54] 0 (1 marks the sort
// padding ~0, which therefore sorts after every real point), [53:24]
// confidence bits 30..1 (a positive float without its sign bit and its last
// mantissa bit: relative 2^-23), [23:0] in-voxel offsets x, y, z in cell/256
// steps.
__device__ __forceinline__ unsigned q8(float f) {
    return (unsigned)min(max(__float2int_rd(f * 256.0f), 0), 255);
}
__device__ __forceinline__ unsigned long long bn_payload(int cx, int cy, int cz, float fx, float fy, float fz,
                                                         float conf) {
    const unsigned l = (unsigned)(cz & 7) | ((unsigned)(cy & 7) << 3) | ((unsigned)(cx & 7) << 6);
    const unsigned off = (q8(fx) << 16) | (q8(fy) << 8) | q8(fz);
    return ((unsigned long long)l << 55) | ((unsigned long long)((__float_as_uint(conf) >> 1) & 0x3FFFFFFFu) << 24) |
           off;
}

struct SpanState {
    unsigned long long carry;  // bin key of the span's last valid point so far
    uint32_t nv, nh;           // valid points, runs
};

// One 32-point slice of a span (every lane calls): compacts the valid points
// into the span's payload region in lane order and records run heads
// (id << BN_LENB | start entry; id BN_IDMASK = dropped, bins full).
__device__ __forceinline__ void span_slice(const BinTab& tab, WarpCache& wc, bool valid, unsigned long long bk,
                                           unsigned long long pay, unsigned long long* __restrict__ pay_span,
                                           uint32_t* hrec, SpanState& s) {
    const int lane = threadIdx.x & 31;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (vm == 0u) return;
    const unsigned below = vm & lanemask_lt();
    const int src = below ? 31 - __clz(below) : lane;
    const unsigned long long pk = __shfl_sync(0xffffffffu, bk, src);
    const unsigned long long prev = below ? pk : s.carry;
    const bool head = valid && bk != prev;
    const unsigned hm = __ballot_sync(0xffffffffu, head);
    const uint32_t e = s.nv + __popc(below);
    if (valid) pay_span[e] = pay;
    const int id = bf_bin_id(tab, wc, head, bk);
    if (head) hrec[s.nh + __popc(hm & lanemask_lt())] = ((id >= 0 ? (uint32_t)id : BN_IDMASK) << BN_LENB) | e;
    s.nv += __popc(vm);
    s.nh += __popc(hm);
    s.carry = __shfl_sync(0xffffffffu, bk, 31 - __clz(vm));
}

struct BnOut {
    BinTab tab;
    uint32_t* bin_nrun;
    unsigned long long* pay;
    uint2* runs;
    uint32_t* span_nh;
    unsigned long long* ctr;
    uint32_t entry0;  // first entry of this launch (a multiple of BN_CTA)
};

// Run records of a finished span.  Returns the points dropped (bin table
// overflow).
__device__ __forceinline__ unsigned span_finish(const BnOut& o, const uint32_t* hrec, const SpanState& s,
                                                uint32_t span_entry0) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    unsigned dropped = 0;
    uint2* out = o.runs + span_entry0;
    const uint32_t emask = (1u << BN_LENB) - 1u;
    for (uint32_t i = lane; i < s.nh; i += 32) {
        const uint32_t h = hrec[i];
        const uint32_t st = h & emask, en = (i + 1 < s.nh) ? (hrec[i + 1] & emask) : s.nv;
        const uint32_t id = h >> BN_LENB;
        if (id != BN_IDMASK) {
            out[i] = make_uint2(span_entry0 + st, (id << BN_LENB) | (en - st));
            atomicAdd(&o.bin_nrun[id], 1u);
        } else {
            out[i] = make_uint2(0u, BN_DROP);
            dropped += en - st;
        }
    }
    if (lane == 0) {
        o.span_nh[span_entry0 / BN_SPAN] = s.nh;
        if (s.nh) atomicAdd(&o.ctr[C_RUNS], (unsigned long long)s.nh);
    }
    return dropped;
}

struct BnSmem {
    WarpCache wc[BN_WARPS];
    uint32_t hrec[BN_WARPS][BN_SPAN];
    unsigned long long cnt[4];
};

__device__ __forceinline__ void bn_flush_counters(BnSmem& sm, const BnOut& o, unsigned n_in, unsigned n_oor,
                                                  unsigned n_drop, unsigned n_slow) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        n_in += __shfl_xor_sync(0xffffffffu, n_in, off);
        n_oor += __shfl_xor_sync(0xffffffffu, n_oor, off);
        n_drop += __shfl_xor_sync(0xffffffffu, n_drop, off);
        n_slow += __shfl_xor_sync(0xffffffffu, n_slow, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (n_in) atomicAdd(&sm.cnt[0], (unsigned long long)n_in);
        if (n_oor) atomicAdd(&sm.cnt[1], (unsigned long long)n_oor);
        if (n_drop) atomicAdd(&sm.cnt[2], (unsigned long long)n_drop);
        if (n_slow) atomicAdd(&sm.cnt[3], (unsigned long long)n_slow);
    }
    __syncthreads();
    if (threadIdx.x < 4 && sm.cnt[threadIdx.x]) atomicAdd(&o.ctr[threadIdx.x], sm.cnt[threadIdx.x]);
}

// Cell of one pixel (u, v) of listed frame slot `slot` (the per-pixel form of
// frame_cells4): fast float32 fold, exact float64 re-run near faces.
__device__ __forceinline__ bool pixel_cell(const FrameGeom& a, float4 Au, float4 Bv, float4 Tm, int slot, int u, int v,
                                           float z, float c, int& cx, int& cy, int& cz, float& fx, float& fy,
                                           float& fz, unsigned& n_in, unsigned& n_oor, unsigned& n_slow) {
    const float inv = a.inv_cell_f;
    const float dx = Au.x + Bv.x, dy = Au.y + Bv.y, dz = Au.z + Bv.z;
    const float x = fmaf(z, dx, Tm.x), y = fmaf(z, dy, Tm.y), zz = fmaf(z, dz, Tm.z);
    const float ax = fabsf(x) + fabsf(y) + fabsf(zz);
    const float err = 2.384185791015625e-07f * (2.0f * z * (Au.w + Bv.w) + Tm.w + 2.0f * ax) + 1e-9f;
    const float margin = err * inv + 3.6e-7f;
    const float qx = x * inv, qy = y * inv, qz = zz * inv;
    const float flx = floorf(qx), fly = floorf(qy), flz = floorf(qz);
    const float dev = fmaxf(fmaxf(fabsf(qx - flx - 0.5f), fabsf(qy - fly - 0.5f)), fabsf(qz - flz - 0.5f));
    const float qmax = fmaxf(fmaxf(fabsf(qx), fabsf(qy)), fabsf(qz));
    bool valid = z > 0.f && c > 0.f;
    n_in += valid;
    cx = (int)flx; cy = (int)fly; cz = (int)flz;
    if (valid && !(dev < 0.5f - margin && qmax <= 1.0e6f)) {
        long long cc[3];
        exact_cells(a.slot_poses + 8 * slot, a.slot_globals + 8 * slot, ray_coef(u, a.cx, a.fx), ray_coef(v, a.cy, a.fy),
                    z, a.cell, cc);
        ++n_slow;
        if (cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2])) {
            cx = (int)cc[0]; cy = (int)cc[1]; cz = (int)cc[2];
        } else {
            ++n_oor;
            valid = false;
        }
    }
    fx = qx - (float)cx; fy = qy - (float)cy; fz = qz - (float)cz;
    return valid;
}

// TMA bulk copies (global -> shared, completion on an mbarrier)
__device__ __forceinline__ uint32_t bn_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bn_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     bn_smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(bn_smem_u32(bar))
                 : "memory");
}

// Grid (CTA regions of BN_CTA pixels, listed frames).  The region's depth
// and confidence (2 x 8 KB) are staged in shared memory by two TMA bulk
// copies (cooperative loads when the planes are not 16-byte aligned); warp
// w then owns the span [BN_SPAN * w, + BN_SPAN) of the region and each lane
// walks every 32nd pixel of it.
__global__ void __launch_bounds__(BN_NT, 4) bn_bin_frames_kernel(FrameGeom a, BnOut o) {
    extern __shared__ float4 sA[];  // A[W]
    __shared__ BnSmem sm;
    __shared__ __align__(128) float sz[BN_CTA];
    __shared__ __align__(128) float sc[BN_CTA];
    __shared__ __align__(8) uint64_t bar;
    const int W = a.W, H = a.H;
    const int HW = H * W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.y;
    const int slot = a.slots[j];
    const int pc = blockIdx.x * BN_CTA;             // first pixel of the region
    const int np = min(BN_CTA, HW - pc);             // pixels in the region
    const float* dsrc = a.depth + (size_t)slot * HW + pc;
    const float* csrc = a.conf + (size_t)slot * HW + pc;
    const bool bulk = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.depth) | reinterpret_cast<uintptr_t>(a.conf)) &
                                          15) == 0;
    if (bulk && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bn_smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bn_smem_u32(&bar)),
                     "r"((uint32_t)(8 * np))
                     : "memory");
        bn_bulk_load(sz, dsrc, 4u * np, &bar);
        bn_bulk_load(sc, csrc, 4u * np, &bar);
    }
    WarpCache& wc = sm.wc[warp];
    for (int i = lane; i < BN_WC; i += 32) wc.ckey[i] = kEmpty;
    if (threadIdx.x < 4) sm.cnt[threadIdx.x] = 0ull;
    const float4* tab = a.ftab + (size_t)j * (W + H + 1);
    for (int u = threadIdx.x; u < W; u += BN_NT) sA[u] = __ldg(tab + u);
    const float4 Tm = __ldg(tab + W + H);
    if (!bulk)
        for (int i = threadIdx.x; i < np; i += BN_NT) { sz[i] = __ldcs(dsrc + i); sc[i] = __ldcs(csrc + i); }
    __syncthreads();
    if (bulk) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(bn_smem_u32(&bar))
            : "memory");
    }
    const uint32_t span_entry0 = o.entry0 + (uint32_t)(blockIdx.y * gridDim.x + blockIdx.x) * BN_CTA +
                                 (uint32_t)warp * BN_SPAN;
    const int q0 = warp * BN_SPAN;  // span start within the region
    unsigned n_in = 0, n_oor = 0, n_slow = 0, n_drop = 0;
    SpanState s{kEmpty, 0u, 0u};
    if (q0 < np) {
        int q = q0 + lane;
        int v = (pc + q) / W, u = (pc + q) - v * W;
        unsigned long long* pay_span = o.pay + span_entry0;
        uint32_t* hr = sm.hrec[warp];
#pragma unroll 2
        for (int k = 0; k < BN_SPAN / 32; ++k) {
            const bool in = q < np;
            const float z = in ? sz[q] : 0.f, c = in ? sc[q] : 0.f;
            int cx = 0, cy = 0, cz = 0;
            float fx = 0.f, fy = 0.f, fz = 0.f;
            bool valid = false;
            if (in) valid = pixel_cell(a, sA[u], __ldg(tab + W + v), Tm, slot, u, v, z, c, cx, cy, cz, fx, fy, fz,
                                       n_in, n_oor, n_slow);
            const unsigned long long bk = pack_block(cx >> 3, cy >> 3, cz >> 3);
            span_slice(o.tab, wc, valid, bk, bn_payload(cx, cy, cz, fx, fy, fz, c), pay_span, hr, s);
            q += 32;
            u += 32;
            while (u >= W) { u -= W; ++v; }
        }
        n_drop = span_finish(o, hr, s, span_entry0);
    } else if (lane == 0) {
        o.span_nh[span_entry0 / BN_SPAN] = 0u;
    }
    bn_flush_counters(sm, o, n_in, n_oor, n_drop, n_slow);
}

// Explicit float64 points under one Sim(3) (exact transform): warp spans of
// BN_SPAN consecutive points.
__global__ void __launch_bounds__(BN_NT) bn_bin_points_kernel(const double* __restrict__ pts,
                                                              const double* __restrict__ conf, int64_t n, Sim3Arg g,
                                                              double cell, BnOut o) {
    __shared__ BnSmem sm;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpCache& wc = sm.wc[warp];
    for (int i = lane; i < BN_WC; i += 32) wc.ckey[i] = kEmpty;
    if (threadIdx.x < 4) sm.cnt[threadIdx.x] = 0ull;
    __syncthreads();
    const uint32_t span_entry0 = o.entry0 + (uint32_t)blockIdx.x * BN_CTA + (uint32_t)warp * BN_SPAN;
    const int64_t p0 = (int64_t)blockIdx.x * BN_CTA + warp * BN_SPAN;
    unsigned n_in = 0, n_oor = 0, n_drop = 0;
    SpanState s{kEmpty, 0u, 0u};
    if (p0 < n) {
        uint32_t* hr = sm.hrec[warp];
        for (int k = 0; k < BN_SPAN / 32; ++k) {
            const int64_t i = p0 + 32 * k + lane;
            bool valid = false;
            unsigned long long bk = kEmpty, pv = 0ull;
            if (i < n) {
                const double c = conf[i];
                if (c > 0) {
                    ++n_in;
                    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
                    double x[3];
                    sim3_apply_exact(g.v, p, x);
                    long long cc[3];
#pragma unroll
                    for (int q = 0; q < 3; ++q) cc[q] = (long long)floor(__ddiv_rn(x[q], cell));
                    if (cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2])) {
                        valid = true;
                        bk = pack_block((int)(cc[0] >> 3), (int)(cc[1] >> 3), (int)(cc[2] >> 3));
                        pv = bn_payload((int)cc[0], (int)cc[1], (int)cc[2], (float)((x[0] - (double)cc[0] * cell) / cell),
                                        (float)((x[1] - (double)cc[1] * cell) / cell),
                                        (float)((x[2] - (double)cc[2] * cell) / cell), (float)c);
                    } else {
                        ++n_oor;
                    }
                }
            }
            span_slice(o.tab, wc, valid, bk, pv, o.pay + span_entry0, hr, s);
        }
        n_drop = span_finish(o, hr, s, span_entry0);
    } else if (lane == 0) {
        o.span_nh[span_entry0 / BN_SPAN] = 0u;
    }
    bn_flush_counters(sm, o, n_in, n_oor, n_drop, 0u);
}

// ---------------------------------------------------------------------------
// 2. run records by bin (counting sort: offsets from a scan of bin_nrun)

__global__ void bn_run_scatter_kernel(const uint32_t* __restrict__ span_nh, int64_t n_spans,
                                      const uint2* __restrict__ runs, const uint32_t* __restrict__ run_off,
                                      uint32_t* __restrict__ cursor, uint2* __restrict__ sorted) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sp = w0; sp < n_spans; sp += nw) {
        const uint32_t nh = span_nh[sp];
        const uint2* r = runs + sp * BN_SPAN;
        for (uint32_t i = lane; i < nh; i += 32) {
            const uint2 rec = r[i];
            if (rec.y == BN_DROP) continue;
            const uint32_t id = rec.y >> BN_LENB;
            sorted[run_off[id] + atomicAdd(&cursor[id], 1u)] = rec;
        }
    }
}

// ---------------------------------------------------------------------------
// 3. per-bin aggregation

struct Sums5 {
    unsigned long long c, x, y, z;
    uint32_t n;
};
struct Sums5Add {
    __device__ __forceinline__ Sums5 operator()(const Sums5& a, const Sums5& b) const {
        return Sums5{a.c + b.c, a.x + b.x, a.y + b.y, a.z + b.z, a.n + b.n};
    }
};

__device__ __forceinline__ Sums5 bn_values(unsigned long long k) {
    if (k == ~0ull) return Sums5{0ull, 0ull, 0ull, 0ull, 0u};
    const float c = __uint_as_float(((uint32_t)(k >> 24) & 0x3FFFFFFFu) << 1);
    const unsigned long long cf = __float2ull_rn(c * kConfScale);
    return Sums5{cf, cf * (2u * ((uint32_t)(k >> 16) & 255u) + 1u), cf * (2u * ((uint32_t)(k >> 8) & 255u) + 1u),
                 cf * (2u * ((uint32_t)k & 255u) + 1u), 1u};
}

struct AgArgs {
    const unsigned long long* bin_keys;
    const uint32_t* run_off;
    const uint2* sorted;
    const unsigned long long* pay;
    double cell;
    int64_t max_voxels, max_bins;
    unsigned long long* ctr;
    unsigned long long* st_key;
    float4* st_sum;
    int32_t* st_cnt;
    uint32_t* st_tag;
    uint8_t* colcnt;
};

__global__ void __launch_bounds__(AG_NT, 2) bn_aggregate_kernel(AgArgs g) {
    typedef cub::BlockRadixSort<unsigned long long, AG_NT, AG_IPT, cub::NullType, 5> Sort;
    typedef cub::BlockScan<Sums5, AG_NT> Scan5;
    typedef cub::BlockScan<uint32_t, AG_NT> ScanU;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename Scan5::TempStorage scan5;
        typename ScanU::TempStorage scanu;
    } tmp;
    __shared__ unsigned long long acc[4][BN_SBV];
    __shared__ uint32_t cnt[BN_SBV];
    __shared__ uint32_t ex[BN_SBV + 1];
    __shared__ uint32_t rs[AG_NT];
    __shared__ uint32_t rx[AG_NT];
    __shared__ uint8_t ridx[AG_CH];
    __shared__ uint32_t last_idx[AG_NT], first_idx[AG_NT];
    __shared__ int bin_s;
    __shared__ uint32_t P_s;
    __shared__ unsigned long long base_s;
    const int t = threadIdx.x;
    const int64_t n_bins = min((int64_t)g.ctr[C_BINS], g.max_bins);
    const double k_len = g.cell * kConfInv / 512.0;  // fixed-point offset sums -> metres
    for (;;) {
        if (t == 0) bin_s = (int)atomicAdd(&g.ctr[C_WORK], 1ull);
        for (int i = t; i < BN_SBV; i += AG_NT) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q][i] = 0ull;
            cnt[i] = 0u;
        }
        __syncthreads();
        const int b = bin_s;
        if (b >= n_bins) break;
        uint32_t r0 = g.run_off[b];
        const uint32_t r1 = g.run_off[b + 1];
        while (r0 < r1) {
            // chunk: the longest prefix of the remaining runs with <= AG_CH points
            const bool has = r0 + (uint32_t)t < r1;
            uint2 rec = make_uint2(0u, 0u);
            if (has) rec = g.sorted[r0 + t];
            const uint32_t len = has ? (rec.y & ((1u << BN_LENB) - 1u)) : 0u;
            uint32_t incl;
            ScanU(tmp.scanu).InclusiveSum(len, incl);
            const bool take = has && incl <= (uint32_t)AG_CH;
            const int n_take = __syncthreads_count(take);
            if (take) {
                rs[t] = rec.x;
                rx[t] = incl - len;
                for (uint32_t q = 0; q < len; ++q) ridx[incl - len + q] = (uint8_t)t;
            }
            if (t == n_take - 1) P_s = incl;
            __syncthreads();
            const uint32_t P = P_s;
            unsigned long long keys[AG_IPT];
#pragma unroll
            for (int i = 0; i < AG_IPT; ++i) {
                const uint32_t f = (uint32_t)(i * AG_NT + t);
                keys[i] = ~0ull;
                if (f < P) {
                    const int r = ridx[f];
                    keys[i] = __ldcs(g.pay + rs[r] + (f - rx[r]));
                }
            }
            Sort(tmp.sort).Sort(keys, 54, 64);  // blocked: thread t holds sorted items t*IPT .. +IPT-1
            // voxel index per item (0xFFFF: padding, which sorts last); the
            // neighbours across thread boundaries through shared memory
            uint32_t idx[AG_IPT];
#pragma unroll
            for (int i = 0; i < AG_IPT; ++i) idx[i] = keys[i] == ~0ull ? 0xFFFFu : (uint32_t)(keys[i] >> 55);
            last_idx[t] = idx[AG_IPT - 1];
            first_idx[t] = idx[0];
            Sums5 tot{0ull, 0ull, 0ull, 0ull, 0u};
#pragma unroll
            for (int i = 0; i < AG_IPT; ++i) tot = Sums5Add()(tot, bn_values(keys[i]));
            __syncthreads();  // sort storage free; last / first indices visible
            Sums5 run;
            Scan5(tmp.scan5).ExclusiveScan(tot, run, Sums5{0ull, 0ull, 0ull, 0ull, 0u}, Sums5Add());
            const uint32_t before = t > 0 ? last_idx[t - 1] : 0xFFFFFFFFu;
            const uint32_t after = t + 1 < AG_NT ? first_idx[t + 1] : 0xFFFFFFFFu;
            // a voxel's run total is (inclusive prefix at its tail) - (exclusive
            // prefix at its head): heads subtract, then tails add (one writer
            // per voxel and phase; unsigned wrap-around keeps it exact)
            {
                Sums5 r = run;
                uint32_t p = before;
#pragma unroll
                for (int i = 0; i < AG_IPT; ++i) {
                    const uint32_t l = idx[i];
                    if (l != 0xFFFFu && l != p) {
                        acc[0][l] -= r.c; acc[1][l] -= r.x; acc[2][l] -= r.y; acc[3][l] -= r.z; cnt[l] -= r.n;
                    }
                    r = Sums5Add()(r, bn_values(keys[i]));
                    p = l;
                }
            }
            __syncthreads();
            {
                Sums5 r = run;
#pragma unroll
                for (int i = 0; i < AG_IPT; ++i) {
                    r = Sums5Add()(r, bn_values(keys[i]));
                    const uint32_t l = idx[i];
                    const uint32_t nx = i + 1 < AG_IPT ? idx[i + 1] : after;
                    if (l != 0xFFFFu && l != nx) {
                        acc[0][l] += r.c; acc[1][l] += r.x; acc[2][l] += r.y; acc[3][l] += r.z; cnt[l] += r.n;
                    }
                }
            }
            __syncthreads();
            r0 += (uint32_t)n_take;
        }
        // occupied voxels in in-bin order (x major): exclusive positions
        const int l0 = 2 * t;
        uint32_t f[2] = {cnt[l0] ? 1u : 0u, cnt[l0 + 1] ? 1u : 0u};
        uint32_t e[2], total;
        {
            typedef cub::BlockScan<uint32_t, AG_NT> BS2;
            BS2(tmp.scanu).ExclusiveSum(f, e, total);
        }
        ex[l0] = e[0];
        ex[l0 + 1] = e[1];
        if (t == 0) {
            ex[BN_SBV] = total;
            base_s = atomicAdd(&g.ctr[C_VOX], (unsigned long long)total);
        }
        __syncthreads();
        const unsigned long long base = base_s;
        const long long room = g.max_voxels - (long long)base;
        const uint32_t kept = room <= 0 ? 0u : (room < (long long)total ? (uint32_t)room : total);
        if (t == 0 && kept < total) atomicAdd(&g.ctr[C_VOX_OVF], (unsigned long long)(total - kept));
        if (t < 64) {
            // column (x, y) of the bin: voxels 8*col .. 8*col+7 (z ascending)
            const uint32_t a0 = min(ex[8 * t], kept), a1 = min(ex[8 * t + 8], kept);
            g.colcnt[(size_t)b * 64 + t] = (uint8_t)(a1 - a0);
        }
        long long bx, by, bz;
        unpack_cells(g.bin_keys[b], bx, by, bz);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int l = l0 + h;
            if (!f[h] || e[h] >= kept) continue;
            const unsigned long long o = base + e[h];
            const long long cx = 8 * bx + (l >> 6), cy = 8 * by + ((l >> 3) & 7), cz = 8 * bz + (l & 7);
            g.st_key[o] = pack_cells(cx, cy, cz);
            g.st_sum[o] = make_float4((float)((double)acc[1][l] * k_len), (float)((double)acc[2][l] * k_len),
                                      (float)((double)acc[3][l] * k_len), (float)((double)acc[0][l] * kConfInv));
            g.st_cnt[o] = (int32_t)cnt[l];
            g.st_tag[o] = ((uint32_t)b << 9) | ((uint32_t)(l >> 3) << 3) | (e[h] - ex[l & ~7]);
        }
        __syncthreads();  // acc / cnt / ex reuse by the next bin
    }
}

// ---------------------------------------------------------------------------
// 4. ordered emit

__device__ __forceinline__ int lower_bound_u64(const unsigned long long* a, int n, unsigned long long v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void bf_iota_kernel(uint32_t* v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

__global__ void bf_groups_kernel(const unsigned long long* __restrict__ skeys, const uint32_t* __restrict__ sids,
                                 int n, BinGroup* __restrict__ grp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = skeys[i];
    const unsigned long long x = k >> 42, xy = k >> 21;
    const int sx = lower_bound_u64(skeys, n, x << 42), ex_ = lower_bound_u64(skeys, n, (x + 1) << 42);
    const int sxy = lower_bound_u64(skeys, n, xy << 21), exy = lower_bound_u64(skeys, n, (xy + 1) << 21);
    grp[sids[i]] = BinGroup{sx, ex_ - sx, sxy - sx, exy - sxy, i - sxy, 0};
}

__device__ __forceinline__ int64_t col_pos(const BinGroup& g, int col) {
    const int lx = col >> 3, ly = col & 7;
    return (int64_t)g.start_x * 64 + (int64_t)lx * 8 * g.n_x + (int64_t)g.off_xy * 8 + (int64_t)ly * g.n_xy + g.r_z;
}

__global__ void bf_colpos_kernel(const BinGroup* __restrict__ grp, const uint8_t* __restrict__ colcnt, int n,
                                 uint32_t* __restrict__ scan_in) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * 64) return;
    const int b = (int)(t >> 6), col = (int)(t & 63);
    scan_in[col_pos(grp[b], col)] = colcnt[t];
}

__global__ void bf_permute_kernel(const unsigned long long* __restrict__ ctr, int64_t max_voxels,
                                  const BinGroup* __restrict__ grp, const uint32_t* __restrict__ col_base,
                                  const unsigned long long* __restrict__ st_key, const float4* __restrict__ st_sum,
                                  const int32_t* __restrict__ st_cnt, const uint32_t* __restrict__ st_tag, double cell,
                                  int64_t* __restrict__ keys, float* __restrict__ cen, float* __restrict__ wsum,
                                  int32_t* __restrict__ count, int64_t* __restrict__ n_out) {
    const int64_t U = min((int64_t)ctr[C_VOX], max_voxels);
    if (blockIdx.x == 0 && threadIdx.x == 0 && n_out) *n_out = U;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < U; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t tag = st_tag[i];
        const int b = (int)(tag >> 9), col = (int)((tag >> 3) & 63);
        const int64_t d = (int64_t)col_base[col_pos(grp[b], col)] + (tag & 7);
        const unsigned long long k = st_key[i];
        const float4 s = st_sum[i];
        long long cx, cy, cz;
        unpack_cells(k, cx, cy, cz);
        const double w = s.w;
        keys[d] = (int64_t)k;
        cen[3 * d + 0] = (float)((double)cx * cell + (double)s.x / w);
        cen[3 * d + 1] = (float)((double)cy * cell + (double)s.y / w);
        cen[3 * d + 2] = (float)((double)cz * cell + (double)s.z / w);
        wsum[d] = s.w;
        count[d] = st_cnt[i];
    }
}

// owner = mix64(key) % n_ranks (dist.owner_of)
__global__ void bf_owner_count_kernel(const unsigned long long* __restrict__ keys, const unsigned long long* ctr,
                                      int64_t max_voxels, int n_ranks, unsigned long long* __restrict__ rank_counts) {
    __shared__ unsigned int hist[64];
    for (int r = threadIdx.x; r < n_ranks; r += blockDim.x) hist[r] = 0u;
    __syncthreads();
    const int64_t n = min((int64_t)ctr[C_VOX], max_voxels);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[mix64(keys[i]) % (unsigned long long)n_ranks], 1u);
    __syncthreads();
    for (int r = threadIdx.x; r < n_ranks; r += blockDim.x)
        if (hist[r]) atomicAdd(&rank_counts[r], (unsigned long long)hist[r]);
}

__global__ void bf_owner_write_kernel(const unsigned long long* __restrict__ skeys, const float4* __restrict__ ssum,
                                      const int32_t* __restrict__ scnt, const unsigned long long* ctr,
                                      int64_t max_voxels, int n_ranks, const unsigned long long* __restrict__ rank_base,
                                      unsigned long long* __restrict__ cursors, int64_t* __restrict__ okeys,
                                      float* __restrict__ sums4, int32_t* __restrict__ cnt) {
    const int64_t n = min((int64_t)ctr[C_VOX], max_voxels);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = skeys[i];
        const int r = (int)(mix64(k) % (unsigned long long)n_ranks);
        const unsigned peers = __match_any_sync(__activemask(), r);
        const int lead = __ffs(peers) - 1;
        const unsigned below = peers & ((1u << (threadIdx.x & 31)) - 1u);
        unsigned long long base = 0;
        if ((int)(threadIdx.x & 31) == lead) base = atomicAdd(&cursors[r], (unsigned long long)__popc(peers));
        base = __shfl_sync(peers, base, lead);
        const unsigned long long o = rank_base[r] + base + __popc(below);
        okeys[o] = (int64_t)k;
        reinterpret_cast<float4*>(sums4)[o] = ssum[i];
        cnt[o] = scnt[i];
    }
}

// ---------------------------------------------------------------------------
// clearing

__global__ void bf_clear_table_kernel(BinEntry* __restrict__ t, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        BinEntry e;
        e.key = kEmpty;
        e.id = -1;
        e.pad = 0;
        t[i] = e;
    }
}

__global__ void bf_clear_used_kernel(BinEntry* __restrict__ table, int64_t tcap, const uint32_t* __restrict__ bin_slot,
                                     uint32_t* __restrict__ bin_nrun, const unsigned long long* __restrict__ ctr,
                                     int64_t max_bins) {
    const unsigned long long used_raw = ctr[C_BINS];
    const bool full = (int64_t)used_raw > max_bins;
    const int64_t used = full ? max_bins : (int64_t)used_raw;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    BinEntry empty;
    empty.key = kEmpty;
    empty.id = -1;
    empty.pad = 0;
    const int64_t n_tab = full ? tcap : used;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_tab; i += stride)
        table[full ? i : (int64_t)bin_slot[i]] = empty;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < used; i += stride) bin_nrun[i] = 0u;
}

// ---------------------------------------------------------------------------
// host side

static BinTab tab_of(const BinFuse* b) {
    return BinTab{b->table, b->tmask, b->bin_keys, b->bin_slot, b->ctr, b->max_bins};
}

BinFuse* bf_create(int64_t max_voxels, int64_t max_bins, double cell, cudaStream_t st, int* rc) {
    BinFuse* b = new BinFuse();
    b->max_voxels = max_voxels;
    // st_tag holds bin << 9, run records bin << BN_LENB: 22-bit bin ids
    b->max_bins = std::min<int64_t>(std::max<int64_t>(max_bins, 8192), (1 << 22) - 2);
    b->cell = cell;
    int64_t tcap = 1;
    while (tcap < 4 * b->max_bins) tcap <<= 1;
    b->tmask = (unsigned long long)(tcap - 1);
    bool ok = cudaMalloc(&b->table, sizeof(BinEntry) * (size_t)tcap) == cudaSuccess &&
              cudaMalloc(&b->bin_keys, sizeof(unsigned long long) * (size_t)b->max_bins) == cudaSuccess &&
              cudaMalloc(&b->bin_slot, sizeof(uint32_t) * (size_t)b->max_bins) == cudaSuccess &&
              cudaMalloc(&b->bin_nrun, sizeof(uint32_t) * (size_t)(b->max_bins + 1)) == cudaSuccess &&
              cudaMalloc(&b->ctr, sizeof(unsigned long long) * 16) == cudaSuccess;
    if (!ok) {
        set_last_error("cudaMalloc(binned fusion)", cudaGetLastError());
        bf_destroy(b);
        *rc = EC3R_ENOMEM;
        return nullptr;
    }
    cudaMemsetAsync(b->bin_nrun, 0, sizeof(uint32_t) * (size_t)(b->max_bins + 1), st);
    cudaMemsetAsync(b->ctr, 0, sizeof(unsigned long long) * 16, st);
    bf_clear_table_kernel<<<(unsigned)((tcap + 255) / 256), 256, 0, st>>>(b->table, tcap);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) {
        bf_destroy(b);
        *rc = EC3R_ECUDA;
        return nullptr;
    }
    *rc = EC3R_OK;
    return b;
}

void bf_destroy(BinFuse* b) {
    if (!b) return;
    cudaFree(b->table);
    cudaFree(b->bin_keys);
    cudaFree(b->bin_slot);
    cudaFree(b->bin_nrun);
    cudaFree(b->ctr);
    cudaFree(b->pay);
    cudaFree(b->runs);
    cudaFree(b->span_nh);
    cudaFree(b->ws);
    delete b;
}

int bf_clear(BinFuse* b, cudaStream_t st) {
    bf_clear_used_kernel<<<kNumSMs * 4, 256, 0, st>>>(b->table, (int64_t)b->tmask + 1, b->bin_slot, b->bin_nrun,
                                                      b->ctr, b->max_bins);
    EC3R_CHECK_LAUNCH("bf_clear_used_kernel");
    EC3R_CUDA_TRY(cudaMemsetAsync(b->ctr, 0, sizeof(unsigned long long) * 16, st));
    b->used = 0;
    b->dirty = true;
    return EC3R_OK;
}

// room for `entries` more payload entries (a multiple of BN_CTA)
static int bf_reserve(BinFuse* b, int64_t entries, cudaStream_t st) {
    if (b->used + entries > (int64_t)0xFFFFFFFFll) {
        set_last_error_msg("binned fusion: more than 2^32 points in one map");
        return EC3R_EARG;
    }
    if (b->used + entries > b->cap) {
        const int64_t cap = std::max<int64_t>(b->used + entries, b->cap + b->cap / 2);
        unsigned long long* pay = nullptr;
        uint2* runs = nullptr;
        uint32_t* nh = nullptr;
        if (cudaMalloc(&pay, sizeof(unsigned long long) * (size_t)cap) != cudaSuccess ||
            cudaMalloc(&runs, sizeof(uint2) * (size_t)cap) != cudaSuccess ||
            cudaMalloc(&nh, sizeof(uint32_t) * (size_t)(cap / BN_SPAN + 1)) != cudaSuccess) {
            cudaFree(pay);
            cudaFree(runs);
            set_last_error("cudaMalloc(binned fusion payload)", cudaGetLastError());
            return EC3R_ENOMEM;
        }
        if (b->used) {
            EC3R_CUDA_TRY(cudaMemcpyAsync(pay, b->pay, sizeof(unsigned long long) * (size_t)b->used,
                                          cudaMemcpyDeviceToDevice, st));
            EC3R_CUDA_TRY(cudaMemcpyAsync(runs, b->runs, sizeof(uint2) * (size_t)b->used, cudaMemcpyDeviceToDevice,
                                          st));
            EC3R_CUDA_TRY(cudaMemcpyAsync(nh, b->span_nh, sizeof(uint32_t) * (size_t)(b->used / BN_SPAN),
                                          cudaMemcpyDeviceToDevice, st));
            EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        }
        cudaFree(b->pay);
        cudaFree(b->runs);
        cudaFree(b->span_nh);
        b->pay = pay;
        b->runs = runs;
        b->span_nh = nh;
        b->cap = cap;
    }
    return EC3R_OK;
}

static BnOut out_of(BinFuse* b) {
    BnOut o;
    o.tab = tab_of(b);
    o.bin_nrun = b->bin_nrun;
    o.pay = b->pay;
    o.runs = b->runs;
    o.span_nh = b->span_nh;
    o.ctr = b->ctr;
    o.entry0 = (uint32_t)b->used;
    return o;
}

int bf_insert_frames(BinFuse* b, const FrameGeom& g, cudaStream_t st) {
    const int64_t HW = (int64_t)g.H * g.W;
    const int per_frame = (int)((HW + BN_CTA - 1) / BN_CTA);
    const int64_t n_cta = (int64_t)per_frame * g.n;
    int rc = bf_reserve(b, n_cta * BN_CTA, st);
    if (rc) return rc;
    const BnOut o = out_of(b);
    const size_t smem = sizeof(float4) * (size_t)g.W;
    if (smem > 64 * 1024) {
        set_last_error_msg("binned fusion: image wider than 4096 px");
        return EC3R_EARG;
    }
    static bool attr = false;
    if (!attr) {
        EC3R_CUDA_TRY(cudaFuncSetAttribute(bn_bin_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           64 * 1024));
        attr = true;
    }
    KernelTimer tk(TK_FUSE_INSERT, st);
    bn_bin_frames_kernel<<<dim3(per_frame, g.n), BN_NT, smem, st>>>(g, o);
    EC3R_CHECK_LAUNCH("bn_bin_frames_kernel");
    tk.stop();
    b->used += n_cta * BN_CTA;
    b->dirty = true;
    return EC3R_OK;
}

int bf_insert_points(BinFuse* b, const double* pts, const double* conf, int64_t n, const double* sim3_h,
                     cudaStream_t st) {
    const int64_t n_cta = (n + BN_CTA - 1) / BN_CTA;
    int rc = bf_reserve(b, n_cta * BN_CTA, st);
    if (rc) return rc;
    const BnOut o = out_of(b);
    Sim3Arg g;
    for (int k = 0; k < 8; ++k) g.v[k] = sim3_h[k];
    bn_bin_points_kernel<<<(unsigned)n_cta, BN_NT, 0, st>>>(pts, conf, n, g, b->cell, o);
    EC3R_CHECK_LAUNCH("bn_bin_points_kernel");
    b->used += n_cta * BN_CTA;
    b->dirty = true;
    return EC3R_OK;
}

int bf_stats(BinFuse* b, int64_t out[5], cudaStream_t st) {
    unsigned long long c[16];
    EC3R_CUDA_TRY(cudaMemcpyAsync(c, b->ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    out[0] = (int64_t)c[C_IN];
    out[1] = (int64_t)c[C_OOR];
    out[2] = (int64_t)(c[C_OVF] + c[C_VOX_OVF]);
    out[3] = (int64_t)c[C_SLOW];
    out[4] = (int64_t)std::min<unsigned long long>(c[C_BINS], (unsigned long long)b->max_bins);
    if (getenv("EC3R_DEBUG_BINS"))
        fprintf(stderr, "[vbin] points %llu bins %llu runs %llu (%.2f points/run) voxels %llu\n", c[C_IN], c[C_BINS],
                c[C_RUNS], c[C_RUNS] ? (double)c[C_IN] / (double)c[C_RUNS] : 0.0, c[C_VOX]);
    return EC3R_OK;
}

static size_t bf_ws_layout(BinFuse* b, int64_t n_runs_cap, BfWs* w) {
    const int64_t nb = b->max_bins;
    size_t cub1 = 0, cub2 = 0, cub3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub1, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(nb + 1));
    cub::DeviceRadixSort::SortPairs(nullptr, cub2, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)nb, 0, 63);
    cub::DeviceScan::ExclusiveSum(nullptr, cub3, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(nb * 64));
    const size_t cubb = std::max(cub1, std::max(cub2, cub3));
    Carver cv{w ? b->ws : nullptr, 0};
    const size_t V = (size_t)b->max_voxels;
    BfWs t;
    t.run_off = cv.take<uint32_t>(nb + 1);
    t.cursor = cv.take<uint32_t>(nb + 1);
    t.sorted = cv.take<uint2>(std::max<int64_t>(n_runs_cap, 1));
    t.st_key = cv.take<unsigned long long>(V);
    t.st_sum = cv.take<float4>(V);
    t.st_cnt = cv.take<int32_t>(V);
    t.st_tag = cv.take<uint32_t>(V);
    t.colcnt = cv.take<uint8_t>(nb * 64 + 64);
    t.skeys = cv.take<unsigned long long>(nb + 1);
    t.ids = cv.take<uint32_t>(nb + 1);
    t.sids = cv.take<uint32_t>(nb + 1);
    t.grp = cv.take<BinGroup>(nb + 1);
    t.scan_in = cv.take<uint32_t>(nb * 64 + 1);
    t.col_base = cv.take<uint32_t>(nb * 64 + 1);
    t.cub_tmp = cv.take<char>(cubb);
    t.cub_bytes = cubb;
    if (w) *w = t;
    return cv.used;
}

// Aggregation (phase A): run records -> per-bin voxels in staging.  No host
// round trip: every launch is sized by the map's capacities and reads the
// live counts on the device.
static int bf_aggregate(BinFuse* b, BfWs* w, cudaStream_t st) {
    // run records <= entries used (one per point at most)
    const size_t need = bf_ws_layout(b, b->used, nullptr);
    if (need > b->ws_cap) {
        EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(b->ws);
        b->ws = nullptr;
        b->ws_cap = 0;
        const size_t cap = need + need / 4;
        if (cudaMalloc(&b->ws, cap) != cudaSuccess) {
            set_last_error("cudaMalloc(binned fusion workspace)", cudaGetLastError());
            return EC3R_ENOMEM;
        }
        b->ws_cap = cap;
    }
    bf_ws_layout(b, b->used, &b->view);
    *w = b->view;
    const int64_t nb = b->max_bins;
    EC3R_CUDA_TRY(cudaMemsetAsync(b->ctr + C_VOX, 0, sizeof(unsigned long long) * 3, st));  // VOX, VOX_OVF, WORK
    size_t tb = w->cub_bytes;
    if (cub::DeviceScan::ExclusiveSum(w->cub_tmp, tb, b->bin_nrun, w->run_off, (int)(nb + 1), st) != cudaSuccess) {
        set_last_error("cub::DeviceScan::ExclusiveSum(bins)", cudaGetLastError());
        return EC3R_ECUDA;
    }
    count_launch();
    EC3R_CUDA_TRY(cudaMemsetAsync(w->cursor, 0, sizeof(uint32_t) * (size_t)nb, st));
    const int64_t n_spans = b->used / BN_SPAN;
    if (n_spans > 0) {
        bn_run_scatter_kernel<<<(unsigned)std::min<int64_t>((n_spans + 7) / 8, (int64_t)kNumSMs * 16), 256, 0, st>>>(
            b->span_nh, n_spans, b->runs, w->run_off, w->cursor, w->sorted);
        EC3R_CHECK_LAUNCH("bn_run_scatter_kernel");
    }
    AgArgs g;
    g.bin_keys = b->bin_keys;
    g.run_off = w->run_off;
    g.sorted = w->sorted;
    g.pay = b->pay;
    g.cell = b->cell;
    g.max_voxels = b->max_voxels;
    g.max_bins = b->max_bins;
    g.ctr = b->ctr;
    g.st_key = w->st_key;
    g.st_sum = w->st_sum;
    g.st_cnt = w->st_cnt;
    g.st_tag = w->st_tag;
    g.colcnt = w->colcnt;
    static int ag_ctas = 0;
    if (!ag_ctas) {
        int per_sm = 0;
        EC3R_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bn_aggregate_kernel, AG_NT, 0));
        ag_ctas = kNumSMs * std::max(per_sm, 1);
    }
    bn_aggregate_kernel<<<(unsigned)ag_ctas, AG_NT, 0, st>>>(g);
    EC3R_CHECK_LAUNCH("bn_aggregate_kernel");
    b->dirty = false;
    return EC3R_OK;
}

static int bf_ensure_aggregated(BinFuse* b, BfWs* w, cudaStream_t st) {
    if (b->dirty) return bf_aggregate(b, w, st);
    *w = b->view;
    return EC3R_OK;
}

int bf_count(BinFuse* b, int64_t* U, cudaStream_t st) {
    BfWs w;
    int rc = bf_ensure_aggregated(b, &w, st);
    if (rc) return rc;
    unsigned long long v = 0;
    EC3R_CUDA_TRY(cudaMemcpyAsync(&v, b->ctr + C_VOX, sizeof(v), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    *U = std::min<int64_t>((int64_t)v, b->max_voxels);
    return EC3R_OK;
}

int bf_extract(BinFuse* b, int64_t* keys, float* centroid, float* wsum, int32_t* count, int64_t* n_out,
               int64_t* U_host, cudaStream_t st) {
    BfWs w;
    int rc = bf_ensure_aggregated(b, &w, st);
    if (rc) return rc;
    // one round trip: the bin count sizes the emit launches
    unsigned long long c[16];
    EC3R_CUDA_TRY(cudaMemcpyAsync(c, b->ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t nb = std::min<int64_t>((int64_t)c[C_BINS], b->max_bins);
    b->n_bins = nb;
    if (nb > 0) {
        bf_iota_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(w.ids, (int)nb);
        EC3R_CHECK_LAUNCH("bf_iota_kernel");
        size_t tb = w.cub_bytes;
        if (cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, b->bin_keys, w.skeys, w.ids, w.sids, (int)nb, 0, 63, st) !=
            cudaSuccess) {
            set_last_error("cub::DeviceRadixSort::SortPairs(bins)", cudaGetLastError());
            return EC3R_ECUDA;
        }
        count_launch();
        bf_groups_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(w.skeys, w.sids, (int)nb, w.grp);
        EC3R_CHECK_LAUNCH("bf_groups_kernel");
        const int64_t ncol = nb * 64;
        bf_colpos_kernel<<<(unsigned)((ncol + 255) / 256), 256, 0, st>>>(w.grp, w.colcnt, (int)nb, w.scan_in);
        EC3R_CHECK_LAUNCH("bf_colpos_kernel");
        tb = w.cub_bytes;
        if (cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.scan_in, w.col_base, (int)ncol, st) != cudaSuccess) {
            set_last_error("cub::DeviceScan::ExclusiveSum(columns)", cudaGetLastError());
            return EC3R_ECUDA;
        }
        count_launch();
    }
    bf_permute_kernel<<<kNumSMs * 8, 256, 0, st>>>(b->ctr, b->max_voxels, w.grp, w.col_base, w.st_key, w.st_sum,
                                                  w.st_cnt, w.st_tag, b->cell, keys, centroid, wsum, count, n_out);
    EC3R_CHECK_LAUNCH("bf_permute_kernel");
    if (U_host) *U_host = std::min<int64_t>((int64_t)c[C_VOX], b->max_voxels);
    return EC3R_OK;
}

int bf_extract_partials(BinFuse* b, int n_ranks, int64_t* keys, float* sums4, int32_t* count, int64_t* rank_counts,
                        cudaStream_t st) {
    BfWs w;
    int rc = bf_ensure_aggregated(b, &w, st);
    if (rc) return rc;
    unsigned long long* base = nullptr;
    EC3R_CUDA_TRY(cudaMallocAsync((void**)&base, sizeof(unsigned long long) * 2 * n_ranks, st));
    unsigned long long* cursors = base + n_ranks;
    EC3R_CUDA_TRY(cudaMemsetAsync(rank_counts, 0, sizeof(int64_t) * n_ranks, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(cursors, 0, sizeof(unsigned long long) * n_ranks, st));
    bf_owner_count_kernel<<<kNumSMs * 8, 256, 0, st>>>(w.st_key, b->ctr, b->max_voxels, n_ranks,
                                                      (unsigned long long*)rank_counts);
    EC3R_CHECK_LAUNCH("bf_owner_count_kernel");
    std::vector<unsigned long long> rc_h(n_ranks), rb(n_ranks);
    EC3R_CUDA_TRY(cudaMemcpyAsync(rc_h.data(), rank_counts, sizeof(int64_t) * n_ranks, cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long acc = 0;
    for (int r = 0; r < n_ranks; ++r) { rb[r] = acc; acc += rc_h[r]; }
    EC3R_CUDA_TRY(cudaMemcpyAsync(base, rb.data(), sizeof(unsigned long long) * n_ranks, cudaMemcpyHostToDevice, st));
    bf_owner_write_kernel<<<kNumSMs * 8, 256, 0, st>>>(w.st_key, w.st_sum, w.st_cnt, b->ctr, b->max_voxels, n_ranks,
                                                      base, cursors, keys, sums4, count);
    EC3R_CHECK_LAUNCH("bf_owner_write_kernel");
    EC3R_CUDA_TRY(cudaFreeAsync(base, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));  // rb is a host temporary
    return EC3R_OK;
}

}  // namespace ec3r
