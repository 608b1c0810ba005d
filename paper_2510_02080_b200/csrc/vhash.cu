// K1+K4: Sim(3) transform + voxel-block hash fusion + downsample emit, on
// sm_100a.
//
// Replaces Submap.world_points / Mapping.fused_cloud (mapping.py:56-57,
// 332-338) under the declared fusion rule of oracle/fuse.py.  Keys are
// _pack(floor(x / cell)) (_kernels/_numpy.py:50-55) and must be bit-exact
// against the reference's float64 chain  x = G.apply(P_f.apply(ray))
// (backend.py:89-90, liegroups.py:90-95,208-209,259-260).
//
// Keys — fast path (every pixel): the composite G o P_f is folded per frame
// into a float32 affine map evaluated as x = z * (A[u] + B[v]) + T (per-column
// / per-row tables in shared memory): 3 FADD + 3 FFMA per pixel instead of
// ~70 float64 operations.  Its rounding error is bounded per pixel; when a
// coordinate lies within that bound of a voxel boundary the pixel re-runs
// the reference's exact float64 sequence (slow path), so keys are bit-exact
// by construction.
//
// Storage — voxel-block hash: voxels are grouped in 4x4x4 blocks; a small
// open-addressing table maps block keys to dense 64-voxel blocks of a pool
// (float4 sum of conf * (x - voxel corner) and conf, uint32 count).  Measured
// on this part (tools/atomics_probe.cu) random atomics run at ~180 G op/s
// when their targets sit in L2 and ~25-33 G op/s when they miss to HBM; dense
// blocks pack the voxels a few concurrently fused frames touch into ~tens of
// MB, so the update stream stays L2-resident, and the block table (a few MB)
// is looked up once per distinct block per warp (__match_any_sync).

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "fuse_common.cuh"
#include "vbin.cuh"

namespace ec3r {

constexpr int kBlockVox = 64;                 // 4 x 4 x 4

struct __align__(16) BlockEntry {
    unsigned long long key;  // packed block coordinates (cell >> 2)
    int idx;                 // pool block index; -1 while being published, -2 pool overflow
    int pad;
};

}  // namespace ec3r

struct ec3r_vhash {
    int64_t max_voxels;  // emit capacity
    int64_t max_blocks;
    unsigned long long tmask;
    double cell;
    ec3r::BlockEntry* table;
    unsigned long long* block_keys;  // max_blocks
    uint32_t* block_slot;            // max_blocks: table position of each allocated block
    float4* sums;                    // max_blocks * 64
    unsigned int* counts;            // max_blocks * 64
    unsigned long long* counters;    // [n_in, n_oor, n_overflow, n_slow, blocks_used, ...]
    float4* ftab;                    // per-frame affine tables of the last insert_frames
    int64_t ftab_cap;                // float4 entries
    int64_t last_count;              // voxels of the last sorted extract (host-known), -1 if unknown
    bool emit_key32;                 // the last read-back extent fit the emit's 32-bit block keys
    // binned super-block engine (vbin.cu, EC3R_FUSE_ENGINE=binned): frame and
    // point inserts go there; partial merges (multi-GPU owner maps) always use
    // the block hash.  A map holds one kind of content between clears.
    ec3r::BinFuse* bf;
    // reduction-floor diagnostic: the next insert_frames logs its runs here
    uint2* diag_runs;
    unsigned long long* diag_n;
    int64_t diag_cap;
    bool binned;
    bool bf_active, legacy_active;
};

namespace ec3r {

struct VB {
    BlockEntry* table;
    unsigned long long tmask;
    unsigned long long* block_keys;
    uint32_t* block_slot;
    float4* sums;
    unsigned int* counts;
    unsigned long long* counters;
    int64_t max_blocks;
};

static VB vb_of(const ec3r_vhash* h) {
    return VB{h->table, h->tmask, h->block_keys, h->block_slot, h->sums, h->counts, h->counters, h->max_blocks};
}

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ void red_add_u32(unsigned int* addr, uint32_t v) {
    asm volatile("red.global.add.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

// One 16-byte L2 read of a table entry {key, idx} (relaxed, gpu scope: the
// table is only written by this kernel's atomics, so L2 is the coherence
// point; a volatile access would compile to .STRONG.SYS and two round trips).
__device__ __forceinline__ void load_entry(const BlockEntry* e, unsigned long long& key, int& idx) {
    unsigned long long lo, hi;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(e) : "memory");
    key = lo;
    idx = (int)(unsigned)(hi & 0xFFFFFFFFull);
}

__device__ __forceinline__ int load_idx(const BlockEntry* e) {
    int idx;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(idx) : "l"(&e->idx) : "memory");
    return idx;
}

// Find or allocate the pool block of block key bk (one thread).  Returns the
// block index, or -2 when the pool or the table is full.
__device__ __noinline__ int vb_find_or_insert(const VB& v, unsigned long long bk) {
    unsigned long long h = table_slot(bk, v.tmask);
    for (unsigned long long probe = 0; probe <= v.tmask; ++probe) {
        BlockEntry* e = v.table + h;
        unsigned long long k;
        int idx;
        load_entry(e, k, idx);
        if (k == bk) {
            while (idx == -1) idx = load_idx(e);  // winner is publishing
            return idx;
        }
        if (k == kEmpty) {
            const unsigned long long prev = atomicCAS(&e->key, kEmpty, bk);
            if (prev == kEmpty) {
                // warp-aggregated allocation: the lanes that won a CAS together
                // share one atomic on the (single, contended) block counter
                cg::coalesced_group g = cg::coalesced_threads();
                unsigned long long base = 0;
                if (g.thread_rank() == 0) base = atomicAdd(&v.counters[4], (unsigned long long)g.size());
                const unsigned long long slot = g.shfl(base, 0) + g.thread_rank();
                int got = -2;
                if ((int64_t)slot < v.max_blocks) {
                    got = (int)slot;
                    v.block_keys[slot] = bk;  // read by later kernels only: no fence needed
                    v.block_slot[slot] = (uint32_t)h;
                }
                atomicExch(&e->idx, got);
                return got;
            }
            if (prev == bk) {
                int i2 = load_idx(e);
                while (i2 == -1) i2 = load_idx(e);
                return i2;
            }
        }
        h = (h + 1) & v.tmask;
    }
    return -2;
}

// Warp-cooperative insert: every lane of the warp calls it (valid = has a
// point).  Lanes sharing a block key elect one leader for the table lookup.
// Returns 1 when this lane's point was dropped (pool / table overflow).
// (cbk, cidx): the lane's last (block key, block index); consecutive points
// of a lane usually fall in the same 8 cm block and skip the table.
__device__ __forceinline__ unsigned vb_insert_warp(const VB& v, bool valid, long long cx, long long cy, long long cz,
                                                   float wx, float wy, float wz, float w, unsigned cnt,
                                                   unsigned long long& cbk, int& cidx) {
    const int lane = threadIdx.x & 31;
    const unsigned long long bk = valid ? pack_cells(cx >> 2, cy >> 2, cz >> 2) : kEmpty;
    const bool need = valid && bk != cbk;
    int idx = cidx;
    if (__any_sync(0xffffffffu, need)) {
        const unsigned peers = __match_any_sync(0xffffffffu, need ? bk : kEmpty);
        const int leader = __ffs(peers) - 1;
        int got = -2;
        if (need && lane == leader) got = vb_find_or_insert(v, bk);
        got = __shfl_sync(0xffffffffu, got, leader);
        if (need) {
            idx = got;
            cbk = bk;
            cidx = got;
        }
    }
    if (!valid) return 0u;
    if (idx < 0) return 1u;
    const int local = (int)(cx & 3) | ((int)(cy & 3) << 2) | ((int)(cz & 3) << 4);
    const size_t s = (size_t)idx * kBlockVox + local;
    red_add_v4(v.sums + s, wx, wy, wz, w);
    atomicAdd(v.counts + s, cnt);
    return 0u;
}

// ---------------------------------------------------------------------------
// clearing

__global__ void vb_clear_table_kernel(BlockEntry* __restrict__ t, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        BlockEntry e;
        e.key = kEmpty;
        e.idx = -1;
        e.pad = 0;
        t[i] = e;
    }
}

__global__ void vb_clear_used_kernel(BlockEntry* __restrict__ table, int64_t tcap, const uint32_t* __restrict__ block_slot,
                                     float4* __restrict__ sums, unsigned int* __restrict__ counts,
                                     const unsigned long long* __restrict__ counters, int64_t max_blocks) {
    const unsigned long long used_raw = counters[4];
    const bool full = (int64_t)used_raw > max_blocks;
    const int64_t used = full ? max_blocks : (int64_t)used_raw;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    BlockEntry empty;
    empty.key = kEmpty;
    empty.idx = -1;
    empty.pad = 0;
    const int64_t n_tab = full ? tcap : used;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_tab; i += stride)
        table[full ? i : (int64_t)block_slot[i]] = empty;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < used * kBlockVox; i += stride) {
        sums[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        counts[i] = 0u;
    }
}

// ---------------------------------------------------------------------------
// frame insertion

#ifndef EC3R_FI_NT
#define EC3R_FI_NT 256  // threads per insert CTA
#endif
constexpr int FI_NT = EC3R_FI_NT;
constexpr int kSmallCtaWaves = 6;  // 128-thread insert CTAs from this many waves of them (see the launch)
#ifndef EC3R_FI_ROWS
#define EC3R_FI_ROWS 64  // image rows per CTA
#endif
constexpr int FI_ROWS = EC3R_FI_ROWS;
#ifndef EC3R_FI_MINB
#define EC3R_FI_MINB 2  // resident CTAs per SM the register budget is sized for
#endif

struct FuseArgs : FrameGeom {
    VB vb;
    uint2* log_runs;                // LOG instance only (see RunLog)
    unsigned long long* log_n;
    unsigned long long log_cap;
};

// Per listed frame j, the composite G o P_f folded into a float32 affine map
// x = z * (A[u] + B[v]) + T: A[u] = M[:,0] x_u + M[:,2], B[v] = M[:,1] y_v,
// each with its |.|-sum in .w for the rounding bound; T = (t, |t|-sum).
__global__ void vh_frame_tables_kernel(FrameGeom a, float4* __restrict__ ftab) {
    const int j = blockIdx.x;
    const int slot = a.slots[j];
    const double* P = a.slot_poses + 8 * slot;
    const double* G = a.slot_globals + 8 * slot;
    double RG[3][3], RP[3][3], M[3][3], T[3];
    quat_to_mat(G + 1, RG);
    quat_to_mat(P + 1, RP);
    for (int i = 0; i < 3; ++i) {
        for (int k = 0; k < 3; ++k) M[i][k] = G[0] * (RG[i][0] * RP[0][k] + RG[i][1] * RP[1][k] + RG[i][2] * RP[2][k]);
        T[i] = G[0] * (RG[i][0] * P[5] + RG[i][1] * P[6] + RG[i][2] * P[7]) + G[5 + i];
    }
    float4* tab = ftab + (size_t)j * (a.W + a.H + 1);
    for (int u = threadIdx.x; u < a.W; u += blockDim.x) {
        const double x = ray_coef(u, a.cx, a.fx);
        const float ax = (float)(M[0][0] * x + M[0][2]), ay = (float)(M[1][0] * x + M[1][2]),
                    az = (float)(M[2][0] * x + M[2][2]);
        tab[u] = make_float4(ax, ay, az, fabsf(ax) + fabsf(ay) + fabsf(az));
    }
    for (int v = threadIdx.x; v < a.H; v += blockDim.x) {
        const double y = ray_coef(v, a.cy, a.fy);
        const float bx = (float)(M[0][1] * y), by = (float)(M[1][1] * y), bz = (float)(M[2][1] * y);
        tab[a.W + v] = make_float4(bx, by, bz, fabsf(bx) + fabsf(by) + fabsf(bz));
    }
    if (threadIdx.x == 0) {
        const float tx = (float)T[0], ty = (float)T[1], tz = (float)T[2];
        tab[a.W + a.H] = make_float4(tx, ty, tz, fabsf(tx) + fabsf(ty) + fabsf(tz));
    }
}

// Frame insertion.  Grid = (bands of FI_ROWS rows, listed frames); a CTA's
// warps take 8 x 16 pixel sub-tiles of its band (lane = 4 horizontally
// adjacent pixels) independently -- no CTA barriers in the loop.  A 2-D
// sub-tile touches ~13 distinct blocks where a 128-pixel row run touches ~36,
// so the per-warp block lookups (lane reuse, one leader per block per pixel
// slot, the 4 slots' first probes in flight together) drop ~3x.  The next
// sub-tile's depth / confidence are loaded before this one's lookups.
//
// Measured on the bench workload (72M points, tools/fuse_timing.py): keys +
// lookups alone run in ~0.9 ms; the two scattered reductions per point add
// ~0.9 ms.  Scattered 16 B + 4 B updates cost one L1 wavefront per lane
// (tools/atomics_probe3.cu: ~93 G point-updates/s for random voxels, up to
// ~300 G when a warp's lanes hit consecutive voxels), and the sweep order
// (frame-major ... all frames interleaved) and pool working set changed the
// time by < 10%, so the pool's L2 residency is not the limiter.
// Reduction-floor diagnostic (ec3r_vhash_diag_*): the insert's LOG
// instance writes every run's reduction target and count (vid, n) in issue
// order instead of reducing; exp_replay_kernel then issues exactly those
// reductions (constant conf-weighted payload, or the logged count), so the
// replay time is the cost of the kernel's own reduction stream without the
// keys, loads and lookups around it.
struct RunLog {
    uint2* runs;                    // (vid, n)
    unsigned long long* n;          // device counter
    unsigned long long cap;
};
__device__ __forceinline__ void log_run(const RunLog& lg, uint32_t vid, uint32_t n) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(lg.n, (unsigned long long)g.size());
    const unsigned long long i = g.shfl(base, 0) + g.thread_rank();
    if (i < lg.cap) lg.runs[i] = make_uint2(vid, n);
}
__global__ void vh_replay_runs_kernel(const uint2* __restrict__ runs, const unsigned long long* __restrict__ n_ptr,
                                      unsigned long long cap, float4* __restrict__ sums,
                                      unsigned int* __restrict__ counts, int with_count) {
    const unsigned long long n = min(*n_ptr, cap);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const uint2 v = __ldcs(runs + i);
        red_add_v4(sums + v.x, 1e-3f, 1e-3f, 1e-3f, 0.5f);
        if (with_count) red_add_u32(counts + v.x, v.y);
    }
}

#ifndef EC3R_FI_PX
#define EC3R_FI_PX 4  // horizontally adjacent pixels per lane (4 or 2; sub-tile 8 x 4*FI_PX)
#endif
constexpr int FI_PX = EC3R_FI_PX;
static_assert(FI_PX == 4 || FI_PX == 2, "FI_PX");
constexpr int ST_H = 8, ST_W = 4 * FI_PX;
#ifndef EC3R_BC_BITS
#define EC3R_BC_BITS 11
#endif
constexpr int BC_BITS = EC3R_BC_BITS;  // shared-memory block cache: 2048 entries (16 KB)

#ifndef EC3R_FI_G
#define EC3R_FI_G 1  // consecutive listed frames per CTA (same band): the block cache carries over
#endif
constexpr int FI_G = EC3R_FI_G;

#ifndef EC3R_FI_DEDUP
#define EC3R_FI_DEDUP 0  // 1: merge a reduction slot's equal-voxel run ends across lanes before issuing
                         // (halves the reduction floor, but the hand-off makes the insert slower:
                         // 1.36 vs 1.19 ms on configs[1], profiles/r02g_fusion_conflicts.json)
#endif
constexpr bool FI_DEDUP = EC3R_FI_DEDUP != 0;

// Opt-in (EC3R_FI_TMA=1): on the bench workload the strip ring measured 1.4 %
// slower than the register-prefetched 64-bit loads (1.198 vs 1.181 ms,
// profiles/r02ag_*): the kernel runs at its reduction floor, and the strip
// hand-offs add barrier waits without removing any reduction.
static bool tma_requested() {
    const char* e = getenv("EC3R_FI_TMA");
    return e != nullptr && e[0] == '1';
}

// TMA form (TMA = true, one frame per CTA): the band's depth and confidence
// stream through shared memory as 8-row strips (one sub-tile row), each a
// contiguous 8 W-float span of both planes moved by two cp.async.bulk copies
// into a 2-stage ring; a warp waits on a strip's mbarrier before its first
// sub-tile there, and the last warp to leave a strip refills its stage with
// the strip two ahead.  Requires H W % 4 == 0 and 16-byte aligned planes.
__device__ __forceinline__ uint32_t vh_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <bool LOG, bool TMA, int NT = FI_NT>
__global__ void __launch_bounds__(NT, EC3R_FI_MINB * FI_NT / NT) vh_insert_frames_kernel(FuseArgs a) {
    extern __shared__ float4 sA[];  // A[W], then (TMA) the strip ring [2 stages][2 planes][8 W]
    __shared__ float4 sB[FI_ROWS];
    __shared__ __align__(8) uint64_t strip_full[2];
    __shared__ unsigned long long cta_cnt[4];
    __shared__ unsigned long long bcache[1 << BC_BITS];  // (tag << 32) | pool block, tag 0 = empty
    __shared__ float4 dd_sum[FI_DEDUP ? NT : 1];      // per-slot run hand-off to the group's lowest lane
    __shared__ float dd_n[FI_DEDUP ? NT : 1];
    const int W = a.W, H = a.H;
    const int HW = H * W;
    const int v_band = blockIdx.x * FI_ROWS;
    const int rows = min(FI_ROWS, H - v_band);
    if (threadIdx.x < 4) cta_cnt[threadIdx.x] = 0;
    for (int i = threadIdx.x; i < (1 << BC_BITS); i += NT) bcache[i] = 0ull;
    // cache keys are block coordinates relative to the first frame's camera block
    int3 ob;
    {
        const float4 T0 = __ldg(a.ftab + (size_t)(blockIdx.y * FI_G) * (W + H + 1) + W + H);
        ob = make_int3((int)floorf(T0.x * a.inv_cell_f * 0.25f), (int)floorf(T0.y * a.inv_cell_f * 0.25f),
                       (int)floorf(T0.z * a.inv_cell_f * 0.25f));
    }
    const float inv = a.inv_cell_f, cellf = a.cell_f;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int dv = lane >> 2, du = FI_PX * (lane & 3);
    const int stx = (W + ST_W - 1) / ST_W;
    const bool pairs = (W & 1) == 0;
    unsigned int n_in = 0, n_oor = 0, n_ovf = 0, n_slow = 0;
    const int j_end = min(a.n, (int)(blockIdx.y + 1) * FI_G);
    for (int j = blockIdx.y * FI_G; j < j_end; ++j) {
    const int slot = a.slots[j];
    const float4* tab = a.ftab + (size_t)j * (W + H + 1);
    __syncthreads();  // the previous frame's tables are no longer read
    for (int u = threadIdx.x; u < W; u += NT) sA[u] = __ldg(tab + u);
    if (threadIdx.x < rows) sB[threadIdx.x] = __ldg(tab + W + v_band + threadIdx.x);
    const float4 Tm = __ldg(tab + W + H);
    __syncthreads();
    const float* dbase = a.depth + (size_t)slot * HW;
    const float* cbase = a.conf + (size_t)slot * HW;
    const int n_strips = (rows + ST_H - 1) / ST_H;
    float* ring = reinterpret_cast<float*>(sA + W);
    auto issue_strip = [&](int s) {  // one thread: strip s of the band into stage s & 1
        const int r0 = s * ST_H, nr = min(ST_H, rows - r0);
        const uint32_t bytes = 4u * (uint32_t)(nr * W);
        const uint32_t bar = vh_smem_u32(strip_full + (s & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2u * bytes) : "memory");
        const size_t off = (size_t)(v_band + r0) * W;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         vh_smem_u32(ring + (size_t)((s & 1) * 2 + 0) * ST_H * W)),
                     "l"(dbase + off), "r"(bytes), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         vh_smem_u32(ring + (size_t)((s & 1) * 2 + 1) * ST_H * W)),
                     "l"(cbase + off), "r"(bytes), "r"(bar)
                     : "memory");
    };
    if constexpr (TMA) {
        if (threadIdx.x == 0) {
            for (int q = 0; q < 2; ++q) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(vh_smem_u32(strip_full + q)) : "memory");
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int q = 0; q < 2 && q < n_strips; ++q) issue_strip(q);
        }
        __syncthreads();
    }
    int cur_strip = -1;
    // warp-wide: strips are entered in order, each after its copy landed
    // (full[stage] mbarrier).  Leaving strip s is a named barrier (id 1 +
    // stage): warps 1..7 arrive, warp 0 syncs -- so it knows every warp is
    // done with the stage -- and refills it with strip s + 2.
    auto mbar_wait_vh = [&](uint64_t* bar, uint32_t par) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "VH_WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra VH_WAIT_%=;\n"
            "}\n" ::"r"(vh_smem_u32(bar)),
            "r"(par)
            : "memory");
    };
    auto enter_strip = [&](int s) {
        while (cur_strip < s) {
            if (cur_strip >= 0) {
                const int id = 1 + (cur_strip & 1);
                if (warp != 0) {
                    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(NT) : "memory");
                } else {
                    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NT) : "memory");
                    if (lane == 0 && cur_strip + 2 < n_strips) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue_strip(cur_strip + 2);
                    }
                    __syncwarp();
                }
            }
            ++cur_strip;
            if (cur_strip < n_strips) mbar_wait_vh(strip_full + (cur_strip & 1), (uint32_t)(cur_strip >> 1) & 1u);
        }
    };

    const int n_sy = (rows + ST_H - 1) / ST_H;
    auto row_of = [&](int sy_) { return sy_ * ST_H + dv; };
    // sub-tile st = sy * stx + sx, walked incrementally (no divisions)
    auto advance = [&](int& sy, int& sx) {
        sx += NT / 32;
        while (sx >= stx) { sx -= stx; ++sy; }
    };
    auto load4 = [&](int sy, int sx, float (&z)[FI_PX], float (&c)[FI_PX]) {
        const int r = row_of(sy), u0 = sx * ST_W + du;
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) { z[k] = 0.f; c[k] = 0.f; }
        if (r >= rows) return;
        const size_t off = (size_t)(v_band + r) * W + u0;
        if (pairs) {
#pragma unroll
            for (int h = 0; h < FI_PX / 2; ++h)
                if (u0 + 2 * h + 1 < W) {
                    const float2 z2 = __ldcs(reinterpret_cast<const float2*>(dbase + off + 2 * h));
                    const float2 c2 = __ldcs(reinterpret_cast<const float2*>(cbase + off + 2 * h));
                    z[2 * h] = z2.x; z[2 * h + 1] = z2.y;
                    c[2 * h] = c2.x; c[2 * h + 1] = c2.y;
                }
        } else {
#pragma unroll
            for (int k = 0; k < FI_PX; ++k)
                if (u0 + k < W) { z[k] = __ldcs(dbase + off + k); c[k] = __ldcs(cbase + off + k); }
        }
    };

    int sy = 0, sx = warp;
    while (sx >= stx) { sx -= stx; ++sy; }
    int py = sy, px = sx;  // prefetch cursor
    float nz[FI_PX], nc[FI_PX];
    if constexpr (!TMA) {
        if (py < n_sy) load4(py, px, nz, nc);
    }
    for (; sy < n_sy; advance(sy, sx)) {
        const int r = row_of(sy), u0 = sx * ST_W + du;
        float zs[FI_PX], cs[FI_PX];
        if constexpr (TMA) {
            enter_strip(sy);
            const float* zr = ring + (size_t)((sy & 1) * 2) * ST_H * W + dv * W + u0;
            const float* cr = zr + ST_H * W;
#pragma unroll
            for (int k = 0; k < FI_PX; ++k) { zs[k] = 0.f; cs[k] = 0.f; }
            if (r < rows) {
                if (pairs) {
#pragma unroll
                    for (int h = 0; h < FI_PX / 2; ++h)
                        if (u0 + 2 * h + 1 < W) {
                            const float2 z2 = *reinterpret_cast<const float2*>(zr + 2 * h);
                            const float2 c2 = *reinterpret_cast<const float2*>(cr + 2 * h);
                            zs[2 * h] = z2.x; zs[2 * h + 1] = z2.y;
                            cs[2 * h] = c2.x; cs[2 * h + 1] = c2.y;
                        }
                } else {
#pragma unroll
                    for (int k = 0; k < FI_PX; ++k)
                        if (u0 + k < W) { zs[k] = zr[k]; cs[k] = cr[k]; }
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < FI_PX; ++k) { zs[k] = nz[k]; cs[k] = nc[k]; }
            advance(py, px);
            if (py < n_sy) load4(py, px, nz, nc);
        }
        const float4 Bv = sB[min(r, rows - 1)];

        // phase A: keys and contributions of the lane's 4 pixels, branch-free
        // except the (rare) exact float64 re-run near a voxel face
        bool valid[FI_PX];
        int cx[FI_PX], cy[FI_PX], cz[FI_PX];
        float ox[FI_PX], oy[FI_PX], oz[FI_PX];
        unsigned slow = 0;
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            const float z = zs[k], c = cs[k];
            const float4 Au = sA[min(u0 + k, W - 1)];  // columns past W are zero-filled (invalid)
            const float dx = Au.x + Bv.x, dy = Au.y + Bv.y, dz = Au.z + Bv.z;
            const float x = fmaf(z, dx, Tm.x), y = fmaf(z, dy, Tm.y), zz = fmaf(z, dz, Tm.z);
            // first-order float32 error bound (x4 safety), see header; +1 ulp(0.5)
            // for the folded face test below
            const float ax = fabsf(x) + fabsf(y) + fabsf(zz);
            const float err = 2.384185791015625e-07f * (2.0f * z * (Au.w + Bv.w) + Tm.w + 2.0f * ax) + 1e-9f;
            const float margin = err * inv + 3.6e-7f;
            const float qx = x * inv, qy = y * inv, qz = zz * inv;
            const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
            // |frac - 1/2| > 1/2 - margin  <=>  within margin of a face (q - floor(q) and - 1/2 are exact)
            const float dev = fmaxf(fmaxf(fabsf(qx - fx - 0.5f), fabsf(qy - fy - 0.5f)), fabsf(qz - fz - 0.5f));
            const float qmax = fmaxf(fmaxf(fabsf(qx), fabsf(qy)), fabsf(qz));
            valid[k] = z > 0.f && c > 0.f;
            n_in += valid[k];
            if (valid[k] && !(dev < 0.5f - margin && qmax <= 1.0e6f)) slow |= 1u << k;
            // |q| <= 1e6 < 2^20: fast-path cells are always inside the key range
            cx[k] = (int)fx; cy[k] = (int)fy; cz[k] = (int)fz;
            ox[k] = x; oy[k] = y; oz[k] = zz;
        }
        if (slow) {
#pragma unroll
            for (int k = 0; k < FI_PX; ++k) {
                if (!(slow & (1u << k))) continue;
                long long cc[3];
                exact_cells(a.slot_poses + 8 * slot, a.slot_globals + 8 * slot, ray_coef(u0 + k, a.cx, a.fx),
                            ray_coef(v_band + r, a.cy, a.fy), zs[k], a.cell, cc);
                ++n_slow;
                if (cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2])) {
                    cx[k] = (int)cc[0]; cy[k] = (int)cc[1]; cz[k] = (int)cc[2];
                } else {
                    ++n_oor;
                    valid[k] = false;
                }
            }
        }
        // phase B: block indices.  The CTA's shared-memory block cache maps
        // an exact 30-bit block key relative to the frame's camera block to
        // the pool block; the four lookups of a lane are independent LDS.64.
        // A miss (first touch of a block by this CTA, a block > 40 m from
        // the camera, or a cache collision) resolves through the global
        // table and refills the cache.
        int got[FI_PX], local[FI_PX];
        uint32_t tag[FI_PX], slot[FI_PX];
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            local[k] = (cx[k] & 3) | ((cy[k] & 3) << 2) | ((cz[k] & 3) << 4);
            const unsigned rx = (unsigned)((cx[k] >> 2) - ob.x + 512), ry = (unsigned)((cy[k] >> 2) - ob.y + 512),
                           rz = (unsigned)((cz[k] >> 2) - ob.z + 512);
            tag[k] = (valid[k] && (rx | ry | rz) < 1024u) ? (rx | (ry << 10) | (rz << 20)) + 1u : 0u;
            slot[k] = (tag[k] * 0x9E3779B1u) >> (32 - BC_BITS);
            const unsigned long long e = tag[k] ? bcache[slot[k]] : 0ull;
            got[k] = ((uint32_t)(e >> 32) == tag[k] && tag[k]) ? (int)(uint32_t)e : -3;
        }
        // misses: lanes sharing a block elect one leader per pixel slot; the
        // leaders' first probes of the 4 slots are in flight together and
        // only a first-probe miss walks the probe chain / inserts
        bool miss[FI_PX];
        int leader[FI_PX];
        unsigned long long bk[FI_PX];
        unsigned lead = 0;
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            miss[k] = valid[k] && got[k] == -3;
            leader[k] = -1;
            bk[k] = pack_block(cx[k] >> 2, cy[k] >> 2, cz[k] >> 2);
            if (__any_sync(0xffffffffu, miss[k])) {
                const unsigned peers = __match_any_sync(0xffffffffu, miss[k] ? bk[k] : kEmpty);
                leader[k] = __ffs(peers) - 1;
                if (miss[k] && lane == leader[k]) lead |= 1u << k;
            }
        }
        if (lead) {
            unsigned long long ek[FI_PX];
            int gk[FI_PX];
#pragma unroll
            for (int k = 0; k < FI_PX; ++k) {
                ek[k] = kEmpty;
                gk[k] = -1;
                if (lead & (1u << k)) load_entry(a.vb.table + table_slot(bk[k], a.vb.tmask), ek[k], gk[k]);
            }
#pragma unroll
            for (int k = 0; k < FI_PX; ++k) {
                if (!(lead & (1u << k))) continue;
                if (ek[k] != bk[k] || gk[k] == -1) gk[k] = vb_find_or_insert(a.vb, bk[k]);
                got[k] = gk[k];
                // the cache is lock-free: entries are single 64-bit words validated by
                // their tag on read, so a racing reader sees the old or the new entry;
                // the (rare) refill is an atomic exchange so the sanitizer sees it too
                if (tag[k] && gk[k] >= 0)
                    atomicExch(&bcache[slot[k]], ((unsigned long long)tag[k] << 32) | (uint32_t)gk[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            if (leader[k] >= 0) {
                const int g = __shfl_sync(0xffffffffu, got[k], leader[k]);
                if (miss[k]) got[k] = g;
            }
        }
        // phase C: reductions into the pool.  Consecutive pixels of the lane
        // in the same voxel form a run whose sums ride along (FFMA with a
        // 0/1 continuation flag); only a run's last pixel issues the two
        // reductions (predicated, no branches).
        uint32_t vid[FI_PX];
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            if (valid[k] && got[k] < 0) ++n_ovf;
            vid[k] = (valid[k] && got[k] >= 0) ? (((uint32_t)got[k] << 6) | (uint32_t)local[k]) : 0xFFFFFFFFu;
        }
        float rx = 0.f, ry = 0.f, rz = 0.f, rw = 0.f, rn = 0.f;
#pragma unroll
        for (int k = 0; k < FI_PX; ++k) {
            const float c = cs[k];
            const float cont = (k > 0 && vid[k] == vid[k - 1]) ? 1.f : 0.f;
            rx = fmaf(cont, rx, c * (ox[k] - (float)cx[k] * cellf));
            ry = fmaf(cont, ry, c * (oy[k] - (float)cy[k] * cellf));
            rz = fmaf(cont, rz, c * (oz[k] - (float)cz[k] * cellf));
            rw = fmaf(cont, rw, c);
            rn = fmaf(cont, rn, 1.f);
            bool last = vid[k] != 0xFFFFFFFFu && (k == FI_PX - 1 || vid[k + 1 < FI_PX ? k + 1 : FI_PX - 1] != vid[k]);
            float sx = rx, sy = ry, sz = rz, sw = rw, sn = rn;
            if constexpr (FI_DEDUP) {
                // Lanes of one reduction instruction that target the same
                // voxel serialise in the memory pipeline (the replayed log
                // with each 32-run group's equal voxels merged takes 0.60 ms
                // instead of 1.13 ms for 14 % fewer runs,
                // tools/fuse_order_probe.py), so equal run ends of this slot
                // (mostly vertical neighbours) are summed into their lowest
                // lane first and issued once.  Opt-in: the live kernel is
                // latency-bound at 16 warps per SM, and the shared-memory
                // hand-off costs more than the reductions it removes.
                const unsigned peers = __match_any_sync(0xffffffffu, last ? vid[k] : 0xFFFFFFFFu);
                const bool grp = last && (peers & (peers - 1u)) != 0u;
                if (__any_sync(0xffffffffu, grp)) {
                    if (grp) {
                        dd_sum[threadIdx.x] = make_float4(rx, ry, rz, rw);
                        dd_n[threadIdx.x] = rn;
                    }
                    __syncwarp();
                    if (grp) {
                        if (lane == __ffs(peers) - 1) {
                            unsigned o = peers & (peers - 1u);  // the other members
                            while (o) {
                                const int b = (threadIdx.x & ~31) + __ffs(o) - 1;
                                o &= o - 1u;
                                const float4 v = dd_sum[b];
                                sx += v.x; sy += v.y; sz += v.z; sw += v.w;
                                sn += dd_n[b];
                            }
                        } else {
                            last = false;
                        }
                    }
                    __syncwarp();
                }
            }
            if (last) {
                if constexpr (LOG) {
                    log_run(RunLog{a.log_runs, a.log_n, a.log_cap}, vid[k], (uint32_t)sn);
                } else {
                    red_add_v4(a.vb.sums + vid[k], sx, sy, sz, sw);
                    red_add_u32(a.vb.counts + vid[k], (uint32_t)sn);
                }
            }
        }
    }
    if constexpr (TMA) enter_strip(n_strips);  // count this warp out of the remaining strips
    }  // frames of this CTA
    // counters: warp reduce then one shared atomic per warp, one global per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
        n_oor += __shfl_xor_sync(0xffffffffu, n_oor, o);
        n_ovf += __shfl_xor_sync(0xffffffffu, n_ovf, o);
        n_slow += __shfl_xor_sync(0xffffffffu, n_slow, o);
    }
    if (lane == 0) {
        atomicAdd(&cta_cnt[0], (unsigned long long)n_in);
        atomicAdd(&cta_cnt[1], (unsigned long long)n_oor);
        atomicAdd(&cta_cnt[2], (unsigned long long)n_ovf);
        atomicAdd(&cta_cnt[3], (unsigned long long)n_slow);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cta_cnt[threadIdx.x]) atomicAdd(&a.vb.counters[threadIdx.x], cta_cnt[threadIdx.x]);
}

// Explicit points (float64) under one Sim(3): exact float64 transform.
__global__ void vh_insert_points_kernel(const double* __restrict__ pts, const double* __restrict__ conf, int64_t n,
                                        Sim3Arg g, double cell, VB vb) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        bool valid = i < n;
        long long cc[3] = {0, 0, 0};
        float ox = 0.f, oy = 0.f, oz = 0.f, w = 0.f;
        unsigned c_in = 0, c_oor = 0;
        if (valid) {
            const double c = conf[i];
            valid = c > 0;
            if (valid) {
                c_in = 1;
                const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
                double x[3];
                sim3_apply_exact(g.v, p, x);
#pragma unroll
                for (int k = 0; k < 3; ++k) cc[k] = (long long)floor(__ddiv_rn(x[k], cell));
                if (cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2])) {
                    w = (float)c;
                    ox = (float)(c * (x[0] - (double)cc[0] * cell));
                    oy = (float)(c * (x[1] - (double)cc[1] * cell));
                    oz = (float)(c * (x[2] - (double)cc[2] * cell));
                } else {
                    valid = false;
                    c_oor = 1;
                }
            }
        }
        unsigned long long cbk = kEmpty;
        int cidx = -2;
        const unsigned ovf = vb_insert_warp(vb, valid, cc[0], cc[1], cc[2], ox, oy, oz, w, 1u, cbk, cidx);
        if (c_in) atomicAdd(&vb.counters[0], 1ull);
        if (c_oor) atomicAdd(&vb.counters[1], 1ull);
        if (ovf) atomicAdd(&vb.counters[2], 1ull);
    }
}

// ---------------------------------------------------------------------------
// extraction

__global__ void vb_gather32_kernel(const float4* __restrict__ sums, const unsigned int* __restrict__ counts,
                                   const unsigned long long* __restrict__ block_keys, const uint32_t* __restrict__ i32,
                                   const int64_t* __restrict__ n_ptr, double cell, int64_t* __restrict__ okeys,
                                   float* __restrict__ cen, float* __restrict__ wsum, int32_t* __restrict__ cnt) {
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = i32[i];
        const float4 s = sums[v];
        long long bx, by, bz;
        unpack_cells(block_keys[v / kBlockVox], bx, by, bz);
        const int local = (int)(v % kBlockVox);
        const long long cx = bx * 4 + (local & 3), cy = by * 4 + ((local >> 2) & 3), cz = bz * 4 + (local >> 4);
        okeys[i] = (int64_t)pack_cells(cx, cy, cz);
        const double w = s.w;
        cen[3 * i + 0] = (float)((double)cx * cell + (double)s.x / w);
        cen[3 * i + 1] = (float)((double)cy * cell + (double)s.y / w);
        cen[3 * i + 2] = (float)((double)cz * cell + (double)s.z / w);
        wsum[i] = s.w;
        cnt[i] = (int32_t)counts[v];
    }
}

__global__ void vb_gather_kernel(const float4* __restrict__ sums, const unsigned int* __restrict__ counts,
                                 const unsigned long long* __restrict__ keys, const int64_t* __restrict__ idx,
                                 const int64_t* __restrict__ n_ptr, double cell, int64_t* __restrict__ okeys,
                                 float* __restrict__ cen, float* __restrict__ wsum, int32_t* __restrict__ cnt) {
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 s = sums[idx[i]];
        const unsigned long long k = keys[i];
        long long cx, cy, cz;
        unpack_cells(k, cx, cy, cz);
        okeys[i] = (int64_t)k;
        const double w = s.w;
        cen[3 * i + 0] = (float)((double)cx * cell + (double)s.x / w);
        cen[3 * i + 1] = (float)((double)cy * cell + (double)s.y / w);
        cen[3 * i + 2] = (float)((double)cz * cell + (double)s.z / w);
        wsum[i] = s.w;
        cnt[i] = (int32_t)counts[idx[i]];
    }
}

// partial sums for the multi-GPU all-to-all: owner = mix64(key) % n_ranks
__global__ void vb_partition_count_kernel(const unsigned long long* __restrict__ keys, const int64_t* __restrict__ n_ptr,
                                          int n_ranks, unsigned long long* __restrict__ rank_counts) {
    // per-CTA histogram in shared memory, one global add per (CTA, rank):
    // a global atomic per voxel on <= n_ranks words serialises at L2
    __shared__ unsigned int hist[64];
    for (int r = threadIdx.x; r < n_ranks; r += blockDim.x) hist[r] = 0u;
    __syncthreads();
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&hist[mix64(keys[i]) % (unsigned long long)n_ranks], 1u);
    __syncthreads();
    for (int r = threadIdx.x; r < n_ranks; r += blockDim.x)
        if (hist[r]) atomicAdd(&rank_counts[r], (unsigned long long)hist[r]);
}

__global__ void vb_partition_write_kernel(const float4* __restrict__ sums, const unsigned int* __restrict__ counts,
                                          const unsigned long long* __restrict__ keys,
                                          const int64_t* __restrict__ idx, const int64_t* __restrict__ n_ptr,
                                          int n_ranks, const unsigned long long* __restrict__ rank_base,
                                          unsigned long long* __restrict__ cursors, int64_t* __restrict__ okeys,
                                          float* __restrict__ sums4, int32_t* __restrict__ cnt) {
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        const int r = (int)(mix64(k) % (unsigned long long)n_ranks);
        // warp-aggregated cursor: one atomic per (warp, owner rank)
        const unsigned peers = __match_any_sync(__activemask(), r);
        const int lead = __ffs(peers) - 1;
        const unsigned lanes_below = peers & ((1u << (threadIdx.x & 31)) - 1u);
        unsigned long long base = 0;
        if ((int)(threadIdx.x & 31) == lead) base = atomicAdd(&cursors[r], (unsigned long long)__popc(peers));
        base = __shfl_sync(peers, base, lead);
        const unsigned long long o = rank_base[r] + base + __popc(lanes_below);
        okeys[o] = (int64_t)k;
        reinterpret_cast<float4*>(sums4)[o] = sums[idx[i]];
        cnt[o] = (int32_t)counts[idx[i]];
    }
}

__global__ void vb_merge_kernel(const int64_t* __restrict__ keys, const float* __restrict__ sums4,
                                const int32_t* __restrict__ cnt, int64_t n, VB vb) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        const bool valid = i < n;
        long long cx = 0, cy = 0, cz = 0;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned c = 0;
        if (valid) {
            unpack_cells((unsigned long long)keys[i], cx, cy, cz);
            s = reinterpret_cast<const float4*>(sums4)[i];
            c = (unsigned)cnt[i];
        }
        unsigned long long cbk = kEmpty;
        int cidx = -2;
        if (vb_insert_warp(vb, valid, cx, cy, cz, s.x, s.y, s.z, s.w, c, cbk, cidx))
            atomicAdd(&vb.counters[2], 1ull);
    }
}

static unsigned grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)kNumSMs * 16) g = (int64_t)kNumSMs * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

__global__ void bbox_init_kernel(int* bbox) {
    if (threadIdx.x < 3) { bbox[threadIdx.x] = INT_MAX; bbox[3 + threadIdx.x] = INT_MIN; }
    if (threadIdx.x == 6 || threadIdx.x == 7) bbox[threadIdx.x] = 0;  // column emit: the 32-bit key overflow flag
}

// Compaction, pass 1 (one warp per pool block): occupied voxels per block
// and the bounding box of the used blocks (cells, conservative to the block).
__global__ void vb_block_count_kernel(const unsigned int* __restrict__ counts,
                                      const unsigned long long* __restrict__ block_keys,
                                      const unsigned long long* __restrict__ counters, int64_t max_blocks,
                                      int* __restrict__ blk_cnt, int* __restrict__ bbox) {
    const int lane = threadIdx.x & 31;
    const int64_t used = min((int64_t)counters[4], max_blocks);
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < max_blocks;
         b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int n = 0;
        if (b < used) {
            const unsigned m0 = __ballot_sync(0xffffffffu, counts[b * kBlockVox + lane] != 0u);
            const unsigned m1 = __ballot_sync(0xffffffffu, counts[b * kBlockVox + 32 + lane] != 0u);
            n = __popc(m0) + __popc(m1);
            if (n && lane < 3) {
                long long c[3];
                unpack_cells(block_keys[b], c[0], c[1], c[2]);
                mn[lane] = min(mn[lane], (int)(4 * c[lane]));
                mx[lane] = max(mx[lane], (int)(4 * c[lane] + 3));
            }
        }
        if (lane == 0) blk_cnt[b] = n;
    }
    // bounding box: shared-memory reduction first, then one global atomic
    // per CTA and component (every warp hitting the six global words
    // serialised them at L2)
    __shared__ int sbox[6];
    if (threadIdx.x < 3) { sbox[threadIdx.x] = INT_MAX; sbox[3 + threadIdx.x] = INT_MIN; }
    __syncthreads();
    if (lane < 3 && mn[lane] <= mx[lane]) {
        atomicMin(&sbox[lane], mn[lane]);
        atomicMax(&sbox[3 + lane], mx[lane]);
    }
    __syncthreads();
    if (threadIdx.x < 3 && sbox[threadIdx.x] <= sbox[3 + threadIdx.x]) {
        atomicMin(&bbox[threadIdx.x], sbox[threadIdx.x]);
        atomicMax(&bbox[3 + threadIdx.x], sbox[3 + threadIdx.x]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) blk_cnt[max_blocks] = 0;
}

// Compaction, pass 2 (one warp per pool block): voxel j of block b goes to
// blk_off[b] + (occupied voxels before it in the block) -- block order, no
// atomics.  pack32: keys relative to the box in 32 bits (lexicographic order
// preserved), else _pack keys + int64 voxel indices.  At most max_voxels
// are written; the excess is counted in counters[5].
__global__ void vb_block_emit_kernel(const unsigned int* __restrict__ counts,
                                     const unsigned long long* __restrict__ block_keys,
                                     const unsigned long long* __restrict__ counters, int64_t max_blocks,
                                     const int* __restrict__ blk_off, int64_t max_voxels, const int* __restrict__ bbox,
                                     int pack32, int by_bits, int bz_bits, uint32_t* __restrict__ k32,
                                     uint32_t* __restrict__ i32, unsigned long long* __restrict__ k64,
                                     int64_t* __restrict__ i64, unsigned long long* __restrict__ ovf,
                                     int64_t* __restrict__ n_out) {
    const int lane = threadIdx.x & 31;
    const int64_t used = min((int64_t)counters[4], max_blocks);
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = min((int64_t)blk_off[max_blocks], max_voxels);
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < used;
         b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const bool o0 = counts[b * kBlockVox + lane] != 0u, o1 = counts[b * kBlockVox + 32 + lane] != 0u;
        const unsigned m0 = __ballot_sync(0xffffffffu, o0), m1 = __ballot_sync(0xffffffffu, o1);
        if (!(m0 | m1)) continue;
        long long bx, by, bz;
        unpack_cells(block_keys[b], bx, by, bz);
        const unsigned lt = (1u << lane) - 1u;
        const int64_t base = blk_off[b];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (!(h ? o1 : o0)) continue;
            const int64_t o = base + (h ? __popc(m0) + __popc(m1 & lt) : __popc(m0 & lt));
            if (o >= max_voxels) { atomicAdd(ovf, 1ull); continue; }
            const int local = lane + 32 * h;
            const long long cx = bx * 4 + (local & 3), cy = by * 4 + ((local >> 2) & 3), cz = bz * 4 + (local >> 4);
            const int64_t v = b * kBlockVox + local;
            if (pack32) {
                k32[o] = ((uint32_t)(cx - bbox[0]) << (by_bits + bz_bits)) | ((uint32_t)(cy - bbox[1]) << bz_bits) |
                         (uint32_t)(cz - bbox[2]);
                i32[o] = (uint32_t)v;
            } else {
                k64[o] = pack_cells(cx, cy, cz);
                i64[o] = v;
            }
        }
    }
}

static int bits_for(int range) {  // bits to hold values 0..range
    int b = 0;
    while (b < 31 && (1u << b) <= (unsigned)range) ++b;
    return b;
}

// Compact + (optional) sort.  *n_out (device) receives U.  Without sort, or
// with the 64-bit key sort, (*ks, *is) are the arrays to gather from and
// *i32 = nullptr; with the 32-bit key sort (bounding box fits 32 bits: the
// usual case, 4 radix passes instead of 8) *i32 holds the sorted pool
// indices.
static size_t scan_temp_bytes(int64_t n) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (int*)nullptr, (int*)nullptr, (int)n);
    return t;
}

static int compact_sorted(ec3r_vhash* h, int sort, void* workspace, size_t workspace_bytes, int64_t* n_out,
                          const unsigned long long** ks, const int64_t** is, const uint32_t** i32,
                          cudaStream_t st) {
    const size_t cap = (size_t)h->max_voxels;
    const int64_t nb = h->max_blocks;
    h->last_count = -1;
    Carver cv{(char*)workspace, 0};
    unsigned long long* k0 = cv.take<unsigned long long>(cap);
    int64_t* i0 = cv.take<int64_t>(cap);
    unsigned long long* k1 = cv.take<unsigned long long>(cap);
    int64_t* i1 = cv.take<int64_t>(cap);
    unsigned long long* cursor = cv.take<unsigned long long>(8);  // [1..3] bbox (6 ints)
    int* bbox = reinterpret_cast<int*>(cursor + 1);
    int* blk_cnt = cv.take<int>(nb + 1);
    int* blk_off = cv.take<int>(nb + 1);
    size_t scan_bytes = scan_temp_bytes(nb + 1);
    void* scan_tmp = cv.take<char>(scan_bytes);
    size_t cub_bytes = workspace_bytes - cv.used;
    void* cub_tmp = cv.base + cv.used;
    if (cv.used > workspace_bytes) return EC3R_EWORKSPACE;
    bbox_init_kernel<<<1, 32, 0, st>>>(bbox);
    EC3R_CHECK_LAUNCH("bbox_init_kernel");
    const unsigned grid = (unsigned)std::min<int64_t>((nb * 32 + 255) / 256, (int64_t)kNumSMs * 16);
    vb_block_count_kernel<<<grid, 256, 0, st>>>(h->counts, h->block_keys, h->counters, nb, blk_cnt, bbox);
    EC3R_CHECK_LAUNCH("vb_block_count_kernel");
    if (cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, blk_cnt, blk_off, (int)(nb + 1), st) != cudaSuccess) {
        set_last_error("cub::DeviceScan::ExclusiveSum", cudaGetLastError());
        return EC3R_ECUDA;
    }
    *ks = k0;
    *is = i0;
    *i32 = nullptr;
    if (!sort) {
        vb_block_emit_kernel<<<grid, 256, 0, st>>>(h->counts, h->block_keys, h->counters, nb, blk_off, h->max_voxels,
                                                   bbox, 0, 0, 0, nullptr, nullptr, k0, i0, h->counters + 5, n_out);
        EC3R_CHECK_LAUNCH("vb_block_emit_kernel");
        return EC3R_OK;
    }
    // one host round trip: the voxel count and the box decide the sort key
    int hst[8];
    EC3R_CUDA_TRY(cudaMemcpyAsync(hst, blk_off + nb, sizeof(int), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaMemcpyAsync(hst + 1, bbox, 6 * sizeof(int), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t nh = std::min<int64_t>(hst[0], h->max_voxels);
    h->last_count = nh;
    const int* bb = hst + 1;
    if (nh <= 0) {
        vb_block_emit_kernel<<<1, 32, 0, st>>>(h->counts, h->block_keys, h->counters, 0, blk_off + nb, h->max_voxels,
                                               bbox, 0, 0, 0, nullptr, nullptr, k0, i0, h->counters + 5, n_out);
        EC3R_CHECK_LAUNCH("vb_block_emit_kernel");
        return EC3R_OK;
    }
    const int bx = bits_for(bb[3] - bb[0]), by = bits_for(bb[4] - bb[1]), bz = bits_for(bb[5] - bb[2]);
    const int total = bx + by + bz;
    if (total <= 32 && cap <= 0xFFFFFFFFull) {
        uint32_t* k32 = reinterpret_cast<uint32_t*>(k1);
        uint32_t* v32 = reinterpret_cast<uint32_t*>(i1);
        uint32_t* k32s = k32 + cap;
        uint32_t* v32s = v32 + cap;
        vb_block_emit_kernel<<<grid, 256, 0, st>>>(h->counts, h->block_keys, h->counters, nb, blk_off, h->max_voxels,
                                                   bbox, 1, by, bz, k32, v32, nullptr, nullptr, h->counters + 5,
                                                   n_out);
        EC3R_CHECK_LAUNCH("vb_block_emit_kernel");
        if (cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k32, k32s, v32, v32s, (int)nh, 0,
                                            total > 0 ? total : 1, st) != cudaSuccess) {
            set_last_error("cub::DeviceRadixSort::SortPairs(u32)", cudaGetLastError());
            return EC3R_ECUDA;
        }
        *i32 = v32s;
        return EC3R_OK;
    }
    vb_block_emit_kernel<<<grid, 256, 0, st>>>(h->counts, h->block_keys, h->counters, nb, blk_off, h->max_voxels, bbox,
                                               0, 0, 0, nullptr, nullptr, k0, i0, h->counters + 5, n_out);
    EC3R_CHECK_LAUNCH("vb_block_emit_kernel");
    if (cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k0, k1, i0, i1, (int)nh, 0, 63, st) != cudaSuccess) {
        set_last_error("cub::DeviceRadixSort::SortPairs", cudaGetLastError());
        return EC3R_ECUDA;
    }
    *ks = k1;
    *is = i1;
    return EC3R_OK;
}


// ---------------------------------------------------------------------------
// Sorted emit without a voxel sort.  The output is ordered by _pack key, i.e.
// by (cx, cy, cz).  A pool block (bx, by, bz) holds 16 voxel columns (lx, ly)
// of 4 voxels (lz); the key order of all columns is the lexicographic order
// of (bx, lx, by, ly, bz).  So only the USED BLOCKS are sorted (by block key,
// ~1/37 of the voxels here); per block, the closed-form position of each of
// its columns in that order follows from the block's x-group (blocks with
// the same bx) and xy-group (same bx, by):
//   pos = 16 * start_x + 4 * n_x * lx + 4 * off_xy + n_xy * ly + r_z
// One exclusive scan of the columns' occupied counts in that order gives each
// column its first output row, and each occupied voxel its row
// (+ its rank among the column's occupied lz).  Reference: the declared
// fusion rule's "output sorted by key" (oracle/fuse.py, _numpy.py:50-55).

struct ColGroup {
    int start_x, n_x, off_xy, n_xy, r_z, pad;
};

__device__ __forceinline__ int64_t vc_used(const unsigned long long* counters, int64_t max_blocks) {
    return min((int64_t)counters[4], max_blocks);
}

// per pool block: 16 column counts and its sort key (_pack key; unused
// blocks sort last)
__global__ void vc_block_prep_kernel(const unsigned int* __restrict__ counts,
                                     const unsigned long long* __restrict__ block_keys,
                                     const unsigned long long* __restrict__ counters, int64_t nb,
                                     uint8_t* __restrict__ colcnt, unsigned long long* __restrict__ skey,
                                     uint32_t* __restrict__ ids) {
    const int lane = threadIdx.x & 31;
    const int64_t used = vc_used(counters, nb);
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb;
         b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        if (b < used) {
            const unsigned m0 = __ballot_sync(0xffffffffu, counts[b * kBlockVox + lane] != 0u);
            const unsigned m1 = __ballot_sync(0xffffffffu, counts[b * kBlockVox + 32 + lane] != 0u);
            if (lane < 16) {
                const unsigned long long m = ((unsigned long long)m1 << 32) | m0;
                colcnt[b * 16 + lane] = (uint8_t)__popcll(m & (0x0001000100010001ull << lane));
            }
        }
        if (lane == 16) {
            skey[b] = b < used ? block_keys[b] : ~0ull;
            ids[b] = (uint32_t)b;
        }
    }
}

// 32-bit sort keys relative to the used blocks' minimum corner: x 11 | y 11 |
// z 10 bits (the _pack key order).  bb[0..2] = min block coordinates,
// bb[3..5] = max; bb[6] set when the extent does not fit (the caller then
// re-runs with the 64-bit keys).
constexpr int VC_XB = 11, VC_YB = 11, VC_ZB = 10;

__global__ void vc_bbox_kernel(const unsigned long long* __restrict__ block_keys,
                               const unsigned long long* __restrict__ counters, int64_t nb, int* __restrict__ bb) {
    const int64_t used = vc_used(counters, nb);
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < used; b += (int64_t)gridDim.x * blockDim.x) {
        long long c[3];
        unpack_cells(block_keys[b], c[0], c[1], c[2]);
#pragma unroll
        for (int a = 0; a < 3; ++a) { mn[a] = min(mn[a], (int)c[a]); mx[a] = max(mx[a], (int)c[a]); }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a)
            if (mn[a] <= mx[a]) { atomicMin(&bb[a], mn[a]); atomicMax(&bb[3 + a], mx[a]); }
}

__global__ void vc_key32_kernel(const unsigned long long* __restrict__ block_keys,
                                unsigned long long* __restrict__ counters, int64_t nb, int* __restrict__ bb,
                                uint32_t* __restrict__ skey, uint32_t* __restrict__ ids, int report) {
    const int64_t used = vc_used(counters, nb);
    const bool fits = used == 0 || ((unsigned)(bb[3] - bb[0]) < (1u << VC_XB) &&
                                    (unsigned)(bb[4] - bb[1]) < (1u << VC_YB) &&
                                    (unsigned)(bb[5] - bb[2]) < (1u << VC_ZB));
    // a map that outgrew the 32-bit keys: the host-read emit re-runs with
    // 64-bit keys; the host-sync-free emit reports it as emit overflow
    // (counters[5], stats n_overflow), so its caller re-runs synced
    if (blockIdx.x == 0 && threadIdx.x == 0 && !fits) {
        bb[6] = 1;
        if (report) atomicAdd(&counters[5], 1ull);
    }
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t k = 0xFFFFFFFFu;
        if (b < used && fits) {
            long long c[3];
            unpack_cells(block_keys[b], c[0], c[1], c[2]);
            k = ((uint32_t)(c[0] - bb[0]) << (VC_YB + VC_ZB)) | ((uint32_t)(c[1] - bb[1]) << VC_ZB) |
                (uint32_t)(c[2] - bb[2]);
        }
        skey[b] = k;
        ids[b] = (uint32_t)b;
    }
}

template <typename K>
__device__ __forceinline__ int64_t lb_key(const K* a, int64_t n, unsigned long long v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((unsigned long long)a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// x-group (same bx) and xy-group (same bx, by) of every used block from the
// key-sorted blocks: x = key >> sx, xy = key >> sy
template <typename K>
__global__ void vc_groups_kernel(const K* __restrict__ skeys, const uint32_t* __restrict__ sids,
                                 const unsigned long long* __restrict__ counters, int64_t nb, int sx, int sy,
                                 ColGroup* __restrict__ grp) {
    const int64_t n = vc_used(counters, nb);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = (unsigned long long)skeys[i];
        const unsigned long long x = k >> sx, xy = k >> sy;
        const int64_t s_x = lb_key(skeys, n, x << sx), e_x = lb_key(skeys, n, (x + 1) << sx);
        const int64_t s_xy = lb_key(skeys, n, xy << sy), e_xy = lb_key(skeys, n, (xy + 1) << sy);
        grp[sids[i]] = ColGroup{(int)s_x, (int)(e_x - s_x), (int)(s_xy - s_x), (int)(e_xy - s_xy), (int)(i - s_xy), 0};
    }
}

__device__ __forceinline__ int64_t vc_col_pos(const ColGroup& g, int col) {
    const int lx = col & 3, ly = col >> 2;
    return (int64_t)g.start_x * 16 + (int64_t)lx * 4 * g.n_x + (int64_t)g.off_xy * 4 + (int64_t)ly * g.n_xy + g.r_z;
}

// column counts in key order (scan input) and the column behind each position
__global__ void vc_colpos_kernel(const ColGroup* __restrict__ grp, const uint8_t* __restrict__ colcnt,
                                 const unsigned long long* __restrict__ counters, int64_t nb,
                                 uint32_t* __restrict__ scan_in, uint32_t* __restrict__ colsrc) {
    const int64_t n16 = vc_used(counters, nb) * 16;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n16; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = vc_col_pos(grp[t >> 4], (int)(t & 15));
        scan_in[p] = colcnt[t];
        colsrc[p] = (uint32_t)t;
    }
}

// one thread per column position, in key order: the column's occupied voxels
// go to consecutive output rows (coalesced writes)
__global__ void vc_gather_kernel(const float4* __restrict__ sums, const unsigned int* __restrict__ counts,
                                 const unsigned long long* __restrict__ block_keys,
                                 const unsigned long long* __restrict__ counters, int64_t nb,
                                 const uint32_t* __restrict__ colsrc, const uint32_t* __restrict__ scan_in,
                                 const uint32_t* __restrict__ col_base, int64_t max_voxels, double cell,
                                 int64_t* __restrict__ okeys, float* __restrict__ cen, float* __restrict__ wsum,
                                 int32_t* __restrict__ cnt, unsigned long long* __restrict__ ovf,
                                 int64_t* __restrict__ n_out) {
    const int64_t n16 = vc_used(counters, nb) * 16;
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = min((int64_t)col_base[n16], max_voxels);
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n16; p += (int64_t)gridDim.x * blockDim.x) {
        if (!scan_in[p]) continue;
        const uint32_t t = colsrc[p];
        const int64_t b = t >> 4;
        const int col = (int)(t & 15);
        int64_t d = col_base[p];
        long long bx, by, bz;
        unpack_cells(block_keys[b], bx, by, bz);
        const long long cx = bx * 4 + (col & 3), cy = by * 4 + (col >> 2);
#pragma unroll
        for (int lz = 0; lz < 4; ++lz) {
            const int64_t v = b * kBlockVox + col + 16 * lz;
            const unsigned c = counts[v];
            if (!c) continue;
            if (d >= max_voxels) { atomicAdd(ovf, 1ull); continue; }
            const float4 s = sums[v];
            const long long cz = bz * 4 + lz;
            okeys[d] = (int64_t)pack_cells(cx, cy, cz);
            const double w = s.w;
            cen[3 * d + 0] = (float)((double)cx * cell + (double)s.x / w);
            cen[3 * d + 1] = (float)((double)cy * cell + (double)s.y / w);
            cen[3 * d + 2] = (float)((double)cz * cell + (double)s.z / w);
            wsum[d] = s.w;
            cnt[d] = (int32_t)c;
            ++d;
        }
    }
}

struct ColWs {
    uint8_t* colcnt;
    int* bb;  // bounding box + overflow flag of the 32-bit keys
    uint32_t *skey32, *skey32_s;
    unsigned long long *skey, *skey_s;
    uint32_t *ids, *ids_s;
    ColGroup* grp;
    uint32_t *scan_in, *colsrc, *col_base;
    void* cub_tmp;
    size_t cub_bytes;
};

static size_t col_ws_layout(int64_t nb, char* base, ColWs* w) {
    size_t cs = 0, cc = 0, c32 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, cs, (unsigned long long*)nullptr, (unsigned long long*)nullptr,
                                    (uint32_t*)nullptr, (uint32_t*)nullptr, (int)nb, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, c32, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)nb, 0, 32);
    cs = std::max(cs, c32);
    cub::DeviceScan::ExclusiveSum(nullptr, cc, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(nb * 16 + 1));
    Carver cv{base, 0};
    ColWs t;
    t.colcnt = cv.take<uint8_t>(nb * 16);
    t.bb = cv.take<int>(8);
    t.skey32 = cv.take<uint32_t>(nb);
    t.skey32_s = cv.take<uint32_t>(nb);
    t.skey = cv.take<unsigned long long>(nb);
    t.skey_s = cv.take<unsigned long long>(nb);
    t.ids = cv.take<uint32_t>(nb);
    t.ids_s = cv.take<uint32_t>(nb);
    t.grp = cv.take<ColGroup>(nb);
    t.scan_in = cv.take<uint32_t>(nb * 16 + 1);
    t.colsrc = cv.take<uint32_t>(nb * 16);
    t.col_base = cv.take<uint32_t>(nb * 16 + 1);
    t.cub_bytes = std::max(cs, cc);
    t.cub_tmp = cv.take<char>(t.cub_bytes);
    if (w) *w = t;
    return cv.used;
}

// No host round trip until the end (the caller needs U): every launch is
// sized by the map's capacity and reads the used-block count on the device.
static int column_emit(ec3r_vhash* h, int64_t* keys, float* centroid, float* wsum, int32_t* count, int64_t* n_out,
                       void* workspace, size_t workspace_bytes, bool read_count, cudaStream_t st) {
    const int64_t nb = h->max_blocks;
    ColWs w;
    if (col_ws_layout(nb, (char*)workspace, &w) > workspace_bytes) return EC3R_EWORKSPACE;
    h->last_count = -1;
    // 32-bit sort keys (4 radix passes instead of 8) when the host knows the
    // map's block extent fit them at the last read-back; a map that outgrew
    // them is caught by the flag read below and re-emitted with 64-bit keys
    const bool k32 = h->emit_key32;  // fit established by an earlier host-read emit (checked on the device)
    EC3R_CUDA_TRY(cudaMemsetAsync(w.scan_in, 0, sizeof(uint32_t) * (size_t)(nb * 16 + 1), st));
    const unsigned gw = (unsigned)std::min<int64_t>((nb * 32 + 255) / 256, (int64_t)kNumSMs * 16);
    vc_block_prep_kernel<<<gw, 256, 0, st>>>(h->counts, h->block_keys, h->counters, nb, w.colcnt, w.skey, w.ids);
    EC3R_CHECK_LAUNCH("vc_block_prep_kernel");
    if (read_count || k32) {  // the box decides the next emit's key width (host read) / this emit's keys
        bbox_init_kernel<<<1, 32, 0, st>>>(w.bb);
        EC3R_CHECK_LAUNCH("bbox_init_kernel");
        const unsigned gb = (unsigned)std::min<int64_t>((nb + 255) / 256, (int64_t)kNumSMs * 4);
        vc_bbox_kernel<<<gb, 256, 0, st>>>(h->block_keys, h->counters, nb, w.bb);
        EC3R_CHECK_LAUNCH("vc_bbox_kernel");
    }
    const unsigned gt = (unsigned)std::min<int64_t>((nb + 255) / 256, (int64_t)kNumSMs * 8);
    size_t cb = w.cub_bytes;
    if (k32) {
        vc_key32_kernel<<<gt, 256, 0, st>>>(h->block_keys, h->counters, nb, w.bb, w.skey32, w.ids, read_count ? 0 : 1);
        EC3R_CHECK_LAUNCH("vc_key32_kernel");
        if (cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.skey32, w.skey32_s, w.ids, w.ids_s, (int)nb, 0, 32,
                                            st) != cudaSuccess) {
            set_last_error("cub::DeviceRadixSort::SortPairs(blocks, 32-bit)", cudaGetLastError());
            return EC3R_ECUDA;
        }
        count_launch();
        vc_groups_kernel<uint32_t><<<gt, 256, 0, st>>>(w.skey32_s, w.ids_s, h->counters, nb, VC_YB + VC_ZB, VC_ZB,
                                                       w.grp);
        EC3R_CHECK_LAUNCH("vc_groups_kernel");
    } else {
        if (cub::DeviceRadixSort::SortPairs(w.cub_tmp, cb, w.skey, w.skey_s, w.ids, w.ids_s, (int)nb, 0, 64, st) !=
            cudaSuccess) {
            set_last_error("cub::DeviceRadixSort::SortPairs(blocks)", cudaGetLastError());
            return EC3R_ECUDA;
        }
        count_launch();
        vc_groups_kernel<unsigned long long><<<gt, 256, 0, st>>>(w.skey_s, w.ids_s, h->counters, nb, 42, 21, w.grp);
        EC3R_CHECK_LAUNCH("vc_groups_kernel");
    }
    const unsigned gc = (unsigned)std::min<int64_t>((nb * 16 + 255) / 256, (int64_t)kNumSMs * 16);
    vc_colpos_kernel<<<gc, 256, 0, st>>>(w.grp, w.colcnt, h->counters, nb, w.scan_in, w.colsrc);
    EC3R_CHECK_LAUNCH("vc_colpos_kernel");
    cb = w.cub_bytes;
    if (cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.scan_in, w.col_base, (int)(nb * 16 + 1), st) != cudaSuccess) {
        set_last_error("cub::DeviceScan::ExclusiveSum(columns)", cudaGetLastError());
        return EC3R_ECUDA;
    }
    count_launch();
    vc_gather_kernel<<<gc, 256, 0, st>>>(h->sums, h->counts, h->block_keys, h->counters, nb, w.colsrc, w.scan_in,
                                         w.col_base, h->max_voxels, h->cell, keys, centroid, wsum, count,
                                         h->counters + 5, n_out);
    EC3R_CHECK_LAUNCH("vc_gather_kernel");
    if (!read_count) return EC3R_OK;  // *n_out (device) holds U
    int64_t U = 0;
    int bb[8];
    EC3R_CUDA_TRY(cudaMemcpyAsync(&U, n_out, sizeof(U), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaMemcpyAsync(bb, w.bb, sizeof(bb), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    const bool fits = bb[0] > bb[3] || ((unsigned)(bb[3] - bb[0]) < (1u << VC_XB) &&
                                        (unsigned)(bb[4] - bb[1]) < (1u << VC_YB) &&
                                        (unsigned)(bb[5] - bb[2]) < (1u << VC_ZB));
    h->emit_key32 = fits;
    if (k32 && !fits)  // the map outgrew the 32-bit keys since the last emit: redo with 64-bit keys
        return column_emit(h, keys, centroid, wsum, count, n_out, workspace, workspace_bytes, read_count, st);
    h->last_count = U;
    return EC3R_OK;
}


// Fixed-slab partials for a host-sync-free all-to-all: owner r's rows go to
// [r * cap, r * cap + min(count_r, cap)); rows past a full slab are counted
// in *overflow (the caller re-runs with a larger cap).  slab_counts[r] =
// min(count_r, cap) after the launch.
__global__ void vb_partition_fixed_kernel(const float4* __restrict__ sums, const unsigned int* __restrict__ counts,
                                          const unsigned long long* __restrict__ keys,
                                          const int64_t* __restrict__ idx, const int64_t* __restrict__ n_ptr,
                                          int n_ranks, int64_t cap, unsigned long long* __restrict__ cursors,
                                          int64_t* __restrict__ okeys, float* __restrict__ sums4,
                                          int32_t* __restrict__ cnt, unsigned long long* __restrict__ overflow) {
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        const int r = (int)(mix64(k) % (unsigned long long)n_ranks);
        const unsigned peers = __match_any_sync(__activemask(), r);
        const int lead = __ffs(peers) - 1;
        const unsigned lanes_below = peers & ((1u << (threadIdx.x & 31)) - 1u);
        unsigned long long base = 0;
        if ((int)(threadIdx.x & 31) == lead) base = atomicAdd(&cursors[r], (unsigned long long)__popc(peers));
        base = __shfl_sync(peers, base, lead);
        const unsigned long long pos = base + __popc(lanes_below);
        if ((int64_t)pos >= cap) {
            atomicAdd(overflow, 1ull);
            continue;
        }
        const int64_t o = (int64_t)r * cap + (int64_t)pos;
        okeys[o] = (int64_t)k;
        reinterpret_cast<float4*>(sums4)[o] = sums[idx[i]];
        cnt[o] = (int32_t)counts[idx[i]];
    }
}

__global__ void vb_slab_counts_kernel(const unsigned long long* __restrict__ cursors, int n_ranks, int64_t cap,
                                      int64_t* __restrict__ slab_counts) {
    const int r = threadIdx.x;
    if (r < n_ranks) slab_counts[r] = min((int64_t)cursors[r], cap);
}

// merge received slabs: row i of slab s is valid iff i < slab_counts[s]
__global__ void vb_merge_slabs_kernel(const int64_t* __restrict__ keys, const float* __restrict__ sums4,
                                      const int32_t* __restrict__ cnt, int n_slabs, int64_t cap,
                                      const int64_t* __restrict__ slab_counts, VB vb) {
    const int64_t n = (int64_t)n_slabs * cap;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const int64_t i = i0 + threadIdx.x;
        bool valid = i < n;
        if (valid) {
            const int64_t sl = i / cap;
            valid = (i - sl * cap) < slab_counts[sl];
        }
        long long cx = 0, cy = 0, cz = 0;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned c = 0;
        if (valid) {
            unpack_cells((unsigned long long)keys[i], cx, cy, cz);
            s = reinterpret_cast<const float4*>(sums4)[i];
            c = (unsigned)cnt[i];
        }
        unsigned long long cbk = kEmpty;
        int cidx = -2;
        if (vb_insert_warp(vb, valid, cx, cy, cz, s.x, s.y, s.z, s.w, c, cbk, cidx))
            atomicAdd(&vb.counters[2], 1ull);
    }
}

}  // namespace ec3r

using namespace ec3r;

static int mixed_error() {
    set_last_error_msg("ec3r_vhash: frame/point inserts and partial merges cannot share a map between clears");
    return EC3R_EARG;
}

extern "C" int ec3r_vhash_create_sized(ec3r_vhash** out, int64_t max_voxels, int64_t max_blocks,
                                       int64_t table_entries, double cell_size, void* stream) {
    if (!out || max_voxels < 2 || max_blocks < 1 || !(cell_size > 0)) return EC3R_EARG;
    ec3r_vhash* h = new ec3r_vhash();
    h->last_count = -1;
    h->emit_key32 = false;
    h->bf = nullptr;
    h->bf_active = h->legacy_active = false;
    {
        // Engine: the binned super-block engine (vbin.cu: sort-based,
        // atomic-free per point, deterministic integer sums) for cells up to
        // 2.56 cm, where its cell/256 offset quantisation keeps centroids
        // within 50 um; the voxel-block hash otherwise.  EC3R_FUSE_ENGINE=hash
        // forces the block hash, =binned the binned engine where it applies.
        const char* e = getenv("EC3R_FUSE_ENGINE");
        const bool want = e && std::string(e) == "binned";
        h->binned = want && cell_size <= 0.0256;
    }
    h->max_voxels = max_voxels > 65536 ? max_voxels : 65536;
    h->max_blocks = max_blocks > 4096 ? max_blocks : 4096;
    // frame fusion addresses voxels as 32-bit (block << 6 | local) ids
    if (h->max_blocks > (1 << 26) - 2) h->max_blocks = (1 << 26) - 2;
    // table: a power of two >= 2x the pool (or the caller's, larger, choice:
    // a sparse table inserts faster — concurrent first touches of neighbouring
    // blocks contend less for L2 lines)
    int64_t tcap = 1;
    const int64_t want = table_entries > 2 * h->max_blocks ? table_entries : 2 * h->max_blocks;
    while (tcap < want) tcap <<= 1;
    if (tcap > (int64_t)1 << 32) return EC3R_EARG;
    h->tmask = (unsigned long long)(tcap - 1);
    h->cell = cell_size;
    const size_t nv = (size_t)h->max_blocks * kBlockVox;
    bool ok = cudaMalloc(&h->table, sizeof(BlockEntry) * (size_t)tcap) == cudaSuccess &&
              cudaMalloc(&h->block_keys, sizeof(unsigned long long) * (size_t)h->max_blocks) == cudaSuccess &&
              cudaMalloc(&h->block_slot, sizeof(uint32_t) * (size_t)h->max_blocks) == cudaSuccess &&
              cudaMalloc(&h->sums, sizeof(float4) * nv) == cudaSuccess &&
              cudaMalloc(&h->counts, sizeof(unsigned int) * nv) == cudaSuccess &&
              cudaMalloc(&h->counters, sizeof(unsigned long long) * 8) == cudaSuccess;
    if (!ok) {
        set_last_error("cudaMalloc(vhash)", cudaGetLastError());
        cudaFree(h->table); cudaFree(h->block_keys); cudaFree(h->block_slot); cudaFree(h->sums); cudaFree(h->counts); cudaFree(h->counters);
        delete h;
        return EC3R_ENOMEM;
    }
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemsetAsync(h->sums, 0, sizeof(float4) * nv, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(h->counts, 0, sizeof(unsigned int) * nv, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(h->counters, 0, sizeof(unsigned long long) * 8, st));
    // the whole table starts empty (later clears touch only the used entries)
    vb_clear_table_kernel<<<(unsigned)((tcap + 255) / 256), 256, 0, st>>>(h->table, tcap);
    EC3R_CHECK_LAUNCH("vb_clear_table_kernel");
    if (h->binned) {
        int rc = EC3R_OK;
        h->bf = bf_create(h->max_voxels, h->max_blocks, cell_size, st, &rc);
        if (!h->bf) {
            ec3r_vhash_destroy(h);
            return rc;
        }
    }
    *out = h;
    return EC3R_OK;
}

// capacity = voxels to emit at most; the pool holds capacity / 4 blocks
// (surface blocks are far fuller than 4 of 64 voxels; sparse inputs
// overflow, are reported and re-run on a larger handle)
extern "C" int ec3r_vhash_create(ec3r_vhash** out, int64_t capacity, double cell_size, void* stream) {
    if (capacity < 2) return EC3R_EARG;
    return ec3r_vhash_create_sized(out, capacity, capacity / 4 > 1 ? capacity / 4 : 1, 0, cell_size, stream);
}

extern "C" int ec3r_vhash_destroy(ec3r_vhash* h) {
    if (!h) return EC3R_OK;
    cudaFree(h->table);
    cudaFree(h->block_keys);
    cudaFree(h->block_slot);
    cudaFree(h->sums);
    cudaFree(h->counts);
    cudaFree(h->counters);
    cudaFree(h->ftab);
    bf_destroy(h->bf);
    delete h;
    return EC3R_OK;
}

extern "C" int64_t ec3r_vhash_capacity(const ec3r_vhash* h) { return h ? h->max_voxels : 0; }

extern "C" int ec3r_vhash_clear(ec3r_vhash* h, void* stream) {
    if (!h) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    const int64_t tcap = (int64_t)h->tmask + 1;
    // only the entries and pool blocks the last fill used (the whole table
    // when that fill overflowed the pool and left unallocated entries)
    vb_clear_used_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->table, tcap, h->block_slot, h->sums, h->counts, h->counters,
                                                      h->max_blocks);
    EC3R_CHECK_LAUNCH("vb_clear_used_kernel");
    EC3R_CUDA_TRY(cudaMemsetAsync(h->counters, 0, sizeof(unsigned long long) * 8, st));
    h->last_count = -1;
    h->legacy_active = false;
    if (h->bf) {
        const int rc = bf_clear(h->bf, st);
        if (rc) return rc;
    }
    h->bf_active = false;
    return EC3R_OK;
}

extern "C" int ec3r_vhash_insert_frames(ec3r_vhash* h, const float* depth_pool, const float* conf_pool, int H, int W,
                                        const double* K4_h, const double* slot_poses, const double* slot_globals,
                                        const int32_t* slots, int n, void* stream) {
    if (!h || H <= 0 || W <= 0 || !K4_h || n < 0) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    FuseArgs a;
    a.depth = depth_pool; a.conf = conf_pool; a.slot_poses = slot_poses; a.slot_globals = slot_globals;
    a.slots = slots; a.n = n; a.H = H; a.W = W;
    a.fx = K4_h[0]; a.fy = K4_h[1]; a.cx = K4_h[2]; a.cy = K4_h[3];
    a.cell = h->cell; a.inv_cell_f = (float)(1.0 / h->cell); a.cell_f = (float)h->cell;
    a.vb = vb_of(h);
    const int64_t need = (int64_t)n * (W + H + 1);
    if (need > h->ftab_cap) {  // grows once per workload shape
        cudaFree(h->ftab);
        h->ftab = nullptr;
        h->ftab_cap = 0;
        if (cudaMalloc(&h->ftab, sizeof(float4) * (size_t)need) != cudaSuccess) {
            set_last_error("cudaMalloc(vhash frame tables)", cudaGetLastError());
            return EC3R_ENOMEM;
        }
        h->ftab_cap = need;
    }
    a.ftab = h->ftab;
    cudaStream_t st = as_stream(stream);
    vh_frame_tables_kernel<<<n, 256, 0, st>>>(a, h->ftab);
    EC3R_CHECK_LAUNCH("vh_frame_tables_kernel");
    if (h->bf) {
        if (h->legacy_active) return mixed_error();
        h->bf_active = true;
        return bf_insert_frames(h->bf, a, st);
    }
    h->legacy_active = true;
    const size_t smem = sizeof(float4) * (size_t)W;
    if (smem > 48 * 1024)
        EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel<false, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // TMA strip ring: 2 stages x 2 planes x 8 rows of W floats after A[W]
    const size_t smem_tma = smem + sizeof(float) * 2 * 2 * ST_H * (size_t)W;
    const bool tma = FI_G == 1 && ((int64_t)H * W) % 4 == 0 &&
                     ((reinterpret_cast<uintptr_t>(depth_pool) | reinterpret_cast<uintptr_t>(conf_pool)) & 15) == 0 &&
                     smem_tma <= 160 * 1024 && tma_requested();
    if (tma) {
        EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel<false, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tma));
        EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel<true, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tma));
    }
    const dim3 grid((H + FI_ROWS - 1) / FI_ROWS, (n + FI_G - 1) / FI_G);
    a.log_runs = nullptr; a.log_n = nullptr; a.log_cap = 0;
    if (h->diag_runs) {  // diagnostic: log this insert's runs instead of reducing (one call)
        a.log_runs = h->diag_runs; a.log_n = h->diag_n; a.log_cap = (unsigned long long)h->diag_cap;
        h->diag_runs = nullptr; h->diag_n = nullptr; h->diag_cap = 0;
        if (tma) vh_insert_frames_kernel<true, true><<<grid, FI_NT, smem_tma, st>>>(a);
        else {
            if (smem > 48 * 1024)
                EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel<true, false>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            vh_insert_frames_kernel<true, false><<<grid, FI_NT, smem, st>>>(a);
        }
        EC3R_CHECK_LAUNCH("vh_insert_frames_kernel<log>");
        return EC3R_OK;
    }
    // CTA size: 128-thread CTAs (4 per SM, the same 16 warps and register
    // budget) when the launch is long enough that their finer granularity
    // pays; 256-thread CTAs when 128-thread ones would leave a heavy last
    // wave (measured, profiles/r02g24_fusion_cta_size.json: configs[3], 21
    // waves of 128: 5.31 vs 5.55 ms; configs[4] shard, 7.0 waves: 1.655 vs
    // 1.70 ms; configs[1], 4.3 waves: 1.255 vs 1.20 ms).
    // EC3R_FI_NT128=0/1 forces either form.
    const int64_t ctas = (int64_t)grid.x * grid.y;
    bool small = ctas >= (int64_t)kSmallCtaWaves * 4 * kNumSMs;
    if (const char* e = getenv("EC3R_FI_NT128")) small = e[0] == '1';
    KernelTimer tk(TK_FUSE_INSERT, st);
    if (tma) vh_insert_frames_kernel<false, true><<<grid, FI_NT, smem_tma, st>>>(a);
    else if (small) {
        if (smem > 48 * 1024)
            EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel<false, false, 128>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        vh_insert_frames_kernel<false, false, 128><<<grid, 128, smem, st>>>(a);
    } else vh_insert_frames_kernel<false, false><<<grid, FI_NT, smem, st>>>(a);
    EC3R_CHECK_LAUNCH("vh_insert_frames_kernel");
    tk.stop();
    return EC3R_OK;
}

extern "C" int ec3r_vhash_insert_points(ec3r_vhash* h, const double* points, const double* conf, int64_t n,
                                        const double* sim3_h, void* stream) {
    if (!h || n < 0 || !sim3_h) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    if (h->bf) {
        if (h->legacy_active) return mixed_error();
        h->bf_active = true;
        return bf_insert_points(h->bf, points, conf, n, sim3_h, as_stream(stream));
    }
    h->legacy_active = true;
    Sim3Arg g;
    for (int k = 0; k < 8; ++k) g.v[k] = sim3_h[k];
    vh_insert_points_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(points, conf, n, g, h->cell, vb_of(h));
    EC3R_CHECK_LAUNCH("vh_insert_points_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_stats_get(ec3r_vhash* h, ec3r_vhash_stats* out_h, void* stream) {
    if (!h || !out_h) return EC3R_EARG;
    if (h->bf_active) {
        int64_t v[5];
        const int rc = bf_stats(h->bf, v, as_stream(stream));
        if (rc) return rc;
        out_h->n_points_in = v[0];
        out_h->n_out_of_range = v[1];
        out_h->n_overflow = v[2];
        out_h->n_slow_path = v[3];
        out_h->n_blocks = v[4];
        return EC3R_OK;
    }
    unsigned long long c[8];
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemcpyAsync(c, h->counters, sizeof(c), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    out_h->n_points_in = (int64_t)c[0];
    out_h->n_out_of_range = (int64_t)c[1];
    out_h->n_overflow = (int64_t)(c[2] + c[5]);  // dropped points + voxels beyond the emit capacity
    out_h->n_slow_path = (int64_t)c[3];
    out_h->n_blocks = (int64_t)(c[4] < (unsigned long long)h->max_blocks ? c[4] : (unsigned long long)h->max_blocks);
    return EC3R_OK;
}

__global__ void vb_count_kernel(const unsigned int* __restrict__ counts, const unsigned long long* __restrict__ counters,
                                int64_t max_blocks, unsigned long long* __restrict__ out) {
    const int64_t n = min((int64_t)counters[4], max_blocks) * kBlockVox;
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += counts[i] != 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

extern "C" int ec3r_vhash_count(ec3r_vhash* h, int64_t* n_out, void* stream) {
    if (!h || !n_out) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    if (h->bf_active) {
        int64_t U = 0;
        const int rc = bf_count(h->bf, &U, st);
        if (rc) return rc;
        EC3R_CUDA_TRY(cudaMemcpyAsync(n_out, &U, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        return EC3R_OK;
    }
    EC3R_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int64_t), st));
    vb_count_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->counts, h->counters, h->max_blocks, (unsigned long long*)n_out);
    EC3R_CHECK_LAUNCH("vb_count_kernel");
    return EC3R_OK;
}

extern "C" size_t ec3r_vhash_extract_workspace(const ec3r_vhash* h) {
    if (!h) return 0;
    const size_t cap = (size_t)h->max_voxels;
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs<unsigned long long, int64_t>(nullptr, cub_bytes, (unsigned long long*)nullptr,
                                                                 (unsigned long long*)nullptr, (int64_t*)nullptr,
                                                                 (int64_t*)nullptr, (int)cap, 0, 63);
    size_t cub32 = 0;
    cub::DeviceRadixSort::SortPairs<uint32_t, uint32_t>(nullptr, cub32, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                                        (uint32_t*)nullptr, (uint32_t*)nullptr, (int)cap, 0, 32);
    if (cub32 > cub_bytes) cub_bytes = cub32;
    const int64_t nb = h->max_blocks;
    const size_t legacy = 4 * align256(sizeof(int64_t) * cap) + align256(64) +
                          2 * align256(sizeof(int) * (size_t)(nb + 1)) + align256(scan_temp_bytes(nb + 1)) +
                          align256(cub_bytes);
    return std::max(legacy, col_ws_layout(nb, nullptr, nullptr));
}

extern "C" int ec3r_vhash_extract(ec3r_vhash* h, int64_t* keys, float* centroid, float* wsum, int32_t* count,
                                  int64_t* n_out, int sort, void* workspace, size_t workspace_bytes, void* stream) {
    if (!h || !keys || !centroid || !wsum || !count || !n_out) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    if (h->bf_active) {  // always key-sorted; the workspace is the engine's own
        int64_t U = -1;
        const int rc = bf_extract(h->bf, keys, centroid, wsum, count, n_out, &U, st);
        h->last_count = U;
        return rc;
    }
    if (!workspace || workspace_bytes < ec3r_vhash_extract_workspace(h)) return EC3R_EWORKSPACE;
    if (sort && !getenv("EC3R_EMIT_VOXEL_SORT"))
        return column_emit(h, keys, centroid, wsum, count, n_out, workspace, workspace_bytes, sort != 2, st);
    const unsigned long long* ks;
    const int64_t* is;
    const uint32_t* i32;
    const int rc = compact_sorted(h, sort, workspace, workspace_bytes, n_out, &ks, &is, &i32, st);
    if (rc) return rc;
    if (i32) {
        vb_gather32_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->sums, h->counts, h->block_keys, i32, n_out, h->cell, keys,
                                                        centroid, wsum, count);
        EC3R_CHECK_LAUNCH("vb_gather32_kernel");
        return EC3R_OK;
    }
    vb_gather_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->sums, h->counts, ks, is, n_out, h->cell, keys, centroid, wsum,
                                                  count);
    EC3R_CHECK_LAUNCH("vb_gather_kernel");
    return EC3R_OK;
}

// Voxel count of the last sorted ec3r_vhash_extract on this handle (the
// library read it on the host to size the sort), or -1.  Saves the caller a
// device round trip.
extern "C" int64_t ec3r_vhash_extract_count(const ec3r_vhash* h) { return h ? h->last_count : -1; }

extern "C" int ec3r_vhash_extract_partials(ec3r_vhash* h, int n_ranks, int64_t* keys, float* sums4, int32_t* count,
                                           int64_t* rank_counts, void* workspace, size_t workspace_bytes,
                                           void* stream) {
    if (!h || n_ranks < 1 || n_ranks > 64 || !keys || !sums4 || !count || !rank_counts) return EC3R_EARG;
    if (h->bf_active) return bf_extract_partials(h->bf, n_ranks, keys, sums4, count, rank_counts, as_stream(stream));
    const size_t need = ec3r_vhash_extract_workspace(h) + 4 * align256(sizeof(unsigned long long) * n_ranks);
    if (!workspace || workspace_bytes < need) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    Carver cv{(char*)workspace, 0};
    unsigned long long* base = cv.take<unsigned long long>(n_ranks);
    unsigned long long* cursors = cv.take<unsigned long long>(n_ranks);
    int64_t* n_dev = cv.take<int64_t>(1);
    void* cws = cv.base + cv.used;
    const unsigned long long* ks;
    const int64_t* is;
    const uint32_t* i32;
    const int rc = compact_sorted(h, 0, cws, workspace_bytes - cv.used, n_dev, &ks, &is, &i32, st);
    if (rc) return rc;
    EC3R_CUDA_TRY(cudaMemsetAsync(rank_counts, 0, sizeof(int64_t) * n_ranks, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(cursors, 0, sizeof(unsigned long long) * n_ranks, st));
    vb_partition_count_kernel<<<kNumSMs * 8, 256, 0, st>>>(ks, n_dev, n_ranks, (unsigned long long*)rank_counts);
    EC3R_CHECK_LAUNCH("vb_partition_count_kernel");
    std::vector<unsigned long long> rc_h(n_ranks), rb(n_ranks);
    EC3R_CUDA_TRY(cudaMemcpyAsync(rc_h.data(), rank_counts, sizeof(int64_t) * n_ranks, cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long acc = 0;
    for (int r = 0; r < n_ranks; ++r) { rb[r] = acc; acc += rc_h[r]; }
    EC3R_CUDA_TRY(cudaMemcpyAsync(base, rb.data(), sizeof(unsigned long long) * n_ranks, cudaMemcpyHostToDevice, st));
    vb_partition_write_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->sums, h->counts, ks, is, n_dev, n_ranks, base, cursors,
                                                           keys, sums4, count);
    EC3R_CHECK_LAUNCH("vb_partition_write_kernel");
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));  // rb is a host temporary
    return EC3R_OK;
}

extern "C" int ec3r_vhash_merge_partials(ec3r_vhash* h, const int64_t* keys, const float* sums4, const int32_t* count,
                                         int64_t n, void* stream) {
    if (!h || n < 0) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    if (h->bf_active) return mixed_error();
    h->legacy_active = true;
    vb_merge_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(keys, sums4, count, n, vb_of(h));
    EC3R_CHECK_LAUNCH("vb_merge_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_extract_partials_fixed(ec3r_vhash* h, int n_ranks, int64_t cap, int64_t* keys, float* sums4,
                                                 int32_t* count, int64_t* slab_counts, int64_t* overflow,
                                                 void* workspace, size_t workspace_bytes, void* stream) {
    if (!h || n_ranks < 1 || n_ranks > 1024 || cap < 1 || !keys || !sums4 || !count || !slab_counts || !overflow)
        return EC3R_EARG;
    if (h->bf_active) {
        set_last_error_msg("ec3r_vhash_extract_partials_fixed: the binned engine emits partials with a host count "
                           "(ec3r_vhash_extract_partials)");
        return EC3R_EARG;
    }
    const size_t need = ec3r_vhash_extract_workspace(h) + 2 * align256(sizeof(unsigned long long) * n_ranks) + 1024;
    if (!workspace || workspace_bytes < need) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    Carver cv{(char*)workspace, 0};
    unsigned long long* cursors = cv.take<unsigned long long>(n_ranks);
    int64_t* n_dev = cv.take<int64_t>(1);
    void* cws = cv.base + cv.used;
    const unsigned long long* ks;
    const int64_t* is;
    const uint32_t* i32;
    const int rc = compact_sorted(h, 0, cws, workspace_bytes - cv.used, n_dev, &ks, &is, &i32, st);
    if (rc) return rc;
    EC3R_CUDA_TRY(cudaMemsetAsync(cursors, 0, sizeof(unsigned long long) * n_ranks, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(overflow, 0, sizeof(int64_t), st));
    vb_partition_fixed_kernel<<<kNumSMs * 8, 256, 0, st>>>(h->sums, h->counts, ks, is, n_dev, n_ranks, cap, cursors,
                                                           keys, sums4, count, (unsigned long long*)overflow);
    EC3R_CHECK_LAUNCH("vb_partition_fixed_kernel");
    vb_slab_counts_kernel<<<1, 1024, 0, st>>>(cursors, n_ranks, cap, slab_counts);
    EC3R_CHECK_LAUNCH("vb_slab_counts_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_merge_partials_slabs(ec3r_vhash* h, const int64_t* keys, const float* sums4,
                                               const int32_t* count, int n_slabs, int64_t cap,
                                               const int64_t* slab_counts, void* stream) {
    if (!h || n_slabs < 1 || cap < 1 || !keys || !sums4 || !count || !slab_counts) return EC3R_EARG;
    if (h->bf_active) return mixed_error();
    h->legacy_active = true;
    vb_merge_slabs_kernel<<<grid_for((int64_t)n_slabs * cap), 256, 0, as_stream(stream)>>>(keys, sums4, count, n_slabs,
                                                                                          cap, slab_counts, vb_of(h));
    EC3R_CHECK_LAUNCH("vb_merge_slabs_kernel");
    return EC3R_OK;
}

// Device-side map counters (n_points_in, n_out_of_range, n_overflow (dropped
// points + voxels past the emit capacity), n_slow_path, n_blocks) into a
// caller device buffer of 5 int64, without a host round trip.
__global__ void vb_stats_dev_kernel(const unsigned long long* __restrict__ c, int64_t max_blocks,
                                    int64_t* __restrict__ out) {
    if (threadIdx.x == 0) {
        out[0] = (int64_t)c[0];
        out[1] = (int64_t)c[1];
        out[2] = (int64_t)(c[2] + c[5]);
        out[3] = (int64_t)c[3];
        out[4] = (int64_t)min(c[4], (unsigned long long)max_blocks);
    }
}

extern "C" int ec3r_vhash_stats_device(ec3r_vhash* h, int64_t* out5, void* stream) {
    if (!h || !out5) return EC3R_EARG;
    if (h->bf_active) {
        set_last_error_msg("ec3r_vhash_stats_device: block-hash maps only");
        return EC3R_EARG;
    }
    vb_stats_dev_kernel<<<1, 32, 0, as_stream(stream)>>>(h->counters, h->max_blocks, out5);
    EC3R_CHECK_LAUNCH("vb_stats_dev_kernel");
    return EC3R_OK;
}


// ---------------------------------------------------------------------------
// Reduction-floor diagnostic (bench.py extras, tools/fuse_timing.py).
// ec3r_vhash_diag_log arms the next ec3r_vhash_insert_frames call to write
// its runs' (pool voxel, count) pairs, in issue order, to runs[0..cap) with
// *n_dev counting them (the map itself is left unchanged); *n_dev must be
// zero.  ec3r_vhash_diag_replay issues exactly those reductions into the
// map's pool (with_count = 0: the float4 sums only) and nothing else.

extern "C" int ec3r_vhash_diag_log(ec3r_vhash* h, void* runs, int64_t cap, unsigned long long* n_dev) {
    if (!h || !runs || !n_dev || cap <= 0) return EC3R_EARG;
    if (h->bf) return EC3R_EARG;  // the block-hash engine's reductions only (the binned engine has none)
    h->diag_runs = static_cast<uint2*>(runs);
    h->diag_n = n_dev;
    h->diag_cap = cap;
    return EC3R_OK;
}

extern "C" int ec3r_vhash_diag_replay(ec3r_vhash* h, const void* runs, const unsigned long long* n_dev, int64_t cap,
                                      int with_count, void* stream) {
    if (!h || !runs || !n_dev || cap <= 0) return EC3R_EARG;
    ec3r::vh_replay_runs_kernel<<<ec3r::kNumSMs * 8, 256, 0, as_stream(stream)>>>(
        static_cast<const uint2*>(runs), n_dev, (unsigned long long)cap, h->sums, h->counts, with_count);
    EC3R_CHECK_LAUNCH("vh_replay_runs_kernel");
    return EC3R_OK;
}
