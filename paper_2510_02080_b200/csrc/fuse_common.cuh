// Shared pieces of the stage-(c) fusion kernels (vhash.cu: voxel-block hash,
// vbin.cu: binned super-block fusion): _pack keys, the per-frame float32
// affine tables and the exact-by-construction voxel cells of a pixel.
//
// Keys are _pack(floor(x / cell)) (_kernels/_numpy.py:50-55) of the
// reference's float64 chain  x = G.apply(P_f.apply(ray))  (backend.py:89-90,
// liegroups.py:90-95,208-209,259-260).  Fast path: the composite G o P_f is
// folded per frame into x = z * (A[u] + B[v]) + T (float32, 3 FADD + 3 FFMA
// per pixel); when a coordinate lies within the fold's rounding bound of a
// voxel face the pixel re-runs the exact float64 sequence, so cells are
// bit-exact.
#pragma once

#include "common.cuh"

namespace ec3r {

constexpr unsigned long long kEmpty = ~0ull;  // never a _pack key (max is 2^63-1)
constexpr int64_t kPackOffset = 1 << 20;

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// table position of a key: a 32-bit mix (tables have < 2^32 entries)
__device__ __forceinline__ unsigned long long table_slot(unsigned long long bk, unsigned long long tmask) {
    uint32_t h = (uint32_t)bk * 0x9E3779B1u ^ (uint32_t)(bk >> 32) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return (unsigned long long)h & tmask;
}

__host__ __device__ __forceinline__ unsigned long long pack_cells(long long cx, long long cy, long long cz) {
    return ((unsigned long long)(cx + kPackOffset) << 42) | ((unsigned long long)(cy + kPackOffset) << 21) |
           (unsigned long long)(cz + kPackOffset);
}

// pack_cells of int32 coordinates with 32-bit operations
__device__ __forceinline__ unsigned long long pack_block(int bx, int by, int bz) {
    const unsigned X = (unsigned)(bx + (int)kPackOffset), Y = (unsigned)(by + (int)kPackOffset),
                   Z = (unsigned)(bz + (int)kPackOffset);
    const unsigned lo = (Y << 21) | Z, hi = (X << 10) | (Y >> 11);
    return ((unsigned long long)hi << 32) | lo;
}

__host__ __device__ __forceinline__ void unpack_cells(unsigned long long k, long long& cx, long long& cy,
                                                      long long& cz) {
    cx = (long long)((k >> 42) & 0x1FFFFF) - kPackOffset;
    cy = (long long)((k >> 21) & 0x1FFFFF) - kPackOffset;
    cz = (long long)(k & 0x1FFFFF) - kPackOffset;
}

__device__ __forceinline__ bool cell_in_range(long long c) { return c >= -kPackOffset && c < kPackOffset; }

// Frame geometry of a fusion launch: the resident pool, the listed slots and
// their affine tables.
struct FrameGeom {
    const float* depth;
    const float* conf;
    const double* slot_poses;    // anchor_from_cam per slot
    const double* slot_globals;  // world_from_anchor (submap global Sim3) per slot
    const int32_t* slots;        // slot ids to fuse
    const float4* ftab;          // per listed frame: A[W], B[H], T (see vh_frame_tables_kernel)
    int n, H, W;
    double fx, fy, cx, cy;
    double cell;
    float inv_cell_f, cell_f;
};

// Per listed frame j, the composite G o P_f folded into a float32 affine map
// x = z * (A[u] + B[v]) + T: A[u] = M[:,0] x_u + M[:,2], B[v] = M[:,1] y_v,
// each with its |.|-sum in .w for the rounding bound; T = (t, |t|-sum).
// (defined in vhash.cu)
__global__ void vh_frame_tables_kernel(FrameGeom a, float4* __restrict__ ftab);

// Exact reference chain for one pixel: cells of  G.apply(P.apply(ray)).
// Out of line by default (rare path, keeps the caller's registers free);
// EC3R_EXACT_INLINE=1 inlines it (needed under tight register caps).
#if defined(EC3R_EXACT_INLINE) && EC3R_EXACT_INLINE
#define EC3R_EXACT_ATTR __forceinline__
#else
#define EC3R_EXACT_ATTR __noinline__ inline
#endif
__device__ EC3R_EXACT_ATTR void exact_cells(const double* P, const double* G, double xcoef, double ycoef,
                                                float zf, double cell, long long c[3]) {
    const double z = (double)zf;
    const double ray[3] = {xm(xcoef, z), xm(ycoef, z), z};
    double pa[3], pw[3];
    pose_apply_exact(P, ray, pa);
    sim3_apply_exact(G, pa, pw);
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = (long long)floor(__ddiv_rn(pw[k], cell));
}

// Cells of four horizontally adjacent pixels (u0..u0+3, row v) of listed
// frame slot `slot`: valid = depth > 0 and conf > 0 (backend.py:87,262 and the
// fusion rule's conf > 0); (x, y, z) are the float32 fast-path coordinates
// (used for the in-voxel offsets), (cx, cy, cz) the exact cells.  Counters:
// n_in valid pixels, n_oor cells outside the _pack range (dropped), n_slow
// exact re-runs.
struct Cells4 {
    bool valid[4];
    int cx[4], cy[4], cz[4];
    float x[4], y[4], z[4];
};

__device__ __forceinline__ void frame_cells4(const FrameGeom& a, const float4* sA, float4 Bv, float4 Tm, int slot,
                                             int u0, int v, const float (&zs)[4], const float (&cs)[4], Cells4& o,
                                             unsigned& n_in, unsigned& n_oor, unsigned& n_slow) {
    const float inv = a.inv_cell_f;
    const int W = a.W;
    unsigned slow = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float z = zs[k], c = cs[k];
        const float4 Au = sA[min(u0 + k, W - 1)];  // columns past W are masked below
        const float dx = Au.x + Bv.x, dy = Au.y + Bv.y, dz = Au.z + Bv.z;
        const float x = fmaf(z, dx, Tm.x), y = fmaf(z, dy, Tm.y), zz = fmaf(z, dz, Tm.z);
        // first-order float32 error bound (x4 safety) + 1 ulp(0.5) for the
        // folded face test below
        const float ax = fabsf(x) + fabsf(y) + fabsf(zz);
        const float err = 2.384185791015625e-07f * (2.0f * z * (Au.w + Bv.w) + Tm.w + 2.0f * ax) + 1e-9f;
        const float margin = err * inv + 3.6e-7f;
        const float qx = x * inv, qy = y * inv, qz = zz * inv;
        const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
        // |frac - 1/2| > 1/2 - margin  <=>  within margin of a face
        const float dev = fmaxf(fmaxf(fabsf(qx - fx - 0.5f), fabsf(qy - fy - 0.5f)), fabsf(qz - fz - 0.5f));
        const float qmax = fmaxf(fmaxf(fabsf(qx), fabsf(qy)), fabsf(qz));
        o.valid[k] = z > 0.f && c > 0.f && u0 + k < W;
        n_in += o.valid[k];
        if (o.valid[k] && !(dev < 0.5f - margin && qmax <= 1.0e6f)) slow |= 1u << k;
        // |q| <= 1e6 < 2^20: fast-path cells are always inside the key range
        o.cx[k] = (int)fx; o.cy[k] = (int)fy; o.cz[k] = (int)fz;
        o.x[k] = x; o.y[k] = y; o.z[k] = zz;
    }
    if (slow) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!(slow & (1u << k))) continue;
            long long cc[3];
            exact_cells(a.slot_poses + 8 * slot, a.slot_globals + 8 * slot, ray_coef(u0 + k, a.cx, a.fx),
                        ray_coef(v, a.cy, a.fy), zs[k], a.cell, cc);
            ++n_slow;
            if (cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2])) {
                o.cx[k] = (int)cc[0]; o.cy[k] = (int)cc[1]; o.cz[k] = (int)cc[2];
            } else {
                ++n_oor;
                o.valid[k] = false;
            }
        }
    }
}

}  // namespace ec3r
