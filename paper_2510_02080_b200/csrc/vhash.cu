// K1+K4: Sim(3) transform + open-addressing voxel-hash fusion + downsample
// emit, on sm_100a.
//
// Replaces Submap.world_points / Mapping.fused_cloud (mapping.py:56-57,
// 332-338) under the declared fusion rule of oracle/fuse.py.  Keys are
// _pack(floor(x / cell)) (_kernels/_numpy.py:50-55) and must be bit-exact
// against the reference's float64 chain  x = G.apply(P_f.apply(ray))
// (backend.py:89-90, liegroups.py:90-95,208-209,259-260).
//
// Fast path (every pixel): the composite G o P_f is folded per frame into a
// float32 affine map evaluated as  x = z * (A[u] + B[v]) + T  (A, B are
// per-column / per-row tables in shared memory), i.e. 3 FADD + 3 FFMA per
// pixel instead of ~70 float64 operations.  Its rounding error is bounded
// per pixel; when a coordinate lies within that bound of a voxel boundary
// the pixel re-runs the reference's exact float64 sequence (slow path,
// ~0.1% of pixels), so keys are bit-exact by construction.  Accumulators are
// float32 sums of conf * (x - voxel corner), so centroids keep ~1e-7 m
// precision at any map extent.

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace ec3r {

constexpr unsigned long long kEmpty = ~0ull;  // never a _pack key (max is 2^63-1)
constexpr int64_t kPackOffset = 1 << 20;

// 32-byte slot: 16-byte aligned float4 accumulator first (vector red), then
// the key and the count.
struct __align__(32) Slot {
    float sx, sy, sz, sw;
    unsigned long long key;
    unsigned int cnt;
    unsigned int pad;
};

}  // namespace ec3r

struct ec3r_vhash {
    int64_t capacity;
    unsigned long long mask;
    double cell;
    ec3r::Slot* slots;
    unsigned long long* counters;  // [n_in, n_oor, n_overflow, n_slow, n_occupied]
};

namespace ec3r {

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

__device__ __forceinline__ unsigned long long pack_cells(long long cx, long long cy, long long cz) {
    return ((unsigned long long)(cx + kPackOffset) << 42) | ((unsigned long long)(cy + kPackOffset) << 21) |
           (unsigned long long)(cz + kPackOffset);
}

__device__ __forceinline__ bool cell_in_range(long long c) { return c >= -kPackOffset && c < kPackOffset; }

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// Insert (key, w*dx, w*dy, w*dz, w, +1).  Returns false when the table is full.
__device__ __forceinline__ bool vh_insert(Slot* __restrict__ slots, unsigned long long mask, unsigned long long key,
                                          float wx, float wy, float wz, float w) {
    unsigned long long idx = mix64(key) & mask;
    for (unsigned long long probe = 0; probe <= mask; ++probe) {
        Slot* s = slots + idx;
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&s->key);
        if (k == kEmpty) {
            const unsigned long long prev = atomicCAS(&s->key, kEmpty, key);
            k = (prev == kEmpty) ? key : prev;
        }
        if (k == key) {
            red_add_v4(&s->sx, wx, wy, wz, w);
            atomicAdd(&s->cnt, 1u);
            return true;
        }
        idx = (idx + 1) & mask;
    }
    return false;
}

__global__ void vh_clear_kernel(Slot* __restrict__ slots, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        float4* p = reinterpret_cast<float4*>(slots + i);
        p[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        ulonglong2 t;
        t.x = kEmpty;
        t.y = 0;
        reinterpret_cast<ulonglong2*>(p + 1)[0] = t;
    }
}

// ---------------------------------------------------------------------------
// frame insertion

constexpr int FI_NT = 256;
constexpr int FI_ROWS = 8;  // image rows per CTA

struct FuseArgs {
    const float* depth;
    const float* conf;
    const double* slot_poses;    // anchor_from_cam per slot
    const double* slot_globals;  // world_from_anchor (submap global Sim3) per slot
    const int32_t* slots;        // slot ids to fuse
    int H, W;
    double fx, fy, cx, cy;
    double cell;
    float inv_cell_f, cell_f;
    Slot* table;
    unsigned long long mask;
    unsigned long long* counters;
};

// Exact reference chain for one pixel: cells of  G.apply(P.apply(ray)).
__device__ __noinline__ void exact_cells(const double* P, const double* G, double xcoef, double ycoef, float zf,
                                         double cell, long long c[3]) {
    const double z = (double)zf;
    const double ray[3] = {xm(xcoef, z), xm(ycoef, z), z};
    double pa[3], pw[3];
    pose_apply_exact(P, ray, pa);
    sim3_apply_exact(G, pa, pw);
#pragma unroll
    for (int k = 0; k < 3; ++k) c[k] = (long long)floor(__ddiv_rn(pw[k], cell));
}

__global__ void __launch_bounds__(FI_NT) vh_insert_frames_kernel(FuseArgs a) {
    extern __shared__ unsigned char fsm[];
    const int W = a.W;
    // smem: A[W] float4 (xyz + |.|sum), xc[W] double, B[ROWS] float4, yc[ROWS] double
    float4* A = reinterpret_cast<float4*>(fsm);
    double* xc = reinterpret_cast<double*>(A + W);
    __shared__ float4 B[FI_ROWS];
    __shared__ double yc[FI_ROWS];
    __shared__ double Pd[8], Gd[8];
    __shared__ float Tm[4];
    __shared__ unsigned long long cta_cnt[4];

    const int slot = a.slots[blockIdx.y];
    const int v0 = blockIdx.x * FI_ROWS;
    const int nrows = min(FI_ROWS, a.H - v0);
    if (threadIdx.x < 8) {
        Pd[threadIdx.x] = a.slot_poses[8 * slot + threadIdx.x];
        Gd[threadIdx.x] = a.slot_globals[8 * slot + threadIdx.x];
    }
    if (threadIdx.x < 4) cta_cnt[threadIdx.x] = 0;
    __syncthreads();
    // composite M = G o P in float64: rotation sG*RG*RP, translation sG*RG*tP + tG
    double RG[3][3], RP[3][3], M[3][3], T[3];
    quat_to_mat(Gd + 1, RG);
    quat_to_mat(Pd + 1, RP);
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) M[i][j] = Gd[0] * (RG[i][0] * RP[0][j] + RG[i][1] * RP[1][j] + RG[i][2] * RP[2][j]);
        T[i] = Gd[0] * (RG[i][0] * Pd[5] + RG[i][1] * Pd[6] + RG[i][2] * Pd[7]) + Gd[5 + i];
    }
    for (int u = threadIdx.x; u < W; u += FI_NT) {
        const double x = ray_coef(u, a.cx, a.fx);
        xc[u] = x;
        const float ax = (float)(M[0][0] * x + M[0][2]), ay = (float)(M[1][0] * x + M[1][2]),
                    az = (float)(M[2][0] * x + M[2][2]);
        A[u] = make_float4(ax, ay, az, fabsf(ax) + fabsf(ay) + fabsf(az));
    }
    if (threadIdx.x < nrows) {
        const int v = v0 + threadIdx.x;
        const double y = ray_coef(v, a.cy, a.fy);
        yc[threadIdx.x] = y;
        const float bx = (float)(M[0][1] * y), by = (float)(M[1][1] * y), bz = (float)(M[2][1] * y);
        B[threadIdx.x] = make_float4(bx, by, bz, fabsf(bx) + fabsf(by) + fabsf(bz));
    }
    if (threadIdx.x == 0) {
        Tm[0] = (float)T[0]; Tm[1] = (float)T[1]; Tm[2] = (float)T[2];
        Tm[3] = fabsf(Tm[0]) + fabsf(Tm[1]) + fabsf(Tm[2]);
    }
    __syncthreads();
    const float tx = Tm[0], ty = Tm[1], tz = Tm[2], tabs = Tm[3];
    const float inv = a.inv_cell_f, cellf = a.cell_f;
    const size_t HW = (size_t)a.H * W;
    const float* dp = a.depth + (size_t)slot * HW + (size_t)v0 * W;
    const float* cp = a.conf + (size_t)slot * HW + (size_t)v0 * W;
    const int npix = nrows * W;
    const bool vec = ((((size_t)slot * HW + (size_t)v0 * W) & 3) == 0) && ((npix & 3) == 0);
    unsigned int n_in = 0, n_oor = 0, n_ovf = 0, n_slow = 0;  // per-thread counts

    for (int base = 4 * threadIdx.x; base < npix; base += 4 * FI_NT) {
        float zs[4], cs[4];
        if (vec) {
            const float4 z4 = __ldcs(reinterpret_cast<const float4*>(dp + base));
            const float4 c4 = __ldcs(reinterpret_cast<const float4*>(cp + base));
            zs[0] = z4.x; zs[1] = z4.y; zs[2] = z4.z; zs[3] = z4.w;
            cs[0] = c4.x; cs[1] = c4.y; cs[2] = c4.z; cs[3] = c4.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool in = base + k < npix;
                zs[k] = in ? dp[base + k] : 0.f;
                cs[k] = in ? cp[base + k] : 0.f;
            }
        }
        int r = base / W;
        int u = base - r * W;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float z = zs[k], c = cs[k];
            if (z > 0.f && c > 0.f) {
                ++n_in;
                const float4 Au = A[u], Bv = B[r];
                const float dx = Au.x + Bv.x, dy = Au.y + Bv.y, dz = Au.z + Bv.z;
                const float x = fmaf(z, dx, tx), y = fmaf(z, dy, ty), zz = fmaf(z, dz, tz);
                // first-order float32 error bound (x4 safety), see header
                const float ax = fabsf(x) + fabsf(y) + fabsf(zz);
                const float err = 2.384185791015625e-07f * (2.0f * z * (Au.w + Bv.w) + tabs + 2.0f * ax) + 1e-9f;
                const float margin = err * inv + 2.4e-7f;
                const float qx = x * inv, qy = y * inv, qz = zz * inv;
                const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
                const bool near = (qx - fx < margin) || (fx + 1.0f - qx < margin) || (qy - fy < margin) ||
                                  (fy + 1.0f - qy < margin) || (qz - fz < margin) || (fz + 1.0f - qz < margin) ||
                                  fabsf(qx) > 1.0e6f || fabsf(qy) > 1.0e6f || fabsf(qz) > 1.0e6f;
                long long cxl, cyl, czl;
                if (!near) {
                    cxl = (long long)fx; cyl = (long long)fy; czl = (long long)fz;
                } else {
                    long long cc[3];
                    exact_cells(Pd, Gd, xc[u], yc[r], z, a.cell, cc);
                    cxl = cc[0]; cyl = cc[1]; czl = cc[2];
                    ++n_slow;
                }
                if (cell_in_range(cxl) && cell_in_range(cyl) && cell_in_range(czl)) {
                    const unsigned long long key = pack_cells(cxl, cyl, czl);
                    const float ox = x - (float)cxl * cellf, oy = y - (float)cyl * cellf, oz = zz - (float)czl * cellf;
                    if (!vh_insert(a.table, a.mask, key, c * ox, c * oy, c * oz, c)) ++n_ovf;
                } else {
                    ++n_oor;
                }
            }
            if (++u == W) { u = 0; ++r; }
        }
    }
    // counters: warp reduce then one shared atomic per warp, one global per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
        n_oor += __shfl_xor_sync(0xffffffffu, n_oor, o);
        n_ovf += __shfl_xor_sync(0xffffffffu, n_ovf, o);
        n_slow += __shfl_xor_sync(0xffffffffu, n_slow, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&cta_cnt[0], (unsigned long long)n_in);
        atomicAdd(&cta_cnt[1], (unsigned long long)n_oor);
        atomicAdd(&cta_cnt[2], (unsigned long long)n_ovf);
        atomicAdd(&cta_cnt[3], (unsigned long long)n_slow);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cta_cnt[threadIdx.x]) atomicAdd(&a.counters[threadIdx.x], cta_cnt[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Grouped insertion with CTA-level aggregation.
//
// Measured on this part (tools/atomics_probe.cu): random global atomics into a
// DRAM-resident table run at ~22-33 G op/s, shared-memory integer atomics at
// ~2 T op/s.  Frames of a submap (and of neighbouring submaps) see the same
// surface, so a CTA takes one band of AG_ROWS image rows across every frame of
// a slot group, accumulates the voxels in a shared-memory open-addressing
// table with fixed-point integer atomics, and flushes each distinct voxel to
// the global hash once.  Keys use the same exact fast/slow path as above.

constexpr int AG_NT = 512;
constexpr int AG_ROWS = 4;
constexpr int AG_SLOTS = 3840;  // 8 B key + 5 x 4 B accumulators: 105 KB, two CTAs per SM
constexpr int AG_PROBES = 32;

struct GroupArgs {
    FuseArgs f;
    const int32_t* group_off;  // n_groups + 1 offsets into f.slots
    float qscale;              // fixed-point scale of the shared accumulators
};

__device__ __forceinline__ bool sm_insert(unsigned long long* skeys, unsigned int* sacc, unsigned long long key,
                                          unsigned int qx, unsigned int qy, unsigned int qz, unsigned int qw) {
    unsigned int h = (unsigned int)(((mix64(key) >> 32) * (unsigned long long)AG_SLOTS) >> 32);
#pragma unroll 1
    for (int probe = 0; probe < AG_PROBES; ++probe) {
        unsigned long long k = skeys[h];
        if (k == kEmpty) {
            const unsigned long long prev = atomicCAS(&skeys[h], kEmpty, key);
            k = (prev == kEmpty) ? key : prev;
        }
        if (k == key) {
            atomicAdd(&sacc[0 * AG_SLOTS + h], qx);
            atomicAdd(&sacc[1 * AG_SLOTS + h], qy);
            atomicAdd(&sacc[2 * AG_SLOTS + h], qz);
            atomicAdd(&sacc[3 * AG_SLOTS + h], qw);
            atomicAdd(&sacc[4 * AG_SLOTS + h], 1u);
            return true;
        }
        h = (h + 1 == AG_SLOTS) ? 0u : h + 1;
    }
    return false;
}

__global__ void __launch_bounds__(AG_NT, 2) vh_insert_groups_kernel(GroupArgs ga) {
    const FuseArgs& a = ga.f;
    extern __shared__ __align__(16) unsigned char gsm[];
    unsigned long long* skeys = reinterpret_cast<unsigned long long*>(gsm);
    unsigned int* sacc = reinterpret_cast<unsigned int*>(skeys + AG_SLOTS);  // [5][AG_SLOTS]
    float* xcf = reinterpret_cast<float*>(sacc + 5 * AG_SLOTS);               // [W]
    __shared__ float ycf[AG_ROWS];
    __shared__ float Mf[12];
    __shared__ double Pd[8], Gd[8];
    __shared__ unsigned long long cta_cnt[4];

    const int W = a.W;
    const int v0 = blockIdx.x * AG_ROWS;
    const int nrows = min(AG_ROWS, a.H - v0);
    const int g0 = ga.group_off[blockIdx.y], g1 = ga.group_off[blockIdx.y + 1];
    for (int i = threadIdx.x; i < AG_SLOTS; i += AG_NT) skeys[i] = kEmpty;
    for (int i = threadIdx.x; i < 5 * AG_SLOTS; i += AG_NT) sacc[i] = 0u;
    for (int u = threadIdx.x; u < W; u += AG_NT) xcf[u] = (float)((u - a.cx) / a.fx);
    if (threadIdx.x < nrows) ycf[threadIdx.x] = (float)((v0 + threadIdx.x - a.cy) / a.fy);
    if (threadIdx.x < 4) cta_cnt[threadIdx.x] = 0;
    const float inv = a.inv_cell_f, cellf = a.cell_f, qs = ga.qscale;
    const float qcell = qs / cellf;
    unsigned int n_in = 0, n_oor = 0, n_ovf = 0, n_slow = 0;  // per-thread counts
    const size_t HW = (size_t)a.H * W;
    const int npix = nrows * W;

    for (int gi = g0; gi < g1; ++gi) {
        const int slot = a.slots[gi];
        __syncthreads();  // previous frame's Mf / Pd / Gd consumers are done
        if (threadIdx.x < 8) {
            Pd[threadIdx.x] = a.slot_poses[8 * slot + threadIdx.x];
            Gd[threadIdx.x] = a.slot_globals[8 * slot + threadIdx.x];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double RG[3][3], RP[3][3];
            quat_to_mat(Gd + 1, RG);
            quat_to_mat(Pd + 1, RP);
            for (int i = 0; i < 3; ++i) {
                for (int j = 0; j < 3; ++j)
                    Mf[3 * i + j] =
                        (float)(Gd[0] * (RG[i][0] * RP[0][j] + RG[i][1] * RP[1][j] + RG[i][2] * RP[2][j]));
                Mf[9 + i] = (float)(Gd[0] * (RG[i][0] * Pd[5] + RG[i][1] * Pd[6] + RG[i][2] * Pd[7]) + Gd[5 + i]);
            }
        }
        __syncthreads();
        // composite rotation*scale row-major m{i}{j} = M[i][j]; translation Mf[9..11]
        const float m00 = Mf[0], m01 = Mf[1], m02 = Mf[2], m10 = Mf[3], m11 = Mf[4], m12 = Mf[5];
        const float m20 = Mf[6], m21 = Mf[7], m22 = Mf[8], tx = Mf[9], ty = Mf[10], tz = Mf[11];
        const float tabs = fabsf(tx) + fabsf(ty) + fabsf(tz);
        const float* dp = a.depth + (size_t)slot * HW + (size_t)v0 * W;
        const float* cp = a.conf + (size_t)slot * HW + (size_t)v0 * W;
        const bool vec = ((((size_t)slot * HW + (size_t)v0 * W) & 3) == 0) && ((npix & 3) == 0);
        for (int base = 4 * threadIdx.x; base < npix; base += 4 * AG_NT) {
            float zs[4], cs[4];
            if (vec) {
                const float4 z4 = __ldcs(reinterpret_cast<const float4*>(dp + base));
                const float4 c4 = __ldcs(reinterpret_cast<const float4*>(cp + base));
                zs[0] = z4.x; zs[1] = z4.y; zs[2] = z4.z; zs[3] = z4.w;
                cs[0] = c4.x; cs[1] = c4.y; cs[2] = c4.z; cs[3] = c4.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool in = base + k < npix;
                    zs[k] = in ? dp[base + k] : 0.f;
                    cs[k] = in ? cp[base + k] : 0.f;
                }
            }
            int r = base / W;
            int u = base - r * W;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float z = zs[k], c = cs[k];
                if (z > 0.f && c > 0.f) {
                    ++n_in;
                    const float xu = xcf[u], yv = ycf[r];
                    const float ax = m00 * xu, ay = m10 * xu, az = m20 * xu;
                    const float bx = m01 * yv, by = m11 * yv, bz = m21 * yv;
                    const float dx = ax + bx + m02, dy = ay + by + m12, dz = az + bz + m22;
                    const float x = fmaf(z, dx, tx), y = fmaf(z, dy, ty), zz = fmaf(z, dz, tz);
                    const float sa = fabsf(ax) + fabsf(ay) + fabsf(az) + fabsf(bx) + fabsf(by) + fabsf(bz) +
                                     fabsf(m02) + fabsf(m12) + fabsf(m22);
                    const float axs = fabsf(x) + fabsf(y) + fabsf(zz);
                    // first-order float32 error bound of x,y,z (x8 safety), see vh_insert_frames_kernel
                    const float err = 4.76837158203125e-07f * (2.0f * z * sa + tabs + 2.0f * axs) + 1e-9f;
                    const float margin = err * inv + 2.4e-7f;
                    const float qx = x * inv, qy = y * inv, qz = zz * inv;
                    const float fx = floorf(qx), fy = floorf(qy), fz = floorf(qz);
                    const bool near = (qx - fx < margin) || (fx + 1.0f - qx < margin) || (qy - fy < margin) ||
                                      (fy + 1.0f - qy < margin) || (qz - fz < margin) || (fz + 1.0f - qz < margin) ||
                                      fabsf(qx) > 1.0e6f || fabsf(qy) > 1.0e6f || fabsf(qz) > 1.0e6f;
                    long long cxl, cyl, czl;
                    if (!near) {
                        cxl = (long long)fx; cyl = (long long)fy; czl = (long long)fz;
                    } else {
                        long long cc[3];
                        exact_cells(Pd, Gd, ray_coef(u, a.cx, a.fx), ray_coef(v0 + r, a.cy, a.fy), z, a.cell, cc);
                        cxl = cc[0]; cyl = cc[1]; czl = cc[2];
                        ++n_slow;
                    }
                    if (cell_in_range(cxl) && cell_in_range(cyl) && cell_in_range(czl)) {
                        const unsigned long long key = pack_cells(cxl, cyl, czl);
                        const float ox = x - (float)cxl * cellf, oy = y - (float)cyl * cellf,
                                    oz = zz - (float)czl * cellf;
                        const unsigned int ux = __float2uint_rn(fminf(fmaxf(c * ox * qcell, 0.f), qs));
                        const unsigned int uy = __float2uint_rn(fminf(fmaxf(c * oy * qcell, 0.f), qs));
                        const unsigned int uz = __float2uint_rn(fminf(fmaxf(c * oz * qcell, 0.f), qs));
                        const unsigned int uw = __float2uint_rn(c * qs);
                        if (!sm_insert(skeys, sacc, key, ux, uy, uz, uw)) {
                            // shared table saturated: this point goes straight to the global hash
                            if (!vh_insert(a.table, a.mask, key, c * ox, c * oy, c * oz, c)) ++n_ovf;
                        }
                    } else {
                        ++n_oor;
                    }
                }
                if (++u == W) { u = 0; ++r; }
            }
        }
    }
    __syncthreads();
    // flush: one global insert per distinct voxel of this CTA
    const float back = cellf / qs, wback = 1.0f / qs;
    for (int i = threadIdx.x; i < AG_SLOTS; i += AG_NT) {
        const unsigned long long key = skeys[i];
        if (key == kEmpty) continue;
        const float sx = (float)sacc[i] * back, sy = (float)sacc[AG_SLOTS + i] * back;
        const float sz = (float)sacc[2 * AG_SLOTS + i] * back, sw = (float)sacc[3 * AG_SLOTS + i] * wback;
        const unsigned int cnt = sacc[4 * AG_SLOTS + i];
        unsigned long long idx = mix64(key) & a.mask;
        bool done = false;
        for (unsigned long long probe = 0; probe <= a.mask; ++probe) {
            Slot* s = a.table + idx;
            unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&s->key);
            if (k == kEmpty) {
                const unsigned long long prev = atomicCAS(&s->key, kEmpty, key);
                k = (prev == kEmpty) ? key : prev;
            }
            if (k == key) {
                red_add_v4(&s->sx, sx, sy, sz, sw);
                atomicAdd(&s->cnt, cnt);
                done = true;
                break;
            }
            idx = (idx + 1) & a.mask;
        }
        if (!done) n_ovf += cnt;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        n_in += __shfl_xor_sync(0xffffffffu, n_in, o);
        n_oor += __shfl_xor_sync(0xffffffffu, n_oor, o);
        n_ovf += __shfl_xor_sync(0xffffffffu, n_ovf, o);
        n_slow += __shfl_xor_sync(0xffffffffu, n_slow, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&cta_cnt[0], (unsigned long long)n_in);
        atomicAdd(&cta_cnt[1], (unsigned long long)n_oor);
        atomicAdd(&cta_cnt[2], (unsigned long long)n_ovf);
        atomicAdd(&cta_cnt[3], (unsigned long long)n_slow);
    }
    __syncthreads();
    if (threadIdx.x < 4 && cta_cnt[threadIdx.x]) atomicAdd(&a.counters[threadIdx.x], cta_cnt[threadIdx.x]);
}

// Explicit points (float64) under one Sim(3): exact float64 transform.
__global__ void vh_insert_points_kernel(const double* __restrict__ pts, const double* __restrict__ conf, int64_t n,
                                        Sim3Arg g, double cell, float cellf, Slot* table, unsigned long long mask,
                                        unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c = conf[i];
    if (!(c > 0)) return;
    atomicAdd(&counters[0], 1ull);
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double x[3];
    sim3_apply_exact(g.v, p, x);
    long long cc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) cc[k] = (long long)floor(__ddiv_rn(x[k], cell));
    if (!(cell_in_range(cc[0]) && cell_in_range(cc[1]) && cell_in_range(cc[2]))) {
        atomicAdd(&counters[1], 1ull);
        return;
    }
    const unsigned long long key = pack_cells(cc[0], cc[1], cc[2]);
    const float w = (float)c;
    const float ox = (float)(x[0] - (double)cc[0] * cell), oy = (float)(x[1] - (double)cc[1] * cell),
                oz = (float)(x[2] - (double)cc[2] * cell);
    (void)cellf;
    if (!vh_insert(table, mask, key, w * ox, w * oy, w * oz, w)) atomicAdd(&counters[2], 1ull);
}

// ---------------------------------------------------------------------------
// extraction

__global__ void vh_count_kernel(const Slot* __restrict__ slots, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += slots[i].key != kEmpty;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Compact occupied slots: (key, slot index), warp-aggregated append.
__global__ void vh_compact_kernel(const Slot* __restrict__ slots, int64_t n, unsigned long long* __restrict__ keys,
                                  int64_t* __restrict__ idx, unsigned long long* __restrict__ cursor) {
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        const unsigned long long k = i < n ? slots[i].key : kEmpty;
        const bool occ = k != kEmpty;
        const unsigned m = __ballot_sync(0xffffffffu, occ);
        unsigned long long base = 0;
        const int lane = threadIdx.x & 31;
        if (lane == 0 && m) base = atomicAdd(cursor, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (occ) {
            const unsigned long long o = base + __popc(m & ((1u << lane) - 1u));
            keys[o] = k;
            idx[o] = i;
        }
    }
}

__global__ void vh_gather_kernel(const Slot* __restrict__ slots, const unsigned long long* __restrict__ keys,
                                 const int64_t* __restrict__ idx, const int64_t* __restrict__ n_ptr, double cell,
                                 int64_t* __restrict__ okeys, float* __restrict__ cen, float* __restrict__ wsum,
                                 int32_t* __restrict__ cnt) {
    const int64_t n = *n_ptr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Slot s = slots[idx[i]];
        const unsigned long long k = keys[i];
        const long long cx = (long long)((k >> 42) & 0x1FFFFF) - kPackOffset;
        const long long cy = (long long)((k >> 21) & 0x1FFFFF) - kPackOffset;
        const long long cz = (long long)(k & 0x1FFFFF) - kPackOffset;
        okeys[i] = (int64_t)k;
        const double w = s.sw;
        cen[3 * i + 0] = (float)((double)cx * cell + (double)s.sx / w);
        cen[3 * i + 1] = (float)((double)cy * cell + (double)s.sy / w);
        cen[3 * i + 2] = (float)((double)cz * cell + (double)s.sz / w);
        wsum[i] = s.sw;
        cnt[i] = (int32_t)s.cnt;
    }
}

// partial sums for the multi-GPU all-to-all: owner = mix64(key) % n_ranks
__global__ void vh_partition_count_kernel(const Slot* __restrict__ slots, int64_t n, int n_ranks,
                                          unsigned long long* __restrict__ rank_counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = slots[i].key;
        if (k != kEmpty) atomicAdd(&rank_counts[mix64(k) % (unsigned long long)n_ranks], 1ull);
    }
}

__global__ void vh_partition_write_kernel(const Slot* __restrict__ slots, int64_t n, int n_ranks,
                                          const unsigned long long* __restrict__ rank_base,
                                          unsigned long long* __restrict__ cursors, int64_t* __restrict__ okeys,
                                          float* __restrict__ sums4, int32_t* __restrict__ cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Slot s = slots[i];
        if (s.key == kEmpty) continue;
        const int r = (int)(mix64(s.key) % (unsigned long long)n_ranks);
        const unsigned long long o = rank_base[r] + atomicAdd(&cursors[r], 1ull);
        okeys[o] = (int64_t)s.key;
        reinterpret_cast<float4*>(sums4)[o] = make_float4(s.sx, s.sy, s.sz, s.sw);
        cnt[o] = (int32_t)s.cnt;
    }
}

__global__ void vh_merge_kernel(const int64_t* __restrict__ keys, const float* __restrict__ sums4,
                                const int32_t* __restrict__ cnt, int64_t n, Slot* table, unsigned long long mask,
                                unsigned long long* counters) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = (unsigned long long)keys[i];
    const float4 s = reinterpret_cast<const float4*>(sums4)[i];
    unsigned long long idx = mix64(key) & mask;
    for (unsigned long long probe = 0; probe <= mask; ++probe) {
        Slot* sl = table + idx;
        unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&sl->key);
        if (k == kEmpty) {
            const unsigned long long prev = atomicCAS(&sl->key, kEmpty, key);
            k = (prev == kEmpty) ? key : prev;
        }
        if (k == key) {
            red_add_v4(&sl->sx, s.x, s.y, s.z, s.w);
            atomicAdd(&sl->cnt, (unsigned)cnt[i]);
            return;
        }
        idx = (idx + 1) & mask;
    }
    atomicAdd(&counters[2], 1ull);
}

}  // namespace ec3r

using namespace ec3r;

extern "C" int ec3r_vhash_create(ec3r_vhash** out, int64_t capacity, double cell_size, void* stream) {
    if (!out || capacity < 2 || !(cell_size > 0)) return EC3R_EARG;
    int64_t cap = 1;
    while (cap < capacity) cap <<= 1;
    ec3r_vhash* h = new ec3r_vhash();
    h->capacity = cap;
    h->mask = (unsigned long long)(cap - 1);
    h->cell = cell_size;
    if (cudaMalloc(&h->slots, sizeof(Slot) * (size_t)cap) != cudaSuccess) {
        set_last_error("cudaMalloc(vhash slots)", cudaGetLastError());
        delete h;
        return EC3R_ENOMEM;
    }
    if (cudaMalloc(&h->counters, sizeof(unsigned long long) * 8) != cudaSuccess) {
        set_last_error("cudaMalloc(vhash counters)", cudaGetLastError());
        cudaFree(h->slots);
        delete h;
        return EC3R_ENOMEM;
    }
    *out = h;
    return ec3r_vhash_clear(h, stream);
}

extern "C" int ec3r_vhash_destroy(ec3r_vhash* h) {
    if (!h) return EC3R_OK;
    cudaFree(h->slots);
    cudaFree(h->counters);
    delete h;
    return EC3R_OK;
}

extern "C" int64_t ec3r_vhash_capacity(const ec3r_vhash* h) { return h ? h->capacity : 0; }

extern "C" int ec3r_vhash_clear(ec3r_vhash* h, void* stream) {
    if (!h) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    vh_clear_kernel<<<(unsigned)((h->capacity + 255) / 256), 256, 0, st>>>(h->slots, h->capacity);
    EC3R_CHECK_LAUNCH("vh_clear_kernel");
    EC3R_CUDA_TRY(cudaMemsetAsync(h->counters, 0, sizeof(unsigned long long) * 8, st));
    return EC3R_OK;
}

extern "C" int ec3r_vhash_insert_frames(ec3r_vhash* h, const float* depth_pool, const float* conf_pool, int H, int W,
                                        const double* K4_h, const double* slot_poses, const double* slot_globals,
                                        const int32_t* slots, int n, void* stream) {
    if (!h || H <= 0 || W <= 0 || !K4_h || n < 0) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    FuseArgs a;
    a.depth = depth_pool; a.conf = conf_pool; a.slot_poses = slot_poses; a.slot_globals = slot_globals;
    a.slots = slots; a.H = H; a.W = W;
    a.fx = K4_h[0]; a.fy = K4_h[1]; a.cx = K4_h[2]; a.cy = K4_h[3];
    a.cell = h->cell; a.inv_cell_f = (float)(1.0 / h->cell); a.cell_f = (float)h->cell;
    a.table = h->slots; a.mask = h->mask; a.counters = h->counters;
    const size_t smem = (size_t)W * (sizeof(float4) + sizeof(double));
    if (smem > 48 * 1024)
        EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
    dim3 grid((H + FI_ROWS - 1) / FI_ROWS, n);
    vh_insert_frames_kernel<<<grid, FI_NT, smem, as_stream(stream)>>>(a);
    EC3R_CHECK_LAUNCH("vh_insert_frames_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_insert_frame_groups(ec3r_vhash* h, const float* depth_pool, const float* conf_pool, int H,
                                              int W, const double* K4_h, const double* slot_poses,
                                              const double* slot_globals, const int32_t* slots,
                                              const int32_t* group_off, int n_groups, int max_frames_per_group,
                                              void* stream) {
    if (!h || H <= 0 || W <= 0 || !K4_h || n_groups < 0 || max_frames_per_group < 1) return EC3R_EARG;
    if (n_groups == 0) return EC3R_OK;
    GroupArgs ga;
    FuseArgs& a = ga.f;
    a.depth = depth_pool; a.conf = conf_pool; a.slot_poses = slot_poses; a.slot_globals = slot_globals;
    a.slots = slots; a.H = H; a.W = W;
    a.fx = K4_h[0]; a.fy = K4_h[1]; a.cx = K4_h[2]; a.cy = K4_h[3];
    a.cell = h->cell; a.inv_cell_f = (float)(1.0 / h->cell); a.cell_f = (float)h->cell;
    a.table = h->slots; a.mask = h->mask; a.counters = h->counters;
    ga.group_off = group_off;
    // fixed-point scale: every point adds <= qscale per accumulator and a CTA
    // sees <= max_frames * AG_ROWS * W points, so sums stay below 2^32
    const double max_pts = (double)max_frames_per_group * AG_ROWS * W;
    double qs = 65536.0;
    while (qs > 1.0 && qs * max_pts >= 4294967295.0) qs *= 0.5;
    ga.qscale = (float)qs;
    const size_t smem = (size_t)AG_SLOTS * (8 + 5 * 4) + (size_t)W * 4;
    EC3R_CUDA_TRY(cudaFuncSetAttribute(vh_insert_groups_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((H + AG_ROWS - 1) / AG_ROWS, n_groups);
    vh_insert_groups_kernel<<<grid, AG_NT, smem, as_stream(stream)>>>(ga);
    EC3R_CHECK_LAUNCH("vh_insert_groups_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_insert_points(ec3r_vhash* h, const double* points, const double* conf, int64_t n,
                                        const double* sim3_h, void* stream) {
    if (!h || n < 0 || !sim3_h) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    Sim3Arg g;
    for (int k = 0; k < 8; ++k) g.v[k] = sim3_h[k];
    vh_insert_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        points, conf, n, g, h->cell, (float)h->cell, h->slots, h->mask, h->counters);
    EC3R_CHECK_LAUNCH("vh_insert_points_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_stats_get(ec3r_vhash* h, ec3r_vhash_stats* out_h, void* stream) {
    if (!h || !out_h) return EC3R_EARG;
    unsigned long long c[8];
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemcpyAsync(c, h->counters, sizeof(c), cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    out_h->n_points_in = (int64_t)c[0];
    out_h->n_out_of_range = (int64_t)c[1];
    out_h->n_overflow = (int64_t)c[2];
    out_h->n_slow_path = (int64_t)c[3];
    return EC3R_OK;
}

static unsigned grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)kNumSMs * 16) g = (int64_t)kNumSMs * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

extern "C" int ec3r_vhash_count(ec3r_vhash* h, int64_t* n_out, void* stream) {
    if (!h || !n_out) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    EC3R_CUDA_TRY(cudaMemsetAsync(n_out, 0, sizeof(int64_t), st));
    vh_count_kernel<<<grid_for(h->capacity), 256, 0, st>>>(h->slots, h->capacity, (unsigned long long*)n_out);
    EC3R_CHECK_LAUNCH("vh_count_kernel");
    return EC3R_OK;
}

extern "C" size_t ec3r_vhash_extract_workspace(const ec3r_vhash* h) {
    if (!h) return 0;
    size_t cub_bytes = 0;
    cub::DeviceRadixSort::SortPairs<unsigned long long, int64_t>(nullptr, cub_bytes, (unsigned long long*)nullptr,
                                                                 (unsigned long long*)nullptr, (int64_t*)nullptr,
                                                                 (int64_t*)nullptr, (int)h->capacity, 0, 63);
    return 4 * align256(sizeof(int64_t) * (size_t)h->capacity) + align256(64) + align256(cub_bytes);
}

extern "C" int ec3r_vhash_extract(ec3r_vhash* h, int64_t* keys, float* centroid, float* wsum, int32_t* count,
                                  int64_t* n_out, int sort, void* workspace, size_t workspace_bytes, void* stream) {
    if (!h || !keys || !centroid || !wsum || !count || !n_out) return EC3R_EARG;
    if (!workspace || workspace_bytes < ec3r_vhash_extract_workspace(h)) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    const size_t cap = (size_t)h->capacity;
    Carver cv{(char*)workspace, 0};
    unsigned long long* k0 = cv.take<unsigned long long>(cap);
    int64_t* i0 = cv.take<int64_t>(cap);
    unsigned long long* k1 = cv.take<unsigned long long>(cap);
    int64_t* i1 = cv.take<int64_t>(cap);
    unsigned long long* cursor = cv.take<unsigned long long>(8);
    size_t cub_bytes = workspace_bytes - cv.used;
    void* cub_tmp = cv.base + cv.used;
    EC3R_CUDA_TRY(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), st));
    vh_compact_kernel<<<grid_for(h->capacity), 256, 0, st>>>(h->slots, h->capacity, k0, i0, cursor);
    EC3R_CHECK_LAUNCH("vh_compact_kernel");
    EC3R_CUDA_TRY(cudaMemcpyAsync(n_out, cursor, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    const unsigned long long* ks = k0;
    const int64_t* is = i0;
    if (sort) {
        unsigned long long nh = 0;
        EC3R_CUDA_TRY(cudaMemcpyAsync(&nh, cursor, sizeof(nh), cudaMemcpyDeviceToHost, st));
        EC3R_CUDA_TRY(cudaStreamSynchronize(st));
        if (nh > 0) {
            if (cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k0, k1, i0, i1, (int)nh, 0, 63, st) !=
                cudaSuccess) {
                set_last_error("cub::DeviceRadixSort::SortPairs", cudaGetLastError());
                return EC3R_ECUDA;
            }
        }
        ks = k1;
        is = i1;
    }
    vh_gather_kernel<<<grid_for(h->capacity), 256, 0, st>>>(h->slots, ks, is, n_out, h->cell, keys, centroid, wsum,
                                                            count);
    EC3R_CHECK_LAUNCH("vh_gather_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_vhash_extract_partials(ec3r_vhash* h, int n_ranks, int64_t* keys, float* sums4, int32_t* count,
                                           int64_t* rank_counts, void* workspace, size_t workspace_bytes,
                                           void* stream) {
    if (!h || n_ranks < 1 || !keys || !sums4 || !count || !rank_counts) return EC3R_EARG;
    if (!workspace || workspace_bytes < sizeof(unsigned long long) * 2 * (size_t)n_ranks) return EC3R_EWORKSPACE;
    cudaStream_t st = as_stream(stream);
    unsigned long long* base = (unsigned long long*)workspace;
    unsigned long long* cursors = base + n_ranks;
    EC3R_CUDA_TRY(cudaMemsetAsync(rank_counts, 0, sizeof(int64_t) * n_ranks, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(cursors, 0, sizeof(unsigned long long) * n_ranks, st));
    vh_partition_count_kernel<<<grid_for(h->capacity), 256, 0, st>>>(h->slots, h->capacity, n_ranks,
                                                                     (unsigned long long*)rank_counts);
    EC3R_CHECK_LAUNCH("vh_partition_count_kernel");
    std::vector<unsigned long long> rc(n_ranks), rb(n_ranks);
    EC3R_CUDA_TRY(cudaMemcpyAsync(rc.data(), rank_counts, sizeof(int64_t) * n_ranks, cudaMemcpyDeviceToHost, st));
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));
    unsigned long long acc = 0;
    for (int r = 0; r < n_ranks; ++r) { rb[r] = acc; acc += rc[r]; }
    EC3R_CUDA_TRY(cudaMemcpyAsync(base, rb.data(), sizeof(unsigned long long) * n_ranks, cudaMemcpyHostToDevice, st));
    vh_partition_write_kernel<<<grid_for(h->capacity), 256, 0, st>>>(h->slots, h->capacity, n_ranks, base, cursors,
                                                                     keys, sums4, count);
    EC3R_CHECK_LAUNCH("vh_partition_write_kernel");
    EC3R_CUDA_TRY(cudaStreamSynchronize(st));  // rb is a host temporary
    return EC3R_OK;
}

extern "C" int ec3r_vhash_merge_partials(ec3r_vhash* h, const int64_t* keys, const float* sums4, const int32_t* count,
                                         int64_t n, void* stream) {
    if (!h || n < 0) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    vh_merge_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(keys, sums4, count, n, h->slots,
                                                                                h->mask, h->counters);
    EC3R_CHECK_LAUNCH("vh_merge_kernel");
    return EC3R_OK;
}
