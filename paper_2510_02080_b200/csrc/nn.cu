// K7: the reference's native-kernel plugin slot on sm_100a — grid-hash
// nearest neighbours (nn_query / nn_dists) and the room / box ray caster
// (raycast).  Drop-in for submap_slam._kernels (_kernels/__init__.py:12-33,
// semantics of _kernels/_numpy.py), results bit-identical to it:
//
// nn_query (_numpy.py:66-132)
//   build: cells = floor(ref / cell) (float64), keys = _pack(cells) in
//          wrapping int64 arithmetic (:50-55), a stable radix sort of
//          (key, original index) (= np.argsort(kind="stable"), :82-84), the
//          points gathered in key order, and an open-addressing table
//          key -> first sorted position of the cell;
//   query: one thread per query walks Chebyshev rings r = 0..8 with shells
//          in meshgrid "ij" order (:58-62); candidates are visited in
//          (shell order, sorted order), a ring's best is its first minimum
//          and replaces the running best only when strictly smaller
//          (:108-120); done once best <= r * cell (:121-122).  Distances are
//          sqrt(dx^2 + dy^2 + dz^2) in float64 with numpy's operation order
//          (:105-106, explicit _rn intrinsics: no FMA contraction);
//   strays: queries open after ring 8 get the brute-force first minimum over
//          all reference points in original order (:126-131), one CTA each.
// raycast (_numpy.py:14-47): one thread per ray, slab test per solid with the
//   inside / outside rule for axis-parallel rays; first hit, 0 for none.

#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <curand_kernel.h>

#include "common.cuh"

namespace ec3r {

constexpr int NN_RING = 8;          // _BRUTE_RING

static unsigned nn_grid(int64_t n, int nt) {
    const int64_t g = (n + nt - 1) / nt;
    return (unsigned)(g < 1 ? 1 : (g > kNumSMs * 32 ? kNumSMs * 32 : g));
}
constexpr int64_t NN_PACK = 1 << 20;  // _PACK_OFFSET

// _pack on int64 cells, wrapping exactly like numpy's int64 shifts / ors
__device__ __forceinline__ long long nn_pack(long long cx, long long cy, long long cz) {
    const unsigned long long x = (unsigned long long)(cx + NN_PACK), y = (unsigned long long)(cy + NN_PACK),
                             z = (unsigned long long)(cz + NN_PACK);
    return (long long)((x << 42) | (y << 21) | z);
}

__device__ __forceinline__ long long cell_of(double v, double cell) {
    return (long long)floor(__ddiv_rn(v, cell));
}

__device__ __forceinline__ double nn_dist(double px, double py, double pz, double qx, double qy, double qz) {
    const double dx = __dsub_rn(px, qx), dy = __dsub_rn(py, qy), dz = __dsub_rn(pz, qz);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__device__ __forceinline__ unsigned long long nn_hash(long long k) {
    unsigned long long h = (unsigned long long)k;
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    return h;
}

struct NnTable {
    long long* keys;  // cap
    int* start;       // cap, -1 = empty
    unsigned long long mask;
};

__global__ void nn_keys_kernel(const double* __restrict__ ref, int64_t n, double cell, long long* __restrict__ keys,
                               int* __restrict__ idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = nn_pack(cell_of(ref[3 * i], cell), cell_of(ref[3 * i + 1], cell), cell_of(ref[3 * i + 2], cell));
        idx[i] = (int)i;
    }
}

// sorted points + one table entry per cell (inserted by the cell's first
// sorted position; every key is inserted exactly once, so a claimed slot
// never needs a key comparison during the build)
__global__ void nn_build_kernel(const double* __restrict__ ref, const long long* __restrict__ skeys,
                                const int* __restrict__ order, int64_t n, double* __restrict__ sref, NnTable t) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int o = order[i];
        sref[3 * i] = ref[3 * (int64_t)o];
        sref[3 * i + 1] = ref[3 * (int64_t)o + 1];
        sref[3 * i + 2] = ref[3 * (int64_t)o + 2];
        const long long k = skeys[i];
        if (i == 0 || skeys[i - 1] != k) {
            unsigned long long h = nn_hash(k) & t.mask;
            while (atomicCAS(t.start + h, -1, (int)i) != -1) h = (h + 1) & t.mask;
            t.keys[h] = k;
        }
    }
}

__device__ __forceinline__ int nn_find(const NnTable& t, long long k) {
    unsigned long long h = nn_hash(k) & t.mask;
    while (true) {
        const int s = __ldg(t.start + h);
        if (s < 0) return -1;
        if (__ldg(t.keys + h) == k) return s;
        h = (h + 1) & t.mask;
    }
}

__global__ void nn_query_kernel(const double* __restrict__ query, int64_t nq, const double* __restrict__ sref,
                                const long long* __restrict__ skeys, const int* __restrict__ order, int64_t nr,
                                double cell, NnTable t, double* __restrict__ out_d, int64_t* __restrict__ out_i,
                                int* __restrict__ strays, unsigned long long* __restrict__ n_strays) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        const double qx = query[3 * q], qy = query[3 * q + 1], qz = query[3 * q + 2];
        const long long cx = cell_of(qx, cell), cy = cell_of(qy, cell), cz = cell_of(qz, cell);
        double best = INFINITY;
        int bi = -1;
        bool done = false;
        for (int r = 0; r <= NN_RING && !done; ++r) {
            double rb = INFINITY;
            int rbi = -1;
            for (int i = -r; i <= r; ++i) {
                for (int j = -r; j <= r; ++j) {
                    const bool face = (i == -r || i == r || j == -r || j == r);
                    const int kstep = (face || r == 0) ? 1 : 2 * r;  // interior rows: only k = -r, r
                    for (int k = -r; k <= r; k += kstep) {
                        const long long ck = nn_pack(cx + i, cy + j, cz + k);
                        int s = nn_find(t, ck);
                        if (s < 0) continue;
                        for (; s < nr && __ldg(skeys + s) == ck; ++s) {
                            const double d = nn_dist(__ldg(sref + 3 * s), __ldg(sref + 3 * s + 1),
                                                     __ldg(sref + 3 * s + 2), qx, qy, qz);
                            if (d < rb) { rb = d; rbi = s; }
                        }
                    }
                }
            }
            if (rb < best) { best = rb; bi = rbi; }
            done = best <= __dmul_rn((double)r, cell);
        }
        if (done) {
            out_d[q] = best;
            out_i[q] = order[bi];
        } else {
            strays[atomicAdd(n_strays, 1ull)] = (int)q;
        }
    }
}

// Stray queries: brute force over all reference points in original order.
__global__ void nn_brute_kernel(const double* __restrict__ query, const double* __restrict__ ref, int64_t nr,
                                const int* __restrict__ strays, const unsigned long long* __restrict__ n_strays,
                                double* __restrict__ out_d, int64_t* __restrict__ out_i) {
    __shared__ double sd[32];
    __shared__ long long si[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ns = (int64_t)*n_strays;
    for (int64_t t = blockIdx.x; t < ns; t += gridDim.x) {
        const int q = strays[t];
        const double qx = query[3 * (int64_t)q], qy = query[3 * (int64_t)q + 1], qz = query[3 * (int64_t)q + 2];
        double best = INFINITY;
        long long bi = LLONG_MAX;
        for (int64_t j = threadIdx.x; j < nr; j += blockDim.x) {
            const double d = nn_dist(ref[3 * j], ref[3 * j + 1], ref[3 * j + 2], qx, qy, qz);
            if (d < best) { best = d; bi = j; }  // per thread: ascending j, first minimum
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, best, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (od < best || (od == best && oi < bi)) { best = od; bi = oi; }
        }
        if (lane == 0) { sd[warp] = best; si[warp] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (sd[w] < best || (sd[w] == best && si[w] < bi)) { best = sd[w]; bi = si[w]; }
            out_d[q] = best;
            out_i[q] = bi;
        }
        __syncthreads();
    }
}

__global__ void nn_empty_kernel(int64_t nq, double* __restrict__ out_d, int64_t* __restrict__ out_i) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
        out_d[q] = INFINITY;
        out_i[q] = -1;
    }
}

// ---------------------------------------------------------------------------
// raycast

// numpy's minimum / maximum propagate NaN (a denormal direction component
// gives 0 * inf); CUDA's fmin / fmax would drop it
__device__ __forceinline__ double np_min(double a, double b) { return (a != a || b != b) ? NAN : fmin(a, b); }
__device__ __forceinline__ double np_max(double a, double b) { return (a != a || b != b) ? NAN : fmax(a, b); }

constexpr int RC_MAX_SOLIDS = 64;
struct RcSolids {
    double lo[RC_MAX_SOLIDS][3];
    double hi[RC_MAX_SOLIDS][3];
    int n;
};

// first hit of one ray (_numpy.py:29-47 for one row), 0 for none
__device__ __forceinline__ double rc_first_hit(const double (&o)[3], const double (&d)[3], const RcSolids& s) {
    constexpr double EPS = 1e-9;
    double inv[3];
    for (int a = 0; a < 3; ++a) inv[a] = __ddiv_rn(1.0, d[a]);
    double best = INFINITY;
    for (int b = 0; b < s.n; ++b) {
        double near = -INFINITY, far = INFINITY;
        for (int a = 0; a < 3; ++a) {
            double t1, t2;
            if (d[a] == 0.0) {
                const bool inside = o[a] >= s.lo[b][a] && o[a] <= s.hi[b][a];
                t1 = inside ? -INFINITY : INFINITY;
                t2 = inside ? INFINITY : -INFINITY;
            } else {
                t1 = __dmul_rn(__dsub_rn(s.lo[b][a], o[a]), inv[a]);
                t2 = __dmul_rn(__dsub_rn(s.hi[b][a], o[a]), inv[a]);
            }
            near = np_max(near, np_min(t1, t2));
            far = np_min(far, np_max(t1, t2));
        }
        if (near <= far && far > EPS) best = fmin(best, near > EPS ? near : far);
    }
    return isfinite(best) ? best : 0.0;
}

__global__ void rc_kernel(const double* __restrict__ org, const double* __restrict__ dir, int64_t n, RcSolids s,
                          double* __restrict__ out_t) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double o[3], d[3];
        for (int a = 0; a < 3; ++a) {
            o[a] = org[3 * i + a];
            d[a] = dir[3 * i + a];
        }
        out_t[i] = rc_first_hit(o, d, s);
    }
}

// ---------------------------------------------------------------------------
// §8(f) rank 3: the synthetic producer on the device -- SyntheticBackend.decode
// (backend.py:228-281) over render_depth (scenesim.py:145-163).  One thread
// per pixel of every listed frame:
//   dir_cam = ((u - cx) / fx, (v - cy) / fy, 1)           (scenesim.py:155-158)
//   dir_world = dir_cam @ R_wc^T  as numpy's BLAS evaluates it here: an FMA
//               chain in column order (d0 r0, + d1 r1, + d2 r2)   (:159)
//   t = first hit (rc_first_hit, bit-exact with _kernels raycast)  (:161)
//   depth = t * scale; with sigma > 0: depth *= exp(sigma xi), conf =
//   1 / (1 + |xi|); conf = 0 where depth <= 0              (backend.py:253-262)
// xi is a standard normal from a counter-based Philox stream keyed by
// (seed, decode call) and indexed by (frame, pixel): the same distribution as
// the reference's default_rng normals, not the same numbers (numpy's
// ziggurat over PCG64 is sequential).  With sigma = 0 the decode is
// bit-exact (depth rounded to float32, the pool's format).
__global__ void dec_kernel(RcSolids s, const double* __restrict__ frames, int F, int H, int W, double fx, double fy,
                           double cx, double cy, double scale, double sigma, unsigned long long key,
                           float* __restrict__ depth, float* __restrict__ conf) {
    const int64_t HW = (int64_t)H * W, n = HW * F;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)(p / HW);
        const int64_t q = p - (int64_t)f * HW;
        const int v = (int)(q / W), u = (int)(q - (int64_t)v * W);
        const double* R = frames + 12 * f;
        const double dc[3] = {__ddiv_rn(__dsub_rn((double)u, cx), fx), __ddiv_rn(__dsub_rn((double)v, cy), fy), 1.0};
        double o[3], d[3];
        for (int i = 0; i < 3; ++i) {
            d[i] = __fma_rn(dc[2], R[3 * i + 2], __fma_rn(dc[1], R[3 * i + 1], __dmul_rn(dc[0], R[3 * i])));
            o[i] = R[9 + i];
        }
        double z = __dmul_rn(rc_first_hit(o, d, s), scale);
        double c = 1.0;
        if (sigma > 0.0) {
            curandStatePhilox4_32_10_t st;
            curand_init(key, (unsigned long long)p, 0ull, &st);
            const double xi = curand_normal_double(&st);
            z = __dmul_rn(z, exp(__dmul_rn(sigma, xi)));
            c = __ddiv_rn(1.0, __dadd_rn(1.0, fabs(xi)));
        }
        depth[p] = (float)z;
        conf[p] = z > 0.0 ? (float)c : 0.f;
    }
}

static int64_t nn_table_cap(int64_t nr) {
    int64_t c = 1024;
    while (c < 2 * nr) c <<= 1;
    return c;
}

static size_t nn_sort_bytes(int64_t nr) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (long long*)nullptr, (long long*)nullptr, (int*)nullptr,
                                    (int*)nullptr, (int)(nr > 0 ? nr : 1));
    return b;
}

}  // namespace ec3r

using namespace ec3r;

extern "C" size_t ec3r_nn_workspace(int64_t n_ref, int64_t n_query) {
    if (n_ref < 0 || n_query < 0) return 0;
    const int64_t cap = nn_table_cap(n_ref);
    return 2 * align256(sizeof(long long) * (size_t)n_ref) + 2 * align256(sizeof(int) * (size_t)n_ref) +
           align256(sizeof(double) * 3 * (size_t)n_ref) + align256(sizeof(long long) * (size_t)cap) +
           align256(sizeof(int) * (size_t)cap) + align256(sizeof(int) * (size_t)n_query) + align256(64) +
           align256(nn_sort_bytes(n_ref));
}

extern "C" int ec3r_nn_query(const double* query, int64_t n_query, const double* ref, int64_t n_ref, double cell,
                             double* out_dist, int64_t* out_idx, void* workspace, size_t workspace_bytes,
                             void* stream) {
    if (n_query < 0 || n_ref < 0 || !(cell > 0) || n_ref > INT32_MAX) return EC3R_EARG;
    if (n_query == 0) return EC3R_OK;
    if (!query || !out_dist || !out_idx || (n_ref && !ref)) return EC3R_EARG;
    cudaStream_t st = as_stream(stream);
    if (n_ref == 0) {
        nn_empty_kernel<<<nn_grid(n_query, 256), 256, 0, st>>>(n_query, out_dist, out_idx);
        EC3R_CHECK_LAUNCH("nn_empty_kernel");
        return EC3R_OK;
    }
    if (!workspace || workspace_bytes < ec3r_nn_workspace(n_ref, n_query)) return EC3R_EWORKSPACE;
    const int64_t cap = nn_table_cap(n_ref);
    Carver cv{(char*)workspace, 0};
    long long* k0 = cv.take<long long>(n_ref);
    long long* k1 = cv.take<long long>(n_ref);
    int* i0 = cv.take<int>(n_ref);
    int* i1 = cv.take<int>(n_ref);
    double* sref = cv.take<double>(3 * n_ref);
    NnTable t;
    t.keys = cv.take<long long>(cap);
    t.start = cv.take<int>(cap);
    t.mask = (unsigned long long)(cap - 1);
    int* strays = cv.take<int>(n_query);
    unsigned long long* n_strays = cv.take<unsigned long long>(8);
    size_t sort_bytes = nn_sort_bytes(n_ref);
    void* sort_tmp = cv.take<char>(sort_bytes);
    EC3R_CUDA_TRY(cudaMemsetAsync(t.start, 0xFF, sizeof(int) * (size_t)cap, st));
    EC3R_CUDA_TRY(cudaMemsetAsync(n_strays, 0, sizeof(unsigned long long), st));
    nn_keys_kernel<<<nn_grid(n_ref, 256), 256, 0, st>>>(ref, n_ref, cell, k0, i0);
    EC3R_CHECK_LAUNCH("nn_keys_kernel");
    if (cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, k0, k1, i0, i1, (int)n_ref, 0, 64, st) !=
        cudaSuccess) {
        set_last_error("cub::DeviceRadixSort::SortPairs(nn)", cudaGetLastError());
        return EC3R_ECUDA;
    }
    nn_build_kernel<<<nn_grid(n_ref, 256), 256, 0, st>>>(ref, k1, i1, n_ref, sref, t);
    EC3R_CHECK_LAUNCH("nn_build_kernel");
    nn_query_kernel<<<nn_grid(n_query, 128), 128, 0, st>>>(query, n_query, sref, k1, i1, n_ref, cell, t, out_dist,
                                                       out_idx, strays, n_strays);
    EC3R_CHECK_LAUNCH("nn_query_kernel");
    nn_brute_kernel<<<kNumSMs * 2, 256, 0, st>>>(query, ref, n_ref, strays, n_strays, out_dist, out_idx);
    EC3R_CHECK_LAUNCH("nn_brute_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_raycast(const double* origins, const double* dirs, int64_t n, const double* solids_h,
                            int n_solids, double* out_t, void* stream) {
    if (n < 0 || n_solids < 0 || n_solids > RC_MAX_SOLIDS || (n_solids && !solids_h)) return EC3R_EARG;
    if (n == 0) return EC3R_OK;
    if (!origins || !dirs || !out_t) return EC3R_EARG;
    RcSolids s;
    s.n = n_solids;
    for (int b = 0; b < n_solids; ++b)
        for (int a = 0; a < 3; ++a) {
            s.lo[b][a] = solids_h[6 * b + a];
            s.hi[b][a] = solids_h[6 * b + 3 + a];
        }
    rc_kernel<<<nn_grid(n, 256), 256, 0, as_stream(stream)>>>(origins, dirs, n, s, out_t);
    EC3R_CHECK_LAUNCH("rc_kernel");
    return EC3R_OK;
}

extern "C" int ec3r_synthetic_decode(const double* solids_h, int n_solids, const double* frames, int n_frames, int H,
                                     int W, const double* K4_h, double scale, double sigma, uint64_t key,
                                     float* out_depth, float* out_conf, void* stream) {
    if (n_frames < 0 || H <= 0 || W <= 0 || n_solids < 0 || n_solids > RC_MAX_SOLIDS || (n_solids && !solids_h) ||
        !K4_h || !(sigma >= 0.0))
        return EC3R_EARG;
    if (n_frames == 0) return EC3R_OK;
    if (!frames || !out_depth || !out_conf) return EC3R_EARG;
    RcSolids s;
    s.n = n_solids;
    for (int b = 0; b < n_solids; ++b)
        for (int a = 0; a < 3; ++a) {
            s.lo[b][a] = solids_h[6 * b + a];
            s.hi[b][a] = solids_h[6 * b + 3 + a];
        }
    const int64_t n = (int64_t)n_frames * H * W;
    dec_kernel<<<nn_grid(n, 256), 256, 0, as_stream(stream)>>>(s, frames, n_frames, H, W, K4_h[0], K4_h[1], K4_h[2],
                                                               K4_h[3], scale, sigma, (unsigned long long)key,
                                                               out_depth, out_conf);
    EC3R_CHECK_LAUNCH("dec_kernel");
    return EC3R_OK;
}
