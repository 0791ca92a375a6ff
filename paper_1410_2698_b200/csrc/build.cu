// build.cu — GPU index build (§4, build steps A1-A5 of DESIGN.md).
//
//   A1 validate + extents      P:571-573 (t_min, t_max), P:807-815 (spatial extents,
//                              maximum per-segment extents)
//   A2 sort by t_start         P:569-571 ("sorting the entries in D by ascending
//                              t_start values, re-numbering the entry segments")
//   A3 temporal bins           P:573-590 (b = (t_max - t_min)/m, bin of l_i,
//                              B_j^first / B_j^last / B_j^end)
//   A5 subbin arrays X, Y, Z   P:816-886 (v slabs per dimension, ids stored per
//                              subbin in (slab, bin) lexicographic order)
//   A4 FSG                     P:282-361 (rasterise each MBB to cells; lookup array A)
#include <float.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>

#include "tds_internal.cuh"

namespace tds {

namespace {

constexpr int NT = 256;

__device__ __forceinline__ void atomic_min_key(uint32_t *a, float v) { atomicMin(a, float_key(v)); }
__device__ __forceinline__ void atomic_max_key(uint32_t *a, float v) { atomicMax(a, float_key(v)); }

__host__ __device__ inline float key_float(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

// A1: validate + reduce extents.  red[] layout (order-preserving keys):
// 0 t_min, 1 t_max, 2..4 lo, 5..7 hi, 8..10 maxext, 11 max duration (rounded up)
__global__ void k_validate_extents(const float4 *__restrict__ rec, uint64_t n,
                                   unsigned long long *__restrict__ bad, uint32_t *__restrict__ red) {
    float tmin = FLT_MAX, tmax = -FLT_MAX, lo[3], hi[3], mx[3], dur = 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) { lo[c] = FLT_MAX; hi[c] = -FLT_MAX; mx[c] = 0.f; }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        float4 a = rec[2 * i], b = rec[2 * i + 1];
        bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w) && isfinite(b.x) &&
                  isfinite(b.y) && isfinite(b.z) && isfinite(b.w) && (b.w > a.w);
        if (!ok) { atomicMin(bad, (unsigned long long)i); continue; }
        tmin = fminf(tmin, a.w);
        tmax = fmaxf(tmax, b.w);
        dur = fmaxf(dur, __fsub_ru(b.w, a.w));
        float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = fminf(lo[c], fminf(p0[c], p1[c]));
            hi[c] = fmaxf(hi[c], fmaxf(p0[c], p1[c]));
            mx[c] = fmaxf(mx[c], fabsf(__fsub_rn(p1[c], p0[c])));
        }
    }
    // warp reduce, then block reduce through shared memory, then one set of atomics per block
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        dur = fmaxf(dur, __shfl_xor_sync(0xffffffffu, dur, o));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
            mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
    }
    __shared__ float sred[NT / 32][12];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sred[w][0] = tmin; sred[w][1] = tmax;
        for (int c = 0; c < 3; ++c) { sred[w][2 + c] = lo[c]; sred[w][5 + c] = hi[c]; sred[w][8 + c] = mx[c]; }
        sred[w][11] = dur;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
        const int k = threadIdx.x;
        const bool is_min = (k == 0) || (k >= 2 && k <= 4);
        float v = sred[0][k];
        for (int ww = 1; ww < NT / 32; ++ww) v = is_min ? fminf(v, sred[ww][k]) : fmaxf(v, sred[ww][k]);
        if (is_min) atomic_min_key(&red[k], v); else atomic_max_key(&red[k], v);
    }
}

__global__ void k_init_red(uint32_t *red, unsigned long long *bad) {
    int i = threadIdx.x;
    if (i < 12) {
        bool is_min = (i == 0) || (i >= 2 && i <= 4);
        red[i] = is_min ? 0xffffffffu : 0u;
    }
    if (i == 0) *bad = ~0ull;
}

__global__ void k_time_keys(const float4 *__restrict__ rec, uint64_t n, uint32_t *__restrict__ keys,
                            uint32_t *__restrict__ vals) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        keys[i] = float_key(rec[2 * i].w);
        vals[i] = (uint32_t)i;
    }
}

// spatial renumbering (default order): key of input row i = (temporal bin, Morton
// code of the start point's cell on a 1024^3 grid over D's extent)
__device__ __forceinline__ uint32_t spread3b(uint32_t x) {       // 10 bits -> every third bit
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void k_gather_keys(const uint32_t *__restrict__ src, const uint32_t *__restrict__ idx, uint64_t n,
                              uint32_t *__restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

__global__ void k_fsg_tkeys(const float4 *__restrict__ rec, const uint32_t *__restrict__ ent, uint64_t len,
                            uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) {
        keys[i] = float_key(rec[2 * (uint64_t)ent[i]].w);
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_gather_records(const float4 *__restrict__ src, const uint32_t *__restrict__ perm, uint64_t n,
                                 float4 *__restrict__ dst) {
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one float4 per thread
    if (t < 2 * n) {
        uint64_t i = t >> 1;
        dst[t] = src[2 * (uint64_t)perm[i] + (t & 1)];
    }
}

// window boxes: one warp per aligned window of WBOX_W candidate positions (lane
// takes positions lane + 32 k); the segments' MBB and time span, reduced over
// order-preserving keys (exact min / max of the stored floats)
__global__ void k_window_boxes(const float4 *__restrict__ rec, const uint32_t *__restrict__ arr, uint64_t len,
                               float4 *__restrict__ out) {
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (len + WBOX_W - 1) / WBOX_W;
    if (w >= nw) return;                       // warp-uniform
    uint32_t lx = 0xffffffffu, ly = 0xffffffffu, lz = 0xffffffffu, lt = 0xffffffffu;
    uint32_t hx = 0, hy = 0, hz = 0, ht = 0;
#pragma unroll
    for (int k = 0; k < (int)(WBOX_W / 32); ++k) {
        const uint64_t c = w * WBOX_W + lane + 32 * k;
        if (c < len) {
            const uint64_t j = arr ? arr[c] : c;
            const float4 a = rec[2 * j], b = rec[2 * j + 1];
            lx = min(lx, float_key(fminf(a.x, b.x))); hx = max(hx, float_key(fmaxf(a.x, b.x)));
            ly = min(ly, float_key(fminf(a.y, b.y))); hy = max(hy, float_key(fmaxf(a.y, b.y)));
            lz = min(lz, float_key(fminf(a.z, b.z))); hz = max(hz, float_key(fmaxf(a.z, b.z)));
            lt = min(lt, float_key(a.w));             ht = max(ht, float_key(b.w));
        }
    }
    lx = __reduce_min_sync(0xffffffffu, lx); ly = __reduce_min_sync(0xffffffffu, ly);
    lz = __reduce_min_sync(0xffffffffu, lz); lt = __reduce_min_sync(0xffffffffu, lt);
    hx = __reduce_max_sync(0xffffffffu, hx); hy = __reduce_max_sync(0xffffffffu, hy);
    hz = __reduce_max_sync(0xffffffffu, hz); ht = __reduce_max_sync(0xffffffffu, ht);
    if (lane == 0) {
        out[2 * w] = make_float4(key_float(lx), key_float(ly), key_float(lz), key_float(lt));
        out[2 * w + 1] = make_float4(key_float(hx), key_float(hy), key_float(hz), key_float(ht));
    }
}

// A3: bin of each sorted entry, literal (P:575-576 with reading C12), in fp64
__global__ void k_bin_of(const float4 *__restrict__ rec, uint64_t n, double t_min, double b, int m,
                         uint32_t *__restrict__ bin) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        double j = floor(((double)rec[2 * i].w - t_min) / b);
        int k = j < 0.0 ? 0 : (j >= (double)m ? m - 1 : (int)j);
        bin[i] = (uint32_t)k;
    }
}

// off[k] = first i with key[i] >= k, k = 0..nk (keys sorted, all < nk)
__global__ void k_bucket_offsets(const uint32_t *__restrict__ key, uint64_t n, uint32_t nk,
                                 uint32_t *__restrict__ off) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t prev = (i == 0) ? -1 : (int64_t)key[i - 1];
    int64_t cur = (i == n) ? (int64_t)nk : (int64_t)key[i];
    for (int64_t k = prev + 1; k <= cur; ++k) off[k] = (uint32_t)i;
}

// A3: per bin, one warp reduces max t_end and min t_start over its members
// (+inf / -inf for an empty bin; the min is suffix-filled afterwards)
__global__ void k_bin_extents(const float4 *__restrict__ rec, uint64_t n, const uint32_t *__restrict__ off, int m,
                              float *__restrict__ bin_lo, float *__restrict__ bin_hi) {
    int j = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (j >= m) return;
    uint32_t a = off[j], b = off[j + 1];
    float hmax = -INFINITY, lmin = INFINITY;
    for (uint32_t i = a + lane; i < b; i += 32) {
        hmax = fmaxf(hmax, rec[2 * (uint64_t)i + 1].w);
        lmin = fminf(lmin, rec[2 * (uint64_t)i].w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
        lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
    }
    if (lane == 0) {
        bin_hi[j] = hmax;
        bin_lo[j] = lmin;
    }
}

// lo_j = min over bins j' >= j of the members' min t_start (empty bins take the
// next non-empty bin's; non-decreasing in j), single block of 1024 threads
__global__ void __launch_bounds__(1024) k_suffix_min(float *__restrict__ lo, int m) {
    __shared__ float wmin[32];
    __shared__ float carry_s;
    if (threadIdx.x == 0) carry_s = INFINITY;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < m; b0 += 1024) {
        const int k = m - 1 - (b0 + threadIdx.x);                  // walk from the end
        float x = (k >= 0) ? lo[k] : INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = fminf(x, y);
        }
        if (lane == 31) wmin[w] = x;
        __syncthreads();
        if (w == 0) {
            float y = wmin[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y = fminf(y, z);
            }
            wmin[lane] = y;
        }
        __syncthreads();
        const float carry = carry_s;
        float r = fminf(x, carry);
        if (w > 0) r = fminf(r, wmin[w - 1]);
        if (k >= 0) lo[k] = r;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = r;
        __syncthreads();
    }
}

// prefix max over m values, single block of 1024 threads
__global__ void __launch_bounds__(1024) k_prefix_max(const float *__restrict__ in, float *__restrict__ out, int m) {
    __shared__ float wmax[32];
    __shared__ float carry_s;
    if (threadIdx.x == 0) carry_s = -INFINITY;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b0 = 0; b0 < m; b0 += 1024) {
        int k = b0 + threadIdx.x;
        float x = (k < m) ? in[k] : -INFINITY;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            float y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = fmaxf(x, y);
        }
        if (lane == 31) wmax[w] = x;
        __syncthreads();
        if (w == 0) {
            float v = wmax[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                float y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v = fmaxf(v, y);
            }
            wmax[lane] = v;
        }
        __syncthreads();
        float pre = (w > 0) ? wmax[w - 1] : -INFINITY;
        float r = fmaxf(fmaxf(x, pre), carry_s);
        if (k < m) out[k] = r;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = r;
        __syncthreads();
    }
}

// A5 / A4: number of slabs (cells) of each entry in dimension c / in 3-D
struct Grid3 {
    float o[3], w[3];
    int g[3];
};

__device__ __forceinline__ void cell_box(const float4 &a, const float4 &b, const Grid3 &G, int lo[3], int hi[3]) {
    float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        lo[c] = cell_of(fminf(p0[c], p1[c]), G.o[c], G.w[c], G.g[c]);
        hi[c] = cell_of(fmaxf(p0[c], p1[c]), G.o[c], G.w[c], G.g[c]);
    }
}

// cell-ordered copies for the GPUSpatial pair kernel: record, original row and
// min cell of entry A[i] at position i (the duplicate-avoidance test needs only
// the min corner: 4 B per pair test instead of 8 for min / max)
__global__ void k_fsg_materialise(const float4 *__restrict__ rec, const uint32_t *__restrict__ perm,
                                  const uint32_t *__restrict__ A, uint64_t len, Grid3 G, float4 *__restrict__ frec,
                                  uint32_t *__restrict__ fperm, uint32_t *__restrict__ ecell) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    const uint32_t e = A[i];
    const float4 a = rec[2 * (uint64_t)e], b = rec[2 * (uint64_t)e + 1];
    int lo[3], hi[3];
    cell_box(a, b, G, lo, hi);
    frec[2 * i] = a;
    frec[2 * i + 1] = b;
    fperm[i] = perm[e];
    ecell[i] = pack_cell(lo[0], lo[1], lo[2]);
}

// A5 + A4 phase 1 in one pass over the records: per entry, the number of slabs
// it overlaps in x / y / z and the number of FSG cells
struct StGeom {
    float o[3], w[3];
    int v;
};

__global__ void k_bin_cell_keys(const float4 *__restrict__ rec, uint64_t n, double t_min, double b, int m,
                                StGeom M, uint32_t *__restrict__ kb, uint32_t *__restrict__ km,
                                uint32_t *__restrict__ vals) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 a = rec[2 * i];
    const double j = floor(((double)a.w - t_min) / b);                 // the bin formula of k_bin_of
    kb[i] = (uint32_t)(j < 0.0 ? 0 : (j >= (double)m ? m - 1 : (int)j));
    const uint32_t cx = (uint32_t)cell_of(a.x, M.o[0], M.w[0], 1024), cy = (uint32_t)cell_of(a.y, M.o[1], M.w[1], 1024),
                   cz = (uint32_t)cell_of(a.z, M.o[2], M.w[2], 1024);
    km[i] = (spread3b(cx) << 2) | (spread3b(cy) << 1) | spread3b(cz);
    vals[i] = (uint32_t)i;
}


__global__ void k_count_all(const float4 *__restrict__ rec, uint64_t n, int want_st, StGeom S, int want_fsg,
                            Grid3 G, uint32_t *__restrict__ cx, uint32_t *__restrict__ cy,
                            uint32_t *__restrict__ cz, uint32_t *__restrict__ cf,
                            unsigned long long *__restrict__ fsg_total) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (i < n) {
        const float4 a = rec[2 * i], b = rec[2 * i + 1];
        if (want_st) {
            const float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
            uint32_t *outs[3] = {cx, cy, cz};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int s0 = cell_of(fminf(p0[d], p1[d]), S.o[d], S.w[d], S.v);
                const int s1 = cell_of(fmaxf(p0[d], p1[d]), S.o[d], S.w[d], S.v);
                outs[d][i] = (uint32_t)(s1 - s0 + 1);
            }
        }
        if (want_fsg) {
            int lo[3], hi[3];
            cell_box(a, b, G, lo, hi);
            c = (unsigned long long)(hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
            cf[i] = (uint32_t)c;
        }
    }
    if (want_fsg) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(fsg_total, c);
    }
}

// A5 + A4 phase 2 emission in one pass: (subbin key, entry) pairs of the three
// subbin arrays and (cell key, entry) pairs of the FSG
struct EmitOut {
    const uint32_t *pos[4];          // x, y, z, fsg
    uint32_t *keys[4], *vals[4];
};

__global__ void k_emit_all(const float4 *__restrict__ rec, uint64_t n, int want_st, StGeom S, int mbits,
                           const uint32_t *__restrict__ bin, int want_fsg, Grid3 G, EmitOut E) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 a = rec[2 * i], b = rec[2 * i + 1];
    if (want_st) {
        const float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
        const uint32_t bi = bin[i];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int s0 = cell_of(fminf(p0[d], p1[d]), S.o[d], S.w[d], S.v);
            const int s1 = cell_of(fmaxf(p0[d], p1[d]), S.o[d], S.w[d], S.v);
            uint32_t k = E.pos[d][i];
            for (int sl = s0; sl <= s1; ++sl, ++k) {
                E.keys[d][k] = ((uint32_t)sl << mbits) | bi;     // subbin (slab j, bin i)
                E.vals[d][k] = (uint32_t)i;
            }
        }
    }
    if (want_fsg) {
        int lo[3], hi[3];
        cell_box(a, b, G, lo, hi);
        uint32_t k = E.pos[3][i];
        for (int x = lo[0]; x <= hi[0]; ++x)
            for (int y = lo[1]; y <= hi[1]; ++y)
                for (int z = lo[2]; z <= hi[2]; ++z, ++k) {
                    E.keys[3][k] = (uint32_t)(((uint64_t)x * G.g[1] + y) * G.g[2] + z);   // row-major h
                    E.vals[3][k] = (uint32_t)i;
                }
    }
}

inline unsigned nblk(uint64_t n, int nt = NT) { return (unsigned)((n + nt - 1) / nt); }

float4 *window_boxes(const float4 *rec, const uint32_t *arr, uint64_t len, cudaStream_t s) {
    const uint64_t nw = (len + WBOX_W - 1) / WBOX_W;
    DBuf<float4> wb(std::max<uint64_t>(2 * nw, 2), s);
    if (nw) {
        k_window_boxes<<<nblk(nw * 32), NT, 0, s>>>(rec, arr, len, wb.p);
        TDS_CHECK_LAUNCH();
    }
    return wb.release();
}



int bits_for(uint64_t nk) {
    int b = 0;
    while ((1ull << b) < nk) ++b;
    return b;
}

// st_off[j*m + i] = first position of subbin (slab j, bin i) in keys sorted by
// (j << mbits) | i (one thread per subbin, binary search)
__global__ void k_subbin_offsets(const uint32_t *__restrict__ keys, uint64_t len, int v, int m, int mbits,
                                 uint32_t *__restrict__ off) {
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > (uint64_t)v * m) return;
    uint32_t key = (t == (uint64_t)v * m) ? 0xffffffffu
                                          : (((uint32_t)(t / m) << mbits) | (uint32_t)(t % m));
    uint64_t lo = 0, hi = len;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    off[t] = (uint32_t)lo;
}

// group (key, val) pairs by key with a stable radix sort; vals -> out ids,
// offsets of the nk buckets -> off[nk+1]
void group_by_key(DBuf<uint32_t> &keys, DBuf<uint32_t> &vals, uint64_t len, uint64_t nk, uint32_t *off,
                  cudaStream_t s) {
    radix_sort_pairs(keys, vals, len, 0, bits_for(nk), s);
    k_bucket_offsets<<<nblk(len + 1), NT, 0, s>>>(keys.p, len, (uint32_t)nk, off);
    TDS_CHECK_LAUNCH();
}

}  // namespace

uint64_t validate_segments(const float4 *rec, uint64_t n, cudaStream_t s) {
    DBuf<unsigned long long> bad(1, s);
    DBuf<uint32_t> red(16, s);
    k_init_red<<<1, 32, 0, s>>>(red.p, bad.p);
    TDS_CHECK_LAUNCH();
    k_validate_extents<<<std::min<uint64_t>(nblk(n), 4096), NT, 0, s>>>(rec, n, bad.p, red.p);
    TDS_CHECK_LAUNCH();
    unsigned long long h = 0;
    TDS_CUDA(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    return h;
}

void build_index(const tds_seg *entries, uint64_t n, const tds_index_params *p, cudaStream_t s,
                 tds_index_s *idx) {
    const float4 *in = reinterpret_cast<const float4 *>(entries);
    Trace tr(s);
    idx->n = n;
    idx->m = p->m_bins;
    idx->v = p->v_subbins;
    for (int c = 0; c < 3; ++c) idx->grid[c] = p->grid[c];
    idx->kinds = p->kinds | TDS_TEMPORAL;

    // ---- A1: validate + extents --------------------------------------------
    DBuf<unsigned long long> bad(1, s);
    DBuf<uint32_t> red(16, s);
    k_init_red<<<1, 32, 0, s>>>(red.p, bad.p);
    TDS_CHECK_LAUNCH();
    k_validate_extents<<<std::min<uint64_t>(nblk(n), (uint64_t)num_sms() * 8), NT, 0, s>>>(in, n, bad.p, red.p);
    TDS_CHECK_LAUNCH();
    unsigned long long hbad;
    uint32_t hred[16];
    TDS_CUDA(cudaMemcpyAsync(&hbad, bad.p, 8, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaMemcpyAsync(hred, red.p, 12 * 4, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    if (hbad != ~0ull)
        fail(TDS_EDATA, "entry segment %llu has a non-finite value or t_end <= t_start", hbad);
    Extents &E = idx->ext;
    E.t_min = key_float(hred[0]);
    E.t_max = key_float(hred[1]);
    for (int c = 0; c < 3; ++c) {
        E.lo[c] = key_float(hred[2 + c]);
        E.hi[c] = key_float(hred[5 + c]);
        E.maxext[c] = key_float(hred[8 + c]);
    }
    E.max_dur = key_float(hred[11]);
    const bool want_st = (p->kinds & TDS_SPATIOTEMPORAL) != 0;
    const bool want_fsg = (p->kinds & TDS_SPATIAL) != 0;
    if (want_st) {   // admissible v: v <= (c_max - c_min) / max |c_start - c_end|
        for (int c = 0; c < 3; ++c) {
            double ext = (double)E.hi[c] - (double)E.lo[c];
            if (E.maxext[c] > 0.f && (double)idx->v > ext / (double)E.maxext[c])
                fail(TDS_EINVAL, "v_subbins=%d exceeds the admissible bound %.3f in dimension %d (P:816-821)",
                     idx->v, ext / (double)E.maxext[c], c);
        }
    }

    tr.mark("validate+sync");
    // ---- A2: stable radix sort by t_start, renumber, gather -----------------
    // (default: by temporal bin, then Morton code of the start cell; TDS_INDEX_TIME_ORDER:
    // by t_start; both stable, so ties keep the input order)
    const int m = idx->m;
    double t_min = E.t_min, b = ((double)E.t_max - (double)E.t_min) / (double)m;
    if (!(b > 0.0)) b = 1.0;
    idx->time_order = (p->flags & TDS_INDEX_TIME_ORDER) != 0;
    DBuf<uint32_t> keys(n, s), perm(n, s);
    if (idx->time_order) {
        k_time_keys<<<nblk(n), NT, 0, s>>>(in, n, keys.p, perm.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(keys.p, perm.p, n, 0, 32, s);
    } else {
        StGeom M{};
        for (int c = 0; c < 3; ++c) {
            const float ext = E.hi[c] - E.lo[c];
            M.o[c] = E.lo[c];
            M.w[c] = ext > 0.f ? ext / 1024.f : 1.0f;
        }
        DBuf<uint32_t> km(n, s), kb2(n, s);
        k_bin_cell_keys<<<nblk(n), NT, 0, s>>>(in, n, t_min, b, m, M, keys.p, km.p, perm.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(km.p, perm.p, n, 0, 30, s);
        k_gather_keys<<<nblk(n), NT, 0, s>>>(keys.p, perm.p, n, kb2.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(kb2.p, perm.p, n, 0, bits_for((uint64_t)m), s);
    }
    DBuf<float4> rec(2 * n, s);
    k_gather_records<<<nblk(2 * n), NT, 0, s>>>(in, perm.p, n, rec.p);
    TDS_CHECK_LAUNCH();
    keys.reset();

    tr.mark("tsort+gather");
    // ---- A3: temporal bins ---------------------------------------------------
    DBuf<uint32_t> bin(n, s), bin_off(m + 1, s);
    DBuf<float> bin_lo(m, s), bin_hi(m, s), bin_pmhi(m, s);
    k_bin_of<<<nblk(n), NT, 0, s>>>(rec.p, n, t_min, b, m, bin.p);
    TDS_CHECK_LAUNCH();
    k_bucket_offsets<<<nblk(n + 1), NT, 0, s>>>(bin.p, n, (uint32_t)m, bin_off.p);
    TDS_CHECK_LAUNCH();
    k_bin_extents<<<nblk((uint64_t)m * 32), NT, 0, s>>>(rec.p, n, bin_off.p, m, bin_lo.p, bin_hi.p);
    TDS_CHECK_LAUNCH();
    k_prefix_max<<<1, 1024, 0, s>>>(bin_hi.p, bin_pmhi.p, m);
    TDS_CHECK_LAUNCH();
    k_suffix_min<<<1, 1024, 0, s>>>(bin_lo.p, m);
    TDS_CHECK_LAUNCH();

    tr.mark("bins");
    // ---- A5 + A4, phase 1: membership counts and their prefix sums for the three
    // subbin arrays and the FSG, read back with ONE synchronisation
    const int v = idx->v;
    Grid3 G{};
    uint64_t ncell = 1;
    if (want_fsg) {
        for (int c = 0; c < 3; ++c) {
            if (idx->grid[c] < 1) fail(TDS_EINVAL, "grid[%d] = %d < 1", c, idx->grid[c]);
            float ext = E.hi[c] - E.lo[c];
            G.o[c] = E.lo[c];
            G.g[c] = idx->grid[c];
            G.w[c] = ext > 0.f ? ext / (float)idx->grid[c] : 1.0f;
            idx->w_fsg[c] = G.w[c];
            ncell *= (uint64_t)idx->grid[c];
        }
        if (ncell >= (1ull << 31)) fail(TDS_EINVAL, "grid has %llu cells (limit 2^31)", (unsigned long long)ncell);
        if (idx->grid[0] > FSG_MAX_X || idx->grid[1] > FSG_MAX_Y || idx->grid[2] > FSG_MAX_Z)
            fail(TDS_EINVAL, "grid %d x %d x %d exceeds %d x %d x %d", idx->grid[0], idx->grid[1], idx->grid[2],
                 FSG_MAX_X, FSG_MAX_Y, FSG_MAX_Z);
    }
    // one pass over the records counts the slab memberships of x / y / z and the
    // FSG cells of every entry; one batched scan turns them into emit positions
    DBuf<uint32_t> st_pos[3];
    DBuf<uint32_t> fsg_pos;
    DBuf<unsigned long long> totals(4, s);       // ST x, y, z lengths; FSG length
    TDS_CUDA(cudaMemsetAsync(totals.p, 0, 32, s));
    StGeom SG{};
    SG.v = v;
    for (int c = 0; c < 3; ++c) {
        float ext = E.hi[c] - E.lo[c];
        E.w_st[c] = ext > 0.f ? ext / (float)v : 1.0f;
        SG.o[c] = E.lo[c];
        SG.w[c] = E.w_st[c];
    }
    if (want_st || want_fsg) {
        DBuf<uint32_t> cnt(4 * n, s);
        if (want_st)
            for (int c = 0; c < 3; ++c) st_pos[c] = DBuf<uint32_t>(n, s);
        if (want_fsg) fsg_pos = DBuf<uint32_t>(n, s);
        k_count_all<<<nblk(n), NT, 0, s>>>(rec.p, n, want_st, SG, want_fsg, G, cnt.p, cnt.p + n, cnt.p + 2 * n,
                                           cnt.p + 3 * n, totals.p + 3);
        TDS_CHECK_LAUNCH();
        const uint32_t *in[4];
        uint32_t *out[4], *tot32[4];
        int k = 0;
        if (want_st)
            for (int c = 0; c < 3; ++c, ++k) {
                in[k] = cnt.p + (uint64_t)c * n;
                out[k] = st_pos[c].p;
                tot32[k] = (uint32_t *)(totals.p + c);
            }
        if (want_fsg) {
            in[k] = cnt.p + 3 * n;
            out[k] = fsg_pos.p;
            tot32[k] = nullptr;                     // the FSG total is summed in 64 bits above
            ++k;
        }
        exclusive_scan_u32_batch(k, in, out, tot32, n, s);
    }
    unsigned long long tot[4] = {0, 0, 0, 0};
    if (want_st || want_fsg) {
        TDS_CUDA(cudaMemcpyAsync(tot, totals.p, 32, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
    }

    tr.mark("counts+sync");
    // ---- phase 2: emission of all four structures in one pass over the records,
    // then per structure the grouping sort and its offsets
    const int mbits = bits_for((uint64_t)m);
    DBuf<uint32_t> sk[3], sv[3], fk, fv;
    EmitOut EO{};
    if (want_st)
        for (int c = 0; c < 3; ++c) {
            const uint64_t len = tot[c] & 0xffffffffull;
            sk[c] = DBuf<uint32_t>(len, s);
            sv[c] = DBuf<uint32_t>(len, s);
            EO.pos[c] = st_pos[c].p;
            EO.keys[c] = sk[c].p;
            EO.vals[c] = sv[c].p;
        }
    if (want_fsg) {
        if (tot[3] >= (1ull << 32) - 1)
            fail(TDS_EINVAL, "FSG lookup array would hold %llu ids (limit 2^32); use a coarser grid", tot[3]);
        fk = DBuf<uint32_t>(tot[3], s);
        fv = DBuf<uint32_t>(tot[3], s);
        EO.pos[3] = fsg_pos.p;
        EO.keys[3] = fk.p;
        EO.vals[3] = fv.p;
    }
    if (want_st || want_fsg) {
        k_emit_all<<<nblk(n), NT, 0, s>>>(rec.p, n, want_st, SG, mbits, bin.p, want_fsg, G, EO);
        TDS_CHECK_LAUNCH();
    }
    for (int c = 0; c < 3; ++c) st_pos[c].reset();
    fsg_pos.reset();

    // ---- A5, phase 2: spatiotemporal subbin arrays ------------------
    if (want_st) {
        for (int c = 0; c < 3; ++c) {
            const uint64_t len = tot[c] & 0xffffffffull;
            DBuf<uint32_t> off((uint64_t)v * m + 1, s);
            // emitted in sorted-position order, so within a slab the bins are already
            // ascending: a stable sort on the slab bits alone groups the subbins
            radix_sort_pairs(sk[c], sv[c], len, mbits, mbits + bits_for((uint64_t)v), s);
            k_subbin_offsets<<<nblk((uint64_t)v * m + 1), NT, 0, s>>>(sk[c].p, len, v, m, mbits, off.p);
            TDS_CHECK_LAUNCH();
            // optional materialised records in X/Y/Z order (ablation): the
            // range kernel then streams them instead of gathering rec[X[i]]
            if (!st_indirect()) {
                DBuf<float4> srec(2 * len, s, 2 * len * sizeof(float4) > (256ull << 20));
                if (len) {
                    k_gather_records<<<nblk(2 * len), NT, 0, s>>>(rec.p, sv[c].p, len, srec.p);
                    TDS_CHECK_LAUNCH();
                }
                idx->st_rec[c] = srec.release();
            }
            sk[c].reset();
            idx->wb_st[c] = window_boxes(rec.p, sv[c].p, len, s);
            idx->st_arr[c] = sv[c].release();
            idx->st_len[c] = len;
            idx->st_off[c] = off.release();
        }
    }

    // ---- A4, phase 2: FSG (dense CSR over all cells) -----------------
    if (want_fsg) {
        const unsigned long long len = tot[3];
        DBuf<uint32_t> off(ncell + 1, s);
        if (!idx->time_order && len > 1) {
            // the cells' entries in t_start order (the per-cell time trimming of the
            // search binary-searches it): stable sort by t_start before the stable
            // grouping by cell (the sorted D is in (bin, Morton) order)
            DBuf<uint32_t> tk(len, s), ix(len, s), k2(len, s), v2(len, s);
            k_fsg_tkeys<<<nblk(len), NT, 0, s>>>(rec.p, fv.p, len, tk.p, ix.p);
            TDS_CHECK_LAUNCH();
            radix_sort_pairs(tk, ix, len, 0, 32, s);
            k_gather_keys<<<nblk(len), NT, 0, s>>>(fk.p, ix.p, len, k2.p);
            TDS_CHECK_LAUNCH();
            k_gather_keys<<<nblk(len), NT, 0, s>>>(fv.p, ix.p, len, v2.p);
            TDS_CHECK_LAUNCH();
            std::swap(fk.p, k2.p);
            std::swap(fv.p, v2.p);
        }
        group_by_key(fk, fv, len, ncell, off.p, s);
        fk.reset();
        DBuf<uint32_t> ecell(len, s);
        DBuf<float4> frec(2 * len, s);
        DBuf<uint32_t> fperm(len, s);
        k_fsg_materialise<<<nblk(len), NT, 0, s>>>(rec.p, perm.p, fv.p, len, G, frec.p, fperm.p, ecell.p);
        TDS_CHECK_LAUNCH();
        idx->wb_fsg = window_boxes(frec.p, nullptr, len, s);
        idx->fsg_ecell = ecell.release();
        idx->fsg_rec = frec.release();
        idx->fsg_perm = fperm.release();
        idx->fsg_A = fv.release();
        idx->A_len = len;
        idx->cell_off = off.release();
        idx->n_cells = ncell;
    }
    bin.s = s;
    tr.mark("st+fsg");

    idx->wb_rec = window_boxes(rec.p, nullptr, n, s);
    idx->rec = rec.release();
    idx->perm = perm.release();
    idx->bin_off = bin_off.release();
    idx->bin_lo = bin_lo.release();
    idx->bin_hi = bin_hi.release();
    idx->bin_pmhi = bin_pmhi.release();
    TDS_CUDA(cudaStreamSynchronize(s));
}

// GPUSpatioTemporal reads candidates through X/Y/Z as in the paper; the
// materialised X/Y/Z-ordered record copies are an ablation,
// TDS_ST_MATERIALISE=1: on B200 they measured no faster (the range kernel is
// issue-bound and L1/L2 absorb the gather) and cost build time
bool st_indirect() {
    const char *e = getenv("TDS_ST_MATERIALISE");
    return !(e && e[0] == '1');
}

void free_index(tds_index_s *idx) {
    cudaStream_t s = 0;
    auto f = [&](void *p) { if (p) dfree(p, s); };
    f(idx->rec); f(idx->perm); f(idx->bin_off); f(idx->bin_lo); f(idx->bin_hi); f(idx->bin_pmhi);
    for (int c = 0; c < 3; ++c) { f(idx->st_arr[c]); f(idx->st_off[c]); f(idx->st_rec[c]); }
    f(idx->cell_off); f(idx->fsg_A); f(idx->fsg_ecell); f(idx->fsg_rec); f(idx->fsg_perm);
    f(idx->wb_rec); f(idx->wb_fsg);
    for (int c = 0; c < 3; ++c) f(idx->wb_st[c]);
    cudaStreamSynchronize(s);
}

}  // namespace tds
