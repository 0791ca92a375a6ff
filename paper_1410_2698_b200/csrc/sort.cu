// sort.cu — device primitives hand-written for sm_100a: exclusive scan
// (reduce-then-scan) and a stable LSD radix sort of (uint32 key, uint32 value)
// pairs.  Used by the index build (t_start sort P:569-571, subbin / cell
// grouping P:347-361) and by query preparation (sort Q by t_start,
// P:681-682; sort S by the array selector).
#include <algorithm>

#include "tds_internal.cuh"

namespace tds {

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;   // 4096 elements per block

template <class T>
__device__ __forceinline__ T warp_incl_scan(T x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, writes the block total to *total.
template <class T, int NT>
__device__ __forceinline__ T block_excl_scan(T x, T *total) {
    __shared__ T wsum[NT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T inc = warp_incl_scan(x);
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        T v = (lane < NT / 32) ? wsum[lane] : T(0);
        T vi = warp_incl_scan(v);
        if (lane < NT / 32) wsum[lane] = vi - v;
        if (lane == NT / 32 - 1) *total = vi;
    }
    __syncthreads();
    T r = inc - x + wsum[w];
    __syncthreads();
    return r;
}

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const T *__restrict__ in, uint64_t n,
                                                              T *__restrict__ partial) {
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        uint64_t k = base + (uint64_t)i * SCAN_THREADS + threadIdx.x;
        if (k < n) s += in[k];
    }
    __shared__ T tot;
    block_excl_scan<T, SCAN_THREADS>(s, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// single block: exclusive scan of partial[0..nb) in place, total -> *d_total
template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(T *partial, uint64_t nb, T *d_total) {
    __shared__ T tot;
    T carry = 0;
    for (uint64_t b0 = 0; b0 < nb; b0 += SCAN_THREADS) {
        uint64_t k = b0 + threadIdx.x;
        T x = (k < nb) ? partial[k] : T(0);
        T e = block_excl_scan<T, SCAN_THREADS>(x, &tot);
        if (k < nb) partial[k] = carry + e;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(const T *__restrict__ in, T *out, uint64_t n,
                                                             const T *__restrict__ partial) {
    __shared__ T buf[SCAN_TILE];
    __shared__ T tot;
    uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {        // coalesced load (striped)
        int j = i * SCAN_THREADS + threadIdx.x;
        uint64_t k = base + j;
        buf[j] = (k < n) ? in[k] : T(0);
    }
    __syncthreads();
    T v[SCAN_ITEMS];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {        // blocked: thread owns 8 consecutive
        v[i] = buf[threadIdx.x * SCAN_ITEMS + i];
        s += v[i];
    }
    T e = block_excl_scan<T, SCAN_THREADS>(s, &tot) + partial[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        buf[threadIdx.x * SCAN_ITEMS + i] = e;
        e += v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int j = i * SCAN_THREADS + threadIdx.x;
        uint64_t k = base + j;
        if (k < n) out[k] = buf[j];
    }
}

// ---------------------------------------------------------------------------
// radix sort
// ---------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;                        // keys per thread
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;     // 2048 keys per tile

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t *__restrict__ keys, uint64_t n,
                                                        int shift, uint32_t mask, uint32_t *__restrict__ hist,
                                                        uint32_t ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    uint64_t base = (uint64_t)blockIdx.x * RS_TILE;
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        uint64_t k = base + (uint64_t)r * RS_THREADS + threadIdx.x;
        if (k < n) atomicAdd(&h[(keys[k] >> shift) & mask], 1u);
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint32_t *__restrict__ kin,
                                                           const uint32_t *__restrict__ vin,
                                                           uint32_t *__restrict__ kout,
                                                           uint32_t *__restrict__ vout, uint64_t n, int shift,
                                                           uint32_t mask, const uint32_t *__restrict__ offs,
                                                           uint32_t ntiles) {
    __shared__ uint32_t cnt[RS_WARPS][256];
    __shared__ uint32_t base[256];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&cnt[0][0])[i] = 0;
    base[threadIdx.x] = offs[(uint64_t)threadIdx.x * ntiles + blockIdx.x];
    __syncthreads();
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t key[RS_ROUNDS], val[RS_ROUNDS], rank[RS_ROUNDS];
    int dig[RS_ROUNDS];
    uint64_t tbase = (uint64_t)blockIdx.x * RS_TILE + (uint64_t)w * (32 * RS_ROUNDS);
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        uint64_t k = tbase + (uint64_t)r * 32 + lane;
        bool valid = k < n;
        key[r] = valid ? kin[k] : 0u;
        val[r] = valid ? vin[k] : 0u;
        int d = valid ? (int)((key[r] >> shift) & mask) : 256;
        dig[r] = d;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t lt = __popc(peers & lt_mask);
        uint32_t c = (d < 256) ? cnt[w][d] : 0u;
        rank[r] = c + lt;
        __syncwarp();
        if (d < 256 && lt == 0) cnt[w][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // exclusive prefix over warps, per digit (thread = digit)
        uint32_t run = 0;
        const int d = threadIdx.x;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            uint32_t t = cnt[ww][d];
            cnt[ww][d] = run + base[d];
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        if (dig[r] < 256) {
            uint32_t pos = cnt[w][dig[r]] + rank[r];
            kout[pos] = key[r];
            vout[pos] = val[r];
        }
    }
}

// ---------------------------------------------------------------------------
// single-pass chained scan (decoupled look-back): one launch per scan
// status word per tile: flag (2 high bits: 1 = aggregate, 2 = inclusive prefix)
// | 62-bit value
// ---------------------------------------------------------------------------
constexpr unsigned long long ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t ld_volatile32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// warp 0 of the block: exclusive prefix of tile t from its predecessors
__device__ __forceinline__ unsigned long long lookback(unsigned long long *status, long long t) {
    const int lane = threadIdx.x & 31;
    unsigned long long prefix = 0;
    long long k = t - 1;
    while (k >= 0) {
        long long idx = k - lane;
        unsigned long long s = ST_INC;            // beyond tile 0: inclusive 0
        if (idx >= 0) {
            do { s = ld_volatile(status + idx); } while ((s >> 62) == 0);
        }
        unsigned inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        unsigned long long v = s & ST_VAL;
        int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long part = (lane <= stop) ? v : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        prefix += part;
        if (inc) break;
        k -= 32;
    }
    return prefix;
}

template <class T>
__device__ __forceinline__ void scan_chained_tile(const T *__restrict__ in, T *out, uint64_t n,
                                                  unsigned long long *status, unsigned *tile_ctr, T *d_total,
                                                  uint64_t ntiles) {
    __shared__ T buf[SCAN_TILE];
    __shared__ T tot;
    __shared__ unsigned long long s_prefix;
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint64_t t = s_tile;
    const uint64_t base = t * SCAN_TILE;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int j = i * SCAN_THREADS + threadIdx.x;
        uint64_t k = base + j;
        buf[j] = (k < n) ? in[k] : T(0);
    }
    __syncthreads();
    T v[SCAN_ITEMS];
    T sum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = buf[threadIdx.x * SCAN_ITEMS + i];
        sum += v[i];
    }
    T e = block_excl_scan<T, SCAN_THREADS>(sum, &tot);
    if (threadIdx.x < 32) {
        if (t == 0) {
            if (threadIdx.x == 0) {
                atomicExch(status, ST_INC | (unsigned long long)tot);
                s_prefix = 0;
            }
        } else {
            if (threadIdx.x == 0) atomicExch(status + t, ST_AGG | (unsigned long long)tot);
            unsigned long long pre = lookback(status, (long long)t);
            if (threadIdx.x == 0) {
                atomicExch(status + t, ST_INC | (pre + (unsigned long long)tot));
                s_prefix = pre;
            }
        }
    }
    __syncthreads();
    e += (T)s_prefix;
    if (t == ntiles - 1 && threadIdx.x == 0 && d_total) *d_total = (T)s_prefix + tot;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        buf[threadIdx.x * SCAN_ITEMS + i] = e;
        e += v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int j = i * SCAN_THREADS + threadIdx.x;
        uint64_t k = base + j;
        if (k < n) out[k] = buf[j];
    }
}

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_chained(const T *__restrict__ in, T *out, uint64_t n,
                                                               unsigned long long *status, unsigned *tile_ctr,
                                                               T *d_total, uint64_t ntiles) {
    scan_chained_tile<T>(in, out, n, status, tile_ctr, d_total, ntiles);
}

// up to 4 independent scans of n elements in one launch (blockIdx.y = scan)
struct ScanBatch {
    const uint32_t *in[4];
    uint32_t *out[4];
    uint32_t *total[4];
};

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_chained_batch(ScanBatch B, uint64_t n,
                                                                     unsigned long long *status, uint64_t ntiles) {
    const int y = blockIdx.y;
    unsigned long long *st = status + (uint64_t)y * (ntiles + 1);
    scan_chained_tile<uint32_t>(B.in[y], B.out[y], n, st, (unsigned *)(st + ntiles), B.total[y], ntiles);
}


// ---------------------------------------------------------------------------
// onesweep radix sort: one histogram pass for all digits, then one
// decoupled-look-back scatter per digit (status per (tile, digit): 2-bit flag |
// 30-bit count)
// ---------------------------------------------------------------------------
constexpr uint32_t RS_AGG = 1u << 30, RS_INC = 2u << 30, RS_VAL = (1u << 30) - 1;

__global__ void __launch_bounds__(RS_THREADS) k_rs_upsweep(const uint32_t *__restrict__ keys, uint64_t n,
                                                           int begin_bit, int npass, int end_bit,
                                                           uint32_t *__restrict__ ghist) {
    __shared__ uint32_t h[4][256];
    for (int i = threadIdx.x; i < 4 * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t k = (uint64_t)blockIdx.x * RS_THREADS + threadIdx.x; k < n; k += (uint64_t)gridDim.x * RS_THREADS) {
        uint32_t key = keys[k];
        for (int p = 0; p < npass; ++p) {
            int shift = begin_bit + 8 * p;
            int nb = end_bit - shift < 8 ? end_bit - shift : 8;
            atomicAdd(&h[p][(key >> shift) & ((1u << nb) - 1u)], 1u);
        }
    }
    __syncthreads();
    for (int p = 0; p < npass; ++p) {
        uint32_t c = h[p][threadIdx.x];
        if (c) atomicAdd(&ghist[p * 256 + threadIdx.x], c);
    }
}

constexpr int OS_ROUNDS = 16;                       // keys per thread (onesweep)
constexpr int OS_TILE = RS_THREADS * OS_ROUNDS;      // 4096 keys per tile

struct __align__(16) OsSmem {
    uint32_t cnt[RS_WARPS][256];     // per-warp digit counts -> warp offsets in the tile
    uint32_t tstart[256];            // digit start in the tile-sorted order
    uint32_t gpos[256];              // global start of this tile's run of digit d
    uint32_t key[OS_TILE];           // tile staged in digit order
    uint32_t val[OS_TILE];
    unsigned tile;
    uint32_t tot;
};

// One onesweep pass: rank the tile's keys per digit (warp match + per-warp
// counts), publish per-digit tile counts and look back over predecessor tiles
// (decoupled look-back), stage the tile in digit order in shared memory, then
// write each digit's run to its global position with consecutive threads on
// consecutive addresses (coalesced).
__global__ void __launch_bounds__(RS_THREADS) k_rs_onesweep(const uint32_t *__restrict__ kin,
                                                            const uint32_t *__restrict__ vin,
                                                            uint32_t *__restrict__ kout, uint32_t *__restrict__ vout,
                                                            uint64_t n, int shift, uint32_t mask,
                                                            const uint32_t *__restrict__ ghist,
                                                            uint32_t *status, unsigned *tile_ctr) {
    extern __shared__ __align__(16) unsigned char os_raw[];
    OsSmem &S = *reinterpret_cast<OsSmem *>(os_raw);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) S.tile = atomicAdd(tile_ctr, 1u);
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&S.cnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = S.tile;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t key[OS_ROUNDS], val[OS_ROUNDS];
    uint32_t rank[OS_ROUNDS];
    const uint64_t tbase = (uint64_t)tile * OS_TILE + (uint64_t)w * (32 * OS_ROUNDS);
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; ++r) {
        uint64_t k = tbase + (uint64_t)r * 32 + lane;
        bool valid = k < n;
        key[r] = valid ? kin[k] : 0u;
        val[r] = valid ? vin[k] : 0u;
    }
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; ++r) {
        uint64_t k = tbase + (uint64_t)r * 32 + lane;
        int d = (k < n) ? (int)((key[r] >> shift) & mask) : 256;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t lt = __popc(peers & lt_mask);
        uint32_t c = (d < 256) ? S.cnt[w][d] : 0u;
        rank[r] = (d < 256) ? (c + lt) : 0xffffffffu;
        __syncwarp();
        if (d < 256 && lt == 0) S.cnt[w][d] = c + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // thread = digit: exclusive over warps, tile count, publish, look back
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ++ww) {
        uint32_t t = S.cnt[ww][d];
        S.cnt[ww][d] = run;
        run += t;
    }
    uint32_t *st = status + (uint64_t)tile * 256 + d;
    uint32_t excl = 0;
    if (tile == 0) {
        atomicExch(st, RS_INC | run);
    } else {
        atomicExch(st, RS_AGG | run);
        // look back 8 predecessor tiles per step (independent loads in flight)
        int64_t k = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
            uint32_t sv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) sv[j] = (k - j >= 0) ? ld_volatile32(status + (uint64_t)(k - j) * 256 + d)
                                                          : RS_INC;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (done) break;
                while ((sv[j] >> 30) == 0) sv[j] = ld_volatile32(status + (uint64_t)(k - j) * 256 + d);
                excl += sv[j] & RS_VAL;
                if ((sv[j] >> 30) == 2) done = true;
            }
            k -= 8;
        }
        atomicExch(st, RS_INC | (excl + run));
    }
    const uint32_t tstart = block_excl_scan<uint32_t, RS_THREADS>(run, &S.tot);
    const uint32_t gex = block_excl_scan<uint32_t, RS_THREADS>(ghist[d], &S.tot);
    S.tstart[d] = tstart;
    S.gpos[d] = gex + excl;
    __syncthreads();
    // stage the tile in digit order
#pragma unroll
    for (int r = 0; r < OS_ROUNDS; ++r) {
        if (rank[r] != 0xffffffffu) {
            const int dd = (int)((key[r] >> shift) & mask);
            const uint32_t pos = S.tstart[dd] + S.cnt[w][dd] + rank[r];
            S.key[pos] = key[r];
            S.val[pos] = val[r];
        }
    }
    __syncthreads();
    // coalesced write-out: position i of the tile-sorted order
    const uint64_t tile_n = min((uint64_t)OS_TILE, n - (uint64_t)tile * OS_TILE);
    for (uint32_t i = threadIdx.x; i < tile_n; i += RS_THREADS) {
        const uint32_t kk = S.key[i];
        const int dd = (int)((kk >> shift) & mask);
        const uint32_t pos = S.gpos[dd] + (i - S.tstart[dd]);
        kout[pos] = kk;
        vout[pos] = S.val[i];
    }
}

template <class T>
void exclusive_scan_impl(const T *in, T *out, uint64_t n, T *d_total, cudaStream_t s) {
    if (n == 0) {
        if (d_total) TDS_CUDA(cudaMemsetAsync(d_total, 0, sizeof(T), s));
        return;
    }
    uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    DBuf<unsigned long long> status(nb + 1, s);          // last word: tile counter
    TDS_CUDA(cudaMemsetAsync(status.p, 0, 8 * (nb + 1), s));
    k_scan_chained<T><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, status.p, (unsigned *)(status.p + nb),
                                                            d_total, nb);
    TDS_CHECK_LAUNCH();
}

}  // namespace

void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, uint32_t *d_total, cudaStream_t s) {
    exclusive_scan_impl<uint32_t>(in, out, n, d_total, s);
}

void exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *d_total, cudaStream_t s) {
    exclusive_scan_impl<uint64_t>(in, out, n, d_total, s);
}

void exclusive_scan_u32_batch(int k, const uint32_t *const *in, uint32_t *const *out, uint32_t *const *d_total,
                              uint64_t n, cudaStream_t s) {
    if (k < 1 || k > 4) fail(TDS_EINVAL, "exclusive_scan_u32_batch: k = %d", k);
    if (n == 0) {
        for (int y = 0; y < k; ++y)
            if (d_total[y]) TDS_CUDA(cudaMemsetAsync(d_total[y], 0, 4, s));
        return;
    }
    ScanBatch B{};
    for (int y = 0; y < k; ++y) { B.in[y] = in[y]; B.out[y] = out[y]; B.total[y] = d_total[y]; }
    const uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    DBuf<unsigned long long> status((uint64_t)k * (nb + 1), s);   // per scan: tile states + tile counter
    TDS_CUDA(cudaMemsetAsync(status.p, 0, 8 * (uint64_t)k * (nb + 1), s));
    k_scan_chained_batch<<<dim3((unsigned)nb, (unsigned)k), SCAN_THREADS, 0, s>>>(B, n, status.p, nb);
    TDS_CHECK_LAUNCH();
}

// the passes; returns true if the sorted data ended in (k2, v2) (odd pass count)
static bool radix_sort_passes(uint32_t *keys, uint32_t *vals, uint32_t *k2p, uint32_t *v2p, uint64_t n,
                              int begin_bit, int end_bit, cudaStream_t s) {
    const uint32_t ntiles = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
    const uint32_t os_tiles = (uint32_t)((n + OS_TILE - 1) / OS_TILE);
    const int npass = (end_bit - begin_bit + 7) / 8;
    uint32_t *ka = keys, *va = vals, *kb = k2p, *vb = v2p;
    if (n < (1ull << 30)) {
        // onesweep: 1 upsweep + 1 scatter per digit
        const uint64_t status_words = (uint64_t)npass * os_tiles * 256;
        static bool attr_set = false;
        if (!attr_set) {
            TDS_CUDA(cudaFuncSetAttribute(k_rs_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sizeof(OsSmem)));
            attr_set = true;
        }
        DBuf<uint32_t> aux(npass * 256 + npass + status_words, s);
        uint32_t *ghist = aux.p, *ctr = aux.p + npass * 256, *status = ctr + npass;
        TDS_CUDA(cudaMemsetAsync(aux.p, 0, 4 * (npass * 256 + npass + status_words), s));
        unsigned ublk = std::min<unsigned>(os_tiles, (unsigned)num_sms() * 4);
        k_rs_upsweep<<<ublk, RS_THREADS, 0, s>>>(keys, n, begin_bit, npass, end_bit, ghist);
        TDS_CHECK_LAUNCH();
        for (int p = 0; p < npass; ++p) {
            int shift = begin_bit + 8 * p;
            int nb = end_bit - shift < 8 ? end_bit - shift : 8;
            k_rs_onesweep<<<os_tiles, RS_THREADS, sizeof(OsSmem), s>>>(ka, va, kb, vb, n, shift, (1u << nb) - 1u,
                                                                        ghist + 256 * p,
                                                                        status + (uint64_t)p * os_tiles * 256, ctr + p);
            TDS_CHECK_LAUNCH();
            std::swap(ka, kb);
            std::swap(va, vb);
        }
    } else {
        DBuf<uint32_t> hist((uint64_t)256 * ntiles, s);
        for (int p = 0; p < npass; ++p) {
            int shift = begin_bit + 8 * p;
            int nb = end_bit - shift < 8 ? end_bit - shift : 8;
            uint32_t mask = (1u << nb) - 1u;
            k_rs_hist<<<ntiles, RS_THREADS, 0, s>>>(ka, n, shift, mask, hist.p, ntiles);
            TDS_CHECK_LAUNCH();
            exclusive_scan_u32(hist.p, hist.p, (uint64_t)256 * ntiles, nullptr, s);
            k_rs_scatter<<<ntiles, RS_THREADS, 0, s>>>(ka, va, kb, vb, n, shift, mask, hist.p, ntiles);
            TDS_CHECK_LAUNCH();
            std::swap(ka, kb);
            std::swap(va, vb);
        }
    }
    return (npass & 1) != 0;
}

void radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint64_t n, int begin_bit, int end_bit, cudaStream_t s) {
    if (n <= 1 || end_bit <= begin_bit) return;
    if (n >= (1ull << 32)) fail(TDS_EINVAL, "radix_sort_pairs: n too large");
    DBuf<uint32_t> k2(n, s), v2(n, s);
    if (radix_sort_passes(keys, vals, k2.p, v2.p, n, begin_bit, end_bit, s)) {
        TDS_CUDA(cudaMemcpyAsync(keys, k2.p, n * 4, cudaMemcpyDeviceToDevice, s));
        TDS_CUDA(cudaMemcpyAsync(vals, v2.p, n * 4, cudaMemcpyDeviceToDevice, s));
    }
}

// same, owning buffers: an odd pass count swaps the buffers instead of copying back
void radix_sort_pairs(DBuf<uint32_t> &keys, DBuf<uint32_t> &vals, uint64_t n, int begin_bit, int end_bit,
                      cudaStream_t s) {
    if (n <= 1 || end_bit <= begin_bit) return;
    if (n >= (1ull << 32)) fail(TDS_EINVAL, "radix_sort_pairs: n too large");
    DBuf<uint32_t> k2(keys.n, s), v2(vals.n, s);
    if (radix_sort_passes(keys.p, vals.p, k2.p, v2.p, n, begin_bit, end_bit, s)) {
        std::swap(keys.p, k2.p);
        std::swap(vals.p, v2.p);
        k2.s = keys.s; v2.s = vals.s;          // free the old buffers on their own streams
        keys.s = s; vals.s = s;
    }
}

}  // namespace tds
