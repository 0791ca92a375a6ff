// tds_internal.cuh — internal declarations of the B200 distance threshold
// search library (see include/tds.h for the C-ABI and DESIGN.md for the
// design).  Shared by the .cu translation units of the library only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <string>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/tds.h"

namespace tds {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Error {
    int code;
    std::string msg;
};
void set_error(int code, const char *fmt, ...);
const char *last_error();

#define TDS_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t _e = (call);                                                    \
        if (_e != cudaSuccess) {                                                    \
            if (_e == cudaErrorMemoryAllocation) {                                  \
                ::tds::set_error(TDS_ENOMEM, "%s:%d %s: %s", __FILE__, __LINE__,    \
                                 #call, cudaGetErrorString(_e));                    \
                throw ::tds::Error{TDS_ENOMEM, ""};                                 \
            }                                                                       \
            ::tds::set_error(TDS_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,  \
                             cudaGetErrorString(_e));                               \
            throw ::tds::Error{TDS_ECUDA, ""};                                      \
        }                                                                           \
    } while (0)

void count_launch();
#define TDS_CHECK_LAUNCH()                 \
    do {                                   \
        ::tds::count_launch();             \
        TDS_CUDA(cudaGetLastError());      \
    } while (0)

[[noreturn]] void fail(int code, const char *fmt, ...);

// ---------------------------------------------------------------------------
// stream-ordered device memory (cudaMallocAsync from the default pool)
// ---------------------------------------------------------------------------
void *dalloc(size_t bytes, cudaStream_t s);
void *dalloc_big(size_t bytes, cudaStream_t s);   // large result buffers (separate pool)
void *pinned_alloc(uint64_t bytes);                // pinned host blocks (cached)
void pinned_free(void *p);
void dfree(void *p, cudaStream_t s);

template <class T>
struct DBuf {                      // RAII device buffer, freed stream-ordered
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DBuf() = default;
    DBuf(size_t n_, cudaStream_t s_, bool big = false) : n(n_), s(s_) {
        p = (T *)(big ? dalloc_big((n_ ? n_ : 1) * sizeof(T), s_) : dalloc((n_ ? n_ : 1) * sizeof(T), s_));
    }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { reset(); p = o.p; n = o.n; s = o.s; o.p = nullptr; }
        return *this;
    }
    void reset() { if (p) dfree(p, s); p = nullptr; n = 0; }
    T *release() { T *q = p; p = nullptr; return q; }
    ~DBuf() { reset(); }
};

// ---------------------------------------------------------------------------
// the resident index (§4)
// ---------------------------------------------------------------------------
struct Extents {                   // export layout (tds_index_export what=11)
    float t_min, t_max;
    float lo[3], hi[3], maxext[3], w_st[3];
    float max_dur;                 // max (t_end - t_start) over D, rounded up
    float pad;
};

}  // namespace tds

struct tds_index_s {
    uint64_t n = 0;
    uint32_t kinds = 0;
    int m = 0, v = 0;
    int grid[3] = {0, 0, 0};
    tds::Extents ext{};
    float w_fsg[3] = {0, 0, 0};
    // temporal: sorted records, renumbering, bins
    float4 *rec = nullptr;          // [2n] sorted by t_start: (x0,y0,z0,t0),(x1,y1,z1,t1)
    uint32_t *perm = nullptr;       // [n]  sorted position -> original row
    uint32_t *bin_off = nullptr;    // [m+1]
    float *bin_lo = nullptr;        // [m]  first member t_start (suffix-filled over empty bins)
    float *bin_hi = nullptr;        // [m]  max member t_end (-inf if empty)
    float *bin_pmhi = nullptr;      // [m]  prefix max of bin_hi
    // spatiotemporal
    uint32_t *st_arr[3] = {nullptr, nullptr, nullptr};   // X, Y, Z (sorted positions)
    uint64_t st_len[3] = {0, 0, 0};
    uint32_t *st_off[3] = {nullptr, nullptr, nullptr};   // [v*m+1], subbin (slab j, bin i) at j*m+i
    float4 *st_rec[3] = {nullptr, nullptr, nullptr};     // [2*len] records in X/Y/Z order (ablation; null by default)
    // FSG as a dense CSR over all cells + lookup array A
    uint32_t *cell_off = nullptr;   // [gx*gy*gz+1]
    uint32_t *fsg_A = nullptr;      // [A_len] sorted positions
    uint32_t *fsg_ecell = nullptr;  // [A_len] min cell of entry A[i]'s MBB, packed x<<21 | y<<10 | z
    float4 *fsg_rec = nullptr;      // [2 A_len] record of entry A[i] (cell-ordered copy, coalesced streaming)
    uint32_t *fsg_perm = nullptr;   // [A_len] original row of entry A[i]
    uint64_t A_len = 0;
    uint64_t n_cells = 0;
    int device = 0;
    uint64_t mem_budget = 0;        // device bytes available for result buffers (at build)
    bool time_order = false;        // entries renumbered by t_start (else by (bin, Morton))
    // window boxes (DESIGN.md §7 "Window boxes"): per aligned window of WBOX_W
    // consecutive candidate positions, (min x, min y, min z, min t0), (max x,
    // max y, max z, max t1) of the segments there; the range kernel tests a
    // group's query boxes against it before loading the window
    float4 *wb_rec = nullptr;                            // [2 ceil(n / WBOX_W)] over rec
    float4 *wb_st[3] = {nullptr, nullptr, nullptr};      // over rec[X[i]], rec[Y[i]], rec[Z[i]]
    float4 *wb_fsg = nullptr;                            // over the cell-ordered copy fsg_rec
};

namespace tds {

// ---------------------------------------------------------------------------
// device helpers shared by build and search
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint32_t float_key(float f) {
    // order-preserving map float -> uint32 (finite values)
    uint32_t u;
#ifdef __CUDA_ARCH__
    u = __float_as_uint(f);
#else
    memcpy(&u, &f, 4);
#endif
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

constexpr uint32_t WBOX_W = 128;    // window-box granularity = the range kernel's window

// slab / cell of coordinate c: clamp(floor((c - o) / w), 0, g - 1) in fp32 RN.
// The SAME expression is used for entries (build) and queries (search): it is
// monotone non-decreasing in c, which is what completeness relies on
// (DESIGN.md "Completeness under rounding").
__device__ __forceinline__ int cell_of(float c, float o, float w, int g) {
    float f = floorf(__fdiv_rn(__fsub_rn(c, o), w));
    int k = (f < 0.f) ? 0 : (f >= (float)g ? g - 1 : (int)f);
    return k;
}

// FSG cell coordinates packed in 32 bits (grid limits 2048 x 2048 x 1024)
constexpr int FSG_MAX_X = 2048, FSG_MAX_Y = 2048, FSG_MAX_Z = 1024;
__host__ __device__ __forceinline__ uint32_t pack_cell(int x, int y, int z) {
    return ((uint32_t)x << 21) | ((uint32_t)y << 10) | (uint32_t)z;
}

// ---------------------------------------------------------------------------
// radix sort / scan primitives (sort.cu)
// ---------------------------------------------------------------------------
// Stable LSD radix sort of (key, value) pairs on bits [begin_bit, end_bit).
// keys/vals are sorted in place (double-buffered with caller-free temporaries).
bool st_indirect();                 // no materialised X/Y/Z records unless TDS_ST_MATERIALISE=1 (ablation)
void radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint64_t n, int begin_bit, int end_bit,
                      cudaStream_t s);
void radix_sort_pairs(DBuf<uint32_t> &keys, DBuf<uint32_t> &vals, uint64_t n, int begin_bit, int end_bit,
                      cudaStream_t s);
// Exclusive scan of n uint32 values into out (out may alias in); optional
// total written to *d_total (device pointer, may be null).  64-bit variant too.
// k (<= 4) independent exclusive scans of n uint32 in one launch (totals optional)
void exclusive_scan_u32_batch(int k, const uint32_t *const *in, uint32_t *const *out, uint32_t *const *d_total,
                              uint64_t n, cudaStream_t s);
void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, uint32_t *d_total,
                        cudaStream_t s);
void exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *d_total,
                        cudaStream_t s);

// ---------------------------------------------------------------------------
// build (build.cu) / search (search.cu)
// ---------------------------------------------------------------------------
void build_index(const tds_seg *entries, uint64_t n, const tds_index_params *p, cudaStream_t s,
                 tds_index_s *idx);
void free_index(tds_index_s *idx);

// validate n segments: returns first bad row or UINT64_MAX (synchronises)
uint64_t validate_segments(const float4 *rec, uint64_t n, cudaStream_t s);

int num_sms();

// opt-in phase trace (env TDS_TRACE=1): CUDA events on a stream, printed to stderr
struct Trace {
    bool on = false;
    cudaStream_t s = 0;
    std::vector<std::pair<const char *, cudaEvent_t>> ev;
    std::vector<double> host_ms;       // host wall clock at each mark
    explicit Trace(cudaStream_t s_);
    void mark(const char *name);
    std::string notes;                 // extra key=value pairs printed with the trace
    void note(const char *key, double v) {
        if (!on) return;
        char b[64];
        snprintf(b, sizeof b, " %s=%.3f", key, v);
        notes += b;
    }
    ~Trace();
};
// free device memory + memory reserved but unused in the default mempool (bytes)
uint64_t device_budget_bytes();        // snapshot minus pool use since (cheap)
void device_budget_refresh();          // new snapshot (cudaMemGetInfo), after ENOMEM
std::mutex &big_alloc_mutex();

// ---------------------------------------------------------------------------
// result records (16 B): (query row, entry row, t_in, t_out)
// ---------------------------------------------------------------------------
struct Rec {
    uint32_t qid, eid;
    float t_in, t_out;
};

}  // namespace tds

struct tds_result_s {
    // chunked form (pass 1 without overflow): records live in buf, in chunks of
    // CS slots; chunk k holds chunk_used[k] records starting at slot k*CS.
    tds::Rec *buf = nullptr;
    uint64_t cap = 0;
    uint32_t CS = 0;
    uint64_t nchunks = 0;
    uint32_t *chunk_used = nullptr;
    uint64_t *chunk_off = nullptr;    // exclusive prefix of chunk_used
    // contiguous form (after overflow handling): store[0..n)
    tds::Rec *store = nullptr;
    bool chunked = true;
    uint64_t n = 0;
    tds_stats stats{};
    int device = 0;
    cudaStream_t stream = 0;          // stream of the last operation (frees are ordered after it)
    uint64_t nq = 0, ne = 0;          // query / entry counts of the search (trajectory merge checks)
    // host-resident form (tds_search_stream): records in pinned host blocks
    std::vector<std::pair<tds::Rec *, uint64_t>> host_blocks;
    bool host = false;
};

namespace tds {
struct SearchOpts {
    uint32_t part = 0, nparts = 1;            // tds_search_part: this part of a work-balanced split
    int32_t *plan_sel = nullptr;              // tds_plan: host outputs per query row (range variants);
    uint32_t *plan_lo = nullptr, *plan_hi = nullptr;   // set -> schedule only, no pair kernel
};
// tds_search_stream: host queries in chunks, records to pinned host memory (search.cu)
void search_stream(tds_index_s *idx, int kind, const float4 *q_host, uint64_t nq, double d, float T0, float T1,
                   uint64_t chunk, cudaStream_t s, tds_result_s *res, const SearchOpts &opt);
void search(tds_index_s *idx, int kind, const float4 *q, uint64_t nq, double d, float T0, float T1,
            uint64_t capacity, cudaStream_t s, tds_result_s *res, const SearchOpts &opt = SearchOpts());
void fetch(tds_result_s *r, uint64_t first, uint64_t count, uint32_t *qid, uint32_t *eid, float *tin,
           float *tout, bool dst_dev, bool sorted, cudaStream_t s);
void free_result(tds_result_s *r);
// rows of D owned by part `part` of `nparts` (partition.cu); rows: device, >= n / nparts + 1
uint64_t time_partition(const float *t_start, uint64_t n, uint32_t part, uint32_t nparts, uint32_t *rows,
                        cudaStream_t s);
void merge_trajectories(tds_result_s *r, const uint32_t *q_traj, uint64_t nq, const uint32_t *e_traj, uint64_t ne,
                        float gap, cudaStream_t s, tds_result_s *out);
}  // namespace tds
