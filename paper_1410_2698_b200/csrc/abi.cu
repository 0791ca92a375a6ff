// abi.cu — the extern "C" boundary declared in include/tds.h: argument
// checking, host/device input detection, error reporting, handle lifetime.
#include <map>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <new>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3 (CUDA toolkit): ranges for profilers
#include "tds_internal.cuh"

// NVTX range over one C-ABI call (visible in nsys / ncu timelines; a few ns
// when no tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

namespace tds {

static thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    (void)code;
    g_err = buf;
}

const char *last_error() { return g_err.c_str(); }

void fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    throw Error{code, buf};
}

// Two private stream-ordered pools per device (the device's default pool and its
// attributes are left alone: other libraries in the process may use it):
//  * the small pool for temporaries (schedules, scans, work lists: up to several
//    GB for large GPUSpatial searches);
//  * the big pool for result buffers, so that their tens-of-GB blocks are reused by
//    later searches instead of being split by small temporaries.
// Both keep freed memory mapped (re-mapping GBs per search measured tens of ms:
// Merger-shaped GPUSpatial 22 -> 72 ms per search with a 4 GB keep limit) until
// tds_trim() releases it; the result-buffer budget counts that memory as free.
constexpr int MAX_DEV = 64;
constexpr uint64_t SMALL_KEEP = UINT64_MAX;

static cudaMemPool_t make_pool(int dev, uint64_t keep) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    return pool;
}

static cudaMemPool_t device_pool(int which) {   // 0 small, 1 big
    static cudaMemPool_t pools[2][MAX_DEV] = {};
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= MAX_DEV) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[which][dev]) pools[which][dev] = make_pool(dev, which ? UINT64_MAX : SMALL_KEEP);
    return pools[which][dev];
}

static cudaMemPool_t small_pool() { return device_pool(0); }
static cudaMemPool_t big_pool() { return device_pool(1); }

void *dalloc(size_t bytes, cudaStream_t s) {
    void *p = nullptr;
    cudaMemPool_t pool = small_pool();
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&p, bytes, pool, s) : cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? TDS_ENOMEM : TDS_ECUDA, "cudaMallocAsync(%zu bytes): %s", bytes,
             cudaGetErrorString(e));
    }
    return p;
}

void dfree(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// Pinned host blocks for host-resident results (tds_search_stream): pinning
// GBs of host memory costs ~0.1-0.3 s per GB, so freed blocks are cached (up to
// PINNED_KEEP bytes) and reused by later results of the same or smaller size.
constexpr uint64_t PINNED_KEEP = 64ull << 30;
std::map<void *, uint64_t> &g_pin_size();
static std::mutex g_pin_mu;
static std::multimap<uint64_t, void *> g_pin_cache;
static uint64_t g_pin_bytes = 0;

void *pinned_alloc(uint64_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_cache.lower_bound(bytes);
        if (it != g_pin_cache.end() && it->first <= 2 * bytes + (64ull << 20)) {
            void *p = it->second;
            g_pin_bytes -= it->first;
            g_pin_cache.erase(it);
            return p;
        }
    }
    const uint64_t sz = std::max<uint64_t>(bytes, 1) + (bytes >> 3);     // room to be reused by larger results
    void *p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, sz, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(TDS_ENOMEM, "cudaHostAlloc(%llu bytes): %s", (unsigned long long)sz, cudaGetErrorString(e));
    }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_size()[p] = sz;
    return p;
}

std::map<void *, uint64_t> &g_pin_size() {
    static std::map<void *, uint64_t> m;
    return m;
}

void pinned_free(void *p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    const uint64_t sz = g_pin_size()[p];
    if (g_pin_bytes + sz <= PINNED_KEEP) {
        g_pin_cache.emplace(sz, p);
        g_pin_bytes += sz;
    } else {
        g_pin_size().erase(p);
        cudaFreeHost(p);
    }
}

// release the memory both pools of the current device hold unused, and the cached
// pinned host blocks (tds_trim)
void trim_pools() {
    cudaDeviceSynchronize();          // stream-ordered frees must have happened
    for (int w = 0; w < 2; ++w)
        if (cudaMemPool_t pool = device_pool(w)) cudaMemPoolTrimTo(pool, 0);
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (auto &kv : g_pin_cache) {
        g_pin_size().erase(kv.second);
        cudaFreeHost(kv.second);
    }
    g_pin_cache.clear();
    g_pin_bytes = 0;
}

void *dalloc_big(size_t bytes, cudaStream_t s);

static uint64_t device_budget_bytes_now();

// Memory budget for result buffers.  cudaMemGetInfo is slow (measured 2-80 ms per
// call on B200 between large searches), so it is called once per device (and
// again after an allocation failure): the budget is that snapshot (free memory +
// memory the two pools held unused) minus what the pools hand out since, read
// from their cheap used-memory counters.  Concurrent searches therefore see each
// other's buffers; allocations by other libraries after the snapshot are not
// tracked (the 0.45 factor and the halving retry on ENOMEM cover them).
static uint64_t pools_used_bytes(int dev) {
    (void)dev;
    cudaMemPool_t pools[2] = {small_pool(), big_pool()};
    uint64_t tot = 0;
    for (cudaMemPool_t pool : pools) {
        uint64_t used = 0;
        if (pool && cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess) tot += used;
    }
    return tot;
}

static std::mutex g_budget_mu;
static int g_budget_dev = -1;
static uint64_t g_budget_avail0 = 0, g_budget_used0 = 0;

static void budget_snapshot_locked(int dev) {
    g_budget_avail0 = device_budget_bytes_now();
    g_budget_used0 = pools_used_bytes(dev);
    g_budget_dev = dev;
}

void device_budget_refresh() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_budget_mu);
    budget_snapshot_locked(dev);
}

uint64_t device_budget_bytes() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_budget_mu);
    if (dev != g_budget_dev || g_budget_avail0 == 0) budget_snapshot_locked(dev);
    const uint64_t cap = g_budget_avail0 + g_budget_used0, used = pools_used_bytes(dev);
    return used < cap ? cap - used : 0;
}

// the lock under which searches size and allocate result buffers above 1 GB
// (concurrent searches then see each other's allocations in the pool counters)
std::mutex &big_alloc_mutex() {
    static std::mutex m;
    return m;
}

static uint64_t device_budget_bytes_now() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    uint64_t extra = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    (void)dev;
    cudaMemPool_t pools[2] = {small_pool(), big_pool()};
    for (cudaMemPool_t pool : pools) {
        if (!pool) continue;
        uint64_t reserved = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
            extra += reserved - used;
    }
    return (uint64_t)fr + extra;
}

// Fault injection for tests (tds_test_inject_enomem): the next k large
// allocations fail with TDS_ENOMEM; g_injected counts the failures injected.
static std::atomic<int> g_inject_left{0}, g_inject_skip{0};
static std::atomic<uint64_t> g_injected{0};

static bool inject_enomem() {
    if (g_inject_left.load(std::memory_order_relaxed) <= 0) return false;
    if (g_inject_skip.load() > 0 && g_inject_skip.fetch_sub(1) > 0) return false;   // let `skip` through first
    if (g_inject_left.fetch_sub(1) <= 0) return false;
    g_injected.fetch_add(1);
    return true;
}

void *dalloc_big(size_t bytes, cudaStream_t s) {
    if (inject_enomem()) fail(TDS_ENOMEM, "injected allocation failure (tds_test_inject_enomem), %zu bytes", bytes);
    cudaMemPool_t pool = big_pool();
    if (!pool) return dalloc(bytes, s);
    void *p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? TDS_ENOMEM : TDS_ECUDA, "cudaMallocFromPoolAsync(%zu bytes): %s", bytes,
             cudaGetErrorString(e));
    }
    return p;
}

Trace::Trace(cudaStream_t s_) : s(s_) {
    const char *e = getenv("TDS_TRACE");
    on = e && e[0] == '1';
    if (on) mark("start");
}

void Trace::mark(const char *name) {
    nvtxMarkA(name);                   // phase ends as NVTX markers (always)
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
    host_ms.push_back(std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now().time_since_epoch()).count());
}

Trace::~Trace() {
    if (!on) return;
    cudaEventSynchronize(ev.back().second);
    std::string line = "[tds trace]";
    for (size_t i = 1; i < ev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
        char b[96];
        snprintf(b, sizeof b, " %s %.3f (host %.3f)", ev[i].first, ms, host_ms[i] - host_ms[i - 1]);
        line += b;
    }
    line += notes;
    {   // pool reservations (GB): default pool, result pool
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pools[2] = {nullptr, big_pool()};
        cudaDeviceGetDefaultMemPool(&pools[0], dev);
        for (cudaMemPool_t pool : pools) {
            uint64_t reserved = 0, used = 0;
            if (pool) {
                cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
                cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
            }
            char b[64];
            snprintf(b, sizeof b, " | pool %.2f/%.2f GB", used / 1e9, reserved / 1e9);
            line += b;
        }
    }
    fprintf(stderr, "%s\n", line.c_str());
    for (auto &x : ev) cudaEventDestroy(x.second);
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// device copy of a caller buffer that may live in host memory
struct Staged {
    const float4 *p = nullptr;
    DBuf<float4> own;
};

static void stage(const tds_seg *src, uint64_t n, cudaStream_t s, Staged &out) {
    if (!src) fail(TDS_EINVAL, "NULL segment pointer");
    if (((uintptr_t)src & 15) != 0) fail(TDS_EINVAL, "segment array must be 16-byte aligned");
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, src);
    if (e != cudaSuccess) cudaGetLastError();
    bool dev = (e == cudaSuccess) && (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    if (dev) {
        out.p = reinterpret_cast<const float4 *>(src);
        return;
    }
    out.own = DBuf<float4>(2 * n, s);
    TDS_CUDA(cudaMemcpyAsync(out.own.p, src, n * sizeof(tds_seg), cudaMemcpyHostToDevice, s));
    out.p = out.own.p;
}

// device copy of a uint32 array that may live in host memory
struct StagedU32 {
    const uint32_t *p = nullptr;
    DBuf<uint32_t> own;
};

static void stage_u32(const uint32_t *src, uint64_t n, cudaStream_t s, StagedU32 &out) {
    if (!src) fail(TDS_EINVAL, "NULL id array");
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, src);
    if (e != cudaSuccess) cudaGetLastError();
    bool dev = (e == cudaSuccess) && (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    if (dev) {
        out.p = src;
        return;
    }
    out.own = DBuf<uint32_t>(n, s);
    TDS_CUDA(cudaMemcpyAsync(out.own.p, src, n * 4, cudaMemcpyHostToDevice, s));
    out.p = out.own.p;
}

}  // namespace tds

using namespace tds;

#define ABI_TRY try {
#define ABI_CATCH                                                   \
    }                                                               \
    catch (const tds::Error &err) {                                 \
        return err.code;                                            \
    }                                                               \
    catch (const std::bad_alloc &) {                                \
        tds::set_error(TDS_ENOMEM, "host allocation failed");       \
        return TDS_ENOMEM;                                          \
    }                                                               \
    catch (...) {                                                   \
        tds::set_error(TDS_ECUDA, "unexpected exception");          \
        return TDS_ECUDA;                                           \
    }

extern "C" {

const char *tds_last_error(void) { return tds::last_error(); }

const char *tds_version(void) { return "tds-b200 0.1 (sm_100a)"; }

uint64_t tds_kernel_launches(void) { return tds::g_launches.load(); }

void tds_trim(void) { tds::trim_pools(); }

uint64_t tds_test_inject_enomem(int k, int skip) {
    if (k >= 0) {
        tds::g_inject_skip.store(skip > 0 ? skip : 0);
        tds::g_inject_left.store(k);
    }
    return tds::g_injected.load();
}

int tds_build_index(const tds_seg *entries, uint64_t n, const tds_index_params *params, void *stream,
                    tds_index *out) {
    NvtxRange nvtx_range("tds_build_index");
    ABI_TRY
    tds::set_error(0, "");
    if (!out || !params) fail(TDS_EINVAL, "NULL argument");
    *out = nullptr;
    if (n == 0) fail(TDS_EINVAL, "n == 0");
    if (n >= (1ull << 32) - 1) fail(TDS_EINVAL, "n = %llu exceeds 2^32 - 2", (unsigned long long)n);
    if (params->m_bins < 1) fail(TDS_EINVAL, "m_bins = %d < 1", params->m_bins);
    if ((params->kinds & TDS_SPATIOTEMPORAL) && params->v_subbins < 1)
        fail(TDS_EINVAL, "v_subbins = %d < 1", params->v_subbins);
    if ((params->kinds & TDS_SPATIAL))
        for (int c = 0; c < 3; ++c)
            if (params->grid[c] < 1) fail(TDS_EINVAL, "grid[%d] = %d < 1", c, params->grid[c]);
    if (params->kinds & ~(uint32_t)TDS_ALL) fail(TDS_EINVAL, "unknown kinds bits 0x%x", params->kinds);
    if ((uint64_t)params->m_bins * (uint64_t)std::max(params->v_subbins, 1) >= (1ull << 31))
        fail(TDS_EINVAL, "m * v too large");
    cudaStream_t s = (cudaStream_t)stream;
    Staged in;
    stage(entries, n, s, in);
    tds_index_s *idx = new tds_index_s();
    cudaGetDevice(&idx->device);
    try {
        build_index(reinterpret_cast<const tds_seg *>(in.p), n, params, s, idx);
    } catch (...) {
        free_index(idx);
        delete idx;
        throw;
    }
    *out = idx;
    return TDS_OK;
    ABI_CATCH
}

}  // extern "C"

namespace {

// argument checks shared by tds_search / tds_search_part / tds_plan
void check_search_args(tds_index idx, int kind, double d, float t_start, float t_end) {
    if (!idx) fail(TDS_EINVAL, "NULL argument");
    if (kind != TDS_TEMPORAL && kind != TDS_SPATIAL && kind != TDS_SPATIOTEMPORAL && kind != TDS_AUTO)
        fail(TDS_EINVAL, "kind = %d is not one of TDS_TEMPORAL/SPATIAL/SPATIOTEMPORAL/AUTO", kind);
    if (kind != TDS_AUTO && !(idx->kinds & (uint32_t)kind))
        fail(TDS_EINVAL, "index was not built for kind %d", kind);
    if (!(d > 0.0) || !isfinite(d) || d > 3.0e38) fail(TDS_EINVAL, "d = %g must be finite and > 0", d);
    if (isnan(t_start) || isnan(t_end) || t_start > t_end) fail(TDS_EINVAL, "bad window [%g, %g]",
                                                               (double)t_start, (double)t_end);
}

void run_search(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start, float t_end,
                uint64_t capacity, void *stream, tds_result *out, uint64_t *n_results, const tds::SearchOpts &opt) {
    if (!out) fail(TDS_EINVAL, "NULL argument");
    *out = nullptr;
    check_search_args(idx, kind, d, t_start, t_end);
    cudaStream_t s = (cudaStream_t)stream;
    tds_result_s *r = new tds_result_s();
    cudaGetDevice(&r->device);
    try {
        if (nq > 0) {
            Staged in;
            stage(queries, nq, s, in);
            tds::search(idx, kind, in.p, nq, d, t_start, t_end, capacity, s, r, opt);
        }
    } catch (...) {
        free_result(r);
        delete r;
        throw;
    }
    *out = r;
    if (n_results) *n_results = r->n;
}

}  // namespace

extern "C" {

int tds_search(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start, float t_end,
               uint64_t capacity, void *stream, tds_result *out, uint64_t *n_results) {
    NvtxRange nvtx_range("tds_search");
    ABI_TRY
    tds::set_error(0, "");
    run_search(idx, kind, queries, nq, d, t_start, t_end, capacity, stream, out, n_results, tds::SearchOpts());
    return TDS_OK;
    ABI_CATCH
}

int tds_search_part(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start,
                    float t_end, uint64_t capacity, uint32_t part, uint32_t nparts, void *stream, tds_result *out,
                    uint64_t *n_results) {
    NvtxRange nvtx_range("tds_search_part");
    ABI_TRY
    tds::set_error(0, "");
    if (nparts < 1 || part >= nparts) fail(TDS_EINVAL, "part %u of %u", part, nparts);
    tds::SearchOpts opt;
    opt.part = part;
    opt.nparts = nparts;
    run_search(idx, kind, queries, nq, d, t_start, t_end, capacity, stream, out, n_results, opt);
    return TDS_OK;
    ABI_CATCH
}

int tds_time_partition(const float *t_start, uint64_t n, uint32_t part, uint32_t nparts, void *stream,
                       uint32_t *rows, uint64_t *n_rows) {
    NvtxRange nvtx_range("tds_time_partition");
    ABI_TRY
    tds::set_error(0, "");
    if (!t_start || !rows || !n_rows) fail(TDS_EINVAL, "NULL argument");
    if (n == 0 || n >= (1ull << 32) - 1) fail(TDS_EINVAL, "n = %llu", (unsigned long long)n);
    if (nparts < 1 || part >= nparts) fail(TDS_EINVAL, "part %u of %u", part, nparts);
    cudaStream_t s = (cudaStream_t)stream;
    StagedU32 in;
    stage_u32(reinterpret_cast<const uint32_t *>(t_start), n, s, in);
    *n_rows = tds::time_partition(reinterpret_cast<const float *>(in.p), n, part, nparts, rows, s);
    return TDS_OK;
    ABI_CATCH
}

int tds_search_stream(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start,
                      float t_end, uint64_t chunk, uint32_t part, uint32_t nparts, void *stream, tds_result *out,
                      uint64_t *n_results) {
    NvtxRange nvtx_range("tds_search_stream");
    ABI_TRY
    tds::set_error(0, "");
    if (!out) fail(TDS_EINVAL, "NULL argument");
    *out = nullptr;
    check_search_args(idx, kind, d, t_start, t_end);
    if (nq > 0 && !queries) fail(TDS_EINVAL, "NULL query pointer");
    if (((uintptr_t)queries & 15) != 0) fail(TDS_EINVAL, "segment array must be 16-byte aligned");
    if (chunk == 0) fail(TDS_EINVAL, "chunk == 0");
    if (nparts < 1 || part >= nparts) fail(TDS_EINVAL, "part %u of %u", part, nparts);
    cudaPointerAttributes at{};
    if (nq > 0 && cudaPointerGetAttributes(&at, queries) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
        fail(TDS_EINVAL, "tds_search_stream takes queries in host memory (use tds_search for device queries)");
    cudaGetLastError();
    tds_result_s *r = new tds_result_s();
    cudaGetDevice(&r->device);
    try {
        tds::SearchOpts opt;
        opt.part = part;
        opt.nparts = nparts;
        tds::search_stream(idx, kind, reinterpret_cast<const float4 *>(queries), nq, d, t_start, t_end, chunk,
                           (cudaStream_t)stream, r, opt);
    } catch (...) {
        free_result(r);
        delete r;
        throw;
    }
    *out = r;
    if (n_results) *n_results = r->n;
    return TDS_OK;
    ABI_CATCH
}

int tds_plan(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start, float t_end,
             void *stream, int32_t *sel, uint32_t *lo, uint32_t *hi) {
    NvtxRange nvtx_range("tds_plan");
    ABI_TRY
    tds::set_error(0, "");
    check_search_args(idx, kind, d, t_start, t_end);
    if (kind == TDS_SPATIAL || kind == TDS_AUTO) fail(TDS_EINVAL, "tds_plan: kind must be TDS_TEMPORAL or TDS_SPATIOTEMPORAL");
    if (nq > 0 && (!sel || !lo || !hi)) fail(TDS_EINVAL, "NULL argument");
    if (nq == 0) return TDS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    tds_result_s r;
    cudaGetDevice(&r.device);
    tds::SearchOpts opt;
    opt.plan_sel = sel;
    opt.plan_lo = lo;
    opt.plan_hi = hi;
    Staged in;
    stage(queries, nq, s, in);
    tds::search(idx, kind, in.p, nq, d, t_start, t_end, 0, s, &r, opt);
    return TDS_OK;
    ABI_CATCH
}

}  // extern "C"

namespace {

// persistent worker threads for tds_search_many (detached; they wait on a queue)
class SearchPool {
  public:
    void run(std::vector<std::function<void()>> &tasks) {
        if (tasks.empty()) return;
        std::mutex m;
        std::condition_variable cv;
        size_t left = tasks.size() - 1;
        {
            std::lock_guard<std::mutex> lk(mu_);
            while (idle_ < (int)left) {
                std::thread(&SearchPool::loop, this).detach();
                ++idle_;
            }
            idle_ -= (int)left;
            for (size_t i = 1; i < tasks.size(); ++i)
                q_.push_back([&, i] {
                    tasks[i]();
                    std::lock_guard<std::mutex> l2(m);
                    if (--left == 0) cv.notify_one();
                });
        }
        cv_.notify_all();
        tasks[0]();                           // the caller drives the first request
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return left == 0; });
    }

  private:
    void loop() {
        for (;;) {
            std::function<void()> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return !q_.empty(); });
                f = std::move(q_.front());
                q_.pop_front();
            }
            f();
            std::lock_guard<std::mutex> lk(mu_);
            ++idle_;
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    int idle_ = 0;
};

SearchPool &search_pool() {
    static SearchPool *p = new SearchPool();  // never destroyed: workers are detached
    return *p;
}

}  // namespace

extern "C" {

int tds_search_many(tds_index idx, int n, const tds_search_req *reqs, tds_result *out, uint64_t *n_results) {
    NvtxRange nvtx_range("tds_search_many");
    ABI_TRY
    tds::set_error(0, "");
    if (n < 0 || (n > 0 && (!reqs || !out))) fail(TDS_EINVAL, "bad request list");
    for (int i = 0; i < n; ++i) out[i] = nullptr;
    if (n == 0) return TDS_OK;
    // requests sharing a stream form one serial lane (request order kept)
    std::vector<std::vector<int>> lanes;
    for (int i = 0; i < n; ++i) {
        size_t k = 0;
        while (k < lanes.size() && reqs[lanes[k][0]].stream != reqs[i].stream) ++k;
        if (k == lanes.size()) lanes.emplace_back();
        lanes[k].push_back(i);
    }
    std::vector<int> code(n, TDS_OK);
    std::vector<std::string> msg(n);
    int dev = 0;
    cudaGetDevice(&dev);
    std::vector<std::function<void()>> tasks;
    for (auto &lane : lanes)
        tasks.push_back([&, lane] {
            cudaSetDevice(dev);
            for (int i : lane) {
                const tds_search_req &r = reqs[i];
                code[i] = tds_search(idx, r.kind, r.queries, r.nq, r.d, r.t_start, r.t_end, r.capacity, r.stream,
                                     &out[i], n_results ? &n_results[i] : nullptr);
                if (code[i] != TDS_OK) {
                    msg[i] = tds_last_error();
                    break;
                }
            }
        });
    search_pool().run(tasks);
    for (int i = 0; i < n; ++i)
        if (code[i] != TDS_OK) {
            for (int j = 0; j < n; ++j)
                if (out[j]) { tds_result_free(out[j]); out[j] = nullptr; }
            tds::set_error(code[i], "%s", msg[i].c_str());
            return code[i];
        }
    return TDS_OK;
    ABI_CATCH
}

int tds_fetch_results(tds_result r, uint64_t first, uint64_t count, uint32_t *query_id, uint32_t *entry_id,
                      float *t_in, float *t_out, int dst_is_device, int sorted, void *stream) {
    NvtxRange nvtx_range("tds_fetch_results");
    ABI_TRY
    tds::set_error(0, "");
    if (!r) fail(TDS_EINVAL, "NULL result");
    tds::fetch(r, first, count, query_id, entry_id, t_in, t_out, dst_is_device != 0, sorted != 0,
               (cudaStream_t)stream);
    return TDS_OK;
    ABI_CATCH
}

int tds_merge_trajectories(tds_result r, const uint32_t *q_traj, uint64_t nq, const uint32_t *e_traj, uint64_t ne,
                           float gap, void *stream, tds_result *out, uint64_t *n_out) {
    NvtxRange nvtx_range("tds_merge_trajectories");
    ABI_TRY
    tds::set_error(0, "");
    if (!r || !out) fail(TDS_EINVAL, "NULL argument");
    *out = nullptr;
    if (nq != r->nq) fail(TDS_EINVAL, "q_traj has %llu ids, the search had %llu queries", (unsigned long long)nq,
                          (unsigned long long)r->nq);
    if (ne != r->ne) fail(TDS_EINVAL, "e_traj has %llu ids, the index has %llu entries", (unsigned long long)ne,
                          (unsigned long long)r->ne);
    if (!(gap >= 0.f) || !isfinite(gap)) fail(TDS_EINVAL, "gap = %g must be finite and >= 0", (double)gap);
    if (r->host) fail(TDS_EINVAL, "the result of tds_search_stream is host-resident: fetch it and merge on the host");
    cudaStream_t s = (cudaStream_t)stream;
    tds_result_s *m = new tds_result_s();
    cudaGetDevice(&m->device);
    try {
        if (r->n > 0) {
            StagedU32 qt, et;
            stage_u32(q_traj, nq, s, qt);
            stage_u32(e_traj, ne, s, et);
            tds::merge_trajectories(r, qt.p, nq, et.p, ne, gap, s, m);
        }
    } catch (...) {
        free_result(m);
        delete m;
        throw;
    }
    m->nq = r->nq;
    m->ne = r->ne;
    *out = m;
    if (n_out) *n_out = m->n;
    return TDS_OK;
    ABI_CATCH
}

int tds_result_stats(tds_result r, tds_stats *out) {
    if (!r || !out) {
        tds::set_error(TDS_EINVAL, "NULL argument");
        return TDS_EINVAL;
    }
    *out = r->stats;
    return TDS_OK;
}

uint64_t tds_result_count(tds_result r) { return r ? r->n : 0; }

int tds_result_host_block(tds_result r, uint64_t i, const void **records, uint64_t *count) {
    ABI_TRY
    tds::set_error(0, "");
    if (!r || !records || !count) fail(TDS_EINVAL, "NULL argument");
    if (!r->host) fail(TDS_EINVAL, "not a host-resident result (tds_search_stream)");
    if (i >= r->host_blocks.size()) {
        *records = nullptr;
        *count = 0;
        return TDS_OK;
    }
    *records = r->host_blocks[i].first;
    *count = r->host_blocks[i].second;
    return TDS_OK;
    ABI_CATCH
}

void tds_result_free(tds_result r) {
    if (!r) return;
    free_result(r);
    delete r;
}

void tds_index_free(tds_index idx) {
    if (!idx) return;
    free_index(idx);
    delete idx;
}

int tds_index_info(tds_index idx, uint64_t *n, int32_t *m, int32_t *v, int32_t *grid3, uint32_t *kinds) {
    if (!idx) {
        tds::set_error(TDS_EINVAL, "NULL index");
        return TDS_EINVAL;
    }
    if (n) *n = idx->n;
    if (m) *m = idx->m;
    if (v) *v = idx->v;
    if (grid3) for (int c = 0; c < 3; ++c) grid3[c] = idx->grid[c];
    if (kinds) *kinds = idx->kinds;
    return TDS_OK;
}

int tds_index_export(tds_index idx, int what, void *dst, uint64_t cap_bytes, uint64_t *n_bytes) {
    ABI_TRY
    if (!idx) fail(TDS_EINVAL, "NULL index");
    const void *src = nullptr;
    uint64_t bytes = 0;
    bool host = false;
    std::vector<float> tmp;
    switch (what) {
        case 0: src = idx->perm; bytes = 4 * idx->n; break;
        case 1: src = idx->bin_off; bytes = 4ull * (idx->m + 1); break;
        case 2: src = idx->bin_hi; bytes = 4ull * idx->m; break;
        case 3: case 4: case 5:
            src = idx->st_arr[what - 3]; bytes = 4 * idx->st_len[what - 3]; break;
        case 6: case 7: case 8:
            src = idx->st_off[what - 6];
            bytes = idx->st_off[what - 6] ? 4ull * ((uint64_t)idx->v * idx->m + 1) : 0; break;
        case 9: src = idx->cell_off; bytes = idx->cell_off ? 4 * (idx->n_cells + 1) : 0; break;
        case 10: src = idx->fsg_A; bytes = 4 * idx->A_len; break;
        case 11: src = &idx->ext; bytes = sizeof(tds::Extents); host = true; break;
        case 12: {
            tmp.resize(idx->n);
            std::vector<float4> r(2 * idx->n);
            TDS_CUDA(cudaMemcpy(r.data(), idx->rec, 32 * idx->n, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < idx->n; ++i) tmp[i] = r[2 * i].w;
            src = tmp.data(); bytes = 4 * idx->n; host = true; break;
        }
        case 13: case 14: case 15: case 16: case 17: {   // window boxes
            const float4 *wb = what == 13 ? idx->wb_rec : what == 17 ? idx->wb_fsg : idx->wb_st[what - 14];
            const uint64_t len = what == 13 ? idx->n : what == 17 ? idx->A_len : idx->st_len[what - 14];
            src = wb;
            bytes = wb ? 32 * ((len + tds::WBOX_W - 1) / tds::WBOX_W) : 0;
            break;
        }
        default: fail(TDS_EINVAL, "unknown export %d", what);
    }
    if (!src && what != 11 && what != 12) fail(TDS_EINVAL, "array %d was not built", what);
    if (n_bytes) *n_bytes = bytes;
    if (dst && bytes) {
        uint64_t b = bytes < cap_bytes ? bytes : cap_bytes;
        if (host) memcpy(dst, src, b);
        else TDS_CUDA(cudaMemcpy(dst, src, b, cudaMemcpyDeviceToHost));
    }
    return TDS_OK;
    ABI_CATCH
}

}  // extern "C"
