/*
 * tds.h — C-ABI of the B200 distance threshold search over 4-D trajectory
 * line segments (Gowanlock & Casanova, arXiv 1410.2698).
 *
 * Citations: "P:a-b" = lines of the paper text; section / figure /
 * algorithm named beside it.  Readings of silent or garbled points are listed
 * in DESIGN.md ("Readings", C1-C24).
 *
 * The operation (§3.1 "Problem Definition"):
 *   D is a database of n entry line segments, each a 4-D segment from
 *   (x,y,z,t)_start to (x,y,z,t)_end, moving linearly in between
 *   (P:102-104).  For a query set Q, a threshold d and a window [T0,T1], the
 *   result set is every (query q, entry e, [t_in, t_out]) such that the shared
 *   span [a,b] = [max(t0q,t0e,T0), min(t1q,t1e,T1)] has a < b and
 *   [t_in,t_out] = { t in [a,b] : ||Pq(t) - Pe(t)||_2 <= d } is non-empty
 *   ("(q1, l1, [0.1, 0.3])").  Distance is synchronous Euclidean
 *   3-D distance.
 *
 * Candidate selection, chosen per search:
 *   TDS_TEMPORAL        GPUTemporal  (§4.2, Alg. 2)
 *   TDS_SPATIAL         GPUSpatial   (§4.1, Alg. 1)
 *   TDS_SPATIOTEMPORAL  GPUSpatioTemporal (§4.3, Alg. 3)
 * Every variant returns the same result set (the indexes are filters).
 *
 * Conventions for every entry point:
 *   - Return 0 (TDS_OK) on success, else a tds_status; a message describing
 *     the failure is available from tds_last_error() (thread-local).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Calls enqueue work on it and synchronise it before returning
 *     unless stated otherwise.
 *   - Input pointers may be DEVICE or HOST memory (detected with
 *     cudaPointerGetAttributes); host inputs are copied to the device inside
 *     the call.  Inputs are read only during the call and never retained.
 *   - Ids in results are row numbers in the caller's input arrays (reading
 *     C9), not positions after the internal sorts.
 *   - The library never falls back to a CPU implementation.
 */
#ifndef TDS_H
#define TDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One segment, 32 bytes: (x0,y0,z0,t0, x1,y1,z1,t1) in float32.
 * Arrays of tds_seg must be 16-byte aligned. */
typedef struct { float x0, y0, z0, t0, x1, y1, z1, t1; } tds_seg;

/* Index variants (bit flags for tds_index_params.kinds; one value for tds_search). */
enum {
    TDS_TEMPORAL = 1,          /* temporal bins */
    TDS_SPATIAL = 2,           /* flatly structured grid */
    TDS_SPATIOTEMPORAL = 4,    /* temporal bins split into spatial subbins */
    TDS_ALL = 7,
    TDS_AUTO = 8               /* tds_search only: per batch, GPUSpatioTemporal or GPUTemporal,
                                  whichever has the lower estimated cost = scheduled pair tests x
                                  measured cost per pair test (the index choice of P:776-777,
                                  P:1693-1696); needs both built, else GPUTemporal */
};

typedef enum {
    TDS_OK = 0,
    TDS_EINVAL = 1,     /* bad argument: n==0, d<=0 or not finite, T0>T1, m<1, v<1 or v above the
                           admissible bound of P:816-821, grid<1, NULL pointer, unbuilt variant */
    TDS_EDATA = 2,      /* a segment has a non-finite value or t_end <= t_start (message: first index) */
    TDS_ENOMEM = 3,     /* device allocation failed */
    TDS_ECAPACITY = 4,  /* one query alone produces more records than `capacity` */
    TDS_ECUDA = 5       /* CUDA runtime error (message carries cudaGetErrorString) */
} tds_status;

typedef struct {
    uint32_t kinds;     /* OR of TDS_TEMPORAL / TDS_SPATIAL / TDS_SPATIOTEMPORAL to build
                           (the temporal structure is always built: ST refines it) */
    int32_t m_bins;     /* m, number of temporal bins, >= 1 (10,000 for S1, 1,000 S2/S3) */
    int32_t v_subbins;  /* v, spatial subbins per dimension per bin, 1 <= v <= floor(extent_c /
                           max per-segment extent_c) for c = x,y,z */
    int32_t grid[3];    /* FSG cells per dimension, >= 1 (50 each in P:1391) */
    uint32_t flags;     /* 0, or TDS_INDEX_TIME_ORDER (below) */
} tds_index_params;

/* tds_index_params.flags.  The build renumbers D.  Default: by
 * temporal bin, and inside a bin by the Morton code of the segment's start cell on
 * a 1024^3 grid over D's extent, so that the range
 * kernel's candidate windows are spatially compact and whole windows can be
 * rejected against a query's box.  TDS_INDEX_TIME_ORDER: by t_start as the paper
 * states (every bin, range and result is the same; only the order of the entries
 * inside a bin differs). */
enum { TDS_INDEX_TIME_ORDER = 1 };

typedef struct tds_index_s *tds_index;
typedef struct tds_result_s *tds_result;

typedef struct {
    uint64_t n_results;         /* records in the result set */
    uint64_t n_queries;         /* queries searched (after dropping empty windows) */
    uint64_t pair_tests;        /* candidate pairs the schedule assigns (sum of range lengths;
                                   GPUSpatial: sum over (query, cell) of cell sizes) */
    uint64_t pairs_executed;    /* pairs the kernel actually evaluated (tiles cover unions) */
    uint64_t refined_pairs;     /* pairs re-evaluated in fp64 (near threshold or hits) */
    uint64_t passes;            /* pair-kernel passes (1 + overflow re-launches) */
    uint64_t spilled;           /* records moved out of the pass buffer on overflow */
    uint64_t fallback_queries;  /* GPUSpatioTemporal queries using the temporal fallback */
    float ms_schedule;          /* device time of query sort + schedule (CUDA events) */
    float ms_pairs;             /* device time of the pair kernel passes */
    float ms_compact;           /* device time of overflow compaction / re-planning */
    float ms_total;             /* tds_search device time */
    int32_t kind;               /* the variant that ran (TDS_TEMPORAL / TDS_SPATIAL / TDS_SPATIOTEMPORAL) */
    int32_t reserved;
    uint64_t pair_tests_alt;    /* TDS_AUTO: scheduled pair tests of the variant not chosen (else 0) */
    uint64_t capacity;          /* records the pass buffer held (after any halving on ENOMEM) */
    uint64_t refined32;         /* filter passes evaluated by the fp32 interval step (refine) */
    uint64_t direct_records;    /* records appended by the whole-span test of dense windows */
} tds_stats;

/*
 * tds_build_index — build the resident index over D (D is stored
 * once on the GPU and queried many times; build time is excluded from the
 * paper's response times).
 *
 *   entries : n segments (device or host memory), copied into index-owned memory
 *   n       : number of entry segments (>= 1, < 2^32)
 *   params  : see tds_index_params
 *   out     : receives the index handle; free with tds_index_free
 *
 * Steps: validate + extents;
 * stable radix sort by t_start and renumbering; bins;
 * optional subbin arrays X/Y/Z and FSG cell lists G/A.
 * Errors: TDS_EINVAL, TDS_EDATA, TDS_ENOMEM, TDS_ECUDA.  Synchronises stream.
 */
int tds_build_index(const tds_seg *entries, uint64_t n, const tds_index_params *params,
                    void *stream, tds_index *out);

/*
 * tds_search — the distance threshold search of Q against the index
 * (Alg. 1 / 2 / 3).
 *
 *   kind      : TDS_TEMPORAL, TDS_SPATIAL or TDS_SPATIOTEMPORAL (must have been built), or
 *               TDS_AUTO (see above; the chosen variant is reported in tds_stats.kind)
 *   queries   : nq segments (device or host memory); nq == 0 gives an empty result
 *   d         : distance threshold, finite and > 0 ("within d" is <= d, reading C4); a double:
 *               the hit decision and interval are exact for this d (fp32 filters use d
 *               rounded up, which only adds candidates)
 *   t_start, t_end : query window [T0, T1]; pass -INFINITY / +INFINITY for none
 *   capacity  : records the pass buffer holds (the paper's fixed result buffer);
 *               0 = automatic.  When a pass overflows, the records of the queries that
 *               lost records are discarded and those queries are re-run in batches that
 *               fit (reading C22); never duplicates, always progresses.
 *   out       : receives the result handle (free with tds_result_free)
 *   n_results : receives the number of records (may be NULL)
 * Errors: TDS_EINVAL, TDS_EDATA (bad query segment), TDS_ENOMEM, TDS_ECAPACITY, TDS_ECUDA.
 * Synchronises stream (one host synchronisation per pass).
 */
int tds_search(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d,
               float t_start, float t_end, uint64_t capacity, void *stream,
               tds_result *out, uint64_t *n_results);

/*
 * tds_search_part — part `part` of a work-balanced split of one tds_search into
 * `nparts` parts (multi-GPU query sharding; the paper's
 * search is data-parallel over query segments, one thread per query, P:430,
 * P:698-701).  Every part computes the same schedule from the full query set
 * and evaluates a contiguous slice of it:
 *   GPUTemporal / GPUSpatioTemporal: the slice of the schedule, sorted by
 *     (selector, range start), whose exact pair-test prefix sum crosses
 *     part/nparts and (part+1)/nparts of the total (sum of hi - lo);
 *   GPUSpatial: the queries (input order) whose flattened (query, cell) slot
 *     prefix crosses the same fractions.
 * The parts' result sets are disjoint and their union is the tds_search
 * result (query ids stay rows of the full query set).  tds_stats.pair_tests
 * and n_queries count this part only.  Arguments as tds_search, plus
 *   part, nparts : 0 <= part < nparts (nparts = 1 is tds_search)
 * Errors: those of tds_search; TDS_EINVAL for part >= nparts.
 */
int tds_search_part(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d,
                    float t_start, float t_end, uint64_t capacity, uint32_t part, uint32_t nparts,
                    void *stream, tds_result *out, uint64_t *n_results);

/*
 * tds_plan — the candidate-range schedule of a search without evaluating it
 * (query prep + candidate-range lookup: GPUTemporal P:680-698 "E_k", and the
 * GPUSpatioTemporal dimension choice P:1033-1083).  For every
 * query row k (HOST output arrays of nq elements):
 *   sel[k] : -1 temporal range (GPUTemporal, or a GPUSpatioTemporal fallback),
 *            0 / 1 / 2 a subbin range of X / Y / Z, 3 no candidates
 *   [lo[k], hi[k]) : the range in the sorted entries (sel = -1) or in X/Y/Z
 *            (sorted-entry positions; see tds_index_export what = 0, 3-5)
 * kind must be TDS_TEMPORAL or TDS_SPATIOTEMPORAL.  For tests and work
 * planning.  Errors: TDS_EINVAL, TDS_EDATA, TDS_ENOMEM, TDS_ECUDA.
 * Synchronises stream.
 */
int tds_plan(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start,
             float t_end, void *stream, int32_t *sel, uint32_t *lo, uint32_t *hi);

/*
 * tds_time_partition — the entries of D owned by part `part` of `nparts` under
 * time-partitioned sharding (the paper's distributed scenario, P:215-217;
 * SURVEY §8f-1, reading C27): the positions [part*n/nparts, (part+1)*n/nparts)
 * of the stable (t_start, row) order — contiguous time ranges of equal entry
 * count.  The order is a device radix sort of the t_start column (the sort of
 * the index build), so only 4 B per entry need to be resident.
 *   t_start : n floats (device or host memory), t_start of every row of D
 *   rows    : DEVICE output, room for n/nparts + 1 row numbers; receives the
 *             rows of D of this part in (t_start, row) order
 *   n_rows  : receives their count
 * Errors: TDS_EINVAL (NULL, n == 0, part >= nparts), TDS_EDATA (non-finite
 * t_start), TDS_ENOMEM, TDS_ECUDA.  Synchronises stream.
 */
int tds_time_partition(const float *t_start, uint64_t n, uint32_t part, uint32_t nparts, void *stream,
                       uint32_t *rows, uint64_t *n_rows);

/*
 * tds_search_stream — tds_search of a query set in HOST memory, processed
 * `chunk` queries at a time (the chunked processing of a large query set of
 * the prior work): while chunk k is searched on the
 * device, chunk k+1 is copied in and chunk k-1's records are copied out to
 * pinned host memory, on a second stream.  The device holds two chunks of
 * queries and one chunk's records at a time, so Q and the result may exceed
 * device memory.
 *   queries : nq segments in host memory (pinned: copied directly; pageable:
 *             through a pinned bounce buffer)
 *   chunk   : queries per chunk (>= 1)
 *   part, nparts : as tds_search_part, applied to every chunk (0, 1: all)
 * The result is host-resident: query ids are rows of the full query set;
 * tds_fetch_results copies from host memory (sorted fetches and device
 * destinations upload the records first); tds_merge_trajectories is not
 * available for it (TDS_EINVAL).  tds_stats sums the chunks' counters;
 * ms_total is wall-clock time.  Other arguments and errors as tds_search
 * (TDS_EINVAL also for device-resident queries and chunk == 0).
 * Synchronises stream.
 */
int tds_search_stream(tds_index idx, int kind, const tds_seg *queries, uint64_t nq, double d, float t_start,
                      float t_end, uint64_t chunk, uint32_t part, uint32_t nparts, void *stream, tds_result *out,
                      uint64_t *n_results);

/* one request of tds_search_many: the arguments of tds_search */
typedef struct tds_search_req {
    int kind;
    const tds_seg *queries;
    uint64_t nq;
    double d;
    float t_start, t_end;
    uint64_t capacity;
    void *stream;
} tds_search_req;

/*
 * tds_search_many — n independent searches of one index (the same operation as
 * n tds_search calls; serving several query sets, or one set under several
 * variants).  Requests on distinct streams
 * run concurrently: each is driven by its own host thread (a persistent
 * internal pool), so their host synchronisations and launch chains overlap;
 * requests sharing a stream run one after another in request order.
 *
 *   reqs      : n requests (see tds_search for the meaning of each field)
 *   out       : n result handles (out[i] for reqs[i]; free each with tds_result_free)
 *   n_results : n counts (may be NULL)
 * Errors: those of tds_search.  On any failure no result is returned (all are
 * freed, out[i] = NULL) and the error of the first failing request in request
 * order is reported.  Synchronises every request stream.
 */
int tds_search_many(tds_index idx, int n, const tds_search_req *reqs, tds_result *out,
                    uint64_t *n_results);

/*
 * tds_fetch_results — copy records [first, first+count) into caller arrays
 * (each `count` long): query_id / entry_id (row numbers of the caller's Q and
 * D), t_in / t_out (the closed interval, float32).  Any output pointer may be
 * NULL to skip that column.  dst_is_device: 1 = outputs are device memory,
 * 0 = host memory.  sorted: 1 = records ordered by (query_id, entry_id)
 * (the order is otherwise unspecified: atomic appends).
 * Device destinations: the copy is enqueued on `stream` and the call returns
 * without synchronising (stream order makes the outputs valid for later work
 * on that stream).  Host destinations: synchronises stream.
 * Errors: TDS_EINVAL (range outside the result), TDS_ECUDA.
 */
int tds_fetch_results(tds_result r, uint64_t first, uint64_t count, uint32_t *query_id,
                      uint32_t *entry_id, float *t_in, float *t_out, int dst_is_device,
                      int sorted, void *stream);

/*
 * tds_merge_trajectories — the trajectory-level answer ("find all
 * trajectories within d ... over [t_start, t_end]", "and corresponding
 * time periods").  Segments belong to trajectories:
 * q_traj[k] / e_traj[i] is the trajectory id of query row k / entry row i
 * (device or host memory; nq must equal the searched query count, ne the
 * index's entry count).  For every (query trajectory, entry trajectory) pair
 * the closed intervals of its segment-pair records are merged into maximal
 * disjoint intervals (an interval merges with the next when the next starts
 * no later than `gap` after it ends; gap = 0: overlapping or touching, e.g.
 * contacts across a shared timestep).  The new result holds records
 * (query trajectory id, entry trajectory id, t_in, t_out), fetched with
 * tds_fetch_results (query_id / entry_id columns carry the trajectory ids).
 * Errors: TDS_EINVAL (NULL, size mismatch, bad gap), TDS_ENOMEM, TDS_ECUDA.
 * Synchronises stream.
 */
int tds_merge_trajectories(tds_result r, const uint32_t *q_traj, uint64_t nq, const uint32_t *e_traj,
                           uint64_t ne, float gap, void *stream, tds_result *out, uint64_t *n_out);

/* tds_result_stats — counters and device timings of the search that made r. */
int tds_result_stats(tds_result r, tds_stats *out);

/* tds_result_count — number of records in r. */
uint64_t tds_result_count(tds_result r);

/* tds_result_host_block — zero-copy access to a host-resident result
 * (tds_search_stream): block i (i = 0, 1, ... until *count == 0 and *records
 * == NULL) holds *count records of 16 B, (query_id, entry_id, t_in, t_out) as
 * uint32, uint32, float, float, in pinned host memory owned by r (valid until
 * tds_result_free).  Errors: TDS_EINVAL (NULL, or not a host-resident result). */
int tds_result_host_block(tds_result r, uint64_t i, const void **records, uint64_t *count);

void tds_result_free(tds_result r);
void tds_index_free(tds_index idx);

/* tds_last_error — message of the last failed call on this thread ("" if none). */
const char *tds_last_error(void);

/*
 * tds_index_export — copy one internal index array to HOST memory, for tests
 * that pin the build against the paper's figures.  `what` selects:
 *   0 perm       uint32[n]      original row of sorted entry i (renumbering)
 *   1 bin_off    uint32[m+1]    first sorted entry of bin j (B_j^first; B_j^last = next-1)
 *   2 bin_hi     float[m]       max t_end over bin j's members (-inf if empty) (B_j^end)
 *   3 st_x/4 st_y/5 st_z uint32[len]   arrays X, Y, Z of sorted-entry ids
 *   6/7/8 st_off_x/y/z uint32[v*m+1]  start of subbin (slab j, bin i) at [j*m+i]
 *   9 fsg_cell_off uint32[gx*gy*gz+1]  dense CSR of cell h (row-major)
 *  10 fsg_A     uint32[len]     lookup array A of sorted-entry ids
 *  11 extents   float[16]       t_min, t_max, lo[3], hi[3], maxext[3], w_st[3], max_dur, pad
 *  12 sorted_t0 float[n]        t_start of the sorted entries
 *  13 wb_rec / 14-16 wb_x, wb_y, wb_z / 17 wb_fsg  float[8 * ceil(len / 128)]
 *               window boxes over the candidate orders (sorted entries, X/Y/Z, the
 *               FSG cell-ordered copy): per aligned window of 128 positions
 *               (min x, min y, min z, min t_start, max x, max y, max z, max t_end)
 *               of its segments (the range kernel's window test)
 * Writes min(cap_bytes, size) bytes to dst (may be NULL to query the size) and the
 * full size to *n_bytes.  Errors: TDS_EINVAL (unknown / unbuilt array).
 */
int tds_index_export(tds_index idx, int what, void *dst, uint64_t cap_bytes, uint64_t *n_bytes);

/* tds_index_info — n, m, v, grid of a built index (any pointer may be NULL). */
int tds_index_info(tds_index idx, uint64_t *n, int32_t *m, int32_t *v, int32_t *grid3,
                   uint32_t *kinds);

/* tds_kernel_launches — number of CUDA kernels this process has launched through
 * the library so far (a monotone counter; benchmarks difference it). */
uint64_t tds_kernel_launches(void);

/* tds_trim — release the device memory the library's pools hold unused (result
 * buffers are kept for reuse by later searches until this call or until an
 * allocation fails).  Current device; call when no search is running. */
void tds_trim(void);

/* tds_test_inject_enomem — TEST HOOK (fault injection, not for production use):
 * k >= 0: after letting the next `skip` large (result buffer) allocations
 * through, make the following k fail with TDS_ENOMEM.  Returns the number of
 * failures injected so far in the process (k < 0: only query the counter). */
uint64_t tds_test_inject_enomem(int k, int skip);

/* tds_version — library build string. */
const char *tds_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TDS_H */
