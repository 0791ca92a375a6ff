// trajectory.cu — trajectory-level answers: the paper's problem
// statement asks for the *trajectories* within d of the query trajectories and
// the corresponding time periods; the search returns
// segment pairs.  This merges a result set into maximal disjoint intervals per
// (query trajectory, entry trajectory):
//   1. flatten the records; keys: t_in, then entry trajectory, then query
//      trajectory (three stable radix sorts = one sort by (q_traj, e_traj, t_in))
//   2. group heads where (q_traj, e_traj) changes; group starts by scan
//   3. one thread per group sweeps its intervals in t_in order and emits the
//      maximal ones (next.t_in <= current end + gap -> extend)
//   4. compaction into the output store
#include <algorithm>

#include "tds_internal.cuh"

namespace tds {

namespace {

inline unsigned nblk(uint64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

__global__ void k_flat_chunks(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                              const uint32_t *__restrict__ used, const uint64_t *__restrict__ off,
                              Rec *__restrict__ out) {
    uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    uint32_t u = used[c];
    uint64_t o = off[c];
    for (uint32_t k = lane; k < u; k += 32) out[o + k] = buf[c * CS + k];
}

__global__ void k_max_u32(const uint32_t *__restrict__ a, uint64_t n, uint32_t *__restrict__ mx) {
    uint32_t m = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, a[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// keys of the records in the current order `ord`: which = 0 t_in, 1 e_traj, 2 q_traj
__global__ void k_traj_key(const Rec *__restrict__ rs, const uint32_t *__restrict__ ord, uint64_t n, int which,
                           const uint32_t *__restrict__ q_traj, const uint32_t *__restrict__ e_traj,
                           uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t src = ord ? ord[i] : (uint32_t)i;
    const Rec r = rs[src];
    keys[i] = which == 0 ? float_key(r.t_in) : (which == 1 ? e_traj[r.eid] : q_traj[r.qid]);
    vals[i] = src;
}

__global__ void k_traj_gather(const Rec *__restrict__ rs, const uint32_t *__restrict__ ord, uint64_t n,
                              const uint32_t *__restrict__ q_traj, const uint32_t *__restrict__ e_traj,
                              Rec *__restrict__ out, uint32_t *__restrict__ head) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Rec r = rs[ord[i]];
    const uint32_t qt = q_traj[r.qid], et = e_traj[r.eid];
    out[i] = Rec{qt, et, r.t_in, r.t_out};
    bool h = true;
    if (i > 0) {
        const Rec p = rs[ord[i - 1]];
        h = (q_traj[p.qid] != qt) || (e_traj[p.eid] != et);
    }
    head[i] = h ? 1u : 0u;
}

__global__ void k_group_starts(const uint32_t *__restrict__ head, const uint32_t *__restrict__ gid, uint64_t n,
                               uint32_t *__restrict__ gstart, uint32_t ngroups) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && head[i]) gstart[gid[i]] = (uint32_t)i;
    if (i == 0) gstart[ngroups] = (uint32_t)n;
}

// one thread per group: sweep the group's intervals (t_in order), emit maximal ones
__global__ void k_merge_groups(const Rec *__restrict__ srt, const uint32_t *__restrict__ gstart, uint32_t ngroups,
                               float gap, Rec *__restrict__ tmp, uint32_t *__restrict__ cnt) {
    uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const uint32_t a = gstart[g], b = gstart[g + 1];
    Rec cur = srt[a];
    uint32_t k = 0;
    for (uint32_t i = a + 1; i < b; ++i) {
        const Rec r = srt[i];
        if (r.t_in <= cur.t_out + gap) {
            cur.t_out = fmaxf(cur.t_out, r.t_out);
        } else {
            tmp[a + k++] = cur;
            cur = r;
        }
    }
    tmp[a + k++] = cur;
    cnt[g] = k;
}

__global__ void k_merge_compact(const Rec *__restrict__ tmp, const uint32_t *__restrict__ gstart,
                                const uint32_t *__restrict__ cnt, const uint32_t *__restrict__ pos, uint32_t ngroups,
                                Rec *__restrict__ out) {
    uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const uint32_t a = gstart[g], p = pos[g];
    for (uint32_t k = 0; k < cnt[g]; ++k) out[p + k] = tmp[a + k];
}

}  // namespace

void merge_trajectories(tds_result_s *r, const uint32_t *q_traj, uint64_t nq, const uint32_t *e_traj, uint64_t ne,
                        float gap, cudaStream_t s, tds_result_s *out) {
    memset(&out->stats, 0, sizeof out->stats);
    out->stream = s;
    out->chunked = false;
    out->n = 0;
    const uint64_t n = r->n;
    if (n == 0) return;
    if (n >= (1ull << 32)) fail(TDS_EINVAL, "merge_trajectories: %llu records (limit 2^32)", (unsigned long long)n);
    // flat records
    DBuf<Rec> flat;
    const Rec *rs = r->store;
    if (r->chunked) {
        flat = DBuf<Rec>(n, s, n * sizeof(Rec) > (256ull << 20));
        k_flat_chunks<<<nblk(r->nchunks * 32), 256, 0, s>>>(r->buf, r->CS, r->nchunks, r->chunk_used, r->chunk_off,
                                                            flat.p);
        TDS_CHECK_LAUNCH();
        rs = flat.p;
    }
    // bits needed for the trajectory keys
    DBuf<uint32_t> mx(2, s);
    TDS_CUDA(cudaMemsetAsync(mx.p, 0, 8, s));
    k_max_u32<<<std::min<unsigned>(nblk(nq), 1024), 256, 0, s>>>(q_traj, nq, mx.p);
    TDS_CHECK_LAUNCH();
    k_max_u32<<<std::min<unsigned>(nblk(ne), 1024), 256, 0, s>>>(e_traj, ne, mx.p + 1);
    TDS_CHECK_LAUNCH();
    uint32_t hmx[2] = {0, 0};
    TDS_CUDA(cudaMemcpyAsync(hmx, mx.p, 8, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    auto bits = [](uint32_t m) { int b = 1; while (b < 32 && (1ull << b) <= m) ++b; return b; };
    // three stable sorts = sort by (q_traj, e_traj, t_in)
    DBuf<uint32_t> keys(n, s), ord(n, s), ord2(n, s);
    k_traj_key<<<nblk(n), 256, 0, s>>>(rs, nullptr, n, 0, q_traj, e_traj, keys.p, ord.p);
    TDS_CHECK_LAUNCH();
    radix_sort_pairs(keys, ord, n, 0, 32, s);
    k_traj_key<<<nblk(n), 256, 0, s>>>(rs, ord.p, n, 1, q_traj, e_traj, keys.p, ord2.p);
    TDS_CHECK_LAUNCH();
    radix_sort_pairs(keys, ord2, n, 0, bits(hmx[1]), s);
    k_traj_key<<<nblk(n), 256, 0, s>>>(rs, ord2.p, n, 2, q_traj, e_traj, keys.p, ord.p);
    TDS_CHECK_LAUNCH();
    radix_sort_pairs(keys, ord, n, 0, bits(hmx[0]), s);
    // sorted records with trajectory ids, group heads, group starts
    DBuf<Rec> srt(n, s, n * sizeof(Rec) > (256ull << 20));
    DBuf<uint32_t> head(n + 1, s), gid(n + 1, s);
    TDS_CUDA(cudaMemsetAsync(head.p + n, 0, 4, s));
    k_traj_gather<<<nblk(n), 256, 0, s>>>(rs, ord.p, n, q_traj, e_traj, srt.p, head.p);
    TDS_CHECK_LAUNCH();
    flat.reset();
    exclusive_scan_u32(head.p, gid.p, n + 1, nullptr, s);
    uint32_t ngroups = 0;
    TDS_CUDA(cudaMemcpyAsync(&ngroups, gid.p + n, 4, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    DBuf<uint32_t> gstart(ngroups + 1, s), cnt(ngroups + 1, s), pos(ngroups + 1, s);
    k_group_starts<<<nblk(n), 256, 0, s>>>(head.p, gid.p, n, gstart.p, ngroups);
    TDS_CHECK_LAUNCH();
    DBuf<Rec> tmp(n, s, n * sizeof(Rec) > (256ull << 20));
    TDS_CUDA(cudaMemsetAsync(cnt.p + ngroups, 0, 4, s));
    k_merge_groups<<<nblk(ngroups), 128, 0, s>>>(srt.p, gstart.p, ngroups, gap, tmp.p, cnt.p);
    TDS_CHECK_LAUNCH();
    exclusive_scan_u32(cnt.p, pos.p, ngroups + 1, nullptr, s);
    uint32_t nout = 0;
    TDS_CUDA(cudaMemcpyAsync(&nout, pos.p + ngroups, 4, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    DBuf<Rec> store(nout, s, nout * sizeof(Rec) > (256ull << 20));
    k_merge_compact<<<nblk(ngroups), 128, 0, s>>>(tmp.p, gstart.p, cnt.p, pos.p, ngroups, store.p);
    TDS_CHECK_LAUNCH();
    TDS_CUDA(cudaStreamSynchronize(s));
    out->store = store.release();
    out->n = nout;
    out->stats.n_results = nout;
    out->stats.n_queries = r->stats.n_queries;
}

}  // namespace tds
