// partition.cu — time-partitioned sharding of D (the paper's
// distributed-memory scenario of "a number of GPU-equipped compute nodes",
// PAPER.md §3.2, reading C27): part k of K owns the entries at
// positions [k n / K, (k+1) n / K) of the stable (t_start, row) order, so the
// parts are contiguous time ranges of equal entry count.  The order comes from
// the same stable LSD radix sort of order-preserving t_start keys the index
// build uses, applied to the t_start column only (4 B per entry:
// a D too large for one GPU still has a t_start column that fits).
#include "tds_internal.cuh"

namespace tds {

namespace {

inline unsigned nblk(uint64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

__global__ void k_tkeys(const float *__restrict__ t, uint64_t n, uint32_t *__restrict__ keys,
                        uint32_t *__restrict__ vals, unsigned long long *__restrict__ bad) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float x = t[i];
    if (!isfinite(x)) atomicMax(bad, ~(unsigned long long)i);
    keys[i] = float_key(x);
    vals[i] = (uint32_t)i;
}

}  // namespace

uint64_t time_partition(const float *t_start, uint64_t n, uint32_t part, uint32_t nparts, uint32_t *rows,
                        cudaStream_t s) {
    DBuf<uint32_t> keys(n, s), vals(n, s);
    DBuf<unsigned long long> bad(1, s);
    TDS_CUDA(cudaMemsetAsync(bad.p, 0, 8, s));
    k_tkeys<<<nblk(n), 256, 0, s>>>(t_start, n, keys.p, vals.p, bad.p);
    TDS_CHECK_LAUNCH();
    radix_sort_pairs(keys, vals, n, 0, 32, s);
    const uint64_t lo = n * part / nparts, hi = n * (part + 1) / nparts;
    if (hi > lo)
        TDS_CUDA(cudaMemcpyAsync(rows, vals.p + lo, 4 * (hi - lo), cudaMemcpyDeviceToDevice, s));
    unsigned long long hb = 0;
    TDS_CUDA(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    if (hb) fail(TDS_EDATA, "t_start[%llu] is not finite", ~hb);
    return hi - lo;
}

}  // namespace tds
