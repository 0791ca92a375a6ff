// search.cu — the distance threshold search on the GPU (DESIGN.md steps A6-A11).
//
//   A6  query prep: sort Q by t_start, clip to the window [T0,T1]
//   A7  schedule: candidate range per query (temporal E_k; spatiotemporal
//       dimension choice; FSG cell rows)
//   A8  pair kernels (Alg. 1/2/3), B200 mapping:
//       lane = query, warp = 32 consecutive schedule entries, candidate records
//       broadcast to the warp (GPUTemporal / GPUSpatioTemporal); lane = candidate
//       over a flattened (query, cell-row) work list (GPUSpatial)
//   A9  pair test: fp32 certified filter + fp64 evaluation of the closed form
//   A10 result append: warp-aggregated, chunk-reserved; overflow -> exact re-plan
//       of the affected queries (reading C22)
//   A11 fetch
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "tds_internal.cuh"

namespace tds {

namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef TDS_RANGE_PT
#define TDS_RANGE_PT 256
#endif
constexpr int PT = TDS_RANGE_PT;         // threads per block of the pair kernel
#ifndef TDS_APPEND_FAST
#define TDS_APPEND_FAST 1                // appendK: warp-uniform fast path when the batch fits the chunk
#endif
#ifndef TDS_RANGE_BPS
#define TDS_RANGE_BPS 2
#endif
constexpr int RANGE_BPS = TDS_RANGE_BPS;       // resident blocks per SM (range kernel)
#ifndef TDS_ITEMS_PER_WARP
#define TDS_ITEMS_PER_WARP 64             // measured: 4 -> 32 = -14 % (d=0.03 ST) .. -22 % (d=0.01); 64 (final kernel): -0.7 % d=0.03, -1.7 % Merger, +1.3 % d=0.01 vs 48
#endif
#ifndef TDS_PRED_STORE
#define TDS_PRED_STORE 1                 // appendK: predicated record stores (inline PTX)
#endif
#ifndef TDS_DENSE_START
#define TDS_DENSE_START 8                // items start dense when the probe's pass fraction is >= this % (else
#endif                                   // the dense/sparse state carries over from the warp's last item)
#ifndef TDS_SPARSE_ONLY
#define TDS_SPARSE_ONLY 3                // sparse-only kernel when the probe's pass fraction is below this %
#endif
#ifndef TDS_HYST_HI
#define TDS_HYST_HI 25
#endif
#ifndef TDS_HYST_LO
#define TDS_HYST_LO 12
#endif
constexpr int HYST_HI = TDS_HYST_HI, HYST_LO = TDS_HYST_LO;
constexpr unsigned long long CAP_PROBE_MIN = 1ull << 24;     // result-size probe above this many pair tests
constexpr uint64_t CAP_FLOOR = 1ull << 22;                   // records: floor of the probed capacity
constexpr double ST_PAIR_COST = 1.5;     // TDS_AUTO: GPUSpatioTemporal cost per pair test / GPUTemporal's
constexpr uint32_t WIN = 128;            // range kernel window: 4 candidates per lane
static_assert(WIN == WBOX_W, "the range kernel's windows are the index's window-box windows");
// fp32 filter margin: eta = KU * M with M an l1 magnitude bound of the pair
// (derived bound 20 u M, u = 2^-24; 64 u used)
constexpr float KU = 64.0f / 16777216.0f;

struct DevStats {
    unsigned long long reserved;     // slots reserved in the pass buffer
    unsigned long long hits;         // records produced (kept or dropped)
    unsigned long long dropped;      // records dropped (buffer full)
    unsigned long long refined;      // pairs evaluated in fp64
    unsigned long long refined32;    // filter passes evaluated by refine_rel
    unsigned long long direct;       // records appended by the whole-span test
    unsigned long long executed;     // lane-pair slots evaluated
    unsigned long long pair_tests;   // algorithmic candidate pairs
    unsigned long long fallback;     // ST temporal fallbacks
    unsigned long long total_slots;  // spatial: flattened slots
    unsigned long long bad;          // ~(first invalid query row), 0 = none (atomicMax)
    unsigned long long union_total;  // sum of tile union lengths (chunk sizing)
    unsigned long long pair_tests_t; // TDS_AUTO: the GPUTemporal plan's pair tests
    unsigned int work_ctr;           // dynamic work distribution
    unsigned int total_items;
    unsigned int ch;                 // candidates per work item
    unsigned int cat_cnt[5];         // schedule entries per category
    unsigned int probe_pass, probe_total;   // density probe (k_density_probe)
    unsigned int part_lo, part_hi;   // tds_search_part: schedule entries / query rows of this part
    double probe_est;                // result-size probe: sum over sampled entries of len x pass fraction
    unsigned int probe_entries;      // sampled live entries
    unsigned int n_static;           // stationary query segments (k_count_static)
    unsigned long long part_slot_lo, part_slot_hi;   // GPUSpatial part: flattened slot range
    unsigned int pad[1];
};

struct Sched {                       // 16 B schedule entry
    uint32_t qid;                    // query row
    uint32_t lo, hi;                 // candidate range [lo, hi) in D (sel<0) or in X/Y/Z[sel]
    int32_t sel;                     // -1 temporal, 0/1/2 = X/Y/Z, 3 = empty
};

struct Tile {
    uint32_t tb, te;                 // schedule entries [tb, te), te - tb <= 32, one category
    uint32_t ulo, uhi;               // union of their ranges
    int32_t sel;
    uint32_t pad[3];
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Morton interleave helper: 10 bits -> every third bit
__device__ __forceinline__ uint32_t spread3(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

// ---------------------------------------------------------------------------
// A9: pair test
// ---------------------------------------------------------------------------
struct QConst {                      // per-lane query constants for the fp32 filter
    float px, py, pz;                // start point
    float vx, vy, vz;                // velocity
    float t0;                        // t_start
    float t0c, t1c;                  // span clipped to the window
    float ext;                       // |p1 - p0|_1
};

__device__ __forceinline__ QConst make_qconst(float4 a, float4 b, float T0, float T1) {
    QConst q;
    float dx = __fsub_rn(b.x, a.x), dy = __fsub_rn(b.y, a.y), dz = __fsub_rn(b.z, a.z);
    float r = rcp_approx(__fsub_rn(b.w, a.w));
    q.px = a.x; q.py = a.y; q.pz = a.z;
    q.vx = dx * r; q.vy = dy * r; q.vz = dz * r;
    q.t0 = a.w;
    q.t0c = fmaxf(a.w, T0);
    q.t1c = fminf(b.w, T1);
    q.ext = fabsf(dx) + fabsf(dy) + fabsf(dz);
    return q;
}

// candidate-side terms of the filter, computed once per loaded candidate and
// reused for every query of the group
struct ECand {
    float px, py, pz, t0;
    float vx, vy, vz, t1;
    float ext;
};

__device__ __forceinline__ ECand make_ecand(float4 a, float4 b) {
    ECand e;
    float dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    float r = rcp_approx(b.w - a.w);
    e.px = a.x; e.py = a.y; e.pz = a.z; e.t0 = a.w;
    e.vx = dx * r; e.vy = dy * r; e.vz = dz * r; e.t1 = b.w;
    e.ext = fabsf(dx) + fabsf(dy) + fabsf(dz);
    return e;
}

// The hot-loop filter (certified): false only if the pair is
// certainly not within d — empty shared span, or fp32 closest approach > d + eta
// with eta = 64 u M >= the derived error bound 20 u M, M = |p0q - p0e|_1 +
// |p1q - p0q|_1 + |p1e - p0e|_1, u = 2^-24.  q0 = (p0, t0), q1 = (v, ext) of the
// query, [t0c, t1c] its window-clipped span, e the candidate's terms.
__device__ __forceinline__ bool filter_pair(float4 q0, float4 q1, float t0c, float t1c, const ECand &e, float d) {
    const float a = fmaxf(t0c, e.t0), b = fminf(t1c, e.t1);
    const float aq = a - q0.w, ae = a - e.t0;
    const float dpx = q0.x - e.px, dpy = q0.y - e.py, dpz = q0.z - e.pz;
    const float Dx = fmaf(-ae, e.vx, fmaf(aq, q1.x, dpx));
    const float Dy = fmaf(-ae, e.vy, fmaf(aq, q1.y, dpy));
    const float Dz = fmaf(-ae, e.vz, fmaf(aq, q1.z, dpz));
    const float Vx = q1.x - e.vx, Vy = q1.y - e.vy, Vz = q1.z - e.vz;
    const float L = b - a;
    const float A = fmaf(Vx, Vx, fmaf(Vy, Vy, Vz * Vz));
    const float B = fmaf(Dx, Vx, fmaf(Dy, Vy, Dz * Vz));
    const float s = fminf(fmaxf(-B * rcp_approx(A), 0.f), L);
    const float yx = fmaf(s, Vx, Dx), yy = fmaf(s, Vy, Dy), yz = fmaf(s, Vz, Dz);
    const float h = fmaf(yx, yx, fmaf(yy, yy, yz * yz));
    const float M = fabsf(dpx) + fabsf(dpy) + fabsf(dpz) + (q1.w + e.ext);
    const float thr = fmaf(KU, M, d);
    return (a < b) & (h <= thr * thr);
}

// Absolute-time form of the certified filter ("absolute form"),
// used by the range kernel's sparse windows.  Times are shifted by a constant
// origin tc (the middle of the index's time extent): t' = fl(t - tc), monotone
// in t.  Each segment is written as P(t') = c + v t' with c = P0 - v t0', so
// the relative motion is C + V t' and the closest approach over the shared span
// [a', b'] is at clamp(-(C.V)/A, a', b') — no per-pair time offsets.  Its fp32
// error is <= 12 u (m_q + m_e) with the per-segment magnitude
// m = |c|_1 + |P1 - P0|_1 + max(|t0'|, |t1'|) |v|_1, so the margin
// eta = 64 u (m_q + m_e) keeps a factor > 5.  The span test is a' <= b' (a
// superset of a < b: rounding t - tc may merge a' and b').
struct FSeg {
    float cx, cy, cz, m;
    float vx, vy, vz, t0, t1;        // t0, t1 shifted by tc
};

__device__ __forceinline__ FSeg make_fseg(float4 a, float4 b, float tc) {
    FSeg f;
    const float dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    const float r = rcp_approx(b.w - a.w);
    f.t0 = a.w - tc; f.t1 = b.w - tc;
    f.vx = dx * r; f.vy = dy * r; f.vz = dz * r;
    f.cx = fmaf(-f.vx, f.t0, a.x); f.cy = fmaf(-f.vy, f.t0, a.y); f.cz = fmaf(-f.vz, f.t0, a.z);
    const float T = fmaxf(fabsf(f.t0), fabsf(f.t1));
    f.m = fmaf(T, fabsf(f.vx) + fabsf(f.vy) + fabsf(f.vz),
               (fabsf(f.cx) + fabsf(f.cy) + fabsf(f.cz)) + (fabsf(dx) + fabsf(dy) + fabsf(dz)));
    return f;
}

// ---- packed fp32x2 (FFMA2 / FADD2 / FMUL2, sm_100): the lane's two candidates
// against one query in one instruction stream.  Each lane of a pair is an IEEE
// round-to-nearest fp32 operation, so filter_abs2 computes bit-for-bit what
// the scalar arithmetic computes for each candidate (same bound); it halves the FMA-pipe
// instructions, which bound the pair loop (B300_MICROARCH: 3-register FFMA
// issues at most every second cycle per SMSP).
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f32x2 r, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ f32x2 bc2(float x) { return pk2(x, x); }
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

struct FSeg2 {                       // two candidates, packed per field
    f32x2 cx, cy, cz, m, vx, vy, vz;
    float t0a, t0b, t1a, t1b;
};

__device__ __forceinline__ FSeg2 make_fseg2(const FSeg &p, const FSeg &q) {
    FSeg2 e;
    e.cx = pk2(p.cx, q.cx); e.cy = pk2(p.cy, q.cy); e.cz = pk2(p.cz, q.cz); e.m = pk2(p.m, q.m);
    e.vx = pk2(p.vx, q.vx); e.vy = pk2(p.vy, q.vy); e.vz = pk2(p.vz, q.vz);
    e.t0a = p.t0; e.t0b = q.t0; e.t1a = p.t1; e.t1b = q.t1;
    return e;
}

// The absolute-form filter for the two candidates of e.  Per candidate:
// a = max(t0c, t0e), b = min(t1c, t1e); C = c_q - c_e, V = v_q - v_e;
// t* = clamp(-(C.V)/|V|^2, a, b); h = |C + V t*|^2; pass iff a <= b and
// h <= (df + 64u (m_q + m_e))^2 (bound in the FSeg comment / DESIGN.md §5);
// n0 = (c, m), n1 = (v, -) of the query, [t0c, t1c] its shifted clipped span.
__device__ __forceinline__ void filter_abs2(float4 n0, float4 n1, float t0c, float t1c, const FSeg2 &e, float df,
                                            bool &pass0, bool &pass1) {
    const float a0 = fmaxf(t0c, e.t0a), b0 = fminf(t1c, e.t1a);
    const float a1 = fmaxf(t0c, e.t0b), b1 = fminf(t1c, e.t1b);
    const f32x2 Cx = sub2(bc2(n0.x), e.cx), Cy = sub2(bc2(n0.y), e.cy), Cz = sub2(bc2(n0.z), e.cz);
    const f32x2 Vx = sub2(bc2(n1.x), e.vx), Vy = sub2(bc2(n1.y), e.vy), Vz = sub2(bc2(n1.z), e.vz);
    const f32x2 A = fma2(Vx, Vx, fma2(Vy, Vy, mul2(Vz, Vz)));
    const f32x2 B = fma2(Cx, Vx, fma2(Cy, Vy, mul2(Cz, Vz)));
    float A0, A1;
    upk2(A, A0, A1);
    float u0, u1;
    upk2(mul2(B, pk2(rcp_approx(A0), rcp_approx(A1))), u0, u1);
    const float s0 = fminf(fmaxf(-u0, a0), b0), s1 = fminf(fmaxf(-u1, a1), b1);
    const f32x2 t = pk2(s0, s1);
    const f32x2 yx = fma2(t, Vx, Cx), yy = fma2(t, Vy, Cy), yz = fma2(t, Vz, Cz);
    const f32x2 h = fma2(yx, yx, fma2(yy, yy, mul2(yz, yz)));
    const f32x2 thr = fma2(bc2(KU), add2(bc2(n0.w), e.m), bc2(df));
    const f32x2 thr2 = mul2(thr, thr);
    float h0, h1, r0, r1;
    upk2(h, h0, h1);
    upk2(thr2, r0, r1);
    pass0 = (a0 <= b0) & (h0 <= r0);
    pass1 = (a1 <= b1) & (h1 <= r1);
}

// filter_abs2 for a stationary query (P1 = P0: the supernova case (i) of
// P:84-88, a point over a time interval): V = -v_e exactly, so
// A = |v_e|^2 and its reciprocal rA are per-candidate terms computed once per
// window (rA packed for the pair), and B, t*, y lose the query-velocity terms.
// Every operation rounds to the same value as in filter_abs2 (negation is exact),
// so the decisions are bit-identical to the general filter's.
__device__ __forceinline__ void filter_static2(float4 n0, float t0c, float t1c, const FSeg2 &e, f32x2 rA, float df,
                                               bool &pass0, bool &pass1) {
    const float a0 = fmaxf(t0c, e.t0a), b0 = fminf(t1c, e.t1a);
    const float a1 = fmaxf(t0c, e.t0b), b1 = fminf(t1c, e.t1b);
    const f32x2 Cx = sub2(bc2(n0.x), e.cx), Cy = sub2(bc2(n0.y), e.cy), Cz = sub2(bc2(n0.z), e.cz);
    const f32x2 nB = fma2(Cx, e.vx, fma2(Cy, e.vy, mul2(Cz, e.vz)));       // -(C.V)
    float u0, u1;
    upk2(mul2(nB, rA), u0, u1);                                              // -(C.V)/A
    const float s0 = fminf(fmaxf(u0, a0), b0), s1 = fminf(fmaxf(u1, a1), b1);
    const f32x2 nt = pk2(-s0, -s1);
    const f32x2 yx = fma2(nt, e.vx, Cx), yy = fma2(nt, e.vy, Cy), yz = fma2(nt, e.vz, Cz);
    const f32x2 h = fma2(yx, yx, fma2(yy, yy, mul2(yz, yz)));
    const f32x2 thr = fma2(bc2(KU), add2(bc2(n0.w), e.m), bc2(df));
    float h0, h1, r0, r1;
    upk2(h, h0, h1);
    upk2(mul2(thr, thr), r0, r1);
    pass0 = (a0 <= b0) & (h0 <= r0);
    pass1 = (a1 <= b1) & (h1 <= r1);
}

// reciprocal of |v|^2 for the two candidates of e (stationary queries)
__device__ __forceinline__ f32x2 static_rA(const FSeg2 &e) {
    float A0, A1;
    upk2(fma2(e.vx, e.vx, fma2(e.vy, e.vy, mul2(e.vz, e.vz))), A0, A1);
    return pk2(rcp_approx(A0), rcp_approx(A1));
}

// filter_abs2 plus the whole-span test of dense windows: in0 / in1 = both ends of
// the shared span certainly within d (squared distance at a' and b' below
// (dlo - 64u (m_q + m_e))^2, the same certified margin: the bound holds at every
// point of the span, the rounded span ends included), so the pair's interval is
// exactly [a, b] (convexity in t).  qin = dlo - 64u m_q of the query.
__device__ __forceinline__ void filter_abs2x(float4 n0, float4 n1, float t0c, float t1c, float qin, const FSeg2 &e,
                                             float df, bool &pass0, bool &pass1, bool &in0, bool &in1) {
    const float a0 = fmaxf(t0c, e.t0a), b0 = fminf(t1c, e.t1a);
    const float a1 = fmaxf(t0c, e.t0b), b1 = fminf(t1c, e.t1b);
    const f32x2 Cx = sub2(bc2(n0.x), e.cx), Cy = sub2(bc2(n0.y), e.cy), Cz = sub2(bc2(n0.z), e.cz);
    const f32x2 Vx = sub2(bc2(n1.x), e.vx), Vy = sub2(bc2(n1.y), e.vy), Vz = sub2(bc2(n1.z), e.vz);
    const f32x2 A = fma2(Vx, Vx, fma2(Vy, Vy, mul2(Vz, Vz)));
    const f32x2 B = fma2(Cx, Vx, fma2(Cy, Vy, mul2(Cz, Vz)));
    float A0, A1;
    upk2(A, A0, A1);
    float u0, u1;
    upk2(mul2(B, pk2(rcp_approx(A0), rcp_approx(A1))), u0, u1);
    const f32x2 pa = pk2(a0, a1), pb = pk2(b0, b1);
    const f32x2 t = pk2(fminf(fmaxf(-u0, a0), b0), fminf(fmaxf(-u1, a1), b1));
    const f32x2 yx = fma2(t, Vx, Cx), yy = fma2(t, Vy, Cy), yz = fma2(t, Vz, Cz);
    const f32x2 h = fma2(yx, yx, fma2(yy, yy, mul2(yz, yz)));
    const f32x2 ax = fma2(pa, Vx, Cx), ay = fma2(pa, Vy, Cy), az = fma2(pa, Vz, Cz);
    const f32x2 bx = fma2(pb, Vx, Cx), by = fma2(pb, Vy, Cy), bz = fma2(pb, Vz, Cz);
    const f32x2 ha = fma2(ax, ax, fma2(ay, ay, mul2(az, az)));
    const f32x2 hb = fma2(bx, bx, fma2(by, by, mul2(bz, bz)));
    const f32x2 thr = fma2(bc2(KU), add2(bc2(n0.w), e.m), bc2(df));
    const f32x2 tin = fma2(bc2(-KU), e.m, bc2(qin));
    float h0, h1, r0, r1, ha0, ha1, hb0, hb1, ti0, ti1, q0, q1;
    upk2(h, h0, h1);
    upk2(mul2(thr, thr), r0, r1);
    upk2(ha, ha0, ha1);
    upk2(hb, hb0, hb1);
    upk2(tin, ti0, ti1);
    upk2(mul2(tin, tin), q0, q1);
    pass0 = (a0 <= b0) & (h0 <= r0);
    pass1 = (a1 <= b1) & (h1 <= r1);
    in0 = (a0 < b0) & (ti0 > 0.f) & (ha0 < q0) & (hb0 < q0);
    in1 = (a1 < b1) & (ti1 > 0.f) & (ha1 < q1) & (hb1 < q1);
}

// fp64 evaluation of the closed form (SURVEY §8c / DESIGN.md "Pair test"):
// the sublevel interval of the convex quadratic ||Pq(t)-Pe(t)||^2 <= d^2 on [a,b].
__device__ __forceinline__ bool pair64(float4 qa, float4 qb, float4 ea, float4 eb, double d, double T0, double T1,
                                    float &t_in, float &t_out) {
    double t0q = qa.w, t1q = qb.w, t0e = ea.w, t1e = eb.w;
    double a = fmax(fmax(t0q, t0e), T0);
    double b = fmin(fmin(t1q, t1e), T1);
    if (!(a < b)) return false;
    const double rq = 1.0 / (t1q - t0q), re = 1.0 / (t1e - t0e);   // 2 divisions instead of 6
    double vqx = ((double)qb.x - (double)qa.x) * rq, vqy = ((double)qb.y - (double)qa.y) * rq,
           vqz = ((double)qb.z - (double)qa.z) * rq;
    double vex = ((double)eb.x - (double)ea.x) * re, vey = ((double)eb.y - (double)ea.y) * re,
           vez = ((double)eb.z - (double)ea.z) * re;
    double Dx = ((double)qa.x + (a - t0q) * vqx) - ((double)ea.x + (a - t0e) * vex);
    double Dy = ((double)qa.y + (a - t0q) * vqy) - ((double)ea.y + (a - t0e) * vey);
    double Dz = ((double)qa.z + (a - t0q) * vqz) - ((double)ea.z + (a - t0e) * vez);
    double Vx = vqx - vex, Vy = vqy - vey, Vz = vqz - vez;
    double L = b - a;
    double A = Vx * Vx + Vy * Vy + Vz * Vz;
    double d2 = d * d;
    if (A == 0.0) {
        double h = Dx * Dx + Dy * Dy + Dz * Dz;
        if (h <= d2) { t_in = (float)a; t_out = (float)b; return true; }
        return false;
    }
    const double iA = 1.0 / A;
    double su = -(Dx * Vx + Dy * Vy + Dz * Vz) * iA;
    double ss = su < 0.0 ? 0.0 : (su > L ? L : su);
    double xs = Dx + ss * Vx, ys = Dy + ss * Vy, zs = Dz + ss * Vz;
    double hs = xs * xs + ys * ys + zs * zs;
    if (!(hs <= d2)) return false;
    double xu = Dx + su * Vx, yu = Dy + su * Vy, zu = Dz + su * Vz;
    double hu = xu * xu + yu * yu + zu * zu;
    double rem = d2 - hu;
    if (rem < 0.0) rem = 0.0;
    double w = sqrt(rem * iA);
    double lo = fmin(fmax(su - w, 0.0), L), hi = fmin(fmax(su + w, 0.0), L);
    t_in = (float)(a + lo);
    t_out = (float)(a + hi);
    return true;
}

// Refine one queued pair in the relative form (P(t) = P0 + (t - t0) v) with
// first-order error bounds evaluated from the pair's own magnitudes (DESIGN.md
// §5 "refine"): 0 = miss, 1 = undecided (fp64), 2 = certain hit with an fp32
// interval within 8e-6 (b - a) of the exact one.  dlo / dhi: d rounded down / up;
// d2h + d2l = d^2 (fp32 head and remainder).
__device__ __forceinline__ int refine_rel(float4 q0, float4 q1, float t0c, float t1c, float4 e0, float t1e, float vex,
                                          float vey, float vez, float dlo, float dhi, float d2h, float d2l, float &tin,
                                          float &tout) {
    constexpr float U = 1.0f / 16777216.0f;
    const float a = fmaxf(t0c, e0.w), b = fminf(t1c, t1e);
    if (!(a < b)) return 0;                                    // C5
    const float L = b - a, aq = a - q0.w, ae = a - e0.w;
    const float dpx = q0.x - e0.x, dpy = q0.y - e0.y, dpz = q0.z - e0.z;
    const float ix = fmaf(aq, q1.x, dpx), iy = fmaf(aq, q1.y, dpy), iz = fmaf(aq, q1.z, dpz);
    const float Dx = fmaf(-ae, vex, ix), Dy = fmaf(-ae, vey, iy), Dz = fmaf(-ae, vez, iz);
    const float Vx = q1.x - vex, Vy = q1.y - vey, Vz = q1.z - vez;
    // position error over the span: eD at s = 0 (roundings of dp, a - t0, the
    // velocities (<= 4u each) and the two FMAs), eV per unit s (velocities and V)
    const float V1e = fabsf(vex) + fabsf(vey) + fabsf(vez);
    const float D1 = fabsf(Dx) + fabsf(Dy) + fabsf(Dz), W1 = fabsf(Vx) + fabsf(Vy) + fabsf(Vz);
    const float eD = U * fmaf(7.f, fabsf(aq) * q1.w + fabsf(ae) * V1e, fabsf(dpx) + fabsf(dpy) + fabsf(dpz) + 2.f * D1);
    const float eV = U * fmaf(5.f, q1.w + V1e, W1);
    const float eP0 = fmaf(L, eV, eD);                         // first-order position error on [0, L]
    const float eP = 1.5f * eP0;                               // x1.5 for the distance decisions
    const float mg = fmaf(4.f * U, dhi, eP);                   // + rounding of the squared norms
    const float din = dlo - mg, dout = dhi + mg;
    // both span ends certainly within d: the whole span (convexity)
    const float ybx = fmaf(L, Vx, Dx), yby = fmaf(L, Vy, Dy), ybz = fmaf(L, Vz, Dz);
    const float ha = fmaf(Dx, Dx, fmaf(Dy, Dy, Dz * Dz)), hb = fmaf(ybx, ybx, fmaf(yby, yby, ybz * ybz));
    const float din2 = din * din;
    if (din > 0.f && ha < din2 && hb < din2) { tin = a; tout = b; return 2; }
    const float A = fmaf(Vx, Vx, fmaf(Vy, Vy, Vz * Vz));
    const float B = fmaf(Dx, Vx, fmaf(Dy, Vy, Dz * Vz));
    const float rA = rcp_approx(A);
    const float su = -B * rA;
    const float s = fminf(fmaxf(su, 0.f), L);
    const float yx = fmaf(s, Vx, Dx), yy = fmaf(s, Vy, Dy), yz = fmaf(s, Vz, Dz);
    const float h = fmaf(yx, yx, fmaf(yy, yy, yz * yz));
    if (!(h <= dout * dout)) return 0;                         // certain miss
    if (!(din > 0.f && h < din2)) return 1;                    // near the threshold
    // the interval: roots of A s^2 + 2 B s + Cd = 0 (Cd = |D|^2 - d^2) in the
    // cancellation-free form q = -(B + sgn(B) sqrt(Delta)), Delta = A (d^2 - h_u)
    // = B^2 - A Cd, roots q / A and Cd / q (the form s_u -+ w loses the digits of
    // s_u and w when both are large against the span: DESIGN.md §5)
    const float ux = fmaf(su, Vx, Dx), uy = fmaf(su, Vy, Dy), uz = fmaf(su, Vz, Dz);
    const float hu = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
    const float rem = fmaxf((d2h - hu) + d2l, 0.f);
    const float sq = sqrt_approx(A * rem);                     // sqrt(Delta) = A w = |y . V| at a root
    const bool bpos = B >= 0.f;
    const float q = bpos ? -(B + sq) : sq - B;
    const float rq = rcp_approx(q), rsq = rcp_approx(sq);
    const float Cd = (ha - d2h) - d2l;
    const float rbig = q * rA, rsmall = Cd * rq;
    const float lo = bpos ? rbig : rsmall, hi = bpos ? rsmall : rbig;
    // rounding error of each root for the computed D, V (first order): q from B
    // (3u sum|D_i V_i|), sqrt(Delta) (A: 3u, d^2 - h_u: 5u h_u + 2.1u rem, the
    // product, sqrt.approx: 2u) and its own rounding; q / A adds A, rcp and the
    // product (6u); Cd / q adds Cd (3u |D|^2 + 2.1u |Cd|), rcp and the product
    const float sdv = fabsf(Dx * Vx) + fabsf(Dy * Vy) + fabsf(Dz * Vz);
    const float dq = fmaf(3.f * U, sdv, fmaf(5.05f * U, sq, fmaf((2.5f * U) * hu, A * rsq, U * fabsf(q))));
    const float eq = dq * fabsf(rq);
    const float ebig = fabsf(rbig) * (eq + 6.f * U);
    const float esmall = fmaf(U * fmaf(3.f, ha, 2.1f * fabsf(Cd)), fabsf(rq), fabsf(rsmall) * (eq + 3.f * U));
    // input errors (the roundings of D and V against the exact motion): a root
    // moves by (y . dP) / |y . V| = (y . dP) / sqrt(Delta) for a position error
    // dP at the root, y = D + s V the relative position there (|y| = d), dP_i <=
    // eD_i + L eV_i per component (roundings of dp, a - t0, the velocities (<= 5u
    // each) and the FMAs)
    const float ex = U * fmaf(6.f, fabsf(aq * q1.x) + fabsf(ae * vex), fabsf(Dx) + fabsf(ix) + fabsf(dpx)) +
                     L * U * fmaf(5.f, fabsf(q1.x) + fabsf(vex), fabsf(Vx));
    const float ey = U * fmaf(6.f, fabsf(aq * q1.y) + fabsf(ae * vey), fabsf(Dy) + fabsf(iy) + fabsf(dpy)) +
                     L * U * fmaf(5.f, fabsf(q1.y) + fabsf(vey), fabsf(Vy));
    const float ez = U * fmaf(6.f, fabsf(aq * q1.z) + fabsf(ae * vez), fabsf(Dz) + fabsf(iz) + fabsf(dpz)) +
                     L * U * fmaf(5.f, fabsf(q1.z) + fabsf(vez), fabsf(Vz));
    const float yl = fabsf(fmaf(lo, Vx, Dx)) * ex + fabsf(fmaf(lo, Vy, Dy)) * ey + fabsf(fmaf(lo, Vz, Dz)) * ez;
    const float yh = fabsf(fmaf(hi, Vx, Dx)) * ex + fabsf(fmaf(hi, Vy, Dy)) * ey + fabsf(fmaf(hi, Vz, Dz)) * ez;
    const float dlt_lo = 1.25f * fmaf(yl, rsq, bpos ? ebig : esmall);
    const float dlt_hi = 1.25f * fmaf(yh, rsq, bpos ? esmall : ebig);
    tin = a + fminf(fmaxf(lo, 0.f), L);
    tout = a + fminf(fmaxf(hi, 0.f), L);
    const float tol = 8e-6f * L;
    const bool in_ok = (lo + dlt_lo < 0.f) || (dlt_lo <= tol);
    const bool out_ok = (hi - dlt_hi > L) || (dlt_hi <= tol);
    return (in_ok && out_ok) ? 2 : 1;
}

// ---------------------------------------------------------------------------
// A10: result append
// ---------------------------------------------------------------------------
struct OutArgs {
    Rec *buf;                        // pass buffer (chunked) or store (exact)
    unsigned long long cap;          // pass buffer slots
    uint32_t CS;                     // chunk size (slots), a power of two
    uint32_t cs_shift;               // log2(CS)
    uint32_t *chunk_used;            // [ceil(cap/CS)]
    uint8_t *redo;                   // [nq] 1 = query lost a record
    uint32_t *qcount;                // [nq] records produced per query
    const unsigned long long *qoff;  // exact mode: per-query output offset
    uint32_t *qfill;                 // exact mode: per-query fill
    DevStats *st;
};

// Per-warp shared state (warp-uniform; lane 0 writes, every lane reads):
// the result chunk being filled and the queue of pairs awaiting fp64 evaluation.
constexpr int RQ_CAP = 192;          // refine queue capacity (32 + up to 5 x 32 additions)

struct WarpState {
    unsigned long long ap_base;
    uint32_t ap_used, ap_size, ap_full;
    uint32_t refined, hits, r32;
    unsigned long long exec, direct; // range kernel: executed pair tests, whole-span records (lane 0)
    uint32_t fn;                     // fp64 queue fill (< 32 between flushes)
    uint16_t rq[RQ_CAP];             // refine queue: group slot g | window slot << 5
    uint32_t fq[64], fj[64];         // fp64 queue: pairs the fp32 stages could not decide
};

__device__ __forceinline__ void warp_state_init(WarpState &W, int lane) {
    if (lane == 0) {
        W.ap_base = 0; W.ap_used = 0; W.ap_size = 0; W.ap_full = 0; W.refined = 0; W.hits = 0; W.fn = 0; W.r32 = 0;
        W.exec = 0; W.direct = 0;
    }
    __syncwarp();
}

// predicated 16-B record store (no branch around it): the result buffer is
// write-only in the pair kernel, so the store needs no ordering with other accesses
__device__ __forceinline__ void st_rec_if(bool h, uint4 *p, const Rec &r) {
#if TDS_PRED_STORE
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q st.global.v4.u32 [%1], {%2, %3, %4, %5};\n\t}"
                 :: "r"((int)h), "l"(p), "r"(r.qid), "r"(r.eid), "r"(__float_as_uint(r.t_in)),
                    "r"(__float_as_uint(r.t_out)));
#else
    if (h) *p = make_uint4(r.qid, r.eid, __float_as_uint(r.t_in), __float_as_uint(r.t_out));
#endif
}

// warp-wide: every lane calls with its own hit flag / record.  Pass 1 appends
// into chunks of CS slots reserved with one atomic per chunk (warp-aggregated,
// no per-record global atomics); EXACT (re-plan passes) writes the record at
// its query's planned offset.
template <bool EXACT>
__device__ __forceinline__ void append(const OutArgs &o, WarpState &W, bool hit, const Rec &r, int lane) {
    const unsigned hm = __ballot_sync(FULL, hit);
    if (!hm) return;
    if (EXACT) {
        if (hit) {   // one atomic per (warp, query): lanes of the same query share it
            const unsigned peers = __match_any_sync(hm, r.qid);
            const int leader = __ffs(peers) - 1;
            uint32_t k = 0;
            if (lane == leader) k = atomicAdd(&o.qfill[r.qid], (uint32_t)__popc(peers));
            k = __shfl_sync(peers, k, leader) + __popc(peers & ((1u << lane) - 1u));
            unsigned long long slot = o.qoff[r.qid] + k;
            reinterpret_cast<uint4 *>(o.buf)[slot] = make_uint4(r.qid, r.eid, __float_as_uint(r.t_in),
                                                                __float_as_uint(r.t_out));
        }
        return;
    }
    const uint32_t k = __popc(hm);
    unsigned long long base = W.ap_base;
    uint32_t used = W.ap_used, size = W.ap_size, full = W.ap_full;
    if (!full && used + k > size) {
        if (size && lane == 0) o.chunk_used[base >> o.cs_shift] = used;
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(&o.st->reserved, (unsigned long long)o.CS);
        nb = __shfl_sync(FULL, nb, 0);
        if (nb >= o.cap) {
            full = 1; size = 0; used = 0;
        } else {
            base = nb;
            used = 0;
            unsigned long long room = o.cap - nb;
            size = room < o.CS ? (uint32_t)room : o.CS;
        }
    }
    const uint32_t rk = __popc(hm & ((1u << lane) - 1u));
    if (TDS_APPEND_FAST && !full && used + k <= size) {   // warp-uniform: the batch fits the chunk
        uint4 *out = reinterpret_cast<uint4 *>(o.buf) + (base + used);
        asm("mov.b64 %0, %0;" : "+l"(out));
        st_rec_if(hit, out + rk, r);
    } else if (hit) {
        if (!full && used + rk < size) {
            reinterpret_cast<uint4 *>(o.buf)[base + used + rk] =
                make_uint4(r.qid, r.eid, __float_as_uint(r.t_in), __float_as_uint(r.t_out));
        } else {
            o.redo[r.qid] = 1;
            atomicAdd(&o.st->dropped, 1ull);
        }
    }
    if (!full) used = min(used + k, size);
    __syncwarp();
    if (lane == 0) { W.ap_base = base; W.ap_used = used; W.ap_size = size; W.ap_full = full; }
    __syncwarp();
}

// K appends of one warp step (a lane's K candidates of one query) with one chunk
// reservation and one warp-state update: the records of set i follow those of
// sets 0..i-1 (k <= 32 K <= CS, so one chunk refresh always makes room).
template <bool EXACT, int K>
__device__ __forceinline__ void appendK(const OutArgs &o, WarpState &W, const bool (&h)[K], const unsigned (&hm)[K],
                                        const Rec (&r)[K], int lane) {
    if (EXACT) {
#pragma unroll
        for (int i = 0; i < K; ++i) append<EXACT>(o, W, h[i], r[i], lane);
        return;
    }
    uint32_t k = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) k += __popc(hm[i]);
    unsigned long long base = W.ap_base;
    uint32_t used = W.ap_used, size = W.ap_size, full = W.ap_full;
    if (!full && used + k > size) {
        if (size && lane == 0) o.chunk_used[base >> o.cs_shift] = used;
        unsigned long long nb = 0;
        if (lane == 0) nb = atomicAdd(&o.st->reserved, (unsigned long long)o.CS);
        nb = __shfl_sync(FULL, nb, 0);
        if (nb >= o.cap) {
            full = 1; size = 0; used = 0;
        } else {
            base = nb;
            used = 0;
            unsigned long long room = o.cap - nb;
            size = room < o.CS ? (uint32_t)room : o.CS;
        }
    }
    const unsigned lt = (1u << lane) - 1u;
    if (TDS_APPEND_FAST && !full && used + k <= size) {   // warp-uniform: the whole batch fits the chunk
        uint4 *out = reinterpret_cast<uint4 *>(o.buf) + (base + used);
        asm("mov.b64 %0, %0;" : "+l"(out));   // opaque base: one IMAD.WIDE per record address
        uint32_t pre = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            st_rec_if(h[i], out + (pre + __popc(hm[i] & lt)), r[i]);
            pre += __popc(hm[i]);
        }
    } else {
        uint4 *out = reinterpret_cast<uint4 *>(o.buf) + base;
        uint32_t pre = used;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const uint32_t slot = pre + __popc(hm[i] & lt);
            if (h[i]) {
                if (!full && slot < size) {
                    out[slot] = make_uint4(r[i].qid, r[i].eid, __float_as_uint(r[i].t_in), __float_as_uint(r[i].t_out));
                } else {
                    o.redo[r[i].qid] = 1;
                    atomicAdd(&o.st->dropped, 1ull);
                }
            }
            pre += __popc(hm[i]);
        }
    }
    if (!full) used = min(used + k, size);
    __syncwarp();
    if (lane == 0) { W.ap_base = base; W.ap_used = used; W.ap_size = size; W.ap_full = full; }
    __syncwarp();
}

template <bool EXACT>
__device__ __forceinline__ void append2(const OutArgs &o, WarpState &W, bool ha, bool hb, unsigned hma, unsigned hmb,
                                        const Rec &ra, const Rec &rb, int lane) {
    const bool h[2] = {ha, hb};
    const unsigned hm[2] = {hma, hmb};
    const Rec r[2] = {ra, rb};
    appendK<EXACT, 2>(o, W, h, hm, r, lane);
}

template <bool EXACT>
__device__ __forceinline__ void warp_state_finish(const OutArgs &o, WarpState &W, int lane) {
    __syncwarp();
    if (lane == 0) {
        if (!EXACT && !W.ap_full && W.ap_size) o.chunk_used[W.ap_base >> o.cs_shift] = W.ap_used;
        if (W.refined) atomicAdd(&o.st->refined, (unsigned long long)W.refined);
        if (W.r32) atomicAdd(&o.st->refined32, (unsigned long long)W.r32);
        if (W.hits) atomicAdd(&o.st->hits, (unsigned long long)W.hits);
    }
}

struct PairCtx {                     // what the fp64 path needs
    const float4 *Q;                 // queries (original rows)
    const float4 *rec;               // sorted entries
    const uint32_t *perm;            // sorted position -> entry row
    float d, T0, T1;                 // d: the threshold rounded up to float (fp32 paths)
    OutArgs o;
    double d64;                      // the caller's threshold (fp64 path)
    float dlo;                       // d rounded down to float (certain-hit tests of refine_rel)
    float d2h, d2l;                  // d^2 = d2h + d2l (fp32 head and the rounded remainder: refine_rel roots)
};

// Evaluate queued pairs 0..n-1 in fp64 (lane k takes pair k) and append the hits.
// Out of line: called once per 32 queued pairs from several sites of the pair
// kernels; inlining it (and pair64) at each site bloated the kernels past the
// instruction cache (ncu: no_instruction stalls on output-bound searches).
// Evaluate the first n (<= 32) pairs of the fp64 queue (lane k takes pair k, all
// lanes busy) and append the hits; the rest moves to the front.
template <bool EXACT>
__device__ __forceinline__ void flush64(const PairCtx *C, WarpState *W, uint32_t n) {
    const int lane = threadIdx.x & 31;
    const bool v = (uint32_t)lane < n;
    const uint32_t q = v ? W->fq[lane] : 0u, j = v ? W->fj[lane] : 0u;
    const uint32_t fn = W->fn;
    const uint32_t t1 = (uint32_t)lane + n < fn ? W->fq[n + lane] : 0u;
    const uint32_t t2 = (uint32_t)lane + n < fn ? W->fj[n + lane] : 0u;
    __syncwarp();
    if ((uint32_t)lane + n < fn) { W->fq[lane] = t1; W->fj[lane] = t2; }
    float tin = 0.f, tout = 0.f;
    bool hit = false;
    if (v) {
        hit = pair64(__ldg(C->Q + 2 * (uint64_t)q), __ldg(C->Q + 2 * (uint64_t)q + 1), __ldg(C->rec + 2 * (uint64_t)j),
                     __ldg(C->rec + 2 * (uint64_t)j + 1), C->d64, (double)C->T0, (double)C->T1, tin, tout);
    }
    const uint32_t eid = hit ? __ldg(C->perm + j) : 0u;
    Rec r{q, eid, tin, tout};
    append<EXACT>(C->o, *W, hit, r, lane);
    const unsigned hm = __ballot_sync(FULL, hit);
    if (hit) {   // per-query counts, aggregated over the lanes of the same query
        const unsigned peers = __match_any_sync(hm, q);
        if ((peers & ((1u << lane) - 1u)) == 0) atomicAdd(&C->o.qcount[q], (uint32_t)__popc(peers));
    }
    __syncwarp();
    if (lane == 0) { W->refined += n; W->hits += __popc(hm); W->fn = fn - n; }
    __syncwarp();
}

// warp-wide: queue four candidate slots at once (branch-free; the queue holds
// < 32 entries before, so at most 32 + 4 x 32 after, within RQ_CAP)
__device__ __forceinline__ void queue_add4(WarpState &W, uint32_t &qn, bool m0, bool m1, bool m2, bool m3,
                                           uint32_t qid, uint32_t j0, uint32_t j1, uint32_t j2, uint32_t j3,
                                           int lane) {
    const unsigned b0 = __ballot_sync(FULL, m0), b1 = __ballot_sync(FULL, m1);
    const unsigned b2 = __ballot_sync(FULL, m2), b3 = __ballot_sync(FULL, m3);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t p = qn;
    if (m0) W.rq[p + __popc(b0 & lt)] = (uint16_t)(qid | (j0 << 5));
    p += __popc(b0);
    if (m1) W.rq[p + __popc(b1 & lt)] = (uint16_t)(qid | (j1 << 5));
    p += __popc(b1);
    if (m2) W.rq[p + __popc(b2 & lt)] = (uint16_t)(qid | (j2 << 5));
    p += __popc(b2);
    if (m3) W.rq[p + __popc(b3 & lt)] = (uint16_t)(qid | (j3 << 5));
    qn = p + __popc(b3);
}

struct SchedArgs {
    const float4 *Q;
    const uint32_t *order;           // t_start-sorted query rows (or a redo list)
    uint32_t nq;
    float d, T0, T1;
    int m, v;
    const uint32_t *bin_off;
    const float *bin_lo, *bin_pmhi;
    const uint32_t *st_off0, *st_off1, *st_off2;
    float st_o[3], st_w[3];
    int use_st;
    Sched *out;
    uint32_t *keys;                  // sort keys: category << 13 | lo >> lo_shift (16 bits)
    uint32_t *vals;                  // identity (sort payload)
    int lo_shift;
    float mo[3], mw[3];              // Morton grid (1024 cells per dimension over D's extent)
    int count_t;                     // TDS_AUTO: also sum the temporal ranges (pair_tests_t)
    const float4 *rec;               // sorted entries (tight ranges)
    int tight;                       // trim the bin hull to entry-exact ends
    DevStats *st;
};

// first j in [0, m) with a[j] > x (a non-decreasing); m if none
__device__ __forceinline__ int upper_bound_f(const float *a, int m, float x) {
    int lo = 0, hi = m;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}
// first j with a[j] >= x
__device__ __forceinline__ int lower_bound_f(const float *a, int m, float x) {
    int lo = 0, hi = m;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] >= x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__global__ void k_schedule(SchedArgs A) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long work = 0, fb = 0, work_t = 0;
    if (p < A.nq) {
        uint32_t k = A.order ? A.order[p] : p;
        float4 a = A.Q[2 * (uint64_t)k], b = A.Q[2 * (uint64_t)k + 1];
        const bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w) && isfinite(b.x) &&
                        isfinite(b.y) && isfinite(b.z) && isfinite(b.w) && (b.w > a.w);
        if (!ok) atomicMax(&A.st->bad, ~(unsigned long long)k);
        float t0c = fmaxf(a.w, A.T0), t1c = fminf(b.w, A.T1);
        Sched S{k, 0u, 0u, 3};
        if (t0c < t1c) {
            // temporal bins overlapping (t0c, t1c): strict member-extent tests (C13)
            int jlo = upper_bound_f(A.bin_pmhi, A.m, t0c);     // first bin with PMhi > t0c
            int jhe = lower_bound_f(A.bin_lo, A.m, t1c);       // first bin with lo >= t1c
            if (jlo < jhe) {
                S.lo = A.bin_off[jlo];
                S.hi = A.bin_off[jhe];
                if (A.tight && S.lo < S.hi) {
                    // entry-exact ends (bin-free tight range).  hi: only bin
                    // jhe-1 can hold entries with t_start >= t1c (every earlier bin ends
                    // before the next bin's first t_start < t1c); t_start is sorted, so a
                    // binary search there gives the first one.  lo: the prefix max of t_end
                    // before bin jlo is <= t0c, so entries of bin jlo are skipped while
                    // their own t_end <= t0c (at most 64 tested; the skipped ones cannot
                    // overlap under C5, so stopping early stays complete).
                    uint32_t b = max(S.lo, A.bin_off[jhe - 1]), e = S.hi;
                    while (b < e) {
                        const uint32_t mid = (b + e) >> 1;
                        if (__ldg(&A.rec[2 * (uint64_t)mid].w) < t1c) b = mid + 1; else e = mid;
                    }
                    S.hi = b;
                    const uint32_t cap = min(S.hi, S.lo + 64u);
                    uint32_t l = S.lo;
                    while (l < cap && !(__ldg(&A.rec[2 * (uint64_t)l + 1].w) > t0c)) ++l;
                    S.lo = l;
                    if (S.lo > S.hi) S.lo = S.hi;
                }
                S.sel = S.lo < S.hi ? -1 : 3;
                work_t = S.hi - S.lo;
                if (A.use_st && S.sel == -1) {
                    // per dimension, the subbins (slabs) the d-inflated MBB
                    // overlaps; a dimension is usable only with a single slab
                    float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
                    const uint32_t *offs[3] = {A.st_off0, A.st_off1, A.st_off2};
                    uint32_t best = 0xffffffffu;
                    for (int c = 0; c < 3; ++c) {
                        float lo = __fsub_rd(fminf(p0[c], p1[c]), A.d);
                        float hi = __fadd_ru(fmaxf(p0[c], p1[c]), A.d);
                        int s0 = cell_of(lo, A.st_o[c], A.st_w[c], A.v);
                        int s1 = cell_of(hi, A.st_o[c], A.st_w[c], A.v);
                        if (s0 != s1) continue;
                        uint32_t r0 = offs[c][(uint64_t)s0 * A.m + jlo];
                        uint32_t r1 = offs[c][(uint64_t)s0 * A.m + jhe];
                        if (r1 - r0 < best) {               // ties -> lowest dimension (C15)
                            best = r1 - r0;
                            S.sel = c;
                            S.lo = r0;
                            S.hi = r1;
                        }
                    }
                    if (S.sel == -1) fb = 1;
                    if (S.lo >= S.hi) S.sel = 3;
                }
                if (S.sel == 3) { S.lo = S.hi = 0; }
                work = S.hi - S.lo;
            }
        }
        A.out[p] = S;
        // sort key: category, range start (top 13 bits), then the Morton code of the
        // query's start cell (top 16 of 30 bits): the groups of 32 consecutive
        // entries are then compact in space as well, which the window boxes exploit
        const uint32_t mx = (uint32_t)cell_of(a.x, A.mo[0], A.mw[0], 1024),
                       my = (uint32_t)cell_of(a.y, A.mo[1], A.mw[1], 1024),
                       mz = (uint32_t)cell_of(a.z, A.mo[2], A.mw[2], 1024);
        const uint32_t mort = (spread3(mx) << 2) | (spread3(my) << 1) | spread3(mz);
        A.keys[p] = ((uint32_t)(S.sel + 1) << 29) | ((S.lo >> A.lo_shift) << 16) | (mort >> 14);
        A.vals[p] = p;
        atomicAdd(&A.st->cat_cnt[S.sel + 1], 1u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        work += __shfl_xor_sync(FULL, work, o);
        fb += __shfl_xor_sync(FULL, fb, o);
        work_t += __shfl_xor_sync(FULL, work_t, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (work) atomicAdd(&A.st->pair_tests, work);
        if (fb) atomicAdd(&A.st->fallback, fb);
        if (A.count_t && work_t) atomicAdd(&A.st->pair_tests_t, work_t);
    }
}

__global__ void k_permute_sched(const Sched *__restrict__ in, const uint32_t *__restrict__ idx, uint32_t n,
                                Sched *__restrict__ out) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = in[idx[p]];
}

// tiles: runs of <= 32 consecutive schedule entries within one category
__global__ void k_make_tiles(const Sched *__restrict__ S, uint32_t n_base, uint32_t n_total_entries,
                             DevStats *__restrict__ st_w, uint32_t range_lo, uint32_t range_hi,
                             Tile *__restrict__ tiles, uint32_t max_tiles, uint32_t *__restrict__ nchunk_len,
                             int part_range) {
    const DevStats *st = st_w;
    if (part_range) { range_lo = st->part_lo; range_hi = st->part_hi; }   // tds_search_part
    // one warp per tile slot; the tile layout is derived from the category counts
    uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (t >= max_tiles) return;
    // category boundaries among entries [range_lo, range_hi) of the sorted schedule
    uint32_t start[6];
    start[0] = 0;
    for (int c = 0; c < 5; ++c) start[c + 1] = start[c] + st->cat_cnt[c];
    (void)n_base; (void)n_total_entries;
    // tiles per category (only categories 0..3 carry work; empties are skipped)
    uint32_t tb = 0, te = 0;
    int sel = 3;
    uint32_t acc = 0;
    bool found = false;
    for (int c = 0; c < 4 && !found; ++c) {
        uint32_t a = max(start[c], range_lo), b = min(start[c + 1], range_hi);
        uint32_t cnt = b > a ? b - a : 0;
        uint32_t nt = (cnt + 31) / 32;
        if (t < acc + nt) {
            tb = a + 32 * (t - acc);
            te = min(tb + 32, b);
            sel = c - 1;
            found = true;
        }
        acc += nt;
    }
    Tile T{0, 0, 0, 0, 3, {0, 0, 0}};
    if (found) {
        uint32_t lo = 0xffffffffu, hi = 0;
        uint32_t p = tb + lane;
        if (p < te) {
            Sched e = S[p];
            if (e.lo < e.hi) { lo = e.lo; hi = e.hi; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(FULL, lo, o));
            hi = max(hi, __shfl_xor_sync(FULL, hi, o));
        }
        T.tb = tb; T.te = te; T.sel = sel;
        // union start aligned down to a window (WIN): the kernel's windows are the
        // index's window-box windows (the slots' own ranges mask the extra candidates)
        if (lo < hi) { T.ulo = lo & ~(WIN - 1); T.uhi = hi; } else { T.ulo = T.uhi = 0; }
    }
    if (lane == 0) {
        tiles[t] = T;
        nchunk_len[t] = T.uhi - T.ulo;
        if (T.uhi > T.ulo) atomicAdd(&st_w->union_total, (unsigned long long)(T.uhi - T.ulo));
        if (t == max_tiles - 1) nchunk_len[max_tiles] = 0;
    }
}

// chunk size from the total union length, then chunks per tile
__global__ void k_tile_chunks(uint32_t *len_to_chunks, uint32_t ntiles, const unsigned long long *total_len,
                              DevStats *st, uint32_t target_items) {
    unsigned long long tl = *total_len;
    unsigned long long ch = (tl + target_items - 1) / (target_items ? target_items : 1);
    ch = ch < WIN ? WIN : ch;                 // items <= target_items + ntiles (the item -> tile map)
    ch = (ch + WIN - 1) / WIN * WIN;          // chunks of whole windows
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) st->ch = (uint32_t)ch;
    if (t < ntiles) len_to_chunks[t] = (uint32_t)((len_to_chunks[t] + ch - 1) / ch);
}

// item -> tile map (one warp per tile fills its items): the pair kernel finds an
// item's tile with one load instead of a binary search over item_start
__global__ void k_item_tiles(const uint32_t *__restrict__ item_start, uint32_t ntiles, uint32_t *__restrict__ item_tile,
                             uint32_t cap) {
    const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= ntiles) return;
    const uint32_t a = item_start[t], b = min(item_start[t + 1], cap);
    for (uint32_t i = a + lane; i < b; i += 32) item_tile[i] = t;
}

// ---------------------------------------------------------------------------
// A8: pair kernel for GPUTemporal / GPUSpatioTemporal (Alg. 2 / Alg. 3)
// ---------------------------------------------------------------------------
struct RangeArgs {
    PairCtx pc;                      // Q, rec, perm, d, window, output
    const uint32_t *arr[3];          // X, Y, Z
    const float4 *srec[3];           // records in X/Y/Z order (null: gather rec[X[i]])
    const Sched *sched;
    const Tile *tiles;
    const uint32_t *item_start;      // [ntiles+1]
    const uint32_t *item_tile;       // [items] tile of each work item
    uint32_t ntiles;
    float df;                        // filter_abs threshold: d * (1 + 2^-20), rounded up
    float d2u;                       // d^2 rounded up (window-box distance test)
    float tc;                        // filter_abs time origin (middle of the index's time extent)
    // GPUSpatial through this kernel (entries = (query, FSG cell) slices of the
    // cell-ordered record copy): per entry its cell and the query box's low corner
    // (packed), per candidate the min cell of its MBB; null for the range variants
    const uint32_t *sp_cell, *sp_qlo, *ecell;
    // window boxes of the candidate order: [0] the sorted (GPUSpatial: cell-ordered)
    // records, [1 + c] X/Y/Z order (tile category sel = c)
    const float4 *wb[4];
    int static_ok;                   // stationary-query filter allowed (default; TDS_NO_STATIC=1: off)
    int hyst_hi, hyst_lo;            // dense-window hysteresis, % of a window's evaluated pairs passing
    int start_dense;                 // every work item starts with a dense window (hit-heavy search)
};

// GPUSpatial duplicate avoidance (replaces the host filter of P:558-559): a pair
// (q, e) is tested only in the first cell (index-space min corner) of
// cells(e) ∩ cells(q), i.e. the cell max(min cell of e, low corner of q's box)
__device__ __forceinline__ bool ref_cell(uint32_t m0, uint32_t qlo, uint32_t cell) {
    const uint32_t rx = max(m0 >> 21, qlo >> 21), ry = max((m0 >> 10) & 0x7ffu, (qlo >> 10) & 0x7ffu),
                   rz = max(m0 & 0x3ffu, qlo & 0x3ffu);
    return ((rx << 21) | (ry << 10) | rz) == cell;
}

// threshold of filter_abs: d (already rounded up) times 1 + 2^-20, rounded up,
// so the rounding of thr and thr^2 never turns a pass into a reject
inline float time_origin(const tds_index_s *idx) {
    return (float)(0.5 * ((double)idx->ext.t_min + (double)idx->ext.t_max));
}

inline float filter_threshold(float d) {
    float df = (float)((double)d * (1.0 + 0x1p-20));
    if ((double)df < (double)d * (1.0 + 0x1p-20)) df = nextafterf(df, INFINITY);
    return df;
}

// Result-size probe of a range search (per search, before the pair kernel): the
// fraction of filter passes on sampled schedule entries (one warp each, spread
// over the sorted schedule) x 128 candidates from the middle of their ranges,
// with the relative-form filter; sizes the automatic pass buffer.
__global__ void k_density_probe(const Sched *__restrict__ S, uint32_t n, const float4 *__restrict__ Q,
                                const float4 *__restrict__ rec, const uint32_t *__restrict__ arr0,
                                const uint32_t *__restrict__ arr1, const uint32_t *__restrict__ arr2, float d, float T0,
                                float T1, const uint32_t *__restrict__ ecell, const uint32_t *__restrict__ sp_cell,
                                const uint32_t *__restrict__ sp_qlo, DevStats *st) {
    const int lane = threadIdx.x & 31;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    if (n == 0) return;
    const uint32_t p = (uint32_t)(((uint64_t)w * n) / nw + n / (2 * nw));
    if (p >= n) return;
    const Sched e = S[p];
    if (lane == 0) atomicAdd(&st->probe_entries, 1u);   // every sampled entry (empty ones estimate 0)
    if (e.sel == 3 || e.hi <= e.lo) return;
    const uint32_t *arr = e.sel == 0 ? arr0 : e.sel == 1 ? arr1 : e.sel == 2 ? arr2 : nullptr;
    const QConst qc = make_qconst(__ldg(Q + 2 * (uint64_t)e.qid), __ldg(Q + 2 * (uint64_t)e.qid + 1), T0, T1);
    const float4 q0 = make_float4(qc.px, qc.py, qc.pz, qc.t0), q1 = make_float4(qc.vx, qc.vy, qc.vz, qc.ext);
    const uint32_t len = e.hi - e.lo, m = min(len, 128u);
    uint32_t pass = 0;
    for (uint32_t k = lane; k < m; k += 32) {
        // spread over the whole range (a contiguous block of an id-ordered range
        // can be unrepresentative, e.g. the boundary between two clusters)
        const uint32_t c = e.lo + (uint32_t)(((uint64_t)k * len) / m), j = arr ? __ldg(arr + c) : c;
        const ECand ec = make_ecand(__ldg(rec + 2 * (uint64_t)j), __ldg(rec + 2 * (uint64_t)j + 1));
        const bool ref = !ecell || ref_cell(__ldg(ecell + j), sp_qlo[p], sp_cell[p]);   // GPUSpatial: no duplicates
        pass += (ref && filter_pair(q0, q1, qc.t0c, qc.t1c, ec, d)) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pass += __shfl_xor_sync(FULL, pass, o);
    if (lane == 0) {
        atomicAdd(&st->probe_pass, pass);
        atomicAdd(&st->probe_total, m);
        atomicAdd(&st->probe_est, (double)len * pass / m);   // this entry's estimated records
    }
}

struct __align__(16) RangeWarpSmem {
    float4 q[32][6];                 // group query slot g: (p0, t0) (v, |v|_1) (t0c, t1c, |p1 - p0|_1, -)
                                     // and the absolute form (c, m) (v, t0c') (t1c', lo, hi, qid)
    WarpState ws;                    // append chunk, refine queue (slot g, sorted position j), fp64 queue
    uint32_t cnt[32];                // records of slot g found by the refine path in this work item
    struct __align__(16) Cand {      // the window's candidates (slot = lane + 32 k), relative form
        float4 p;                    // (x0, y0, z0, t0)
        float4 v;                    // (vx, vy, vz, t1)
        uint4 id;                    // (entry row, sorted / cell-ordered position j, min cell, -)
    } cw[WIN];
    uint32_t spc[32], spq[32];       // GPUSpatial: cell and query-box low corner of slot g
    float4 qb[32][2];                // slot g's segment MBB and clipped span: (lo, t0c) (hi, t1c)
    uint32_t qn;                     // refine queue fill
};

// Evaluate refine-queue entries [base, base + n), n <= 32 (lane k takes entry
// k): (slot g, sorted entry position j) -> refine_rel with the query's terms from
// shared memory; certain hits are appended, undecided pairs go to the fp64 queue.
template <bool EXACT, bool SPATIAL>
__device__ __noinline__ void range_refine(const RangeArgs *A, RangeWarpSmem *W, uint32_t n, uint32_t base) {
    const int lane = threadIdx.x & 31;
    const bool v = (uint32_t)lane < n;
    const uint32_t e = v ? W->ws.rq[base + lane] : 0u, g = e & 31u, slot = e >> 5;
    __syncwarp();                    // queue slots read: later queue additions may reuse them
    float tin = 0.f, tout = 0.f;
    int k = 0;
    uint32_t qid = 0;
    const uint4 id = W->cw[slot].id;  // (entry row, position j, min cell)
    if (v) {
        const float4 q0 = W->q[g][0], q1 = W->q[g][1], q2 = W->q[g][2];
        qid = __float_as_uint(W->q[g][5].w);
        if (!SPATIAL || ref_cell(id.z, W->spq[g], W->spc[g])) {
            const float4 ep = W->cw[slot].p;
            const float4 ev = W->cw[slot].v;
            k = refine_rel(q0, q1, q2.x, q2.y, ep, ev.w, ev.x, ev.y, ev.z, A->pc.dlo, A->pc.d, A->pc.d2h, A->pc.d2l,
                           tin, tout);
        }
    }
    const uint32_t j = id.y;
    const bool hit = (k == 2), need64 = (k == 1);
    const Rec r{qid, hit ? id.x : 0u, tin, tout};
    append<EXACT>(A->pc.o, W->ws, hit, r, lane);
    if (hit) atomicAdd(&W->cnt[g], 1u);
    const unsigned hm = __ballot_sync(FULL, hit), m64 = __ballot_sync(FULL, need64);
    const uint32_t fn = W->ws.fn;
    if (need64) {
        const uint32_t pos = fn + __popc(m64 & ((1u << lane) - 1u));
        W->ws.fq[pos] = qid;
        W->ws.fj[pos] = j;
    }
    __syncwarp();
    if (lane == 0) { W->ws.hits += __popc(hm); W->ws.fn = fn + __popc(m64); W->ws.r32 += n; }
    __syncwarp();
    if (fn + __popc(m64) >= 32) flush64<EXACT>(&A->pc, &W->ws, 32);
}

// warp-wide: evaluate the newest 32 queued pairs while >= 32 are queued
template <bool EXACT, bool SPATIAL>
__device__ __forceinline__ void range_drain(const RangeArgs *A, RangeWarpSmem &W, uint32_t &qn) {
    while (qn >= 32) {
        __syncwarp();
        qn -= 32;
        range_refine<EXACT, SPATIAL>(A, &W, 32, qn);
    }
}

// Mapping: a work item is a group of <= 32
// consecutive schedule entries (one category) and a chunk of the union of their
// candidate ranges.  Lane g owns query slot g of the group (its constants are
// staged in shared memory); the warp walks the chunk 128 candidates at a time
// with lane = candidate (4 per lane).  A ballot over the owners gives the
// queries whose range meets the window, so each loaded candidate is tested
// against every query that needs it and gaps between ranges are skipped.
// Sparse windows: the absolute-form filter (packed, two chains); passes are
// queued (slot, candidate) and evaluated 32 at a time by range_refine.  Dense
// windows (hysteresis on the window's pass fraction): the fused relative-form
// step dense_test2 appends whole-span hits at once and queues the rest.
template <bool EXACT, bool STATIC, bool SPATIAL, bool SPARSE>
#ifdef TDS_RANGE_MAXNREG
__global__ void __maxnreg__(TDS_RANGE_MAXNREG) k_pair_range(
#else
__global__ void __launch_bounds__(PT, RANGE_BPS) k_pair_range(
#endif
    const __grid_constant__ RangeArgs A) {
    extern __shared__ __align__(16) unsigned char range_smem[];     // PT / 32 x RangeWarpSmem (> 48 KB)
    const int lane = threadIdx.x & 31;
    RangeWarpSmem &W = reinterpret_cast<RangeWarpSmem *>(range_smem)[threadIdx.x >> 5];
    DevStats *st = A.pc.o.st;
    const uint32_t total = A.item_start[A.ntiles];
    const uint32_t CH = st->ch;
    const float df = A.df;
    warp_state_init(W.ws, lane);
    W.cnt[lane] = 0;
    uint32_t qn = 0;                         // refine queue fill (warp-uniform)
    __syncwarp();
    uint32_t direct_hits = 0;               // per work item (added to the warp's total at the item end)
    bool dense = false;                      // warp-uniform: the last window was hit-heavy
    while (true) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(&st->work_ctr, 1u);
        item = __shfl_sync(FULL, item, 0);
        if (item >= total) break;
        const uint32_t lo = A.item_tile[item];
        const Tile T = A.tiles[lo];
        const uint32_t chunk = item - A.item_start[lo];
        if (A.start_dense) dense = true;     // hit-heavy search (probe): every item starts dense
        const uint32_t c_lo = T.ulo + chunk * CH;
        const uint32_t c_hi = min(c_lo + CH, T.uhi);
        // ---- owner side: lane g stages query slot g of the group
        const uint32_t p = T.tb + lane;
        const bool active = p < T.te;
        Sched S{0, 0, 0, 3};
        if (active) S = A.sched[p];
        uint32_t my_lo = max(S.lo, c_lo), my_hi = min(S.hi, c_hi);
        if (!active || my_lo >= my_hi) { my_lo = 0xffffffffu; my_hi = 0; }
        {
            float4 qa = make_float4(0.f, 0.f, 0.f, 0.f), qb = make_float4(0.f, 0.f, 0.f, 1.f);
            if (active) { qa = __ldg(A.pc.Q + 2 * (uint64_t)S.qid); qb = __ldg(A.pc.Q + 2 * (uint64_t)S.qid + 1); }
            const QConst qc = make_qconst(qa, qb, A.pc.T0, A.pc.T1);
            const FSeg qf = make_fseg(qa, qb, A.tc);
            __syncwarp();
            W.q[lane][0] = make_float4(qc.px, qc.py, qc.pz, qc.t0);
            W.q[lane][1] = make_float4(qc.vx, qc.vy, qc.vz, fabsf(qc.vx) + fabsf(qc.vy) + fabsf(qc.vz));
            W.q[lane][2] = make_float4(qc.t0c, qc.t1c, qc.ext, 0.f);
            W.q[lane][3] = make_float4(qf.cx, qf.cy, qf.cz, qf.m);
            W.q[lane][4] = make_float4(qf.vx, qf.vy, qf.vz, qc.t0c - A.tc);
            W.q[lane][5] = make_float4(qc.t1c - A.tc, __uint_as_float(my_lo), __uint_as_float(my_hi),
                                       __uint_as_float(S.qid));
            if (SPATIAL) {
                W.spc[lane] = active ? A.sp_cell[p] : 0xffffffffu;
                W.spq[lane] = active ? A.sp_qlo[p] : 0u;
            }
            W.qb[lane][0] = make_float4(fminf(qa.x, qb.x), fminf(qa.y, qb.y), fminf(qa.z, qb.z), qc.t0c);
            W.qb[lane][1] = make_float4(fmaxf(qa.x, qb.x), fmaxf(qa.y, qb.y), fmaxf(qa.z, qb.z), qc.t1c);
            __syncwarp();
        }
        uint32_t wlo = my_lo, whi = my_hi;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wlo = min(wlo, __shfl_xor_sync(FULL, wlo, o));
            whi = max(whi, __shfl_xor_sync(FULL, whi, o));
        }
        // every query of the group stationary (P1 = P0): the sparse windows use
        // filter_static2 (TDS_NO_STATIC=1 disables it, for the A/B)
        bool stat = false;
        {
            const bool st_q = !active || (__float_as_uint(W.q[lane][1].w) == 0u);   // |v|_1 == +0
            stat = STATIC && A.static_ok && __all_sync(FULL, st_q);
        }
        const uint32_t *arr = (T.sel >= 0) ? A.arr[T.sel] : nullptr;
        uint32_t owner_hits = 0;             // whole-span hits of this lane's query slot (dense path)
        // records: sorted entries (temporal), the materialised X/Y/Z-ordered copy
        // (TDS_ST_MATERIALISE=1: streamed, independent of the id load), or rec[X[i]]
        const float4 *srec = (T.sel >= 0) ? A.srec[T.sel] : nullptr;
        auto load_cand = [&](uint32_t c, bool v, uint32_t &j, float4 &a, float4 &b) {
            j = 0;
            a = make_float4(0.f, 0.f, 0.f, 0.f);
            b = make_float4(0.f, 0.f, 0.f, 1.f);
            if (v) {
                j = arr ? __ldg(arr + c) : c;
                const float4 *src = srec ? srec + 2 * (uint64_t)c : A.pc.rec + 2 * (uint64_t)j;
                a = __ldg(src);
                b = __ldg(src + 1);
            }
        };
        const float4 *wbt = A.wb[T.sel + 1];
        uint32_t base = wlo & ~(WIN - 1);      // windows aligned with the index's window boxes
        while (base < whi) {
            const uint32_t cend = min(base + WIN, whi);
            unsigned mask = __ballot_sync(FULL, my_lo < cend && my_hi > base);
            if (!mask) {                       // skip the gap to the next range start
                uint32_t nxt = (my_lo >= cend && my_lo < my_hi) ? my_lo : 0xffffffffu;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) nxt = min(nxt, __shfl_xor_sync(FULL, nxt, o));
                if (nxt == 0xffffffffu) break;
                base = nxt & ~(WIN - 1);
                continue;
            }
            // window box (built with the index): a pair within d at time t has
            // P_q(t) in the query segment's MBB and P_e(t) in the window box, so a
            // query whose MBB is farther than d from the box (Euclidean box-box
            // distance, gaps and squares rounded down, compared with d^2 rounded
            // up), or whose window-clipped span misses the box's time span (C5), has
            // no pair in the window; if no query is left the window is never loaded
            {
                const float4 *wp = wbt + 2 * (size_t)(base / WIN);
                const float4 bl = __ldg(wp), bh = __ldg(wp + 1);
                const float4 ql = W.qb[lane][0], qh = W.qb[lane][1];
                const float gx = fmaxf(0.f, fmaxf(__fsub_rd(ql.x, bh.x), __fsub_rd(bl.x, qh.x)));
                const float gy = fmaxf(0.f, fmaxf(__fsub_rd(ql.y, bh.y), __fsub_rd(bl.y, qh.y)));
                const float gz = fmaxf(0.f, fmaxf(__fsub_rd(ql.z, bh.z), __fsub_rd(bl.z, qh.z)));
                const float g2 = __fadd_rd(__fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)), __fmul_rd(gz, gz));
                const bool ov = ((mask >> lane) & 1u) & (g2 <= A.d2u) & (ql.w < bh.w) & (qh.w > bl.w);
                mask = __ballot_sync(FULL, ov);
            }
            if (!mask) { base = cend; continue; }
            const unsigned mask_eval = mask;   // queries evaluated in this window
            const uint32_t wn = cend - max(base, wlo);   // candidates of the window inside the union
            if (lane == 0) W.ws.exec += (unsigned long long)wn * __popc(mask);   // stats: executed pair tests
            // ---- worker side: lane = candidate
            const uint32_t c0 = base + lane, c1 = c0 + 32, c2 = c0 + 64, c3 = c0 + 96;
            uint32_t j0, j1, j2, j3;
            uint32_t wpass = 0;                // filter passes of this window (all queries)
            // ---- the window: the lane's four candidates as absolute-form filter terms
            // (registers, two packed pairs) and in the relative form with their rows
            // (shared memory slots lane + 32 k, read by the refine step)
            FSeg2 f01, f23;
            {
                auto stage = [&](int k, uint32_t c, uint32_t j, float4 a, float4 b, const FSeg &f) {
                    const bool v = c < cend;
                    RangeWarpSmem::Cand &cd = W.cw[lane + 32 * k];
                    cd.p = a;
                    cd.v = make_float4(f.vx, f.vy, f.vz, b.w);        // make_ecand's velocity (same rcp)
                    cd.id = make_uint4(v ? __ldg(A.pc.perm + j) : 0u, j, (SPATIAL && v) ? __ldg(A.ecell + j) : 0u, 0u);
                };
                float4 a0, b0, a1, b1;
                load_cand(c0, c0 < cend, j0, a0, b0);
                load_cand(c1, c1 < cend, j1, a1, b1);
                {
                    const FSeg fa = make_fseg(a0, b0, A.tc), fb = make_fseg(a1, b1, A.tc);
                    f01 = make_fseg2(fa, fb);
                    stage(0, c0, j0, a0, b0, fa);
                    stage(1, c1, j1, a1, b1, fb);
                }
                load_cand(c2, c2 < cend, j2, a0, b0);
                load_cand(c3, c3 < cend, j3, a1, b1);
                {
                    const FSeg fa = make_fseg(a0, b0, A.tc), fb = make_fseg(a1, b1, A.tc);
                    f23 = make_fseg2(fa, fb);
                    stage(2, c2, j2, a0, b0, fa);
                    stage(3, c3, j3, a1, b1, fb);
                }
                __syncwarp();
            }
            const uint32_t s0 = lane, s1 = lane + 32, s2 = lane + 64, s3 = lane + 96;   // window slots
            if (!SPARSE && dense) {
                // fused step: the filter and the whole-span test for the lane's four
                // candidates (two packed pairs); whole-span hits are appended at once
                // with [a, b] from the raw times, other passes go to the refine queue
                while (mask) {
                    const int g = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const float4 n0 = W.q[g][3], n1 = W.q[g][4], n2 = W.q[g][5];
                    const uint32_t glo = __float_as_uint(n2.y), ghi = __float_as_uint(n2.z);
                    const float qin = fmaf(-KU, n0.w, A.pc.dlo);
                    bool m[4], in[4];
                    filter_abs2x(n0, n1, n1.w, n2.x, qin, f01, df, m[0], m[1], in[0], in[1]);
                    filter_abs2x(n0, n1, n1.w, n2.x, qin, f23, df, m[2], m[3], in[2], in[3]);
                    if (glo > base || ghi - base < WIN) {    // slots outside the query's range
                        const uint32_t r0 = c0 - glo, gw = ghi - glo;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const bool ok = r0 + 32u * k < gw;
                            m[k] &= ok;
                            in[k] &= ok;
                        }
                    }
                    if (SPATIAL) {                         // GPUSpatial: the pair's reference cell only
                        const uint32_t sq = W.spq[g], sc = W.spc[g];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const bool ok = ref_cell(W.cw[lane + 32 * k].id.z, sq, sc);
                            m[k] &= ok;
                            in[k] &= ok;
                        }
                    }
                    unsigned bi[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        m[k] &= !in[k];
                        bi[k] = __ballot_sync(FULL, in[k]);
                    }
                    const uint32_t nin = __popc(bi[0]) + __popc(bi[1]) + __popc(bi[2]) + __popc(bi[3]);
                    if (nin) {
                        const float4 q2 = W.q[g][2];
                        const uint32_t qid = __float_as_uint(n2.w);
                        Rec r[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const RangeWarpSmem::Cand &cd = W.cw[lane + 32 * k];
                            r[k] = Rec{qid, cd.id.x, fmaxf(q2.x, cd.p.w), fminf(q2.y, cd.v.w)};
                        }
                        appendK<EXACT, 4>(A.pc.o, W.ws, in, bi, r, lane);
                        direct_hits += nin;
                        if (lane == g) owner_hits += nin;
                    }
                    wpass += nin;
                    if (__any_sync(FULL, (m[0] | m[1]) | (m[2] | m[3]))) {
                        const uint32_t q0n = qn;
                        queue_add4(W.ws, qn, m[0], m[1], m[2], m[3], (uint32_t)g, s0, s1, s2, s3, lane);
                        wpass += qn - q0n;
                        range_drain<EXACT, SPATIAL>(&A, W, qn);
                    }
                }
            } else {
                f32x2 rA01 = 0ull, rA23 = 0ull;
                if (stat) { rA01 = static_rA(f01); rA23 = static_rA(f23); }
                while (mask) {
                    const int g = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const float4 n0 = W.q[g][3], n1 = W.q[g][4], n2 = W.q[g][5];
                    const uint32_t glo = __float_as_uint(n2.y), ghi = __float_as_uint(n2.z);
                    bool m0, m1, m2, m3;
                    if (stat) {
                        filter_static2(n0, n1.w, n2.x, f01, rA01, df, m0, m1);
                        filter_static2(n0, n1.w, n2.x, f23, rA23, df, m2, m3);
                    } else {
                        filter_abs2(n0, n1, n1.w, n2.x, f01, df, m0, m1);
                        filter_abs2(n0, n1, n1.w, n2.x, f23, df, m2, m3);
                    }
                    // warp-uniform: unless the query's range covers all WIN candidate slots
                    // (then all are valid: ghi <= whi), test each slot against the range
                    // (c < ghi <= whi implies c < cend: no separate validity test)
                    if (glo > base || ghi - base < WIN) {
                        const uint32_t r0 = c0 - glo, gw = ghi - glo;
                        m0 &= r0 < gw; m1 &= r0 + 32 < gw; m2 &= r0 + 64 < gw; m3 &= r0 + 96 < gw;
                    }
                    if (!__any_sync(FULL, (m0 | m1) | (m2 | m3))) continue;
                    if (SPATIAL) {                         // GPUSpatial: the pair's reference cell only
                        const uint32_t sq = W.spq[g], sc = W.spc[g];
                        m0 &= ref_cell(W.cw[s0].id.z, sq, sc);
                        m1 &= ref_cell(W.cw[s1].id.z, sq, sc);
                        m2 &= ref_cell(W.cw[s2].id.z, sq, sc);
                        m3 &= ref_cell(W.cw[s3].id.z, sq, sc);
                    }
                    const uint32_t q0n = qn;
                    queue_add4(W.ws, qn, m0, m1, m2, m3, (uint32_t)g, s0, s1, s2, s3, lane);
                    wpass += qn - q0n;
                    range_drain<EXACT, SPATIAL>(&A, W, qn);
                }
            }
            // switch to the fused dense path once >= HYST_HI % of the window's pairs pass,
            // back to the sparse path below HYST_LO % (hysteresis: a window mix near one
            // threshold would toggle between the paths)
            if (qn) {                          // the queue refers to this window's slots
                __syncwarp();
                range_refine<EXACT, SPATIAL>(&A, &W, qn, 0);
                qn = 0;
            }
            dense = 100u * wpass >= (uint32_t)(dense ? A.hyst_lo : A.hyst_hi) * __popc(mask_eval) * wn;
            base = cend;
        }
        // ---- item end: the queue refers to this group's slots
        if (qn) {
            __syncwarp();
            range_refine<EXACT, SPATIAL>(&A, &W, qn, 0);
            qn = 0;
        }
        __syncwarp();
        if (lane == 0) W.ws.direct += direct_hits;
        direct_hits = 0;
        const uint32_t cq = owner_hits + W.cnt[lane];
        W.cnt[lane] = 0;
        // an inactive slot never has a record (its mask bit is never set); its query
        // row is read back from the staged slot instead of kept in a register
        if (cq) atomicAdd(&A.pc.o.qcount[__float_as_uint(W.q[lane][5].w)], cq);
        __syncwarp();
    }
    __syncwarp();
    if (W.ws.fn) flush64<EXACT>(&A.pc, &W.ws, W.ws.fn);
    warp_state_finish<EXACT>(A.pc.o, W.ws, lane);
    if (lane == 0 && W.ws.exec) atomicAdd(&st->executed, W.ws.exec);
    if (lane == 0 && W.ws.direct) { atomicAdd(&st->hits, W.ws.direct); atomicAdd(&st->direct, W.ws.direct); }
}

// ---------------------------------------------------------------------------
// GPUSpatial (Alg. 1) work list: per query, the rows (cx, cy) of FSG cells its
// d-inflated MBB overlaps; a row's cells cz_lo..cz_hi are contiguous in the
// dense CSR, so one row is one contiguous slice of the lookup array A.
// ---------------------------------------------------------------------------
struct FsgGrid {
    float o[3], w[3];
    int g[3];
};

__device__ __forceinline__ void query_box(float4 a, float4 b, float d, const FsgGrid &G, int lo[3], int hi[3]) {
    float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        lo[c] = cell_of(__fsub_rd(fminf(p0[c], p1[c]), d), G.o[c], G.w[c], G.g[c]);
        hi[c] = cell_of(__fadd_ru(fmaxf(p0[c], p1[c]), d), G.o[c], G.w[c], G.g[c]);
    }
}

// GPUSpatial query order (a locality order only; the result set does not
// depend on it): by t_start, then by the Morton code of the start point's cell,
// so that warps working at the same time read the same (cell, time) slices and
// the slices are reused from L2.  Keys for two stable radix sorts (cell first,
// then t_start).

__global__ void k_fsg_order_keys(const float4 *__restrict__ Q, uint32_t n, FsgGrid G, uint32_t *__restrict__ kcell,
                                 uint32_t *__restrict__ kt, uint32_t *__restrict__ vals) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float4 a = Q[2 * (uint64_t)p];
    const uint32_t cx = (uint32_t)cell_of(a.x, G.o[0], G.w[0], G.g[0]), cy = (uint32_t)cell_of(a.y, G.o[1], G.w[1], G.g[1]),
                   cz = (uint32_t)cell_of(a.z, G.o[2], G.w[2], G.g[2]);
    kcell[p] = (spread3(cx) << 2) | (spread3(cy) << 1) | spread3(cz);
    kt[p] = float_key(isfinite(a.w) ? a.w : 0.f);
    vals[p] = p;
}

__global__ void k_gather_u32(const uint32_t *__restrict__ src, const uint32_t *__restrict__ idx, uint32_t n,
                             uint32_t *__restrict__ out) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = src[idx[p]];
}

// GPUSpatial schedule entries from the (query, cell) items: entry r = (query row,
// time-trimmed slice [alo, alo + len) of the cell-ordered copy), its cell and the
// query box's low corner for the reference-cell rule; sort key = slice start
// (empty slices last, key empty_key)
__global__ void k_fsg_sched(uint32_t nrows, const uint32_t *__restrict__ row_q, const uint32_t *__restrict__ row_alo,
                            const uint32_t *__restrict__ row_len, const uint32_t *__restrict__ row_cxy,
                            const int4 *__restrict__ qbox, uint32_t empty_key, Sched *__restrict__ out,
                            uint32_t *__restrict__ keys, uint32_t *__restrict__ vals, uint32_t *__restrict__ sp_cell,
                            uint32_t *__restrict__ sp_qlo, DevStats *st) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long work = 0;
    uint32_t live = 0;
    if (r < nrows) {
        const int4 lo = qbox[2 * row_q[r]];
        const uint32_t a0 = row_alo[r], len = row_len[r];
        out[r] = len ? Sched{(uint32_t)lo.w, a0, a0 + len, -1} : Sched{(uint32_t)lo.w, 0u, 0u, 3};
        keys[r] = len ? a0 : empty_key;
        vals[r] = r;
        sp_cell[r] = row_cxy[r];
        sp_qlo[r] = pack_cell(lo.x, lo.y, lo.z);
        work = len;
        live = len ? 1u : 0u;
    }
    uint32_t empty = (r < nrows) ? 1u - live : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        work += __shfl_xor_sync(FULL, work, o);
        live += __shfl_xor_sync(FULL, live, o);
        empty += __shfl_xor_sync(FULL, empty, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (work) atomicAdd(&st->pair_tests, work);
        if (live) atomicAdd(&st->cat_cnt[0], live);
        if (empty) atomicAdd(&st->cat_cnt[4], empty);
    }
}

__global__ void k_fsg_count(const float4 *__restrict__ Q, const uint32_t *__restrict__ list, uint32_t n, float d,
                            float T0, float T1, FsgGrid G, uint32_t *__restrict__ nitems, int4 *__restrict__ qbox,
                            unsigned long long *__restrict__ total, unsigned long long *__restrict__ bad) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t k = list ? list[p] : p;
    float4 a = Q[2 * (uint64_t)k], b = Q[2 * (uint64_t)k + 1];
    const bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w) && isfinite(b.x) &&
                    isfinite(b.y) && isfinite(b.z) && isfinite(b.w) && (b.w > a.w);
    if (!ok) atomicMax(bad, ~(unsigned long long)k);
    int lo[3], hi[3];
    query_box(a, b, d, G, lo, hi);
    bool live = fmaxf(a.w, T0) < fminf(b.w, T1);
    const unsigned long long cnt =
        live ? (unsigned long long)(hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1) : 0ull;
    nitems[p] = (uint32_t)min(cnt, 0xffffffffull);
    atomicAdd(total, cnt);
    qbox[2 * p] = make_int4(lo[0], lo[1], lo[2], (int)k);
    qbox[2 * p + 1] = make_int4(hi[0], hi[1], hi[2], 0);
}

// first i in [lo, hi) with t_start(i) > x (ge = false) or >= x (ge = true); the
// entries of one cell are in t_start order (stable grouping of the sorted D)
__device__ __forceinline__ uint32_t cell_time_bound(const float4 *__restrict__ frec, uint32_t lo, uint32_t hi, float x,
                                                    bool ge) {
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        float t = __ldg(&frec[2 * (uint64_t)mid].w);
        bool right = ge ? (t >= x) : (t > x);
        if (right) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// one warp per query: work items = the (query, cell) pairs of its d-inflated
// box, each a slice of the cell-ordered arrays.  Unless `literal`,
// the slice is trimmed to the entries that can overlap the query in time:
// t_start < t1q and t_start > t0q - max_dur (a time filter the paper's FSG does
// not apply; the result set is unchanged).
__global__ void k_fsg_items(const uint32_t *__restrict__ item_start, uint32_t n, const int4 *__restrict__ qbox,
                            const float4 *__restrict__ Q, FsgGrid G, const uint32_t *__restrict__ cell_off,
                            const float4 *__restrict__ frec, float T0, float T1, float max_dur, int literal,
                            uint32_t *__restrict__ item_q, uint32_t *__restrict__ item_alo,
                            uint32_t *__restrict__ item_len, uint32_t *__restrict__ item_cell) {
    const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n) return;
    const uint32_t r0 = item_start[p], r1 = item_start[p + 1];
    if (r0 == r1) return;
    const int4 lo = qbox[2 * p], hi = qbox[2 * p + 1];
    const uint32_t k = (uint32_t)lo.w;
    const float t0c = fmaxf(Q[2 * (uint64_t)k].w, T0), t1c = fminf(Q[2 * (uint64_t)k + 1].w, T1);
    const float tlo = __fsub_rd(t0c, max_dur);
    const int ny = hi.y - lo.y + 1, nz = hi.z - lo.z + 1;
    for (uint32_t c = lane; c < r1 - r0; c += 32) {
        const int z = lo.z + (int)(c % nz), y = lo.y + (int)((c / nz) % ny), x = lo.x + (int)(c / (nz * ny));
        const uint64_t h = ((uint64_t)x * G.g[1] + y) * G.g[2] + z;
        uint32_t a0 = cell_off[h], a1 = cell_off[h + 1];
        if (!literal && a0 < a1) {                 // a cell's entries are in t_start order (build)
            a1 = cell_time_bound(frec, a0, a1, t1c, true);      // first t_start >= t1c
            a0 = cell_time_bound(frec, a0, a1, tlo, false);     // first t_start > t0c - max_dur
        }
        const uint32_t r = r0 + c;
        item_q[r] = p;                        // index into the query list / qbox
        item_alo[r] = a0;
        item_len[r] = a1 > a0 ? a1 - a0 : 0u;
        item_cell[r] = pack_cell(x, y, z);
    }
}

// ---------------------------------------------------------------------------
// overflow handling (A10): keep records of complete queries, re-plan the rest
// ---------------------------------------------------------------------------
// records of each chunk of the pass buffer to keep (their query did not lose a
// record, so it is not re-run); one warp per chunk
__global__ void k_chunk_kept(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                             const uint32_t *__restrict__ chunk_used, const uint8_t *__restrict__ redo,
                             uint64_t *__restrict__ kept) {
    uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (c > nchunks) return;
    uint32_t cnt = 0;
    if (c < nchunks) {
        const uint32_t u = chunk_used[c];
        for (uint32_t k = lane; k < u; k += 32) cnt += redo[buf[c * CS + k].qid] ? 0u : 1u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    if (lane == 0) kept[c] = cnt;                 // kept[nchunks] = 0 (total after the scan)
}

// kept records straight from the chunked pass buffer into the exact store, in
// chunk order (warp per chunk; positions by ballot within the chunk)
__global__ void k_scatter_kept_chunked(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                                       const uint32_t *__restrict__ chunk_used, const uint8_t *__restrict__ redo,
                                       const uint64_t *__restrict__ kept_off, Rec *__restrict__ out) {
    uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    const uint32_t u = chunk_used[c];
    uint64_t base = kept_off[c];
    for (uint32_t k0 = 0; k0 < u; k0 += 32) {
        const uint32_t k = k0 + lane;
        Rec r{0u, 0u, 0.f, 0.f};
        bool keep = false;
        if (k < u) {
            r = buf[c * CS + k];
            keep = !redo[r.qid];
        }
        const unsigned m = __ballot_sync(FULL, keep);
        if (keep) out[base + __popc(m & ((1u << lane) - 1u))] = r;
        base += __popc(m);
    }
}

__global__ void k_flatten(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                          const uint32_t *__restrict__ chunk_used, const uint64_t *__restrict__ chunk_off,
                          Rec *__restrict__ flat) {
    uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    uint32_t u = chunk_used[c];
    uint64_t o = chunk_off[c];
    for (uint32_t k = lane; k < u; k += 32) flat[o + k] = buf[c * CS + k];
}


__global__ void k_chunk_offsets_u64(const uint32_t *__restrict__ used, uint64_t n, uint64_t *__restrict__ out) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = used[i];
}

// overflow re-plan: the schedule entries of the queries in the current batch
__global__ void k_mark_rows(const uint32_t *__restrict__ rows, uint32_t n, uint8_t *__restrict__ mark) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mark[rows[i]] = 1;
}

__global__ void k_redo_flags_sched(const Sched *__restrict__ S, uint32_t n, const uint8_t *__restrict__ inbatch,
                                   uint32_t *__restrict__ flag) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) flag[p] = (S[p].sel != 3 && inbatch[S[p].qid]) ? 1u : 0u;
}

__global__ void k_compact_sched(const Sched *__restrict__ S, uint32_t n, const uint32_t *__restrict__ flag,
                                const uint32_t *__restrict__ pos, Sched *__restrict__ out,
                                const uint32_t *__restrict__ cell, const uint32_t *__restrict__ qlo,
                                uint32_t *__restrict__ cell_out, uint32_t *__restrict__ qlo_out) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && flag[p]) {
        out[pos[p]] = S[p];
        if (cell_out) { cell_out[pos[p]] = cell[p]; qlo_out[pos[p]] = qlo[p]; }
    }
}

__global__ void k_cat_counts(const Sched *__restrict__ S, uint32_t n, DevStats *st) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) atomicAdd(&st->cat_cnt[S[p].sel + 1], 1u);
}

// ---------------------------------------------------------------------------
// A11: fetch
// ---------------------------------------------------------------------------
// one warp per chunk; each lane keeps 4 record loads in flight (16 B, streaming:
// the records are read once) and writes the four SoA columns with streaming
// stores.  FULL: the whole result is fetched (no per-record range test).
template <bool FULL>
__global__ void __launch_bounds__(256) k_fetch_chunked(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                                const uint32_t *__restrict__ used, const uint64_t *__restrict__ off, uint64_t first,
                                uint64_t count, uint32_t *qid, uint32_t *eid, float *tin, float *tout) {
    uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    const uint32_t u = used[c];
    const uint64_t o = off[c];
    if (!FULL && (o + u <= first || o >= first + count)) return;
    const uint4 *src = reinterpret_cast<const uint4 *>(buf + c * CS);
    for (uint32_t k0 = 0; k0 < u; k0 += 128) {
        uint4 r[4];
        bool v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t k = k0 + lane + 32 * i;
            v[i] = k < u;
            if (!FULL) v[i] = v[i] && o + k >= first && o + k < first + count;
            if (v[i]) r[i] = __ldcs(src + k);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!v[i]) continue;
            const uint64_t j = o + k0 + lane + 32 * i - first;
            if (qid) __stcs(qid + j, r[i].x);
            if (eid) __stcs(eid + j, r[i].y);
            if (tin) __stcs(reinterpret_cast<uint32_t *>(tin) + j, r[i].z);
            if (tout) __stcs(reinterpret_cast<uint32_t *>(tout) + j, r[i].w);
        }
    }
}

__global__ void k_fetch_flat(const Rec *__restrict__ rs, const uint32_t *__restrict__ order, uint64_t first,
                             uint64_t count, uint32_t *qid, uint32_t *eid, float *tin, float *tout) {
    uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= count) return;
    uint64_t g = first + j;
    Rec r = rs[order ? order[g] : g];
    if (qid) qid[j] = r.qid;
    if (eid) eid[j] = r.eid;
    if (tin) tin[j] = r.t_in;
    if (tout) tout[j] = r.t_out;
}

// records of one chunk's result with the chunk's first query row added to the
// query ids (tds_search_stream), from the chunked or the contiguous form
__global__ void k_pack_chunked(const Rec *__restrict__ buf, uint32_t CS, uint64_t nchunks,
                               const uint32_t *__restrict__ used, const uint64_t *__restrict__ off, uint32_t qoff,
                               Rec *__restrict__ out) {
    const uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    const uint32_t u = used[c];
    const uint64_t o = off[c];
    for (uint32_t k = lane; k < u; k += 32) {
        Rec r = buf[c * CS + k];
        r.qid += qoff;
        out[o + k] = r;
    }
}

__global__ void k_pack_flat(const Rec *__restrict__ in, uint64_t n, uint32_t qoff, Rec *__restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        Rec r = in[i];
        r.qid += qoff;
        out[i] = r;
    }
}

__global__ void k_rec_field(const Rec *__restrict__ rs, uint64_t n, int which, const uint32_t *__restrict__ order,
                            uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t src = order ? order[i] : (uint32_t)i;
    Rec r = rs[src];
    keys[i] = which == 0 ? r.qid : r.eid;
    vals[i] = src;
}

// ---------------------------------------------------------------------------
// work-balanced parts of one search (tds_search_part): part k of K
// takes the contiguous slice of the sorted schedule whose exact pair-test prefix
// sum crosses k/K and (k+1)/K of the total (prefix sum + binary search)
// ---------------------------------------------------------------------------
__global__ void k_sched_work(const Sched *__restrict__ S, uint32_t n, uint64_t *__restrict__ w) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) w[p] = S[p].sel == 3 ? 0ull : (uint64_t)(S[p].hi - S[p].lo);
    if (p == n) w[p] = 0ull;
}

// first index p in [0, n] with pre(p) >= target, pre non-decreasing
template <class F>
__device__ __forceinline__ uint32_t part_lower_bound(F pre, uint32_t n, unsigned long long target) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pre(mid) >= target) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ unsigned long long part_target(unsigned long long total, uint32_t k, uint32_t K) {
    return (unsigned long long)(((unsigned __int128)total * k) / K);
}

// range variants: pre = exclusive prefix of the sorted schedule's range lengths
__global__ void k_part_bounds(const uint64_t *__restrict__ pre, uint32_t n, uint32_t part, uint32_t nparts,
                              DevStats *st) {
    if (threadIdx.x || blockIdx.x) return;
    const unsigned long long total = pre[n];
    auto f = [&](uint32_t p) { return pre[p]; };
    const uint32_t lo = part == 0 ? 0u : part_lower_bound(f, n, part_target(total, part, nparts));
    uint32_t hi = part + 1 >= nparts ? n : part_lower_bound(f, n, part_target(total, part + 1, nparts));
    if (hi < lo) hi = lo;
    st->part_lo = lo;
    st->part_hi = hi;
    st->pair_tests = pre[hi] - pre[lo];
}

inline unsigned nblk(uint64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
struct Timer {
    cudaEvent_t e[6];
    cudaStream_t s;
    explicit Timer(cudaStream_t s_) : s(s_) {
        for (auto &x : e) cudaEventCreate(&x);
    }
    ~Timer() {
        for (auto &x : e) cudaEventDestroy(x);
    }
    void mark(int k) { cudaEventRecord(e[k], s); }
    float ms(int a, int b) {
        float t = 0.f;
        cudaEventElapsedTime(&t, e[a], e[b]);
        return t;
    }
};

int persistent_blocks(int bps) { return num_sms() * bps; }

// per-thread reusable CUDA events and pinned host copy of DevStats (avoid
// creating events / staging pageable copies on every search)
Timer &timer_for(cudaStream_t s) {
    static thread_local Timer *t = nullptr;
    if (!t) t = new Timer(s);
    t->s = s;
    return *t;
}

DevStats *pinned_stats() {
    static thread_local DevStats *p = nullptr;
    if (!p && cudaMallocHost(&p, sizeof(DevStats)) != cudaSuccess) {
        cudaGetLastError();
        static thread_local DevStats fallback;
        p = &fallback;
    }
    return p;
}

// TDS_FSG_LITERAL=1: GPUSpatial candidates are whole cells, as in the paper
// (no per-cell time trimming) — for ablation
// TDS_TIGHT_RANGE=1: entry-exact candidate range ends instead of the hull of the
// overlapping bins (the paper's granularity).  An ablation, off by default: on
// Random-1M-shaped data it removes < 1 bin of slack per side and measured within
// noise, while its extra schedule loads shift the overlap of the concurrent
// searches of a bench step
int tight_ranges() {
    const char *e = getenv("TDS_TIGHT_RANGE");
    return (e && e[0] == '1') ? 1 : 0;
}

// work items per resident warp of the range kernel (the dynamic distribution's
// granularity: more, smaller items shorten the tail of the launch);
// TDS_ITEMS_PER_WARP overrides (A/B)
uint32_t items_per_warp() {
    const char *e = getenv("TDS_ITEMS_PER_WARP");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? (uint32_t)v : (uint32_t)TDS_ITEMS_PER_WARP;
}

int fsg_literal() {
    const char *e = getenv("TDS_FSG_LITERAL");
    return (e && e[0] == '1') ? 1 : 0;
}

// STATIC: the instantiation with the stationary-query filter (compiled only
// where the query set holds a stationary segment: the path costs registers)
template <bool EXACT, bool STATIC, bool SPATIAL, bool SPARSE>
void launch_range_k(const RangeArgs &a, cudaStream_t s) {
    constexpr size_t smem = sizeof(RangeWarpSmem) * (PT / 32);
    // RANGE_BPS resident blocks per SM: 228 KB of shared memory per SM, 1 KB reserved per block
    static_assert(RANGE_BPS * (smem + 1024) <= 228 * 1024, "range kernel shared memory exceeds RANGE_BPS blocks/SM");
    static bool attr_set[64] = {};   // per instantiation and device (first launch)
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 64 || !attr_set[dev]) {
        TDS_CUDA(cudaFuncSetAttribute(k_pair_range<EXACT, STATIC, SPATIAL, SPARSE>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (dev < 64) attr_set[dev] = true;
    }
    k_pair_range<EXACT, STATIC, SPATIAL, SPARSE><<<persistent_blocks(RANGE_BPS), PT, smem, s>>>(a);
}

template <bool EXACT, bool SPARSE>
void launch_range_m(const RangeArgs &a, bool with_static, cudaStream_t s) {
    // GPUSpatial (reference-cell rule) and the stationary-query filter are
    // compile-time variants: each costs registers where it is not needed
    if (a.ecell) {
        if (with_static) launch_range_k<EXACT, true, true, SPARSE>(a, s);
        else launch_range_k<EXACT, false, true, SPARSE>(a, s);
    } else {
        if (with_static) launch_range_k<EXACT, true, false, SPARSE>(a, s);
        else launch_range_k<EXACT, false, false, SPARSE>(a, s);
    }
}

// hit-sparse searches (the probe's pass fraction below TDS_SPARSE_ONLY %) run the
// instantiation without the dense-window step (first passes only)
template <bool EXACT>
void launch_range(const RangeArgs &a, bool with_static, bool sparse_only, cudaStream_t s) {
    if constexpr (!EXACT) {
        if (sparse_only) {
            launch_range_m<EXACT, true>(a, with_static, s);
            return;
        }
    }
    (void)sparse_only;
    launch_range_m<EXACT, false>(a, with_static, s);
}

// stationary query segments (P1 = P0, the supernova case of P:84-88) in Q
__global__ void k_count_static(const float4 *__restrict__ Q, uint32_t n, DevStats *st) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    bool sq = false;
    if (p < n) {
        const float4 a = Q[2 * (uint64_t)p], b = Q[2 * (uint64_t)p + 1];
        sq = a.x == b.x && a.y == b.y && a.z == b.z;
    }
    const unsigned m = __ballot_sync(FULL, sq);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&st->n_static, (unsigned)__popc(m));
}

// build tiles + work items for schedule entries [lo, hi) of the sorted schedule
// (the category counts in st describe the whole sorted schedule)
uint32_t plan_items(const Sched *sched, uint32_t lo, uint32_t hi, DevStats *st, DBuf<Tile> &tiles,
                    DBuf<uint32_t> &item_start, DBuf<uint32_t> &item_tile, cudaStream_t s, int part_range = 0) {
    uint32_t n = hi - lo;
    uint32_t max_tiles = n / 32 + 5;     // also bounds the tiles of any sub-range (part_range)
    tiles = DBuf<Tile>(max_tiles, s);
    item_start = DBuf<uint32_t>(max_tiles + 1, s);
    k_make_tiles<<<nblk((uint64_t)max_tiles * 32), 256, 0, s>>>(sched, lo, n, st, lo, hi, tiles.p, max_tiles,
                                                                item_start.p, part_range);
    TDS_CHECK_LAUNCH();
    uint32_t target = (uint32_t)persistent_blocks(RANGE_BPS) * (PT / 32) * items_per_warp();
    k_tile_chunks<<<nblk(max_tiles), 256, 0, s>>>(item_start.p, max_tiles, &st->union_total, st, target);
    TDS_CHECK_LAUNCH();
    exclusive_scan_u32(item_start.p, item_start.p, max_tiles + 1, nullptr, s);
    const uint32_t cap = target + max_tiles + 1;   // bounds the items (k_tile_chunks)
    item_tile = DBuf<uint32_t>(cap, s);
    k_item_tiles<<<nblk((uint64_t)max_tiles * 32), 256, 0, s>>>(item_start.p, max_tiles, item_tile.p, cap);
    TDS_CHECK_LAUNCH();
    return max_tiles;
}

struct Ctx {
    tds_index_s *idx;
    int kind;
    const float4 *Q;
    uint64_t nq;
    float d, T0, T1;
    cudaStream_t s;
};

}  // namespace

void search(tds_index_s *idx, int kind, const float4 *Q, uint64_t nq, double d64, float T0, float T1,
            uint64_t capacity, cudaStream_t s, tds_result_s *res, const SearchOpts &opt) {
    const uint32_t part = opt.nparts > 1 ? opt.part : 0u, nparts = std::max<uint32_t>(opt.nparts, 1u);
    // fp32 paths use d rounded up (conservative: never drops a pair within the
    // caller's d); the fp64 evaluation uses the caller's d exactly
    float d = (float)d64;
    if ((double)d < d64) d = nextafterf(d, INFINITY);
    float dlo = (float)d64;                               // rounded down (certain-hit tests)
    if ((double)dlo > d64) dlo = nextafterf(dlo, 0.f);
    tds_stats &S = res->stats;
    memset(&S, 0, sizeof S);
    res->stream = s;
    res->nq = nq;
    res->ne = idx->n;
    res->n = 0;
    res->chunked = false;
    if (nq == 0) return;
    if (nq >= (1ull << 31)) fail(TDS_EINVAL, "nq = %llu too large", (unsigned long long)nq);
    Timer &tm = timer_for(s);
    tm.mark(0);
    Trace tr(s);
    const uint32_t n = (uint32_t)nq;
    // one zeroed header allocation: device stats, per-query counts, redo flags
    const size_t hdr = (sizeof(DevStats) + 4ull * n + n + 15) & ~(size_t)15;
    DBuf<uint8_t> header(hdr, s);
    TDS_CUDA(cudaMemsetAsync(header.p, 0, hdr, s));
    DevStats *dstp = reinterpret_cast<DevStats *>(header.p);
    uint32_t *qcount_p = reinterpret_cast<uint32_t *>(header.p + sizeof(DevStats));
    uint8_t *redo_p = header.p + sizeof(DevStats) + 4ull * n;
    struct { DevStats *p; } dst{dstp};
    struct { uint32_t *p; } qcount{qcount_p};
    struct { uint8_t *p; } redo{redo_p};
    // stationary query segments decide whether the pair kernel carries the
    // stationary-query filter (launch_range)
    k_count_static<<<nblk(n), 256, 0, s>>>(Q, n, dstp);
    TDS_CHECK_LAUNCH();

    // ---- A6: queries are validated inside the schedule kernels; GPUTemporal /
    // GPUSpatioTemporal order them by (selector, range start) below, which subsumes
    // the t_start sort of P:681-682 (range starts are monotone in t_start)
    // TDS_AUTO: schedule GPUSpatioTemporal (counting the GPUTemporal ranges too),
    // then keep whichever plan has the lower estimated cost (below)
    const int req_kind = kind;
    if (kind == TDS_AUTO) kind = (idx->kinds & TDS_SPATIOTEMPORAL) ? TDS_SPATIOTEMPORAL : TDS_TEMPORAL;
    const bool spatial = (kind == TDS_SPATIAL);
    DBuf<uint32_t> keys, order;
    if (!spatial) { keys = DBuf<uint32_t>(n, s); order = DBuf<uint32_t>(n, s); }

    // ---- A7: schedule ---------------------------------------------------------
    // Every variant ends in a sorted schedule of ns entries (query row, candidate
    // range, selector) for the pair kernel: one per query for GPUTemporal /
    // GPUSpatioTemporal (a range of the sorted entries or of X/Y/Z), one per
    // (query, FSG cell) for GPUSpatial (a time-trimmed slice of the cell-ordered
    // record copy, with the cell and the query box for the reference-cell rule).
    DBuf<Sched> sched;
    DBuf<uint32_t> sp_cell, sp_qlo;      // GPUSpatial entries: cell, query-box low corner (packed)
    DBuf<Tile> tiles;
    DBuf<uint32_t> item_start, item_tile;
    uint32_t ntiles = 0;
    uint32_t ns = n;                     // schedule entries
    int key_bits = 16;
    if (!spatial) {
        sched = DBuf<Sched>(n, s);
        SchedArgs a{};
        a.Q = Q; a.order = nullptr; a.nq = n; a.d = d; a.T0 = T0; a.T1 = T1;
        a.m = idx->m; a.v = idx->v;
        a.bin_off = idx->bin_off; a.bin_lo = idx->bin_lo; a.bin_pmhi = idx->bin_pmhi;
        a.use_st = kind == TDS_SPATIOTEMPORAL;
        if (a.use_st) {
            a.st_off0 = idx->st_off[0]; a.st_off1 = idx->st_off[1]; a.st_off2 = idx->st_off[2];
            for (int c = 0; c < 3; ++c) { a.st_o[c] = idx->ext.lo[c]; a.st_w[c] = idx->ext.w_st[c]; }
        }
        a.out = sched.p;
        a.keys = keys.p;
        a.vals = order.p;
        uint64_t lo_max = idx->n;
        if (a.use_st)
            for (int c = 0; c < 3; ++c) lo_max = std::max<uint64_t>(lo_max, idx->st_len[c]);
        int lo_bits = 1;
        while ((1ull << lo_bits) <= lo_max) ++lo_bits;
        // the order only shapes the groups of 32 (the category must be exact): the
        // top 13 bits of the range start suffice, so the key has 16 bits = 2 passes
        a.lo_shift = std::max(0, lo_bits - 13);
        for (int c = 0; c < 3; ++c) {
            const float ext = idx->ext.hi[c] - idx->ext.lo[c];
            a.mo[c] = idx->ext.lo[c];
            a.mw[c] = ext > 0.f ? ext / 1024.f : 1.0f;
        }
        key_bits = 32;
        a.st = dst.p;
        a.count_t = (req_kind == TDS_AUTO && a.use_st) ? 1 : 0;
        a.rec = idx->rec;
        a.tight = tight_ranges() && idx->time_order;      // needs t_start order inside the bins
        k_schedule<<<nblk(n), 256, 0, s>>>(a);
        TDS_CHECK_LAUNCH();
        if (a.count_t) {
            // index choice per batch: estimated cost = scheduled
            // pair tests x cost per pair test; GPUSpatioTemporal's indirect candidates
            // measured ST_PAIR_COST x GPUTemporal's per pair test
            DevStats &h0 = *pinned_stats();
            TDS_CUDA(cudaMemcpyAsync(&h0, dst.p, sizeof h0, cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            const unsigned long long p_st = h0.pair_tests, p_t = h0.pair_tests_t;
            if ((double)p_t < ST_PAIR_COST * (double)p_st) {
                TDS_CUDA(cudaMemsetAsync(dst.p, 0, sizeof(DevStats), s));
                a.use_st = 0;
                a.count_t = 0;
                kind = TDS_TEMPORAL;
                k_schedule<<<nblk(n), 256, 0, s>>>(a);
                TDS_CHECK_LAUNCH();
                S.pair_tests_alt = p_st;
            } else {
                S.pair_tests_alt = p_t;
            }
        }
        if (opt.plan_sel) {
            // tds_plan: the schedule entry of every query row (query order, before the sort)
            std::vector<Sched> hsched(n);
            TDS_CUDA(cudaMemcpyAsync(hsched.data(), sched.p, sizeof(Sched) * n, cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaMemcpyAsync(pinned_stats(), dst.p, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            if (pinned_stats()->bad)
                fail(TDS_EDATA, "query segment %llu has a non-finite value or t_end <= t_start", ~pinned_stats()->bad);
            for (uint32_t p = 0; p < n; ++p) {
                opt.plan_sel[p] = hsched[p].sel;
                opt.plan_lo[p] = hsched[p].lo;
                opt.plan_hi[p] = hsched[p].hi;
            }
            S.kind = kind;
            return;
        }
    } else {
        FsgGrid G{};
        for (int c = 0; c < 3; ++c) { G.o[c] = idx->ext.lo[c]; G.w[c] = idx->w_fsg[c]; G.g[c] = idx->grid[c]; }
        DBuf<int4> qbox(2ull * n, s);
        DBuf<uint32_t> row_start(n + 1, s), nr(n + 1, s);
        DBuf<unsigned long long> ntot(1, s);
        TDS_CUDA(cudaMemsetAsync(nr.p + n, 0, 4, s));
        TDS_CUDA(cudaMemsetAsync(ntot.p, 0, 8, s));
        // query order: (t_start, Morton cell of the start point); equal slices of
        // queries at the same time end up next to each other after the entry sort
        DBuf<uint32_t> kc(n, s), kt(n, s), kt2(n, s), fsg_order(n, s);
        k_fsg_order_keys<<<nblk(n), 256, 0, s>>>(Q, n, G, kc.p, kt.p, fsg_order.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(kc.p, fsg_order.p, n, 0, 30, s);
        k_gather_u32<<<nblk(n), 256, 0, s>>>(kt.p, fsg_order.p, n, kt2.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(kt2.p, fsg_order.p, n, 0, 32, s);
        k_fsg_count<<<nblk(n), 256, 0, s>>>(Q, fsg_order.p, n, d, T0, T1, G, nr.p, qbox.p, ntot.p, &dst.p->bad);
        TDS_CHECK_LAUNCH();
        exclusive_scan_u32(nr.p, row_start.p, n + 1, nullptr, s);
        unsigned long long items64 = 0;
        TDS_CUDA(cudaMemcpyAsync(&items64, ntot.p, 8, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
        if (items64 >= (1ull << 31))
            fail(TDS_EINVAL, "the d-inflated query boxes cover %llu grid cells (limit 2^31): use a coarser grid",
                 items64);
        const uint32_t nrows = (uint32_t)items64;
        DBuf<uint32_t> row_q(nrows, s), row_alo(nrows, s), row_len(nrows + 1, s), row_cxy(nrows, s);
        k_fsg_items<<<nblk((uint64_t)n * 32), 256, 0, s>>>(row_start.p, n, qbox.p, Q, G, idx->cell_off, idx->fsg_rec,
                                                          T0, T1, idx->ext.max_dur, fsg_literal(), row_q.p,
                                                          row_alo.p, row_len.p, row_cxy.p);
        TDS_CHECK_LAUNCH();
        // (query, cell) items -> schedule entries, sorted by slice start: the entries
        // of queries that share a (cell, time) slice form the groups of 32
        ns = std::max<uint32_t>(nrows, 1u);
        sched = DBuf<Sched>(ns, s);
        keys = DBuf<uint32_t>(ns, s);
        order = DBuf<uint32_t>(ns, s);
        sp_cell = DBuf<uint32_t>(ns, s);
        sp_qlo = DBuf<uint32_t>(ns, s);
        if (nrows == 0) {
            TDS_CUDA(cudaMemsetAsync(sched.p, 0, sizeof(Sched), s));
            ns = 0;
        } else {
            int lo_bits = 1;
            while ((1ull << lo_bits) <= idx->A_len) ++lo_bits;     // A_len < 2^31 (build check)
            key_bits = std::min(lo_bits + 1, 32);
            k_fsg_sched<<<nblk(nrows), 256, 0, s>>>(nrows, row_q.p, row_alo.p, row_len.p, row_cxy.p, qbox.p,
                                                    1u << lo_bits, sched.p, keys.p, order.p, sp_cell.p, sp_qlo.p,
                                                    dst.p);
            TDS_CHECK_LAUNCH();
        }
    }
    if (ns) {
        // sort the entries by (category, range start): one stable radix sort
        tr.mark("sched_kernel");
        radix_sort_pairs(keys.p, order.p, ns, 0, key_bits, s);
        tr.mark("sort");
        {
            DBuf<Sched> tmp(ns, s);
            k_permute_sched<<<nblk(ns), 256, 0, s>>>(sched.p, order.p, ns, tmp.p);
            TDS_CHECK_LAUNCH();
            std::swap(sched.p, tmp.p);
        }
        if (spatial) {
            DBuf<uint32_t> tc(ns, s), tq(ns, s);
            k_gather_u32<<<nblk(ns), 256, 0, s>>>(sp_cell.p, order.p, ns, tc.p);
            TDS_CHECK_LAUNCH();
            k_gather_u32<<<nblk(ns), 256, 0, s>>>(sp_qlo.p, order.p, ns, tq.p);
            TDS_CHECK_LAUNCH();
            std::swap(sp_cell.p, tc.p);
            std::swap(sp_qlo.p, tq.p);
        }
        tr.mark("permute");
        if (nparts > 1) {
            // this part's slice of the sorted schedule: equal shares of the exact pair tests
            DBuf<uint64_t> w(ns + 1, s);
            k_sched_work<<<nblk(ns + 1), 256, 0, s>>>(sched.p, ns, w.p);
            TDS_CHECK_LAUNCH();
            exclusive_scan_u64(w.p, w.p, ns + 1, nullptr, s);
            k_part_bounds<<<1, 32, 0, s>>>(w.p, ns, part, nparts, dst.p);
            TDS_CHECK_LAUNCH();
            ntiles = plan_items(sched.p, 0, ns, dst.p, tiles, item_start, item_tile, s, /*part_range=*/1);
        } else {
            ntiles = plan_items(sched.p, 0, ns, dst.p, tiles, item_start, item_tile, s);
        }
    }
    const float4 *prec = spatial ? idx->fsg_rec : idx->rec;
    const uint32_t *pperm = spatial ? idx->fsg_perm : idx->perm;
    // result-size probe (automatic capacity): launched before the host reads the
    // schedule's totals, so one synchronisation returns both (its estimate is used
    // for large searches only, below); its counters start zeroed with the header
    tr.mark("tiles");
    const bool probe_run = capacity == 0 && ns;
    if (probe_run) {
        k_density_probe<<<32, 256, 0, s>>>(sched.p, ns, Q, prec, spatial ? nullptr : idx->st_arr[0],
                                           spatial ? nullptr : idx->st_arr[1], spatial ? nullptr : idx->st_arr[2], d,
                                           T0, T1, spatial ? idx->fsg_ecell : nullptr, sp_cell.p, sp_qlo.p, dst.p);
        TDS_CHECK_LAUNCH();
    }
    tr.mark("schedule");
    // pair tests bound the result count: size the pass buffer
    DevStats &hs = *pinned_stats();
    TDS_CUDA(cudaMemcpyAsync(&hs, dst.p, sizeof hs, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    if (hs.bad) fail(TDS_EDATA, "query segment %llu has a non-finite value or t_end <= t_start", ~hs.bad);
    tm.mark(1);
    tr.mark("sync");
    S.pair_tests = hs.pair_tests;
    S.fallback_queries = hs.fallback;
    const char *ns_env0 = getenv("TDS_NO_STATIC");
    const bool with_static = hs.n_static > 0 && !(ns_env0 && ns_env0[0] == '1');
    S.kind = kind;
    S.n_queries = spatial ? nq : (nq - hs.cat_cnt[4]);
    if (nparts > 1 && !spatial) {
        const uint32_t live = (uint32_t)(nq - hs.cat_cnt[4]);
        S.n_queries = std::min(hs.part_hi, live) > hs.part_lo ? std::min(hs.part_hi, live) - hs.part_lo : 0;
    }
    // result-size probe (automatic capacity, large searches): the pass fraction of a
    // sample of the pair tests bounds the result count; the pass buffer takes three
    // times the estimate (a pass that overflows re-plans exactly, C22) instead of one
    // slot per pair test, which on hit-sparse searches meant a buffer 10-40x the
    // result and a compaction copy after the pass
    uint64_t est_hits = 0;
    bool probed = false;
    int start_dense = 0;
    bool sparse_only = false;
    if (probe_run && hs.probe_total >= 1024) {
        const char *e = getenv("TDS_DENSE_START");            // A/B override (%)
        const double thr = (e ? atof(e) : (double)TDS_DENSE_START) / 100.0;
        start_dense = (double)hs.probe_pass >= thr * (double)hs.probe_total ? 1 : 0;
        const char *e2 = getenv("TDS_SPARSE_ONLY");           // A/B override (%)
        const double thr2 = (e2 ? atof(e2) : (double)TDS_SPARSE_ONLY) / 100.0;
        sparse_only = (double)hs.probe_pass < thr2 * (double)hs.probe_total;
    }
    if (probe_run && hs.pair_tests >= CAP_PROBE_MIN) {
        if (hs.probe_total >= 1024 && hs.probe_entries) {
            // unbiased for entries sampled evenly over the schedule: the mean of the
            // sampled entries' estimated records times the number of entries
            probed = true;
            const double scale = (double)(nparts > 1 ? hs.part_hi - hs.part_lo : ns) / hs.probe_entries;
            est_hits = (uint64_t)(hs.probe_est * scale);
        }
        tr.note("probe_est_hits", (double)est_hits);
    }

    uint64_t cap = capacity;
    std::unique_lock<std::mutex> big_lock;
    if (cap == 0) {
        // budget: the device memory available at the last snapshot minus what the
        // pools hand out since (abi.cu; no cudaMemGetInfo per search).  Buffers above
        // 1 GB are sized and allocated under a process-wide lock, so concurrent
        // searches (tds_search_many) do not over-commit the device.
        uint64_t want = hs.pair_tests + 64;
        if (probed) want = std::min<uint64_t>(want, 3 * est_hits + CAP_FLOOR);
        // + one partly filled chunk per warp (chunks of <= 1024 slots are reserved whole),
        // rounded up to 4 sizes per octave so that later searches reuse the pool's blocks
        want += (uint64_t)persistent_blocks(RANGE_BPS) * (PT / 32) * 1024;
        {
            int e = 0;
            while ((4ull << e) < want) ++e;
            const uint64_t q = 1ull << e;                        // want in (4q, 8q]
            want = (want + q - 1) / q * q;
        }
        if (want * sizeof(Rec) > (1ull << 30)) big_lock = std::unique_lock<std::mutex>(big_alloc_mutex());
        const uint64_t budget_bytes = device_budget_bytes();
        cap = std::min<uint64_t>(want, (uint64_t)(budget_bytes * 0.45) / sizeof(Rec));
        cap = std::max<uint64_t>(cap, 1024);
        tr.mark(big_lock.owns_lock() ? "budget(locked)" : "budget");
    }
    cap = std::min<uint64_t>(cap, (1ull << 40));
    const uint64_t nwarps = (uint64_t)persistent_blocks(RANGE_BPS) * (PT / 32);
    const uint64_t cs_want = std::min<uint64_t>(1024, std::max<uint64_t>(128, cap / (16 * nwarps)));  // >= 128: appendK
    uint32_t cs_shift = 7;
    while ((2ull << cs_shift) <= cs_want) ++cs_shift;
    const uint32_t CS = 1u << cs_shift;             // a power of two: chunk index by shift
    const uint64_t nchunks = (cap + CS - 1) / CS;
    DBuf<Rec> buf;
    for (;;) {
        try {
            buf = DBuf<Rec>(cap, s, /*big=*/true);
            break;
        } catch (const Error &e) {
            if (e.code != TDS_ENOMEM || capacity != 0 || cap <= (1ull << 20)) throw;
            cap /= 2;                     // auto capacity: retry smaller (overflow re-plan covers the rest)
            device_budget_refresh();      // memory use changed outside the pools
            set_error(0, "");
        }
    }
    tr.mark("alloc");
    tr.note("cap_GB", cap * sizeof(Rec) / 1e9);
    S.capacity = cap;
    if (big_lock.owns_lock()) big_lock.unlock();   // the pool counts the buffer from here on
    DBuf<uint32_t> chunk_used(nchunks, s);
    TDS_CUDA(cudaMemsetAsync(chunk_used.p, 0, 4 * nchunks, s));

    OutArgs o{};
    o.buf = buf.p; o.cap = cap; o.CS = CS; o.cs_shift = cs_shift; o.chunk_used = chunk_used.p;
    o.redo = redo.p; o.qcount = qcount.p; o.st = dst.p;

    auto range_args = [&](const OutArgs &oo) {
        RangeArgs a{};
        a.df = filter_threshold(d);
        {
            float d2 = d * d;                              // d (float, rounded up) squared, rounded up
            if ((double)d2 < (double)d * (double)d) d2 = nextafterf(d2, INFINITY);
            a.d2u = d2;
        }
        a.tc = time_origin(idx);
        const double dd = d64 * d64;
        const float d2h = (float)dd, d2l = (float)(dd - (double)d2h);
        a.pc = PairCtx{Q, prec, pperm, d, T0, T1, oo, d64, dlo, d2h, d2l};
        for (int c = 0; c < 3; ++c) {
            a.arr[c] = spatial ? nullptr : idx->st_arr[c];
            a.srec[c] = spatial ? nullptr : idx->st_rec[c];
        }
        if (spatial) { a.ecell = idx->fsg_ecell; }
        a.wb[0] = spatial ? idx->wb_fsg : idx->wb_rec;
        for (int c = 0; c < 3; ++c) a.wb[1 + c] = spatial ? nullptr : idx->wb_st[c];
        const char *ns_env = getenv("TDS_NO_STATIC");
        a.static_ok = (ns_env && ns_env[0] == '1') ? 0 : 1;
        const char *hh = getenv("TDS_HYST_HI"), *hl = getenv("TDS_HYST_LO");   // tuning (A/B)
        a.hyst_hi = hh ? atoi(hh) : HYST_HI;
        a.hyst_lo = hl ? atoi(hl) : HYST_LO;
        a.start_dense = start_dense;
        return a;
    };

    // ---- A8-A10: pass 1 --------------------------------------------------------
    tr.mark("sync+alloc");
    tm.mark(2);
    if (ns && hs.pair_tests > 0) {
        RangeArgs a = range_args(o);
        a.sched = sched.p; a.tiles = tiles.p; a.item_start = item_start.p; a.item_tile = item_tile.p;
        a.ntiles = ntiles;
        a.sp_cell = sp_cell.p; a.sp_qlo = sp_qlo.p;
        launch_range<false>(a, with_static, sparse_only, s);
        TDS_CHECK_LAUNCH();
    }
    tm.mark(3);
    tr.mark("pairs");
    TDS_CUDA(cudaMemcpyAsync(&hs, dst.p, sizeof hs, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    S.passes = 1;
    S.refined_pairs = hs.refined;
    S.refined32 = hs.refined32;
    S.direct_records = hs.direct;
    S.pairs_executed = hs.executed;

    // only the first nres chunks were ever reserved (reservations are sequential)
    const uint64_t nres = std::min<uint64_t>(nchunks, (std::min<unsigned long long>(hs.reserved, cap) + CS - 1) / CS);
    DBuf<uint64_t> chunk_off(std::max<uint64_t>(nres, 1), s);
    k_chunk_offsets_u64<<<nblk(std::max<uint64_t>(nres, 1)), 256, 0, s>>>(chunk_used.p, nres, chunk_off.p);
    TDS_CHECK_LAUNCH();
    exclusive_scan_u64(chunk_off.p, chunk_off.p, nres, nullptr, s);

    if (hs.dropped == 0 && cap >= (1ull << 26) && hs.hits <= cap / 8) {
        // few results in a large (>= 1 GB) pass buffer: compact them into a
        // right-sized store and return the buffer to the pool for the next search
        DBuf<Rec> store(hs.hits, s, /*big=*/hs.hits * sizeof(Rec) > (256ull << 20));
        if (nres) {
            k_flatten<<<nblk(nres * 32), 256, 0, s>>>(buf.p, CS, nres, chunk_used.p, chunk_off.p, store.p);
            TDS_CHECK_LAUNCH();
        }
        res->chunked = false;
        res->store = store.release();
        res->n = hs.hits;
        tm.mark(4);
        TDS_CUDA(cudaEventSynchronize(tm.e[4]));
        S.n_results = res->n;
        S.ms_schedule = tm.ms(0, 1);
        S.ms_pairs = tm.ms(2, 3);
        S.ms_compact = tm.ms(3, 4);
        S.ms_total = tm.ms(0, 4);
        return;
    }
    if (hs.dropped == 0) {
        res->chunked = true;
        res->buf = buf.release();
        res->cap = cap;
        res->CS = CS;
        res->nchunks = nres;
        res->chunk_used = chunk_used.release();
        res->chunk_off = chunk_off.release();
        res->n = hs.hits;
        tm.mark(4);
        TDS_CUDA(cudaEventSynchronize(tm.e[4]));
        S.n_results = res->n;
        S.ms_schedule = tm.ms(0, 1);
        S.ms_pairs = tm.ms(2, 3);
        S.ms_total = tm.ms(0, 4);
        return;
    }

    // ---- overflow: keep complete queries, re-plan the others exactly ------------
    // memory: the pass buffer + 8 B per chunk + the exact store; kept records move
    // from the chunked buffer straight into the store
    DBuf<uint64_t> kept_off(nres + 1, s);
    k_chunk_kept<<<nblk((nres + 1) * 32), 256, 0, s>>>(buf.p, CS, nres, chunk_used.p, redo.p, kept_off.p);
    TDS_CHECK_LAUNCH();
    exclusive_scan_u64(kept_off.p, kept_off.p, nres + 1, nullptr, s);
    uint64_t nkept = 0;
    TDS_CUDA(cudaMemcpyAsync(&nkept, kept_off.p + nres, 8, cudaMemcpyDeviceToHost, s));
    // queries to re-run (input order) with their exact record counts
    std::vector<uint8_t> hr(n);
    std::vector<uint32_t> hq(n);
    TDS_CUDA(cudaMemcpyAsync(hr.data(), redo.p, n, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaMemcpyAsync(hq.data(), qcount.p, 4ull * n, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> rl, hcnt;
    uint64_t redo_total = 0;
    for (uint32_t k = 0; k < n; ++k)
        if (hr[k]) {
            if (hq[k] > cap)
                fail(TDS_ECAPACITY, "one query produces %u records, more than capacity %llu", hq[k],
                     (unsigned long long)cap);
            rl.push_back(k);
            hcnt.push_back(hq[k]);
            redo_total += hq[k];
        }
    const uint32_t nredo = (uint32_t)rl.size();
    const uint64_t total = nkept + redo_total;
    DBuf<Rec> store;
    try {
        store = DBuf<Rec>(total, s, /*big=*/true);
    } catch (const Error &e) {
        if (e.code != TDS_ENOMEM) throw;
        set_error(0, "");
    }
    if (store.p) {
        if (nres) {
            k_scatter_kept_chunked<<<nblk(nres * 32), 256, 0, s>>>(buf.p, CS, nres, chunk_used.p, redo.p,
                                                                   kept_off.p, store.p);
            TDS_CHECK_LAUNCH();
        }
        buf.reset();
    } else {
        // not enough device memory for the pass buffer and the exact store at once:
        // spill the kept records to mapped pinned host memory, release the pass
        // buffer, then allocate the store and copy them back (peak = the larger one)
        Rec *host = nullptr, *host_dev = nullptr;
        TDS_CUDA(cudaHostAlloc((void **)&host, std::max<uint64_t>(nkept, 1) * sizeof(Rec), cudaHostAllocMapped));
        struct HostFree { Rec *p; ~HostFree() { cudaFreeHost(p); } } host_guard{host};
        TDS_CUDA(cudaHostGetDevicePointer((void **)&host_dev, host, 0));
        if (nres) {
            k_scatter_kept_chunked<<<nblk(nres * 32), 256, 0, s>>>(buf.p, CS, nres, chunk_used.p, redo.p,
                                                                   kept_off.p, host_dev);
            TDS_CHECK_LAUNCH();
        }
        buf.reset();
        TDS_CUDA(cudaStreamSynchronize(s));
        device_budget_refresh();
        store = DBuf<Rec>(total, s, /*big=*/true);
        if (nkept) TDS_CUDA(cudaMemcpyAsync(store.p, host, nkept * sizeof(Rec), cudaMemcpyHostToDevice, s));
        TDS_CUDA(cudaStreamSynchronize(s));
        tr.note("spilled_to_host", (double)nkept);
    }
    kept_off.reset();
    S.spilled = nkept;

    // per-query exact offsets (redo order after the kept records)
    DBuf<unsigned long long> qoff(n, s);
    DBuf<uint32_t> qfill(n, s);
    TDS_CUDA(cudaMemsetAsync(qfill.p, 0, 4ull * n, s));
    {
        std::vector<unsigned long long> hoff(n, 0);
        uint64_t acc = nkept;
        for (uint32_t k = 0; k < nredo; ++k) { hoff[rl[k]] = acc; acc += hcnt[k]; }
        TDS_CUDA(cudaMemcpyAsync(qoff.p, hoff.data(), 8ull * n, cudaMemcpyHostToDevice, s));
        TDS_CUDA(cudaStreamSynchronize(s));
    }
    tm.mark(4);
    // batches of re-run queries with sum(count) <= cap (the paper's incremental
    // processing of Q): the schedule entries of the batch's queries
    // are compacted and re-evaluated, records written at exact per-query offsets
    o.buf = store.p;
    o.qoff = qoff.p;
    o.qfill = qfill.p;
    DBuf<uint32_t> qcount2(n, s);      // counts are recomputed, not needed again
    TDS_CUDA(cudaMemsetAsync(qcount2.p, 0, 4ull * n, s));
    o.qcount = qcount2.p;
    DBuf<uint8_t> inbatch(n, s);
    DBuf<uint32_t> dl(std::max<uint32_t>(nredo, 1), s);
    if (nredo) TDS_CUDA(cudaMemcpyAsync(dl.p, rl.data(), 4ull * nredo, cudaMemcpyHostToDevice, s));
    uint32_t b0 = 0;
    while (b0 < nredo) {
        uint64_t acc = 0;
        uint32_t b1 = b0;
        while (b1 < nredo && acc + hcnt[b1] <= cap) acc += hcnt[b1++];
        TDS_CUDA(cudaMemsetAsync(inbatch.p, 0, n, s));
        k_mark_rows<<<nblk(b1 - b0), 256, 0, s>>>(dl.p + b0, b1 - b0, inbatch.p);
        TDS_CHECK_LAUNCH();
        DBuf<uint32_t> flag(ns + 1, s), fpos(ns + 1, s);
        TDS_CUDA(cudaMemsetAsync(flag.p + ns, 0, 4, s));
        k_redo_flags_sched<<<nblk(ns), 256, 0, s>>>(sched.p, ns, inbatch.p, flag.p);
        TDS_CHECK_LAUNCH();
        exclusive_scan_u32(flag.p, fpos.p, ns + 1, nullptr, s);
        uint32_t nb = 0;
        TDS_CUDA(cudaMemcpyAsync(&nb, fpos.p + ns, 4, cudaMemcpyDeviceToHost, s));
        DBuf<Sched> rsched(std::max<uint32_t>(ns, 1), s);
        DBuf<uint32_t> rcell, rqlo;
        if (spatial) { rcell = DBuf<uint32_t>(ns, s); rqlo = DBuf<uint32_t>(ns, s); }
        k_compact_sched<<<nblk(ns), 256, 0, s>>>(sched.p, ns, flag.p, fpos.p, rsched.p, sp_cell.p, sp_qlo.p, rcell.p,
                                                 rqlo.p);
        TDS_CHECK_LAUNCH();
        // category counts of the batch (for the tile layout)
        DBuf<DevStats> bst(1, s);
        TDS_CUDA(cudaMemsetAsync(bst.p, 0, sizeof(DevStats), s));
        TDS_CUDA(cudaStreamSynchronize(s));
        if (nb) {
            k_cat_counts<<<nblk(nb), 256, 0, s>>>(rsched.p, nb, bst.p);
            TDS_CHECK_LAUNCH();
            DBuf<Tile> bt;
            DBuf<uint32_t> bis, bit;
            const uint32_t bnt = plan_items(rsched.p, 0, nb, bst.p, bt, bis, bit, s);
            RangeArgs a = range_args(o);
            a.pc.o.st = bst.p;
            a.sched = rsched.p; a.tiles = bt.p; a.item_start = bis.p; a.item_tile = bit.p; a.ntiles = bnt;
            a.sp_cell = rcell.p; a.sp_qlo = rqlo.p;
            launch_range<true>(a, with_static, false, s);
            TDS_CHECK_LAUNCH();
            TDS_CUDA(cudaStreamSynchronize(s));
            DevStats hb2;
            TDS_CUDA(cudaMemcpy(&hb2, bst.p, sizeof hb2, cudaMemcpyDeviceToHost));
            S.refined_pairs += hb2.refined;
            S.refined32 += hb2.refined32;
            S.direct_records += hb2.direct;
            S.pairs_executed += hb2.executed;
        }
        S.passes++;
        b0 = b1;
    }
    tm.mark(5);
    TDS_CUDA(cudaStreamSynchronize(s));
    res->chunked = false;
    res->store = store.release();
    res->n = total;
    S.n_results = total;
    S.ms_schedule = tm.ms(0, 1);
    S.ms_pairs = tm.ms(2, 3) + tm.ms(4, 5);
    S.ms_compact = tm.ms(3, 4);
    S.ms_total = tm.ms(0, 5);
}

void fetch(tds_result_s *r, uint64_t first, uint64_t count, uint32_t *qid, uint32_t *eid, float *tin, float *tout,
           bool dst_dev, bool sorted, cudaStream_t s) {
    if (first > r->n || count > r->n - first) fail(TDS_EINVAL, "fetch range [%llu, +%llu) outside %llu records",
                                                   (unsigned long long)first, (unsigned long long)count,
                                                   (unsigned long long)r->n);
    r->stream = s;
    if (count == 0) return;
    if (r->host) {
        // host-resident records (tds_search_stream): unsorted host destinations are
        // filled on the host; otherwise the range is uploaded and fetched as a store
        if (!dst_dev && !sorted) {
            uint64_t pos = 0, j = 0;
            for (auto &bk : r->host_blocks) {
                const uint64_t lo = std::max(first, pos), hi = std::min(first + count, pos + bk.second);
                for (uint64_t i = lo; i < hi; ++i, ++j) {
                    const Rec &x = bk.first[i - pos];
                    if (qid) qid[j] = x.qid;
                    if (eid) eid[j] = x.eid;
                    if (tin) tin[j] = x.t_in;
                    if (tout) tout[j] = x.t_out;
                }
                pos += bk.second;
            }
            return;
        }
        tds_result_s tmp;
        tmp.chunked = false;
        tmp.n = r->n;
        tmp.stream = s;
        DBuf<Rec> all(r->n, s, r->n * sizeof(Rec) > (256ull << 20));
        uint64_t pos = 0;
        for (auto &bk : r->host_blocks) {
            TDS_CUDA(cudaMemcpyAsync(all.p + pos, bk.first, bk.second * sizeof(Rec), cudaMemcpyHostToDevice, s));
            pos += bk.second;
        }
        tmp.store = all.p;
        fetch(&tmp, first, count, qid, eid, tin, tout, dst_dev, sorted, s);
        TDS_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // device staging for host destinations
    DBuf<uint32_t> dq, de;
    DBuf<float> di, doo;
    uint32_t *oq = qid, *oe = eid;
    float *oi = tin, *oo = tout;
    if (!dst_dev) {
        if (qid) { dq = DBuf<uint32_t>(count, s); oq = dq.p; }
        if (eid) { de = DBuf<uint32_t>(count, s); oe = de.p; }
        if (tin) { di = DBuf<float>(count, s); oi = di.p; }
        if (tout) { doo = DBuf<float>(count, s); oo = doo.p; }
    }
    if (!sorted) {
        if (r->chunked) {
            if (first == 0 && count == r->n)
                k_fetch_chunked<true><<<nblk(r->nchunks * 32), 256, 0, s>>>(r->buf, r->CS, r->nchunks, r->chunk_used,
                                                                        r->chunk_off, first, count, oq, oe, oi, oo);
            else
                k_fetch_chunked<false><<<nblk(r->nchunks * 32), 256, 0, s>>>(r->buf, r->CS, r->nchunks,
                                                                         r->chunk_used, r->chunk_off, first, count,
                                                                         oq, oe, oi, oo);
        } else {
            k_fetch_flat<<<nblk(count), 256, 0, s>>>(r->store, nullptr, first, count, oq, oe, oi, oo);
        }
        TDS_CHECK_LAUNCH();
    } else {
        // flatten, then stable radix sort by entry id, then by query id
        const uint64_t n = r->n;
        DBuf<Rec> flat;
        const Rec *rs = r->store;
        if (r->chunked) {
            flat = DBuf<Rec>(n, s);
            k_flatten<<<nblk(r->nchunks * 32), 256, 0, s>>>(r->buf, r->CS, r->nchunks, r->chunk_used, r->chunk_off,
                                                            flat.p);
            TDS_CHECK_LAUNCH();
            rs = flat.p;
        }
        DBuf<uint32_t> k1(n, s), ord(n, s), k2(n, s), ord2(n, s);
        k_rec_field<<<nblk(n), 256, 0, s>>>(rs, n, 1, nullptr, k1.p, ord.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(k1.p, ord.p, n, 0, 32, s);
        k_rec_field<<<nblk(n), 256, 0, s>>>(rs, n, 0, ord.p, k2.p, ord2.p);
        TDS_CHECK_LAUNCH();
        radix_sort_pairs(k2.p, ord2.p, n, 0, 32, s);
        k_fetch_flat<<<nblk(count), 256, 0, s>>>(rs, ord2.p, first, count, oq, oe, oi, oo);
        TDS_CHECK_LAUNCH();
    }
    if (!dst_dev) {
        if (qid) TDS_CUDA(cudaMemcpyAsync(qid, oq, 4 * count, cudaMemcpyDeviceToHost, s));
        if (eid) TDS_CUDA(cudaMemcpyAsync(eid, oe, 4 * count, cudaMemcpyDeviceToHost, s));
        if (tin) TDS_CUDA(cudaMemcpyAsync(tin, oi, 4 * count, cudaMemcpyDeviceToHost, s));
        if (tout) TDS_CUDA(cudaMemcpyAsync(tout, oo, 4 * count, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
    }
}

// tds_search_stream (the chunked processing of Q of the prior work,
// P:178-183): queries in host memory, `chunk` at a time.  The copy stream uploads
// chunk k+1 while chunk k is searched on `s`, and copies chunk k's records
// (query ids offset to rows of the full set) into pinned host memory while
// chunk k+1 is searched, so the device holds two query chunks and one chunk's
// records at a time; the result is host-resident.
void search_stream(tds_index_s *idx, int kind, const float4 *qh, uint64_t nq, double d64, float T0, float T1,
                   uint64_t chunk, cudaStream_t s, tds_result_s *res, const SearchOpts &opt) {
    res->host = true;
    res->chunked = false;
    res->stream = s;
    res->nq = nq;
    res->ne = idx->n;
    res->n = 0;
    tds_stats &S = res->stats;
    memset(&S, 0, sizeof S);
    if (nq == 0) return;
    chunk = std::max<uint64_t>(1, std::min<uint64_t>(chunk, nq));
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, qh) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    cudaStream_t cs = nullptr;
    TDS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t c; ~StreamGuard() { cudaStreamSynchronize(c); cudaStreamDestroy(c); } } sg{cs};
    cudaEvent_t up[2], used[2], packed;
    for (auto &e : up) TDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : used) TDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TDS_CUDA(cudaEventCreateWithFlags(&packed, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t *a; cudaEvent_t *b; cudaEvent_t c;
        ~EvGuard() { for (int i = 0; i < 2; ++i) { cudaEventDestroy(a[i]); cudaEventDestroy(b[i]); } cudaEventDestroy(c); }
    } eg{up, used, packed};
    DBuf<float4> qb[2] = {DBuf<float4>(2 * chunk, s), DBuf<float4>(2 * chunk, s)};
    TDS_CUDA(cudaStreamSynchronize(s));                 // buffers allocated before the copy stream uses them
    // pageable queries go through a pinned bounce buffer (one per device buffer)
    std::vector<float4 *> bounce(2, nullptr);
    struct BounceGuard { std::vector<float4 *> &b; ~BounceGuard() { for (auto p : b) if (p) cudaFreeHost(p); } } bg{bounce};
    if (!pinned)
        for (auto &p : bounce) TDS_CUDA(cudaHostAlloc((void **)&p, 2 * chunk * sizeof(float4), cudaHostAllocDefault));
    const uint64_t nch = (nq + chunk - 1) / chunk;
    auto upload = [&](uint64_t k) {
        const uint64_t q0 = k * chunk, nk = std::min(chunk, nq - q0);
        const int b = (int)(k & 1);
        TDS_CUDA(cudaStreamWaitEvent(cs, used[b], 0));  // the search of chunk k-2 is done with it
        const float4 *src = qh + 2 * q0;
        if (!pinned) {
            TDS_CUDA(cudaEventSynchronize(used[b]));    // the bounce buffer's last copy has completed
            memcpy(bounce[b], src, nk * sizeof(tds_seg));
            src = bounce[b];
        }
        TDS_CUDA(cudaMemcpyAsync(qb[b].p, src, nk * sizeof(tds_seg), cudaMemcpyHostToDevice, cs));
        TDS_CUDA(cudaEventRecord(up[b], cs));
    };
    for (int b = 0; b < 2; ++b) TDS_CUDA(cudaEventRecord(used[b], s));
    upload(0);
    auto t0 = std::chrono::steady_clock::now();
    for (uint64_t k = 0; k < nch; ++k) {
        const uint64_t q0 = k * chunk, nk = std::min(chunk, nq - q0);
        const int b = (int)(k & 1);
        if (k + 1 < nch) upload(k + 1);
        TDS_CUDA(cudaStreamWaitEvent(s, up[b], 0));
        tds_result_s r;
        try {
            search(idx, kind, qb[b].p, nk, d64, T0, T1, 0, s, &r, opt);
        } catch (...) {
            free_result(&r);
            throw;
        }
        TDS_CUDA(cudaEventRecord(used[b], s));
        // this chunk's records, query ids offset, to a device staging buffer, then to
        // pinned host memory on the copy stream (overlapping the next search)
        const uint64_t nr = r.n;
        if (nr) {
            DBuf<Rec> st(nr, s, nr * sizeof(Rec) > (256ull << 20));
            if (r.chunked)
                k_pack_chunked<<<nblk(r.nchunks * 32), 256, 0, s>>>(r.buf, r.CS, r.nchunks, r.chunk_used, r.chunk_off,
                                                                    (uint32_t)q0, st.p);
            else
                k_pack_flat<<<nblk(nr), 256, 0, s>>>(r.store, nr, (uint32_t)q0, st.p);
            TDS_CHECK_LAUNCH();
            TDS_CUDA(cudaEventRecord(packed, s));
            free_result(&r);
            Rec *hb = reinterpret_cast<Rec *>(pinned_alloc(nr * sizeof(Rec)));
            res->host_blocks.emplace_back(hb, nr);
            TDS_CUDA(cudaStreamWaitEvent(cs, packed, 0));
            TDS_CUDA(cudaMemcpyAsync(hb, st.p, nr * sizeof(Rec), cudaMemcpyDeviceToHost, cs));
            st.s = cs;                                   // freed after the copy, in copy-stream order
        } else {
            free_result(&r);
        }
        res->n += nr;
        S.pair_tests += r.stats.pair_tests;
        S.pairs_executed += r.stats.pairs_executed;
        S.refined_pairs += r.stats.refined_pairs;
        S.refined32 += r.stats.refined32;
        S.direct_records += r.stats.direct_records;
        S.passes += r.stats.passes;
        S.fallback_queries += r.stats.fallback_queries;
        S.n_queries += r.stats.n_queries;
        S.ms_pairs += r.stats.ms_pairs;
        S.ms_schedule += r.stats.ms_schedule;
        S.kind = r.stats.kind;
    }
    TDS_CUDA(cudaStreamSynchronize(cs));
    TDS_CUDA(cudaStreamSynchronize(s));
    S.n_results = res->n;
    S.ms_total = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void free_result(tds_result_s *r) {
    if (!r->host_blocks.empty()) cudaStreamSynchronize(r->stream);   // copies into the blocks are done
    for (auto &b : r->host_blocks) pinned_free(b.first);
    r->host_blocks.clear();
    cudaStream_t s = r->stream;      // ordered after the last fetch on that stream
    if (r->buf) dfree(r->buf, s);
    if (r->chunk_used) dfree(r->chunk_used, s);
    if (r->chunk_off) dfree(r->chunk_off, s);
    if (r->store) dfree(r->store, s);
    r->buf = nullptr; r->chunk_used = nullptr; r->chunk_off = nullptr; r->store = nullptr;
}

}  // namespace tds
