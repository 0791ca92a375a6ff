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
constexpr int PT = 256;                  // threads per block of the pair kernels
#ifndef TDS_RANGE_BPS
#define TDS_RANGE_BPS 2
#endif
#ifndef TDS_SPATIAL_BPS
#define TDS_SPATIAL_BPS 3
#endif
constexpr int RANGE_BPS = TDS_RANGE_BPS;       // resident blocks per SM (range kernel)
constexpr int SPATIAL_BPS = TDS_SPATIAL_BPS;
constexpr int SP_PER_LANE = 8;           // slots per lane per grab (spatial kernel)
#ifndef TDS_HYST_HI
#define TDS_HYST_HI 50
#endif
#ifndef TDS_HYST_LO
#define TDS_HYST_LO 25
#endif
constexpr int HYST_HI = TDS_HYST_HI, HYST_LO = TDS_HYST_LO;
constexpr unsigned long long CAP_PROBE_MIN = 1ull << 24;     // result-size probe above this many pair tests
constexpr uint64_t CAP_FLOOR = 1ull << 22;                   // records: floor of the probed capacity
constexpr double ST_PAIR_COST = 1.5;     // TDS_AUTO: GPUSpatioTemporal cost per pair test / GPUTemporal's
constexpr uint32_t WIN = 128;            // range kernel window: 4 candidates per lane
constexpr unsigned long long SP_GRAB = 32ull * SP_PER_LANE;
// fp32 filter margin: eta = KU * M with M an l1 magnitude bound of the pair
// (derived bound 20 u M, u = 2^-24; 64 u used)
constexpr float KU = 64.0f / 16777216.0f;

struct DevStats {
    unsigned long long reserved;     // slots reserved in the pass buffer
    unsigned long long hits;         // records produced (kept or dropped)
    unsigned long long dropped;      // records dropped (buffer full)
    unsigned long long refined;      // pairs evaluated in fp64
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

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
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

// For a pair that passed a filter: 0 = no shared span (a >= b), 2 = certain hit (fp32 closest approach
// < d - eta) whose fp32 interval [tin, tout] is within its first-order error
// bound of the exact one, the bound being <= 1e-6 * max(b - a, min(|a|, |b|))
// for every end not certainly clamped to a or b (clamped ends are exact);
// 1 = evaluate in fp64 (pair64).
template <bool CHECK_MISS = false>
__device__ __forceinline__ int hit_kind(float4 q0, float4 q1, float t0c, float t1c, const ECand &e, float d,
                                        float &tin, float &tout) {
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
    const float rA = rcp_approx(A);
    const float su = -B * rA;
    const float s = fminf(fmaxf(su, 0.f), L);
    const float yx = fmaf(s, Vx, Dx), yy = fmaf(s, Vy, Dy), yz = fmaf(s, Vz, Dz);
    const float h = fmaf(yx, yx, fmaf(yy, yy, yz * yz));
    const float M = fabsf(dpx) + fabsf(dpy) + fabsf(dpz) + (q1.w + e.ext);
    if (!(a < b)) return 0;                                     // C5 (filter_abs passes a == b)
    if (CHECK_MISS) {                                           // fused filter (dense windows)
        const float thr = fmaf(KU, M, d);
        if (!(h <= thr * thr)) return 0;
    }
    const float dl = d - KU * M;
    if (!(dl > 0.f) || !(h < dl * dl)) return 1;
    const float ux = fmaf(su, Vx, Dx), uy = fmaf(su, Vy, Dy), uz = fmaf(su, Vz, Dz);
    const float hu = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
    const float d2 = d * d;
    const float rem = fmaxf(d2 - hu, 0.f);
    const float w = sqrt_approx(rem * rA);                     // MUFU.SQRT: |rel err| <= 2^-22, in dw
    const float V1 = fabsf(q1.x) + fabsf(q1.y) + fabsf(q1.z) + fabsf(e.vx) + fabsf(e.vy) + fabsf(e.vz);
    constexpr float U = 1.0f / 16777216.0f;
    // the bound itself needs no IEEE division / sqrt: approximate MUFU results,
    // covered by the x2 safety factor
    const float rsA = rsqrt_approx(A);                         // 1 / sqrt(A)
    // s_u may lie far outside [0, L]: magnitudes along the line up to |s_u| enter M_u,
    // and the relative errors of A and of the reciprocal scale |s_u| and w
    // first-order bounds: |dDa| <= 11 u M_u, |dDV| <= 6 u V1,
    // s_u = -(Da.DV)/A -> |ds_u| <= 14 u M_u/sqrt(A) + 6 u V1 M_u/A + |s_u| (dA/A + 2u);
    // rem = d^2 - h_u -> |drem| <= 2 d 14 u M_u + A ds_u^2 + 2 u (d^2 + rem)
    const float Su = fmaxf(fabsf(su), L);
    const float Mu = M + Su * V1;
    const float relA = (12.f * U) * V1 * rsA + 5.f * U;
    const float dsu = (14.f * U) * Mu * rsA + (6.f * U) * V1 * Mu * rA + fabsf(su) * relA;
    const float drem = (28.f * U) * d * Mu + A * dsu * dsu + (2.f * U) * (d2 + rem);
    const float dw = w * (0.5f * drem * rcp_approx(rem) + 0.5f * relA + 4.f * U);
    // x2 safety on the first-order terms, + the rounding of s_u -+ w
    const float dst = fmaf(U, fabsf(su) + w, 2.f * (dsu + dw));
    const float lo = su - w, hi = su + w;
    tin = a + fminf(fmaxf(lo, 0.f), L);
    tout = a + fminf(fmaxf(hi, 0.f), L);
    // accepted offsets are within 8e-6 (b - a) of the exact ones; the output adds
    // its fp32 rounding (<= 0.5 ulp(t)): |t - t_exact| <= 1e-5 (b - a) + ulp(t)
    const float tol = (8e-6f) * L;
    const bool in_ok = (lo + dst < 0.f) || (dst <= tol);
    const bool out_ok = (hi - dst > L) || (dst <= tol);
    return (in_ok && out_ok) ? 2 : 1;
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
// interval within 8e-6 (b - a) of the exact one.  dlo / dhi: d rounded down / up.
__device__ __forceinline__ int refine_rel(float4 q0, float4 q1, float t0c, float t1c, float4 e0, float t1e, float vex,
                                          float vey, float vez, float dlo, float dhi, float &tin, float &tout) {
    constexpr float U = 1.0f / 16777216.0f;
    const float a = fmaxf(t0c, e0.w), b = fminf(t1c, t1e);
    if (!(a < b)) return 0;                                    // C5
    const float L = b - a, aq = a - q0.w, ae = a - e0.w;
    const float dpx = q0.x - e0.x, dpy = q0.y - e0.y, dpz = q0.z - e0.z;
    const float Dx = fmaf(-ae, vex, fmaf(aq, q1.x, dpx));
    const float Dy = fmaf(-ae, vey, fmaf(aq, q1.y, dpy));
    const float Dz = fmaf(-ae, vez, fmaf(aq, q1.z, dpz));
    const float Vx = q1.x - vex, Vy = q1.y - vey, Vz = q1.z - vez;
    // position error over the span: eD at s = 0 (roundings of dp, a - t0, the
    // velocities (<= 4u each) and the two FMAs), eV per unit s (velocities and V)
    const float V1e = fabsf(vex) + fabsf(vey) + fabsf(vez);
    const float D1 = fabsf(Dx) + fabsf(Dy) + fabsf(Dz), W1 = fabsf(Vx) + fabsf(Vy) + fabsf(Vz);
    const float eD = U * fmaf(7.f, fabsf(aq) * q1.w + fabsf(ae) * V1e, fabsf(dpx) + fabsf(dpy) + fabsf(dpz) + 2.f * D1);
    const float eV = U * fmaf(5.f, q1.w + V1e, W1);
    const float eP = 1.5f * fmaf(L, eV, eD);                   // x1.5 on the first-order bound
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
    const float ux = fmaf(su, Vx, Dx), uy = fmaf(su, Vy, Dy), uz = fmaf(su, Vz, Dz);
    const float hu = fmaf(ux, ux, fmaf(uy, uy, uz * uz));
    const float rem = fmaxf(fmaf(dhi, dhi, -hu), 0.f);
    const float w = sqrt_approx(rem * rA);
    const float lo = su - w, hi = su + w;
    // error of the unclamped ends: root sensitivity d eP / (A w) to the position
    // error, + roundings of h_u and d^2, of B (3u |D|_1 |V|_1 / A), of s_u and w
    const float dlt = fmaf(U, fabsf(su) + w,
                           1.5f * fmaf(fmaf(dhi, eP, (4.5f * U) * dhi * dhi), rcp_approx(A * w),
                                       fmaf((3.f * U) * D1 * W1, rA, U * fmaf(7.f, fabsf(su), 5.f * w))));
    tin = a + fminf(fmaxf(lo, 0.f), L);
    tout = a + fminf(fmaxf(hi, 0.f), L);
    const float tol = 8e-6f * L;
    const bool in_ok = (lo + dlt < 0.f) || (dlt <= tol);
    const bool out_ok = (hi - dlt > L) || (dlt <= tol);
    return (in_ok && out_ok) ? 2 : 1;
}

// ---------------------------------------------------------------------------
// A10: result append
// ---------------------------------------------------------------------------
struct OutArgs {
    Rec *buf;                        // pass buffer (chunked) or store (exact)
    unsigned long long cap;          // pass buffer slots
    uint32_t CS;                     // chunk size (slots)
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
    uint32_t refined, hits;
    uint32_t fn;                     // fp64 queue fill (< 32 between flushes)
    uint32_t rq[RQ_CAP], rj[RQ_CAP]; // refine queue: query row (| F64_FLAG), sorted entry position
    uint32_t fq[64], fj[64];         // fp64 queue: pairs the fp32 stages could not decide
};
constexpr uint32_t F64_FLAG = 0x80000000u;   // refine-queue entry already known to need fp64

__device__ __forceinline__ void warp_state_init(WarpState &W, int lane) {
    if (lane == 0) {
        W.ap_base = 0; W.ap_used = 0; W.ap_size = 0; W.ap_full = 0; W.refined = 0; W.hits = 0; W.fn = 0;
    }
    __syncwarp();
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
        if (size && lane == 0) o.chunk_used[base / o.CS] = used;
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
    if (hit) {
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
        if (size && lane == 0) o.chunk_used[base / o.CS] = used;
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
        if (!EXACT && !W.ap_full && W.ap_size) o.chunk_used[W.ap_base / o.CS] = W.ap_used;
        if (W.refined) atomicAdd(&o.st->refined, (unsigned long long)W.refined);
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

// Evaluate queued pairs [base, base + n), n <= 32 (lane k takes pair k): certain
// hits with an accurate fp32 interval are appended; the undecided go to the fp64
// queue, which is evaluated 32 at a time (a warp-wide fp64 pass per 32 pairs that
// need it, not per flush).  Entries flagged F64_FLAG skip the fp32 stage.
template <bool EXACT>
__device__ __forceinline__ void flush_refine(const PairCtx *C, WarpState *W, uint32_t n, uint32_t base = 0) {
    const int lane = threadIdx.x & 31;
    const bool v = (uint32_t)lane < n;
    const uint32_t qraw = v ? W->rq[base + lane] : 0u, j = v ? W->rj[base + lane] : 0u;
    const uint32_t q = qraw & ~F64_FLAG;
    __syncwarp();                    // queue slots read: later queue_add may reuse them
    float tin = 0.f, tout = 0.f;
    int k = 0;
    if (v) {
        if (qraw & F64_FLAG) {
            k = 1;
        } else {
            const float4 qa = __ldg(C->Q + 2 * (uint64_t)q), qb = __ldg(C->Q + 2 * (uint64_t)q + 1);
            const float4 ea = __ldg(C->rec + 2 * (uint64_t)j), eb = __ldg(C->rec + 2 * (uint64_t)j + 1);
            const QConst qc = make_qconst(qa, qb, C->T0, C->T1);
            const ECand e = make_ecand(ea, eb);
            k = refine_rel(make_float4(qc.px, qc.py, qc.pz, qc.t0),
                           make_float4(qc.vx, qc.vy, qc.vz, fabsf(qc.vx) + fabsf(qc.vy) + fabsf(qc.vz)), qc.t0c, qc.t1c,
                           make_float4(e.px, e.py, e.pz, e.t0), e.t1, e.vx, e.vy, e.vz, C->dlo, C->d, tin, tout);
        }
    }
    const bool hit = (k == 2), need64 = (k == 1);
    const uint32_t eid = hit ? __ldg(C->perm + j) : 0u;
    Rec r{q, eid, tin, tout};
    append<EXACT>(C->o, *W, hit, r, lane);
    const unsigned hm = __ballot_sync(FULL, hit);
    if (hit) {   // per-query counts, aggregated over the lanes of the same query
        const unsigned peers = __match_any_sync(hm, q);
        if ((peers & ((1u << lane) - 1u)) == 0) atomicAdd(&C->o.qcount[q], (uint32_t)__popc(peers));
    }
    // undecided pairs -> fp64 queue
    const unsigned m64 = __ballot_sync(FULL, need64);
    const uint32_t fn = W->fn;
    if (need64) {
        const uint32_t pos = fn + __popc(m64 & ((1u << lane) - 1u));
        W->fq[pos] = q;
        W->fj[pos] = j;
    }
    __syncwarp();
    if (lane == 0) { W->hits += __popc(hm); W->fn = fn + __popc(m64); }
    __syncwarp();
    if (fn + __popc(m64) >= 32) flush64<EXACT>(C, W, 32);
}

// warp-wide: queue the pairs whose fp32 filter passed (no flush here)
__device__ __forceinline__ void queue_add(WarpState &W, uint32_t &qn, bool maybe, uint32_t qid, uint32_t j, int lane) {
    const unsigned mb = __ballot_sync(FULL, maybe);
    if (!mb) return;
    const uint32_t pos = qn + __popc(mb & ((1u << lane) - 1u));
    if (maybe) { W.rq[pos] = qid; W.rj[pos] = j; }
    qn += __popc(mb);
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
    if (m0) { const uint32_t k = p + __popc(b0 & lt); W.rq[k] = qid; W.rj[k] = j0; }
    p += __popc(b0);
    if (m1) { const uint32_t k = p + __popc(b1 & lt); W.rq[k] = qid; W.rj[k] = j1; }
    p += __popc(b1);
    if (m2) { const uint32_t k = p + __popc(b2 & lt); W.rq[k] = qid; W.rj[k] = j2; }
    p += __popc(b2);
    if (m3) { const uint32_t k = p + __popc(b3 & lt); W.rq[k] = qid; W.rj[k] = j3; }
    qn = p + __popc(b3);
}

// warp-wide: evaluate queued pairs in fp64, 32 at a time, while >= 32 are queued
template <bool EXACT>
__device__ __forceinline__ void queue_drain(const PairCtx *C, WarpState &W, uint32_t &qn, int lane) {
    if (qn < 32) return;
    __syncwarp();
    uint32_t head = 0;
    do {                                 // flush 32 at a time in place
        flush_refine<EXACT>(C, &W, 32, head);
        head += 32;
    } while (qn - head >= 32);
    const uint32_t rest = qn - head;     // move the remainder to the front
    uint32_t t1 = 0, t2 = 0;
    if ((uint32_t)lane < rest) { t1 = W.rq[head + lane]; t2 = W.rj[head + lane]; }
    __syncwarp();
    if ((uint32_t)lane < rest) { W.rq[lane] = t1; W.rj[lane] = t2; }
    __syncwarp();
    qn = rest;
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
        A.keys[p] = ((uint32_t)(S.sel + 1) << 13) | (S.lo >> A.lo_shift);
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
        if (lo < hi) { T.ulo = lo; T.uhi = hi; } else { T.ulo = T.uhi = 0; }
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
    ch = ch < 64 ? 64 : (ch > 8192 ? 8192 : ch);
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) st->ch = (uint32_t)ch;
    if (t < ntiles) len_to_chunks[t] = (uint32_t)((len_to_chunks[t] + ch - 1) / ch);
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
    uint32_t ntiles;
    float df;                        // filter_abs threshold: d * (1 + 2^-20), rounded up
    float tc;                        // filter_abs time origin (middle of the index's time extent)
};

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
                                float T1, DevStats *st) {
    const int lane = threadIdx.x & 31;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    if (n == 0) return;
    const uint32_t p = (uint32_t)(((uint64_t)w * n) / nw + n / (2 * nw));
    if (p >= n) return;
    const Sched e = S[p];
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
        pass += filter_pair(q0, q1, qc.t0c, qc.t1c, ec, d) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pass += __shfl_xor_sync(FULL, pass, o);
    if (lane == 0) {
        atomicAdd(&st->probe_pass, pass);
        atomicAdd(&st->probe_total, m);
    }
}

struct __align__(16) RangeWarpSmem {
    float4 q[32][6];                 // group query slot g: (p0, t0) (v, |v|_1) (t0c, t1c, |p1 - p0|_1, -)
                                     // and the absolute form (c, m) (v, t0c') (t1c', lo, hi, qid)
    WarpState ws;                    // append chunk, refine queue (slot g, sorted position j), fp64 queue
    uint32_t cnt[32];                // records of slot g found by the refine path in this work item
    uint32_t qn;                     // refine queue fill
};

// Evaluate refine-queue entries [base, base + n), n <= 32 (lane k takes entry
// k): (slot g, sorted entry position j) -> refine_rel with the query's terms from
// shared memory; certain hits are appended, undecided pairs go to the fp64 queue.
template <bool EXACT>
__device__ __noinline__ void range_refine(const RangeArgs *A, RangeWarpSmem *W, uint32_t n, uint32_t base) {
    const int lane = threadIdx.x & 31;
    const bool v = (uint32_t)lane < n;
    const uint32_t g = v ? W->ws.rq[base + lane] : 0u, j = v ? W->ws.rj[base + lane] : 0u;
    __syncwarp();                    // queue slots read: later queue additions may reuse them
    float tin = 0.f, tout = 0.f;
    int k = 0;
    uint32_t qid = 0;
    if (v) {
        const float4 q0 = W->q[g][0], q1 = W->q[g][1], q2 = W->q[g][2];
        qid = __float_as_uint(W->q[g][5].w);
        const ECand e = make_ecand(__ldg(A->pc.rec + 2 * (uint64_t)j), __ldg(A->pc.rec + 2 * (uint64_t)j + 1));
        k = refine_rel(q0, q1, q2.x, q2.y, make_float4(e.px, e.py, e.pz, e.t0), e.t1, e.vx, e.vy, e.vz, A->pc.dlo,
                       A->pc.d, tin, tout);
    }
    const bool hit = (k == 2), need64 = (k == 1);
    const Rec r{qid, hit ? __ldg(A->pc.perm + j) : 0u, tin, tout};
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
    if (lane == 0) { W->ws.hits += __popc(hm); W->ws.fn = fn + __popc(m64); }
    __syncwarp();
    if (fn + __popc(m64) >= 32) flush64<EXACT>(&A->pc, &W->ws, 32);
}

// warp-wide: evaluate the newest 32 queued pairs while >= 32 are queued
template <bool EXACT>
__device__ __forceinline__ void range_drain(const RangeArgs *A, RangeWarpSmem &W, uint32_t &qn) {
    while (qn >= 32) {
        __syncwarp();
        qn -= 32;
        range_refine<EXACT>(A, &W, 32, qn);
    }
}

// Dense windows: for the lane's two candidates against query slot g, in the
// relative form: in0/in1 = both span ends certainly within d (then the whole
// shared span [a, b] is within d: the squared distance is convex in t; the
// pair's interval is exactly [a, b]), ps0/ps1 = the closest approach passes the
// filter.  Certainty margin KU M, M = |p0q - p0e|_1 + |p1q - p0q|_1 + |p1e -
// p0e|_1 (the relative-form bound of DESIGN.md §5 holds at every point of the
// span, so at both ends).  Packed FP32x2 per candidate pair.
__device__ __forceinline__ void dense_test2(float4 q0, float4 q1, float4 q2, const ECand &e0, const ECand &e1, float d,
                                            bool &in0, bool &in1, bool &ps0, bool &ps1, float &a0, float &b0,
                                            float &a1, float &b1) {
    a0 = fmaxf(q2.x, e0.t0); b0 = fminf(q2.y, e0.t1);
    a1 = fmaxf(q2.x, e1.t0); b1 = fminf(q2.y, e1.t1);
    const f32x2 a = pk2(a0, a1);
    const f32x2 L = sub2(pk2(b0, b1), a);
    const f32x2 aq = sub2(a, bc2(q0.w)), nae = sub2(pk2(e0.t0, e1.t0), a);
    const f32x2 dpx = sub2(bc2(q0.x), pk2(e0.px, e1.px)), dpy = sub2(bc2(q0.y), pk2(e0.py, e1.py)),
                dpz = sub2(bc2(q0.z), pk2(e0.pz, e1.pz));
    const f32x2 evx = pk2(e0.vx, e1.vx), evy = pk2(e0.vy, e1.vy), evz = pk2(e0.vz, e1.vz);
    const f32x2 Dx = fma2(nae, evx, fma2(aq, bc2(q1.x), dpx));
    const f32x2 Dy = fma2(nae, evy, fma2(aq, bc2(q1.y), dpy));
    const f32x2 Dz = fma2(nae, evz, fma2(aq, bc2(q1.z), dpz));
    const f32x2 Vx = sub2(bc2(q1.x), evx), Vy = sub2(bc2(q1.y), evy), Vz = sub2(bc2(q1.z), evz);
    const f32x2 ybx = fma2(L, Vx, Dx), yby = fma2(L, Vy, Dy), ybz = fma2(L, Vz, Dz);
    const f32x2 ha = fma2(Dx, Dx, fma2(Dy, Dy, mul2(Dz, Dz)));
    const f32x2 hb = fma2(ybx, ybx, fma2(yby, yby, mul2(ybz, ybz)));
    float x0, x1, y0, y1, z0, z1;
    upk2(dpx, x0, x1);
    upk2(dpy, y0, y1);
    upk2(dpz, z0, z1);
    const f32x2 M = add2(pk2(fabsf(x0) + fabsf(y0) + fabsf(z0), fabsf(x1) + fabsf(y1) + fabsf(z1)),
                         add2(bc2(q2.z), pk2(e0.ext, e1.ext)));
    const f32x2 thr = fma2(bc2(KU), M, bc2(d)), dl = fma2(bc2(-KU), M, bc2(d));
    const f32x2 A = fma2(Vx, Vx, fma2(Vy, Vy, mul2(Vz, Vz)));
    const f32x2 B = fma2(Dx, Vx, fma2(Dy, Vy, mul2(Dz, Vz)));
    float A0, A1, L0, L1, u0, u1;
    upk2(A, A0, A1);
    upk2(L, L0, L1);
    upk2(mul2(B, pk2(rcp_approx(A0), rcp_approx(A1))), u0, u1);
    const f32x2 sv = pk2(fminf(fmaxf(-u0, 0.f), L0), fminf(fmaxf(-u1, 0.f), L1));
    const f32x2 yx = fma2(sv, Vx, Dx), yy = fma2(sv, Vy, Dy), yz = fma2(sv, Vz, Dz);
    const f32x2 h = fma2(yx, yx, fma2(yy, yy, mul2(yz, yz)));
    float ha0, ha1, hb0, hb1, h0, h1, t0, t1, l0, l1, dl0, dl1;
    upk2(ha, ha0, ha1);
    upk2(hb, hb0, hb1);
    upk2(h, h0, h1);
    upk2(mul2(thr, thr), t0, t1);
    upk2(mul2(dl, dl), l0, l1);
    upk2(dl, dl0, dl1);
    in0 = (a0 < b0) & (dl0 > 0.f) & (ha0 < l0) & (hb0 < l0);
    in1 = (a1 < b1) & (dl1 > 0.f) & (ha1 < l1) & (hb1 < l1);
    ps0 = (a0 < b0) & (h0 <= t0);
    ps1 = (a1 < b1) & (h1 <= t1);
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
template <bool EXACT>
__global__ void __launch_bounds__(PT, RANGE_BPS) k_pair_range(const __grid_constant__ RangeArgs A) {
    __shared__ RangeWarpSmem sm[PT / 32];
    const int lane = threadIdx.x & 31;
    RangeWarpSmem &W = sm[threadIdx.x >> 5];
    DevStats *st = A.pc.o.st;
    const uint32_t total = A.item_start[A.ntiles];
    const uint32_t CH = st->ch;
    const float d = A.pc.d;
    const float df = A.df;
    warp_state_init(W.ws, lane);
    W.cnt[lane] = 0;
    uint32_t qn = 0;                         // refine queue fill (warp-uniform)
    __syncwarp();
    unsigned long long exec = 0, direct_hits = 0;
    bool dense = false;                      // warp-uniform: the last window was hit-heavy
    while (true) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(&st->work_ctr, 1u);
        item = __shfl_sync(FULL, item, 0);
        if (item >= total) break;
        uint32_t lo = 0, hi = A.ntiles;
        while (hi - lo > 1) {
            uint32_t mid = (lo + hi) >> 1;
            if (A.item_start[mid] <= item) lo = mid; else hi = mid;
        }
        const Tile T = A.tiles[lo];
        const uint32_t chunk = item - A.item_start[lo];
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
            __syncwarp();
        }
        uint32_t wlo = my_lo, whi = my_hi;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wlo = min(wlo, __shfl_xor_sync(FULL, wlo, o));
            whi = max(whi, __shfl_xor_sync(FULL, whi, o));
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
        uint32_t base = wlo;
        while (base < whi) {
            const uint32_t cend = min(base + WIN, whi);
            unsigned mask = __ballot_sync(FULL, my_lo < cend && my_hi > base);
            const unsigned wmask = mask;
            if (!mask) {                       // skip the gap to the next range start
                uint32_t nxt = (my_lo >= cend && my_lo < my_hi) ? my_lo : 0xffffffffu;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) nxt = min(nxt, __shfl_xor_sync(FULL, nxt, o));
                base = nxt;
                continue;
            }
            // ---- worker side: lane = candidate
            const uint32_t c0 = base + lane, c1 = c0 + 32, c2 = c0 + 64, c3 = c0 + 96;
            uint32_t j0, j1, j2, j3;
            exec += (unsigned long long)(cend - base) * __popc(mask);
            uint32_t wpass = 0;                // filter passes of this window (all queries)
            if (dense) {
                // the window in two halves of 64 candidates (two per lane), each against
                // every query slot: one copy of the step, two candidate terms live
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const uint32_t ca = c0 + 64u * h, cb = ca + 32u;
                    if (ca - lane >= cend) break;
                    uint32_t ja, jb;
                    float4 a, b;
                    load_cand(ca, ca < cend, ja, a, b);
                    const ECand ea = make_ecand(a, b);
                    load_cand(cb, cb < cend, jb, a, b);
                    const ECand eb = make_ecand(a, b);
                    // entry rows, loaded once per window (not per hit)
                    const uint32_t ida = ca < cend ? __ldg(A.pc.perm + ja) : 0u, idb = cb < cend ? __ldg(A.pc.perm + jb) : 0u;
                    unsigned m = wmask;
                    while (m) {
                        const int g = __ffs(m) - 1;
                        m &= m - 1;
                        const float4 q0 = W.q[g][0], q1 = W.q[g][1], q2 = W.q[g][2], q5 = W.q[g][5];
                        const uint32_t glo = __float_as_uint(q5.y), ghi = __float_as_uint(q5.z);
                        const uint32_t qid = __float_as_uint(q5.w);
                        bool in0, in1, ps0, ps1;
                        float a0, b0, a1, b1;
                        dense_test2(q0, q1, q2, ea, eb, d, in0, in1, ps0, ps1, a0, b0, a1, b1);
                        // slot c valid for slot g iff glo <= c < ghi (ghi <= whi) and c < cend
                        const bool r0 = (ca - glo < ghi - glo) && (ca < cend);
                        const bool r1 = (cb - glo < ghi - glo) && (cb < cend);
                        in0 &= r0; in1 &= r1;
                        ps0 = ps0 & r0 & !in0;
                        ps1 = ps1 & r1 & !in1;
                        const unsigned bi0 = __ballot_sync(FULL, in0), bi1 = __ballot_sync(FULL, in1);
                        const unsigned bp0 = __ballot_sync(FULL, ps0), bp1 = __ballot_sync(FULL, ps1);
                        wpass += __popc(bi0) + __popc(bi1) + __popc(bp0) + __popc(bp1);
                        if (bi0 | bi1) {
                            append2<EXACT>(A.pc.o, W.ws, in0, in1, bi0, bi1, Rec{qid, ida, a0, b0},
                                           Rec{qid, idb, a1, b1}, lane);
                            const uint32_t hg = __popc(bi0) + __popc(bi1);
                            direct_hits += hg;
                            if (lane == g) owner_hits += hg;
                        }
                        if (bp0 | bp1) {
                            queue_add(W.ws, qn, ps0, (uint32_t)g, ja, lane);
                            queue_add(W.ws, qn, ps1, (uint32_t)g, jb, lane);
                            range_drain<EXACT>(&A, W, qn);
                        }
                    }
                }
            } else {
                FSeg2 f01, f23;
                {
                    float4 a0, b0, a1, b1;
                    load_cand(c0, c0 < cend, j0, a0, b0);
                    load_cand(c1, c1 < cend, j1, a1, b1);
                    f01 = make_fseg2(make_fseg(a0, b0, A.tc), make_fseg(a1, b1, A.tc));
                    load_cand(c2, c2 < cend, j2, a0, b0);
                    load_cand(c3, c3 < cend, j3, a1, b1);
                    f23 = make_fseg2(make_fseg(a0, b0, A.tc), make_fseg(a1, b1, A.tc));
                }
                while (mask) {
                    const int g = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const float4 n0 = W.q[g][3], n1 = W.q[g][4], n2 = W.q[g][5];
                    const uint32_t glo = __float_as_uint(n2.y), ghi = __float_as_uint(n2.z);
                    bool m0, m1, m2, m3;
                    filter_abs2(n0, n1, n1.w, n2.x, f01, df, m0, m1);
                    filter_abs2(n0, n1, n1.w, n2.x, f23, df, m2, m3);
                    // warp-uniform: unless the query's range covers all WIN candidate slots
                    // (then all are valid: ghi <= whi), test each slot against the range
                    // (c < ghi <= whi implies c < cend: no separate validity test)
                    if (glo > base || ghi - base < WIN) {
                        const uint32_t r0 = c0 - glo, gw = ghi - glo;
                        m0 &= r0 < gw; m1 &= r0 + 32 < gw; m2 &= r0 + 64 < gw; m3 &= r0 + 96 < gw;
                    }
                    if (!__any_sync(FULL, (m0 | m1) | (m2 | m3))) continue;
                    const uint32_t q0n = qn;
                    queue_add4(W.ws, qn, m0, m1, m2, m3, (uint32_t)g, j0, j1, j2, j3, lane);
                    wpass += qn - q0n;
                    range_drain<EXACT>(&A, W, qn);
                }
            }
            // switch to the fused dense path once >= HYST_HI % of the window's pairs pass,
            // back to the sparse path below HYST_LO % (hysteresis: a window mix near one
            // threshold would toggle between the paths)
            dense = 100u * wpass >= (uint32_t)(dense ? HYST_LO : HYST_HI) * __popc(wmask) * (cend - base);
            base = cend;
        }
        // ---- item end: the queue refers to this group's slots
        if (qn) {
            __syncwarp();
            range_refine<EXACT>(&A, &W, qn, 0);
            qn = 0;
        }
        __syncwarp();
        const uint32_t cq = owner_hits + W.cnt[lane];
        W.cnt[lane] = 0;
        if (active && cq) atomicAdd(&A.pc.o.qcount[S.qid], cq);
        __syncwarp();
    }
    __syncwarp();
    if (W.ws.fn) flush64<EXACT>(&A.pc, &W.ws, W.ws.fn);
    warp_state_finish<EXACT>(A.pc.o, W.ws, lane);
    if (lane == 0 && exec) atomicAdd(&st->executed, exec);
    if (lane == 0 && direct_hits) atomicAdd(&st->hits, direct_hits);
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
__device__ __forceinline__ uint32_t spread3(uint32_t x) {      // 10 bits -> every third bit
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

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
        if (!literal && a0 < a1) {
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

struct SpatialArgs {
    PairCtx pc;                      // rec / perm = the cell-ordered copies (indexed by A position)
    const uint32_t *ecell;           // packed min cell of entry A[i]
    const uint32_t *grab_row;        // [ngrab + 1] row of the first slot of each grab
    const uint32_t *cell_off;
    const int4 *qbox;                // [2 * nlist]: lo (w = query row), hi
    const uint32_t *row_q, *row_alo, *row_cxy;   // work items (query, cell): query, slice start, packed cell
    const unsigned long long *slot_start;   // [nrows + 1]
    const uint32_t *slot_row;        // [slots] row of each slot (small searches), else nullptr
    unsigned long long slot_lo, slot_hi;   // the slots this launch evaluates (tds_search_part: a sub-range)
    uint32_t nrows;
    FsgGrid G;
};

// Small searches (<= SLOT_ROW_MAX slots): the row of every slot, found by one
// thread per slot in parallel, so the pair kernel needs one load per row change
// instead of a dependent binary search (most (query, cell-row) items of a small
// search are empty after time trimming: on Random-1M-shaped data a row change
// per slot, each a ~10-level chain of L2 loads, set the kernel time).
constexpr unsigned long long SLOT_ROW_MAX = 1ull << 22;

__device__ __forceinline__ uint32_t find_row(const unsigned long long *ss, uint32_t lo, uint32_t hi,
                                             unsigned long long s) {
    // last r in [lo, hi) with ss[r] <= s
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (ss[mid] <= s) lo = mid; else hi = mid;
    }
    return lo;
}

// slot_row[k] = row of slot base + k
__global__ void k_slot_rows(const unsigned long long *__restrict__ ss, uint32_t nrows, unsigned long long base,
                            uint64_t nslots, uint32_t *__restrict__ slot_row) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nslots) slot_row[k] = find_row(ss, 0, nrows, base + k);
}

// grab_row[k] = row of slot base + k * SP_GRAB (clamped to the last slot < end)
__global__ void k_grab_rows(const unsigned long long *__restrict__ ss, uint32_t nrows, unsigned long long base,
                            unsigned long long end, uint64_t ngrab, uint32_t *__restrict__ grab_row) {
    uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > ngrab) return;
    unsigned long long s = base + k * SP_GRAB;
    if (s >= end) s = end > base ? end - 1 : base;
    grab_row[k] = find_row(ss, 0, nrows, s);
}

// Result-size probe of a GPUSpatial search: the fraction of passing pair tests
// (relative-form filter + the reference-cell rule) on slots sampled evenly over
// [s_lo, s_hi), one per thread.
__global__ void k_density_probe_spatial(const unsigned long long *__restrict__ ss, uint32_t nrows,
                                        unsigned long long s_lo, unsigned long long s_hi,
                                        const uint32_t *__restrict__ row_q, const uint32_t *__restrict__ row_alo,
                                        const uint32_t *__restrict__ row_cxy, const int4 *__restrict__ qbox,
                                        const uint32_t *__restrict__ ecell, const float4 *__restrict__ Q,
                                        const float4 *__restrict__ frec, float d, float T0, float T1, DevStats *st) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    const unsigned long long n = s_hi - s_lo;
    uint32_t pass = 0, tot = 0;
    if (n) {
        const unsigned long long sl = s_lo + (unsigned long long)(((unsigned __int128)n * (2 * t + 1)) / (2ull * nt));
        const uint32_t r = find_row(ss, 0, nrows, sl);
        const uint32_t i = row_alo[r] + (uint32_t)(sl - ss[r]);
        const int4 qlo = qbox[2 * row_q[r]];
        const uint32_t m0 = ecell[i];
        const int rx = max((int)(m0 >> 21), qlo.x), ry = max((int)((m0 >> 10) & 0x7ffu), qlo.y);
        const int rz = max((int)(m0 & 0x3ffu), qlo.z);
        tot = 1;
        if (pack_cell(rx, ry, rz) == row_cxy[r]) {
            const QConst qc = make_qconst(__ldg(Q + 2 * (uint64_t)qlo.w), __ldg(Q + 2 * (uint64_t)qlo.w + 1), T0, T1);
            pass = filter_pair(make_float4(qc.px, qc.py, qc.pz, qc.t0), make_float4(qc.vx, qc.vy, qc.vz, qc.ext),
                               qc.t0c, qc.t1c, make_ecand(__ldg(frec + 2 * (uint64_t)i), __ldg(frec + 2 * (uint64_t)i + 1)),
                               d) ? 1u : 0u;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pass += __shfl_xor_sync(FULL, pass, o);
        tot += __shfl_xor_sync(FULL, tot, o);
    }
    if ((threadIdx.x & 31) == 0 && tot) {
        atomicAdd(&st->probe_pass, pass);
        atomicAdd(&st->probe_total, tot);
    }
}

// lane = candidate slot of the flattened (query, cell row) work list; warps grab
// 32 x SP_PER_LANE consecutive slots at a time (dynamic load balance).
template <bool EXACT>
__global__ void __launch_bounds__(PT, SPATIAL_BPS) k_pair_spatial(const __grid_constant__ SpatialArgs A) {
    __shared__ WarpState sm[PT / 32];
    const int lane = threadIdx.x & 31;
    WarpState &W = sm[threadIdx.x >> 5];
    DevStats *st = A.pc.o.st;
    const unsigned long long total = A.slot_hi;
    warp_state_init(W, lane);
    uint32_t qn = 0;
    unsigned long long exec = 0, direct_hits = 0;
    uint32_t cur_p = 0xffffffffu;
    uint32_t cur_qrow = 0;
    QConst q = make_qconst(make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 1.f), A.pc.T0, A.pc.T1);
    int4 qlo = make_int4(0, 0, 0, 0);
    constexpr int SB = 4;                       // slots per lane per batch (loads hoisted)
    while (true) {
        unsigned gi = 0;
        if (lane == 0) gi = atomicAdd(&st->work_ctr, 1u);
        gi = __shfl_sync(FULL, gi, 0);
        const unsigned long long B = A.slot_lo + (unsigned long long)gi * SP_GRAB;
        if (B >= total) break;
        const unsigned long long Bend = min(B + SP_GRAB, total);
        const uint32_t rlo = A.grab_row[gi], rhi = A.grab_row[gi + 1] + 1;
        // row of this lane's first slot (small search inside the grab's row range);
        // later slots advance the row linearly (rows are consecutive in slot order)
        uint32_t r = A.slot_row ? A.slot_row[min(B + lane, Bend - 1) - A.slot_lo]
                                : find_row(A.slot_start, rlo, rhi, min(B + lane, Bend - 1));
        unsigned long long r_start = A.slot_start[r], r_next = A.slot_start[r + 1];
        uint32_t r_alo = A.row_alo[r], r_cxy = A.row_cxy[r], r_p = A.row_q[r];
        exec += Bend - B;
#pragma unroll 1
        for (int u0 = 0; u0 < SP_PER_LANE; u0 += SB) {
            uint32_t ii[SB], cxy[SB], pp[SB];
            bool vv[SB];
#pragma unroll
            for (int u = 0; u < SB; ++u) {
                const unsigned long long s = B + (unsigned long long)(u0 + u) * 32 + lane;
                vv[u] = s < Bend;
                if (vv[u] && s >= r_next) {
                    // next item holding slot s (binary search: many (query, cell) items are empty)
                    r = A.slot_row ? A.slot_row[s - A.slot_lo] : find_row(A.slot_start, r + 1, rhi, s);
                    r_start = A.slot_start[r];
                    r_next = A.slot_start[r + 1];
                    r_alo = A.row_alo[r];
                    r_cxy = A.row_cxy[r];
                    r_p = A.row_q[r];
                }
                ii[u] = vv[u] ? r_alo + (uint32_t)(s - r_start) : 0u;
                cxy[u] = r_cxy;
                pp[u] = r_p;
            }
            float4 ea[SB], eb[SB];
            uint32_t ec[SB];
#pragma unroll
            for (int u = 0; u < SB; ++u) {          // coalesced: consecutive slots, consecutive i
                ea[u] = __ldg(A.pc.rec + 2 * (uint64_t)ii[u]);
                eb[u] = __ldg(A.pc.rec + 2 * (uint64_t)ii[u] + 1);
                ec[u] = __ldg(A.ecell + ii[u]);
            }
#pragma unroll
            for (int u = 0; u < SB; ++u) {
                int kk = 0;
                if (vv[u]) {
                    if (pp[u] != cur_p) {
                        cur_p = pp[u];
                        qlo = A.qbox[2 * cur_p];
                        cur_qrow = (uint32_t)qlo.w;
                        q = make_qconst(__ldg(A.pc.Q + 2 * (uint64_t)cur_qrow),
                                        __ldg(A.pc.Q + 2 * (uint64_t)cur_qrow + 1), A.pc.T0, A.pc.T1);
                    }
                    // duplicate avoidance: test (q, e) only in the first cell (index-space
                    // min corner) of cells(e) ∩ cells(q) (replaces the host filter of P:558-559)
                    const uint32_t m0 = ec[u];
                    const int rx = max((int)(m0 >> 21), qlo.x), ry = max((int)((m0 >> 10) & 0x7ffu), qlo.y);
                    const int rz = max((int)(m0 & 0x3ffu), qlo.z);
                    const bool first = pack_cell(rx, ry, rz) == cxy[u];
                    if (first) kk = filter_pair(make_float4(q.px, q.py, q.pz, q.t0),
                                                make_float4(q.vx, q.vy, q.vz, q.ext), q.t0c, q.t1c,
                                                make_ecand(ea[u], eb[u]), A.pc.d) ? 1 : 0;
                }
                // passes are queued; the flush classifies (fp32 interval or fp64) 32 at a time
                queue_add(W, qn, kk == 1, cur_qrow, ii[u], lane);
            }
            queue_drain<EXACT>(&A.pc, W, qn, lane);
        }
    }
    __syncwarp();                    // last queue_add writes -> flush reads
    if (qn) flush_refine<EXACT>(&A.pc, &W, qn);
    if (W.fn) flush64<EXACT>(&A.pc, &W, W.fn);
    warp_state_finish<EXACT>(A.pc.o, W, lane);
    if (lane == 0 && exec) atomicAdd(&st->executed, exec);
    if (lane == 0 && direct_hits) atomicAdd(&st->hits, direct_hits);
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

// redo flags of schedule entries (range variants) / query list (spatial)
__global__ void k_redo_flags_sched(const Sched *__restrict__ S, uint32_t n, const uint8_t *__restrict__ redo,
                                   uint32_t *__restrict__ flag) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) flag[p] = redo[S[p].qid];
}

__global__ void k_compact_sched(const Sched *__restrict__ S, uint32_t n, const uint32_t *__restrict__ flag,
                                const uint32_t *__restrict__ pos, Sched *__restrict__ out,
                                const uint32_t *__restrict__ qcount, uint32_t *__restrict__ cnt_out) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && flag[p]) {
        out[pos[p]] = S[p];
        cnt_out[pos[p]] = qcount[S[p].qid];
    }
}

__global__ void k_set_qoff(const Sched *__restrict__ S, uint32_t n, const uint64_t *__restrict__ off,
                           unsigned long long base, unsigned long long *__restrict__ qoff) {
    uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) qoff[S[p].qid] = base + off[p];
}

__global__ void k_u32_to_u64(const uint32_t *__restrict__ a, uint64_t n, uint64_t *__restrict__ b) {
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
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

// GPUSpatial: parts at query granularity; query p's slots start at ss[row_start[p]]
__global__ void k_part_bounds_spatial(const unsigned long long *__restrict__ ss, const uint32_t *__restrict__ row_start,
                                      uint32_t n, uint32_t part, uint32_t nparts, DevStats *st) {
    if (threadIdx.x || blockIdx.x) return;
    auto f = [&](uint32_t p) { return ss[row_start[p]]; };
    const unsigned long long total = f(n);
    const uint32_t lo = part == 0 ? 0u : part_lower_bound(f, n, part_target(total, part, nparts));
    uint32_t hi = part + 1 >= nparts ? n : part_lower_bound(f, n, part_target(total, part + 1, nparts));
    if (hi < lo) hi = lo;
    st->part_lo = lo;
    st->part_hi = hi;
    st->part_slot_lo = f(lo);
    st->part_slot_hi = f(hi);
    st->pair_tests = f(hi) - f(lo);
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

int fsg_literal() {
    const char *e = getenv("TDS_FSG_LITERAL");
    return (e && e[0] == '1') ? 1 : 0;
}

// build tiles + work items for schedule entries [lo, hi) of the sorted schedule
// (the category counts in st describe the whole sorted schedule)
uint32_t plan_items(const Sched *sched, uint32_t lo, uint32_t hi, DevStats *st, DBuf<Tile> &tiles,
                    DBuf<uint32_t> &item_start, cudaStream_t s, int part_range = 0) {
    uint32_t n = hi - lo;
    uint32_t max_tiles = n / 32 + 5;     // also bounds the tiles of any sub-range (part_range)
    tiles = DBuf<Tile>(max_tiles, s);
    item_start = DBuf<uint32_t>(max_tiles + 1, s);
    k_make_tiles<<<nblk((uint64_t)max_tiles * 32), 256, 0, s>>>(sched, lo, n, st, lo, hi, tiles.p, max_tiles,
                                                                item_start.p, part_range);
    TDS_CHECK_LAUNCH();
    uint32_t target = (uint32_t)persistent_blocks(RANGE_BPS) * (PT / 32) * 4;
    k_tile_chunks<<<nblk(max_tiles), 256, 0, s>>>(item_start.p, max_tiles, &st->union_total, st, target);
    TDS_CHECK_LAUNCH();
    exclusive_scan_u32(item_start.p, item_start.p, max_tiles + 1, nullptr, s);
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

    // ---- A6: queries are validated inside the schedule kernels; GPUTemporal /
    // GPUSpatioTemporal order them by (selector, range start) below, which subsumes
    // the t_start sort of P:681-682 (range starts are monotone in t_start); FSG
    // keeps input order
    // TDS_AUTO: schedule GPUSpatioTemporal (counting the GPUTemporal ranges too),
    // then keep whichever plan has the lower estimated cost (below)
    const int req_kind = kind;
    if (kind == TDS_AUTO) kind = (idx->kinds & TDS_SPATIOTEMPORAL) ? TDS_SPATIOTEMPORAL : TDS_TEMPORAL;
    const bool spatial = (kind == TDS_SPATIAL);
    DBuf<uint32_t> keys, order;
    if (!spatial) { keys = DBuf<uint32_t>(n, s); order = DBuf<uint32_t>(n, s); }

    // ---- A7: schedule ---------------------------------------------------------
    DBuf<Sched> sched;
    DBuf<Tile> tiles;
    DBuf<uint32_t> item_start;
    uint32_t ntiles = 0;
    // spatial work list
    FsgGrid G{};
    DBuf<int4> qbox;
    DBuf<uint32_t> row_start, row_q, row_alo, row_len, row_cxy;
    DBuf<unsigned long long> slot_start;
    DBuf<uint32_t> fsg_order;          // GPUSpatial query order (rows of Q)
    uint32_t nrows = 0;
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
        a.st = dst.p;
        a.count_t = (req_kind == TDS_AUTO && a.use_st) ? 1 : 0;
        a.rec = idx->rec;
        a.tight = tight_ranges();
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
        // sort S by (array selector, range start): one stable radix sort
        radix_sort_pairs(keys.p, order.p, n, 0, 16, s);
        {
            DBuf<Sched> tmp(n, s);
            k_permute_sched<<<nblk(n), 256, 0, s>>>(sched.p, order.p, n, tmp.p);
            TDS_CHECK_LAUNCH();
            std::swap(sched.p, tmp.p);
        }
        if (nparts > 1) {
            // this part's slice of the sorted schedule: equal shares of the exact pair tests
            DBuf<uint64_t> w(n + 1, s);
            k_sched_work<<<nblk(n + 1), 256, 0, s>>>(sched.p, n, w.p);
            TDS_CHECK_LAUNCH();
            exclusive_scan_u64(w.p, w.p, n + 1, nullptr, s);
            k_part_bounds<<<1, 32, 0, s>>>(w.p, n, part, nparts, dst.p);
            TDS_CHECK_LAUNCH();
            ntiles = plan_items(sched.p, 0, n, dst.p, tiles, item_start, s, /*part_range=*/1);
        } else {
            ntiles = plan_items(sched.p, 0, n, dst.p, tiles, item_start, s);
        }
    } else {
        for (int c = 0; c < 3; ++c) { G.o[c] = idx->ext.lo[c]; G.w[c] = idx->w_fsg[c]; G.g[c] = idx->grid[c]; }
        qbox = DBuf<int4>(2ull * n, s);
        row_start = DBuf<uint32_t>(n + 1, s);
        DBuf<uint32_t> nr(n + 1, s);
        DBuf<unsigned long long> ntot(1, s);
        TDS_CUDA(cudaMemsetAsync(nr.p + n, 0, 4, s));
        TDS_CUDA(cudaMemsetAsync(ntot.p, 0, 8, s));
        // query order: (t_start, Morton cell of the start point), for L2 reuse of the slices
        DBuf<uint32_t> kc(n, s), kt(n, s), kt2(n, s);
        fsg_order = DBuf<uint32_t>(n, s);
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
        if (items64 >= (1ull << 32) - 1)
            fail(TDS_EINVAL, "the d-inflated query boxes cover %llu grid cells (limit 2^32): use a coarser grid",
                 items64);
        nrows = (uint32_t)items64;
        row_q = DBuf<uint32_t>(nrows, s);
        row_alo = DBuf<uint32_t>(nrows, s);
        row_len = DBuf<uint32_t>(nrows + 1, s);
        row_cxy = DBuf<uint32_t>(nrows, s);
        TDS_CUDA(cudaMemsetAsync(row_len.p + nrows, 0, 4, s));
        k_fsg_items<<<nblk((uint64_t)n * 32), 256, 0, s>>>(row_start.p, n, qbox.p, Q, G, idx->cell_off, idx->fsg_rec,
                                                          T0, T1, idx->ext.max_dur, fsg_literal(), row_q.p,
                                                          row_alo.p, row_len.p, row_cxy.p);
        TDS_CHECK_LAUNCH();
        DBuf<uint64_t> rl64(nrows + 1, s);
        k_u32_to_u64<<<nblk(nrows + 1), 256, 0, s>>>(row_len.p, nrows + 1, rl64.p);
        TDS_CHECK_LAUNCH();
        slot_start = DBuf<unsigned long long>(nrows + 1, s);
        exclusive_scan_u64(rl64.p, (uint64_t *)slot_start.p, nrows + 1, (uint64_t *)&dst.p->pair_tests, s);
        if (nparts > 1) {   // this part: the queries whose slots cross equal shares of the total
            k_part_bounds_spatial<<<1, 32, 0, s>>>(slot_start.p, row_start.p, n, part, nparts, dst.p);
            TDS_CHECK_LAUNCH();
        }
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
    S.kind = kind;
    S.n_queries = spatial ? nq : (nq - hs.cat_cnt[4]);
    unsigned long long slot_lo = 0, slot_hi = hs.pair_tests;   // GPUSpatial slots of this call
    if (nparts > 1) {
        if (spatial) {
            S.n_queries = hs.part_hi - hs.part_lo;
            slot_lo = hs.part_slot_lo;
            slot_hi = hs.part_slot_hi;
        } else {
            const uint32_t live = (uint32_t)(nq - hs.cat_cnt[4]);
            S.n_queries = std::min(hs.part_hi, live) > hs.part_lo ? std::min(hs.part_hi, live) - hs.part_lo : 0;
        }
    }
    // result-size probe (automatic capacity, large searches): the pass fraction of a
    // sample of the pair tests bounds the result count; the pass buffer takes three
    // times the estimate (a pass that overflows re-plans exactly, C22) instead of one
    // slot per pair test, which on hit-sparse searches meant a buffer 10-40x the
    // result and a compaction copy after the pass
    uint64_t est_hits = 0;
    bool probed = false;
    const unsigned long long probe_pairs = spatial ? slot_hi - slot_lo : hs.pair_tests;
    if (capacity == 0 && probe_pairs >= CAP_PROBE_MIN) {
        TDS_CUDA(cudaMemsetAsync(&dst.p->probe_pass, 0, 8, s));
        if (!spatial) {
            k_density_probe<<<32, 256, 0, s>>>(sched.p, n, Q, idx->rec, idx->st_arr[0], idx->st_arr[1],
                                               idx->st_arr[2], d, T0, T1, dst.p);
        } else {
            k_density_probe_spatial<<<32, 256, 0, s>>>(slot_start.p, nrows, slot_lo, slot_hi, row_q.p, row_alo.p,
                                                       row_cxy.p, qbox.p, idx->fsg_ecell, Q, idx->fsg_rec, d, T0, T1,
                                                       dst.p);
        }
        TDS_CHECK_LAUNCH();
        TDS_CUDA(cudaMemcpyAsync(&hs, dst.p, sizeof hs, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
        if (hs.probe_total >= 1024) {
            probed = true;
            est_hits = (uint64_t)((double)probe_pairs * hs.probe_pass / hs.probe_total);
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
        uint64_t want = probe_pairs + 64;
        if (probed) want = std::min<uint64_t>(want, 3 * est_hits + CAP_FLOOR);
        if (want * sizeof(Rec) > (1ull << 30)) big_lock = std::unique_lock<std::mutex>(big_alloc_mutex());
        const uint64_t budget_bytes = device_budget_bytes();
        cap = std::min<uint64_t>(want, (uint64_t)(budget_bytes * 0.45) / sizeof(Rec));
        cap = std::max<uint64_t>(cap, 1024);
        tr.mark(big_lock.owns_lock() ? "budget(locked)" : "budget");
    }
    cap = std::min<uint64_t>(cap, (1ull << 40));
    const int bps = spatial ? SPATIAL_BPS : RANGE_BPS;
    const uint64_t nwarps = (uint64_t)persistent_blocks(bps) * (PT / 32);
    uint32_t CS = (uint32_t)std::min<uint64_t>(1024, std::max<uint64_t>(128, cap / (16 * nwarps)));  // >= 128: appendK
    CS = (CS + 31) / 32 * 32;
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
    o.buf = buf.p; o.cap = cap; o.CS = CS; o.chunk_used = chunk_used.p;
    o.redo = redo.p; o.qcount = qcount.p; o.st = dst.p;

    // ---- A8-A10: pass 1 --------------------------------------------------------
    tr.mark("sync+alloc");
    tm.mark(2);
    if (!spatial) {
        RangeArgs a{};
        a.df = filter_threshold(d);
        a.tc = time_origin(idx);
        a.pc = PairCtx{Q, idx->rec, idx->perm, d, T0, T1, o, d64, dlo};
        for (int c = 0; c < 3; ++c) { a.arr[c] = idx->st_arr[c]; a.srec[c] = idx->st_rec[c]; }
        a.sched = sched.p; a.tiles = tiles.p; a.item_start = item_start.p; a.ntiles = ntiles;
        k_pair_range<false><<<persistent_blocks(RANGE_BPS), PT, 0, s>>>(a);
        TDS_CHECK_LAUNCH();
    } else if (nrows > 0 && hs.pair_tests > 0) {
        const uint64_t nslots = slot_hi - slot_lo;
        const uint64_t ngrab = (nslots + SP_GRAB - 1) / SP_GRAB;
        DBuf<uint32_t> grab_row(ngrab + 1, s);
        k_grab_rows<<<nblk(ngrab + 1), 256, 0, s>>>(slot_start.p, nrows, slot_lo, slot_hi, ngrab, grab_row.p);
        TDS_CHECK_LAUNCH();
        DBuf<uint32_t> slot_row;
        if (nslots <= SLOT_ROW_MAX) {
            slot_row = DBuf<uint32_t>(nslots, s);
            k_slot_rows<<<nblk(nslots), 256, 0, s>>>(slot_start.p, nrows, slot_lo, nslots, slot_row.p);
            TDS_CHECK_LAUNCH();
        }
        SpatialArgs a{};
        a.slot_row = slot_row.p;
        a.slot_lo = slot_lo;
        a.slot_hi = slot_hi;
        a.pc = PairCtx{Q, idx->fsg_rec, idx->fsg_perm, d, T0, T1, o, d64, dlo};
        a.ecell = idx->fsg_ecell; a.cell_off = idx->cell_off; a.grab_row = grab_row.p;
        a.qbox = qbox.p; a.row_q = row_q.p; a.row_alo = row_alo.p; a.row_cxy = row_cxy.p;
        a.slot_start = slot_start.p; a.nrows = nrows; a.G = G;
        // persistent grid, but no more blocks than grabs / warps per block: a small
        // search (Random-1M-shaped: a few hundred grabs) does not launch 444 blocks
        // that mostly find no work
        const int sp_blocks = (int)std::min<uint64_t>(persistent_blocks(SPATIAL_BPS), (ngrab + PT / 32 - 1) / (PT / 32));
        k_pair_spatial<false><<<sp_blocks, PT, 0, s>>>(a);
        TDS_CHECK_LAUNCH();
    }
    tm.mark(3);
    tr.mark("pairs");
    TDS_CUDA(cudaMemcpyAsync(&hs, dst.p, sizeof hs, cudaMemcpyDeviceToHost, s));
    TDS_CUDA(cudaStreamSynchronize(s));
    S.passes = 1;
    S.refined_pairs = hs.refined;
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

    // redo list with exact counts, in schedule order (range) / input order (spatial)
    std::vector<uint32_t> hcnt;
    DBuf<Sched> rsched;
    DBuf<uint32_t> rlist;              // spatial: redo query rows
    uint32_t nredo = 0;
    if (!spatial) {
        DBuf<uint32_t> flag(n + 1, s), fpos(n + 1, s), cnt(n, s);
        TDS_CUDA(cudaMemsetAsync(flag.p + n, 0, 4, s));
        k_redo_flags_sched<<<nblk(n), 256, 0, s>>>(sched.p, n, redo.p, flag.p);
        TDS_CHECK_LAUNCH();
        exclusive_scan_u32(flag.p, fpos.p, n + 1, nullptr, s);
        rsched = DBuf<Sched>(n, s);
        k_compact_sched<<<nblk(n), 256, 0, s>>>(sched.p, n, flag.p, fpos.p, rsched.p, qcount.p, cnt.p);
        TDS_CHECK_LAUNCH();
        TDS_CUDA(cudaMemcpyAsync(&nredo, fpos.p + n, 4, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
        hcnt.resize(nredo);
        if (nredo) TDS_CUDA(cudaMemcpyAsync(hcnt.data(), cnt.p, 4ull * nredo, cudaMemcpyDeviceToHost, s));
    } else {
        std::vector<uint8_t> hr(n);
        std::vector<uint32_t> hq(n);
        TDS_CUDA(cudaMemcpyAsync(hr.data(), redo.p, n, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaMemcpyAsync(hq.data(), qcount.p, 4ull * n, cudaMemcpyDeviceToHost, s));
        TDS_CUDA(cudaStreamSynchronize(s));
        std::vector<uint32_t> rl;
        for (uint32_t k = 0; k < n; ++k)
            if (hr[k]) { rl.push_back(k); hcnt.push_back(hq[k]); }
        nredo = (uint32_t)rl.size();
        rlist = DBuf<uint32_t>(nredo, s);
        if (nredo) TDS_CUDA(cudaMemcpyAsync(rlist.p, rl.data(), 4ull * nredo, cudaMemcpyHostToDevice, s));
    }
    TDS_CUDA(cudaStreamSynchronize(s));
    uint64_t redo_total = 0;
    for (uint32_t c : hcnt) {
        if (c > cap) fail(TDS_ECAPACITY, "one query produces %u records, more than capacity %llu", c,
                          (unsigned long long)cap);
        redo_total += c;
    }
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

    // per-query exact offsets in redo order
    DBuf<unsigned long long> qoff(n, s);
    DBuf<uint32_t> qfill(n, s);
    TDS_CUDA(cudaMemsetAsync(qfill.p, 0, 4ull * n, s));
    {
        std::vector<uint64_t> off(nredo);
        uint64_t acc = nkept;
        for (uint32_t k = 0; k < nredo; ++k) { off[k] = acc; acc += hcnt[k]; }
        DBuf<uint64_t> doff(nredo, s);
        if (nredo) TDS_CUDA(cudaMemcpyAsync(doff.p, off.data(), 8ull * nredo, cudaMemcpyHostToDevice, s));
        if (!spatial) {
            if (nredo) k_set_qoff<<<nblk(nredo), 256, 0, s>>>(rsched.p, nredo, doff.p, 0ull, qoff.p);
        } else {
            // spatial: scatter offsets by query row
            std::vector<uint32_t> rl(nredo);
            if (nredo) TDS_CUDA(cudaMemcpyAsync(rl.data(), rlist.p, 4ull * nredo, cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            std::vector<unsigned long long> hq(n, 0);
            for (uint32_t k = 0; k < nredo; ++k) hq[rl[k]] = off[k];
            TDS_CUDA(cudaMemcpyAsync(qoff.p, hq.data(), 8ull * n, cudaMemcpyHostToDevice, s));
        }
        TDS_CHECK_LAUNCH();
        TDS_CUDA(cudaStreamSynchronize(s));
    }
    tm.mark(4);
    // batches: consecutive redo entries with sum(count) <= cap (paper's incremental
    // processing of Q)
    o.buf = store.p;
    o.qoff = qoff.p;
    o.qfill = qfill.p;
    DBuf<uint32_t> qcount2(n, s);      // counts are recomputed, not needed again
    TDS_CUDA(cudaMemsetAsync(qcount2.p, 0, 4ull * n, s));
    o.qcount = qcount2.p;
    uint32_t b0 = 0;
    while (b0 < nredo) {
        uint64_t acc = 0;
        uint32_t b1 = b0;
        while (b1 < nredo && acc + hcnt[b1] <= cap) acc += hcnt[b1++];
        TDS_CUDA(cudaMemsetAsync(&dst.p->work_ctr, 0, 4, s));
        TDS_CUDA(cudaMemsetAsync(&dst.p->total_slots, 0, 8, s));
        if (!spatial) {
            // category counts of the batch: re-derive by planning on the compacted list
            DBuf<DevStats> bst(1, s);
            TDS_CUDA(cudaMemsetAsync(bst.p, 0, sizeof(DevStats), s));
            DBuf<uint32_t> ck(b1 - b0, s);
            // count categories of [b0, b1)
            std::vector<Sched> hsched(b1 - b0);
            TDS_CUDA(cudaMemcpyAsync(hsched.data(), rsched.p + b0, sizeof(Sched) * (b1 - b0),
                                     cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            DevStats hb{};
            for (auto &e : hsched) hb.cat_cnt[e.sel + 1]++;
            TDS_CUDA(cudaMemcpyAsync(bst.p, &hb, sizeof hb, cudaMemcpyHostToDevice, s));
            DBuf<Tile> bt;
            DBuf<uint32_t> bis;
            uint32_t bnt = plan_items(rsched.p + b0, 0, b1 - b0, bst.p, bt, bis, s);
            RangeArgs a{};
            a.df = filter_threshold(d);
            a.tc = time_origin(idx);
            a.pc = PairCtx{Q, idx->rec, idx->perm, d, T0, T1, o, d64, dlo};
            a.pc.o.st = bst.p;
            for (int c = 0; c < 3; ++c) { a.arr[c] = idx->st_arr[c]; a.srec[c] = idx->st_rec[c]; }
            a.sched = rsched.p + b0; a.tiles = bt.p; a.item_start = bis.p; a.ntiles = bnt;
            k_pair_range<true><<<persistent_blocks(RANGE_BPS), PT, 0, s>>>(a);
            TDS_CHECK_LAUNCH();
            TDS_CUDA(cudaStreamSynchronize(s));
            DevStats hb2;
            TDS_CUDA(cudaMemcpy(&hb2, bst.p, sizeof hb2, cudaMemcpyDeviceToHost));
            S.refined_pairs += hb2.refined;
            S.pairs_executed += hb2.executed;
        } else {
            uint32_t nb = b1 - b0;
            DBuf<int4> bq(2ull * nb, s);
            DBuf<uint32_t> bnr(nb + 1, s), brs(nb + 1, s);
            DBuf<unsigned long long> btot(1, s);
            TDS_CUDA(cudaMemsetAsync(bnr.p + nb, 0, 4, s));
            TDS_CUDA(cudaMemsetAsync(btot.p, 0, 8, s));
            k_fsg_count<<<nblk(nb), 256, 0, s>>>(Q, rlist.p + b0, nb, d, T0, T1, G, bnr.p, bq.p, btot.p,
                                                 &dst.p->bad);
            TDS_CHECK_LAUNCH();
            exclusive_scan_u32(bnr.p, brs.p, nb + 1, nullptr, s);
            uint32_t bnrows = 0;
            TDS_CUDA(cudaMemcpyAsync(&bnrows, brs.p + nb, 4, cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            DBuf<uint32_t> rq(bnrows, s), ra(bnrows, s), rlen(bnrows + 1, s), rc(bnrows, s);
            TDS_CUDA(cudaMemsetAsync(rlen.p + bnrows, 0, 4, s));
            k_fsg_items<<<nblk((uint64_t)nb * 32), 256, 0, s>>>(brs.p, nb, bq.p, Q, G, idx->cell_off, idx->fsg_rec, T0,
                                                                T1, idx->ext.max_dur, fsg_literal(), rq.p, ra.p,
                                                                rlen.p, rc.p);
            TDS_CHECK_LAUNCH();
            DBuf<uint64_t> rl64(bnrows + 1, s);
            DBuf<unsigned long long> ss(bnrows + 1, s);
            k_u32_to_u64<<<nblk(bnrows + 1), 256, 0, s>>>(rlen.p, bnrows + 1, rl64.p);
            TDS_CHECK_LAUNCH();
            exclusive_scan_u64(rl64.p, (uint64_t *)ss.p, bnrows + 1, nullptr, s);
            unsigned long long bslots = 0;
            TDS_CUDA(cudaMemcpyAsync(&bslots, ss.p + bnrows, 8, cudaMemcpyDeviceToHost, s));
            TDS_CUDA(cudaStreamSynchronize(s));
            const uint64_t ngrab = (bslots + SP_GRAB - 1) / SP_GRAB;
            DBuf<uint32_t> grab_row(ngrab + 1, s);
            k_grab_rows<<<nblk(ngrab + 1), 256, 0, s>>>(ss.p, bnrows, 0ull, bslots, ngrab, grab_row.p);
            TDS_CHECK_LAUNCH();
            DBuf<uint32_t> slot_row;
            if (bslots && bslots <= SLOT_ROW_MAX) {
                slot_row = DBuf<uint32_t>(bslots, s);
                k_slot_rows<<<nblk(bslots), 256, 0, s>>>(ss.p, bnrows, 0ull, bslots, slot_row.p);
                TDS_CHECK_LAUNCH();
            }
            SpatialArgs a{};
            a.slot_row = slot_row.p;
            a.slot_lo = 0;
            a.slot_hi = bslots;
            a.pc = PairCtx{Q, idx->fsg_rec, idx->fsg_perm, d, T0, T1, o, d64, dlo};
            a.ecell = idx->fsg_ecell; a.cell_off = idx->cell_off; a.grab_row = grab_row.p;
            a.qbox = bq.p; a.row_q = rq.p; a.row_alo = ra.p; a.row_cxy = rc.p; a.slot_start = ss.p;
            a.nrows = bnrows; a.G = G;
            if (bnrows && bslots) {
                const int sp_blocks =
                    (int)std::min<uint64_t>(persistent_blocks(SPATIAL_BPS), (ngrab + PT / 32 - 1) / (PT / 32));
                k_pair_spatial<true><<<sp_blocks, PT, 0, s>>>(a);
                TDS_CHECK_LAUNCH();
            }
            TDS_CUDA(cudaStreamSynchronize(s));
            DevStats hb2;
            TDS_CUDA(cudaMemcpy(&hb2, dst.p, sizeof hb2, cudaMemcpyDeviceToHost));
            S.refined_pairs = hb2.refined;
            S.pairs_executed = hb2.executed;
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

void free_result(tds_result_s *r) {
    cudaStream_t s = r->stream;      // ordered after the last fetch on that stream
    if (r->buf) dfree(r->buf, s);
    if (r->chunk_used) dfree(r->chunk_used, s);
    if (r->chunk_off) dfree(r->chunk_off, s);
    if (r->store) dfree(r->store, s);
    r->buf = nullptr; r->chunk_used = nullptr; r->chunk_off = nullptr; r->store = nullptr;
}

}  // namespace tds
