/*
 * tds_oracle.c — plain, slow, obviously-correct CPU oracle for the distance
 * threshold search over 4-D line segments (Gowanlock & Casanova,
 * arXiv 1410.2698; PAPER.md = /root/reference/PAPER.md, cited as P:line).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header or constant with the CUDA path
 * (paper_1410_2698_b200/csrc, include/tds.h) and includes neither.
 *
 * What it computes (the plain definition):
 *   A segment moves linearly between its endpoints:
 *     P(t) = P0 + (t - t0) * (P1 - P0) / (t1 - t0).
 *   For a query q and an entry e, over the shared span
 *     a = max(t0q, t0e, T0),  b = min(t1q, t1e, T1)   (window [T0,T1])
 *   the pair interacts iff a < b (reading C5) and the set
 *     I = { t in [a,b] : ||Pq(t) - Pe(t)||_2 <= d }
 *   is non-empty; the result is (q, e, min I, max I)  ("(q1,l1,[0.1,0.3])").
 *   ||Pq(t)-Pe(t)||^2 is a convex quadratic in t, so I is one closed interval,
 *   evaluated here in closed form in double precision from the float32 inputs.
 *   The search is brute force over ALL pairs: no index (the three indexes of
 *   P:253-1173 are filters that must reach exactly this set).
 *
 * Parity pins: tests/test_oracle_compare.py (hand-worked cases E1-E10 in
 * tests/golden/compare_cases.txt, dense sampling + bisection, symmetry,
 * monotonicity) and tests/test_oracle_search.py (pure-Python brute force).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o liboracle.so tds_oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* One segment: 8 float32 values (x0,y0,z0,t0,x1,y1,z1,t1). */

/*
 * oracle_compare — the interaction of query segment q with entry segment e.
 *
 * Returns 1 if the shared span is non-empty (a < b) and the pair comes within
 * d somewhere on it; then *t_in, *t_out hold the closed interval I.  In every
 * case with a < b, *dmin holds the minimum distance over [a,b]; returns 0 and
 * *dmin = +inf when a >= b.
 */
int oracle_compare(const float *q, const float *e, double d, double T0, double T1,
                   double *t_in, double *t_out, double *dmin)
{
    double t0q = q[3], t1q = q[7], t0e = e[3], t1e = e[7];
    double a = t0q;
    if (t0e > a) a = t0e;
    if (T0 > a) a = T0;
    double b = t1q;
    if (t1e < b) b = t1e;
    if (T1 < b) b = T1;
    *dmin = INFINITY;
    if (!(a < b)) return 0;                       /* reading C5: need a < b */

    double dq = t1q - t0q, de = t1e - t0e;
    double Da[3], DV[3];
    for (int c = 0; c < 3; ++c) {
        double vq = ((double)q[4 + c] - (double)q[c]) / dq;   /* velocity of q */
        double ve = ((double)e[4 + c] - (double)e[c]) / de;   /* velocity of e */
        double pq = (double)q[c] + (a - t0q) * vq;            /* Pq(a) */
        double pe = (double)e[c] + (a - t0e) * ve;            /* Pe(a) */
        Da[c] = pq - pe;                                      /* Delta(a) */
        DV[c] = vq - ve;                                      /* d Delta / dt */
    }
    double L = b - a;
    double A = DV[0] * DV[0] + DV[1] * DV[1] + DV[2] * DV[2];
    double d2 = d * d;

    if (A == 0.0) {                               /* constant separation */
        double h = Da[0] * Da[0] + Da[1] * Da[1] + Da[2] * Da[2];
        *dmin = sqrt(h);
        if (h <= d2) { *t_in = a; *t_out = b; return 1; }
        return 0;
    }
    /* ||Delta(a + s)||^2 = A s^2 + 2 (Da.DV) s + Da.Da, minimised at s_u */
    double s_u = -(Da[0] * DV[0] + Da[1] * DV[1] + Da[2] * DV[2]) / A;
    double s_star = s_u < 0.0 ? 0.0 : (s_u > L ? L : s_u);
    double h_star = 0.0, h_u = 0.0;
    for (int c = 0; c < 3; ++c) {
        double x = Da[c] + s_star * DV[c];
        double y = Da[c] + s_u * DV[c];
        h_star += x * x;
        h_u += y * y;
    }
    *dmin = sqrt(h_star);
    if (!(h_star <= d2)) return 0;
    /* roots of A s^2 + 2 (Da.DV) s + Da.Da = d^2 are s_u -/+ w */
    double rem = d2 - h_u;
    if (rem < 0.0) rem = 0.0;
    double w = sqrt(rem / A);
    double lo = s_u - w, hi = s_u + w;
    if (lo < 0.0) lo = 0.0;
    if (lo > L) lo = L;
    if (hi < 0.0) hi = 0.0;
    if (hi > L) hi = L;
    *t_in = a + lo;
    *t_out = a + hi;
    return 1;
}

/* one output record of the all-pairs search */
typedef struct {
    int64_t qid, eid;
    double t_in, t_out, dmin;
    int32_t hit;       /* 1 = within d; 0 = near miss kept for the exclusion band */
    int32_t pad;
} oracle_rec;

typedef struct { oracle_rec *v; int64_t n, cap; } rec_vec;

static void push(rec_vec *r, oracle_rec x)
{
    if (r->n == r->cap) {
        r->cap = r->cap ? 2 * r->cap : 16;
        r->v = (oracle_rec *)realloc(r->v, (size_t)r->cap * sizeof(oracle_rec));
    }
    r->v[r->n++] = x;
}

static rec_vec g_out;   /* result of the last oracle_search (not thread safe) */

/*
 * oracle_search — all-pairs brute force.  For every q in Q and every e in D
 * evaluates oracle_compare; keeps every hit and every miss whose minimum
 * distance is <= near * d (near >= 1, for the parity exclusion band).
 * Records are ordered by (qid, eid).  Returns the record count; fetch with
 * oracle_fetch().  Parallel over queries (OpenMP), threads = nthreads (<=0:
 * OpenMP default).
 */
int64_t oracle_search(const float *D, int64_t nD, const float *Q, int64_t nQ,
                      double d, double T0, double T1, double near, int nthreads)
{
    free(g_out.v);
    memset(&g_out, 0, sizeof g_out);
    rec_vec *per_q = (rec_vec *)calloc((size_t)(nQ > 0 ? nQ : 1), sizeof(rec_vec));
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k = 0; k < nQ; ++k) {
        const float *q = Q + 8 * k;
        for (int64_t i = 0; i < nD; ++i) {
            const float *e = D + 8 * i;
            double ti = 0.0, to = 0.0, dm = INFINITY;
            int hit = oracle_compare(q, e, d, T0, T1, &ti, &to, &dm);
            if (hit || dm <= near * d) {
                oracle_rec r;
                r.qid = k; r.eid = i; r.t_in = hit ? ti : 0.0; r.t_out = hit ? to : 0.0;
                r.dmin = dm; r.hit = hit; r.pad = 0;
                push(&per_q[k], r);
            }
        }
    }
    int64_t total = 0;
    for (int64_t k = 0; k < nQ; ++k) total += per_q[k].n;
    g_out.v = (oracle_rec *)malloc((size_t)(total > 0 ? total : 1) * sizeof(oracle_rec));
    g_out.cap = total;
    for (int64_t k = 0; k < nQ; ++k) {
        if (per_q[k].n)
            memcpy(g_out.v + g_out.n, per_q[k].v, (size_t)per_q[k].n * sizeof(oracle_rec));
        g_out.n += per_q[k].n;
        free(per_q[k].v);
    }
    free(per_q);
    return total;
}

/* oracle_search_subset — like oracle_search but only for the query rows listed
 * in qsel[0..nsel); record qid is the ORIGINAL row number qsel[j]. */
int64_t oracle_search_subset(const float *D, int64_t nD, const float *Q, const int64_t *qsel,
                             int64_t nsel, double d, double T0, double T1, double near,
                             int nthreads)
{
    float *sub = (float *)malloc((size_t)(nsel > 0 ? nsel : 1) * 8 * sizeof(float));
    for (int64_t j = 0; j < nsel; ++j) memcpy(sub + 8 * j, Q + 8 * qsel[j], 8 * sizeof(float));
    int64_t n = oracle_search(D, nD, sub, nsel, d, T0, T1, near, nthreads);
    for (int64_t r = 0; r < n; ++r) g_out.v[r].qid = qsel[g_out.v[r].qid];
    free(sub);
    return n;
}

/* copy the records of the last search into caller arrays (each of length n) */
void oracle_fetch(int64_t *qid, int64_t *eid, double *t_in, double *t_out, double *dmin,
                  int32_t *hit)
{
    for (int64_t r = 0; r < g_out.n; ++r) {
        qid[r] = g_out.v[r].qid;
        eid[r] = g_out.v[r].eid;
        t_in[r] = g_out.v[r].t_in;
        t_out[r] = g_out.v[r].t_out;
        dmin[r] = g_out.v[r].dmin;
        hit[r] = g_out.v[r].hit;
    }
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
