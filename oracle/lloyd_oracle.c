/*
 * oracle/lloyd_oracle.c -- plain, slow, obviously-correct FP64 Lloyd's algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2412_02244_b200/, libkm.so) never links, imports or calls it, and this
 * file shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:Lnn" = its line nn):
 *   - Eq. 1: k-means minimises sum_j sum_{p in S_j} ||p - c_j||^2, with
 *     c_j the mean of S_j.
 *   - Lloyd's algorithm: "assigning each spatial vector to its nearest
 *     centroid and iteratively refining the centroids" -- n x k distances per
 *     iteration.  Dask-means yields "the same results as Lloyd's algorithm"
 *     (P:L104), so plain Lloyd is the definition the GPU path must reproduce.
 *   - Refine (Alg. 1 line 12): c_j <- sv(j)/|S_j|, and the drift
 *     Delta[j] = ||c_j - c'_j||.
 *   - Loop (Alg. 1): repeat until no centroid moves.
 * Readings where the paper is silent (DESIGN.md "Readings" R1-R10):
 *   - squared Euclidean distance in direct (difference) form, FP64 (R1);
 *   - ties go to the lowest centroid index (R2), i.e. strict '<' scanning j upward;
 *   - an empty cluster keeps its centroid, drift 0 (R5);
 *   - mode A (the parity gate) stores centroids as float32 (round-to-nearest-even)
 *     between iterations; mode B keeps them in FP64 (R8);
 *   - tol < 0: exactly max_iter iterations; tol >= 0: stop after an iteration
 *     whose max drift <= tol, or (t >= 1) in which no label changed (R6);
 *   - returned pair is (labels of the last assignment, centroids after the last
 *     refine); out_sse is Eq. 1 of that pair (R3, R4).
 *
 * Arithmetic is written out in the order stated: for each point, D_ij =
 * sum_m (double(p_im) - double(c_jm))^2 accumulated m = 0..d-1 (multiply, then
 * add; compile with -ffp-contract=off so no FMA is formed).  Sums are sequential
 * in point-index order.  Only the assignment loop is parallelised (OpenMP over
 * points); labels do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* squared Euclidean distance, FP64, direct form (Eq. 1 summand). */
static double sqdist(const float *p, const double *c, int d)
{
    double s = 0.0;
    for (int m = 0; m < d; ++m) {
        double t = (double)p[m] - c[m];
        s = s + t * t;
    }
    return s;
}

/* Neumaier-compensated running sum (used for every SSE value). */
typedef struct { double s, comp; } ksum;
static void ksum_add(ksum *a, double x)
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->comp += (a->s - t) + x;
    else                       a->comp += (x - t) + a->s;
    a->s = t;
}
static double ksum_get(const ksum *a) { return a->s + a->comp; }

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Assignment step: labels[i] = lowest j attaining min_j D_ij.
 * best[i] = D_{i,labels[i]}; second[i] = smallest D_ij over j != labels[i]
 * (+inf when k == 1).  Either output pointer may be NULL.
 */
void oracle_assign(const float *P, int64_t n, int d, const double *C, int k,
                   int32_t *labels, double *best, double *second, int threads)
{
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
        const float *p = P + i * d;
        double b1 = INFINITY, b2 = INFINITY;
        int32_t a = -1;
        for (int j = 0; j < k; ++j) {
            double D = sqdist(p, C + (int64_t)j * d, d);
            if (D < b1) { b2 = b1; b1 = D; a = j; }
            else if (D < b2) { b2 = D; }
        }
        labels[i] = a;
        if (best) best[i] = b1;
        if (second) second[i] = b2;
    }
    (void)threads;
}

/*
 * Refine step (Alg. 1 line 12; sums sv(j) of P:L411-413 taken from
 * scratch).  counts[j] = |S_j|; S_j = sum of the member points, sequential in
 * index order in FP64; Cnew[j] = S_j / |S_j| (FP64 divide), rounded to float32
 * when round_f32 != 0 (mode A).  Empty cluster: Cnew[j] = Cold[j].
 * drift[j] = ||Cnew[j] - Cold[j]|| (FP64, on the stored values).  Returns max drift.
 * sums (k*d doubles) is caller scratch or NULL.
 */
double oracle_update(const float *P, int64_t n, int d, const int32_t *labels,
                     int k, const double *Cold, double *Cnew, int64_t *counts,
                     double *drift, int round_f32)
{
    double *S = (double *)calloc((size_t)k * d, sizeof(double));
    int64_t *cnt = counts ? counts : (int64_t *)malloc((size_t)k * sizeof(int64_t));
    memset(cnt, 0, (size_t)k * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {
        int32_t j = labels[i];
        cnt[j] += 1;
        for (int m = 0; m < d; ++m) S[(int64_t)j * d + m] += (double)P[i * d + m];
    }
    double maxdrift = 0.0;
    for (int j = 0; j < k; ++j) {
        double dd = 0.0;
        for (int m = 0; m < d; ++m) {
            int64_t q = (int64_t)j * d + m;
            double c;
            if (cnt[j] > 0) {
                c = S[q] / (double)cnt[j];
                if (round_f32) c = (double)(float)c;
            } else {
                c = Cold[q];
            }
            double t = c - Cold[q];
            dd = dd + t * t;
            Cnew[q] = c;
        }
        double dr = sqrt(dd);
        if (drift) drift[j] = dr;
        if (dr > maxdrift) maxdrift = dr;
    }
    free(S);
    if (!counts) free(cnt);
    return maxdrift;
}

/* Eq. 1 of a given partition and centroid set, Neumaier sum in index order. */
double oracle_sse(const float *P, int64_t n, int d, const int32_t *labels,
                  const double *C)
{
    ksum a = {0.0, 0.0};
    for (int64_t i = 0; i < n; ++i)
        ksum_add(&a, sqdist(P + i * d, C + (int64_t)labels[i] * d, d));
    return ksum_get(&a);
}

/*
 * Whole loop (Alg. 1 skeleton, without the index: plain Lloyd).
 * C0/Cout are k*d doubles (mode A: C0 must hold float32-representable values).
 * For t = 0..max_iter-1: assign against C_t, record SSE_t = sum_i min_j D_ij
 * and changed_t, refine to C_{t+1}, record max drift; stop early per tol.
 * Outputs: Cout = C_{t_last+1}, labels = a_{t_last}, *out_sse = Eq. 1 of that
 * pair.  Traces (length >= max_iter, nullable).  Returns iterations executed.
 */
int oracle_lloyd(const float *P, int64_t n, int d, int k, const double *C0,
                 int max_iter, double tol, int round_f32,
                 double *Cout, int32_t *labels, double *out_sse,
                 double *sse_trace, int64_t *changed_trace, double *drift_trace,
                 int threads)
{
    double *C = (double *)malloc((size_t)k * d * sizeof(double));
    double *Cn = (double *)malloc((size_t)k * d * sizeof(double));
    double *best = (double *)malloc((size_t)n * sizeof(double));
    int32_t *prev = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    memcpy(C, C0, (size_t)k * d * sizeof(double));
    int it = 0;
    for (int t = 0; t < max_iter; ++t) {
        oracle_assign(P, n, d, C, k, labels, best, NULL, threads);
        ksum a = {0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) ksum_add(&a, best[i]);
        int64_t changed = 0;
        if (t == 0) changed = n;
        else for (int64_t i = 0; i < n; ++i) changed += (labels[i] != prev[i]);
        double md = oracle_update(P, n, d, labels, k, C, Cn, NULL, NULL, round_f32);
        if (sse_trace) sse_trace[t] = ksum_get(&a);
        if (changed_trace) changed_trace[t] = changed;
        if (drift_trace) drift_trace[t] = md;
        memcpy(C, Cn, (size_t)k * d * sizeof(double));
        memcpy(prev, labels, (size_t)n * sizeof(int32_t));
        it = t + 1;
        if (tol >= 0.0 && (md <= tol || (t >= 1 && changed == 0))) break;
    }
    memcpy(Cout, C, (size_t)k * d * sizeof(double));
    if (out_sse) *out_sse = oracle_sse(P, n, d, labels, C);
    free(C); free(Cn); free(best); free(prev);
    return it;
}
