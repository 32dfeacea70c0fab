// km_small.cuh -- the whole Lloyd run for small problems in ONE launch of ONE CTA.
//
// For n up to a few 10^4 points (config 1: n = 10^4, d = 2, k = 10) an iteration is ~10^5
// pairs: every multi-kernel schedule is launch- and latency-bound (each launch, grid-wide
// ticket and reduction costs microseconds).  One CTA of 1024 threads keeps the centroids, their
// negated SoA copy and the privatised fixed-point sums (accumulate_point_priv) in shared memory
// and runs, with __syncthreads between the phases:
//   bounding box -> fixed-point scale (make_quant, as quant_kernel)
//   for t < max_iter: assignment (the packed FP32 scan of K1 + FP64 certification, exact labels,
//     P:L99) with SSE_t, changed_t and the sums sv(j), |S_j|; refine
//     c_j = RN_f32(sv(j)/|S_j|), drift, traces, convergence (Alg. 1 line 12)
//   Eq. 1 of the returned pair as the 128-bit fixed-point sum (sse_kernel's rounding).
// Every value is computed with the arithmetic of the multi-kernel brute-force path, so labels,
// centroids, changed_t, drift and out_sse are identical to it bit for bit (SSE_t up to FP64
// summation order).
#pragma once
#include "km_kernels.cuh"
#include "km_assign_fast.cuh"

namespace km {

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxN = 1 << 16;   // km_api.cu uses this kernel for n <= kSmallMaxN, k <= kSmallMaxK
constexpr int kSmallMaxK = 1024;

template <int D>
__host__ __device__ constexpr size_t small_smem(int k, int kpad)
{
    return (size_t)D * kpad * 4 + (size_t)k * D * 4 + priv_bytes<D>(k);
}

template <int D>
__global__ void __launch_bounds__(kSmallThreads, 1)
lloyd_small_kernel(const float* __restrict__ pts, int n, float* __restrict__ Cio, int k, int kpad,
                   int32_t* __restrict__ labels, int max_iter, float tol, Quant* __restrict__ quant_out,
                   double* __restrict__ sse_trace, long long* __restrict__ chg_trace, double* __restrict__ drift_trace,
                   Ctl* __restrict__ ctl, SseFix* __restrict__ sse_out)
{
    extern __shared__ __align__(16) float ssm[];
    float* nc = ssm;                                   // [D][kpad] negated centroids (-inf padding)
    float* Cs = ssm + D * kpad;                        // [k][D] current centroids
    unsigned int* sp = reinterpret_cast<unsigned int*>(Cs + k * D);   // privatised sums and counts
    __shared__ float s_box[2 * D][32];
    __shared__ double s_d[32];
    __shared__ int s_done;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int NW = kSmallThreads / 32;

    // ---- bounding box -> the fixed-point scale (same formula as quant_kernel)
    float lo[D], hi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = INFINITY; hi[m] = -INFINITY; }
    for (int i = tid; i < n; i += kSmallThreads)
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const float v = pts[(int64_t)i * D + m];
            lo[m] = fminf(lo[m], v);
            hi[m] = fmaxf(hi[m], v);
        }
#pragma unroll
    for (int m = 0; m < D; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
        if (lane == 0) { s_box[m][w] = lo[m]; s_box[D + m][w] = hi[m]; }
    }
    for (int j = tid; j < k * D; j += kSmallThreads) Cs[j] = Cio[j];
    __syncthreads();
#pragma unroll
    for (int m = 0; m < D; ++m)
        for (int ww = 0; ww < NW; ++ww) { lo[m] = fminf(lo[m], s_box[m][ww]); hi[m] = fmaxf(hi[m], s_box[D + m][ww]); }
    Quant q;
    make_quant(q, lo, hi, D, n);
    if (tid == 0) *quant_out = q;

    int t = 0, conv = 0;
    for (; t < max_iter; ++t) {
        // ---- stage the negated SoA centroids; clear the sums
        for (int j = tid; j < kpad; j += kSmallThreads)
#pragma unroll
            for (int m = 0; m < D; ++m) nc[m * kpad + j] = j < k ? -Cs[j * D + m] : -INFINITY;
        priv_clear<D>(sp, k);
        __syncthreads();
        // ---- assignment + SSE_t + changed_t + sums (as assign_scan_kernel, one point at a time)
        const float4* nc4 = reinterpret_cast<const float4*>(nc);
        const int kq = kpad >> 2;
        double sse = 0.0;
        unsigned long long chg = 0;
        for (int i = tid; i < n; i += kSmallThreads) {
            Pt<D> p;
#pragma unroll
            for (int m = 0; m < D; ++m) p.v[m] = pts[(int64_t)i * D + m];
            float m1 = INFINITY, m2 = INFINITY;
            int b1 = 0;
            for (int g = 0; g < kq; ++g) {
                float4 c[D];
#pragma unroll
                for (int m = 0; m < D; ++m) c[m] = nc4[m * kq + g];
                const float2 s0 = pair2<D>(p, c, false);
                const float2 s1 = pair2<D>(p, c, true);
                const float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
                const bool lt = v < m1;
                m2 = fmaxf(m1, fminf(m2, v));
                m1 = fminf(m1, v);
                b1 = lt ? g : b1;
            }
            const int a = certify_label<D, 4>(p, m1, m2, b1, nc, kpad, k);
            sse += dist64n<D>(p, nc, kpad, a);
            chg += t == 0 ? 1ull : (unsigned long long)(labels[i] != a);
            labels[i] = a;
            accumulate_point_priv<D>(p.v, a, q, sp, k);
        }
        block_sum2<kSmallThreads>(sse, chg);   // thread 0 holds the totals
        __syncthreads();
        // ---- refine (finalize_block's arithmetic), max drift
        double md = 0.0;
        for (int j = tid; j < k; j += kSmallThreads) {
            const unsigned int cnt = sp[2 * k * D + j];
            double dd = 0.0;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const int idx = j * D + m;
                const float old = Cs[idx];
                float nw = old;
                if (cnt > 0) {
                    const unsigned long long sv = ((unsigned long long)sp[k * D + idx] << 32) | sp[idx];
                    const double mean = __dadd_rn(q.o[m], __dmul_rn(__ddiv_rn((double)sv, (double)cnt), q.inv[m]));
                    nw = __double2float_rn(mean);
                }
                const double tt = __dsub_rn((double)nw, (double)old);
                dd = __dadd_rn(dd, __dmul_rn(tt, tt));
                Cs[idx] = nw;
            }
            md = fmax(md, sqrt(dd));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
        if (lane == 0) s_d[w] = md;
        __syncthreads();
        if (tid == 0) {
            for (int ww = 1; ww < NW; ++ww) md = fmax(md, s_d[ww]);
            if (sse_trace) sse_trace[t] = sse;
            if (chg_trace) chg_trace[t] = (long long)chg;
            if (drift_trace) drift_trace[t] = md;
            s_done = tol >= 0.0f && (md <= (double)tol || (t >= 1 && chg == 0));
        }
        __syncthreads();
        if (s_done) { ++t; conv = 1; break; }
    }
    const int iters = t;
    // ---- Eq. 1 of the returned pair: bound (sse_bound_kernel), 128-bit fixed point (sse_kernel)
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = (float)q.o[m]; hi[m] = q.hi[m]; }
    for (int j = tid; j < k; j += kSmallThreads)
#pragma unroll
        for (int m = 0; m < D; ++m) { lo[m] = fminf(lo[m], Cs[j * D + m]); hi[m] = fmaxf(hi[m], Cs[j * D + m]); }
#pragma unroll
    for (int m = 0; m < D; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
        if (lane == 0) { s_box[m][w] = lo[m]; s_box[D + m][w] = hi[m]; }
    }
    __syncthreads();
    double b = 0.0;
    for (int m = 0; m < D; ++m) {
        float a0 = s_box[m][0], z = s_box[D + m][0];
        for (int ww = 1; ww < NW; ++ww) { a0 = fminf(a0, s_box[m][ww]); z = fmaxf(z, s_box[D + m][ww]); }
        const double e = (double)z - (double)a0;
        b += e * e;
    }
    const int s3 = sse_shift(b, q.n);
    const double scale = ldexp(1.0, s3);
    u128 acc = 0;
    for (int i = tid; i < n; i += kSmallThreads) {
        const int a = labels[i];
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double tt = __dsub_rn((double)pts[(int64_t)i * D + m], (double)Cs[a * D + m]);
            v = __dadd_rn(v, __dmul_rn(tt, tt));
        }
        add_fix(acc, v, scale);
    }
    acc = block_sum128(acc);
    for (int j = tid; j < k * D; j += kSmallThreads) Cio[j] = Cs[j];
    if (tid == 0) {
        const double inv = ldexp(1.0, -s3);
        const double hv = (double)(unsigned long long)(acc >> 64), lv = (double)(unsigned long long)acc;
        sse_out->value = __dmul_rn(__dadd_rn(__dmul_rn(hv, 0x1p64), lv), inv);
        sse_out->inv = inv;
        const unsigned long long m48 = (1ull << 48) - 1;
        sse_out->limb[0] = (unsigned long long)acc & m48;
        sse_out->limb[1] = (unsigned long long)(acc >> 48) & m48;
        sse_out->limb[2] = (unsigned long long)(acc >> 96);
        ctl->iter = iters;
        ctl->done = conv;
    }
}

}  // namespace km
