// km_kernels.cuh -- sm_100a kernels of the exact Lloyd step (libkm).
//
// Paper: arXiv 2412.02244 (Dask-means), cited P:Lnn = /root/reference/PAPER.md line nn.
//   assign   : nearest centroid per point (Alg. 1 Assign P:L306-358 without
//              the index), ties -> lowest index, EXACT w.r.t. the FP64 distance.
//   update   : sv(j) = sum of members as exact 64-bit fixed point,
//              fused into the assign epilogue (one RED per coordinate).
//   finalize : c_j <- sv(j)/|S_j| (Alg. 1 line 12), drift Delta[j]
//              (P:L135), convergence "whether any of the centroids move".
// Layouts, roofline and the exactness argument: DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace km {

constexpr int kAssignThreads = 256;
constexpr int kFinalizeThreads = 1024;
constexpr int kReduceThreads = 1024;
constexpr int kMaxAccCopies = 8;   // private copies of the tile path's running sums (km_api.cu kAccCopies)

// Fixed-point quantisation of coordinates for the exact sums sv(j):
//   qv(p_m) = rint((double(p_m) - o_m) * scale_m) >= 0, scale_m = 2^s_m,
// s_m chosen so that n * extent_m * 2^s_m < 2^61 (no int64 overflow for any cluster).
struct Quant {
    double o[3];
    double scale[3];
    double inv[3];
    float hi[3];        // bounding-box maximum (the minimum is o)
    double sse_scale;   // 2^s2: SSE_t summands as fixed point (tile path), n * E^2 * 2^s2 < 2^62
    double sse_inv;     // 2^-s2
    long long n;        // points of the (global) problem
};

// The quantisation of a problem with n points and bounding box [lo, hi] (host and device:
// the data-parallel path computes it on the host from the global box, bit-identically).
// E^2 = sum_m extent_m^2 bounds every point-centroid squared distance (centroids are means
// of points, so they lie in the box), hence every SSE summand.
__host__ __device__ inline void make_quant(Quant& q, const float* lo, const float* hi, int d, int64_t n)
{
    int nb = 0;
    while (nb < 63 && (n >> nb) != 0) ++nb;   // n < 2^nb
    double e2 = 0.0;
    for (int m = 0; m < 3; ++m) {
        if (m < d) {
            const double ext = (double)hi[m] - (double)lo[m];
            int e = 0;
            if (ext > 0.0) frexp(ext, &e);              // ext < 2^e
            const int s = ext > 0.0 ? 61 - nb - e : 0;   // n * ext * 2^s < 2^61
            q.o[m] = (double)lo[m];
            q.hi[m] = hi[m];
            q.scale[m] = ldexp(1.0, s);
            q.inv[m] = ldexp(1.0, -s);
            e2 += ext * ext;
        } else {
            q.o[m] = 0.0; q.hi[m] = 0.f; q.scale[m] = 1.0; q.inv[m] = 1.0;
        }
    }
    const double tot = (double)n * e2 * (1.0 + 0x1p-20);
    int e = 0;
    if (tot > 0.0) frexp(tot, &e);                       // tot < 2^e
    const int s2 = tot > 0.0 ? 62 - e : 0;
    q.sse_scale = ldexp(1.0, s2);
    q.sse_inv = ldexp(1.0, -s2);
    q.n = (long long)n;
}

// One SSE_t summand (a squared distance or a tile's moment sum) as fixed point.
// The same for an FP32 summand when 2^-100 <= scale <= 2^100: v * 2^s2 is then exact in FP32
// (a normal float below 2^62, or below 2^-126 where both forms round to 0), so the integer is
// bit-identical to sse_q((double)v, scale) with one FMUL + one F2I instead of FP64 work.
__device__ __forceinline__ unsigned long long sse_qf(float v, float scale_f)
{
    return (unsigned long long)__float2ll_rn(__fmul_rn(v, scale_f));
}

__device__ __forceinline__ unsigned long long sse_q(double v, double scale)
{
    return (unsigned long long)__double2ll_rn(__dmul_rn(v, scale));
}

// Device control words of a run.
struct Ctl {
    int done;   // set by finalize when converged (R6); later kernels return at once
    int iter;   // iterations completed
};

// --------------------------------------------------------------------------
// FP64 distance in exactly the oracle's order (R1): the exact label
// is defined by this value.  __dmul_rn/__dadd_rn forbid FMA contraction.
template <int D>
__device__ __forceinline__ double dist64(const float (&p)[D], const float* const (&sc)[D], int j)
{
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        double t = __dsub_rn((double)p[m], (double)sc[m][j]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

// FP32 direct-form distance used by the filter scan.  Relative error <= 5u
// (u = 2^-24) against the exact value; see DESIGN.md "Exactness".
template <int D>
__device__ __forceinline__ float dist32(const float (&p)[D], const float (&c)[D])
{
    float dx = __fsub_rn(p[0], c[0]);
    float s = __fmul_rn(dx, dx);
#pragma unroll
    for (int m = 1; m < D; ++m) {
        float t = __fsub_rn(p[m], c[m]);
        s = __fmaf_rn(t, t, s);
    }
    return s;
}

// Slow path: exact FP64 scan of all k centroids (used only when the FP32 filter
// cannot certify the winner: near-ties within 2^-19 relative, or overflow).
template <int D>
__device__ __noinline__ int exact_scan(const float (&p)[D], const float* const (&sc)[D], int k)
{
    double best = INFINITY;
    int a = 0;
    for (int j = 0; j < k; ++j) {
        double v = dist64<D>(p, sc, j);
        if (v < best) { best = v; a = j; }
    }
    return a;
}

// Certification threshold: any centroid whose FP32 distance exceeds thr(m1) cannot
// be the FP64 argmin (|D32 - D64| <= 5.01u * D64 + subnormal slack; thr uses 32u).
__device__ __forceinline__ float certify_thr(float m1)
{
    return __fmaf_ru(m1, 1.0f + 0x1p-19f, 0x1p-120f);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block reduction (fixed tree) of one double and one u64.
template <int NT>
__device__ __forceinline__ void block_sum2(double& a, unsigned long long& b)
{
    __shared__ double sa[NT / 32];
    __shared__ unsigned long long sb[NT / 32];
    a = warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sa[w] = a; sb[w] = b; }
    __syncthreads();
    if (w == 0) {
        a = l < NT / 32 ? sa[l] : 0.0;
        b = l < NT / 32 ? sb[l] : 0ull;
        a = warp_sum(a);
        b = warp_sum(b);
    }
}

// Stage C (row-major [k][D]) into shared memory as SoA sc[m][0..kpad), padding
// with +inf (pads never win: their FP32 distance is +inf).
template <int D>
__device__ __forceinline__ void stage_centroids(float* smem, const float* __restrict__ C, int k, int kpad)
{
    for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) smem[m * kpad + j] = j < k ? C[(int64_t)j * D + m] : INFINITY;
    }
    __syncthreads();
}

// Fixed-point accumulation of one point into sv(a) and |S_a| (global REDs).
template <int D>
__device__ __forceinline__ void accumulate_point(const float (&p)[D], int a, const Quant& q,
                                                 unsigned long long* __restrict__ acc_sum,
                                                 unsigned int* __restrict__ acc_cnt)
{
#pragma unroll
    for (int m = 0; m < D; ++m) {
        double v = __dmul_rn(__dsub_rn((double)p[m], q.o[m]), q.scale[m]);
        atomicAdd(&acc_sum[(int64_t)a * D + m], (unsigned long long)__double2ll_rn(v));
    }
    atomicAdd(&acc_cnt[a], 1u);
}

// Privatised update (A4, north_star (b): per-block shared-memory partial sums and counts, then
// one global reduction).  Each CTA keeps sv(j) of its own points as two 32-bit shared words
// per coordinate (native ATOMS.ADD; 64-bit shared atomics are CAS loops) and |S_j| as one:
// the low word's atomic returns the old value, so a wrap (old + lo < old) carries one into
// the high word -- every wrap happens in exactly one atomic, hence hi:lo is the exact 64-bit
// sum (a CTA's sum of one coordinate is < 2^61, Quant).  The flush adds each nonzero (hi:lo)
// and count to the global sums with one RED: k(d+1) REDs per CTA instead of d+1 per point.
// Integer sums are order-independent, so results equal the unprivatised form bit for bit.
template <int D>
__host__ __device__ constexpr size_t priv_bytes(int k) { return (size_t)k * (2 * D + 1) * 4; }

template <int D>
__device__ __forceinline__ void priv_clear(unsigned int* __restrict__ sp, int k)
{
    for (int i = threadIdx.x; i < k * (2 * D + 1); i += blockDim.x) sp[i] = 0u;
}

template <int D>
__device__ __forceinline__ void accumulate_point_priv(const float (&p)[D], int a, const Quant& q,
                                                      unsigned int* __restrict__ sp, int k)
{
    unsigned int* slo = sp;
    unsigned int* shi = sp + k * D;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const unsigned long long v = (unsigned long long)__double2ll_rn(
            __dmul_rn(__dsub_rn((double)p[m], q.o[m]), q.scale[m]));
        const unsigned int lo = (unsigned int)v;
        const unsigned int old = atomicAdd(&slo[a * D + m], lo);
        const unsigned int hi = (unsigned int)(v >> 32) + (old + lo < old ? 1u : 0u);
        if (hi) atomicAdd(&shi[a * D + m], hi);
    }
    atomicAdd(&sp[2 * k * D + a], 1u);
}

// The running sums of the incremental update (sv(j) += p when p moves in, -= p when it moves
// out): a point that changed label adds its fixed-point value to the new cluster's
// private partial and its two's complement (mod 2^64, the same carry logic) to the old one's;
// counts +1 / -1 (mod 2^32).  The global running sums are exact integers in [0, 2^63), so the
// modular partials add up to them exactly in any order.
template <int D>
__device__ __forceinline__ void move_point_priv(const float (&p)[D], int from, int to, const Quant& q,
                                                unsigned int* __restrict__ sp, int k)
{
    unsigned int* slo = sp;
    unsigned int* shi = sp + k * D;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const unsigned long long v = (unsigned long long)__double2ll_rn(
            __dmul_rn(__dsub_rn((double)p[m], q.o[m]), q.scale[m]));
        {
            const unsigned int lo = (unsigned int)v;
            const unsigned int old = atomicAdd(&slo[to * D + m], lo);
            const unsigned int hi = (unsigned int)(v >> 32) + (old + lo < old ? 1u : 0u);
            if (hi) atomicAdd(&shi[to * D + m], hi);
        }
        if (from >= 0) {
            const unsigned long long w = 0ull - v;
            const unsigned int lo = (unsigned int)w;
            const unsigned int old = atomicAdd(&slo[from * D + m], lo);
            const unsigned int hi = (unsigned int)(w >> 32) + (old + lo < old ? 1u : 0u);
            if (hi) atomicAdd(&shi[from * D + m], hi);
        }
    }
    atomicAdd(&sp[2 * k * D + to], 1u);
    if (from >= 0) atomicAdd(&sp[2 * k * D + from], 0xffffffffu);
}

// after a __syncthreads(): the CTA's partials into the global sums
template <int D>
__device__ __forceinline__ void priv_flush(const unsigned int* __restrict__ sp, int k,
                                           unsigned long long* __restrict__ acc_sum,
                                           unsigned int* __restrict__ acc_cnt)
{
    for (int i = threadIdx.x; i < k * D; i += blockDim.x) {
        const unsigned long long v = ((unsigned long long)sp[k * D + i] << 32) | sp[i];
        if (v) atomicAdd(&acc_sum[i], v);
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const unsigned int c = sp[2 * k * D + j];
        if (c) atomicAdd(&acc_cnt[j], c);
    }
}

// --------------------------------------------------------------------------
// K1 (v1): assignment, P points per thread, FP32 top-2 filter + exact FP64 certification.
// Persistent grid: CTA b handles point tiles b, b+grid, ... (tile = blockDim * P).
// Outputs per point: labels[i]; fused: changed count, SSE_t partial (FP64 exact
// distance of the chosen centroid), and (FUSE) the fixed-point sums.
template <int D, int P, bool FUSE>
__global__ void __launch_bounds__(kAssignThreads)
assign_simple_kernel(const float* __restrict__ pts, int64_t n, const float* __restrict__ C, int k, int kpad,
                     int32_t* __restrict__ labels, int first, double* __restrict__ sse_part,
                     unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                     unsigned int* __restrict__ acc_cnt, const Quant* __restrict__ quant,
                     const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    extern __shared__ float smem[];
    stage_centroids<D>(smem, C, k, kpad);
    const float* sc[D];
#pragma unroll
    for (int m = 0; m < D; ++m) sc[m] = smem + m * kpad;
    Quant q;
    if (FUSE) q = *quant;

    double sse = 0.0;
    unsigned long long chg = 0;
    const int64_t tile = (int64_t)blockDim.x * P;
    for (int64_t base = (int64_t)blockIdx.x * tile; base < n; base += (int64_t)gridDim.x * tile) {
        float p[P][D];
        float m1[P], m2[P];
        int j1[P];
#pragma unroll
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
#pragma unroll
            for (int m = 0; m < D; ++m) p[r][m] = i < n ? pts[i * D + m] : 0.0f;
            m1[r] = INFINITY; m2[r] = INFINITY; j1[r] = 0;
        }
#pragma unroll 4
        for (int j = 0; j < kpad; ++j) {
            float c[D];
#pragma unroll
            for (int m = 0; m < D; ++m) c[m] = sc[m][j];
#pragma unroll
            for (int r = 0; r < P; ++r) {
                float v = dist32<D>(p[r], c);
                bool lt = v < m1[r];
                m2[r] = lt ? m1[r] : fminf(m2[r], v);
                j1[r] = lt ? j : j1[r];
                m1[r] = fminf(m1[r], v);
            }
        }
#pragma unroll
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
            if (i >= n) continue;
            int a = j1[r];
            if (!(m2[r] > certify_thr(m1[r]))) a = exact_scan<D>(p[r], sc, k);
            sse += dist64<D>(p[r], sc, a);
            if (first) chg += 1;
            else chg += (labels[i] != a);
            labels[i] = a;
            if (FUSE) accumulate_point<D>(p[r], a, q, acc_sum, acc_cnt);
        }
    }
    block_sum2<kAssignThreads>(sse, chg);
    if (threadIdx.x == 0) { sse_part[blockIdx.x] = sse; chg_part[blockIdx.x] = chg; }
}

// Fixed-point accumulation from given labels (standalone km_update).  PRIV: per-CTA shared
// partials (accumulate_point_priv), one flush per CTA.
template <int D, bool PRIV>
__global__ void __launch_bounds__(256)
accumulate_kernel(const float* __restrict__ pts, int64_t n, const int32_t* __restrict__ labels,
                  unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt,
                  const Quant* __restrict__ quant, int k)
{
    extern __shared__ unsigned int s_priv[];
    if (PRIV) {
        priv_clear<D>(s_priv, k);
        __syncthreads();
    }
    const Quant q = *quant;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float p[D];
#pragma unroll
        for (int m = 0; m < D; ++m) p[m] = pts[i * D + m];
        if (PRIV) accumulate_point_priv<D>(p, labels[i], q, s_priv, k);
        else accumulate_point<D>(p, labels[i], q, acc_sum, acc_cnt);
    }
    if (PRIV) {
        __syncthreads();
        priv_flush<D>(s_priv, k, acc_sum, acc_cnt);
    }
}

// --------------------------------------------------------------------------
// Bounding box (per-CTA partial min/max, then quant_kernel) -> Quant.
template <int D>
__global__ void __launch_bounds__(256)
bbox_kernel(const float* __restrict__ pts, int64_t n, float* __restrict__ part)
{
    float lo[D], hi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = INFINITY; hi[m] = -INFINITY; }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) {
            float v = pts[i * D + m];
            lo[m] = fminf(lo[m], v);
            hi[m] = fmaxf(hi[m], v);
        }
    }
    __shared__ float s[2 * D][8];
#pragma unroll
    for (int m = 0; m < D; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
#pragma unroll
        for (int m = 0; m < D; ++m) { s[m][w] = lo[m]; s[D + m][w] = hi[m]; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) {
#pragma unroll
            for (int m = 0; m < D; ++m) { lo[m] = fminf(lo[m], s[m][ww]); hi[m] = fmaxf(hi[m], s[D + m][ww]); }
        }
#pragma unroll
        for (int m = 0; m < D; ++m) { part[blockIdx.x * 2 * D + m] = lo[m]; part[blockIdx.x * 2 * D + D + m] = hi[m]; }
    }
}

template <int D>
__global__ void __launch_bounds__(256) quant_kernel(const float* __restrict__ part, int nparts, int64_t n,
                                                    Quant* __restrict__ q, const Ctl* __restrict__ ctl)
{
    float lo[D], hi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = INFINITY; hi[m] = -INFINITY; }
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) { lo[m] = fminf(lo[m], part[b * 2 * D + m]); hi[m] = fmaxf(hi[m], part[b * 2 * D + D + m]); }
    }
    __shared__ float s[2 * D][8];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int m = 0; m < D; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
        if (l == 0) { s[m][w] = lo[m]; s[D + m][w] = hi[m]; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
#pragma unroll
            for (int m = 0; m < D; ++m) { lo[m] = fminf(lo[m], s[m][ww]); hi[m] = fmaxf(hi[m], s[D + m][ww]); }
        Quant h;
        make_quant(h, lo, hi, D, n);
        *q = h;
    }
    (void)ctl;
}

// --------------------------------------------------------------------------
// Data-parallel partials (one CTA): export the local fixed-point sums / counts / changed /
// SSE_t as one u64 vector + one double (and clear the accumulators), or import the
// all-reduced vector back into the accumulators for finalize.
__global__ void __launch_bounds__(1024)
export_partials_kernel(unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt, int kd, int k,
                       int ncopy, int clear, const double* __restrict__ sse_part, const unsigned long long* __restrict__ sseq_part,
                       const unsigned long long* __restrict__ chg_part, int nparts, unsigned long long* __restrict__ out_u,
                       const Quant* __restrict__ quant, unsigned long long* __restrict__ tot_reset,
                       const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    // clear = 1: per-iteration sums (brute force); 0: the tile path's running sums persist
    // ncopy > 1: the running sums are kept in ncopy private copies (summed here, exact)
    for (int i = threadIdx.x; i < kd; i += blockDim.x) {
        unsigned long long v = 0ull;
        for (int c = 0; c < ncopy; ++c) v += acc_sum[(int64_t)c * kd + i];
        out_u[i] = v;
        if (clear) acc_sum[i] = 0ull;
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        unsigned int v = 0u;
        for (int c = 0; c < ncopy; ++c) v += acc_cnt[(int64_t)c * k + j];
        out_u[kd + j] = v;
        if (clear) acc_cnt[j] = 0u;
    }
    double s = 0.0;
    unsigned long long c = 0, sq = 0;
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        if (sseq_part) sq += sseq_part[b]; else s += sse_part[b];
        c += chg_part[b];
    }
    block_sum2<1024>(s, c);
    __syncthreads();
    double dummy = 0.0;
    block_sum2<1024>(dummy, sq);
    if (threadIdx.x == 0) {
        if (tot_reset) { tot_reset[0] = 0ull; tot_reset[1] = 0ull; }
        out_u[kd + k] = c;
        // SSE_t as one fixed-point word at the GLOBAL scale 2^s2 (n_global E^2 2^s2 < 2^62):
        // the ranks' words add exactly in the same all-reduce as the sums
        out_u[kd + k + 1] = sseq_part ? sq : sse_q(s, quant->sse_scale);
    }
}

__global__ void __launch_bounds__(1024)
import_partials_kernel(const unsigned long long* __restrict__ in_u, int kd, int k,
                       unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt,
                       double* __restrict__ sse_part, unsigned long long* __restrict__ chg_part,
                       const Quant* __restrict__ quant, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    for (int i = threadIdx.x; i < kd; i += blockDim.x) acc_sum[i] = in_u[i];
    for (int j = threadIdx.x; j < k; j += blockDim.x) acc_cnt[j] = (unsigned int)in_u[kd + j];
    if (threadIdx.x == 0) {
        sse_part[0] = __dmul_rn((double)in_u[kd + k + 1], quant->sse_inv);
        chg_part[0] = in_u[kd + k];
    }
}

// --------------------------------------------------------------------------
// K3 finalize (one CTA of NT threads): new centroids from the fixed-point sums, drift, traces,
// convergence flag; clears the accumulators for the next iteration.  Used as its own kernel
// (finalize_kernel) and as the tail of the brute-force assignment (the CTA that finishes last,
// assign_scan_kernel), so a brute-force iteration is one launch.
struct FinArgs {
    const float* Cold;
    float* Cnew;
    int k;
    unsigned long long* acc_sum;
    unsigned int* acc_cnt;
    int ncopy, clear;
    const Quant* quant;
    int32_t* counts_out;
    double* maxdrift_out;
    const double* sse_part;
    const unsigned long long* sseq_part;
    const unsigned long long* chg_part;
    int nparts;
    double* sse_trace;
    long long* chg_trace;
    double* drift_trace;
    unsigned int* cb2_reset;
    unsigned long long* tot_reset;
    Ctl* ctl;
    float tol;
};

template <int D, int NT>
__device__ __forceinline__ void finalize_block(const FinArgs& f)
{
    const Quant q = *f.quant;
    const int k = f.k;
    double md = 0.0;
    for (int j = threadIdx.x; j < k; j += NT) {
        unsigned int c = 0u;   // ncopy (<= kMaxAccCopies) private copies of the running sums add up exactly
#pragma unroll
        for (int cp = 0; cp < kMaxAccCopies; ++cp)
            if (cp < f.ncopy) c += f.acc_cnt[(int64_t)cp * k + j];   // all loads in flight at once
        double dd = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            int64_t idx = (int64_t)j * D + m;
            float old = f.Cold[idx];
            float nw = old;
            if (c > 0) {
                unsigned long long sv = 0ull;
#pragma unroll
                for (int cp = 0; cp < kMaxAccCopies; ++cp)
                    if (cp < f.ncopy) sv += f.acc_sum[(int64_t)cp * k * D + idx];
                double mean = __dadd_rn(q.o[m], __dmul_rn(__ddiv_rn((double)sv, (double)c), q.inv[m]));
                nw = __double2float_rn(mean);
            }
            double t = __dsub_rn((double)nw, (double)old);
            dd = __dadd_rn(dd, __dmul_rn(t, t));
            f.Cnew[idx] = nw;
            if (f.clear) f.acc_sum[idx] = 0ull;
        }
        if (f.clear) f.acc_cnt[j] = 0u;
        if (f.cb2_reset) f.cb2_reset[j] = 0x7f800000u;   // +inf: the next inter-bound pass takes minima
        if (f.counts_out) f.counts_out[j] = (int32_t)c;
        md = fmax(md, sqrt(dd));
    }
    // deterministic reductions: max drift, SSE_t, changed_t
    __shared__ double s_md[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if ((threadIdx.x & 31) == 0) s_md[threadIdx.x >> 5] = md;
    double sse = 0.0;
    unsigned long long chg = 0, sq = 0;
    for (int b = threadIdx.x; b < f.nparts; b += NT) {
        if (f.sseq_part) sq += f.sseq_part[b]; else sse += f.sse_part[b];
        chg += f.chg_part[b];
    }
    __syncthreads();
    block_sum2<NT>(sse, chg);
    __syncthreads();
    double dummy = 0.0;
    block_sum2<NT>(dummy, sq);
    if (threadIdx.x == 0) {
        if (f.tot_reset) { f.tot_reset[0] = 0ull; f.tot_reset[1] = 0ull; }   // the tile path's totals, read above
        if (f.sseq_part) sse = __dmul_rn((double)sq, q.sse_inv);   // integer sum: order-independent
        for (int w = 1; w < NT / 32; ++w) md = fmax(md, s_md[w]);
        if (f.maxdrift_out) *f.maxdrift_out = md;
        if (f.ctl) {
            Ctl* ctl = f.ctl;
            int t = ctl->iter;
            if (f.sse_trace) f.sse_trace[t] = sse;
            if (f.chg_trace) f.chg_trace[t] = (long long)chg;
            if (f.drift_trace) f.drift_trace[t] = md;
            ctl->iter = t + 1;
            if (f.tol >= 0.0f && (md <= (double)f.tol || (t >= 1 && chg == 0))) ctl->done = 1;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kFinalizeThreads)
finalize_kernel(FinArgs f)
{
    if (f.ctl && f.ctl->done) return;
    finalize_block<D, kFinalizeThreads>(f);
}

// --------------------------------------------------------------------------
// The tile path's refine spread over ceil(k / 256) CTAs (the single-CTA finalize_kernel is
// latency-bound at k = 10^3): each CTA refines its centroids from the ncopy private running
// sums (exact integers) and folds its max drift into fin[0] (FP64 bits, atomicMax); the last
// CTA to finish (ticket fin[1]) writes the traces and the convergence flag and resets the
// iteration totals.  Same arithmetic and results as finalize_kernel.
template <int D>
__global__ void __launch_bounds__(256)
finalize_grid_kernel(float* __restrict__ C, int k, const unsigned long long* __restrict__ acc_sum,
                     const unsigned int* __restrict__ acc_cnt, int ncopy, const Quant* __restrict__ quant,
                     unsigned long long* __restrict__ tot, unsigned int* __restrict__ cb2_reset,
                     unsigned long long* __restrict__ fin, double* __restrict__ sse_trace,
                     long long* __restrict__ chg_trace, double* __restrict__ drift_trace, Ctl* __restrict__ ctl,
                     float tol)
{
    if (ctl && ctl->done) return;
    const Quant q = *quant;
    double md = 0.0;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) {
        unsigned int c = 0u;
#pragma unroll
        for (int cp = 0; cp < kMaxAccCopies; ++cp)
            if (cp < ncopy) c += acc_cnt[(int64_t)cp * k + j];
        double dd = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const int64_t idx = (int64_t)j * D + m;
            const float old = C[idx];
            float nw = old;
            if (c > 0) {
                unsigned long long sv = 0ull;
#pragma unroll
                for (int cp = 0; cp < kMaxAccCopies; ++cp)
                    if (cp < ncopy) sv += acc_sum[(int64_t)cp * k * D + idx];
                const double mean = __dadd_rn(q.o[m], __dmul_rn(__ddiv_rn((double)sv, (double)c), q.inv[m]));
                nw = __double2float_rn(mean);
            }
            const double t = __dsub_rn((double)nw, (double)old);
            dd = __dadd_rn(dd, __dmul_rn(t, t));
            C[idx] = nw;
        }
        cb2_reset[j] = 0x7f800000u;   // +inf: the next inter-bound pass takes minima
        md = sqrt(dd);
    }
    __shared__ double s_md[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if ((threadIdx.x & 31) == 0) s_md[threadIdx.x >> 5] = md;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) md = fmax(md, s_md[w]);
        if (md > 0.0) atomicMax(&fin[0], (unsigned long long)__double_as_longlong(md));
        __threadfence();
        const unsigned long long ticket = atomicAdd(&fin[1], 1ull);
        if (ticket == gridDim.x - 1) {   // the last CTA: every other CTA's drift is in fin[0]
            __threadfence();
            const double mdall = __longlong_as_double((long long)atomicAdd(&fin[0], 0ull));
            const unsigned long long chg = tot[1];
            const double sse = __dmul_rn((double)tot[0], q.sse_inv);
            const int t = ctl->iter;
            if (sse_trace) sse_trace[t] = sse;
            if (chg_trace) chg_trace[t] = (long long)chg;
            if (drift_trace) drift_trace[t] = mdall;
            ctl->iter = t + 1;
            if (tol >= 0.0f && (mdall <= (double)tol || (t >= 1 && chg == 0))) ctl->done = 1;
            tot[0] = 0ull;
            tot[1] = 0ull;
            fin[0] = 0ull;
            fin[1] = 0ull;
        }
    }
}

// --------------------------------------------------------------------------
// Eq. 1 of the returned pair as an ORDER-INDEPENDENT sum: each point's FP64
// distance D_i (oracle order) is rounded to an integer multiple of 2^-s3 and the integers are
// added in 128 bits, so out_sse is the same number for any grid, work order, path (tiles or
// brute force) and sharding (km_dp_end / km_dp_sse).  s3: n * B * 2^s3 (1 + 2^-20) < 2^126,
// where B bounds every D_i (low-d: the squared diagonal of the points' box united with the
// centroids' box); the error is <= n * 2^-(s3+1), i.e. ~2^-100 of n * B.
typedef unsigned __int128 u128;

struct SseFix {                       // device result of sse_fix_reduce_kernel (64 B)
    double value;                     // the sum as FP64: (hi * 2^64 + lo) * 2^-s3
    double inv;                       // 2^-s3
    unsigned long long limb[3];       // the 128-bit sum in 48-bit limbs (carry-free sums over ranks)
    unsigned long long pad[3];
};

__device__ __forceinline__ int sse_shift(double bound, long long n)
{
    const double tot = (double)n * bound * (1.0 + 0x1p-20);
    int e = 0;
    if (tot > 0.0) frexp(tot, &e);   // tot < 2^e
    return tot > 0.0 ? 126 - e : 0;
}

__device__ __forceinline__ void add_fix(u128& acc, double d, double scale)
{
    const double v = rint(__dmul_rn(d, scale));                          // exact scaling, one rounding
    const unsigned long long hi = (unsigned long long)__dmul_rn(v, 0x1p-64);
    const double rem = __dsub_rn(v, __dmul_rn((double)hi, 0x1p64));     // exact: a subset of v's bits
    acc += ((u128)hi << 64) + (unsigned long long)rem;
}

__device__ __forceinline__ u128 warp_sum128(u128 v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
        const unsigned long long hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(v >> 64), o);
        v += ((u128)hi << 64) | lo;
    }
    return v;
}

// block sum (blockDim <= 1024) -> thread 0
__device__ __forceinline__ u128 block_sum128(u128 v)
{
    __shared__ unsigned long long s_lo[32], s_hi[32];
    v = warp_sum128(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { s_lo[w] = (unsigned long long)v; s_hi[w] = (unsigned long long)(v >> 64); }
    __syncthreads();
    v = 0;
    if (w == 0) {
        if (l < (int)(blockDim.x >> 5)) v = ((u128)s_hi[l] << 64) | s_lo[l];
        v = warp_sum128(v);
    }
    return v;
}

// s3 of the low-d path (one CTA): B = squared diagonal of the points' box united with the
// centroids' box.
template <int D>
__global__ void __launch_bounds__(kReduceThreads)
sse_bound_kernel(const Quant* __restrict__ quant, const float* __restrict__ C, int k, int* __restrict__ s3_out)
{
    __shared__ float s_b[2 * D][32];
    const Quant q = *quant;
    float lo[D], hi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = (float)q.o[m]; hi[m] = q.hi[m]; }
    for (int j = threadIdx.x; j < k; j += blockDim.x)
#pragma unroll
        for (int m = 0; m < D; ++m) { lo[m] = fminf(lo[m], C[(int64_t)j * D + m]); hi[m] = fmaxf(hi[m], C[(int64_t)j * D + m]); }
#pragma unroll
    for (int m = 0; m < D; ++m)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0)
#pragma unroll
        for (int m = 0; m < D; ++m) { s_b[m][w] = lo[m]; s_b[D + m][w] = hi[m]; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int m = 0; m < D; ++m) {
            float a = s_b[m][0], z = s_b[D + m][0];
            for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww) { a = fminf(a, s_b[m][ww]); z = fmaxf(z, s_b[D + m][ww]); }
            const double e = (double)z - (double)a;
            b += e * e;
        }
        *s3_out = sse_shift(b, q.n);
    }
}

// Eq. 1 of (labels, C), low d: per-CTA 128-bit partials part[2b], part[2b + 1].
template <int D>
__global__ void __launch_bounds__(256)
sse_kernel(const float* __restrict__ pts, int64_t n, const int32_t* __restrict__ labels,
           const float* __restrict__ C, const int* __restrict__ s3, unsigned long long* __restrict__ part)
{
    const double scale = ldexp(1.0, *s3);
    u128 acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int a = labels[i];
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double t = __dsub_rn((double)pts[i * D + m], (double)C[(int64_t)a * D + m]);
            v = __dadd_rn(v, __dmul_rn(t, t));
        }
        add_fix(acc, v, scale);
    }
    acc = block_sum128(acc);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = (unsigned long long)acc;
        part[2 * blockIdx.x + 1] = (unsigned long long)(acc >> 64);
    }
}

// The 128-bit total of nparts partials (one CTA) -> SseFix.
__global__ void __launch_bounds__(kReduceThreads)
sse_fix_reduce_kernel(const unsigned long long* __restrict__ part, int nparts, const int* __restrict__ s3,
                      SseFix* __restrict__ out)
{
    u128 acc = 0;
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) acc += ((u128)part[2 * b + 1] << 64) | part[2 * b];
    acc = block_sum128(acc);
    if (threadIdx.x == 0) {
        const double inv = ldexp(1.0, -*s3);
        const double hi = (double)(unsigned long long)(acc >> 64), lo = (double)(unsigned long long)acc;
        out->value = __dmul_rn(__dadd_rn(__dmul_rn(hi, 0x1p64), lo), inv);
        out->inv = inv;
        const unsigned long long m48 = (1ull << 48) - 1;
        out->limb[0] = (unsigned long long)acc & m48;
        out->limb[1] = (unsigned long long)(acc >> 48) & m48;
        out->limb[2] = (unsigned long long)(acc >> 96);
    }
}

// Sum per-CTA partials in a fixed order into out[0] (double) / out_u (nullable).
__global__ void __launch_bounds__(kReduceThreads)
reduce_parts_kernel(const double* __restrict__ part, const unsigned long long* __restrict__ upart, int nparts,
                    double* __restrict__ out, unsigned long long* __restrict__ out_u)
{
    double s = 0.0;
    unsigned long long u = 0;
    for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
        s += part[b];
        if (upart) u += upart[b];
    }
    block_sum2<kReduceThreads>(s, u);
    if (threadIdx.x == 0) {
        if (out) *out = s;
        if (out_u) *out_u = u;
    }
}

}  // namespace km
