// km_assign_fast.cuh -- K1 (fast): the brute-force assignment scan with packed FP32x2 math.
//
// Per point, the exact label is argmin_j of the FP64 direct-form distance (R1, R2;
// Lloyd's assignment).  The scan computes the FP32 direct-form distance
//     D32_j = fma(dz,dz, fma(dy,dy, dx*dx)),  dm = p_m + (-c_jm)   (RN everywhere)
// for two centroids at a time with FADD2/FMUL2/FFMA2 and keeps, per point, the best
// BLOCK of centroids (its minimum m1 and index b1) and the second-best block minimum
// m2.  A block is a group of 4 centroids (GROUP bookkeeping: per 4 pairs) or a chunk
// of kChunk centroids (CHUNK bookkeeping: a lazy running minimum, one FMNMX3 per 2
// pairs, block update once per chunk).  Certification:
// |D32 - D64| <= 5.01u D64 (u = 2^-24), so every j with D32_j > thr(m1) =
// m1 (1 + 2^-19) is not the FP64 argmin.  If m2 > thr, the FP64 argmin lies in block
// b1: re-evaluate its centroids with the identical FP32 operations; if exactly one is
// <= thr it is the label, otherwise compare the block in FP64.  If m2 <= thr (a
// cross-block near-tie) the point takes the exact FP64 scan of all k.
#pragma once
#include <cuda_runtime.h>
#include "km_kernels.cuh"

namespace km {

constexpr int kChunk = 32;

template <int D>
struct Pt {
    float v[D];
};

// FP64 distance against a NEGATED centroid (p + (-c) == p - c exactly), oracle order.
template <int D>
__device__ __forceinline__ double dist64n(const Pt<D>& p, const float* __restrict__ nc, int kpad, int j)
{
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        double t = __dadd_rn((double)p.v[m], (double)nc[m * kpad + j]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

// Exact FP64 argmin over j in [j0, j1), lowest index on ties (strict <, ascending j).
template <int D>
__device__ __noinline__ int exact_scan_v(Pt<D> p, const float* __restrict__ nc, int kpad, int j0, int j1)
{
    double best = INFINITY;
    int a = j0;
    for (int j = j0; j < j1; ++j) {
        double v = dist64n<D>(p, nc, kpad, j);
        if (v < best) { best = v; a = j; }
    }
    return a;
}

template <int D>
__device__ __forceinline__ float dist32n(const Pt<D>& p, const float* __restrict__ nc, int kpad, int j)
{
    float t = __fadd_rn(p.v[0], nc[j]);
    float s = __fmul_rn(t, t);
#pragma unroll
    for (int m = 1; m < D; ++m) {
        t = __fadd_rn(p.v[m], nc[m * kpad + j]);
        s = __fmaf_rn(t, t, s);
    }
    return s;
}

// Certified label of one point given (m1, b1, m2) over blocks of B centroids.
template <int D, int B>
__device__ __forceinline__ int certify_label(const Pt<D>& p, float m1, float m2, int b1, const float* __restrict__ nc,
                                             int kpad, int k)
{
    const float thr = certify_thr(m1);
    if (!(m2 > thr)) return exact_scan_v<D>(p, nc, kpad, 0, k);
    const int j0 = b1 * B;
    const int lane = threadIdx.x & 31;
    int cnt = 0, a = 0x7fffffff;
#pragma unroll 4
    for (int u = 0; u < B; ++u) {
        const int j = j0 + ((u + lane) & (B - 1));   // lane swizzle: conflict-free shared reads
        if (dist32n<D>(p, nc, kpad, j) <= thr) { ++cnt; a = min(a, j); }
    }
    if (cnt != 1) a = exact_scan_v<D>(p, nc, kpad, j0, min(j0 + B, k));
    return a;
}

// certify_label that also returns sec: the smallest FP32 distance over j != a (the second
// smallest block minimum m2 and the rest of block b1), or -1 when the label came from an FP64
// scan (no bound: the point is scanned again next iteration).
template <int D, int B>
__device__ __forceinline__ int certify_label_sec(const Pt<D>& p, float m1, float m2, int b1,
                                                 const float* __restrict__ nc, int kpad, int k, float& sec)
{
    const float thr = certify_thr(m1);
    sec = -1.0f;
    if (!(m2 > thr)) return exact_scan_v<D>(p, nc, kpad, 0, k);
    const int j0 = b1 * B;
    const int lane = threadIdx.x & 31;
    int cnt = 0, a = 0x7fffffff;
    float dj[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
        const int j = j0 + ((u + lane) & (B - 1));   // lane swizzle: conflict-free shared reads
        dj[u] = dist32n<D>(p, nc, kpad, j);
        if (dj[u] <= thr) { ++cnt; a = min(a, j); }
    }
    if (cnt != 1) return exact_scan_v<D>(p, nc, kpad, j0, min(j0 + B, k));
    float s2 = m2;
#pragma unroll
    for (int u = 0; u < B; ++u)
        if (j0 + ((u + lane) & (B - 1)) != a) s2 = fminf(s2, dj[u]);   // (-inf padding: +inf distances)
    sec = s2;
    return a;
}

// Two pairs (centroids 2h, 2h+1 of the float4 group) for one point: packed direct form.
template <int D>
__device__ __forceinline__ float2 pair2(const Pt<D>& p, const float4 (&c)[D], bool hi)
{
    float2 t = __fadd2_rn(make_float2(p.v[0], p.v[0]), hi ? make_float2(c[0].z, c[0].w) : make_float2(c[0].x, c[0].y));
    float2 s = __fmul2_rn(t, t);
#pragma unroll
    for (int m = 1; m < D; ++m) {
        t = __fadd2_rn(make_float2(p.v[m], p.v[m]), hi ? make_float2(c[m].z, c[m].w) : make_float2(c[m].x, c[m].y));
        s = __ffma2_rn(t, t, s);
    }
    return s;
}

// Hamerly bounds in distance units, rounded outward.  lower_dist: a lower bound of
// the true distance from an FP32 direct-form squared distance D32 (|D32 - D| <= 5.01u D +
// subnormal slack, u = 2^-24): sqrt((D32 - 2^-120)(1 - 2^-20)) rounded down; -1 -> 0.
__device__ __forceinline__ float lower_dist(float d32)
{
    if (!(d32 > 0x1p-120f)) return 0.0f;
    return __fsqrt_rd(__fmul_rd(__fsub_rd(d32, 0x1p-120f), 1.0f - 0x1p-20f));
}

// One round of the scan: PP points per thread, points base + r * blockDim + tid (r < PP) --
// or, with a queue qi (bounds kernel), the points qi[base + r * blockDim + tid] (base + ... < hi),
// whose new lower bound of the second-nearest distance goes to lbv (Hamerly bounds).
template <int D, int PP, bool CHUNKED, int FUSE>
__device__ __forceinline__ void scan_round(int64_t base, int64_t hi, const float* __restrict__ pts,
                                           const float* smem, int k, int kpad, int32_t* __restrict__ labels,
                                           int first, const Quant& q, unsigned long long* __restrict__ acc_sum,
                                           unsigned int* __restrict__ acc_cnt, unsigned int* spriv, double& sse,
                                           unsigned long long& chg, const int* qi = nullptr,
                                           float* __restrict__ lbv = nullptr)
{
    const float4* nc4 = reinterpret_cast<const float4*>(smem);
    const int kq = kpad >> 2;   // float4 groups per coordinate
    const int ngroups = kq;
    Pt<D> p[PP];
    float m1[PP], m2[PP];
    int b1[PP], old[PP];
    int64_t ii[PP];
#pragma unroll
    for (int r = 0; r < PP; ++r) {
        const int64_t e = base + (int64_t)r * blockDim.x + threadIdx.x;
        ii[r] = e < hi ? (qi ? (int64_t)qi[e] : e) : -1;
    }
    // a warp without points skips the round (the tail rounds of a short queue)
    if (!__any_sync(0xffffffffu, base + (int64_t)(threadIdx.x & ~31) < hi)) return;
#pragma unroll
    for (int r = 0; r < PP; ++r) {
        const int64_t i = ii[r];
#pragma unroll
        for (int m = 0; m < D; ++m) p[r].v[m] = i >= 0 ? pts[i * D + m] : 0.0f;
        // the previous labels load with the points (their latency hides behind the scan)
        old[r] = (!first && i >= 0) ? labels[i] : -1;
        m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0;
    }
    if (CHUNKED) {
        constexpr int GPC = kChunk / 4;   // float4 groups per chunk
        const int nchunks = ngroups / GPC;
        for (int ch = 0; ch < nchunks; ++ch) {
            float mc[PP];
#pragma unroll
            for (int r = 0; r < PP; ++r) mc[r] = INFINITY;
#pragma unroll
            for (int gg = 0; gg < GPC; ++gg) {
                const int g = ch * GPC + gg;
                float4 c[D];
#pragma unroll
                for (int m = 0; m < D; ++m) c[m] = nc4[m * kq + g];
#pragma unroll
                for (int r = 0; r < PP; ++r) {
                    float2 s0 = pair2<D>(p[r], c, false);
                    float2 s1 = pair2<D>(p[r], c, true);
                    mc[r] = fminf(fminf(mc[r], s0.x), s0.y);
                    mc[r] = fminf(fminf(mc[r], s1.x), s1.y);
                }
            }
#pragma unroll
            for (int r = 0; r < PP; ++r) {
                bool lt = mc[r] < m1[r];
                m2[r] = fmaxf(m1[r], fminf(m2[r], mc[r]));   // second smallest of {m1, m2, mc}
                m1[r] = fminf(m1[r], mc[r]);
                b1[r] = lt ? ch : b1[r];
            }
        }
    } else {
#pragma unroll 2
        for (int g = 0; g < ngroups; ++g) {
            float4 c[D];
#pragma unroll
            for (int m = 0; m < D; ++m) c[m] = nc4[m * kq + g];
#pragma unroll
            for (int r = 0; r < PP; ++r) {
                float2 s0 = pair2<D>(p[r], c, false);
                float2 s1 = pair2<D>(p[r], c, true);
                float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
                bool lt = v < m1[r];
                m2[r] = fmaxf(m1[r], fminf(m2[r], v));
                m1[r] = fminf(m1[r], v);
                b1[r] = lt ? g : b1[r];
            }
        }
    }
#pragma unroll
    for (int r = 0; r < PP; ++r) {
        const int64_t i = ii[r];
        if (i < 0) continue;
        int a;
        if (lbv) {
            float sec;
            a = certify_label_sec<D, CHUNKED ? kChunk : 4>(p[r], m1[r], m2[r], b1[r], smem, kpad, k, sec);
            lbv[i] = lower_dist(sec);
        } else {
            a = certify_label<D, CHUNKED ? kChunk : 4>(p[r], m1[r], m2[r], b1[r], smem, kpad, k);
        }
        sse += dist64n<D>(p[r], smem, kpad, a);
        chg += old[r] != a ? 1ull : 0ull;
        if (old[r] != a) labels[i] = a;
        if (FUSE == 1) accumulate_point<D>(p[r].v, a, q, acc_sum, acc_cnt);
        if (FUSE == 2) accumulate_point_priv<D>(p[r].v, a, q, spriv, k);
        if (FUSE == 3 && old[r] != a) move_point_priv<D>(p[r].v, old[r], a, q, spriv, k);
    }
}

// FUSE: 0 labels only (km_assign), 1 fused update with per-point global REDs, 2 fused update
// privatised in shared memory (accumulate_point_priv; the default when k(2d+1)*4 B fits),
// 3 the same privatised partials of an INCREMENTAL update: only points whose label changed
// (all of them at t = 0) move their value between the running sums (move_point_priv), which
// the refine keeps (km_run_ctx's brute-force loop).
template <int D, int P, int MINB, bool CHUNKED, int FUSE>
__global__ void __launch_bounds__(kAssignThreads, MINB)
assign_scan_kernel(const float* __restrict__ pts, int64_t n, const float* C, int k, int kpad,
                   int32_t* __restrict__ labels, int first, double* __restrict__ sse_part,
                   unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                   unsigned int* __restrict__ acc_cnt, const Quant* __restrict__ quant, const Ctl* ctl,
                   unsigned int* __restrict__ tick, const FinArgs fin)
{
    // tick != nullptr: the CTA that finishes last runs the refine (finalize_block) -- one launch
    // per brute-force iteration (C is then rewritten in place, after every CTA has read it)
    if (ctl && ctl->done) return;
    extern __shared__ __align__(16) float smem[];
    // stage NEGATED centroids, SoA, padded with -inf (p + -inf = -inf, squared = +inf: pads never win)
    for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) smem[m * kpad + j] = j < k ? -C[(int64_t)j * D + m] : -INFINITY;
    }
    unsigned int* const spriv = reinterpret_cast<unsigned int*>(smem + D * kpad);
    if (FUSE >= 2) priv_clear<D>(spriv, k);
    __syncthreads();
    Quant q;
    if (FUSE) q = *quant;
    double sse = 0.0;
    unsigned long long chg = 0;
    // CTA b scans the contiguous range [b n / grid, (b + 1) n / grid): rounds of P points per
    // thread, the remainder in ONE round of P/2 or P/4 points per thread (no CTA runs a whole
    // extra round for a few points)
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    const int64_t tile = (int64_t)blockDim.x * P;
    int64_t base = lo;
    for (; hi - base > tile / 2; base += tile)
        scan_round<D, P, CHUNKED, FUSE>(base, hi, pts, smem, k, kpad, labels, first, q, acc_sum, acc_cnt, spriv, sse, chg);
    if (P >= 4 && hi - base > tile / 4)
        scan_round<D, (P >= 2 ? P / 2 : 1), CHUNKED, FUSE>(base, hi, pts, smem, k, kpad, labels, first, q, acc_sum,
                                                        acc_cnt, spriv, sse, chg);
    else if (hi - base > 0)
        scan_round<D, (P >= 4 ? P / 4 : 1), CHUNKED, FUSE>(base, hi, pts, smem, k, kpad, labels, first, q, acc_sum,
                                                        acc_cnt, spriv, sse, chg);
    if (FUSE >= 2) {
        __syncthreads();
        priv_flush<D>(spriv, k, acc_sum, acc_cnt);
    }
    block_sum2<kAssignThreads>(sse, chg);
    if (threadIdx.x == 0) { sse_part[blockIdx.x] = sse; chg_part[blockIdx.x] = chg; }
    if (tick) {
        __shared__ bool s_last;
        __threadfence();   // this CTA's partials and sum REDs before its ticket
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(tick, 1u) == gridDim.x - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            finalize_block<D, kAssignThreads>(fin);
            if (threadIdx.x == 0) *tick = 0u;
        }
    }
}

// K1b: the brute-force iteration with per-point Hamerly bounds (KM_MODE_BOUNDS; the drift lower
// bound of P:L135 applied to the second-nearest centroid, the inter bound of Eq. 4).
// Every point keeps lb[i], a lower bound of its distance to every centroid other than its label
// a(i).  Per iteration, for every point (t >= 1):
//   D64 = ||p - c_a||^2 in FP64, oracle order      (its exact distance; also its SSE_t term)
//   lb' = lb - dmax                                 (dmax >= max_j ||c_j^t - c_j^(t-1)||)
//   D64 (1 + 2^-40) < RD(B^2), B = max(lb', s_a) > 0, s_a = min_{l != a} ||c_a - c_l|| / 2
//   rounded down (Eq. 4): every other centroid is strictly farther -> a(i) stays, no scan;
//   lb[i] = lb'.
// The other points (all of them at t = 0) are queued in shared memory and scanned densely
// (scan_round over the queue: FP32 scan + FP64 certification, new lb from the second-best FP32
// distance).  Bounds are rounded outward, so a skip is never wrong; the result
// is the brute-force path's bit for bit.  Incremental privatised sums (FUSE 3).
//
// The refine of iteration t-1 runs at the START of launch t, in every CTA (the same arithmetic
// as finalize_block: c_j = RN_f32(o + sv(j)/|S_j| / scale), drift): no CTA waits
// for a last one, and every CTA has the drift bound and the convergence decision it
// needs.  CTA 0 stores C^t (double-buffered: CTAs of launch t read C^(t-1)), the traces of
// iteration t-1 and the iteration count; the partials are double-buffered the same way.
// bounds_tail_kernel refines the last iteration.
constexpr int kBoundsChunk = 2048;   // points tested per CTA before the queued ones are scanned
constexpr int kBoundsMaxKS = 256;    // the s_a test (k^2 distances per CTA) only for k <= 256
template <int D>
__host__ __device__ constexpr size_t bounds_smem_extra(int k)
{
    return (size_t)kBoundsChunk * 8 + (size_t)k * 4;
}

struct BoundsIO {
    const float* cprev;                    // t == 0: C^0; t >= 1: C^(t-1)
    float* cout;                           // t >= 1: C^t (written by CTA 0)
    // running sums S_(t-1) = S_(t-2) + D_(t-1), double-buffered S and triple-buffered deltas D
    const unsigned long long* s_prev;      // S_(t-2) (zero for t = 1)
    const unsigned int* sn_prev;
    const unsigned long long* d_prev;      // D_(t-1): the deltas launch t-1 flushed
    const unsigned int* dn_prev;
    unsigned long long* s_out;             // S_(t-1), written by CTA 0
    unsigned int* sn_out;
    unsigned long long* d_zero;            // D_(t+1): zeroed by CTA 0 (last read by launch t-1)
    unsigned int* dn_zero;
    unsigned long long* d_cur;             // this launch's deltas (privatised flush)
    unsigned int* dn_cur;
    const double* sse_prev;                // iteration t-1's per-CTA partials (double-buffered)
    const unsigned long long* chg_prev;
    double* sse_cur;
    unsigned long long* chg_cur;
    int nparts;                            // CTAs of the scan launches
    double* sse_trace;
    long long* chg_trace;
    double* drift_trace;
    Ctl* ctl;
    float tol;
    int t;
};

// The refine of iteration t-1 from S_(t-1) (finalize_block's arithmetic), into the negated SoA
// copy nc (nullable) and, by the publishing CTA, into io.cout with S_(t-1), the traces of
// iteration t-1 and the iteration count.  Returns true when the run has converged;
// *dmax: the largest drift rounded up to float.
template <int D, int NT>
__device__ __forceinline__ bool bounds_refine(const BoundsIO& io, const Quant& q, int k, int kpad, float* nc,
                                              bool publish, bool need_chg, float* dmax)
{
    __shared__ double s_md[NT / 32];
    __shared__ unsigned long long s_chg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double md = 0.0;
    for (int j = threadIdx.x; j < kpad; j += NT) {
        if (j >= k) {
            if (nc)
#pragma unroll
                for (int m = 0; m < D; ++m) nc[m * kpad + j] = -INFINITY;
            continue;
        }
        const unsigned int c = io.sn_prev[j] + io.dn_prev[j];   // (mod 2^32: exact)
        if (publish) { io.sn_out[j] = c; io.dn_zero[j] = 0u; }
        double dd = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const int64_t idx = (int64_t)j * D + m;
            const unsigned long long sv = io.s_prev[idx] + io.d_prev[idx];   // (mod 2^64: exact)
            if (publish) { io.s_out[idx] = sv; io.d_zero[idx] = 0ull; }
            const float old = io.cprev[idx];
            float nw = old;
            if (c > 0) {
                const double mean = __dadd_rn(q.o[m], __dmul_rn(__ddiv_rn((double)sv, (double)c), q.inv[m]));
                nw = __double2float_rn(mean);
            }
            const double tt = __dsub_rn((double)nw, (double)old);
            dd = __dadd_rn(dd, __dmul_rn(tt, tt));
            if (nc) nc[m * kpad + j] = -nw;
            if (publish) io.cout[idx] = nw;
        }
        md = fmax(md, sqrt(dd));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
    if (lane == 0) s_md[wid] = md;
    // changed_(t-1) (convergence test; trace) and SSE_(t-1) (trace)
    double sse = 0.0;
    unsigned long long chg = 0;
    if (need_chg || publish)
        for (int b = threadIdx.x; b < io.nparts; b += NT) {
            chg += io.chg_prev[b];
            if (publish) sse += io.sse_prev[b];
        }
    __syncthreads();
    md = s_md[0];
    for (int w = 1; w < NT / 32; ++w) md = fmax(md, s_md[w]);
    block_sum2<NT>(sse, chg);   // (thread 0 holds the totals)
    if (threadIdx.x == 0) {
        s_chg = chg;
        if (publish) {
            const int tp = io.t - 1;
            if (io.sse_trace) io.sse_trace[tp] = sse;
            if (io.chg_trace) io.chg_trace[tp] = (long long)chg;
            if (io.drift_trace) io.drift_trace[tp] = md;
            io.ctl->iter = io.t;
        }
    }
    __syncthreads();
    *dmax = __double2float_ru(__dmul_ru(md, 1.0 + 0x1p-40));
    const bool conv = io.tol >= 0.0f && (md <= (double)io.tol || (io.t - 1 >= 1 && s_chg == 0));
    if (conv && publish && threadIdx.x == 0) io.ctl->done = 1;
    return conv;
}

template <int D, int P, int MINB>
__global__ void __launch_bounds__(kAssignThreads, MINB)
bounds_scan_kernel(const float* __restrict__ pts, int64_t n, int k, int kpad, int32_t* __restrict__ labels,
                   float* __restrict__ lbv, const Quant* __restrict__ quant, unsigned long long* __restrict__ nscan,
                   const BoundsIO io)
{
    // programmatic dependent launch: the next iteration's grid may be scheduled as this one's
    // CTAs retire; this grid reads the previous one's outputs only after it has completed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef KM_BPROF
    // (profiling builds) phase times of thread 0 summed over CTAs into nscan[1..5] (ns)
    unsigned long long tp0, tp1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp0));
#define KM_BP(slot) do { if (threadIdx.x == 0 && nscan) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1)); \
        atomicAdd(nscan + (slot), tp1 - tp0); tp0 = tp1; } } while (0)
#else
#define KM_BP(slot) do { } while (0)
#endif
    if (io.ctl->done) return;
    extern __shared__ __align__(16) float smem[];
    unsigned int* const spriv = reinterpret_cast<unsigned int*>(smem + D * kpad);
    int* const sq = reinterpret_cast<int*>(spriv + (size_t)k * (2 * D + 1));   // per-warp queues [kBoundsChunk]
    int* const sq2 = sq + kBoundsChunk;                                       // the dense queue [kBoundsChunk]
    float* const s_half = reinterpret_cast<float*>(sq2 + kBoundsChunk);      // s_a [k]
    __shared__ int s_wq[kAssignThreads / 32];
    const int wid = threadIdx.x >> 5;
    int* const sqw = sq + wid * (kBoundsChunk / (kAssignThreads / 32));
    int wq = 0;
    const int first = io.t == 0;
    const Quant q = *quant;
    const int lane = threadIdx.x & 31;
    float dmax = 0.0f;
    if (first) {
        for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
#pragma unroll
            for (int m = 0; m < D; ++m) smem[m * kpad + j] = j < k ? -io.cprev[(int64_t)j * D + m] : -INFINITY;
        }
        if (blockIdx.x == 0)   // D_1 (zero before launch 1 flushes into it)
            for (int i = threadIdx.x; i < k * (D + 1); i += blockDim.x) {
                if (i < k * D) io.d_zero[i] = 0ull;
                else io.dn_zero[i - k * D] = 0u;
            }
    } else if (bounds_refine<D, kAssignThreads>(io, q, k, kpad, smem, blockIdx.x == 0, io.tol >= 0.0f, &dmax)) {
        return;   // converged: C^t (in io.cout) is the result
    }
    KM_BP(1);
    priv_clear<D>(spriv, k);
    __syncthreads();
    const bool use_s = k <= kBoundsMaxKS && !first;
    if (use_s) {
        // s_a: the minimum FP32 squared distance from c_a to every other centroid, the l range
        // split over tpc threads per centroid (float bits of non-negative values order like
        // integers: atomicMin), then half the distance's lower bound
        const int tpc = max(1, (int)blockDim.x / k);
        for (int a = threadIdx.x; a < k; a += blockDim.x) s_half[a] = INFINITY;
        __syncthreads();
        for (int x = threadIdx.x; x < k * tpc; x += blockDim.x) {
            const int a = x / tpc, part = x - a * tpc;
            float ca[D], mn = INFINITY;
#pragma unroll
            for (int m = 0; m < D; ++m) ca[m] = smem[m * kpad + a];
#pragma unroll 4
            for (int l = part; l < k; l += tpc) {
                float t = __fsub_rn(ca[0], smem[l]);
                float d2 = __fmul_rn(t, t);
#pragma unroll
                for (int m = 1; m < D; ++m) { t = __fsub_rn(ca[m], smem[m * kpad + l]); d2 = __fmaf_rn(t, t, d2); }
                mn = l == a ? mn : fminf(mn, d2);
            }
            atomicMin(reinterpret_cast<unsigned int*>(s_half) + a, __float_as_uint(mn));
        }
        __syncthreads();
        for (int a = threadIdx.x; a < k; a += blockDim.x) s_half[a] = 0.5f * lower_dist(s_half[a]);
        __syncthreads();
    }
    KM_BP(2);
    double sse = 0.0;
    unsigned long long chg = 0;
    unsigned long long nq_tot = 0;   // (every thread computes the same nq; thread 0 reports it)
    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    for (int64_t c0 = lo; c0 < hi; c0 += kBoundsChunk) {
        const int64_t c1 = min(hi, c0 + (int64_t)kBoundsChunk);
        // (1) the bound test of every point of the chunk (kBT per thread, all loads in flight at
        // once); the others join the queue
        constexpr int kBT = kBoundsChunk / kAssignThreads;
        Pt<D> p[kBT];
        int a[kBT];
        float lb[kBT];
        if (!first) {
#pragma unroll
            for (int r = 0; r < kBT; ++r) {
                const int64_t i = c0 + (int64_t)r * blockDim.x + threadIdx.x;
                const bool ok = i < c1;
#pragma unroll
                for (int m = 0; m < D; ++m) p[r].v[m] = ok ? pts[i * D + m] : 0.0f;
                a[r] = ok ? labels[i] : 0;
                lb[r] = ok ? lbv[i] : 0.0f;
            }
        }
        // the tests of the thread's kBT points first (independent chains), the queue after
        unsigned needm = 0u;
#pragma unroll
        for (int r = 0; r < kBT; ++r) {
            const int64_t i = c0 + (int64_t)r * blockDim.x + threadIdx.x;
            if (i < c1) {
                if (first) {
                    needm |= 1u << r;
                } else {
                    const double d64 = dist64n<D>(p[r], smem, kpad, a[r]);
                    const float lbp = __fsub_rd(lb[r], dmax);
                    const float bound = use_s ? fmaxf(lbp, s_half[a[r]]) : lbp;
                    // ||p - c_a|| < bound, squared: D64 (1 + 2^-40) bounds the true squared
                    // distance from above, RD(bound^2) the squared bound from below (no sqrt)
                    if (bound > 0.0f && __dmul_ru(d64, 1.0 + 0x1p-40) < (double)__fmul_rd(bound, bound)) {
                        sse += d64;
                        lbv[i] = lbp;
                    } else {
                        needm |= 1u << r;
                    }
                }
            }
        }
        // the warp's own queue, in point order (deterministic: the SSE_t partials then sum in
        // the same order every run)
#pragma unroll
        for (int r = 0; r < kBT; ++r) {
            const bool need = (needm >> r) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, need);
            if (need) sqw[wq + __popc(bal & ((1u << lane) - 1u))] = (int)(c0 + (int64_t)r * blockDim.x + threadIdx.x);
            wq += __popc(bal);
        }
        if (lane == 0) s_wq[wid] = wq;
        __syncthreads();
        // the warps' queues, concatenated in warp order
        int wbase = 0, nq = 0;
#pragma unroll
        for (int w = 0; w < kAssignThreads / 32; ++w) {
            wbase += w < wid ? s_wq[w] : 0;
            nq += s_wq[w];
        }
        for (int e = lane; e < wq; e += 32) sq2[wbase + e] = sqw[e];
        wq = 0;
        __syncthreads();
        KM_BP(3);
        // (2) the queued points, densely: rounds of P per thread, the remainder in one shorter round
        nq_tot += (unsigned long long)nq;
        const int64_t tile = (int64_t)blockDim.x * P;
        int64_t b = 0;
        for (; nq - b > tile / 2; b += tile)
            scan_round<D, P, false, 3>(b, nq, pts, smem, k, kpad, labels, first, q, nullptr, nullptr, spriv, sse,
                                       chg, sq2, lbv);
        if (P >= 4 && nq - b > tile / 4)
            scan_round<D, (P >= 2 ? P / 2 : 1), false, 3>(b, nq, pts, smem, k, kpad, labels, first, q, nullptr,
                                                          nullptr, spriv, sse, chg, sq2, lbv);
        else if (nq - b > 0)
            scan_round<D, (P >= 4 ? P / 4 : 1), false, 3>(b, nq, pts, smem, k, kpad, labels, first, q, nullptr,
                                                          nullptr, spriv, sse, chg, sq2, lbv);
        __syncthreads();
    }
    KM_BP(4);
    priv_flush<D>(spriv, k, io.d_cur, io.dn_cur);
    if (nscan && threadIdx.x == 0 && nq_tot) atomicAdd(nscan, nq_tot);
    block_sum2<kAssignThreads>(sse, chg);
    if (threadIdx.x == 0) { io.sse_cur[blockIdx.x] = sse; io.chg_cur[blockIdx.x] = chg; }
    KM_BP(5);
#undef KM_BP
}

// After the last launch (io.t = T, io.cout = C[]): converged earlier at launch t (done) -> the
// result C^t sits in buffer t % 2: copy buffer 1 to C[]; else the refine of iteration T-1 into
// C[] with its traces, the iteration count and the convergence flag.
template <int D>
__global__ void __launch_bounds__(kFinalizeThreads)
bounds_tail_kernel(const BoundsIO io, const float* __restrict__ buf1, int k, const Quant* __restrict__ quant)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (io.ctl->done) {
        if (io.ctl->iter & 1)
            for (int i = threadIdx.x; i < k * D; i += blockDim.x) io.cout[i] = buf1[i];
        return;
    }
    const Quant q = *quant;
    float dmax;
    bounds_refine<D, kFinalizeThreads>(io, q, k, k, nullptr, true, false, &dmax);
}

// Variant table (km_debug_set_variant): 1.. -> (bookkeeping, points/thread, min CTAs/SM)
struct ScanVariant {
    bool chunked;
    int P, minb;
};
constexpr int kNumScanVariants = 8;
__host__ __device__ inline ScanVariant scan_variant(int v)
{
    switch (v) {
        case 1: return {false, 4, 2};
        case 2: return {true, 4, 2};
        case 3: return {false, 4, 3};
        case 4: return {true, 4, 3};
        case 5: return {false, 2, 4};
        case 6: return {true, 2, 4};
        case 7: return {false, 8, 2};
        default: return {true, 8, 2};   // 8
    }
}

inline int assign_points_per_thread(int variant) { return variant == 0 ? 2 : scan_variant(variant).P; }
inline int assign_kpad(int variant, int k)
{
    if (variant >= 1 && scan_variant(variant).chunked) return ((k + kChunk - 1) / kChunk) * kChunk;
    return (k + 3) & ~3;
}

template <int D, int P, int MINB, bool CH>
int configure_scan(size_t smem, size_t priv, int* blocks_per_sm)
{
    cudaError_t e = cudaFuncSetAttribute(assign_scan_kernel<D, P, MINB, CH, 1>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncSetAttribute(assign_scan_kernel<D, P, MINB, CH, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return (int)e;
    if (priv) {
        e = cudaFuncSetAttribute(assign_scan_kernel<D, P, MINB, CH, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(smem + priv));
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(assign_scan_kernel<D, P, MINB, CH, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(smem + priv));
        if (e != cudaSuccess) return (int)e;
        return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, assign_scan_kernel<D, P, MINB, CH, 2>,
                                                                  kAssignThreads, smem + priv);
    }
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, assign_scan_kernel<D, P, MINB, CH, 1>,
                                                              kAssignThreads, smem);
}

template <int D>
int configure_assign_fast(int variant, size_t smem, size_t priv, int* blocks_per_sm)
{
    switch (variant) {
        case 1: return configure_scan<D, 4, 2, false>(smem, priv, blocks_per_sm);
        case 2: return configure_scan<D, 4, 2, true>(smem, priv, blocks_per_sm);
        case 3: return configure_scan<D, 4, 3, false>(smem, priv, blocks_per_sm);
        case 4: return configure_scan<D, 4, 3, true>(smem, priv, blocks_per_sm);
        case 5: return configure_scan<D, 2, 4, false>(smem, priv, blocks_per_sm);
        case 6: return configure_scan<D, 2, 4, true>(smem, priv, blocks_per_sm);
        case 7: return configure_scan<D, 8, 2, false>(smem, priv, blocks_per_sm);
        default: return configure_scan<D, 8, 2, true>(smem, priv, blocks_per_sm);
    }
}

#define KM_SCAN_LAUNCH(P_, MB_, CH_)                                                                           \
    assign_scan_kernel<D, P_, MB_, CH_, FUSE><<<grid, kAssignThreads, smem, s>>>(                              \
        pts, n, C, k, kpad, labels, first, sse_part, chg_part, acc_sum, acc_cnt, quant, ctl, tick, fin)

template <int D, int FUSE>
void launch_assign_fast(int variant, int grid, size_t smem, cudaStream_t s, const float* pts, int64_t n,
                        const float* C, int k, int kpad, int32_t* labels, int first, double* sse_part,
                        unsigned long long* chg_part, unsigned long long* acc_sum, unsigned int* acc_cnt,
                        const Quant* quant, const Ctl* ctl, unsigned int* tick, const FinArgs& fin)
{
    switch (variant) {
        case 1: KM_SCAN_LAUNCH(4, 2, false); break;
        case 2: KM_SCAN_LAUNCH(4, 2, true); break;
        case 3: KM_SCAN_LAUNCH(4, 3, false); break;
        case 4: KM_SCAN_LAUNCH(4, 3, true); break;
        case 5: KM_SCAN_LAUNCH(2, 4, false); break;
        case 6: KM_SCAN_LAUNCH(2, 4, true); break;
        case 7: KM_SCAN_LAUNCH(8, 2, false); break;
        default: KM_SCAN_LAUNCH(8, 2, true); break;
    }
}
#undef KM_SCAN_LAUNCH

}  // namespace km
