// km_small.cuh -- the whole Lloyd run for small problems in ONE launch of ONE thread-block
// cluster (8 CTAs on 8 SMs, distributed shared memory).
//
// For n up to a few 10^4 points (config 1: n = 10^4, d = 2, k = 10) an iteration is ~10^5
// pairs: a multi-kernel schedule is launch- and latency-bound (each launch, grid-wide ticket
// and reduction costs microseconds).  Here one cluster runs the whole loop; CTA r owns the
// points [r n / 8, (r+1) n / 8), holds them and their labels in shared memory for the whole run
// (one global read, one write of the labels at the end), and keeps its own copy of the
// centroids, their negated SoA form and its privatised fixed-point RUNNING sums in shared
// memory.  Per iteration:
//   assign its points (the packed FP32 scan of K1 + FP64 certification: exact labels),
//     SSE_t and changed_t partials; a point whose label changed moves its value between the
//     running sums sv(j), |S_j| (at t = 0 every point adds);
//   cluster barrier;
//   CTA r refines the centroids j = r (mod 8): it adds the 8 CTAs' sums of j through DSMEM
//     (exact integers), c_j = RN_f32(sv(j)/|S_j|) (Alg. 1 line 12) and stores c_j
//     into all 8 copies; partial max drift;
//   cluster barrier; every CTA reads the 8 partials in rank order, so all take the same
//     convergence decision; CTA 0 writes the traces.
// Before the loop: the bounding box over the cluster -> the fixed-point scale (make_quant).
// After it: Eq. 1 of the returned pair as the 128-bit fixed-point sum (sse_kernel's rounding).
// The arithmetic is the multi-kernel brute-force path's, so labels, centroids, changed_t, drift
// and out_sse are identical to it bit for bit (SSE_t up to FP64 summation order).
#pragma once
#include <cooperative_groups.h>
#include "km_kernels.cuh"
#include "km_assign_fast.cuh"

namespace km {

constexpr int kSmallCtas = 8;         // portable cluster size
constexpr int kSmallThreads = 512;
constexpr int kSmallMaxN = 1 << 16;   // km_api.cu uses this kernel for n <= kSmallMaxN, k <= kSmallMaxK
constexpr int kSmallMaxK = 1024;

template <int D>
__host__ __device__ constexpr int small_cap(int64_t n) { return (int)((n + kSmallCtas - 1) / kSmallCtas); }
template <int D>
__host__ __device__ constexpr size_t small_smem(int k, int kpad, int64_t n)
{
    return (size_t)D * kpad * 4 + (size_t)k * D * 4 + priv_bytes<D>(k) + (size_t)small_cap<D>(n) * (D + 1) * 4;
}

// Everything one run reads and writes (the kernel is the whole device work of a km_run_ctx call:
// no memset or copy nodes around it).
struct SmallIO {
    const float* cin;          // initial centroids [k][D]
    float* cout;               // final centroids (the context's working copy)
    float* cout2;              // nullable: the caller's device output as well
    double* sse_trace;         // [max_iter] (entries past the executed iterations: NaN / -1)
    long long* chg_trace;
    double* drift_trace;
    double* sse_user;          // nullable: the caller's device traces
    long long* chg_user;
    Ctl* ctl;
    SseFix* sse_out;
    double* host_sse;          // nullable: mapped pinned host record (Eq. 1, iterations)
    Ctl* host_ctl;
};

template <int D>
__global__ void __cluster_dims__(kSmallCtas, 1, 1) __launch_bounds__(kSmallThreads, 1)
lloyd_small_kernel(const float* __restrict__ pts, int n, int k, int kpad, int32_t* __restrict__ labels,
                   int max_iter, float tol, Quant* __restrict__ quant_out, const SmallIO io)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    extern __shared__ __align__(16) float ssm[];
    float* nc = ssm;                                   // [D][kpad] negated centroids (-inf padding)
    float* Cs = ssm + D * kpad;                        // [k][D] this CTA's copy of the centroids
    unsigned int* sp = reinterpret_cast<unsigned int*>(Cs + k * D);   // privatised running sums and counts
    float* ps = reinterpret_cast<float*>(sp + (size_t)k * (2 * D + 1));   // [cap][D] this CTA's points
    int* pl = reinterpret_cast<int*>(ps + (size_t)small_cap<D>(n) * D);  // [cap] their labels
    __shared__ float s_box[2 * D][32];
    __shared__ float s_cbox[2 * D];                    // this CTA's points' box (read by the cluster)
    __shared__ double s_sse[2], s_md[2];               // per-iteration partials, double-buffered by parity
    __shared__ unsigned long long s_chg[2];
    __shared__ double s_w[32];
    __shared__ double s_dec[2];                        // this iteration's SSE_t and max drift
    __shared__ unsigned long long s_decc;              // and changed_t
    __shared__ unsigned long long s_fix[2];            // this CTA's 128-bit Eq. 1 partial
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int NW = kSmallThreads / 32;
    const int i0 = (int)((long long)n * rank / kSmallCtas), i1 = (int)((long long)n * (rank + 1) / kSmallCtas);

    // ---- bounding box of the cluster's points -> the fixed-point scale (as quant_kernel)
    float lo[D], hi[D];
#pragma unroll
    for (int m = 0; m < D; ++m) { lo[m] = INFINITY; hi[m] = -INFINITY; }
    for (int i = i0 + tid; i < i1; i += kSmallThreads)
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const float v = pts[(int64_t)i * D + m];
            ps[(i - i0) * D + m] = v;
            lo[m] = fminf(lo[m], v);
            hi[m] = fmaxf(hi[m], v);
        }
    priv_clear<D>(sp, k);
#pragma unroll
    for (int m = 0; m < D; ++m) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[m] = fminf(lo[m], __shfl_xor_sync(0xffffffffu, lo[m], o));
            hi[m] = fmaxf(hi[m], __shfl_xor_sync(0xffffffffu, hi[m], o));
        }
        if (lane == 0) { s_box[m][w] = lo[m]; s_box[D + m][w] = hi[m]; }
    }
    for (int j = tid; j < k * D; j += kSmallThreads) Cs[j] = io.cin[j];
    __syncthreads();
    if (tid < D) {
        float a = INFINITY, z = -INFINITY;
        for (int ww = 0; ww < NW; ++ww) { a = fminf(a, s_box[tid][ww]); z = fmaxf(z, s_box[D + tid][ww]); }
        s_cbox[tid] = a;
        s_cbox[D + tid] = z;
    }
    cluster.sync();
#pragma unroll
    for (int m = 0; m < D; ++m) {
        lo[m] = INFINITY;
        hi[m] = -INFINITY;
        for (int q2 = 0; q2 < kSmallCtas; ++q2) {
            const float* rb = cluster.map_shared_rank(s_cbox, q2);
            lo[m] = fminf(lo[m], rb[m]);
            hi[m] = fmaxf(hi[m], rb[D + m]);
        }
    }
    Quant q;
    make_quant(q, lo, hi, D, n);
    if (rank == 0 && tid == 0) *quant_out = q;

    int t = 0, conv = 0;
    for (; t < max_iter; ++t) {
        const int par = t & 1;
        // ---- stage the negated SoA centroids
        for (int j = tid; j < kpad; j += kSmallThreads)
#pragma unroll
            for (int m = 0; m < D; ++m) nc[m * kpad + j] = j < k ? -Cs[j * D + m] : -INFINITY;
        __syncthreads();
        // ---- assignment + SSE_t + changed_t + sums (as assign_scan_kernel, one point at a time)
        const float4* nc4 = reinterpret_cast<const float4*>(nc);
        const int kq = kpad >> 2;
        double sse = 0.0;
        unsigned long long chg = 0;
        for (int i = tid; i < i1 - i0; i += kSmallThreads) {
            Pt<D> p;
#pragma unroll
            for (int m = 0; m < D; ++m) p.v[m] = ps[i * D + m];
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
            const int old = t == 0 ? -1 : pl[i];
            if (old != a) {   // (incremental: only moved points touch the running sums)
                ++chg;
                pl[i] = a;
                move_point_priv<D>(p.v, old, a, q, sp, k);
            }
        }
        block_sum2<kSmallThreads>(sse, chg);
        if (tid == 0) { s_sse[par] = sse; s_chg[par] = chg; }
        cluster.sync();   // every CTA's sums and partials are complete
        // ---- refine the centroids j = rank (mod 8) from the 8 CTAs' sums; store into every copy
        double md = 0.0;
        for (int j = rank + kSmallCtas * tid; j < k; j += kSmallCtas * kSmallThreads) {
            unsigned int cnt = 0;
            unsigned long long sv[D];
#pragma unroll
            for (int m = 0; m < D; ++m) sv[m] = 0ull;
            for (int q2 = 0; q2 < kSmallCtas; ++q2) {
                const unsigned int* rp = cluster.map_shared_rank(sp, q2);
                cnt += rp[2 * k * D + j];
#pragma unroll
                for (int m = 0; m < D; ++m)
                    sv[m] += ((unsigned long long)rp[k * D + j * D + m] << 32) | rp[j * D + m];
            }
            double dd = 0.0;
            float nw[D];
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const float old = Cs[j * D + m];
                nw[m] = old;
                if (cnt > 0) {
                    const double mean = __dadd_rn(q.o[m], __dmul_rn(__ddiv_rn((double)sv[m], (double)cnt), q.inv[m]));
                    nw[m] = __double2float_rn(mean);
                }
                const double tt = __dsub_rn((double)nw[m], (double)old);
                dd = __dadd_rn(dd, __dmul_rn(tt, tt));
            }
            for (int q2 = 0; q2 < kSmallCtas; ++q2) {
                float* rc = cluster.map_shared_rank(Cs, q2);
#pragma unroll
                for (int m = 0; m < D; ++m) rc[j * D + m] = nw[m];
            }
            md = fmax(md, sqrt(dd));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
        if (lane == 0) s_w[w] = md;
        __syncthreads();
        if (tid == 0) {
            for (int ww = 1; ww < NW; ++ww) md = fmax(md, s_w[ww]);
            s_md[par] = md;
        }
        cluster.sync();   // every copy of the centroids and every partial is final
        // ---- the same decision in every CTA: the 8 partials in rank order (lanes 0..7 of warp 0
        // read them through DSMEM at once; lane 0 adds them in rank order; shared with the CTA)
        if (w == 0) {
            double a = 0.0, mdq = 0.0;
            unsigned long long c2 = 0;
            if (lane < kSmallCtas) {
                a = *cluster.map_shared_rank(&s_sse[par], lane);
                c2 = *cluster.map_shared_rank(&s_chg[par], lane);
                mdq = *cluster.map_shared_rank(&s_md[par], lane);
            }
            double st = 0.0, mt = 0.0;
            unsigned long long ct = 0;
            for (int q2 = 0; q2 < kSmallCtas; ++q2) {
                st += __shfl_sync(0xffffffffu, a, q2);
                ct += __shfl_sync(0xffffffffu, c2, q2);
                mt = fmax(mt, __shfl_sync(0xffffffffu, mdq, q2));
            }
            if (lane == 0) { s_dec[0] = st; s_dec[1] = mt; s_decc = ct; }
        }
        __syncthreads();
        const double sse_t = s_dec[0], md_t = s_dec[1];
        const unsigned long long chg_t = s_decc;
        if (rank == 0 && tid == 0) {
            io.sse_trace[t] = sse_t;
            io.chg_trace[t] = (long long)chg_t;
            io.drift_trace[t] = md_t;
            if (io.sse_user) io.sse_user[t] = sse_t;
            if (io.chg_user) io.chg_user[t] = (long long)chg_t;
        }
        if (tol >= 0.0f && (md_t <= (double)tol || (t >= 1 && chg_t == 0))) { ++t; conv = 1; break; }
    }
    const int iters = t;
    // labels back to global memory (input order); traces past the executed iterations
    for (int i = tid; i < i1 - i0; i += kSmallThreads) labels[i0 + i] = pl[i];
    if (rank == 0)
        for (int u = iters + tid; u < max_iter; u += kSmallThreads) {
            io.sse_trace[u] = __longlong_as_double(-1ll);   // all bits set: NaN
            io.chg_trace[u] = -1ll;
            io.drift_trace[u] = __longlong_as_double(-1ll);
            if (io.sse_user) io.sse_user[u] = __longlong_as_double(-1ll);
            if (io.chg_user) io.chg_user[u] = -1ll;
        }
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
    for (int i = tid; i < i1 - i0; i += kSmallThreads) {
        const int a = pl[i];
        double v = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double tt = __dsub_rn((double)ps[i * D + m], (double)Cs[a * D + m]);
            v = __dadd_rn(v, __dmul_rn(tt, tt));
        }
        add_fix(acc, v, scale);
    }
    acc = block_sum128(acc);
    if (tid == 0) { s_fix[0] = (unsigned long long)acc; s_fix[1] = (unsigned long long)(acc >> 64); }
    if (rank == 0)
        for (int j = tid; j < k * D; j += kSmallThreads) {
            io.cout[j] = Cs[j];
            if (io.cout2) io.cout2[j] = Cs[j];
        }
    cluster.sync();
    if (rank == 0 && tid == 0) {
        u128 tot = 0;
        for (int q2 = 0; q2 < kSmallCtas; ++q2) {
            const unsigned long long* rf = cluster.map_shared_rank(s_fix, q2);
            tot += ((u128)rf[1] << 64) | rf[0];
        }
        const double inv = ldexp(1.0, -s3);
        const double hv = (double)(unsigned long long)(tot >> 64), lv = (double)(unsigned long long)tot;
        const double sv = __dmul_rn(__dadd_rn(__dmul_rn(hv, 0x1p64), lv), inv);
        io.sse_out->value = sv;
        io.sse_out->inv = inv;
        const unsigned long long m48 = (1ull << 48) - 1;
        io.sse_out->limb[0] = (unsigned long long)tot & m48;
        io.sse_out->limb[1] = (unsigned long long)(tot >> 48) & m48;
        io.sse_out->limb[2] = (unsigned long long)(tot >> 96);
        io.ctl->iter = iters;
        io.ctl->done = conv;
        if (io.host_sse) {   // mapped pinned host record: no copy nodes after the kernel
            *reinterpret_cast<volatile double*>(io.host_sse) = sv;
            reinterpret_cast<volatile Ctl*>(io.host_ctl)->iter = iters;
            reinterpret_cast<volatile Ctl*>(io.host_ctl)->done = conv;
        }
    }
    cluster.sync();   // no CTA exits while rank 0 still reads its shared memory
}

}  // namespace km
