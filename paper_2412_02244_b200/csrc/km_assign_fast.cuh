// km_assign_fast.cuh -- K1 (fast): the assignment scan with packed FP32x2 math.
//
// Per point, the exact label is argmin_j of the FP64 direct-form distance (R1, R2;
// Lloyd's assignment).  The scan computes the FP32 direct-form distance
//     D32_j = fma(dz,dz, fma(dy,dy, dx*dx)),  dm = p_m + (-c_jm)   (RN everywhere)
// for two centroids at a time with FADD2/FMUL2/FFMA2, keeps per point the best
// group of 4 centroids (min m1, its group g1) and the second-best group minimum m2,
// and certifies the winner: |D32 - D64| <= 5.01u D64 (u = 2^-24), so every j with
// D32_j > thr(m1) = m1 (1 + 2^-19) is not the FP64 argmin.  If m2 > thr, the FP64
// argmin lies in group g1: rescan its 4 centroids (identical FP32 ops) and, when
// exactly one is within thr, that is the label; otherwise compare them in FP64.
// If m2 <= thr (a near-tie across groups) the point takes the exact FP64 scan.
// DESIGN.md "Exactness" has the argument, "K1" the roofline.
#pragma once
#include <cuda_runtime.h>
#include "km_kernels.cuh"

namespace km {

constexpr int kFastP = 4;   // points per thread

inline int assign_points_per_thread(int variant) { return variant == 0 ? 2 : kFastP; }

// FP64 distance against a NEGATED centroid (p + (-c) == p - c exactly).
template <int D>
__device__ __forceinline__ double dist64n(const float (&p)[D], const float* const (&nc)[D], int j)
{
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        double t = __dadd_rn((double)p[m], (double)nc[m][j]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

template <int D>
__device__ __noinline__ int exact_scan_n(const float (&p)[D], const float* const (&nc)[D], int j0, int j1)
{
    double best = INFINITY;
    int a = j0;
    for (int j = j0; j < j1; ++j) {
        double v = dist64n<D>(p, nc, j);
        if (v < best) { best = v; a = j; }
    }
    return a;
}

template <int D>
__device__ __forceinline__ float dist32n(const float (&p)[D], const float* const (&nc)[D], int j)
{
    float t = __fadd_rn(p[0], nc[0][j]);
    float s = __fmul_rn(t, t);
#pragma unroll
    for (int m = 1; m < D; ++m) {
        t = __fadd_rn(p[m], nc[m][j]);
        s = __fmaf_rn(t, t, s);
    }
    return s;
}

template <int D, int P, bool FUSE>
__global__ void __launch_bounds__(kAssignThreads, 2)
assign_fast_kernel(const float* __restrict__ pts, int64_t n, const float* __restrict__ C, int k, int kpad,
                   int32_t* __restrict__ labels, int first, double* __restrict__ sse_part,
                   unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                   unsigned int* __restrict__ acc_cnt, const Quant* __restrict__ quant, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    extern __shared__ __align__(16) float smem[];
    // stage NEGATED centroids, SoA, padded with -inf (p + -inf = -inf, squared = +inf: pads never win)
    for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) smem[m * kpad + j] = j < k ? -C[(int64_t)j * D + m] : -INFINITY;
    }
    __syncthreads();
    const float* nc[D];
#pragma unroll
    for (int m = 0; m < D; ++m) nc[m] = smem + m * kpad;
    const float4* nc4[D];
#pragma unroll
    for (int m = 0; m < D; ++m) nc4[m] = reinterpret_cast<const float4*>(nc[m]);
    const int ngroups = kpad >> 2;

    Quant q;
    if (FUSE) q = *quant;
    double sse = 0.0;
    unsigned long long chg = 0;
    const int64_t tile = (int64_t)blockDim.x * P;
    for (int64_t base = (int64_t)blockIdx.x * tile; base < n; base += (int64_t)gridDim.x * tile) {
        float p[P][D];
        float2 pp[P][D];
        float m1[P], m2[P];
        int g1[P];
#pragma unroll
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                p[r][m] = i < n ? pts[i * D + m] : 0.0f;
                pp[r][m] = make_float2(p[r][m], p[r][m]);
            }
            m1[r] = INFINITY; m2[r] = INFINITY; g1[r] = 0;
        }
#pragma unroll 2
        for (int g = 0; g < ngroups; ++g) {
            float4 c[D];
#pragma unroll
            for (int m = 0; m < D; ++m) c[m] = nc4[m][g];
#pragma unroll
            for (int r = 0; r < P; ++r) {
                float2 t0 = __fadd2_rn(pp[r][0], make_float2(c[0].x, c[0].y));
                float2 t1 = __fadd2_rn(pp[r][0], make_float2(c[0].z, c[0].w));
                float2 s0 = __fmul2_rn(t0, t0);
                float2 s1 = __fmul2_rn(t1, t1);
#pragma unroll
                for (int m = 1; m < D; ++m) {
                    t0 = __fadd2_rn(pp[r][m], make_float2(c[m].x, c[m].y));
                    t1 = __fadd2_rn(pp[r][m], make_float2(c[m].z, c[m].w));
                    s0 = __ffma2_rn(t0, t0, s0);
                    s1 = __ffma2_rn(t1, t1, s1);
                }
                float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
                bool lt = v < m1[r];
                m2[r] = fmaxf(m1[r], fminf(m2[r], v));   // second smallest of {m1, m2, v}
                m1[r] = fminf(m1[r], v);
                g1[r] = lt ? g : g1[r];
            }
        }
#pragma unroll
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
            if (i >= n) continue;
            const float thr = certify_thr(m1[r]);
            int a;
            if (!(m2[r] > thr)) {
                a = exact_scan_n<D>(p[r], nc, 0, k);
            } else {
                const int j0 = g1[r] * 4;
                int cnt = 0;
                a = j0;
#pragma unroll
                for (int u = 3; u >= 0; --u) {
                    if (dist32n<D>(p[r], nc, j0 + u) <= thr) { ++cnt; a = j0 + u; }
                }
                if (cnt != 1) a = exact_scan_n<D>(p[r], nc, j0, min(j0 + 4, k));
            }
            sse += dist64n<D>(p[r], nc, a);
            if (first) chg += 1;
            else chg += (labels[i] != a);
            labels[i] = a;
            if (FUSE) accumulate_point<D>(p[r], a, q, acc_sum, acc_cnt);
        }
    }
    block_sum2<kAssignThreads>(sse, chg);
    if (threadIdx.x == 0) { sse_part[blockIdx.x] = sse; chg_part[blockIdx.x] = chg; }
}

template <int D>
int configure_assign_fast(size_t smem, int* blocks_per_sm)
{
    cudaError_t e;
    e = cudaFuncSetAttribute(assign_fast_kernel<D, kFastP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = cudaFuncSetAttribute(assign_fast_kernel<D, kFastP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, assign_fast_kernel<D, kFastP, true>,
                                                      kAssignThreads, smem);
    return (int)e;
}

template <int D, bool FUSE>
void launch_assign_fast(int grid, size_t smem, cudaStream_t s, const float* pts, int64_t n, const float* C, int k,
                        int kpad, int32_t* labels, int first, double* sse_part, unsigned long long* chg_part,
                        unsigned long long* acc_sum, unsigned int* acc_cnt, const Quant* quant, const Ctl* ctl)
{
    assign_fast_kernel<D, kFastP, FUSE><<<grid, kAssignThreads, smem, s>>>(
        pts, n, C, k, kpad, labels, first, sse_part, chg_part, acc_sum, acc_cnt, quant, ctl);
}

}  // namespace km
