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

// FUSE: 0 labels only (km_assign), 1 fused update with per-point global REDs, 2 fused update
// privatised in shared memory (accumulate_point_priv; the default when k(2d+1)*4 B fits).
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
    if (FUSE == 2) priv_clear<D>(spriv, k);
    __syncthreads();
    const float4* nc4 = reinterpret_cast<const float4*>(smem);
    const int kq = kpad >> 2;   // float4 groups per coordinate
    const int ngroups = kq;

    Quant q;
    if (FUSE) q = *quant;
    double sse = 0.0;
    unsigned long long chg = 0;
    const int64_t tile = (int64_t)blockDim.x * P;
    for (int64_t base = (int64_t)blockIdx.x * tile; base < n; base += (int64_t)gridDim.x * tile) {
        Pt<D> p[P];
        float m1[P], m2[P];
        int b1[P];
#pragma unroll
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
#pragma unroll
            for (int m = 0; m < D; ++m) p[r].v[m] = i < n ? pts[i * D + m] : 0.0f;
            m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0;
        }
        if (CHUNKED) {
            constexpr int GPC = kChunk / 4;   // float4 groups per chunk
            const int nchunks = ngroups / GPC;
            for (int ch = 0; ch < nchunks; ++ch) {
                float mc[P];
#pragma unroll
                for (int r = 0; r < P; ++r) mc[r] = INFINITY;
#pragma unroll
                for (int gg = 0; gg < GPC; ++gg) {
                    const int g = ch * GPC + gg;
                    float4 c[D];
#pragma unroll
                    for (int m = 0; m < D; ++m) c[m] = nc4[m * kq + g];
#pragma unroll
                    for (int r = 0; r < P; ++r) {
                        float2 s0 = pair2<D>(p[r], c, false);
                        float2 s1 = pair2<D>(p[r], c, true);
                        mc[r] = fminf(fminf(mc[r], s0.x), s0.y);
                        mc[r] = fminf(fminf(mc[r], s1.x), s1.y);
                    }
                }
#pragma unroll
                for (int r = 0; r < P; ++r) {
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
                for (int r = 0; r < P; ++r) {
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
        for (int r = 0; r < P; ++r) {
            int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
            if (i >= n) continue;
            const int a = certify_label<D, CHUNKED ? kChunk : 4>(p[r], m1[r], m2[r], b1[r], smem, kpad, k);
            sse += dist64n<D>(p[r], smem, kpad, a);
            if (first) chg += 1;
            else chg += (labels[i] != a);
            labels[i] = a;
            if (FUSE == 1) accumulate_point<D>(p[r].v, a, q, acc_sum, acc_cnt);
            if (FUSE == 2) accumulate_point_priv<D>(p[r].v, a, q, spriv, k);
        }
    }
    if (FUSE == 2) {
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
