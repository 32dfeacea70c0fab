// km_hd.cuh -- the high-dimensional variant (the paper's check on embedded
// trajectories, d = 128 / 256, Table tab:high_dimension): the same exact Lloyd
// step, with the assignment as a dense contraction on the 5th-generation tensor cores.
//
// For a point p and centroids c_j (both centred on the bounding-box midpoint o, p' = p - o,
// c' = c - o, FP32) the nearest centroid maximises
//       v_j = p'.c'_j - ||c'_j||^2 / 2            (||p' - c'_j||^2 = ||p'||^2 - 2 v_j).
// hd_gemm_kernel computes p'.c'_j for a 128-point tile against all k centroids on the tensor
// cores in split form (TF32 hi.hi with tcgen05.mma kind::tf32 + the BF16 corrections lo.hi and
// hi.lo with kind::f16; operands TMA-staged in swizzled shared memory, 128 x 128 accumulators in
// four TMEM buffers (all 512 columns); the TMA and MMA warps converged with one elect.sync lane
// issuing) and
// keeps, per point and column half, the 4 (k <= 2048) or 8 largest v_j (ascending j on ties),
// dropping at once every score below max(v_last, v1 - 2E).  The scores carry a bound E_i
// (DESIGN.md 12): hd_certify_kernel accepts the top label when v1 - v2 > 2 E_i, otherwise
// decides among the in-band candidates (v_j >= v1 - 2 E_i, all among the kept ones) with the
// oracle's FP64 direct-form distance on the ORIGINAL coordinates, otherwise sends the point to
// the FP64 fallback over all k (hd_fb_slice / hd_fb_settle, hd_fallback_kernel).  Labels are
// therefore exactly the FP64 argmin (lowest index on ties), as in the low-dimensional path.
// The update keeps running 64-bit fixed-point sums sv(j) and moment sums Q_j:
// only points whose label changed move; SSE_t comes from the moments in hd_finalize_kernel.
#pragma once
#include "km_kernels.cuh"
#include <cuda.h>
#include <cuda_bf16.h>

namespace km {
namespace hd {

constexpr int kBM = 128;   // points per tile (UMMA M, TMEM lanes)
constexpr int kBN = 128;   // centroids per accumulator (UMMA N, TMEM columns)
constexpr int kBK = 32;    // K chunk: 32 FP32 = one 128-B swizzle row
constexpr int kTopMax = 8;          // scores kept per point and column half (TOP = 4 or 8; value desc., lower j first)
#ifndef KM_HD_ACC
#define KM_HD_ACC 4
#endif
constexpr int kAccN = KM_HD_ACC;    // TMEM accumulator buffers of kBN columns (2: 256 columns, 4: all 512)
constexpr int kEpiWarps = 8;        // two per TMEM lane quadrant, each scanning half the columns
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;   // warp 0 TMA, warp 1 MMA + TMEM owner, 2.. epilogue
// instruction descriptors: D = F32 (bits 4-5), A = B = TF32 (2) or BF16 (1) (bits 7-9, 10-12),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);
constexpr uint32_t kIdescBf = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                              ((uint32_t)(kBM >> 4) << 24);

// Split products: x = x_hi + x_lo with x_hi = x rounded to TF32 (exact as a TF32 operand) and
// x_lo = x - x_hi (exact in FP32, |x_lo| <= 2^-11 |x|).  p.c ~ p_hi.c_hi (kind::tf32, K = 8)
// + bf16(p_lo).bf16(c_hi) + bf16(p_hi).bf16(c_lo) (kind::f16 with BF16 operands, K = 16, twice
// the TF32 rate), all into one FP32 accumulator (DESIGN.md 12 bounds the error).  Per 32-wide K
// chunk a tile holds the TF32 hi part (16 KB, 128-B swizzle) and the BF16 hi and lo parts (8 KB
// each, 64-B swizzle).  The point tile stays resident in shared memory (D <= 128; at D = 256 its
// BF16 parts stream with the centroid chunks).
template <int D>
struct GemmCfg {
    static constexpr int KC = D / kBK;
    static constexpr bool kALoRes = D <= 128;
    static constexpr int kAChunk = kBM * kBK * 4;    // 16 KB: TF32 hi
    static constexpr int kAHalf = kBM * kBK * 2;     // 8 KB: one BF16 part
    static constexpr int kBChunk = kBN * kBK * 4;    // 16 KB
    static constexpr int kBHalf = kBN * kBK * 2;     // 8 KB
    static constexpr int kABytes = KC * (kAChunk + (kALoRes ? 2 * kAHalf : 0));
    static constexpr int kStageBytes = kBChunk + 2 * kBHalf + (kALoRes ? 0 : 2 * kAHalf);
    static constexpr int kFixed = 1024 + kABytes + 256;
    static constexpr int kFit = (232448 - kFixed) / kStageBytes;
    static constexpr int kStages = kFit > 4 ? 4 : kFit;
    static constexpr int kSmem = kFixed + kStages * kStageBytes;
    static_assert(kStages >= 2, "shared memory");
};

struct HdState {
    double sse_scale, sse_inv;   // SSE_t summands in fixed point (as the low-d path)
    unsigned long long sse_q;    // SSE_t of the iteration (fixed point)
    unsigned long long chg;      // changed_t
    unsigned long long md_bits;  // max drift of the iteration (FP64 bits; non-negative)
    unsigned int cmax_bits;      // max_j ||c'_j|| rounded up (FP32 bits)
    int nfb;                     // points sent to the FP64 fallback this iteration
    unsigned long long n_cert, n_band, n_full;   // cumulative decision counts (diagnostics)
};

// ---------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "HD_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra HD_WAIT_%=;\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// Elected-lane forms for a converged warp (no per-instruction divergence loops in SASS)
__device__ __forceinline__ void bar_expect_elect(uint64_t* b, uint32_t bytes)
{
    asm volatile(
        "{\n .reg .pred pe;\n elect.sync _|pe, 0xffffffff;\n"
        "@pe mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(su32(b)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void tma_2d_elect(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* b)
{
    asm volatile(
        "{\n .reg .pred pe;\n elect.sync _|pe, 0xffffffff;\n"
        "@pe cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n}\n" ::
            "r"(su32(dst)),
        "l"((uint64_t)tm), "r"(x), "r"(y), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int x, int y, uint64_t* b)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(su32(dst)),
        "l"((uint64_t)tm), "r"(x), "r"(y), "r"(su32(b))
        : "memory");
}
// UMMA shared-memory descriptor: K-major operand, 128-B swizzle, 8-row groups 1024 B apart
// (SBO), version 1 (sm_100).  Advancing K by 8 TF32 inside the swizzle atom adds 32 B to the
// start address.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO
    d |= (uint64_t)1 << 46;              // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}
// The same for BF16 K-major operands with 64-B rows (32 BF16): 64-B swizzle, 8-row groups 512 B
// apart; K advances by 16 BF16 = 32 B.
__device__ __forceinline__ uint64_t sdesc64(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;              // SWIZZLE_64B
    return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
// One 32-wide K chunk: 4 TF32 MMAs (hi.hi, K = 8) + 2 x 2 BF16 MMAs (lo.hi, hi.lo, K = 16) in one
// statement (one issue sequence instead of eight); K steps add 2 (32 B) to the descriptors.
__device__ __forceinline__ void mma_chunk(uint32_t dtmem, uint64_t dah, uint64_t dbh, uint64_t dabl, uint64_t dabh,
                                          uint64_t dbbh, uint64_t dbbl, uint32_t acc)
{
    asm volatile(
        "{\n"
        ".reg .pred pa, pt, pe;\n"
        ".reg .b64 x1, y1, x2, y2, x3, y3;\n"
        "elect.sync _|pe, 0xffffffff;\n"   // the whole warp arrives; one lane issues
        "setp.ne.b32 pa, %7, 0;\n"
        "setp.eq.b32 pt, 0, 0;\n"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %8, pa;\n"
        "add.u64 x1, %1, 2;\n add.u64 y1, %2, 2;\n"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], x1, y1, %8, pt;\n"
        "add.u64 x2, %1, 4;\n add.u64 y2, %2, 4;\n"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], x2, y2, %8, pt;\n"
        "add.u64 x3, %1, 6;\n add.u64 y3, %2, 6;\n"
        "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], x3, y3, %8, pt;\n"
        "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %5, %9, pt;\n"
        "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %6, %9, pt;\n"
        "add.u64 x1, %3, 2;\n add.u64 y1, %5, 2;\n"
        "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], x1, y1, %9, pt;\n"
        "add.u64 x2, %4, 2;\n add.u64 y2, %6, 2;\n"
        "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], x2, y2, %9, pt;\n"
        "}\n" ::"r"(dtmem),
        "l"(dah), "l"(dbh), "l"(dabl), "l"(dabh), "l"(dbbh), "l"(dbbl), "r"(acc), "r"(kIdesc), "r"(kIdescBf)
        : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(dtmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* b)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}
// tcgen05.commit by one elected lane of a converged warp
__device__ __forceinline__ void mma_commit_elect(uint64_t* b)
{
    asm volatile(
        "{\n"
        ".reg .pred pe;\n"
        "elect.sync _|pe, 0xffffffff;\n"
        "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
        "}\n" ::"r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// 32 lanes x 32 columns of 32-bit accumulators -> 32 registers per thread (row = lane)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");   // the load and its wait in one statement: no use of r[] can move above the wait
}

// 32 lanes x 64 columns -> 64 registers per thread, and the wait, in one statement
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr)
        : "memory");
}

// ------------------------------------------------------------------------- index build
// Per-CTA bounding-box partials [grid][2d] (lo, hi) of the [n][d] points (d | 256).
__global__ void __launch_bounds__(256)
hd_bbox_kernel(const float* __restrict__ P, int64_t n, int d, float* __restrict__ part)
{
    __shared__ float s_lo[256], s_hi[256];
    const int m = threadIdx.x % d, r0 = threadIdx.x / d, rs = 256 / d;
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * rs + r0; i < n; i += (int64_t)gridDim.x * rs) {
        const float v = P[i * d + m];
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    s_lo[threadIdx.x] = lo;
    s_hi[threadIdx.x] = hi;
    __syncthreads();
    if (threadIdx.x < d) {
        for (int t = threadIdx.x + d; t < 256; t += d) { lo = fminf(lo, s_lo[t]); hi = fmaxf(hi, s_hi[t]); }
        part[(int64_t)blockIdx.x * 2 * d + threadIdx.x] = lo;
        part[(int64_t)blockIdx.x * 2 * d + d + threadIdx.x] = hi;
    }
}

// One CTA: the box, the per-dimension fixed point of the sums (origin lo_m, scale 2^s_m with
// n * extent_m * 2^s_m < 2^61: the low-d rule of DESIGN.md 5), the centring origin o_m (FP32
// midpoint) and the SSE_t fixed-point scale (n * sum_m extent_m^2 * 2^s2 < 2^62).
__global__ void __launch_bounds__(1024)
hd_quant_kernel(const float* __restrict__ part, int nparts, int64_t n, int d, double* __restrict__ qo,
                double* __restrict__ qs, double* __restrict__ qi, float* __restrict__ ctr,
                HdState* __restrict__ st)
{
    // thread t: dimension t % d over the partials t / d, t / d + G, ... (G = 1024 / d groups)
    __shared__ float s_lo[1024], s_hi[1024];
    __shared__ double s_e2[256];
    const int m0 = threadIdx.x % d, g = threadIdx.x / d, G = 1024 / d;
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll 4
    for (int b = g; b < nparts; b += G) {
        lo = fminf(lo, part[(int64_t)b * 2 * d + m0]);
        hi = fmaxf(hi, part[(int64_t)b * 2 * d + d + m0]);
    }
    s_lo[threadIdx.x] = lo;
    s_hi[threadIdx.x] = hi;
    __syncthreads();
    int nb = 0;
    while (nb < 63 && (n >> nb) != 0) ++nb;
    double e2 = 0.0;
    if (threadIdx.x < d) {
        const int m = threadIdx.x;
        for (int q = 1; q < G; ++q) { lo = fminf(lo, s_lo[q * d + m]); hi = fmaxf(hi, s_hi[q * d + m]); }
        const double ext = (double)hi - (double)lo;
        int e = 0;
        if (ext > 0.0) frexp(ext, &e);
        const int s = ext > 0.0 ? 61 - nb - e : 0;
        qo[m] = (double)lo;
        qs[m] = ldexp(1.0, s);
        qi[m] = ldexp(1.0, -s);
        ctr[m] = __double2float_rn(0.5 * ((double)lo + (double)hi));
        e2 = ext * ext;
    }
    if (threadIdx.x < 256) s_e2[threadIdx.x] = e2;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 256; ++i) t += s_e2[i];   // m = 0 .. d-1 in order (host: hd_host_quant)
        const double tot = (double)n * t * (1.0 + 0x1p-20);
        int e = 0;
        if (tot > 0.0) frexp(tot, &e);
        const int s2 = tot > 0.0 ? 62 - e : 0;
        st->sse_scale = ldexp(1.0, s2);
        st->sse_inv = ldexp(1.0, -s2);
    }
}

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// x_hi = x rounded to TF32 (nearest, ties away; low 13 bits zero), x_lo = x - x_hi (exact).
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo)
{
    uint32_t u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    hi = __uint_as_float(u);
    lo = __fsub_rn(x, hi);
}

// Centred copy p' = fl(p - o) split into TF32 hi / lo parts (the A operands) and an upper
// bound of ||p'|| per point.
template <int D>
__global__ void __launch_bounds__(256)
hd_center_kernel(const float* __restrict__ P, int64_t n, const float* __restrict__ ctr, float* __restrict__ Pc,
                 __nv_bfloat16* __restrict__ Pbh, __nv_bfloat16* __restrict__ Pbl, float* __restrict__ pn,
                 const double* __restrict__ qo, const HdState* __restrict__ st, unsigned long long* __restrict__ pq2)
{
    const double ss = st->sse_scale;
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float o[D / 32];
#pragma unroll
    for (int u = 0; u < D / 32; ++u) o[u] = ctr[lane + 32 * u];
    for (int64_t i = w0; i < n; i += nw) {
        double s = 0.0, s2 = 0.0;
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const float pm = P[i * D + lane + 32 * u];
            const double e = (double)pm - qo[lane + 32 * u];   // from the fixed-point origin (exact)
            s2 = fma(e, e, s2);
            const float v = __fsub_rn(pm, o[u]);
            float hi, lo;
            split_tf32(v, hi, lo);
            Pc[i * D + lane + 32 * u] = hi;
            Pbh[i * D + lane + 32 * u] = __float2bfloat16_rn(hi);
            Pbl[i * D + lane + 32 * u] = __float2bfloat16_rn(lo);
            s = fma((double)v, (double)v, s);
        }
        s = warp_sum_d(s);
        s2 = warp_sum_d(s2);
        if (lane == 0) {
            pn[i] = __double2float_ru(__dsqrt_ru(s * (1.0 + 0x1p-40)));
            pq2[i] = sse_q(s2, ss);   // ||p - o_q||^2 in the SSE fixed point: the moment sums Q_j
        }
    }
}

// Per iteration: centred centroids c' = fl(c - o) (the B operand), h_j = -||c'_j||^2 / 2
// (FP32; -inf for the padding j >= k, which then never wins) and max_j ||c'_j|| (rounded up).
template <int D>
__global__ void __launch_bounds__(256)
hd_prep_kernel(const float* __restrict__ C, int k, int kpad, const float* __restrict__ ctr, float* __restrict__ Cc,
               __nv_bfloat16* __restrict__ Cbh, __nv_bfloat16* __restrict__ Cbl, float* __restrict__ h,
               HdState* __restrict__ st, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int j = w0; j < kpad; j += nw) {
        if (j >= k) {
            if (lane == 0) h[j] = -INFINITY;
            continue;
        }
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const int m = lane + 32 * u;
            const float v = __fsub_rn(C[(int64_t)j * D + m], ctr[m]);
            float hi, lo;
            split_tf32(v, hi, lo);
            Cc[(int64_t)j * D + m] = hi;
            Cbh[(int64_t)j * D + m] = __float2bfloat16_rn(hi);
            Cbl[(int64_t)j * D + m] = __float2bfloat16_rn(lo);
            s = fma((double)v, (double)v, s);
        }
        s = warp_sum_d(s);
        if (lane == 0) {
            h[j] = __double2float_rn(-0.5 * s);
            atomicMax(&st->cmax_bits, __float_as_uint(__double2float_ru(__dsqrt_ru(s * (1.0 + 0x1p-40)))));
        }
    }
}

// Error bound of the tensor-core scores: |v~_j - v_j| <= E for every j, plus
// the centring and FP64 slack, for a point with ||p'|| <= A and centroids with ||c'|| <= B.
template <int D>
__device__ __forceinline__ double hd_bound(double A, double B)
{
    // split representation error (TF32 hi.hi exact; BF16 rounding of the hi and lo parts in the
    // two correction products; the dropped lo.lo) <= 2^-17 sum|p'_m c'_m|; FP32 accumulation: at
    // most one rounding (<= 2 ulp, 2^-22) per MMA instruction (D/8 TF32 + D/8 BF16 of them)
    // relative to sum|terms|
    const double beta = 0x1p-17 + (double)(D / 4 + 2) * 0x1p-22 * (1.0 + 0x1p-9);
    // (the last two terms: TF32 flushing of subnormal operands, absolute)
    const double E = beta * A * B + 0x1p-23 * (A * B + 0.5 * B * B) + 0x1p-25 * B * B + 0x1p-22 * (A + B) * (A + B) +
                     (double)D * 0x1p-126 * (A + B) + 0x1p-140;
    return E * (1.0 + 0x1p-20);
}

// ---------------------------------------------------------------------- the contraction
// Persistent: CTA b takes point tiles b, b + grid, ...; per tile the whole A (128 x D FP32)
// is loaded once and every centroid tile of 256 streams through a K-chunk ring.  The MMA
// thread accumulates 128 x 256 scores in one of two TMEM buffers while the four epilogue
// warps scan the other (thread = point = TMEM lane): v = acc + h_j, a 32-column max first,
// the top-8 insertion only for columns that can enter it.
template <int D, int TOP>
__global__ void __launch_bounds__(kGemmThreads, 1)
hd_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAh,
               const __grid_constant__ CUtensorMap tmAl, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
               const float* __restrict__ h, int64_t n, int n_tiles_k, int m_tiles, float4* __restrict__ topv,
               int4* __restrict__ topj, const float* __restrict__ pn, const HdState* __restrict__ st,
               const Ctl* __restrict__ ctl)
{
    using G = GemmCfg<D>;
    if (ctl && ctl->done) return;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* sA = base;
    unsigned char* sB = base + G::kABytes;   // stage s: [B_hi | B_lo | (A_lo if not resident)]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + G::kStages * G::kStageBytes);
    uint64_t* full = bars;                       // [kStages] TMA -> MMA
    uint64_t* empty = bars + G::kStages;         // [kStages] MMA -> TMA
    // per K chunk of the point tile: chunk c of the next tile loads as soon as the last centroid
    // tile's chunk-c MMAs of this one are done (overlaps most of the load with the tile's tail)
    uint64_t* afull = bars + 2 * G::kStages;     // [KC] A chunk landed
    uint64_t* aempty = afull + G::KC;            // [KC] A chunk consumed
    uint64_t* tfull = aempty + G::KC;            // [kAccN] accumulator ready
    uint64_t* tempty = tfull + kAccN;            // [kAccN] accumulator drained
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + kAccN);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < G::kStages; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
        for (int c = 0; c < G::KC; ++c) { bar_init(&afull[c], 1); bar_init(&aempty[c], 1); }
        for (int a = 0; a < kAccN; ++a) { bar_init(&tfull[a], 1); bar_init(&tempty[a], kEpiWarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmAh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmAl) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmBl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                     "n"(kAccN * kBN) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tslot;

    if (warp == 0) {
        {   // ---- TMA producer: the whole warp waits, one elected lane issues
            int stage = 0;
            uint32_t sph = 0, aph = 0;
            for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
                // A chunk c: [TF32 hi 16 KB | BF16 hi 8 KB | BF16 lo 8 KB] (BF16 parts only if resident)
                for (int c = 0; c < G::KC; ++c) {
                    bar_wait(&aempty[c], aph ^ 1u);
                    bar_expect_elect(&afull[c], (uint32_t)(G::kABytes / G::KC));
                    unsigned char* ac = sA + c * (G::kABytes / G::KC);
                    tma_2d_elect(ac, &tmA, c * kBK, mt * kBM, &afull[c]);
                    if (G::kALoRes) {
                        tma_2d_elect(ac + G::kAChunk, &tmAh, c * kBK, mt * kBM, &afull[c]);
                        tma_2d_elect(ac + G::kAChunk + G::kAHalf, &tmAl, c * kBK, mt * kBM, &afull[c]);
                    }
                }
                aph ^= 1u;
                for (int nt = 0; nt < n_tiles_k; ++nt)
                    for (int c = 0; c < G::KC; ++c) {
                        bar_wait(&empty[stage], sph ^ 1u);
                        unsigned char* st = sB + stage * G::kStageBytes;
                        bar_expect_elect(&full[stage], (uint32_t)G::kStageBytes);
                        // stage: [B TF32 hi 16 KB | B BF16 hi 8 KB | B BF16 lo 8 KB | (A BF16 hi, lo)]
                        tma_2d_elect(st, &tmB, c * kBK, nt * kBN, &full[stage]);
                        tma_2d_elect(st + G::kBChunk, &tmBh, c * kBK, nt * kBN, &full[stage]);
                        tma_2d_elect(st + G::kBChunk + G::kBHalf, &tmBl, c * kBK, nt * kBN, &full[stage]);
                        if (!G::kALoRes) {
                            tma_2d_elect(st + G::kBChunk + 2 * G::kBHalf, &tmAh, c * kBK, mt * kBM, &full[stage]);
                            tma_2d_elect(st + G::kBChunk + 2 * G::kBHalf + G::kAHalf, &tmAl, c * kBK, mt * kBM,
                                   &full[stage]);
                        }
                        if (++stage == G::kStages) { stage = 0; sph ^= 1u; }
                    }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        {   // ---- MMA issuer: the whole warp waits, one elected lane issues (no divergent loops)
            int stage = 0, acc = 0;
            uint32_t sph = 0, aph = 0, tph = 0;
            const uint32_t a0 = su32(sA), b0 = su32(sB);
            for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
                for (int nt = 0; nt < n_tiles_k; ++nt) {
                    bar_wait(&tempty[acc], tph ^ 1u);
                    tc_after();
                    const uint32_t dt = tmem + (uint32_t)(acc * kBN);
                    for (int c = 0; c < G::KC; ++c) {
                        if (nt == 0) bar_wait(&afull[c], aph);   // this tile's A chunk c
                        bar_wait(&full[stage], sph);
                        tc_after();
                        const uint32_t ah = a0 + c * (G::kABytes / G::KC);
                        const uint32_t bh = b0 + stage * G::kStageBytes;
                        const uint32_t bbh = bh + G::kBChunk, bbl = bbh + G::kBHalf;
                        const uint32_t abh = G::kALoRes ? ah + G::kAChunk : bbl + G::kBHalf;
                        const uint32_t abl = abh + G::kAHalf;
                        // descriptors built once per stage; a K step of 32 B adds 2 to the start
                        // address field (addresses < 256 KB: no carry out of its 14 bits)
                        const uint64_t dah = sdesc(ah), dbh = sdesc(bh);
                        const uint64_t dabl = sdesc64(abl), dabh = sdesc64(abh);
                        const uint64_t dbbh = sdesc64(bbh), dbbl = sdesc64(bbl);
                        mma_chunk(dt, dah, dbh, dabl, dabh, dbbh, dbbl, c != 0 ? 1u : 0u);
                        mma_commit_elect(&empty[stage]);   // frees the B stage when these MMAs complete
                        if (nt == n_tiles_k - 1) mma_commit_elect(&aempty[c]);   // A chunk c is free
                        if (++stage == G::kStages) { stage = 0; sph ^= 1u; }
                    }
                    mma_commit_elect(&tfull[acc]);
                    if (++acc == kAccN) { acc = 0; tph ^= 1u; }
                }
                aph ^= 1u;
            }
        }
        __syncwarp();
    } else {
        // ---- epilogue: 4 warps, thread = point row (TMEM lane 32 (warp % 4) + lane)
        // warp w: TMEM lane quadrant w % 4 (rows 32 (w % 4) ..), column half (w - 2) / 4.  The
        // warp's 64 h_j come straight from global memory (L1-broadcast loads issued before the
        // accumulator wait: no shared staging, no barrier between the epilogue warps).
        const int ew = warp - 2;
        const int lb = 32 * (warp & 3), half = ew >> 2;
        const int row = lb + lane;
        const uint32_t tq = tmem + ((uint32_t)lb << 16) + (uint32_t)(64 * half);
        int acc = 0;
        uint32_t tph = 0;
        const double Bc = (double)__uint_as_float(st->cmax_bits);
        for (int mt = blockIdx.x; mt < m_tiles; mt += gridDim.x) {
            float tv[TOP];
            int tj[TOP];
#pragma unroll
            for (int q = 0; q < TOP; ++q) { tv[q] = -INFINITY; tj[q] = -1; }
            // Only scores >= v1 - 2E can matter to hd_certify_kernel (same bound, rounded so this
            // threshold never exceeds certify's): t = max(v8, v1 - 2E) rejects the rest at once.
            const int64_t ir = (int64_t)mt * kBM + row;
            const float two_e = __double2float_ru(2.0 * hd_bound<D>(ir < n ? (double)pn[ir] : 0.0, Bc));
            float t = -INFINITY;
            for (int nt = 0; nt < n_tiles_k; ++nt) {
                float4 hq[16];
                const float4* h4 = reinterpret_cast<const float4*>(h + nt * kBN + 64 * half);
#pragma unroll
                for (int q = 0; q < 16; ++q) hq[q] = __ldg(h4 + q);
                bar_wait(&tfull[acc], tph);
                tc_after();
                uint32_t r[64];
                tmem_ld64(tq + (uint32_t)(acc * kBN), r);   // this warp's 64 columns; TMEM goes back at once
                tc_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[acc]);
#pragma unroll
                for (int q = 0; q < 16; ++q) {   // packed FADD2: two columns per instruction (RN, as FADD)
                    const float2 s0 = __fadd2_rn(make_float2(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1])),
                                                 make_float2(hq[q].x, hq[q].y));
                    const float2 s1 = __fadd2_rn(make_float2(__uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])),
                                                 make_float2(hq[q].z, hq[q].w));
                    r[4 * q] = __float_as_uint(s0.x);
                    r[4 * q + 1] = __float_as_uint(s0.y);
                    r[4 * q + 2] = __float_as_uint(s1.x);
                    r[4 * q + 3] = __float_as_uint(s1.y);
                }
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {   // unrolled: r[] stays in registers
                    const float* v = reinterpret_cast<const float*>(r + 32 * ch);
                    float mx = fmaxf(fmaxf(v[0], v[1]), v[2]);
#pragma unroll
                    for (int c = 3; c < 32; c += 2) mx = fmaxf(fmaxf(mx, v[c]), c + 1 < 32 ? v[c + 1] : v[c]);
                    if (mx > t) {
                        // the final v1 >= mx, so nothing below mx - 2E can reach the band: raise t
                        // first (the first chunk of a tile would otherwise qualify all 32 columns)
                        t = fmaxf(t, __fsub_rd(mx, two_e));
                        // the columns that can enter the top 8, then one compact insertion loop
                        // (a select tree fetches v[c] without local memory)
                        unsigned msk = 0u;
#pragma unroll
                        for (int c = 0; c < 32; ++c) msk |= (v[c] > t ? 1u : 0u) << c;
                        const int jb = nt * kBN + 64 * half + ch * 32;
                        while (msk) {
                            const int c = __ffs(msk) - 1;
                            msk &= msk - 1u;
                            float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
                            for (int q = 0; q < 16; ++q) t16[q] = (c & 16) ? v[q + 16] : v[q];
#pragma unroll
                            for (int q = 0; q < 8; ++q) t8[q] = (c & 8) ? t16[q + 8] : t16[q];
#pragma unroll
                            for (int q = 0; q < 4; ++q) t4[q] = (c & 4) ? t8[q + 4] : t8[q];
#pragma unroll
                            for (int q = 0; q < 2; ++q) t2[q] = (c & 2) ? t4[q + 2] : t4[q];
                            const float x = (c & 1) ? t2[1] : t2[0];
                            if (x > t) {   // strict: an equal value at a larger j stays behind
                                const int j = jb + c;
#pragma unroll
                                for (int q = TOP - 1; q > 0; --q) {   // shift down, branch-free
                                    const bool gp = x > tv[q - 1], gq = x > tv[q];
                                    tv[q] = gp ? tv[q - 1] : (gq ? x : tv[q]);
                                    tj[q] = gp ? tj[q - 1] : (gq ? j : tj[q]);
                                }
                                const bool g0 = x > tv[0];
                                tv[0] = g0 ? x : tv[0];
                                tj[0] = g0 ? j : tj[0];
                                t = fmaxf(tv[TOP - 1], __fsub_rd(tv[0], two_e));
                            }
                        }
                    }
                }
                if (++acc == kAccN) { acc = 0; tph ^= 1u; }
            }
            const int64_t i = (int64_t)mt * kBM + row;
            if (i < n) {   // this half's top 8; hd_certify_kernel merges the two halves
                float4* ov = topv + (2 * i + half) * (TOP / 4);
                int4* oj = topj + (2 * i + half) * (TOP / 4);
#pragma unroll
                for (int w = 0; w < TOP / 4; ++w) {
                    ov[w] = make_float4(tv[4 * w], tv[4 * w + 1], tv[4 * w + 2], tv[4 * w + 3]);
                    oj[w] = make_int4(tj[4 * w], tj[4 * w + 1], tj[4 * w + 2], tj[4 * w + 3]);
                }
            }
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAccN * kBN) : "memory");
}

// ---------------------------------------------------------------------- certification
// FP64 distance in exactly the oracle's order (sequential m, multiply then add, no FMA).
template <int D>
__device__ __forceinline__ double d64_seq(const float* __restrict__ p, const float* __restrict__ c)
{
    double s = 0.0;
#pragma unroll 8
    for (int m = 0; m < D; ++m) {
        const double t = __dsub_rn((double)p[m], (double)c[m]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

// FP64 distance with lanes over coordinates (fma, any summation order), the sum on every lane.
// |D^ - D64| <= 2^-44 D for d <= 256: both are within (d + 5) 2^-53 D of the exact value.
template <int D>
__device__ __forceinline__ double d64_par(int lane, const float (&pv)[D / 32], const float* __restrict__ c)
{
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < D / 32; ++u) {
        const double t = (double)pv[u] - (double)c[lane + 32 * u];
        s = fma(t, t, s);
    }
    return warp_sum_d(s);
}

constexpr double kTieRel = 0x1p-42;   // D^ within this relative band of the minimum: decide in d64_seq

// Warp-cooperative: point i (coordinates pv, lanes over m) takes label a whose FP64 distance
// is s -> SSE_t summand, changed_t, and the running sums move.
template <int D>
__device__ __forceinline__ void hd_settle(int lane, int64_t i, int a, double s, const float (&pv)[D / 32], int prev,
                                          int32_t* __restrict__ labels, const double* __restrict__ qo,
                                          const double* __restrict__ qs, unsigned long long* __restrict__ acc_sum,
                                          unsigned int* __restrict__ acc_cnt, unsigned long long* __restrict__ acc_q,
                                          const unsigned long long* __restrict__ pq2, double sse_scale,
                                          unsigned long long& sq, unsigned long long& chg)
{
    // acc_q given: SSE_t comes from the moment sums in hd_finalize_kernel; else per point here
    if (!acc_q && lane == 0) sq += sse_q(s, sse_scale);
    if (prev != a) {
        if (lane == 0) {
            labels[i] = a;
            ++chg;
        }
        if (!acc_sum) return;   // km_assign: labels and SSE only
        if (lane == 0) {
            atomicAdd(&acc_cnt[a], 1u);
            if (prev >= 0) atomicAdd(&acc_cnt[prev], 0xffffffffu);
            if (acc_q) {
                atomicAdd(&acc_q[a], pq2[i]);
                if (prev >= 0) atomicAdd(&acc_q[prev], 0ull - pq2[i]);
            }
        }
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const int m = lane + 32 * u;
            const unsigned long long q =
                (unsigned long long)__double2ll_rn(__dmul_rn(__dsub_rn((double)pv[u], qo[m]), qs[m]));
            atomicAdd(&acc_sum[(int64_t)a * D + m], q);
            if (prev >= 0) atomicAdd(&acc_sum[(int64_t)prev * D + m], 0ull - q);
        }
    }
}

// Two phases per group of 32 points.  A (lane = point): merge the two column halves' top 8
// (value descending, lower j first), the bound E_i, and the decision class: top-2 gap > 2E ->
// certified; the band [v1 - 2E, v1] within the top 8 -> FP64 among those; else the point goes
// to hd_fallback_kernel.  B (warp per point, lanes over coordinates, next point's rows
// prefetched): the FP64 distance of the label (SSE_t) or of the band candidates (parallel sum;
// the oracle's sequential form only for FP64 near-ties), then the label change and the sums.
template <int D, int TOP>
__global__ void __launch_bounds__(256)
hd_certify_kernel(const float* __restrict__ P, const float* __restrict__ C, int64_t n, const float4* __restrict__ topv,
                  const int4* __restrict__ topj, const float* __restrict__ pn, HdState* __restrict__ st,
                  int32_t* __restrict__ labels, int first, const double* __restrict__ qo, const double* __restrict__ qs,
                  unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt,
                  unsigned long long* __restrict__ acc_q, const unsigned long long* __restrict__ pq2, int* __restrict__ fb,
                  const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double B = (double)__uint_as_float(st->cmax_bits);
    const double ss = st->sse_scale;
    const bool all_fb = first == 2;   // (debug: every point to the fallback)
    if (all_fb) first = 1;
    unsigned long long sq = 0, chg = 0, ncert = 0, nband = 0, nfull = 0;
    for (int64_t base = gw * 32; base < n; base += nw * 32) {
        // ---- A: lane = point
        const int64_t i = base + lane;
        float v[TOP];
        int jj[TOP];
#pragma unroll
        for (int q = 0; q < TOP; ++q) { v[q] = -INFINITY; jj[q] = 0x7fffffff; }
        int kind = 3, prev = -1;
        double two_e = 0.0;
        if (i < n) {
            float av[TOP], bv[TOP];
            int aj[TOP], bj[TOP];
            {
                const float4* pa = topv + 2 * (TOP / 4) * i;   // [half 0: TOP/4 x float4][half 1]
                const int4* ja = topj + 2 * (TOP / 4) * i;
#pragma unroll
                for (int w = 0; w < TOP / 4; ++w) {
                    const float4 x = pa[w], y = pa[TOP / 4 + w];
                    const int4 xj = ja[w], yj = ja[TOP / 4 + w];
                    av[4 * w] = x.x; av[4 * w + 1] = x.y; av[4 * w + 2] = x.z; av[4 * w + 3] = x.w;
                    bv[4 * w] = y.x; bv[4 * w + 1] = y.y; bv[4 * w + 2] = y.z; bv[4 * w + 3] = y.w;
                    aj[4 * w] = xj.x; aj[4 * w + 1] = xj.y; aj[4 * w + 2] = xj.z; aj[4 * w + 3] = xj.w;
                    bj[4 * w] = yj.x; bj[4 * w + 1] = yj.y; bj[4 * w + 2] = yj.z; bj[4 * w + 3] = yj.w;
                }
#pragma unroll
                for (int q = 0; q < TOP; ++q) {   // empty slots (-inf, -1) sort last
                    aj[q] = aj[q] < 0 ? 0x7fffffff : aj[q];
                    bj[q] = bj[q] < 0 ? 0x7fffffff : bj[q];
                }
            }
#pragma unroll
            for (int o = 0; o < TOP; ++o) {   // merge of two sorted lists, static indices only
                const bool ta = av[0] > bv[0] || (av[0] == bv[0] && aj[0] < bj[0]);
                v[o] = ta ? av[0] : bv[0];
                jj[o] = ta ? aj[0] : bj[0];
#pragma unroll
                for (int q = 0; q < TOP - 1; ++q) {
                    av[q] = ta ? av[q + 1] : av[q];
                    aj[q] = ta ? aj[q + 1] : aj[q];
                    bv[q] = ta ? bv[q] : bv[q + 1];
                    bj[q] = ta ? bj[q] : bj[q + 1];
                }
                av[TOP - 1] = ta ? -INFINITY : av[TOP - 1];
                aj[TOP - 1] = ta ? 0x7fffffff : aj[TOP - 1];
                bv[TOP - 1] = ta ? bv[TOP - 1] : -INFINITY;
                bj[TOP - 1] = ta ? bj[TOP - 1] : 0x7fffffff;
            }
            two_e = 2.0 * hd_bound<D>((double)pn[i], B);
            const double v1 = v[0];
            kind = all_fb ? 2 : (v1 - (double)v[1] > two_e) ? 0 : ((double)v[TOP - 1] < v1 - two_e) ? 1 : 2;
            prev = first ? -1 : labels[i];
        }
        const unsigned fm = __ballot_sync(full, kind == 2);
        if (fm) {
            int pos = 0;
            if (lane == __ffs(fm) - 1) pos = atomicAdd(&st->nfb, __popc(fm));
            pos = __shfl_sync(full, pos, __ffs(fm) - 1);
            if (kind == 2) fb[pos + __popc(fm & lt)] = (int)i;
        }
        ncert += kind == 0;
        nband += kind == 1;
        nfull += kind == 2;
        // ---- B: warp per point
        // with moment sums (acc_q) a certified point that keeps its label needs nothing more
        unsigned todo = __ballot_sync(full, kind == 1 || (kind == 0 && (!acc_q || prev != jj[0])));
        int q = todo ? __ffs(todo) - 1 : -1;
        float pv[D / 32], cv[D / 32];
        auto load_rows = [&](int qq, float (&pr)[D / 32], float (&cr)[D / 32]) {
            const int a0 = __shfl_sync(full, jj[0], qq);
#pragma unroll
            for (int u = 0; u < D / 32; ++u) {
                pr[u] = P[(base + qq) * D + lane + 32 * u];
                cr[u] = C[(int64_t)a0 * D + lane + 32 * u];
            }
        };
        if (q >= 0) load_rows(q, pv, cv);
        while (q >= 0) {
            todo &= todo - 1;
            const int qn = todo ? __ffs(todo) - 1 : -1;
            float pnx[D / 32], cnx[D / 32];
            if (qn >= 0) load_rows(qn, pnx, cnx);   // the next point's rows while this one is settled
            const int64_t iq = base + q;
            const int kq = __shfl_sync(full, kind, q);
            const int pq = __shfl_sync(full, prev, q);
            int a = __shfl_sync(full, jj[0], q);
            double s;
            {
                double t2 = 0.0;
#pragma unroll
                for (int u = 0; u < D / 32; ++u) {
                    const double t = (double)pv[u] - (double)cv[u];
                    t2 = fma(t, t, t2);
                }
                s = warp_sum_d(t2);
            }
            if (kq == 1) {
                // every centroid outside the top 8 has v <= v8 < v1 - 2E: the FP64 argmin (and all
                // its ties) is among the in-band top entries (at least two)
                const double te = __shfl_sync(full, two_e, q);
                const double v1 = __shfl_sync(full, v[0], q);
                double dh[TOP];
                int tjj[TOP];
                double b1 = s, b2 = INFINITY;
                int j1 = a;
                dh[0] = s;
                tjj[0] = a;
#pragma unroll
                for (int c = 1; c < TOP; ++c) {
                    const float vc = __shfl_sync(full, v[c], q);
                    tjj[c] = __shfl_sync(full, jj[c], q);
                    dh[c] = INFINITY;
                    if (tjj[c] != 0x7fffffff && (double)vc >= v1 - te)
                        dh[c] = d64_par<D>(lane, pv, C + (int64_t)tjj[c] * D);
                    if (dh[c] < b1 || (dh[c] == b1 && tjj[c] < j1)) { b2 = b1; b1 = dh[c]; j1 = tjj[c]; }
                    else if (dh[c] < b2) b2 = dh[c];
                }
                a = j1;
                s = b1;
                if (!(b2 > b1 * (1.0 + kTieRel))) {
                    // an FP64 near-tie: the oracle's own sequential form decides (lowest j on ties)
                    double dv = INFINITY;
                    int jv = 0x7fffffff;
                    double myd = INFINITY;
                    int myj = 0x7fffffff;
#pragma unroll
                    for (int c = 0; c < TOP; ++c)
                        if (lane == c) { myd = dh[c]; myj = tjj[c]; }
                    if (lane < TOP && myd <= b1 * (1.0 + kTieRel)) {
                        jv = myj;
                        dv = d64_seq<D>(P + iq * D, C + (int64_t)jv * D);
                    }
#pragma unroll
                    for (int o = TOP / 2; o > 0; o >>= 1) {   // lanes 0 .. TOP-1 hold the candidates
                        const double od = __shfl_xor_sync(full, dv, o);
                        const int oj = __shfl_xor_sync(full, jv, o);
                        if (od < dv || (od == dv && oj < jv)) { dv = od; jv = oj; }
                    }
                    a = __shfl_sync(full, jv, 0);
                    s = __shfl_sync(full, dv, 0);
                }
            }
            hd_settle<D>(lane, iq, a, s, pv, pq, labels, qo, qs, acc_sum, acc_cnt, acc_q, pq2, ss, sq, chg);
            q = qn;
#pragma unroll
            for (int u = 0; u < D / 32; ++u) { pv[u] = pnx[u]; cv[u] = cnx[u]; }
        }
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, chg);
    __syncthreads();
    unsigned long long c3 = ncert;
    block_sum2<256>(dummy, c3);
    __syncthreads();
    unsigned long long b3 = nband;
    block_sum2<256>(dummy, b3);
    __syncthreads();
    unsigned long long f3 = nfull;
    block_sum2<256>(dummy, f3);
    if (threadIdx.x == 0) {
        atomicAdd(&st->sse_q, sq);
        atomicAdd(&st->chg, chg);
        atomicAdd(&st->n_cert, c3);
        atomicAdd(&st->n_band, b3);
        atomicAdd(&st->n_full, f3);
    }
}

// Points the certification could not decide: FP64 over all k.  A CTA takes 8 of them at once
// (every centroid row is read once for the 8): warp w scans j = w, w + 8, ..., lanes over
// coordinates; the 8 partial sums are reduce-scattered so lane l ends with point l >> 2's
// D^.  Per point the CTA minimum decides unless an FP64 near-tie remains, which the oracle's
// sequential form settles (lowest j on ties).
constexpr int kFbPts = 8;
constexpr int kFbSlices = 32;   // hd_fb_slice_kernel: slices of the k centroids per undecided point
constexpr int kFbCap = 4096;    // undecided points handled by the sliced pair; the rest: all k per CTA

template <int D>
__global__ void __launch_bounds__(256)
hd_fallback_kernel(const float* __restrict__ P, const float* __restrict__ C, int k, const int* __restrict__ fb,
                   HdState* __restrict__ st, int32_t* __restrict__ labels, int first, const double* __restrict__ qo,
                   const double* __restrict__ qs, unsigned long long* __restrict__ acc_sum,
                   unsigned int* __restrict__ acc_cnt, unsigned long long* __restrict__ acc_q,
                   const unsigned long long* __restrict__ pq2, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    __shared__ double s_b1[8][kFbPts], s_b2[8][kFbPts];
    __shared__ int s_j1[8][kFbPts];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nfb = st->nfb;   // points [0, kFbCap) go through hd_fb_slice / hd_fb_settle
    const double ss = st->sse_scale;
    unsigned long long sq = 0, chg = 0;
    const int nbatch = nfb > kFbCap ? (nfb - kFbCap + kFbPts - 1) / kFbPts : 0;
    for (int bi = blockIdx.x; bi < nbatch; bi += gridDim.x) {
        const int q0 = kFbCap + bi * kFbPts, nq = min(kFbPts, nfb - q0);
        float pv[kFbPts][D / 32];
#pragma unroll
        for (int q = 0; q < kFbPts; ++q) {
            const int64_t i = q < nq ? fb[q0 + q] : fb[q0];
#pragma unroll
            for (int u = 0; u < D / 32; ++u) pv[q][u] = P[i * D + lane + 32 * u];
        }
        const int myq = lane >> 2;   // the point this lane's reduced value belongs to
        double b1 = INFINITY, b2 = INFINITY;
        int j1 = 0x7fffffff;
        for (int j = warp; j < k; j += 8) {
            double v[kFbPts];
#pragma unroll
            for (int q = 0; q < kFbPts; ++q) v[q] = 0.0;
#pragma unroll
            for (int u = 0; u < D / 32; ++u) {
                const double c = (double)C[(int64_t)j * D + lane + 32 * u];
#pragma unroll
                for (int q = 0; q < kFbPts; ++q) {
                    const double t = (double)pv[q][u] - c;
                    v[q] = fma(t, t, v[q]);
                }
            }
            // reduce-scatter of 8 values over 32 lanes (xor 16, 8, 4 halve the vector; 2, 1 finish)
            const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
            double w4[4], w2[2];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const double keep = h4 ? v[x + 4] : v[x], send = h4 ? v[x] : v[x + 4];
                w4[x] = keep + __shfl_xor_sync(full, send, 16);
            }
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                const double keep = h3 ? w4[x + 2] : w4[x], send = h3 ? w4[x] : w4[x + 2];
                w2[x] = keep + __shfl_xor_sync(full, send, 8);
            }
            double y = (h2 ? w2[1] : w2[0]) + __shfl_xor_sync(full, h2 ? w2[0] : w2[1], 4);
            y += __shfl_xor_sync(full, y, 2);
            y += __shfl_xor_sync(full, y, 1);
            if (y < b1) { b2 = b1; b1 = y; j1 = j; }   // j ascending per warp: the first minimum stays
            else if (y < b2) b2 = y;
        }
        if ((lane & 3) == 0) { s_b1[warp][myq] = b1; s_b2[warp][myq] = b2; s_j1[warp][myq] = j1; }
        __syncthreads();
        if (warp < nq) {
            const int q = warp;
            const int64_t i = fb[q0 + q];
            double e1 = lane < 8 ? s_b1[lane][q] : INFINITY, e2 = lane < 8 ? s_b2[lane][q] : INFINITY;
            int f1 = lane < 8 ? s_j1[lane][q] : 0x7fffffff;
            double B1 = e1;
            int J1 = f1;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(full, B1, o);
                const int oj = __shfl_xor_sync(full, J1, o);
                if (od < B1 || (od == B1 && oj < J1)) { B1 = od; J1 = oj; }
            }
            double B2 = (f1 == J1) ? e2 : e1;   // the winning warp offers its second, the others their first
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) B2 = fmin(B2, __shfl_xor_sync(full, B2, o));
            // lanes 0-7 hold the reduction: every lane takes theirs (uniform control flow below)
            B1 = __shfl_sync(full, B1, 0);
            B2 = __shfl_sync(full, B2, 0);
            J1 = __shfl_sync(full, J1, 0);
            float pq[D / 32];
#pragma unroll
            for (int u = 0; u < D / 32; ++u) pq[u] = P[i * D + lane + 32 * u];
            int a = J1;
            double s = B1;
            if (!(B2 > B1 * (1.0 + kTieRel)) && first != 3) {
                // FP64 near-tie: the oracle's sequential form over the band (rare: exact ties)
                const double thr = B1 * (1.0 + kTieRel);
                double best = INFINITY;
                int bj = 0x7fffffff;
                for (int j = 0; j < k; ++j) {
                    const double dj = d64_par<D>(lane, pq, C + (int64_t)j * D);
                    if (dj <= thr) {
                        const double e = d64_seq<D>(P + i * D, C + (int64_t)j * D);
                        if (e < best) { best = e; bj = j; }
                    }
                }
                a = bj;
                s = best;
            }
            const int prev = first ? -1 : labels[i];
            hd_settle<D>(lane, i, a, s, pq, prev, labels, qo, qs, acc_sum, acc_cnt, acc_q, pq2, ss, sq, chg);
        }
        __syncthreads();   // the per-point tables are rewritten by the next batch
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, chg);
    if (threadIdx.x == 0 && (sq | chg)) {
        atomicAdd(&st->sse_q, sq);
        atomicAdd(&st->chg, chg);
    }
}

// Few undecided points (the usual case): each point's k centroids are split into kFbSlices
// slices scanned by different CTAs (8 points per CTA as above), every slice leaving its (best,
// index, second) in a scratch table; hd_fb_settle_kernel then decides per point.  Points beyond
// kFbCap take hd_fallback_kernel (all k per CTA).
template <int D>
__global__ void __launch_bounds__(256)
hd_fb_slice_kernel(const float* __restrict__ P, const float* __restrict__ C, int k, const int* __restrict__ fb,
                   const HdState* __restrict__ st, double* __restrict__ sb1, double* __restrict__ sb2,
                   int* __restrict__ sj1, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    __shared__ double s_b1[8][kFbPts], s_b2[8][kFbPts];
    __shared__ int s_j1[8][kFbPts];
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nfb = min(st->nfb, kFbCap);
    const int nbatch = (nfb + kFbPts - 1) / kFbPts;
    const int kc = (k + kFbSlices - 1) / kFbSlices;
    for (int item = blockIdx.x; item < nbatch * kFbSlices; item += gridDim.x) {
        const int bi = item / kFbSlices, sl = item % kFbSlices;
        const int q0 = bi * kFbPts, nq = min(kFbPts, nfb - q0);
        float pv[kFbPts][D / 32];
#pragma unroll
        for (int q = 0; q < kFbPts; ++q) {
            const int64_t i = q < nq ? fb[q0 + q] : fb[q0];
#pragma unroll
            for (int u = 0; u < D / 32; ++u) pv[q][u] = P[i * D + lane + 32 * u];
        }
        const int myq = lane >> 2;
        double b1 = INFINITY, b2 = INFINITY;
        int j1 = 0x7fffffff;
        const int jend = min(k, (sl + 1) * kc);
        for (int j = sl * kc + warp; j < jend; j += 8) {
            double v[kFbPts];
#pragma unroll
            for (int q = 0; q < kFbPts; ++q) v[q] = 0.0;
#pragma unroll
            for (int u = 0; u < D / 32; ++u) {
                const double c = (double)C[(int64_t)j * D + lane + 32 * u];
#pragma unroll
                for (int q = 0; q < kFbPts; ++q) {
                    const double t = (double)pv[q][u] - c;
                    v[q] = fma(t, t, v[q]);
                }
            }
            // reduce-scatter of 8 values over 32 lanes (xor 16, 8, 4 halve the vector; 2, 1 finish)
            const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
            double w4[4], w2[2];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                const double keep = h4 ? v[x + 4] : v[x], send = h4 ? v[x] : v[x + 4];
                w4[x] = keep + __shfl_xor_sync(full, send, 16);
            }
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                const double keep = h3 ? w4[x + 2] : w4[x], send = h3 ? w4[x] : w4[x + 2];
                w2[x] = keep + __shfl_xor_sync(full, send, 8);
            }
            double y = (h2 ? w2[1] : w2[0]) + __shfl_xor_sync(full, h2 ? w2[0] : w2[1], 4);
            y += __shfl_xor_sync(full, y, 2);
            y += __shfl_xor_sync(full, y, 1);
            if (y < b1) { b2 = b1; b1 = y; j1 = j; }   // j ascending per warp: the first minimum stays
            else if (y < b2) b2 = y;
        }
        if ((lane & 3) == 0) { s_b1[warp][myq] = b1; s_b2[warp][myq] = b2; s_j1[warp][myq] = j1; }
        __syncthreads();
        if (warp < nq) {
            const int q = warp;
            double e1 = lane < 8 ? s_b1[lane][q] : INFINITY, e2 = lane < 8 ? s_b2[lane][q] : INFINITY;
            int f1 = lane < 8 ? s_j1[lane][q] : 0x7fffffff;
            double B1 = e1;
            int J1 = f1;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(full, B1, o);
                const int oj = __shfl_xor_sync(full, J1, o);
                if (od < B1 || (od == B1 && oj < J1)) { B1 = od; J1 = oj; }
            }
            double B2 = (f1 == J1) ? e2 : e1;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) B2 = fmin(B2, __shfl_xor_sync(full, B2, o));
            if (lane == 0) {
                const int64_t slot = (int64_t)(q0 + q) * kFbSlices + sl;
                sb1[slot] = B1;
                sb2[slot] = B2;
                sj1[slot] = J1;
            }
        }
        __syncthreads();
    }
}

// Warp per undecided point (< kFbCap): the slices' results -> the minimum (lowest j on ties)
// and the runner-up; an FP64 near-tie takes the oracle's sequential form over all k.
template <int D>
__global__ void __launch_bounds__(256)
hd_fb_settle_kernel(const float* __restrict__ P, const float* __restrict__ C, int k, const int* __restrict__ fb,
                    HdState* __restrict__ st, int32_t* __restrict__ labels, int first, const double* __restrict__ qo,
                    const double* __restrict__ qs, unsigned long long* __restrict__ acc_sum,
                    unsigned int* __restrict__ acc_cnt, unsigned long long* __restrict__ acc_q,
                    const unsigned long long* __restrict__ pq2, const double* __restrict__ sb1,
                    const double* __restrict__ sb2, const int* __restrict__ sj1, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int nfb = min(st->nfb, kFbCap);
    const double ss = st->sse_scale;
    unsigned long long sq = 0, chg = 0;
    for (int p = w0; p < nfb; p += nw) {
        const int64_t i = fb[p];
        const int64_t slot = (int64_t)p * kFbSlices + lane;
        const double e1 = lane < kFbSlices ? sb1[slot] : INFINITY, e2 = lane < kFbSlices ? sb2[slot] : INFINITY;
        const int f1 = lane < kFbSlices ? sj1[slot] : 0x7fffffff;
        double B1 = e1;
        int J1 = f1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(full, B1, o);
            const int oj = __shfl_xor_sync(full, J1, o);
            if (od < B1 || (od == B1 && oj < J1)) { B1 = od; J1 = oj; }
        }
        double B2 = (f1 == J1) ? e2 : e1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) B2 = fmin(B2, __shfl_xor_sync(full, B2, o));
        float pq[D / 32];
#pragma unroll
        for (int u = 0; u < D / 32; ++u) pq[u] = P[i * D + lane + 32 * u];
        int a = J1;
        double s = B1;
        if (!(B2 > B1 * (1.0 + kTieRel)) && first != 3) {
            const double thr = B1 * (1.0 + kTieRel);
            double best = INFINITY;
            int bj = 0x7fffffff;
            for (int j = 0; j < k; ++j) {
                const double dj = d64_par<D>(lane, pq, C + (int64_t)j * D);
                if (dj <= thr) {
                    const double e = d64_seq<D>(P + i * D, C + (int64_t)j * D);
                    if (e < best) { best = e; bj = j; }
                }
            }
            a = bj;
            s = best;
        }
        const int prev = first ? -1 : labels[i];
        hd_settle<D>(lane, i, a, s, pq, prev, labels, qo, qs, acc_sum, acc_cnt, acc_q, pq2, ss, sq, chg);
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, chg);
    if (threadIdx.x == 0 && (sq | chg)) {
        atomicAdd(&st->sse_q, sq);
        atomicAdd(&st->chg, chg);
    }
}

// ------------------------------------------------------------------------------ refine
// Warp per centroid: c_j = o + sv(j) / |S_j| * 2^-s (FP64, rounded to FP32; empty keeps c_j),
// drift ||c_new - c_old||.  The running sums persist (incremental).
template <int D>
__global__ void __launch_bounds__(256)
hd_finalize_kernel(float* __restrict__ C, int k, const unsigned long long* __restrict__ acc_sum,
                   const unsigned int* __restrict__ acc_cnt, const double* __restrict__ qo,
                   const double* __restrict__ qi, int32_t* __restrict__ counts_out, HdState* __restrict__ st,
                   const Ctl* __restrict__ ctl, const unsigned long long* __restrict__ acc_q = nullptr)
{
    if (ctl && ctl->done) return;
    const double ss = st->sse_scale, sinv = st->sse_inv;
    unsigned long long sq = 0;
    const int lane = threadIdx.x & 31;
    const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    double md = 0.0;
    for (int j = w0; j < k; j += nw) {
        const unsigned int c = acc_cnt[j];
        double dd = 0.0, cs = 0.0, cc = 0.0;   // (c - o).S and ||c - o||^2 with the assignment's c
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const int m = lane + 32 * u;
            const int64_t idx = (int64_t)j * D + m;
            const float old = C[idx];
            if (acc_q) {
                const double co = (double)old - qo[m];
                cs = fma(co, (double)acc_sum[idx] * qi[m], cs);
                cc = fma(co, co, cc);
            }
            float nw_ = old;
            if (c > 0) {
                const double mean =
                    __dadd_rn(qo[m], __dmul_rn(__ddiv_rn((double)acc_sum[idx], (double)c), qi[m]));
                nw_ = __double2float_rn(mean);
            }
            const double t = __dsub_rn((double)nw_, (double)old);
            dd = fma(t, t, dd);
            C[idx] = nw_;
        }
        dd = warp_sum_d(dd);
        md = fmax(md, sqrt(dd));
        if (lane == 0 && counts_out) counts_out[j] = (int32_t)c;
        if (acc_q) {
            // SSE_t of cluster j from its moments: sum_i ||p_i - c||^2 = Q_j - 2 (c - o).S_j +
            // |S_j| ||c - o||^2 (o = the fixed-point origin; Q_j, S_j exact integers)
            cs = warp_sum_d(cs);
            cc = warp_sum_d(cc);
            if (lane == 0 && c > 0) {
                const double sj = (double)acc_q[j] * sinv - 2.0 * cs + (double)c * cc;
                sq += sse_q(fmax(sj, 0.0), ss);
            }
        }
    }
    if (acc_q && lane == 0 && sq) atomicAdd(&st->sse_q, sq);
    if (lane == 0 && md > 0.0) atomicMax(&st->md_bits, (unsigned long long)__double_as_longlong(md));
}

// km_update: every point's fixed-point coordinates into sv(label), |S_label| += 1 (warp per point).
template <int D>
__global__ void __launch_bounds__(256)
hd_accumulate_kernel(const float* __restrict__ P, int64_t n, const int32_t* __restrict__ labels,
                     const double* __restrict__ qo, const double* __restrict__ qs,
                     unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        const int a = labels[i];
        if (lane == 0) atomicAdd(&acc_cnt[a], 1u);
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const int m = lane + 32 * u;
            atomicAdd(&acc_sum[(int64_t)a * D + m], (unsigned long long)__double2ll_rn(
                                                        __dmul_rn(__dsub_rn((double)P[i * D + m], qo[m]), qs[m])));
        }
    }
}

// km_assign / km_update: the state's SSE_t and max drift to device scalars (nullable).
__global__ void hd_scalars_kernel(const HdState* __restrict__ st, double* __restrict__ sse, double* __restrict__ md)
{
    if (sse) *sse = __dmul_rn((double)st->sse_q, st->sse_inv);
    if (md) *md = __longlong_as_double((long long)st->md_bits);
}

// Data-parallel (km_dp_*): the shard's running sums, counts, changed_t and SSE_t as one u64
// vector + one double; and the all-reduced vector back as the global sums for the refine.
__global__ void __launch_bounds__(1024)
hd_export_kernel(const unsigned long long* __restrict__ acc_sum, const unsigned int* __restrict__ acc_cnt,
                 const unsigned long long* __restrict__ acc_q, int kd, int k, const HdState* __restrict__ st,
                 unsigned long long* __restrict__ out_u, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    for (int i = threadIdx.x; i < kd; i += blockDim.x) out_u[i] = acc_sum[i];
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        out_u[kd + j] = acc_cnt[j];
        out_u[kd + k + 1 + j] = acc_q[j];   // the moment sums Q_j (layout: sums, counts, changed, Q)
    }
    if (threadIdx.x == 0) {
        out_u[kd + k] = st->chg;   // (SSE_t comes from the all-reduced moment sums Q)
    }
}

__global__ void __launch_bounds__(1024)
hd_import_kernel(const unsigned long long* __restrict__ in_u, int kd, int k,
                 unsigned long long* __restrict__ g_sum, unsigned int* __restrict__ g_cnt,
                 unsigned long long* __restrict__ g_q, HdState* __restrict__ st, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    for (int i = threadIdx.x; i < kd; i += blockDim.x) g_sum[i] = in_u[i];
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        g_cnt[j] = (unsigned int)in_u[kd + j];
        g_q[j] = in_u[kd + k + 1 + j];
    }
    if (threadIdx.x == 0) {
        st->chg = in_u[kd + k];   // the global changed_t (hd_tail_kernel); SSE_t: hd_finalize_kernel
        st->sse_q = 0ull;         // from the global moment sums
    }
}

// One thread: the iteration's traces and the convergence decision (R6), then reset.
__global__ void hd_tail_kernel(HdState* __restrict__ st, double* __restrict__ sse_trace,
                               long long* __restrict__ chg_trace, double* __restrict__ drift_trace,
                               Ctl* __restrict__ ctl, float tol)
{
    if (ctl->done) return;
    const int t = ctl->iter;
    const double sse = __dmul_rn((double)st->sse_q, st->sse_inv);
    const unsigned long long chg = st->chg;
    const double md = __longlong_as_double((long long)st->md_bits);
    if (sse_trace) sse_trace[t] = sse;
    if (chg_trace) chg_trace[t] = (long long)chg;
    if (drift_trace) drift_trace[t] = md;
    ctl->iter = t + 1;
    if (tol >= 0.0f && (md <= (double)tol || (t >= 1 && chg == 0))) ctl->done = 1;
    st->sse_q = 0;
    st->chg = 0;
    st->md_bits = 0;
    st->cmax_bits = 0;
    st->nfb = 0;
}

// s3 of Eq. 1's fixed-point sum (km_kernels.cuh sse_kernel) for the high-d variant (one CTA):
// B = squared diagonal of the points' box united with the centroids' box; the points' box from
// the fixed-point origin o_m = min (qo) and the FP32 midpoint ctr_m = RN(0.5 (lo + hi)), so
// hi_m <= 2 ctr_m - lo_m + 4 ulp(ctr_m) -- available identically on every data-parallel rank.
template <int D>
__global__ void __launch_bounds__(1024)
hd_sse_bound_kernel(const double* __restrict__ qo, const float* __restrict__ ctr, const float* __restrict__ C,
                    int k, long long n, int* __restrict__ s3_out)
{
    __shared__ double s_b[32];
    double b = 0.0;
    for (int m = threadIdx.x; m < D; m += blockDim.x) {
        const double lo0 = qo[m];
        const double cm = (double)ctr[m];
        double lo = lo0, hi = 2.0 * cm - lo0 + 4.0 * fabs(cm) * 0x1p-24 + 0x1p-126;
        for (int j = 0; j < k; ++j) {
            const double v = (double)C[(int64_t)j * D + m];
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
        b += (hi - lo) * (hi - lo);
    }
    unsigned long long dummy = 0;
    block_sum2<1024>(b, dummy);
    if (threadIdx.x == 0) *s3_out = sse_shift(b * (1.0 + 0x1p-30), n);
}

// Eq. 1 of the returned pair (labels, C): warp per point, D_i summed over the lanes in a fixed
// tree (deterministic per point), then added in 128-bit fixed point (order-independent).
template <int D>
__global__ void __launch_bounds__(256)
hd_sse_kernel(const float* __restrict__ P, int64_t n, const int32_t* __restrict__ labels, const float* __restrict__ C,
              const int* __restrict__ s3, unsigned long long* __restrict__ part)
{
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double scale = ldexp(1.0, *s3);
    u128 acc = 0;
    for (int64_t i = w0; i < n; i += nw) {
        const int a = labels[i];
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < D / 32; ++u) {
            const double t = (double)P[i * D + lane + 32 * u] - (double)C[(int64_t)a * D + lane + 32 * u];
            s = fma(t, t, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) add_fix(acc, s, scale);
    }
    acc = block_sum128(acc);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = (unsigned long long)acc;
        part[2 * blockIdx.x + 1] = (unsigned long long)(acc >> 64);
    }
}

}  // namespace hd
}  // namespace km
