// km_tiles.cuh -- the paper's spatial-vector index (Dask-means, arXiv 2412.02244)
// re-designed for the GPU: a flat tree over Morton-sorted points (built once per call, Alg. 1
// line 1):
//   * a TILE is 128 consecutive sorted points owned by one warp (4 per lane): a ball node N
//     with pivot p* = o (tile mean), radius r, |N|, moments and its exact fixed-point sum; a
//     tile whose points straddle a large Morton jump also carries two tight sub-balls;
//   * level-1 nodes group 8 or 16 tiles (km_ctx::st_shift), higher levels kFanout nodes (km_levels.cuh).
// Per iteration (Alg. 1 loop): the inter bound settles tiles and points (Eq. 3-5,
// km_bounds.cuh); every node prunes its parent's candidate list with its ball (Eq. 7-8,
// km_levels.cuh); the assignment kernel (km_tiles_assign.cuh) prunes each listed tile's
// level-1 list with the tile ball(s): one candidate -> the whole tile is assigned in batch
// (Eq. 6, Alg. 1) and moves as N.p*.|N| (exactly, in integers);
// otherwise its points scan the candidates (FP32 + FP64 certification).  Pruning removes only
// centroids that are strictly farther, by a relative margin >> FP64 rounding, for every point
// of the ball, so labels are identical to plain Lloyd's and to KM_MODE_BRUTE.
// This file: tile/index data layouts, the Morton sort helpers, tile geometry, the prune
// threshold, async-copy helpers and the shared-memory layout of the assignment kernel.
#pragma once
#include <cuda_runtime.h>
#include "km_kernels.cuh"
#include "km_assign_fast.cuh"

namespace km {

#ifndef KM_SPLIT_RATIO
#define KM_SPLIT_RATIO 0.3   // sub-balls used when both radii are <= this fraction of the tile radius
#endif
constexpr int kTileThreads = 256;                        // CTA size: 8 independent warps
constexpr int kWarpsPerCta = kTileThreads / 32;
constexpr int kTilePoints = 128;                         // one warp x 4 consecutive points per lane
#ifndef KM_ST_CACHE
#define KM_ST_CACHE 0
#endif
constexpr int kCandCap = 2048;                           // super-tile list capacity
#ifndef KM_WCAP
#define KM_WCAP 64
#endif
constexpr int kWCap = KM_WCAP;                           // per-warp slots for the chunked scan of long candidate lists
constexpr int kMaxPruneRounds = 64;                      // st_prune: k <= 64 * 256
constexpr int kTC = 32;                                  // candidates per tile precomputed by the level-1 prune

struct __align__(16) StGeom {
    float o[3];
    float r;   // max_t (||o_t - o|| + r_t), rounded up: bounds every point of the super-tile
};

struct __align__(16) TileGeom {
    float o[3];   // centre (float), pivot p* of the ball
    float r;      // radius, rounded up: max_i ||p_i - o|| <= r
    int cnt;      // points in the tile
    int pad[3];   // 32 B: one bulk-copy unit
};

struct __align__(16) TileMom {
    double s1[3];                // sum_i (p_i - o)
    double s2;                   // sum_i ||p_i - o||^2
    unsigned long long q[3];     // sum_i qv(p_i): exact fixed-point tile sum
    unsigned long long pad;      // 64 B: one bulk-copy unit
};

// Two sub-balls of a tile split at its largest Morton-key jump (points [0, split) and
// [split, cnt)): a tile whose consecutive sorted points come from two distant regions gets two
// tight balls instead of one huge one (TileGeom.pad[0] = 1 when they are used).
struct __align__(16) TileSub {
    float o1[3];
    float r1;
    float o2[3];
    float r2;
};

struct __align__(16) TileInfo {   // constant per run: one 128 B copy
    TileGeom g;
    TileSub sb;
    TileMom m;
};

// Per-tile inputs of the assignment kernel written each iteration by the index kernels:
// pre by tile_filter_kernel (tiles whose previous labels were all a), ncand / off by the level-1
// prune (tile_cands_warp).  The candidates themselves live in the tile's SoA block of tcand
// ((D + 1) * kTC words: negated coordinates [D][kTC], then the centroid indices [kTC]) when
// ncand <= kTC, else in the overflow pool at off (CRec records; off < 0: pool full, the
// assignment kernel scans the whole level-1 list, a superset).
struct __align__(16) TileAux {
    float4 pre;   // Eq. 4 record of the previous label a: {c_a, lower bound of (cb[a]/2)^2}
    int ncand;
    int off;
    int pad[2];
};

template <int D>
__host__ __device__ constexpr int cand_block_words() { return (D + 1) * kTC; }

struct __align__(16) TileState {
    int lab[4];   // per warp (32 points) of the tile: >= 0 every label of the warp's points; -1 mixed
};

// The tile's label state: a >= 0 iff every label of the tile equals a (all four warp slots agree;
// writers set all four for a whole-tile decision, K1b each live warp's own).
__device__ __forceinline__ int tile_lab(const TileState& s)
{
    return (s.lab[0] >= 0 && s.lab[0] == s.lab[1] && s.lab[0] == s.lab[2] && s.lab[0] == s.lab[3]) ? s.lab[0] : -1;
}
__device__ __forceinline__ void tile_lab_set(TileState* s, int v) { *reinterpret_cast<int4*>(s) = make_int4(v, v, v, v); }

constexpr int kStCache = KM_ST_CACHE;   // per-warp cache of the parent's list (coordinates + index)

__device__ __forceinline__ unsigned int spread_bits2(unsigned int x)   // 15 bits -> every 2nd bit
{
    x &= 0x7fff;
    x = (x | (x << 8)) & 0x00ff00ff;
    x = (x | (x << 4)) & 0x0f0f0f0f;
    x = (x | (x << 2)) & 0x33333333;
    x = (x | (x << 1)) & 0x55555555;
    return x;
}

__device__ __forceinline__ unsigned int spread_bits3(unsigned int x)   // 10 bits -> every 3rd bit
{
    x &= 0x3ff;
    x = (x | (x << 16)) & 0x030000ff;
    x = (x | (x << 8)) & 0x0300f00f;
    x = (x | (x << 4)) & 0x030c30c3;
    x = (x | (x << 2)) & 0x09249249;
    return x;
}

// Bits per coordinate of the Morton key: 2 x 15 (d = 2) and 3 x 10 (d = 3); for n >= 4M, 24-bit
// keys (2 x 12, 3 x 8) = three radix passes instead of four.  Coarser cells cost some tile
// compactness (a slightly slower assignment per iteration) against ~1/4 of the sort: measured
// -4 % per run at config 4 (20 iterations) and -3 % at config 5 (10 iterations); n = 1M sets
// keep the fine keys (+3 % at config 3 otherwise).
#ifndef KM_MORTON2_LARGE
#define KM_MORTON2_LARGE 12   // 24-bit keys for large 2-D sets: config 5 -3 % per 10-iteration run
#endif
#ifndef KM_MORTON3_LARGE
#define KM_MORTON3_LARGE 8   // bits per coordinate of 3-D keys when n >= 4M (3 x 8 = 24: three radix passes)
#endif
inline int morton_bits(int d, int64_t n)
{
    return d == 2 ? (n >= (4ll << 20) ? KM_MORTON2_LARGE : 15) : (n >= (4ll << 20) ? KM_MORTON3_LARGE : 10);
}

// Morton key of every point on a grid of 2^(D*B) cells over the bounding box (Quant.o = min).
template <int D>
__global__ void __launch_bounds__(256)
morton_kernel(const float* __restrict__ pts, int64_t n, const Quant* __restrict__ quant, int B,
              unsigned int* __restrict__ keys, unsigned int* __restrict__ idx)
{
    const Quant q = *quant;
    float lo[D], sc[D];
#pragma unroll
    for (int m = 0; m < D; ++m) {
        lo[m] = (float)q.o[m];
        float ext = q.hi[m] - lo[m];
        sc[m] = ext > 0.f ? (float)((1 << B) - 1) / ext : 0.f;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned int key = 0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            float g = (pts[i * D + m] - lo[m]) * sc[m];
            unsigned int u = (unsigned int)fminf(fmaxf(g, 0.f), (float)((1 << B) - 1));   // B <= 15 (2-D) / 10 (3-D)
            key |= (D == 2 ? spread_bits2(u) : spread_bits3(u)) << m;
        }
        keys[i] = key;
        idx[i] = (unsigned int)i;
    }
}

// Labels back to input order (once per run): out[idx[i]] = lab_sorted[i] for the i whose
// destination lies in [w0, w1).  The caller sweeps windows small enough to stay resident in
// the 126 MB L2, so the random 4-B stores merge in L2 and reach HBM as whole sectors
// (one pass over 400 MB of labels at config 5 would be a random read-modify-write per label).
// SSE (the first window's launch): Eq. 1 of the returned pair over the sorted points, fused
// into the same pass (sse_kernel's arithmetic: 128-bit fixed-point partials per CTA).
template <int D, bool SSE>
__global__ void __launch_bounds__(256)
scatter_labels_kernel(const int32_t* __restrict__ lab_sorted, int64_t n, const unsigned int* __restrict__ idx,
                      int32_t* __restrict__ out, unsigned int w0, unsigned int w1, const float* __restrict__ ps,
                      const float* __restrict__ C, const int* __restrict__ s3, unsigned long long* __restrict__ part)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double scale = SSE ? ldexp(1.0, *s3) : 0.0;
    u128 acc = 0;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
        unsigned int d[4];
        int32_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool ok = i0 + u * stride < n;
            d[u] = ok ? idx[i0 + u * stride] : 0xffffffffu;
            v[u] = ok ? lab_sorted[i0 + u * stride] : 0;
        }
        if (SSE) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (i0 + u * stride < n) {
                    const int64_t i = i0 + u * stride;
                    double sd = 0.0;
#pragma unroll
                    for (int m = 0; m < D; ++m) {
                        const double tt = __dsub_rn((double)ps[i * D + m], (double)C[(int64_t)v[u] * D + m]);
                        sd = __dadd_rn(sd, __dmul_rn(tt, tt));
                    }
                    add_fix(acc, sd, scale);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (d[u] >= w0 && d[u] < w1) out[d[u]] = v[u];
    }
    if (SSE) {
        acc = block_sum128(acc);
        if (threadIdx.x == 0) {
            part[2 * blockIdx.x] = (unsigned long long)acc;
            part[2 * blockIdx.x + 1] = (unsigned long long)(acc >> 64);
        }
    }
}

// More than one destination window (n > the window): the first pass (which reads every label,
// its destination and, for Eq. 1, every point anyway) stores window 0's labels and appends every
// other (destination, label) pair to its window's bucket -- bucket w holds exactly the window's
// size, so its region is fixed; a CTA reserves its share per window with one atomic after
// counting in shared memory -- and each later window reads only its own bucket
// (scatter_window_kernel) instead of all n pairs again.  Results are the same: every label goes
// to its own destination.
constexpr int kScatterMaxWin = 64;
template <int D, bool SSE>
__global__ void __launch_bounds__(256)
scatter_bucket_kernel(const int32_t* __restrict__ lab_sorted, int64_t n, const unsigned int* __restrict__ idx,
                      int32_t* __restrict__ out, unsigned int win, int nwin, const float* __restrict__ ps,
                      const float* __restrict__ C, const int* __restrict__ s3, unsigned long long* __restrict__ part,
                      unsigned long long* __restrict__ bucket, unsigned long long* __restrict__ cursor)
{
    __shared__ unsigned int s_cnt[kScatterMaxWin];
    __shared__ unsigned long long s_base[kScatterMaxWin];
    const double scale = SSE ? ldexp(1.0, *s3) : 0.0;
    u128 acc = 0;
    constexpr int U = 4;
    const int64_t chunk = (int64_t)blockDim.x * U;
    for (int64_t c0 = (int64_t)blockIdx.x * chunk; c0 < n; c0 += (int64_t)gridDim.x * chunk) {
        for (int w = threadIdx.x; w < nwin; w += blockDim.x) s_cnt[w] = 0u;
        __syncthreads();
        unsigned int d[U];
        int32_t v[U];
        unsigned int slot[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = c0 + (int64_t)u * blockDim.x + threadIdx.x;
            const bool ok = i < n;
            d[u] = ok ? idx[i] : 0xffffffffu;
            v[u] = ok ? lab_sorted[i] : 0;
            if (SSE && ok) {
                double sd = 0.0;
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    const double tt = __dsub_rn((double)ps[i * D + m], (double)C[(int64_t)v[u] * D + m]);
                    sd = __dadd_rn(sd, __dmul_rn(tt, tt));
                }
                add_fix(acc, sd, scale);
            }
            slot[u] = 0xffffffffu;
            if (ok) {
                if (d[u] < win) out[d[u]] = v[u];
                else slot[u] = atomicAdd(&s_cnt[d[u] / win], 1u);
            }
        }
        __syncthreads();
        for (int w = 1 + threadIdx.x; w < nwin; w += blockDim.x)
            s_base[w] = s_cnt[w] ? atomicAdd(&cursor[w], (unsigned long long)s_cnt[w]) : 0ull;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (slot[u] != 0xffffffffu) {
                const int w = (int)(d[u] / win);
                // bucket w occupies [(w - 1) win, min(n, (w + 1) win) - win)
                bucket[(int64_t)(w - 1) * win + s_base[w] + slot[u]] = ((unsigned long long)d[u] << 32) | (unsigned int)v[u];
            }
        __syncthreads();
    }
    if (SSE) {
        acc = block_sum128(acc);
        if (threadIdx.x == 0) {
            part[2 * blockIdx.x] = (unsigned long long)acc;
            part[2 * blockIdx.x + 1] = (unsigned long long)(acc >> 64);
        }
    }
}

__global__ void __launch_bounds__(256)
scatter_window_kernel(const unsigned long long* __restrict__ bucket, int64_t cnt, int32_t* __restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long e = bucket[i];
        out[e >> 32] = (int32_t)(unsigned int)e;
    }
}

template <typename T>
__device__ __forceinline__ T warp_allsum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-tile geometry and moments (once per run; points are fixed).  One warp per tile; each
// lane holds its 4 consecutive points in registers (one load each).  Any centre gives a valid
// ball as long as r bounds the distances to it, so the centres (tile mean, and the means of
// the two halves split at the largest Morton-key jump) are FP32 sums; r, the moments
// s1 = sum (p - o), s2 = sum ||p - o||^2 (FP64) and the exact tile sums are relative to them.
// GATHER: the tile's points are first gathered from the caller's array through the sort's
// permutation and written to the sorted copy ps (fused gather: ps is not read back).  The level-0
// balls (StGeom) of the index are written beside the TileInfo.
template <int D, bool GATHER>
__global__ void __launch_bounds__(256)
tile_geom_kernel(const float* __restrict__ pin, const unsigned int* __restrict__ perm, float* __restrict__ ps,
                 int64_t n, int ntiles, const Quant* __restrict__ quant, const unsigned int* __restrict__ keys,
                 TileInfo* __restrict__ info, StGeom* __restrict__ balls)
{
    const Quant q = *quant;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int t = gw; t < ntiles; t += nwarps) {
        const int64_t b = (int64_t)t * kTilePoints;
        const int cnt = (int)min((int64_t)kTilePoints, n - b);
        const int nv = max(0, min(4, cnt - 4 * lane));
        float v[4][D];
        unsigned kk[4];
        if (GATHER) {
            unsigned src[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) src[r] = r < nv ? perm[b + 4 * lane + r] : 0u;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int m = 0; m < D; ++m) v[r][m] = r < nv ? __ldg(pin + (int64_t)src[r] * D + m) : 0.f;
            float* dst = ps + (b + 4 * lane) * D;
            if (nv == 4) {   // 4 D floats = D float4s, 16-B aligned
                float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
                for (int u = 0; u < D; ++u) {
                    const int e0 = 4 * u;
                    d4[u] = make_float4(v[e0 / D][e0 % D], v[(e0 + 1) / D][(e0 + 1) % D], v[(e0 + 2) / D][(e0 + 2) % D],
                                        v[(e0 + 3) / D][(e0 + 3) % D]);
                }
            } else {
                for (int r = 0; r < nv; ++r)
#pragma unroll
                    for (int m = 0; m < D; ++m) dst[r * D + m] = v[r][m];
            }
        } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int m = 0; m < D; ++m) v[r][m] = r < nv ? ps[(b + 4 * lane + r) * D + m] : 0.f;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) kk[r] = r < nv ? keys[b + 4 * lane + r] : 0u;
        // split at the largest Morton jump: highest differing key bit between consecutive points
        const unsigned kprev = __shfl_up_sync(full, kk[3], 1);
        int best = -1;   // (bit << 8) | (255 - i): largest bit, then the first i
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = 4 * lane + r;
            if (r < nv && i >= 1) {
                const unsigned x = kk[r] ^ (r ? kk[r - 1] : kprev);
                const int bit = x ? 31 - __clz(x) : 0;
                best = max(best, (bit << 8) | (255 - i));
            }
        }
        best = __reduce_max_sync(full, best);
        const int split = best < 0 ? 0 : 255 - (best & 255);   // 0: single point
        float o[D], o1[D], o2[D];
#pragma unroll
        for (int m = 0; m < D; ++m) {
            float st = 0.f, s1p = 0.f;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                st += v[r][m];   // zeros past the end
                if (4 * lane + r < split) s1p += v[r][m];
            }
            st = warp_allsum(st);
            s1p = warp_allsum(s1p);
            o[m] = st / (float)cnt;
            o1[m] = split > 0 ? s1p / (float)split : o[m];
            o2[m] = split > 0 ? (st - s1p) / (float)(cnt - split) : o[m];
        }
        double s1[D], s2 = 0.0;
        float rmax = 0.f, rs1 = 0.f, rs2 = 0.f;   // squared radii (rounded up), square roots at the end
        unsigned long long qs[D];
#pragma unroll
        for (int m = 0; m < D; ++m) { s1[m] = 0.0; qs[m] = 0ull; }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r < nv) {
                double d2 = 0.0, e2 = 0.0;
                const bool h1 = 4 * lane + r < split;
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    const double t1 = (double)v[r][m] - (double)o[m];
                    const double t2 = (double)v[r][m] - (double)(h1 ? o1[m] : o2[m]);
                    s1[m] += t1;
                    d2 += t1 * t1;
                    e2 += t2 * t2;
                    qs[m] += (unsigned long long)__double2ll_rn(
                        __dmul_rn(__dsub_rn((double)v[r][m], q.o[m]), q.scale[m]));
                }
                s2 += d2;
                rmax = fmaxf(rmax, __double2float_ru(d2));
                if (h1) rs1 = fmaxf(rs1, __double2float_ru(e2));
                else rs2 = fmaxf(rs2, __double2float_ru(e2));
            }
        }
#pragma unroll
        for (int m = 0; m < D; ++m) { s1[m] = warp_allsum(s1[m]); qs[m] = warp_allsum(qs[m]); }
        s2 = warp_allsum(s2);
        // non-negative floats order like their bits: one REDUX each; sqrt rounded up keeps the bound
        rmax = __fsqrt_ru(__uint_as_float(__reduce_max_sync(full, __float_as_uint(rmax))));
        rs1 = __fsqrt_ru(__uint_as_float(__reduce_max_sync(full, __float_as_uint(rs1))));
        rs2 = __fsqrt_ru(__uint_as_float(__reduce_max_sync(full, __float_as_uint(rs2))));
        if (lane == 0) {
            TileGeom g;
#pragma unroll
            for (int m = 0; m < 3; ++m) g.o[m] = m < D ? o[m] : 0.f;
            // rounded up (above), plus a relative margin for the FP64 rounding of the distances
            g.r = __fmul_ru(rmax, 1.0f + 0x1p-20f);
            g.cnt = cnt;
            // the sub-balls are used when they are much tighter than the tile ball
            g.pad[0] = split > 0 && fmaxf(rs1, rs2) <= (float)KM_SPLIT_RATIO * rmax ? 1 : 0;
            g.pad[1] = split;
            g.pad[2] = 0;
            info[t].g = g;
            TileSub sb;
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                sb.o1[m] = m < D ? o1[m] : 0.f;
                sb.o2[m] = m < D ? o2[m] : 0.f;
            }
            sb.r1 = __fmul_ru(rs1, 1.0f + 0x1p-20f);
            sb.r2 = __fmul_ru(rs2, 1.0f + 0x1p-20f);
            info[t].sb = sb;
            TileMom mm;
#pragma unroll
            for (int m = 0; m < 3; ++m) { mm.s1[m] = m < D ? s1[m] : 0.0; mm.q[m] = m < D ? qs[m] : 0ull; }
            mm.s2 = s2;
            mm.pad = 0ull;
            info[t].m = mm;
            StGeom bg;
            bg.o[0] = g.o[0]; bg.o[1] = g.o[1]; bg.o[2] = g.o[2];
            bg.r = g.r;
            balls[t] = bg;
        }
    }
}

// Conservative inclusion threshold for a ball (o, r): include j iff delta_j^2 <= T2 where
// T = (sqrt(min delta^2)(1 + 2^-16) + 2r)(1 + 2^-14).  sqrt.approx (rel. error < 2^-21) is
// covered by the 2^-16 factor; every later RN rounding (<= 2^-24 each) and the FP32
// rounding of delta (< 3 * 2^-24) by the 2^-14 margins.
// KM_PRUNE_DIAM exists only so that a fault-injection build (-DKM_PRUNE_DIAM=1.0f: the ball's
// radius instead of its diameter, i.e. a wrong Eq. 8) can show the full-size parity tests fail.
#ifndef KM_PRUNE_DIAM
#define KM_PRUNE_DIAM 2.0f
#endif
__device__ __forceinline__ float prune_thr2(float dmin2, float r)
{
    float s;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(dmin2));
    const float mg = 1.0f + 0x1p-14f;
    const float T = (s * (1.0f + 0x1p-16f) + KM_PRUNE_DIAM * r) * mg;
    return T * T * mg;
}

template <int D>
__device__ __forceinline__ float delta2(const float (&o)[3], const float* __restrict__ C, int j)
{
    float s = 0.f;
#pragma unroll
    for (int m = 0; m < D; ++m) { const float t1 = __fsub_rn(o[m], C[(int64_t)j * D + m]); s = __fmaf_rn(t1, t1, s); }
    return s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// One warp's shared memory: double-buffered tile (ball + moments, label state, the per-tile
// inputs of this iteration and its candidate block, points, previous labels) and the chunk
// buffer of the overflow scan.
template <int D>
struct WarpSmem {
    struct Buf {
        TileInfo info;
        TileState st;
        TileAux aux;
        float cand[cand_block_words<D>()];
        float pts[kTilePoints * D];
        int lab[kTilePoints];
    } buf[2];
    float cnc[D][kWCap];          // overflow scan: candidate chunk (negated)
    unsigned long long mbar[2];   // K1t bulk staging: completion barrier of each buffer
};


// FP32 / FP64 distances against a centroid read from global memory (same operation order
// as the shared-memory versions: p + (-c) == p - c exactly).
template <int D>
__device__ __forceinline__ float dist32g(const Pt<D>& p, const float* __restrict__ C, int j)
{
    float t = __fsub_rn(p.v[0], C[(int64_t)j * D]);
    float s = __fmul_rn(t, t);
#pragma unroll
    for (int m = 1; m < D; ++m) {
        t = __fsub_rn(p.v[m], C[(int64_t)j * D + m]);
        s = __fmaf_rn(t, t, s);
    }
    return s;
}

// Exact FP64 argmin over entries [e0, e1) of a centroid list (list == nullptr: identity),
// lowest j on ties whatever the list order.
template <int D>
__device__ __noinline__ int exact_scan_list(Pt<D> p, const float* __restrict__ C, const int* list, int e0, int e1)
{
    double best = INFINITY;
    int a = list ? list[e0] : e0;
    for (int e = e0; e < e1; ++e) {
        const int j = list ? list[e] : e;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double t = __dsub_rn((double)p.v[m], (double)C[(int64_t)j * D + m]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        if (s < best || (s == best && j < a)) { best = s; a = j; }   // ties: lowest j, in any list order
    }
    return a;
}

// Packed group scan of 4 points over slots [0, nslots) of the warp's SoA candidate buffer.
template <int D>
__device__ __forceinline__ void scan_slots(const Pt<D> (&p)[4], const float (*cnc)[kWCap], int nslots, int gbase,
                                           float (&m1)[4], float (&m2)[4], int (&b1)[4])
{
    for (int gi = 0; gi < (nslots >> 2); ++gi) {
        float4 c[D];
#pragma unroll
        for (int m = 0; m < D; ++m) c[m] = reinterpret_cast<const float4*>(cnc[m])[gi];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            float2 s0 = pair2<D>(p[r], c, false);
            float2 s1 = pair2<D>(p[r], c, true);
            float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
            bool lt = v < m1[r];
            m2[r] = fmaxf(m1[r], fminf(m2[r], v));
            m1[r] = fminf(m1[r], v);
            b1[r] = lt ? gbase + gi : b1[r];
        }
    }
}

// Run-length + warp aggregation of the fixed-point sums of a lane's 4 consecutive points.
// A warp whose points share one label sums with one butterfly and one lane issues the
// REDs; otherwise every lane issues one RED group per label run of its own points.
template <int D>
__device__ __forceinline__ void accumulate_runs(const Pt<D> (&p)[4], const int (&a)[4], int nvalid, bool warp_uni,
                                                int L, const Quant& q, unsigned long long* __restrict__ acc_sum,
                                                unsigned int* __restrict__ acc_cnt)
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long qv[4][D];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int m = 0; m < D; ++m)
            qv[r][m] = r < nvalid ? (unsigned long long)__double2ll_rn(
                                        __dmul_rn(__dsub_rn((double)p[r].v[m], q.o[m]), q.scale[m]))
                                  : 0ull;
    if (warp_uni) {
#pragma unroll
        for (int m = 0; m < D; ++m) {
            unsigned long long s = warp_allsum(qv[0][m] + qv[1][m] + qv[2][m] + qv[3][m]);
            if (lane == 0) atomicAdd(&acc_sum[(int64_t)L * D + m], s);
        }
        const int c = (int)__reduce_add_sync(full, (unsigned)nvalid);
        if (lane == 0) atomicAdd(&acc_cnt[L], (unsigned int)c);
        return;
    }
    unsigned long long s[D];
#pragma unroll
    for (int m = 0; m < D; ++m) s[m] = 0ull;
    int cur = a[0], cnt = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (r < nvalid) {
            if (cnt > 0 && a[r] != cur) {
#pragma unroll
                for (int m = 0; m < D; ++m) { atomicAdd(&acc_sum[(int64_t)cur * D + m], s[m]); s[m] = 0ull; }
                atomicAdd(&acc_cnt[cur], (unsigned int)cnt);
                cnt = 0;
            }
            cur = a[r];
#pragma unroll
            for (int m = 0; m < D; ++m) s[m] += qv[r][m];
            ++cnt;
        }
    }
    if (cnt > 0) {
#pragma unroll
        for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)cur * D + m], s[m]);
        atomicAdd(&acc_cnt[cur], (unsigned int)cnt);
    }
}

}  // namespace km
