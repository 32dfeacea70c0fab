// km_tiles.cuh -- the paper's batch assignment (Dask-means, arXiv 2412.02244) re-designed
// for the GPU: Morton-sorted point tiles act as the ball nodes N of the spatial-vector
// index (pivot p* = tile centre o, radius r, |N| = tile size), and each CTA
// prunes the centroid set for its tile before any point is touched.
//
//   * Candidate pruning (Eq. 5-8, with N = tile): every point p of the tile
//     satisfies | ||p - c_j|| - ||o - c_j|| | <= r, so centroid j can be nearest to some
//     point only if  delta_j <= min_l delta_l + 2r  (delta_j = ||o - c_j||).  All other
//     centroids are pruned -- exactly the gap test "d2 - d1 > 2 N.r" (Eq. 6) generalised
//     to a candidate list, with FP margins that keep it conservative.
//   * Batch assignment (Alg. 1): if one candidate remains, the whole tile
//     goes to it; sums use the tile's precomputed fixed-point sum ("p can be replaced by
//     N.p*.|N| if a node N moves", P:L412 -- here exactly, in integers), the SSE uses the
//     tile's moments, and labels are rewritten only if the tile's label changed.
//   * Otherwise every point scans only the candidates (FP32 packed scan + FP64
//     certification, as in the brute-force kernel) -- "Assign(N', ...)" per point.
// Labels are identical to plain Lloyd's: pruning only removes centroids that are
// strictly farther (by a relative margin >> FP64 rounding) for every point of the tile.
#pragma once
#include <cuda_runtime.h>
#include "km_kernels.cuh"
#include "km_assign_fast.cuh"

namespace km {

constexpr int kTileThreads = 256;
constexpr int kTileP = 4;                                // points per thread
constexpr int kTilePoints = kTileThreads * kTileP;       // 1024 points per tile
constexpr int kCandCap = 2048;                           // candidate slots held in shared memory

struct __align__(16) TileGeom {
    float o[3];   // centre (float), pivot p* of the ball
    float r;      // radius, rounded up: max_i ||p_i - o|| <= r
    int cnt;      // points in the tile
    int pad[3];   // 32 B: one bulk copy unit
};

struct TileMom {
    double s1[3];                // sum_i (p_i - o)
    double s2;                   // sum_i ||p_i - o||^2
    unsigned long long q[3];     // sum_i qv(p_i): exact fixed-point tile sum
};

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

// Morton key of every point on a 2^30-cell grid over the bounding box (Quant.o = min).
template <int D>
__global__ void __launch_bounds__(256)
morton_kernel(const float* __restrict__ pts, int64_t n, const Quant* __restrict__ quant,
              unsigned int* __restrict__ keys, unsigned int* __restrict__ idx)
{
    constexpr int B = D == 2 ? 15 : 10;
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
            unsigned int u = (unsigned int)fminf(fmaxf(g, 0.f), (float)((1 << B) - 1));
            key |= (D == 2 ? spread_bits2(u) : spread_bits3(u)) << m;
        }
        keys[i] = key;
        idx[i] = (unsigned int)i;
    }
}

template <int D>
__global__ void __launch_bounds__(256)
gather_kernel(const float* __restrict__ pts, int64_t n, const unsigned int* __restrict__ idx, float* __restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = idx[i];
#pragma unroll
        for (int m = 0; m < D; ++m) out[i * D + m] = pts[s * D + m];
    }
}

__global__ void __launch_bounds__(256)
scatter_labels_kernel(const int32_t* __restrict__ lab_sorted, int64_t n, const unsigned int* __restrict__ idx,
                      int32_t* __restrict__ out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[idx[i]] = lab_sorted[i];
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* scratch /* >= 32 */)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) scratch[w] = v;
    __syncthreads();
    v = scratch[0];
    for (int i = 1; i < nw; ++i) v = op(v, scratch[i]);
    return v;
}

// Per-tile geometry and moments (once per run; points are fixed).  One CTA per tile.
template <int D>
__global__ void __launch_bounds__(kTileThreads)
tile_geom_kernel(const float* __restrict__ ps, int64_t n, int ntiles, const Quant* __restrict__ quant,
                 TileGeom* __restrict__ geom, TileMom* __restrict__ mom)
{
    __shared__ double sd[32];
    __shared__ unsigned long long su[32];
    __shared__ float sf[32];
    const Quant q = *quant;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t b = (int64_t)t * kTilePoints;
        const int cnt = (int)min((int64_t)kTilePoints, n - b);
        // mean (FP64) -> centre o (float)
        float o[D];
#pragma unroll
        for (int m = 0; m < D; ++m) {
            double s = 0.0;
            for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += (double)ps[(b + i) * D + m];
            s = block_reduce(s, [](double x, double y) { return x + y; }, sd);
            o[m] = (float)(s / cnt);
        }
        double s1[D], s2 = 0.0, rmax = 0.0;
        unsigned long long qs[D];
#pragma unroll
        for (int m = 0; m < D; ++m) { s1[m] = 0.0; qs[m] = 0ull; }
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            double d2 = 0.0;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const float pv = ps[(b + i) * D + m];
                const double t1 = (double)pv - (double)o[m];
                s1[m] += t1;
                d2 += t1 * t1;
                qs[m] += (unsigned long long)__double2ll_rn(__dmul_rn(__dsub_rn((double)pv, q.o[m]), q.scale[m]));
            }
            s2 += d2;
            rmax = fmax(rmax, sqrt(d2));
        }
#pragma unroll
        for (int m = 0; m < D; ++m) {
            s1[m] = block_reduce(s1[m], [](double x, double y) { return x + y; }, sd);
            qs[m] = block_reduce(qs[m], [](unsigned long long x, unsigned long long y) { return x + y; }, su);
        }
        s2 = block_reduce(s2, [](double x, double y) { return x + y; }, sd);
        rmax = block_reduce(rmax, [](double x, double y) { return fmax(x, y); }, sd);
        (void)sf;
        if (threadIdx.x == 0) {
            TileGeom g;
#pragma unroll
            for (int m = 0; m < 3; ++m) g.o[m] = m < D ? o[m] : 0.f;
            // round up, plus a relative margin for the FP64 rounding of the distances themselves
            g.r = __fmul_ru(__double2float_ru(rmax), 1.0f + 0x1p-20f);
            g.cnt = cnt;
            geom[t] = g;
            TileMom mm;
#pragma unroll
            for (int m = 0; m < 3; ++m) { mm.s1[m] = m < D ? s1[m] : 0.0; mm.q[m] = m < D ? qs[m] : 0ull; }
            mm.s2 = s2;
            mom[t] = mm;
        }
        __syncthreads();
    }
}

// Warp-aggregated fixed-point accumulation: lanes with equal labels are summed with a
// butterfly and one lane issues the REDs (sorted tiles make warps label-coherent).
template <int D>
__device__ __forceinline__ void warp_accumulate(bool valid, int a, const float (&p)[D], const Quant& q,
                                                unsigned long long* __restrict__ acc_sum,
                                                unsigned int* __restrict__ acc_cnt)
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long qv[D];
#pragma unroll
    for (int m = 0; m < D; ++m)
        qv[m] = valid ? (unsigned long long)__double2ll_rn(__dmul_rn(__dsub_rn((double)p[m], q.o[m]), q.scale[m])) : 0ull;
    unsigned act = __ballot_sync(full, valid);
    while (act) {
        const int leader = __ffs(act) - 1;
        const int L = __shfl_sync(full, a, leader);
        const bool mine = valid && a == L;
        const unsigned mask = __ballot_sync(full, mine);
#pragma unroll
        for (int m = 0; m < D; ++m) {
            unsigned long long s = mine ? qv[m] : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(full, s, o);
            if (lane == leader) atomicAdd(&acc_sum[(int64_t)L * D + m], s);
        }
        if (lane == leader) atomicAdd(&acc_cnt[L], (unsigned int)__popc(mask));
        act &= ~mask;
    }
}

// Exact FP64 argmin over candidate slots [s0, s1) (ascending slot == ascending j).
template <int D>
__device__ __noinline__ int exact_scan_slots(Pt<D> p, const float* __restrict__ cnc, int cap,
                                             const int* __restrict__ cj, int s0, int s1)
{
    double best = INFINITY;
    int a = s0;
    for (int s = s0; s < s1; ++s) {
        double v = dist64n<D>(p, cnc, cap, s);
        if (v < best) { best = v; a = s; }
    }
    return cj[a];
}

// ---- TMA bulk copies (cp.async.bulk, global -> shared, completion on an mbarrier) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Tile staging buffer: geometry, points (float, [cnt][D]) and previous labels.
template <int D>
struct TileBuf {
    TileGeom g;
    float pts[kTilePoints * D];
    int lab[kTilePoints];
};

// Issue the bulk copies of tile t into buffer b (one elected thread).
template <int D>
__device__ __forceinline__ void stage_tile(TileBuf<D>* buf, unsigned long long* bar, int t, const TileGeom* geom,
                                           const float* ps, const int32_t* labels, int64_t n, bool want_labels)
{
    const int64_t base = (int64_t)t * kTilePoints;
    const int cnt = (int)min((int64_t)kTilePoints, n - base);
    const uint32_t pb = ((uint32_t)cnt * D * 4 + 15) & ~15u;   // sources are padded to 16 B in HBM
    const uint32_t lb = want_labels ? (((uint32_t)cnt * 4 + 15) & ~15u) : 0u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)sizeof(TileGeom) + pb + lb);
    bulk_g2s(&buf->g, geom + t, (uint32_t)sizeof(TileGeom), bar);
    bulk_g2s(buf->pts, ps + base * D, pb, bar);
    if (want_labels) bulk_g2s(buf->lab, labels + base, lb, bar);
}

// K1t: tile-pruned assignment + fused update.  Persistent CTAs, tile t = blockIdx.x + i*gridDim.x;
// the next tile's points/labels/geometry are bulk-copied into shared memory (double buffer)
// while the current tile is pruned and scanned.
template <int D>
__global__ void __launch_bounds__(kTileThreads, 2)
assign_tiles_kernel(const float* __restrict__ ps, int64_t n, int ntiles, const TileGeom* __restrict__ geom,
                    const TileMom* __restrict__ mom, int* __restrict__ tile_lab, const float* __restrict__ C, int k,
                    int kpad, int32_t* __restrict__ labels, int first, double* __restrict__ sse_part,
                    unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                    unsigned int* __restrict__ acc_cnt, const Quant* __restrict__ quant, const Ctl* __restrict__ ctl,
                    unsigned long long* __restrict__ stats)
{
    if (ctl && ctl->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileBuf<D>* tb = reinterpret_cast<TileBuf<D>*>(smem_raw);             // [2]
    float* nc = reinterpret_cast<float*>(smem_raw + 2 * sizeof(TileBuf<D>));  // [D][kpad]  negated centroids
    float* cnc = nc + D * kpad;                                            // [D][kCandCap] negated candidates
    int* cj = reinterpret_cast<int*>(cnc + D * kCandCap);                 // [kCandCap] candidate -> centroid
    __shared__ unsigned long long bars[2];
    __shared__ int s_scan[32];
    __shared__ float s_min[32];
    __shared__ int s_wlab[32];

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool want_labels = !first;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < ntiles) stage_tile<D>(&tb[0], &bars[0], blockIdx.x, geom, ps, labels, n, want_labels);
    for (int j = threadIdx.x; j < kpad; j += blockDim.x) {
#pragma unroll
        for (int m = 0; m < D; ++m) nc[m * kpad + j] = j < k ? -C[(int64_t)j * D + m] : -INFINITY;
    }
    __syncthreads();
    const Quant q = *quant;
    const int per = (k + blockDim.x - 1) / blockDim.x;   // contiguous centroid range per thread
    const int jb = min(k, threadIdx.x * per), je = min(k, jb + per);

    double sse = 0.0;
    unsigned long long chg = 0, st_pairs = 0, st_pts = 0, st_batch = 0;
    int prev_t = -1;        // tile whose label state is pending in s_wlab
    uint32_t phase[2] = {0u, 0u};

    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        // prefetch the next tile into the other buffer (freed by the barrier that ended the last tile)
        const int tn = t + gridDim.x;
        if (threadIdx.x == 0 && tn < ntiles) stage_tile<D>(&tb[b ^ 1], &bars[b ^ 1], tn, geom, ps, labels, n, want_labels);
        // finish the previous tile's label state (s_wlab written before the last barrier)
        if (threadIdx.x == 0 && prev_t >= 0) {
            int L = -2;
            bool ok = true;
            for (int i = 0; i < nw; ++i) {
                const int v = s_wlab[i];
                if (v == -2) continue;
                if (v < 0 || (L >= 0 && v != L)) { ok = false; break; }
                L = v;
            }
            tile_lab[prev_t] = ok && L >= 0 ? L : -1;
        }
        prev_t = -1;
        mbar_wait(&bars[b], phase[b]);
        phase[b] ^= 1u;
        const TileBuf<D>& B = tb[b];
        const TileGeom g = B.g;
        const int64_t base = (int64_t)t * kTilePoints;

        // --- prune: delta_j^2 = ||o - c_j||^2; include j iff delta_j <= delta_min + 2r ----------
        float dmin2 = INFINITY;
        for (int j = jb; j < je; ++j) {
            float s = 0.f;
#pragma unroll
            for (int m = 0; m < D; ++m) { float t1 = g.o[m] + nc[m * kpad + j]; s = __fmaf_rn(t1, t1, s); }
            dmin2 = fminf(dmin2, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dmin2 = fminf(dmin2, __shfl_xor_sync(0xffffffffu, dmin2, o));
        if (lane == 0) s_min[w] = dmin2;
        __syncthreads();
        dmin2 = s_min[0];
        for (int i = 1; i < nw; ++i) dmin2 = fminf(dmin2, s_min[i]);
        // conservative threshold: margin 2^-14 >> the FP32 rounding of delta
        const float mg = 1.0f + 0x1p-14f;
        const float T = __fmul_ru(__fadd_ru(__fsqrt_ru(dmin2), __fmul_ru(2.0f, g.r)), mg);
        const float T2 = __fmul_ru(__fmul_ru(T, T), mg);
        int cnt = 0;
        for (int j = jb; j < je; ++j) {
            float s = 0.f;
#pragma unroll
            for (int m = 0; m < D; ++m) { float t1 = g.o[m] + nc[m * kpad + j]; s = __fmaf_rn(t1, t1, s); }
            cnt += (s <= T2);
        }
        int x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
        if (lane == 31) s_scan[w] = x;
        __syncthreads();
        int wofs = 0, ncand = 0;
        for (int i = 0; i < nw; ++i) { const int v = s_scan[i]; wofs += i < w ? v : 0; ncand += v; }
        const bool overflow = ncand > kCandCap;
        if (!overflow) {
            int off = wofs + x - cnt;
            for (int j = jb; j < je; ++j) {
                float s = 0.f;
#pragma unroll
                for (int m = 0; m < D; ++m) { float t1 = g.o[m] + nc[m * kpad + j]; s = __fmaf_rn(t1, t1, s); }
                if (s <= T2) {
#pragma unroll
                    for (int m = 0; m < D; ++m) cnc[m * kCandCap + off] = nc[m * kpad + j];
                    cj[off] = j;
                    ++off;
                }
            }
            const int padded = (ncand + 3) & ~3;
            if (threadIdx.x < padded - ncand) {
                const int s = ncand + threadIdx.x;
#pragma unroll
                for (int m = 0; m < D; ++m) cnc[m * kCandCap + s] = -INFINITY;
                cj[s] = 0x7fffffff;
            }
        }
        __syncthreads();

        if (ncand == 1) {
            // --- batch assignment of the whole tile (Eq. 6 / Alg. 1) ---------
            const int cstar = cj[0];
            const int prev = tile_lab[t];
            int changed = 0;
            if (first || prev != cstar) {
                if (first || prev >= 0) {
                    changed = threadIdx.x == 0 ? g.cnt : 0;
                    for (int i = threadIdx.x; i < g.cnt; i += blockDim.x) labels[base + i] = cstar;
                } else {
                    for (int i = threadIdx.x; i < g.cnt; i += blockDim.x) {
                        changed += B.lab[i] != cstar;
                        labels[base + i] = cstar;
                    }
                }
            }
            chg += (unsigned long long)changed;
            if (threadIdx.x == 0) {
                const TileMom mm = mom[t];
                double dot = 0.0, oc2 = 0.0;
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    const double oc = (double)g.o[m] + (double)nc[m * kpad + cstar];   // o - c
                    dot += oc * mm.s1[m];
                    oc2 += oc * oc;
                }
                sse += mm.s2 + 2.0 * dot + (double)g.cnt * oc2;
#pragma unroll
                for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)cstar * D + m], mm.q[m]);
                atomicAdd(&acc_cnt[cstar], (unsigned int)g.cnt);
                tile_lab[t] = cstar;
                st_batch += 1;
            }
        } else {
            // --- per-point scan over the candidates (or all k on overflow) --------------
            const float* sb = overflow ? nc : cnc;
            const int stride = overflow ? kpad : kCandCap;
            const int nslots = overflow ? kpad : ((ncand + 3) & ~3);
            const int nreal = overflow ? k : ncand;
            const float4* sb4 = reinterpret_cast<const float4*>(sb);
            const int kq = stride >> 2;
            Pt<D> p[kTileP];
            float m1[kTileP], m2[kTileP];
            int b1[kTileP];
#pragma unroll
            for (int r = 0; r < kTileP; ++r) {
                const int i = r * blockDim.x + threadIdx.x;
#pragma unroll
                for (int m = 0; m < D; ++m) p[r].v[m] = i < g.cnt ? B.pts[i * D + m] : 0.0f;
                m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0;
            }
            for (int gi = 0; gi < (nslots >> 2); ++gi) {
                float4 c[D];
#pragma unroll
                for (int m = 0; m < D; ++m) c[m] = sb4[m * kq + gi];
#pragma unroll
                for (int r = 0; r < kTileP; ++r) {
                    float2 s0 = pair2<D>(p[r], c, false);
                    float2 s1 = pair2<D>(p[r], c, true);
                    float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
                    bool lt = v < m1[r];
                    m2[r] = fmaxf(m1[r], fminf(m2[r], v));
                    m1[r] = fminf(m1[r], v);
                    b1[r] = lt ? gi : b1[r];
                }
            }
            int wl = -2;   // this warp's common label (-2: no valid point, -1: mixed)
#pragma unroll
            for (int r = 0; r < kTileP; ++r) {
                const int i = r * blockDim.x + threadIdx.x;
                const bool valid = i < g.cnt;
                int a = 0;
                if (valid) {
                    const float thr = certify_thr(m1[r]);
                    if (!(m2[r] > thr)) {
                        a = overflow ? exact_scan_v<D>(p[r], nc, kpad, 0, k)
                                     : exact_scan_slots<D>(p[r], cnc, kCandCap, cj, 0, nreal);
                    } else {
                        const int s0 = b1[r] * 4;
                        int cn = 0, slot = 0x7fffffff;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int s = s0 + ((u + lane) & 3);
                            if (dist32n<D>(p[r], sb, stride, s) <= thr) { ++cn; slot = min(slot, s); }
                        }
                        if (cn == 1) a = overflow ? slot : cj[slot];
                        else a = overflow ? exact_scan_v<D>(p[r], nc, kpad, s0, min(s0 + 4, k))
                                          : exact_scan_slots<D>(p[r], cnc, kCandCap, cj, s0, min(s0 + 4, nreal));
                    }
                    sse += dist64n<D>(p[r], nc, kpad, a);
                    if (first) chg += 1;
                    else chg += (B.lab[i] != a);
                    labels[base + i] = a;
                }
                // warp-uniform label bookkeeping for the tile label state
                const unsigned vm = __ballot_sync(0xffffffffu, valid);
                if (vm) {
                    const int L = __shfl_sync(0xffffffffu, a, __ffs(vm) - 1);
                    const bool uni = __all_sync(0xffffffffu, !valid || a == L);
                    const int cur = uni ? L : -1;
                    wl = wl == -2 ? cur : (wl == cur ? wl : -1);
                }
                warp_accumulate<D>(valid, a, p[r].v, q, acc_sum, acc_cnt);
            }
            if (lane == 0) s_wlab[w] = wl;
            prev_t = t;
            if (threadIdx.x == 0) {
                st_pairs += (unsigned long long)g.cnt * (unsigned long long)nreal;
                st_pts += (unsigned long long)g.cnt;
            }
        }
        __syncthreads();   // shared buffers (candidates, tile buffer b, s_wlab) are reused next
    }
    if (threadIdx.x == 0 && prev_t >= 0) {
        int L = -2;
        bool ok = true;
        for (int i = 0; i < nw; ++i) {
            const int v = s_wlab[i];
            if (v == -2) continue;
            if (v < 0 || (L >= 0 && v != L)) { ok = false; break; }
            L = v;
        }
        tile_lab[prev_t] = ok && L >= 0 ? L : -1;
    }
    block_sum2<kTileThreads>(sse, chg);
    if (threadIdx.x == 0) {
        sse_part[blockIdx.x] = sse;
        chg_part[blockIdx.x] = chg;
        if (stats) {
            atomicAdd(&stats[0], st_pairs);
            atomicAdd(&stats[1], st_pts);
            atomicAdd(&stats[2], st_batch);
            atomicAdd(&stats[3], (unsigned long long)((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x));
        }
    }
}

}  // namespace km
