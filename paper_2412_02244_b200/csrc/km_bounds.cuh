// km_bounds.cuh -- the paper's inter bound (Dask-means, arXiv 2412.02244, Eq. 3-5,
// P:L236-251) on the GPU:
//   cb[j] = min_{l != j} ||c_j - c_l||                                   (Eq. 3)
//   a point keeps its previous cluster a(i) if ||p_i - c_a(i)|| < cb[a(i)] / 2     (Eq. 4)
//   a node N keeps a(N) if ||N.p* - c_a(N)|| + N.r < cb[a(N)] / 2                   (Eq. 5)
// (Alg. 1 Assign).  Here a node is a tile (128 Morton-sorted
// points; km_tiles.cuh) whose points all carried label a in the previous iteration.
//
// Exactness.  In exact arithmetic ||p - c_a|| < cb/2 gives, for j != a,
// ||p - c_j|| >= ||c_a - c_j|| - ||p - c_a|| > ||p - c_a||, i.e. a is the unique nearest
// centroid.  The tests below use a lower bound of (cb/2)^2 with a relative margin of 2^-17
// (cbh2), far above the FP32/FP64 rounding of the quantities compared, so a passing point is
// strictly nearer to c_a by a relative gap >> FP64 rounding, and its FP64 label (the oracle's)
// is a.  Passing tiles/points keep their labels; their cluster sums need no update because
// the sums are maintained incrementally (sv(j) +- p only when p moves).
#pragma once
#include "km_tiles.cuh"

namespace km {

// (cb/2)^2 lower bound from the FP32 bits of min_l ||c_j - c_l||^2 (computed in the direct
// form with RN: relative error < 6u, u = 2^-24).  0.25 * (1 - 2^-17) covers it plus the
// strictness margin; -2^-118 covers subnormal absolute error; +inf stays +inf (k = 1).
__device__ __forceinline__ float inter_half2(unsigned int cb2_bits)
{
    return __fmaf_rd(__uint_as_float(cb2_bits), 0.25f - 0x1p-19f, -0x1p-118f);
}

// Eq. 3 for all j: grid (ceil(k / (256 JB)), S); CTA (bx, s) takes centroids l in chunk s
// (staged in shared memory) and folds min_{l != j} ||c_j - c_l||^2 into cb2[j] for JB centroids
// per thread (each staged centroid read once per JB pairs; uint atomicMin on the non-negative
// float bits; finalize resets cb2 to +inf after each refine).
template <int D, int JB>
__global__ void __launch_bounds__(256)
interbound_kernel(const float* __restrict__ C, int k, int chunk, unsigned int* __restrict__ cb2,
                  int* __restrict__ work_cnt, const Ctl* __restrict__ ctl)
{
    if (ctl && ctl->done) return;
    // the work lists' counters this stream owns; slot 4 (the level-1 pool cursor) belongs to the
    // main stream's level-1 prune, which may run concurrently, and is reset there
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 8 && threadIdx.x != 4) work_cnt[threadIdx.x] = 0;
    extern __shared__ float s_c[];   // [D][chunk]
    const int l0 = blockIdx.y * chunk, l1 = min(k, l0 + chunk);
    for (int l = l0 + threadIdx.x; l < l1; l += blockDim.x)
#pragma unroll
        for (int m = 0; m < D; ++m) s_c[m * chunk + (l - l0)] = C[(int64_t)l * D + m];
    __syncthreads();
    const int j0 = blockIdx.x * blockDim.x * JB + threadIdx.x;
    float cj[JB][D], best[JB];
#pragma unroll
    for (int u = 0; u < JB; ++u) {
        const int j = min(j0 + u * (int)blockDim.x, k - 1);
#pragma unroll
        for (int m = 0; m < D; ++m) cj[u][m] = C[(int64_t)j * D + m];
        best[u] = INFINITY;
    }
    const int cnt = l1 - l0;
#pragma unroll 2
    for (int e = 0; e < cnt; ++e) {
        float cl[D];
#pragma unroll
        for (int m = 0; m < D; ++m) cl[m] = s_c[m * chunk + e];
#pragma unroll
        for (int u = 0; u < JB; ++u) {
            float t = __fsub_rn(cj[u][0], cl[0]);
            float s = __fmul_rn(t, t);
#pragma unroll
            for (int m = 1; m < D; ++m) { t = __fsub_rn(cj[u][m], cl[m]); s = __fmaf_rn(t, t, s); }
            best[u] = (e + l0 == j0 + u * (int)blockDim.x) ? best[u] : fminf(best[u], s);
        }
    }
#pragma unroll
    for (int u = 0; u < JB; ++u) {
        const int j = j0 + u * (int)blockDim.x;
        if (j < k && best[u] < INFINITY) atomicMin(&cb2[j], __float_as_uint(best[u]));
    }
}

// Sum_{p in tile} ||p - c||^2 from the tile moments (o, s1 = sum (p - o), s2 = sum ||p - o||^2).
template <int D>
__device__ __forceinline__ double tile_sse(const TileGeom& g, const TileMom& mm, const float (&cc)[3])
{
    double dot = 0.0, oc2 = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const double oc = (double)g.o[m] - (double)cc[m];
        dot += oc * mm.s1[m];
        oc2 += oc * oc;
    }
    return mm.s2 + 2.0 * dot + (double)g.cnt * oc2;
}

// Eq. 5 on every tile whose previous labels were all a (tile_lab = a >= 0): FP64
// U = ||o - c_a|| + r (r already rounded up); pass iff U^2 (1 + 2^-40) < cbh2(a).  Passing
// tiles add their SSE_t share (moments) and are done for this iteration; the others go to
// the work list of assign_tiles_kernel (ascending within a warp) and mark their level-1 node
// as needed.  first = 1 (no previous labels): every tile is listed.
template <int D>
__global__ void __launch_bounds__(256)
tile_filter_kernel(const TileInfo* __restrict__ info, const TileState* __restrict__ tstate, int ntiles,
                   const float* __restrict__ C, const unsigned int* __restrict__ cb2, int first, int* __restrict__ work,
                   int* __restrict__ work_cnt, int* __restrict__ l1need, const unsigned char* __restrict__ theavy,
                   TileAux* __restrict__ aux,
                   unsigned long long* __restrict__ sseq_part,
                   unsigned long long* __restrict__ chg_part, const Quant* __restrict__ quant,
                   const Ctl* __restrict__ ctl, unsigned long long* __restrict__ stats, int st_shift)
{
    if (ctl && ctl->done) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const double ss = quant->sse_scale;
    unsigned long long sq = 0, npass = 0;
    for (int base = blockIdx.x * blockDim.x; base < ntiles; base += gridDim.x * blockDim.x) {
        const int t = base + threadIdx.x;
        bool need = false;
        if (t < ntiles) {
            const int a = first ? -1 : tile_lab(tstate[t]);
            need = true;
            if (a >= 0) {
                const TileGeom g = info[t].g;
                float cc[3] = {0.f, 0.f, 0.f};
#pragma unroll
                for (int m = 0; m < D; ++m) cc[m] = C[(int64_t)a * D + m];
                // U bounds ||p - c_a|| over the tile: one ball, or the larger of the two sub-balls
                auto ub = [&](const float* oo, float rr) {
                    double d2 = 0.0;
#pragma unroll
                    for (int m = 0; m < D; ++m) { const double x = (double)oo[m] - (double)cc[m]; d2 += x * x; }
                    return sqrt(d2) + (double)rr;
                };
                double U = ub(g.o, g.r);
                if (g.pad[0]) {
                    const TileSub sb = info[t].sb;
                    U = fmax(ub(sb.o1, sb.r1), ub(sb.o2, sb.r2));
                }
                const float h2 = inter_half2(cb2[a]);
                if (U * U * (1.0 + 0x1p-40) < (double)h2) {
                    need = false;
                    ++npass;
                    sq += sse_q(tile_sse<D>(g, info[t].m, cc), ss);
                } else {
                    // listed: the point-level Eq. 4 record for the assignment kernel (staged with the tile)
                    aux[t].pre = make_float4(cc[0], cc[1], cc[2], h2);
                }
            }
        }
        // tiles K1t found expensive last iteration (long lists) go to the top end of the list,
        // which K1t hands out first: they start early instead of ending the kernel late
        const bool hv = need && theavy && theavy[t];
        const unsigned bal = __ballot_sync(full, need && !hv);
        const unsigned balh = __ballot_sync(full, hv);
        const unsigned lt = (1u << lane) - 1u;
        if (bal) {
            const int leader = __ffs(bal) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(work_cnt, __popc(bal));
            pos = __shfl_sync(full, pos, leader);
            if (need && !hv) work[pos + __popc(bal & lt)] = t;
        }
        if (balh) {
            const int leader = __ffs(balh) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(work_cnt + 5, __popc(balh));
            pos = __shfl_sync(full, pos, leader);
            if (hv) work[ntiles - 1 - (pos + __popc(balh & lt))] = t;
        }
        if (need) l1need[t >> st_shift] = 1;
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, npass);
    if (threadIdx.x == 0) {
        atomicAdd(sseq_part, sq);   // the iteration's SSE_t total (integers: order-independent)
        if (stats) atomicAdd(&stats[12], npass);
    }
}

}  // namespace km
