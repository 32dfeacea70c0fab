// km_tiles2.cuh -- the tile path split in two high-occupancy kernels (replaces the fused
// warp-per-tile K1t of km_tiles_assign.cuh, which was latency-bound at 16 warps per SM).
//
// Per iteration, after tile_filter_kernel (Eq. 5) and the index-level prunes (Eq. 7-8):
//   K1a tile_prune_kernel   one warp per LISTED tile: prune the tile's level-1 list with the
//                           tile ball -> one candidate: the batch decision of Eq. 6 (Alg. 1
//                           lines 325-329), sums moved as whole nodes and SSE_t from
//                           the tile moments; otherwise the candidate records go to tcand.
//   K1b tile_assign_kernel  one thread per POINT of every tile K1a did not settle: Eq. 4 inter
//                           bound against the previous centroid, else a scan of the tile's
//                           candidates in FP32 + FP64 certification (same argument as K1);
//                           labels, incremental sums (sv(j) +- p), SSE_t, changed.
// Both kernels use only registers and a few hundred bytes of shared memory per warp, so an SM
// runs 64 warps of them (vs 16 for the fused kernel) and memory latency is hidden by TLP.
#pragma once
#include "km_tiles.cuh"
#include "km_levels.cuh"
#include "km_bounds.cuh"

namespace km {

constexpr int kTC = 64;   // candidates stored per tile (more: K1b re-prunes the tile's level-1 list)


// FP32 direct-form squared distance (RN), same operation order as the other kernels.
template <int D>
__device__ __forceinline__ float d32(const float (&p)[D], const CRec& c)
{
    float t = __fsub_rn(p[0], c.x);
    float s = __fmul_rn(t, t);
    t = __fsub_rn(p[1], c.y);
    s = __fmaf_rn(t, t, s);
    if (D == 3) { t = __fsub_rn(p[D - 1], c.z); s = __fmaf_rn(t, t, s); }
    return s;
}

template <int D>
__device__ __forceinline__ double d64(const float (&p)[D], const CRec& c)
{
    const float cv[3] = {c.x, c.y, c.z};
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const double t = __dsub_rn((double)p[m], (double)cv[m]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

template <int D>
__device__ __forceinline__ unsigned long long qcoord(float v, const Quant& q, int m)
{
    return (unsigned long long)__double2ll_rn(__dmul_rn(__dsub_rn((double)v, q.o[m]), q.scale[m]));
}

// Same, reading the quantisation through the pointer (keeps K1b's register count down).
__device__ __forceinline__ unsigned long long qcoordp(float v, const Quant* __restrict__ q, int m)
{
    return (unsigned long long)__double2ll_rn(__dmul_rn(__dsub_rn((double)v, __ldg(&q->o[m])), __ldg(&q->scale[m])));
}

// ------------------------------------------------------------------------------------------
// K1a: warp per listed tile (static stride over the work list).
template <int D>
__global__ void __launch_bounds__(256)
tile_prune_kernel(const int* __restrict__ work, const int* __restrict__ work_cnt, int64_t n, const TileInfo* __restrict__ info,
                  TileState* __restrict__ tstate, const CRec* __restrict__ pool, const NodeRef* __restrict__ l1ref,
                  const float* __restrict__ C, int k, int first, TileRes* __restrict__ work2, int* __restrict__ work2_cnt,
                  CRec* __restrict__ tcand, CRec* __restrict__ ovf, int* __restrict__ ovf_cursor, int ovf_cap,
                  unsigned long long* __restrict__ sseq_part, unsigned long long* __restrict__ chg_part,
                  unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt, int ncopy,
                  const Quant* __restrict__ quant, const Ctl* __restrict__ ctl, unsigned long long* __restrict__ stats,
                  int st_shift)
{
    acc_sum += (int64_t)(blockIdx.x % ncopy) * k * D;   // this CTA's private copy of the running sums
    acc_cnt += (int64_t)(blockIdx.x % ncopy) * k;
    if (ctl && ctl->done) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, W = (gridDim.x * blockDim.x) >> 5;
    const int nheavy = work_cnt[5];   // (heavy tiles are stored downward from the top end)
    const int nwork = work_cnt[0] + nheavy;
    const int ntl = (int)((n + kTilePoints - 1) / kTilePoints);
    auto entry = [&](int v) { return v < nheavy ? work[ntl - 1 - v] : work[v - nheavy]; };
    const double ss = quant->sse_scale;
    unsigned long long sq = 0, chg = 0, st_batch = 0, st_tiles = 0, st_plen = 0;
    int tnext = gw < nwork ? entry(gw) : 0;
    for (int wi = gw; wi < nwork; wi += W) {
        const int t = tnext;
        if (wi + W < nwork) tnext = entry(wi + W);   // consumed next round
        const TileGeom g = info[t].g;
        const int prev = first ? -1 : tile_lab(tstate[t]);
        const NodeRef R = l1ref[t >> st_shift];
        const CRec* src = R.off >= 0 ? pool + R.off : nullptr;
        const int plen = R.len;
        auto rec = [&](int e) { return src ? src[e] : make_rec<D>(C, e); };
        ++st_tiles;
        st_plen += plen;
        // pass 1: nearest list centroid to the pivot (two record loads per lane in flight)
        float dmin2 = INFINITY;
        for (int e0 = 0; e0 < plen; e0 += 64) {
            const int e1 = e0 + lane, e2 = e0 + 32 + lane;
            CRec c1, c2;
            if (e1 < plen) c1 = rec(e1);
            if (e2 < plen) c2 = rec(e2);
            if (e1 < plen) dmin2 = fminf(dmin2, rec_delta2<D>(g.o, c1));
            if (e2 < plen) dmin2 = fminf(dmin2, rec_delta2<D>(g.o, c2));
        }
        dmin2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dmin2)));   // >= 0: uint order
        const float T2 = prune_thr2(dmin2, g.r);
        // pass 2: ordered compaction of the candidates (ascending j) into tcand
        int ncand = 0, cfirst = -1;
        float fx = 0.f, fy = 0.f, fz = 0.f;   // coordinates of the first candidate (its lane)
        CRec* out = tcand + (int64_t)t * kTC;
        for (int e0 = 0; e0 < plen; e0 += 32) {
            const int e = e0 + lane;
            CRec c;
            bool f = false;
            if (e < plen) { c = rec(e); f = rec_delta2<D>(g.o, c) <= T2; }
            const unsigned bal = __ballot_sync(full, f);
            if (f) {
                const int slot = ncand + __popc(bal & lt);
                if (slot < kTC) out[slot] = c;
                if (slot == 0) { cfirst = c.j; fx = c.x; fy = c.y; fz = c.z; }
            }
            ncand += __popc(bal);
        }
        TileRes r;
        r.t = t;
        r.prev = prev;
        r.ncand = ncand;
        r.cstar = -1;
        r.T2 = T2;
        r.coff = 0;
        r.pad = 0;
        if (ncand == 1) {
            // --- batch assignment of the whole tile (Eq. 6 / Alg. 1) -------------
            const int sl = __ffs(__ballot_sync(full, cfirst >= 0)) - 1;
            const int cstar = __shfl_sync(full, cfirst, sl);
            const float cc[3] = {__shfl_sync(full, fx, sl), __shfl_sync(full, fy, sl), __shfl_sync(full, fz, sl)};
            r.cstar = cstar;
            r.mode = (first || prev != cstar) ? kTileBatch : kTileNoop;
            if (lane == 0) {
                const TileMom mm = info[t].m;
                sq += sse_q(tile_sse<D>(g, mm, cc), ss);
                if (first || (prev >= 0 && prev != cstar)) {
                    // the whole node moves: sv(n1) += N.p* |N|, sv(a(N)) -= N.p* |N|
#pragma unroll
                    for (int m = 0; m < D; ++m) {
                        atomicAdd(&acc_sum[(int64_t)cstar * D + m], mm.q[m]);
                        if (!first) atomicAdd(&acc_sum[(int64_t)prev * D + m], 0ull - mm.q[m]);
                    }
                    atomicAdd(&acc_cnt[cstar], (unsigned int)g.cnt);
                    if (!first) atomicAdd(&acc_cnt[prev], 0u - (unsigned int)g.cnt);
                    chg += (unsigned long long)g.cnt;
                }
                if (prev != cstar) tile_lab_set(&tstate[t], cstar);
                ++st_batch;
            }
        } else {
            r.mode = ncand <= kTC && ncand > 0 ? kTileScan : kTileScanList;
            if (ncand > kTC) {
                // long candidate list: a second emission into the overflow pool (rare)
                int off = 0;
                if (lane == 0) off = atomicAdd(ovf_cursor, ncand);
                off = __shfl_sync(full, off, 0);
                if ((long long)off + ncand <= (long long)ovf_cap) {
                    r.mode = kTileScan;
                    r.coff = off;
                    int cnt = 0;
                    for (int e0 = 0; e0 < plen; e0 += 32) {
                        const int e = e0 + lane;
                        CRec c;
                        bool f = false;
                        if (e < plen) { c = rec(e); f = rec_delta2<D>(g.o, c) <= T2; }
                        const unsigned bal = __ballot_sync(full, f);
                        if (f) ovf[off + cnt + __popc(bal & lt)] = c;
                        cnt += __popc(bal);
                    }
                }
            }
        }
        // tiles with per-point work go to K1b's list (one 32-B record each)
        if (lane == 0 && r.mode != kTileNoop) work2[atomicAdd(work2_cnt, 1)] = r;
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, chg);
    if (threadIdx.x == 0) {
        atomicAdd(sseq_part, sq);   // the iteration's totals (integers: order-independent)
        atomicAdd(chg_part, chg);
    }
    if (stats && lane == 0) {
        atomicAdd(&stats[2], st_batch);
        atomicAdd(&stats[3], st_tiles);
        atomicAdd(&stats[10], st_plen);
    }
}

// ------------------------------------------------------------------------------------------
// K1b: one thread per point over K1a's records; CTA = 2 tiles (256 threads), persistent, the
// next record prefetched while the current tile is processed.
#ifndef KM_K1B_MINB
#define KM_K1B_MINB 3
#endif
template <int D>
__global__ void __launch_bounds__(256, KM_K1B_MINB)
tile_assign_kernel(const float* __restrict__ ps, int64_t n, const TileRes* __restrict__ work2,
                   const int* __restrict__ work2_cnt, const TileInfo* __restrict__ info, const CRec* __restrict__ tcand,
                   const CRec* __restrict__ ovf, int ctab,
                   TileState* __restrict__ tstate, const CRec* __restrict__ pool, const NodeRef* __restrict__ l1ref,
                   const float* __restrict__ C, int k, const unsigned int* __restrict__ cb2, int32_t* __restrict__ labels,
                   int first, unsigned long long* __restrict__ sseq_part, unsigned long long* __restrict__ chg_part,
                   unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt, int ncopy,
                   const Quant* __restrict__ quant, const Ctl* __restrict__ ctl, unsigned long long* __restrict__ stats,
                   int st_shift)
{
    acc_sum += (int64_t)(blockIdx.x % ncopy) * k * D;   // this CTA's private copy of the running sums
    acc_cnt += (int64_t)(blockIdx.x % ncopy) * k;
    if (ctl && ctl->done) return;
    __shared__ CRec s_c[8][32];   // per warp: one chunk of candidate records
    extern __shared__ float4 s_tab[];   // ctab: {c_j, (cb[j]/2)^2 lower bound} for Eq. 4, all k
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    if (ctab && !first) {
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const CRec c = make_rec<D>(C, j);
            s_tab[j] = make_float4(c.x, c.y, c.z, inter_half2(cb2[j]));
        }
        __syncthreads();
    }
    const Quant* const q = quant;
    const double ss = quant->sse_scale;
    const int nw2 = work2_cnt[0];
    unsigned long long sq = 0, chg = 0, st_pairs = 0, st_pts = 0, st_pskip = 0;
    const int half = threadIdx.x >> 7;
    const int stride = 2 * gridDim.x;
    const int pt = threadIdx.x & 127;
    // software pipeline: the next tile's record, point and previous label are loaded while the
    // current tile is processed (and the record after that), so each warp keeps two tiles of
    // HBM reads in flight
    int ei = 2 * blockIdx.x + half;
    TileRes r_nxt;
    float p_nxt[D];
    int old_nxt = -1;
    CRec c_nxt;   // this lane's record of the first candidate chunk of the next tile
    auto load_pt = [&](const TileRes& rr, float (&pp)[D], int& oo, CRec& cc) {
        const int64_t ix = (int64_t)rr.t * kTilePoints + pt;
        const bool v = ix < n;
#pragma unroll
        for (int m = 0; m < D; ++m) pp[m] = v ? ps[ix * D + m] : 0.f;
        oo = (first || !v) ? -1 : labels[ix];
        if (rr.mode == kTileScan && lane < rr.ncand)
            cc = (rr.ncand <= kTC ? tcand + (int64_t)rr.t * kTC : ovf + rr.coff)[lane];
    };
    if (ei < nw2) { r_nxt = work2[ei]; load_pt(r_nxt, p_nxt, old_nxt, c_nxt); }
    TileRes r_nn;
    if (ei + stride < nw2) r_nn = work2[ei + stride];
    for (; ei < nw2; ei += stride) {
        const TileRes r = r_nxt;
        float p[D];
#pragma unroll
        for (int m = 0; m < D; ++m) p[m] = p_nxt[m];
        const int old = old_nxt;
        const CRec c0 = c_nxt;
        if (ei + stride < nw2) {
            r_nxt = r_nn;
            load_pt(r_nxt, p_nxt, old_nxt, c_nxt);                    // consumed next round
            if (ei + 2 * stride < nw2) r_nn = work2[ei + 2 * stride];   // consumed in two rounds
        }
        const int t = r.t;
        const int64_t idx = (int64_t)t * kTilePoints + pt;
        const bool valid = idx < n;
        if (__ballot_sync(full, valid) == 0u) continue;   // a warp past the end of the last tile
        int a = old;
        if (r.mode == kTileBatch) {
            a = r.cstar;
            if (valid && !first && r.prev < 0 && old != a) {
                // mixed -> uniform: move this point (uniform/first tiles were moved whole by K1a)
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    const unsigned long long qv = qcoordp(p[m], q, m);
                    atomicAdd(&acc_sum[(int64_t)a * D + m], qv);
                    atomicAdd(&acc_sum[(int64_t)old * D + m], 0ull - qv);
                }
                atomicAdd(&acc_cnt[a], 1u);
                atomicAdd(&acc_cnt[old], 0xffffffffu);
                ++chg;
            }
            if (valid && (first || old != a)) labels[idx] = a;
            continue;
        }
        // --- kTileScan / kTileScanList ---------------------------------------------------------
        float m1 = INFINITY;
        bool done = !valid;
        if (valid && !first) {
            // Eq. 4: ||p - c_a(i)|| < cb[a(i)] / 2 keeps the previous label
            CRec co;
            float h2;
            if (ctab) {
                const float4 e = s_tab[old];
                co.x = e.x; co.y = e.y; co.z = e.z; co.j = old;
                h2 = e.w;
            } else {
                co = make_rec<D>(C, old);
                h2 = inter_half2(cb2[old]);
            }
            const float dv = d32<D>(p, co);
            if (dv < h2) { done = true; m1 = dv; ++st_pskip; }
        }
        if (__any_sync(full, !done)) {
            // scan the candidates in chunks of 32 staged in shared memory; kTileScanList
            // re-prunes the tile's level-1 list on the fly with K1a's threshold
            const bool inlist = r.mode == kTileScan;
            const CRec* src;
            int len;
            float o[3] = {0.f, 0.f, 0.f};
            if (inlist) {
                src = r.ncand <= kTC ? tcand + (int64_t)t * kTC : ovf + r.coff;
                len = r.ncand;
            } else {
                const NodeRef R = l1ref[t >> st_shift];
                src = R.off >= 0 ? pool + R.off : nullptr;
                len = R.len;
                const TileGeom g = info[t].g;
                o[0] = g.o[0]; o[1] = g.o[1]; o[2] = g.o[2];
            }
            float m2 = INFINITY, s1 = INFINITY;
            int bj = 0, nscan = 0;
            for (int e0 = 0; e0 < len; e0 += 32) {
                const int e = e0 + lane;
                CRec c;
                bool f = e < len;
                if (f) c = (inlist && e0 == 0) ? c0 : (src ? src[e] : make_rec<D>(C, e));
                if (!inlist && f) f = rec_delta2<D>(o, c) <= r.T2;
                const unsigned bal = __ballot_sync(full, f);
                __syncwarp();
                if (f) s_c[w][__popc(bal & lt)] = c;   // ascending j preserved
                __syncwarp();
                const int cl = __popc(bal);
                nscan += cl;
                if (!done) {
                    for (int u = 0; u < cl; ++u) {
                        const CRec cu = s_c[w][u];
                        const float v = d32<D>(p, cu);
                        const bool lt1 = v < s1;
                        m2 = lt1 ? s1 : fminf(m2, v);   // second smallest over the other candidates
                        bj = lt1 ? cu.j : bj;           // the FIRST (lowest j) candidate at the minimum
                        s1 = fminf(s1, v);
                    }
                }
            }
            if (!done) {
                m1 = s1;
                st_pairs += (unsigned long long)nscan;
                ++st_pts;
                if (m2 > certify_thr(m1)) {
                    a = bj;   // the unique FP32 argmin is the FP64 argmin
                } else {
                    // near-tie: exact FP64 over the whole list, lowest j on ties (ascending list)
                    double best = INFINITY;
                    for (int e = 0; e < len; ++e) {
                        const CRec c = src ? src[e] : make_rec<D>(C, e);
                        const double v = d64<D>(p, c);
                        if (v < best) { best = v; a = c.j; }
                    }
                }
            }
        }
        if (valid) {
            sq += sse_q((double)m1, ss);
            const bool moved = first || old != a;
            chg += moved;
            if (moved) labels[idx] = a;
        }
        // sums: iteration 0 adds every point (warp-aggregated when the warp is uniform);
        // later iterations move only the points whose label changed
        const int L0 = __shfl_sync(full, a, 0);   // lane 0 of a live warp is always valid
        const bool wuni = __all_sync(full, !valid || a == L0);
        if (first) {
            if (wuni) {
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    unsigned long long qv = valid ? qcoordp(p[m], q, m) : 0ull;
#pragma unroll
                    for (int of = 16; of > 0; of >>= 1) qv += __shfl_xor_sync(full, qv, of);
                    if (lane == 0) atomicAdd(&acc_sum[(int64_t)L0 * D + m], qv);
                }
                const unsigned c = __popc(__ballot_sync(full, valid));
                if (lane == 0) atomicAdd(&acc_cnt[L0], c);
            } else if (valid) {
#pragma unroll
                for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)a * D + m], qcoordp(p[m], q, m));
                atomicAdd(&acc_cnt[a], 1u);
            }
        } else if (valid && old != a) {
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const unsigned long long qv = qcoordp(p[m], q, m);
                atomicAdd(&acc_sum[(int64_t)a * D + m], qv);
                atomicAdd(&acc_sum[(int64_t)old * D + m], 0ull - qv);
            }
            atomicAdd(&acc_cnt[a], 1u);
            atomicAdd(&acc_cnt[old], 0xffffffffu);
        }
        // tile label state: this warp's slot (no read-back; readers combine the four slots)
        if (lane == 0) tstate[t].lab[w & 3] = wuni ? L0 : -1;
    }
    double dummy = 0.0;
    block_sum2<256>(dummy, sq);
    __syncthreads();
    block_sum2<256>(dummy, chg);
    if (threadIdx.x == 0) {
        atomicAdd(sseq_part, sq);   // the iteration's totals (integers: order-independent)
        atomicAdd(chg_part, chg);
    }
    if (stats) {
        st_pairs = warp_sum(st_pairs);
        st_pts = warp_sum(st_pts);
        st_pskip = warp_sum(st_pskip);
        if (lane == 0) {
            atomicAdd(&stats[0], st_pairs);
            atomicAdd(&stats[1], st_pts);
            atomicAdd(&stats[22], st_pskip);
        }
    }
}

}  // namespace km
