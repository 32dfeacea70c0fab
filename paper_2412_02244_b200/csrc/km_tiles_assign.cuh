// km_tiles_assign.cuh -- K1t, the tile-pruned assignment + fused update (see km_tiles.cuh
// for the index and the pruning argument).  One warp = one tile (ball node) at a time.
//
// Per warp: a contiguous range of tiles (so consecutive tiles share a parent list, which the
// warp caches in shared memory), TMA bulk copies of the next tile's geometry, moments, label
// state, points and previous labels (double buffer, mbarrier completion), then
//   prune the cached parent list with the tile ball (Eq. 7-8)  ->  batch (1 candidate,
//   Eq. 6 / Alg. 1)  or  per-point packed scan + FP64 certification.
#pragma once
#include "km_tiles.cuh"
#include "km_levels.cuh"

namespace km {

#ifndef KM_CHUNK_TILES
#define KM_CHUNK_TILES 1
#endif
constexpr int kChunkTiles = KM_CHUNK_TILES;   // consecutive tiles per work chunk of a warp

template <int D>
__global__ void __launch_bounds__(kTileThreads, 2)
assign_tiles_kernel(const float* __restrict__ ps, int64_t n, int ntiles, const TileGeom* __restrict__ geom,
                    const TileMom* __restrict__ mom, TileState* __restrict__ tstate, const int* __restrict__ pool,
                    const NodeRef* __restrict__ l1ref, const float* __restrict__ C, int k,
                    int32_t* __restrict__ labels, int first, double* __restrict__ sse_part,
                    unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                    unsigned int* __restrict__ acc_cnt, const Quant* __restrict__ quant, const Ctl* __restrict__ ctl,
                    unsigned long long* __restrict__ stats)
{
    if (ctl && ctl->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem<D>& S = reinterpret_cast<WarpSmem<D>*>(smem_raw)[w];
    const unsigned full = 0xffffffffu;
    const unsigned ltmask = (1u << lane) - 1u;
    const bool want_labels = !first;
    // tiles of this warp: chunks of kChunkTiles consecutive tiles, chunks interleaved over all
    // warps (locality for the parent-list cache, balance across the grid)
    const int gw = blockIdx.x * kWarpsPerCta + w, W = gridDim.x * kWarpsPerCta;
    auto next_tile = [&](int t) {
        const int nt = (t + 1) % kChunkTiles ? t + 1 : t + 1 + (W - 1) * kChunkTiles;
        return nt;
    };
    const int tstart = gw * kChunkTiles;
    if (lane == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (tstart < ntiles) stage_tile<D>(&S.buf[0], &S.bar[0], tstart, geom, mom, tstate, ps, labels, n, want_labels);
    }
    __syncwarp();
    const Quant q = *quant;

    double sse = 0.0;
    unsigned long long chg = 0, st_pairs = 0, st_pts = 0, st_batch = 0, st_tiles = 0;
    uint32_t phase[2] = {0u, 0u};
    int cached_st = -1, plen = 0;
    const int* srcp = nullptr;   // parent list in global memory (nullptr: identity over all k)
    bool pcached = false;        // parent list cached in S.pc / S.pj

    int it = 0;
    for (int t = tstart; t < ntiles; t = next_tile(t), ++it) {
        const int b = it & 1;
        const int tn = next_tile(t);
        if (lane == 0 && tn < ntiles)
            stage_tile<D>(&S.buf[b ^ 1], &S.bar[b ^ 1], tn, geom, mom, tstate, ps, labels, n, want_labels);
        const int st = t / kStTiles;
        if (st != cached_st) {   // new parent: (re)load its list
            cached_st = st;
            const NodeRef R = l1ref[st];
            srcp = R.off >= 0 ? pool + R.off : nullptr;
            plen = R.len;
            pcached = plen <= kStCache;
            if (pcached) {
                __syncwarp();
                for (int e = lane; e < plen; e += 32) {
                    const int j = srcp ? __ldg(srcp + e) : e;
                    S.pj[e] = j;
#pragma unroll
                    for (int m = 0; m < D; ++m) S.pc[m][e] = __ldg(C + (int64_t)j * D + m);
                }
                __syncwarp();
            }
        }
        mbar_wait(&S.bar[b], phase[b]);
        phase[b] ^= 1u;
        const auto& B = S.buf[b];
        const TileGeom g = B.g;
        const int64_t base = (int64_t)t * kTilePoints;
        ++st_tiles;

        // --- warp prune of the parent's list with the tile ball (Eq. 7-8) -------------------
        auto pj = [&](int e) { return pcached ? S.pj[e] : (srcp ? __ldg(srcp + e) : e); };
        auto pd2 = [&](int e, int j) {
            float s = 0.f;
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const float c = pcached ? S.pc[m][e] : __ldg(C + (int64_t)j * D + m);
                const float t1 = __fsub_rn(g.o[m], c);
                s = __fmaf_rn(t1, t1, s);
            }
            return s;
        };
        float dmin2 = INFINITY;
        for (int e = lane; e < plen; e += 32) dmin2 = fminf(dmin2, pd2(e, pj(e)));
#pragma unroll
        for (int of = 16; of > 0; of >>= 1) dmin2 = fminf(dmin2, __shfl_xor_sync(full, dmin2, of));
        const float T2 = prune_thr2(dmin2, g.r);
        int ncand = 0, cfirst = -1;
        for (int e0 = 0; e0 < plen; e0 += 32) {
            const int e = e0 + lane;
            int j = 0;
            bool f = false;
            if (e < plen) { j = pj(e); f = pd2(e, j) <= T2; }
            const unsigned bal = __ballot_sync(full, f);
            if (f) {
                const int off = ncand + __popc(bal & ltmask);
                if (off < kWCap) {
#pragma unroll
                    for (int m = 0; m < D; ++m) S.cnc[m][off] = -(pcached ? S.pc[m][e] : __ldg(C + (int64_t)j * D + m));
                    S.cj[off] = j;
                }
                if (off == 0) cfirst = j;
            }
            ncand += __popc(bal);
        }
        const bool overflow = ncand > kWCap || ncand == 0;
        if (!overflow) {
            const int padded = (ncand + 3) & ~3;
            if (lane < padded - ncand) {
#pragma unroll
                for (int m = 0; m < D; ++m) S.cnc[m][ncand + lane] = -INFINITY;
                S.cj[ncand + lane] = 0x7fffffff;
            }
        }
        __syncwarp();

        const int i0 = 4 * lane;
        const int nvalid = max(0, min(4, g.cnt - i0));
        if (ncand == 1) {
            // --- batch assignment of the whole tile (Eq. 6 / Alg. 1) ---------
            const int cstar = __shfl_sync(full, cfirst, __ffs(__ballot_sync(full, cfirst >= 0)) - 1);
            const int prev = B.st.lab;
            if (first || prev != cstar) {
                int changed = 0;
                if (!first && prev < 0) {
                    for (int r = 0; r < nvalid; ++r) changed += B.lab[i0 + r] != cstar;
                } else {
                    changed = nvalid;
                }
                chg += (unsigned long long)changed;
                if (nvalid == 4) *reinterpret_cast<int4*>(&labels[base + i0]) = make_int4(cstar, cstar, cstar, cstar);
                else for (int r = 0; r < nvalid; ++r) labels[base + i0 + r] = cstar;
            }
            if (lane == 0) {
                const TileMom& mm = B.mom;
                double dot = 0.0, oc2 = 0.0;
#pragma unroll
                for (int m = 0; m < D; ++m) {
                    const double oc = (double)g.o[m] - (double)__ldg(C + (int64_t)cstar * D + m);   // o - c
                    dot += oc * mm.s1[m];
                    oc2 += oc * oc;
                }
                sse += mm.s2 + 2.0 * dot + (double)g.cnt * oc2;
#pragma unroll
                for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)cstar * D + m], mm.q[m]);
                atomicAdd(&acc_cnt[cstar], (unsigned int)g.cnt);
                if (prev != cstar) tstate[t].lab = cstar;
                st_batch += 1;
            }
        } else {
            // --- per-point scan over the candidates (the parent list, chunked, on overflow) ----
            Pt<D> p[4];
            {
                const float4* bp = reinterpret_cast<const float4*>(B.pts + i0 * D);
                float v[4 * D];
#pragma unroll
                for (int u = 0; u < D; ++u) {
                    const float4 x4 = bp[u];
                    v[4 * u] = x4.x; v[4 * u + 1] = x4.y; v[4 * u + 2] = x4.z; v[4 * u + 3] = x4.w;
                }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int m = 0; m < D; ++m) p[r].v[m] = r < nvalid ? v[r * D + m] : 0.0f;
            }
            float m1[4], m2[4];
            int b1[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) { m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0; }
            if (!overflow) {
                scan_slots<D>(p, S.cnc, (ncand + 3) & ~3, 0, m1, m2, b1);
            } else {
                // stage the parent list itself in chunks; group index = list position / 4
                for (int e0 = 0; e0 < plen; e0 += kWCap) {
                    __syncwarp();
                    const int cl = min(kWCap, plen - e0), lp = (cl + 3) & ~3;
                    for (int s = lane; s < lp; s += 32) {
                        const int j = s < cl ? (srcp ? __ldg(srcp + e0 + s) : e0 + s) : 0;
#pragma unroll
                        for (int m = 0; m < D; ++m) S.cnc[m][s] = s < cl ? -__ldg(C + (int64_t)j * D + m) : -INFINITY;
                    }
                    __syncwarp();
                    scan_slots<D>(p, S.cnc, lp, e0 >> 2, m1, m2, b1);
                }
            }
            int a[4];
            const int4 old = *reinterpret_cast<const int4*>(&B.lab[i0]);
            const int oldv[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                a[r] = 0;
                if (r < nvalid) {
                    const float thr = certify_thr(m1[r]);
                    if (!(m2[r] > thr)) {
                        a[r] = overflow ? exact_scan_list<D>(p[r], C, srcp, 0, plen)
                                        : exact_scan_list<D>(p[r], C, S.cj, 0, ncand);
                    } else {
                        const int s0 = b1[r] * 4;
                        int cn = 0, slot = 0x7fffffff;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int s = s0 + ((u + lane) & 3);
                            float dv;
                            if (overflow) dv = s < plen ? dist32g<D>(p[r], C, srcp ? __ldg(srcp + s) : s) : INFINITY;
                            else dv = dist32n<D>(p[r], &S.cnc[0][0], kWCap, s);
                            if (dv <= thr) { ++cn; slot = min(slot, s); }
                        }
                        if (cn == 1) a[r] = overflow ? (srcp ? __ldg(srcp + slot) : slot) : S.cj[slot];
                        else a[r] = overflow ? exact_scan_list<D>(p[r], C, srcp, s0, min(s0 + 4, plen))
                                             : exact_scan_list<D>(p[r], C, S.cj, s0, min(s0 + 4, ncand));
                    }
                    // SSE_t summand: the certified FP32 distance (|D32 - D64| <= 1e-6 D64)
                    sse += (double)m1[r];
                    chg += first ? 1u : (unsigned)(oldv[r] != a[r]);
                }
            }
            if (nvalid == 4) *reinterpret_cast<int4*>(&labels[base + i0]) = make_int4(a[0], a[1], a[2], a[3]);
            else for (int r = 0; r < nvalid; ++r) labels[base + i0 + r] = a[r];
            // is the whole tile on one label?  -> tile label state + one-butterfly sums
            const bool tu = nvalid == 0 || ((nvalid < 2 || a[1] == a[0]) && (nvalid < 3 || a[2] == a[0]) &&
                                            (nvalid < 4 || a[3] == a[0]));
            const int L = __shfl_sync(full, a[0], 0);   // lane 0 always has a valid point
            const bool uni = __all_sync(full, nvalid == 0 || (tu && a[0] == L));
            accumulate_runs<D>(p, a, nvalid, uni, L, q, acc_sum, acc_cnt);
            if (lane == 0) {
                const int ns = uni ? L : -1;
                if (ns != B.st.lab) tstate[t].lab = ns;
                st_pairs += (unsigned long long)g.cnt * (unsigned long long)(overflow ? plen : ncand);
                st_pts += (unsigned long long)g.cnt;
            }
        }
        __syncwarp();   // the candidate buffer and tile buffer b are reused next
    }
    block_sum2<kTileThreads>(sse, chg);
    __shared__ unsigned long long s_st[4][kWarpsPerCta];
    if (lane == 0) { s_st[0][w] = st_pairs; s_st[1][w] = st_pts; s_st[2][w] = st_batch; s_st[3][w] = st_tiles; }
    __syncthreads();
    if (threadIdx.x == 0) {
        sse_part[blockIdx.x] = sse;
        chg_part[blockIdx.x] = chg;
        if (stats) {
            unsigned long long v[4] = {0, 0, 0, 0};
            for (int i = 0; i < kWarpsPerCta; ++i)
                for (int c = 0; c < 4; ++c) v[c] += s_st[c][i];
            for (int c = 0; c < 4; ++c) atomicAdd(&stats[c], v[c]);
        }
    }
}

}  // namespace km
