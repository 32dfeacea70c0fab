// km_tiles_assign.cuh -- K1t, the tile-pruned assignment + fused update (see km_tiles.cuh
// for the index and the pruning argument, km_levels.cuh for the node lists and the per-tile
// candidate lists, km_bounds.cuh for the inter bound).
//
// One warp = one tile (ball node of 128 Morton-consecutive points) at a time; warps are
// independent (no CTA barrier in the loop).  Everything a tile needs arrives with one batch of
// 16-B cp.async copies issued one tile ahead (double buffer): its points and previous labels,
// its ball + moments, its label state, and this iteration's per-tile inputs -- the Eq. 4
// record of its previous label (tile_filter_kernel) and its candidate list, pruned from the
// level-1 node's list with the tile's ball by the level-1 prune (tile_cands_warp, Eq. 7-8).
// Per tile:
//   0. (t > 0, previous labels all a) Eq. 4 for every point against c_a: all pass -> labels,
//      sums and tile state unchanged, SSE_t from the FP32 distances; done.
//   1. one candidate -> batch assignment of the whole tile (Eq. 6, Alg. 1): the
//      tile moves as N.p*|N|, SSE_t from its moments;
//   2. otherwise a packed FP32 scan of the candidates (4 points x 4 centroids per step) and
//      FP64 certification; more than kTC candidates are scanned in chunks
//      from the overflow pool.
//   3. sums: iteration 0 adds every point (the tile sum when the tile is uniform); later
//      iterations move only the points whose label changed (incremental sv(j)).
#pragma once
#include "km_tiles.cuh"
#include "km_levels.cuh"
#include "km_bounds.cuh"

#ifndef KM_HEAVY_CAND
#define KM_HEAVY_CAND 24   // a tile with more candidates is scheduled first next iteration
#endif

#ifndef KM_STATIC_FRAC
#define KM_STATIC_FRAC 50   // percent of the work list assigned round-robin before atomic claiming
#endif

#ifndef KM_CLAIM
#define KM_CLAIM 4          // entries of the dynamic part claimed per atomic
#endif

#ifndef KM_K1T_WARPS
#define KM_K1T_WARPS 4      // warps per CTA of K1t (4: config 4 -3 %, config 3 -4 % against 8)
#endif

namespace km {

constexpr int kK1tWarps = KM_K1T_WARPS;
constexpr int kK1tThreads = 32 * kK1tWarps;

template <int D>
__device__ __forceinline__ CRec get_rec(const CRec* recs, const float* __restrict__ C, int e)
{
    return recs ? recs[e] : make_rec<D>(C, e);
}

// Exact FP64 argmin over records [e0, e1) of a list (recs == nullptr: all k), lowest j on ties
// whatever the list order (the overflow pool is filled in no fixed order).
template <int D>
__device__ __noinline__ int exact_scan_recs(Pt<D> p, const CRec* recs, const float* __restrict__ C, int e0, int e1)
{
    double best = INFINITY;
    int a = get_rec<D>(recs, C, e0).j;
    for (int e = e0; e < e1; ++e) {
        const CRec c = get_rec<D>(recs, C, e);
        const float cv[3] = {c.x, c.y, c.z};
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double t = __dsub_rn((double)p.v[m], (double)cv[m]);
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        if (s < best || (s == best && c.j < a)) { best = s; a = c.j; }   // ties: lowest j, in any list order
    }
    return a;
}

template <int D>
__device__ __forceinline__ float dist32_rec(const Pt<D>& p, const CRec& c)
{
    float t = __fsub_rn(p.v[0], c.x);
    float s = __fmul_rn(t, t);
    t = __fsub_rn(p.v[1], c.y);
    s = __fmaf_rn(t, t, s);
    if (D == 3) { t = __fsub_rn(p.v[2], c.z); s = __fmaf_rn(t, t, s); }
    return s;
}

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// All lanes: 16-B async copies of tile t (points, previous labels, ball + moments, label
// state, per-tile inputs, candidate block).
template <int D>
__device__ __forceinline__ void stage_tile_cp(typename WarpSmem<D>::Buf* buf, int t, const TileInfo* info,
                                              const TileState* tstate, const TileAux* aux, const float* tcand,
                                              const float* ps, const int32_t* labels, int64_t n, bool want_labels,
                                              int lane)
{
    const int64_t base = (int64_t)t * kTilePoints;
    const int cnt = (int)min((int64_t)kTilePoints, n - base);
    const int pch = (cnt * D * 4 + 15) >> 4;   // sources are padded to 16 B in HBM
    const char* src = reinterpret_cast<const char*>(ps + base * D);
    char* dst = reinterpret_cast<char*>(buf->pts);
    for (int c = lane; c < pch; c += 32) cp16(dst + 16 * c, src + 16 * c);
    if (want_labels && lane < ((cnt * 4 + 15) >> 4)) cp16(buf->lab + 4 * lane, labels + base + 4 * lane);
    constexpr int kCb = cand_block_words<D>() / 4;   // 16-B chunks of the candidate block (24 / 32)
    const float* cb = tcand + (int64_t)t * cand_block_words<D>();
    if (lane < kCb) cp16(buf->cand + 4 * lane, cb + 4 * lane);
    if (lane < (int)(sizeof(TileInfo) / 16))
        cp16(reinterpret_cast<char*>(&buf->info) + 16 * lane, reinterpret_cast<const char*>(info + t) + 16 * lane);
    else if (lane == 29)
        cp16(&buf->st, tstate + t);
    else if (lane >= 30)
        cp16(reinterpret_cast<char*>(&buf->aux) + 16 * (lane - 30), reinterpret_cast<const char*>(aux + t) + 16 * (lane - 30));
}

#ifndef KM_K1T_BULK
#define KM_K1T_BULK 1   // 1: one lane stages a tile with bulk copies (TMA engine) + an mbarrier; 0: 16-B cp.async per lane
#endif
__device__ __forceinline__ void k1t_bulk(void* sdst, const void* gsrc, uint32_t bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void k1t_bar_wait(unsigned long long* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "K1T_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra K1T_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Lane 0: tile t's points, previous labels, ball + moments, label state, per-tile inputs and
// candidate block as six bulk copies completing on one mbarrier (the buffer's previous readers
// have passed a __syncwarp; the proxy fence orders their generic reads before the async writes).
template <int D>
__device__ __forceinline__ void stage_tile_bulk(typename WarpSmem<D>::Buf* buf, unsigned long long* bar, int t,
                                                const TileInfo* info, const TileState* tstate, const TileAux* aux,
                                                const float* tcand, const float* ps, const int32_t* labels, int64_t n,
                                                bool want_labels)
{
    const int64_t base = (int64_t)t * kTilePoints;
    const int cnt = (int)min((int64_t)kTilePoints, n - base);
    const uint32_t pb = (uint32_t)((cnt * D * 4 + 15) & ~15);   // sources are padded to 16 B in HBM
    const uint32_t lb = want_labels ? (uint32_t)((cnt * 4 + 15) & ~15) : 0u;
    constexpr uint32_t cbb = cand_block_words<D>() * 4;
    const uint32_t bytes = (uint32_t)(sizeof(TileInfo) + sizeof(TileState) + sizeof(TileAux)) + cbb + pb + lb;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    k1t_bulk(&buf->info, info + t, (uint32_t)sizeof(TileInfo), bar);
    k1t_bulk(&buf->st, tstate + t, (uint32_t)sizeof(TileState), bar);
    k1t_bulk(&buf->aux, aux + t, (uint32_t)sizeof(TileAux), bar);
    k1t_bulk(buf->cand, tcand + (int64_t)t * cand_block_words<D>(), cbb, bar);
    k1t_bulk(buf->pts, ps + base * D, pb, bar);
    if (lb) k1t_bulk(buf->lab, labels + base, lb, bar);
}

// Packed scan of 4 points over the candidate slots [0, nslots) of an SoA block (negated
// coordinates, row stride STRIDE) tracking, per point, the FP32 minimum m1, its FIRST slot b1
// and the second-smallest value m2 over all other slots.
template <int D, int STRIDE>
__device__ __forceinline__ void scan_block(const Pt<D> (&p)[4], const float* cnc, int nslots, float (&m1)[4],
                                           float (&m2)[4], int (&b1)[4])
{
    for (int gi = 0; gi < (nslots >> 2); ++gi) {
        float4 c[D];
#pragma unroll
        for (int m = 0; m < D; ++m) c[m] = reinterpret_cast<const float4*>(cnc + m * STRIDE)[gi];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const float2 s0 = pair2<D>(p[r], c, false);
            const float2 s1 = pair2<D>(p[r], c, true);
            const float v[4] = {s0.x, s0.y, s1.x, s1.y};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool lt = v[u] < m1[r];
                m2[r] = fmaxf(m1[r], fminf(m2[r], v[u]));   // second smallest of {m1, m2, v}
                m1[r] = fminf(m1[r], v[u]);
                b1[r] = lt ? 4 * gi + u : b1[r];
            }
        }
    }
}

// Incremental sums ("sv(j) = sv(j) + p" when p moves in, "- p" when it moves
// out): for every valid point r whose label changed from old[r] to neu[r], add its fixed-point
// vector to sv(neu) and subtract it from sv(old) (mod 2^64: the running sums are exact).
template <int D>
__device__ __forceinline__ void move_points(const Pt<D> (&p)[4], const int (&old)[4], const int (&neu)[4], int nvalid,
                                            const Quant* __restrict__ qp, unsigned long long* __restrict__ acc_sum,
                                            unsigned int* __restrict__ acc_cnt)
{
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (r < nvalid && old[r] != neu[r]) {
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const unsigned long long qv = (unsigned long long)__double2ll_rn(
                    __dmul_rn(__dsub_rn((double)p[r].v[m], __ldg(&qp->o[m])), __ldg(&qp->scale[m])));
                atomicAdd(&acc_sum[(int64_t)neu[r] * D + m], qv);
                atomicAdd(&acc_sum[(int64_t)old[r] * D + m], 0ull - qv);
            }
            atomicAdd(&acc_cnt[neu[r]], 1u);
            atomicAdd(&acc_cnt[old[r]], 0xffffffffu);
        }
    }
}

// K1t.  Tiles come from the work list of tile_filter_kernel (those not settled by Eq. 5);
// warps take entries round-robin for the first KM_STATIC_FRAC percent, then through an atomic
// counter (results do not depend on the order: labels are exact, sums and SSE_t are integers).
// Lane 0 runs a 3-stage prefetch pipeline: the index of tile i+2 (atomic), the id of tile i+1
// (work list load) and the copies of tile i+1, each consumed one tile later.
// FIRST (iteration 0: no previous labels) is a template parameter so that each instantiation
// carries only its own paths.  MINB (CTAs per SM the register budget targets): chosen by
// configure_tiles from the tile count (KM_DBG_K1T_MINB overrides).
template <int D, bool FIRST, int MINB>
__global__ void __launch_bounds__(kK1tThreads, MINB)
assign_tiles_kernel(const float* __restrict__ ps, int64_t n, const int* __restrict__ work,
                    int* __restrict__ work_cnt, const TileInfo* __restrict__ info,
                    TileState* __restrict__ tstate, const TileAux* __restrict__ aux, const float* __restrict__ tcand,
                    const CRec* __restrict__ pool, const NodeRef* __restrict__ l1ref, const float* __restrict__ C,
                    int k, int32_t* __restrict__ labels, unsigned long long* __restrict__ sseq_part,
                    unsigned long long* __restrict__ chg_part, unsigned long long* __restrict__ acc_sum,
                    unsigned int* __restrict__ acc_cnt, int ncopy, const CRec* __restrict__ ovf,
                    unsigned char* __restrict__ theavy, const Quant* __restrict__ quant, const Ctl* __restrict__ ctl,
                    unsigned long long* __restrict__ stats, int st_shift)
{
    acc_sum += (int64_t)(blockIdx.x % ncopy) * k * D;   // this CTA's private copy of the running sums
    acc_cnt += (int64_t)(blockIdx.x % ncopy) * k;
    if (ctl && ctl->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem<D>& S = reinterpret_cast<WarpSmem<D>*>(smem_raw)[w];
    const unsigned full = 0xffffffffu;
    constexpr bool first = FIRST;
    const bool want_labels = !first;
    // the work list: heavy tiles (work_cnt[5], stored downward from the top end) first, then the rest
    const int ntl = (int)((n + kTilePoints - 1) / kTilePoints);
    const int nheavy = work_cnt[5];
    const int nwork = work_cnt[0] + nheavy;
    auto entry = [&](int v) { return v < nheavy ? work[ntl - 1 - v] : work[v - nheavy]; };
    int* const wnext = work_cnt + 1;   // next unclaimed entry of the dynamic part
    const int W = gridDim.x * kK1tWarps, gw = blockIdx.x * kK1tWarps + w;
    const int nstatic = (int)((long long)nwork * KM_STATIC_FRAC / 100);
    // the dynamic part is claimed KM_CLAIM entries at a time (one atomic on the shared counter per
    // batch: with one per tile, ~2400 warps contending for that one address stalled the kernel)
    int bnext = 0, bend = 0;   // lane 0: the current batch of the dynamic part
    auto claim = [&](int prev) -> int {   // lane 0: the entry after prev (-1: first)
        const int nx = prev < 0 ? gw : prev + W;
        if (prev < nstatic && nx < nstatic) return nx;
        if (bnext >= bend) {
            bnext = nstatic + atomicAdd(wnext, KM_CLAIM);
            bend = bnext + KM_CLAIM;
        }
        return bnext++;
    };

    int cur_t = -1;
    int pf_t = -1, pf_idx = nwork;   // lane 0: id of tile i+1, index of tile i+2
    if (lane == 0) {
        const int i0 = claim(-1);
        if (i0 < nwork) {
            const int i1 = claim(i0);
            cur_t = entry(i0);
            if (i1 < nwork) {
                pf_t = entry(i1);
                pf_idx = claim(i1);
            }
        }
    }
    cur_t = __shfl_sync(full, cur_t, 0);
#if KM_K1T_BULK
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (cur_t >= 0) stage_tile_bulk<D>(&S.buf[0], &S.mbar[0], cur_t, info, tstate, aux, tcand, ps, labels, n, want_labels);
    }
    __syncwarp();
#else
    if (cur_t >= 0) stage_tile_cp<D>(&S.buf[0], cur_t, info, tstate, aux, tcand, ps, labels, n, want_labels, lane);
    cp_commit();
#endif
    // (the fixed-point origin and scales are read from the Quant record when a point moves:
    // keeping them in registers cost 12 of K1t's 128)
    const double ss = quant->sse_scale;
    const float ssf = (float)ss;
    const bool ssf_ok = ss >= 0x1p-100 && ss <= 0x1p100;   // FP32 quantisation of SSE_t summands is exact

    unsigned long long sq = 0, chg = 0;
    // per-warp work counters in shared memory (lane 0 updates them; in registers they cost 7 of 128)
    __shared__ unsigned int s_cntr[kK1tWarps][7];
    if (lane < 7) s_cntr[w][lane] = 0u;
    unsigned int* const cw = s_cntr[w];   // [0] pairs [1] points [2] batch [3] tiles [4] Eq. 4 [5] overflow [6] split

    for (int it = 0; cur_t >= 0; ++it) {
        const int t = cur_t;
        const int b = it & 1;
        int tn = -1;
        if (lane == 0) {
            tn = pf_t;
            // advance the pipeline: the load and the atomic are independent; both results are
            // consumed one tile later
            const int idx = pf_idx;
            pf_idx = idx < nwork ? claim(idx) : nwork;
            pf_t = idx < nwork ? entry(idx) : -1;
        }
        tn = __shfl_sync(full, tn, 0);
#if KM_K1T_BULK
        if (lane == 0 && tn >= 0)
            stage_tile_bulk<D>(&S.buf[b ^ 1], &S.mbar[b ^ 1], tn, info, tstate, aux, tcand, ps, labels, n, want_labels);
        k1t_bar_wait(&S.mbar[b], (uint32_t)(it >> 1) & 1u);   // tile i (the (it/2)-th use of buffer b) has landed
#else
        if (tn >= 0) stage_tile_cp<D>(&S.buf[b ^ 1], tn, info, tstate, aux, tcand, ps, labels, n, want_labels, lane);
        cp_commit();
        cp_wait<1>();   // pending: [tile i, tile i+1] -> tile i has landed
        __syncwarp();
#endif
        const auto& B = S.buf[b];
        const TileGeom g = B.info.g;
        const int64_t base = (int64_t)t * kTilePoints;
        const int i0 = 4 * lane;
        const int nvalid = max(0, min(4, g.cnt - i0));
        if (lane == 0) cw[3] += 1u;

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
        int oldv[4] = {0, 0, 0, 0};
        const int prev = first ? -1 : tile_lab(B.st);
        const int ncand = B.aux.ncand;
        bool skip = false;
        if (!first) {
            const int4 old = *reinterpret_cast<const int4*>(&B.lab[i0]);
            oldv[0] = old.x; oldv[1] = old.y; oldv[2] = old.z; oldv[3] = old.w;
            // (one candidate and a uniform previous label: the batch step below settles the
            // tile from its moments without the Eq. 4 pass over its points)
            if (prev >= 0 && ncand != 1) {
                // --- Eq. 4: ||p - c_a|| < cb[a] / 2 for every point keeps every label ----------
                // (the tile's previous labels were all a; the record {c_a, (cb[a]/2)^2 lower
                // bound} came with the tile; mixed tiles almost never pass for all 128 points)
                const float4 e = B.aux.pre;
                float dv[4];
                bool ok = true;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    dv[r] = 0.f;
                    if (r < nvalid) {
                        float tt = __fsub_rn(p[r].v[0], e.x);
                        float sd = __fmul_rn(tt, tt);
                        tt = __fsub_rn(p[r].v[1], e.y);
                        sd = __fmaf_rn(tt, tt, sd);
                        if (D == 3) { tt = __fsub_rn(p[r].v[D - 1], e.z); sd = __fmaf_rn(tt, tt, sd); }
                        dv[r] = sd;
                        ok = ok && sd < e.w;
                    }
                }
                skip = __all_sync(full, ok);
                if (skip) {
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (r < nvalid) sq += ssf_ok ? sse_qf(dv[r], ssf) : sse_q((double)dv[r], ss);
                    if (lane == 0) cw[4] += 1u;
                }
            }
        }

        const float* cblk = B.cand;
        const int* cjb = reinterpret_cast<const int*>(B.cand + D * kTC);
        if (skip) {
            // Eq. 4 settled every point: nothing else to do
        } else if (ncand == 1) {
            // --- batch assignment of the whole tile (Eq. 6 / Alg. 1) ---------
            const int cstar = cjb[0];
            if (first || prev != cstar) {
                int changed = 0;
                if (!first && prev < 0) {
                    for (int r = 0; r < nvalid; ++r) changed += oldv[r] != cstar;
                } else {
                    changed = nvalid;
                }
                chg += (unsigned long long)changed;
                if (nvalid == 4) *reinterpret_cast<int4*>(&labels[base + i0]) = make_int4(cstar, cstar, cstar, cstar);
                else for (int r = 0; r < nvalid; ++r) labels[base + i0 + r] = cstar;
            }
            const TileMom& mm = B.info.m;
            if (!first && prev < 0) {
                // mixed -> uniform: move the points that were elsewhere
                const int neu[4] = {cstar, cstar, cstar, cstar};
                move_points<D>(p, oldv, neu, nvalid, quant, acc_sum, acc_cnt);
            }
            if (lane == 0) {
                const float cc[3] = {-cblk[0], -cblk[kTC], D == 3 ? -cblk[2 * kTC] : 0.f};
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
                }
                if (prev != cstar) tile_lab_set(&tstate[t], cstar);
                cw[2] += 1u;
            }
        } else {
            // --- per-point scan over the candidates + FP64 certification ---------------------
            float m1[4], m2[4];
            int b1[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) { m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0; }
            const bool inblk = ncand <= kTC;
            const CRec* orecs = nullptr;   // more than kTC candidates: the overflow pool or the level-1 list
            int olen = ncand;
            if (inblk) {
                scan_block<D, kTC>(p, cblk, (ncand + 3) & ~3, m1, m2, b1);
            } else {
                if (lane == 0) cw[5] += 1u;
                const int off = B.aux.off;
                if (off >= 0) {
                    orecs = ovf + off;
                } else {   // pool full: the whole level-1 list (a superset of the candidates)
                    const NodeRef R = l1ref[t >> st_shift];
                    orecs = R.off >= 0 ? pool + R.off : nullptr;
                    olen = R.len;
                }
                // stage the candidates in chunks; group index = position / 4
                for (int e0 = 0; e0 < olen; e0 += kWCap) {
                    __syncwarp();
                    const int cl = min(kWCap, olen - e0), lp = (cl + 3) & ~3;
                    for (int s2 = lane; s2 < lp; s2 += 32) {
                        CRec c;
                        if (s2 < cl) c = get_rec<D>(orecs, C, e0 + s2);
                        S.cnc[0][s2] = s2 < cl ? -c.x : -INFINITY;
                        S.cnc[1][s2] = s2 < cl ? -c.y : -INFINITY;
                        if (D == 3) S.cnc[D - 1][s2] = s2 < cl ? -c.z : -INFINITY;
                    }
                    __syncwarp();
                    scan_slots<D>(p, S.cnc, lp, e0 >> 2, m1, m2, b1);
                }
            }
            int a[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                a[r] = 0;
                if (r < nvalid) {
                    const float thr = certify_thr(m1[r]);
                    if (inblk) {
                        // b1 is the FP32 argmin slot; every other slot has D32 >= m2
                        a[r] = m2[r] > thr ? cjb[b1[r]] : exact_scan_list<D>(p[r], C, cjb, 0, ncand);
                    } else if (!(m2[r] > thr)) {
                        a[r] = exact_scan_recs<D>(p[r], orecs, C, 0, olen);
                    } else {
                        const int s0 = b1[r] * 4;
                        int cn = 0, slot = 0x7fffffff;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int s2 = s0 + ((u + lane) & 3);
                            const float dv = s2 < olen ? dist32_rec<D>(p[r], get_rec<D>(orecs, C, s2)) : INFINITY;
                            if (dv <= thr) { ++cn; slot = min(slot, s2); }
                        }
                        a[r] = cn == 1 ? get_rec<D>(orecs, C, slot).j
                                       : exact_scan_recs<D>(p[r], orecs, C, s0, min(s0 + 4, olen));
                    }
                    // SSE_t summand: the certified FP32 distance (|D32 - D64| <= 1e-6 D64)
                    sq += ssf_ok ? sse_qf(m1[r], ssf) : sse_q((double)m1[r], ss);
                    chg += first ? 1u : (unsigned)(oldv[r] != a[r]);
                }
            }
            if (nvalid == 4) *reinterpret_cast<int4*>(&labels[base + i0]) = make_int4(a[0], a[1], a[2], a[3]);
            else for (int r = 0; r < nvalid; ++r) labels[base + i0 + r] = a[r];
            // is the whole tile on one label?  -> tile label state; sums from the tile moments
            const bool tu = nvalid == 0 || ((nvalid < 2 || a[1] == a[0]) && (nvalid < 3 || a[2] == a[0]) &&
                                            (nvalid < 4 || a[3] == a[0]));
            const int L = __shfl_sync(full, a[0], 0);   // lane 0 always has a valid point
            const bool uni = __all_sync(full, nvalid == 0 || (tu && a[0] == L));
            if (first) {
                if (uni) {
                    if (lane == 0) {
#pragma unroll
                        for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)L * D + m], B.info.m.q[m]);
                        atomicAdd(&acc_cnt[L], (unsigned int)g.cnt);
                    }
                } else {
                    accumulate_runs<D>(p, a, nvalid, false, L, *quant, acc_sum, acc_cnt);
                }
            } else {
                bool moved = false;
#pragma unroll
                for (int r = 0; r < 4; ++r) moved = moved || (r < nvalid && a[r] != oldv[r]);
                if (__any_sync(full, moved)) move_points<D>(p, oldv, a, nvalid, quant, acc_sum, acc_cnt);
            }
            if (lane == 0) {
                const int ns = uni ? L : -1;
                if (ns != prev) tile_lab_set(&tstate[t], ns);
                cw[0] += (unsigned)(g.cnt * olen);
                cw[1] += (unsigned)g.cnt;
            }
        }
        if (!skip && lane == 0) {
            theavy[t] = ncand > KM_HEAVY_CAND ? 1 : 0;
            cw[6] += g.pad[0] ? 1u : 0u;   // pruned with its two sub-balls
        }
        cur_t = tn;
        __syncwarp();   // the tile buffer b is reused next
    }
    double dummy = 0.0;
    block_sum2<kK1tThreads>(dummy, sq);
    __syncthreads();
    block_sum2<kK1tThreads>(dummy, chg);
    __shared__ unsigned long long s_st[7][kK1tWarps];
    if (lane == 0) {
        for (int c = 0; c < 7; ++c) s_st[c][w] = cw[c];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(sseq_part, sq);   // the iteration's totals (integers: order-independent)
        atomicAdd(chg_part, chg);
        if (stats) {
            unsigned long long v[7] = {0, 0, 0, 0, 0, 0, 0};
            for (int i = 0; i < kK1tWarps; ++i)
                for (int c = 0; c < 7; ++c) v[c] += s_st[c][i];
            for (int c = 0; c < 4; ++c) atomicAdd(&stats[c], v[c]);
            atomicAdd(&stats[13], v[4]);
            atomicAdd(&stats[14], v[5]);
            atomicAdd(&stats[29], v[6]);
        }
    }
}

}  // namespace km
