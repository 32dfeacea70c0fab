// km_tiles_assign.cuh -- K1t, the tile-pruned assignment + fused update (see km_tiles.cuh
// for the index and the pruning argument, km_levels.cuh for the parent lists).
// One warp = one tile (ball node) at a time; warps are independent (no CTA barrier in the
// loop).  Per tile, lane 0 keeps two TMA bulk-copy streams ahead of the warp:
//   * the NEXT tile's info (ball + moments), label state, points and previous labels
//     (double buffer, one mbarrier per buffer), issued when the current tile starts;
//   * the NEXT tile's parent list records {c, j} (single buffer, own mbarrier), issued
//     as soon as the current tile's prune has consumed the buffer.
// Then: prune the parent list with the tile ball (Eq. 7-8) -> batch (1 candidate, Eq. 6 /
// Alg. 1) or per-point packed scan + FP64 certification.
#pragma once
#include "km_tiles.cuh"
#include "km_levels.cuh"
#include "km_bounds.cuh"

// KM_PROF builds (tools only) accumulate clock64() per section into stats[4..9].
#ifdef KM_PROF
#define KM_TICK(v) const long long v = clock64()
#define KM_ACC(i, a, b) prof[i] += (unsigned long long)((b) - (a))
#else
#define KM_TICK(v)
#define KM_ACC(i, a, b)
#endif

#ifndef KM_PRUNE_REGQ
#define KM_PRUNE_REGQ 4   // lists up to 32 * KM_PRUNE_REGQ keep their delta^2 in registers during the prune
#endif

#ifndef KM_HEAVY_PLEN
#define KM_HEAVY_PLEN 512   // a tile pruning a longer level-1 list is scheduled first next iteration
#endif

#ifndef KM_STATIC_FRAC
#define KM_STATIC_FRAC 50   // percent of the work list assigned round-robin before atomic claiming
#endif

// Eq. 4 point pretest: 0 = every listed tile; 1 = tiles whose previous labels were uniform
// (default: a mixed tile almost never passes for all 128 points; config 4 -1.4 %); 2 = none
#ifndef KM_PRETEST_UNIFORM_ONLY
#define KM_PRETEST_UNIFORM_ONLY 1
#endif

#ifndef KM_LATE_STAGE
#define KM_LATE_STAGE 0   // 1: issue the next tile's bulk copies after the prune (tuning)
#endif

namespace km {

#ifndef KM_GU
#define KM_GU 2
#endif
constexpr int kGU = KM_GU;   // record loads in flight per lane when a list is read from global memory

template <int D>
__device__ __forceinline__ CRec get_rec(const CRec* recs, const float* __restrict__ C, int e)
{
    return recs ? recs[e] : make_rec<D>(C, e);
}

// Exact FP64 argmin over records [e0, e1) of a list (recs == nullptr: all k), lowest j on ties.
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
        if (s < best) { best = s; a = c.j; }
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

#ifndef KM_CPASYNC
#define KM_CPASYNC 1   // 1: per-lane 16-B cp.async copies; 0: one-lane TMA bulk copies + mbarriers
#endif

__device__ __forceinline__ void cp16(void* sdst, const void* gsrc)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// All lanes: 16-B async copies of tile t (points, previous labels, ball + moments, label state).
template <int D>
__device__ __forceinline__ void stage_tile_cp(typename WarpSmem<D>::Buf* buf, int t, const TileInfo* info,
                                              const TileState* tstate, const float* ps, const int32_t* labels,
                                              int64_t n, bool want_labels, int lane)
{
    const int64_t base = (int64_t)t * kTilePoints;
    const int cnt = (int)min((int64_t)kTilePoints, n - base);
    const int pch = (cnt * D * 4 + 15) >> 4;   // sources are padded to 16 B in HBM
    const char* src = reinterpret_cast<const char*>(ps + base * D);
    char* dst = reinterpret_cast<char*>(buf->pts);
    for (int c = lane; c < pch; c += 32) cp16(dst + 16 * c, src + 16 * c);
    if (want_labels && lane < ((cnt * 4 + 15) >> 4)) cp16(buf->lab + 4 * lane, labels + base + 4 * lane);
    if (lane < (int)(sizeof(TileInfo) / 16))
        cp16(reinterpret_cast<char*>(&buf->info) + 16 * lane, reinterpret_cast<const char*>(info + t) + 16 * lane);
    else if (lane == 31)
        cp16(&buf->st, tstate + t);
}

// Issue the bulk copy of a level-1 list into the warp's list buffer (lane 0).
__device__ __forceinline__ bool stage_list(float4* dst, unsigned long long* bar, const CRec* pool, const NodeRef& R)
{
    if (R.off < 0 || R.len <= 0 || R.len > kL1Cap) return false;
#ifndef KM_NO_PROXY_FENCE
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
    mbar_expect_tx(bar, (uint32_t)R.len * 16u);
    bulk_g2s(dst, pool + R.off, (uint32_t)R.len * 16u, bar);
    return true;
}

// Packed scan of 4 points over candidate slots [0, nslots) tracking, per point, the FP32
// minimum m1, its FIRST slot b1 and the second-smallest value m2 over all other slots.
template <int D>
__device__ __forceinline__ void scan_slots_exact(const Pt<D> (&p)[4], const float (*cnc)[kWCap], int nslots,
                                                 float (&m1)[4], float (&m2)[4], int (&b1)[4])
{
    for (int gi = 0; gi < (nslots >> 2); ++gi) {
        float4 c[D];
#pragma unroll
        for (int m = 0; m < D; ++m) c[m] = reinterpret_cast<const float4*>(cnc[m])[gi];
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
                                            const Quant& q, unsigned long long* __restrict__ acc_sum,
                                            unsigned int* __restrict__ acc_cnt)
{
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (r < nvalid && old[r] != neu[r]) {
#pragma unroll
            for (int m = 0; m < D; ++m) {
                const unsigned long long qv = (unsigned long long)__double2ll_rn(
                    __dmul_rn(__dsub_rn((double)p[r].v[m], q.o[m]), q.scale[m]));
                atomicAdd(&acc_sum[(int64_t)neu[r] * D + m], qv);
                atomicAdd(&acc_sum[(int64_t)old[r] * D + m], 0ull - qv);
            }
            atomicAdd(&acc_cnt[neu[r]], 1u);
            atomicAdd(&acc_cnt[old[r]], 0xffffffffu);
        }
    }
}

// K1t.  Tiles come from the work list of tile_filter_kernel (those not settled by Eq. 5);
// warps take entries dynamically (atomic counter; results do not depend on the order: labels
// are exact, sums and SSE_t are integers).  Lane 0 runs a 3-stage prefetch pipeline: the
// index of tile i+2 (atomic), the id of tile i+1 (work list load) and the TMA copies of tile
// i+1, each consumed one tile later so its latency hides behind tile i.  Per tile:
//   0. (t > 0) Eq. 4 for every point against its previous centroid: all pass -> labels,
//      sums and tile state unchanged, SSE_t from the FP32 distances; done.
//   1. prune the parent list with the tile ball (Eq. 7-8) -> one candidate: batch (Eq. 6);
//      otherwise per-point packed scan over the candidates + FP64 certification.
//   2. sums: iteration 0 adds every point (tile moments when the tile is uniform);
//      later iterations move only the points whose label changed (incremental sv(j)).
#ifndef KM_K1T_MINB
#define KM_K1T_MINB 2
#endif
// FIRST (iteration 0: no previous labels) is a template parameter so that each instantiation
// carries only its own paths (smaller hot loop for the instruction caches).
// MINB (CTAs per SM the register budget targets): 2 (128 registers, 16 warps/SM) for large
// problems; 1 (no spills, 8 warps/SM) measured faster when there are few tiles (config 3:
// 0.088 -> 0.078 ms/iter; config 4 prefers 2), chosen by configure_tiles.
template <int D, bool FIRST, int MINB = KM_K1T_MINB>
__global__ void __launch_bounds__(kTileThreads, MINB)
assign_tiles_kernel(const float* __restrict__ ps, int64_t n, const int* __restrict__ work,
                    int* __restrict__ work_cnt, const TileInfo* __restrict__ info,
                    TileState* __restrict__ tstate, const CRec* __restrict__ pool,
                    const NodeRef* __restrict__ l1ref, const float* __restrict__ C, int k,
                    const unsigned int* __restrict__ cb2, const float* __restrict__ cpk, int32_t* __restrict__ labels,
                    unsigned long long* __restrict__ sseq_part, unsigned long long* __restrict__ chg_part,
                    unsigned long long* __restrict__ acc_sum, unsigned int* __restrict__ acc_cnt, int ncopy,
                    CRec* __restrict__ ovf, int* __restrict__ ovf_cursor, int ovf_cap, unsigned char* __restrict__ theavy,
                    const Quant* __restrict__ quant, const Ctl* __restrict__ ctl,
                    unsigned long long* __restrict__ stats, int st_shift)
{
    acc_sum += (int64_t)(blockIdx.x % ncopy) * k * D;   // this CTA's private copy of the running sums
    acc_cnt += (int64_t)(blockIdx.x % ncopy) * k;
    if (ctl && ctl->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem<D>& S = reinterpret_cast<WarpSmem<D>*>(smem_raw)[w];
    const CRec* slst = reinterpret_cast<const CRec*>(S.lst);
    const unsigned full = 0xffffffffu;
    const unsigned ltmask = (1u << lane) - 1u;
    constexpr bool first = FIRST;
    const bool want_labels = !first;
    // the work list: heavy tiles (work_cnt[5], stored downward from the top end) first, then the rest
    const int ntl = (int)((n + kTilePoints - 1) / kTilePoints);
    const int nheavy = work_cnt[5];
    const int nwork = work_cnt[0] + nheavy;
    auto entry = [&](int v) { return v < nheavy ? work[ntl - 1 - v] : work[v - nheavy]; };
    int* const wnext = work_cnt + 1;   // next unclaimed entry of the dynamic part
    // work-list entries [0, nstatic) go round-robin (warp gw: gw, gw + W, ...; no atomics), the
    // rest is claimed one entry at a time through an atomic counter (balances the tail)
    const int W = gridDim.x * kWarpsPerCta, gw = blockIdx.x * kWarpsPerCta + w;
    const int nstatic = (int)((long long)nwork * KM_STATIC_FRAC / 100);
    auto claim = [&](int prev) -> int {   // lane 0: the entry after prev (-1: first)
        const int nx = prev < 0 ? gw : prev + W;
        if (prev < nstatic && nx < nstatic) return nx;
        return nstatic + atomicAdd(wnext, 1);
    };

    // current tile's parent list: (off, len) and whether it sits in S.lst
    long long cur_off = 0;
    int cur_len = 0, cur_sm = 0, cur_t = -1;
    int pf_t = -1, pf_idx = nwork;     // lane 0: id of tile i+1, index of tile i+2
#if KM_CPASYNC
    if (lane == 0) {
        const int i0 = claim(-1);
        if (i0 < nwork) {
            const int i1 = claim(i0);
            cur_t = entry(i0);
            if (i1 < nwork) {
                pf_t = entry(i1);
                pf_idx = claim(i1);
            }
            const NodeRef R = l1ref[cur_t >> st_shift];
            cur_off = R.off;
            cur_len = R.len;
            cur_sm = R.off >= 0 && R.len > 0 && R.len <= kL1Cap;
        }
    }
    cur_off = __shfl_sync(full, cur_off, 0);
    cur_len = __shfl_sync(full, cur_len, 0);
    cur_sm = __shfl_sync(full, cur_sm, 0);
    cur_t = __shfl_sync(full, cur_t, 0);
    if (cur_t >= 0) stage_tile_cp<D>(&S.buf[0], cur_t, info, tstate, ps, labels, n, want_labels, lane);
    cp_commit();
    if (cur_sm)
        for (int e = lane; e < cur_len; e += 32) cp16(&S.lst[e], pool + cur_off + e);
    cp_commit();
#else
    if (lane == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        mbar_init(&S.lbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int i0 = claim(-1);
        if (i0 < nwork) {
            const int i1 = claim(i0);
            cur_t = entry(i0);
            if (i1 < nwork) {
                pf_t = entry(i1);
                pf_idx = claim(i1);
            }
            stage_tile<D>(&S.buf[0], &S.bar[0], cur_t, info, tstate, ps, labels, n, want_labels);
            const NodeRef R = l1ref[cur_t >> st_shift];
            cur_off = R.off;
            cur_len = R.len;
            cur_sm = stage_list(S.lst, &S.lbar, pool, R) ? 1 : 0;
        }
    }
    cur_off = __shfl_sync(full, cur_off, 0);
    cur_len = __shfl_sync(full, cur_len, 0);
    cur_sm = __shfl_sync(full, cur_sm, 0);
    cur_t = __shfl_sync(full, cur_t, 0);
#endif
    const Quant q = *quant;
    const double ss = q.sse_scale;
    const float ssf = (float)ss;
    const bool ssf_ok = ss >= 0x1p-100 && ss <= 0x1p100;   // FP32 quantisation of SSE_t summands is exact

    unsigned long long sq = 0, chg = 0;
    unsigned int st_pairs = 0, st_pts = 0, st_batch = 0, st_tiles = 0, st_plen = 0, st_sm = 0, st_pskip = 0, st_gl = 0,
                 st_glplen = 0, st_split = 0;   // per-warp work counters (32 bit: fewer registers)
    uint32_t phase[2] = {0u, 0u}, lphase = 0u;
#ifdef KM_PROF
    unsigned long long prof[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

    int it = 0;
    for (; cur_t >= 0; ++it) {
        KM_TICK(t0);
        const int t = cur_t;
        const int b = it & 1;
        int tn = -1;
        NodeRef nref;
        nref.off = -1; nref.len = 0;
        if (lane == 0) {
            tn = pf_t;
            if (tn >= 0) {
#if !KM_LATE_STAGE && !KM_CPASYNC
                stage_tile<D>(&S.buf[b ^ 1], &S.bar[b ^ 1], tn, info, tstate, ps, labels, n, want_labels);
#endif
                nref = l1ref[tn >> st_shift];   // consumed after the prune: latency hidden
            }
            // advance the pipeline: the load and the atomic are independent; both results are
            // consumed one tile later
            const int idx = pf_idx;
            pf_idx = idx < nwork ? claim(idx) : nwork;
            pf_t = idx < nwork ? entry(idx) : -1;
        }
        const CRec* grecs = cur_off >= 0 ? pool + cur_off : nullptr;   // global view of the list
        const int plen = cur_len;
        __syncwarp();
        KM_TICK(t0l);
        KM_ACC(12, t0, t0l);
#if KM_CPASYNC
        tn = __shfl_sync(full, tn, 0);
        if (tn >= 0) stage_tile_cp<D>(&S.buf[b ^ 1], tn, info, tstate, ps, labels, n, want_labels, lane);
        cp_commit();
        KM_TICK(t0a);
        KM_ACC(10, t0, t0a);
        cp_wait<2>();   // pending: [tile i, list i, tile i+1] -> tile i has landed
        __syncwarp();
        KM_TICK(t0b);
        KM_ACC(11, t0a, t0b);
#else
        KM_TICK(t0a);
        KM_ACC(10, t0, t0a);
        if (cur_sm) { mbar_wait(&S.lbar, lphase); lphase ^= 1u; }
        KM_TICK(t0b);
        KM_ACC(11, t0a, t0b);
        mbar_wait(&S.bar[b], phase[b]);
        phase[b] ^= 1u;
#endif
        const auto& B = S.buf[b];
        const TileGeom g = B.info.g;
        const int64_t base = (int64_t)t * kTilePoints;
        const int i0 = 4 * lane;
        const int nvalid = max(0, min(4, g.cnt - i0));
        ++st_tiles;
        KM_TICK(t1);
        KM_ACC(0, t0, t1);

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
        bool skip = false;
        if (!first) {
            const int4 old = *reinterpret_cast<const int4*>(&B.lab[i0]);
            oldv[0] = old.x; oldv[1] = old.y; oldv[2] = old.z; oldv[3] = old.w;
            // --- Eq. 4: ||p - c_a(i)|| < cb[a(i)] / 2 for every point keeps every label ------
            float dv[4];
#if KM_PRETEST_UNIFORM_ONLY == 2
            bool ok = false;                 // (tuning) no point pretest
#elif KM_PRETEST_UNIFORM_ONLY
            bool ok = tile_lab(B.st) >= 0;   // (tuning) mixed tiles rarely pass for every point
#else
            bool ok = true;
#endif
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                dv[r] = 0.f;
                if (r < nvalid) {
                    // one 16-B load: {c_a, (cb[a]/2)^2 lower bound} packed by tile_filter_kernel
                    const float4 e = __ldg(reinterpret_cast<const float4*>(cpk) + oldv[r]);
                    float t = __fsub_rn(p[r].v[0], e.x);
                    float sd = __fmul_rn(t, t);
                    t = __fsub_rn(p[r].v[1], e.y);
                    sd = __fmaf_rn(t, t, sd);
                    if (D == 3) { t = __fsub_rn(p[r].v[D - 1], e.z); sd = __fmaf_rn(t, t, sd); }
                    dv[r] = sd;
                    ok = ok && sd < e.w;
                }
            }
            skip = __all_sync(full, ok);
            if (skip) {
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    if (r < nvalid) sq += ssf_ok ? sse_qf(dv[r], ssf) : sse_q((double)dv[r], ss);
                st_pskip += lane == 0;
            }
        }

        KM_TICK(t1b);
        KM_ACC(6, t1, t1b);
#if KM_CPASYNC
        cp_wait<1>();   // the list of tile i has landed (tile i+1 may still be in flight)
        __syncwarp();
#endif
        int ncand = 0, cfirst = -1;
        bool overflow = false;
        float T2 = 0.f, T2b = -1.f;   // T2b >= 0: second sub-ball threshold (split tiles)
        auto keep = [&](const CRec& c) {
            return T2b >= 0.f ? (rec_delta2<D>(B.info.sb.o1, c) <= T2 || rec_delta2<D>(B.info.sb.o2, c) <= T2b)
                              : rec_delta2<D>(g.o, c) <= T2;
        };
        const CRec* orecs = grecs;   // overflow scan: the candidates (pool) or the whole parent list
        int olen = plen;
        if (!skip) {
            // --- warp prune of the parent's list with the tile ball (Eq. 7-8) ---------------
            st_plen += (unsigned)plen;
            st_sm += (unsigned)cur_sm;
            auto emit = [&](bool f, const CRec& c) {
                const unsigned bal = __ballot_sync(full, f);
                if (f) {
                    const int off = ncand + __popc(bal & ltmask);
                    if (off < kWCap) {
                        S.cnc[0][off] = -c.x;
                        S.cnc[1][off] = -c.y;
                        if (D == 3) S.cnc[D - 1][off] = -c.z;
                        S.cj[off] = c.j;
                    }
                    if (off == 0) cfirst = c.j;
                }
                ncand += __popc(bal);
            };
            if (g.pad[0]) {
                // a tile split at a Morton jump: keep j if it can be nearest to a point of EITHER
                // sub-ball (the union of the two Eq. 7-8 tests; both balls cover their points)
                const TileSub sb = B.info.sb;
                st_split += lane == 0;
                auto rec = [&](int e) { return cur_sm ? slst[e] : get_rec<D>(grecs, C, e); };
                float dm1 = INFINITY, dm2 = INFINITY;
                for (int e = lane; e < plen; e += 32) {
                    const CRec c = rec(e);
                    dm1 = fminf(dm1, rec_delta2<D>(sb.o1, c));
                    dm2 = fminf(dm2, rec_delta2<D>(sb.o2, c));
                }
                dm1 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dm1)));
                dm2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dm2)));
                T2 = prune_thr2(dm1, sb.r1);
                T2b = prune_thr2(dm2, sb.r2);
                for (int e0 = 0; e0 < plen; e0 += 32) {
                    const int e = e0 + lane;
                    CRec c;
                    bool f = false;
                    if (e < plen) { c = rec(e); f = keep(c); }
                    emit(f, c);
                }
            } else if (cur_sm && plen <= 32 * KM_PRUNE_REGQ) {
                // single pass over the shared-memory list: delta^2 kept in registers
                constexpr int kQ = KM_PRUNE_REGQ;
                float dvq[kQ];
                float dmin2 = INFINITY;
#pragma unroll
                for (int qq = 0; qq < kQ; ++qq) {
                    if (qq * 32 >= plen) break;
                    const int e = qq * 32 + lane;
                    dvq[qq] = e < plen ? rec_delta2<D>(g.o, slst[e]) : INFINITY;
                    dmin2 = fminf(dmin2, dvq[qq]);
                }
                dmin2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dmin2)));   // >= 0: uint order
                T2 = prune_thr2(dmin2, g.r);
#pragma unroll
                for (int qq = 0; qq < kQ; ++qq) {
                    if (qq * 32 >= plen) break;
                    const int e = qq * 32 + lane;
                    const bool f = dvq[qq] <= T2;
                    CRec c;
                    if (f) c = slst[e];
                    emit(f, c);
                }
            } else {
                // long list (in shared memory beyond the register cache, or in global memory,
                // L2-resident): two passes, kGU independent record loads per lane in flight
                auto rec = [&](int e) { return cur_sm ? slst[e] : get_rec<D>(grecs, C, e); };
                float dmin2 = INFINITY;
                for (int e0 = 0; e0 < plen; e0 += 32 * kGU) {
                    CRec cr[kGU];
#pragma unroll
                    for (int u = 0; u < kGU; ++u) {
                        const int e = e0 + 32 * u + lane;
                        if (e < plen) cr[u] = rec(e);
                    }
#pragma unroll
                    for (int u = 0; u < kGU; ++u)
                        if (e0 + 32 * u + lane < plen) dmin2 = fminf(dmin2, rec_delta2<D>(g.o, cr[u]));
                }
#pragma unroll
                for (int of = 16; of > 0; of >>= 1) dmin2 = fminf(dmin2, __shfl_xor_sync(full, dmin2, of));
                T2 = prune_thr2(dmin2, g.r);
                for (int e0 = 0; e0 < plen; e0 += 32 * kGU) {
                    CRec cr[kGU];
#pragma unroll
                    for (int u = 0; u < kGU; ++u) {
                        const int e = e0 + 32 * u + lane;
                        if (e < plen) cr[u] = rec(e);
                    }
#pragma unroll
                    for (int u = 0; u < kGU; ++u) {
                        if (e0 + 32 * u >= plen) break;
                        const bool f = e0 + 32 * u + lane < plen && rec_delta2<D>(g.o, cr[u]) <= T2;
                        emit(f, cr[u]);
                    }
                }
            }
            overflow = ncand > kWCap || ncand == 0;
            if (ncand > kWCap) {
                // more candidates than the shared buffer: compact them (ascending j) into the
                // overflow pool so the scan and the FP64 fallback see only candidates
                int off = 0;
                if (lane == 0) off = atomicAdd(ovf_cursor, ncand);
                off = __shfl_sync(full, off, 0);
                if ((long long)off + ncand <= (long long)ovf_cap) {
                    int cnt = 0;
                    for (int e0 = 0; e0 < plen; e0 += 32) {
                        const int e = e0 + lane;
                        CRec c;
                        bool f = false;
                        if (e < plen) { c = cur_sm ? slst[e] : get_rec<D>(grecs, C, e); f = keep(c); }
                        const unsigned bal = __ballot_sync(full, f);
                        if (f) ovf[off + cnt + __popc(bal & ltmask)] = c;
                        cnt += __popc(bal);
                    }
                    __syncwarp();
                    orecs = ovf + off;
                    olen = ncand;
                }
            }
            if (!overflow) {
                const int padded = (ncand + 3) & ~3;
                if (lane < padded - ncand) {
#pragma unroll
                    for (int m = 0; m < D; ++m) S.cnc[m][ncand + lane] = -INFINITY;
                    S.cj[ncand + lane] = 0x7fffffff;
                }
            }
        }
        if (!skip && lane == 0) theavy[t] = (plen > KM_HEAVY_PLEN || ncand > kWCap) ? 1 : 0;
        __syncwarp();
        KM_TICK(t2a);
        KM_ACC(7, t1b, t2a);
        if (!skip) {
            if (cur_sm) { KM_ACC(8, t1b, t2a); } else { KM_ACC(9, t1b, t2a); st_gl += 1; st_glplen += plen; }
        }
        // the list buffer is free: bring in the next tile's parent list
        int nsm = 0;
#if KM_CPASYNC
        const long long n_off = __shfl_sync(full, nref.off, 0);
        const int n_len = __shfl_sync(full, nref.len, 0);
        nsm = tn >= 0 && n_off >= 0 && n_len > 0 && n_len <= kL1Cap;
        if (nsm)
            for (int e = lane; e < n_len; e += 32) cp16(&S.lst[e], pool + n_off + e);
        cp_commit();
#else
        if (lane == 0 && tn >= 0) {
#if KM_LATE_STAGE
            stage_tile<D>(&S.buf[b ^ 1], &S.bar[b ^ 1], tn, info, tstate, ps, labels, n, want_labels);
#endif
            nsm = stage_list(S.lst, &S.lbar, pool, nref) ? 1 : 0;
        }
        const long long n_off = __shfl_sync(full, nref.off, 0);
        const int n_len = __shfl_sync(full, nref.len, 0);
        nsm = __shfl_sync(full, nsm, 0);
        tn = __shfl_sync(full, tn, 0);
#endif
        KM_TICK(t2);
        KM_ACC(1, t2a, t2);

        if (skip) {
            // Eq. 4 settled every point: nothing else to do
        } else if (ncand == 1) {
            // --- batch assignment of the whole tile (Eq. 6 / Alg. 1) ---------
            const int cstar = __shfl_sync(full, cfirst, __ffs(__ballot_sync(full, cfirst >= 0)) - 1);
            const int prev = tile_lab(B.st);
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
                move_points<D>(p, oldv, neu, nvalid, q, acc_sum, acc_cnt);
            }
            if (lane == 0) {
                const float cc[3] = {-S.cnc[0][0], -S.cnc[1][0], D == 3 ? -S.cnc[D - 1][0] : 0.f};
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
                st_batch += 1;
            }
            KM_TICK(t3);
            KM_ACC(2, t2, t3);
        } else {
            // --- per-point scan over the candidates (the parent list, chunked, on overflow) ----
            float m1[4], m2[4];
            int b1[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) { m1[r] = INFINITY; m2[r] = INFINITY; b1[r] = 0; }
            if (!overflow) {
                scan_slots_exact<D>(p, S.cnc, (ncand + 3) & ~3, m1, m2, b1);
            } else {
                // stage the candidates (pool) or the parent list in chunks; group index = position / 4
                for (int e0 = 0; e0 < olen; e0 += kWCap) {
                    __syncwarp();
                    const int cl = min(kWCap, olen - e0), lp = (cl + 3) & ~3;
                    for (int s = lane; s < lp; s += 32) {
                        CRec c;
                        if (s < cl) c = get_rec<D>(orecs, C, e0 + s);
                        S.cnc[0][s] = s < cl ? -c.x : -INFINITY;
                        S.cnc[1][s] = s < cl ? -c.y : -INFINITY;
                        if (D == 3) S.cnc[D - 1][s] = s < cl ? -c.z : -INFINITY;
                    }
                    __syncwarp();
                    scan_slots<D>(p, S.cnc, lp, e0 >> 2, m1, m2, b1);
                }
            }
            KM_TICK(t3);
            KM_ACC(3, t2, t3);
            int a[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                a[r] = 0;
                if (r < nvalid) {
                    const float thr = certify_thr(m1[r]);
                    if (!overflow) {
                        // b1 is the FP32 argmin slot; every other slot has D32 >= m2
                        a[r] = m2[r] > thr ? S.cj[b1[r]] : exact_scan_list<D>(p[r], C, S.cj, 0, ncand);
                    } else if (!(m2[r] > thr)) {
                        a[r] = exact_scan_recs<D>(p[r], orecs, C, 0, olen);
                    } else {
                        const int s0 = b1[r] * 4;
                        int cn = 0, slot = 0x7fffffff;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int s = s0 + ((u + lane) & 3);
                            const float dv = s < olen ? dist32_rec<D>(p[r], get_rec<D>(orecs, C, s)) : INFINITY;
                            if (dv <= thr) { ++cn; slot = min(slot, s); }
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
            KM_TICK(t4);
            KM_ACC(4, t3, t4);
            if (first) {
                if (uni) {
                    if (lane == 0) {
#pragma unroll
                        for (int m = 0; m < D; ++m) atomicAdd(&acc_sum[(int64_t)L * D + m], B.info.m.q[m]);
                        atomicAdd(&acc_cnt[L], (unsigned int)g.cnt);
                    }
                } else {
                    accumulate_runs<D>(p, a, nvalid, false, L, q, acc_sum, acc_cnt);
                }
            } else {
                bool moved = false;
#pragma unroll
                for (int r = 0; r < 4; ++r) moved = moved || (r < nvalid && a[r] != oldv[r]);
                if (__any_sync(full, moved)) move_points<D>(p, oldv, a, nvalid, q, acc_sum, acc_cnt);
            }
            KM_TICK(t5);
            KM_ACC(5, t4, t5);
            if (lane == 0) {
                const int ns = uni ? L : -1;
                if (ns != tile_lab(B.st)) tile_lab_set(&tstate[t], ns);
                st_pairs += (unsigned)(g.cnt * (overflow ? olen : ncand));
                st_pts += (unsigned)g.cnt;
            }
        }
        cur_off = n_off;
        cur_len = n_len;
        cur_sm = nsm;
        cur_t = tn;
        __syncwarp();   // the candidate buffer and tile buffer b are reused next
#ifdef KM_PROF
        {   // per-tile duration histogram: [24] > 20k cycles, [25] > 50k, [26] > 200k, [27] max, [28] cycles in > 50k tiles
            KM_TICK(tz);
            const unsigned long long dt = (unsigned long long)(tz - t0);
            if (lane == 0 && stats) {
                if (dt > 20000) atomicAdd(&stats[24], 1ull);
                if (dt > 50000) { atomicAdd(&stats[25], 1ull); atomicAdd(&stats[28], dt); }
                if (dt > 200000) atomicAdd(&stats[26], 1ull);
                atomicMax(&stats[27], dt);
            }
        }
#endif
    }
    double dummy = 0.0;
    block_sum2<kTileThreads>(dummy, sq);
    __syncthreads();
    block_sum2<kTileThreads>(dummy, chg);
    __shared__ unsigned long long s_st[5][kWarpsPerCta];
    if (lane == 0) {
        s_st[0][w] = st_pairs; s_st[1][w] = st_pts; s_st[2][w] = st_batch; s_st[3][w] = st_tiles;
        s_st[4][w] = st_pskip;
    }
#ifdef KM_PROF
    if (lane == 0 && stats)
    {
        for (int i = 0; i < 6; ++i) atomicAdd(&stats[4 + i], prof[i]);
        atomicAdd(&stats[14], prof[6]);
        atomicAdd(&stats[15], prof[7]);
        atomicAdd(&stats[16], prof[8]);
        atomicAdd(&stats[17], prof[9]);
        atomicAdd(&stats[20], prof[10]);
        atomicAdd(&stats[21], prof[11]);
        atomicAdd(&stats[23], prof[12]);
    }
#endif
    if (lane == 0 && stats) {
        atomicAdd(&stats[10], (unsigned long long)st_plen); atomicAdd(&stats[11], (unsigned long long)st_sm);
        atomicAdd(&stats[18], (unsigned long long)st_gl); atomicAdd(&stats[19], (unsigned long long)st_glplen);
        atomicAdd(&stats[29], (unsigned long long)st_split);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(sseq_part, sq);   // the iteration's totals (integers: order-independent)
        atomicAdd(chg_part, chg);
        if (stats) {
            unsigned long long v[5] = {0, 0, 0, 0, 0};
            for (int i = 0; i < kWarpsPerCta; ++i)
                for (int c = 0; c < 5; ++c) v[c] += s_st[c][i];
            for (int c = 0; c < 4; ++c) atomicAdd(&stats[c], v[c]);
            atomicAdd(&stats[13], v[4]);
        }
    }
}

}  // namespace km
