// km_levels.cuh -- the upper levels of the point index: a flat tree whose level-0 nodes are
// the tiles (128 sorted points) and whose level-l node covers lev_fan[l] consecutive
// level-(l-1) nodes (level 1: 8 or 16 tiles, above: kFanout).  Every node is a ball
// (o, r) bounding all its points; per iteration each node keeps the centroids that can be
// nearest to one of its points, pruned from its PARENT's list -- the kNN bounds inherited
// from parent nodes of Eq. 7-8, evaluated top-down, the roots pruning all k.
//
// Lists hold records {c_x, c_y, c_z, j} (ascending j) so that a child prunes and scans
// from one contiguous, TMA-copyable block without gathering C.  NodeRef {off, len}:
// off >= 0 -> pool[off .. off+len); off < 0 -> all k (read C directly).  A node whose list
// would exceed its capacity inherits its parent's reference (a correct superset).
#pragma once
#include "km_tiles.cuh"

namespace km {

constexpr int kFanout = 16;   // children per node above level 1
constexpr int kL1Store = 1024; // level-1 list storage per node (longer lists inherit the parent's)

struct __align__(16) CRec {
    float x, y, z;
    int j;
};

struct __align__(16) NodeRef {
    long long off;
    int len;
    int pad;
};

template <int D>
__device__ __forceinline__ CRec make_rec(const float* __restrict__ C, int j)
{
    CRec r;
    r.x = __ldg(C + (int64_t)j * D);
    r.y = __ldg(C + (int64_t)j * D + 1);
    r.z = D == 3 ? __ldg(C + (int64_t)j * D + 2) : 0.f;
    r.j = j;
    return r;
}

template <int D>
__device__ __forceinline__ float rec_delta2(const float (&o)[3], const CRec& c)
{
    float t1 = __fsub_rn(o[0], c.x);
    float s = __fmul_rn(t1, t1);
    t1 = __fsub_rn(o[1], c.y);
    s = __fmaf_rn(t1, t1, s);
    if (D == 3) { t1 = __fsub_rn(o[2], c.z); s = __fmaf_rn(t1, t1, s); }
    return s;
}

// Per-tile candidate lists, computed where the level-1 node's list already is (Eq. 7-8 with the
// tile's ball, or the union of its two sub-balls, against the node's list; the bounds the tile
// inherits from its parent): one warp, up to 8 tiles per pass -- each list record
// is loaded once and tested against every ball.  The test and the threshold are exactly the
// tile-level prune of DESIGN.md 3b (rec_delta2, prune_thr2), so the candidate set contains the
// FP64 argmin of every point of the tile and all its ties.  Up to kTC candidates go to the
// tile's SoA block (negated coordinates, indices; ascending j; padded to a multiple of 4 with
// -inf / INT_MAX); more go to the overflow pool as CRec records (ascending j).
struct TileCandOut {
    const TileInfo* info;
    float* tcand;        // [ntiles][(D + 1) * kTC]
    TileAux* aux;        // [ntiles]
    CRec* ovf;           // overflow pool
    int* ovf_cur;        // [8]: [0] its cursor, [1] the flat prune's node counter, [2] heavy nodes, [3] tile_cands_kernel's
                         // item counter, [4] heavy nodes with multi-pass lists (all reset every iteration
                         // before the level-1 prune)
    int* heavy;          // [nnodes] level-1 nodes whose list is longer than kShortList: from index 0 upward,
                         // those with multi-pass lists (queue_heavy) from the top end downward
    int ovf_cap;
    int ntiles;
    int st_shift;        // tiles per level-1 node = 1 << st_shift
    unsigned long long* stats;   // [10] summed node-list lengths, [11] nodes, [15] tile candidates (nullable)
    int nnodes;          // level-1 nodes
    int short_list;      // lists up to this length (<= kShortList) get their tiles' candidates in the prune kernel
};

// once per warp at the end of a level-1 prune kernel (no per-tile global atomics)
__device__ __forceinline__ void flush_cand_stats(const TileCandOut& out, unsigned long long (&st)[3])
{
    if (!out.stats) return;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) st[i] += __shfl_xor_sync(0xffffffffu, st[i], o);
    if ((threadIdx.x & 31) == 0) {
        if (st[1] | st[2]) {   // (tile_cands_kernel's warps count candidates only)
            atomicAdd(&out.stats[10], st[0]);
            atomicAdd(&out.stats[11], st[1]);
            atomicAdd(&out.stats[15], st[2]);
        }
    }
}

template <int D>
__device__ __forceinline__ float ball_delta2(const float4& b, const CRec& c)
{
    const float o[3] = {b.x, b.y, b.z};
    return rec_delta2<D>(o, c);
}

// get(e): record e of the node's list (in whatever memory holds it).  Lane layout: 4 lanes per
// tile, 8 tiles per pass; each lane scans every 4th record of the list against its tile's ball
// (split tiles: both sub-balls), the group's minimum gives the threshold, and the kept records
// are appended through a shared-memory counter.  The order of a tile's candidates is therefore
// not fixed; nothing depends on it: the scan keeps the FP32 minimum (order-free), certification
// accepts only a unique FP32 winner, and every FP64 decision breaks ties by the lowest j.
// st[3] (per lane, flushed by the caller once per warp): summed list lengths, nodes, candidates.
// Long lists (L > kShortList): one tile at a time, the 32 lanes over the records (ballot
// compaction in list order), so that a node with a long list is not a long serial chain.
#ifndef KM_SHORT_LIST
#define KM_SHORT_LIST 64
#endif
#ifndef KM_TC_RQ
#define KM_TC_RQ 4          // tile_cands_long: list records per lane held in registers (8: +0.5 % / +1.1 % at configs 4 / 5)
#endif
#ifndef KM_TC_MINB
#define KM_TC_MINB 1        // tile_cands_kernel: CTAs per SM the register budget targets
#endif
#ifndef KM_TC_LPT
#define KM_TC_LPT 1        // multi-pass lists queued first (config 4: tile_cands_kernel 23.8 -> 23.0 us; config 5 -0.7 % per run)
#endif
constexpr int kShortList = KM_SHORT_LIST;

// One thread: queue level-1 node v (list length L > kShortList) for tile_cands_kernel.  Lists
// that take several load rounds per tile (L > 32 * KM_TC_RQ) are stored from the top end of
// heavy[] and taken first, so the longest items start first instead of forming the kernel's tail.
__device__ __forceinline__ void queue_heavy(const TileCandOut& tco, int v, int L)
{
    if (KM_TC_LPT && L > 32 * KM_TC_RQ) tco.heavy[tco.nnodes - 1 - atomicAdd(tco.ovf_cur + 4, 1)] = v;
    else tco.heavy[atomicAdd(tco.ovf_cur + 2, 1)] = v;
}

template <int D, typename Get>
__device__ void tile_cands_long(Get get, int L, int t, const TileCandOut& out, unsigned long long (&st)[3])
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const TileInfo& ti = out.info[t];
    const TileGeom g = ti.g;
    const bool split = g.pad[0] != 0;
    float4 b0, b1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (split) {
        const TileSub sb = ti.sb;
        b0 = make_float4(sb.o1[0], sb.o1[1], sb.o1[2], sb.r1);
        b1 = make_float4(sb.o2[0], sb.o2[1], sb.o2[2], sb.r2);
    } else {
        b0 = make_float4(g.o[0], g.o[1], g.o[2], g.r);
    }
    float* blk = out.tcand + (int64_t)t * cand_block_words<D>();
    // lists up to 32 * kRQ records: every record of the lane loaded once (all loads in flight) and
    // its distances to the ball(s) kept in registers for the compaction
    constexpr int kRQ = KM_TC_RQ;
    if (L <= 32 * kRQ) {
        CRec cr[kRQ];
        float d0[kRQ], d1[kRQ];
#pragma unroll
        for (int q = 0; q < kRQ; ++q) {
            cr[q].x = cr[q].y = cr[q].z = INFINITY;
            cr[q].j = 0;
            if (q * 32 + lane < L) cr[q] = get(q * 32 + lane);
        }
        float m0 = INFINITY, m1 = INFINITY;
#pragma unroll
        for (int q = 0; q < kRQ; ++q) {
            d0[q] = ball_delta2<D>(b0, cr[q]);
            d1[q] = split ? ball_delta2<D>(b1, cr[q]) : INFINITY;
            m0 = fminf(m0, d0[q]);
            m1 = fminf(m1, d1[q]);
        }
        const float T0 = prune_thr2(__uint_as_float(__reduce_min_sync(full, __float_as_uint(m0))), b0.w);
        const float T1 = split ? prune_thr2(__uint_as_float(__reduce_min_sync(full, __float_as_uint(m1))), b1.w) : -1.0f;
        int cnt = 0;
#pragma unroll
        for (int q = 0; q < kRQ; ++q) {
            if (q * 32 >= L) break;
            const bool f = q * 32 + lane < L && (d0[q] <= T0 || d1[q] <= T1);
            const unsigned bal = __ballot_sync(full, f);
            if (!bal) continue;
            const int pos = cnt + __popc(bal & lt);
            if (f && pos < kTC) {
                blk[pos] = -cr[q].x;
                blk[kTC + pos] = -cr[q].y;
                if (D == 3) blk[2 * kTC + pos] = -cr[q].z;
                reinterpret_cast<int*>(blk)[D * kTC + pos] = cr[q].j;
            }
            cnt += __popc(bal);
        }
        int off = 0;
        if (cnt <= kTC) {
            if (lane < ((cnt + 3) & ~3) - cnt) {
                const int s2 = cnt + lane;
                blk[s2] = -INFINITY;
                blk[kTC + s2] = -INFINITY;
                if (D == 3) blk[2 * kTC + s2] = -INFINITY;
                reinterpret_cast<int*>(blk)[D * kTC + s2] = 0x7fffffff;
            }
        } else {
            if (lane == 0) off = atomicAdd(out.ovf_cur, cnt);
            off = __shfl_sync(full, off, 0);
            if ((long long)off + cnt <= (long long)out.ovf_cap) {
                int wpos = 0;
#pragma unroll
                for (int q = 0; q < kRQ; ++q) {
                    if (q * 32 >= L) break;
                    const bool f = q * 32 + lane < L && (d0[q] <= T0 || d1[q] <= T1);
                    const unsigned bal = __ballot_sync(full, f);
                    if (f) out.ovf[off + wpos + __popc(bal & lt)] = cr[q];
                    wpos += __popc(bal);
                }
            } else {
                off = -1;
            }
        }
        if (lane == 0) {
            out.aux[t].ncand = cnt;
            out.aux[t].off = off;
            st[2] += (unsigned long long)cnt;
        }
        return;
    }
    // longer lists: kLU independent record loads per lane in flight per pass (the list is in L2:
    // a chain of dependent loads would serialise the tile)
    constexpr int kLU = 4;
    float m0 = INFINITY, m1 = INFINITY;
    for (int e0 = lane; e0 < L; e0 += 32 * kLU) {
        CRec cr[kLU];
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            cr[u].x = cr[u].y = cr[u].z = INFINITY;
            cr[u].j = 0;
            if (e0 + 32 * u < L) cr[u] = get(e0 + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            m0 = fminf(m0, ball_delta2<D>(b0, cr[u]));
            if (split) m1 = fminf(m1, ball_delta2<D>(b1, cr[u]));
        }
    }
    const float T0 = prune_thr2(__uint_as_float(__reduce_min_sync(full, __float_as_uint(m0))), b0.w);
    const float T1 = split ? prune_thr2(__uint_as_float(__reduce_min_sync(full, __float_as_uint(m1))), b1.w) : -1.0f;
    auto keep = [&](const CRec& c) {
        return ball_delta2<D>(b0, c) <= T0 || (split && ball_delta2<D>(b1, c) <= T1);
    };
    int cnt = 0;
    for (int e00 = 0; e00 < L; e00 += 32 * kLU) {
        CRec cr[kLU];
#pragma unroll
        for (int u = 0; u < kLU; ++u)
            if (e00 + 32 * u + lane < L) cr[u] = get(e00 + 32 * u + lane);
#pragma unroll
        for (int u = 0; u < kLU; ++u) {
            if (e00 + 32 * u >= L) break;
            const bool f = e00 + 32 * u + lane < L && keep(cr[u]);
            const unsigned bal = __ballot_sync(full, f);
            const int pos = cnt + __popc(bal & lt);
            if (f && pos < kTC) {
                blk[pos] = -cr[u].x;
                blk[kTC + pos] = -cr[u].y;
                if (D == 3) blk[2 * kTC + pos] = -cr[u].z;
                reinterpret_cast<int*>(blk)[D * kTC + pos] = cr[u].j;
            }
            cnt += __popc(bal);
        }
    }
    int off = 0;
    if (cnt <= kTC) {
        if (lane < ((cnt + 3) & ~3) - cnt) {
            const int s2 = cnt + lane;
            blk[s2] = -INFINITY;
            blk[kTC + s2] = -INFINITY;
            if (D == 3) blk[2 * kTC + s2] = -INFINITY;
            reinterpret_cast<int*>(blk)[D * kTC + s2] = 0x7fffffff;
        }
    } else {
        if (lane == 0) off = atomicAdd(out.ovf_cur, cnt);
        off = __shfl_sync(full, off, 0);
        if ((long long)off + cnt <= (long long)out.ovf_cap) {
            int wpos = 0;
            for (int e0 = 0; e0 < L; e0 += 32) {
                const int e = e0 + lane;
                CRec c;
                bool f = false;
                if (e < L) { c = get(e); f = keep(c); }
                const unsigned bal = __ballot_sync(full, f);
                if (f) out.ovf[off + wpos + __popc(bal & lt)] = c;
                wpos += __popc(bal);
            }
        } else {
            off = -1;   // pool full: the assignment kernel scans the whole level-1 list
        }
    }
    if (lane == 0) {
        out.aux[t].ncand = cnt;
        out.aux[t].off = off;
        st[2] += (unsigned long long)cnt;
    }
}

template <int D, typename Get>
__device__ void tile_cands_warp(Get get, int L, int t0, int nt, const TileCandOut& out, int* scnt,
                                unsigned long long (&st)[3])
{
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int grp = lane >> 2, sub = lane & 3;
    for (int g0 = 0; g0 < nt; g0 += 8) {
        const bool act = g0 + grp < nt;
        const int t = t0 + g0 + grp;
        float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
        bool split = false;
        if (act) {
            const TileInfo& ti = out.info[t];
            const TileGeom g = ti.g;
            split = g.pad[0] != 0;
            if (split) {
                const TileSub sb = ti.sb;
                b0 = make_float4(sb.o1[0], sb.o1[1], sb.o1[2], sb.r1);
                b1 = make_float4(sb.o2[0], sb.o2[1], sb.o2[2], sb.r2);
            } else {
                b0 = make_float4(g.o[0], g.o[1], g.o[2], g.r);
            }
        }
        float m0 = INFINITY, m1 = INFINITY;
        for (int e = sub; e < L; e += 4) {
            const CRec c = get(e);
            m0 = fminf(m0, ball_delta2<D>(b0, c));
            if (split) m1 = fminf(m1, ball_delta2<D>(b1, c));
        }
        m0 = fminf(m0, __shfl_xor_sync(full, m0, 1));
        m0 = fminf(m0, __shfl_xor_sync(full, m0, 2));
        m1 = fminf(m1, __shfl_xor_sync(full, m1, 1));
        m1 = fminf(m1, __shfl_xor_sync(full, m1, 2));
        const float T0 = prune_thr2(m0, b0.w);
        const float T1 = split ? prune_thr2(m1, b1.w) : -1.0f;
        auto keep = [&](const CRec& c) {
            return ball_delta2<D>(b0, c) <= T0 || (split && ball_delta2<D>(b1, c) <= T1);
        };
        if (sub == 0) { scnt[grp] = 0; scnt[8 + grp] = 0; }
        __syncwarp();
        float* blk = out.tcand + (int64_t)t * cand_block_words<D>();
        if (act)
            for (int e = sub; e < L; e += 4) {
                const CRec c = get(e);
                if (keep(c)) {
                    const int pos = atomicAdd(&scnt[grp], 1);
                    if (pos < kTC) {
                        blk[pos] = -c.x;
                        blk[kTC + pos] = -c.y;
                        if (D == 3) blk[2 * kTC + pos] = -c.z;
                        reinterpret_cast<int*>(blk)[D * kTC + pos] = c.j;
                    }
                }
            }
        __syncwarp();
        const int cnt = scnt[grp];
        int off = 0;
        if (cnt > kTC) {   // more than kTC: all of them into the overflow pool
            if (sub == 0) off = atomicAdd(out.ovf_cur, cnt);
        }
        off = __shfl_sync(full, off, lane & ~3);
        if (act) {
            if (cnt <= kTC) {
                for (int s2 = cnt + sub; s2 < ((cnt + 3) & ~3); s2 += 4) {
                    blk[s2] = -INFINITY;
                    blk[kTC + s2] = -INFINITY;
                    if (D == 3) blk[2 * kTC + s2] = -INFINITY;
                    reinterpret_cast<int*>(blk)[D * kTC + s2] = 0x7fffffff;
                }
            } else if ((long long)off + cnt <= (long long)out.ovf_cap) {
                for (int e = sub; e < L; e += 4) {
                    const CRec c = get(e);
                    if (keep(c)) out.ovf[off + atomicAdd(&scnt[8 + grp], 1)] = c;
                }
            } else {
                off = -1;   // pool full: the assignment kernel scans the whole level-1 list
            }
            if (sub == 0) {
                out.aux[t].ncand = cnt;
                out.aux[t].off = off;
                st[2] += (unsigned long long)cnt;
            }
        }
        __syncwarp();
    }
}

// Ball of every node of a level from its children's balls: o = mean of child centres,
// r = max (||o_c - o|| + r_c) in FP64, rounded up (triangle inequality).
template <int D>
__global__ void level_geom_kernel(const StGeom* __restrict__ child, int nchild, int fan, int nnodes,
                                  StGeom* __restrict__ out)
{
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nnodes; v += gridDim.x * blockDim.x) {
        const int c0 = v * fan, c1 = min(nchild, c0 + fan);
        double c[3] = {0.0, 0.0, 0.0};
        for (int i = c0; i < c1; ++i)
#pragma unroll
            for (int m = 0; m < D; ++m) c[m] += child[i].o[m];
        StGeom o;
        o.o[0] = o.o[1] = o.o[2] = 0.f;
#pragma unroll
        for (int m = 0; m < D; ++m) o.o[m] = (float)(c[m] / (c1 - c0));
        double R = 0.0;
        for (int i = c0; i < c1; ++i) {
            double d2 = 0.0;
#pragma unroll
            for (int m = 0; m < D; ++m) { const double x = (double)child[i].o[m] - (double)o.o[m]; d2 += x * x; }
            R = fmax(R, sqrt(d2) + (double)child[i].r);
        }
        o.r = __fmul_ru(__double2float_ru(R), 1.0f + 0x1p-20f);
        out[v] = o;
    }
}

// Upper levels: one CTA per node prunes its parent's list (pref == nullptr: the roots, all k
// centroids) with the node ball; block-wide ordered compaction (ascending parent position,
// hence ascending j).  Level storage holds up to k records per node, so no list overflows.
template <int D>
__global__ void __launch_bounds__(kTileThreads)
cta_prune_kernel(const StGeom* __restrict__ sg, int nnodes, int fan, const NodeRef* __restrict__ pref,
                 const float* __restrict__ C, int k, CRec* __restrict__ pool, long long pool_base, int cap,
                 NodeRef* __restrict__ ref, int* __restrict__ need, int* __restrict__ dyn_cursor,
                 const Ctl* __restrict__ ctl, TileCandOut tco)
{
    // tco.tcand != nullptr (level 1): each warp then computes the candidate lists of up to 8 of
    // the node's tiles from the node's list (tile_cands_warp)
    __shared__ int s_tcnt[kWarpsPerCta][16];
    __shared__ CRec s_nl[kShortList];   // a short node list, for its tiles' candidate pass
    unsigned long long tst[3] = {0ull, 0ull, 0ull};
    // dyn_cursor != nullptr: the level's pool region (nnodes * cap records) is allocated per node
    // with exact list lengths (atomic cursor, reset every iteration), so a long list of one node
    // does not force it to inherit its parent's much longer list
    if (ctl && ctl->done) return;
    __shared__ long long s_off;
    __shared__ int s_pfx[kMaxPruneRounds * kWarpsPerCta + 1];
    __shared__ float s_min[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int v = blockIdx.x; v < nnodes; v += gridDim.x) {
        if (need) {   // level 1: only nodes with a listed tile (block-uniform)
            if (!need[v]) continue;
            __syncthreads();
            if (threadIdx.x == 0) need[v] = 0;
        }
        NodeRef P;
        if (pref) P = pref[v / fan];
        else { P.off = -1; P.len = k; P.pad = 0; }
        const CRec* src = P.off >= 0 ? pool + P.off : nullptr;
        auto rec = [&](int e) { return src ? src[e] : make_rec<D>(C, e); };
        const int plen = P.len;
        const int rounds = (plen + blockDim.x - 1) / blockDim.x;
        const StGeom g = sg[v];
        float dmin2 = INFINITY;
        for (int rr = 0; rr < rounds; ++rr) {
            const int e = rr * blockDim.x + threadIdx.x;
            if (e < plen) dmin2 = fminf(dmin2, rec_delta2<D>(g.o, rec(e)));
        }
        // squared distances are >= 0: their float bits order like unsigned integers
        dmin2 = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(dmin2)));
        if (lane == 0) s_min[w] = dmin2;
        __syncthreads();
        dmin2 = s_min[0];
        for (int i = 1; i < nw; ++i) dmin2 = fminf(dmin2, s_min[i]);
        const float T2 = prune_thr2(dmin2, g.r);
        unsigned long long fl = 0ull;
        for (int rr = 0; rr < rounds; ++rr) {
            const int e = rr * blockDim.x + threadIdx.x;
            const bool f = e < plen && rec_delta2<D>(g.o, rec(e)) <= T2;
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (f) fl |= 1ull << rr;
            if (lane == 0) s_pfx[rr * nw + w] = __popc(bal);
        }
        __syncthreads();
        if (w == 0) {   // exclusive prefix over (round, warp) in place; total at the end
            const int tot = rounds * nw;
            int carry = 0;
            for (int c0 = 0; c0 < tot; c0 += 32) {
                const int x0 = c0 + lane < tot ? s_pfx[c0 + lane] : 0;
                int x = x0;
#pragma unroll
                for (int of = 1; of < 32; of <<= 1) { int y = __shfl_up_sync(0xffffffffu, x, of); if (lane >= of) x += y; }
                if (c0 + lane < tot) s_pfx[c0 + lane] = carry + x - x0;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) s_pfx[kMaxPruneRounds * kWarpsPerCta] = carry;
        }
        __syncthreads();
        const int total = s_pfx[kMaxPruneRounds * kWarpsPerCta];
        bool fits;
        long long off;
        if (dyn_cursor) {
            if (threadIdx.x == 0) {
                const long long o = atomicAdd(dyn_cursor, total);
                s_off = o + total <= (long long)nnodes * cap ? o : -1;
            }
            __syncthreads();
            fits = s_off >= 0;
            off = pool_base + s_off;
        } else {
            fits = total <= cap;
            off = pool_base + (long long)v * cap;
        }
        if (fits) {
            const unsigned lt = (1u << lane) - 1u;
            for (int rr = 0; rr < rounds; ++rr) {
                const bool f = (fl >> rr) & 1ull;
                const unsigned bal = __ballot_sync(0xffffffffu, f);
                if (f) {
                    const int pos = s_pfx[rr * nw + w] + __popc(bal & lt);
                    const CRec c = rec(rr * blockDim.x + threadIdx.x);
                    pool[off + pos] = c;
                    if (tco.tcand && pos < kShortList) s_nl[pos] = c;   // the tiles' pass reads it from here
                }
            }
        }
        if (threadIdx.x == 0) {
            NodeRef r;
            r.off = fits ? off : P.off;
            r.len = fits ? total : P.len;
            r.pad = 0;
            ref[v] = r;
        }
        __syncthreads();
        if (tco.tcand) {
            const int t0 = v << tco.st_shift;
            const int nt = min(1 << tco.st_shift, tco.ntiles - t0);
            const long long lo = fits ? off : P.off;
            const int L = fits ? total : P.len;
            const CRec* list = lo >= 0 ? pool + lo : nullptr;
            auto get = [&](int e) { return fits ? s_nl[e] : (list ? list[e] : make_rec<D>(C, e)); };
            if (L > tco.short_list) {   // one warp per tile in tile_cands_kernel
                if (threadIdx.x == 0) queue_heavy(tco, v, L);
                if (lane == 0 && w == 0) { tst[0] += (unsigned long long)L; tst[1] += 1ull; }
            } else {
                if (lane == 0 && w == 0) { tst[0] += (unsigned long long)L; tst[1] += 1ull; }
                if (w * 8 < nt) tile_cands_warp<D>(get, L, t0 + w * 8, min(8, nt - w * 8), tco, s_tcnt[w], tst);
            }
            __syncthreads();
        }
    }
    if (tco.tcand) flush_cand_stats(tco, tst);
}

// Lower levels: a CTA takes 8 consecutive nodes (one warp each) that share one parent (the
// parent fan is a multiple of 8), stages the parent's list in shared memory once (coalesced),
// and every warp prunes it with its node ball (ordered warp compaction into the pool).
constexpr int kPruneGroup = kTileThreads / 32;
#ifndef KM_NODE_REGQ
#define KM_NODE_REGQ 32
#endif
constexpr int kNodeRegQ = KM_NODE_REGQ;   // staged lists up to 32 * kNodeRegQ: single pass, delta^2 in registers
static_assert(kFanout % kPruneGroup == 0, "a prune group must share one parent");

template <int D>
__global__ void __launch_bounds__(kTileThreads)
node_prune_kernel(const StGeom* __restrict__ sg, int nnodes, int fan, const NodeRef* __restrict__ pref,
                  const float* __restrict__ C, int k, CRec* __restrict__ pool, long long pool_base, int cap,
                  NodeRef* __restrict__ ref, int* __restrict__ need, const Ctl* __restrict__ ctl, TileCandOut tco)
{
    if (ctl && ctl->done) return;
    __shared__ CRec s_list[kCandCap];
    __shared__ int s_tcnt[kPruneGroup][16];   // tile_cands_warp's counters, per warp
    unsigned long long tst[3] = {0ull, 0ull, 0ull};
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    const int ngroups = (nnodes + kPruneGroup - 1) / kPruneGroup;
    for (int gidx = blockIdx.x; gidx < ngroups; gidx += gridDim.x) {
        const int v = gidx * kPruneGroup + w;
        // need (level 1 only): set by tile_filter_kernel for nodes with a listed tile; cleared here
        bool mine = v < nnodes;
        if (mine && need) mine = need[v] != 0;
        if (!__syncthreads_or(mine)) continue;
        NodeRef P;
        if (pref) P = pref[(gidx * kPruneGroup) / fan];
        else { P.off = -1; P.len = k; P.pad = 0; }   // single level: the parent is all k
        const int plen = P.len;
        const bool staged = plen <= kCandCap;
        if (staged) {
            for (int e = threadIdx.x; e < plen; e += blockDim.x)
                s_list[e] = P.off >= 0 ? pool[P.off + e] : make_rec<D>(C, e);
        }
        __syncthreads();
        if (mine) {
            if (need && lane == 0) need[v] = 0;
            const StGeom g = sg[v];
            const CRec* src = P.off >= 0 ? pool + P.off : nullptr;
            auto rec = [&](int e) { return staged ? s_list[e] : (src ? src[e] : make_rec<D>(C, e)); };
            const long long off = pool_base + (long long)v * cap;
            int cnt = 0;
            if (staged && plen <= 32 * kNodeRegQ) {
                // one pass over the staged list: delta^2 kept in registers for the compaction
                float dv[kNodeRegQ];
                float dmin2 = INFINITY;
#pragma unroll
                for (int qq = 0; qq < kNodeRegQ; ++qq) {
                    const int e = qq * 32 + lane;
                    dv[qq] = e < plen ? rec_delta2<D>(g.o, s_list[e]) : INFINITY;
                    dmin2 = fminf(dmin2, dv[qq]);
                }
                dmin2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dmin2)));   // >= 0: uint order
                const float T2 = prune_thr2(dmin2, g.r);
#pragma unroll
                for (int qq = 0; qq < kNodeRegQ; ++qq) {
                    if (qq * 32 >= plen) break;
                    const int e = qq * 32 + lane;
                    const bool f = dv[qq] <= T2;
                    const unsigned bal = __ballot_sync(full, f);
                    const int o2 = cnt + __popc(bal & lt);
                    if (f && o2 < cap) pool[off + o2] = s_list[e];
                    cnt += __popc(bal);
                }
            } else {
                float dmin2 = INFINITY;
                for (int e = lane; e < plen; e += 32) dmin2 = fminf(dmin2, rec_delta2<D>(g.o, rec(e)));
                dmin2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dmin2)));   // >= 0: uint order
                const float T2 = prune_thr2(dmin2, g.r);
                for (int e0 = 0; e0 < plen; e0 += 32) {
                    const int e = e0 + lane;
                    CRec c;
                    bool f = false;
                    if (e < plen) { c = rec(e); f = rec_delta2<D>(g.o, c) <= T2; }
                    const unsigned bal = __ballot_sync(full, f);
                    const int o2 = cnt + __popc(bal & lt);
                    if (f && o2 < cap) pool[off + o2] = c;
                    cnt += __popc(bal);
                }
            }
            if (lane == 0) {
                NodeRef r;
                if (cnt <= cap) { r.off = off; r.len = cnt; }
                else { r.off = P.off; r.len = P.len; }   // inherit the parent's (superset) list
                r.pad = 0;
                ref[v] = r;
            }
            if (tco.tcand) {   // the tiles' candidate lists from this node's list (written above by this warp)
                __syncwarp();
                const int t0 = v << tco.st_shift;
                const bool own = cnt <= cap;
                const long long lo = own ? off : P.off;
                const CRec* list = own ? pool + lo : (lo >= 0 ? pool + lo : nullptr);
                auto get = [&](int e) { return list ? list[e] : make_rec<D>(C, e); };
                const int L = own ? cnt : P.len;
                if (lane == 0) { tst[0] += (unsigned long long)L; tst[1] += 1ull; }
                if (L > tco.short_list) {
                    if (lane == 0) queue_heavy(tco, v, L);
                } else {
                    tile_cands_warp<D>(get, L, t0, min(1 << tco.st_shift, tco.ntiles - t0), tco, s_tcnt[w], tst);
                }
            }
        }
        __syncthreads();   // s_list is rewritten by the next group
    }
    if (tco.tcand) flush_cand_stats(tco, tst);
}

// The flat index (k <= kNodeRegQ * 32, level 1 prunes all k directly): all k records staged once
// per CTA in shared memory; every warp then takes level-1 nodes on its own (no CTA barrier):
// the node's list from all k (delta^2 in registers, one pass), then its tiles' candidate lists
// from the node's list, read back from shared memory through the kept positions.
constexpr int kFlatIdxCap = kShortList;   // kept positions per warp (longer lists go to tile_cands_kernel)
template <int D>
__host__ __device__ constexpr size_t flat_prune_smem(int k)
{
    return (size_t)k * sizeof(CRec) + (size_t)kWarpsPerCta * kFlatIdxCap * 2 + (size_t)kWarpsPerCta * 16 * 4;
}

#ifndef KM_FLAT_MINB
#define KM_FLAT_MINB 4
#endif
template <int D>
__global__ void __launch_bounds__(kTileThreads, KM_FLAT_MINB)
node_prune_flat_kernel(const StGeom* __restrict__ sg, int nnodes, const float* __restrict__ C, int k,
                       CRec* __restrict__ pool, long long pool_base, int cap, NodeRef* __restrict__ ref,
                       const Ctl* __restrict__ ctl, TileCandOut tco)
{
    if (ctl && ctl->done) return;
    extern __shared__ __align__(16) unsigned char fsm[];
    CRec* s_list = reinterpret_cast<CRec*>(fsm);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned short* s_idx = reinterpret_cast<unsigned short*>(fsm + (size_t)k * sizeof(CRec)) + w * kFlatIdxCap;
    int* s_tcnt = reinterpret_cast<int*>(fsm + (size_t)k * sizeof(CRec) + (size_t)kWarpsPerCta * kFlatIdxCap * 2) + w * 16;
    const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
    unsigned long long tst[3] = {0ull, 0ull, 0ull};
    for (int e = threadIdx.x; e < k; e += blockDim.x) s_list[e] = make_rec<D>(C, e);
    __syncthreads();
    // nodes are claimed dynamically (a node's cost grows with its list length, which varies
    // widely): the first one round-robin, then through the counter tco.ovf_cur[1]
    const int nwarps = gridDim.x * kWarpsPerCta;
    int v = blockIdx.x * kWarpsPerCta + w;
    int vnext = 0;
    if (lane == 0) vnext = nwarps + atomicAdd(tco.ovf_cur + 1, 1);
    for (; v < nnodes;) {
        const StGeom g = sg[v];
        float dv[kNodeRegQ];
        float dmin2 = INFINITY;
#pragma unroll
        for (int qq = 0; qq < kNodeRegQ; ++qq) {
            const int e = qq * 32 + lane;
            dv[qq] = e < k ? rec_delta2<D>(g.o, s_list[e]) : INFINITY;
            dmin2 = fminf(dmin2, dv[qq]);
        }
        dmin2 = __uint_as_float(__reduce_min_sync(full, __float_as_uint(dmin2)));   // >= 0: uint order
        const float T2 = prune_thr2(dmin2, g.r);
        const long long off = pool_base + (long long)v * cap;
        int cnt = 0;
#pragma unroll
        for (int qq = 0; qq < kNodeRegQ; ++qq) {
            if (qq * 32 >= k) break;
            const int e = qq * 32 + lane;
            const bool f = dv[qq] <= T2;
            const unsigned bal = __ballot_sync(full, f);
            if (!bal) continue;   // (most chunks keep nothing)
            const int o2 = cnt + __popc(bal & lt);
            if (f && o2 < cap) {
                pool[off + o2] = s_list[e];
                if (o2 < kFlatIdxCap) s_idx[o2] = (unsigned short)e;
            }
            cnt += __popc(bal);
        }
        const bool own = cnt <= cap;
        if (lane == 0) {
            NodeRef r;
            r.off = own ? off : -1;   // longer than the capacity: all k
            r.len = own ? cnt : k;
            r.pad = 0;
            ref[v] = r;
        }
        const int L = own ? cnt : k;
        if (lane == 0) { tst[0] += (unsigned long long)L; tst[1] += 1ull; }
        if (L > tco.short_list) {   // the tiles of a long list get one warp each in tile_cands_kernel
            if (lane == 0) queue_heavy(tco, v, L);
        } else {
            __syncwarp();
            const int t0 = v << tco.st_shift;
            auto get = [&](int e) { return own ? s_list[s_idx[e]] : s_list[e]; };
            tile_cands_warp<D>(get, L, t0, min(1 << tco.st_shift, tco.ntiles - t0), tco, s_tcnt, tst);
        }
        v = __shfl_sync(full, vnext, 0);
        if (lane == 0 && v < nnodes) vnext = nwarps + atomicAdd(tco.ovf_cur + 1, 1);
    }
    flush_cand_stats(tco, tst);
}

// The tiles of the long-list nodes queued by the level-1 prune kernels: one warp per tile (lanes
// over the node's list in the pool, tile_cands_long), claimed dynamically, so the few nodes with
// hundreds of candidates spread over the whole GPU instead of serialising one warp.  (Staging
// the list in shared memory per (node, 8 tiles) item was measured slower: config 4 +13 %,
// config 5 +26 % per run -- fewer warps per SM and 8 tiles in series per warp.)
template <int D>
__global__ void __launch_bounds__(kTileThreads, KM_TC_MINB)
tile_cands_kernel(const NodeRef* __restrict__ ref, const CRec* __restrict__ pool, const float* __restrict__ C,
                  const Ctl* __restrict__ ctl, TileCandOut tco)
{
    if (ctl && ctl->done) return;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long tst[3] = {0ull, 0ull, 0ull};
    const int per = 1 << tco.st_shift;
    const int nvh = tco.ovf_cur[4], nh = tco.ovf_cur[2];
    const int nitems = (nvh + nh) * per;
    if (tco.stats && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&tco.stats[16], (unsigned long long)(nvh + nh));
    // item i = (queued node i / per, tile i % per); the multi-pass nodes first
    auto node_of = [&](int i) {
        const int q = i >> tco.st_shift;
        return q < nvh ? tco.heavy[tco.nnodes - 1 - q] : tco.heavy[q - nvh];
    };
    // (later items claimed one ahead, with the node of the next item loaded while the current one
    // runs, was measured slower: 29.2 vs 23.0 us per launch at config 4)
    // every warp's first item is static (no counter round trip before the first tile), the rest
    // are claimed through the counter (config 3 -2.0 %, config 4 -1.3 % per run; all items static:
    // +1.8 % / +5 % at configs 4 / 5; 2-8 items per claim: +3...+70 % -- the kernel is bound by the
    // serial chain per tile, so tiles in series per warp cost more than the atomics they save)
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < nitems;) {
        const int v = node_of(i);
        const int t = (v << tco.st_shift) + (i & (per - 1));
        if (t < tco.ntiles) {
            const NodeRef R = ref[v];
            const CRec* list = R.off >= 0 ? pool + R.off : nullptr;
            auto get = [&](int e) { return list ? list[e] : make_rec<D>(C, e); };
            tile_cands_long<D>(get, R.len, t, tco, tst);
        }
        if (lane == 0) i = nwarps + atomicAdd(tco.ovf_cur + 3, 1);
        i = __shfl_sync(full, i, 0);
    }
    flush_cand_stats(tco, tst);
}

}  // namespace km
