// km_api.cu -- the C ABI of libkm (include/km.h): validation, workspace, launches,
// the device-side Lloyd loop, timing.  No torch types cross this boundary.
//
// Loop (Alg. 1 skeleton, with the index replaced by a brute-force
// shared-memory scan):
//   bbox -> quant                                   (once per run: fixed-point origin/scale)
//   for t < max_iter:  assign+accumulate (K1) ; finalize (K3)   -- early-exit on ctl.done
//   sse (Eq. 1 of the returned pair) ; reduce
#include "../../include/km.h"
#include "km_kernels.cuh"
#include "km_assign_fast.cuh"
#include "km_tiles_assign.cuh"
#include "km_hd.cuh"
#include "km_small.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <algorithm>
#include <new>
#include <vector>

namespace {

thread_local int t_last_cuda_error = 0;

constexpr int kMaxParts = 4096;   // per-CTA partial slots
constexpr size_t kPrivMax = 48 * 1024;      // K1's privatised update partials (k <= 2457 at d = 2, 1755 at d = 3)
constexpr size_t kAccPrivMax = 96 * 1024;   // accumulate_kernel's
constexpr int kGraphMaxIter = 128;          // longer runs launch eagerly (graph size)
#ifndef KM_ACC_COPIES
#define KM_ACC_COPIES 8
#endif
constexpr int kAccCopies = KM_ACC_COPIES;   // private copies of the tile path's running sums
static_assert(kAccCopies >= 1 && kAccCopies <= km::kMaxAccCopies, "finalize unrolls up to kMaxAccCopies");
#ifndef KM_FLAT_K
#define KM_FLAT_K 1024
#endif
#ifndef KM_SCATTER_WIN
#define KM_SCATTER_WIN (12ll << 20)
#endif

struct TimedLaunch {
    int kind;  // 0 assign, 1 update, 2 other
    cudaEvent_t a, b;
};

// The device-side arguments of one km_run_ctx call (also the CUDA-graph cache key; compared
// with memcmp, so every member is set explicitly and the padding is zeroed by {}-init).
struct RunIO {
    const float* P;             // device points (the caller's or the staged copy)
    int32_t* L;                 // device labels
    const float* init_dev;      // device initial centroids (nullptr: staged from the host before)
    float* outc_dev;            // device output centroids (nullptr: copied to the host after)
    double* sse_trace;          // optional device traces
    int64_t* chg_trace;
    int max_iter;
    float tol;
    int path;                   // 0 brute force, 1 tiles, 2 high-d, 3 brute force + bounds; -1: no graph
};

struct HostScalars {            // pinned: the scalars every call reads back
    double sse;
    km::Ctl ctl;
};

}  // namespace

struct km_ctx {
    int64_t n = 0;
    int d = 0, k = 0, kpad = 0;
    int du = 0;                             // caller's d when it is zero-padded to d (high-d variant)
    float* pad_c = nullptr;                 // [k][d] padded new centroids (km_update, du != 0)
    int device = 0, num_sms = 0;
    cudaStream_t stream = nullptr;
    // workspace (device)
    unsigned long long* acc_sum = nullptr;  // [k][d]
    unsigned int* acc_cnt = nullptr;        // [k]
    double* sse_part = nullptr;             // [kMaxParts]
    unsigned long long* chg_part = nullptr; // [kMaxParts]
    float* bbox_part = nullptr;             // [kMaxParts][2d]
    km::Quant* quant = nullptr;
    km::Ctl* ctl = nullptr;
    double* scal = nullptr;                 // km::SseFix: Eq. 1 of the returned pair (value, scale, limbs)
    int* s3 = nullptr;                      // its fixed-point exponent
    unsigned int* tick = nullptr;           // K1's CTA ticket (the last CTA runs the refine)
    unsigned long long* sse128 = nullptr;   // [2 * kMaxParts] per-CTA 128-bit partials of Eq. 1
    long long n_global = 0;                 // data-parallel run: points over all ranks (0: this context's n)
    double dp_sse_inv = 0.0;                // 2^-s3 of the last km_dp_end (km_dp_sse)
    float* cwork = nullptr;                 // [k][d] working centroids
    double* sse_trace = nullptr;
    long long* chg_trace = nullptr;
    double* drift_trace = nullptr;
    int trace_cap = 0;
    int last_iters = 0;
    // host-pointer staging (lazily allocated)
    float* stage_pts = nullptr;
    int32_t* stage_lab = nullptr;
    // launch geometry
    int assign_grid = 0;
    int assign_variant = 1;   // 0 simple, 1.. km::scan_variant()
    size_t priv_smem = 0;     // K1's shared-memory update partials (0: per-point global REDs)
    size_t acc_priv = 0;      // the same for accumulate_kernel (km_update)
    int aux_grid = 0;
    // tile-pruned path (km_tiles.cuh)
    int mode = KM_MODE_AUTO;
    bool tiles_ready = false;
    float* ps = nullptr;                    // [n][d] Morton-sorted points
    int32_t* ls = nullptr;                  // [n] labels in sorted order
    unsigned int* keys[2] = {nullptr, nullptr};
    unsigned int* idx[2] = {nullptr, nullptr};
    unsigned int* perm = nullptr;           // sorted position -> input index (points to idx[0] or idx[1])
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    km::TileInfo* tgeom = nullptr;          // [ntiles] ball + moments (constant per run)
    km::TileState* tlab = nullptr;          // [ntiles] per-tile label state
    unsigned long long* stats = nullptr;    // [4]
    // index levels above the tiles (km_levels.cuh): level 0 = tile balls
    static constexpr int kMaxLev = 10;
    int nlev = 0;                           // levels 1..nlev-1 carry candidate lists
    int lev_n[kMaxLev] = {0};
    int lev_fan[kMaxLev] = {0};             // children per node of level l
    int lev_cap[kMaxLev] = {0};
    long long lev_off[kMaxLev] = {0};       // pool offset of level l's lists
    km::StGeom* lev_geom[kMaxLev] = {nullptr};
    km::NodeRef* lev_ref[kMaxLev] = {nullptr};
    km::CRec* lpool = nullptr;              // candidate lists (records) of all levels
    // inter bound (km_bounds.cuh) and the work list of the tiles Eq. 5 does not settle
    unsigned int* cb2 = nullptr;            // [k] FP32 bits of min_l ||c_j - c_l||^2
    km::TileAux* taux = nullptr;            // [ntiles] per-tile inputs of K1t (Eq. 4 record, candidate count)
    float* tcand = nullptr;                 // [ntiles][(d + 1) * kTC] per-tile candidate blocks
    int* ovf_cur = nullptr;                 // [8] overflow pool cursor, node / heavy / item counters of the level-1 prune
    int* heavy = nullptr;                   // [level-1 nodes] nodes with long lists (tile_cands_kernel)
    unsigned long long* sbucket = nullptr;  // [n - window] label scatter: (destination, label) of windows >= 1
    unsigned long long* scursor = nullptr;  // [kScatterMaxWin] their fill cursors
    int* work = nullptr;                    // [ntiles]
    int* work_cnt = nullptr;                // [8]: listed tiles, next entry to claim (K1t), K1b records,
                                            //      overflow pool cursor, level-1 pool cursor
    int* l1need = nullptr;                  // [lev_n[1]]
    unsigned long long* ttot = nullptr;     // [2] tile path: SSE_t (fixed point) and changed_t of the iteration
    unsigned long long* tfin = nullptr;     // [2] finalize_grid_kernel: max drift bits, CTA ticket
    unsigned long long* tacc_sum = nullptr; // [kAccCopies][k][d] running sums sv(j) of the tile path (persist
    unsigned int* tacc_cnt = nullptr;       // [kAccCopies][k]   across iterations: incremental, P:L411-413;
                                            //  CTA b updates copy b % kAccCopies: spreads the hot REDs)
    int filter_grid = 0, ib_chunk = 0, ib_gx = 0, ib_gy = 0, ib_jb = 1;
    int np_res = 1, npf_res = 1, tc_res = 1;   // resident node_prune / node_prune_flat / tile_cands CTAs per SM
    // A6: the whole run (index build, max_iter iterations, final SSE, labels) as one CUDA graph,
    // captured on a private stream and replayed while the arguments it depends on are unchanged
    cudaStream_t cap = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    RunIO gkey;                             // the arguments the captured graph was built for
    int64_t graph_launches = 0;             // kernels per replay (km_launch_count)
    bool use_graph = true;                  // km_debug_set(KM_DBG_GRAPH, 0): eager launches
    bool use_small = true;                  // km_debug_set(KM_DBG_SMALL, 0): the multi-kernel brute force
    bool use_pdl = true;                    // km_debug_set(KM_DBG_PDL, 0): no programmatic dependent launches
    // KM_MODE_BOUNDS: per-point Hamerly bounds (bounds_scan_kernel)
    float* lbv = nullptr;                   // [n] lower bound of each point's second-nearest distance
    float* cbuf1 = nullptr;                 // [k][d] second centroid buffer (launch t writes C^t to buffer t % 2)
    unsigned long long* bsum = nullptr;     // [5][k][d] running sums S (2 buffers), deltas D (3 buffers)
    unsigned int* bcnt = nullptr;           // [5][k] their counts
    unsigned long long* bscan = nullptr;    // points scanned (summed over the run's iterations)
    int bounds_grid = 0;
    bool last_run_bounds = false;
    HostScalars* hscal = nullptr;           // pinned host record of Eq. 1 and the iteration count
    HostScalars* dscal = nullptr;           // its device-side address (mapped), nullptr if unavailable
    // second stream: the inter bound + tile filter run beside the index-level prunes
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_c = nullptr, ev_f = nullptr;
    km::CRec* ovf = nullptr;                // [ovf_cap] K1t candidate lists longer than its shared buffer
    unsigned char* theavy = nullptr;        // [ntiles] K1t: the tile pruned a long list (schedule it first)
    int ovf_cap = 0;
    int ntiles = 0, tiles_grid = 0, tiles_kpad = 0;
    int k1t_minb = 2;                       // K1t register-budget variant (km_tiles_assign.cuh)
    int st_shift = 4;                       // level-1 nodes (super-tiles) group 1 << st_shift tiles
    // test/tuning overrides (km_debug_set; 0 = the per-context default)
    int dbg_st_shift = 0, dbg_minb = 0, hd_dbg = 0, dbg_short_list = 0;
    int short_list = km::kShortList;        // level-1 lists up to this length are expanded in the prune kernel
    size_t tiles_smem = 0;
    bool last_run_tiles = false;
    // data-parallel run state (km_dp_*)
    const float* dp_points = nullptr;
    int dp_iter = 0;
    int32_t* dp_lab = nullptr;              // labels of the brute-force DP path
    int32_t* stage_lab_dp()
    {
        if (!dp_lab && cudaMalloc((void**)&dp_lab, sizeof(int32_t) * (size_t)n) != cudaSuccess) {
            cudaGetLastError();
            dp_lab = nullptr;
        }
        return dp_lab;
    }
    // high-dimensional variant (km_hd.cuh; d in {32, 64, 128, 256})
    bool hd = false;
    float* hpc = nullptr;                   // [n][d] centred points, TF32 hi part: the A operand
    __nv_bfloat16* hpbh = nullptr;          // [n][d] BF16 of the hi part
    __nv_bfloat16* hpbl = nullptr;          // [n][d] BF16 of the lo part
    __nv_bfloat16* hcbh = nullptr;          // [hd_kpad][d] centred centroids: BF16 hi
    __nv_bfloat16* hcbl = nullptr;          // [hd_kpad][d] BF16 lo
    float* hpn = nullptr;                   // [n] upper bound of ||p'||
    float* hcc = nullptr;                   // [hd_kpad][d] centred centroids: the B operand
    float* hh = nullptr;                    // [hd_kpad] -||c'_j||^2 / 2 (-inf padding)
    float4* htopv = nullptr;                // [n][2][kTop/4] largest scores per point and column half
    int4* htopj = nullptr;                  // [n][2][kTop/4] their centroid indices
    int32_t* hlab = nullptr;                // [n] working labels
    int* hfb = nullptr;                     // [n] points for the FP64 fallback
    double* hq = nullptr;                   // [3][d] fixed-point origin, scale, inverse scale
    float* hctr = nullptr;                  // [d] centring origin (box midpoint, FP32)
    km::hd::HdState* hst = nullptr;
    CUtensorMap tmA, tmAh, tmAl, tmB, tmBh, tmBl;   // TMA descriptors (fixed at create)
    int hd_kpad = 0, hd_ntk = 0, hd_mt = 0, hd_grid = 0, hd_bbox_grid = 0;
    unsigned long long* hacc_q = nullptr;   // [k] running moment sums Q_j = sum ||p - o||^2 (SSE fixed point)
    unsigned long long* hpq2 = nullptr;     // [n] ||p - o||^2 per point (SSE fixed point)
    unsigned long long* hg_q = nullptr;     // [k] data-parallel: the all-reduced Q_j
    double* hfb_b = nullptr;                // [2][kFbCap][kFbSlices] sliced fallback: best, runner-up
    int* hfb_j = nullptr;                   // [kFbCap][kFbSlices] index of the best
    unsigned long long* hg_sum = nullptr;   // [k][d] data-parallel: the all-reduced sums (refine input)
    unsigned int* hg_cnt = nullptr;         // [k]
    // timing
    bool timing = false;
    std::vector<TimedLaunch> pending;
    std::vector<cudaEvent_t> pool;
    double tot_ms[3] = {0, 0, 0};
    int64_t tot_launches[3] = {0, 0, 0};
    int64_t launches = 0;
};

namespace {

int cuda_fail(cudaError_t e)
{
    t_last_cuda_error = (int)e;
    return KM_E_CUDA;
}

#define KM_CUDA(call)                                  \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_);   \
    } while (0)

cudaEvent_t take_event(km_ctx* c)
{
    if (!c->pool.empty()) {
        cudaEvent_t e = c->pool.back();
        c->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Every kernel launch goes through begin/end: launch counting, event timing and
// the post-launch error check.
struct LaunchScope {
    km_ctx* c;
    int kind;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    LaunchScope(km_ctx* c_, int kind_) : LaunchScope(c_, kind_, c_->stream) {}
    LaunchScope(km_ctx* c_, int kind_, cudaStream_t s_) : c(c_), kind(kind_), s(s_)
    {
        if (c->timing) {
            a = take_event(c);
            cudaEventRecord(a, s);
        }
    }
    int end()
    {
        c->launches++;
        cudaError_t e = cudaGetLastError();
        if (c->timing) {
            cudaEvent_t b = take_event(c);
            cudaEventRecord(b, s);
            c->pending.push_back({kind, a, b});
        }
        if (e != cudaSuccess) return cuda_fail(e);
        return KM_OK;
    }
};

int round_up4(int k) { return (k + 3) & ~3; }

size_t assign_smem_bytes(int d, int kpad) { return (size_t)d * kpad * sizeof(float); }

bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb)
{
    if (!a || !b || !na || !nb) return false;
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

// 1 = device memory on this context's device, 0 = host memory, -1 = other device
int pointer_kind(const km_ctx* c, const void* p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (at.type == cudaMemoryTypeDevice) return at.device == c->device ? 1 : -1;
    if (at.type == cudaMemoryTypeManaged) return 1;
    return 0;
}

km::FinArgs fin_args(km_ctx* c, const float* Cold, float* Cnew, int32_t* counts, double* maxdrift, bool traces,
                     km::Ctl* ctl, float tol, int nparts, bool tiles, bool dp);

// K1.  fin_tol: the brute-force loop fuses the refine into the CTA that finishes last (one
// launch per iteration; traces, flag and tol as finalize_kernel); NAN: no fused refine.
// incr (with a fused refine and the privatised update): the incremental update -- running sums
// kept by the refine, only changed points move (the caller zeroes the sums before t = 0).
template <int D>
int launch_assign(km_ctx* c, const float* pts, const float* C, int32_t* labels, int first, bool fuse,
                  const km::Ctl* ctl, float fin_tol = NAN, bool incr = false)
{
    size_t smem = assign_smem_bytes(D, c->kpad);
    const bool fin = fuse && ctl && fin_tol == fin_tol && c->assign_variant != 0;
    km::FinArgs fa = fin ? fin_args(c, c->cwork, c->cwork, nullptr, nullptr, true, const_cast<km::Ctl*>(ctl),
                                    fin_tol, c->assign_grid, false, false)
                         : km::FinArgs{};
    incr = incr && fin && c->priv_smem;
    if (incr) fa.clear = 0;
    unsigned int* tick = fin ? c->tick : nullptr;
    LaunchScope ls(c, 0);
    if (c->assign_variant == 0) {
        if (fuse)
            km::assign_simple_kernel<D, 2, true><<<c->assign_grid, km::kAssignThreads, smem, c->stream>>>(
                pts, c->n, C, c->k, c->kpad, labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt,
                c->quant, ctl);
        else
            km::assign_simple_kernel<D, 2, false><<<c->assign_grid, km::kAssignThreads, smem, c->stream>>>(
                pts, c->n, C, c->k, c->kpad, labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt,
                c->quant, ctl);
    } else if (!fuse) {
        km::launch_assign_fast<D, 0>(c->assign_variant, c->assign_grid, smem, c->stream, pts, c->n, C, c->k, c->kpad,
                                     labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt, c->quant, ctl,
                                     tick, fa);
    } else if (incr) {   // privatised partials of the incremental update
        km::launch_assign_fast<D, 3>(c->assign_variant, c->assign_grid, smem + c->priv_smem, c->stream, pts, c->n, C,
                                     c->k, c->kpad, labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt,
                                     c->quant, ctl, tick, fa);
    } else if (c->priv_smem) {   // the update privatised per CTA in shared memory (A4)
        km::launch_assign_fast<D, 2>(c->assign_variant, c->assign_grid, smem + c->priv_smem, c->stream, pts, c->n, C,
                                     c->k, c->kpad, labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt,
                                     c->quant, ctl, tick, fa);
    } else {
        km::launch_assign_fast<D, 1>(c->assign_variant, c->assign_grid, smem, c->stream, pts, c->n, C, c->k, c->kpad,
                                     labels, first, c->sse_part, c->chg_part, c->acc_sum, c->acc_cnt, c->quant, ctl,
                                     tick, fa);
    }
    return ls.end();
}

// K1b (KM_MODE_BOUNDS): launch t refines iteration t-1 in every CTA, then assigns (the buffers
// of km::BoundsIO); t == max_iter: the tail kernel (refine of the last iteration into cwork).
km::BoundsIO bounds_io(km_ctx* c, int t, float tol)
{
    const int64_t kd = (int64_t)c->k * c->d;
    auto S = [&](int x) { return c->bsum + x * kd; };
    auto SN = [&](int x) { return c->bcnt + (int64_t)x * c->k; };
    auto Dd = [&](int y) { return c->bsum + (2 + y) * kd; };
    auto DN = [&](int y) { return c->bcnt + (int64_t)(2 + y) * c->k; };
    float* buf[2] = {c->cwork, c->cbuf1};
    km::BoundsIO io{};
    io.cprev = t == 0 ? buf[0] : buf[(t - 1) % 2];
    io.cout = buf[t % 2];
    io.s_prev = S(t % 2);
    io.sn_prev = SN(t % 2);
    io.d_prev = Dd((t + 2) % 3);
    io.dn_prev = DN((t + 2) % 3);
    io.s_out = S((t + 1) % 2);
    io.sn_out = SN((t + 1) % 2);
    io.d_zero = Dd((t + 1) % 3);
    io.dn_zero = DN((t + 1) % 3);
    io.d_cur = Dd(t % 3);
    io.dn_cur = DN(t % 3);
    const int half = kMaxParts / 2;
    io.sse_prev = c->sse_part + ((t + 1) % 2) * half;
    io.chg_prev = c->chg_part + ((t + 1) % 2) * half;
    io.sse_cur = c->sse_part + (t % 2) * half;
    io.chg_cur = c->chg_part + (t % 2) * half;
    io.nparts = c->bounds_grid;
    io.sse_trace = c->sse_trace;
    io.chg_trace = c->chg_trace;
    io.drift_trace = c->drift_trace;
    io.ctl = c->ctl;
    io.tol = tol;
    io.t = t;
    return io;
}

template <int D>
int launch_bounds(km_ctx* c, const float* pts, int32_t* labels, int t, float tol)
{
    const km::BoundsIO io = bounds_io(c, t, tol);
    const size_t smem = assign_smem_bytes(D, c->kpad) + km::priv_bytes<D>(c->k) + km::bounds_smem_extra<D>(c->k);
    LaunchScope ls(c, 0);
    // programmatic dependent launch (t >= 1): scheduled while launch t-1's CTAs retire
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c->bounds_grid);
    cfg.blockDim = dim3(km::kAssignThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = t > 0 && c->use_pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KM_CUDA(cudaLaunchKernelEx(&cfg, km::bounds_scan_kernel<D, 4, 2>, pts, c->n, c->k, c->kpad, labels, c->lbv,
                               (const km::Quant*)c->quant, c->bscan, io));
    return ls.end();
}

template <int D>
int launch_bounds_tail(km_ctx* c, int T, float tol)
{
    km::BoundsIO io = bounds_io(c, T, tol);
    io.cout = c->cwork;
    LaunchScope ls(c, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(km::kFinalizeThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = c->use_pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KM_CUDA(cudaLaunchKernelEx(&cfg, km::bounds_tail_kernel<D>, io, (const float*)c->cbuf1, c->k,
                               (const km::Quant*)c->quant));
    return ls.end();
}

int launch_assign_d(km_ctx* c, const float* pts, const float* C, int32_t* labels, int first, bool fuse,
                    const km::Ctl* ctl, float fin_tol = NAN, bool incr = false)
{
    return c->d == 2 ? launch_assign<2>(c, pts, C, labels, first, fuse, ctl, fin_tol, incr)
                     : launch_assign<3>(c, pts, C, labels, first, fuse, ctl, fin_tol, incr);
}

int launch_quant(km_ctx* c, const float* pts)
{
    {
        LaunchScope ls(c, 2);
        if (c->d == 2) km::bbox_kernel<2><<<c->aux_grid, 256, 0, c->stream>>>(pts, c->n, c->bbox_part);
        else km::bbox_kernel<3><<<c->aux_grid, 256, 0, c->stream>>>(pts, c->n, c->bbox_part);
        int rc = ls.end();
        if (rc) return rc;
    }
    LaunchScope ls(c, 2);
    if (c->d == 2) km::quant_kernel<2><<<1, 256, 0, c->stream>>>(c->bbox_part, c->aux_grid, c->n, c->quant, nullptr);
    else km::quant_kernel<3><<<1, 256, 0, c->stream>>>(c->bbox_part, c->aux_grid, c->n, c->quant, nullptr);
    return ls.end();
}

// The refine's arguments (finalize_kernel, or the fused tail of the brute-force assignment).
// tiles: running sums in tacc (kept), SSE_t partials in fixed point, inter bound reset.
// dp: the all-reduced partials were imported into acc_sum / sse_part[0].
km::FinArgs fin_args(km_ctx* c, const float* Cold, float* Cnew, int32_t* counts, double* maxdrift, bool traces,
                     km::Ctl* ctl, float tol, int nparts, bool tiles, bool dp)
{
    km::FinArgs f{};
    f.Cold = Cold;
    f.Cnew = Cnew;
    f.k = c->k;
    f.acc_sum = tiles && !dp ? c->tacc_sum : c->acc_sum;
    f.acc_cnt = tiles && !dp ? c->tacc_cnt : c->acc_cnt;
    f.ncopy = tiles && !dp ? kAccCopies : 1;
    f.clear = tiles && !dp ? 0 : 1;
    f.quant = c->quant;
    f.counts_out = counts;
    f.maxdrift_out = maxdrift;
    f.sse_part = c->sse_part;
    f.sseq_part = tiles && !dp ? c->ttot : nullptr;
    f.chg_part = tiles && !dp ? c->ttot + 1 : c->chg_part;
    f.nparts = tiles && !dp ? 1 : nparts;
    f.sse_trace = traces ? c->sse_trace : nullptr;
    f.chg_trace = traces ? c->chg_trace : nullptr;
    f.drift_trace = traces ? c->drift_trace : nullptr;
    f.cb2_reset = tiles ? c->cb2 : nullptr;
    f.tot_reset = tiles && !dp ? c->ttot : nullptr;
    f.ctl = ctl;
    f.tol = tol;
    return f;
}

int launch_finalize(km_ctx* c, const float* Cold, float* Cnew, int32_t* counts, double* maxdrift, bool traces,
                    km::Ctl* ctl, float tol, int nparts, bool tiles = false, bool dp = false)
{
    // tiles: running sums in tacc (kept), SSE_t partials in fixed point, inter bound reset.
    // dp: the all-reduced partials were imported into acc_sum / sse_part[0].
    if (tiles && !dp && traces && ctl && !counts && !maxdrift) {
        // the tile path inside km_run_ctx: the multi-CTA refine
        LaunchScope ls(c, 1);
        const int g = (c->k + 255) / 256;
        if (c->d == 2)
            km::finalize_grid_kernel<2><<<g, 256, 0, c->stream>>>(Cnew, c->k, c->tacc_sum, c->tacc_cnt, kAccCopies,
                                                                   c->quant, c->ttot, c->cb2, c->tfin, c->sse_trace,
                                                                   c->chg_trace, c->drift_trace, ctl, tol);
        else
            km::finalize_grid_kernel<3><<<g, 256, 0, c->stream>>>(Cnew, c->k, c->tacc_sum, c->tacc_cnt, kAccCopies,
                                                                   c->quant, c->ttot, c->cb2, c->tfin, c->sse_trace,
                                                                   c->chg_trace, c->drift_trace, ctl, tol);
        return ls.end();
    }
    LaunchScope ls(c, 1);
    const km::FinArgs f = fin_args(c, Cold, Cnew, counts, maxdrift, traces, ctl, tol, nparts, tiles, dp);
    if (c->d == 2) km::finalize_kernel<2><<<1, km::kFinalizeThreads, 0, c->stream>>>(f);
    else km::finalize_kernel<3><<<1, km::kFinalizeThreads, 0, c->stream>>>(f);
    return ls.end();
}

// ---------------------------------------------------------------- tile-pruned path
template <typename T>
int dmalloc(T** p, size_t count);

size_t tiles_smem_bytes(int d)
{
    return (size_t)km::kK1tWarps * (d == 2 ? sizeof(km::WarpSmem<2>) : sizeof(km::WarpSmem<3>));
}

int morton_key_bits(int d, int64_t n) { return d * km::morton_bits(d, n); }

bool tiles_supported(const km_ctx* c) { return !c->hd && c->k <= km::kMaxPruneRounds * km::kTileThreads; }

// KM_MODE_AUTO: the index pays off once the brute-force scan is long; below ~3e8 point-centroid
// pairs per iteration the one-launch brute-force iteration is faster (measured: config 2, n = 1e6,
// k = 100: 34 vs 49 us per iteration; config 3, k = 1000: 264 vs 83 us)
bool bounds_supported(const km_ctx* c) { return !c->hd && c->bounds_grid > 0 && c->n <= (int64_t)INT32_MAX; }
// AUTO takes the bounds for the brute-force problems whose s_a test fits every CTA (k <= 256)
bool auto_bounds(const km_ctx* c) { return bounds_supported(c) && c->k <= km::kBoundsMaxKS; }
bool small_run(const km_ctx* c);
bool auto_tiles(const km_ctx* c);
// km_run_ctx's path: 0 brute force (or the one-cluster small run), 1 tiles, 2 high-d, 3 bounds
int run_path(const km_ctx* c)
{
    if (c->hd) return 2;
    if (c->mode == KM_MODE_TILES || (c->mode == KM_MODE_AUTO && auto_tiles(c))) return 1;
    if (c->mode == KM_MODE_BOUNDS) return 3;
    if (c->mode == KM_MODE_AUTO && !small_run(c) && auto_bounds(c)) return 3;
    return 0;
}

int ensure_bounds(km_ctx* c)
{
    if (c->lbv) return KM_OK;
    if (dmalloc(&c->lbv, (size_t)c->n) || dmalloc(&c->cbuf1, (size_t)c->k * c->d) || dmalloc(&c->bscan, 8) ||
        dmalloc(&c->bsum, (size_t)5 * c->k * c->d) || dmalloc(&c->bcnt, (size_t)5 * c->k)) {
        cudaFree(c->lbv); cudaFree(c->cbuf1); cudaFree(c->bscan); cudaFree(c->bsum); cudaFree(c->bcnt);
        c->lbv = nullptr; c->cbuf1 = nullptr; c->bscan = nullptr; c->bsum = nullptr; c->bcnt = nullptr;
        return KM_E_NOMEM;
    }
    return KM_OK;
}

bool auto_tiles(const km_ctx* c) { return tiles_supported(c) && c->n >= 16384 && (double)c->n * c->k >= 3e8; }

// K1t's shared-memory attribute and residency for register budget MB (FIRST and later variants)
template <int D, int MB>
int k1t_setup(km_ctx* c, int* nb, int* nb0)
{
    KM_CUDA(cudaFuncSetAttribute(km::assign_tiles_kernel<D, true, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)c->tiles_smem));
    KM_CUDA(cudaFuncSetAttribute(km::assign_tiles_kernel<D, false, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)c->tiles_smem));
    KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, km::assign_tiles_kernel<D, false, MB>, km::kK1tThreads,
                                                          c->tiles_smem));
    KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb0, km::assign_tiles_kernel<D, true, MB>, km::kK1tThreads,
                                                          c->tiles_smem));
    return KM_OK;
}

template <int D>
int configure_tiles(km_ctx* c)
{
    c->tiles_kpad = round_up4(c->k);
    c->tiles_smem = tiles_smem_bytes(D);
#ifndef KM_K1T_SMALL_TILES
#define KM_K1T_SMALL_TILES 40000
#endif
    const int64_t ntl = (c->n + km::kTilePoints - 1) / km::kTilePoints;
#ifndef KM_K1T_MINB_LARGE
#define KM_K1T_MINB_LARGE (16 / KM_K1T_WARPS)   // 128 registers: 16 warps per SM
#endif
    // 2-D problems (config 5) run K1t at 5 CTAs of 4 warps per SM (96 registers, 60 B of spills:
    // -4 % per launch), 3-D ones at 4 (128 registers: the 96-register build is +7 % at config 4)
    c->k1t_minb = ntl < KM_K1T_SMALL_TILES ? 1 : (D == 2 && KM_K1T_WARPS == 4 ? 5 : KM_K1T_MINB_LARGE);
    // super-tiles of 8 tiles in 3-D (configs 3 / 4: -4 % / -2 % against 16), 16 or 32 tiles in 2-D
    // (configs 2 / 5: 8 would cost +5 % / +7 %; profiles/r01/s2/super_tile_ab.txt); km_debug_set
    // overrides (KM_DBG_ST_SHIFT 2..5, KM_DBG_K1T_MINB 1 / 2 / 3)
    c->st_shift = D == 3 ? 3 : (c->k >= 4096 ? 5 : 4);   // 2-D, k >= 4096: 32 tiles (config 5 -0.6 %)
    if (c->dbg_st_shift) c->st_shift = c->dbg_st_shift;
    // few tiles (config 3: 7.8 k tiles, 977 level-1 nodes): the node-per-warp prune does not fill the
    // GPU, so shorter lists already hand their tiles to tile_cands_kernel (one warp per tile).
    // Config 3, ms per run: 64 -> 1.59, 48 -> 1.53, 32 -> 1.48, 16 -> 1.46, <= 12 -> 1.45;
    // config 4: 64 -> 3.68, 48 -> 3.67, 32 -> 3.71; config 5: no change (gpurun A/B, round 2)
    c->short_list = c->dbg_short_list ? c->dbg_short_list : (ntl < 16384 ? 12 : ntl < 32768 ? 32 : km::kShortList);
    if (c->dbg_minb) c->k1t_minb = c->dbg_minb;
    int nb = 0, nb0 = 0;
    int rc0 = c->k1t_minb == 1 ? k1t_setup<D, 1>(c, &nb, &nb0)
              : c->k1t_minb == 3 ? k1t_setup<D, 3>(c, &nb, &nb0)
#if KM_K1T_WARPS < 8
              : c->k1t_minb == 4 ? k1t_setup<D, 4>(c, &nb, &nb0)
              : c->k1t_minb == 5 ? k1t_setup<D, 5>(c, &nb, &nb0)
#endif
                                 : k1t_setup<D, 2>(c, &nb, &nb0);
    if (rc0) return rc0;
    nb = std::min(nb, nb0);
    if (nb < 1) return KM_E_UNSUPPORTED;
    nb = std::min(nb, 64 / km::kK1tWarps);
    c->ntiles = (int)((c->n + km::kTilePoints - 1) / km::kTilePoints);
    // level sizes: level 1 groups 1 << st_shift tiles, higher levels kFanout nodes, up to <= 256 roots
    c->lev_n[0] = c->ntiles;
    c->nlev = 1;
    while (c->nlev < km_ctx::kMaxLev) {
        const int fan = c->nlev == 1 ? (1 << c->st_shift) : km::kFanout;
        const int nn = (c->lev_n[c->nlev - 1] + fan - 1) / fan;
        c->lev_fan[c->nlev] = fan;
        c->lev_n[c->nlev] = nn;
        // level 1 stores up to min(k, 1024) records per node (a longer list inherits the parent's)
        c->lev_cap[c->nlev] = c->nlev == 1 ? std::min(c->k, km::kL1Store) : c->k;
        c->nlev++;
        if (nn <= 256) break;
        // small k: level 1 prunes all k directly (one launch instead of a chain of levels)
        if (c->k <= KM_FLAT_K && c->nlev == 2) break;
    }
    c->tiles_grid = std::max(1, std::min((c->ntiles + km::kK1tWarps - 1) / km::kK1tWarps, c->num_sms * nb));
    c->filter_grid = std::max(1, std::min((c->ntiles + 255) / 256, c->num_sms * 8));
    KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->np_res, km::node_prune_kernel<D>, km::kTileThreads, 0));
    c->np_res = std::max(1, c->np_res);
    KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->tc_res, km::tile_cands_kernel<D>, km::kTileThreads, 0));
    c->tc_res = std::max(1, c->tc_res);
    if (c->k <= km::kNodeRegQ * 32) {
        const size_t fsm = km::flat_prune_smem<D>(c->k);
        KM_CUDA(cudaFuncSetAttribute(km::node_prune_flat_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
        KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->npf_res, km::node_prune_flat_kernel<D>,
                                                              km::kTileThreads, fsm));
        c->npf_res = std::max(1, c->npf_res);
    }
    c->ovf_cap = (int)std::min<long long>((long long)c->ntiles * 16 + (1 << 20), 1ll << 30);
    // Eq. 3: grid (ceil(k/256), S), S chunks of the k centroids, ~2 CTAs per SM in total
    c->ib_jb = c->k > 2048 ? 4 : 1;   // centroids per thread (register blocking for large k)
    c->ib_gx = (c->k + 256 * c->ib_jb - 1) / (256 * c->ib_jb);
    c->ib_gy = std::max(1, std::min((c->k + 63) / 64, (2 * c->num_sms + c->ib_gx - 1) / c->ib_gx));
    c->ib_chunk = (c->k + c->ib_gy - 1) / c->ib_gy;
    c->ib_gy = (c->k + c->ib_chunk - 1) / c->ib_chunk;
    if ((size_t)c->ib_chunk * D * 4 > 48 * 1024) {
        KM_CUDA(cudaFuncSetAttribute(km::interbound_kernel<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((size_t)c->ib_chunk * D * 4)));
        KM_CUDA(cudaFuncSetAttribute(km::interbound_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((size_t)c->ib_chunk * D * 4)));
    }
    return KM_OK;
}

void free_tiles(km_ctx* c)
{
    auto f = [](auto*& p) { cudaFree((void*)p); p = nullptr; };
    f(c->ps); f(c->ls); f(c->keys[0]); f(c->keys[1]); f(c->idx[0]); f(c->idx[1]); f(c->tgeom); f(c->tlab);
    f(c->stats); f(c->lpool); f(c->cb2); f(c->taux); f(c->tcand); f(c->ovf_cur); f(c->heavy); f(c->sbucket); f(c->scursor); f(c->work); f(c->work_cnt); f(c->l1need); f(c->ttot);
    f(c->tfin); f(c->tacc_sum); f(c->tacc_cnt); f(c->ovf); f(c->theavy); f(c->cub_tmp);
    for (int l = 0; l < km_ctx::kMaxLev; ++l) { f(c->lev_geom[l]); f(c->lev_ref[l]); }
    c->perm = nullptr;
}

int ensure_tiles_alloc(km_ctx* c)
{
    const size_t n = (size_t)c->n;
    int rc = c->d == 2 ? configure_tiles<2>(c) : configure_tiles<3>(c);
    if (rc) return rc;
    // +16 elements: the last tile's bulk copies round their size up to 16 B
    if (dmalloc(&c->ps, n * c->d + 16) || dmalloc(&c->ls, n + 16) || dmalloc(&c->keys[0], n) || dmalloc(&c->keys[1], n) ||
        dmalloc(&c->idx[0], n) || dmalloc(&c->idx[1], n) || dmalloc(&c->tgeom, (size_t)c->ntiles) ||
        dmalloc(&c->tlab, (size_t)c->ntiles) || dmalloc(&c->stats, 32) ||
        dmalloc(&c->lev_geom[0], (size_t)c->ntiles))
        return KM_E_NOMEM;
    long long pool_sz = 0;
    for (int l = 1; l < c->nlev; ++l) {
        c->lev_off[l] = pool_sz;
        pool_sz += (long long)c->lev_n[l] * c->lev_cap[l];
        if (dmalloc(&c->lev_geom[l], (size_t)c->lev_n[l]) || dmalloc(&c->lev_ref[l], (size_t)c->lev_n[l]))
            return KM_E_NOMEM;
    }
    if (dmalloc(&c->lpool, (size_t)pool_sz)) return KM_E_NOMEM;
    if (!c->aux) KM_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    if (!c->ev_c) KM_CUDA(cudaEventCreateWithFlags(&c->ev_c, cudaEventDisableTiming));
    if (!c->ev_f) KM_CUDA(cudaEventCreateWithFlags(&c->ev_f, cudaEventDisableTiming));
    if (dmalloc(&c->cb2, (size_t)c->k) || dmalloc(&c->taux, (size_t)c->ntiles) ||
        dmalloc(&c->tcand, (size_t)c->ntiles * (c->d + 1) * km::kTC) || dmalloc(&c->ovf_cur, 8) || dmalloc(&c->heavy, (size_t)std::max(1, c->lev_n[1])) ||
        dmalloc(&c->work, (size_t)c->ntiles) || dmalloc(&c->work_cnt, 8) ||
        dmalloc(&c->l1need, (size_t)std::max(1, c->lev_n[1])) || dmalloc(&c->ttot, 2) || dmalloc(&c->tfin, 2) ||
        dmalloc(&c->tacc_sum, (size_t)kAccCopies * c->k * c->d) || dmalloc(&c->tacc_cnt, (size_t)kAccCopies * c->k) ||
        dmalloc(&c->ovf, (size_t)c->ovf_cap) || dmalloc(&c->theavy, (size_t)c->ntiles))
        return KM_E_NOMEM;
    if (c->n > KM_SCATTER_WIN && (int64_t)((c->n + KM_SCATTER_WIN - 1) / KM_SCATTER_WIN) <= km::kScatterMaxWin) {
        // the label scatter's window buckets (optional: without them every window re-reads all n)
        if (dmalloc(&c->sbucket, (size_t)(c->n - KM_SCATTER_WIN)) || dmalloc(&c->scursor, (size_t)km::kScatterMaxWin)) {
            cudaFree(c->sbucket); cudaFree(c->scursor);
            c->sbucket = nullptr; c->scursor = nullptr;
            cudaGetLastError();
        }
    }
    size_t bytes = 0;
    KM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, c->keys[0], c->keys[1], c->idx[0], c->idx[1], (int)n, 0,
                                            morton_key_bits(c->d, c->n), c->stream));
    c->cub_bytes = bytes;
    if (dmalloc((char**)&c->cub_tmp, bytes + 256)) return KM_E_NOMEM;
    return KM_OK;
}

// Tile-path workspace, allocated at the first tile run; on failure everything allocated so far
// is released (a later call retries from scratch).
int ensure_tiles(km_ctx* c)
{
    if (c->tiles_ready) return KM_OK;
    int rc = ensure_tiles_alloc(c);
    if (rc) {
        free_tiles(c);
        return rc;
    }
    c->tiles_ready = true;
    return KM_OK;
}

// Once per run: Morton keys, sort, gather, per-tile geometry and moments (the paper's
// "Create Ball-tree on D", Alg. 1 line 1, as a flat tile index).  Needs quant.
int prepare_tiles(km_ctx* c, const float* P)
{
    const int64_t n = c->n;
    {
        LaunchScope ls(c, 2);
        if (c->d == 2) km::morton_kernel<2><<<c->aux_grid, 256, 0, c->stream>>>(P, n, c->quant, km::morton_bits(2, n),
                                                                          c->keys[0], c->idx[0]);
        else km::morton_kernel<3><<<c->aux_grid, 256, 0, c->stream>>>(P, n, c->quant, km::morton_bits(3, n),
                                                                          c->keys[0], c->idx[0]);
        int rc = ls.end();
        if (rc) return rc;
    }
    {
        LaunchScope ls(c, 2);
        size_t bytes = c->cub_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(c->cub_tmp, bytes, c->keys[0], c->keys[1], c->idx[0],
                                                        c->idx[1], (int)n, 0, morton_key_bits(c->d, c->n), c->stream);
        if (e != cudaSuccess) return cuda_fail(e);
        int rc = ls.end();
        if (rc) return rc;
        c->perm = c->idx[1];
    }
    {   // gather into the sorted copy + per-tile geometry + level-0 balls, one pass
        LaunchScope ls(c, 2);
        const int g = std::min((c->ntiles + 7) / 8, c->num_sms * 8);
        if (c->d == 2)
            km::tile_geom_kernel<2, true><<<g, km::kTileThreads, 0, c->stream>>>(P, c->perm, c->ps, n, c->ntiles, c->quant,
                                                                                c->keys[1], c->tgeom, c->lev_geom[0]);
        else
            km::tile_geom_kernel<3, true><<<g, km::kTileThreads, 0, c->stream>>>(P, c->perm, c->ps, n, c->ntiles, c->quant,
                                                                                c->keys[1], c->tgeom, c->lev_geom[0]);
        int rc = ls.end();
        if (rc) return rc;
    }
    for (int l = 1; l < c->nlev; ++l) {
        LaunchScope ls(c, 2);
        const int g = std::min((c->lev_n[l] + 127) / 128, 4096);
        if (c->d == 2)
            km::level_geom_kernel<2><<<g, 128, 0, c->stream>>>(c->lev_geom[l - 1], c->lev_n[l - 1], c->lev_fan[l],
                                                               c->lev_n[l], c->lev_geom[l]);
        else
            km::level_geom_kernel<3><<<g, 128, 0, c->stream>>>(c->lev_geom[l - 1], c->lev_n[l - 1], c->lev_fan[l],
                                                               c->lev_n[l], c->lev_geom[l]);
        int rc = ls.end();
        if (rc) return rc;
    }
    KM_CUDA(cudaMemsetAsync(c->tlab, 0xff, sizeof(km::TileState) * c->ntiles, c->stream));
    KM_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(unsigned long long) * 32, c->stream));
    // running sums start at 0; cb2 bytes 0x7f -> 3.4e38 (no bound) until the first Eq. 3 pass
    KM_CUDA(cudaMemsetAsync(c->tacc_sum, 0, sizeof(unsigned long long) * kAccCopies * c->k * c->d, c->stream));
    KM_CUDA(cudaMemsetAsync(c->tacc_cnt, 0, sizeof(unsigned int) * kAccCopies * c->k, c->stream));
    KM_CUDA(cudaMemsetAsync(c->cb2, 0x7f, sizeof(unsigned int) * c->k, c->stream));
    KM_CUDA(cudaMemsetAsync(c->l1need, 0, sizeof(int) * std::max(1, c->lev_n[1]), c->stream));
    KM_CUDA(cudaMemsetAsync(c->theavy, 0, (size_t)c->ntiles, c->stream));
    KM_CUDA(cudaMemsetAsync(c->ttot, 0, 2 * sizeof(unsigned long long), c->stream));
    KM_CUDA(cudaMemsetAsync(c->tfin, 0, 2 * sizeof(unsigned long long), c->stream));
    KM_CUDA(cudaMemsetAsync(c->work_cnt, 0, 8 * sizeof(int), c->stream));
    return KM_OK;
}


int launch_assign_tiles(km_ctx* c, const float* C, int first)
{
    const int D = c->d;
    // fork: [inter bound -> tile filter] on the aux stream, the index levels >= 2 on the main
    // stream; join before the level-1 prune (it needs the filter's node marks)
    KM_CUDA(cudaEventRecord(c->ev_c, c->stream));
    KM_CUDA(cudaStreamWaitEvent(c->aux, c->ev_c, 0));
    // Eq. 3: inter bound cb[j] of this iteration's centroids (also clears the work counter)
    if (!first) {
        LaunchScope ls(c, 2, c->aux);
        dim3 g(c->ib_gx, c->ib_gy);
        const size_t sm = (size_t)c->ib_chunk * D * 4;
        if (D == 2 && c->ib_jb == 4)
            km::interbound_kernel<2, 4><<<g, 256, sm, c->aux>>>(C, c->k, c->ib_chunk, c->cb2, c->work_cnt, c->ctl);
        else if (D == 2)
            km::interbound_kernel<2, 1><<<g, 256, sm, c->aux>>>(C, c->k, c->ib_chunk, c->cb2, c->work_cnt, c->ctl);
        else if (c->ib_jb == 4)
            km::interbound_kernel<3, 4><<<g, 256, sm, c->aux>>>(C, c->k, c->ib_chunk, c->cb2, c->work_cnt, c->ctl);
        else
            km::interbound_kernel<3, 1><<<g, 256, sm, c->aux>>>(C, c->k, c->ib_chunk, c->cb2, c->work_cnt, c->ctl);
        int rc = ls.end();
        if (rc) return rc;
    } else {
        // slots 0-3 and 5-7 (slot 4, the level-1 pool cursor, is the main stream's: below)
        KM_CUDA(cudaMemsetAsync(c->work_cnt, 0, 4 * sizeof(int), c->aux));
        KM_CUDA(cudaMemsetAsync(c->work_cnt + 5, 0, 3 * sizeof(int), c->aux));
    }
    // Eq. 5 on every tile -> work list of the rest, level-1 nodes they need
    {
        LaunchScope ls(c, 2, c->aux);
        if (D == 2)
            km::tile_filter_kernel<2><<<c->filter_grid, 256, 0, c->aux>>>(
                c->tgeom, c->tlab, c->ntiles, C, c->cb2, first, c->work, c->work_cnt, c->l1need, c->theavy, c->taux,
                c->ttot, c->ttot + 1, c->quant, c->ctl, c->stats, c->st_shift);
        else
            km::tile_filter_kernel<3><<<c->filter_grid, 256, 0, c->aux>>>(
                c->tgeom, c->tlab, c->ntiles, C, c->cb2, first, c->work, c->work_cnt, c->l1need, c->theavy, c->taux,
                c->ttot, c->ttot + 1, c->quant, c->ctl, c->stats, c->st_shift);
        int rc = ls.end();
        if (rc) return rc;
    }
    KM_CUDA(cudaEventRecord(c->ev_f, c->aux));
    // candidate lists top-down for this iteration's centroids (Eq. 7-8 bounds from the parent):
    // levels >= 2 one CTA per node (the roots from all k), level 1 one warp per needed node
    const int top = c->nlev - 1;
    for (int l = top; l >= 2; --l) {
        LaunchScope ls(c, 2);
        const int g = std::min(c->lev_n[l], c->num_sms * 8);
        const km::NodeRef* pref = l == top ? nullptr : c->lev_ref[l + 1];
        const int fan = l == top ? 1 : c->lev_fan[l + 1];
        if (D == 2)
            km::cta_prune_kernel<2><<<g, km::kTileThreads, 0, c->stream>>>(c->lev_geom[l], c->lev_n[l], fan, pref, C,
                                                                          c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                                                                          c->lev_ref[l], nullptr, nullptr, c->ctl, km::TileCandOut{});
        else
            km::cta_prune_kernel<3><<<g, km::kTileThreads, 0, c->stream>>>(c->lev_geom[l], c->lev_n[l], fan, pref, C,
                                                                          c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                                                                          c->lev_ref[l], nullptr, nullptr, c->ctl, km::TileCandOut{});
        int rc = ls.end();
        if (rc) return rc;
    }
    // flat index (level 1 prunes all k): no level chain to hide the filter behind, so level 1
    // prunes every node (no need mask) beside the filter and the join moves after it
    const bool flat = top == 1;
    if (!flat) KM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_f, 0));   // join
    int* const l1need = flat ? nullptr : c->l1need;
    // level 1: one CTA per needed node when the parent lists are long (k > 2048: measured faster
    // at config 5), else one warp per node with the parent list staged once per 8 nodes
#ifndef KM_L1_CTA_MINK
#define KM_L1_CTA_MINK 2048
#endif
    // the level-1 prune also writes every tile's candidate list (tile_cands_warp): its overflow
    // pool cursor is reset on this stream, ordered before the prune
    KM_CUDA(cudaMemsetAsync(c->ovf_cur, 0, 8 * sizeof(int), c->stream));
    const km::TileCandOut tco{c->tgeom, c->tcand, c->taux, c->ovf, c->ovf_cur, c->heavy, c->ovf_cap, c->ntiles,
                              c->st_shift, c->stats, c->lev_n[1], c->short_list};
    if (c->k > KM_L1_CTA_MINK) {
        // the pool cursor of the per-node allocation: reset on this stream, ordered before the
        // prune (the aux stream's counter resets never touch slot 4)
        KM_CUDA(cudaMemsetAsync(c->work_cnt + 4, 0, sizeof(int), c->stream));
        LaunchScope ls(c, 2);
        const int l = 1;
        const int g = std::min(c->lev_n[l], c->num_sms * 8);
        const km::NodeRef* pref = top == 1 ? nullptr : c->lev_ref[l + 1];
        const int fan = top == 1 ? 1 : c->lev_fan[l + 1];
        if (D == 2)
            km::cta_prune_kernel<2><<<g, km::kTileThreads, 0, c->stream>>>(c->lev_geom[l], c->lev_n[l], fan, pref, C,
                                                                          c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                                                                          c->lev_ref[l], l1need, c->work_cnt + 4,
                                                                          c->ctl, tco);
        else
            km::cta_prune_kernel<3><<<g, km::kTileThreads, 0, c->stream>>>(c->lev_geom[l], c->lev_n[l], fan, pref, C,
                                                                          c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                                                                          c->lev_ref[l], l1need, c->work_cnt + 4,
                                                                          c->ctl, tco);
        int rc = ls.end();
        if (rc) return rc;
    } else if (flat && c->k <= km::kNodeRegQ * 32) {
        // all k staged once per CTA; warps take level-1 nodes independently
        LaunchScope ls(c, 2);
        const int g = std::min((c->lev_n[1] + km::kWarpsPerCta - 1) / km::kWarpsPerCta, c->num_sms * c->npf_res);
        const size_t sm = D == 2 ? km::flat_prune_smem<2>(c->k) : km::flat_prune_smem<3>(c->k);
        if (D == 2)
            km::node_prune_flat_kernel<2><<<g, km::kTileThreads, sm, c->stream>>>(
                c->lev_geom[1], c->lev_n[1], C, c->k, c->lpool, c->lev_off[1], c->lev_cap[1], c->lev_ref[1], c->ctl, tco);
        else
            km::node_prune_flat_kernel<3><<<g, km::kTileThreads, sm, c->stream>>>(
                c->lev_geom[1], c->lev_n[1], C, c->k, c->lpool, c->lev_off[1], c->lev_cap[1], c->lev_ref[1], c->ctl, tco);
        int rc = ls.end();
        if (rc) return rc;
    } else {
        LaunchScope ls(c, 2);
        const int l = 1;
        const int g = std::min((c->lev_n[l] + km::kPruneGroup - 1) / km::kPruneGroup, c->num_sms * c->np_res);
        const km::NodeRef* pref = top == 1 ? nullptr : c->lev_ref[l + 1];
        const int fan = top == 1 ? 1 : c->lev_fan[l + 1];
        if (D == 2)
            km::node_prune_kernel<2><<<g, km::kTileThreads, 0, c->stream>>>(
                c->lev_geom[l], c->lev_n[l], fan, pref, C, c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                c->lev_ref[l], l1need, c->ctl, tco);
        else
            km::node_prune_kernel<3><<<g, km::kTileThreads, 0, c->stream>>>(
                c->lev_geom[l], c->lev_n[l], fan, pref, C, c->k, c->lpool, c->lev_off[l], c->lev_cap[l],
                c->lev_ref[l], l1need, c->ctl, tco);
        int rc = ls.end();
        if (rc) return rc;
    }
    {   // the tiles of long level-1 lists: one warp each
        LaunchScope ls(c, 2);
        if (D == 2)
            km::tile_cands_kernel<2><<<c->num_sms * c->tc_res, km::kTileThreads, 0, c->stream>>>(
                c->lev_ref[1], c->lpool, C, c->ctl, tco);
        else
            km::tile_cands_kernel<3><<<c->num_sms * c->tc_res, km::kTileThreads, 0, c->stream>>>(
                c->lev_ref[1], c->lpool, C, c->ctl, tco);
        int rc = ls.end();
        if (rc) return rc;
    }
    if (flat) KM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_f, 0));   // join
    LaunchScope ls(c, 0);
#define KM_K1T_ARGS                                                                                           \
    c->ps, c->n, c->work, c->work_cnt, c->tgeom, c->tlab, c->taux, c->tcand, c->lpool, c->lev_ref[1], C, c->k,   \
        c->ls, c->ttot, c->ttot + 1, c->tacc_sum, c->tacc_cnt, kAccCopies, c->ovf, c->theavy, c->quant, c->ctl,   \
        c->stats, c->st_shift
#define KM_K1T_LAUNCH(DD, FF, MB) \
    km::assign_tiles_kernel<DD, FF, MB><<<c->tiles_grid, km::kK1tThreads, c->tiles_smem, c->stream>>>(KM_K1T_ARGS)
    if (c->k1t_minb == 1) {
        if (D == 2 && first) KM_K1T_LAUNCH(2, true, 1);
        else if (D == 2) KM_K1T_LAUNCH(2, false, 1);
        else if (first) KM_K1T_LAUNCH(3, true, 1);
        else KM_K1T_LAUNCH(3, false, 1);
    } else if (c->k1t_minb == 3) {
        if (D == 2 && first) KM_K1T_LAUNCH(2, true, 3);
        else if (D == 2) KM_K1T_LAUNCH(2, false, 3);
        else if (first) KM_K1T_LAUNCH(3, true, 3);
        else KM_K1T_LAUNCH(3, false, 3);
#if KM_K1T_WARPS < 8
    } else if (c->k1t_minb == 4) {
        if (D == 2 && first) KM_K1T_LAUNCH(2, true, 4);
        else if (D == 2) KM_K1T_LAUNCH(2, false, 4);
        else if (first) KM_K1T_LAUNCH(3, true, 4);
        else KM_K1T_LAUNCH(3, false, 4);
    } else if (c->k1t_minb == 5) {
        if (D == 2 && first) KM_K1T_LAUNCH(2, true, 5);
        else if (D == 2) KM_K1T_LAUNCH(2, false, 5);
        else if (first) KM_K1T_LAUNCH(3, true, 5);
        else KM_K1T_LAUNCH(3, false, 5);
#endif
    } else {
        if (D == 2 && first) KM_K1T_LAUNCH(2, true, 2);
        else if (D == 2) KM_K1T_LAUNCH(2, false, 2);
        else if (first) KM_K1T_LAUNCH(3, true, 2);
        else KM_K1T_LAUNCH(3, false, 2);
    }
#undef KM_K1T_LAUNCH
#undef KM_K1T_ARGS
    return ls.end();
}


// Labels back to input order, windowed; the first window's pass also sums Eq. 1 of the returned
// pair over the sorted points (the bound kernel before it, the 128-bit total after it).
int launch_scatter_labels(km_ctx* c, int32_t* out)
{
    {
        LaunchScope ls(c, 2);
        if (c->d == 2) km::sse_bound_kernel<2><<<1, km::kReduceThreads, 0, c->stream>>>(c->quant, c->cwork, c->k, c->s3);
        else km::sse_bound_kernel<3><<<1, km::kReduceThreads, 0, c->stream>>>(c->quant, c->cwork, c->k, c->s3);
        int rc = ls.end();
        if (rc) return rc;
    }
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 4, (c->n + 255) / 256));
    // destination windows of KM_SCATTER_WIN labels (default 12 M = 48 MB): the scattered stores
    // stay L2-resident
    constexpr int64_t kWin = KM_SCATTER_WIN;
    const int nwin = (int)((c->n + kWin - 1) / kWin);
    if (nwin > 1 && nwin <= km::kScatterMaxWin && c->sbucket) {
        {   // window 0 + Eq. 1 + the other windows' buckets
            KM_CUDA(cudaMemsetAsync(c->scursor, 0, sizeof(unsigned long long) * nwin, c->stream));
            LaunchScope ls(c, 2);
            if (c->d == 2)
                km::scatter_bucket_kernel<2, true><<<g, 256, 0, c->stream>>>(c->ls, c->n, c->perm, out, (unsigned)kWin,
                                                                           nwin, c->ps, c->cwork, c->s3, c->sse128,
                                                                           c->sbucket, c->scursor);
            else
                km::scatter_bucket_kernel<3, true><<<g, 256, 0, c->stream>>>(c->ls, c->n, c->perm, out, (unsigned)kWin,
                                                                           nwin, c->ps, c->cwork, c->s3, c->sse128,
                                                                           c->sbucket, c->scursor);
            int rc = ls.end();
            if (rc) return rc;
        }
        for (int w = 1; w < nwin; ++w) {
            LaunchScope ls(c, 2);
            const int64_t cnt = std::min<int64_t>(c->n, (int64_t)(w + 1) * kWin) - (int64_t)w * kWin;
            km::scatter_window_kernel<<<c->num_sms * 4, 256, 0, c->stream>>>(c->sbucket + (int64_t)(w - 1) * kWin, cnt,
                                                                            out);
            int rc = ls.end();
            if (rc) return rc;
        }
        LaunchScope ls(c, 2);
        km::sse_fix_reduce_kernel<<<1, km::kReduceThreads, 0, c->stream>>>(c->sse128, g, c->s3,
                                                                            reinterpret_cast<km::SseFix*>(c->scal));
        return ls.end();
    }
    for (int64_t w0 = 0; w0 < c->n; w0 += kWin) {
        LaunchScope ls(c, 2);
        const int64_t w1 = std::min<int64_t>(c->n, w0 + kWin);
        if (w0 == 0) {
            if (c->d == 2)
                km::scatter_labels_kernel<2, true><<<g, 256, 0, c->stream>>>(c->ls, c->n, c->perm, out, (unsigned)w0,
                                                                           (unsigned)w1, c->ps, c->cwork, c->s3,
                                                                           c->sse128);
            else
                km::scatter_labels_kernel<3, true><<<g, 256, 0, c->stream>>>(c->ls, c->n, c->perm, out, (unsigned)w0,
                                                                           (unsigned)w1, c->ps, c->cwork, c->s3,
                                                                           c->sse128);
        } else {
            km::scatter_labels_kernel<2, false><<<g, 256, 0, c->stream>>>(c->ls, c->n, c->perm, out, (unsigned)w0,
                                                                        (unsigned)w1, nullptr, nullptr, nullptr,
                                                                        nullptr);
        }
        int rc = ls.end();
        if (rc) return rc;
    }
    LaunchScope ls(c, 2);
    km::sse_fix_reduce_kernel<<<1, km::kReduceThreads, 0, c->stream>>>(c->sse128, g, c->s3,
                                                                        reinterpret_cast<km::SseFix*>(c->scal));
    return ls.end();
}

// Eq. 1 of (labels, C) as an order-independent 128-bit fixed-point sum -> c->scal
// (km::SseFix): the bound B of every term and its exponent, the per-CTA partials, the total.
int launch_final_sse(km_ctx* c, const float* pts, const int32_t* labels, const float* C)
{
    {
        LaunchScope ls(c, 2);
        if (c->d == 2) km::sse_bound_kernel<2><<<1, km::kReduceThreads, 0, c->stream>>>(c->quant, C, c->k, c->s3);
        else km::sse_bound_kernel<3><<<1, km::kReduceThreads, 0, c->stream>>>(c->quant, C, c->k, c->s3);
        int rc = ls.end();
        if (rc) return rc;
    }
    {
        LaunchScope ls(c, 2);
        if (c->d == 2) km::sse_kernel<2><<<c->aux_grid, 256, 0, c->stream>>>(pts, c->n, labels, C, c->s3, c->sse128);
        else km::sse_kernel<3><<<c->aux_grid, 256, 0, c->stream>>>(pts, c->n, labels, C, c->s3, c->sse128);
        int rc = ls.end();
        if (rc) return rc;
    }
    LaunchScope ls(c, 2);
    km::sse_fix_reduce_kernel<<<1, km::kReduceThreads, 0, c->stream>>>(c->sse128, c->aux_grid, c->s3,
                                                                        reinterpret_cast<km::SseFix*>(c->scal));
    return ls.end();
}

// The same for the high-dimensional variant (warp per point, hd_sse_kernel).
template <int D>
int hd_final_sse(km_ctx* c, const float* P, const int32_t* labels)
{
    const int64_t n = c->n;
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (n + 7) / 8));
    {
        LaunchScope ls(c, 2);
        km::hd::hd_sse_bound_kernel<D><<<1, 1024, 0, c->stream>>>(c->hq, c->hctr, c->cwork, c->k,
                                                                  c->n_global ? c->n_global : n, c->s3);
        int rc = ls.end();
        if (rc) return rc;
    }
    {
        LaunchScope ls(c, 2);
        km::hd::hd_sse_kernel<D><<<wgrid, 256, 0, c->stream>>>(P, n, labels, c->cwork, c->s3, c->sse128);
        int rc = ls.end();
        if (rc) return rc;
    }
    LaunchScope ls(c, 2);
    km::sse_fix_reduce_kernel<<<1, km::kReduceThreads, 0, c->stream>>>(c->sse128, wgrid, c->s3,
                                                                        reinterpret_cast<km::SseFix*>(c->scal));
    return ls.end();
}

template <typename T>
int dmalloc(T** p, size_t count)
{
    if (cudaMalloc((void**)p, count * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return KM_E_NOMEM;
    }
    return KM_OK;
}

int ensure_traces(km_ctx* c, int max_iter)
{
    if (max_iter <= c->trace_cap) return KM_OK;
    cudaFree(c->sse_trace);
    cudaFree(c->chg_trace);
    cudaFree(c->drift_trace);
    c->sse_trace = nullptr; c->chg_trace = nullptr; c->drift_trace = nullptr;
    c->trace_cap = 0;
    int cap = std::max(max_iter, 64);
    if (dmalloc(&c->sse_trace, cap) || dmalloc(&c->chg_trace, cap) || dmalloc(&c->drift_trace, cap))
        return KM_E_NOMEM;
    c->trace_cap = cap;
    return KM_OK;
}

// ------------------------------------------------------------------ high-dimensional path
typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

TmapEncodeFn tmap_encoder()
{
    static TmapEncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (TmapEncodeFn)p;
        else
            cudaGetLastError();
    }
    return fn;
}

// [rows][d] row-major, boxes of 32 columns x box_rows rows: FP32 with 128-B swizzle (128-B
// rows) or BF16 with 64-B swizzle (64-B rows) -- the UMMA K-major canonical layouts; rows past
// the end read as zero.
int make_tmap(CUtensorMap* m, const void* base, int64_t rows, int d, int box_rows, bool bf16)
{
    TmapEncodeFn enc = tmap_encoder();
    if (!enc) return KM_E_UNSUPPORTED;
    const int es_bytes = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * es_bytes};
    cuuint32_t box[2] = {(cuuint32_t)km::hd::kBK, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? KM_OK : KM_E_CUDA;
}

bool hd_dim(int d) { return d == 32 || d == 64 || d == 128 || d == 256; }
// any other 4 <= d <= 256 runs the high-d variant on points zero-padded to the next native width:
// padded coordinates add exact zeros to every product, sum and distance (oracle pin
// test_high_d_zero_padding_is_exact), so labels, centroids and SSE are those of the unpadded problem
int hd_pad_dim(int d) { return d < 4 || d > 256 ? 0 : d <= 32 ? 32 : d <= 64 ? 64 : d <= 128 ? 128 : 256; }

// caller rows [rows][du] -> zero-padded context rows [rows][d] (pad columns of dst must be zero)
int pad_rows(km_ctx* c, float* dst, const float* src, int64_t rows, bool src_host)
{
    KM_CUDA(cudaMemcpy2DAsync(dst, (size_t)c->d * 4, src, (size_t)c->du * 4, (size_t)c->du * 4, (size_t)rows,
                              src_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
    return KM_OK;
}
int unpad_rows(km_ctx* c, float* dst, const float* src, int64_t rows, bool dst_host)
{
    KM_CUDA(cudaMemcpy2DAsync(dst, (size_t)c->du * 4, src, (size_t)c->d * 4, (size_t)c->du * 4, (size_t)rows,
                              dst_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream));
    return KM_OK;
}
// padded copy of the caller's points in stage_pts (allocated and zeroed once)
int pad_points(km_ctx* c, const float* points, bool host)
{
    if (!c->stage_pts) {
        if (dmalloc(&c->stage_pts, (size_t)c->n * c->d)) return KM_E_NOMEM;
        KM_CUDA(cudaMemsetAsync(c->stage_pts, 0, sizeof(float) * c->n * c->d, c->stream));
    }
    return pad_rows(c, c->stage_pts, points, c->n, host);
}
int pad_centroids(km_ctx* c, float* dst, const float* src, bool host)
{
    KM_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * c->k * c->d, c->stream));
    return pad_rows(c, dst, src, c->k, host);
}

template <int D>
int hd_configure(km_ctx* c)
{
    using G = km::hd::GemmCfg<D>;
    c->hd_kpad = (c->k + km::hd::kBN - 1) / km::hd::kBN * km::hd::kBN;
    c->hd_ntk = c->hd_kpad / km::hd::kBN;
    c->hd_mt = (int)((c->n + km::hd::kBM - 1) / km::hd::kBM);
    c->hd_grid = std::max(1, std::min(c->num_sms, c->hd_mt));
    c->hd_bbox_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 4, (c->n + (256 / D) - 1) / (256 / D)));
    KM_CUDA(cudaFuncSetAttribute(km::hd::hd_gemm_kernel<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem));
    KM_CUDA(cudaFuncSetAttribute(km::hd::hd_gemm_kernel<D, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem));
    const int64_t n = c->n;
    if (dmalloc(&c->hpc, (size_t)n * D) || dmalloc(&c->hpn, (size_t)n) || dmalloc(&c->hcc, (size_t)c->hd_kpad * D) ||
        dmalloc(&c->hh, (size_t)c->hd_kpad) || dmalloc(&c->htopv, (size_t)2 * n * (km::hd::kTopMax / 4)) || dmalloc(&c->htopj, (size_t)2 * n * (km::hd::kTopMax / 4)) ||
        dmalloc(&c->hlab, (size_t)n) || dmalloc(&c->hfb, (size_t)n) || dmalloc(&c->hq, (size_t)3 * D) ||
        dmalloc(&c->hctr, (size_t)D) || dmalloc(&c->hst, 1) || dmalloc(&c->hpbh, (size_t)n * D) ||
        dmalloc(&c->hpbl, (size_t)n * D) || dmalloc(&c->hcbh, (size_t)c->hd_kpad * D) ||
        dmalloc(&c->hcbl, (size_t)c->hd_kpad * D) || dmalloc(&c->hacc_q, (size_t)c->k) || dmalloc(&c->hpq2, (size_t)n) ||
        dmalloc(&c->hfb_b, (size_t)2 * km::hd::kFbCap * km::hd::kFbSlices) ||
        dmalloc(&c->hfb_j, (size_t)km::hd::kFbCap * km::hd::kFbSlices))
        return KM_E_NOMEM;
    int rc = make_tmap(&c->tmA, c->hpc, n, D, km::hd::kBM, false);
    if (!rc) rc = make_tmap(&c->tmAh, c->hpbh, n, D, km::hd::kBM, true);
    if (!rc) rc = make_tmap(&c->tmAl, c->hpbl, n, D, km::hd::kBM, true);
    if (!rc) rc = make_tmap(&c->tmB, c->hcc, c->k, D, km::hd::kBN, false);
    if (!rc) rc = make_tmap(&c->tmBh, c->hcbh, c->k, D, km::hd::kBN, true);
    if (!rc) rc = make_tmap(&c->tmBl, c->hcbl, c->k, D, km::hd::kBN, true);
    return rc;
}

// The whole loop on the device (iterations early-exit through ctl->done):
//   once: box -> fixed point + centring origin -> centred copy p' and ||p'||
//   per iteration: prep (c', h, max ||c'||) -> tensor-core scores + top 4 -> certification
//                  (+ FP64 fallback) with label changes moving the running sums -> refine -> tail
// Per call: state reset, box, fixed point, centring origin (+ the centred hi/lo copy of the
// points when center is set).
template <int D>
int hd_setup(km_ctx* c, const float* P, bool center)
{
    const int64_t n = c->n;
    double* qo = c->hq;
    double* qs = c->hq + D;
    double* qi = c->hq + 2 * D;
    KM_CUDA(cudaMemsetAsync(c->hst, 0, sizeof(km::hd::HdState), c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * (size_t)c->k * D, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * (size_t)c->k, c->stream));
    KM_CUDA(cudaMemsetAsync(c->hacc_q, 0, sizeof(unsigned long long) * (size_t)c->k, c->stream));
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (n + 7) / 8));
    {
        LaunchScope ls(c, 2);
        km::hd::hd_bbox_kernel<<<c->hd_bbox_grid, 256, 0, c->stream>>>(P, n, D, c->bbox_part);
        int rc = ls.end();
        if (rc) return rc;
    }
    {
        LaunchScope ls(c, 2);
        km::hd::hd_quant_kernel<<<1, 1024, 0, c->stream>>>(c->bbox_part, c->hd_bbox_grid, n, D, qo, qs, qi, c->hctr,
                                                          c->hst);
        int rc = ls.end();
        if (rc) return rc;
    }
    if (center) {
        LaunchScope ls(c, 2);
        km::hd::hd_center_kernel<D><<<wgrid, 256, 0, c->stream>>>(P, n, c->hctr, c->hpc, c->hpbh, c->hpbl, c->hpn,
                                                                      qo, c->hst, c->hpq2);
        int rc = ls.end();
        if (rc) return rc;
    }
    return KM_OK;
}

// One assignment against C (prep, scores, certification, fallback).  acc = the running sums
// (km_run) or null (km_assign: labels and SSE_t only).
template <int D>
int hd_assign_step(km_ctx* c, const float* P, const float* C, int32_t* labels, int first, bool acc, int dbg,
                   const km::Ctl* ctl)
{
    const int64_t n = c->n;
    const int k = c->k;
    double* qo = c->hq;
    double* qs = c->hq + D;
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (n + 7) / 8));
    const int pgrid = std::max(1, std::min(c->num_sms * 8, (c->hd_kpad + 7) / 8));
    unsigned long long* as = acc ? c->acc_sum : nullptr;
    unsigned int* ac = acc ? c->acc_cnt : nullptr;
    unsigned long long* aq = acc ? c->hacc_q : nullptr;
    {
        LaunchScope ls(c, 2);
        km::hd::hd_prep_kernel<D><<<pgrid, 256, 0, c->stream>>>(C, k, c->hd_kpad, c->hctr, c->hcc, c->hcbh, c->hcbl, c->hh,
                                                                c->hst, ctl);
        int rc = ls.end();
        if (rc) return rc;
    }
    // scores kept per point and column half: 4, or 8 when k is large (bands get more crowded)
    const bool top8 = c->k > 2048;
    {
        LaunchScope ls(c, 0);
#define KM_HD_GEMM_ARGS                                                                                        \
    c->tmA, c->tmAh, c->tmAl, c->tmB, c->tmBh, c->tmBl, c->hh, n, c->hd_ntk, c->hd_mt, c->htopv, c->htopj, c->hpn, \
        c->hst, ctl
        if (top8)
            km::hd::hd_gemm_kernel<D, 8><<<c->hd_grid, km::hd::kGemmThreads, km::hd::GemmCfg<D>::kSmem, c->stream>>>(
                KM_HD_GEMM_ARGS);
        else
            km::hd::hd_gemm_kernel<D, 4><<<c->hd_grid, km::hd::kGemmThreads, km::hd::GemmCfg<D>::kSmem, c->stream>>>(
                KM_HD_GEMM_ARGS);
#undef KM_HD_GEMM_ARGS
        int rc = ls.end();
        if (rc) return rc;
    }
    if (!(dbg & 1)) {
        LaunchScope ls(c, 2);
#define KM_HD_CERT_ARGS                                                                                         \
    P, C, n, c->htopv, c->htopj, c->hpn, c->hst, labels, (dbg & 4) ? 2 : first, qo, qs, as, ac, aq, c->hpq2, c->hfb, ctl
        if (top8) km::hd::hd_certify_kernel<D, 8><<<wgrid, 256, 0, c->stream>>>(KM_HD_CERT_ARGS);
        else km::hd::hd_certify_kernel<D, 4><<<wgrid, 256, 0, c->stream>>>(KM_HD_CERT_ARGS);
#undef KM_HD_CERT_ARGS
        int rc = ls.end();
        if (rc) return rc;
    }
    if (!(dbg & 2)) {
        // undecided points: the first kFbCap through the sliced pair, the rest all-k per CTA
        const int fbf = (dbg & 8) ? 3 : first;
        double* sb1 = c->hfb_b;
        double* sb2 = c->hfb_b + (size_t)km::hd::kFbCap * km::hd::kFbSlices;
        {
            LaunchScope ls(c, 2);
            km::hd::hd_fb_slice_kernel<D><<<c->num_sms * 2, 256, 0, c->stream>>>(P, C, k, c->hfb, c->hst, sb1, sb2,
                                                                               c->hfb_j, ctl);
            int rc = ls.end();
            if (rc) return rc;
        }
        {
            LaunchScope ls(c, 2);
            km::hd::hd_fb_settle_kernel<D><<<c->num_sms, 256, 0, c->stream>>>(
                P, C, k, c->hfb, c->hst, labels, fbf, qo, qs, as, ac, aq, c->hpq2, sb1, sb2, c->hfb_j, ctl);
            int rc = ls.end();
            if (rc) return rc;
        }
        LaunchScope ls(c, 2);
        km::hd::hd_fallback_kernel<D><<<c->num_sms * 4, 256, 0, c->stream>>>(
            P, C, k, c->hfb, c->hst, labels, (dbg & 8) ? 3 : first, qo, qs, as, ac, aq, c->hpq2, ctl);
        int rc = ls.end();
        if (rc) return rc;
    }
    return KM_OK;
}

template <int D>
int hd_run_loop(km_ctx* c, const float* P, int max_iter, float tol)
{
    const int64_t n = c->n;
    const int k = c->k;
    double* qo = c->hq;
    double* qi = c->hq + 2 * D;
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (n + 7) / 8));
    int rc = hd_setup<D>(c, P, true);
    if (rc) return rc;
    // (km_debug_set KM_DBG_HD) 1: no certify, 2: no fallback, 4: every point to the fallback,
    // 8: no sequential tie path
    const int dbg = c->hd_dbg;
    const int fgrid = std::max(1, std::min(c->num_sms * 8, (k + 7) / 8));
    for (int t = 0; t < max_iter; ++t) {
        const int first = t == 0;
        rc = hd_assign_step<D>(c, P, c->cwork, c->hlab, first, true, dbg, c->ctl);
        if (rc) return rc;
        {
            LaunchScope ls(c, 1);
            km::hd::hd_finalize_kernel<D><<<fgrid, 256, 0, c->stream>>>(c->cwork, k, c->acc_sum, c->acc_cnt, qo, qi,
                                                                        nullptr, c->hst, c->ctl, c->hacc_q);
            int rc = ls.end();
            if (rc) return rc;
        }
        {
            LaunchScope ls(c, 1);
            km::hd::hd_tail_kernel<<<1, 1, 0, c->stream>>>(c->hst, c->sse_trace, c->chg_trace, c->drift_trace, c->ctl,
                                                           tol);
            int rc = ls.end();
            if (rc) return rc;
        }
    }
    return hd_final_sse<D>(c, P, c->hlab);
}

template <int D>
int hd_assign_call(km_ctx* c, const float* P, const float* C, int32_t* labels, double* sse_dev)
{
    int rc = hd_setup<D>(c, P, true);
    if (!rc) rc = hd_assign_step<D>(c, P, C, labels, 1, false, 0, nullptr);
    if (rc || !sse_dev) return rc;
    LaunchScope ls(c, 2);
    km::hd::hd_scalars_kernel<<<1, 1, 0, c->stream>>>(c->hst, sse_dev, nullptr);
    return ls.end();
}

template <int D>
int hd_update_call(km_ctx* c, const float* P, const int32_t* labels, const float* Cold, float* Cnew, int32_t* counts,
                   double* md_dev)
{
    int rc = hd_setup<D>(c, P, false);
    if (rc) return rc;
    const int64_t n = c->n;
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (n + 7) / 8));
    {
        LaunchScope ls(c, 1);
        km::hd::hd_accumulate_kernel<D><<<wgrid, 256, 0, c->stream>>>(P, n, labels, c->hq, c->hq + D, c->acc_sum,
                                                                      c->acc_cnt);
        rc = ls.end();
        if (rc) return rc;
    }
    if (Cnew != Cold)
        KM_CUDA(cudaMemcpyAsync(Cnew, Cold, sizeof(float) * (size_t)c->k * D, cudaMemcpyDeviceToDevice, c->stream));
    {
        LaunchScope ls(c, 1);
        const int fgrid = std::max(1, std::min(c->num_sms * 8, (c->k + 7) / 8));
        km::hd::hd_finalize_kernel<D><<<fgrid, 256, 0, c->stream>>>(Cnew, c->k, c->acc_sum, c->acc_cnt, c->hq,
                                                                    c->hq + 2 * D, counts, c->hst, nullptr);
        rc = ls.end();
        if (rc) return rc;
    }
    if (!md_dev) return KM_OK;
    LaunchScope ls(c, 2);
    km::hd::hd_scalars_kernel<<<1, 1, 0, c->stream>>>(c->hst, nullptr, md_dev);
    return ls.end();
}

// ---- data parallel (km_dp_*) for the high-dimensional variant -----------------------------
// The fixed point and the centring origin of the GLOBAL problem, from the all-reduced box:
// the formulas of hd_quant_kernel (same operations, same order), so any sharding is
// bit-identical to one context holding the union of the shards.
void hd_host_quant(const float* lo_hi, int d, int64_t n, double* q3, float* ctr, double* sse2)
{
    int nb = 0;
    while (nb < 63 && (n >> nb) != 0) ++nb;
    double t = 0.0;
    for (int m = 0; m < d; ++m) {
        const float lo = lo_hi[m], hi = lo_hi[d + m];
        const double ext = (double)hi - (double)lo;
        int e = 0;
        if (ext > 0.0) frexp(ext, &e);
        const int sc = ext > 0.0 ? 61 - nb - e : 0;
        q3[m] = (double)lo;
        q3[d + m] = ldexp(1.0, sc);
        q3[2 * d + m] = ldexp(1.0, -sc);
        ctr[m] = (float)(0.5 * ((double)lo + (double)hi));
        t += ext * ext;
    }
    const double tot = (double)n * t * (1.0 + 0x1p-20);
    int e = 0;
    if (tot > 0.0) frexp(tot, &e);
    const int s2 = tot > 0.0 ? 62 - e : 0;
    sse2[0] = ldexp(1.0, s2);
    sse2[1] = ldexp(1.0, -s2);
}

template <int D>
int hd_dp_bbox(km_ctx* c, const float* P, float* lo_hi)
{
    {
        LaunchScope ls(c, 2);
        km::hd::hd_bbox_kernel<<<c->hd_bbox_grid, 256, 0, c->stream>>>(P, c->n, D, c->bbox_part);
        int rc = ls.end();
        if (rc) return rc;
    }
    std::vector<float> part((size_t)c->hd_bbox_grid * 2 * D);
    KM_CUDA(cudaMemcpyAsync(part.data(), c->bbox_part, part.size() * 4, cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaStreamSynchronize(c->stream));
    for (int m = 0; m < D; ++m) {
        float lo = INFINITY, hi = -INFINITY;
        for (int b = 0; b < c->hd_bbox_grid; ++b) {
            lo = std::min(lo, part[(size_t)b * 2 * D + m]);
            hi = std::max(hi, part[(size_t)b * 2 * D + D + m]);
        }
        lo_hi[m] = lo;
        lo_hi[D + m] = hi;
    }
    return KM_OK;
}

template <int D>
int hd_dp_begin(km_ctx* c, const float* P, const float* init, int ki, const float* lo_hi, int64_t n_global)
{
    std::vector<double> q3(3 * D);
    std::vector<float> ctr(D);
    double sse2[2];
    hd_host_quant(lo_hi, D, n_global, q3.data(), ctr.data(), sse2);
    if (!c->hg_sum && (dmalloc(&c->hg_sum, (size_t)c->k * D) || dmalloc(&c->hg_cnt, (size_t)c->k) ||
                       dmalloc(&c->hg_q, (size_t)c->k)))
        return KM_E_NOMEM;
    KM_CUDA(cudaMemsetAsync(c->hacc_q, 0, sizeof(unsigned long long) * (size_t)c->k, c->stream));
    KM_CUDA(cudaMemsetAsync(c->hst, 0, sizeof(km::hd::HdState), c->stream));
    KM_CUDA(cudaMemcpyAsync(c->hst, sse2, sizeof(sse2), cudaMemcpyHostToDevice, c->stream));   // sse_scale, sse_inv
    KM_CUDA(cudaMemcpyAsync(c->hq, q3.data(), q3.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    KM_CUDA(cudaMemcpyAsync(c->hctr, ctr.data(), ctr.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * (size_t)c->k * D, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * (size_t)c->k, c->stream));
    KM_CUDA(cudaMemcpyAsync(c->cwork, init, (size_t)c->k * D * 4, ki ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            c->stream));
    KM_CUDA(cudaMemsetAsync(c->ctl, 0, sizeof(km::Ctl), c->stream));
    const int wgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 8, (c->n + 7) / 8));
    LaunchScope ls(c, 2);
    km::hd::hd_center_kernel<D><<<wgrid, 256, 0, c->stream>>>(P, c->n, c->hctr, c->hpc, c->hpbh, c->hpbl, c->hpn,
                                                              c->hq, c->hst, c->hpq2);
    return ls.end();
}

template <int D>
int hd_dp_step(km_ctx* c, uint64_t* partial)
{
    int rc = hd_assign_step<D>(c, c->dp_points, c->cwork, c->hlab, c->dp_iter == 0, true, 0, c->ctl);
    if (rc) return rc;
    LaunchScope ls(c, 1);
    km::hd::hd_export_kernel<<<1, 1024, 0, c->stream>>>(c->acc_sum, c->acc_cnt, c->hacc_q, c->k * D, c->k, c->hst,
                                                        (unsigned long long*)partial, c->ctl);
    return ls.end();
}

template <int D>
int hd_dp_apply(km_ctx* c, const uint64_t* partial, float tol)
{
    {
        LaunchScope ls(c, 1);
        km::hd::hd_import_kernel<<<1, 1024, 0, c->stream>>>((const unsigned long long*)partial, c->k * D, c->k,
                                                            c->hg_sum, c->hg_cnt, c->hg_q, c->hst, c->ctl);
        int rc = ls.end();
        if (rc) return rc;
    }
    {
        LaunchScope ls(c, 1);
        const int fgrid = std::max(1, std::min(c->num_sms * 8, (c->k + 7) / 8));
        km::hd::hd_finalize_kernel<D><<<fgrid, 256, 0, c->stream>>>(c->cwork, c->k, c->hg_sum, c->hg_cnt, c->hq,
                                                                    c->hq + 2 * D, nullptr, c->hst, c->ctl, c->hg_q);
        int rc = ls.end();
        if (rc) return rc;
    }
    LaunchScope ls(c, 1);
    km::hd::hd_tail_kernel<<<1, 1, 0, c->stream>>>(c->hst, c->sse_trace, c->chg_trace, c->drift_trace, c->ctl, tol);
    return ls.end();
}

template <int D>
int hd_dp_end(km_ctx* c, int32_t* out_labels)
{
    int rc = hd_final_sse<D>(c, c->dp_points, c->hlab);
    if (rc) return rc;
    KM_CUDA(cudaMemcpyAsync(out_labels, c->hlab, (size_t)c->n * 4, cudaMemcpyDeviceToDevice, c->stream));
    return KM_OK;
}

#define KM_HD_DISPATCH(fn, ...)                                  \
    (c->d == 32    ? fn<32>(__VA_ARGS__)                         \
     : c->d == 64  ? fn<64>(__VA_ARGS__)                         \
     : c->d == 128 ? fn<128>(__VA_ARGS__)                        \
                   : fn<256>(__VA_ARGS__))

int hd_run(km_ctx* c, const float* P, int max_iter, float tol)
{
    switch (c->d) {
        case 32: return hd_run_loop<32>(c, P, max_iter, tol);
        case 64: return hd_run_loop<64>(c, P, max_iter, tol);
        case 128: return hd_run_loop<128>(c, P, max_iter, tol);
        case 256: return hd_run_loop<256>(c, P, max_iter, tol);
        default: return KM_E_UNSUPPORTED;
    }
}

// The device work of one km_run_ctx call after the inputs are staged (Alg. 1: index, the loop
// P:L286-301 with its convergence flag, Eq. 1 of the returned pair): a fixed launch sequence
// (converged iterations return at once through ctl.done), hence capturable as one graph.
// Small brute-force problems run as one launch of one CTA (the default scan variants only)
bool small_run(const km_ctx* c)
{
    return c->use_small && c->assign_variant != 0 && c->n <= km::kSmallMaxN && c->k <= km::kSmallMaxK;
}

// The whole device work of a small km_run_ctx call: ONE kernel (it reads the initial centroids,
// writes the outputs, the traces and the host scalars itself).
int run_small(km_ctx* c, const RunIO& io)
{
    km::SmallIO so{};
    so.cin = io.init_dev ? io.init_dev : c->cwork;
    so.cout = c->cwork;
    so.cout2 = c->du ? nullptr : io.outc_dev;
    so.sse_trace = c->sse_trace;
    so.chg_trace = c->chg_trace;
    so.drift_trace = c->drift_trace;
    so.sse_user = io.sse_trace;
    so.chg_user = reinterpret_cast<long long*>(io.chg_trace);
    so.ctl = c->ctl;
    so.sse_out = reinterpret_cast<km::SseFix*>(c->scal);
    so.host_sse = c->dscal ? &c->dscal->sse : nullptr;
    so.host_ctl = c->dscal ? &c->dscal->ctl : nullptr;
    LaunchScope ls(c, 0);
    const size_t sm = c->d == 2 ? km::small_smem<2>(c->k, c->kpad, c->n) : km::small_smem<3>(c->k, c->kpad, c->n);
    if (c->d == 2)
        km::lloyd_small_kernel<2><<<km::kSmallCtas, km::kSmallThreads, sm, c->stream>>>(
            io.P, (int)c->n, c->k, c->kpad, io.L, io.max_iter, io.tol, c->quant, so);
    else
        km::lloyd_small_kernel<3><<<km::kSmallCtas, km::kSmallThreads, sm, c->stream>>>(
            io.P, (int)c->n, c->k, c->kpad, io.L, io.max_iter, io.tol, c->quant, so);
    int rc = ls.end();
    if (rc) return rc;
    if (!c->dscal) {   // (no mapped host record: copy the scalars)
        KM_CUDA(cudaMemcpyAsync(&c->hscal->sse, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        KM_CUDA(cudaMemcpyAsync(&c->hscal->ctl, c->ctl, sizeof(km::Ctl), cudaMemcpyDeviceToHost, c->stream));
    }
    return KM_OK;
}

int run_body(km_ctx* c, const float* P, int32_t* L, int max_iter, float tol, int path)
{
    KM_CUDA(cudaMemsetAsync(c->ctl, 0, sizeof(km::Ctl), c->stream));
    // trace entries of iterations a converged run does not execute read as NaN / -1 (all bits set)
    KM_CUDA(cudaMemsetAsync(c->sse_trace, 0xff, sizeof(double) * max_iter, c->stream));
    KM_CUDA(cudaMemsetAsync(c->chg_trace, 0xff, sizeof(long long) * max_iter, c->stream));
    KM_CUDA(cudaMemsetAsync(c->drift_trace, 0xff, sizeof(double) * max_iter, c->stream));
    int rc;
    if (path == 2) {
        rc = hd_run(c, P, max_iter, tol);
        if (rc) return rc;
        KM_CUDA(cudaMemcpyAsync(L, c->hlab, (size_t)c->n * 4, cudaMemcpyDeviceToDevice, c->stream));
        return KM_OK;
    }
    rc = launch_quant(c, P);
    if (rc) return rc;
    if (path == 1) {
        rc = prepare_tiles(c, P);
        if (rc) return rc;
        for (int t = 0; t < max_iter; ++t) {
            rc = launch_assign_tiles(c, c->cwork, t == 0);
            if (rc) return rc;
            rc = launch_finalize(c, c->cwork, c->cwork, nullptr, nullptr, true, c->ctl, tol, 1, true);
            if (rc) return rc;
        }
        return launch_scatter_labels(c, L);   // + Eq. 1 of the returned pair
    }
    // the incremental update's running sums start at zero
    KM_CUDA(cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * c->k * c->d, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * c->k, c->stream));
    if (path == 3) {   // KM_MODE_BOUNDS: running sums and deltas start at zero
        KM_CUDA(cudaMemsetAsync(c->bscan, 0, 8 * sizeof(unsigned long long), c->stream));
        KM_CUDA(cudaMemsetAsync(c->bsum, 0, sizeof(unsigned long long) * 5 * c->k * c->d, c->stream));
        KM_CUDA(cudaMemsetAsync(c->bcnt, 0, sizeof(unsigned int) * 5 * c->k, c->stream));
        for (int t = 0; t < max_iter; ++t) {
            rc = c->d == 2 ? launch_bounds<2>(c, P, L, t, tol) : launch_bounds<3>(c, P, L, t, tol);
            if (rc) return rc;
        }
        rc = c->d == 2 ? launch_bounds_tail<2>(c, max_iter, tol) : launch_bounds_tail<3>(c, max_iter, tol);
        if (rc) return rc;
        return launch_final_sse(c, P, L, c->cwork);
    }
    for (int t = 0; t < max_iter; ++t) {
        if (c->assign_variant == 0) {   // (debug variant: separate refine launch)
            rc = launch_assign_d(c, P, c->cwork, L, t == 0, true, c->ctl);
            if (!rc) rc = launch_finalize(c, c->cwork, c->cwork, nullptr, nullptr, true, c->ctl, tol, c->assign_grid);
        } else {
            rc = launch_assign_d(c, P, c->cwork, L, t == 0, true, c->ctl, tol, true);   // refine fused into the last CTA
        }
        if (rc) return rc;
    }
    // (zero again between calls: km_update and the data-parallel path start from zero sums)
    KM_CUDA(cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * c->k * c->d, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * c->k, c->stream));
    return launch_final_sse(c, P, L, c->cwork);
}

void drop_graph(km_ctx* c)
{
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->graph) cudaGraphDestroy(c->graph);
    c->gexec = nullptr;
    c->graph = nullptr;
    c->gkey.path = -1;
}

// The device work of one km_run_ctx call: the device-side input copy, run_body, the device-side
// output copies and the scalars (Eq. 1, iterations) into the context's pinned host record.
int run_device(km_ctx* c, const RunIO& io)
{
    if (io.path == 0 && small_run(c)) return run_small(c, io);
    const size_t cb = (size_t)c->k * (c->du ? c->du : c->d) * 4;
    int rc = KM_OK;
    if (io.init_dev) {
        if (c->du) rc = pad_centroids(c, c->cwork, io.init_dev, false);
        else KM_CUDA(cudaMemcpyAsync(c->cwork, io.init_dev, cb, cudaMemcpyDeviceToDevice, c->stream));
        if (rc) return rc;
    }
    rc = run_body(c, io.P, io.L, io.max_iter, io.tol, io.path);
    if (rc) return rc;
    if (io.outc_dev) {
        if (c->du) rc = unpad_rows(c, io.outc_dev, c->cwork, c->k, false);
        else KM_CUDA(cudaMemcpyAsync(io.outc_dev, c->cwork, cb, cudaMemcpyDeviceToDevice, c->stream));
        if (rc) return rc;
    }
    if (io.sse_trace)
        KM_CUDA(cudaMemcpyAsync(io.sse_trace, c->sse_trace, sizeof(double) * io.max_iter, cudaMemcpyDeviceToDevice,
                                c->stream));
    if (io.chg_trace)
        KM_CUDA(cudaMemcpyAsync(io.chg_trace, c->chg_trace, sizeof(int64_t) * io.max_iter, cudaMemcpyDeviceToDevice,
                                c->stream));
    KM_CUDA(cudaMemcpyAsync(&c->hscal->sse, c->scal, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaMemcpyAsync(&c->hscal->ctl, c->ctl, sizeof(km::Ctl), cudaMemcpyDeviceToHost, c->stream));
    return KM_OK;
}

// A6: capture run_device once per argument set (RunIO) on the private stream, then replay it on
// the context stream: one graph launch per call instead of 5-9 host launches per iteration and
// the copies around them.  Kernels read every per-run value from device memory (ctl, quant,
// centroids), so a replay is the same computation as the eager sequence.
int run_graph(km_ctx* c, const RunIO& io)
{
    if (!c->gexec || memcmp(&io, &c->gkey, sizeof(io)) != 0) {
        drop_graph(c);
        if (!c->cap) KM_CUDA(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
        KM_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
        cudaStream_t user = c->stream;
        c->stream = c->cap;
        const int64_t l0 = c->launches;
        int rc = run_device(c, io);
        c->stream = user;
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->cap, &g);
        c->graph_launches = c->launches - l0;
        c->launches = l0;
        if (rc || e != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return rc ? rc : cuda_fail(e);
        }
        c->graph = g;
        e = cudaGraphInstantiate(&c->gexec, g, 0);
        if (e != cudaSuccess) {
            drop_graph(c);
            return cuda_fail(e);
        }
        c->gkey = io;
    }
    KM_CUDA(cudaGraphLaunch(c->gexec, c->stream));
    c->launches += c->graph_launches;
    return KM_OK;
}

template <int D>
int configure_kernels(km_ctx* c)
{
    c->kpad = km::assign_kpad(c->assign_variant, c->k);
    size_t smem = assign_smem_bytes(D, c->kpad);
    int nb = 0;
    if (c->assign_variant == 0) {
        KM_CUDA(cudaFuncSetAttribute(km::assign_simple_kernel<D, 2, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        KM_CUDA(cudaFuncSetAttribute(km::assign_simple_kernel<D, 2, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, km::assign_simple_kernel<D, 2, true>,
                                                              km::kAssignThreads, smem));
    } else {
        // privatised update when the k(2d+1) shared words fit beside the centroids
        c->priv_smem = km::priv_bytes<D>(c->k) <= kPrivMax ? km::priv_bytes<D>(c->k) : 0;
        int rc = km::configure_assign_fast<D>(c->assign_variant, smem, c->priv_smem, &nb);
        if (rc) return cuda_fail((cudaError_t)rc);
    }
    c->acc_priv = km::priv_bytes<D>(c->k) <= kAccPrivMax ? km::priv_bytes<D>(c->k) : 0;
    if (c->n <= km::kSmallMaxN && c->k <= km::kSmallMaxK)
        KM_CUDA(cudaFuncSetAttribute(km::lloyd_small_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)km::small_smem<D>(c->k, c->kpad, c->n)));
    if (c->acc_priv)
        KM_CUDA(cudaFuncSetAttribute(km::accumulate_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)c->acc_priv));
    if (nb < 1) return KM_E_UNSUPPORTED;
    nb = std::min(nb, 4);
    {
        const size_t bsm = smem + km::priv_bytes<D>(c->k) + km::bounds_smem_extra<D>(c->k);
        int nbb = 0;
        if (bsm <= 227 * 1024) {
            KM_CUDA(cudaFuncSetAttribute(km::bounds_scan_kernel<D, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bsm));
            KM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbb, km::bounds_scan_kernel<D, 4, 2>,
                                                                  km::kAssignThreads, bsm));
        }
        const int64_t chunks = (c->n + km::kBoundsChunk - 1) / km::kBoundsChunk;
        c->bounds_grid = nbb < 1 ? 0 : (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * std::min(nbb, 4), chunks));
    }
    int64_t tile = (int64_t)km::kAssignThreads * km::assign_points_per_thread(c->assign_variant);
    int64_t tiles = (c->n + tile - 1) / tile;
    c->assign_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * nb, tiles));
    c->aux_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 4, (c->n + 255) / 256));
    return KM_OK;
}

}  // namespace

extern "C" {

int32_t km_max_k(int32_t d)
{
    if (hd_dim(d) || hd_pad_dim(d)) return 1 << 20;   // high-dimensional variant: centroids stream from HBM/L2
    if (d != 2 && d != 3) return 0;
    // all centroids staged as SoA float32 in <= 227 KB of shared memory (minus 4 KB reserve)
    return (int32_t)(((227 * 1024 - 4096) / (4 * d)) & ~3);
}

int km_create(km_ctx** out, int64_t n, int32_t d, int32_t k, void* cuda_stream)
{
    if (!out) return KM_E_INVALID;
    *out = nullptr;
    if (n < 1 || k < 1 || (int64_t)k > n || n > (int64_t)INT32_MAX) return KM_E_INVALID;
    if (d != 2 && d != 3 && !hd_dim(d) && !hd_pad_dim(d)) return KM_E_UNSUPPORTED;
    if (k > km_max_k(d)) return KM_E_UNSUPPORTED;
    km_ctx* c = new (std::nothrow) km_ctx();
    if (!c) return KM_E_NOMEM;
    if (d != 2 && d != 3 && !hd_dim(d)) {
        c->du = d;
        d = hd_pad_dim(d);
    }
    c->n = n; c->d = d; c->k = k; c->kpad = round_up4(k);
    c->stream = (cudaStream_t)cuda_stream;
    int rc = KM_OK;
    if (cudaGetDevice(&c->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError());
        delete c;
        return rc;
    }
    if (dmalloc(&c->acc_sum, (size_t)k * d) || dmalloc(&c->acc_cnt, (size_t)k) || dmalloc(&c->sse_part, kMaxParts) ||
        dmalloc(&c->chg_part, kMaxParts) || dmalloc(&c->bbox_part, (size_t)kMaxParts * 2 * d) ||
        dmalloc(&c->quant, 1) || dmalloc(&c->ctl, 1) || dmalloc(&c->scal, 8) || dmalloc(&c->s3, 1) || dmalloc(&c->tick, 1) || dmalloc(&c->sse128, 2 * kMaxParts) || dmalloc(&c->cwork, (size_t)k * d) ||
        ensure_traces(c, 64)) {
        km_destroy(c);
        return KM_E_NOMEM;
    }
    if (cudaHostAlloc((void**)&c->hscal, sizeof(HostScalars), cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        c->hscal = nullptr;
        km_destroy(c);
        return KM_E_NOMEM;
    }
    if (cudaHostGetDevicePointer((void**)&c->dscal, c->hscal, 0) != cudaSuccess) {
        cudaGetLastError();
        c->dscal = nullptr;
    }
    if (cudaMemsetAsync(c->tick, 0, sizeof(unsigned int), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * k * d, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * k, c->stream) != cudaSuccess) {
        rc = cuda_fail(cudaGetLastError());
        km_destroy(c);
        return rc;
    }
    if (hd_dim(d)) {
        c->hd = true;
        c->aux_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * 4, (n + 255) / 256));
        rc = d == 32 ? hd_configure<32>(c) : d == 64 ? hd_configure<64>(c) : d == 128 ? hd_configure<128>(c)
                                                                                      : hd_configure<256>(c);
    } else {
        // chunked bookkeeping (a lazy running minimum per 32 centroids) for long scans: config 4
        // brute force 2.37 -> 2.30 ms per launch; per-group bookkeeping below (config 2: 37 vs 52 us)
        c->assign_variant = k >= 512 ? 2 : 1;
        rc = d == 2 ? configure_kernels<2>(c) : configure_kernels<3>(c);
    }
    if (rc) {
        km_destroy(c);
        return rc;
    }
    *out = c;
    return KM_OK;
}

int km_destroy(km_ctx* c)
{
    if (!c) return KM_OK;
    if (c->stream) cudaStreamSynchronize(c->stream);
    else cudaDeviceSynchronize();
    cudaFree(c->acc_sum); cudaFree(c->acc_cnt); cudaFree(c->sse_part); cudaFree(c->chg_part);
    cudaFree(c->bbox_part); cudaFree(c->quant); cudaFree(c->ctl); cudaFree(c->scal); cudaFree(c->s3); cudaFree(c->tick); cudaFree(c->sse128); cudaFree(c->cwork);
    cudaFree(c->sse_trace); cudaFree(c->chg_trace); cudaFree(c->drift_trace);
    cudaFree(c->stage_pts); cudaFree(c->stage_lab); cudaFree(c->pad_c);
    free_tiles(c);
    cudaFree(c->lbv); cudaFree(c->cbuf1); cudaFree(c->bscan); cudaFree(c->bsum); cudaFree(c->bcnt);
    cudaFree(c->dp_lab);
    cudaFree(c->hpc); cudaFree(c->hpbh); cudaFree(c->hpbl); cudaFree(c->hcbh); cudaFree(c->hcbl); cudaFree(c->hpn); cudaFree(c->hg_sum); cudaFree(c->hg_cnt); cudaFree(c->hacc_q); cudaFree(c->hpq2); cudaFree(c->hg_q); cudaFree(c->hfb_b); cudaFree(c->hfb_j); cudaFree(c->hcc); cudaFree(c->hh); cudaFree(c->htopv); cudaFree(c->htopj);
    cudaFree(c->hlab); cudaFree(c->hfb); cudaFree(c->hq); cudaFree(c->hctr); cudaFree(c->hst);
    drop_graph(c);
    if (c->hscal) cudaFreeHost(c->hscal);
    if (c->cap) cudaStreamDestroy(c->cap);
    if (c->aux) { cudaStreamSynchronize(c->aux); cudaStreamDestroy(c->aux); }
    if (c->ev_c) cudaEventDestroy(c->ev_c);
    if (c->ev_f) cudaEventDestroy(c->ev_f);
    for (auto& t : c->pending) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
    for (auto e : c->pool) cudaEventDestroy(e);
    delete c;
    return KM_OK;
}

int km_set_mode(km_ctx* c, int mode)
{
    if (!c || mode < KM_MODE_AUTO || mode > KM_MODE_BOUNDS) return KM_E_INVALID;
    if (mode == KM_MODE_TILES && !tiles_supported(c)) return KM_E_UNSUPPORTED;
    if (mode == KM_MODE_BOUNDS && !bounds_supported(c)) return KM_E_UNSUPPORTED;
    c->mode = mode;
    return KM_OK;
}

int km_read_stats(km_ctx* c, int64_t* out4)
{
    if (!c || !out4) return KM_E_INVALID;
    KM_CUDA(cudaStreamSynchronize(c->stream));
    if (c->last_run_bounds && c->bscan) {   // points that failed their bound test were scanned
        unsigned long long ns = 0;
        KM_CUDA(cudaMemcpy(&ns, c->bscan, sizeof(ns), cudaMemcpyDeviceToHost));
        out4[0] = (int64_t)ns * c->k;
        out4[1] = (int64_t)ns;
        out4[2] = 0;
        out4[3] = 0;
        return 0;
    }
    if (!c->last_run_tiles || !c->stats) {
        out4[0] = c->last_iters * (int64_t)c->n * c->k;
        out4[1] = c->last_iters * (int64_t)c->n;
        out4[2] = 0;
        out4[3] = 0;
        return 0;
    }
    unsigned long long h[4];
    KM_CUDA(cudaMemcpy(h, c->stats, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; ++i) out4[i] = (int64_t)h[i];
    return 1;
}

int km_set_stream(km_ctx* c, void* s)
{
    if (!c) return KM_E_INVALID;
    c->stream = (cudaStream_t)s;
    return KM_OK;
}

int km_assign(km_ctx* c, const float* points, const float* centroids, int32_t* labels, double* sse_dev)
{
    if (!c || !points || !centroids || !labels) return KM_E_INVALID;
    if (c->hd) {
        if (((uintptr_t)points | (uintptr_t)centroids | (uintptr_t)labels | (uintptr_t)sse_dev) & 3) return KM_E_INVALID;
        if (pointer_kind(c, points) != 1 || pointer_kind(c, centroids) != 1 || pointer_kind(c, labels) != 1 ||
            (sse_dev && pointer_kind(c, sse_dev) != 1))
            return KM_E_UNSUPPORTED;
        if (c->du) {
            int rc = pad_points(c, points, false);
            if (!rc) rc = pad_centroids(c, c->cwork, centroids, false);
            if (rc) return rc;
            points = c->stage_pts;
            centroids = c->cwork;
        }
        switch (c->d) {
            case 32: return hd_assign_call<32>(c, points, centroids, labels, sse_dev);
            case 64: return hd_assign_call<64>(c, points, centroids, labels, sse_dev);
            case 128: return hd_assign_call<128>(c, points, centroids, labels, sse_dev);
            default: return hd_assign_call<256>(c, points, centroids, labels, sse_dev);
        }
    }
    if (((uintptr_t)points | (uintptr_t)centroids | (uintptr_t)labels | (uintptr_t)sse_dev) & 3) return KM_E_INVALID;
    size_t pb = (size_t)c->n * c->d * 4, cb = (size_t)c->k * c->d * 4, lb = (size_t)c->n * 4;
    if (ranges_overlap(labels, lb, points, pb) || ranges_overlap(labels, lb, centroids, cb) ||
        ranges_overlap(sse_dev, 8, points, pb) || ranges_overlap(sse_dev, 8, labels, lb))
        return KM_E_INVALID;
    if (pointer_kind(c, points) != 1 || pointer_kind(c, centroids) != 1 || pointer_kind(c, labels) != 1 ||
        (sse_dev && pointer_kind(c, sse_dev) != 1))
        return KM_E_UNSUPPORTED;
    int rc = launch_assign_d(c, points, centroids, labels, 1, false, nullptr);
    if (rc) return rc;
    if (sse_dev) {
        LaunchScope ls(c, 2);
        km::reduce_parts_kernel<<<1, km::kReduceThreads, 0, c->stream>>>(c->sse_part, nullptr, c->assign_grid,
                                                                          sse_dev, nullptr);
        return ls.end();
    }
    return KM_OK;
}

int km_update(km_ctx* c, const float* points, const int32_t* labels, const float* old_centroids,
              float* new_centroids, int32_t* counts, double* max_drift_dev)
{
    if (!c || !points || !labels || !old_centroids || !new_centroids) return KM_E_INVALID;
    if (((uintptr_t)points | (uintptr_t)labels | (uintptr_t)old_centroids | (uintptr_t)new_centroids |
         (uintptr_t)counts | (uintptr_t)max_drift_dev) & 3)
        return KM_E_INVALID;
    const int du = c->du ? c->du : c->d;
    size_t pb = (size_t)c->n * du * 4, cb = (size_t)c->k * du * 4, lb = (size_t)c->n * 4;
    if (ranges_overlap(new_centroids, cb, points, pb) || ranges_overlap(new_centroids, cb, labels, lb) ||
        ranges_overlap(counts, (size_t)c->k * 4, points, pb) || ranges_overlap(counts, (size_t)c->k * 4, new_centroids, cb))
        return KM_E_INVALID;
    if (new_centroids != old_centroids && ranges_overlap(new_centroids, cb, old_centroids, cb)) return KM_E_INVALID;
    if (pointer_kind(c, points) != 1 || pointer_kind(c, labels) != 1 || pointer_kind(c, old_centroids) != 1 ||
        pointer_kind(c, new_centroids) != 1 || (counts && pointer_kind(c, counts) != 1) ||
        (max_drift_dev && pointer_kind(c, max_drift_dev) != 1))
        return KM_E_UNSUPPORTED;
    if (c->hd && c->du) {
        if (!c->pad_c && dmalloc(&c->pad_c, (size_t)c->k * c->d)) return KM_E_NOMEM;
        int rc = pad_points(c, points, false);
        if (!rc) rc = pad_centroids(c, c->cwork, old_centroids, false);
        if (rc) return rc;
        switch (c->d) {
            case 32: rc = hd_update_call<32>(c, c->stage_pts, labels, c->cwork, c->pad_c, counts, max_drift_dev); break;
            case 64: rc = hd_update_call<64>(c, c->stage_pts, labels, c->cwork, c->pad_c, counts, max_drift_dev); break;
            case 128: rc = hd_update_call<128>(c, c->stage_pts, labels, c->cwork, c->pad_c, counts, max_drift_dev); break;
            default: rc = hd_update_call<256>(c, c->stage_pts, labels, c->cwork, c->pad_c, counts, max_drift_dev); break;
        }
        if (rc) return rc;
        return unpad_rows(c, new_centroids, c->pad_c, c->k, false);
    }
    if (c->hd) {
        switch (c->d) {
            case 32: return hd_update_call<32>(c, points, labels, old_centroids, new_centroids, counts, max_drift_dev);
            case 64: return hd_update_call<64>(c, points, labels, old_centroids, new_centroids, counts, max_drift_dev);
            case 128: return hd_update_call<128>(c, points, labels, old_centroids, new_centroids, counts, max_drift_dev);
            default: return hd_update_call<256>(c, points, labels, old_centroids, new_centroids, counts, max_drift_dev);
        }
    }
    int rc = launch_quant(c, points);
    if (rc) return rc;
    {
        LaunchScope ls(c, 1);
        const size_t ap = c->acc_priv;
        if (c->d == 2 && ap)
            km::accumulate_kernel<2, true><<<c->aux_grid, 256, ap, c->stream>>>(points, c->n, labels, c->acc_sum,
                                                                                c->acc_cnt, c->quant, c->k);
        else if (c->d == 2)
            km::accumulate_kernel<2, false><<<c->aux_grid, 256, 0, c->stream>>>(points, c->n, labels, c->acc_sum,
                                                                                c->acc_cnt, c->quant, c->k);
        else if (ap)
            km::accumulate_kernel<3, true><<<c->aux_grid, 256, ap, c->stream>>>(points, c->n, labels, c->acc_sum,
                                                                                c->acc_cnt, c->quant, c->k);
        else
            km::accumulate_kernel<3, false><<<c->aux_grid, 256, 0, c->stream>>>(points, c->n, labels, c->acc_sum,
                                                                                c->acc_cnt, c->quant, c->k);
        rc = ls.end();
        if (rc) return rc;
    }
    return launch_finalize(c, old_centroids, new_centroids, counts, max_drift_dev, false, nullptr, -1.0f, 0);
}

int km_run_ctx(km_ctx* c, const float* points, const float* init_centroids, int32_t max_iter, float tol,
               float* out_centroids, int32_t* out_labels, double* out_sse, double* sse_trace_dev,
               int64_t* changed_trace_dev)
{
    if (!c || !points || !init_centroids || !out_centroids || !out_labels || max_iter < 1) return KM_E_INVALID;
    if (((uintptr_t)points | (uintptr_t)init_centroids | (uintptr_t)out_centroids | (uintptr_t)out_labels) & 3)
        return KM_E_INVALID;
    if (tol != tol) return KM_E_INVALID;
    const int du = c->du ? c->du : c->d;
    size_t pb = (size_t)c->n * du * 4, cb = (size_t)c->k * du * 4, lb = (size_t)c->n * 4;
    if (ranges_overlap(out_centroids, cb, points, pb) || ranges_overlap(out_centroids, cb, init_centroids, cb) ||
        ranges_overlap(out_labels, lb, points, pb) || ranges_overlap(out_labels, lb, init_centroids, cb) ||
        ranges_overlap(out_labels, lb, out_centroids, cb))
        return KM_E_INVALID;
    int kp = pointer_kind(c, points), ki = pointer_kind(c, init_centroids);
    int kc = pointer_kind(c, out_centroids), kl = pointer_kind(c, out_labels);
    if (kp < 0 || ki < 0 || kc < 0 || kl < 0) return KM_E_UNSUPPORTED;
    if ((sse_trace_dev && pointer_kind(c, sse_trace_dev) != 1) ||
        (changed_trace_dev && pointer_kind(c, changed_trace_dev) != 1))
        return KM_E_UNSUPPORTED;
    int rc = ensure_traces(c, max_iter);
    if (rc) return rc;
    c->n_global = 0;
    c->dp_points = nullptr;

    // inputs: host -> device staging (part of the call, hence of e2e timing)
    const float* P = points;
    if (c->du) {
        rc = pad_points(c, points, kp == 0);
        if (rc) return rc;
        P = c->stage_pts;
    } else if (kp == 0) {
        if (!c->stage_pts && dmalloc(&c->stage_pts, (size_t)c->n * c->d)) return KM_E_NOMEM;
        KM_CUDA(cudaMemcpyAsync(c->stage_pts, points, pb, cudaMemcpyHostToDevice, c->stream));
        P = c->stage_pts;
    }
    int32_t* L = out_labels;
    if (kl == 0) {
        if (!c->stage_lab && dmalloc(&c->stage_lab, (size_t)c->n)) return KM_E_NOMEM;
        L = c->stage_lab;
    }
    // host initial centroids: staged before the (captured) device work
    if (ki == 0) {
        if (c->du) rc = pad_centroids(c, c->cwork, init_centroids, true);
        else KM_CUDA(cudaMemcpyAsync(c->cwork, init_centroids, cb, cudaMemcpyHostToDevice, c->stream));
        if (rc) return rc;
    }
    const int path = run_path(c);
    if (path == 1) {
        if (!tiles_supported(c)) return KM_E_UNSUPPORTED;
        rc = ensure_tiles(c);   // allocations stay outside the captured region
        if (rc) return rc;
    }
    if (path == 3) {
        rc = ensure_bounds(c);
        if (rc) return rc;
    }
    c->last_run_tiles = path == 1;
    c->last_run_bounds = path == 3;
    RunIO io;
    memset(&io, 0, sizeof(io));   // (padding too: the graph cache compares keys with memcmp)
    io.P = P;
    io.L = L;
    io.init_dev = ki ? init_centroids : nullptr;
    io.outc_dev = kc ? out_centroids : nullptr;
    io.sse_trace = sse_trace_dev;
    io.chg_trace = changed_trace_dev;
    io.max_iter = max_iter;
    io.tol = tol;
    io.path = path;
    const bool graph = c->use_graph && !c->timing && max_iter <= kGraphMaxIter;
    rc = graph ? run_graph(c, io) : run_device(c, io);
    if (rc) return rc;

    // host outputs
    if (kc == 0) {
        if (c->du) rc = unpad_rows(c, out_centroids, c->cwork, c->k, true);
        else KM_CUDA(cudaMemcpyAsync(out_centroids, c->cwork, cb, cudaMemcpyDeviceToHost, c->stream));
        if (rc) return rc;
    }
    if (kl == 0) KM_CUDA(cudaMemcpyAsync(out_labels, L, lb, cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaStreamSynchronize(c->stream));
    if (out_sse) *out_sse = c->hscal->sse;
    c->last_iters = c->hscal->ctl.iter;
    return c->hscal->ctl.iter;
}

int km_run(const float* points, int64_t n, int32_t d, int32_t k, const float* init_centroids, int32_t max_iter,
           float tol, float* out_centroids, int32_t* out_labels, double* out_sse)
{
    if (!points || !init_centroids || !out_centroids || !out_labels || max_iter < 1) return KM_E_INVALID;
    km_ctx* c = nullptr;
    int rc = km_create(&c, n, d, k, nullptr);
    if (rc) return rc;
    rc = km_run_ctx(c, points, init_centroids, max_iter, tol, out_centroids, out_labels, out_sse, nullptr, nullptr);
    km_destroy(c);
    return rc;
}

int km_read_traces(km_ctx* c, double* sse, int64_t* changed, double* max_drift, int32_t count)
{
    if (!c || count < 0) return KM_E_INVALID;
    int m = std::min(count, c->last_iters);
    m = std::min(m, c->trace_cap);
    KM_CUDA(cudaStreamSynchronize(c->stream));
    if (m > 0) {
        if (sse) KM_CUDA(cudaMemcpy(sse, c->sse_trace, sizeof(double) * m, cudaMemcpyDeviceToHost));
        if (changed) KM_CUDA(cudaMemcpy(changed, c->chg_trace, sizeof(int64_t) * m, cudaMemcpyDeviceToHost));
        if (max_drift) KM_CUDA(cudaMemcpy(max_drift, c->drift_trace, sizeof(double) * m, cudaMemcpyDeviceToHost));
    }
    return c->last_iters;
}

int km_timing_enable(km_ctx* c, int on)
{
    if (!c) return KM_E_INVALID;
    c->timing = on != 0;
    return KM_OK;
}

int km_timing_read(km_ctx* c, km_timing* out, int reset)
{
    if (!c || !out) return KM_E_INVALID;
    KM_CUDA(cudaStreamSynchronize(c->stream));
    for (auto& t : c->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t.a, t.b);
        c->tot_ms[t.kind] += ms;
        c->tot_launches[t.kind] += 1;
        c->pool.push_back(t.a);
        c->pool.push_back(t.b);
    }
    c->pending.clear();
    out->assign_ms = c->tot_ms[0];
    out->update_ms = c->tot_ms[1];
    out->other_ms = c->tot_ms[2];
    out->assign_launches = c->tot_launches[0];
    out->update_launches = c->tot_launches[1];
    out->other_launches = c->tot_launches[2];
    if (reset) {
        for (int i = 0; i < 3; ++i) { c->tot_ms[i] = 0; c->tot_launches[i] = 0; }
    }
    return KM_OK;
}

int64_t km_launch_count(km_ctx* c, int reset)
{
    if (!c) return KM_E_INVALID;
    int64_t v = c->launches;
    if (reset) c->launches = 0;
    return v;
}

const char* km_strerror(int code)
{
    switch (code) {
        case KM_OK: return "ok";
        case KM_E_INVALID: return "invalid argument";
        case KM_E_UNSUPPORTED: return "unsupported (d not in {2,3}, k too large, or pointer not on the context device)";
        case KM_E_NOMEM: return "device allocation failed";
        case KM_E_CUDA: return "CUDA error (see km_last_cuda_error)";
        case KM_E_STATE: return "context state / shape mismatch";
        default: return "unknown status";
    }
}

int km_last_cuda_error(void) { return t_last_cuda_error; }

// Internal knobs for tests/benchmarks (not part of km.h's stable surface).
int km_debug_set_variant(km_ctx* c, int variant)
{
    if (!c || variant < 0 || variant > km::kNumScanVariants) return KM_E_INVALID;
    if (c->hd) return KM_E_UNSUPPORTED;
    c->assign_variant = variant;
    drop_graph(c);
    return c->d == 2 ? configure_kernels<2>(c) : configure_kernels<3>(c);
}

int km_debug_assign_grid(km_ctx* c) { return c ? c->assign_grid : KM_E_INVALID; }

// The bounds path's counters of the last run: [0] points scanned, [1..5] phase times (ns, summed
// over CTAs; KM_BPROF builds only).  Synchronises.
int km_debug_bounds(km_ctx* c, int64_t* out8)
{
    if (!c || !out8) return KM_E_INVALID;
    if (!c->bscan) return KM_E_STATE;
    KM_CUDA(cudaStreamSynchronize(c->stream));
    KM_CUDA(cudaMemcpy(out8, c->bscan, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    return KM_OK;
}

int km_debug_set(km_ctx* c, int what, int value)
{
    if (!c) return KM_E_INVALID;
    switch (what) {
        case KM_DBG_ST_SHIFT:
            if (value != 0 && (value < 2 || value > 5)) return KM_E_INVALID;
            if (c->tiles_ready) return KM_E_STATE;   // the index shape is fixed at the first tile run
            c->dbg_st_shift = value;
            return KM_OK;
        case KM_DBG_K1T_MINB:
            if (value < 0 || value > (KM_K1T_WARPS < 8 ? 5 : 3)) return KM_E_INVALID;
            if (c->tiles_ready) return KM_E_STATE;
            c->dbg_minb = value;
            return KM_OK;
        case KM_DBG_SHORT_LIST:
            if (value < 0 || value > km::kShortList) return KM_E_INVALID;
            if (c->tiles_ready) return KM_E_STATE;
            c->dbg_short_list = value;
            return KM_OK;
        case KM_DBG_HD:
            if (value < 0 || value > 15) return KM_E_INVALID;
            if (!c->hd) return KM_E_STATE;
            c->hd_dbg = value;
            drop_graph(c);
            return KM_OK;
        case KM_DBG_GRAPH:
            if (value < 0 || value > 1) return KM_E_INVALID;
            c->use_graph = value != 0;
            return KM_OK;
        case KM_DBG_PDL:
            if (value < 0 || value > 1) return KM_E_INVALID;
            c->use_pdl = value != 0;
            drop_graph(c);
            return KM_OK;
        case KM_DBG_SMALL:
            if (value < 0 || value > 1) return KM_E_INVALID;
            c->use_small = value != 0;
            drop_graph(c);
            return KM_OK;
        default: return KM_E_INVALID;
    }
}

// ---------------------------------------------------------------- data-parallel (km.h "DP")
int km_dp_bbox(km_ctx* c, const float* points, float* lo_hi)
{
    if (!c || !points || !lo_hi || ((uintptr_t)points & 3)) return KM_E_INVALID;
    if (pointer_kind(c, points) != 1) return KM_E_UNSUPPORTED;
    if (c->du) {   // padded width: box of the padded copy (pad dimensions are [0, 0]), caller's d returned
        std::vector<float> box(2 * (size_t)c->d);
        int rc = pad_points(c, points, false);
        if (!rc) rc = KM_HD_DISPATCH(hd_dp_bbox, c, c->stage_pts, box.data());
        if (rc) return rc;
        for (int m = 0; m < c->du; ++m) {
            lo_hi[m] = box[m];
            lo_hi[c->du + m] = box[c->d + m];
        }
        return KM_OK;
    }
    if (c->hd) return KM_HD_DISPATCH(hd_dp_bbox, c, points, lo_hi);
    int rc = launch_quant(c, points);   // local bbox into Quant.o / Quant.hi
    if (rc) return rc;
    km::Quant h;
    KM_CUDA(cudaMemcpyAsync(&h, c->quant, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaStreamSynchronize(c->stream));
    for (int m = 0; m < c->d; ++m) {
        lo_hi[m] = (float)h.o[m];
        lo_hi[c->d + m] = h.hi[m];
    }
    return KM_OK;
}

int km_dp_begin(km_ctx* c, const float* points, const float* init_centroids, const float* lo_hi, int64_t n_global,
                int32_t max_iter)
{
    if (!c || !points || !init_centroids || !lo_hi || n_global < c->n || max_iter < 1) return KM_E_INVALID;
    if (((uintptr_t)points | (uintptr_t)init_centroids) & 3) return KM_E_INVALID;
    if (pointer_kind(c, points) != 1) return KM_E_UNSUPPORTED;
    const int ki = pointer_kind(c, init_centroids);
    if (ki < 0) return KM_E_UNSUPPORTED;
    int rc = ensure_traces(c, max_iter);
    if (rc) return rc;
    std::vector<float> box;
    if (c->du) {   // padded width: padded points, centroids and box (pad dimensions [0, 0])
        box.assign(2 * (size_t)c->d, 0.0f);
        for (int m = 0; m < c->du; ++m) {
            box[m] = lo_hi[m];
            box[c->d + m] = lo_hi[c->du + m];
        }
        if (!c->pad_c && dmalloc(&c->pad_c, (size_t)c->k * c->d)) return KM_E_NOMEM;
        rc = pad_points(c, points, false);
        if (!rc) rc = pad_centroids(c, c->pad_c, init_centroids, ki == 0);
        if (rc) return rc;
        points = c->stage_pts;
        init_centroids = c->pad_c;
        lo_hi = box.data();
    }
    c->n_global = n_global;
    if (c->hd) {
        c->last_run_tiles = false;
        rc = KM_HD_DISPATCH(hd_dp_begin, c, points, init_centroids, c->du ? 1 : ki, lo_hi, n_global);
        if (rc) return rc;
        c->dp_points = points;
        c->dp_iter = 0;
        return KM_OK;
    }
    // the quantisation of the GLOBAL problem: same formula as quant_kernel, so sums (and
    // centroids) are bit-identical to a single-GPU run over the union of the shards
    km::Quant h;
    memset(&h, 0, sizeof(h));
    km::make_quant(h, lo_hi, lo_hi + c->d, c->d, n_global);
    KM_CUDA(cudaMemcpyAsync(c->quant, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    KM_CUDA(cudaMemcpyAsync(c->cwork, init_centroids, (size_t)c->k * c->d * 4,
                            ki ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    KM_CUDA(cudaMemsetAsync(c->ctl, 0, sizeof(km::Ctl), c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_sum, 0, sizeof(unsigned long long) * c->k * c->d, c->stream));
    KM_CUDA(cudaMemsetAsync(c->acc_cnt, 0, sizeof(unsigned int) * c->k, c->stream));
    c->dp_points = points;
    c->dp_iter = 0;
    c->last_run_tiles = c->mode == KM_MODE_TILES ||
                        (c->mode == KM_MODE_AUTO && auto_tiles(c));
    c->last_run_bounds = false;
    if (c->last_run_tiles) {
        rc = ensure_tiles(c);
        if (rc) return rc;
        rc = prepare_tiles(c, points);
        if (rc) return rc;
    }
    return KM_OK;
}

int64_t km_dp_partial_len(km_ctx* c)
{
    if (!c) return KM_E_INVALID;
    // low d: sums [k][d], counts [k], changed_t, SSE_t (fixed point); high d: sums [k][d'],
    // counts [k], changed_t, moment sums Q [k] (SSE_t follows from them)
    return (int64_t)c->k * c->d + c->k + 1 + (c->hd ? c->k : 1);
}

int km_dp_step(km_ctx* c, uint64_t* partial_dev)
{
    if (!c || !c->dp_points || !partial_dev) return KM_E_STATE;
    if (c->hd) return KM_HD_DISPATCH(hd_dp_step, c, partial_dev);
    if (!c->last_run_tiles && !c->stage_lab_dp()) return KM_E_NOMEM;
    int rc = c->last_run_tiles ? launch_assign_tiles(c, c->cwork, c->dp_iter == 0)
                               : launch_assign_d(c, c->dp_points, c->cwork, c->stage_lab_dp(), c->dp_iter == 0, true,
                                                 c->ctl);
    if (rc) return rc;
    LaunchScope ls(c, 1);
    const bool t = c->last_run_tiles;
    km::export_partials_kernel<<<1, 1024, 0, c->stream>>>(
        t ? c->tacc_sum : c->acc_sum, t ? c->tacc_cnt : c->acc_cnt, c->k * c->d, c->k, t ? kAccCopies : 1, t ? 0 : 1,
        c->sse_part, t ? c->ttot : nullptr, t ? c->ttot + 1 : c->chg_part, t ? 1 : c->assign_grid,
        (unsigned long long*)partial_dev, c->quant, t ? c->ttot : nullptr, c->ctl);
    return ls.end();
}

int km_dp_apply(km_ctx* c, const uint64_t* partial_dev, float tol, int* done_host)
{
    if (!c || !c->dp_points || !partial_dev) return KM_E_STATE;
    if (c->dp_iter >= c->trace_cap) return KM_E_STATE;
    if (c->hd) {
        int rc = KM_HD_DISPATCH(hd_dp_apply, c, partial_dev, tol);
        if (rc) return rc;
    } else {
        {
            LaunchScope ls(c, 1);
            km::import_partials_kernel<<<1, 1024, 0, c->stream>>>((const unsigned long long*)partial_dev, c->k * c->d,
                                                                   c->k, c->acc_sum, c->acc_cnt, c->sse_part,
                                                                   c->chg_part, c->quant, c->ctl);
            int rc = ls.end();
            if (rc) return rc;
        }
        int rc = launch_finalize(c, c->cwork, c->cwork, nullptr, nullptr, true, c->ctl, tol, 1, c->last_run_tiles,
                                 true);
        if (rc) return rc;
    }
    c->dp_iter++;
    if (done_host) {
        km::Ctl h;
        KM_CUDA(cudaMemcpyAsync(&h, c->ctl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        KM_CUDA(cudaStreamSynchronize(c->stream));
        *done_host = h.done;
    }
    return c->dp_iter;
}

int km_dp_end(km_ctx* c, float* out_centroids, int32_t* out_labels, double* out_sse_local, uint64_t* out_sse_fixed3)
{
    if (!c || !c->dp_points || !out_centroids || !out_labels) return KM_E_STATE;
    if (pointer_kind(c, out_centroids) != 1 || pointer_kind(c, out_labels) != 1) return KM_E_UNSUPPORTED;
    int rc;
    if (c->hd) {
        rc = KM_HD_DISPATCH(hd_dp_end, c, out_labels);
    } else if (c->last_run_tiles) {
        rc = launch_scatter_labels(c, out_labels);   // + Eq. 1 of the shard
    } else {
        rc = launch_final_sse(c, c->dp_points, c->stage_lab_dp(), c->cwork);
        if (!rc) KM_CUDA(cudaMemcpyAsync(out_labels, c->stage_lab_dp(), (size_t)c->n * 4, cudaMemcpyDeviceToDevice,
                                         c->stream));
    }
    if (rc) return rc;
    if (c->du) {
        rc = unpad_rows(c, out_centroids, c->cwork, c->k, false);
        if (rc) return rc;
    } else {
        KM_CUDA(cudaMemcpyAsync(out_centroids, c->cwork, (size_t)c->k * c->d * 4, cudaMemcpyDeviceToDevice,
                                c->stream));
    }
    km::Ctl h;
    km::SseFix f;
    KM_CUDA(cudaMemcpyAsync(&f, c->scal, sizeof(f), cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaMemcpyAsync(&h, c->ctl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KM_CUDA(cudaStreamSynchronize(c->stream));
    if (out_sse_local) *out_sse_local = f.value;
    if (out_sse_fixed3)
        for (int i = 0; i < 3; ++i) out_sse_fixed3[i] = f.limb[i];
    c->dp_sse_inv = f.inv;
    c->last_iters = h.iter;
    c->dp_points = nullptr;
    c->n_global = 0;
    return h.iter;
}

// Eq. 1 over all ranks from the SUM over ranks of their km_dp_end limbs: the same formula as
// sse_fix_reduce_kernel, so the value equals a single context's out_sse bit for bit.
double km_dp_sse(km_ctx* c, const uint64_t* sse_fixed3_sum)
{
    if (!c || !sse_fixed3_sum || c->dp_sse_inv == 0.0) return NAN;
    const km::u128 acc = (km::u128)sse_fixed3_sum[0] + ((km::u128)sse_fixed3_sum[1] << 48) +
                         ((km::u128)sse_fixed3_sum[2] << 96);
    const double hi = (double)(unsigned long long)(acc >> 64), lo = (double)(unsigned long long)acc;
    volatile double t = hi * 0x1p64;   // (no contraction: the device form rounds the same two steps)
    volatile double u = t + lo;
    return u * c->dp_sse_inv;
}

// All 16 internal counters of the last tile run (KM_PROF builds fill [4..9] with cycles).

// All 16 internal counters of the last tile run (KM_PROF builds fill [4..9] with cycles).
int km_hd_stats(km_ctx* c, int64_t* out3)
{
    if (!c || !out3) return KM_E_INVALID;
    if (!c->hd) return KM_E_STATE;
    KM_CUDA(cudaStreamSynchronize(c->stream));
    km::hd::HdState h;
    KM_CUDA(cudaMemcpy(&h, c->hst, sizeof(h), cudaMemcpyDeviceToHost));
    out3[0] = (int64_t)h.n_cert;
    out3[1] = (int64_t)h.n_band;
    out3[2] = (int64_t)h.n_full;
    return KM_OK;
}

int km_debug_stats(km_ctx* c, int64_t* out32)
{
    if (!c || !out32 || !c->stats) return KM_E_INVALID;
    KM_CUDA(cudaStreamSynchronize(c->stream));
    KM_CUDA(cudaMemcpy(out32, c->stats, sizeof(int64_t) * 32, cudaMemcpyDeviceToHost));
    return KM_OK;
}

}  // extern "C"
