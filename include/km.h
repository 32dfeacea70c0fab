/*
 * km.h -- C ABI of libkm: the exact Lloyd step (k-means) for low-dimensional
 * spatial vectors (d = 2 geo-locations, d = 3 point clouds) on one B200.
 *
 * What the library computes (PAPER.md = arXiv 2412.02244 "Dask-means", cited as
 * P:Lnn = line nn of its LaTeX source):
 *   - the k-means objective, Eq. 1: partition D = {p_1..p_n} in R^{n x d}
 *     into k sets minimising sum_j sum_{p in S_j} ||p - c_j||^2, c_j = mean(S_j);
 *   - Lloyd's algorithm: assign every point to its nearest centroid, then
 *     refine each centroid to the mean of its members (Alg. 1 line 12,
 *     c_j <- sv(j)/|S_j|, drift Delta[j] = ||c_j - c'_j||);
 *   - "checks whether any of the centroids move; if so, it continues".
 *   Dask-means' pruning "yield[s] the same results as Lloyd's algorithm",
 *   so the result defined here is plain Lloyd's.  Readings where the paper is
 *   silent:
 *     R1 distance = squared Euclidean; R2 ties -> lowest centroid index;
 *     R3 outputs = (labels of the last assignment, centroids after the last
 *        refine); R4 out_sse = Eq. 1 of that pair;
 *     R5 an empty cluster keeps its centroid (drift 0);
 *     R6 tol < 0 runs exactly max_iter iterations; tol >= 0 stops after an
 *        iteration whose max drift <= tol or (from the 2nd on) in which no label
 *        changed;
 *     R8 centroids are float32 between iterations: the new centroid is the FP64
 *        mean rounded once to float32 (round-to-nearest-even).
 *   Labels are EXACT: label i is the lowest j minimising the FP64 value
 *   sum_m (double(p_im) - double(c_jm))^2 (summed m = 0..d-1, multiply then add),
 *   i.e. bit-identical to the FP64 oracle given the same float32 centroids.
 *
 * Conventions for every entry point:
 *   - Arrays are row-major and contiguous: points [n][d] float32, centroids
 *     [k][d] float32, labels [n] int32, counts [k] int32.  Pointers must be
 *     4-byte aligned.
 *   - The caller owns every buffer.  The library never frees or retains a
 *     caller pointer past the call that received it.  Outputs must not
 *     overlap inputs.
 *   - d must be 2 or 3 (the spatial path), or 32, 64, 128 or 256 (the high-dimensional
 *     variant: the paper's embedded-trajectory check, Table
 *     tab:high_dimension; tensor-core scores + exact FP64 certification;
 *     km_run, km_run_ctx, km_assign, km_update and the km_dp_* calls).  Any other
 *     4 <= d <= 256 runs the same variant on a zero-padded copy (next width of 32, 64,
 *     128, 256; padded coordinates add exact zeros, so results are those of the
 *     unpadded problem) through every call, the km_dp_* ones included (lo_hi and
 *     centroids in the caller's d; the opaque partial in the padded width, see
 *     km_dp_partial_len).  d = 1 or d > 256: KM_E_UNSUPPORTED
 *     (no CPU fallback).
 *     1 <= k <= n, k <= km_max_k(d) (d = 2, 3: all k staged in shared memory).
 *   - Inputs must be finite; |coordinates| < 1e18 is assumed so squared FP32
 *     distances are finite (larger values stay correct but take the slow path).
 *   - Status codes: KM_OK, or a negative KM_E_*; nothing is launched when
 *     validation fails.  Asynchronous device faults surface as KM_E_CUDA from the
 *     next synchronising call; km_last_cuda_error() gives the cudaError_t.
 *   - A km_ctx is not thread-safe; distinct contexts are independent.  Work is
 *     stream-ordered on the context's stream.
 */
#ifndef KM_H
#define KM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct km_ctx km_ctx;

enum {
    KM_OK = 0,
    KM_E_INVALID = -1,      /* bad argument: n<1, n>2^31-1, k<1, k>n, max_iter<1, NULL, misaligned, overlap */
    KM_E_UNSUPPORTED = -2,  /* d < 2 or d > 256; k > km_max_k(d); pointer not on the context's device */
    KM_E_NOMEM = -3,        /* workspace allocation failed */
    KM_E_CUDA = -4,         /* CUDA launch / runtime error (see km_last_cuda_error) */
    KM_E_STATE = -5         /* context / shape mismatch */
};

/* Create a context for problems of shape (n, d, k) on the current CUDA device.
 * 1 <= n <= 2^31 - 1 (the index sorts and scatters with 32-bit positions; KM_E_INVALID
 * otherwise).  cuda_stream: a cudaStream_t (NULL = legacy default stream).  Allocates the
 * workspace (accumulators k*(d+1) words, per-CTA partials, traces); no
 * allocation happens later except host-staging buffers on the first km_run_ctx
 * call that passes host pointers.  *out is set to NULL on failure. */
int km_create(km_ctx **out, int64_t n, int32_t d, int32_t k, void *cuda_stream);

/* Free the workspace.  NULL is a no-op.  Use after destroy is undefined. */
int km_destroy(km_ctx *ctx);

/* Change the stream later work is ordered on (NULL = legacy default). */
int km_set_stream(km_ctx *ctx, void *cuda_stream);

/* Largest k supported for dimension d (shared-memory-resident centroids); 0 if d unsupported. */
int32_t km_max_k(int32_t d);

/* Assignment strategy of km_run_ctx / km_run (results are identical in every mode):
 *   KM_MODE_BRUTE: every point scans all k centroids (Lloyd's n x k distances).
 *   KM_MODE_TILES: the paper's index-based assignment (Alg. 1 Assign) on the GPU.
 *     Once per call (Alg. 1 line 1, "Create Ball-tree on D") the points are Morton-sorted
 *     into tiles of 128 points -- ball nodes with pivot, radius, moments and exact
 *     fixed-point sums -- grouped in a flat tree (8 tiles per level-1 node in 3-D; 16, or 32
 *     when k >= 4096, in 2-D; 16 children per node above).  Per iteration:
 *       - inter bound cb[j] = min_{l != j} ||c_j - c_l|| (Eq. 3); a tile whose
 *         points all carried label a keeps it if ||o - c_a|| + r < cb[a]/2 (Eq. 5), a point
 *         keeps a(i) if ||p - c_a(i)|| < cb[a(i)]/2 (Eq. 4) -- with FP margins that make
 *         the tests conservative;
 *       - every tree node keeps the centroids that can be nearest to one of its points,
 *         pruned from its parent's list (bounds inherited from the parent, Eq. 7-8); a tile
 *         left with one candidate is assigned in batch (Eq. 6), otherwise its points scan
 *         the candidates (FP32 + FP64 certification, as in BRUTE);
 *       - the sums sv(j) change only when a tile or point moves, in exact
 *         integers, so they equal the from-scratch sums bit for bit.
 *     Needs k <= 16384 (KM_E_UNSUPPORTED otherwise).
 *   KM_MODE_BOUNDS: BRUTE with per-point Hamerly bounds: every point keeps a lower bound lb
 *     of its distance to every centroid but its own (the second-best FP32 distance of its last
 *     scan, rounded down); per iteration lb shrinks by the largest centroid drift and
 *     the point keeps its label without a scan when the exact distance to its centroid
 *     (rounded up) is below max(lb, s_a), s_a = half the distance from c_a to its nearest
 *     other centroid (the inter bound of Eq. 4; computed when k <= 256).  One
 *     launch per iteration; n <= 2^31 - 1.  Uses 4n bytes of device memory for the bounds.
 *   KM_MODE_AUTO (default): TILES when supported, n >= 16384 and n*k >= 3e8 (below that
 *     the brute-force scan, one launch per iteration, is faster); else the one-cluster
 *     brute-force run for n <= 65536 and k <= 1024; else BOUNDS when k <= 256; else BRUTE.
 * km_assign / km_update are always brute force (no index). */
enum { KM_MODE_AUTO = 0, KM_MODE_BRUTE = 1, KM_MODE_TILES = 2, KM_MODE_BOUNDS = 3 };
int km_set_mode(km_ctx *ctx, int mode);

/* Work counters of the last km_run_ctx, copied to HOST out4[4] (synchronises):
 *   [0] point-centroid distances evaluated by the scans, [1] points scanned individually,
 *   [2] tiles assigned in batch (Eq. 6), [3] tiles that reached the assignment kernel
 *   (not settled by Eq. 5).  Returns 1 if the last run used tiles, 0 for brute force
 *   (counters derived: n*k*iterations, n*iterations, 0, 0). */
int km_read_stats(km_ctx *ctx, int64_t *out4);

/* Diagnostics (tests, benchmarks, tuning; not needed to use the library).
 * km_debug_stats: all 32 internal counters of the last tile run to HOST out32[32]
 *   ([0..3] as km_read_stats, [10] summed parent-list lengths, [12] tiles settled by Eq. 5,
 *   [13] tiles settled by Eq. 4 in the fused kernel, [22] points settled by Eq. 4 in the
 *   split kernels, [29] tiles pruned with their two sub-balls, other slots: cycle counters
 *   of profiling builds).  Synchronises.
 * km_debug_set_variant: brute-force scan kernel variant (0 simple, 1.. packed FP32x2).
 * km_debug_assign_grid: grid size of the brute-force scan kernel.
 * km_debug_set: per-context overrides for tests and tuning (results never change; 0 restores
 *   the default).  The library reads no environment variables.
 *     KM_DBG_ST_SHIFT (2..5): tiles per level-1 node = 2^value (default 8 in 3-D; 16, or 32
 *       for k >= 4096, in 2-D); KM_DBG_K1T_MINB (1..5): register budget of the tile
 *       assignment kernel (CTAs of 4 warps per SM it targets; default 4 = 128 registers).  Both: KM_E_STATE once the context has run the tile path.
 *     KM_DBG_SHORT_LIST (1..64): level-1 candidate lists up to this length get their tiles' lists
 *       in the prune kernel, longer ones one warp per tile (default 12 below 16 Ki tiles, 32 below 32 Ki, else 64);
 *       KM_E_STATE once the context has run the tile path.
 *     KM_DBG_HD (high-d contexts only; bit mask): 1 no certification kernel, 2 no fallback
 *       kernels, 4 every point through the FP64 fallback, 8 fallback without the sequential
 *       tie path.  Values 1, 2, 8 are for fault-injection tests and break exactness.
 *     KM_DBG_GRAPH (0 / 1): km_run_ctx without / with the CUDA graph (default 1).
 *     KM_DBG_SMALL (0 / 1): small brute-force runs without / with the one-cluster kernel (default 1).
 *     KM_DBG_PDL (0 / 1): without / with programmatic dependent launches between consecutive
 *       iterations' kernels (default 1).
 *   KM_E_INVALID for an unknown key or value. */
enum { KM_DBG_ST_SHIFT = 1, KM_DBG_K1T_MINB = 2, KM_DBG_HD = 3, KM_DBG_GRAPH = 4, KM_DBG_SMALL = 5, KM_DBG_PDL = 6,
       KM_DBG_SHORT_LIST = 7 };
int km_debug_stats(km_ctx *ctx, int64_t *out32);
int km_debug_set_variant(km_ctx *ctx, int variant);
int km_debug_assign_grid(km_ctx *ctx);
int km_debug_set(km_ctx *ctx, int what, int value);
/* KM_MODE_BOUNDS counters of the last run: [0] points scanned; [1..5] phase times in ns summed
 * over CTAs (refine, s_a pass, bound test, queued scan, flush; -DKM_BPROF builds only). */
int km_debug_bounds(km_ctx *ctx, int64_t *out8);

/* High-dimensional variant: how the assignments of the last run were decided, summed over its
 * iterations, to HOST out3[3]: [0] certified from the tensor-core top two (gap > 2E),
 * [1] decided in FP64 among the in-band top-4 candidates (top-8 when k > 2048), [2] FP64 scan over all k.
 * KM_E_STATE for a d = 2 / 3 context.  Synchronises. */
int km_hd_stats(km_ctx *ctx, int64_t *out3);

/* One assignment step (Alg. 1 Assign, without the index).
 *   points [n][d], centroids [k][d]: DEVICE, read-only.
 *   labels [n]: DEVICE, written: labels[i] = lowest j minimising the FP64 distance.
 *   sse_dev: DEVICE double, nullable: written with sum_i min_j D_ij (FP64 sum).
 * Asynchronous on the context stream. */
int km_assign(km_ctx *ctx, const float *points, const float *centroids,
              int32_t *labels, double *sse_dev);

/* One refine step (Alg. 1 line 12):
 *   new_centroids[j] = RN_f32(mean of points with labels == j), or
 *   old_centroids[j] if there are none (R5).
 *   points [n][d], labels [n], old_centroids [k][d]: DEVICE, read-only; labels in [0,k).
 *   new_centroids [k][d]: DEVICE, written (may equal old_centroids for in-place).
 *   counts [k]: DEVICE int32, nullable: |S_j|.
 *   max_drift_dev: DEVICE double, nullable: max_j ||new_j - old_j|| (FP64).
 * Sums are exact 64-bit fixed point (order-independent, bit-reproducible).
 * Asynchronous on the context stream. */
int km_update(km_ctx *ctx, const float *points, const int32_t *labels,
              const float *old_centroids, float *new_centroids, int32_t *counts,
              double *max_drift_dev);

/* The whole loop on a reusable context (no allocation after the first call).
 *   points [n][d], init_centroids [k][d]: HOST or DEVICE (detected per pointer; managed
 *     memory is treated as device memory and must be accessible from the context's device).
 *   out_centroids [k][d], out_labels [n]: HOST or DEVICE, written (R3).
 *   out_sse: HOST double, nullable: Eq. 1 of (out_labels, out_centroids) (R4): every point's
 *     FP64 distance rounded to a multiple of 2^-s3 (n * bound * 2^s3 < 2^126, relative error
 *     ~1e-30 of the bound) and summed as a 128-bit integer, so the value does not depend on
 *     the work order, the path (tiles / brute force) or the sharding.
 *   sse_trace_dev [max_iter] double, changed_trace_dev [max_iter] int64:
 *     DEVICE, nullable: SSE_t = sum_i min_j D(p_i, c_t,j) and the number of
 *     labels that changed in iteration t (t = 0 counts n).  All max_iter entries are
 *     written: those of iterations a converged run (tol >= 0) did not execute are NaN
 *     (SSE) and -1 (changed).
 *   tol: < 0 -> exactly max_iter iterations; >= 0 -> stop per R6.
 * Centroids: the exact fixed-point mean (sums in 64-bit integers at the scale 2^s_m of
 * each coordinate, s_m set by n and the bounding box) rounded once to float32.  It equals
 * the FP64 mean of the oracle within 2^-(s_m+1) absolute (plus the final rounding), which
 * is below a float32 ulp for centroids of magnitude comparable to the box extent; a
 * centroid very near 0 inside a wide box can differ from the FP64 mean by a few ulps.
 * Execution: for max_iter <= 128 the device work of the call (index build, iterations,
 * final SSE) is captured once as a CUDA graph and replayed while points, labels, max_iter,
 * tol and the mode are unchanged (km_debug_set(KM_DBG_GRAPH, 0) launches eagerly; timing
 * mode always does).  Results are identical either way.
 * Synchronous: returns the number of iterations executed (>= 1) after the
 * context stream has drained, or a negative KM_E_* code. */
int km_run_ctx(km_ctx *ctx, const float *points, const float *init_centroids,
               int32_t max_iter, float tol, float *out_centroids, int32_t *out_labels,
               double *out_sse, double *sse_trace_dev, int64_t *changed_trace_dev);

/* Stateless form with exactly the north-star parameter list: creates a
 * context on the legacy default stream, runs km_run_ctx, destroys it.
 * Pointers as in km_run_ctx (host or device).  Returns iterations or KM_E_*. */
int km_run(const float *points, int64_t n, int32_t d, int32_t k,
           const float *init_centroids, int32_t max_iter, float tol,
           float *out_centroids, int32_t *out_labels, double *out_sse);

/* ---- Data-parallel Lloyd over shards (one context per rank / GPU) -------------------
 * The points are split into shards; every rank holds all k centroids.  Per iteration each
 * rank assigns its shard and exports ONE vector of partials (fixed-point sums, counts,
 * changed_t and SSE_t, all 64-bit integers); the CALLER sums it over the ranks (one
 * all-reduce, e.g. NCCL); every rank then applies the identical refine.  Integer sums are
 * order-independent, so any sharding gives labels and centroids bit-identical to one GPU
 * holding the union, and the final Eq. 1 (km_dp_end limbs summed -> km_dp_sse) equals a
 * single context's out_sse bit for bit.  (The paper names distribution as future work,
 * P:L886.)
 * Sequence: km_dp_bbox -> (all-reduce MIN of lo, MAX of hi; SUM of n) -> km_dp_begin ->
 *   repeat { km_dp_step -> all-reduce SUM of the partial -> km_dp_apply } -> km_dp_end ->
 *   all-reduce SUM of the 3 limbs -> km_dp_sse.
 * points/labels are this rank's shard (DEVICE, n = the context's n); all async on the
 * context stream unless stated. */

/* Local bounding box of the shard: HOST lo_hi[2d] = {min_0..min_{d-1}, max_0..max_{d-1}}.
 * Synchronous. */
int km_dp_bbox(km_ctx *ctx, const float *points, float *lo_hi);

/* Start a run: lo_hi = GLOBAL bounding box, n_global = total points over all ranks (sets
 * the shared fixed-point scales), init_centroids [k][d] HOST or DEVICE (same on all ranks),
 * max_iter = capacity of the traces.  Builds the tile index of the shard in TILES mode. */
int km_dp_begin(km_ctx *ctx, const float *points, const float *init_centroids, const float *lo_hi,
                int64_t n_global, int32_t max_iter);

/* Length (uint64 elements) of this context's partial: k*d + k + 2 (sums [k][d], counts [k],
 * changed_t, SSE_t at the global scale 2^s2), or k*d' + 2k + 1 for the high-dimensional
 * variant (sums over the padded width d', counts, changed_t, moment sums Q [k] from which
 * SSE_t follows).  KM_E_INVALID for a NULL context. */
int64_t km_dp_partial_len(km_ctx *ctx);

/* One local assignment + accumulation against the current centroids; writes DEVICE
 * partial_dev[km_dp_partial_len(ctx)] (uint64, layout above). */
int km_dp_step(km_ctx *ctx, uint64_t *partial_dev);

/* Refine from the all-reduced partial (Alg. 1 line 12; R5, R6, R8).  done_host (nullable;
 * synchronises when given) receives the convergence flag.  Returns the number of
 * iterations applied so far. */
int km_dp_apply(km_ctx *ctx, const uint64_t *partial_dev, float tol, int *done_host);

/* Finish: DEVICE out_centroids [k][d], DEVICE out_labels [n] of the shard; HOST
 * out_sse_local (nullable) = Eq. 1 over the shard; HOST out_sse_fixed3[3] (nullable) = the
 * same as a 128-bit fixed-point integer in 48-bit limbs (sum them over the ranks, then
 * km_dp_sse).  Synchronous; returns the iterations executed. */
int km_dp_end(km_ctx *ctx, float *out_centroids, int32_t *out_labels, double *out_sse_local,
              uint64_t *out_sse_fixed3);

/* Eq. 1 over all ranks from the limb-wise SUM of every rank's km_dp_end limbs (host only;
 * NaN before a km_dp_end).  Bit-identical to km_run_ctx's out_sse on the union. */
double km_dp_sse(km_ctx *ctx, const uint64_t *sse_fixed3_sum);

/* Per-iteration traces of the last km_run_ctx on this context, copied to HOST
 * arrays of length >= count (nullable each): SSE_t, changed_t, max drift_t.
 * Synchronises the context stream.  Returns the number of iterations recorded. */
int km_read_traces(km_ctx *ctx, double *sse, int64_t *changed, double *max_drift, int32_t count);

/* Device timing of the library's own kernels (CUDA events recorded on the
 * context stream around every launch while enabled). */
typedef struct km_timing {
    double assign_ms;         /* total device time of assignment kernels (high-d variant: the
                                 tensor-core score kernel only; its certification is "other") */
    double update_ms;         /* refine/finalize kernels */
    double other_ms;          /* bbox, final SSE, reductions */
    int64_t assign_launches;
    int64_t update_launches;
    int64_t other_launches;
} km_timing;
int km_timing_enable(km_ctx *ctx, int on);
/* Synchronises the context stream; reset != 0 clears the totals. */
int km_timing_read(km_ctx *ctx, km_timing *out, int reset);

/* Number of kernels this context has launched since creation (or the last reset). */
int64_t km_launch_count(km_ctx *ctx, int reset);

const char *km_strerror(int code);
int km_last_cuda_error(void);   /* cudaError_t of the last KM_E_CUDA on this thread */

#ifdef __cplusplus
}
#endif
#endif /* KM_H */
