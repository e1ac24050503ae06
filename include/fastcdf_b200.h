/*
 * fastcdf_b200.h — C-ABI of the B200-native generalized-ECDF / Laplacian-KDE hot path.
 *
 * The reference (`fastcdf`, arXiv 2005.03246, /root/reference/pkg/src/fastcdf) is a pure
 * Python/numba package with no FFI of its own.  Each entry point below is the native body of
 * one public reference function; the Python package `paper_2005_03246_b200` binds them with
 * ctypes and keeps the reference's Python signatures on top.
 *
 * Conventions (all entry points):
 *   - Array arguments named x, w, knots, out, lattice, ... are DEVICE pointers (cudaMalloc'd or
 *     torch CUDA storage).  Small per-dimension parameter arrays (m, delta, dims, h, centre) are
 *     HOST pointers of length d.
 *   - x is row-major (n, d) fp64, exactly the reference's `Sample.points` layout (core.py:49-74).
 *   - w == NULL means unit weights y == 1 (core.py:270-271).  Unit-weight grid paths accumulate
 *     in int32 lattices (exact; n < 2^31) and are bit-exact with the reference.
 *   - Grids are rectilinear: knots = the d knot vectors concatenated (dim 0 first), m[k] knots in
 *     dim k, each strictly increasing (core.py:77-141).  Output grid order is lexicographic with
 *     the last dimension fastest (core.py:137-141).
 *   - delta[k] = +1 selects "<=" and -1 selects "<" (core.py:144-172).
 *   - Every call only enqueues work on `stream` (a cudaStream_t; NULL = legacy default stream).
 *     Calls documented as "syncs" read a device scalar back and block on the stream.  The
 *     read-back goes through a 4 KB mapped pinned host buffer (allocated once per host thread)
 *     written by a one-warp kernel, never through a copy engine, so it does not queue behind
 *     bulk transfers the caller has in flight on other streams.
 *   - Workspace protocol (CUB style): call with ws == NULL to receive the byte count in
 *     *ws_bytes; then call again with a device buffer of at least that size.  The library never
 *     allocates device memory itself and keeps no state between calls (reentrant).
 *   - Return value: FCG_OK or an error code; fcg_last_error() gives a thread-local message.
 *     No C++ exception crosses this boundary.
 */
#ifndef FASTCDF_B200_H
#define FASTCDF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCG_ABI_VERSION 1
#define FCG_MAX_DIM 8

/* status codes */
#define FCG_OK 0
#define FCG_EINVAL 22      /* bad argument (maps to ParameterError / ShapeError host-side) */
#define FCG_EUNSUPPORTED 95 /* shape outside what the kernels implement (e.g. d > FCG_MAX_DIM) */
#define FCG_ERANGE 34      /* exponential overflow guard (maps to OverflowGuardError host-side) */
#define FCG_ECUDA 100      /* a CUDA launch or copy failed */
#define FCG_EWORKSPACE 101 /* ws too small */

/* lattice element kinds */
#define FCG_LAT_I32 0      /* exact unit-weight counts */
#define FCG_LAT_F64 1      /* weighted sums */

int fcg_abi_version(void);
const char *fcg_last_error(void);
/* Number of SMs of the current device (for host-side sizing / reporting). */
int fcg_device_sm_count(void);

/* Launch profiler (the B200 stand-in for the reference's runtime_seconds metadata,
 * fastsum.py:79,89-92): when enabled, every kernel launch of this library is bracketed by CUDA
 * events recorded on its own stream.  fcg_profile_report() synchronises those events and
 * writes "name count total_ms launches\n" lines (one per kernel label) into buf, then clears
 * the records.  Returns the number of bytes written (truncated to cap-1), or -1 on error.
 * fcg_profile_launches() returns the number of launches recorded since the last report. */
int fcg_profile_enable(int on);
int fcg_profile_report(char *buf, size_t cap);
int64_t fcg_profile_launches(void);

/* ---------------------------------------------------------------------------------------
 * Grid path (Algorithm 1, lexicographic sweep)
 * ------------------------------------------------------------------------------------- */

/* Generalized local sums, Eq. (4): lattice[(M_1+1) x ... x (M_d+1)] = per-cell sums of w
 * (or counts when w == NULL) with the delta-dependent bin rule b_k = #knots < x (delta=+1) or
 * #knots <= x (delta=-1).
 * Replaces: histogram.py:191-217 local_sums / local_sums_sorted / local_sums_uniform
 *           (= flat_bin_indices histogram.py:153-174 + scatter_flat histogram.py:177-181). */
int fcg_local_sums(const double *x, int64_t n, int32_t d, const double *w,
                   const double *knots, const int64_t *m, const int32_t *delta,
                   int32_t lat_kind, void *lattice,
                   void *ws, size_t *ws_bytes, void *stream);

/* In-place directional sweep of a dense lattice: inclusive prefix sums along every axis,
 * forward where delta=+1 and suffix (reverse) where delta=-1.
 * Replaces: fastsum.py:60-66 directional_sweep (_cumsum_directional fastsum.py:45-57). */
int fcg_directional_sweep(void *lattice, int32_t lat_kind, int32_t d, const int64_t *dims,
                          const int32_t *delta, void *ws, size_t *ws_bytes, void *stream);

/* Generalized ECDF on the grid, Eq. (3) at every grid node (survival == 0) — replaces
 * fastsum.py:69-92 ecdf_fastsum — or the survival function Eq. (2) (survival == 1, delta is
 * ignored; all comparisons strict ">") — replaces fastsum.py:95-111 esf_fastsum.
 * out: prod(m) values.  out_kind 0: fp64 (count or sum, divided by n when scaled);
 *                       out_kind 1: int64 raw counts (requires w == NULL). */
int fcg_ecdf_grid(const double *x, int64_t n, int32_t d, const double *w,
                  const double *knots, const int64_t *m, const int32_t *delta,
                  int32_t survival, int32_t scaled, int32_t out_kind, void *out,
                  void *ws, size_t *ws_bytes, void *stream);

/* Per-dimension min / max of x: out_minmax[0:d] = min, out_minmax[d:2d] = max (device).
 * Feeds the centring / overflow guard of fastsum.py:114-129 and dnc.py:598-605,656. */
int fcg_minmax(const double *x, int64_t n, int32_t d, double *out_minmax,
               void *ws, size_t *ws_bytes, void *stream);

/* Laplacian KDE on the grid by the 2^d-term CDF decomposition, Eq. (12).
 * h: host (d,) diagonal bandwidth; centre: host (d,) centring point c (the caller computes the
 * reference's hull midrange and overflow guard).  out: prod(m) fp64 densities.
 * Replaces: fastsum.py:204-233 kde_fastsum for family "laplacian"
 *           (_kde_exponential_fastsum fastsum.py:139-169,179-182). */
int fcg_kde_grid_laplacian(const double *x, int64_t n, int32_t d, const double *w,
                           const double *knots, const int64_t *m, const double *h,
                           const double *centre, double *out,
                           void *ws, size_t *ws_bytes, void *stream);

/* matern32-additive KDE on the grid through the same 2^d terms, Eq. (29): per term the d + 1
 * channels w e and w e (x_l - c_l) are binned and swept like the Laplacian term and combined as
 * zfac * (coef * S_0 - sum_l (delta_l / h_l) S_l), coef = 1 + sum_k delta_k (z_k - c_k) / h_k,
 * scaled by 1 / (2^d N prod h (1 + d)).  Arguments as fcg_kde_grid_laplacian.
 * Replaces: fastsum.py:204-233 kde_fastsum for family "matern32-additive"
 *           (_kde_exponential_fastsum fastsum.py:139-181 with additive_matern). */
int fcg_kde_grid_matern32(const double *x, int64_t n, int32_t d, const double *w,
                          const double *knots, const int64_t *m, const double *h,
                          const double *centre, double *out,
                          void *ws, size_t *ws_bytes, void *stream);

/* Multilinear interpolation of grid-aligned values at nq query points (device arrays; knots
 * concatenated per dimension, m host (d,), every m_k >= 2).  Queries are clamped to the knot
 * hull per coordinate; out[t] is bit-identical to the reference.  *clamp_count (host, may be
 * NULL; non-NULL synchronises the stream) receives the number of clamped queries.
 * Replaces: interp.py:24-75 multilinear_interp. */
int fcg_multilinear_interp(const double *knots, const int64_t *m, int32_t d, const double *values,
                           const double *q, int64_t nq, double *out, int64_t *clamp_count,
                           void *ws, size_t *ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU slab decomposition along axis 1 (used by paper_2005_03246_b200.distributed)
 * ------------------------------------------------------------------------------------- */

/* owner[i] = r with bounds[r] <= c < bounds[r+1] where c = b - shift is point i's cell along
 * `axis` (b = #knots_axis < x, or <= x when le), or -1 when no slab holds it.  G <= 64. */
int fcg_axis_owner(const double *x, int64_t n, int32_t d, int32_t axis, const double *knots_axis,
                   int64_t m, int32_t le, int32_t shift, const int64_t *bounds, int32_t G,
                   int32_t *owner, void *stream);

/* Stable partition of the rows of x (and w, may be NULL) by owner (rows with owner -1 are
 * dropped): x_out / w_out hold owner 0's rows, then owner 1's, ...; counts (host, G) per owner.
 * Syncs (the counts size the all-to-all). */
int fcg_partition_rows(const double *x, int64_t n, int32_t d, const double *w,
                       const int32_t *owner, int32_t G, double *x_out, double *w_out,
                       int64_t *counts, void *ws, size_t *ws_bytes, void *stream);

/* out[a][j][b] = (local[a][j][b] + carry[a][b]) / div (div <= 0: no division); kind 0: local and
 * carry are int64 counts, 1: fp64.  The carry plane is the all-gathered axis-1 prefix of the
 * lower slabs (or suffix of the higher slabs). */
int fcg_slab_finish(const void *local, int32_t kind, const void *carry, int64_t A, int64_t J,
                    int64_t B, double div, double *out, void *stream);

/* fcg_kde_grid_laplacian with extras: n_scale is the N of the normalisation (the global N on a
 * slab); u_bound (> 0 when known) bounds sum_k max_i |x_ik - c_k| / h_k and, when <= 600, lets
 * the kernels build each term's weights from per-point exponential factors instead of one exp
 * per point and term (the reference's fastsum.py:114-129 guard bounds the span per dimension);
 * when planes != NULL, slot `code` of planes[code * (M_0 * M_2 * ... * M_{d-1})] receives the
 * slab-boundary plane of S (last axis-1 plane for delta_1 = +1, first for -1) weighted by the
 * term's factors zf_k(i_k) = exp(-delta_k (z_k - c_k) / h_k) of the axes k >= kw, kw =
 * max(2, d - 2); terms that differ only in the signs of those axes may be summed into the slot
 * of the lowest such code (the other slots are then zero).  Linear, so the exchange is a sum. */
/* centre == NULL (auto centre): the kernels take the hull of the data and the knot ends while
 * binning (no separate min/max pass), derive c = (lo + hi) / 2 and u_bound themselves and fail
 * with FCG_ERANGE when some span_k / h_k > 600 (fastsum.py:114-129, core.py:22); this
 * synchronises the stream once, after the binning pass.  u_bound is then ignored. */
int fcg_kde_grid_laplacian_ex(const double *x, int64_t n, int32_t d, const double *w,
                              const double *knots, const int64_t *m, const double *h,
                              const double *centre, double n_scale, double u_bound,
                              double *planes, double *out, void *ws, size_t *ws_bytes,
                              void *stream);

/* out[i] += sum_code prod_{k<kw} zf_code,k(i_k) * C_code[i_0, i_2, ...] / (2^d n_scale prod h):
 * the exchanged carry planes (weighted as fcg_kde_grid_laplacian_ex stores them) folded into a
 * slab's KDE (zfac is linear in S). */
int fcg_kde_carry_fixup(double *out, int32_t d, const int64_t *m, const double *knots,
                        const double *h, const double *centre, const double *planes,
                        double n_scale, void *ws, size_t *ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Ranking (subsystem 1): device LSD radix sort of fp64 keys.
 * keys: device, element i at keys[i*stride].  Outputs (device int32, any may be NULL):
 *   order[p]  = index of the element at sorted position p (stable)
 *   pos[i]    = sorted position of element i
 *   lower[i]  = #keys <  keys[i]      upper[i] = #keys <= keys[i]
 *   dense[i]  = #distinct keys < keys[i]
 * n must be < 2^31.  -0.0 and +0.0 rank equal.  Replaces the np.argsort(kind="stable") calls
 * at histogram.py:131 and dnc.py:517,527,544 and the tie scan of core.py:278-281. */
int fcg_rank_f64(const double *keys, int64_t n, int64_t stride,
                 int32_t *order, int32_t *pos, int32_t *lower, int32_t *upper, int32_t *dense,
                 void *ws, size_t *ws_bytes, void *stream);

/* Distinct-per-dimension flags (core.py:278-281): flags[k] = 1 when the n coordinates of
 * dimension k are pairwise distinct.  flags: host (d,).  Syncs. */
int fcg_distinct(const double *x, int64_t n, int32_t d, int32_t *flags,
                 void *ws, size_t *ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * Host <-> device transfers of the drop-in numpy path (numpy in, numpy out)
 * ------------------------------------------------------------------------------------- */

/* Pageable host -> device copy staged through a pinned ring with multi-threaded host copies;
 * enqueued on `stream`, returns once the source may be reused (like cudaMemcpyAsync from
 * pageable memory).  Replaces the implicit np.asarray upload of every reference call. */
int fcg_copy_h2d(void *dst_dev, const void *src_host, size_t bytes, void *stream);
/* Device -> pageable host copy after the work queued on `stream`; returns when dst is filled. */
int fcg_copy_d2h(void *dst_host, const void *src_dev, size_t bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * At-points path (subsystem 4)
 * ------------------------------------------------------------------------------------- */

/* Generalized ECDF at the sample points with ties allowed, Eq. (3) exactly as naive.py:90-114
 * implements it (i == j included): out[j] = sum_i w_i prod_k [x_ik <= x_jk] (delta=+1) or
 * [x_ik < x_jk] (delta=-1); survival == 1 gives Eq. (2), sum_i w_i prod_k [x_ik > x_jk].
 * Divided by n when scaled.  Syncs (reads the distinct-level counts to pick the rank lattice
 * or the dominance kernel).  Routes: rank lattice when the grid of distinct levels is small;
 * rank-space dominance otherwise (d = 2: coarse grid + per-chunk solvers; 3 <= d <= 6 and
 * n >= 8192: coarse G^d grid + per-dimension slab phases, csrc/points_nd.cuh; direct tiles
 * only for d >= 7 or fewer points). */
int fcg_ecdf_points(const double *x, int64_t n, int32_t d, const double *w,
                    const int32_t *delta, int32_t survival, int32_t scaled, double *out,
                    void *ws, size_t *ws_bytes, void *stream);

/* Both at-points outputs of BASELINE config 2 from one ranking of every dimension:
 * out_ecdf as fcg_ecdf_points(delta, survival = 0) and out_esf as fcg_ecdf_points(survival = 1)
 * (naive.py:90-114, 210-217).  One host sync (the distinct-level counts). */
int fcg_ecdf_esf_points(const double *x, int64_t n, int32_t d, const double *w,
                        const int32_t *delta, int32_t scaled, double *out_ecdf, double *out_esf,
                        void *ws, size_t *ws_bytes, void *stream);

/* Strict-dominance ECDF at the sample points (requires pairwise-distinct coordinates per
 * dimension, checked by the caller): out[j] = sum_{i != j, x_i < x_j in every dim} w_i,
 * + w_j when include_self, / n when scaled.  Replaces dnc.py:531-561 ecdf_dnc (and, for
 * d >= 3, the MergeND recursion dnc.py:65-135, 307-410 behind it: the rank-space coarse grid +
 * slab phases of csrc/points_nd.cuh for 3 <= d <= 6). */
int fcg_dnc_ecdf(const double *x, int64_t n, int32_t d, const double *w,
                 int32_t include_self, int32_t scaled, double *out,
                 void *ws, size_t *ws_bytes, void *stream);

/* Laplacian KDE at the sample points via 2^d all-delta strict-dominance sums
 * (dnc.py:635-690 kde_dnc, _run_all_delta dnc.py:564-585).  Requires distinct coordinates.
 * h, centre: host (d,).  nw weight vectors w[v*n + i] (v < nw) are evaluated in one pass;
 * out[v*n + j] receives the density numerator of weight vector v (self term and
 * 1/(2^d n prod h) included, exactly the reference's kde_dnc output).  3 <= d <= 6: every
 * sign code's far field from a coarse rank grid, pairs sharing a rank chunk summed directly
 * (csrc/points_nd.cuh). */
int fcg_kde_points_laplacian(const double *x, int64_t n, int32_t d, const double *w,
                             int32_t nw, const double *h, const double *centre, double *out,
                             void *ws, size_t *ws_bytes, void *stream);

/* Query-sharded forms for one process per GPU ("sample-point queries are sharded
 * with the ranked data replicated"); d = 2 (the dominance route).  Every shard ranks and
 * groups all n sources (replicated) but evaluates only its own queries: the points whose
 * rank along dimension 1 falls in chunks [P s / G, P (s+1) / G) of the P = ceil(n / 2048)
 * chunks (a contiguous 1/G slice of the queries in rank order).  Other entries of out are
 * set to exactly 0, so a SUM all-reduce over the G shards gathers the result (the owned values
 * are computed by exactly the unsharded arithmetic).  Same arguments as the unsharded calls plus
 * shard s in [0, G) and G. */
int fcg_kde_points_laplacian_shard(const double *x, int64_t n, int32_t d, const double *w,
                                   int32_t nw, const double *h, const double *centre,
                                   int32_t shard, int32_t nshards, double *out,
                                   void *ws, size_t *ws_bytes, void *stream);
int fcg_dnc_ecdf_shard(const double *x, int64_t n, int32_t d, const double *w,
                       int32_t include_self, int32_t scaled, int32_t shard, int32_t nshards,
                       double *out, void *ws, size_t *ws_bytes, void *stream);

/* As fcg_kde_points_laplacian for d = 2, with one pointer per weight vector (NULL = unit
 * weights for that channel), so callers mixing a unit density and a response need no stacked
 * copy (the config-4 pair: w0 = NULL, w1 = y). */
int fcg_kde_points_laplacian_w2(const double *x, int64_t n, int32_t d, const double *w0,
                                const double *w1, int32_t nw, const double *h,
                                const double *centre, double *out, void *ws, size_t *ws_bytes,
                                void *stream);

/* All-delta strict-dominance tables (dnc.py:608-632 kde_terms_dnc, _run_all_delta): psi and
 * table are (n, 2^d) row-major; table[j][b] = sum of psi[i][b] over the points i != j with
 * x_ik < x_jk where bit k of b is 0 and x_ik > x_jk where it is 1.  Requires distinct
 * coordinates per dimension; d <= 6.  One rank-space dominance sum per code (3 <= d <= 6,
 * n >= 8192: csrc/points_nd.cuh), direct tiled pairs otherwise. */
int fcg_dominance_terms(const double *x, int64_t n, int32_t d, const double *psi, double *table,
                        void *ws, size_t *ws_bytes, void *stream);

/* matern32-additive KDE at the sample points (dnc.py:635-690 with family "matern32-additive"):
 * the d + 1 channels of dnc.py:661-669 are run as 2d + 1 Laplacian dominance channels whose
 * weights only change sign with the term (A = w e, B_k = s_k w e, C_l = s_l w xc_l e / h_l),
 * combined as A + sum_k (xc_k / h_k) B_k - sum_l C_l, + w, * 1 / (2^d n prod h (1 + d)).
 * One weight vector (or NULL); requires distinct coordinates; h, centre host (d,).
 * d = 3, 4 (n >= 8192): per sign code the two far-field channels sum w psi and sum w U psi
 * (U = sum_k s_k u_k) on the coarse rank grid, pairs sharing a rank chunk summed directly as
 * (1 + U_s - U_t) psi_s / psi_t from per-point tables (csrc/points_nd.cuh); d >= 5: direct
 * tiles. */
int fcg_kde_points_matern32(const double *x, int64_t n, int32_t d, const double *w,
                            const double *h, const double *centre, double *out,
                            void *ws, size_t *ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTCDF_B200_H */
