/*
 * ORACLE — test infrastructure only.  CPU restatement of the reference fastcdf algorithms
 * (/root/reference/pkg/src/fastcdf) used as the parity checker by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference leg.  The product
 * path (paper_2005_03246_b200) never links, imports or calls this file.
 *
 * Pinned against the reference's own outputs: the tests/golden npz fixtures were produced by importing
 * the reference package in the build container (tests/golden/make_golden.py) and
 * tests/test_oracle_golden.py checks every function here against them.
 *
 * Each function cites the reference code it restates.  Summation orders follow the reference
 * (np.bincount input order, sequential np.cumsum along an axis), so unit- and integer-weight
 * results are bit-identical and fp64 results match to the last ulp in practice.
 * Thread parallelism (pthreads; the image has no libgomp) is only over independent work items
 * (points, whole scan lines), which preserves every per-value summation order.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORC_API __attribute__((visibility("default")))

static int g_threads = 1;

ORC_API int orc_max_threads(void) {
  long v = sysconf(_SC_NPROCESSORS_ONLN);
  return v > 0 ? (int)v : 1;
}

ORC_API void orc_set_threads(int t) { g_threads = t > 0 ? t : 1; }
ORC_API int orc_get_threads(void) { return g_threads; }

/* static-chunk parallel for over [0, n): body(lo, hi, ctx) on up to g_threads threads */
typedef void (*orc_body)(int64_t lo, int64_t hi, void *ctx);
typedef struct {
  orc_body f;
  void *ctx;
  int64_t lo, hi;
} orc_job;

static void *orc_run(void *p) {
  orc_job *j = (orc_job *)p;
  j->f(j->lo, j->hi, j->ctx);
  return NULL;
}

static void parallel_for(int64_t n, orc_body f, void *ctx) {
  int T = g_threads > 64 ? 64 : g_threads;
  if (T <= 1 || n < 2 * (int64_t)T) {
    f(0, n, ctx);
    return;
  }
  pthread_t th[64];
  orc_job jobs[64];
  int spawned[64] = {0};
  const int64_t chunk = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    jobs[t].f = f;
    jobs[t].ctx = ctx;
    jobs[t].lo = t * chunk < n ? t * chunk : n;
    jobs[t].hi = (t + 1) * chunk < n ? (t + 1) * chunk : n;
  }
  for (int t = 1; t < T; ++t)
    if (jobs[t].lo < jobs[t].hi && pthread_create(&th[t], NULL, orc_run, &jobs[t]) == 0)
      spawned[t] = 1;
  f(jobs[0].lo, jobs[0].hi, ctx);
  for (int t = 1; t < T; ++t) {
    if (spawned[t]) pthread_join(th[t], NULL);
    else if (jobs[t].lo < jobs[t].hi) f(jobs[t].lo, jobs[t].hi, ctx);
  }
}

/* _flat_bins_uniform, histogram.py:60-92: mesh-division guess then nudge against the knots;
 * flat = sum_k b_k * prod_{j>k} (M_j + 1).  closed[k] = 1 for delta_k = +1. */
typedef struct {
  const double *points, *z0, *dz, *knots_flat;
  const int64_t *msize, *offsets;
  const uint8_t *closed;
  int d;
  int64_t *out;
} bins_ctx;

static void bins_body(int64_t lo, int64_t hi, void *vp) {
  const bins_ctx *c = (const bins_ctx *)vp;
  for (int64_t i = lo; i < hi; ++i) {
    int64_t flat = 0;
    for (int k = 0; k < c->d; ++k) {
      const double x = c->points[i * c->d + k];
      const double t = (x - c->z0[k]) / c->dz[k];
      const int64_t m = c->msize[k];
      int64_t b;
      if (c->closed[k]) b = (int64_t)ceil(t); /* int(np.ceil(t)) */
      else b = (int64_t)floor(t) + 1;         /* int(np.floor(t)) + 1 */
      if (b < 0) b = 0;
      else if (b > m) b = m;
      const double *kn = c->knots_flat + c->offsets[k];
      if (c->closed[k]) {
        while (b > 0 && x <= kn[b - 1]) --b;
        while (b < m && x > kn[b]) ++b;
      } else {
        while (b > 0 && x < kn[b - 1]) --b;
        while (b < m && x >= kn[b]) ++b;
      }
      flat = flat * (m + 1) + b;
    }
    c->out[i] = flat;
  }
}

ORC_API void orc_flat_bins_uniform(const double *points, int64_t n, int d, const double *z0,
                                   const double *dz, const int64_t *msize, const uint8_t *closed,
                                   const double *knots_flat, const int64_t *offsets,
                                   int64_t *out) {
  bins_ctx c = {points, z0, dz, knots_flat, msize, offsets, closed, d, out};
  parallel_for(n, bins_body, &c);
}

/* _scan_bins_sorted, histogram.py:43-57: two-pointer walk of the stably sorted values
 * (order = np.argsort(kind="stable")) against the knot ladder. */
ORC_API void orc_scan_bins_sorted(const double *values, int64_t stride, const int64_t *order,
                                  int64_t n, const double *knots, int64_t m, int closed,
                                  int64_t *out) {
  int64_t g = 0;
  for (int64_t t = 0; t < n; ++t) {
    const int64_t i = order[t];
    const double x = values[i * stride];
    if (closed) {
      while (g < m && knots[g] < x) ++g;
    } else {
      while (g < m && knots[g] <= x) ++g;
    }
    out[i] = g;
  }
}

/* np.bincount(flat, weights, minlength=L) (histogram.py:177-181): sequential, input order. */
ORC_API void orc_bincount(const int64_t *flat, const double *w, int64_t n, int64_t L,
                          double *out) {
  memset(out, 0, (size_t)L * sizeof(double));
  if (w) {
    for (int64_t i = 0; i < n; ++i) out[flat[i]] += w[i];
  } else {
    for (int64_t i = 0; i < n; ++i) out[flat[i]] += 1.0;
  }
}

/* One axis of _cumsum_directional, fastsum.py:45-57: np.cumsum along `axis` (reverse = flip,
 * cumsum, flip), in place over a C-contiguous array.  Parallel over independent lines. */
typedef struct {
  double *data;
  int64_t D, B;
  int reverse;
} cum_ctx;

static void cum_rows_body(int64_t lo, int64_t hi, void *vp) {
  const cum_ctx *c = (const cum_ctx *)vp;
  for (int64_t a = lo; a < hi; ++a) {
    double *row = c->data + a * c->D;
    double run = 0.0;
    if (!c->reverse) {
      for (int64_t j = 0; j < c->D; ++j) { run += row[j]; row[j] = run; }
    } else {
      for (int64_t j = c->D - 1; j >= 0; --j) { run += row[j]; row[j] = run; }
    }
  }
}

/* strided axis: item = (a, block of 256 b's); walk j with the inner loop over contiguous b */
static void cum_lines_body(int64_t lo, int64_t hi, void *vp) {
  const cum_ctx *c = (const cum_ctx *)vp;
  const int64_t nb = (c->B + 255) / 256;
  for (int64_t item = lo; item < hi; ++item) {
    const int64_t a = item / nb, b0 = (item % nb) * 256;
    const int64_t b1 = b0 + 256 < c->B ? b0 + 256 : c->B;
    double *base = c->data + a * c->D * c->B;
    if (!c->reverse) {
      for (int64_t j = 1; j < c->D; ++j) {
        double *cur = base + j * c->B, *prev = base + (j - 1) * c->B;
        for (int64_t b = b0; b < b1; ++b) cur[b] += prev[b];
      }
    } else {
      for (int64_t j = c->D - 2; j >= 0; --j) {
        double *cur = base + j * c->B, *prev = base + (j + 1) * c->B;
        for (int64_t b = b0; b < b1; ++b) cur[b] += prev[b];
      }
    }
  }
}

ORC_API void orc_cumsum_axis(double *data, int d, const int64_t *dims, int axis, int reverse) {
  int64_t A = 1, B = 1;
  for (int k = 0; k < axis; ++k) A *= dims[k];
  for (int k = axis + 1; k < d; ++k) B *= dims[k];
  cum_ctx c = {data, dims[axis], B, reverse};
  if (B == 1) parallel_for(A, cum_rows_body, &c);
  else parallel_for(A * ((B + 255) / 256), cum_lines_body, &c);
}

/* Compaction of fastsum.py:85-88: core = cum[0:M_1, ..., 0:M_d] (lo[k] = 0) or the shifted
 * slice [1:M+1] (lo[k] = 1, _delta_term_slices fastsum.py:132-136), optionally / n. */
typedef struct {
  const double *cum;
  int d;
  const int64_t *m, *lo;
  double divisor;
  double *out;
} slice_ctx;

static void slice_body(int64_t lo, int64_t hi, void *vp) {
  const slice_ctx *c = (const slice_ctx *)vp;
  for (int64_t j = lo; j < hi; ++j) {
    int64_t rem = j, src = 0, stride = 1;
    for (int k = c->d - 1; k >= 0; --k) {
      const int64_t idx = rem % c->m[k];
      rem /= c->m[k];
      src += (idx + c->lo[k]) * stride;
      stride *= (c->m[k] + 1);
    }
    double v = c->cum[src];
    if (c->divisor > 0.0) v /= c->divisor;
    c->out[j] = v;
  }
}

ORC_API void orc_slice(const double *cum, int d, const int64_t *m, const int64_t *lo,
                       double divisor, double *out) {
  int64_t M = 1;
  for (int k = 0; k < d; ++k) M *= m[k];
  slice_ctx c = {cum, d, m, lo, divisor, out};
  parallel_for(M, slice_body, &c);
}

/* _ecdf_naive_loop, naive.py:90-114: Kahan-compensated direct double loop. */
typedef struct {
  const double *points, *weights, *queries, *signs, *h;
  int64_t n;
  int d, exclude_self;
  double *out;
} naive_ctx;

static void ecdf_naive_body(int64_t lo, int64_t hi, void *vp) {
  const naive_ctx *c = (const naive_ctx *)vp;
  for (int64_t j = lo; j < hi; ++j) {
    double acc = 0.0, comp = 0.0;
    for (int64_t i = 0; i < c->n; ++i) {
      if (c->exclude_self && i == j) continue;
      int ok = 1;
      for (int k = 0; k < c->d; ++k) {
        const double a = c->points[i * c->d + k], z = c->queries[j * c->d + k];
        if (c->signs[k] > 0 ? (a > z) : (a >= z)) { ok = 0; break; }
      }
      if (ok) {
        const double y = c->weights[i] - comp;
        const double t = acc + y;
        comp = (t - acc) - y;
        acc = t;
      }
    }
    c->out[j] = acc;
  }
}

ORC_API void orc_ecdf_naive(const double *points, const double *weights, int64_t n, int d,
                            const double *queries, int64_t q, const double *signs,
                            int exclude_self, double *out) {
  naive_ctx c = {points, weights, queries, signs, NULL, n, d, exclude_self, out};
  parallel_for(q, ecdf_naive_body, &c);
}

/* _kde_naive_diag_loop with the Laplacian profile (naive.py:117-141, _profile1 naive.py:64-72
 * with alpha = 1, betas = (1,), gamma = 1/2, shape_h = 1): sum_i w_i prod_k e^{-|u_k|}/2. */
static void kde_naive_body(int64_t lo, int64_t hi, void *vp) {
  const naive_ctx *c = (const naive_ctx *)vp;
  for (int64_t j = lo; j < hi; ++j) {
    double acc = 0.0, comp = 0.0;
    for (int64_t i = 0; i < c->n; ++i) {
      double val = 1.0;
      for (int k = 0; k < c->d; ++k) {
        const double t = fabs((c->points[i * c->d + k] - c->queries[j * c->d + k]) / c->h[k]);
        const double s = t / 1.0;
        const double poly = 0.0 * s + 1.0;
        val *= (0.5 / 1.0) * poly * exp(-1.0 * s);
        if (val == 0.0) break;
      }
      const double y = c->weights[i] * val - comp;
      const double t2 = acc + y;
      comp = (t2 - acc) - y;
      acc = t2;
    }
    c->out[j] = acc;
  }
}

ORC_API void orc_kde_naive_laplacian(const double *points, const double *weights, int64_t n,
                                     int d, const double *queries, int64_t q, const double *h,
                                     double *out) {
  naive_ctx c = {points, weights, queries, NULL, h, n, d, 0, out};
  parallel_for(q, kde_naive_body, &c);
}

/* ---- divide-and-conquer dominance, d = 2 (dnc.py) -------------------------------------- */

/* _merge1d_ecdf, dnc.py:45-62 */
static void merge1d_ecdf(const double *x0, const int64_t *src, int64_t m1, const int64_t *tgt,
                         int64_t m2, const double *y, double *F) {
  double s = 0.0;
  int64_t j = 0;
  for (int64_t i = 0; i < m2; ++i) {
    const int64_t t = tgt[i];
    while (j < m1 && x0[src[j]] <= x0[t]) { s += y[src[j]]; ++j; }
    F[t] += s;
    if (j == m1) {
      for (int64_t k = i + 1; k < m2; ++k) F[tgt[k]] += s;
      return;
    }
  }
}

#define ORC_BASE 32 /* dnc.py:39 */

/* _recur_split_ecdf for d = 2, dnc.py:138-186.  x is (2, n) row-major (points.T). */
static void recur_split_ecdf2(const double *x, int64_t n, const double *y, double *F,
                              const int64_t *phi0, const int64_t *phi1, int64_t m,
                              uint8_t *mask) {
  if (m <= 1) return;
  if (m <= ORC_BASE) {
    for (int64_t b = 0; b < m; ++b) {
      const int64_t t = phi0[b];
      for (int64_t a = 0; a < m; ++a) {
        const int64_t s = phi0[a];
        if (s == t) continue;
        if (x[s] >= x[t]) continue;
        if (x[n + s] >= x[n + t]) continue;
        F[t] += y[s];
      }
    }
    return;
  }
  const int64_t mid = m / 2;
  /* layout: child1 rows 0/1 [mid each], then child2 rows 0/1 [m - mid each] */
  int64_t *p1 = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)m);
  int64_t *c1r0 = p1, *c1r1 = p1 + mid;
  int64_t *c2r0 = p1 + 2 * mid, *c2r1 = p1 + 2 * mid + (m - mid);
  for (int64_t t = 0; t < mid; ++t) mask[phi1[t]] = 1;
  int64_t a = 0, b = 0;
  for (int64_t t = 0; t < m; ++t) {
    const int64_t p = phi0[t];
    if (mask[p]) c1r0[a++] = p;
    else c2r0[b++] = p;
  }
  memcpy(c1r1, phi1, sizeof(int64_t) * (size_t)mid);
  memcpy(c2r1, phi1 + mid, sizeof(int64_t) * (size_t)(m - mid));
  for (int64_t t = 0; t < mid; ++t) mask[phi1[t]] = 0;
  recur_split_ecdf2(x, n, y, F, c1r0, c1r1, mid, mask);
  recur_split_ecdf2(x, n, y, F, c2r0, c2r1, m - mid, mask);
  merge1d_ecdf(x, c1r0, mid, c2r0, m - mid, y, F);
  free(p1);
}

/* ecdf_dnc's recursion for d = 2 (dnc.py:549-553); phi = stable argsorts per dim. */
ORC_API void orc_dnc_ecdf2(const double *xT, int64_t n, const double *y, const int64_t *phi0,
                           const int64_t *phi1, double *F) {
  uint8_t *mask = (uint8_t *)calloc((size_t)n, 1);
  memset(F, 0, sizeof(double) * (size_t)n);
  recur_split_ecdf2(xT, n, y, F, phi0, phi1, n, mask);
  free(mask);
}

/* _merge1d1_delta / _merge1d2_delta, dnc.py:251-304, restricted to the column list. */
static void merge1d1_delta(const double *x0, const int64_t *src, int64_t m1, const int64_t *tgt,
                           int64_t m2, const double *psi, int ncols, double *F, const int *cols,
                           int nc, double *S) {
  if (nc == 0 || m1 == 0 || m2 == 0) return;
  for (int c = 0; c < nc; ++c) S[cols[c]] = 0.0;
  int64_t j = 0;
  for (int64_t i = 0; i < m2; ++i) {
    const int64_t t = tgt[i];
    while (j < m1 && x0[src[j]] <= x0[t]) {
      const int64_t s = src[j];
      for (int c = 0; c < nc; ++c) S[cols[c]] += psi[s * ncols + cols[c]];
      ++j;
    }
    for (int c = 0; c < nc; ++c) F[t * ncols + cols[c]] += S[cols[c]];
    if (j == m1) {
      for (int64_t k = i + 1; k < m2; ++k)
        for (int c = 0; c < nc; ++c) F[tgt[k] * ncols + cols[c]] += S[cols[c]];
      return;
    }
  }
}

static void merge1d2_delta(const double *x0, const int64_t *src, int64_t m1, const int64_t *tgt,
                           int64_t m2, const double *psi, int ncols, double *F, const int *cols,
                           int nc, double *S) {
  if (nc == 0 || m1 == 0 || m2 == 0) return;
  for (int c = 0; c < nc; ++c) S[cols[c]] = 0.0;
  int64_t j = m1 - 1;
  for (int64_t i = m2 - 1; i >= 0; --i) {
    const int64_t t = tgt[i];
    while (j >= 0 && x0[src[j]] > x0[t]) {
      const int64_t s = src[j];
      for (int c = 0; c < nc; ++c) S[cols[c]] += psi[s * ncols + cols[c]];
      --j;
    }
    for (int c = 0; c < nc; ++c) F[t * ncols + cols[c]] += S[cols[c]];
    if (j < 0) {
      for (int64_t k = 0; k < i; ++k)
        for (int c = 0; c < nc; ++c) F[tgt[k] * ncols + cols[c]] += S[cols[c]];
      return;
    }
  }
}

/* _recur_split_delta for d = 2 (dnc.py:413-468): code bit 0 = dim-0 strict-greater,
 * bit 1 = dim-1 strict-greater; column = code * nch + c. */
static void recur_split_delta2(const double *x, int64_t n, const double *psi, int nch,
                               double *F, const int64_t *phi0, const int64_t *phi1, int64_t m,
                               uint8_t *mask, double *S) {
  const int ncols = 4 * nch;
  if (m <= 1) return;
  if (m <= ORC_BASE) {
    for (int64_t b = 0; b < m; ++b) {
      const int64_t t = phi0[b];
      for (int64_t a = 0; a < m; ++a) {
        const int64_t s = phi0[a];
        if (s == t) continue;
        int code = 0; /* _pair_code dnc.py:193-199 */
        if (x[s] > x[t]) code |= 1;
        if (x[n + s] > x[n + t]) code |= 2;
        for (int c = 0; c < nch; ++c) F[t * ncols + code * nch + c] += psi[s * ncols + code * nch + c];
      }
    }
    return;
  }
  const int64_t mid = m / 2;
  int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)m);
  int64_t *c1r0 = buf, *c1r1 = buf + mid, *c2r0 = buf + 2 * mid, *c2r1 = buf + 2 * mid + (m - mid);
  for (int64_t t = 0; t < mid; ++t) mask[phi1[t]] = 1;
  int64_t a = 0, b = 0;
  for (int64_t t = 0; t < m; ++t) {
    const int64_t p = phi0[t];
    if (mask[p]) c1r0[a++] = p;
    else c2r0[b++] = p;
  }
  memcpy(c1r1, phi1, sizeof(int64_t) * (size_t)mid);
  memcpy(c2r1, phi1 + mid, sizeof(int64_t) * (size_t)(m - mid));
  for (int64_t t = 0; t < mid; ++t) mask[phi1[t]] = 0;
  recur_split_delta2(x, n, psi, nch, F, c1r0, c1r1, mid, mask, S);
  recur_split_delta2(x, n, psi, nch, F, c2r0, c2r1, m - mid, mask, S);
  /* dnc.py:459-468: the four 1-d merges selected by _filter_bits3 over codes 0..3 */
  int cols[4 * 8];
  int nc;
  /* codes with bit0 = 0 and bit1 = 0 (code 0): sources phi1 -> targets phi2, <= merge */
  nc = 0; for (int c = 0; c < nch; ++c) cols[nc++] = 0 * nch + c;
  merge1d1_delta(x, c1r0, mid, c2r0, m - mid, psi, ncols, F, cols, nc, S);
  /* bit0 = 1, bit1 = 0 (code 1): phi1 -> phi2, strictly-above merge */
  nc = 0; for (int c = 0; c < nch; ++c) cols[nc++] = 1 * nch + c;
  merge1d2_delta(x, c1r0, mid, c2r0, m - mid, psi, ncols, F, cols, nc, S);
  /* bit0 = 0, bit1 = 1 (code 2): phi2 -> phi1 */
  nc = 0; for (int c = 0; c < nch; ++c) cols[nc++] = 2 * nch + c;
  merge1d1_delta(x, c2r0, m - mid, c1r0, mid, psi, ncols, F, cols, nc, S);
  /* bit0 = 1, bit1 = 1 (code 3): phi2 -> phi1 */
  nc = 0; for (int c = 0; c < nch; ++c) cols[nc++] = 3 * nch + c;
  merge1d2_delta(x, c2r0, m - mid, c1r0, mid, psi, ncols, F, cols, nc, S);
  free(buf);
}

/* _run_all_delta for d = 2 (dnc.py:564-585). psi, F: (n, 4*nch) row-major. */
ORC_API void orc_run_all_delta2(const double *xT, int64_t n, const double *psi, int nch,
                                const int64_t *phi0, const int64_t *phi1, double *F) {
  uint8_t *mask = (uint8_t *)calloc((size_t)n, 1);
  double *S = (double *)calloc(4 * (size_t)nch, sizeof(double));
  memset(F, 0, sizeof(double) * (size_t)n * 4 * (size_t)nch);
  recur_split_delta2(xT, n, psi, nch, F, phi0, phi1, n, mask, S);
  free(S);
  free(mask);
}
