// Shared binning: the reference's delta-dependent bin rule (histogram.py:3-15,60-92) evaluated
// exactly from the uploaded knot values.
#pragma once
#include "common.cuh"

namespace fcg {

constexpr int kSmemKnots = 4096;  // up to 32 KB of knots staged in (dynamic) shared memory

struct BinGrid {
  int d;
  int64_t m[FCG_MAX_DIM];
  int64_t koff[FCG_MAX_DIM];
  int le[FCG_MAX_DIM];       // 1: count knots <= x (delta=-1); 0: count knots < x (delta=+1)
  int64_t shift[FCG_MAX_DIM];  // lattice cell = b - shift
  int64_t dims[FCG_MAX_DIM];   // lattice extents
  int64_t stride[FCG_MAX_DIM];
  int64_t total_knots;
};

enum WeightKind { W_UNIT = 0, W_F64 = 1, W_PSI = 2 };

struct PsiParams {  // psi_i = w_i * exp(sum_k (x_ik - c_k) * a_k), a_k = delta_k / h_k
  double c[FCG_MAX_DIM];
  double a[FCG_MAX_DIM];
  int poly1;  // l + 1: psi_i also times (x_il - c_l) (matern32 channels); 0: no factor
};

// #knots < x (le = 0) or #knots <= x (le = 1) for a strictly increasing knot vector.
// The mesh guess (exact for uniform grids except right at knots) is verified against the
// uploaded knot values and nudged once; anything farther off falls back to binary search, so
// the result is the exact count for any rectilinear grid.
//
// mesh_ok: the knots were checked to lie within kMeshTol mesh steps of z0 + j dz (mesh_uniform
// below).  Then a point whose mesh coordinate t is farther than kMeshSafe from every integer is
// on the same side of the nearest knots as of the mesh lines (t itself is off by < 1e-13 for
// m <= 2^20), so the guess is the exact count and the knot loads and compares are skipped.
constexpr double kMeshTol = 1e-9, kMeshSafe = 1e-6;

__device__ __forceinline__ int knot_count(double x, const double *kn, int m, int le, double z0,
                                          double inv_dz, bool mesh_ok = false) {
  const double t = (x - z0) * inv_dz;
  // floor(t) + 1 (le) or ceil(t), clamped to [0, m]: the conversions saturate (NaN -> 0)
  const int f = le ? __double2int_rd(t) : __double2int_ru(t - 1.0);
  const int g = min(max(f, -1), m - 1) + 1;
  if (mesh_ok && fabs(t - rint(t)) > kMeshSafe) return g;  // NaN: falls through
  // pred(k) := knot k counts (kn[k] < x, or <= x when le); valid iff pred(g-1) && !pred(g)
  const double a = kn[g > 0 ? g - 1 : 0], b = kn[g < m ? g : m - 1];
  const bool lo_ok = (g == 0) || a < x || (le && a == x);
  const bool hi_ok = (g == m) || x < b || (!le && x == b);
  if (lo_ok && hi_ok) return g;
  const int g2 = lo_ok ? g + 1 : g - 1;  // one nudge (knot hits land one bin off)
  const bool lo2 = (g2 == 0) || (le ? (kn[g2 - 1] <= x) : (kn[g2 - 1] < x));
  const bool hi2 = (g2 == m) || (le ? (x < kn[g2]) : (x <= kn[g2]));
  if (lo2 && hi2) return g2;
  int lo = 0, hi = m;  // first index whose knot fails the predicate
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool pred = le ? (kn[mid] <= x) : (kn[mid] < x);
    if (pred) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Bit k set when dimension k's knots follow the mesh z0 + j dz to kMeshTol steps.  Call from
// every thread of the CTA after stage_knots' barrier (contains barriers).
__device__ __forceinline__ unsigned mesh_uniform(const BinGrid &g, const double *kb,
                                                 const double *s_z0, const double *s_idz) {
  unsigned mask = 0;
  for (int k = 0; k < g.d; ++k) {
    const double *kn = kb + g.koff[k];
    bool ok = true;
    for (int64_t j = threadIdx.x; j < g.m[k]; j += blockDim.x)
      ok = ok && fabs((kn[j] - s_z0[k]) * s_idz[k] - (double)j) <= kMeshTol;
    if (g.m[k] > (int64_t(1) << 20)) ok = false;
    if (__syncthreads_and(ok)) mask |= 1u << k;
  }
  return mask;
}

inline BinGrid make_bin_grid(int d, const int64_t *m, const int *le, const int64_t *shift,
                      const int64_t *dims) {
  BinGrid g{};
  g.d = d;
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    g.m[k] = m[k];
    g.koff[k] = off;
    off += m[k];
    g.le[k] = le[k];
    g.shift[k] = shift[k];
    g.dims[k] = dims[k];
  }
  g.total_knots = off;
  int64_t s = 1;
  for (int k = d - 1; k >= 0; --k) {
    g.stride[k] = s;
    s *= dims[k];
  }
  return g;
}


// Stage the knots (when they fit) and the per-dimension mesh guess parameters in shared
// memory; returns the knot base pointer to use.  Call from every thread, then __syncthreads().
__device__ __forceinline__ const double *stage_knots(const BinGrid &g, const double *knots,
                                                     double *s_knots, double *s_z0,
                                                     double *s_idz) {
  const bool use_smem = g.total_knots <= kSmemKnots;
  if (use_smem)
    for (int64_t i = threadIdx.x; i < g.total_knots; i += blockDim.x) s_knots[i] = knots[i];
  if (threadIdx.x < g.d) {
    const int k = threadIdx.x;
    const double *kn = knots + g.koff[k];
    const int64_t m = g.m[k];
    s_z0[k] = kn[0];
    s_idz[k] = (m > 1) ? (double)(m - 1) / (kn[m - 1] - kn[0]) : 0.0;
  }
  return use_smem ? s_knots : knots;
}

}  // namespace fcg
