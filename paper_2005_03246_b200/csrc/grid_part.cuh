// Partitioned grid pipeline (d >= 3): points are bucketed once by lattice plane (the last two
// axes) with a 2-pass radix partition on 32-bit bucket keys; one CTA per plane then builds the
// plane histogram in shared memory (no memset, no global atomics), scans both in-plane axes
// there and writes the plane once.  The remaining leading axes are walked by the scan engine,
// whose last pass carries the output epilogue.
#pragma once
#include "bin.cuh"
#include "scan.cuh"

namespace fcg {

struct PartPlan {
  bool ok = false;
  int64_t NP = 0;   // planes (product of the leading d-2 extents)
  int64_t H = 0;    // rows per plane (extent of axis d-2)
  int64_t W = 0;    // row length (extent of axis d-1)
  int64_t R = 0;    // rows per shared-memory block
  int64_t nrb = 0;  // row blocks per plane
  int64_t NB = 0;   // buckets
  int nbits = 0;    // radix key bits
  int cell_bits = 0;  // KDE: in-bucket cell bits of the sorted key (0: bucket-only keys)
  bool all = false;   // KDE: every term group from one plane pass (plane_kde_all_kernel)
  int col_bits = 0;
};

// Unit-weight ECDF / ESF over the cell-space lattice `g` (dims = output extents).
PartPlan plan_ecdf_partition(const BinGrid &g, int64_t n);
// Carve (ws == nullptr: size only) and run.  epi: the final epilogue (axis 0).
int ecdf_partitioned(const double *x, int64_t n, const double *knots, const BinGrid &g,
                     const bool *rev, const PartPlan &plan, const Epi &epi, Workspace &W,
                     bool run, cudaStream_t st);

// Slab carry planes of the KDE: a captured plane is weighted by the factors zf_k of the axes
// k >= kde_cap_kw(d) (the in-plane axes the partitioned path folds, never the slab axis 1);
// the carry fix-up applies the factors of the axes below it.
inline int kde_cap_kw(int d) { return d - 2 > 2 ? d - 2 : 2; }

// Laplacian KDE: full-space binning (dims M_k + 1) shared by all 2^d terms.
PartPlan plan_kde_partition(int d, const int64_t *m, int64_t n, bool factored);
// bound_u_sum: an upper bound of sum_k max_i |x_ik - c_k| / h_k (selects the factored psi
// records); n_scale: the N of the 1/(2^d N prod h) normalisation (the global N on a slab);
// planes: optional [2^d][A * B1] capture of each term's slab-boundary S plane (may be null).
int kde_partitioned(const double *x, int64_t n, const double *w, const double *knots,
                    const int64_t *m, int d, const double *h, const double *centre,
                    double bound_u_sum, double n_scale, double *planes, const PartPlan &plan,
                    double *out, Workspace &W, bool run, cudaStream_t st);

// Auto centre of the KDE (centre == NULL): mm[0..d) / mm[d..2d) = order keys of the hull's
// lower / upper ends, seeded with the knot ends by hull_init and widened by the binning pass.
struct HullKnots {
  int d;
  int64_t first[FCG_MAX_DIM], last[FCG_MAX_DIM];
};
int hull_init(const double *knots, int d, const int64_t *m, unsigned long long *mm, cudaStream_t st);
// Synchronises; c = (lo + hi) / 2 and u_bound = sum_k span_k / (2 h_k) (with a 1e-6 margin), or
// FCG_ERANGE past span_k / h_k > 600 (fastsum.py:114-129).
int hull_centre(const unsigned long long *mm, int d, const double *h, double *c, double *u_bound,
                cudaStream_t st);

}  // namespace fcg
