// Directional prefix-sum engine over dense d-dimensional lattices (Algorithm 1's sweep).
//
// A d-dim lattice is scanned one axis at a time.  For axis `ax` the lattice is viewed as
// [A][D][B] (A = product of the leading extents, D = extent of ax, B = product of the trailing
// extents).  Two kernel shapes cover every axis:
//   * rows  (B == 1, the contiguous last axis): one warp per row segment, 32 consecutive
//           elements per step, warp-shuffle inclusive scans, register carry;
//   * lines (B > 1): one thread per (a, b) line, b fastest so that every step of a warp touches
//           32 consecutive elements (coalesced), unrolled loads to keep many bytes in flight.
// When A*B is too small to fill 148 SMs the axis is split into C chunks and scanned in three
// phases (chunk totals -> exclusive scan of the totals -> re-scan with carry-in).
// The last pass of a pipeline carries an epilogue that writes the final result (fp64 value
// with the single division by N of fastsum.py:87-88, int64 counts, or the KDE term
// accumulation zfac * S of fastsum.py:162-168 with the final scale of fastsum.py:179-182) so the
// lattice is never re-read.
#pragma once
#include "common.cuh"

namespace fcg {

enum EpiKind { EPI_INPLACE = 0, EPI_F64 = 1, EPI_I64 = 2, EPI_KDE = 3 };

struct Epi {
  int kind = EPI_INPLACE;
  void *out = nullptr;
  double div = 0.0;        // EPI_F64: divide by div when > 0
  double rdiv = 0.0;       // RN(1 / div) (div_rn)
  // EPI_KDE: out = (accumulate ? out : 0) + zfac * S, then * scale when apply_scale
  const double *zf = nullptr;  // concatenated per-axis factor tables
  int64_t zoff[FCG_MAX_DIM] = {0};
  int d = 0;
  int ax = 0;
  int64_t dims[FCG_MAX_DIM] = {0};
  int accumulate = 0;
  int apply_scale = 0;
  double scale = 1.0;
  // optional side output (axis-0 pass only): the S values of the axis-1 plane plane_idx,
  // weighted by zf_k(i_k) of the axes k >= cap_kw, stored as
  // plane_out[i0 * (dims[2] * ... * dims[d-1]) + rest] (slab carry exchange)
  double *plane_out = nullptr;
  int64_t plane_idx = -1;
  int cap_kw = FCG_MAX_DIM;
};

struct LatShape {
  int d = 0;
  int64_t dims[FCG_MAX_DIM] = {0};
  int64_t size() const {
    int64_t s = 1;
    for (int k = 0; k < d; ++k) s *= dims[k];
    return s;
  }
};

// Size (elements of T) of the chunk-carry scratch the engine may need for one pass.
int64_t scan_scratch_elems(const LatShape &s);
// Upper bound of scan_scratch_elems over every lattice shape (chunking only happens when a
// pass has fewer parallel units than ~3 x resident threads).
int64_t scan_scratch_bound();

// Scan every axis of `lat` (in place) with direction rev[k] (true = suffix sums).  The last
// processed axis (axis 0) applies `epi`.  T = int32_t or double.
template <typename T>
int scan_lattice(T *lat, const LatShape &s, const bool *rev, const Epi &epi, T *scratch,
                 cudaStream_t stream);

// Scan a single axis (used by the sweep pipeline and the dominance kernel's coarse grid).
template <typename T>
int scan_axis(T *lat, const LatShape &s, int ax, bool rev, const Epi &epi, T *scratch,
              cudaStream_t stream);

}  // namespace fcg
