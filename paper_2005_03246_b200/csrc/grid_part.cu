// Partitioned grid pipeline; see grid_part.cuh.
//
// Why: scattering 1e8 points with global atomics into a 1-2 GB lattice is random
// read-modify-write traffic (two 32-byte sectors per point, ~10x the useful bytes, measured at
// 12-16% of HBM peak).  Bucketing by plane first turns it into streaming: each CTA reads its
// bucket's records contiguously, accumulates in shared memory and writes its plane once, with
// the two in-plane scan passes (Algorithm 1's sweeps along axes d-2, d-1) fused in.
#include <math_constants.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "grid_part.cuh"
#include "tma.cuh"
#include "partition.cuh"
#include "sort.cuh"

namespace fcg {

int launch_kde_zf(const double *knots, int d, const int64_t *m, const double *c, const double *h,
                  int code, double *zf, cudaStream_t st);

namespace {

constexpr uint32_t kDead = 0xFFFFFFFFu;
// KDE record keys have <= 31 bits (plan_kde_partition); window lanes past a share's end carry
// kPadKey | lane, distinct per lane so they never form a run (which would cost scan steps)
constexpr uint32_t kPadKey = 0x80000000u;
constexpr int kPlaneThreads = 256;
constexpr int kKdeThreads = 256;
constexpr size_t kEcdfTileBytes = 96 * 1024;   // int32 tile budget (2 CTAs per SM)
constexpr size_t kKdeTileBytes = 110 * 1024;   // two fp64 row-block tiles (2 CTAs per SM)
constexpr int64_t kMinPartitionN = int64_t(1) << 20;

struct PartGeo {
  int d;
  int64_t E[FCG_MAX_DIM];      // extents of the bucketed space
  int64_t shift[FCG_MAX_DIM];  // bucket-space index = b - shift
  int64_t W, R, nrb, H;
  float inv_R;                 // 1 / R (row-block division by reciprocal + one correction)
  int ecdf;                    // 1: val = in-block cell offset; 0: val = point index
  int cell_bits;               // > 0: key = bucket << cell_bits | r_in << col_bits | col
  int col_bits;
};

// LEU: 0 / 1 = every axis counts knots < x / <= x (folded at compile time), 2 = per-axis g.le
template <int D, int LEU = 2>
__device__ __forceinline__ void part_key(const double *xi, int d, const double *kb, const BinGrid &g,
                                         const double *s_z0, const double *s_idz,
                                         const PartGeo &p, int64_t i, uint32_t &key,
                                         int32_t &val, unsigned mesh = 0u) {
  uint32_t plane = 0;
  int row = 0, col = 0;
  bool live = true;
  constexpr int DD = D > 0 ? D : FCG_MAX_DIM;
  int cnt[DD];
  bool counted = false;
  if (D > 0 && mesh == (1u << D) - 1u) {
    // every axis follows its mesh (CTA-uniform): the mesh counts of all axes first, ONE test
    // whether the point is clear of every mesh line (bin.cuh: then they are the exact counts);
    // the rare point near a line takes the verified counts below
    bool safe = true;
#pragma unroll
    for (int k = 0; k < DD; ++k) {
      const int le = LEU == 2 ? g.le[k] : LEU;
      const double t = (xi[k] - s_z0[k]) * s_idz[k];
      const int f = le ? __double2int_rd(t) : __double2int_ru(t - 1.0);
      cnt[k] = min(max(f, -1), (int)g.m[k] - 1) + 1;
      safe = safe && fabs(t - rint(t)) > kMeshSafe;  // NaN: not safe
    }
    counted = safe;
  }
  if (!counted) {
#pragma unroll
    for (int k = 0; k < DD; ++k)
      if (k < d)
        cnt[k] = knot_count(xi[k], kb + g.koff[k], (int)g.m[k], LEU == 2 ? g.le[k] : LEU,
                            s_z0[k], s_idz[k]);
  }
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    if (k < d) {
      const int c = cnt[k] - (int)p.shift[k];
      live = live && c >= 0 && c < (int)p.E[k];
      if (k < d - 2) plane = plane * (uint32_t)p.E[k] + (uint32_t)c;
      else if (k == d - 2) row = c;
      else col = c;
    }
  }
  key = kDead;
  val = (int32_t)i;
  if (live) {
    // row < 2^24: the float quotient is within one of row / R
    const int R = (int)p.R;
    int rb = __float2int_rz((float)row * p.inv_R);
    int r_in = row - rb * R;
    if (r_in < 0) {
      --rb;
      r_in += R;
    } else if (r_in >= R) {
      ++rb;
      r_in -= R;
    }
    key = plane * (uint32_t)p.nrb + (uint32_t)rb;
    if (p.ecdf) val = r_in * (int)p.W + col;
    if (p.cell_bits > 0) key = (key << p.cell_bits) | ((uint32_t)r_in << p.col_bits) | (uint32_t)col;
  }
}


// start[b] = first sorted position whose key >= b << shift, for b in [0, NB]
__global__ void bucket_start_kernel(const uint32_t *__restrict__ keys, int64_t n, int64_t NB,
                                    int shift, int32_t *__restrict__ start) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= NB;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    const int64_t bk = b << shift;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)keys[mid] < bk) lo = mid + 1;
      else hi = mid;
    }
    start[b] = (int32_t)lo;
  }
}

// In-shared-memory scans of an nr x W tile: rows along the last axis (warp per row), then
// columns along axis d-2 (segmented: G threads per column) continuing the carry row.
template <typename T>
__device__ __forceinline__ void tile_scan(T *tile, int nr, int W, bool rev_r, bool rev_c, T *carry,
                                          T *seg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // warp per row, 32 consecutive elements per step (conflict-free), shuffle scans + carry
  for (int r = warp; r < nr; r += nwarps) {
    T *row = tile + (size_t)r * W;
    T run = T(0);
    for (int jb = 0; jb < W; jb += 32) {
      const int jj = jb + lane;
      const int j = rev_c ? W - 1 - jj : jj;
      T v = jj < W ? row[j] : T(0);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      v += run;
      if (jj < W) row[j] = v;
      run = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const int G = (int)blockDim.x >= W ? (int)blockDim.x / W : 1;
  const int Rg = (nr + G - 1) / G;
  // phase A: segment totals
  for (int cc = threadIdx.x; cc < W * G; cc += blockDim.x) {
    const int c = cc % W, g = cc / W;
    T s = T(0);
    for (int q = g * Rg; q < nr && q < (g + 1) * Rg; ++q) {
      const int r = rev_r ? nr - 1 - q : q;
      s += tile[(size_t)r * W + c];
    }
    seg[(size_t)g * W + c] = s;
  }
  __syncthreads();
  // phase B: rescan with carry-in
  for (int cc = threadIdx.x; cc < W * G; cc += blockDim.x) {
    const int c = cc % W, g = cc / W;
    T run = carry[c];
    for (int gg = 0; gg < g; ++gg) run += seg[(size_t)gg * W + c];
    for (int q = g * Rg; q < nr && q < (g + 1) * Rg; ++q) {
      const int r = rev_r ? nr - 1 - q : q;
      run += tile[(size_t)r * W + c];
      tile[(size_t)r * W + c] = run;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    T s = carry[c];
    for (int g = 0; g < G; ++g) s += seg[(size_t)g * W + c];
    carry[c] = s;
  }
  __syncthreads();
}

template <typename T> struct V16 {};
template <> struct V16<double> { using vt = double2; static constexpr int V = 2; };
template <> struct V16<int32_t> { using vt = int4; static constexpr int V = 4; };

template <typename T>
__device__ __forceinline__ void v16_load(const T *p, T *r) {
  if constexpr (sizeof(T) == 8) {
    const double2 a = *reinterpret_cast<const double2 *>(p);
    r[0] = a.x; r[1] = a.y;
  } else {
    const int4 a = *reinterpret_cast<const int4 *>(p);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
  }
}
template <typename T>
__device__ __forceinline__ void v16_store(T *p, const T *r) {
  if constexpr (sizeof(T) == 8) {
    *reinterpret_cast<double2 *>(p) = make_double2(r[0], r[1]);
  } else {
    *reinterpret_cast<int4 *>(p) = make_int4(r[0], r[1], r[2], r[3]);
  }
}

// Vectorised tile scan for rows whose length is a multiple of 32 * V (V = 16 / sizeof(T)):
// every lane owns E = W / 32 consecutive elements read with 16-byte shared accesses
// (conflict-free), scans them serially, and one warp scan stitches the lanes; columns are
// walked V at a time with pointer increments (no per-element index arithmetic).
// Requires W % (32 * V) == 0 and E <= 16.
template <typename T, int EMAX>
__device__ __forceinline__ void tile_scan_vec(T *tile, int nr, int W, bool rev_r, bool rev_c,
                                              T *carry, T *seg) {
  constexpr int V = V16<T>::V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  constexpr int E = EMAX;  // W == 32 * E
  for (int r = warp; r < nr; r += nwarps) {
    T *row = tile + (size_t)r * W;
    // lane-contiguous chunk in scan order: forward [lane*E, lane*E+E), reverse mirrored
    T *chunk = rev_c ? row + (W - (lane + 1) * E) : row + lane * E;
    T v[EMAX];
#pragma unroll
    for (int e = 0; e < EMAX; e += V)
      if (e < E) v16_load<T>(chunk + e, v + e);
    T tot = T(0);
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
      if (e < E) tot += v[e];
    T incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    T run = incl - tot;
    if (!rev_c) {
#pragma unroll
      for (int e = 0; e < EMAX; ++e)
        if (e < E) { run += v[e]; v[e] = run; }
    } else {
#pragma unroll
      for (int e = EMAX - 1; e >= 0; --e)
        if (e < E) { run += v[e]; v[e] = run; }
    }
#pragma unroll
    for (int e = 0; e < EMAX; e += V)
      if (e < E) v16_store<T>(chunk + e, v + e);
  }
  __syncthreads();
  // columns, V adjacent columns per thread, G segments of rows per column group
  const int CG = W / V;
  const int G = (int)blockDim.x >= CG ? (int)blockDim.x / CG : 1;
  const int Rg = (nr + G - 1) / G;
  const long step = rev_r ? -(long)W : (long)W;
  for (int cc = threadIdx.x; cc < CG * G; cc += blockDim.x) {
    const int cgi = cc % CG, g = cc / CG;
    const int q0 = g * Rg, q1 = min(nr, (g + 1) * Rg);
    T s[V];
#pragma unroll
    for (int k = 0; k < V; ++k) s[k] = T(0);
    if (q0 < q1) {
      const T *p = tile + (size_t)(rev_r ? nr - 1 - q0 : q0) * W + cgi * V;
      for (int q = q0; q < q1; ++q, p += step) {
        T a[V];
        v16_load<T>(p, a);
#pragma unroll
        for (int k = 0; k < V; ++k) s[k] += a[k];
      }
    }
    v16_store<T>(seg + (size_t)g * W + cgi * V, s);
  }
  __syncthreads();
  for (int cc = threadIdx.x; cc < CG * G; cc += blockDim.x) {
    const int cgi = cc % CG, g = cc / CG;
    const int q0 = g * Rg, q1 = min(nr, (g + 1) * Rg);
    T run[V];
    v16_load<T>(carry + cgi * V, run);
    for (int gg = 0; gg < g; ++gg) {
      T a[V];
      v16_load<T>(seg + (size_t)gg * W + cgi * V, a);
#pragma unroll
      for (int k = 0; k < V; ++k) run[k] += a[k];
    }
    if (q0 < q1) {
      T *p = tile + (size_t)(rev_r ? nr - 1 - q0 : q0) * W + cgi * V;
      for (int q = q0; q < q1; ++q, p += step) {
        T a[V];
        v16_load<T>(p, a);
#pragma unroll
        for (int k = 0; k < V; ++k) { run[k] += a[k]; a[k] = run[k]; }
        v16_store<T>(p, a);
      }
    }
  }
  __syncthreads();
  for (int cgi = threadIdx.x; cgi < CG; cgi += blockDim.x) {
    T c[V];
    v16_load<T>(carry + cgi * V, c);
    for (int g = 0; g < G; ++g) {
      T a[V];
      v16_load<T>(seg + (size_t)g * W + cgi * V, a);
#pragma unroll
      for (int k = 0; k < V; ++k) c[k] += a[k];
    }
    v16_store<T>(carry + cgi * V, c);
  }
  __syncthreads();
}

// dispatch: compile-time lane chunk for W in {32V, 64V, 128V}, generic scan otherwise
template <typename T, int SE>
__device__ __forceinline__ void tile_scan_any(T *tile, int nr, int W, bool rev_r, bool rev_c,
                                              T *carry, T *seg) {
  if constexpr (SE > 0) tile_scan_vec<T, SE>(tile, nr, W, rev_r, rev_c, carry, seg);
  else tile_scan<T>(tile, nr, W, rev_r, rev_c, carry, seg);
}

// host: the lane chunk E (= W / 32) of the vectorised scan, 0 for the generic scan
int scan_variant(int64_t W, int V) {
  for (int e : {V, 2 * V, 4 * V})
    if (e <= 8 && W == 32 * e) return e;
  return 0;
}

template <typename T>
__device__ __forceinline__ void tile_zero(T *tile, int count) {
  constexpr int V = V16<T>::V;
  if (count % V == 0) {
    using vt = typename V16<T>::vt;
    vt z;
    memset(&z, 0, sizeof(vt));
    vt *t4 = reinterpret_cast<vt *>(tile);
    for (int i = threadIdx.x; i < count / V; i += blockDim.x) t4[i] = z;
  } else {
    for (int i = threadIdx.x; i < count; i += blockDim.x) tile[i] = T(0);
  }
}

template <typename T>
__device__ __forceinline__ void tile_store(T *__restrict__ dst, const T *tile, int64_t count) {
  // 16-byte vector stores when both sides are aligned (they are for whole planes)
  constexpr int V = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && count % V == 0) {
    const int4 *src4 = reinterpret_cast<const int4 *>(tile);
    int4 *dst4 = reinterpret_cast<int4 *>(dst);
    for (int64_t i = threadIdx.x; i < count / V; i += blockDim.x) dst4[i] = src4[i];
  } else {
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = tile[i];
  }
}

// ECDF / ESF counts: CTA per plane, row blocks in scan order.
template <int SE>
__global__ void __launch_bounds__(kPlaneThreads, 3) plane_count_kernel(
    PartGeo p, const int32_t *__restrict__ start, const int32_t *__restrict__ vals, int rev_r,
    int rev_c, int32_t *__restrict__ lat, const uint32_t *__restrict__ pkeys) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = (int)p.W, R = (int)p.R;
  const int G = (int)blockDim.x >= W ? (int)blockDim.x / W : 1;
  int32_t *tile = reinterpret_cast<int32_t *>(smem);
  int32_t *carry = tile + (size_t)R * W;
  int32_t *seg = carry + W;
  const int64_t plane = blockIdx.x;
  for (int c = threadIdx.x; c < W; c += blockDim.x) carry[c] = 0;
  for (int64_t rbi = 0; rbi < p.nrb; ++rbi) {
    const int64_t rb = rev_r ? p.nrb - 1 - rbi : rbi;
    const int64_t r0 = rb * R;
    const int nr = (int)((r0 + R <= p.H) ? R : p.H - r0);
    tile_zero<int32_t>(tile, nr * W);
    __syncthreads();
    const int64_t b = plane * p.nrb + rb;
    const int32_t q0 = start[b], q1 = start[b + 1];
    constexpr int KB = 8;
    for (int32_t qb = q0 + threadIdx.x; qb < q1; qb += KB * blockDim.x) {
      int32_t v[KB];
      if (pkeys) {  // packed keys: in-block cell r_in << col_bits | col
        const uint32_t cm = (1u << p.col_bits) - 1u;
#pragma unroll
        for (int u = 0; u < KB; ++u) {
          const int32_t q = qb + u * (int32_t)blockDim.x;
          const uint32_t kk = q < q1 ? pkeys[q] : 0u;
          v[u] = q < q1 ? (int32_t)(((kk & ((1u << p.cell_bits) - 1u)) >> p.col_bits) * (uint32_t)W +
                                    (kk & cm))
                        : -1;
        }
      } else {
#pragma unroll
        for (int u = 0; u < KB; ++u) {
          const int32_t q = qb + u * (int32_t)blockDim.x;
          v[u] = q < q1 ? vals[q] : -1;
        }
      }
#pragma unroll
      for (int u = 0; u < KB; ++u)
        if (v[u] >= 0) atomicAdd(&tile[v[u]], 1);
    }
    __syncthreads();
    tile_scan_any<int32_t, SE>(tile, nr, W, rev_r, rev_c, carry, seg);
    tile_store<int32_t>(lat + (plane * p.H + r0) * W, tile, (int64_t)nr * W);
    __syncthreads();
  }
  (void)G;
}

// KDE term group: CTA per cell-space plane.  The 2^d terms are folded in groups that share
// the signs of the leading axes (k < kz); inside a group only the in-plane factors differ, so
//   sum_t zfac_t S_t = prod_{k<kz} zf_k  x  S_lead( sum_t zf_r,t(i_r) zf_c,t(i_c) P_t )
// with P_t the term's in-plane 2-D scan (the leading-axis scans are linear and commute with
// multiplication by functions of the in-plane indices).  The CTA builds, per row direction
// (phase), the two column-direction tiles from ONE pass over its bucket's records, scans them,
// weights them by the in-plane factors and writes (phase 0) or adds (phase 1) the plane.
// Records are bucketed by full-space (M+1) row block; a phase with row shift s reads full block
// rb as cell rows [rb*Rf - s, (rb+1)*Rf - s), so every cell row block comes from one bucket.
struct KdeGroup {
  int d;
  int64_t Mr, Mc;                    // cell extents of axes d-2, d-1
  int64_t Rf, nrb;                   // full-space rows per bucket block, blocks per plane
  int64_t lead_m[FCG_MAX_DIM];       // cell extents of leading axes
  int64_t lead_s[FCG_MAX_DIM];       // their shifts (1 where delta = -1)
  int64_t lead_full[FCG_MAX_DIM];    // full (M+1) extents of leading axes
  unsigned lead_neg;                 // leading axes with delta = -1 (bit k)
  int nphase;                        // 1: row sign fixed (rneg[0]); 2: both row signs
  int rneg[2];
  double c[FCG_MAX_DIM], a[FCG_MAX_DIM];  // raw records: centre and 1/h
  const double *zr[2];               // row-axis factor table of each phase (null: factor 1)
  const double *zcp, *zcm;           // column-axis factor tables, delta_c = +1 / -1
  int cell_bits, col_bits;           // sorted key layout: bucket << cell_bits | r_in << col_bits | col
  unsigned fmask[2];                 // factored record fields multiplied into psi per phase
  int nf[2];                         // ... as a list (fast path)
  int fidx[2][FCG_MAX_DIM + 1];
};

// ---- accumulation of cell-sorted records into the two row-block tiles -------------------
// Each warp owns a contiguous share of the bucket and walks it in windows of 32 consecutive
// records.  Runs of equal keys are summed with shuffles; a run strictly inside the warp's
// share holds every record of its cell (the bucket is sorted), so it is written with a plain
// shared store, and a run reaching lane 31 is carried into the next window in registers.  Only
// the first and last run of a share may meet another warp's records and use atomics (fp64
// shared atomics are CAS loops on sm_100).
struct TileTarget {
  double *tp, *tm;
  int W, nr, rowoff, col_bits;
  uint32_t cmask, rmask;
  int swz;  // tiles use the swizzled row layout of kde_tiles_walk
};

// Row layout of the vectorised walk: 16-byte chunk ch of a row is stored at ch ^ ((ch>>3)&7),
// so the lanes' strided 16-byte accesses (E/2 chunks per lane) hit distinct banks.
__device__ __forceinline__ int swz_col(int c) { return c ^ (((c >> 4) & 7) << 1); }

__device__ __forceinline__ void tile_put(const TileTarget &T, uint32_t key, double vp, double vm,
                                         bool atomic) {
  const int cr = (int)((key >> T.col_bits) & T.rmask) + T.rowoff;
  const int col = (int)(key & T.cmask);
  if (cr < 0 || cr >= T.nr) return;
  if (col < T.W) {
    double *p = T.tp + cr * T.W + (T.swz ? swz_col(col) : col);
    if (atomic) atomicAdd(p, vp);
    else *p = vp;
  }
  if (col >= 1) {
    double *m = T.tm + cr * T.W + (T.swz ? swz_col(col - 1) : col - 1);
    if (atomic) atomicAdd(m, vm);
    else *m = vm;
  }
}

struct KdeRec {
  uint32_t key;
  double pp, pm;
};

// psi of the delta_c = +1 / -1 terms of the phase for sorted record q
__device__ __forceinline__ KdeRec kde_load(const uint32_t *__restrict__ keys,
                                           const double *__restrict__ rec, int64_t nrec,
                                           int32_t q, bool in, int factored, unsigned fmask,
                                           int mfield, int d, const double *c, const double *a,
                                           unsigned negmask) {
  KdeRec r;
  r.key = in ? keys[q] : kPadKey | (uint32_t)(threadIdx.x & 31);  // distinct dead keys
  r.pp = 0.0;
  r.pm = 0.0;
  if (!in) return r;
  if (factored) {
    double f[FCG_MAX_DIM + 1];
#pragma unroll
    for (int k = 0; k <= FCG_MAX_DIM; ++k)  // all loads issued before the product
      f[k] = ((fmask >> k) & 1) ? rec[(int64_t)k * nrec + q] : 1.0;
    const double qc = rec[(int64_t)mfield * nrec + q];
    double v = f[0];
#pragma unroll
    for (int k = 1; k <= FCG_MAX_DIM; ++k) v *= f[k];
    r.pp = v;
    r.pm = v * qc;
  } else {
    double sx = 0.0;
    for (int k = 0; k < d - 1; ++k)
      sx += (rec[(int64_t)k * nrec + q] - c[k]) * (((negmask >> k) & 1) ? -a[k] : a[k]);
    const double uc = (rec[(int64_t)(d - 1) * nrec + q] - c[d - 1]) * a[d - 1];
    const double wq = rec[(int64_t)d * nrec + q];
    r.pp = wq * exp(sx + uc);
    r.pm = wq * exp(sx - uc);
  }
  return r;
}

// Factored records: psi_+ = prod of NF fields, psi_- = psi_+ * q_c.  Raw fields of the next
// two windows are loaded ahead of the reduction of the current one (the product would
// otherwise wait on each window's loads in turn).
template <int NF>
struct RawWin {
  uint32_t key;
  double f[NF > 0 ? NF : 1];
  double qc;
};

struct AccParams {
  const uint32_t *keys;
  const double *fp[FCG_MAX_DIM + 1];  // field arrays of the sorted records (field-major)
  const double *fq;
  int32_t q0, q1;
};

template <int NF>
__device__ __forceinline__ void raw_load(RawWin<NF> &r, const uint32_t *__restrict__ keys,
                                         const double *const *fp, const double *fq, int32_t q,
                                         bool in) {
  r.key = in ? keys[q] : kPadKey | (uint32_t)(threadIdx.x & 31);  // distinct dead keys
  const int32_t qq = in ? q : 0;
#pragma unroll
  for (int j = 0; j < NF; ++j) r.f[j] = fp[j][qq];
  r.qc = fq[qq];
}

// one window: segmented run sums, carry handling, tile writes (see the comment above)
struct RunCarry {
  uint32_t key = 0xFFFFFFFFu;
  double p = 0.0, m = 0.0;
  bool first = false;
};

__device__ __forceinline__ void window_reduce(const TileTarget &T, uint32_t key, double pp,
                                              double pm, bool share_first, RunCarry &c,
                                              int lane) {
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = lane == 0 || key != prev;
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const int hl = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
  const int span = lane - hl;
  const int maxspan = __reduce_max_sync(0xffffffffu, span);
  double sp = pp, sm = pm;
  for (int o = 1; o <= maxspan; ++o) {
    const double up = __shfl_up_sync(0xffffffffu, pp, o);
    const double um = __shfl_up_sync(0xffffffffu, pm, o);
    if (o <= span) {
      sp += up;
      sm += um;
    }
  }
  const uint32_t key0 = __shfl_sync(0xffffffffu, key, 0);
  const bool cont = key0 == c.key;
  if (cont && hl == 0) {
    sp += c.p;
    sm += c.m;
  }
  if (!cont && c.key < kPadKey && lane == 0) tile_put(T, c.key, c.p, c.m, c.first);
  const bool ffirst = share_first || (cont && c.first);  // window's first run = share's first
  const bool tail = lane == 31 || ((heads >> (lane + 1)) & 1);
  if (tail && lane != 31 && key < kPadKey) tile_put(T, key, sp, sm, hl == 0 && ffirst);
  c.key = __shfl_sync(0xffffffffu, key, 31);
  c.p = __shfl_sync(0xffffffffu, sp, 31);
  c.m = __shfl_sync(0xffffffffu, sm, 31);
  const int hl31 = __shfl_sync(0xffffffffu, hl, 31);
  c.first = hl31 == 0 && ffirst;
}

template <int NF, int DEPTH = (NF <= 2 ? 2 : 1)>
__device__ __forceinline__ void accumulate_factored(const TileTarget &T, const AccParams &P,
                                                    int wb, int we, int lane) {
  RunCarry c;
  RawWin<NF> buf[DEPTH];  // ring of windows in flight (static indices: k is unrolled)
  const double *fp[NF > 0 ? NF : 1];
#pragma unroll
  for (int j = 0; j < NF; ++j) fp[j] = P.fp[j];
  auto ld = [&](RawWin<NF> &r, int win) {
    const int32_t q = P.q0 + win * 32 + lane;
    raw_load<NF>(r, P.keys, fp, P.fq, q, q < P.q1);
  };
#pragma unroll
  for (int k = 0; k < DEPTH; ++k)
    if (wb + k < we) ld(buf[k], wb + k);
  for (int win = wb; win < we; win += DEPTH) {
#pragma unroll
    for (int k = 0; k < DEPTH; ++k) {
      if (win + k < we) {  // warp-uniform
        const RawWin<NF> cur = buf[k];
        if (win + k + DEPTH < we) ld(buf[k], win + k + DEPTH);
        double pp = 1.0;
#pragma unroll
        for (int j = 0; j < NF; ++j) pp *= cur.f[j];
        if (cur.key >= kPadKey) pp = 0.0;
        window_reduce(T, cur.key, pp, pp * cur.qc, win + k == wb, c, lane);
      }
    }
  }
  if (c.key < kPadKey && lane == 0) tile_put(T, c.key, c.p, c.m, true);
}

// In-plane 2-D scan of the two row-block tiles fused with the factor weighting and the plane
// write, for W == 32 * E: warp g walks row segment g (in scan order) with each lane owning E
// consecutive columns of both tiles in registers.  U accumulates raw column sums (carry of the
// previous row blocks + earlier segments + rows so far), so each row's 2-D scan value is the
// row-direction scan of U (serial over the lane's E columns, one warp scan across lanes):
//   delta_c = +1 tile: prefix over columns, delta_c = -1 tile: suffix.
// Every tile element is read twice (segment sums, walk) and zeroed on the walk, ready for the
// next row block.
template <int E>
__device__ __forceinline__ void kde_tiles_walk(double *tp, double *tm, double *cp, double *cm,
                                               double *segp, double *segm, int nr, int rneg,
                                               const double *zr, const double *zcp_r,
                                               const double *zcm_r, double *g, int ph) {
  constexpr int W = 32 * E, C = E / 2;  // C 16-byte chunks per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int c0 = lane * E;
  int pc[C];  // physical (swizzled) double offsets of the lane's chunks
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int ch = lane * C + j;
    pc[j] = (ch ^ ((ch >> 3) & 7)) * 2;
  }
  const int Rg = (nr + nw - 1) / nw;
  const int q0 = warp * Rg, q1 = min(nr, q0 + Rg);
  // pass 1: raw column sums of this warp's segment
  {
    double sp[E], sm[E];
#pragma unroll
    for (int e = 0; e < E; ++e) sp[e] = sm[e] = 0.0;
    for (int q = q0; q < q1; ++q) {
      const int r = rneg ? nr - 1 - q : q;
#pragma unroll
      for (int j = 0; j < C; ++j) {
        const double2 u = *reinterpret_cast<const double2 *>(tp + r * W + pc[j]);
        const double2 v = *reinterpret_cast<const double2 *>(tm + r * W + pc[j]);
        sp[2 * j] += u.x; sp[2 * j + 1] += u.y;
        sm[2 * j] += v.x; sm[2 * j + 1] += v.y;
      }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      *reinterpret_cast<double2 *>(segp + warp * W + pc[j]) = make_double2(sp[2 * j], sp[2 * j + 1]);
      *reinterpret_cast<double2 *>(segm + warp * W + pc[j]) = make_double2(sm[2 * j], sm[2 * j + 1]);
    }
  }
  __syncthreads();
  // pass 2: walk the segment with the column sums of everything before it
  double up[E], um[E];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const double2 a = *reinterpret_cast<const double2 *>(cp + pc[j]);
    const double2 b = *reinterpret_cast<const double2 *>(cm + pc[j]);
    up[2 * j] = a.x; up[2 * j + 1] = a.y;
    um[2 * j] = b.x; um[2 * j + 1] = b.y;
  }
  for (int w = 0; w < warp; ++w) {
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const double2 a = *reinterpret_cast<const double2 *>(segp + w * W + pc[j]);
      const double2 b = *reinterpret_cast<const double2 *>(segm + w * W + pc[j]);
      up[2 * j] += a.x; up[2 * j + 1] += a.y;
      um[2 * j] += b.x; um[2 * j + 1] += b.y;
    }
  }
  double zp[E], zm[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    zp[e] = zcp_r[c0 + e];
    zm[e] = zcm_r[c0 + e];
  }
  const double2 zero2 = make_double2(0.0, 0.0);
  for (int q = q0; q < q1; ++q) {
    const int r = rneg ? nr - 1 - q : q;
    double2 *o = reinterpret_cast<double2 *>(g + (int64_t)r * W + c0);
    const double zrv = zr ? __ldg(zr + r) : 1.0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      double2 *a = reinterpret_cast<double2 *>(tp + r * W + pc[j]);
      double2 *b = reinterpret_cast<double2 *>(tm + r * W + pc[j]);
      const double2 u = *a, v = *b;
      *a = zero2;
      *b = zero2;
      up[2 * j] += u.x; up[2 * j + 1] += u.y;
      um[2 * j] += v.x; um[2 * j + 1] += v.y;
    }
    double tsp = 0.0, tsm = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      tsp += up[e];
      tsm += um[e];
    }
    double ip = tsp, im = tsm;  // inclusive prefix (p) / suffix (m) of the lane totals
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double xp = __shfl_up_sync(0xffffffffu, ip, off);
      const double xm = __shfl_down_sync(0xffffffffu, im, off);
      if (lane >= off) ip += xp;
      if (lane + off < 32) im += xm;
    }
    double sp[E], sm[E];
    double run = ip - tsp;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      run += up[e];
      sp[e] = run;
    }
    run = im - tsm;
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
      run += um[e];
      sm[e] = run;
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int e = 2 * j;
      double2 v;
      v.x = zrv * (zp[e] * sp[e] + zm[e] * sm[e]);
      v.y = zrv * (zp[e + 1] * sp[e + 1] + zm[e + 1] * sm[e + 1]);
      if (ph > 0) {
        const double2 old = o[j];
        v.x += old.x;
        v.y += old.y;
      }
      o[j] = v;
    }
  }
  __syncthreads();
  // carry for the next row block: column sums through this block (same swizzled layout)
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    double a = cp[c], b = cm[c];
    for (int w = 0; w < nw; ++w) {
      a += segp[w * W + c];
      b += segm[w * W + c];
    }
    cp[c] = a;
    cm[c] = b;
  }
  __syncthreads();
}

template <int SE>
__global__ void __launch_bounds__(kKdeThreads, 2) plane_kde_group_kernel(
    KdeGroup t, const int32_t *__restrict__ start, const double *__restrict__ rec, int64_t nrec,
    const uint32_t *__restrict__ keys, int factored, double *__restrict__ lat) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = (int)t.Mc, H = (int)t.Mr, Rf = (int)t.Rf;
  double *tp = reinterpret_cast<double *>(smem);  // delta_c = +1 tile
  double *tm = tp + (size_t)Rf * W;               // delta_c = -1 tile
  double *cp = tm + (size_t)Rf * W;
  double *cm = cp + W;
  double *zc = cm + W;                            // interleaved (zcp, zcm) per column (SE == 0)
  double *seg = zc + 2 * W;                       // SE > 0: [2][nwarps][W]; else scan segments
  const int d = t.d;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t cplane = blockIdx.x;
  int64_t rem = cplane, fplane = 0, mul = 1;
  for (int k = d - 3; k >= 0; --k) {
    const int64_t i = rem % t.lead_m[k];
    rem /= t.lead_m[k];
    fplane += (i + t.lead_s[k]) * mul;
    mul *= t.lead_full[k];
  }
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    zc[2 * c] = t.zcp[c];
    zc[2 * c + 1] = t.zcm[c];
  }
  if (SE > 0) {  // the walk re-zeroes the tiles as it reads them
    tile_zero<double>(tp, 2 * Rf * W);
  }
  double *plane_out = lat + cplane * H * W;
  const int kr = d - 2, kcol = d - 1;
  const uint32_t cmask = (1u << t.col_bits) - 1u, rmask = (1u << (t.cell_bits - t.col_bits)) - 1u;
  for (int ph = 0; ph < t.nphase; ++ph) {
    const int rneg = t.rneg[ph];
    const int sr = rneg;
    const double *zr = t.zr[ph];
    for (int c = threadIdx.x; c < W; c += blockDim.x) {
      cp[c] = 0.0;
      cm[c] = 0.0;
    }
    for (int64_t rbi = 0; rbi < t.nrb; ++rbi) {
      const int64_t rb = rneg ? t.nrb - 1 - rbi : rbi;
      const int lo = (int)(rb * Rf - sr), hi = lo + Rf;
      const int clo = lo < 0 ? 0 : lo, chi = hi > H ? H : hi;
      if (chi <= clo) continue;
      const int nr = chi - clo;
      if (SE == 0) {
        tile_zero<double>(tp, nr * W);
        tile_zero<double>(tm, nr * W);
      }
      __syncthreads();
      const int64_t b = fplane * t.nrb + rb;
      const int32_t q0 = start[b], q1 = start[b + 1];
      const int rowoff = (int)(rb * Rf) - sr - clo;  // tile row = r_in + rowoff
      TileTarget T;
      T.tp = tp;
      T.tm = tm;
      T.W = W;
      T.nr = nr;
      T.rowoff = rowoff;
      T.col_bits = t.col_bits;
      T.cmask = cmask;
      T.rmask = rmask;
      T.swz = SE > 0;
      const int nwin = (q1 - q0 + 31) >> 5;
      const int per = (nwin + nw - 1) / nw;
      const int wb = warp * per, we = min(nwin, wb + per);
      const int nf = factored ? t.nf[ph] : 0;
      if (nf >= 1 && nf <= 5) {
        AccParams P;
        P.keys = keys;
        for (int j = 0; j < nf; ++j) P.fp[j] = rec + (int64_t)t.fidx[ph][j] * nrec;
        P.fq = rec + (int64_t)(1 + kcol) * nrec;
        P.q0 = q0;
        P.q1 = q1;
        switch (nf) {
          case 1: accumulate_factored<1>(T, P, wb, we, lane); break;
          case 2: accumulate_factored<2>(T, P, wb, we, lane); break;
          case 3: accumulate_factored<3>(T, P, wb, we, lane); break;
          case 4: accumulate_factored<4>(T, P, wb, we, lane); break;
          default: accumulate_factored<5>(T, P, wb, we, lane); break;
        }
      } else {  // raw records (or many factors): product / exp at load time
        const unsigned negmask = t.lead_neg | (rneg ? 1u << kr : 0u);
        RunCarry c;
        for (int win = wb; win < we; ++win) {
          const int32_t q = q0 + win * 32 + lane;
          const KdeRec cur = kde_load(keys, rec, nrec, q, q < q1, factored, t.fmask[ph], 1 + kcol,
                                      d, t.c, t.a, negmask);
          window_reduce(T, cur.key, cur.pp, cur.pm, win == wb, c, lane);
        }
        if (c.key < kPadKey && lane == 0) tile_put(T, c.key, c.p, c.m, true);
      }
      __syncthreads();
      double *g = plane_out + (int64_t)clo * W;
      if constexpr (SE > 0) {
        kde_tiles_walk<SE>(tp, tm, cp, cm, seg, seg + nw * W, nr, rneg, zr ? zr + clo : nullptr, t.zcp, t.zcm, g,
                           ph);
      } else {
        tile_scan<double>(tp, nr, W, rneg, false, cp, seg);
        tile_scan<double>(tm, nr, W, rneg, true, cm, seg);
        // weight by the in-plane factors and write / accumulate this block's rows of the plane
        for (int i = threadIdx.x; i < nr * W; i += blockDim.x) {
          const int r = i / W, c = i - r * W;
          double v = (zr ? __ldg(zr + clo + r) : 1.0) * (zc[2 * c] * tp[i] + zc[2 * c + 1] * tm[i]);
          if (ph > 0) v += g[i];
          g[i] = v;
        }
        __syncthreads();
      }
    }
  }
}

// ---- all term groups in one plane pass (d = 3, 4; factored records) ----------------------
// The groups (leading-axis sign patterns g) differ only in which full-space plane feeds an
// output plane (shift s_g along each leading axis) and in the leading factors q_k of psi.  A
// CTA therefore owns one FULL-space plane F and, from one pass over its bucket's records per
// row sign, builds the column-sign tile pairs of every group (output plane F - s_g), so the
// records are streamed 2 times instead of 2 * 2^(d-2).  Warp g walks group g's tile pair with
// the raw column sums kept in registers across the row blocks (no segment pass), and writes
// the weighted rows of the group's lattice.
constexpr int kAllThreads = 128;
constexpr size_t kAllTileBytes = 55 * 1024;  // 4 CTAs per SM
// Tile layout of the all-groups kernel: 2 NG tiles (group g: column sign + at 2g, - at 2g+1) of
// rows RS = W + 2 fp64 apart and TS fp64 apart, so a row starts 16 bytes further round the banks
// than the row above it and a tile (TS / 2 odd in 16-byte units) likewise: the horizontal
// pre-scan, where 8 consecutive lanes walk 8 different (tile, row) sequences in lock step, and
// the walk, where the lanes read one row's consecutive 16-byte chunks, are both conflict-free
// without an index swizzle.
__host__ __device__ constexpr int all_tile_rows(int ng, int64_t w) {
  return (int)(((int64_t)(kAllTileBytes / (16 * (size_t)ng)) - 2) / (w + 2));
}
__host__ __device__ constexpr int all_tile_stride(int ng, int64_t w) {
  return all_tile_rows(ng, w) * (int)(w + 2) + 2 * (1 - (all_tile_rows(ng, w) & 1));
}

struct KdeAll {
  int d, nlead;
  int64_t Mr, Mc, Rf, nrb;
  int64_t lead_m[FCG_MAX_DIM];
  int cell_bits, col_bits;
  int row_split;              // 1: each row sign has its own lattice (slab planes at d = 3)
  const double *zr_pos, *zr_neg, *zc_pos, *zc_neg;
  double *lat[16];            // output lattice of (group, row sign) -> lat[row_split ? 2g+ph : g]
};

template <int NG>
struct AllVals {
  double v[2 * NG];  // (psi_+, psi_-) per group
};

// 32-bit shared-window stores / loads (no generic-address materialisation per access)
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_f64x2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}

// One run sum into every group's tile pair (raw cell values; the column sign - tile holds the
// cell at column col - 1).  Tiles of groups whose output plane does not exist are written too
// and simply never read (the walk re-zeroes every tile), which keeps the stores unpredicated.
template <int NG, int W, int TSB>
__device__ __forceinline__ void all_put(uint32_t sbase, int nr, int rowoff, int col_bits,
                                        uint32_t rmask, uint32_t cmask, uint32_t key,
                                        const AllVals<NG> &a) {
  const int cr = (int)((key >> col_bits) & rmask) + rowoff;
  const int col = (int)(key & cmask);
  if (cr < 0 || cr >= nr) return;
  // columns XOR-swizzled by 16-byte chunk within aligned 16-column groups: a window's lanes span
  // ~90 columns of a row, and columns 16 apart would otherwise share a bank pair
  const uint32_t rowa = sbase + (uint32_t)(cr * (W + 2)) * 8u;
  if (col < W) {
    const uint32_t ap = rowa + (uint32_t)swz_col(col) * 8u;
#pragma unroll
    for (int g = 0; g < NG; ++g) sts_f64(ap + 2 * g * TSB, a.v[2 * g]);
  }
  if (col >= 1) {
    const uint32_t am = rowa + (uint32_t)swz_col(col - 1) * 8u + TSB;
#pragma unroll
    for (int g = 0; g < NG; ++g) sts_f64(am + 2 * g * TSB, a.v[2 * g + 1]);
  }
}

// Warp shares of every bucket, aligned to run boundaries (no run of equal keys straddles two
// warps): bounds[b * (nw + 1) + w] = first record of warp w's share of bucket b.  Computed once
// for all buckets so the plane kernel reads two numbers instead of searching the keys.
__global__ void share_bounds_kernel(const uint32_t *__restrict__ keys,
                                    const int32_t *__restrict__ start, int64_t NB, int nw,
                                    int32_t *__restrict__ bounds) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < NB * (nw + 1);
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / (nw + 1);
    const int w = (int)(t - b * (nw + 1));
    const int32_t q0 = start[b], q1 = start[b + 1];
    const int32_t per = (q1 - q0 + nw - 1) / nw;
    int32_t p = q0 + w * per;
    if (p > q1) p = q1;
    if (p > q0 && p < q1) {
      const uint32_t k0 = keys[p - 1];
      while (p < q1 && keys[p] == k0) ++p;
    }
    bounds[t] = p;
  }
}

template <int E, int NG>
__global__ void __launch_bounds__(kAllThreads, 4) plane_kde_all_kernel(
    KdeAll t, const int32_t *__restrict__ bounds, const double *__restrict__ rec, int64_t nrec,
    const uint32_t *__restrict__ keys) {
  constexpr int W = 32 * E, C = E / 2;
  constexpr int RS = W + 2;                      // row stride (fp64)
  constexpr int TS = all_tile_stride(NG, W);     // tile stride (fp64); Rf <= all_tile_rows
  constexpr int TSB = TS * (int)sizeof(double);
  static_assert(NG * all_tile_rows(NG, W) <= 64, "pre-scan needs a lane per (group, row) and direction");
  extern __shared__ __align__(16) unsigned char smem[];
  double *tiles = reinterpret_cast<double *>(smem);  // [2 NG][TS] tiles, RS-strided rows
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const int Rf = (int)t.Rf, H = (int)t.Mr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int d = t.d, kr = d - 2, kcol = d - 1;
  // full-space leading indices of this CTA's plane, and each group's output plane
  constexpr int NL = NG == 4 ? 2 : 1;  // leading axes (t.nlead = log2 NG)
  int64_t fidx[NL];
  // Launch order: interior planes first, the boundary planes (first / last index along a leading
  // axis: fewer valid groups, the last layer holds no records) at the end, so the kernel's tail
  // is made of its cheapest CTAs.
  if (NL == 2) {
    const int64_t n0 = t.lead_m[0] + 1, n1 = t.lead_m[1] + 1;
    const int64_t ni = (n0 - 2) * (n1 - 2);
    int64_t e = blockIdx.x;
    if (n0 < 3 || n1 < 3) {
      fidx[0] = e / n1;
      fidx[NL - 1] = e % n1;
    } else if (e < ni) {
      fidx[0] = 1 + e / (n1 - 2);
      fidx[NL - 1] = 1 + e % (n1 - 2);
    } else {
      e -= ni;
      if (e < 2 * n1) {  // the first and the last row
        fidx[0] = e < n1 ? 0 : n0 - 1;
        fidx[NL - 1] = e % n1;
      } else {           // the first and the last column of the rows between
        e -= 2 * n1;
        fidx[0] = 1 + e / 2;
        fidx[NL - 1] = (e & 1) ? n1 - 1 : 0;
      }
    }
  } else {
    const int64_t n0 = t.lead_m[0] + 1;
    const int64_t e = blockIdx.x;
    fidx[0] = n0 < 3 ? e : (e < n0 - 2 ? 1 + e : (e == n0 - 2 ? 0 : n0 - 1));
  }
  unsigned vmask = 0;
  int64_t oplane[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    bool ok = true;
    int64_t pidx = 0;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int64_t i = fidx[k] - ((g >> k) & 1);
      ok = ok && i >= 0 && i < t.lead_m[k];
      pidx = pidx * t.lead_m[k] + i;
    }
    oplane[g] = pidx;
    if (ok) vmask |= 1u << g;
  }
  if (vmask == 0) return;  // uniform
  int64_t fplane = 0;
#pragma unroll
  for (int k = 0; k < NL; ++k) fplane = fplane * (t.lead_m[k] + 1) + fidx[k];
  tile_zero<double>(tiles, 2 * NG * TS);
  const uint32_t cmask = (1u << t.col_bits) - 1u, rmask = (1u << (t.cell_bits - t.col_bits)) - 1u;
  // walk ownership: lane l holds the column pairs (2 l, 2 l + 1) + 64 j, j < C, so a warp's
  // accesses of one row are consecutive 16-byte chunks (tiles and the plane alike)
  double zp[E], zm[E];
#pragma unroll
  for (int j = 0; j < C; ++j) {
    const int c = 64 * j + 2 * lane;
    zp[2 * j] = t.zc_pos[c];
    zp[2 * j + 1] = t.zc_pos[c + 1];
    zm[2 * j] = t.zc_neg[c];
    zm[2 * j + 1] = t.zc_neg[c + 1];
  }
  // field pointers: A, q_lead, q_row, q_col (factored records)
  const double *fA = rec, *fr = rec + (int64_t)(1 + kr) * nrec, *fc = rec + (int64_t)(1 + kcol) * nrec;
  const double *fq0 = rec + nrec, *fq1 = rec + 2 * nrec;
  // this warp's output plane per row sign (selected with compile-time indices so oplane stays in
  // registers)
  double *gbase0 = nullptr, *gbase1 = nullptr;
#pragma unroll
  for (int gg = 0; gg < NG; ++gg)
    if (gg == warp) {
      gbase0 = t.lat[t.row_split ? 2 * gg : gg] + oplane[gg] * H * W;
      gbase1 = t.lat[t.row_split ? 2 * gg + 1 : gg] + oplane[gg] * H * W;
    }
  for (int ph = 0; ph < 2; ++ph) {
    const int rneg = ph, sr = ph;
    const double *zr = t.row_split ? nullptr : (rneg ? t.zr_neg : t.zr_pos);
    double up[E], um[E];  // this warp's group: raw column sums through the rows walked so far
#pragma unroll
    for (int e = 0; e < E; ++e) up[e] = um[e] = 0.0;
    for (int64_t rbi = 0; rbi < t.nrb; ++rbi) {
      const int64_t rb = rneg ? t.nrb - 1 - rbi : rbi;
      const int lo = (int)(rb * Rf - sr), hi = lo + Rf;
      const int clo = lo < 0 ? 0 : lo, chi = hi > H ? H : hi;
      if (chi <= clo) continue;
      const int nr = chi - clo;
      const int rowoff = (int)(rb * Rf) - sr - clo;
      __syncthreads();  // the previous block's walk has re-zeroed the tiles
      // L2 prefetch of the next row block's records and (second row sign) of the plane rows its
      // walk reads back, so their DRAM latency is off the next block's critical path
      if (warp == nw - 1 && lane < 8 + NG) {
        int nph = ph;
        int64_t nrbi = rbi + 1;
        if (nrbi >= t.nrb) {
          nph = ph + 1;
          nrbi = 0;
        }
        if (nph < 2) {
          const int64_t rbn = nph ? t.nrb - 1 - nrbi : nrbi;
          const int64_t bn = fplane * t.nrb + rbn;
          if (lane < 6) {
            const int32_t a0 = bounds[bn * (nw + 1)], a1 = bounds[bn * (nw + 1) + nw];
            const size_t cnt = (size_t)(a1 - a0);
            if (lane == 0) l2_prefetch(keys + a0, cnt * sizeof(uint32_t));
            else if (lane == 1) l2_prefetch(fA + a0, cnt * sizeof(double));
            else if (lane == 2) l2_prefetch(fc + a0, cnt * sizeof(double));
            else if (lane == 3 && t.nlead > 0) l2_prefetch(fq0 + a0, cnt * sizeof(double));
            else if (lane == 4 && t.nlead > 1) l2_prefetch(fq1 + a0, cnt * sizeof(double));
            else if (lane == 5 && nph) l2_prefetch(fr + a0, cnt * sizeof(double));
          } else if (lane >= 8 && nph && !t.row_split) {
            const int g = lane - 8;
            const int nlo = (int)(rbn * Rf - nph), nclo = nlo < 0 ? 0 : nlo;
            const int nchi = nlo + Rf > H ? H : nlo + Rf;
            const double *lp = nullptr;
#pragma unroll
            for (int gg = 0; gg < NG; ++gg)
              if (gg == g) lp = t.lat[gg] + oplane[gg] * H * W;
            if (((vmask >> g) & 1) && nchi > nclo)
              l2_prefetch(lp + (int64_t)nclo * W, (size_t)(nchi - nclo) * W * sizeof(double));
          }
        }
      }
      {
        // warp shares aligned to run boundaries (share_bounds_kernel): every run of equal keys
        // is complete inside one share, so all tile writes are plain stores
        const int64_t b = fplane * t.nrb + rb;
        const int32_t sb = bounds[b * (nw + 1) + warp], se = bounds[b * (nw + 1) + warp + 1];
        uint32_t ckey = 0xFFFFFFFFu;
        AllVals<NG> cv;
#pragma unroll
        for (int i = 0; i < 2 * NG; ++i) cv.v[i] = 0.0;
        // raw fields of the next window are loaded before this one is reduced
        struct Raw {
          uint32_t key;
          double A, qc, q0, q1, qr;
        };
        auto load = [&](Raw &r, int32_t qb) {
          const int32_t q = qb + lane;
          const bool in = q < se;
          const int32_t qq = in ? q : sb;
          r.key = in ? keys[q] : kPadKey | (uint32_t)lane;  // padding: distinct dead keys
          r.A = fA[qq];
          r.qc = fc[qq];
          r.q0 = t.nlead > 0 ? fq0[qq] : 1.0;
          r.q1 = t.nlead > 1 ? fq1[qq] : 1.0;
          r.qr = rneg ? fr[qq] : 1.0;
        };
        Raw nx;
        if (sb < se) load(nx, sb);
        for (int32_t qb = sb; qb < se; qb += 32) {
          const Raw cur = nx;
          const bool more = qb + 32 < se;  // warp-uniform
          if (more) load(nx, qb + 32);
          const uint32_t key = cur.key;
          const double qcv = cur.qc, q0v = cur.q0, q1v = cur.q1;
          AllVals<NG> a;
          const bool valid = key < kPadKey;
          const double base = valid ? cur.A * cur.qr : 0.0;
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            double v = base;
            if (g & 1) v *= q0v;
            if (g & 2) v *= q1v;
            a.v[2 * g] = v;
            a.v[2 * g + 1] = v * qcv;
          }
          // segmented run sums over the window (see window_reduce)
          const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
          const bool head = lane == 0 || key != prev;
          const unsigned heads = __ballot_sync(0xffffffffu, head);
          const int hl = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
          const int span = lane - hl;
          const int maxspan = __reduce_max_sync(0xffffffffu, span);
          // log-step segmented scan (Hillis-Steele bounded by the run head), only as many
          // steps as the longest run needs
          AllVals<NG> sv = a;
          for (int o = 1; o <= maxspan; o <<= 1) {
#pragma unroll
            for (int i = 0; i < 2 * NG; ++i) {
              const double u = __shfl_up_sync(0xffffffffu, sv.v[i], o);
              if (lane - o >= hl) sv.v[i] += u;
            }
          }
          // a run carried in from the previous window continues in this window's first run
          if (ckey != 0xFFFFFFFFu && hl == 0) {
#pragma unroll
            for (int i = 0; i < 2 * NG; ++i) sv.v[i] += cv.v[i];
          }
          // lane 31's run ends here unless the next window starts with the same key (the
          // prefetched next window tells), so only a continuing run is carried
          const uint32_t nk0 = __shfl_sync(0xffffffffu, more ? nx.key : kPadKey, 0);
          const uint32_t k31 = __shfl_sync(0xffffffffu, key, 31);
          const bool cont_out = k31 < kPadKey && k31 == nk0;  // warp-uniform
          const bool tail = lane == 31 ? !cont_out : ((heads >> (lane + 1)) & 1);
          if (tail && valid)
            all_put<NG, W, TSB>(sbase, nr, rowoff, t.col_bits, rmask, cmask, key, sv);
          ckey = 0xFFFFFFFFu;
          if (cont_out) {
            ckey = k31;
#pragma unroll
            for (int i = 0; i < 2 * NG; ++i) cv.v[i] = __shfl_sync(0xffffffffu, sv.v[i], 31);
          }
        }
      }
      __syncthreads();
      // horizontal pre-scan of every tile row in place: warps of even index run the column
      // sign + tiles (inclusive prefix), odd ones the - tiles (inclusive suffix); lane q of a
      // direction owns (group q % NG, row q / NG).  Chunks are loaded 8 at a time ahead of the
      // dependent adds.
      {
        const int dir = warp & 1;
        const int q = (warp >> 1) * 32 + lane;
        const int gq = q % NG, r = q / NG;
        constexpr int SPAN = W;
        if (r < nr) {
          const uint32_t ra = sbase + (uint32_t)((2 * gq + dir) * TS + r * RS) * 8u;
          double run = 0.0;
          if (dir == 0) {
#pragma unroll
            for (int b = 0; b < SPAN / 16; ++b) {
              double2 v[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) v[k] = lds_f64x2(ra + swz_col(16 * b + 2 * k) * 8);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                v[k].x += run;
                v[k].y += v[k].x;
                run = v[k].y;
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) sts_f64x2(ra + swz_col(16 * b + 2 * k) * 8, v[k]);
            }
          } else {
#pragma unroll
            for (int b = 0; b < SPAN / 16; ++b) {
              double2 v[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) v[k] = lds_f64x2(ra + swz_col(SPAN - 2 - 16 * b - 2 * k) * 8);
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                v[k].y += run;
                v[k].x += v[k].y;
                run = v[k].x;
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) sts_f64x2(ra + swz_col(SPAN - 2 - 16 * b - 2 * k) * 8, v[k]);
            }
          }
        }
      }
      __syncthreads();
      // walk: warp g owns group g's tile pair; the rows are already prefix-summed along the
      // columns, so the 2-D prefix is a per-column running sum kept in registers across blocks
      if (warp < NG) {
        const int g = warp;
        const uint32_t tp = sbase + (uint32_t)(2 * g) * TSB, tm = tp + TSB;
        int cj[C];  // this lane's (swizzled) column pairs
#pragma unroll
        for (int j = 0; j < C; ++j) cj[j] = swz_col(64 * j + 2 * lane);
        const bool wr = (vmask >> g) & 1;
        double *gp = wr ? (ph ? gbase1 : gbase0) + (int64_t)clo * W : nullptr;
        const bool rmw = ph > 0 && !t.row_split;
        const double2 zero2 = make_double2(0.0, 0.0);
        constexpr int RMAX = all_tile_rows(NG, W);
        if constexpr (RMAX <= 8) {  // few rows per block: all of them unrolled, loads up front
          // every row's read-back plane values and row factor in flight at once
          double2 oldr[RMAX][C];
          double zrr[RMAX];
  #pragma unroll
          for (int qr = 0; qr < RMAX; ++qr) {
            const int r = rneg ? nr - 1 - qr : qr;
            const bool in = qr < nr && wr;
            zrr[qr] = (in && zr) ? __ldg(zr + clo + r) : 1.0;
  #pragma unroll
            for (int j = 0; j < C; ++j)
              oldr[qr][j] = (in && rmw) ? reinterpret_cast<const double2 *>(gp + (int64_t)r * W + 2 * lane)[32 * j]
                                        : zero2;
          }
  #pragma unroll
          for (int qr = 0; qr < RMAX; ++qr) {
            if (qr < nr) {
              const int r = rneg ? nr - 1 - qr : qr;
  #pragma unroll
              for (int j = 0; j < C; ++j) {
                const uint32_t o = (uint32_t)(r * RS + cj[j]) * 8u;
                const double2 a = lds_f64x2(tp + o), b = lds_f64x2(tm + o);
                sts_f64x2(tp + o, zero2);
                sts_f64x2(tm + o, zero2);
                up[2 * j] += a.x; up[2 * j + 1] += a.y;
                um[2 * j] += b.x; um[2 * j + 1] += b.y;
              }
              if (wr) {  // warp-uniform
                double2 *o = reinterpret_cast<double2 *>(gp + (int64_t)r * W + 2 * lane);
  #pragma unroll
                for (int j = 0; j < C; ++j) {
                  const int e = 2 * j;
                  double2 v;
                  v.x = zrr[qr] * (zp[e] * up[e] + zm[e] * um[e]) + oldr[qr][j].x;
                  v.y = zrr[qr] * (zp[e + 1] * up[e + 1] + zm[e + 1] * um[e + 1]) + oldr[qr][j].y;
                  o[32 * j] = v;
                }
              }
            }
          }
        } else {  // many rows: one row of look-ahead (keeps the registers in budget)
          double2 na[C], nb[C], nold[C];  // next row: tiles and (accumulate pass) plane values
          auto fetch = [&](int qr) {
            const int r = rneg ? nr - 1 - qr : qr;
  #pragma unroll
            for (int j = 0; j < C; ++j) {
              na[j] = lds_f64x2(tp + (uint32_t)(r * RS + cj[j]) * 8u);
              nb[j] = lds_f64x2(tm + (uint32_t)(r * RS + cj[j]) * 8u);
              nold[j] = (wr && rmw) ? reinterpret_cast<const double2 *>(gp + (int64_t)r * W + 2 * lane)[32 * j]
                                    : zero2;
            }
          };
          fetch(0);
          for (int qr = 0; qr < nr; ++qr) {
            const int r = rneg ? nr - 1 - qr : qr;
            double2 ca[C], cb[C], old[C];
  #pragma unroll
            for (int j = 0; j < C; ++j) {
              ca[j] = na[j];
              cb[j] = nb[j];
              old[j] = nold[j];
            }
            if (qr + 1 < nr) fetch(qr + 1);
  #pragma unroll
            for (int j = 0; j < C; ++j) {
              sts_f64x2(tp + (uint32_t)(r * RS + cj[j]) * 8u, zero2);
              sts_f64x2(tm + (uint32_t)(r * RS + cj[j]) * 8u, zero2);
              up[2 * j] += ca[j].x; up[2 * j + 1] += ca[j].y;
              um[2 * j] += cb[j].x; um[2 * j + 1] += cb[j].y;
            }
            if (!wr) continue;  // warp-uniform
            const double zrv = zr ? __ldg(zr + clo + r) : 1.0;
            double2 *o = reinterpret_cast<double2 *>(gp + (int64_t)r * W + 2 * lane);
  #pragma unroll
            for (int j = 0; j < C; ++j) {
              const int e = 2 * j;
              double2 v;
              v.x = zrv * (zp[e] * up[e] + zm[e] * um[e]);
              v.y = zrv * (zp[e + 1] * up[e + 1] + zm[e + 1] * um[e + 1]);
              if (rmw) {
                v.x += old[j].x;
                v.y += old[j].y;
              }
              o[32 * j] = v;
            }
          }
        }
      }
    }
  }
}

// KDE records, built in the coarse partition pass (partition.cuh) from coalesced reads of x, w:
//   factored (f != 0): fields (A, q_0..q_{d-1}) with A = w e^{sum_k u_k}, q_k = e^{-2 u_k},
//                      u_k = (x_k - c_k) / h_k, so a term's psi = A * prod_{k: delta_k=-1} q_k;
//   raw:               fields (x_0..x_{d-1}, w) and psi = w e^{sum_k delta_k u_k}.
// The factored form is used only when sum_k max|u_k| <= 600, which keeps every partial
// product inside e^{+-600} (fp64 overflows past e^709).  The pass groups the records by the
// top 8 bits of the sorted key (256 coarse buckets of ~n/256 records) and writes them
// record-major next to their keys; the full sort then only moves (key, slot) pairs and the
// final gather reads each coarse bucket from L2 (sorted order walks the buckets in turn)
// instead of paying a DRAM line per random record.
template <int D>
struct KdeBuild {
  static constexpr int kD = D;
  int factored;
  PsiParams pp;
  __device__ __forceinline__ void operator()(const double *xi, double wi, double *r) const {
    if (factored) {
      double su = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double u = (xi[k] - pp.c[k]) * pp.a[k];  // a_k = 1 / h_k
        su += u;
        r[1 + k] = exp(-2.0 * u);
      }
      r[0] = wi * exp(su);
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) r[k] = xi[k];
      r[D] = wi;
    }
  }
};

template <int D>
int kde_build_records(const uint32_t *keys, int64_t n, int shift, const double *x, const double *w,
                      int factored, const PsiParams &pp, double *rec_c, uint32_t *keys_c,
                      int32_t *slot, int32_t *hist, int32_t *partial, cudaStream_t st) {
  KdeBuild<D> kb{factored, pp};
  return digit_partition_build<KdeBuild<D>, D + 1>(keys, n, shift, x, w, kb, rec_c, keys_c, slot,
                                                   hist, partial, st, nullptr, "part_emit", true,
                                                   true);
}

// sorted records, field-major (rec[f * n + q], so a warp's loads of one field are coalesced and
// a phase loads only the fields it multiplies), from the coarse-bucketed record-major array
__global__ void __launch_bounds__(256) kde_gather_kernel(const double *__restrict__ rec_c,
                                                        const int32_t *__restrict__ slot,
                                                        int64_t n, int d,
                                                        double *__restrict__ rec) {
  constexpr int U = 4;  // records in flight per thread (slot loads, then all field loads)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < n; q0 += U * stride) {
    int32_t sl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride;
      sl[u] = q < n ? __ldcs(slot + q) : 0;
    }
    double v[U][FCG_MAX_DIM + 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double *r = rec_c + (int64_t)sl[u] * (d + 1);
#pragma unroll
      for (int f = 0; f <= FCG_MAX_DIM; ++f)
        if (f <= d) v[u][f] = r[f];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride;
      if (q < n) {
#pragma unroll
        for (int f = 0; f <= FCG_MAX_DIM; ++f)
          if (f <= d) __stcs(rec + (int64_t)f * n + q, v[u][f]);  // streaming: keep L2 for rec_c
      }
    }
  }
}

// Final axis-0 pass for a group of KDE terms sharing (delta_0, delta_1): each term's lattice is
// scanned along axis 0 (same direction for the whole group) and
//   out (+)= sum_t zfac_t(i) * S_t(i)      (x scale after the last group)
// so the accumulator is read-modify-written once per group instead of once per term
// (fastsum.py:162-168, summed over terms in group order).
constexpr int kMaxGroup = 8;
struct MultiFinal {
  int nt, d;
  const double *lat[kMaxGroup];
  const double *zf[kMaxGroup];
  double *plane[kMaxGroup];   // slab carry capture per term (or null)
  int64_t zoff[FCG_MAX_DIM];
  int64_t dims[FCG_MAX_DIM];
  int64_t plane_idx[kMaxGroup];  // axis-1 index each member captures (-1: none)
  int kz;                     // zf applies on axes k < kz (the in-plane factors are folded in)
  int accumulate, apply_scale;
  double scale;
  double *out;
};

template <int NT, bool REV>
__global__ void __launch_bounds__(256) kde_final_multi(MultiFinal f) {
  const int64_t D0 = f.dims[0];
  int64_t B = 1;
  for (int k = 1; k < f.d; ++k) B *= f.dims[k];
  const int64_t B1 = B / f.dims[1];
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < B;
       b += (int64_t)gridDim.x * blockDim.x) {
    double zo[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) zo[t] = 1.0;
    {
      int64_t rem = b;
      for (int k = f.d - 1; k >= 1; --k) {
        const int64_t i = rem % f.dims[k];
        rem /= f.dims[k];
        if (k >= f.kz) continue;
#pragma unroll
        for (int t = 0; t < NT; ++t)
          if (t < f.nt) zo[t] *= f.zf[t][f.zoff[k] + i];
      }
    }
    int64_t cap[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t)
      cap[t] = (t < f.nt && f.plane_idx[t] >= 0 && b / B1 == f.plane_idx[t]) ? b % B1 : -1;
    double carry[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) carry[t] = 0.0;
    constexpr int U = 4;
    for (int64_t jj0 = 0; jj0 < D0; jj0 += U) {
      double v[U][NT], o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t jj = jj0 + u;
        const int64_t j = REV ? D0 - 1 - jj : jj;
        const bool ok = jj < D0;
#pragma unroll
        for (int t = 0; t < NT; ++t) v[u][t] = (ok && t < f.nt) ? f.lat[t][j * B + b] : 0.0;
        o[u] = (ok && f.accumulate) ? f.out[j * B + b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t jj = jj0 + u;
        if (jj >= D0) break;
        const int64_t j = REV ? D0 - 1 - jj : jj;
        double val = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (t < f.nt) {
            carry[t] += v[u][t];
            val += (zo[t] * f.zf[t][f.zoff[0] + j]) * carry[t];
            if (cap[t] >= 0) f.plane[t][j * B1 + cap[t]] = carry[t];
          }
        }
        double r = o[u] + val;
        if (f.apply_scale) r = r * f.scale;
        f.out[j * B + b] = r;
      }
    }
  }
}

// ---- fused axis-1 + axis-0 final pass (d >= 4) ------------------------------------------
// For up to two group lattices sharing delta_0: the 2-D prefix over (i0, i1) of every in-plane
// column, times the leading factors, accumulated into the density -- replacing a separate
// read + write pass along axis 1 per lattice.  A CTA owns 32 consecutive columns and walks i0;
// the [i1][32] slabs of row i0 + 1 are copied into shared memory (cp.async) while row i0 is
// scanned: thread (column, segment) scans 16 axis-1 positions serially, segments are stitched
// through shared memory, and the axis-0 carries stay in registers.  A lattice running the
// other way along axis 1 hands its values back through its slab so both are combined per cell.
constexpr int kF2Cols = 16, kF2Seg = 8, kF2Segs = 16;  // 16 columns per CTA, axis 1 <= 128
struct Final2D {
  int nt, d, kz;
  const double *lat[2];
  const double *zf[2];
  double *plane[2];
  int64_t plane_idx[2];
  int rev1[2];
  int64_t zoff[FCG_MAX_DIM], dims[FCG_MAX_DIM];
  int accumulate, apply_scale;
  double scale;
  double *out;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct F2Maps {  // TMA boxes [D1][kF2Cols] of the group lattices (0 .. NT-1) and the output (NT)
  CUtensorMap tm[3];
};

template <int NT, bool REV0, bool TMA>
__global__ void __launch_bounds__(256, 2) final2d_kernel(Final2D f, const __grid_constant__ F2Maps maps) {
  extern __shared__ __align__(128) double f2_smem[];
  constexpr int CW = kF2Cols;
  const int64_t D0 = f.dims[0], D1 = f.dims[1];
  int64_t B = 1;
  for (int k = 2; k < f.d; ++k) B *= f.dims[k];
  const int slab = (int)D1 * CW;                        // doubles per [i1][CW] slab
  double *buf = f2_smem;                                // [2][NT + 1][D1][CW] (lattices, density)
  double *segs = buf + 2 * (NT + 1) * slab;             // [NT][kF2Segs][CW]
  double *z1 = segs + NT * kF2Segs * CW;                // [NT][D1] axis-1 factors
  uint64_t *s_bar = reinterpret_cast<uint64_t *>(z1 + NT * D1);  // [2] TMA stage barriers
  const int c = threadIdx.x % CW, sg = threadIdx.x / CW;
  const int64_t b0 = (int64_t)blockIdx.x * CW;
  const int64_t b = b0 + c;
  for (int i = threadIdx.x; i < NT * (int)D1; i += blockDim.x) {
    const int t = i / (int)D1, i1 = i - t * (int)D1;
    z1[i] = f.zf[t][f.zoff[1] + i1];
  }
  // leading factors of the axes 2 .. kz-1 (d >= 5): functions of the column only
  double zb[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) zb[t] = 1.0;
  {
    int64_t rem = b;
    for (int k = f.d - 1; k >= 2; --k) {
      const int64_t i = rem % f.dims[k];
      rem /= f.dims[k];
      if (k < f.kz)
#pragma unroll
        for (int t = 0; t < NT; ++t) zb[t] *= f.zf[t][f.zoff[k] + i];
    }
  }
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  // TMA: one thread issues the [D1][CW] box of every slab of row i0 (no per-thread copies);
  // otherwise 16-byte cp.async chunks from every thread
  auto stage = [&](int64_t jj, int which) {
    const int64_t i0 = REV0 ? D0 - 1 - jj : jj;
    if constexpr (TMA) {
      if (threadIdx.x == 0) {
        const int nsl = NT + (f.accumulate ? 1 : 0);
        mbar_expect_tx(&s_bar[which], (uint32_t)(nsl * slab * sizeof(double)));
#pragma unroll
        for (int t = 0; t <= NT; ++t) {
          if (t == NT && !f.accumulate) break;
          tma_load_2d(buf + (which * (NT + 1) + t) * slab, &maps.tm[t], (int32_t)b0,
                      (int32_t)(i0 * D1), &s_bar[which]);
        }
      }
      return;
    }
#pragma unroll
    for (int t = 0; t <= NT; ++t) {  // t == NT: the density accumulator's row
      if (t == NT && !f.accumulate) break;
      double *dst = buf + (which * (NT + 1) + t) * slab;
      const double *src = (t < NT ? f.lat[t] : f.out) + (i0 * D1) * B + b0;
      for (int ch = threadIdx.x; ch < (int)D1 * (CW / 2); ch += blockDim.x) {  // 16-byte chunks
        const int r = ch / (CW / 2), q = ch % (CW / 2);
        cp_async16(dst + r * CW + q * 2, src + (int64_t)r * B + q * 2);
      }
    }
    cp_async_commit();
  };
  double carry[NT][kF2Seg];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int s = 0; s < kF2Seg; ++s) carry[t][s] = 0.0;
  const int p0 = sg * kF2Seg;
  stage(0, 0);
  for (int64_t jj = 0; jj < D0; ++jj) {
    const int64_t i0 = REV0 ? D0 - 1 - jj : jj;
    const int cur = (int)(jj & 1);
    if constexpr (TMA) {
      if (jj + 1 < D0) stage(jj + 1, cur ^ 1);
      mbar_wait(&s_bar[cur], (uint32_t)((jj >> 1) & 1));
    } else {
      if (jj + 1 < D0) stage(jj + 1, cur ^ 1);
      else cp_async_commit();  // keep the group count uniform
      cp_async_wait1();
      __syncthreads();
    }
    double v[NT][kF2Seg];
    // Cells in order for every lattice: a forward lattice (rev1 = 0) takes inclusive prefixes
    // inside the thread's 8-cell segment plus the totals of the segments below, a reversed one
    // inclusive suffixes plus the totals of the segments above.  A warp holds two segments of
    // the same 16 columns: their totals pair up with one shuffle, so the cross-warp sums run
    // over the 8 warp totals (both lattices in one double2).
    const int warp = threadIdx.x >> 5, upper = (threadIdx.x >> 4) & 1;
    double inner[NT], wtot[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double *sl = buf + (cur * (NT + 1) + t) * slab;
      double x[kF2Seg];
#pragma unroll
      for (int s = 0; s < kF2Seg; ++s) x[s] = p0 + s < D1 ? sl[(p0 + s) * CW + c] : 0.0;
      double run = 0.0;
      if (!f.rev1[t]) {
#pragma unroll
        for (int s = 0; s < kF2Seg; ++s) {
          run += x[s];
          v[t][s] = run;
        }
      } else {
#pragma unroll
        for (int s = kF2Seg - 1; s >= 0; --s) {
          run += x[s];
          v[t][s] = run;
        }
      }
      const double other = __shfl_xor_sync(0xffffffffu, run, 16);
      inner[t] = (f.rev1[t] ? !upper : upper) ? other : 0.0;
      wtot[t] = run + other;
    }
    if (!upper)
      reinterpret_cast<double2 *>(segs)[warp * CW + c] =
          make_double2(wtot[0], NT > 1 ? wtot[NT - 1] : 0.0);
    __syncthreads();
    {
      const int nwarp = blockDim.x >> 5;
      double o0 = inner[0], o1 = inner[NT - 1];
      for (int w = 0; w < nwarp; ++w) {
        if (w == warp) continue;
        const double2 a = reinterpret_cast<const double2 *>(segs)[w * CW + c];
        if (f.rev1[0] ? w > warp : w < warp) o0 += a.x;
        if (NT > 1 && (f.rev1[NT - 1] ? w > warp : w < warp)) o1 += a.y;
      }
      inner[0] = o0;
      if (NT > 1) inner[NT - 1] = o1;
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const double off = inner[t];
#pragma unroll
      for (int s = 0; s < kF2Seg; ++s) carry[t][s] += v[t][s] + off;
      if (f.plane[t] != nullptr) {  // slab carry capture (scanned over axes 0 and 1)
#pragma unroll
        for (int s = 0; s < kF2Seg; ++s)
          if (p0 + s < D1 && p0 + s == f.plane_idx[t]) f.plane[t][i0 * B + b] = carry[t][s];
      }
    }
    const double z00 = f.zf[0][f.zoff[0] + i0] * zb[0];
    const double z01 = NT > 1 ? f.zf[NT - 1][f.zoff[0] + i0] * zb[NT - 1] : 0.0;
    const double *slo = buf + (cur * (NT + 1) + NT) * slab;
#pragma unroll
    for (int s = 0; s < kF2Seg; ++s) {
      const int i1 = p0 + s;
      if (i1 >= D1) continue;
      double val = (z00 * z1[i1]) * carry[0][s];
      if (NT > 1) val += (z01 * z1[(NT - 1) * (int)D1 + i1]) * carry[NT - 1][s];
      double r = f.accumulate ? slo[i1 * CW + c] + val : val;
      if (f.apply_scale) r = r * f.scale;
      f.out[(i0 * D1 + i1) * B + b] = r;
    }
    if constexpr (TMA) fence_proxy_async_smem();  // generic slab accesses before the next TMA
    __syncthreads();  // the slab buffer `cur` is refilled next row
  }
}

int launch_final2d(const Final2D &f, bool rev0, cudaStream_t st) {
  int64_t B = 1;
  for (int k = 2; k < f.d; ++k) B *= f.dims[k];
  const unsigned grid = (unsigned)(B / kF2Cols);
  const size_t smem = (size_t)(2 * (f.nt + 1) * f.dims[1] * kF2Cols + f.nt * kF2Segs * kF2Cols +
                               f.nt * f.dims[1]) * sizeof(double) + 2 * sizeof(uint64_t);
  FCG_PROF("kde_final_group", st);
  // TMA boxes: [D1][kF2Cols] fp64 of each lattice (and of the accumulator), rows i0 * D1 + i1
  // of a 2-D (B, D0 * D1) view
  F2Maps maps{};
  static const bool no_tma = getenv("FCG_NO_TMA") && getenv("FCG_NO_TMA")[0] == '1';
  bool tma = !no_tma && f.dims[1] <= 256;
  const uint64_t rows = (uint64_t)f.dims[0] * f.dims[1];
  for (int t = 0; t < f.nt && tma; ++t)
    tma = tma_map_2d_f64(&maps.tm[t], f.lat[t], B, rows, B, kF2Cols, (uint32_t)f.dims[1]);
  if (tma && f.accumulate)  // box NT: the accumulator
    tma = tma_map_2d_f64(&maps.tm[f.nt], f.out, B, rows, B, kF2Cols, (uint32_t)f.dims[1]);
  auto go = [&](auto kern) -> int {
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 256, smem, st>>>(f, maps);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  };
  if (tma) {
    if (f.nt == 1) return rev0 ? go(final2d_kernel<1, true, true>) : go(final2d_kernel<1, false, true>);
    return rev0 ? go(final2d_kernel<2, true, true>) : go(final2d_kernel<2, false, true>);
  }
  if (f.nt == 1) return rev0 ? go(final2d_kernel<1, true, false>) : go(final2d_kernel<1, false, false>);
  return rev0 ? go(final2d_kernel<2, true, false>) : go(final2d_kernel<2, false, false>);
}

// Fused axis-1 + axis-0 final pass of the partitioned ECDF (d >= 4): int32 counts in, the
// output epilogue (count / N as fp64, or int64 counts) out, 16 columns per CTA as in
// final2d_kernel; the axis-1 lattice pass disappears.
constexpr int kE2Stages = 4;
template <bool REV0, bool REV1, int EK, bool TMA>
__global__ void __launch_bounds__(256, 2) ecdf_final2d_kernel(const int32_t *__restrict__ lat,
                                                              int64_t D0, int64_t D1, int64_t B,
                                                              double div, void *out,
                                                              const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(128) int32_t e2_smem[];
  const double rdiv = div > 0.0 ? 1.0 / div : 0.0;
  constexpr int CW = kF2Cols;
  constexpr int ST = kE2Stages;           // slabs in flight (rows i0 + 1 .. i0 + ST - 1 arriving)
  const int slab = (int)D1 * CW;
  const int sstr = (slab + 31) & ~31;      // buffer stride: 128-byte aligned TMA destinations
  int32_t *buf = e2_smem;                 // [ST][D1][CW]
  int32_t *segs = buf + ST * sstr;        // [kF2Segs][CW]
  uint64_t *bar = reinterpret_cast<uint64_t *>(segs + kF2Segs * CW);  // [ST] TMA barriers
  const int c = threadIdx.x % CW, sg = threadIdx.x / CW;
  const int64_t b0 = (int64_t)blockIdx.x * CW;
  const int64_t b = b0 + c;
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int q = 0; q < ST; ++q) mbar_init(&bar[q], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  auto stage = [&](int64_t jj, int which) {
    const int64_t i0 = REV0 ? D0 - 1 - jj : jj;
    if constexpr (TMA) {  // one thread: the [D1][CW] box of row i0
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bar[which], (uint32_t)(slab * sizeof(int32_t)));
        tma_load_2d(buf + which * sstr, &tm, (int32_t)b0, (int32_t)(i0 * D1), &bar[which]);
      }
      return;
    }
    int32_t *dst = buf + which * sstr;
    const int32_t *src = lat + (i0 * D1) * B + b0;
    for (int ch = threadIdx.x; ch < (int)D1 * (CW / 4); ch += blockDim.x) {  // 16-byte chunks
      const int r = ch / (CW / 4), q = ch % (CW / 4);
      cp_async16(dst + r * CW + q * 4, src + (int64_t)r * B + q * 4);
    }
    cp_async_commit();
  };
  int32_t carry[kF2Seg];
#pragma unroll
  for (int s = 0; s < kF2Seg; ++s) carry[s] = 0;
  const int p0 = sg * kF2Seg;
#pragma unroll
  for (int q = 0; q < ST - 1; ++q) {
    if (q < D0) stage(q, q);
    else if (!TMA) cp_async_commit();
  }
  for (int64_t jj = 0; jj < D0; ++jj) {
    const int64_t i0 = REV0 ? D0 - 1 - jj : jj;
    const int cur = (int)(jj % ST);
    if constexpr (TMA) {
      if (jj + ST - 1 < D0) stage(jj + ST - 1, (int)((jj + ST - 1) % ST));
      mbar_wait(&bar[cur], (uint32_t)((jj / ST) & 1));
    } else {
      if (jj + ST - 1 < D0) stage(jj + ST - 1, (int)((jj + ST - 1) % ST));
      else cp_async_commit();  // keep the group count uniform
      asm volatile("cp.async.wait_group %0;" ::"n"(kE2Stages - 1) : "memory");
      __syncthreads();
    }
    const int32_t *sl = buf + cur * sstr;
    int32_t v[kF2Seg];
    int32_t run = 0;
#pragma unroll
    for (int s = 0; s < kF2Seg; ++s) {
      const int p = p0 + s;
      if (p < D1) run += sl[(REV1 ? (int)D1 - 1 - p : p) * CW + c];
      v[s] = run;
    }
    segs[sg * CW + c] = run;
    __syncthreads();
    int32_t off = 0;
    for (int w = 0; w < sg; ++w) off += segs[w * CW + c];
#pragma unroll
    for (int s = 0; s < kF2Seg; ++s) {
      const int p = p0 + s;
      carry[s] += v[s] + off;
      if (p >= D1) continue;
      const int64_t i1 = REV1 ? D1 - 1 - p : p;
      const int64_t o = (i0 * D1 + i1) * B + b;
      if constexpr (EK == EPI_I64) {
        static_cast<int64_t *>(out)[o] = (int64_t)carry[s];
      } else {
        double r = (double)carry[s];
        if (div > 0.0) r = div_rn(r, div, rdiv);  // the single division of fastsum.py:87-88
        static_cast<double *>(out)[o] = r;
      }
    }
    __syncthreads();  // slab `cur` and the segment totals are rewritten next row
  }
}

int launch_ecdf_final2d(const int32_t *lat, const int64_t *dims, int d, bool rev0, bool rev1,
                        const Epi &epi, cudaStream_t st) {
  int64_t B = 1;
  for (int k = 2; k < d; ++k) B *= dims[k];
  const unsigned grid = (unsigned)(B / kF2Cols);
  const size_t smem = (size_t)(kE2Stages * ((dims[1] * kF2Cols + 31) & ~int64_t(31)) +
                               kF2Segs * kF2Cols) * sizeof(int32_t) + kE2Stages * sizeof(uint64_t);
  FCG_PROF("scan_lines_final", st);
  // TMA box [D1][kF2Cols] int32 of the 2-D (B, D0 * D1) view of the count lattice
  CUtensorMap tm{};
  static const bool no_tma = getenv("FCG_NO_TMA") && getenv("FCG_NO_TMA")[0] == '1';
  const bool tma = !no_tma && dims[1] <= 256 &&
                   tma_map_2d_i32(&tm, lat, B, (uint64_t)dims[0] * dims[1], B, kF2Cols,
                                  (uint32_t)dims[1]);
  auto go = [&](auto kern) -> int {
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, 256, smem, st>>>(lat, dims[0], dims[1], B, epi.div, epi.out, tm);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  };
  auto pick = [&](auto tma_tag) -> int {
    constexpr bool T = decltype(tma_tag)::value;
    if (epi.kind == EPI_I64) {
      if (rev0) return rev1 ? go(ecdf_final2d_kernel<true, true, EPI_I64, T>) : go(ecdf_final2d_kernel<true, false, EPI_I64, T>);
      return rev1 ? go(ecdf_final2d_kernel<false, true, EPI_I64, T>) : go(ecdf_final2d_kernel<false, false, EPI_I64, T>);
    }
    if (rev0) return rev1 ? go(ecdf_final2d_kernel<true, true, EPI_F64, T>) : go(ecdf_final2d_kernel<true, false, EPI_F64, T>);
    return rev1 ? go(ecdf_final2d_kernel<false, true, EPI_F64, T>) : go(ecdf_final2d_kernel<false, false, EPI_F64, T>);
  };
  return tma ? pick(std::true_type{}) : pick(std::false_type{});
}

int launch_final_multi(const MultiFinal &f, bool rev, cudaStream_t st) {
  int64_t B = 1;
  for (int k = 1; k < f.d; ++k) B *= f.dims[k];
  const int grid = grid_for(B, 256, 8);
  FCG_PROF("kde_final_group", st);
if (f.nt <= 2) {
    if (rev) kde_final_multi<2, true><<<grid, 256, 0, st>>>(f);
    else kde_final_multi<2, false><<<grid, 256, 0, st>>>(f);
  } else if (f.nt <= 4) {
    if (rev) kde_final_multi<4, true><<<grid, 256, 0, st>>>(f);
    else kde_final_multi<4, false><<<grid, 256, 0, st>>>(f);
  } else {
    if (rev) kde_final_multi<8, true><<<grid, 256, 0, st>>>(f);
    else kde_final_multi<8, false><<<grid, 256, 0, st>>>(f);
  }
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

// rows of segment totals the tile scans need (scalar or vectorised column pass)
int64_t seg_rows(int threads, int64_t W, int V) {
  int64_t g1 = threads >= W ? threads / W : 1;
  int64_t g2 = threads * V >= W ? threads * V / W : 1;
  return g1 > g2 ? g1 : g2;
}

// plane_kde_group_kernel: two tiles, two carry rows, the column factor pairs, segment totals
// (vectorised walk: [2][warps][W]; generic scan: G rows)
size_t kde_group_smem(int64_t Rf, int64_t W, int64_t G) {
  const int64_t segs = std::max<int64_t>(G, 2 * (kKdeThreads / 32));
  return (size_t)(2 * Rf * W + 2 * W + 2 * W + segs * W) * sizeof(double);
}

int bits_for(int64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 32 && (int64_t(1) << b) <= v) ++b;
  return b;
}

// keys + payloads of one radix tile per CTA, with the tile's histogram of the keys' low byte
// (the first LSD pass's digit-major histogram, so that pass needs no histogram kernel)
template <int D, bool MM, int LEU>
__global__ void __launch_bounds__(256, D == 3 || D == 4 ? 4 : 1) part_bin_tile_kernel(const double *__restrict__ x, int64_t n,
                                                            int drt, const double *__restrict__ knots,
                                                            BinGrid g, PartGeo p,
                                                            uint32_t *__restrict__ keys,
                                                            int32_t *__restrict__ vals,
                                                            int32_t *__restrict__ hist,
                                                            int64_t tiles, int tile, int hshift,
                                                            unsigned long long *__restrict__ mm) {
  extern __shared__ double s_knots[];
  __shared__ double s_z0[FCG_MAX_DIM], s_idz[FCG_MAX_DIM];
  __shared__ int32_t s_hist[8][256];
  __shared__ unsigned long long s_mm[8][2][FCG_MAX_DIM];
  const int d = D > 0 ? D : drt;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x & 31; i < 256; i += 32) s_hist[warp][i] = 0;
  const double *kb = stage_knots(g, knots, s_knots, s_z0, s_idz);
  __syncthreads();
  // uniform axes: points away from the mesh lines skip the knot verification
  const unsigned mesh = g.total_knots <= kSmemKnots ? mesh_uniform(g, kb, s_z0, s_idz) : 0u;
  constexpr int DD = D > 0 ? D : FCG_MAX_DIM;
  const int64_t tile0 = (int64_t)blockIdx.x * tile;
  constexpr int U = 2;  // points in flight per thread
  // data hull (auto centre of the KDE): per-thread, then warp, then CTA, then one atomic each
  double lo[DD], hi[DD];
#pragma unroll
  for (int k = 0; k < DD; ++k) {
    lo[k] = CUDART_INF;
    hi[k] = -CUDART_INF;
  }
  for (int j0 = 0; j0 < tile; j0 += U * 256) {
    double xi[U][DD];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = tile0 + j0 + u * 256 + threadIdx.x;
      const int64_t ii = i < n ? i : 0;
      if constexpr (D == 4) {
        const double2 v0 = __ldcs(reinterpret_cast<const double2 *>(x) + 2 * ii);
        const double2 v1 = __ldcs(reinterpret_cast<const double2 *>(x) + 2 * ii + 1);
        xi[u][0] = v0.x; xi[u][1] = v0.y; xi[u][2] = v1.x; xi[u][3] = v1.y;
      } else {
#pragma unroll
        for (int k = 0; k < DD; ++k)
          if (k < d) xi[u][k] = x[ii * d + k];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = tile0 + j0 + u * 256 + threadIdx.x;
      if (i >= n) continue;
      uint32_t key;
      int32_t val;
      part_key<D, LEU>(xi[u], d, kb, g, s_z0, s_idz, p, i, key, val, mesh);
      keys[i] = key;
      if (vals) vals[i] = val;
      atomicAdd(&s_hist[warp][(key >> hshift) & 0xFFu], 1);
      if constexpr (MM) {
#pragma unroll
        for (int k = 0; k < DD; ++k) {
          if (k < d) {
            lo[k] = fmin(lo[k], xi[u][k]);
            hi[k] = fmax(hi[k], xi[u][k]);
          }
        }
      }
    }
  }
  if constexpr (MM) {  // warp reduce in order-key space: two redux.sync per 64-bit value
#pragma unroll
    for (int k = 0; k < DD; ++k) {
      if (k < d) {
        const uint64_t kl = f64_key(lo[k]), kh = f64_key(hi[k]);
        const unsigned lhi = __reduce_min_sync(0xffffffffu, (unsigned)(kl >> 32));
        const unsigned hhi = __reduce_max_sync(0xffffffffu, (unsigned)(kh >> 32));
        const unsigned llo =
            __reduce_min_sync(0xffffffffu, (unsigned)(kl >> 32) == lhi ? (unsigned)kl : ~0u);
        const unsigned hlo =
            __reduce_max_sync(0xffffffffu, (unsigned)(kh >> 32) == hhi ? (unsigned)kh : 0u);
        if ((threadIdx.x & 31) == 0) {
          s_mm[warp][0][k] = ((unsigned long long)lhi << 32) | llo;
          s_mm[warp][1][k] = ((unsigned long long)hhi << 32) | hlo;
        }
      }
    }
  }
  __syncthreads();
  int32_t tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += s_hist[w][threadIdx.x];
  hist[(int64_t)threadIdx.x * tiles + blockIdx.x] = tot;
  if (MM && threadIdx.x < 2 * d) {
    const int k = threadIdx.x >> 1, side = threadIdx.x & 1;
    unsigned long long key = s_mm[0][side][k];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const unsigned long long v = s_mm[w][side][k];
      key = side ? (v > key ? v : key) : (v < key ? v : key);
    }
    unsigned long long *slot = mm + side * d + k;
    if (side) atomicMax(slot, key);  // result unused: a fire-and-forget RED
    else atomicMin(slot, key);
  }
}


// tile: items per histogram tile (the consuming pass's tile); hshift: the digit's shift
int launch_part_bin_tiles(const double *x, int64_t n, int d, const double *knots, const BinGrid &g,
                          const PartGeo &p, uint32_t *keys, int32_t *vals, int32_t *hist,
                          cudaStream_t st, int tile = kSortTile, int hshift = 0,
                          unsigned long long *mm = nullptr) {
  const size_t smem = g.total_knots <= kSmemKnots ? (size_t)g.total_knots * sizeof(double) : 0;
  const int64_t tiles = ceil_div(n, tile);
  FCG_PROF("part_bin", st);
  const bool al = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const unsigned gr = (unsigned)tiles;
  auto launch = [&](auto kern) {
    kern<<<gr, 256, smem, st>>>(x, n, d, knots, g, p, keys, vals, hist, tiles, tile, hshift, mm);
  };
  bool le0 = true, le1 = true;
  for (int k = 0; k < d; ++k) {
    le0 = le0 && g.le[k] == 0;
    le1 = le1 && g.le[k] == 1;
  }
  auto by_le = [&](auto k0, auto k1, auto k2) {
    if (le0) launch(k0);
    else if (le1) launch(k1);
    else launch(k2);
  };
  if (d == 4 && al) {
    if (mm) by_le(part_bin_tile_kernel<4, true, 0>, part_bin_tile_kernel<4, true, 1>, part_bin_tile_kernel<4, true, 2>);
    else by_le(part_bin_tile_kernel<4, false, 0>, part_bin_tile_kernel<4, false, 1>, part_bin_tile_kernel<4, false, 2>);
  } else if (d == 3) {
    if (mm) by_le(part_bin_tile_kernel<3, true, 0>, part_bin_tile_kernel<3, true, 1>, part_bin_tile_kernel<3, true, 2>);
    else by_le(part_bin_tile_kernel<3, false, 0>, part_bin_tile_kernel<3, false, 1>, part_bin_tile_kernel<3, false, 2>);
  } else {
    mm ? launch(part_bin_tile_kernel<0, true, 2>) : launch(part_bin_tile_kernel<0, false, 2>);
  }
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}


struct PartBufs {
  uint32_t *keys;
  int32_t *vals;
  RadixWs rw;
  int32_t *start;
  SegSortWs sw;
};

void carve_part(Workspace &W, PartBufs &b, int64_t n, int64_t NB) {
  b.keys = W.take<uint32_t>(n);
  b.vals = W.take<int32_t>(n);
  b.rw.keys_alt = reinterpret_cast<uint64_t *>(W.take<uint32_t>(n));
  b.rw.vals_alt = W.take<int32_t>(n);
  // histograms of the radix passes (4096-item tiles) and of the record partition (2048)
  const size_t hist = std::max(std::max(radix_ws_hist_elems(n), digit_hist_elems(n)),
                               (size_t)256 * seg_sort_tiles(n) + 1);
  b.rw.hist = W.take<int32_t>(hist);
  b.rw.partial = W.take<int32_t>(scan_ws_partial_elems((int64_t)hist + 2));
  b.start = W.take<int32_t>(NB + 1);
  b.sw.seg_start = W.take<int32_t>(kSortSegs + 1);
  b.sw.tile_base = W.take<int32_t>(kSortSegs + 1);
  b.sw.tile_seg = W.take<int32_t>(seg_sort_tiles(n));
}

int partition(const double *x, int64_t n, int d, const double *knots, const BinGrid &g,
              const PartGeo &p, int64_t NB, int nbits, PartBufs &b, cudaStream_t st) {
  // equal bucket keys may come out in any order (the plane kernel only groups by bucket).
  // Packed keys (p.cell_bits > 0): bucket << cell_bits | in-block cell, keys only, sorted on
  // the bucket bits [cell_bits, cell_bits + nbits): half the bytes per sort pass.
  const int lo = p.cell_bits;
  int32_t *vals = lo > 0 ? nullptr : b.vals;
  if (nbits > 8 && nbits <= 16) {  // high digit first, then the low digit per segment
    FCG_TRY(launch_part_bin_tiles(x, n, d, knots, g, p, b.keys, vals, b.rw.hist, st, kSortTile,
                                  lo + 8));
    FCG_TRY(msd2_sort_pairs_u32(b.keys, vals, n, nbits, b.rw, b.sw, st, true, lo));
  } else {
    FCG_TRY(launch_part_bin_tiles(x, n, d, knots, g, p, b.keys, vals, b.rw.hist, st, kSortTile,
                                  lo));
    FCG_TRY(radix_sort_pairs<uint32_t>(b.keys, vals, n, lo, lo + ((nbits + 7) / 8) * 8, b.rw, st,
                                       false, true));
  }
  FCG_PROF("part_bucket_start", st);
  bucket_start_kernel<<<grid_for(NB + 1, 256, 4), 256, 0, st>>>(b.keys, n, NB, p.cell_bits,
                                                                 b.start);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

}  // namespace

__global__ void hull_init_kernel(const double *__restrict__ knots, HullKnots hk,
                                 unsigned long long *mm) {
  const int k = threadIdx.x;
  if (k < hk.d) {
    mm[k] = f64_key(knots[hk.first[k]]);
    mm[hk.d + k] = f64_key(knots[hk.last[k]]);
  }
}

int hull_init(const double *knots, int d, const int64_t *m, unsigned long long *mm, cudaStream_t st) {
  HullKnots hk{};
  hk.d = d;
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    hk.first[k] = off;
    hk.last[k] = off + m[k] - 1;
    off += m[k];
  }
  hull_init_kernel<<<1, 32, 0, st>>>(knots, hk, mm);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

static double f64_unkey(uint64_t k) {
  const uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  double v;
  std::memcpy(&v, &u, sizeof v);
  return v;
}

int hull_centre(const unsigned long long *mm, int d, const double *h, double *c, double *u_bound,
                cudaStream_t st) {
  unsigned long long host[2 * FCG_MAX_DIM];
  FCG_TRY(read_small(host, mm, 2 * d * sizeof(unsigned long long), st));
  double ub = 0.0;
  for (int k = 0; k < d; ++k) {
    const double lo = f64_unkey(host[k]), hi = f64_unkey(host[d + k]);
    const double span = hi - lo;
    // fastsum.py:114-129 with EXP_OVERFLOW_GUARD = 600 (core.py:22)
    if (span / h[k] > 600.0) {
      char msg[160];
      std::snprintf(msg, sizeof msg,
                    "dimension %d: span/bandwidth = %.1f exceeds 600; enlarge the bandwidth or rescale",
                    k, span / h[k]);
      return fail(FCG_ERANGE, msg);
    }
    c[k] = 0.5 * (lo + hi);
    ub += span / (2.0 * h[k]);
  }
  *u_bound = ub * 1.000001;
  return FCG_OK;
}

PartPlan plan_ecdf_partition(const BinGrid &g, int64_t n) {
  PartPlan pl;
  const int d = g.d;
  if (d < 3 || n < kMinPartitionN) return pl;
  // Sparse lattices (well under one point per 4 cells, e.g. config 3 at 0.07) keep the atomic
  // scatter: its random updates mostly hit L2 and the partition would cost more than it saves.
  int64_t cells = 1;
  for (int k = 0; k < d; ++k) cells *= g.dims[k];
  if (4 * n < cells) return pl;
  pl.W = g.dims[d - 1];
  pl.H = g.dims[d - 2];
  pl.NP = 1;
  for (int k = 0; k < d - 2; ++k) pl.NP *= g.dims[k];
  if (pl.W > 8192 || pl.NP < 2 * (int64_t)sm_count()) return pl;
  const int64_t G = seg_rows(kPlaneThreads, pl.W, 4);
  // tile + carry + segment totals
  int64_t R = (int64_t)(kEcdfTileBytes / 4 - pl.W - G * pl.W) / pl.W;
  if (R < 1) return pl;
  if (R > pl.H) R = pl.H;
  pl.R = R;
  pl.nrb = ceil_div(pl.H, R);
  pl.NB = pl.NP * pl.nrb;
  if (pl.NB >= (int64_t(1) << 31) - 2 || n >= (int64_t(1) << 31) - 1) return pl;
  pl.nbits = bits_for(pl.NB);  // kDead's low nbits are all ones > NB - 1
  // packed keys bucket << cell_bits | r_in << col_bits | col when they fit 31 bits (the dead
  // key 0xFFFFFFFF then sorts last): keys only through the sort
  static const bool unpacked = getenv("FCG_ECDF_UNPACKED") && getenv("FCG_ECDF_UNPACKED")[0] == '1';
  const int colb = bits_for(pl.W - 1), rowb = pl.R > 1 ? bits_for(pl.R - 1) : 0;
  if (!unpacked && colb + rowb > 0 && pl.nbits + colb + rowb <= 31) {
    pl.col_bits = colb;  // (nbits stays bits_for(NB): the dead key's bucket bits exceed NB - 1)
    pl.cell_bits = colb + rowb;
  }
  pl.ok = true;
  return pl;
}

int ecdf_partitioned(const double *x, int64_t n, const double *knots, const BinGrid &g,
                     const bool *rev, const PartPlan &pl, const Epi &epi, Workspace &W, bool run,
                     cudaStream_t st) {
  const int d = g.d;
  PartBufs b;
  carve_part(W, b, n, pl.NB);
  LatShape s;
  s.d = d;
  for (int k = 0; k < d; ++k) s.dims[k] = g.dims[k];
  int32_t *lat = W.take<int32_t>(s.size());
  int32_t *scratch = W.take<int32_t>(scan_scratch_bound());
  if (!run) return FCG_OK;
  PartGeo p{};
  p.d = d;
  for (int k = 0; k < d; ++k) {
    p.E[k] = g.dims[k];
    p.shift[k] = g.shift[k];
  }
  p.W = pl.W;
  p.R = pl.R;
  p.inv_R = 1.0f / (float)pl.R;
  p.nrb = pl.nrb;
  p.H = pl.H;
  p.ecdf = 1;
  p.cell_bits = pl.cell_bits;  // > 0: packed keys (no value array)
  p.col_bits = pl.col_bits;
  FCG_TRY(partition(x, n, d, knots, g, p, pl.NB, pl.nbits, b, st));
  const int64_t G = seg_rows(kPlaneThreads, pl.W, 4);
  const size_t smem = (size_t)(pl.R * pl.W + pl.W + G * pl.W) * sizeof(int32_t);
  {
    FCG_PROF("plane_count", st);
    const int se = scan_variant(pl.W, 4);
    auto kern = se == 4 ? plane_count_kernel<4> : (se == 8 ? plane_count_kernel<8> : plane_count_kernel<0>);
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)pl.NP, kPlaneThreads, smem, st>>>(p, b.start, b.vals, rev[d - 2], rev[d - 1],
                                                      lat, p.cell_bits > 0 ? b.keys : nullptr);
    FCG_LAUNCH_CHECK();
  }
  Epi inplace;
  int64_t bcols = 1;
  for (int k = 2; k < d; ++k) bcols *= s.dims[k];
  const bool fuse01 = d >= 4 && (epi.kind == EPI_F64 || epi.kind == EPI_I64) &&
                      s.dims[1] <= kF2Seg * kF2Segs && bcols % kF2Cols == 0;
  for (int ax = d - 3; ax >= (fuse01 ? 2 : 1); --ax)
    FCG_TRY(scan_axis<int32_t>(lat, s, ax, rev[ax], inplace, scratch, st));
  if (fuse01) return launch_ecdf_final2d(lat, s.dims, d, rev[0], rev[1], epi, st);
  return scan_axis<int32_t>(lat, s, 0, rev[0], epi, scratch, st);
}

PartPlan plan_kde_partition(int d, const int64_t *m, int64_t n, bool factored) {
  PartPlan pl;
  if (d < 3 || n < kMinPartitionN) return pl;
  pl.W = m[d - 1];
  pl.H = m[d - 2];
  if (pl.W + 1 > 65535 || pl.H + 1 > 65535) return pl;  // packed 16-bit (row, col) offsets
  const int64_t G = seg_rows(kKdeThreads, pl.W, 2);
  const int64_t Hf = pl.H + 1;
  // all term groups in one pass (plane_kde_all_kernel): d = 3, 4, factored records,
  // W = 32 E with E in {2, 4, 8}; otherwise one launch per group (plane_kde_group_kernel)
  const int ng = 1 << (d - 2);
  const int e_all = scan_variant(pl.W, 2);
  pl.all = factored && (d == 3 || d == 4) && (e_all == 2 || e_all == 4);
  // fewest full-space row blocks whose tiles fit the budget
  int64_t nrb = 1, Rf = Hf;
  while (true) {
    Rf = ceil_div(Hf, nrb);
    if (pl.all ? Rf <= all_tile_rows(ng, pl.W) : kde_group_smem(Rf, pl.W, G) <= kKdeTileBytes) break;
    if (Rf == 1) return pl;
    ++nrb;
  }
  pl.NP = 1;
  int64_t np_full = 1;
  for (int k = 0; k < d - 2; ++k) {
    pl.NP *= m[k];
    np_full *= m[k] + 1;
  }
  if (pl.NP < 2 * (int64_t)sm_count()) return pl;
  pl.R = Rf;
  pl.nrb = nrb;
  pl.NB = np_full * nrb;
  if (pl.NB >= (int64_t(1) << 31) - 2 || n >= (int64_t(1) << 31) - 1) return pl;
  // records sorted by full cell: key = bucket << cell_bits | r_in << col_bits | col (< 2^31,
  // so the dead key 0xFFFFFFFF sorts last)
  pl.col_bits = bits_for(pl.W);      // full-space columns 0..W
  pl.cell_bits = pl.col_bits + bits_for(Rf - 1);
  pl.nbits = bits_for(pl.NB - 1) + pl.cell_bits;
  if (pl.nbits > 31) return pl;
  pl.ok = true;
  return pl;
}

int kde_partitioned(const double *x, int64_t n, const double *w, const double *knots,
                    const int64_t *m, int d, const double *h, const double *centre,
                    double bound_u_sum, double n_scale, double *planes, const PartPlan &pl,
                    double *out, Workspace &W, bool run, cudaStream_t st) {
  PartBufs b;
  carve_part(W, b, n, pl.NB);
  double *rec = W.take<double>((size_t)n * (d + 1));
  double *rec_c = W.take<double>((size_t)n * (d + 1));
  uint32_t *keys_c = W.take<uint32_t>(n);
  int32_t *share_b = W.take<int32_t>((size_t)pl.NB * (kAllThreads / 32 + 1));
  const SegSortWs &sw = b.sw;
  LatShape s;
  s.d = d;
  int64_t total_knots = 0;
  for (int k = 0; k < d; ++k) {
    s.dims[k] = m[k];
    total_knots += m[k];
  }
  // Terms are folded in groups sharing the signs of axes k < kz (see plane_kde_group_kernel):
  // kz = d - 2 folds all four in-plane sign pairs; with slab planes requested the folded axes
  // must all be >= 2 (the slab axis 1 factor has to stay outside the captured plane), so d = 3
  // then folds only the column axis.  Groups sharing delta_0 share one final axis-0 pass.
  const int kz = planes ? kde_cap_kw(d) : d - 2;
  const int ngroups = 1 << kz;
  const int per0 = ngroups / 2;  // groups per delta_0 sign
  const int nbatch = per0 < kMaxGroup ? per0 : kMaxGroup;
  // all-groups pass: every group lattice alive at once; else one batch of groups at a time
  double *lats = W.take<double>((size_t)s.size() * (pl.all ? ngroups : nbatch));
  double *scratch = W.take<double>(scan_scratch_bound());
  double *zfs = W.take<double>((size_t)total_knots * (nbatch + 2));
  unsigned long long *mm = W.take<unsigned long long>(2 * FCG_MAX_DIM);
  if (!run) return FCG_OK;
  const bool auto_centre = centre == nullptr;
  double c_auto[FCG_MAX_DIM];

  // one delta=+1 binning in the full (M+1)^d space serves every term (fastsum.py:146-149)
  int le[FCG_MAX_DIM];
  int64_t zero[FCG_MAX_DIM], full[FCG_MAX_DIM];
  for (int k = 0; k < d; ++k) {
    le[k] = 0;
    zero[k] = 0;
    full[k] = m[k] + 1;
  }
  BinGrid g = make_bin_grid(d, m, le, zero, full);
  PartGeo p{};
  p.d = d;
  for (int k = 0; k < d; ++k) {
    p.E[k] = full[k];
    p.shift[k] = 0;
  }
  p.W = full[d - 1];
  p.H = full[d - 2];
  p.R = pl.R;
  p.inv_R = 1.0f / (float)pl.R;
  p.nrb = pl.nrb;
  p.ecdf = 0;
  p.cell_bits = pl.cell_bits;
  p.col_bits = pl.col_bits;
  // factored psi records when every partial product stays inside e^{+-600}: needs
  // sum_k max|u_k| <= 600 with u_k = (x_k - c_k)/h_k; bounded here by the hull of the knots
  // and the data (the caller's centre is that hull's midrange, fastsum.py:118-129)
  // keys -> records grouped by the key's top 8 bits -> sort (key, slot) -> L2-local gather
  const int sort_bits = ((pl.nbits + 7) / 8) * 8;
  const int cshift = pl.nbits > 8 ? pl.nbits - 8 : 0;  // coarse digit: the key's top 8 bits
  if (auto_centre) FCG_TRY(hull_init(knots, d, m, mm, st));
  FCG_TRY(launch_part_bin_tiles(x, n, d, knots, g, p, b.keys, nullptr, b.rw.hist, st, kPartTile,
                                cshift, auto_centre ? mm : nullptr));  // slots come later
  if (auto_centre) {  // the hull came with the binning pass
    FCG_TRY(hull_centre(mm, d, h, c_auto, &bound_u_sum, st));
    centre = c_auto;
  }
  PsiParams pp{};
  for (int k = 0; k < d; ++k) {
    pp.c[k] = centre[k];
    pp.a[k] = 1.0 / h[k];
  }
  const int factored = bound_u_sum <= 600.0 ? 1 : 0;
  // d = 3, 4: the segmented sort's last pass writes the records (no slots, no gather kernel)
  const bool fused_gather = cshift > 0 && (d + 1 == 4 || d + 1 == 5);
  // the all-groups kernel takes factored records only (an auto-centre plan assumed them)
  const bool all_run = pl.all && factored;
  {
    const int shift = cshift;
    const bool al = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    int rc;
    switch (d) {  // the partitioned path runs for d >= 3
      case 3: rc = kde_build_records<3>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                        b.rw.hist, b.rw.partial, st); break;
      case 4:
        if (!al) return fail(FCG_EINVAL, "points must be 16-byte aligned");
        rc = kde_build_records<4>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                  b.rw.hist, b.rw.partial, st); break;
      case 5: rc = kde_build_records<5>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                        b.rw.hist, b.rw.partial, st); break;
      case 6:
        if (!al) return fail(FCG_EINVAL, "points must be 16-byte aligned");
        rc = kde_build_records<6>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                  b.rw.hist, b.rw.partial, st); break;
      case 7: rc = kde_build_records<7>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                        b.rw.hist, b.rw.partial, st); break;
      default:
        if (!al) return fail(FCG_EINVAL, "points must be 16-byte aligned");
        rc = kde_build_records<8>(b.keys, n, shift, x, w, factored, pp, rec_c, keys_c, fused_gather ? nullptr : b.vals,
                                  b.rw.hist, b.rw.partial, st); break;
    }
    FCG_TRY(rc);
  }
  // Records are grouped by the key's top 8 bits (coarse segments); sort every segment by the
  // bits below (equal keys are the same cell: their order is irrelevant).  For d = 3, 4 the last
  // pass writes the records themselves, field-major, from their segment-local slots (no
  // separate gather); otherwise the (key, slot) sort is followed by the gather kernel.
  uint32_t *skeys = keys_c;
  if (fused_gather) {
    FCG_TRY(seg_sort_pairs_u32(keys_c, b.vals, n, cshift, b.rw, sw, st, rec_c, d + 1, rec, &skeys,
                               true));
  } else {
    FCG_TRY(radix_sort_pairs<uint32_t>(keys_c, b.vals, n, 0, sort_bits, b.rw, st, false));
  }
  {
    FCG_PROF("part_bucket_start", st);
    bucket_start_kernel<<<grid_for(pl.NB + 1, 256, 4), 256, 0, st>>>(skeys, n, pl.NB, p.cell_bits,
                                                                      b.start);
    FCG_LAUNCH_CHECK();
    if (all_run) {
      const int nw = kAllThreads / 32;
      share_bounds_kernel<<<grid_for(pl.NB * (nw + 1), 256, 4), 256, 0, st>>>(skeys, b.start, pl.NB,
                                                                              nw, share_b);
      FCG_LAUNCH_CHECK();
    }
  }
  if (!fused_gather) {
    FCG_PROF("kde_materialize", st);
    // two CTAs per SM: the sorted positions in flight span ~half a coarse bucket, so its
    // records are re-read from L2 (a full grid spreads over several buckets and misses)
    kde_gather_kernel<<<grid_for(n, 256, 2), 256, 0, st>>>(rec_c, b.vals, n, d, rec);
    FCG_LAUNCH_CHECK();
  }
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  const double scale = 1.0 / (std::ldexp(1.0, d) * n_scale * prod_h);
  const int64_t G = seg_rows(kKdeThreads, pl.W, 2);
  int64_t plane_sz = m[0];
  for (int k = 2; k < d; ++k) plane_sz *= m[k];
  if (planes)  // slots of codes that are folded into a lower code stay zero
    FCG_CUDA_TRY(cudaMemsetAsync(planes, 0, (size_t)plane_sz * (size_t(1) << d) * sizeof(double), st));
  const size_t smem = kde_group_smem(pl.R, pl.W, G);
  const int se = scan_variant(pl.W, 2);
  auto kde_kern = se == 2 ? plane_kde_group_kernel<2>
                          : (se == 4 ? plane_kde_group_kernel<4>
                                     : (se == 8 ? plane_kde_group_kernel<8> : plane_kde_group_kernel<0>));
  FCG_CUDA_TRY(cudaFuncSetAttribute(kde_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t L = s.size();
  int64_t zoff[FCG_MAX_DIM];
  {
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      zoff[k] = off;
      off += m[k];
    }
  }
  // factor tables of the all-(+1) and all-(-1) sign vectors: the in-plane factors of any term
  double *zpos = zfs + (size_t)nbatch * total_knots, *zneg = zpos + total_knots;
  FCG_TRY(launch_kde_zf(knots, d, m, centre, h, 0, zpos, st));
  FCG_TRY(launch_kde_zf(knots, d, m, centre, h, (1 << d) - 1, zneg, st));
  const int kr = d - 2, kc = d - 1;
  if (all_run) {  // one pass over the records per row sign for every group
    KdeAll ta{};
    ta.d = d;
    ta.nlead = d - 2;
    ta.Mr = m[kr];
    ta.Mc = m[kc];
    ta.Rf = pl.R;
    ta.nrb = pl.nrb;
    for (int k = 0; k < d - 2; ++k) ta.lead_m[k] = m[k];
    ta.cell_bits = pl.cell_bits;
    ta.col_bits = pl.col_bits;
    ta.row_split = kz > kr ? 1 : 0;
    ta.zr_pos = zpos + zoff[kr];
    ta.zr_neg = zneg + zoff[kr];
    ta.zc_pos = zpos + zoff[kc];
    ta.zc_neg = zneg + zoff[kc];
    const int ng = 1 << (d - 2);
    for (int g = 0; g < ng; ++g) {
      if (ta.row_split) {  // lattice of group code gl = lead signs | row sign << kr
        for (int ph = 0; ph < 2; ++ph) ta.lat[2 * g + ph] = lats + (size_t)(g | (ph << kr)) * L;
      } else {
        ta.lat[g] = lats + (size_t)g * L;
      }
    }
    const size_t asmem = (size_t)(2 * ng) * all_tile_stride(ng, pl.W) * sizeof(double);
    int64_t np_full = 1;
    for (int k = 0; k < d - 2; ++k) np_full *= m[k] + 1;
    FCG_PROF("plane_kde", st);
    auto launch = [&](auto kern) -> int {
      FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asmem));
      kern<<<(unsigned)np_full, kAllThreads, asmem, st>>>(ta, share_b, rec, n, skeys);
      FCG_LAUNCH_CHECK();
      return FCG_OK;
    };
    const int E = scan_variant(pl.W, 2);
    if (d == 4) {
      FCG_TRY(E == 2 ? launch(plane_kde_all_kernel<2, 4>) : launch(plane_kde_all_kernel<4, 4>));
    } else {
      FCG_TRY(E == 2 ? launch(plane_kde_all_kernel<2, 2>) : launch(plane_kde_all_kernel<4, 2>));
    }
  }
  for (int s0 = 0; s0 < 2; ++s0) {
    for (int b0 = 0; b0 < per0; b0 += nbatch) {
      const int nt = (per0 - b0) < nbatch ? (per0 - b0) : nbatch;
      // axes 1 and 0 in one pass (final2d_kernel) when the batch, axis 1 and the columns fit
      int64_t bcols = 1;
      for (int k = 2; k < d; ++k) bcols *= m[k];
      const bool fuse01 = d >= 4 && kz >= 2 && nt <= 2 && m[1] <= kF2Seg * kF2Segs &&
                          bcols % kF2Cols == 0;
      Final2D f2{};
      MultiFinal f{};
      f.nt = nt;
      f.d = d;
      f.kz = kz;
      for (int k = 0; k < d; ++k) {
        f.zoff[k] = zoff[k];
        f.dims[k] = m[k];
      }
      for (int tt = 0; tt < nt; ++tt) {
        const int gl = s0 | ((b0 + tt) << 1);  // signs of axes < kz (bit k: delta_k = -1)
        double *lat = lats + (size_t)(all_run ? gl : tt) * L;
        double *zf = zfs + (size_t)tt * total_knots;
        KdeGroup t{};
        t.d = d;
        bool rev[FCG_MAX_DIM];
        for (int k = 0; k < d; ++k) {
          rev[k] = k < kz && ((gl >> k) & 1);
          t.c[k] = centre[k];
          t.a[k] = 1.0 / h[k];
        }
        t.Mr = m[kr];
        t.Mc = m[kc];
        t.Rf = pl.R;
        t.nrb = pl.nrb;
        t.lead_neg = 0;
        for (int k = 0; k < kr; ++k) {
          t.lead_m[k] = m[k];
          t.lead_s[k] = rev[k] ? 1 : 0;
          t.lead_full[k] = m[k] + 1;
          if (rev[k]) t.lead_neg |= 1u << k;
        }
        if (kz > kr) {  // row sign fixed by the group
          t.nphase = 1;
          t.rneg[0] = rev[kr] ? 1 : 0;
        } else {
          t.nphase = 2;
          t.rneg[0] = 0;
          t.rneg[1] = 1;
        }
        for (int ph = 0; ph < t.nphase; ++ph) {
          // a row sign fixed by the group leaves the row factor to the final pass (k < kz)
          t.zr[ph] = kz > kr ? nullptr : (t.rneg[ph] ? zneg : zpos) + zoff[kr];
          t.fmask[ph] = 1u | (t.lead_neg << 1) | (t.rneg[ph] ? 1u << (1 + kr) : 0u);
          t.nf[ph] = 0;
          for (int f = 0; f <= d; ++f)
            if ((t.fmask[ph] >> f) & 1) t.fidx[ph][t.nf[ph]++] = f;
        }
        t.zcp = zpos + zoff[kc];
        t.zcm = zneg + zoff[kc];
        t.cell_bits = pl.cell_bits;
        t.col_bits = pl.col_bits;
        FCG_TRY(launch_kde_zf(knots, d, m, centre, h, gl, zf, st));
        if (!all_run) {
          FCG_PROF("plane_kde", st);
          kde_kern<<<(unsigned)pl.NP, kKdeThreads, smem, st>>>(t, b.start, rec, n, skeys,
                                                               factored, lat);
          FCG_LAUNCH_CHECK();
        }
        Epi inplace;
        for (int ax = d - 3; ax >= (fuse01 ? 2 : 1); --ax)
          FCG_TRY(scan_axis<double>(lat, s, ax, rev[ax], inplace, scratch, st));
        f2.lat[tt] = lat;
        f2.zf[tt] = zf;
        f2.plane[tt] = planes ? planes + (int64_t)gl * plane_sz : nullptr;
        f2.plane_idx[tt] = planes ? (rev[1] ? 0 : m[1] - 1) : -1;
        f2.rev1[tt] = rev[1] ? 1 : 0;
        f.lat[tt] = lat;
        f.zf[tt] = zf;
        f.plane[tt] = planes ? planes + (int64_t)gl * plane_sz : nullptr;
        f.plane_idx[tt] = planes ? (rev[1] ? 0 : m[1] - 1) : -1;
      }
      f.accumulate = (s0 > 0 || b0 > 0) ? 1 : 0;
      f.apply_scale = (s0 == 1 && b0 + nt >= per0) ? 1 : 0;
      f.scale = scale;
      f.out = out;
      if (fuse01) {
        f2.nt = nt;
        f2.d = d;
        f2.kz = kz;
        for (int k = 0; k < d; ++k) {
          f2.zoff[k] = zoff[k];
          f2.dims[k] = m[k];
        }
        f2.accumulate = f.accumulate;
        f2.apply_scale = f.apply_scale;
        f2.scale = scale;
        f2.out = out;
        FCG_TRY(launch_final2d(f2, s0 == 1, st));
      } else {
        FCG_TRY(launch_final_multi(f, s0 == 1, st));
      }
    }
  }
  return FCG_OK;
}

}  // namespace fcg
