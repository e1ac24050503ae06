// Partitioned grid pipeline; see grid_part.cuh.
//
// Why: scattering 1e8 points with global atomics into a 1-2 GB lattice is random
// read-modify-write traffic (two 32-byte sectors per point, ~10x the useful bytes, measured at
// 12-16% of HBM peak).  Bucketing by plane first turns it into streaming: each CTA reads its
// bucket's records contiguously, accumulates in shared memory and writes its plane once, with
// the two in-plane scan passes (Algorithm 1's sweeps along axes d-2, d-1) fused in.
#include "grid_part.cuh"
#include "sort.cuh"

namespace fcg {

int launch_kde_zf(const double *knots, int d, const int64_t *m, const double *c, const double *h,
                  int code, double *zf, cudaStream_t st);

namespace {

constexpr uint32_t kDead = 0xFFFFFFFFu;
constexpr int kPlaneThreads = 512;
constexpr int kKdeThreads = 512;
constexpr size_t kEcdfTileBytes = 96 * 1024;   // int32 tile budget (2 CTAs per SM)
constexpr size_t kKdeTileBytes = 72 * 1024;    // fp64 row-block budget (3 CTAs per SM)
constexpr int64_t kMinPartitionN = int64_t(1) << 20;

struct PartGeo {
  int d;
  int64_t E[FCG_MAX_DIM];      // extents of the bucketed space
  int64_t shift[FCG_MAX_DIM];  // bucket-space index = b - shift
  int64_t W, R, nrb, H;
  int ecdf;                    // 1: val = in-block cell offset; 0: val = point index
};

template <int D>
__global__ void __launch_bounds__(256, 4) part_bin_kernel(const double *__restrict__ x, int64_t n,
                                                       int drt, const double *__restrict__ knots,
                                                       BinGrid g, PartGeo p,
                                                       uint32_t *__restrict__ keys,
                                                       int32_t *__restrict__ vals) {
  extern __shared__ double s_knots[];
  __shared__ double s_z0[FCG_MAX_DIM], s_idz[FCG_MAX_DIM];
  const int d = D > 0 ? D : drt;
  const double *kb = stage_knots(g, knots, s_knots, s_z0, s_idz);
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double xi[D > 0 ? D : FCG_MAX_DIM];
    if constexpr (D == 4) {
      const double2 v0 = reinterpret_cast<const double2 *>(x)[2 * i];
      const double2 v1 = reinterpret_cast<const double2 *>(x)[2 * i + 1];
      xi[0] = v0.x; xi[1] = v0.y; xi[2] = v1.x; xi[3] = v1.y;
    } else {
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : FCG_MAX_DIM); ++k)
        if (k < d) xi[k] = x[i * d + k];
    }
    uint32_t plane = 0;
    int row = 0, col = 0;
    bool live = true;
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : FCG_MAX_DIM); ++k) {
      if (k < d) {
        const int c = knot_count(xi[k], kb + g.koff[k], (int)g.m[k], g.le[k], s_z0[k], s_idz[k]) -
                      (int)p.shift[k];
        live = live && c >= 0 && c < (int)p.E[k];
        if (k < d - 2) plane = plane * (uint32_t)p.E[k] + (uint32_t)c;
        else if (k == d - 2) row = c;
        else col = c;
      }
    }
    uint32_t key = kDead;
    int32_t val = (int32_t)i;
    if (live) {
      const int rb = row / (int)p.R;
      key = plane * (uint32_t)p.nrb + (uint32_t)rb;
      if (p.ecdf) val = (row - rb * (int)p.R) * (int)p.W + col;
    }
    keys[i] = key;
    vals[i] = val;
  }
}

// start[b] = first sorted position whose key >= b, for b in [0, NB]
__global__ void bucket_start_kernel(const uint32_t *__restrict__ keys, int64_t n, int64_t NB,
                                    int32_t *__restrict__ start) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= NB;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)keys[mid] < b) lo = mid + 1;
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
__global__ void __launch_bounds__(kPlaneThreads, 2) plane_count_kernel(
    PartGeo p, const int32_t *__restrict__ start, const int32_t *__restrict__ vals, int rev_r,
    int rev_c, int32_t *__restrict__ lat) {
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
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int32_t q = qb + u * (int32_t)blockDim.x;
        v[u] = q < q1 ? vals[q] : -1;
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

// KDE term: CTA per cell-space plane.  Records are bucketed by full-space (M+1) row block; a
// term with row shift s reads full block rb as cell rows [rb*Rf - s, (rb+1)*Rf - s), so every
// cell row block comes from exactly one bucket.  Blocks are visited in the term's row scan
// direction with a carry row, like the ECDF plane kernel.
struct KdeTerm {
  int d;
  int64_t Mr, Mc;                    // cell extents of axes d-2, d-1
  int64_t sr, sc;                    // shifts (1 where delta = -1)
  int64_t Rf, nrb;                   // full-space rows per bucket block, blocks per plane
  int64_t lead_m[FCG_MAX_DIM];       // cell extents of leading axes
  int64_t lead_s[FCG_MAX_DIM];       // their shifts
  int64_t lead_full[FCG_MAX_DIM];    // full (M+1) extents of leading axes
  double c[FCG_MAX_DIM], a[FCG_MAX_DIM];
};

template <int SE>
__global__ void __launch_bounds__(kKdeThreads, 2) plane_kde_kernel(
    KdeTerm t, const int32_t *__restrict__ start, const double *__restrict__ rec,
    const uint32_t *__restrict__ loc, int factored, unsigned negmask, int rev_r, int rev_c,
    double *__restrict__ lat) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = (int)t.Mc, H = (int)t.Mr, Rf = (int)t.Rf;
  double *tile = reinterpret_cast<double *>(smem);
  double *carry = tile + (size_t)Rf * W;
  double *seg = carry + W;
  const int d = t.d;
  const int64_t cplane = blockIdx.x;
  int64_t rem = cplane, fplane = 0, mul = 1;
  for (int k = d - 3; k >= 0; --k) {
    const int64_t i = rem % t.lead_m[k];
    rem /= t.lead_m[k];
    fplane += (i + t.lead_s[k]) * mul;
    mul *= t.lead_full[k];
  }
  for (int c = threadIdx.x; c < W; c += blockDim.x) carry[c] = 0.0;
  double *plane_out = lat + cplane * H * W;
  for (int64_t rbi = 0; rbi < t.nrb; ++rbi) {
    const int64_t rb = rev_r ? t.nrb - 1 - rbi : rbi;
    int lo = (int)(rb * Rf - t.sr), hi = lo + Rf;
    const int clo = lo < 0 ? 0 : lo, chi = hi > H ? H : hi;
    if (chi <= clo) continue;
    const int nr = chi - clo;
    double *gtile = plane_out + (int64_t)clo * W;  // this block's rows of the lattice
    tile_zero<double>(tile, nr * W);
    __syncthreads();
    const int64_t b = fplane * t.nrb + rb;
    const int32_t q0 = start[b], q1 = start[b + 1];
    constexpr int KB = 2;
    for (int32_t qb = q0 + threadIdx.x; qb < q1; qb += KB * blockDim.x) {
      uint32_t l[KB];
      double psi[KB];  // loads of all KB records issued before the first atomic
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int32_t q = qb + u * (int32_t)blockDim.x;
        const bool ok = q < q1;
        l[u] = ok ? loc[q] : 0xFFFFFFFFu;
        const double *r = rec + (int64_t)(ok ? q : q0) * (d + 1);
        double v;
        if (factored) {
          v = r[0];
          for (int k = 0; k < d; ++k)
            if ((negmask >> k) & 1) v *= r[1 + k];
        } else {
          double sx = 0.0;
          for (int k = 0; k < d; ++k) sx += (r[k] - t.c[k]) * t.a[k];
          v = r[d] * exp(sx);
        }
        psi[u] = v;
      }
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int cr = (int)(l[u] >> 16) - (int)t.sr - clo;
        const int cc = (int)(l[u] & 0xFFFFu) - (int)t.sc;
        if (l[u] == 0xFFFFFFFFu || cr < 0 || cr >= nr || cc < 0 || cc >= W) continue;
        atomicAdd(&tile[cr * W + cc], psi[u]);  // fp64 shared atomic (CAS loop on sm_100)
      }
    }
    __syncthreads();
    tile_scan_any<double, SE>(tile, nr, W, rev_r, rev_c, carry, seg);
    tile_store<double>(gtile, tile, (int64_t)nr * W);
    __syncthreads();
  }
}

// gather the sorted records the KDE terms stream: the in-plane full-space offset packed as
// 16-bit (row, col), and either
//   factored (f != 0): rec[q] = (A, q_0..q_{d-1}) with A = w e^{sum_k u_k}, q_k = e^{-2 u_k},
//                      u_k = (x_k - c_k) / h_k, so term psi = A * prod_{k: delta_k=-1} q_k;
//   raw:               rec[q] = (x_0..x_{d-1}, w) and psi = w e^{sum_k delta_k u_k} per term.
// The factored form is used only when sum_k max|u_k| <= 600, which keeps every partial
// product inside e^{+-600} (fp64 overflows past e^709).
__global__ void kde_materialize_kernel(const double *__restrict__ x, const double *__restrict__ w,
                                       int64_t n, int d, const int32_t *__restrict__ order,
                                       const double *__restrict__ knots, BinGrid g, PsiParams pp,
                                       int factored, double *__restrict__ rec,
                                       uint32_t *__restrict__ loc) {
  extern __shared__ double s_knots[];
  __shared__ double s_z0[FCG_MAX_DIM], s_idz[FCG_MAX_DIM];
  const double *kb = stage_knots(g, knots, s_knots, s_z0, s_idz);
  __syncthreads();
  const int kr = d - 2, kc = d - 1;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = order[q];
    const double wi = w ? w[i] : 1.0;
    double *r = rec + q * (d + 1);
    if (factored) {
      double su = 0.0;
      for (int k = 0; k < d; ++k) {
        const double u = (x[i * d + k] - pp.c[k]) * pp.a[k];  // a_k = 1 / h_k
        su += u;
        r[1 + k] = exp(-2.0 * u);
      }
      r[0] = wi * exp(su);
    } else {
      for (int k = 0; k < d; ++k) r[k] = x[i * d + k];
      r[d] = wi;
    }
    const int br = knot_count(x[i * d + kr], kb + g.koff[kr], (int)g.m[kr], 0, s_z0[kr], s_idz[kr]);
    const int bc = knot_count(x[i * d + kc], kb + g.koff[kc], (int)g.m[kc], 0, s_z0[kc], s_idz[kc]);
    loc[q] = ((uint32_t)br << 16) | (uint32_t)bc;
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
  int64_t plane_idx;          // axis-1 index captured (-1: none)
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
#pragma unroll
        for (int t = 0; t < NT; ++t)
          if (t < f.nt) zo[t] *= f.zf[t][f.zoff[k] + i];
      }
    }
    const int64_t cap = (f.plane_idx >= 0 && b / B1 == f.plane_idx) ? b % B1 : -1;
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
            if (cap >= 0) f.plane[t][j * B1 + cap] = carry[t];
          }
        }
        double r = o[u] + val;
        if (f.apply_scale) r = r * f.scale;
        f.out[j * B + b] = r;
      }
    }
  }
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

int bits_for(int64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 32 && (int64_t(1) << b) <= v) ++b;
  return b;
}

int launch_part_bin(const double *x, int64_t n, int d, const double *knots, const BinGrid &g,
                    const PartGeo &p, uint32_t *keys, int32_t *vals, cudaStream_t st) {
  const size_t smem = g.total_knots <= kSmemKnots ? (size_t)g.total_knots * sizeof(double) : 0;
  const int grid = grid_for(n, 256, 8);
  FCG_PROF("part_bin", st);
  switch (d) {
    case 3: part_bin_kernel<3><<<grid, 256, smem, st>>>(x, n, d, knots, g, p, keys, vals); break;
    case 4:
      if ((reinterpret_cast<uintptr_t>(x) & 15) == 0)
        part_bin_kernel<4><<<grid, 256, smem, st>>>(x, n, d, knots, g, p, keys, vals);
      else
        part_bin_kernel<0><<<grid, 256, smem, st>>>(x, n, d, knots, g, p, keys, vals);
      break;
    default: part_bin_kernel<0><<<grid, 256, smem, st>>>(x, n, d, knots, g, p, keys, vals); break;
  }
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

struct PartBufs {
  uint32_t *keys;
  int32_t *vals;
  RadixWs rw;
  int32_t *start;
};

void carve_part(Workspace &W, PartBufs &b, int64_t n, int64_t NB) {
  b.keys = W.take<uint32_t>(n);
  b.vals = W.take<int32_t>(n);
  b.rw.keys_alt = reinterpret_cast<uint64_t *>(W.take<uint32_t>(n));
  b.rw.vals_alt = W.take<int32_t>(n);
  b.rw.hist = W.take<int32_t>(radix_ws_hist_elems(n));
  b.rw.partial = W.take<int32_t>(scan_ws_partial_elems(256 * (n / kSortTile + 1) + 2));
  b.start = W.take<int32_t>(NB + 1);
}

int partition(const double *x, int64_t n, int d, const double *knots, const BinGrid &g,
              const PartGeo &p, int64_t NB, int nbits, PartBufs &b, cudaStream_t st) {
  FCG_TRY(launch_part_bin(x, n, d, knots, g, p, b.keys, b.vals, st));
  FCG_TRY(radix_sort_pairs<uint32_t>(b.keys, b.vals, n, 0, ((nbits + 7) / 8) * 8, b.rw, st));
  FCG_PROF("part_bucket_start", st);
  bucket_start_kernel<<<grid_for(NB + 1, 256, 4), 256, 0, st>>>(b.keys, n, NB, b.start);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

}  // namespace

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
  p.nrb = pl.nrb;
  p.H = pl.H;
  p.ecdf = 1;
  FCG_TRY(partition(x, n, d, knots, g, p, pl.NB, pl.nbits, b, st));
  const int64_t G = seg_rows(kPlaneThreads, pl.W, 4);
  const size_t smem = (size_t)(pl.R * pl.W + pl.W + G * pl.W) * sizeof(int32_t);
  {
    FCG_PROF("plane_count", st);
    const int se = scan_variant(pl.W, 4);
    auto kern = se == 4 ? plane_count_kernel<4> : (se == 8 ? plane_count_kernel<8> : plane_count_kernel<0>);
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)pl.NP, kPlaneThreads, smem, st>>>(p, b.start, b.vals, rev[d - 2], rev[d - 1],
                                                      lat);
    FCG_LAUNCH_CHECK();
  }
  Epi inplace;
  for (int ax = d - 3; ax >= 1; --ax)
    FCG_TRY(scan_axis<int32_t>(lat, s, ax, rev[ax], inplace, scratch, st));
  return scan_axis<int32_t>(lat, s, 0, rev[0], epi, scratch, st);
}

PartPlan plan_kde_partition(int d, const int64_t *m, int64_t n) {
  PartPlan pl;
  if (d < 3 || n < kMinPartitionN) return pl;
  pl.W = m[d - 1];
  pl.H = m[d - 2];
  if (pl.W + 1 > 65535 || pl.H + 1 > 65535) return pl;  // packed 16-bit (row, col) offsets
  const int64_t G = seg_rows(kKdeThreads, pl.W, 2);
  const int64_t Hf = pl.H + 1;
  // fewest full-space row blocks whose tile fits the budget
  int64_t nrb = 1, Rf = Hf;
  while (true) {
    Rf = ceil_div(Hf, nrb);
    const size_t bytes = (size_t)(Rf * pl.W + pl.W + G * pl.W) * sizeof(double);
    if (bytes <= kKdeTileBytes) break;
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
  pl.nbits = bits_for(pl.NB);
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
  uint32_t *loc = W.take<uint32_t>(n);
  LatShape s;
  s.d = d;
  int64_t total_knots = 0;
  for (int k = 0; k < d; ++k) {
    s.dims[k] = m[k];
    total_knots += m[k];
  }
  // terms are processed in groups sharing (delta_0, delta_1); one lattice + zf table per member
  const int ntg = 1 << (d - 2);
  const int nbatch = ntg < kMaxGroup ? ntg : kMaxGroup;
  double *lats = W.take<double>((size_t)s.size() * nbatch);
  double *scratch = W.take<double>(scan_scratch_bound());
  double *zfs = W.take<double>((size_t)total_knots * nbatch);
  if (!run) return FCG_OK;

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
  p.nrb = pl.nrb;
  p.ecdf = 0;
  FCG_TRY(partition(x, n, d, knots, g, p, pl.NB, pl.nbits, b, st));
  // factored psi records when every partial product stays inside e^{+-600}: needs
  // sum_k max|u_k| <= 600 with u_k = (x_k - c_k)/h_k; bounded here by the hull of the knots
  // and the data (the caller's centre is that hull's midrange, fastsum.py:118-129)
  PsiParams pp{};
  for (int k = 0; k < d; ++k) {
    pp.c[k] = centre[k];
    pp.a[k] = 1.0 / h[k];
  }
  int factored = bound_u_sum <= 600.0 ? 1 : 0;
  {
    const size_t smem = g.total_knots <= kSmemKnots ? (size_t)g.total_knots * sizeof(double) : 0;
    FCG_PROF("kde_materialize", st);
    kde_materialize_kernel<<<grid_for(n, 256, 8), 256, smem, st>>>(x, w, n, d, b.vals, knots, g, pp,
                                                                  factored, rec, loc);
    FCG_LAUNCH_CHECK();
  }
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  const double scale = 1.0 / (std::ldexp(1.0, d) * n_scale * prod_h);
  const int64_t G = seg_rows(kKdeThreads, pl.W, 2);
  int64_t plane_sz = m[0];
  for (int k = 2; k < d; ++k) plane_sz *= m[k];
  const size_t smem = (size_t)(pl.R * pl.W + pl.W + G * pl.W) * sizeof(double);
  const int se = scan_variant(pl.W, 2);
  auto kde_kern = se == 2 ? plane_kde_kernel<2>
                          : (se == 4 ? plane_kde_kernel<4> : (se == 8 ? plane_kde_kernel<8> : plane_kde_kernel<0>));
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
  for (int grp = 0; grp < 4; ++grp) {
    for (int b0 = 0; b0 < ntg; b0 += nbatch) {
      const int nt = (ntg - b0) < nbatch ? (ntg - b0) : nbatch;
      MultiFinal f{};
      f.nt = nt;
      f.d = d;
      for (int k = 0; k < d; ++k) {
        f.zoff[k] = zoff[k];
        f.dims[k] = m[k];
      }
      const bool rev0 = grp & 1, rev1 = (grp >> 1) & 1;
      f.plane_idx = planes ? (rev1 ? 0 : m[1] - 1) : -1;
      for (int tt = 0; tt < nt; ++tt) {
        const int code = grp | ((b0 + tt) << 2);
        double *lat = lats + (size_t)tt * L;
        double *zf = zfs + (size_t)tt * total_knots;
        KdeTerm t{};
        t.d = d;
        bool rev[FCG_MAX_DIM];
        int64_t sh[FCG_MAX_DIM];
        for (int k = 0; k < d; ++k) {
          const double sgn = ((code >> k) & 1) ? -1.0 : 1.0;
          rev[k] = sgn < 0;
          sh[k] = sgn < 0 ? 1 : 0;
          t.c[k] = centre[k];
          t.a[k] = sgn / h[k];
        }
        t.Mr = m[d - 2];
        t.Mc = m[d - 1];
        t.sr = sh[d - 2];
        t.sc = sh[d - 1];
        t.Rf = pl.R;
        t.nrb = pl.nrb;
        for (int k = 0; k < d - 2; ++k) {
          t.lead_m[k] = m[k];
          t.lead_s[k] = sh[k];
          t.lead_full[k] = m[k] + 1;
        }
        FCG_TRY(launch_kde_zf(knots, d, m, centre, h, code, zf, st));
        {
          FCG_PROF("plane_kde", st);
          unsigned negmask = 0;
          for (int k = 0; k < d; ++k)
            if (rev[k]) negmask |= 1u << k;
          kde_kern<<<(unsigned)pl.NP, kKdeThreads, smem, st>>>(
              t, b.start, rec, loc, factored, negmask, rev[d - 2], rev[d - 1], lat);
          FCG_LAUNCH_CHECK();
        }
        Epi inplace;
        for (int ax = d - 3; ax >= 1; --ax)
          FCG_TRY(scan_axis<double>(lat, s, ax, rev[ax], inplace, scratch, st));
        f.lat[tt] = lat;
        f.zf[tt] = zf;
        f.plane[tt] = planes ? planes + (int64_t)code * plane_sz : nullptr;
      }
      f.accumulate = (grp > 0 || b0 > 0) ? 1 : 0;
      f.apply_scale = (grp == 3 && b0 + nt >= ntg) ? 1 : 0;
      f.scale = scale;
      f.out = out;
      FCG_TRY(launch_final_multi(f, rev0, st));
    }
  }
  return FCG_OK;
}

}  // namespace fcg
