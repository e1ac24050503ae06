// Grid path: fused per-point binning + scatter-add (subsystems 1-2 on a rectilinear grid),
// directional sweeps (subsystem 3) and the grid ECDF / ESF / Laplacian-KDE pipelines.
//
// Reference semantics followed:
//   * bin rule, histogram.py:3-15 and _flat_bins_uniform histogram.py:60-92: in dimension k a
//     point lands in bin b = #knots < x (delta_k = +1) or #knots <= x (delta_k = -1), b in
//     [0, M_k].  The device computes exactly that count from the uploaded knot values (a mesh
//     guess verified against the knots, binary search when the guess is off), never from
//     z0 + j*dz, so it is exact for any rectilinear grid and for points sitting on knots.
//   * ecdf_fastsum (fastsum.py:69-92): forward prefix sums over delta-binned local sums, the
//     j_k = M_k overflow layer is dropped, one division by N at the end.
//   * esf_fastsum (fastsum.py:95-111): equals "strictly above" = delta=+1 binning, suffix sums,
//     read one bin later (the reflection identity).
//   * _kde_exponential_fastsum Laplacian branch (fastsum.py:139-169,179-182).
//
// Dead-layer elision: for a forward axis the j = M_k layer never reaches an output, for a
// reverse axis the j = 0 layer never does (_delta_term_slices fastsum.py:132-136).  The fast
// pipelines therefore scatter into an exactly prod(M_k)-cell lattice (cell = b - shift_k,
// points falling in the dead layer are skipped) and the final scan pass writes the output in
// place of the reference's slice + copy.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "common.cuh"
#include "scan.cuh"
#include "bin.cuh"
#include "grid_part.cuh"

namespace fcg {

namespace {

template <int D, int WK, typename T>
__global__ void __launch_bounds__(256, 4) bin_scatter_kernel(const double *__restrict__ x,
                                                          int64_t n, int drt,
                                                          const double *__restrict__ w,
                                                          const double *__restrict__ knots,
                                                          BinGrid g, PsiParams pp,
                                                          T *__restrict__ lat) {
  extern __shared__ double s_knots[];
  __shared__ double s_z0[FCG_MAX_DIM], s_idz[FCG_MAX_DIM];
  const int d = D > 0 ? D : drt;
  const bool use_smem = g.total_knots <= kSmemKnots;
  if (use_smem)
    for (int64_t i = threadIdx.x; i < g.total_knots; i += blockDim.x) s_knots[i] = knots[i];
  if (threadIdx.x < d) {
    const int k = threadIdx.x;
    const double *kn = knots + g.koff[k];
    const int64_t m = g.m[k];
    s_z0[k] = kn[0];
    s_idz[k] = (m > 1) ? (double)(m - 1) / (kn[m - 1] - kn[0]) : 0.0;
  }
  __syncthreads();
  const double *kb = use_smem ? s_knots : knots;
  // uniform axes: points away from the mesh lines skip the knot verification (bin.cuh)
  const unsigned mesh = use_smem ? mesh_uniform(g, kb, s_z0, s_idz) : 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double xi[D > 0 ? D : FCG_MAX_DIM];
    if constexpr (D == 2) {
      const double2 v = reinterpret_cast<const double2 *>(x)[i];
      xi[0] = v.x;
      xi[1] = v.y;
    } else if constexpr (D == 4) {
      const double2 v0 = reinterpret_cast<const double2 *>(x)[2 * i];
      const double2 v1 = reinterpret_cast<const double2 *>(x)[2 * i + 1];
      xi[0] = v0.x; xi[1] = v0.y; xi[2] = v1.x; xi[3] = v1.y;
    } else {
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : FCG_MAX_DIM); ++k)
        if (k < d) xi[k] = x[i * d + k];
    }
    int64_t flat = 0;
    bool live = true;
#pragma unroll
    for (int k = 0; k < (D > 0 ? D : FCG_MAX_DIM); ++k) {
      if (k < d) {
        const int64_t b = knot_count(xi[k], kb + g.koff[k], (int)g.m[k], g.le[k], s_z0[k], s_idz[k],
                                     (mesh >> k) & 1u);
        const int64_t cell = b - g.shift[k];
        live = live && (cell >= 0) && (cell < g.dims[k]);
        flat += cell * g.stride[k];
      }
    }
    if (!live) continue;
    if constexpr (WK == W_UNIT) {
      atomicAdd(reinterpret_cast<int *>(lat) + flat, 1);
    } else if constexpr (WK == W_F64) {
      atomicAdd(reinterpret_cast<double *>(lat) + flat, w[i]);
    } else {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < (D > 0 ? D : FCG_MAX_DIM); ++k)
        if (k < d) s += (xi[k] - pp.c[k]) * pp.a[k];
      const double wi = w ? w[i] : 1.0;
      double v = wi * exp(s);
      if (pp.poly1 > 0) v = v * (xi[pp.poly1 - 1] - pp.c[pp.poly1 - 1]);  // w e xc_l
      atomicAdd(reinterpret_cast<double *>(lat) + flat, v);
    }
  }
}

// ---- one-launch pipeline for small 2-D lattices (BASELINE config 1: 256 x 256) ------------
// Launch-bound sizes spend more in launch gaps than in work (five kernels of a few microseconds
// each).  One cooperative kernel runs the whole ecdf_fastsum pipeline with grid-wide barriers:
// zero the lattice, bin + scatter (global atomics into an L2-resident lattice), scan every row
// along axis 1 (warp per row, shuffles), then the axis-0 pass as kSmallChunks row chunks:
// per-(chunk, column) totals, and each (chunk, column) thread adds the totals of the chunks
// before it (in scan order) and walks its rows writing the epilogue (count / N or int64).
constexpr int kSmallThreads = 256;
constexpr int kSmallChunks = 16;
constexpr int64_t kSmallCells = int64_t(1) << 20;

template <typename T, int EK>
__global__ void __launch_bounds__(kSmallThreads, 4) small2d_kernel(
    const double *__restrict__ x, int64_t n, const double *__restrict__ w,
    const double *__restrict__ knots, BinGrid g, int rev0, int rev1, T *__restrict__ lat,
    T *__restrict__ csum, Epi e, unsigned long long *trace) {
  namespace cg = cooperative_groups;
  auto stamp = [&](int i) {  // dev timing of the phases (trace != nullptr)
    if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[i] = t;
    }
  };
  stamp(0);
  extern __shared__ double s_knots[];
  __shared__ double s_z0[FCG_MAX_DIM], s_idz[FCG_MAX_DIM];
  const double *kb = stage_knots(g, knots, s_knots, s_z0, s_idz);
  // 32-bit indexing: the lattice has <= kSmallCells cells
  const int m0 = (int)g.dims[0], m1 = (int)g.dims[1], L = m0 * m1;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (int i = tid; i < L; i += nth) lat[i] = T(0);
  __syncthreads();
  cg::this_grid().sync();
  stamp(1);
  {
    const double *k0 = kb + g.koff[0], *k1 = kb + g.koff[1];
    const int M0 = (int)g.m[0], M1 = (int)g.m[1], le0 = g.le[0], le1 = g.le[1];
    const int sh0 = (int)g.shift[0], sh1 = (int)g.shift[1];
    const double z00 = s_z0[0], z01 = s_z0[1], i00 = s_idz[0], i01 = s_idz[1];
    for (int64_t i = tid; i < n; i += nth) {
      const double2 v = reinterpret_cast<const double2 *>(x)[i];
      const int c0 = knot_count(v.x, k0, M0, le0, z00, i00) - sh0;
      const int c1 = knot_count(v.y, k1, M1, le1, z01, i01) - sh1;
      if (c0 < 0 || c0 >= m0 || c1 < 0 || c1 >= m1) continue;
      if constexpr (sizeof(T) == 4) atomicAdd(reinterpret_cast<int *>(lat) + c0 * m1 + c1, 1);
      else atomicAdd(reinterpret_cast<double *>(lat) + c0 * m1 + c1, w[i]);
    }
  }
  cg::this_grid().sync();
  stamp(2);
  {  // axis 1: warp per row; rows of <= 256 columns load all 8 segments first (one round trip)
    const int lane = threadIdx.x & 31;
    for (int r = tid >> 5; r < m0; r += nth >> 5) {
      T *row = lat + r * m1;
      if (m1 <= 256) {
        T v[8];
#pragma unroll
        for (int sg = 0; sg < 8; ++sg) {
          const int jj = sg * 32 + lane;
          v[sg] = jj < m1 ? row[rev1 ? m1 - 1 - jj : jj] : T(0);
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
          for (int sg = 0; sg < 8; ++sg) {
            const T u = __shfl_up_sync(0xffffffffu, v[sg], o);
            if (lane >= o) v[sg] += u;
          }
        }
        T carry = T(0);
#pragma unroll
        for (int sg = 0; sg < 8; ++sg) {
          v[sg] += carry;
          carry = __shfl_sync(0xffffffffu, v[sg], 31);
          const int jj = sg * 32 + lane;
          if (jj < m1) row[rev1 ? m1 - 1 - jj : jj] = v[sg];
        }
        continue;
      }
      T carry = T(0);
      for (int j0 = 0; j0 < m1; j0 += 32) {
        const int j = rev1 ? m1 - 1 - (j0 + lane) : j0 + lane;
        const bool in = j0 + lane < m1;
        T v = in ? row[j] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const T u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        v += carry;
        if (in) row[j] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
      }
    }
  }
  cg::this_grid().sync();
  stamp(3);
  // axis 0: C chunks of Dc rows; loops of fixed trip count with independent loads
  const int C = m0 < kSmallChunks ? m0 : kSmallChunks;
  const int Dc = (m0 + C - 1) / C;
  for (int t = tid; t < C * m1; t += nth) {  // chunk totals along axis 0
    const int c = t / m1, col = t - c * m1;
    const int a = c * Dc, b = a + Dc < m0 ? a + Dc : m0;
    T s = T(0);
    for (int r0 = a; r0 < b; r0 += kSmallChunks) {
      T v[kSmallChunks];
#pragma unroll
      for (int u = 0; u < kSmallChunks; ++u) v[u] = r0 + u < b ? lat[(r0 + u) * m1 + col] : T(0);
#pragma unroll
      for (int u = 0; u < kSmallChunks; ++u) s += v[u];
    }
    csum[t] = s;
  }
  cg::this_grid().sync();
  stamp(4);
  double *of = static_cast<double *>(e.out);
  int64_t *oi = static_cast<int64_t *>(e.out);
  const double div = e.div, rdiv = e.div > 0.0 ? 1.0 / e.div : 0.0;
  for (int t = tid; t < C * m1; t += nth) {  // carry-in + walk (scan order) + epilogue
    const int c = t / m1, col = t - c * m1;
    // every load of the thread is issued before the first store (the output may alias the
    // lattice as far as the compiler knows, which would serialise load / store pairs)
    T cs[kSmallChunks];
#pragma unroll
    for (int q = 0; q < kSmallChunks; ++q) cs[q] = csum[(q < C ? q : 0) * m1 + col];
    T run = T(0);
#pragma unroll
    for (int q = 0; q < kSmallChunks; ++q)
      if (q < C && (rev0 ? q > c : q < c)) run += cs[q];
    const int a = c * Dc, b = a + Dc < m0 ? a + Dc : m0;
    for (int k0 = 0; k0 < b - a; k0 += kSmallChunks) {
      T v[kSmallChunks];
#pragma unroll
      for (int u = 0; u < kSmallChunks; ++u) {
        const int k = k0 + u;
        v[u] = k < b - a ? lat[(rev0 ? b - 1 - k : a + k) * m1 + col] : T(0);
      }
#pragma unroll
      for (int u = 0; u < kSmallChunks; ++u) {
        const int k = k0 + u;
        if (k >= b - a) break;
        run += v[u];
        const int f = (rev0 ? b - 1 - k : a + k) * m1 + col;
        if constexpr (EK == EPI_F64) {
          double vv = (double)run;
          if (div > 0.0) {
            // integer counts: the Markstein-corrected reciprocal is the IEEE quotient
            // (common.cuh div_rn, checked by tests/c/div_rn_check.c); weighted sums divide
            if constexpr (sizeof(T) == 4) vv = div_rn(vv, div, rdiv);
            else vv = vv / div;
          }
          of[f] = vv;
        } else {
          oi[f] = (int64_t)run;
        }
      }
    }
  }
  if (trace) {
    cg::this_grid().sync();
    stamp(5);
  }
}

template <typename T, int EK>
int launch_small2d(const double *x, int64_t n, const double *w, const double *knots,
                   const BinGrid &g, bool rev0, bool rev1, T *lat, T *csum, const Epi &e,
                   cudaStream_t st) {
  auto kern = small2d_kernel<T, EK>;
  const size_t smem = g.total_knots <= kSmemKnots ? (size_t)g.total_knots * sizeof(double) : 0;
  // residency of the cooperative grid (a per-instantiation constant: knots <= kSmemKnots use
  // at most 32 KB of shared memory, so the 32 KB figure bounds every launch)
  static int per_sm = -1;
  if (per_sm < 0) {
    int v = 0;
    FCG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kSmallThreads,
                                                               kSmemKnots * sizeof(double)));
    per_sm = v;
  }
  if (per_sm < 1) return fail(FCG_ECUDA, "small2d kernel cannot be resident");
  const int64_t L = g.dims[0] * g.dims[1];
  // few blocks: the grid barriers' cost grows with the block count, the phases are tiny
  static const int64_t per_thread = getenv("FCG_SMALL_PER_THREAD") ? atoll(getenv("FCG_SMALL_PER_THREAD")) : 4;
  const int64_t work = std::max<int64_t>(std::max<int64_t>(n, L / 4), 1);
  int64_t blocks = std::min<int64_t>(ceil_div(work, kSmallThreads * per_thread),
                                     (int64_t)per_sm * sm_count());
  blocks = std::max<int64_t>(blocks, 1);
  int r0 = rev0 ? 1 : 0, r1 = rev1 ? 1 : 0;
  // FCG_SMALL_TRACE=1 (dev): phase timestamps, printed after the launch (synchronises)
  static unsigned long long *trace = nullptr;
  static const bool want_trace = getenv("FCG_SMALL_TRACE") && getenv("FCG_SMALL_TRACE")[0] == '1';
  if (want_trace && !trace) FCG_CUDA_TRY(cudaMalloc(&trace, 8 * sizeof(unsigned long long)));
  void *args[] = {(void *)&x, (void *)&n, (void *)&w, (void *)&knots, (void *)&g, (void *)&r0,
                  (void *)&r1, (void *)&lat, (void *)&csum, (void *)&e, (void *)&trace};
  FCG_PROF(sizeof(T) == 4 ? "small2d_count" : "small2d_w", st);
  FCG_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)blocks),
                                           dim3(kSmallThreads), args, smem, st));
  if (trace) {
    unsigned long long h[8];
    FCG_CUDA_TRY(cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    FCG_CUDA_TRY(cudaStreamSynchronize(st));
    fprintf(stderr, "small2d blocks=%lld phases(us):", (long long)blocks);
    for (int i = 1; i <= 5; ++i) fprintf(stderr, " %.2f", (h[i] - h[i - 1]) * 1e-3);
    fprintf(stderr, "\n");
  }
  return FCG_OK;
}

template <int WK, typename T>
int launch_bin_scatter(const double *x, int64_t n, int d, const double *w, const double *knots,
                       const BinGrid &g, const PsiParams &pp, T *lat, cudaStream_t st) {
  if (n == 0) return FCG_OK;
  const int grid = grid_for(n, 256, 8);
  const size_t smem = g.total_knots <= kSmemKnots ? (size_t)g.total_knots * sizeof(double) : 0;
  const bool vec_ok = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  FCG_PROF(WK == W_UNIT ? "bin_scatter_count" : (WK == W_F64 ? "bin_scatter_w" : "bin_scatter_psi"), st);
  switch (d) {
    case 1: bin_scatter_kernel<1, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat); break;
    case 2:
      if (vec_ok) bin_scatter_kernel<2, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat);
      else bin_scatter_kernel<0, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat);
      break;
    case 3: bin_scatter_kernel<3, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat); break;
    case 4:
      if (vec_ok) bin_scatter_kernel<4, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat);
      else bin_scatter_kernel<0, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat);
      break;
    default: bin_scatter_kernel<0, WK, T><<<grid, 256, smem, st>>>(x, n, d, w, knots, g, pp, lat); break;
  }
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

int check_common(int64_t n, int32_t d, const int64_t *m) {
  if (d < 1 || d > FCG_MAX_DIM)
    return fail(FCG_EUNSUPPORTED, "dimension d must be in [1, " + std::to_string(FCG_MAX_DIM) + "]");
  if (n < 0) return fail(FCG_EINVAL, "n must be >= 0");
  if (n >= (int64_t(1) << 31)) return fail(FCG_EUNSUPPORTED, "n must be < 2^31");
  for (int k = 0; k < d; ++k)
    if (m[k] < 1) return fail(FCG_EINVAL, "every dimension needs at least one knot");
  return FCG_OK;
}

// ---- KDE helpers -------------------------------------------------------------------------

// zf[koff_k + j] = exp(-delta_k * (knot_kj - c_k) / h_k)   (fastsum.py:162-166)
struct ZfParams {
  int d;
  int64_t m[FCG_MAX_DIM], koff[FCG_MAX_DIM];
  double c[FCG_MAX_DIM], h[FCG_MAX_DIM], s[FCG_MAX_DIM];
};

__global__ void zf_kernel(const double *__restrict__ knots, ZfParams p, double *__restrict__ zf,
                          int64_t total) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < p.d && i >= p.koff[k + 1]) ++k;
    const double zc = knots[i] - p.c[k];
    zf[i] = exp((-p.s[k] * zc) / p.h[k]);
  }
}

// ---- min / max ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ord_key(double v) { return f64_key(v); }
__device__ __forceinline__ double ord_val(uint64_t k) {
  uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

__global__ void minmax_init(unsigned long long *mm, int d) {
  int k = threadIdx.x;
  if (k < d) {
    mm[k] = ~0ull;
    mm[d + k] = 0ull;
  }
}

// x is read as a flat stream of n*d doubles, VEC per load; the grid's total stride is a
// multiple of d, so each thread's VEC lanes always hold the same components k0..k0+VEC-1
// (mod d) and it keeps one (lo, hi) pair per lane -- coalesced, no per-point component loop.
template <int VEC>
__global__ void __launch_bounds__(256) minmax_kernel(const double *__restrict__ x, int64_t total,
                                                     int d, unsigned long long *mm) {
  __shared__ unsigned long long s_lo[FCG_MAX_DIM], s_hi[FCG_MAX_DIM];
  if (threadIdx.x < FCG_MAX_DIM) {
    s_lo[threadIdx.x] = ~0ull;
    s_hi[threadIdx.x] = 0ull;
  }
  __syncthreads();
  uint64_t lo[VEC], hi[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    lo[v] = ~0ull;
    hi[v] = 0ull;
  }
  const int64_t t0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * VEC;
  for (int64_t j = t0; j < total; j += stride) {
    if (VEC == 2 && j + 1 < total) {
      const double2 p = __ldcs(reinterpret_cast<const double2 *>(x + j));
      const uint64_t a = ord_key(p.x), b = ord_key(p.y);
      lo[0] = a < lo[0] ? a : lo[0];
      hi[0] = a > hi[0] ? a : hi[0];
      lo[VEC - 1] = b < lo[VEC - 1] ? b : lo[VEC - 1];
      hi[VEC - 1] = b > hi[VEC - 1] ? b : hi[VEC - 1];
    } else {
      const uint64_t a = ord_key(x[j]);
      lo[0] = a < lo[0] ? a : lo[0];
      hi[0] = a > hi[0] ? a : hi[0];
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    const int k = (int)((t0 + v) % d);
    atomicMin(s_lo + k, (unsigned long long)lo[v]);  // idle lanes hold the identities
    atomicMax(s_hi + k, (unsigned long long)hi[v]);
  }
  __syncthreads();
  if (threadIdx.x < d) {
    atomicMin(mm + threadIdx.x, s_lo[threadIdx.x]);
    atomicMax(mm + d + threadIdx.x, s_hi[threadIdx.x]);
  }
}

__global__ void minmax_finish(const unsigned long long *mm, int d, double *out) {
  int k = threadIdx.x;
  if (k < 2 * d) out[k] = ord_val(mm[k]);
}

}  // namespace

int launch_kde_zf(const double *knots, int d, const int64_t *m, const double *c, const double *h,
                  int code, double *zf, cudaStream_t st) {
  ZfParams zp{};
  zp.d = d;
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    zp.m[k] = m[k];
    zp.koff[k] = off;
    off += m[k];
    zp.c[k] = c[k];
    zp.h[k] = h[k];
    zp.s[k] = ((code >> k) & 1) ? -1.0 : 1.0;
  }
  FCG_PROF("kde_zfac", st);
  zf_kernel<<<grid_for(off, 256, 1), 256, 0, st>>>(knots, zp, zf, off);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

// ============================================================================================
// C-ABI entry points
// ============================================================================================

}  // namespace fcg

using namespace fcg;

extern "C" int fcg_local_sums(const double *x, int64_t n, int32_t d, const double *w,
                              const double *knots, const int64_t *m, const int32_t *delta,
                              int32_t lat_kind, void *lattice, void *ws, size_t *ws_bytes,
                              void *stream) {
  FCG_TRY(check_common(n, d, m));
  if (lat_kind == FCG_LAT_I32 && w != nullptr)
    return fail(FCG_EINVAL, "int32 lattices hold unit-weight counts only (pass w = NULL)");
  if (ws == nullptr) {
    *ws_bytes = 256;
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  int le[FCG_MAX_DIM];
  int64_t shift[FCG_MAX_DIM], dims[FCG_MAX_DIM];
  int64_t L = 1;
  for (int k = 0; k < d; ++k) {
    if (delta[k] != 1 && delta[k] != -1) return fail(FCG_EINVAL, "delta entries must be -1 or +1");
    le[k] = delta[k] < 0;
    shift[k] = 0;
    dims[k] = m[k] + 1;  // full (M_k+1) lattice incl. the overflow layer (histogram.py:27-31)
    L *= dims[k];
  }
  BinGrid g = make_bin_grid(d, m, le, shift, dims);
  PsiParams pp{};
  const size_t esz = lat_kind == FCG_LAT_I32 ? 4 : 8;
  FCG_CUDA_TRY(cudaMemsetAsync(lattice, 0, (size_t)L * esz, st));
  if (lat_kind == FCG_LAT_I32)
    return launch_bin_scatter<W_UNIT>(x, n, d, w, knots, g, pp, static_cast<int32_t *>(lattice), st);
  return launch_bin_scatter<W_F64>(x, n, d, w, knots, g, pp, static_cast<double *>(lattice), st);
}

extern "C" int fcg_directional_sweep(void *lattice, int32_t lat_kind, int32_t d,
                                     const int64_t *dims, const int32_t *delta, void *ws,
                                     size_t *ws_bytes, void *stream) {
  if (d < 1 || d > FCG_MAX_DIM) return fail(FCG_EUNSUPPORTED, "dimension out of range");
  LatShape s;
  s.d = d;
  for (int k = 0; k < d; ++k) {
    if (dims[k] < 1) return fail(FCG_EINVAL, "lattice extents must be >= 1");
    s.dims[k] = dims[k];
  }
  const size_t esz = lat_kind == FCG_LAT_I32 ? 4 : 8;
  Workspace W(ws);
  void *scratch = W.take<char>((size_t)scan_scratch_elems(s) * esz);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  bool rev[FCG_MAX_DIM];
  for (int k = 0; k < d; ++k) {
    if (delta[k] != 1 && delta[k] != -1) return fail(FCG_EINVAL, "delta entries must be -1 or +1");
    rev[k] = delta[k] < 0;
  }
  Epi e;  // in place
  cudaStream_t st = as_stream(stream);
  if (lat_kind == FCG_LAT_I32)
    return scan_lattice<int32_t>(static_cast<int32_t *>(lattice), s, rev, e,
                                 static_cast<int32_t *>(scratch), st);
  return scan_lattice<double>(static_cast<double *>(lattice), s, rev, e,
                              static_cast<double *>(scratch), st);
}

extern "C" int fcg_ecdf_grid(const double *x, int64_t n, int32_t d, const double *w,
                             const double *knots, const int64_t *m, const int32_t *delta,
                             int32_t survival, int32_t scaled, int32_t out_kind, void *out,
                             void *ws, size_t *ws_bytes, void *stream) {
  FCG_TRY(check_common(n, d, m));
  if (out_kind == 1 && w != nullptr)
    return fail(FCG_EINVAL, "int64 count output requires unit weights (w = NULL)");
  LatShape s;
  s.d = d;
  for (int k = 0; k < d; ++k) s.dims[k] = m[k];
  const int64_t L = s.size();
  const bool unit = (w == nullptr);
  const size_t esz = unit ? 4 : 8;
  int le[FCG_MAX_DIM];
  int64_t shift[FCG_MAX_DIM];
  bool rev[FCG_MAX_DIM];
  for (int k = 0; k < d; ++k) {
    if (!survival && delta[k] != 1 && delta[k] != -1)
      return fail(FCG_EINVAL, "delta entries must be -1 or +1");
    if (survival) {  // strictly above: #knots < x binning, suffix sums read one bin later
      le[k] = 0;
      shift[k] = 1;
      rev[k] = true;
    } else {
      le[k] = delta[k] < 0;
      shift[k] = 0;
      rev[k] = false;
    }
  }
  BinGrid g = make_bin_grid(d, m, le, shift, s.dims);
  Epi e;
  e.kind = out_kind == 1 ? EPI_I64 : EPI_F64;
  e.out = out;
  e.div = scaled ? (double)n : 0.0;
  e.rdiv = scaled ? 1.0 / (double)n : 0.0;
  cudaStream_t st = as_stream(stream);
  Workspace W(ws);
  // unit weights at scale: plane-partitioned pipeline (grid_part.cu)
  const PartPlan plan = unit ? plan_ecdf_partition(g, n) : PartPlan{};
  if (plan.ok) {
    FCG_TRY(ecdf_partitioned(x, n, knots, g, rev, plan, e, W, ws != nullptr, st));
    if (ws == nullptr) *ws_bytes = W.bytes();
    return FCG_OK;
  }
  void *lat = W.take<char>((size_t)L * esz);
  void *scratch = W.take<char>((size_t)scan_scratch_elems(s) * esz);
  // small 2-D lattices: the whole pipeline in one cooperative launch
  const bool small = d == 2 && L <= kSmallCells && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                     !(getenv("FCG_SMALL2D") && getenv("FCG_SMALL2D")[0] == '0');
  void *csum = small ? W.take<char>((size_t)kSmallChunks * m[1] * esz) : nullptr;
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (small) {
    if (unit)
      return e.kind == EPI_I64
                 ? launch_small2d<int32_t, EPI_I64>(x, n, w, knots, g, rev[0], rev[1],
                                                    static_cast<int32_t *>(lat),
                                                    static_cast<int32_t *>(csum), e, st)
                 : launch_small2d<int32_t, EPI_F64>(x, n, w, knots, g, rev[0], rev[1],
                                                    static_cast<int32_t *>(lat),
                                                    static_cast<int32_t *>(csum), e, st);
    return launch_small2d<double, EPI_F64>(x, n, w, knots, g, rev[0], rev[1],
                                           static_cast<double *>(lat), static_cast<double *>(csum),
                                           e, st);
  }
  PsiParams pp{};
  {
    FCG_PROF("lattice_zero", st);
    FCG_CUDA_TRY(cudaMemsetAsync(lat, 0, (size_t)L * esz, st));
  }
  if (unit) {
    FCG_TRY(launch_bin_scatter<W_UNIT>(x, n, d, w, knots, g, pp, static_cast<int32_t *>(lat), st));
    return scan_lattice<int32_t>(static_cast<int32_t *>(lat), s, rev, e,
                                 static_cast<int32_t *>(scratch), st);
  }
  FCG_TRY(launch_bin_scatter<W_F64>(x, n, d, w, knots, g, pp, static_cast<double *>(lat), st));
  return scan_lattice<double>(static_cast<double *>(lat), s, rev, e,
                              static_cast<double *>(scratch), st);
}

namespace fcg {
// widen the order-key hull mm[0..2d) by the n points of x
static int launch_minmax_accum(const double *x, int64_t n, int d, unsigned long long *mm,
                               cudaStream_t st) {
  if (n <= 0) return FCG_OK;
  // grid: a multiple of d blocks (so the flat stride is a multiple of d), ~4 per SM
  const int64_t total = n * d;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t per = vec ? 512 : 256;
  int64_t blocks = std::min<int64_t>(ceil_div(total, per), 4 * (int64_t)sm_count());
  blocks = ceil_div(blocks, d) * d;
  if (vec)
    minmax_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(x, total, d, mm);
  else
    minmax_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(x, total, d, mm);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}
}  // namespace fcg

extern "C" int fcg_minmax(const double *x, int64_t n, int32_t d, double *out_minmax, void *ws,
                          size_t *ws_bytes, void *stream) {
  if (d < 1 || d > FCG_MAX_DIM) return fail(FCG_EUNSUPPORTED, "dimension out of range");
  Workspace W(ws);
  unsigned long long *mm = W.take<unsigned long long>(2 * d);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  FCG_PROF("minmax", st);
  minmax_init<<<1, 32, 0, st>>>(mm, d);
  FCG_LAUNCH_CHECK();
  FCG_TRY(launch_minmax_accum(x, n, d, mm, st));
  minmax_finish<<<1, 32, 0, st>>>(mm, d, out_minmax);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

namespace fcg {

// Laplacian grid KDE (fastsum.py:139-169,179-182).  n_scale: N of the normalisation;
// planes: optional per-term slab-boundary plane capture (see fcg_kde_grid_laplacian_ex).
static int kde_grid_impl(const double *x, int64_t n, int32_t d, const double *w,
                         const double *knots, const int64_t *m, const double *h,
                         const double *centre, double n_scale, double u_bound, double *planes,
                         double *out, void *ws, size_t *ws_bytes, void *stream) {
  FCG_TRY(check_common(n, d, m));
  LatShape s;
  s.d = d;
  int64_t total_knots = 0;
  for (int k = 0; k < d; ++k) {
    s.dims[k] = m[k];
    total_knots += m[k];
  }
  const int64_t L = s.size();
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  if (planes && d < 2) return fail(FCG_EINVAL, "slab planes need d >= 2");
  cudaStream_t st = as_stream(stream);
  Workspace W(ws);
  // auto centre: plan for factored records (the hull decides at run time)
  const bool auto_centre = centre == nullptr;
  const PartPlan plan =
      plan_kde_partition(d, m, n, auto_centre || (u_bound > 0.0 && u_bound <= 600.0));
  if (plan.ok) {
    FCG_TRY(kde_partitioned(x, n, w, knots, m, d, h, centre, u_bound > 0.0 ? u_bound : 1e300,
                            n_scale, planes, plan, out, W, ws != nullptr, st));
    if (ws == nullptr) *ws_bytes = W.bytes();
    return FCG_OK;
  }
  double *lat = W.take<double>((size_t)L);
  double *scratch = W.take<double>((size_t)scan_scratch_elems(s));
  double *zf = W.take<double>((size_t)total_knots);
  unsigned long long *mm = W.take<unsigned long long>(2 * FCG_MAX_DIM);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  double c_auto[FCG_MAX_DIM];
  if (auto_centre) {
    FCG_TRY(hull_init(knots, d, m, mm, st));
    FCG_TRY(launch_minmax_accum(x, n, d, mm, st));
    FCG_TRY(hull_centre(mm, d, h, c_auto, &u_bound, st));
    centre = c_auto;
  }
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  const double scale = 1.0 / (std::ldexp(1.0, d) * n_scale * prod_h);
  int64_t plane_sz = m[0];
  for (int k = 2; k < d; ++k) plane_sz *= m[k];
  const int ncodes = 1 << d;
  for (int code = 0; code < ncodes; ++code) {
    int le[FCG_MAX_DIM];
    int64_t shift[FCG_MAX_DIM];
    bool rev[FCG_MAX_DIM];
    PsiParams pp{};
    for (int k = 0; k < d; ++k) {
      const double sgn = ((code >> k) & 1) ? -1.0 : 1.0;  // DeltaVector.from_code, core.py:165-168
      le[k] = 0;                                       // one delta=+1 binning for every term
      shift[k] = sgn < 0 ? 1 : 0;                      // -1 axes read [1:M+1]
      rev[k] = sgn < 0;
      pp.c[k] = centre[k];
      pp.a[k] = sgn / h[k];
    }
    BinGrid g = make_bin_grid(d, m, le, shift, s.dims);
    FCG_TRY(launch_kde_zf(knots, d, m, centre, h, code, zf, st));
    {
      FCG_PROF("lattice_zero", st);
      FCG_CUDA_TRY(cudaMemsetAsync(lat, 0, (size_t)L * sizeof(double), st));
    }
    FCG_TRY(launch_bin_scatter<W_PSI>(x, n, d, w, knots, g, pp, lat, st));
    Epi e;
    e.kind = EPI_KDE;
    e.out = out;
    e.zf = zf;
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      e.zoff[k] = off;
      off += m[k];
    }
    e.accumulate = code > 0;
    e.apply_scale = code == ncodes - 1;
    e.scale = scale;
    if (planes) {
      e.plane_out = planes + (int64_t)code * plane_sz;
      e.plane_idx = rev[1] ? 0 : m[1] - 1;
      e.cap_kw = kde_cap_kw(d);
    }
    FCG_TRY(scan_lattice<double>(lat, s, rev, e, scratch, st));
  }
  return FCG_OK;
}

namespace {
// matern32-additive term (fastsum.py:170-178): with S_0 the sweep of w e and S_l that of
// w e xc_l,  acc = coef * S_0 - sum_l (delta_l / h_l) S_l,  coef = 1 + sum_k delta_k zc_k / h_k,
// out (+)= zfac * acc, times the final scale after the last term.
struct MaternP {
  int d;
  int64_t dims[FCG_MAX_DIM], zoff[FCG_MAX_DIM];
  double sgn[FCG_MAX_DIM], c[FCG_MAX_DIM], h[FCG_MAX_DIM];
  int accumulate, apply_scale;
  double scale;
};

__global__ void matern_combine_kernel(double *__restrict__ out, const double *__restrict__ S,
                                      int64_t L, const double *__restrict__ zf,
                                      const double *__restrict__ knots, MaternP p) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < L;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx[FCG_MAX_DIM];
    int64_t rem = t;
    for (int k = p.d - 1; k >= 0; --k) {
      idx[k] = rem % p.dims[k];
      rem /= p.dims[k];
    }
    double zfac = 1.0, coef = 1.0;
    for (int k = 0; k < p.d; ++k) {
      zfac = zfac * zf[p.zoff[k] + idx[k]];
      coef = coef + (p.sgn[k] * (knots[p.zoff[k] + idx[k]] - p.c[k])) / p.h[k];
    }
    double acc = coef * S[t];
    for (int l = 0; l < p.d; ++l) acc -= (p.sgn[l] / p.h[l]) * S[(int64_t)(l + 1) * L + t];
    double r = zfac * acc;
    if (p.accumulate) r = out[t] + r;
    if (p.apply_scale) r = r * p.scale;
    out[t] = r;
  }
}

// out[i] += scale * sum_code zfac_code(i) * C_code[i0, i2, ..]   (slab carry fix-up)
struct FixP {
  int d, ncodes, kw;  // zf of axes k < kw (the captured planes carry the rest)
  int64_t dims[FCG_MAX_DIM];
  int64_t zoff[FCG_MAX_DIM];
  int64_t zsz;        // entries per code in zf
  int64_t plane_sz;   // entries per code in C
  double scale;
};

// Q[b1][pi] = sum over the codes with delta_1 bit b1 of prod_{k<kw, k!=1} zf_code,k(i_k) * C_code[pi]
// (pi = (i0, i2, ..)): the carry planes folded per axis-1 sign, so the lattice pass needs two
// plane reads per element instead of one per code.
__global__ void kde_fixup_fold_kernel(FixP p, const double *__restrict__ zf,
                                      const double *__restrict__ C, double *__restrict__ Q) {
  for (int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pi < p.plane_sz;
       pi += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx[FCG_MAX_DIM];
    int64_t rem = pi;
    for (int k = p.d - 1; k >= 2; --k) {
      idx[k] = rem % p.dims[k];
      rem /= p.dims[k];
    }
    idx[0] = rem;
    double q0 = 0.0, q1 = 0.0;
    for (int code = 0; code < p.ncodes; ++code) {
      const double *z = zf + code * p.zsz;
      double zz = 1.0;
      for (int k = 0; k < p.kw; ++k)
        if (k != 1) zz *= z[p.zoff[k] + idx[k]];
      const double v = zz * C[code * p.plane_sz + pi];
      if ((code >> 1) & 1) q1 += v;
      else q0 += v;
    }
    Q[pi] = q0;
    Q[p.plane_sz + pi] = q1;
  }
}

// out[i] += scale * (zf_{+,1}(i1) Q[0][pi] + zf_{-,1}(i1) Q[1][pi])
__global__ void kde_fixup_kernel(double *__restrict__ out, FixP p, const double *__restrict__ z1p,
                                 const double *__restrict__ z1m, const double *__restrict__ Q) {
  int64_t L = 1;
  for (int k = 0; k < p.d; ++k) L *= p.dims[k];
  const int64_t B = p.plane_sz / p.dims[0];  // extent of the axes 2..d-1
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < L;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t % B;
    const int64_t r = t / B;
    const int64_t i1 = r % p.dims[1];
    const int64_t i0 = r / p.dims[1];
    const int64_t pi = i0 * B + b;
    out[t] += p.scale * (z1p[i1] * Q[pi] + z1m[i1] * Q[p.plane_sz + pi]);
  }
}
}  // namespace

}  // namespace fcg

extern "C" int fcg_kde_grid_laplacian(const double *x, int64_t n, int32_t d, const double *w,
                                      const double *knots, const int64_t *m, const double *h,
                                      const double *centre, double *out, void *ws,
                                      size_t *ws_bytes, void *stream) {
  return kde_grid_impl(x, n, d, w, knots, m, h, centre, (double)n, -1.0, nullptr, out, ws,
                       ws_bytes, stream);
}

extern "C" int fcg_kde_grid_laplacian_ex(const double *x, int64_t n, int32_t d, const double *w,
                                         const double *knots, const int64_t *m, const double *h,
                                         const double *centre, double n_scale, double u_bound,
                                         double *planes, double *out, void *ws, size_t *ws_bytes,
                                         void *stream) {
  return kde_grid_impl(x, n, d, w, knots, m, h, centre, n_scale, u_bound, planes, out, ws,
                       ws_bytes, stream);
}

extern "C" int fcg_kde_grid_matern32(const double *x, int64_t n, int32_t d, const double *w,
                                     const double *knots, const int64_t *m, const double *h,
                                     const double *centre, double *out, void *ws,
                                     size_t *ws_bytes, void *stream) {
  FCG_TRY(check_common(n, d, m));
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  LatShape s;
  s.d = d;
  int64_t total_knots = 0;
  for (int k = 0; k < d; ++k) {
    s.dims[k] = m[k];
    total_knots += m[k];
  }
  const int64_t L = s.size();
  Workspace W(ws);
  double *S = W.take<double>((size_t)L * (d + 1));  // S_0 .. S_d of the current term
  double *scratch = W.take<double>((size_t)scan_scratch_elems(s));
  double *zf = W.take<double>((size_t)total_knots);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (L == 0) return FCG_OK;
  cudaStream_t st = as_stream(stream);
  // scale = 1 / (2^d n prod h), then / (1 + d)   (fastsum.py:179-181)
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  double scale = 1.0 / (std::ldexp(1.0, d) * (double)n * prod_h);
  scale /= 1.0 + d;
  const int ncodes = 1 << d;
  for (int code = 0; code < ncodes; ++code) {
    int le[FCG_MAX_DIM];
    int64_t shift[FCG_MAX_DIM];
    bool rev[FCG_MAX_DIM];
    PsiParams pp{};
    MaternP mp{};
    mp.d = d;
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      const double sgn = ((code >> k) & 1) ? -1.0 : 1.0;  // DeltaVector.from_code
      le[k] = 0;
      shift[k] = sgn < 0 ? 1 : 0;
      rev[k] = sgn < 0;
      pp.c[k] = centre[k];
      pp.a[k] = sgn / h[k];
      mp.dims[k] = m[k];
      mp.zoff[k] = off;
      off += m[k];
      mp.sgn[k] = sgn;
      mp.c[k] = centre[k];
      mp.h[k] = h[k];
    }
    BinGrid g = make_bin_grid(d, m, le, shift, s.dims);
    FCG_TRY(launch_kde_zf(knots, d, m, centre, h, code, zf, st));
    Epi inplace;
    for (int ch = 0; ch <= d; ++ch) {  // channel 0: w e; channel l: w e xc_{l-1}
      double *lat = S + (int64_t)ch * L;
      {
        FCG_PROF("lattice_zero", st);
        FCG_CUDA_TRY(cudaMemsetAsync(lat, 0, (size_t)L * sizeof(double), st));
      }
      pp.poly1 = ch;
      if (n > 0) FCG_TRY(launch_bin_scatter<W_PSI>(x, n, d, w, knots, g, pp, lat, st));
      FCG_TRY(scan_lattice<double>(lat, s, rev, inplace, scratch, st));
    }
    mp.accumulate = code > 0;
    mp.apply_scale = code == ncodes - 1;
    mp.scale = scale;
    FCG_PROF("kde_matern_combine", st);
    matern_combine_kernel<<<grid_for(L, 256), 256, 0, st>>>(out, S, L, zf, knots, mp);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}

extern "C" int fcg_kde_carry_fixup(double *out, int32_t d, const int64_t *m, const double *knots,
                                   const double *h, const double *centre, const double *planes,
                                   double n_scale, void *ws, size_t *ws_bytes, void *stream) {
  if (d < 2 || d > FCG_MAX_DIM) return fail(FCG_EINVAL, "dimension out of range");
  int64_t total_knots = 0;
  for (int k = 0; k < d; ++k) total_knots += m[k];
  const int ncodes = 1 << d;
  int64_t L = 1;
  for (int k = 0; k < d; ++k) L *= m[k];
  Workspace W(ws);
  double *zf = W.take<double>((size_t)ncodes * total_knots);
  double *Q = W.take<double>((size_t)2 * (L / (m[1] > 0 ? m[1] : 1)));
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  for (int code = 0; code < ncodes; ++code)
    FCG_TRY(launch_kde_zf(knots, d, m, centre, h, code, zf + (int64_t)code * total_knots, st));
  FixP p{};
  p.d = d;
  p.ncodes = ncodes;
  p.kw = kde_cap_kw(d);
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    p.dims[k] = m[k];
    p.zoff[k] = off;
    off += m[k];
  }
  p.zsz = total_knots;
  p.plane_sz = L / m[1];
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  p.scale = 1.0 / (std::ldexp(1.0, d) * n_scale * prod_h);
  if (L == 0) return FCG_OK;
  FCG_PROF("dist_kde_fixup", st);
  kde_fixup_fold_kernel<<<grid_for(p.plane_sz, 256), 256, 0, st>>>(p, zf, planes, Q);
  FCG_LAUNCH_CHECK();
  // axis-1 factor tables of the two signs: codes 0 (delta_1 = +1) and 2 (delta_1 = -1)
  kde_fixup_kernel<<<grid_for(L, 256), 256, 0, st>>>(out, p, zf + p.zoff[1],
                                                     zf + 2 * total_knots + p.zoff[1], Q);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}
