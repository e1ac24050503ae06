// At-points path (subsystem 4): generalized ECDF / ESF at the sample points with ties
// (Eq. 3 as naive.py:90-114 implements it), the strict-dominance ECDF of ecdf_dnc
// (dnc.py:531-561) and the all-delta Laplacian KDE of kde_dnc (dnc.py:635-690).
//
// Routes:
//  * rank lattice (any d, few distinct levels — BASELINE config 2): dense ranks per dimension
//    are bin indices on the grid of distinct values, so the grid engine (scatter -> directional
//    scans) computes every orthant sum and a gather reads each point's own node.  This is the
//    reference's own exact route for tied data.
//  * rank-space dominance, d = 2 (continuous data — config 4): after ranking, the points are a
//    permutation in [0,n)^2.  A 3-level decomposition answers every lower-left query
//    F(t) = sum_i psi_i [p0_i < Q0_t][p1_i < Q1_t]:
//      level 1: chunks of S = 2048 consecutive p1 positions x blocks of S p0 positions form a
//               coarse (n/S)^2 grid; a 2-D inclusive prefix gives all fully-dominated cells;
//      level 2: the query's own chunk and own block are solved inside one CTA each: the
//               <= 2048 sources are laid out in shared memory by local slot / local rank, a
//               64x64 grid of cell sums (prefixed per code direction) covers full cells, and the
//               <= 2 x 32 sources of the query's slot cell and threshold rank cells finish.
//    The four sign codes of the KDE (dnc.py:459-468) are the four orientations of the same
//    problem, sharing one ranking, one chunk/block grouping and (self path) one near-field pass.
//  * rank-space dominance, 3 <= d <= 6 (points_nd.cuh): a coarse G^d grid of rank chunks for the
//    far field and one slab phase per dimension for the sources sharing a chunk with the query.
//  * direct O(n^2) tiles (d >= 7, or fewer than 8192 points).
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "scan.cuh"
#include "sort.cuh"
#include "tma.cuh"

namespace fcg {

namespace {

constexpr int LS = 11;
constexpr int S = 1 << LS;    // level-1 block / chunk size
constexpr int SUBL = 5;
constexpr int SUB = 1 << SUBL;  // level-2 sub-block size
constexpr int NSUB = S / SUB;   // 64
constexpr int kSolverThreads = 1024;
// The d = 2 dominance route keeps a (n/S)^2 x channels fp64 coarse grid: up to 48 GB of the
// 180 GB HBM (n ~ 2.5e8 with two channels); larger n is refused up front with a clear error.
constexpr int64_t kMaxCoarseBytes = int64_t(48) << 30;
constexpr int kCoarseRowBytes = 96 * 1024;  // shared-memory row segment of the coarse histogram

// ------------------------------------------------------------------------------------------
// helpers
__global__ void fill_f64(double *p, int64_t n, double v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void gather_sorted_w(const int32_t *__restrict__ order, const double *__restrict__ w,
                                int64_t n, double *__restrict__ ws) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    ws[p] = w ? w[order[p]] : 1.0;
}

// ------------------------------------------------------------------------------------------
// rank lattice route
struct RankLat {
  int d;
  const int32_t *dense[FCG_MAX_DIM];
  int shift[FCG_MAX_DIM];      // cell = dense - shift (ECDF delta=-1: -1, ESF: +1)
  int64_t dims[FCG_MAX_DIM];
  int64_t stride[FCG_MAX_DIM];
};

template <bool UNIT>
__global__ void rank_scatter_kernel(RankLat r, int64_t n, const double *__restrict__ w,
                                    void *lat) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    bool live = true;
    for (int k = 0; k < r.d; ++k) {
      const int64_t c = (int64_t)r.dense[k][i] - r.shift[k];
      live = live && c >= 0 && c < r.dims[k];
      flat += c * r.stride[k];
    }
    if (!live) continue;
    if (UNIT) atomicAdd(static_cast<int *>(lat) + flat, 1);
    else atomicAdd(static_cast<double *>(lat) + flat, w[i]);
  }
}

template <typename T>
__global__ void rank_gather_kernel(RankLat r, int64_t n, const T *__restrict__ lat, double div,
                                   double *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    for (int k = 0; k < r.d; ++k) flat += (int64_t)r.dense[k][t] * r.stride[k];
    double v = (double)lat[flat];
    if (div > 0.0) v = v / div;
    out[t] = v;
  }
}

// ------------------------------------------------------------------------------------------
// dominance, d = 2
struct Dom2 {
  int64_t n, nq, P, npad;
  int nch;
  int f0, f1;
  const int32_t *pos0, *pos1;     // unflipped source positions (permutations of [0, n))
  const int32_t *bychunk;         // sources sorted by (p1 >> LS, p0)
  const int32_t *byblock;         // sources sorted by (p0 >> LS, p1)
  const double *psi;              // [nch][n]
  const int32_t *Q0f, *Q1f;       // query thresholds in the flipped frame, in [0, npad]
  double *out;                    // [nch][nq]
  double *G;                      // [P][P][nch] coarse grid
  const int32_t *qc_list, *qc_start;  // queries bucketed by chunk(Q1f) (P + 1 buckets)
  const int32_t *qb_list, *qb_start;  // queries bucketed by block(Q0f)
};

__device__ __forceinline__ int32_t flipp(int32_t p, int f, int64_t npad) {
  return f ? (int32_t)(npad - 1 - p) : p;
}

// blocks per shared-memory segment of a coarse row
inline int64_t coarse_tb(int nch) { return kCoarseRowBytes / (8 * (int64_t)nch); }

// the d = 2 dominance route's coarse grid fits the device budget
inline bool dom_fits(int64_t n, int nch) {
  const int64_t P = ceil_div(n, S);
  return P * P * nch * 8 <= kMaxCoarseBytes;
}
inline int dom_too_large(int64_t n) {
  return fail(FCG_EUNSUPPORTED,
              "n = " + std::to_string(n) + " points: the d = 2 dominance coarse grids would "
              "exceed the 48 GB device budget (n <= ~3.5e8 for one channel, ~1.2e8 for the "
              "Laplacian KDE with two weight vectors)");
}

// coarse rows: CTA per (flipped chunk c, segment of TB blocks); row[b][ch] accumulated in
// shared memory, so a row of any length is built in ceil(P / TB) segments
__global__ void __launch_bounds__(512) coarse_rows_smem(Dom2 D, int64_t TB) {
  extern __shared__ double s_row[];  // [TB][nch]
  const int64_t c = blockIdx.x;
  const int64_t g = D.f1 ? D.P - 1 - c : c;
  const int64_t P = D.P;
  const int64_t b0 = (int64_t)blockIdx.y * TB, nb = (b0 + TB < P ? TB : P - b0);
  for (int64_t i = threadIdx.x; i < nb * D.nch; i += blockDim.x) s_row[i] = 0.0;
  __syncthreads();
  const int64_t lo = g * S, hi = (g + 1) * S < D.n ? (g + 1) * S : D.n;
  for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
    const int32_t src = D.bychunk[k];
    const int64_t b = (flipp(D.pos0[src], D.f0, D.npad) >> LS) - b0;
    if (b < 0 || b >= nb) continue;
    for (int ch = 0; ch < D.nch; ++ch) atomicAdd(&s_row[b * D.nch + ch], D.psi[ch * D.n + src]);
  }
  __syncthreads();
  double *row = D.G + (c * P + b0) * D.nch;
  for (int64_t i = threadIdx.x; i < nb * D.nch; i += blockDim.x) row[i] = s_row[i];
}

// out = inclusive-prefix coarse grid at (chunk(Q1f) - 1, block(Q0f) - 1)
__global__ void coarse_query(Dom2 D) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < D.nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = D.Q1f[t] >> LS, b = D.Q0f[t] >> LS;
    c = c > D.P ? D.P : c;
    b = b > D.P ? D.P : b;
    for (int ch = 0; ch < D.nch; ++ch) {
      double v = 0.0;
      if (c > 0 && b > 0) v = D.G[((c - 1) * D.P + (b - 1)) * D.nch + ch];
      D.out[ch * D.nq + t] = v;
    }
  }
}

// keys for query bucketing: chunk(Q1f) or block(Q0f), clamped to P
__global__ void query_keys(Dom2 D, int32_t *kc, int32_t *kb) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < D.nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = D.Q1f[t] >> LS, b = D.Q0f[t] >> LS;
    kc[t] = (int32_t)(c > D.P ? D.P : c);
    kb[t] = (int32_t)(b > D.P ? D.P : b);
  }
}

// Query bucketing with warp-aggregated atomics: sorted or clustered keys would otherwise
// serialise thousands of threads on one counter.
__device__ __forceinline__ unsigned lane_lt_mask() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void bucket_count(const int32_t *__restrict__ key, int64_t n, int32_t *cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t t = base + threadIdx.x;
    const bool ok = t < n;
    const int k = ok ? key[t] : -1 - (int)(threadIdx.x & 31);
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[k], __popc(peers));
  }
}

__global__ void bucket_fill(const int32_t *__restrict__ key, int64_t n, int32_t *cursor,
                            int32_t *list) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t t = base + threadIdx.x;
    const bool ok = t < n;
    const int k = ok ? key[t] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int leader = __ffs(peers) - 1;
    int pos = 0;
    if (ok && lane == leader) pos = atomicAdd(&cursor[k], __popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (ok) list[pos + __popc(peers & lane_lt_mask())] = (int32_t)t;
  }
}

// Level-2 solver.  CHUNK: CTA per flipped chunk c, sources of that chunk; slot X = local p1f,
// rank Y = rank of p0f within the chunk; query (qx = Q1f - cS, qy = #sources with p0f < Q0f).
// BLOCK: CTA per flipped block b; slot X = local p0f, rank Y = rank of p1f within the block;
// query (qx = Q0f - bS, qy = #sources with p1f < chunk(Q1f) * S).
template <bool CHUNK, int NCH>
__global__ void __launch_bounds__(kSolverThreads) level2_solver(Dom2 D) {
  extern __shared__ __align__(16) unsigned char smem[];
  double *s_sub = reinterpret_cast<double *>(smem);             // [NCH][NSUB][NSUB]
  double *s_psi = s_sub + NCH * NSUB * NSUB;                    // [NCH][S] by slot X
  int32_t *s_key = reinterpret_cast<int32_t *>(s_psi + NCH * S);  // [S] sorted keys by rank Y
  int16_t *s_yofx = reinterpret_cast<int16_t *>(s_key + S);     // [S]
  int16_t *s_xofy = s_yofx + S;                                 // [S]

  const int64_t cb = blockIdx.x;  // flipped chunk (CHUNK) or flipped block (BLOCK)
  const int fslot = CHUNK ? D.f1 : D.f0;
  const int frank = CHUNK ? D.f0 : D.f1;
  const int64_t g = fslot ? D.P - 1 - cb : cb;  // unflipped group index
  const int64_t lo = g * S;
  const int64_t Sg = (lo + S < D.n ? S : D.n - lo);
  const int32_t *grp = (CHUNK ? D.bychunk : D.byblock) + lo;
  const int32_t *slotpos = CHUNK ? D.pos1 : D.pos0;
  const int32_t *rankpos = CHUNK ? D.pos0 : D.pos1;

  for (int i = threadIdx.x; i < NCH * NSUB * NSUB; i += blockDim.x) s_sub[i] = 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    s_yofx[i] = -1;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) s_psi[ch * S + i] = 0.0;
  }
  __syncthreads();
  // gather the group's sources: batches of KG per thread with every global load of a batch
  // issued before the shared-memory stores (the gathers are random, latency-bound)
  constexpr int KG = 4;
  for (int64_t k0 = threadIdx.x; k0 < Sg; k0 += KG * blockDim.x) {
    int32_t src[KG], sp[KG], rp[KG];
    double ps[KG][NCH];
#pragma unroll
    for (int u = 0; u < KG; ++u) {
      const int64_t k = k0 + u * (int64_t)blockDim.x;
      src[u] = k < Sg ? grp[k] : -1;
    }
#pragma unroll
    for (int u = 0; u < KG; ++u) {
      const int32_t sr = src[u] < 0 ? grp[0] : src[u];
      sp[u] = slotpos[sr];
      rp[u] = rankpos[sr];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) ps[u][ch] = D.psi[ch * D.n + sr];
    }
#pragma unroll
    for (int u = 0; u < KG; ++u) {
      if (src[u] < 0) continue;
      const int64_t k = k0 + u * (int64_t)blockDim.x;
      const int y = frank ? (int)(Sg - 1 - k) : (int)k;
      int x = sp[u] - (int32_t)lo;
      if (fslot) x = S - 1 - x;
      s_yofx[x] = (int16_t)y;
      s_xofy[y] = (int16_t)x;
      s_key[y] = flipp(rp[u], frank, D.npad);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) s_psi[ch * S + x] = ps[u][ch];
    }
  }
  __syncthreads();
  // sub-grid cell sums: thread (channel, sub-row u) owns row u and walks its SUB slots (no
  // fp64 shared atomics, which are CAS loops on sm_100)
  for (int r = threadIdx.x; r < NCH * NSUB; r += blockDim.x) {
    const int ch = r / NSUB, u = r % NSUB;
    double *row = s_sub + (ch * NSUB + u) * NSUB;
    for (int x = u << SUBL; x < (u + 1) << SUBL; ++x) {
      const int y = s_yofx[x];
      if (y >= 0) row[y >> SUBL] += s_psi[ch * S + x];
    }
  }
  __syncthreads();
  // inclusive 2-D prefix of the sub-grid: rows (over y-sub index), then columns
  for (int r = threadIdx.x; r < NCH * NSUB; r += blockDim.x) {
    double *row = s_sub + r * NSUB;
    double run = 0.0;
    for (int v = 0; v < NSUB; ++v) { run += row[v]; row[v] = run; }
  }
  __syncthreads();
  for (int cidx = threadIdx.x; cidx < NCH * NSUB; cidx += blockDim.x) {
    const int ch = cidx / NSUB, v = cidx % NSUB;
    double run = 0.0;
    for (int u = 0; u < NSUB; ++u) {
      double *p = s_sub + (ch * NSUB + u) * NSUB + v;
      run += *p;
      *p = run;
    }
  }
  __syncthreads();

  const int32_t *qlist = CHUNK ? D.qc_list : D.qb_list;
  const int32_t q0 = (CHUNK ? D.qc_start : D.qb_start)[cb];
  const int32_t q1 = (CHUNK ? D.qc_start : D.qb_start)[cb + 1];
  for (int32_t qi = q0 + threadIdx.x; qi < q1; qi += blockDim.x) {
    const int32_t t = qlist[qi];
    int qx, qy;
    {
      int32_t ythr;
      if (CHUNK) {
        qx = (int)(D.Q1f[t] - cb * S);
        ythr = D.Q0f[t];
      } else {
        qx = (int)(D.Q0f[t] - cb * S);
        int64_t c = D.Q1f[t] >> LS;
        ythr = (int32_t)((c > D.P ? D.P : c) * S);
      }
      // qy = #keys < ythr among the Sg sorted keys
      int a = 0, bnd = (int)Sg;
      while (a < bnd) {
        const int mid = (a + bnd) >> 1;
        if (s_key[mid] < ythr) a = mid + 1;
        else bnd = mid;
      }
      qy = a;
    }
    const int u = qx >> SUBL, v = qy >> SUBL;
    double acc[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
      acc[ch] = (u > 0 && v > 0) ? s_sub[(ch * NSUB + (u - 1)) * NSUB + (v - 1)] : 0.0;
    for (int x = u << SUBL; x < qx; ++x) {  // partial slot sub-range, any rank < qy
      const int y = s_yofx[x];
      if (y >= 0 && y < qy) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[ch] += s_psi[ch * S + x];
      }
    }
    const int xfull = u << SUBL;
    for (int y = v << SUBL; y < qy; ++y) {  // partial rank sub-range, full slot sub-blocks
      const int x = s_xofy[y];
      if (x < xfull) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) acc[ch] += s_psi[ch * S + x];
      }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) D.out[ch * D.nq + t] += acc[ch];
  }
}

size_t level2_smem(int nch) {
  return (size_t)nch * NSUB * NSUB * 8 + (size_t)nch * S * 8 + (size_t)S * 4 + (size_t)S * 4;
}

// grouping keys: key[p] = pos_other[order[p]] >> LS, val[p] = order[p]
__global__ void group_keys(const int32_t *__restrict__ order, const int32_t *__restrict__ pos_other,
                           int64_t n, uint64_t *keys, int32_t *vals) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = order[p];
    keys[p] = (uint64_t)(pos_other[i] >> LS);
    vals[p] = i;
  }
}

// ------------------------------------------------------------------------------------------
// brute force (d >= 3): CTA = 256 queries, source tiles staged in shared memory
enum BruteMode { BR_ECDF = 0, BR_KDE = 1, BR_MATERN = 2 };

struct Brute {
  int64_t n;
  int d;
  const double *x;
  const double *w;   // [nw][n] or NULL
  int nw;
  int sign[FCG_MAX_DIM];  // ECDF: +1 <=, -1 <, 2 = strictly greater (survival)
  double inv_h[FCG_MAX_DIM];
  double *out;       // [nw][n]
};

template <int MODE>
__global__ void __launch_bounds__(256) brute_kernel(Brute B) {
  __shared__ double s_x[256 * FCG_MAX_DIM];
  __shared__ double s_w[2][256];
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const bool live = t < B.n;
  double xt[FCG_MAX_DIM];
  for (int k = 0; k < B.d; ++k) xt[k] = live ? B.x[t * B.d + k] : 0.0;
  double acc[2] = {0.0, 0.0};
  for (int64_t base = 0; base < B.n; base += 256) {
    const int64_t i = base + threadIdx.x;
    __syncthreads();
    if (i < B.n) {
      for (int k = 0; k < B.d; ++k) s_x[threadIdx.x * B.d + k] = B.x[i * B.d + k];
      for (int v = 0; v < B.nw; ++v) s_w[v][threadIdx.x] = B.w ? B.w[v * B.n + i] : 1.0;
    }
    __syncthreads();
    const int cnt = (int)((B.n - base) < 256 ? (B.n - base) : 256);
    for (int j = 0; j < cnt; ++j) {
      const double *xs = s_x + j * B.d;
      if (MODE == BR_ECDF) {
        bool ok = true;
        for (int k = 0; k < B.d; ++k) {
          const double a = xs[k], z = xt[k];
          const int s = B.sign[k];
          ok = ok && (s == 1 ? a <= z : (s == -1 ? a < z : a > z));
        }
        if (ok)
          for (int v = 0; v < B.nw; ++v) acc[v] += s_w[v][j];
      } else {
        if (base + j == t) continue;  // self term added in closed form by the caller
        double e = 0.0;
        for (int k = 0; k < B.d; ++k) e += fabs(xs[k] - xt[k]) * B.inv_h[k];
        const double kv = MODE == BR_MATERN ? (1.0 + e) * exp(-e) : exp(-e);
        for (int v = 0; v < B.nw; ++v) acc[v] += s_w[v][j] * kv;
      }
    }
  }
  if (live)
    for (int v = 0; v < B.nw; ++v) B.out[v * B.n + t] = acc[v];
}

// ------------------------------------------------------------------------------------------
// KDE epilogue pieces (dnc.py:661-686)
struct KdeP {
  int d;
  double c[FCG_MAX_DIM], a[FCG_MAX_DIM];  // a_k = s_k / h_k
  int code;                                // the term's sign code (bit k: s_k = -1)
  unsigned smask[2];                       // channel v's psi carries prod_{k in smask} s_k
};

__device__ __forceinline__ double chan_sign(const KdeP &p, int v) {
  return (__popc(p.smask[v] & (unsigned)p.code) & 1) ? -1.0 : 1.0;
}

// expo[i] = sum_k (x_ik - c_k) * a_k ; psi[v][i] = w[v][i] * exp(expo[i])
__global__ void kde_psi_kernel(const double *__restrict__ x, int64_t n, KdeP p,
                               const double *__restrict__ w, int nw, double *__restrict__ expo,
                               double *__restrict__ psi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < p.d; ++k) s += (x[i * p.d + k] - p.c[k]) * p.a[k];
    expo[i] = s;
    const double e = exp(s);
    for (int v = 0; v < nw; ++v) psi[v * n + i] = (w ? w[v * n + i] : 1.0) * e * chan_sign(p, v);
  }
}

// out[v][t] (+)= exp(-expo[t]) * F[v][t]
__global__ void kde_accum_kernel(int64_t n, int nw, const double *__restrict__ expo,
                                 const double *__restrict__ F, double *__restrict__ out, int first) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double z = exp(-expo[t]);
    for (int v = 0; v < nw; ++v) {
      const double r = z * F[v * n + t];
      out[v * n + t] = first ? r : out[v * n + t] + r;
    }
  }
}

// out[v][t] = (out[v][t] + w[v][t]) * scale   (self term, then the shared normalisation)
__global__ void kde_finish_kernel(int64_t n, int nw, const double *__restrict__ w, double scale,
                                  double *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    for (int v = 0; v < nw; ++v) {
      double r = out[v * n + t] + (w ? w[v * n + t] : 1.0);
      out[v * n + t] = r * scale;
    }
}

// final: out[t] = (out[t] + (self ? w[t] : 0)) / div
__global__ void finish_ecdf_kernel(double *__restrict__ out, int64_t n,
                                   const double *__restrict__ w, int include_self, double div) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    double r = out[t];
    if (include_self) r = r + (w ? w[t] : 1.0);
    if (div > 0.0) r = r / div;
    out[t] = r;
  }
}

// d == 1 gather from an inclusive sorted prefix (forward) or suffix (reverse) scan
// mode 0: out[t] = q > 0 ? incl[q-1] : 0   (sources at sorted positions < q)
// mode 1: out[t] = q < n ? suf[q] : 0      (sources at sorted positions >= q)
__global__ void gather1d_kernel(const double *__restrict__ scan, const int32_t *__restrict__ q,
                                int64_t n, int mode, double *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t qq = q[t];
    out[t] = mode == 0 ? (qq > 0 ? scan[qq - 1] : 0.0) : (qq < n ? scan[qq] : 0.0);
  }
}

// srt[p] = vals[order[p]] (vals == NULL: ones); cpy = copy for the in-place scan
__global__ void permute_kernel(const double *__restrict__ vals, const int32_t *__restrict__ order,
                               int64_t n, double *__restrict__ srt, double *__restrict__ cpy) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double v = vals ? vals[order[p]] : 1.0;
    srt[p] = v;
    cpy[p] = v;
  }
}

// dst[order[p]] = incl[p] - srt[p]: "cumsum - self" of dnc.py:543-547 and dnc.py:572-579
__global__ void excl_scatter_kernel(const double *__restrict__ incl, const double *__restrict__ srt,
                                    const int32_t *__restrict__ order, int64_t n,
                                    double *__restrict__ dst) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    dst[order[p]] = incl[p] - srt[p];
}

// flipped-frame thresholds: Q0f = f(base0) etc.  kind: 0 = copy, 1 = npad-1-pos (self, flipped),
// 2 = npad - q (count-type threshold, flipped)
__global__ void make_q_kernel(const int32_t *__restrict__ a, int64_t n, int kind, int64_t npad,
                              int32_t *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = a[t];
    out[t] = kind == 0 ? v : (kind == 1 ? (int32_t)(npad - 1 - v) : (int32_t)(npad - v));
  }
}

__global__ void adjacent_equal_kernel(const uint64_t *__restrict__ keys, int64_t n, int32_t *flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    if (keys[p] == keys[p - 1]) *flag = 1;
}

// ------------------------------------------------------------------------------------------
// Self-query dominance (kde_dnc / ecdf_dnc, d = 2).  The chunk grouping (sources sorted by
// (p1 >> LS, p0)) and the block grouping ((p0 >> LS, p1)) are index lists; the level-2 CTAs and
// the coarse rows gather their sources' records through them (one 32-byte sector per point for
// coordinates and weights, L2-resident after a CTA's first code), and the level-2 results land
// in point order, so the finish is a streaming pass.

// per point (input order): coordinates and weights in one sector
struct __align__(16) PtXW {
  double x0, x1, w0, w1;
};

// per-channel weight vectors of the self path (nullptr = unit weights for that channel)
struct WPtr {
  const double *p[2];
  __host__ __device__ double at(int v, int64_t i) const { return p[v] ? p[v][i] : 1.0; }
};
inline WPtr wptr(const double *w, int nw, int64_t n) {  // the [nw][n] matrix layout
  return WPtr{{w, (w && nw > 1) ? w + n : nullptr}};
}

// Self-path grouping without a global sort.  Group g of the slot dimension (chunk: points with
// p1 in [g S, g S + Sg), i.e. order1[g S ...], slot = p1; block: order0, slot = p0) is ordered
// by its rank-dimension position r (p0 for chunks, p1 for blocks): a shared-memory counting pass
// over the level-1 cells r >> LS of the other dimension (about S / P points per cell) gives every
// point its cell's start, and a count of the smaller keys inside the cell its index k.  Writes
// the (slot, rank) positions and the coordinate / weight sector in group order, for the coarse
// rows and the level-2 CTAs.  Same order as sorting by (slot >> LS, rank).
constexpr int kGroupThreads = 1024;
constexpr int kGroupPer = S / kGroupThreads;

__global__ void __launch_bounds__(kGroupThreads) group_self_kernel(
    const int32_t *__restrict__ order_slot, const int32_t *__restrict__ pos_rank,
    const PtXW *__restrict__ xw, int64_t n, int64_t P, int shift, int2 *__restrict__ gpos,
    PtXW *__restrict__ gxw) {
  // P here: the number of cells key >> shift (the level-1 cells, or coarser ones for very large n)
  extern __shared__ int32_t gs_smem[];
  int32_t *s_cnt = gs_smem;                // [P + 1]: cell counts -> exclusive starts
  int32_t *s_key = gs_smem + P + 1;        // [S]: keys by cell position
  int32_t *s_wsum = s_key + S;             // [32]
  const int64_t lo = (int64_t)blockIdx.x * S;
  const int Sg = (int)(lo + S < n ? S : n - lo);
  for (int64_t i = threadIdx.x; i <= P; i += kGroupThreads) s_cnt[i] = 0;
  __syncthreads();
  int32_t id[kGroupPer], key[kGroupPer], sl[kGroupPer];
#pragma unroll
  for (int j = 0; j < kGroupPer; ++j) {
    const int i = threadIdx.x + j * kGroupThreads;
    id[j] = i < Sg ? order_slot[lo + i] : 0;
  }
#pragma unroll
  for (int j = 0; j < kGroupPer; ++j) {
    const int i = threadIdx.x + j * kGroupThreads;
    key[j] = i < Sg ? pos_rank[id[j]] : 0;
    sl[j] = i < Sg ? atomicAdd(&s_cnt[key[j] >> shift], 1) : 0;
  }
  __syncthreads();
  {  // exclusive scan of the P + 1 counts in place (thread t: a contiguous run of cells)
    const int64_t per = (P + 1 + kGroupThreads - 1) / kGroupThreads;
    const int64_t a = threadIdx.x * per, b = a + per < P + 1 ? a + per : P + 1;
    int32_t tot = 0;
    for (int64_t i = a; i < b; ++i) tot += s_cnt[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    int32_t run = x - tot;
    for (int w = 0; w < warp; ++w) run += s_wsum[w];
    for (int64_t i = a; i < b; ++i) {
      const int32_t c = s_cnt[i];
      s_cnt[i] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kGroupPer; ++j) {
    const int i = threadIdx.x + j * kGroupThreads;
    if (i < Sg) s_key[s_cnt[key[j] >> shift] + sl[j]] = key[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kGroupPer; ++j) {
    const int i = threadIdx.x + j * kGroupThreads;
    if (i >= Sg) continue;
    const int64_t c = key[j] >> shift;
    const int a = s_cnt[c], b = s_cnt[c + 1];
    int k = a;
    for (int m = a; m < b; ++m) k += s_key[m] < key[j];
    gpos[lo + k] = make_int2((int32_t)(lo + i), key[j]);
    gxw[lo + k] = xw[id[j]];
  }
}

constexpr int64_t kGroupMaxCells = 16384;  // shared-memory counters per group CTA
inline int group_self_shift(int64_t n) {
  int sh = LS;
  while ((((n - 1) >> sh) + 1) > kGroupMaxCells) ++sh;
  return sh;
}
inline int64_t group_self_cells(int64_t n) { return ((n - 1) >> group_self_shift(n)) + 1; }
size_t group_self_smem(int64_t n) { return (size_t)(group_self_cells(n) + 1 + S + 32) * 4; }

__global__ void pack_points_kernel(const double *__restrict__ x, WPtr w, int nw, int64_t n,
                                   PtXW *__restrict__ xw) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    PtXW r;
    r.x0 = x[2 * i];
    r.x1 = x[2 * i + 1];
    r.w0 = w.at(0, i);
    r.w1 = nw > 1 ? w.at(1, i) : 0.0;
    xw[i] = r;
  }
}

struct Dom2S {
  int64_t n, P, npad;
  int64_t c_lo, c_hi;  // query shard: points whose (unflipped) chunk p1 >> LS is in [c_lo, c_hi)
  int nch, f0, f1, kde;
  const int2 *gpos_c, *gpos_b;  // (slot, rank) positions in group order
  const PtXW *gxw_c, *gxw_b;    // coordinates and weights in group order
  double *accc, *accb;          // level-2 results [n][nch] in p1 (chunks) / p0 (blocks) order
  double *G;         // coarse grids [ncodes][P][P][nch], each in its code's flipped frame
  KdeP kp;           // the current code (level-2 solvers: psi and z computed on the fly)
};

// The sign codes of one self-dominance call: the 2^2 Laplacian orientations (kde) or the plain
// strict-dominance ECDF (one code, psi = w).
struct Codes {
  int n, kde;
  KdeP kp[4];
};

// exponent s_code(x) = sum_j (x_j - c_j) a_j (dnc.py:661-669: a_j carries the code's sign)
__device__ __forceinline__ double code_s(const KdeP &kp, double x0, double x1) {
  return (x0 - kp.c[0]) * kp.a[0] + (x1 - kp.c[1]) * kp.a[1];
}

// Coarse rows of every code, prefixed along the block axis: CTA per unflipped chunk g.  The
// chunk's points arrive in p0 order, so their blocks are nondecreasing and the inclusive prefix
// at block b is a running sum over the points evaluated at the last point of block <= b: one
// CTA-wide scan per (code, channel), parked in shared memory, and an output-ordered pass where
// every thread finds its block's point by binary search and stores coalesced.  Codes with
// f0 = 1 store their grid flipped along the block axis: suffix sums (second sweep), written at
// P-1-b.  Row f1 ? P-1-g : g.  No atomics.
constexpr int kCoarseThreads = 512;
constexpr int kCoarsePer = S / kCoarseThreads;  // consecutive points per thread

template <int NCH>
__global__ void __launch_bounds__(kCoarseThreads, 2) coarse_rows_codes(Dom2S D, Codes K) {
  constexpr int NV = 2 * NCH, NW = kCoarseThreads / 32;  // channels per sweep (2 codes)
  extern __shared__ __align__(16) double s_scan[];        // [S][NV] scan values by point
  int32_t *s_blk = reinterpret_cast<int32_t *>(s_scan + S * NV);  // [S] blocks by point
  __shared__ double s_wtot[NV][NW];
  const int64_t g = blockIdx.x, P = D.P, lo = g * S;
  const int Sg = (int)(lo + S < D.n ? S : D.n - lo);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nc = K.n > 1 ? 2 : 1, nq = nc * NCH;
#pragma unroll
  for (int j = 0; j < kCoarsePer; ++j) {
    const int k = tid * kCoarsePer + j;
    s_blk[k] = k < Sg ? (D.gpos_c[lo + k].y >> LS) : (int32_t)P;
  }
  for (int sweep = 0; sweep < (K.n > 1 ? 2 : 1); ++sweep) {
    const bool rev = sweep != 0;
    double val[kCoarsePer][NV];
#pragma unroll
    for (int j = 0; j < kCoarsePer; ++j) {
      const int k = tid * kCoarsePer + j;
      const bool live = k < Sg;
      PtXW r = live ? D.gxw_c[lo + k] : PtXW{0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) {
        if (ci >= nc) break;
        const int c = sweep + 2 * ci;
        const double e = (K.kde && live) ? exp(code_s(K.kp[c], r.x0, r.x1)) : (live ? 1.0 : 0.0);
#pragma unroll
        for (int v = 0; v < NCH; ++v)
          val[j][ci * NCH + v] = (v ? r.w1 : r.w0) * e * (K.kde ? chan_sign(K.kp[c], v) : 1.0);
      }
    }
    // inclusive scans over the points: ascending (sweep 0) or descending (sweep 1)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      if (q >= nq) break;
      double run = 0.0;
      if (!rev) {
#pragma unroll
        for (int j = 0; j < kCoarsePer; ++j) val[j][q] = run = run + val[j][q];
      } else {
#pragma unroll
        for (int j = kCoarsePer - 1; j >= 0; --j) val[j][q] = run = run + val[j][q];
      }
      double x = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = rev ? __shfl_down_sync(0xffffffffu, x, o) : __shfl_up_sync(0xffffffffu, x, o);
        if (rev ? lane + o < 32 : lane >= o) x += y;
      }
      if (lane == (rev ? 0 : 31)) s_wtot[q][warp] = x;
      double excl = rev ? __shfl_down_sync(0xffffffffu, x, 1) : __shfl_up_sync(0xffffffffu, x, 1);
      if (lane == (rev ? 31 : 0)) excl = 0.0;  // the lanes before (after) this one
#pragma unroll
      for (int j = 0; j < kCoarsePer; ++j) val[j][q] += excl;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      if (q >= nq) break;
      double carry = 0.0;
      if (!rev) {
        for (int w = 0; w < warp; ++w) carry += s_wtot[q][w];
      } else {
        for (int w = NW - 1; w > warp; --w) carry += s_wtot[q][w];
      }
#pragma unroll
      for (int j = 0; j < kCoarsePer; ++j)
        s_scan[(tid * kCoarsePer + j) * NV + q] = val[j][q] + carry;
    }
    __syncthreads();
    // output pass: block b takes the prefix through its last point (the suffix from its first)
    double *rows[2];
#pragma unroll
    for (int ci = 0; ci < 2; ++ci) {
      const int c = sweep + 2 * ci;
      const int f1 = (c >> 1) & 1;
      rows[ci] = D.G + ((int64_t)c * P + (f1 ? P - 1 - g : g)) * P * NCH;
    }
    const int32_t Pi = (int32_t)P;
    for (int32_t b = tid; b < Pi; b += kCoarseThreads) {
      // number of points with block < thr (dead points hold block P): sweep 0 counts blocks
      // <= b, sweep 1 blocks < b; a fixed-step search over the S entries
      const int32_t thr = rev ? b : b + 1;
      int a = 0;
#pragma unroll
      for (int step = S / 2; step > 0; step >>= 1)
        if (s_blk[a + step - 1] < thr) a += step;
      if (s_blk[a] < thr) ++a;  // a in [0, S]; entries past Sg never count (thr <= P)
      const int idx = rev ? a : a - 1;
      const bool has = rev ? idx < Sg : idx >= 0;
      const int64_t bq = rev ? P - 1 - b : b;
#pragma unroll
      for (int ci = 0; ci < 2; ++ci) {
        if (ci >= nc) break;
#pragma unroll
        for (int v = 0; v < NCH; ++v)
          rows[ci][bq * NCH + v] = has ? s_scan[idx * NV + ci * NCH + v] : 0.0;
      }
    }
    __syncthreads();
  }
}

// All sign codes of one level-2 grouping in one CTA (CHUNK: chunk g, sources = the chunk's
// points by p0 rank; BLOCK: block g by p1 rank).  The CTA loads its sources once (registers:
// thread t holds sources t, t + 1024, ...), and for every code rebuilds the flipped-frame layout,
// the sub-grid and both partial passes.  Each thread owns the same queries in every code (pass A:
// the sources of its unflipped slots, pass B: the sources of its ranks), so the code sum
// z_c * F_c accumulates in registers; the two halves meet in shared memory once and are written
// with plain coalesced stores (no global read-modify-write per code).
//
// Shared-memory discipline (ncu: the first version lost half its shared wavefronts to bank
// conflicts and a third of its warp time to barriers behind 4-warp serial loops): the sub-grid is
// built by one WARP per sub-row with the lanes on the 64 column cells (broadcast reads of the
// sub-row's slots, the row prefix accumulated in registers), the column prefix by all 1024
// threads as 8-row segments plus segment carries, and both partial passes read 4 candidates per
// step (one 8-byte load of four int16 positions, four independent broadcast psi loads).
constexpr int kL2Per = S / kSolverThreads;  // sources per thread
constexpr int16_t kEmptyY = 0x7fff;          // an empty slot: above every rank threshold

// Masked accumulate a += h * p: one select of the mask's high word and an FMA per channel (a
// predicated add compiles to an add plus four 32-bit selects on the ALU pipe).  p is finite
// (validated inputs; empty slots hold 0), so h = 0 adds exactly +0.0.
template <int NCH>
struct PsiT;
template <>
struct PsiT<1> {
  using T = double;
  __device__ static void add(double (&a)[1], double p, bool h) {
    const double m = h ? 1.0 : 0.0;
    a[0] = fma(p, m, a[0]);
  }
};
template <>
struct PsiT<2> {
  using T = double2;
  __device__ static void add(double (&a)[2], double2 p, bool h) {
    const double m = h ? 1.0 : 0.0;
    a[0] = fma(p.x, m, a[0]);
    a[1] = fma(p.y, m, a[1]);
  }
};

template <bool CHUNK, int NCH>
__global__ void __launch_bounds__(kSolverThreads) level2_codes(Dom2S D, Codes K) {
  using PT = typename PsiT<NCH>::T;
  extern __shared__ __align__(16) unsigned char smem[];
  double *s_sub = reinterpret_cast<double *>(smem);               // [NCH][NSUB][NSUB]
  double *s_psi = s_sub + NCH * NSUB * NSUB;                      // [S][NCH] by slot
  double *s_tot = s_psi + NCH * S;                                // [1024] column-scan carries
  double *s_z = s_tot + kSolverThreads;                           // [S] e^{-s} by group index
  int32_t *s_key = reinterpret_cast<int32_t *>(s_z + S);          // [S] rank-dim positions by rank
  int16_t *s_yofx = reinterpret_cast<int16_t *>(s_key + S);       // [S]
  int16_t *s_xofy = s_yofx + S;                                   // [S]
  int16_t *s_kofx = s_xofy + S;                                   // [S] group index by slot
  int16_t *s_qy = s_kofx + S;                                     // [S] rank threshold by
                                                                  // UNFLIPPED slot
  int16_t *s_slot = s_qy + S;                                     // [S] unflipped slot by k
  const PT *s_p = reinterpret_cast<const PT *>(s_psi);

  double *out = CHUNK ? D.accc : D.accb;
  const int64_t g = blockIdx.x + (CHUNK ? D.c_lo : 0);  // unflipped chunk / block
  const int64_t lo = g * S;
  const int Sg = (int)(lo + S < D.n ? S : D.n - lo);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool all_owned = CHUNK || (D.c_lo == 0 && D.c_hi == D.P);
  auto owned_key = [&](int32_t key) {  // BLOCK kind: the query's chunk is the shard's
    const int64_t cu = key >> LS;
    return all_owned || (cu >= D.c_lo && cu < D.c_hi);
  };
  // ranks past the group's end are never written; pass B may read their positions (masked)
  for (int i = Sg + threadIdx.x; i < S; i += blockDim.x) s_xofy[i] = 0;
  const int2 *gpos = CHUNK ? D.gpos_c : D.gpos_b;
  const PtXW *gxw = CHUNK ? D.gxw_c : D.gxw_b;
  // this thread's sources (group indices k = threadIdx.x + j * 1024): rank keys in registers,
  // slots in shared memory, coordinates and weights re-read per code (coalesced; L2 hits after
  // the first code)
  int32_t key_u[kL2Per];
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = threadIdx.x + j * kSolverThreads;
    const int2 pp = k < Sg ? gpos[lo + k] : make_int2(0, 0);
    key_u[j] = pp.y;
    if (k < Sg) s_slot[k] = (int16_t)(pp.x - (int32_t)lo);
  }
  double accA[kL2Per][NCH], accB[kL2Per][NCH];
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) accA[j][ch] = accB[j][ch] = 0.0;
  }

  for (int code = 0; code < K.n; ++code) {
    const KdeP &kp = K.kp[code];
    const int f0 = code & 1, f1 = (code >> 1) & 1;
    const int fslot = CHUNK ? f1 : f0, frank = CHUNK ? f0 : f1;
    // BLOCK thresholds depend on the rank frame only: searched at the first code of each frame
    // (codes run 0..3, so the rank frame f1 changes at codes 0 and 2)
    const bool search = !CHUNK && (code == 0 || code == 2);
    __syncthreads();  // the previous code's passes are done with the shared arrays
    for (int i = threadIdx.x; i < S / 2; i += blockDim.x)
      reinterpret_cast<uint32_t *>(s_yofx)[i] = (uint32_t)(uint16_t)kEmptyY * 0x10001u;
    if (Sg < S)  // empty slots are read (masked) by the passes: keep them finite
      for (int i = threadIdx.x; i < S * NCH; i += blockDim.x) s_psi[i] = 0.0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      const int k = threadIdx.x + j * kSolverThreads;
      if (k >= Sg) continue;
      const int y = frank ? Sg - 1 - k : k;
      const int sl = s_slot[k];
      const int x = fslot ? S - 1 - sl : sl;
      s_yofx[x] = (int16_t)y;
      s_xofy[y] = (int16_t)x;
      s_kofx[x] = (int16_t)k;
      s_key[y] = flipp(key_u[j], frank, D.npad);
      const PtXW r = gxw[lo + k];
      double e = 1.0, z = 1.0;
      if (K.kde) {
        const double sv = code_s(kp, r.x0, r.x1);
        e = exp(sv);
        z = exp(-sv);
        s_z[k] = z;
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
        s_psi[x * NCH + ch] = (ch ? r.w1 : r.w0) * e * (K.kde ? chan_sign(kp, ch) : 1.0);
      if (CHUNK) {
        // level 1: the code's coarse cell below the query's chunk and block (flipped frame).
        // The chunk's points run in p0 order, so a warp's reads walk one grid row in order.
        const int64_t P = D.P, bu = key_u[j] >> LS;
        const int64_t cc = f1 ? P - 1 - g : g, bb = f0 ? P - 1 - bu : bu;
        if (cc > 0 && bb > 0) {
          const double *gv = D.G + (((int64_t)code * P + cc - 1) * P + bb - 1) * NCH;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) accB[j][ch] += z * gv[ch];
        }
      }
    }
    __syncthreads();
    // sub-grid rows: warp per sub-row u, lane l owns column cells l and l + 32; the inclusive
    // row prefix sum_{x in row u, y >> SUBL <= v} psi_x is accumulated directly
    for (int u = warp; u < NSUB; u += kSolverThreads / 32) {
      double a0[NCH], a1[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) a0[ch] = a1[ch] = 0.0;
      const int base = u << SUBL;
      const int lim0 = (lane + 1) << SUBL, lim1 = (lane + 33) << SUBL;  // cells <= l, <= l + 32
#pragma unroll 4
      for (int i = 0; i < SUB; i += 4) {
        const short4 y4 = *reinterpret_cast<const short4 *>(s_yofx + base + i);
        const int yy[4] = {y4.x, y4.y, y4.z, y4.w};
        PT pp[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) pp[t] = s_p[base + i + t];
#pragma unroll
        for (int t = 0; t < 4; ++t) {  // empty slots (kEmptyY) are past every cell
          PsiT<NCH>::add(a0, pp[t], yy[t] < lim0);
          PsiT<NCH>::add(a1, pp[t], yy[t] < lim1);
        }
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        s_sub[(ch * NSUB + u) * NSUB + lane] = a0[ch];
        s_sub[(ch * NSUB + u) * NSUB + lane + 32] = a1[ch];
      }
    }
    __syncthreads();
    // column prefix over the sub-rows: thread (segment sg, column cc), lanes on consecutive
    // columns; segment totals meet in s_tot
    {
      constexpr int NCC = NCH * NSUB, SEGS = kSolverThreads / NCC, RPS = NSUB / SEGS;
      const int cc = threadIdx.x % NCC, sg = threadIdx.x / NCC;
      const int ch = cc / NSUB, v = cc % NSUB;
      double *col = s_sub + (ch * NSUB + sg * RPS) * NSUB + v;
      double vals[RPS];
      double run = 0.0;
#pragma unroll
      for (int r = 0; r < RPS; ++r) vals[r] = col[r * NSUB];
#pragma unroll
      for (int r = 0; r < RPS; ++r) {
        run += vals[r];
        vals[r] = run;
      }
      s_tot[sg * NCC + cc] = run;
      __syncthreads();
      double carry = 0.0;
      for (int t = 0; t < sg; ++t) carry += s_tot[t * NCC + cc];
#pragma unroll
      for (int r = 0; r < RPS; ++r) col[r * NSUB] = vals[r] + carry;
    }
    __syncthreads();
    // pass A: this thread's unflipped slots (a warp's 32 slots stay in one sub-row)
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      const int uu = threadIdx.x + j * kSolverThreads;
      const int x = fslot ? S - 1 - uu : uu;
      const int y = s_yofx[x];
      int k = 0;
      bool occ = y != kEmptyY;
      if (occ) {
        k = s_kofx[x];
        occ = CHUNK || owned_key(flipp(s_key[y], frank, D.npad));
      }
      int qy = 0;
      if (occ) {
        if (CHUNK) {
          qy = y;
          s_qy[uu] = (int16_t)qy;
        } else if (search) {
          const int64_t c = s_key[y] >> LS;  // own chunk (self threshold)
          const int32_t ythr = (int32_t)((c > D.P ? D.P : c) * S);
          int a = 0, bnd = Sg;
          while (a < bnd) {
            const int mid = (a + bnd) >> 1;
            if (s_key[mid] < ythr) a = mid + 1;
            else bnd = mid;
          }
          qy = a;
          s_qy[uu] = (int16_t)qy;
        } else {
          qy = s_qy[uu];  // the previous code's: same rank frame
        }
      }
      const int u = x >> SUBL, v = qy >> SUBL;
      double acc[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
        acc[ch] = (occ && u > 0 && v > 0) ? s_sub[(ch * NSUB + (u - 1)) * NSUB + (v - 1)] : 0.0;
      const int xe = occ ? x : 0;  // candidates c < xe
      const int cend = (int)__reduce_max_sync(0xffffffffu, (unsigned)xe);
      const int xe_t[4] = {xe, xe - 1, xe - 2, xe - 3};  // c0 + t < xe  <=>  c0 < xe - t
      for (int c0 = u << SUBL; c0 < cend; c0 += 4) {
        const uint2 y4 = *reinterpret_cast<const uint2 *>(s_yofx + c0);  // 4 ranks (< 2^15)
        const int yc[4] = {(int)(y4.x & 0xffffu), (int)(y4.x >> 16), (int)(y4.y & 0xffffu),
                           (int)(y4.y >> 16)};
        PT pc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) pc[t] = s_p[c0 + t];
#pragma unroll
        for (int t = 0; t < 4; ++t) PsiT<NCH>::add(acc, pc[t], c0 < xe_t[t] && yc[t] < qy);
      }
      if (occ) {
        const double z = K.kde ? s_z[k] : 1.0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) accA[j][ch] += z * acc[ch];
      }
    }
    __syncthreads();
    // pass B: this thread's ranks (= its own sources k), coalesced
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      const int k = threadIdx.x + j * kSolverThreads;
      const bool ok = k < Sg && (CHUNK || owned_key(key_u[j]));
      const int y = frank ? Sg - 1 - k : k;
      const int x = ok ? s_xofy[y] : 0;
      const int qy = ok ? (int)s_qy[fslot ? S - 1 - x : x] : 0;
      const int xfull = (x >> SUBL) << SUBL;
      const int cbeg = ok ? (qy >> SUBL) << SUBL : S;  // candidates cbeg <= c < qy (none: S, 0)
      const int cstart = (int)__reduce_min_sync(0xffffffffu, (unsigned)cbeg);
      const int cend = (int)__reduce_max_sync(0xffffffffu, ok ? (unsigned)qy : 0u);
      double acc[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.0;
      // cbeg <= c0 + t < qy as one unsigned compare of c0 against per-t bounds:
      // (unsigned)(c0 - (cbeg - t)) < (unsigned)(qy - cbeg)   (idle lanes: cbeg = S, qy = 0)
      const int lo_t[4] = {cbeg, cbeg - 1, cbeg - 2, cbeg - 3};
      const unsigned span = (unsigned)(qy - cbeg);
      for (int c0 = cstart; c0 < cend; c0 += 4) {
        const uint2 x4 = *reinterpret_cast<const uint2 *>(s_xofy + c0);  // 4 slots (< 2^15)
        const int xc[4] = {(int)(x4.x & 0xffffu), (int)(x4.x >> 16), (int)(x4.y & 0xffffu),
                           (int)(x4.y >> 16)};
        PT pc[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) pc[t] = s_p[xc[t]];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          PsiT<NCH>::add(acc, pc[t], (unsigned)(c0 - lo_t[t]) < span && xc[t] < xfull);
      }
      if (ok) {
        const double z = K.kde ? s_z[k] : 1.0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) accB[j][ch] += z * acc[ch];
      }
    }
  }
  // the two halves of every query meet in shared memory (reusing the psi rows) by unflipped slot
  // (the slot-dimension position, so the store is coalesced in that dimension's rank order:
  // chunks write p1 order, blocks p0 order); the pass-B half moves, pass A is already by slot
  __syncthreads();
  double *s_acc = s_psi;  // [S][NCH] by unflipped slot
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = threadIdx.x + j * kSolverThreads;
    if (k >= Sg) continue;
    const int sl = s_slot[k];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) s_acc[sl * NCH + ch] = accB[j][ch];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int uu = threadIdx.x + j * kSolverThreads;
    if (uu >= Sg) continue;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) out[(lo + uu) * NCH + ch] = accA[j][ch] + s_acc[uu * NCH + ch];
  }
}

// ---- level 2, direct form ----------------------------------------------------------------
// The same chunk / block problem in one unflipped frame.  Sources sit in shared memory by slot
// (the slot dimension's local position) with their rank (order along the other dimension), the
// table T[c] = exp(s_c(x)) of the four sign codes and their weights.  A query with slot x and
// rank thresholds (qlo, qhi) -- dominated below: ranks < qlo, above: ranks >= qhi; its own rank
// (chunks) or the ranks outside its own chunk (blocks) -- splits every code's sum into
//   mid field: the 64 x 64 grid of (32 slots) x (32 ranks) cells, cell sums of psi_code
//              scattered with shared atomics, prefixed along each axis in the code's direction,
//              one lookup at the cell diagonal to the query's (slot cell, threshold rank cell);
//   near field: the sources of the query's slot cell (pass A) and of the thresholds' rank cells
//              (below: the cell of qlo; above: the rest of the cell of qhi - 1) outside that slot
//              cell (pass B), visited ONCE for all codes: the pair's quadrant
//              picks the code c, and z_c(t) psi_c(s) = w_s T_s[c] T_t[3 - c] is formed directly
//              (T[3 - c] = exp(-s_c): the opposite code), so nothing is masked out four times.
// The plain ECDF (one code, psi = w) keeps only the pairs of quadrant 0.
template <bool CHUNK, int NCH>
__global__ void __launch_bounds__(kSolverThreads) level2_direct(Dom2S D, Codes K) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RST = NSUB + 1;  // padded row: lookups of one slot cell spread over the banks
  double *s_sub = reinterpret_cast<double *>(smem);               // [NCH][NSUB][RST]
  double *s_tab = s_sub + NCH * NSUB * RST;                       // [S][4] by slot (16-byte aligned)
  double *s_w = s_tab + S * 4;                                    // [S][NCH] by slot
  double *s_tot = s_w + S * NCH;                                  // [kSolverThreads]
  double *s_sgn = s_tot + kSolverThreads;                         // [4][2] channel signs by code
  int32_t *s_key = reinterpret_cast<int32_t *>(s_sgn + 8);        // [S] rank-dimension key by rank
  int16_t *s_yofx = reinterpret_cast<int16_t *>(s_key + S);       // [S] rank by slot
  int16_t *s_xofy = s_yofx + S;                                   // [S] slot by rank
  int16_t *s_qlo = s_xofy + S;                                    // [S] thresholds by slot
  int16_t *s_qhi = s_qlo + S;
  double *out = CHUNK ? D.accc : D.accb;
  const int64_t g = blockIdx.x + (CHUNK ? D.c_lo : 0);  // unflipped chunk / block
  const int64_t lo = g * S;
  const int Sg = (int)(lo + S < D.n ? S : D.n - lo);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool kde = K.kde != 0;
  const bool all_owned = CHUNK || (D.c_lo == 0 && D.c_hi == D.P);
  const int2 *gpos = CHUNK ? D.gpos_c : D.gpos_b;
  const PtXW *gxw = CHUNK ? D.gxw_c : D.gxw_b;
  bool has_sign = false;
  for (int v = 0; v < NCH; ++v) has_sign = has_sign || K.kp[0].smask[v] != 0u;
  // empty slots / ranks: no rank, zero weight and table, key past every threshold
  for (int i = tid; i < S / 2; i += kSolverThreads)
    reinterpret_cast<uint32_t *>(s_yofx)[i] = (uint32_t)(uint16_t)kEmptyY * 0x10001u;
  if (Sg < S) {
    for (int i = tid; i < S * 4; i += kSolverThreads) s_tab[i] = 0.0;
    for (int i = tid; i < S * NCH; i += kSolverThreads) s_w[i] = 0.0;
    for (int i = Sg + tid; i < S; i += kSolverThreads) {
      s_xofy[i] = 0;
      s_key[i] = 0x7fffffff;
    }
  }
  if (tid < 8) s_sgn[tid] = (K.kde && (tid & 1) < NCH) ? chan_sign(K.kp[tid >> 1], tid & 1) : 1.0;
  __syncthreads();
  int32_t key_u[kL2Per];
  int slot[kL2Per];
  double accA[kL2Per][NCH], accB[kL2Per][NCH];
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = tid + j * kSolverThreads;
    const bool live = k < Sg;
    const int2 pp = live ? gpos[lo + k] : make_int2((int32_t)lo, 0);
    key_u[j] = pp.y;
    slot[j] = pp.x - (int32_t)lo;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) accA[j][ch] = accB[j][ch] = 0.0;
    if (!live) continue;
    const PtXW r = gxw[lo + k];
    double4 t4 = make_double4(1.0, 1.0, 1.0, 1.0);
    if (kde) {
      t4.x = exp(code_s(K.kp[0], r.x0, r.x1));
      t4.y = exp(code_s(K.kp[1], r.x0, r.x1));
      t4.z = exp(code_s(K.kp[2], r.x0, r.x1));
      t4.w = exp(code_s(K.kp[3], r.x0, r.x1));
    }
    s_xofy[k] = (int16_t)slot[j];
    s_yofx[slot[j]] = (int16_t)k;
    s_key[k] = pp.y;
    reinterpret_cast<double4 *>(s_tab)[slot[j]] = t4;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) s_w[slot[j] * NCH + ch] = ch ? r.w1 : r.w0;
  }
  __syncthreads();
  if (!CHUNK) {
    // block thresholds by rank: the ranks of the query's own chunk [qlo, qhi) are a run around
    // it (a block holds ~S / P points of a chunk), found by walking the neighbours; a long run
    // (clustered data) falls back to fixed-step searches.  Keys < 2^31 - 1, so a clamped bound
    // still counts every live key of the last chunk; empty ranks hold 2^31 - 1.
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      const int y = tid + j * kSolverThreads;
      if (y >= Sg) continue;
      const int64_t c = key_u[j] >> LS;
      const int32_t t_lo = (int32_t)(c * S);
      const int32_t t_hi = (c + 1) * S > 0x7fffffff ? 0x7fffffff : (int32_t)((c + 1) * S);
      int a = y, b = y + 1, steps = 0;
      while (a > 0 && s_key[a - 1] >= t_lo && steps < 8) --a, ++steps;
      while (b < Sg && s_key[b] < t_hi && steps < 16) ++b, ++steps;
      if (steps >= 8) {
        a = b = 0;
#pragma unroll
        for (int step = S / 2; step > 0; step >>= 1) {
          if (s_key[a + step - 1] < t_lo) a += step;
          if (s_key[b + step - 1] < t_hi) b += step;
        }
        if (s_key[a] < t_lo) ++a;
        if (s_key[b] < t_hi) ++b;
      }
      s_qlo[slot[j]] = (int16_t)a;
      s_qhi[slot[j]] = (int16_t)b;
    }
    __syncthreads();
  }
  // thresholds of this thread's slots (pass A / lookup order)
  int qloA[kL2Per], qhiA[kL2Per];
  bool occA[kL2Per];
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int x = tid + j * kSolverThreads;
    const int y = s_yofx[x];
    occA[j] = y != kEmptyY;
    qloA[j] = qhiA[j] = 0;
    if (!occA[j]) continue;
    if (CHUNK) {
      qloA[j] = y;
      qhiA[j] = y + 1;
    } else {
      const int64_t c = s_key[y] >> LS;
      occA[j] = all_owned || (c >= D.c_lo && c < D.c_hi);
      qloA[j] = s_qlo[x];
      qhiA[j] = s_qhi[x];
    }
  }
  // cell sums without atomics: a warp's 32 sources are one rank cell, so the cell row is the
  // warp's alone; lanes whose sources share a slot cell are grouped once (match.any), the
  // group's lowest lane stores the group's sum
  unsigned grp[kL2Per];
  int gmax[kL2Per];
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = tid + j * kSolverThreads;
    grp[j] = __match_any_sync(0xffffffffu, k < Sg ? (slot[j] >> SUBL) : NSUB + lane);
    gmax[j] = (int)__reduce_max_sync(0xffffffffu, (unsigned)__popc(grp[j]));
  }
  // ---- mid field, one code at a time ----
  for (int code = 0; code < K.n; ++code) {
    const int f0 = code & 1, f1 = (code >> 1) & 1;
    const int fslot = CHUNK ? f1 : f0, frank = CHUNK ? f0 : f1;
    __syncthreads();  // the previous code's lookups are done
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      const int k = tid + j * kSolverThreads;
      const bool live = k < Sg;
      const int u = slot[j] >> SUBL, v = k >> SUBL;
      // the warp's rank-cell row starts from zero (every rank cell has its warp, live or not)
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        s_sub[(ch * NSUB + v) * RST + lane] = 0.0;
        s_sub[(ch * NSUB + v) * RST + lane + 32] = 0.0;
      }
      __syncwarp();
      double psi[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
        psi[ch] = live ? s_w[slot[j] * NCH + ch] * s_tab[slot[j] * 4 + code] * s_sgn[code * 2 + ch]
                       : 0.0;
      double tot[NCH];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) tot[ch] = psi[ch];
      unsigned rem = grp[j] & ~(1u << lane);
      for (int it = 1; it < gmax[j]; ++it) {  // warp-uniform trip count
        const int src = rem ? __ffs(rem) - 1 : lane;
        rem &= rem - 1;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const double o = __shfl_sync(0xffffffffu, psi[ch], src);
          // partners are added in lane order by every member; only the sum's owner stores it
          if (src != lane) tot[ch] += o;
        }
      }
      if (!live) continue;
      if (lane == __ffs(grp[j]) - 1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) s_sub[(ch * NSUB + v) * RST + u] = tot[ch];
      }
      if (CHUNK) {
        // level 1: the code's coarse cell below the query's chunk and block (flipped frame).
        // The chunk's points run in p0 order, so a warp's reads walk one grid row in order.
        const int64_t P = D.P, bu = key_u[j] >> LS;
        const int64_t cc = f1 ? P - 1 - g : g, bb = f0 ? P - 1 - bu : bu;
        if (cc > 0 && bb > 0) {
          const double *gv = D.G + (((int64_t)code * P + cc - 1) * P + bb - 1) * NCH;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) accB[j][ch] += s_tab[slot[j] * 4 + 3 - code] * gv[ch];
        }
      }
    }
    __syncthreads();
    // cells are stored [channel][rank cell][slot cell].  Prefix along the slot cells (ascending,
    // or descending for a reversed slot frame): a warp per (channel, rank cell) row, lanes on
    // cells l and l + 32
    for (int row = warp; row < NCH * NSUB; row += kSolverThreads / 32) {
      double *rp = s_sub + row * RST;
      double a = rp[lane], b = rp[lane + 32];
      if (!fslot) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
          if (lane >= o) {
            a += ya;
            b += yb;
          }
        }
        b += __shfl_sync(0xffffffffu, a, 31);
      } else {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double ya = __shfl_down_sync(0xffffffffu, a, o), yb = __shfl_down_sync(0xffffffffu, b, o);
          if (lane + o < 32) {
            a += ya;
            b += yb;
          }
        }
        a += __shfl_sync(0xffffffffu, b, 0);
      }
      rp[lane] = a;
      rp[lane + 32] = b;
    }
    __syncthreads();
    // prefix along the rank cells: thread (segment sg, column cc), segment totals meet in s_tot
    {
      constexpr int NCC = NCH * NSUB, SEGS = kSolverThreads / NCC, RPS = NSUB / SEGS;
      const int cc = tid % NCC, sg = tid / NCC;
      const int ch = cc / NSUB, v = cc % NSUB;
      double *col = s_sub + (ch * NSUB + sg * RPS) * RST + v;
      double vals[RPS];
      double run = 0.0;
#pragma unroll
      for (int r = 0; r < RPS; ++r) vals[r] = col[r * RST];
      if (!frank) {
#pragma unroll
        for (int r = 0; r < RPS; ++r) vals[r] = run = run + vals[r];
      } else {
#pragma unroll
        for (int r = RPS - 1; r >= 0; --r) vals[r] = run = run + vals[r];
      }
      s_tot[sg * NCC + cc] = run;
      __syncthreads();
      double carry = 0.0;
      if (!frank) {
        for (int t = 0; t < sg; ++t) carry += s_tot[t * NCC + cc];
      } else {
        for (int t = SEGS - 1; t > sg; --t) carry += s_tot[t * NCC + cc];
      }
#pragma unroll
      for (int r = 0; r < RPS; ++r) col[r * RST] = vals[r] + carry;
    }
    __syncthreads();
    // lookup by slot
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
      if (!occA[j]) continue;
      const int x = tid + j * kSolverThreads;
      const int ui = fslot ? (x >> SUBL) + 1 : (x >> SUBL) - 1;
      // above: the cells past the one holding the last excluded rank qhi - 1
      const int vi = frank ? ((qhiA[j] - 1) >> SUBL) + 1 : (qloA[j] >> SUBL) - 1;
      if (ui < 0 || ui >= NSUB || vi < 0 || vi >= NSUB) continue;
      const double z = s_tab[x * 4 + (3 - code)];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) accA[j][ch] += z * s_sub[(ch * NSUB + vi) * RST + ui];
    }
  }
  // ---- near field, all codes at once ----
  // quadrant code of a pair: bit of dimension 0 / 1 set when the source lies above the query
  auto pair_value = [&](int code2, int xs, const double4 &tq) -> double {
    if (!kde) return code2 == 0 ? 1.0 : 0.0;
    // the query's factor is its table entry of the opposite code
    const double tt = (code2 & 2) ? ((code2 & 1) ? tq.x : tq.y) : ((code2 & 1) ? tq.z : tq.w);
    return s_tab[xs * 4 + code2] * tt;
  };
  // pass A: this thread's slots, the 32 slots of their cell (a warp's slots share the cell)
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int x = tid + j * kSolverThreads;
    const int c0 = (x >> SUBL) << SUBL;
    const int qlo = qloA[j], qhi = occA[j] ? qhiA[j] : 0x7ffe;  // idle lanes: nothing passes
    const int qlo_e = occA[j] ? qlo : 0;
    const double4 tq = reinterpret_cast<const double4 *>(s_tab)[x];
    double acc[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.0;
#pragma unroll 2
    for (int c = c0; c < c0 + SUB; c += 4) {
      const uint2 y4 = *reinterpret_cast<const uint2 *>(s_yofx + c);
      const int yc[4] = {(int)(y4.x & 0xffffu), (int)(y4.x >> 16), (int)(y4.y & 0xffffu),
                         (int)(y4.y >> 16)};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool below = yc[t] < qlo_e, above = yc[t] >= qhi && yc[t] != kEmptyY;
        const int sb = c + t > x ? 1 : 0, rb = above ? 1 : 0;
        const int code2 = CHUNK ? (rb | (sb << 1)) : (sb | (rb << 1));
        double kv = pair_value(code2, c + t, tq);
        kv = (below || above) ? kv : 0.0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          double wv = s_w[(c + t) * NCH + ch];
          if (has_sign) wv *= s_sgn[code2 * 2 + ch];
          acc[ch] = fma(wv, kv, acc[ch]);
        }
      }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) accA[j][ch] += acc[ch];
  }
  // pass B: this thread's ranks (its own sources), the threshold cells' ranks outside the
  // query's slot cell
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = tid + j * kSolverThreads;
    const int x = slot[j];
    bool ok = k < Sg;
    int qlo = k, qhi = k + 1;
    if (!CHUNK && ok) {
      const int64_t cu = key_u[j] >> LS;
      ok = all_owned || (cu >= D.c_lo && cu < D.c_hi);
      qlo = s_qlo[x];
      qhi = s_qhi[x];
    }
    const int lo_s = (qlo >> SUBL) << SUBL;
    int hi_e = (((qhi - 1) >> SUBL) << SUBL) + SUB;  // end of the cell holding rank qhi - 1
    hi_e = hi_e > Sg ? Sg : hi_e;
    const unsigned span_lo = ok ? (unsigned)(qlo - lo_s) : 0u;
    const unsigned span_hi = (ok && hi_e > qhi) ? (unsigned)(hi_e - qhi) : 0u;
    const int wmin = (int)__reduce_min_sync(0xffffffffu, ok ? (unsigned)lo_s : (unsigned)S);
    const int wmax = (int)__reduce_max_sync(0xffffffffu, ok ? (unsigned)hi_e : 0u);
    const int xcell = x >> SUBL;
    const double4 tq = reinterpret_cast<const double4 *>(s_tab)[x];
    double acc[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) acc[ch] = 0.0;
    for (int r0 = wmin; r0 < wmax; r0 += 4) {
      const uint2 x4 = *reinterpret_cast<const uint2 *>(s_xofy + r0);
      const int xr[4] = {(int)(x4.x & 0xffffu), (int)(x4.x >> 16), (int)(x4.y & 0xffffu),
                         (int)(x4.y >> 16)};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool below = (unsigned)(r0 + t - lo_s) < span_lo;
        const bool above = (unsigned)(r0 + t - qhi) < span_hi;
        const bool take = (below || above) && (xr[t] >> SUBL) != xcell;
        const int sb = xr[t] > x ? 1 : 0, rb = above ? 1 : 0;
        const int code2 = CHUNK ? (rb | (sb << 1)) : (sb | (rb << 1));
        double kv = pair_value(code2, xr[t], tq);
        kv = take ? kv : 0.0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          double wv = s_w[xr[t] * NCH + ch];
          if (has_sign) wv *= s_sgn[code2 * 2 + ch];
          acc[ch] = fma(wv, kv, acc[ch]);
        }
      }
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) accB[j][ch] += acc[ch];
  }
  // the two halves of every query meet in shared memory by slot; coalesced store in slot order
  __syncthreads();
  double *s_acc = s_sub;  // [S][NCH] by slot
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int k = tid + j * kSolverThreads;
    if (k >= Sg) continue;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) s_acc[slot[j] * NCH + ch] = accB[j][ch];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kL2Per; ++j) {
    const int uu = tid + j * kSolverThreads;
    if (uu >= Sg) continue;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) out[(lo + uu) * NCH + ch] = accA[j][ch] + s_acc[uu * NCH + ch];
  }
}

size_t level2_direct_smem(int nch) {
  return (size_t)nch * NSUB * (NSUB + 1) * 8 + (size_t)S * 32 + (size_t)nch * S * 8 +
         (size_t)kSolverThreads * 8 + 64 + (size_t)S * 4 + (size_t)S * 2 * 4;
}

size_t level2_self_smem(int nch) {
  return (size_t)nch * NSUB * NSUB * 8 + (size_t)nch * S * 8 + (size_t)kSolverThreads * 8 +
         (size_t)S * 8 + (size_t)S * 4 + (size_t)S * 2 * 5;
}

// out[v][t] = (acc_c[p1(t)][v] + acc_b[p0(t)][v] + (add_w ? w[v][t] : 0)) * mult / div
// (mult == 0: none, div == 0: none); acc_c carries the level-1 term
__global__ void self_finish_kernel(int64_t n, int nw,
                                   const double *__restrict__ accc, const double *__restrict__ accb,
                                   WPtr w, int add_w, double mult, double div,
                                   double *__restrict__ out, const int32_t *__restrict__ pos0,
                                   const int32_t *__restrict__ pos1, int64_t c_lo, int64_t c_hi) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cu = pos1[t] >> LS;
    if (cu < c_lo || cu >= c_hi) {  // another shard's query: exact zero (sum-reduce gathers)
      for (int v = 0; v < nw; ++v) out[v * n + t] = 0.0;
      continue;
    }
    const int64_t kc = pos1[t], kb = pos0[t];
    for (int v = 0; v < nw; ++v) {
      double r = accc[kc * nw + v] + accb[kb * nw + v];
      if (add_w) r = r + w.at(v, t);
      if (mult != 0.0) r = r * mult;
      if (div != 0.0) r = r / div;
      out[v * n + t] = r;
    }
  }
}

// ------------------------------------------------------------------------------------------
// host-side composition

struct Ranked {        // per-dimension ranking results (device)
  int32_t *order, *pos, *lower, *upper, *dense;
};

struct PtsWs {
  // ranking
  uint64_t *k;
  int32_t *v;
  RadixWs rw;
  int32_t *heads, *start, *ndist;
  Ranked r[FCG_MAX_DIM];
  // d = 2 dominance
  int32_t *bychunk, *byblock, *Q0f, *Q1f, *kc, *kb, *qc_list, *qc_start, *qb_list, *qb_start,
      *cursor;
  double *G, *psi, *expo, *F, *lat, *scratch;
  int64_t P, npad, lat_cells;
};

int64_t pad_of(int64_t n) { return ceil_div(n, S) * S; }

void carve(Workspace &W, PtsWs &p, int64_t n, int d, int nch, bool need_dom, bool need_kde,
           int64_t lat_cells) {
  p.k = W.take<uint64_t>(n);
  p.v = W.take<int32_t>(n);
  p.rw.keys_alt = W.take<uint64_t>(n);
  p.rw.vals_alt = W.take<int32_t>(n);
  p.rw.hist = W.take<int32_t>(radix_ws_hist_elems(n));
  p.rw.partial = W.take<int32_t>(scan_ws_partial_elems(256 * (n / kSortTile + 1) + n + 2));
  p.heads = W.take<int32_t>(n);
  p.start = W.take<int32_t>(n + 1);
  p.ndist = W.take<int32_t>(FCG_MAX_DIM);
  for (int k = 0; k < d; ++k) {
    p.r[k].order = W.take<int32_t>(n);
    p.r[k].pos = W.take<int32_t>(n);
    p.r[k].lower = W.take<int32_t>(n);
    p.r[k].upper = W.take<int32_t>(n);
    p.r[k].dense = W.take<int32_t>(n);
  }
  p.P = ceil_div(n, S);
  p.npad = p.P * S;
  p.lat_cells = lat_cells;
  if (lat_cells > 0) {
    p.lat = W.take<double>(lat_cells);
  } else {
    p.lat = nullptr;
  }
  p.scratch = W.take<double>(scan_scratch_bound());
  if (need_dom) {
    p.bychunk = W.take<int32_t>(n);
    p.byblock = W.take<int32_t>(n);
    p.Q0f = W.take<int32_t>(n);
    p.Q1f = W.take<int32_t>(n);
    p.kc = W.take<int32_t>(n);
    p.kb = W.take<int32_t>(n);
    p.qc_list = W.take<int32_t>(n);
    p.qb_list = W.take<int32_t>(n);
    p.qc_start = W.take<int32_t>(p.P + 2);
    p.qb_start = W.take<int32_t>(p.P + 2);
    p.cursor = W.take<int32_t>(p.P + 2);
    p.G = W.take<double>(p.P * p.P * nch * (need_kde ? 4 : 1));
    p.psi = W.take<double>((size_t)n * nch);
    p.F = W.take<double>((size_t)n * nch);
  }
  if (need_kde) p.expo = W.take<double>(n);
}

// ties = false: only the order and the positions (distinct coordinates, the self path).
// mask: the dimension's digit mask (radix_digit_masks_f64), or ~0u to compute it here (syncs).
int rank_dim(const double *x, int64_t n, int d, int k, PtsWs &p, cudaStream_t st, bool ties = true,
             uint32_t mask = ~0u) {
  if (!ties && mask != ~0u && __builtin_popcount(mask & 0xFu) >= 2) {
    // continuous data, positions only: sort the keys' top halves, order the short runs of
    // equal top halves by the low halves (falls through when a run is too long)
    bool done = false;
    FCG_TRY(rank_order_split_f64(x + k, n, d, mask, reinterpret_cast<uint32_t *>(p.k), p.v, p.rw,
                                 p.ndist + k, p.r[k].order, p.r[k].pos, &done, st));
    if (done) return FCG_OK;
  }
  FCG_TRY(radix_init_f64(x + k, n, d, p.k, p.v, st));
  if (mask == ~0u) FCG_TRY(radix_sort_pairs_pruned(p.k, p.v, n, p.rw, st));
  else FCG_TRY(radix_sort_pairs_mask(p.k, p.v, n, mask, p.rw, st));
  FCG_CUDA_TRY(cudaMemcpyAsync(p.r[k].order, p.v, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  if (!ties)
    return rank_outputs(p.k, p.v, n, p.r[k].pos, nullptr, nullptr, nullptr, p.heads, p.start,
                        p.rw.partial, nullptr, st);
  return rank_outputs(p.k, p.v, n, p.r[k].pos, p.r[k].lower, p.r[k].upper, p.r[k].dense, p.heads,
                      p.start, p.rw.partial, p.ndist + k, st);
}

int group_by(const int32_t *order, const int32_t *pos_other, int64_t n, int64_t P, int32_t *out,
             PtsWs &p, cudaStream_t st) {
  {
    FCG_PROF("pts_group_keys", st);
    group_keys<<<grid_for(n, 256), 256, 0, st>>>(order, pos_other, n, p.k, p.v);
    FCG_LAUNCH_CHECK();
  }
  int bits = 0;
  while ((int64_t(1) << bits) < P) ++bits;
  FCG_TRY(radix_sort_pairs(p.k, p.v, n, 0, bits < 1 ? 8 : ((bits + 7) / 8) * 8, p.rw, st));
  FCG_CUDA_TRY(cudaMemcpyAsync(out, p.v, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  return FCG_OK;
}

int bucket(const int32_t *keys, int64_t n, int64_t nb, int32_t *list, int32_t *start,
           int32_t *cursor, PtsWs &p, cudaStream_t st) {
  FCG_CUDA_TRY(cudaMemsetAsync(start, 0, (size_t)(nb + 1) * 4, st));
  {
    FCG_PROF("pts_bucket", st);
    bucket_count<<<grid_for(n, 256), 256, 0, st>>>(keys, n, start);
    FCG_LAUNCH_CHECK();
  }
  FCG_TRY(scan_i32(start, start, nb + 1, false, p.rw.partial, st));
  FCG_CUDA_TRY(cudaMemcpyAsync(cursor, start, (size_t)(nb + 1) * 4, cudaMemcpyDeviceToDevice, st));
  FCG_PROF("pts_bucket", st);
  bucket_fill<<<grid_for(n, 256), 256, 0, st>>>(keys, n, cursor, list);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

// Lower-left dominance sums in one orientation (f0, f1) of the shared ranking.
// psi: [nch][n] (nch <= 2), thresholds already in p.Q0f / p.Q1f; out: [nch][n].
int dom2d(PtsWs &p, int64_t n, int nch, int f0, int f1, const double *psi, double *out,
          cudaStream_t st) {
  Dom2 D;
  D.n = n;
  D.nq = n;
  D.P = p.P;
  D.npad = p.npad;
  D.nch = nch;
  D.f0 = f0;
  D.f1 = f1;
  D.pos0 = p.r[0].pos;
  D.pos1 = p.r[1].pos;
  D.bychunk = p.bychunk;
  D.byblock = p.byblock;
  D.psi = psi;
  D.Q0f = p.Q0f;
  D.Q1f = p.Q1f;
  D.out = out;
  D.G = p.G;
  D.qc_list = p.qc_list;
  D.qc_start = p.qc_start;
  D.qb_list = p.qb_list;
  D.qb_start = p.qb_start;
  const int64_t P = p.P;
  {  // general thresholds: bucket the queries by chunk and by block
    {
      FCG_PROF("pts_query_keys", st);
      query_keys<<<grid_for(n, 256), 256, 0, st>>>(D, p.kc, p.kb);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(bucket(p.kc, n, P + 1, p.qc_list, p.qc_start, p.cursor, p, st));
    FCG_TRY(bucket(p.kb, n, P + 1, p.qb_list, p.qb_start, p.cursor, p, st));
  }
  // level 1: coarse grid (rows in shared-memory segments of TB blocks)
  {
    FCG_PROF("pts_coarse_hist", st);
    const int64_t TB = coarse_tb(nch);
    const int64_t nseg = ceil_div(P, TB);
    const size_t row_smem = (size_t)(TB < P ? TB : P) * nch * sizeof(double);
    FCG_CUDA_TRY(cudaFuncSetAttribute(coarse_rows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kCoarseRowBytes));
    coarse_rows_smem<<<dim3((unsigned)P, (unsigned)nseg), 512, row_smem, st>>>(D, TB);
    FCG_LAUNCH_CHECK();
  }
  LatShape gs;
  gs.d = 3;
  gs.dims[0] = P;
  gs.dims[1] = P;
  gs.dims[2] = nch;
  Epi inplace;
  FCG_TRY(scan_axis<double>(p.G, gs, 1, false, inplace, p.scratch, st));
  FCG_TRY(scan_axis<double>(p.G, gs, 0, false, inplace, p.scratch, st));
  {
    FCG_PROF("pts_coarse_query", st);
    coarse_query<<<grid_for(n, 256), 256, 0, st>>>(D);
    FCG_LAUNCH_CHECK();
  }
  // level 2: own chunk, own block
  const size_t sm = level2_smem(nch);
  if (nch == 1) {
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_solver<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_solver<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    {
      FCG_PROF("pts_level2_chunk", st);
      level2_solver<true, 1><<<(unsigned)P, kSolverThreads, sm, st>>>(D);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_level2_block", st);
    level2_solver<false, 1><<<(unsigned)P, kSolverThreads, sm, st>>>(D);
    FCG_LAUNCH_CHECK();
  } else {
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_solver<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_solver<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    {
      FCG_PROF("pts_level2_chunk", st);
      level2_solver<true, 2><<<(unsigned)P, kSolverThreads, sm, st>>>(D);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_level2_block", st);
    level2_solver<false, 2><<<(unsigned)P, kSolverThreads, sm, st>>>(D);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}

// every dimension's ranking after one digit-mask read-back for all of them
int rank_all(const double *x, int64_t n, int d, PtsWs &p, cudaStream_t st, bool ties = true) {
  uint32_t masks[FCG_MAX_DIM];
  FCG_TRY(radix_digit_masks_f64(x, n, d, reinterpret_cast<unsigned long long *>(p.rw.hist),
                                masks, st));
  for (int k = 0; k < d; ++k) FCG_TRY(rank_dim(x, n, d, k, p, st, ties, masks[k]));
  return FCG_OK;
}


// d == 1 dominance: dst[i] = sum over sorted positions before (rev: after) i of vals, as the
// reference computes it (inclusive cumsum minus self).  lat: 2n doubles of scratch.
int sorted_exclusive(const double *vals, const int32_t *order, int64_t n, bool rev, double *lat,
                     double *scratch, double *dst, cudaStream_t st) {
  {
    FCG_PROF("pts_sorted_w", st);
    permute_kernel<<<grid_for(n, 256), 256, 0, st>>>(vals, order, n, lat, lat + n);
    FCG_LAUNCH_CHECK();
  }
  LatShape s1;
  s1.d = 1;
  s1.dims[0] = n;
  Epi inplace;
  FCG_TRY(scan_axis<double>(lat + n, s1, 0, rev, inplace, scratch, st));
  FCG_PROF("pts_gather", st);
  excl_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(lat + n, lat, order, n, dst);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

struct SelfWs {
  PtXW *xw;
  int2 *gpos_c, *gpos_b;
  PtXW *gxw_c, *gxw_b;
  double *accc, *accb;  // [n][nw]
};

void carve_self(Workspace &W, SelfWs &q, int64_t n, int nw) {
  q.xw = W.take<PtXW>(n);
  q.gpos_c = W.take<int2>(n);
  q.gpos_b = W.take<int2>(n);
  q.gxw_c = W.take<PtXW>(n);
  q.gxw_b = W.take<PtXW>(n);
  q.accc = W.take<double>((size_t)n * nw);
  q.accb = W.take<double>((size_t)n * nw);
}

// Strict-dominance sums at the points for d = 2 in group order: the plain ECDF (kde = 0, one
// orientation, psi = w) or the 2^2 Laplacian orientations (kde = 1, psi = w e^{s}, each term
// weighted by e^{-s} at the query).  out[v][t] = (sum + (add_w ? w : 0)) * mult / div.
int self_dom2d(const double *x, WPtr w, int64_t n, int nw, int kde, const double *h,
               const double *centre, int add_w, double mult, double div, PtsWs &p, SelfWs &q,
               double *out, cudaStream_t st, const unsigned *smask = nullptr, int shard = 0,
               int nshards = 1) {
  FCG_TRY(rank_all(x, n, 2, p, st, false));
  const int g = grid_for(n, 256);
  {
    FCG_PROF("pts_group", st);
    pack_points_kernel<<<g, 256, 0, st>>>(x, w, nw, n, q.xw);
    const size_t gsm = group_self_smem(n);
    const int64_t cells = group_self_cells(n);
    const int sh = group_self_shift(n);
    FCG_CUDA_TRY(cudaFuncSetAttribute(group_self_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)gsm));
    group_self_kernel<<<(unsigned)p.P, kGroupThreads, gsm, st>>>(p.r[1].order, p.r[0].pos, q.xw, n,
                                                                  cells, sh, q.gpos_c, q.gxw_c);
    group_self_kernel<<<(unsigned)p.P, kGroupThreads, gsm, st>>>(p.r[0].order, p.r[1].pos, q.xw, n,
                                                                  cells, sh, q.gpos_b, q.gxw_b);
    FCG_LAUNCH_CHECK();
  }
  Dom2S D{};
  D.n = n;
  D.P = p.P;
  D.npad = p.npad;
  D.nch = nw;
  D.kde = kde;
  D.gpos_c = q.gpos_c;
  D.gpos_b = q.gpos_b;
  D.gxw_c = q.gxw_c;
  D.gxw_b = q.gxw_b;
  D.accc = q.accc;
  D.accb = q.accb;
  D.G = p.G;
  const int64_t P = p.P;
  // query shard: a contiguous range of chunks (points in p1 rank order)
  D.c_lo = P * shard / nshards;
  D.c_hi = P * (shard + 1) / nshards;
  const unsigned nchunk = (unsigned)(D.c_hi - D.c_lo);
  const bool direct = [] {  // FCG_LEVEL2=codes: the per-code masked passes (A/B runs, tests)
    const char *e = getenv("FCG_LEVEL2");
    return !(e && std::string(e) == "codes");
  }();
  const size_t sm = direct ? level2_direct_smem(nw) : level2_self_smem(nw);
  if (direct) {
    if (nw == 1) {
      FCG_CUDA_TRY(cudaFuncSetAttribute(level2_direct<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      FCG_CUDA_TRY(cudaFuncSetAttribute(level2_direct<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    } else {
      FCG_CUDA_TRY(cudaFuncSetAttribute(level2_direct<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      FCG_CUDA_TRY(cudaFuncSetAttribute(level2_direct<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    }
  } else if (nw == 1) {
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_codes<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_codes<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  } else {
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_codes<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    FCG_CUDA_TRY(cudaFuncSetAttribute(level2_codes<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  }
  // every code's coarse grid from one pass over the points (rows built in shared-memory
  // segments of TB blocks), both prefix axes of all grids in two scans, one query pass
  Codes K{};
  K.n = kde ? 4 : 1;
  K.kde = kde;
  for (int code = 0; code < K.n; ++code) {
    KdeP &kp = K.kp[code];
    kp.d = 2;
    kp.code = code;
    for (int v = 0; v < nw; ++v) kp.smask[v] = smask ? smask[v] : 0u;
    for (int k = 0; k < 2; ++k) {
      const double sgn = ((code >> k) & 1) ? -1.0 : 1.0;  // DeltaVector.from_code
      kp.c[k] = kde ? centre[k] : 0.0;
      kp.a[k] = kde ? sgn / h[k] : 0.0;
    }
  }
  {
    FCG_PROF("pts_coarse_hist", st);
    const size_t csm = (size_t)S * 2 * nw * sizeof(double) + (size_t)S * sizeof(int32_t);
    if (nw == 1) {
      FCG_CUDA_TRY(cudaFuncSetAttribute(coarse_rows_codes<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
      coarse_rows_codes<1><<<(unsigned)P, kCoarseThreads, csm, st>>>(D, K);
    } else {
      FCG_CUDA_TRY(cudaFuncSetAttribute(coarse_rows_codes<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
      coarse_rows_codes<2><<<(unsigned)P, kCoarseThreads, csm, st>>>(D, K);
    }
    FCG_LAUNCH_CHECK();
  }
  {  // the block axis is prefixed by the row kernel; the chunk axis in one scan pass
    LatShape gs;
    gs.d = 4;
    gs.dims[0] = K.n;
    gs.dims[1] = P;
    gs.dims[2] = P;
    gs.dims[3] = nw;
    Epi inplace;
    FCG_TRY(scan_axis<double>(p.G, gs, 1, false, inplace, p.scratch, st));
  }
  // level 2: every code of a chunk / block in one CTA (the chunk solvers for the shard's chunks)
  {
    FCG_PROF("pts_level2_chunk", st);
    if (nchunk > 0) {
      if (direct) {
        if (nw == 1) level2_direct<true, 1><<<nchunk, kSolverThreads, sm, st>>>(D, K);
        else level2_direct<true, 2><<<nchunk, kSolverThreads, sm, st>>>(D, K);
      } else if (nw == 1) {
        level2_codes<true, 1><<<nchunk, kSolverThreads, sm, st>>>(D, K);
      } else {
        level2_codes<true, 2><<<nchunk, kSolverThreads, sm, st>>>(D, K);
      }
    }
    FCG_LAUNCH_CHECK();
  }
  {
    FCG_PROF("pts_level2_block", st);
    if (direct) {
      if (nw == 1) level2_direct<false, 1><<<(unsigned)P, kSolverThreads, sm, st>>>(D, K);
      else level2_direct<false, 2><<<(unsigned)P, kSolverThreads, sm, st>>>(D, K);
    } else if (nw == 1) {
      level2_codes<false, 1><<<(unsigned)P, kSolverThreads, sm, st>>>(D, K);
    } else {
      level2_codes<false, 2><<<(unsigned)P, kSolverThreads, sm, st>>>(D, K);
    }
    FCG_LAUNCH_CHECK();
  }
  FCG_PROF("pts_finish", st);
  self_finish_kernel<<<g, 256, 0, st>>>(n, nw, q.accc, q.accb, w,
                                       add_w, mult, div, out, p.r[0].pos, p.r[1].pos, D.c_lo,
                                       D.c_hi);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

int make_q(const int32_t *a, int64_t n, int kind, int64_t npad, int32_t *out, cudaStream_t st) {
  FCG_PROF("pts_make_q", st);
  make_q_kernel<<<grid_for(n, 256), 256, 0, st>>>(a, n, kind, npad, out);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

#include "points_nd.cuh"

int check_pts(int64_t n, int32_t d) {
  if (d < 1 || d > FCG_MAX_DIM) return fail(FCG_EUNSUPPORTED, "dimension out of range");
  if (n < 0) return fail(FCG_EINVAL, "n must be >= 0");
  if (n >= (int64_t(1) << 31) - 1) return fail(FCG_EUNSUPPORTED, "n must be < 2^31 - 1");
  return FCG_OK;
}

// lattice budget for the rank-lattice route
int64_t lattice_budget(int64_t n) {
  int64_t b = 4 * n;
  if (b < (int64_t(1) << 22)) b = int64_t(1) << 22;
  if (b > (int64_t(1) << 30)) b = int64_t(1) << 30;
  return b;
}

}  // namespace

}  // namespace fcg

using namespace fcg;

extern "C" int fcg_distinct(const double *x, int64_t n, int32_t d, int32_t *flags, void *ws,
                            size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  Workspace W(ws);
  uint64_t *k = W.take<uint64_t>(n);
  int32_t *v = W.take<int32_t>(n);
  RadixWs rw;
  rw.keys_alt = W.take<uint64_t>(n);
  rw.vals_alt = W.take<int32_t>(n);
  rw.hist = W.take<int32_t>(radix_ws_hist_elems(n));
  rw.partial = W.take<int32_t>(scan_ws_partial_elems(256 * (n / kSortTile + 1) + 2));
  int32_t *dflag = W.take<int32_t>(FCG_MAX_DIM);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  FCG_CUDA_TRY(cudaMemsetAsync(dflag, 0, FCG_MAX_DIM * 4, st));
  for (int kd = 0; kd < d; ++kd) {
    FCG_TRY(radix_init_f64(x + kd, n, d, k, v, st));
    FCG_TRY(radix_sort_pairs_pruned(k, v, n, rw, st));
    if (n > 1) {
      FCG_PROF("pts_distinct", st);
      adjacent_equal_kernel<<<grid_for(n, 256), 256, 0, st>>>(k, n, dflag + kd);
      FCG_LAUNCH_CHECK();
    }
  }
  int32_t h[FCG_MAX_DIM];
  FCG_TRY(read_small(h, dflag, FCG_MAX_DIM * 4, st));
  for (int kd = 0; kd < d; ++kd) flags[kd] = h[kd] ? 0 : 1;
  return FCG_OK;
}

namespace fcg {
namespace {
// One at-points request: out[j] = sum_i w_i prod_k [x_ik <= / < x_jk] (delta) or, survival,
// prod_k [x_ik > x_jk]; divided by n when scaled.
struct PtsReq {
  const int32_t *delta;
  int survival;
  double *out;
};

// Requests sharing one ranking of every dimension (the expensive part at BASELINE config 2).
int ecdf_points_multi(const double *x, int64_t n, int d, const double *w, int scaled,
                      const PtsReq *req, int nreq, void *ws, size_t *ws_bytes, cudaStream_t st) {
  FCG_TRY(check_pts(n, d));
  for (int q = 0; q < nreq; ++q)
    if (!req[q].survival)
      for (int k = 0; k < d; ++k)
        if (req[q].delta[k] != 1 && req[q].delta[k] != -1)
          return fail(FCG_EINVAL, "delta entries must be -1 or +1");
  // Workspace is sized for the worst case of the routes chosen at run time.
  const bool dom_ok = (d == 2 && dom_fits(n, 1));
  const int64_t budget = lattice_budget(n);
  Workspace W(ws);
  PtsWs p;
  carve(W, p, n, d, 1, dom_ok, false, d == 1 ? n : budget);
  NdWs nq{};
  if (nd_route(n, d)) carve_nd(W, nq, n, d, 1, 1, false);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  const double div = scaled ? (double)n : 0.0;

  if (d == 1) {  // sort, prefix (or suffix) scan of sorted weights, gather
    FCG_TRY(rank_dim(x, n, 1, 0, p, st));
    {
      FCG_PROF("pts_sorted_w", st);
      gather_sorted_w<<<grid_for(n, 256), 256, 0, st>>>(p.r[0].order, w, n, p.lat);
      FCG_LAUNCH_CHECK();
    }
    // both scan directions may be requested: the prefix first, the suffix from a fresh copy
    for (int q = 0; q < nreq; ++q) {
      const bool rev = req[q].survival != 0;
      if (q > 0) {
        FCG_PROF("pts_sorted_w", st);
        gather_sorted_w<<<grid_for(n, 256), 256, 0, st>>>(p.r[0].order, w, n, p.lat);
        FCG_LAUNCH_CHECK();
      }
      LatShape s1;
      s1.d = 1;
      s1.dims[0] = n;
      Epi inplace;
      FCG_TRY(scan_axis<double>(p.lat, s1, 0, rev, inplace, p.scratch, st));
      const int32_t *qq = req[q].survival ? p.r[0].upper
                                          : (req[q].delta[0] > 0 ? p.r[0].upper : p.r[0].lower);
      {
        FCG_PROF("pts_gather", st);
        gather1d_kernel<<<grid_for(n, 256), 256, 0, st>>>(p.lat, qq, n, rev ? 1 : 0, req[q].out);
        FCG_LAUNCH_CHECK();
      }
      FCG_PROF("pts_finish", st);
      finish_ecdf_kernel<<<grid_for(n, 256), 256, 0, st>>>(req[q].out, n, w, 0, div);
      FCG_LAUNCH_CHECK();
    }
    return FCG_OK;
  }

  // rank every dimension once; the distinct counts decide the route (host sync)
  FCG_TRY(rank_all(x, n, d, p, st));
  int32_t nd[FCG_MAX_DIM];
  FCG_TRY(read_small(nd, p.ndist, d * 4, st));
  double cells = 1.0;
  for (int k = 0; k < d; ++k) cells *= (double)nd[k];

  if (cells <= (double)budget) {  // rank lattice route
    for (int q = 0; q < nreq; ++q) {
      const int survival = req[q].survival;
      const int32_t *delta = req[q].delta;
      double *out = req[q].out;
      RankLat r;
      LatShape s;
      r.d = s.d = d;
      bool rev[FCG_MAX_DIM];
      int64_t stride = 1;
      for (int k = d - 1; k >= 0; --k) {
        r.dense[k] = p.r[k].dense;
        r.shift[k] = survival ? 1 : (delta[k] > 0 ? 0 : -1);
        r.dims[k] = s.dims[k] = nd[k];
        r.stride[k] = stride;
        stride *= nd[k];
        rev[k] = survival != 0;
      }
      const bool unit = (w == nullptr);
      {
        FCG_PROF("lattice_zero", st);
        FCG_CUDA_TRY(cudaMemsetAsync(p.lat, 0, (size_t)stride * (unit ? 4 : 8), st));
      }
      {
        FCG_PROF("pts_rank_scatter", st);
        if (unit) rank_scatter_kernel<true><<<grid_for(n, 256), 256, 0, st>>>(r, n, w, p.lat);
        else rank_scatter_kernel<false><<<grid_for(n, 256), 256, 0, st>>>(r, n, w, p.lat);
        FCG_LAUNCH_CHECK();
      }
      Epi inplace;
      if (unit) {
        FCG_TRY(scan_lattice<int32_t>(reinterpret_cast<int32_t *>(p.lat), s, rev, inplace,
                                      reinterpret_cast<int32_t *>(p.scratch), st));
        FCG_PROF("pts_gather", st);
        rank_gather_kernel<int32_t><<<grid_for(n, 256), 256, 0, st>>>(
            r, n, reinterpret_cast<const int32_t *>(p.lat), div, out);
      } else {
        FCG_TRY(scan_lattice<double>(p.lat, s, rev, inplace, p.scratch, st));
        FCG_PROF("pts_gather", st);
        rank_gather_kernel<double><<<grid_for(n, 256), 256, 0, st>>>(r, n, p.lat, div, out);
      }
      FCG_LAUNCH_CHECK();
    }
    return FCG_OK;
  }

  if (dom_ok) {  // d == 2 rank-space dominance
    FCG_TRY(group_by(p.r[0].order, p.r[1].pos, n, p.P, p.bychunk, p, st));
    FCG_TRY(group_by(p.r[1].order, p.r[0].pos, n, p.P, p.byblock, p, st));
    {
      FCG_PROF("pts_psi", st);
      if (w) FCG_CUDA_TRY(cudaMemcpyAsync(p.psi, w, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
      else fill_f64<<<grid_for(n, 256), 256, 0, st>>>(p.psi, n, 1.0);
      FCG_LAUNCH_CHECK();
    }
    for (int q = 0; q < nreq; ++q) {
      const int survival = req[q].survival;
      const int32_t *delta = req[q].delta;
      if (survival) {  // [x_i > x_t] <=> flipped p_i < npad - upper_t
        FCG_TRY(make_q(p.r[0].upper, n, 2, p.npad, p.Q0f, st));
        FCG_TRY(make_q(p.r[1].upper, n, 2, p.npad, p.Q1f, st));
      } else {
        FCG_TRY(make_q(delta[0] > 0 ? p.r[0].upper : p.r[0].lower, n, 0, p.npad, p.Q0f, st));
        FCG_TRY(make_q(delta[1] > 0 ? p.r[1].upper : p.r[1].lower, n, 0, p.npad, p.Q1f, st));
      }
      FCG_TRY(dom2d(p, n, 1, survival, survival, p.psi, req[q].out, st));
      FCG_PROF("pts_finish", st);
      finish_ecdf_kernel<<<grid_for(n, 256), 256, 0, st>>>(req[q].out, n, w, 0, div);
      FCG_LAUNCH_CHECK();
    }
    return FCG_OK;
  }

  if (d == 2) return dom_too_large(n);
  if (nd_route(n, d)) {  // coarse grid + slab remainder in rank space
    for (int q = 0; q < nreq; ++q) {
      int rev[FCG_MAX_DIM], qoff[FCG_MAX_DIM];
      const int32_t *thr[FCG_MAX_DIM];
      for (int k = 0; k < d; ++k) {
        rev[k] = req[q].survival ? 1 : 0;  // [x_i > x_t] <=> p_i >= upper_t
        qoff[k] = 0;
        thr[k] = (req[q].survival || req[q].delta[k] > 0) ? p.r[k].upper : p.r[k].lower;
      }
      FCG_TRY(dom_nd(p, nq, n, d, 1, NdW{{w, nullptr}, 1}, rev, qoff, thr, req[q].out, 0, 1, st));
      FCG_PROF("pts_finish", st);
      finish_ecdf_kernel<<<grid_for(n, 256), 256, 0, st>>>(req[q].out, n, w, 0, div);
      FCG_LAUNCH_CHECK();
    }
    return FCG_OK;
  }
  // direct tiles (d >= 7, or too few points for the rank-space route to pay)
  for (int q = 0; q < nreq; ++q) {
    Brute B;
    B.n = n;
    B.d = d;
    B.x = x;
    B.w = w;
    B.nw = 1;
    B.out = req[q].out;
    for (int k = 0; k < d; ++k) B.sign[k] = req[q].survival ? 2 : req[q].delta[k];
    {
      FCG_PROF("pts_brute", st);
      brute_kernel<BR_ECDF><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(B);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_finish", st);
    finish_ecdf_kernel<<<grid_for(n, 256), 256, 0, st>>>(req[q].out, n, w, 0, div);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}
}  // namespace
}  // namespace fcg

extern "C" int fcg_ecdf_points(const double *x, int64_t n, int32_t d, const double *w,
                               const int32_t *delta, int32_t survival, int32_t scaled,
                               double *out, void *ws, size_t *ws_bytes, void *stream) {
  const PtsReq r{delta, survival, out};
  return ecdf_points_multi(x, n, d, w, scaled, &r, 1, ws, ws_bytes, as_stream(stream));
}

extern "C" int fcg_ecdf_esf_points(const double *x, int64_t n, int32_t d, const double *w,
                                   const int32_t *delta, int32_t scaled, double *out_ecdf,
                                   double *out_esf, void *ws, size_t *ws_bytes, void *stream) {
  const PtsReq r[2] = {{delta, 0, out_ecdf}, {delta, 1, out_esf}};
  return ecdf_points_multi(x, n, d, w, scaled, r, 2, ws, ws_bytes, as_stream(stream));
}

extern "C" int fcg_dnc_ecdf(const double *x, int64_t n, int32_t d, const double *w,
                            int32_t include_self, int32_t scaled, double *out, void *ws,
                            size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d == 2 && !dom_fits(n, 1)) return dom_too_large(n);
  const bool dom_ok = d == 2;
  Workspace W(ws);
  PtsWs p;
  const bool nd = nd_route(n, d);
  carve(W, p, n, nd ? d : (d < 2 ? d : 2), 1, dom_ok, false, d == 1 ? 2 * n : 0);
  SelfWs q{};
  if (dom_ok) carve_self(W, q, n, 1);
  NdWs nq{};
  if (nd) carve_nd(W, nq, n, d, 1, 1, false);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  cudaStream_t st = as_stream(stream);
  const double div = scaled ? (double)n : 0.0;
  if (d == 1) {  // argsort, cumsum - self (dnc.py:543-547)
    FCG_TRY(rank_dim(x, n, 1, 0, p, st));
    FCG_TRY(sorted_exclusive(w, p.r[0].order, n, false, p.lat, p.scratch, out, st));
  } else if (dom_ok) {
    return self_dom2d(x, wptr(w, 1, n), n, 1, 0, nullptr, nullptr, include_self, 0.0, div, p, q,
                      out, st);
  } else if (nd) {  // strict dominance in rank space: p_m(s) < p_m(t) for every m
    FCG_TRY(rank_all(x, n, d, p, st, false));
    int rev[FCG_MAX_DIM] = {0}, qoff[FCG_MAX_DIM] = {0};
    const int32_t *thr[FCG_MAX_DIM];
    for (int k = 0; k < d; ++k) thr[k] = p.r[k].pos;
    FCG_TRY(dom_nd(p, nq, n, d, 1, NdW{{w, nullptr}, 1}, rev, qoff, thr, out, 0, 1, st));
  } else {
    Brute B;
    B.n = n;
    B.d = d;
    B.x = x;
    B.w = w;
    B.nw = 1;
    B.out = out;
    for (int k = 0; k < d; ++k) B.sign[k] = -1;
    FCG_PROF("pts_brute", st);
    brute_kernel<BR_ECDF><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(B);
    FCG_LAUNCH_CHECK();
  }
  FCG_PROF("pts_finish", st);
  finish_ecdf_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, w, include_self, div);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

extern "C" int fcg_kde_points_laplacian(const double *x, int64_t n, int32_t d, const double *w,
                                        int32_t nw, const double *h, const double *centre,
                                        double *out, void *ws, size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (nw < 1 || nw > 2) return fail(FCG_EUNSUPPORTED, "nw must be 1 or 2 weight vectors per call");
  if (d == 2 && !dom_fits(n, 4 * nw)) return dom_too_large(n);  // 4 sign codes' grids
  const bool dom_ok = d == 2;
  Workspace W(ws);
  PtsWs p;
  const bool nd = nd_route(n, d);
  carve(W, p, n, nd ? d : (d < 2 ? d : 2), nw, dom_ok, true, d == 1 ? n * 2 : 0);
  SelfWs q{};
  if (dom_ok) carve_self(W, q, n, nw);
  NdWs nq{};
  if (nd) carve_nd(W, nq, n, d, nw, 1 << d, true);
  double *psi1 = nullptr, *F1 = nullptr;
  if (d == 1) {
    psi1 = W.take<double>((size_t)n * nw);
    F1 = W.take<double>((size_t)n * nw);
  }
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  cudaStream_t st = as_stream(stream);
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  const double scale = 1.0 / (std::ldexp(1.0, d) * (double)n * prod_h);

  if (nd) {  // far field per sign code on a coarse rank grid + direct near-field pairs
    FCG_TRY(rank_all(x, n, d, p, st, false));
    FCG_TRY(kde_nd(p, nq, x, n, d, w, nw, h, centre, out, st));
    FCG_PROF("pts_finish", st);
    kde_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, nw, w, scale, out);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }
  if (d >= 3 || !(d == 1 || dom_ok)) {
    Brute B;
    B.n = n;
    B.d = d;
    B.x = x;
    B.w = w;
    B.nw = nw;
    B.out = out;
    for (int k = 0; k < d; ++k) B.inv_h[k] = 1.0 / h[k];
    {
      FCG_PROF("pts_brute", st);
      brute_kernel<BR_KDE><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(B);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_finish", st);
    kde_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, nw, w, scale, out);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }

  if (d == 2)  // group-ordered self dominance over the 4 orientations (dnc.py:459-468)
    return self_dom2d(x, wptr(w, nw, n), n, nw, 1, h, centre, 1, scale, 0.0, p, q, out, st);
  const int ncodes = 1 << d;
  FCG_TRY(rank_dim(x, n, 1, 0, p, st));
  for (int code = 0; code < ncodes; ++code) {
    KdeP kp{};  // smask = 0: plain (unsigned) channels
    kp.d = d;
    for (int k = 0; k < d; ++k) {
      const double sgn = ((code >> k) & 1) ? -1.0 : 1.0;  // DeltaVector.from_code
      kp.c[k] = centre[k];
      kp.a[k] = sgn / h[k];
    }
    {
      FCG_PROF("pts_psi", st);
      kde_psi_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, kp, w, nw, p.expo, psi1);
      FCG_LAUNCH_CHECK();
    }
    {  // d == 1: code 0 = strictly below (prefix), code 1 = strictly above (suffix)
      for (int v = 0; v < nw; ++v)
        FCG_TRY(sorted_exclusive(psi1 + (size_t)v * n, p.r[0].order, n, code == 1, p.lat,
                                 p.scratch, F1 + (size_t)v * n, st));
    }
    FCG_PROF("pts_kde_accum", st);
    kde_accum_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, nw, p.expo, F1, out, code == 0);
    FCG_LAUNCH_CHECK();
  }
  FCG_PROF("pts_finish", st);
  kde_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, nw, w, scale, out);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

namespace fcg {
namespace {
// matern32-additive at the points as signed Laplacian channels.  With s the term's signs,
//   sum_code z_code [(1 + expo_code) F_0 - sum_l (s_l / h_l) F_l]
//     = A + sum_k (xc_k / h_k) B_k - sum_l C_l,
// A = sum_code z F(w e), B_k = sum_code z F(s_k w e), C_l = sum_code z F(s_l w xc_l e / h_l):
// 2d + 1 channels of the Laplacian dominance engine whose psi only changes sign with the code.
__global__ void matern_channels_kernel(const double *__restrict__ x, int64_t n, int d,
                                       const double *__restrict__ w, const double *c,
                                       const double *hinv, double *__restrict__ wv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wi = w ? w[i] : 1.0;
    wv[i] = wi;
    for (int k = 0; k < d; ++k) {
      wv[(int64_t)(1 + k) * n + i] = wi;
      wv[(int64_t)(1 + d + k) * n + i] = wi * (x[i * d + k] - c[k]) * hinv[k];
    }
  }
}

struct MatFin {
  int d;
  double c[FCG_MAX_DIM], hinv[FCG_MAX_DIM];
  double scale;
};

// out = (A + sum_k (xc_k / h_k) B_k - sum_l C_l + w) * scale   (self term, dnc.py:682-686)
__global__ void matern_finish_kernel(const double *__restrict__ acc, const double *__restrict__ x,
                                     int64_t n, const double *__restrict__ w, MatFin f,
                                     double *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    double r = acc[t];
    for (int k = 0; k < f.d; ++k)
      r += (x[t * f.d + k] - f.c[k]) * f.hinv[k] * acc[(int64_t)(1 + k) * n + t];
    for (int l = 0; l < f.d; ++l) r -= acc[(int64_t)(1 + f.d + l) * n + t];
    r = r + (w ? w[t] : 1.0);
    out[t] = r * f.scale;
  }
}
}  // namespace
}  // namespace fcg

extern "C" int fcg_kde_points_matern32(const double *x, int64_t n, int32_t d, const double *w,
                                       const double *h, const double *centre, double *out,
                                       void *ws, size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d == 2 && !dom_fits(n, 8)) return dom_too_large(n);  // 4 codes x 2 channels
  const bool dom_ok = d == 2;
  const int nchan = 2 * d + 1;
  Workspace W(ws);
  PtsWs p;
  const bool nd = nd_route(n, d) && d <= 4;  // table-form near field: d = 3, 4
  carve(W, p, n, nd ? d : (d < 2 ? d : 2), 2, dom_ok, true, d == 1 ? n * 2 : 0);
  SelfWs q{};
  if (dom_ok) carve_self(W, q, n, 2);
  NdWs nq{};
  if (nd) carve_nd(W, nq, n, d, 2, 1 << d, true, true);
  double *wv = W.take<double>((size_t)n * nchan);
  double *acc = W.take<double>((size_t)n * nchan);
  double *psi1 = nullptr, *F1 = nullptr;
  if (d == 1) {
    psi1 = W.take<double>((size_t)n);
    F1 = W.take<double>((size_t)n);
  }
  double *dpar = W.take<double>(2 * FCG_MAX_DIM);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  cudaStream_t st = as_stream(stream);
  double prod_h = 1.0;
  for (int k = 0; k < d; ++k) prod_h *= h[k];
  double scale = 1.0 / (std::ldexp(1.0, d) * (double)n * prod_h);
  scale /= 1.0 + d;  // dnc.py:683-685

  if (nd) {  // far field per sign code (two channels) + table-form near field
    FCG_TRY(rank_all(x, n, d, p, st, false));
    FCG_TRY(kde_nd(p, nq, x, n, d, w, 1, h, centre, out, st, true));
    FCG_PROF("pts_finish", st);
    kde_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, 1, w, scale, out);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }
  if (d >= 3 || !(d == 1 || dom_ok)) {  // direct pairs with the matern32-additive kernel
    Brute B;
    B.n = n;
    B.d = d;
    B.x = x;
    B.w = w;
    B.nw = 1;
    B.out = out;
    for (int k = 0; k < d; ++k) B.inv_h[k] = 1.0 / h[k];
    {
      FCG_PROF("pts_brute", st);
      brute_kernel<BR_MATERN><<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(B);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_finish", st);
    kde_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, 1, w, scale, out);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }
  MatFin f{};
  f.d = d;
  f.scale = scale;
  double hp[2 * FCG_MAX_DIM];
  for (int k = 0; k < d; ++k) {
    f.c[k] = centre[k];
    f.hinv[k] = 1.0 / h[k];
    hp[k] = centre[k];
    hp[FCG_MAX_DIM + k] = 1.0 / h[k];
  }
  FCG_CUDA_TRY(cudaMemcpyAsync(dpar, hp, sizeof(hp), cudaMemcpyHostToDevice, st));
  {
    FCG_PROF("pts_psi", st);
    matern_channels_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, d, w, dpar, dpar + FCG_MAX_DIM, wv);
    FCG_LAUNCH_CHECK();
  }
  if (d == 2) {
    // channels: 0 A, 1-2 B_k (sign s_k), 3-4 C_l (sign s_l); two per pass
    const unsigned m01[2] = {0u, 1u}, m23[2] = {2u, 1u}, m4[1] = {2u};
    FCG_TRY(self_dom2d(x, wptr(wv, 2, n), n, 2, 1, h, centre, 0, 0.0, 0.0, p, q, acc, st, m01));
    FCG_TRY(self_dom2d(x, wptr(wv + 2 * n, 2, n), n, 2, 1, h, centre, 0, 0.0, 0.0, p, q,
                       acc + 2 * n, st, m23));
    FCG_TRY(self_dom2d(x, wptr(wv + 4 * n, 1, n), n, 1, 1, h, centre, 0, 0.0, 0.0, p, q,
                       acc + 4 * n, st, m4));
  } else {  // d == 1: code 0 = strictly below (prefix), code 1 = strictly above (suffix)
    FCG_TRY(rank_dim(x, n, 1, 0, p, st));
    const unsigned masks[3] = {0u, 1u, 1u};
    for (int ch = 0; ch < 3; ++ch) {
      for (int code = 0; code < 2; ++code) {
        KdeP kp{};
        kp.d = 1;
        kp.code = code;
        kp.smask[0] = masks[ch];
        kp.c[0] = centre[0];
        kp.a[0] = (code ? -1.0 : 1.0) / h[0];
        {
          FCG_PROF("pts_psi", st);
          kde_psi_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, kp, wv + (size_t)ch * n, 1, p.expo,
                                                           psi1);
          FCG_LAUNCH_CHECK();
        }
        FCG_TRY(sorted_exclusive(psi1, p.r[0].order, n, code == 1, p.lat, p.scratch, F1, st));
        FCG_PROF("pts_kde_accum", st);
        kde_accum_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, 1, p.expo, F1, acc + (size_t)ch * n,
                                                          code == 0);
        FCG_LAUNCH_CHECK();
      }
    }
  }
  FCG_PROF("pts_finish", st);
  matern_finish_kernel<<<grid_for(n, 256), 256, 0, st>>>(acc, x, n, w, f, out);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

extern "C" int fcg_kde_points_laplacian_shard(const double *x, int64_t n, int32_t d,
                                              const double *w, int32_t nw, const double *h,
                                              const double *centre, int32_t shard,
                                              int32_t nshards, double *out, void *ws,
                                              size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d != 2) return fail(FCG_EUNSUPPORTED, "query sharding is implemented for d = 2");
  if (nshards < 1 || shard < 0 || shard >= nshards) return fail(FCG_EINVAL, "shard out of range");
  if (nw < 1 || nw > 2) return fail(FCG_EUNSUPPORTED, "nw must be 1 or 2 weight vectors per call");
  if (!dom_fits(n, 4 * nw)) return dom_too_large(n);
  Workspace W(ws);
  PtsWs p;
  carve(W, p, n, 2, nw, true, true, 0);
  SelfWs q{};
  carve_self(W, q, n, nw);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  const double scale = 1.0 / (4.0 * (double)n * h[0] * h[1]);
  return self_dom2d(x, wptr(w, nw, n), n, nw, 1, h, centre, 1, scale, 0.0, p, q, out, as_stream(stream),
                    nullptr, shard, nshards);
}

extern "C" int fcg_dnc_ecdf_shard(const double *x, int64_t n, int32_t d, const double *w,
                                  int32_t include_self, int32_t scaled, int32_t shard,
                                  int32_t nshards, double *out, void *ws, size_t *ws_bytes,
                                  void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d != 2) return fail(FCG_EUNSUPPORTED, "query sharding is implemented for d = 2");
  if (nshards < 1 || shard < 0 || shard >= nshards) return fail(FCG_EINVAL, "shard out of range");
  if (!dom_fits(n, 1)) return dom_too_large(n);
  Workspace W(ws);
  PtsWs p;
  carve(W, p, n, 2, 1, true, false, 0);
  SelfWs q{};
  carve_self(W, q, n, 1);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  return self_dom2d(x, wptr(w, 1, n), n, 1, 0, nullptr, nullptr, include_self, 0.0, scaled ? (double)n : 0.0,
                    p, q, out, as_stream(stream), nullptr, shard, nshards);
}

extern "C" int fcg_kde_points_laplacian_w2(const double *x, int64_t n, int32_t d, const double *w0,
                                           const double *w1, int32_t nw, const double *h,
                                           const double *centre, double *out, void *ws,
                                           size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d != 2) return fail(FCG_EUNSUPPORTED, "per-channel weight pointers: d = 2 only");
  if (nw < 1 || nw > 2) return fail(FCG_EUNSUPPORTED, "nw must be 1 or 2 weight vectors per call");
  if (!dom_fits(n, 4 * nw)) return dom_too_large(n);
  Workspace W(ws);
  PtsWs p;
  carve(W, p, n, 2, nw, true, true, 0);
  SelfWs q{};
  carve_self(W, q, n, nw);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  for (int k = 0; k < d; ++k)
    if (!(h[k] > 0.0)) return fail(FCG_EINVAL, "bandwidth must be > 0");
  const double scale = 1.0 / (4.0 * (double)n * h[0] * h[1]);
  return self_dom2d(x, WPtr{{w0, nw > 1 ? w1 : nullptr}}, n, nw, 1, h, centre, 1, scale, 0.0, p,
                    q, out, as_stream(stream));
}

// ---- all-delta dominance tables (kde_terms_dnc, dnc.py:608-632), tiled direct pairs -------
// table[j][b] = sum of psi[i][b] over the points i strictly dominating j under the sign code b
// (bit k of b: delta_k = -1, i.e. x_ik > x_jk; otherwise x_ik < x_jk), i != j.  With distinct
// coordinates every pair (i, j) lands in exactly one code: b(i, j) = sum_k [x_ik > x_jk] << k.
namespace fcg {
namespace {
constexpr int kTermQ = 128;  // queries per CTA (one per thread)
constexpr int kTermS = 64;   // sources per shared-memory tile

__global__ void __launch_bounds__(kTermQ) terms_kernel(const double *__restrict__ x, int64_t n,
                                                       int d, const double *__restrict__ psi,
                                                       double *__restrict__ table) {
  extern __shared__ double t_smem[];
  const int nc = 1 << d, stride = nc + 1;           // per-thread accumulator row (bank skew)
  double *s_acc = t_smem;                           // [kTermQ][stride]
  double *s_x = s_acc + kTermQ * stride;            // [kTermS][d]
  double *s_psi = s_x + kTermS * FCG_MAX_DIM;       // [kTermS][nc]
  const int64_t t = (int64_t)blockIdx.x * kTermQ + threadIdx.x;
  double xt[FCG_MAX_DIM];
  for (int k = 0; k < d; ++k) xt[k] = t < n ? x[t * d + k] : 0.0;
  double *acc = s_acc + threadIdx.x * stride;
  for (int b = 0; b < nc; ++b) acc[b] = 0.0;
  for (int64_t s0 = 0; s0 < n; s0 += kTermS) {
    const int ns = (int)(n - s0 < kTermS ? n - s0 : kTermS);
    __syncthreads();
    for (int i = threadIdx.x; i < ns * d; i += blockDim.x) s_x[i] = x[s0 * d + i];
    for (int i = threadIdx.x; i < ns * nc; i += blockDim.x) s_psi[i] = psi[s0 * nc + i];
    __syncthreads();
    if (t < n) {
      for (int j = 0; j < ns; ++j) {
        if (s0 + j == t) continue;
        int b = 0;
        for (int k = 0; k < d; ++k) b |= (s_x[j * d + k] > xt[k] ? 1 : 0) << k;
        acc[b] += s_psi[j * nc + b];
      }
    }
  }
  if (t < n)
    for (int b = 0; b < nc; ++b) table[t * nc + b] = acc[b];
}
}  // namespace
}  // namespace fcg

extern "C" int fcg_dominance_terms(const double *x, int64_t n, int32_t d, const double *psi,
                                   double *table, void *ws, size_t *ws_bytes, void *stream) {
  FCG_TRY(check_pts(n, d));
  if (d > 6) return fail(FCG_EUNSUPPORTED, "dominance tables support d <= 6 (2^d columns)");
  const bool nd = nd_route(n, d);
  Workspace W(ws);
  PtsWs p;
  NdWs nq{};
  if (nd) {
    carve(W, p, n, d, 1, false, false, 0);
    carve_nd(W, nq, n, d, 1, 1, false);
  }
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  const int nc = 1 << d;
  if (nd) {  // one rank-space dominance sum per sign code (bit k: x_ik > x_jk)
    cudaStream_t st = as_stream(stream);
    FCG_TRY(rank_all(x, n, d, p, st, false));
    for (int b = 0; b < nc; ++b) {
      int rev[FCG_MAX_DIM], qoff[FCG_MAX_DIM];
      const int32_t *thr[FCG_MAX_DIM];
      for (int k = 0; k < d; ++k) {
        rev[k] = qoff[k] = (b >> k) & 1;  // p_k(i) >= p_k(j) + 1
        thr[k] = p.r[k].pos;
      }
      FCG_TRY(dom_nd(p, nq, n, d, 1, NdW{{psi + b, nullptr}, nc}, rev, qoff, thr, table + b, 0,
                     nc, st));
    }
    return FCG_OK;
  }
  const size_t smem = ((size_t)kTermQ * (nc + 1) + (size_t)kTermS * FCG_MAX_DIM +
                       (size_t)kTermS * nc) * sizeof(double);
  cudaStream_t st = as_stream(stream);
  FCG_CUDA_TRY(cudaFuncSetAttribute(terms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  FCG_PROF("pts_terms", st);
  terms_kernel<<<(unsigned)ceil_div(n, kTermQ), kTermQ, smem, st>>>(x, n, d, psi, table);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}
