// Rank-space dominance sums at the sample points for 3 <= d <= 6.  Included by
// points.cu inside namespace fcg { namespace { ... } } after the ranking helpers.
//
// The reference answers these with the MergeND recursion (dnc.py:65-135, 307-410); the sums are
//   F(t) = sum_s w_s prod_m [p_m(s) < Q_m(t)]        (rev_m: [p_m(s) >= Q_m(t)])
// over rank positions p_m (a permutation of [0, n) per dimension) and per-query thresholds Q_m
// (own position: strict dominance; lower / upper tie ranks: < / <= with ties; survival: >).
// Decomposition, one level, in the frame flipped along every reversed dimension (pf = NP-1-p,
// Tf = NP - Q, so every test reads pf < Tf):
//   far field:  chunks of 2^ls consecutive positions per dimension give a G^d coarse grid; its
//               directional prefix sums (the grid engine of scan.cu) hold, for every query, the
//               sources whose chunk is strictly below the threshold's chunk in EVERY dimension;
//   near field: a dominated source outside the far field shares the threshold's chunk in some
//               dimension; phase k takes the sources of chunk(Tf_k) along dimension k whose
//               chunks are strictly below along the dimensions m < k, and compares positions
//               directly for m >= k (each dominated source is met in exactly one phase).
//               Thresholds are nondecreasing along the dimension's rank order, so the queries of
//               chunk(Tf_k) are a contiguous run of that order; a CTA takes 256 of them and stages
//               the chunk's sources below its largest threshold (already gathered in dimension-k
//               order) through shared memory with TMA bulk copies.
// Cost: d n 2^ls pair tests + (2d + 1) G^d lattice cell visits instead of n^2 pairs.
//
// The Laplacian KDE (kde_dnc, dnc.py:635-690) uses the same split over its 2^d sign codes: the
// far field of every code is a coarse-grid dominance sum of psi_code = w prod_m E_m^{+-1}
// (E_m = exp((x_m - c_m) / h_m)); pairs that share a chunk in some dimension are summed directly,
// the kernel value formed as prod_m min(E_sm / E_tm, E_tm / E_sm) (no sign codes, no
// cancellation); phase k takes the pairs whose first shared chunk is along dimension k.  For
// d = 3, 4 every point carries the table of its 2^d signed products instead, so a pair costs one
// table read per side and one multiply.

constexpr int kNdThreads = 128;
constexpr int kNdQPT = 2;                        // queries per thread (ECDF)
constexpr int kNdQ = kNdThreads * kNdQPT;        // queries per CTA
constexpr int kNdTile = 256;                     // sources per shared-memory stage (ECDF)
constexpr int kNdTileK = 128;                    // sources per stage (KDE)
constexpr int kNdMinLs = 8;                      // a chunk is at least one tile
constexpr int64_t kNdMinN = 8192;                // below this the direct tiles are used
constexpr int64_t kNdMaxCoarseBytes = int64_t(2) << 30;

struct NdW {  // up to two weight vectors, element i of vector v at p[v][i * stride]
  const double *p[2];
  int64_t stride;
  __host__ __device__ double at(int v, int64_t i) const { return p[v] ? p[v][i * stride] : 1.0; }
};

struct NdPlan {
  int ls;
  int64_t G, NP, cells;
};

// chunk size by a cost model: pair tests against coarse-lattice passes
inline NdPlan nd_plan(int64_t n, int d, int nch, int ncodes, bool kde) {
  NdPlan best{};
  double best_cost = -1.0;
  for (int ls = kNdMinLs; ls <= 31; ++ls) {  // ends at G == 1 (one cell, always admissible)
    const int64_t G = ceil_div(n, int64_t(1) << ls);
    double cells = 1.0;
    for (int k = 0; k < d; ++k) cells *= (double)G;
    if (cells * 8.0 * nch > (double)kNdMaxCoarseBytes) continue;
    const double near = (double)d * (double)n * (double)(int64_t(1) << ls) / (kde ? (d <= 4 ? 1.25e12 : 6.5e11) : 5e12);
    const double far = (double)ncodes * nch * (cells * 8.0 * (2 * d + 2) / 4e12 + (d + 3) * 4e-6);
    const double cost = near + far;
    if (best_cost < 0.0 || cost < best_cost) {
      best_cost = cost;
      best.ls = ls;
      best.G = G;
      best.NP = G << ls;
      best.cells = (int64_t)cells;
    }
    if (G == 1) break;
  }
  return best;
}

// FCG_ND=off sends every d >= 3 request to the direct tiles (cross-checks in the tests)
inline bool nd_route(int64_t n, int d) {
  const char *e = getenv("FCG_ND");
  if (e && std::string(e) == "off") return false;
  return d >= 3 && d <= 6 && n >= kNdMinN;
}

struct DomN {
  int64_t n, G, NP, cells;
  int d, ls, nch, k;  // k: the near-field phase's dimension
  int rev[FCG_MAX_DIM], qoff[FCG_MAX_DIM];
  const int32_t *pos[FCG_MAX_DIM], *order[FCG_MAX_DIM], *thr[FCG_MAX_DIM];
  int64_t stride[FCG_MAX_DIM];
  NdW w;
  double *H;    // [nch][cells]
  double *out;  // channel v of query t at out[v * out_vs + t * out_ts]
  int64_t out_vs, out_ts;
  int32_t *rec;  // [NP][DP] flipped positions of the sources in dimension-k order
  double *wrec;  // [nch][NP]
  int32_t *qkey, *qstart, *tstart;
};

__device__ __forceinline__ int32_t nd_thr(const DomN &D, int m, int64_t t) {
  const int64_t Q = (int64_t)D.thr[m][t] + D.qoff[m];
  return (int32_t)(D.rev[m] ? D.NP - Q : Q);
}

__global__ void nd_scatter_kernel(DomN D) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < D.n;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    for (int m = 0; m < D.d; ++m) flat += (int64_t)(D.pos[m][s] >> D.ls) * D.stride[m];
    for (int v = 0; v < D.nch; ++v) atomicAdd(D.H + (size_t)v * D.cells + flat, D.w.at(v, s));
  }
}

// far field: the scanned coarse cell just below (above, reversed) the threshold's chunk
__global__ void nd_far_query_kernel(DomN D) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < D.n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    bool live = true;
    for (int m = 0; m < D.d; ++m) {
      const int64_t cq = nd_thr(D, m, t) >> D.ls;
      live = live && cq >= 1;
      flat += (D.rev[m] ? D.G - cq : cq - 1) * D.stride[m];
    }
    for (int v = 0; v < D.nch; ++v)
      D.out[v * D.out_vs + t * D.out_ts] = live ? D.H[(size_t)v * D.cells + flat] : 0.0;
  }
}

__global__ void nd_qkey_kernel(DomN D) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < D.n;
       t += (int64_t)gridDim.x * blockDim.x)
    D.qkey[t] = nd_thr(D, D.k, t) >> D.ls;
}

// tiles of kNdQ queries per bucket (bucket G: thresholds past every source chunk, no tiles)
__global__ void nd_tiles_kernel(DomN D) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < D.G + 2;
       j += (int64_t)gridDim.x * blockDim.x)
    D.tstart[j] = j < D.G ? (D.qstart[j + 1] - D.qstart[j] + kNdQ - 1) / kNdQ : 0;
}

template <int DP>
__global__ void nd_gather_kernel(DomN D) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D.NP;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t r[DP];
#pragma unroll
    for (int m = 0; m < DP; ++m) r[m] = 0x7fffffff;  // padding never passes a test
    const bool live = i < D.n;
    const int32_t s = live ? D.order[D.k][i] : 0;
    if (live) {
#pragma unroll
      for (int m = 0; m < DP; ++m)
        if (m < D.d) {
          const int32_t pp = D.pos[m][s];
          r[m] = D.rev[m] ? (int32_t)(D.NP - 1 - pp) : pp;
        }
    }
    int4 *dst = reinterpret_cast<int4 *>(D.rec + i * DP);
    dst[0] = make_int4(r[0], r[1], r[2], r[3]);
    if (DP == 8) dst[1] = make_int4(r[4 % DP], r[5 % DP], r[6 % DP], r[7 % DP]);
    if (D.wrec)
      for (int v = 0; v < D.nch; ++v) D.wrec[(size_t)v * D.NP + i] = live ? D.w.at(v, s) : 0.0;
  }
}

template <int DD, int NCH, bool UNIT>
__global__ void __launch_bounds__(kNdThreads) nd_near_kernel(DomN A) {
  constexpr int DP = DD <= 4 ? 4 : 8;
  constexpr uint32_t kRecBytes = kNdTile * DP * 4, kWBytes = kNdTile * 8;
  __shared__ __align__(128) int32_t s_rec[2][kNdTile * DP];
  __shared__ __align__(128) double s_w[2][UNIT ? 2 : NCH * kNdTile];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ int s_j;
  __shared__ int32_t s_tmax[kNdThreads / 32];
  const int tid = threadIdx.x;
  if (tid == 0) {  // the bucket this tile belongs to: tstart[j] <= tile < tstart[j + 1]
    const int32_t tile = (int32_t)blockIdx.x;
    int lo = 0, hi = (int)A.G + 1;
    if (tile >= A.tstart[hi]) {
      lo = -1;
    } else {
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (A.tstart[mid] <= tile) lo = mid;
        else hi = mid;
      }
    }
    s_j = lo;
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int j = s_j;
  if (j < 0) return;
  const int k = A.k, ls = A.ls;
  const int64_t qbeg = A.qstart[j] + (int64_t)((int32_t)blockIdx.x - A.tstart[j]) * kNdQ;
  const int64_t qend = A.qstart[j + 1];
  // The queries of a bucket run in the dimension's (flipped) rank order, so their thresholds
  // along k are nondecreasing: the tile only needs the chunk's sources below its largest one.
  int32_t T[kNdQPT][DD];
  int64_t tq[kNdQPT];
  int32_t tkmax = 0;
#pragma unroll
  for (int r = 0; r < kNdQPT; ++r) {
    const int64_t qi = qbeg + tid + r * kNdThreads;
    tq[r] = qi < qend ? (int64_t)A.order[k][A.rev[k] ? A.n - 1 - qi : qi] : -1;
#pragma unroll
    for (int m = 0; m < DD; ++m) {
      int32_t tf = 0;  // dead lanes: nothing is below 0
      if (tq[r] >= 0) {
        tf = nd_thr(A, m, tq[r]);
        if (m < k) tf = (tf >> ls) << ls;
        if (m == k) tkmax = max(tkmax, tf);
      }
      T[r][m] = tf;
    }
  }
  tkmax = __reduce_max_sync(0xffffffffu, tkmax);
  if ((tid & 31) == 0) s_tmax[tid >> 5] = tkmax;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kNdThreads / 32; ++w) tkmax = max(tkmax, s_tmax[w]);
  const bool revk = A.rev[k] != 0;
  const int64_t base = (revk ? A.G - 1 - j : (int64_t)j) << ls;
  const int ctiles = (1 << ls) / kNdTile;
  int ntile = (int)((tkmax - ((int64_t)j << ls) + kNdTile - 1) / kNdTile);  // flipped offsets
  ntile = ntile < 0 ? 0 : (ntile > ctiles ? ctiles : ntile);
  const int32_t *rec = A.rec + base * DP;
  auto issue = [&](int i) {
    const int sg = i & 1;
    const int64_t u = revk ? ctiles - 1 - i : i;  // flipped order runs down the stored chunk
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[sg], kRecBytes + (UNIT ? 0u : (uint32_t)NCH * kWBytes));
    bulk_load_1d(s_rec[sg], rec + u * kNdTile * DP, kRecBytes, &s_bar[sg]);
    if (!UNIT)
      for (int v = 0; v < NCH; ++v)
        bulk_load_1d(&s_w[sg][v * kNdTile], A.wrec + (size_t)v * A.NP + base + u * kNdTile,
                     kWBytes, &s_bar[sg]);
  };
  if (tid == 0 && ntile > 0) issue(0);
  int32_t cnt[kNdQPT] = {0};
  double acc[kNdQPT][NCH] = {{0.0}};
  for (int i = 0; i < ntile; ++i) {
    const int sg = i & 1;
    if (tid == 0 && i + 1 < ntile) issue(i + 1);
    mbar_wait(&s_bar[sg], (uint32_t)(i >> 1) & 1u);
    const int4 *r4 = reinterpret_cast<const int4 *>(s_rec[sg]);
#pragma unroll 4
    for (int jj = 0; jj < kNdTile; ++jj) {
      int32_t pv[DP];
      {
        const int4 a = r4[jj * (DP / 4)];
        pv[0] = a.x, pv[1] = a.y, pv[2] = a.z, pv[3] = a.w;
      }
      if (DP == 8) {
        const int4 b = r4[jj * (DP / 4) + DP / 4 - 1];
        pv[4 % DP] = b.x, pv[5 % DP] = b.y, pv[6 % DP] = b.z, pv[7 % DP] = b.w;
      }
#pragma unroll
      for (int r = 0; r < kNdQPT; ++r) {
        bool ok = true;
#pragma unroll
        for (int m = 0; m < DD; ++m) ok = ok && pv[m] < T[r][m];
        if (UNIT) {
          cnt[r] += ok ? 1 : 0;
        } else {
#pragma unroll
          for (int v = 0; v < NCH; ++v) acc[r][v] += ok ? s_w[sg][v * kNdTile + jj] : 0.0;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < kNdQPT; ++r) {
    if (tq[r] < 0) continue;
#pragma unroll
    for (int v = 0; v < NCH; ++v) {
      double *o = A.out + v * A.out_vs + tq[r] * A.out_ts;
      *o += UNIT ? (double)cnt[r] : acc[r][v];
    }
  }
}

struct NdWs {
  int32_t *rec, *qkey, *qstart, *tstart, *crec;
  double *wrec, *H, *EE, *IE, *erec, *trec, *wq, *UU, *utab;
};

inline int nd_rd(int d, int nw) { return (2 * d + nw + 1) & ~1; }  // doubles per KDE record

void carve_nd(Workspace &W, NdWs &q, int64_t n, int d, int nch, int ncodes, bool kde,
              bool matern = false) {
  const NdPlan pl = nd_plan(n, d, nch, ncodes, kde);
  const int DP = d <= 4 ? 4 : 8;
  q.H = W.take<double>((size_t)pl.cells * nch);
  if (!kde) {
    q.rec = W.take<int32_t>((size_t)pl.NP * DP);
    q.wrec = W.take<double>((size_t)pl.NP * nch);
    q.qkey = W.take<int32_t>(n);
    q.qstart = W.take<int32_t>(pl.G + 3);
    q.tstart = W.take<int32_t>(pl.G + 3);
  } else {
    q.EE = W.take<double>((size_t)n * d);
    q.IE = W.take<double>((size_t)n * d);
    if (matern) {
      q.UU = W.take<double>((size_t)n * d);
      q.utab = W.take<double>((size_t)pl.NP << d);
    }
    if (d <= 4) {  // table form of the near field
      q.trec = W.take<double>((size_t)pl.NP << d);
      q.wq = W.take<double>((size_t)pl.NP * 2);
    } else {
      q.erec = W.take<double>((size_t)pl.NP * nd_rd(d, nch));
    }
    q.crec = W.take<int32_t>((size_t)pl.NP * DP);
  }
}

template <int DD>
int nd_near_launch(const DomN &D, bool unit, unsigned grid, cudaStream_t st) {
  if (unit) nd_near_kernel<DD, 1, true><<<grid, kNdThreads, 0, st>>>(D);
  else if (D.nch == 1) nd_near_kernel<DD, 1, false><<<grid, kNdThreads, 0, st>>>(D);
  else nd_near_kernel<DD, 2, false><<<grid, kNdThreads, 0, st>>>(D);
  return FCG_OK;
}

// out[v][t] = sum_s w_v(s) prod_m [rev_m ? p_m(s) >= thr_m(t) + qoff_m : p_m(s) < thr_m(t) + qoff_m]
// The ranking (p.r[m].pos / order for every m < d) must be in place, and thr_m nondecreasing
// along dimension m's rank order (positions, lower / upper tie ranks).
int dom_nd(PtsWs &p, NdWs &q, int64_t n, int d, int nch, NdW w, const int *rev, const int *qoff,
           const int32_t *const *thr, double *out, int64_t out_vs, int64_t out_ts,
           cudaStream_t st) {
  const NdPlan pl = nd_plan(n, d, nch, 1, false);
  const bool unit = nch == 1 && w.p[0] == nullptr;
  DomN D{};
  D.n = n;
  D.G = pl.G;
  D.NP = pl.NP;
  D.cells = pl.cells;
  D.d = d;
  D.ls = pl.ls;
  D.nch = nch;
  int64_t stride = 1;
  for (int m = d - 1; m >= 0; --m) {
    D.rev[m] = rev[m];
    D.qoff[m] = qoff[m];
    D.pos[m] = p.r[m].pos;
    D.order[m] = p.r[m].order;
    D.thr[m] = thr[m];
    D.stride[m] = stride;
    stride *= pl.G;
  }
  D.w = w;
  D.H = q.H;
  D.out = out;
  D.out_vs = out_vs;
  D.out_ts = out_ts;
  D.rec = q.rec;
  D.wrec = unit ? nullptr : q.wrec;
  D.qkey = q.qkey;
  D.qstart = q.qstart;
  D.tstart = q.tstart;
  // far field
  FCG_CUDA_TRY(cudaMemsetAsync(q.H, 0, (size_t)pl.cells * nch * 8, st));
  {
    FCG_PROF("pts_nd_scatter", st);
    nd_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(D);
    FCG_LAUNCH_CHECK();
  }
  LatShape gs;
  gs.d = d;
  bool brev[FCG_MAX_DIM];
  for (int m = 0; m < d; ++m) {
    gs.dims[m] = pl.G;
    brev[m] = rev[m] != 0;
  }
  Epi inplace;
  for (int v = 0; v < nch; ++v)
    FCG_TRY(scan_lattice<double>(q.H + (size_t)v * pl.cells, gs, brev, inplace, p.scratch, st));
  {
    FCG_PROF("pts_nd_far", st);
    nd_far_query_kernel<<<grid_for(n, 256), 256, 0, st>>>(D);
    FCG_LAUNCH_CHECK();
  }
  // near field, one phase per dimension
  const unsigned tiles = (unsigned)(ceil_div(n, kNdQ) + pl.G + 1);
  for (int k = 0; k < d; ++k) {
    D.k = k;
    {
      FCG_PROF("pts_nd_keys", st);
      nd_qkey_kernel<<<grid_for(n, 256), 256, 0, st>>>(D);
      FCG_LAUNCH_CHECK();
    }
    // bucket starts only: a bucket's queries are a contiguous run of the dimension's rank order
    FCG_CUDA_TRY(cudaMemsetAsync(q.qstart, 0, (size_t)(pl.G + 2) * 4, st));
    {
      FCG_PROF("pts_bucket", st);
      bucket_count<<<grid_for(n, 256), 256, 0, st>>>(q.qkey, n, q.qstart);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(scan_i32(q.qstart, q.qstart, pl.G + 2, false, p.rw.partial, st));
    {
      FCG_PROF("pts_nd_keys", st);
      nd_tiles_kernel<<<grid_for(pl.G + 2, 256), 256, 0, st>>>(D);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(scan_i32(q.tstart, q.tstart, pl.G + 2, false, p.rw.partial, st));
    {
      FCG_PROF("pts_nd_gather", st);
      if (d <= 4) nd_gather_kernel<4><<<grid_for(pl.NP, 256), 256, 0, st>>>(D);
      else nd_gather_kernel<8><<<grid_for(pl.NP, 256), 256, 0, st>>>(D);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_nd_near", st);
    switch (d) {
      case 3: nd_near_launch<3>(D, unit, tiles, st); break;
      case 4: nd_near_launch<4>(D, unit, tiles, st); break;
      case 5: nd_near_launch<5>(D, unit, tiles, st); break;
      default: nd_near_launch<6>(D, unit, tiles, st); break;
    }
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}

// ---- Laplacian KDE -----------------------------------------------------------------------
struct KdeN {
  int64_t n, G, NP, cells;
  int d, ls, nw, k, code, first;
  int matern;  // matern32-additive (dnc.py:659-685): kernel (1 + e) exp(-e), e = sum_m |du_m|
  const int32_t *pos[FCG_MAX_DIM], *order[FCG_MAX_DIM];
  int64_t stride[FCG_MAX_DIM];
  double c[FCG_MAX_DIM], h[FCG_MAX_DIM];
  const double *x;
  const double *w;  // [nw][n] or NULL
  double *EE, *IE;  // [d][n]: exp(+u), exp(-u), u = (x - c) / h
  double *UU;       // [d][n]: u (matern)
  double *utab;     // [NP][2^d]: U[c] = sum_m (bit m of c ? +u_m : -u_m) (matern, d <= 4)
  double *H, *out;  // [nw][cells], [nw][n]
  double *erec;     // [NP][RD]: E_0.., I_0.., w_0..                      (d >= 5)
  double *trec;     // [NP][2^d]: prod_m (bit m of the code ? I_m : E_m)  (d <= 4)
  double *wq;       // [NP][2]: the weights                               (d <= 4)
  int32_t *crec;    // [NP][DP]: position along every dimension (padding: -1)
};

__global__ void nd_kde_exp_kernel(KdeN K) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < K.n;
       s += (int64_t)gridDim.x * blockDim.x)
    for (int m = 0; m < K.d; ++m) {
      const double u = (K.x[s * K.d + m] - K.c[m]) / K.h[m];
      K.EE[(size_t)m * K.n + s] = exp(u);
      K.IE[(size_t)m * K.n + s] = exp(-u);
      if (K.matern) K.UU[(size_t)m * K.n + s] = u;
    }
}

// code bit m set: sources above the query along m (x_s > x_t): source factor exp(-u_s), query
// factor exp(+u_t); clear: source exp(+u_s), query exp(-u_t)   (dnc.py:661-669)
__global__ void nd_kde_scatter_kernel(KdeN K) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < K.n;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    double f = 1.0, U = 0.0;
    for (int m = 0; m < K.d; ++m) {
      const bool up = (K.code >> m) & 1;
      flat += (int64_t)(K.pos[m][s] >> K.ls) * K.stride[m];
      f *= up ? K.IE[(size_t)m * K.n + s] : K.EE[(size_t)m * K.n + s];
      if (K.matern) U += up ? K.UU[(size_t)m * K.n + s] : -K.UU[(size_t)m * K.n + s];
    }
    if (K.matern) {  // channels sum w psi and sum w U psi (one weight vector)
      const double wf = (K.w ? K.w[s] : 1.0) * f;
      atomicAdd(K.H + flat, wf);
      atomicAdd(K.H + K.cells + flat, wf * U);
      continue;
    }
    for (int v = 0; v < K.nw; ++v)
      atomicAdd(K.H + (size_t)v * K.cells + flat, (K.w ? K.w[(size_t)v * K.n + s] : 1.0) * f);
  }
}

__global__ void nd_kde_query_kernel(KdeN K) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < K.n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t flat = 0;
    bool live = true;
    double z = 1.0, U = 0.0;
    for (int m = 0; m < K.d; ++m) {
      const int64_t c = K.pos[m][t] >> K.ls;
      const bool up = (K.code >> m) & 1;
      const int64_t idx = up ? c + 1 : c - 1;
      live = live && idx >= 0 && idx < K.G;
      flat += idx * K.stride[m];
      z *= up ? K.EE[(size_t)m * K.n + t] : K.IE[(size_t)m * K.n + t];
      if (K.matern) U += up ? K.UU[(size_t)m * K.n + t] : -K.UU[(size_t)m * K.n + t];
    }
    if (K.matern) {  // sum_s w (1 + U_s - U_t) psi_s z_t
      const double r = live ? z * ((1.0 - U) * K.H[flat] + K.H[K.cells + flat]) : 0.0;
      double *o = K.out + t;
      *o = K.first ? r : *o + r;
      continue;
    }
    for (int v = 0; v < K.nw; ++v) {
      const double r = live ? z * K.H[(size_t)v * K.cells + flat] : 0.0;
      double *o = K.out + (size_t)v * K.n + t;
      *o = K.first ? r : *o + r;
    }
  }
}

template <int DP>
__global__ void nd_kde_gather_kernel(KdeN K, int RD) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K.NP;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool live = i < K.n;
    const int32_t s = live ? K.order[K.k][i] : 0;
    double *e = K.erec + i * RD;
    int32_t c[DP];
#pragma unroll
    for (int m = 0; m < DP; ++m) c[m] = -1;
    for (int m = 0; m < K.d; ++m) {
      e[m] = live ? K.EE[(size_t)m * K.n + s] : 0.0;
      e[K.d + m] = live ? K.IE[(size_t)m * K.n + s] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < DP; ++m)
      if (m < K.d && live) c[m] = K.pos[m][s] >> K.ls;
    for (int v = 0; v < RD - 2 * K.d; ++v)
      e[2 * K.d + v] = (live && v < K.nw) ? (K.w ? K.w[(size_t)v * K.n + s] : 1.0) : 0.0;
    int4 *dst = reinterpret_cast<int4 *>(K.crec + i * DP);
    dst[0] = make_int4(c[0], c[1], c[2], c[3]);
    if (DP == 8) dst[1] = make_int4(c[4 % DP], c[5 % DP], c[6 % DP], c[7 % DP]);
  }
}

// one query per thread; sources of the query's dimension-k chunk staged by TMA bulk copies
template <int DD, int NW>
__global__ void __launch_bounds__(kNdThreads) nd_kde_near_kernel(KdeN K) {
  constexpr int DP = DD <= 4 ? 4 : 8;
  constexpr int RD = (2 * DD + NW + 1) & ~1;
  constexpr uint32_t kEBytes = kNdTileK * RD * 8, kCBytes = kNdTileK * DP * 4;
  __shared__ __align__(128) double s_e[2][kNdTileK * RD];
  __shared__ __align__(128) int32_t s_c[2][kNdTileK * DP];
  __shared__ __align__(8) uint64_t s_bar[2];
  const int tid = threadIdx.x;
  const int k = K.k, ls = K.ls;
  const int64_t qi = (int64_t)blockIdx.x * kNdThreads + tid;  // dimension-k sorted index
  const int64_t base = (qi >> ls) << ls;                       // uniform over the CTA
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  double Et[DD], It[DD];
  int32_t ct[DD];
  {
    const double *e = K.erec + qi * RD;
    const int32_t *c = K.crec + qi * DP;
#pragma unroll
    for (int m = 0; m < DD; ++m) {
      Et[m] = e[m];
      It[m] = e[DD + m];
      ct[m] = m < k ? c[m] : -2;  // -2: no source chunk equals it, the test passes
    }
  }
  const int32_t self = k == 0 ? (int32_t)(qi - base) : -1;
  const int ntile = (1 << ls) / kNdTileK;
  auto issue = [&](int i) {
    const int sg = i & 1;
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[sg], kEBytes + kCBytes);
    bulk_load_1d(s_e[sg], K.erec + (base + (int64_t)i * kNdTileK) * RD, kEBytes, &s_bar[sg]);
    bulk_load_1d(s_c[sg], K.crec + (base + (int64_t)i * kNdTileK) * DP, kCBytes, &s_bar[sg]);
  };
  if (tid == 0) issue(0);
  double acc[NW] = {0.0};
  for (int i = 0; i < ntile; ++i) {
    const int sg = i & 1;
    if (tid == 0 && i + 1 < ntile) issue(i + 1);
    mbar_wait(&s_bar[sg], (uint32_t)(i >> 1) & 1u);
    const double2 *e2 = reinterpret_cast<const double2 *>(s_e[sg]);
    const int4 *c4 = reinterpret_cast<const int4 *>(s_c[sg]);
    const int32_t self_j = self - i * kNdTileK;
#pragma unroll 2
    for (int jj = 0; jj < kNdTileK; ++jj) {
      double ev[RD];
#pragma unroll
      for (int a = 0; a < RD / 2; ++a) {
        const double2 v = e2[jj * (RD / 2) + a];
        ev[2 * a] = v.x;
        ev[2 * a + 1] = v.y;
      }
      int32_t cs[DP];
      {
        const int4 a = c4[jj * (DP / 4)];
        cs[0] = a.x, cs[1] = a.y, cs[2] = a.z, cs[3] = a.w;
      }
      if (DP == 8) {
        const int4 b = c4[jj * (DP / 4) + DP / 4 - 1];
        cs[4 % DP] = b.x, cs[5 % DP] = b.y, cs[6 % DP] = b.z, cs[7 % DP] = b.w;
      }
      bool ok = jj != self_j;
      double kv = 1.0;
#pragma unroll
      for (int m = 0; m < DD; ++m) {
        ok = ok && cs[m] != ct[m];
        kv *= fmin(ev[m] * It[m], ev[DD + m] * Et[m]);
      }
#pragma unroll
      for (int v = 0; v < NW; ++v) acc[v] += ok ? ev[2 * DD + v] * kv : 0.0;
    }
    __syncthreads();
  }
  if (qi < K.n) {
    const int32_t t = K.order[k][qi];
#pragma unroll
    for (int v = 0; v < NW; ++v) K.out[(size_t)v * K.n + t] += acc[v];
  }
}

template <int DD>
void nd_kde_near_launch(const KdeN &K, unsigned grid, cudaStream_t st) {
  if (K.nw == 1) nd_kde_near_kernel<DD, 1><<<grid, kNdThreads, 0, st>>>(K);
  else nd_kde_near_kernel<DD, 2><<<grid, kNdThreads, 0, st>>>(K);
}

// ---- near field in table form (d = 3, 4) ----------------------------------------------------
// Every point carries the 2^d products P[c] = prod_m (bit m of c ? exp(-u_m) : exp(+u_m)).  For a
// pair the code c has bit m set where the source lies above the query, and the kernel value is
// P_s[c] * P_t[~c]: one table read per side and one multiply instead of per-dimension factors.
template <int DD>
__global__ void nd_kde_tab_gather_kernel(KdeN K) {
  constexpr int NC = 1 << DD;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K.NP;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool live = i < K.n;
    const int32_t s = live ? K.order[K.k][i] : 0;
    double E[DD], I[DD];
    int32_t c[4] = {-1, -1, -1, -1};
#pragma unroll
    for (int m = 0; m < DD; ++m) {
      E[m] = live ? K.EE[(size_t)m * K.n + s] : 0.0;
      I[m] = live ? K.IE[(size_t)m * K.n + s] : 0.0;
      if (live) c[m] = K.pos[m][s];
    }
    double *tb = K.trec + i * NC;
#pragma unroll
    for (int code = 0; code < NC; ++code) {
      double pr = (code & 1) ? I[0] : E[0];
#pragma unroll
      for (int m = 1; m < DD; ++m) pr *= ((code >> m) & 1) ? I[m] : E[m];
      tb[code] = pr;
    }
    if (K.matern) {
      double u[DD];
#pragma unroll
      for (int m = 0; m < DD; ++m) u[m] = live ? K.UU[(size_t)m * K.n + s] : 0.0;
#pragma unroll
      for (int code = 0; code < NC; ++code) {
        double U = 0.0;
#pragma unroll
        for (int m = 0; m < DD; ++m) U += ((code >> m) & 1) ? u[m] : -u[m];
        K.utab[i * NC + code] = U;
      }
    }
    K.wq[2 * i] = live ? (K.w ? K.w[s] : 1.0) : 0.0;
    K.wq[2 * i + 1] = (live && K.nw > 1) ? (K.w ? K.w[(size_t)K.n + s] : 1.0) : 0.0;
    *reinterpret_cast<int4 *>(K.crec + i * 4) = make_int4(c[0], c[1], c[2], c[3]);
  }
}

constexpr int kNdTabQPT = 2;
inline size_t nd_kde_tab_smem(int d, bool matern) {
  const size_t NC = size_t(1) << d, NQ = kNdThreads * kNdTabQPT;
  return (2 * kNdTileK * NC + 2 * kNdTileK * 2 + NC * NQ) * 8 * (matern ? 2 : 1) +
         2 * kNdTileK * 16 + 32;
}

// KK: the phase's dimension (pairs sharing a chunk along an earlier dimension are left to that
// phase; phase 0 skips the query itself)
template <int DD, int NW, int KK, bool MAT>
__global__ void __launch_bounds__(kNdThreads) nd_kde_tab_kernel(KdeN K) {
  constexpr int NC = 1 << DD, QPT = kNdTabQPT, NQ = kNdThreads * QPT, TS = kNdTileK;
  constexpr uint32_t kTBytes = TS * NC * 8, kWBytes = TS * 16, kCBytes = TS * 16;
  extern __shared__ __align__(128) unsigned char nd_smem[];
  double *s_tab = reinterpret_cast<double *>(nd_smem);            // [2][TS][NC]
  double *s_w = s_tab + 2 * TS * NC;                              // [2][TS][2]
  double *s_q = s_w + 2 * TS * 2;                                 // [NC][NQ], complemented codes
  double *s_ut = s_q + NC * NQ;                                   // [2][TS][NC]     (matern)
  double *s_qu = s_ut + (MAT ? 2 * TS * NC : 0);                  // [NC][NQ]        (matern)
  int32_t *s_c = reinterpret_cast<int32_t *>(
      s_qu + (MAT ? NC * NQ + 2 * TS * 2 : 0));                   // [2][TS][4]
  uint64_t *s_bar = reinterpret_cast<uint64_t *>(s_c + 2 * TS * 4);
  const int tid = threadIdx.x;
  const int ls = K.ls;
  const int64_t q0 = (int64_t)blockIdx.x * NQ;  // dimension-k sorted index
  const int64_t base = (q0 >> ls) << ls;        // uniform over the CTA
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  int32_t pt[QPT][DD], self[QPT];
#pragma unroll
  for (int r = 0; r < QPT; ++r) {
    const int64_t qi = q0 + tid + r * kNdThreads;
    const int4 c = *reinterpret_cast<const int4 *>(K.crec + qi * 4);
    const int32_t cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int m = 0; m < DD; ++m) pt[r][m] = cc[m];
#pragma unroll
    for (int code = 0; code < NC; ++code) {
      s_q[(code ^ (NC - 1)) * NQ + r * kNdThreads + tid] = K.trec[qi * NC + code];
      if (MAT) s_qu[code * NQ + r * kNdThreads + tid] = K.utab[qi * NC + code];
    }
    self[r] = (int32_t)(qi - base);
  }
  const int ntile = (1 << ls) / TS;
  auto issue = [&](int i) {
    const int sg = i & 1;
    const int64_t off = base + (int64_t)i * TS;
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar[sg], (MAT ? 2 : 1) * kTBytes + kWBytes + kCBytes);
    if (MAT) bulk_load_1d(s_ut + sg * TS * NC, K.utab + off * NC, kTBytes, &s_bar[sg]);
    bulk_load_1d(s_tab + sg * TS * NC, K.trec + off * NC, kTBytes, &s_bar[sg]);
    bulk_load_1d(s_w + sg * TS * 2, K.wq + off * 2, kWBytes, &s_bar[sg]);
    bulk_load_1d(s_c + sg * TS * 4, K.crec + off * 4, kCBytes, &s_bar[sg]);
  };
  if (tid == 0) issue(0);
  double acc[QPT][NW] = {{0.0}};
  for (int i = 0; i < ntile; ++i) {
    const int sg = i & 1;
    if (tid == 0 && i + 1 < ntile) issue(i + 1);
    mbar_wait(&s_bar[sg], (uint32_t)(i >> 1) & 1u);
    const double *tb = s_tab + sg * TS * NC;
    const double *ub = s_ut + sg * TS * NC;
    const double2 *w2 = reinterpret_cast<const double2 *>(s_w + sg * TS * 2);
    const int4 *c4 = reinterpret_cast<const int4 *>(s_c + sg * TS * 4);
#pragma unroll 2
    for (int jj = 0; jj < TS; ++jj) {
      const int4 c = c4[jj];
      const int32_t ps[4] = {c.x, c.y, c.z, c.w};
      const double2 wv = w2[jj];
      const int32_t sj = i * TS + jj;
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        unsigned code = 0;  // bit m: the source lies above the query along m
#pragma unroll
        for (int m = DD - 1; m >= 0; --m)
          code = __funnelshift_l((unsigned)(pt[r][m] - ps[m]), code, 1);
        double kv = tb[jj * NC + code] * s_q[code * NQ + r * kNdThreads + tid];
        if (MAT) kv *= 1.0 + (ub[jj * NC + code] - s_qu[code * NQ + r * kNdThreads + tid]);
        bool ok = KK > 0 || sj != self[r];
#pragma unroll
        for (int m = 0; m < KK; ++m) ok = ok && ((unsigned)(ps[m] ^ pt[r][m]) >> ls) != 0u;
        kv = ok ? kv : 0.0;
        acc[r][0] = fma(wv.x, kv, acc[r][0]);
        if (NW > 1) acc[r][NW - 1] = fma(wv.y, kv, acc[r][NW - 1]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < QPT; ++r) {
    const int64_t qi = q0 + tid + r * kNdThreads;
    if (qi >= K.n) continue;
    const int32_t t = K.order[KK][qi];
#pragma unroll
    for (int v = 0; v < NW; ++v) K.out[(size_t)v * K.n + t] += acc[r][v];
  }
}

template <int DD, int NW, int KK, bool MAT>
int nd_kde_tab_launch1(const KdeN &K, cudaStream_t st) {
  const size_t sm = nd_kde_tab_smem(DD, MAT);
  FCG_CUDA_TRY(cudaFuncSetAttribute(nd_kde_tab_kernel<DD, NW, KK, MAT>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  nd_kde_tab_kernel<DD, NW, KK, MAT>
      <<<(unsigned)(K.NP / (kNdThreads * kNdTabQPT)), kNdThreads, sm, st>>>(K);
  return FCG_OK;
}
template <int DD, int NW, bool MAT>
int nd_kde_tab_launch(const KdeN &K, cudaStream_t st) {
  constexpr int KL = DD - 1;
  switch (K.k) {
    case 0: return nd_kde_tab_launch1<DD, NW, 0, MAT>(K, st);
    case 1: return nd_kde_tab_launch1<DD, NW, 1, MAT>(K, st);
    case 2: return nd_kde_tab_launch1<DD, NW, 2, MAT>(K, st);
    default: return nd_kde_tab_launch1<DD, NW, KL, MAT>(K, st);
  }
}

// out[v][t] = sum_{s != t} w_v(s) exp(-sum_m |x_sm - x_tm| / h_m)   (before the self term and
// the normalisation, which kde_finish_kernel adds); the ranking must be in place
// matern (d <= 4, nw == 1): the matern32-additive kernel (1 + e) exp(-e) instead; its far field
// needs the two channels sum w psi and sum w U psi per code (workspace carved with nch = 2)
int kde_nd(PtsWs &p, NdWs &q, const double *x, int64_t n, int d, const double *w, int nw,
           const double *h, const double *centre, double *out, cudaStream_t st,
           bool matern = false) {
  const int ncodes = 1 << d;
  const int nchan = matern ? 2 : nw;
  const NdPlan pl = nd_plan(n, d, nchan, ncodes, true);
  KdeN K{};
  K.n = n;
  K.G = pl.G;
  K.NP = pl.NP;
  K.cells = pl.cells;
  K.d = d;
  K.ls = pl.ls;
  K.nw = nw;
  int64_t stride = 1;
  for (int m = d - 1; m >= 0; --m) {
    K.pos[m] = p.r[m].pos;
    K.order[m] = p.r[m].order;
    K.stride[m] = stride;
    stride *= pl.G;
    K.c[m] = centre[m];
    K.h[m] = h[m];
  }
  K.x = x;
  K.w = w;
  K.matern = matern ? 1 : 0;
  K.EE = q.EE;
  K.IE = q.IE;
  K.UU = q.UU;
  K.utab = q.utab;
  K.H = q.H;
  K.out = out;
  K.erec = q.erec;
  K.trec = q.trec;
  K.wq = q.wq;
  K.crec = q.crec;
  {
    FCG_PROF("pts_psi", st);
    nd_kde_exp_kernel<<<grid_for(n, 256), 256, 0, st>>>(K);
    FCG_LAUNCH_CHECK();
  }
  LatShape gs;
  gs.d = d;
  for (int m = 0; m < d; ++m) gs.dims[m] = pl.G;
  Epi inplace;
  for (int code = 0; code < ncodes; ++code) {
    K.code = code;
    K.first = code == 0;
    bool brev[FCG_MAX_DIM];
    for (int m = 0; m < d; ++m) brev[m] = (code >> m) & 1;
    FCG_CUDA_TRY(cudaMemsetAsync(q.H, 0, (size_t)pl.cells * nchan * 8, st));
    {
      FCG_PROF("pts_nd_scatter", st);
      nd_kde_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(K);
      FCG_LAUNCH_CHECK();
    }
    for (int v = 0; v < nchan; ++v)
      FCG_TRY(scan_lattice<double>(q.H + (size_t)v * pl.cells, gs, brev, inplace, p.scratch, st));
    FCG_PROF("pts_nd_far", st);
    nd_kde_query_kernel<<<grid_for(n, 256), 256, 0, st>>>(K);
    FCG_LAUNCH_CHECK();
  }
  const int RD = nd_rd(d, nw);
  const unsigned grid = (unsigned)(pl.NP / kNdThreads);
  for (int k = 0; k < d; ++k) {
    K.k = k;
    if (d <= 4) {
      {
        FCG_PROF("pts_nd_gather", st);
        if (d == 3) nd_kde_tab_gather_kernel<3><<<grid_for(pl.NP, 256), 256, 0, st>>>(K);
        else nd_kde_tab_gather_kernel<4><<<grid_for(pl.NP, 256), 256, 0, st>>>(K);
        FCG_LAUNCH_CHECK();
      }
      FCG_PROF("pts_nd_kde_near", st);
      if (matern) {
        FCG_TRY(d == 3 ? (nd_kde_tab_launch<3, 1, true>(K, st)) : (nd_kde_tab_launch<4, 1, true>(K, st)));
      } else if (d == 3) {
        FCG_TRY(nw == 1 ? (nd_kde_tab_launch<3, 1, false>(K, st)) : (nd_kde_tab_launch<3, 2, false>(K, st)));
      } else {
        FCG_TRY(nw == 1 ? (nd_kde_tab_launch<4, 1, false>(K, st)) : (nd_kde_tab_launch<4, 2, false>(K, st)));
      }
      FCG_LAUNCH_CHECK();
      continue;
    }
    {
      FCG_PROF("pts_nd_gather", st);
      nd_kde_gather_kernel<8><<<grid_for(pl.NP, 256), 256, 0, st>>>(K, RD);
      FCG_LAUNCH_CHECK();
    }
    FCG_PROF("pts_nd_kde_near", st);
    if (d == 5) nd_kde_near_launch<5>(K, grid, st);
    else nd_kde_near_launch<6>(K, grid, st);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}
