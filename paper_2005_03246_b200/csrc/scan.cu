// Directional prefix-sum engine; see scan.cuh.
#include "scan.cuh"

namespace fcg {

namespace {

constexpr int kUnroll = 16;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Product over the axes other than e.ax of zf_k[i_k] for the multi-index of flat line origin
// (a over axes < ax, b over axes > ax).
__device__ __forceinline__ double zprod_other(const Epi &e, int64_t a, int64_t b) {
  double z = 1.0;
  // decompose b over axes d-1 .. ax+1 (last axis fastest)
  for (int k = e.d - 1; k > e.ax; --k) {
    int64_t i = b % e.dims[k];
    b /= e.dims[k];
    z *= e.zf[e.zoff[k] + i];
  }
  for (int k = e.ax - 1; k >= 0; --k) {
    int64_t i = a % e.dims[k];
    a /= e.dims[k];
    z *= e.zf[e.zoff[k] + i];
  }
  return z;
}

template <typename T, int EK>
__device__ __forceinline__ void emit(T *lat, const Epi &e, int64_t f, int64_t j, double zo, T v) {
  if constexpr (EK == EPI_INPLACE) {
    lat[f] = v;
  } else if constexpr (EK == EPI_F64) {
    double r = (double)v;
    if (e.div > 0.0) r = r / e.div;  // (div_rn measured slower in the 16-deep line walk)
    static_cast<double *>(e.out)[f] = r;
  } else if constexpr (EK == EPI_I64) {
    static_cast<int64_t *>(e.out)[f] = (int64_t)v;
  } else {
    double *o = static_cast<double *>(e.out);
    double r = (zo * e.zf[e.zoff[e.ax] + j]) * (double)v;
    if (e.accumulate) r = o[f] + r;
    if (e.apply_scale) r = r * e.scale;
    o[f] = r;
  }
}

// ---- lines: thread per (a, chunk c, b) ----------------------------------------------------
template <typename T, bool REV, int EK>
__global__ void __launch_bounds__(256) lines_kernel(T *__restrict__ lat, int64_t A, int64_t D,
                                                    int64_t B, int64_t Dc, int64_t C,
                                                    const T *__restrict__ carry_in, Epi e) {
  const int64_t total = A * C * B;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t % B;
    const int64_t r = t / B;
    const int64_t c = r % C;
    const int64_t a = r / C;
    T carry = carry_in ? carry_in[(a * C + c) * B + b] : T(0);
    const int64_t j0 = c * Dc;
    const int64_t j1 = (j0 + Dc < D) ? j0 + Dc : D;
    T *base = lat + a * D * B + b;
    double zo = 1.0;
    if constexpr (EK == EPI_KDE) zo = zprod_other(e, a, b);
    // slab carry capture: this line lies in the requested axis-1 plane (axis-0 pass, d >= 2)
    double *pcap = nullptr;
    int64_t pB1 = 0;
    double pw = 1.0;
    if constexpr (EK == EPI_KDE) {
      if (e.plane_out && e.ax == 0 && e.d >= 2) {
        pB1 = B / e.dims[1];
        if (b / pB1 == e.plane_idx) {
          pcap = e.plane_out + (b % pB1);
          int64_t r = b;  // capture weight: zf of the axes >= cap_kw (b spans axes 1..d-1)
          for (int k = e.d - 1; k >= 1; --k) {
            const int64_t i = r % e.dims[k];
            r /= e.dims[k];
            if (k >= e.cap_kw) pw *= e.zf[e.zoff[k] + i];
          }
        }
      }
    }
    int64_t jj = j0;
    for (; jj + kUnroll <= j1; jj += kUnroll) {
      T v[kUnroll];
      double ov[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t j = REV ? (D - 1 - (jj + u)) : (jj + u);
        v[u] = base[j * B];
        // the KDE accumulator is read-modify-written: issue its loads with the lattice loads
        // (the compiler cannot hoist them past the stores on its own)
        if constexpr (EK == EPI_KDE)
          ov[u] = e.accumulate ? static_cast<const double *>(e.out)[a * D * B + j * B + b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t j = REV ? (D - 1 - (jj + u)) : (jj + u);
        carry += v[u];
        if constexpr (EK == EPI_KDE) {
          double r = (zo * e.zf[e.zoff[e.ax] + j]) * (double)carry;
          if (e.accumulate) r = ov[u] + r;
          if (e.apply_scale) r = r * e.scale;
          static_cast<double *>(e.out)[a * D * B + j * B + b] = r;
          if (pcap) pcap[j * pB1] = pw * (double)carry;
        } else {
          emit<T, EK>(lat, e, a * D * B + j * B + b, j, zo, carry);
        }
      }
    }
    for (; jj < j1; ++jj) {
      const int64_t j = REV ? (D - 1 - jj) : jj;
      carry += base[j * B];
      emit<T, EK>(lat, e, a * D * B + j * B + b, j, zo, carry);
      if constexpr (EK == EPI_KDE)
        if (pcap) pcap[j * pB1] = pw * (double)carry;
    }
  }
}

// chunk totals for lines: sums[(a*C + c)*B + b]
template <typename T, bool REV>
__global__ void __launch_bounds__(256) lines_chunk_sums(const T *__restrict__ lat, int64_t A,
                                                        int64_t D, int64_t B, int64_t Dc,
                                                        int64_t C, T *__restrict__ sums) {
  const int64_t total = A * C * B;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t % B;
    const int64_t r = t / B;
    const int64_t c = r % C;
    const int64_t a = r / C;
    const int64_t j0 = c * Dc;
    const int64_t j1 = (j0 + Dc < D) ? j0 + Dc : D;
    const T *base = lat + a * D * B + b;
    T s = T(0);
    int64_t jj = j0;
    for (; jj + kUnroll <= j1; jj += kUnroll) {
      T v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t j = REV ? (D - 1 - (jj + u)) : (jj + u);
        v[u] = base[j * B];
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) s += v[u];
    }
    for (; jj < j1; ++jj) s += base[(REV ? (D - 1 - jj) : jj) * B];
    sums[t] = s;
  }
}

// exclusive scan over c of sums[a][c][b] (in place), thread per (a, b)
template <typename T>
__global__ void chunk_excl_scan(T *__restrict__ sums, int64_t A, int64_t C, int64_t B) {
  const int64_t total = A * B;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t % B;
    const int64_t a = t / B;
    T run = T(0);
    for (int64_t c = 0; c < C; ++c) {
      T *p = sums + (a * C + c) * B + b;
      T v = *p;
      *p = run;
      run += v;
    }
  }
}

// ---- rows (B == 1): warp per (row a, chunk c) ---------------------------------------------
template <typename T, bool REV, int EK>
__global__ void __launch_bounds__(256) rows_kernel(T *__restrict__ lat, int64_t A, int64_t D,
                                                   int64_t Dc, int64_t C,
                                                   const T *__restrict__ carry_in, Epi e) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < A * C;
       w += warps) {
    const int64_t a = w / C;
    const int64_t c = w % C;
    T carry = carry_in ? carry_in[w] : T(0);
    const int64_t j0 = c * Dc;
    const int64_t j1 = (j0 + Dc < D) ? j0 + Dc : D;
    T *row = lat + a * D;
    double zo = 1.0;
    if constexpr (EK == EPI_KDE) zo = zprod_other(e, a, 0);
    constexpr int U = 4;
    for (int64_t jb = j0; jb < j1; jb += 32 * U) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t jj = jb + u * 32 + lane;
        v[u] = (jj < j1) ? row[REV ? (D - 1 - jj) : jj] : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        T s = warp_incl_scan(v[u], lane) + carry;
        carry = __shfl_sync(0xffffffffu, s, 31);
        const int64_t jj = jb + u * 32 + lane;
        if (jj < j1) {
          const int64_t j = REV ? (D - 1 - jj) : jj;
          emit<T, EK>(lat, e, a * D + j, j, zo, s);
        }
      }
    }
  }
}

template <typename T, bool REV>
__global__ void __launch_bounds__(256) rows_chunk_sums(const T *__restrict__ lat, int64_t A,
                                                       int64_t D, int64_t Dc, int64_t C,
                                                       T *__restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < A * C;
       w += warps) {
    const int64_t a = w / C;
    const int64_t c = w % C;
    const int64_t j0 = c * Dc;
    const int64_t j1 = (j0 + Dc < D) ? j0 + Dc : D;
    const T *row = lat + a * D;
    T s = T(0);
    for (int64_t jj = j0 + lane; jj < j1; jj += 32) s += row[REV ? (D - 1 - jj) : jj];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sums[w] = s;
  }
}

struct PassPlan {
  int64_t A, D, B, C, Dc;
};

PassPlan plan_pass(const LatShape &s, int ax) {
  PassPlan p;
  p.A = 1;
  for (int k = 0; k < ax; ++k) p.A *= s.dims[k];
  p.D = s.dims[ax];
  p.B = 1;
  for (int k = ax + 1; k < s.d; ++k) p.B *= s.dims[k];
  const int64_t target = (int64_t)sm_count() * 1536;  // resident threads worth filling
  const int64_t units = (p.B == 1) ? p.A * 32 : p.A * p.B;
  int64_t C = 1;
  if (units < target && p.D >= 128) {
    C = ceil_div(target, units);
    int64_t cmax = p.D / 32;
    if (C > cmax) C = cmax;
    if (C > 512) C = 512;
    if (C < 1) C = 1;
  }
  p.C = C;
  p.Dc = ceil_div(p.D, C);
  p.C = ceil_div(p.D, p.Dc);
  return p;
}

template <typename T, bool REV, int EK>
int launch_pass(T *lat, const PassPlan &p, const Epi &e, T *scratch, cudaStream_t st) {
  const T *carry = nullptr;
  if (p.C > 1) {
    FCG_PROF("scan_chunk_carry", st);
    if (p.B == 1) {
      const int64_t warps = p.A * p.C;
      rows_chunk_sums<T, REV><<<grid_for(warps * 32, 256), 256, 0, st>>>(lat, p.A, p.D, p.Dc,
                                                                       p.C, scratch);
      FCG_LAUNCH_CHECK();
      chunk_excl_scan<T><<<grid_for(p.A, 256), 256, 0, st>>>(scratch, p.A, p.C, 1);
    } else {
      lines_chunk_sums<T, REV><<<grid_for(p.A * p.C * p.B, 256), 256, 0, st>>>(
          lat, p.A, p.D, p.B, p.Dc, p.C, scratch);
      FCG_LAUNCH_CHECK();
      chunk_excl_scan<T><<<grid_for(p.A * p.B, 256), 256, 0, st>>>(scratch, p.A, p.C, p.B);
    }
    FCG_LAUNCH_CHECK();
    carry = scratch;
  }
  const bool fin = EK != EPI_INPLACE;
  if (p.B == 1) {
    FCG_PROF(fin ? "scan_rows_final" : "scan_rows", st);
    rows_kernel<T, REV, EK><<<grid_for(p.A * p.C * 32, 256), 256, 0, st>>>(lat, p.A, p.D, p.Dc,
                                                                          p.C, carry, e);
  } else {
    FCG_PROF(fin ? "scan_lines_final" : "scan_lines", st);
    lines_kernel<T, REV, EK><<<grid_for(p.A * p.C * p.B, 256), 256, 0, st>>>(
        lat, p.A, p.D, p.B, p.Dc, p.C, carry, e);
  }
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

template <typename T, int EK>
int launch_dir(T *lat, const PassPlan &p, bool rev, const Epi &e, T *scratch, cudaStream_t st) {
  return rev ? launch_pass<T, true, EK>(lat, p, e, scratch, st)
             : launch_pass<T, false, EK>(lat, p, e, scratch, st);
}

}  // namespace

int64_t scan_scratch_elems(const LatShape &s) {
  int64_t mx = 0;
  for (int ax = 0; ax < s.d; ++ax) {
    PassPlan p = plan_pass(s, ax);
    if (p.C > 1) {
      int64_t need = p.A * p.C * p.B;
      if (need > mx) mx = need;
    }
  }
  return mx;
}

int64_t scan_scratch_bound() { return (int64_t)sm_count() * 1536 * 3 + 4096; }

template <typename T>
int scan_axis(T *lat, const LatShape &s, int ax, bool rev, const Epi &epi, T *scratch,
              cudaStream_t st) {
  PassPlan p = plan_pass(s, ax);
  Epi e = epi;
  e.ax = ax;
  e.d = s.d;
  for (int k = 0; k < s.d; ++k) e.dims[k] = s.dims[k];
  switch (e.kind) {
    case EPI_INPLACE: return launch_dir<T, EPI_INPLACE>(lat, p, rev, e, scratch, st);
    case EPI_F64: return launch_dir<T, EPI_F64>(lat, p, rev, e, scratch, st);
    case EPI_I64: return launch_dir<T, EPI_I64>(lat, p, rev, e, scratch, st);
    case EPI_KDE: return launch_dir<T, EPI_KDE>(lat, p, rev, e, scratch, st);
  }
  return fail(FCG_EINVAL, "unknown epilogue kind");
}

// ---- fused in-plane pass: axes d-1 (columns) and d-2 (rows) of every plane in one sweep ----
// One CTA per plane of H x W (W = 256 E).  Thread t owns E contiguous columns (the column block
// order is reversed for a suffix along the columns); RB rows at a time are loaded, scanned along
// the columns (thread-local E, then a warp shuffle scan and the warp totals through shared
// memory), added to the per-column running sums along the rows (registers), and stored; the
// next RB rows are in flight meanwhile.  Saves one read + write of the lattice against the two
// separate axis passes.
constexpr int kP2Threads = 256;

template <typename T, int E, int RB, int ST, bool REVR, bool REVC>
__global__ void __launch_bounds__(kP2Threads, 4) plane2d_kernel(T *__restrict__ lat, int64_t H) {
  constexpr int W = kP2Threads * E;
  constexpr int CH = W * (int)sizeof(T) / 16;  // 16-byte chunks per row
  extern __shared__ __align__(16) unsigned char p2_smem[];
  T *s_buf = reinterpret_cast<T *>(p2_smem);  // [ST][RB][W] staged rows (cp.async ring)
  __shared__ T s_w[RB][kP2Threads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int cb = REVC ? kP2Threads - 1 - t : t;  // this thread's column block
  T *pbase = lat + (int64_t)blockIdx.x * H * W;
  const int64_t nb = (H + RB - 1) / RB;
  auto stage = [&](int64_t k) {
    if (k < nb) {
      T *dst = s_buf + (int)(k % ST) * RB * W;
      for (int c = t; c < RB * CH; c += kP2Threads) {
        const int q = c / CH, o = c - q * CH;
        const int64_t rr = k * RB + q;
        if (rr < H) {
          const int64_t r = REVR ? H - 1 - rr : rr;
          const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + q * W + o * (16 / (int)sizeof(T)));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                       "l"(pbase + r * W + o * (16 / (int)sizeof(T)))
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  T carry[E];
#pragma unroll
  for (int e = 0; e < E; ++e) carry[e] = T(0);
#pragma unroll
  for (int k = 0; k < ST - 1; ++k) stage(k);
  for (int64_t k = 0; k < nb; ++k) {
    stage(k + ST - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(ST - 1) : "memory");
    __syncthreads();
    const T *bf = s_buf + (int)(k % ST) * RB * W + cb * E;
    const int64_t r0 = k * RB;
    T v[RB][E], tot[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      T run = T(0);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int ee = REVC ? E - 1 - e : e;
        run += bf[q * W + ee];
        v[q][ee] = run;
      }
      // inclusive scan of the thread totals over the warp
      T x = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      tot[q] = x - run;  // exclusive within the warp
      if (lane == 31) s_w[q][warp] = x;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      T off = tot[q];
      for (int w = 0; w < warp; ++w) off += s_w[q][w];
      const int64_t rr = r0 + q;
      if (rr < H) {
        const int64_t r = REVR ? H - 1 - rr : rr;
        T *row = pbase + r * W + cb * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          carry[e] += v[q][e] + off;
          row[e] = carry[e];
        }
      }
    }
    __syncthreads();  // s_w and the staged slot are rewritten next
  }
}

template <typename T>
static int plane2d_scan(T *lat, const LatShape &s, bool rev_row, bool rev_col, cudaStream_t st) {
  const int d = s.d;
  const int64_t W = s.dims[d - 1], H = s.dims[d - 2];
  int64_t A = 1;
  for (int k = 0; k < d - 2; ++k) A *= s.dims[k];
  const int E = (int)(W / kP2Threads);
  if (W % kP2Threads || (E != 1 && E != 2 && E != 4) || A < 2 * (int64_t)sm_count() || A > 65535 * 32)
    return -1;  // not applicable: the caller runs the two axis passes
  FCG_PROF("scan_plane2d", st);
  constexpr int RB = 8, ST = 3;  // 8 rows per step, 2 steps in flight
  const size_t smem = (size_t)ST * RB * W * sizeof(T);
  int rc = FCG_OK;
  auto go = [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      rc = fail(FCG_ECUDA, "plane2d: shared memory attribute");
    else
      kern<<<(unsigned)A, kP2Threads, smem, st>>>(lat, H);
  };
#define FCG_P2(EE)                                                                         \
  do {                                                                                     \
    if (rev_row) {                                                                         \
      if (rev_col) go(plane2d_kernel<T, EE, RB, ST, true, true>);                              \
      else go(plane2d_kernel<T, EE, RB, ST, true, false>);                                     \
    } else {                                                                               \
      if (rev_col) go(plane2d_kernel<T, EE, RB, ST, false, true>);                             \
      else go(plane2d_kernel<T, EE, RB, ST, false, false>);                                    \
    }                                                                                      \
  } while (0)
  if (E == 1) FCG_P2(1);
  else if (E == 2) FCG_P2(2);
  else FCG_P2(4);
#undef FCG_P2
  FCG_TRY(rc);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

template <typename T>
int scan_lattice(T *lat, const LatShape &s, const bool *rev, const Epi &epi, T *scratch,
                 cudaStream_t st) {
  // last (contiguous) axis first, axis 0 last so that its coalesced line walk carries the
  // epilogue.  With d >= 3 the two in-plane axes go in one fused pass when the shape allows.
  Epi inplace;
  int ax = s.d - 1;
  if (s.d >= 3) {
    const int rc = plane2d_scan<T>(lat, s, rev[s.d - 2], rev[s.d - 1], st);
    if (rc == FCG_OK) ax = s.d - 3;
    else if (rc != -1) return rc;
  }
  for (; ax >= 0; --ax) {
    FCG_TRY(scan_axis<T>(lat, s, ax, rev[ax], ax == 0 ? epi : inplace, scratch, st));
  }
  return FCG_OK;
}

template int scan_lattice<int32_t>(int32_t *, const LatShape &, const bool *, const Epi &,
                                   int32_t *, cudaStream_t);
template int scan_lattice<double>(double *, const LatShape &, const bool *, const Epi &, double *,
                                  cudaStream_t);
template int scan_axis<int32_t>(int32_t *, const LatShape &, int, bool, const Epi &, int32_t *,
                                cudaStream_t);
template int scan_axis<double>(double *, const LatShape &, int, bool, const Epi &, double *,
                               cudaStream_t);

}  // namespace fcg
