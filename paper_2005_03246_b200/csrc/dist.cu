// Multi-GPU slab decomposition support: the lattice is split along axis 1 into
// contiguous slabs, one per rank.  These kernels route points to the rank owning their axis-1
// cell and finish a slab with the carry plane the ranks exchange over NCCL.
#include "bin.cuh"
#include "common.cuh"
#include "partition.cuh"
#include "sort.cuh"

namespace fcg {
namespace {

// owner[i] = rank whose [bounds[r], bounds[r+1]) holds the point's axis cell, or -1 (dead)
struct OwnerP {
  int d, axis, m, le, shift, G;
  int64_t bounds[65];
};

__global__ void axis_owner_kernel(const double *__restrict__ x, int64_t n,
                                  const double *__restrict__ kn, OwnerP p,
                                  int32_t *__restrict__ owner) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double z0 = kn[0];
    const double idz = p.m > 1 ? (double)(p.m - 1) / (kn[p.m - 1] - kn[0]) : 0.0;
    const int c = knot_count(x[i * p.d + p.axis], kn, p.m, p.le, z0, idz) - p.shift;
    int r = -1;
    for (int q = 0; q < p.G; ++q)
      if (c >= p.bounds[q] && c < p.bounds[q + 1]) r = q;
    owner[i] = r;
  }
}

__global__ void owner_keys_kernel(const int32_t *__restrict__ owner, int64_t n,
                                  uint32_t *__restrict__ keys, int32_t *__restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = owner[i];
    keys[i] = o < 0 ? 0xFFu : (uint32_t)o;
    vals[i] = (int32_t)i;
  }
}

__global__ void gather_rows_kernel(const double *__restrict__ x, const double *__restrict__ w,
                                   int64_t n, int d, const int32_t *__restrict__ order,
                                   double *__restrict__ xo, double *__restrict__ wo) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = order[q];
    for (int k = 0; k < d; ++k) xo[q * d + k] = x[i * d + k];
    if (w) wo[q] = w[i];
  }
}

__global__ void owner_counts_kernel(const uint32_t *__restrict__ keys, int64_t n, int G,
                                    int64_t *__restrict__ start) {
  const int r = threadIdx.x;
  if (r > G) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)keys[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  start[r] = lo;
}

// routing records: the point's row and its weight (split again on the way out)
template <int D>
struct RouteBuild {
  static constexpr int kD = D;
  __device__ __forceinline__ void operator()(const double *xi, double wi, double *out) const {
#pragma unroll
    for (int k = 0; k < D; ++k) out[k] = xi[k];
    out[D] = wi;
  }
};

// start[r] = first position of owner r in the partitioned order (digit-major scanned counts)
__global__ void route_starts_kernel(const int32_t *__restrict__ hist, int64_t tiles, int G,
                                    int64_t *__restrict__ start) {
  const int r = threadIdx.x;
  if (r <= G) start[r] = hist[(int64_t)r * tiles];
}

template <int D>
int route_partition(const uint32_t *keys, int64_t n, const double *x, const double *w,
                    double *x_out, double *w_out, int32_t *hist, int32_t *partial, cudaStream_t st) {
  RouteBuild<D> rb;
  return digit_partition_build<RouteBuild<D>, D + 1>(keys, n, 0, x, w, rb, x_out, nullptr, nullptr,
                                                     hist, partial, st, w_out, "dist_partition",
                                                     false, true);
}

// out[a][j][b] = (local[a][j][b] + carry[a][b]) / div   (div <= 0: no division)
template <typename T>
__global__ void slab_finish_kernel(const T *__restrict__ local, const T *__restrict__ carry,
                                   int64_t A, int64_t J, int64_t B, double div,
                                   double *__restrict__ out) {
  const int64_t total = A * J * B;
  const double rdiv = div > 0.0 ? 1.0 / div : 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t % B;
    const int64_t a = t / (J * B);
    T v = local[t];
    if (carry) v += carry[a * B + b];
    double r = (double)v;
    if (div > 0.0) r = div_rn(r, div, rdiv);
    out[t] = r;
  }
}

}  // namespace
}  // namespace fcg

using namespace fcg;

extern "C" int fcg_axis_owner(const double *x, int64_t n, int32_t d, int32_t axis,
                              const double *knots_axis, int64_t m, int32_t le, int32_t shift,
                              const int64_t *bounds, int32_t G, int32_t *owner, void *stream) {
  if (d < 1 || d > FCG_MAX_DIM || axis < 0 || axis >= d) return fail(FCG_EINVAL, "bad axis");
  if (G < 1 || G > 64) return fail(FCG_EUNSUPPORTED, "1..64 slabs supported");
  if (n == 0) return FCG_OK;
  OwnerP p{};
  p.d = d;
  p.axis = axis;
  p.m = (int)m;
  p.le = le;
  p.shift = shift;
  p.G = G;
  for (int q = 0; q <= G; ++q) p.bounds[q] = bounds[q];
  cudaStream_t st = as_stream(stream);
  FCG_PROF("dist_axis_owner", st);
  axis_owner_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, knots_axis, p, owner);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

extern "C" int fcg_partition_rows(const double *x, int64_t n, int32_t d, const double *w,
                                  const int32_t *owner, int32_t G, double *x_out, double *w_out,
                                  int64_t *counts, void *ws, size_t *ws_bytes, void *stream) {
  if (G < 1 || G > 64) return fail(FCG_EUNSUPPORTED, "1..64 owners supported");
  if (d < 1 || d > FCG_MAX_DIM) return fail(FCG_EINVAL, "dimension out of range");
  Workspace W(ws);
  uint32_t *keys = W.take<uint32_t>(n);
  int32_t *vals = W.take<int32_t>(n);
  const size_t hist_elems = digit_hist_elems(n);
  int32_t *hist = W.take<int32_t>(hist_elems);
  int32_t *partial = W.take<int32_t>(scan_ws_partial_elems((int64_t)hist_elems + 2));
  int64_t *start = W.take<int64_t>(G + 1);
  double *w_scratch = W.take<double>(w_out ? 0 : n);  // unit weights: the routed w is dropped
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  if (n > 0) {
    {
      FCG_PROF("dist_partition", st);
      owner_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(owner, n, keys, vals);
      FCG_LAUNCH_CHECK();
    }
    // one payload-carrying pass: rows and weights read once (coalesced), written by owner
    if ((d % 2 == 0) && (reinterpret_cast<uintptr_t>(x) & 15) != 0)
      return fail(FCG_EINVAL, "points must be 16-byte aligned");
    double *wo = w_out ? w_out : w_scratch;
    int rc;
    switch (d) {
      case 1: rc = route_partition<1>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 2: rc = route_partition<2>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 3: rc = route_partition<3>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 4: rc = route_partition<4>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 5: rc = route_partition<5>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 6: rc = route_partition<6>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      case 7: rc = route_partition<7>(keys, n, x, w, x_out, wo, hist, partial, st); break;
      default: rc = route_partition<8>(keys, n, x, w, x_out, wo, hist, partial, st); break;
    }
    FCG_TRY(rc);
    route_starts_kernel<<<1, 128, 0, st>>>(hist, ceil_div(n, kPartTile), G, start);
    FCG_LAUNCH_CHECK();
  } else {
    FCG_CUDA_TRY(cudaMemsetAsync(start, 0, (G + 1) * sizeof(int64_t), st));
  }
  int64_t h[66];
  FCG_TRY(read_small(h, start, (G + 1) * sizeof(int64_t), st));
  for (int r = 0; r < G; ++r) counts[r] = h[r + 1] - h[r];
  return FCG_OK;
}

extern "C" int fcg_slab_finish(const void *local, int32_t kind, const void *carry, int64_t A,
                               int64_t J, int64_t B, double div, double *out, void *stream) {
  const int64_t total = A * J * B;
  if (total == 0) return FCG_OK;
  cudaStream_t st = as_stream(stream);
  FCG_PROF("dist_slab_finish", st);
  if (kind == 0)  // int64 counts
    slab_finish_kernel<int64_t><<<grid_for(total, 256), 256, 0, st>>>(
        static_cast<const int64_t *>(local), static_cast<const int64_t *>(carry), A, J, B, div, out);
  else
    slab_finish_kernel<double><<<grid_for(total, 256), 256, 0, st>>>(
        static_cast<const double *>(local), static_cast<const double *>(carry), A, J, B, div, out);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}
