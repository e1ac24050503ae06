// Multilinear interpolation of grid-aligned values at query points (the
// grid -> points bridge of interp.py:24-75).  One thread per query: per coordinate the query is
// clamped to the knot hull, its cell is #knots <= q minus one (the exact device knot count of
// bin.cuh, clipped to [0, m-2]) and t = (q - z[cell]) / (z[cell+1] - z[cell]); the 2^d corners
// are summed in the reference's order with explicitly rounded fp64 operations (no FMA
// contraction), so the result is bit-identical to the reference's numpy evaluation.
#include "bin.cuh"
#include "common.cuh"

namespace fcg {
namespace {

struct InterpP {
  int d;
  int64_t m[FCG_MAX_DIM], koff[FCG_MAX_DIM];
};

__global__ void __launch_bounds__(256) interp_kernel(const double *__restrict__ knots, InterpP p,
                                                     const double *__restrict__ vals,
                                                     const double *__restrict__ q, int64_t nq,
                                                     double *__restrict__ out,
                                                     unsigned long long *__restrict__ clamp) {
  unsigned local = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nq;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t cell[FCG_MAX_DIM];
    double fr[FCG_MAX_DIM];
    bool cl = false;
    for (int k = 0; k < p.d; ++k) {
      const double *z = knots + p.koff[k];
      const int m = (int)p.m[k];
      double col = q[t * p.d + k];
      const double lo = z[0], hi = z[m - 1];
      cl = cl || col < lo || col > hi;
      col = fmin(fmax(col, lo), hi);  // np.clip
      const double idz = (double)(m - 1) / (hi - lo);
      int c = knot_count(col, z, m, 1, lo, idz) - 1;  // searchsorted(right) - 1
      c = c < 0 ? 0 : (c > m - 2 ? m - 2 : c);
      cell[k] = c;
      fr[k] = __ddiv_rn(__dsub_rn(col, z[c]), __dsub_rn(z[c + 1], z[c]));
    }
    double acc = 0.0;
    for (int corner = 0; corner < (1 << p.d); ++corner) {
      double w = 1.0;
      int64_t flat = 0;
      for (int k = 0; k < p.d; ++k) {
        const int bit = (corner >> k) & 1;
        w = __dmul_rn(w, bit ? fr[k] : __dsub_rn(1.0, fr[k]));
        flat = flat * p.m[k] + cell[k] + bit;
      }
      acc = __dadd_rn(acc, __dmul_rn(w, vals[flat]));
    }
    out[t] = acc;
    local += cl ? 1u : 0u;
  }
  // clamp count: warp sum, one atomic per warp
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(clamp, (unsigned long long)local);
}

}  // namespace
}  // namespace fcg

using namespace fcg;

extern "C" int fcg_multilinear_interp(const double *knots, const int64_t *m, int32_t d,
                                      const double *values, const double *q, int64_t nq,
                                      double *out, int64_t *clamp_count, void *ws,
                                      size_t *ws_bytes, void *stream) {
  if (d < 1 || d > FCG_MAX_DIM) return fail(FCG_EUNSUPPORTED, "dimension out of range");
  for (int k = 0; k < d; ++k)
    if (m[k] < 2) return fail(FCG_EINVAL, "interpolation needs at least 2 knots per dimension");
  if (nq < 0) return fail(FCG_EINVAL, "nq must be >= 0");
  Workspace W(ws);
  unsigned long long *cnt = W.take<unsigned long long>(1);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  cudaStream_t st = as_stream(stream);
  InterpP p{};
  p.d = d;
  int64_t off = 0;
  for (int k = 0; k < d; ++k) {
    p.m[k] = m[k];
    p.koff[k] = off;
    off += m[k];
  }
  FCG_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
  if (nq > 0) {
    FCG_PROF("interp", st);
    interp_kernel<<<grid_for(nq, 256), 256, 0, st>>>(knots, p, values, q, nq, out, cnt);
    FCG_LAUNCH_CHECK();
  }
  if (clamp_count) {  // host scalar: synchronises the stream
    unsigned long long h = 0;
    FCG_TRY(read_small(&h, cnt, sizeof(h), st));
    *clamp_count = (int64_t)h;
  }
  return FCG_OK;
}
