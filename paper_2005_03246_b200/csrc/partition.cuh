// Stable partition of n items by one 8-bit digit of a 32-bit key that builds a record of
// `words` doubles per item on the way (build(i, out) writes item i's record): the pass that
// groups the items also writes their records, record-major, next to their keys and slots.
// A tile (kPartTile items) is ranked exactly like the radix sort's scatter (match_any peers +
// per-warp digit counters, digit-major global offsets, so items of one digit keep their input
// order), built into shared memory in digit order, and written out with consecutive threads on
// consecutive doubles of each digit's run.
#pragma once
#include "sort.cuh"

namespace fcg {

constexpr int kPartThreads = 256;
constexpr int kPartItems = 16;
constexpr int kPartTile = kPartThreads * kPartItems;  // 4096 items per CTA

namespace part_detail {

__device__ __forceinline__ unsigned lane_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

static __global__ void __launch_bounds__(kPartThreads) digit_hist_kernel(const uint32_t *__restrict__ keys,
                                                                  int64_t n, int shift,
                                                                  int32_t *__restrict__ hist,
                                                                  int64_t tiles) {
  __shared__ int32_t s_hist[kPartThreads / 32][256];
  const int warp = threadIdx.x >> 5;
  for (int d = threadIdx.x & 31; d < 256; d += 32) s_hist[warp][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kPartTile;
  uint32_t k[kPartItems];  // every key of the tile in flight before the counting
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int64_t i = base + (int64_t)j * kPartThreads + threadIdx.x;
    k[j] = i < n ? keys[i] : 0u;
  }
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int64_t i = base + (int64_t)j * kPartThreads + threadIdx.x;
    if (i < n) atomicAdd(&s_hist[warp][(k[j] >> shift) & 0xFFu], 1);
  }
  __syncthreads();
  int32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kPartThreads / 32; ++w) tot += s_hist[w][threadIdx.x];
  hist[(int64_t)threadIdx.x * tiles + blockIdx.x] = tot;
}

// Build: struct with `static constexpr int kD` (point dimension, > 0) and
//   void operator()(const double *xi, double wi, double *out) const  (writes kWords doubles)
template <class Build, int WORDS>
__global__ void __launch_bounds__(kPartThreads, 2) digit_stage_kernel(
    const uint32_t *__restrict__ keys, int64_t n, int shift, const int32_t *__restrict__ offs,
    int64_t tiles, const double *__restrict__ x, const double *__restrict__ w, Build build,
    double *__restrict__ rec_out, uint32_t *__restrict__ keys_out, int32_t *__restrict__ slot_out,
    double *__restrict__ last_out) {
  constexpr int D = Build::kD;
  extern __shared__ __align__(16) unsigned char ps_smem[];
  double *s_rec = reinterpret_cast<double *>(ps_smem);                       // [tile][WORDS]
  uint32_t *s_key = reinterpret_cast<uint32_t *>(s_rec + (size_t)kPartTile * WORDS);
  int32_t *s_cnt = reinterpret_cast<int32_t *>(s_key + kPartTile);            // [8][256]
  int32_t *s_goff = s_cnt + (kPartThreads / 32) * 256;
  int32_t *s_tstart = s_goff + 256;
  int32_t *s_wsum = s_tstart + 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) s_cnt[warp * 256 + d] = 0;
  s_goff[threadIdx.x] = offs[(int64_t)threadIdx.x * tiles + blockIdx.x];
  __syncwarp();
  const int64_t tile0 = (int64_t)blockIdx.x * kPartTile;
  const int64_t base = tile0 + (int64_t)warp * (kPartTile / 8);
  const int tile_n = (int)((n - tile0) < kPartTile ? (n - tile0) : kPartTile);
  uint32_t k[kPartItems];
  int32_t r[kPartItems];
  double xs[kPartItems][D], ws[kPartItems];
  // every item's key, point and weight in flight before the ranking needs them
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int64_t i = base + (int64_t)j * 32 + lane;
    const bool ok = i < n;
    const int64_t ii = ok ? i : 0;
    k[j] = ok ? keys[i] : 0u;
    if constexpr (D % 2 == 0) {
#pragma unroll
      for (int c = 0; c < D; c += 2) {
        const double2 v = reinterpret_cast<const double2 *>(x + ii * D)[c / 2];
        xs[j][c] = v.x;
        xs[j][c + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < D; ++c) xs[j][c] = x[ii * D + c];
    }
    ws[j] = w ? w[ii] : 1.0;
  }
  const unsigned lt = lane_lt();
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int64_t i = base + (int64_t)j * 32 + lane;
    const bool ok = i < n;
    const unsigned dig = ok ? ((k[j] >> shift) & 0xFFu) : 256u + lane;
    const unsigned peers = digit_peers(dig);
    int32_t before = 0;
    if (ok) before = s_cnt[warp * 256 + dig];
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) s_cnt[warp * 256 + dig] = before + __popc(peers);
    __syncwarp();
    r[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    int32_t run = 0;
#pragma unroll
    for (int wp = 0; wp < kPartThreads / 32; ++wp) {
      const int32_t t = s_cnt[wp * 256 + d];
      s_cnt[wp * 256 + d] = run;
      run += t;
    }
    int32_t xx = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, xx, o);
      if (lane >= o) xx += y;
    }
    if (lane == 31) s_wsum[warp] = xx;
    __syncthreads();
    int32_t wpre = 0;
    for (int wp = 0; wp < warp; ++wp) wpre += s_wsum[wp];
    s_tstart[d] = wpre + xx - run;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int64_t i = base + (int64_t)j * 32 + lane;
    if (i < n) {
      const unsigned dig = (k[j] >> shift) & 0xFFu;
      const int pos = s_tstart[dig] + s_cnt[warp * 256 + dig] + r[j];
      s_key[pos] = k[j];
      build(xs[j], ws[j], s_rec + (size_t)pos * WORDS);
    }
  }
  __syncthreads();
  if (keys_out || slot_out) {
    for (int pos = threadIdx.x; pos < tile_n; pos += kPartThreads) {
      const uint32_t key = s_key[pos];
      const unsigned dig = (key >> shift) & 0xFFu;
      const int64_t dst = (int64_t)s_goff[dig] + (pos - s_tstart[dig]);
      if (keys_out) keys_out[dst] = key;
      if (slot_out) slot_out[dst] = (int32_t)dst;
    }
  }
  if (last_out == nullptr) {
    const int tw = tile_n * WORDS;
    for (int idx = threadIdx.x; idx < tw; idx += kPartThreads) {
      const int pos = idx / WORDS;  // compile-time divisor
      const unsigned dig = (s_key[pos] >> shift) & 0xFFu;
      const int64_t dst = (int64_t)s_goff[dig] + (pos - s_tstart[dig]);
      rec_out[dst * WORDS + (idx - pos * WORDS)] = s_rec[idx];
    }
  } else {  // split records: the first WORDS-1 words to rec_out, the last word to last_out
    constexpr int W1 = WORDS - 1;
    const int tw = tile_n * W1;
    for (int idx = threadIdx.x; idx < tw; idx += kPartThreads) {
      const int pos = idx / W1;
      const int wd = idx - pos * W1;
      const unsigned dig = (s_key[pos] >> shift) & 0xFFu;
      const int64_t dst = (int64_t)s_goff[dig] + (pos - s_tstart[dig]);
      rec_out[dst * W1 + wd] = s_rec[pos * WORDS + wd];
    }
    for (int pos = threadIdx.x; pos < tile_n; pos += kPartThreads) {
      const unsigned dig = (s_key[pos] >> shift) & 0xFFu;
      const int64_t dst = (int64_t)s_goff[dig] + (pos - s_tstart[dig]);
      last_out[dst] = s_rec[pos * WORDS + W1];
    }
  }
}

// Variant for costly builds (the KDE records: d + 1 exponentials per item).  The tile is ranked
// from its keys alone and only (key, item index) is staged in shared memory; each item's record
// is built at write-out time from x / w re-read in tile order (a 4096-item window, so the
// re-read is sector-dense and the points are fetched from DRAM once).  6 bytes of shared
// memory and a handful of registers per item instead of a staged record (3 CTAs per SM: the
// record build keeps its exponentials in registers).
template <class Build, int WORDS>
__global__ void __launch_bounds__(kPartThreads, 3) digit_stage_late_kernel(
    const uint32_t *__restrict__ keys, int64_t n, int shift, const int32_t *__restrict__ offs,
    int64_t tiles, const double *__restrict__ x, const double *__restrict__ w, Build build,
    double *__restrict__ rec_out, uint32_t *__restrict__ keys_out, int32_t *__restrict__ slot_out,
    double *__restrict__ last_out) {
  constexpr int D = Build::kD;
  __shared__ uint32_t s_key[kPartTile];
  __shared__ uint16_t s_src[kPartTile];
  __shared__ int32_t s_cnt[(kPartThreads / 32) * 256];
  __shared__ int32_t s_goff[256], s_tstart[256], s_wsum[kPartThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) s_cnt[warp * 256 + d] = 0;
  s_goff[threadIdx.x] = offs[(int64_t)threadIdx.x * tiles + blockIdx.x];
  __syncwarp();
  const int64_t tile0 = (int64_t)blockIdx.x * kPartTile;
  const int wbase = warp * (kPartTile / 8);
  const int tile_n = (int)((n - tile0) < kPartTile ? (n - tile0) : kPartTile);
  uint32_t k[kPartItems];
  int32_t r[kPartItems];
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int li = wbase + j * 32 + lane;
    k[j] = li < tile_n ? keys[tile0 + li] : 0u;
  }
  const unsigned lt = lane_lt();
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const bool ok = wbase + j * 32 + lane < tile_n;
    const unsigned dig = ok ? ((k[j] >> shift) & 0xFFu) : 256u + lane;
    const unsigned peers = digit_peers(dig);
    int32_t before = 0;
    if (ok) before = s_cnt[warp * 256 + dig];
    __syncwarp();
    if (ok && lane == __ffs(peers) - 1) s_cnt[warp * 256 + dig] = before + __popc(peers);
    __syncwarp();
    r[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    int32_t run = 0;
#pragma unroll
    for (int wp = 0; wp < kPartThreads / 32; ++wp) {
      const int32_t t = s_cnt[wp * 256 + d];
      s_cnt[wp * 256 + d] = run;
      run += t;
    }
    int32_t xx = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, xx, o);
      if (lane >= o) xx += y;
    }
    if (lane == 31) s_wsum[warp] = xx;
    __syncthreads();
    int32_t wpre = 0;
    for (int wp = 0; wp < warp; ++wp) wpre += s_wsum[wp];
    s_tstart[d] = wpre + xx - run;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPartItems; ++j) {
    const int li = wbase + j * 32 + lane;
    if (li < tile_n) {
      const unsigned dig = (k[j] >> shift) & 0xFFu;
      const int pos = s_tstart[dig] + s_cnt[warp * 256 + dig] + r[j];
      s_key[pos] = k[j];
      s_src[pos] = (uint16_t)li;
    }
  }
  __syncthreads();
  // write-out in grouped order: two items per thread step, their point loads issued together
  for (int p0 = threadIdx.x; p0 < tile_n; p0 += 2 * kPartThreads) {
    double xs[2][D], ws[2];
    uint32_t kk[2];
    int64_t dst[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int pos = p0 + u * kPartThreads;
      ok[u] = pos < tile_n;
      const int pp = ok[u] ? pos : p0;
      kk[u] = s_key[pp];
      const unsigned dig = (kk[u] >> shift) & 0xFFu;
      dst[u] = (int64_t)s_goff[dig] + (pp - s_tstart[dig]);
      const int64_t i = tile0 + s_src[pp];
      if constexpr (D % 2 == 0) {
#pragma unroll
        for (int c = 0; c < D; c += 2) {
          const double2 v = reinterpret_cast<const double2 *>(x + i * D)[c / 2];
          xs[u][c] = v.x;
          xs[u][c + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) xs[u][c] = x[i * D + c];
      }
      ws[u] = w ? w[i] : 1.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      double rr[WORDS];
      build(xs[u], ws[u], rr);
      if (last_out == nullptr) {
        double *o = rec_out + dst[u] * WORDS;
#pragma unroll
        for (int f = 0; f < WORDS; ++f) o[f] = rr[f];
      } else {  // split records: the first WORDS-1 words to rec_out, the last to last_out
        double *o = rec_out + dst[u] * (WORDS - 1);
#pragma unroll
        for (int f = 0; f < WORDS - 1; ++f) o[f] = rr[f];
        last_out[dst[u]] = rr[WORDS - 1];
      }
      if (keys_out) keys_out[dst[u]] = kk[u];
      if (slot_out) slot_out[dst[u]] = (int32_t)dst[u];
    }
  }
}

}  // namespace part_detail

inline size_t digit_stage_smem(int words) {
  return (size_t)kPartTile * (words * sizeof(double) + sizeof(uint32_t)) +
         ((kPartThreads / 32) * 256 + 256 + 256 + 8) * sizeof(int32_t);
}

inline size_t digit_hist_elems(int64_t n) { return (size_t)256 * (size_t)ceil_div(n, kPartTile) + 1; }

// Workspace: hist = digit_hist_elems(n) ints, partial = scan_ws_partial_elems(hist elems).
// x: (n, Build::kD) row-major points (16-byte aligned when kD is even), w: weights or NULL.
template <class Build, int WORDS>
int digit_partition_build(const uint32_t *keys, int64_t n, int shift, const double *x,
                          const double *w, const Build &build, double *rec_out,
                          uint32_t *keys_out, int32_t *slot_out, int32_t *hist, int32_t *partial,
                          cudaStream_t st, double *last_out = nullptr,
                          const char *label = "part_emit", bool hist_ready = false,
                          bool late_build = false) {
  if (n <= 0) return FCG_OK;
  const int64_t tiles = ceil_div(n, kPartTile);
  if (!hist_ready) {  // else: the key producer already wrote the per-tile digit histogram
    FCG_PROF("part_hist", st);
    part_detail::digit_hist_kernel<<<(unsigned)tiles, kPartThreads, 0, st>>>(keys, n, shift, hist,
                                                                            tiles);
    FCG_LAUNCH_CHECK();
  }
  FCG_TRY(scan_i32(hist, hist, 256 * tiles, false, partial, st));
  FCG_PROF(label, st);
  if (late_build) {
    part_detail::digit_stage_late_kernel<Build, WORDS><<<(unsigned)tiles, kPartThreads, 0, st>>>(
        keys, n, shift, hist, tiles, x, w, build, rec_out, keys_out, slot_out, last_out);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }
  const size_t sm = digit_stage_smem(WORDS);
  auto kern = part_detail::digit_stage_kernel<Build, WORDS>;
  FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  kern<<<(unsigned)tiles, kPartThreads, sm, st>>>(keys, n, shift, hist, tiles, x, w, build,
                                                  rec_out, keys_out, slot_out, last_out);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

}  // namespace fcg
