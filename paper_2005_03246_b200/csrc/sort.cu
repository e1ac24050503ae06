// Subsystem 1 (ranking): stable LSD radix sort of order-preserving fp64 keys, device-wide
// scans and the rank outputs of fcg_rank_f64.  Replaces np.argsort(kind="stable")
// (histogram.py:131, dnc.py:517,527,544) and the tie scan of core.py:278-281.
//
// One radix pass (8-bit digit) = digit histogram per 4096-item tile (warp-aggregated shared
// atomics) -> exclusive scan of the digit-major histogram -> stable scatter: every warp ranks
// its 512 items with __match_any_sync peers and per-warp digit counters, so equal digits keep
// their input order (stability across tiles comes from the digit-major global offsets).
#include "sort.cuh"

namespace fcg {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one int per thread (blockDim = 1024); returns the exclusive
// prefix, *total receives the block total.
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t *s_warp, int32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t t = (lane < (int)(blockDim.x >> 5)) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;  // inclusive warp-total prefix
  }
  __syncthreads();
  const int32_t warp_excl = warp ? s_warp[warp - 1] : 0;
  *total = s_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// single CTA, whole array (small scans: one launch instead of three)
__global__ void __launch_bounds__(kScanThreads) scan_single_kernel(const int32_t *in, int32_t *out,
                                                                   int64_t n, int inclusive) {
  __shared__ int32_t s_warp[32];
  int32_t carry = 0;
  for (int64_t b0 = 0; b0 < n; b0 += kScanTile) {
    const int64_t base = b0 + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    int32_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      v[j] = (base + j < n) ? in[base + j] : 0;
      s += v[j];
    }
    int32_t tot;
    int32_t run = block_excl_scan(s, s_warp, &tot) + carry;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
      if (base + j < n) out[base + j] = inclusive ? run + v[j] : run;
      run += v[j];
    }
    carry += tot;
    __syncthreads();
  }
}

// ---- single-pass scan with decoupled look-back ------------------------------------------
// One launch per scan (plus a memset of the tile status words): tile t publishes its aggregate
// (flag 1), then its inclusive prefix (flag 2) as soon as the look-back over its predecessors
// (a warp reading 32 status words at a time) has found one.  Tiles are taken in blockIdx order
// (lower tiles are dispatched first, so every tile waited on is resident or done).
constexpr int kLbThreads = 512;
constexpr int kLbItems = 8;
constexpr int kLbTile = kLbThreads * kLbItems;

__device__ __forceinline__ void lb_publish(unsigned long long *p, unsigned flag, int32_t v) {
  const unsigned long long w = ((unsigned long long)flag << 32) | (uint32_t)v;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long lb_read(const unsigned long long *p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

__global__ void __launch_bounds__(kLbThreads) scan_lookback_kernel(
    const int32_t *in, int32_t *out, int64_t n, int inclusive, unsigned long long *status) {
  __shared__ int32_t s_warp[32];
  __shared__ int32_t s_prefix;
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * kLbTile + (int64_t)threadIdx.x * kLbItems;
  int32_t v[kLbItems];
  int32_t sum = 0;
  if (base + kLbItems <= n && (reinterpret_cast<uintptr_t>(in + base) & 15) == 0) {
    const int4 a = reinterpret_cast<const int4 *>(in + base)[0];
    const int4 b = reinterpret_cast<const int4 *>(in + base)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int j = 0; j < kLbItems; ++j) v[j] = base + j < n ? in[base + j] : 0;
  }
#pragma unroll
  for (int j = 0; j < kLbItems; ++j) sum += v[j];
  int32_t agg;
  const int32_t excl = block_excl_scan(sum, s_warp, &agg);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int32_t prefix = 0;
    if (tile == 0) {
      if (lane == 0) lb_publish(status, 2u, agg);
    } else {
      if (lane == 0) lb_publish(status + tile, 1u, agg);
      int64_t idx = tile - 1;
      while (true) {
        const int64_t j = idx - lane;
        unsigned long long w = 0;
        unsigned flag = 2;  // before tile 0: an inclusive 0
        if (j >= 0) {
          do {
            w = lb_read(status + j);
            flag = (unsigned)(w >> 32);
          } while (flag == 0);
        }
        const int32_t val = j >= 0 ? (int32_t)(uint32_t)w : 0;
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2);
        if (inc) {
          const int first = __ffs(inc) - 1;  // nearest predecessor with its inclusive prefix
          int32_t x = lane <= first ? val : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          prefix += x;
          break;
        }
        int32_t x = val;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        prefix += x;
        idx -= 32;
      }
      if (lane == 0) lb_publish(status + tile, 2u, prefix + agg);
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  int32_t run = s_prefix + excl;
#pragma unroll
  for (int j = 0; j < kLbItems; ++j) {
    const int32_t o = inclusive ? run + v[j] : run;
    run += v[j];
    v[j] = o;
  }
  if (base + kLbItems <= n && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
    reinterpret_cast<int4 *>(out + base)[0] = make_int4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<int4 *>(out + base)[1] = make_int4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int j = 0; j < kLbItems; ++j)
      if (base + j < n) out[base + j] = v[j];
  }
}

__global__ void radix_init_kernel(const double *__restrict__ x, int64_t n, int64_t stride,
                                  uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = f64_key(x[i * stride]);
    vals[i] = (int32_t)i;
  }
}

// Tile maps: which items tile g covers and where its digit counts live in the histogram that
// the exclusive scan turns into global offsets.
//   FlatMap: tile g = items [g T, min(n, g T + T)), counts digit-major over all tiles.
//   SegMap:  items are grouped in segments (seg_start[s] .. seg_start[s+1]); tiles never straddle
//            a segment, counts are laid out [segment][digit][tile of the segment], so one scan
//            yields offsets that keep every item inside its segment (a segmented LSD pass).
struct FlatMap {
  int64_t n, tiles;
  __device__ __forceinline__ bool range(int64_t g, int64_t &start, int &len) const {
    start = g * kSortTile;
    const int64_t r = n - start;
    len = (int)(r < kSortTile ? r : kSortTile);
    return true;
  }
  __device__ __forceinline__ int64_t hidx(int64_t g, int d) const { return (int64_t)d * tiles + g; }
};

struct SegMap {
  const int32_t *seg_start, *tile_base, *tile_seg;
  __device__ __forceinline__ bool range(int64_t g, int64_t &start, int &len) const {
    if (g >= tile_base[kSortSegs]) return false;  // past the last segment's tiles
    const int s = tile_seg[g];
    const int64_t t = g - tile_base[s];
    start = seg_start[s] + t * kSortTile;
    const int64_t r = seg_start[s + 1] - start;
    len = (int)(r < kSortTile ? r : kSortTile);
    return true;
  }
  __device__ __forceinline__ int64_t hidx(int64_t g, int d) const {
    const int s = tile_seg[g];
    const int64_t nt = tile_base[s + 1] - tile_base[s];
    return (int64_t)256 * tile_base[s] + (int64_t)d * nt + (g - tile_base[s]);
  }
};

template <typename KeyT, class Map>
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const KeyT *__restrict__ keys,
                                                                  Map map, int shift,
                                                                  int32_t *__restrict__ hist) {
  __shared__ int32_t s_hist[kSortThreads / 32][256];
  int64_t base;
  int len;
  if (!map.range(blockIdx.x, base, len)) return;
  const int warp = threadIdx.x >> 5;
  for (int d = threadIdx.x & 31; d < 256; d += 32) s_hist[warp][d] = 0;
  __syncwarp();
  KeyT k[kSortItems];  // every key of the tile in flight before the counting
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int ii = j * kSortThreads + threadIdx.x;
    k[j] = ii < len ? keys[base + ii] : KeyT(0);
  }
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int ii = j * kSortThreads + threadIdx.x;
    if (ii < len) atomicAdd(&s_hist[warp][(unsigned)((k[j] >> shift) & 0xFF)], 1);
  }
  __syncthreads();
  int32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) tot += s_hist[w][threadIdx.x];
  hist[map.hidx(blockIdx.x, threadIdx.x)] = tot;
}

// Stable scatter of one tile (4096 items) by one 8-bit digit.  Items are first ranked inside
// the tile (warp peers via __match_any_sync + per-warp digit counters), staged in shared memory
// in digit order, then written out so that consecutive threads write consecutive addresses of
// each digit's run (coalesced) instead of 32 scattered 4-byte stores per warp.
// STABLE = false (first LSD pass of a sort whose equal keys may come out in any order): items
// are ranked by a shared-memory atomic on their warp's digit counter instead of peer masks.
// GW > 0 (record gather, last pass of a segmented sort): instead of the value, item v's record
// rec_in[v * GW + f] is written field-major to rec_out[f * rec_n + dst].
template <typename KeyT, bool STABLE, class Map, int GW>
__global__ void __launch_bounds__(kSortThreads, 3) radix_scatter_kernel(
    const KeyT *__restrict__ kin, const int32_t *__restrict__ vin, KeyT *__restrict__ kout,
    int32_t *__restrict__ vout, Map map, int shift, const int32_t *__restrict__ offs,
    const double *__restrict__ rec_in, double *__restrict__ rec_out, int64_t rec_n) {
  extern __shared__ __align__(16) unsigned char rs_smem[];
  KeyT *s_key = reinterpret_cast<KeyT *>(rs_smem);                       // [kSortTile]
  int32_t *s_val = reinterpret_cast<int32_t *>(s_key + kSortTile);        // [kSortTile]
  int32_t *s_cnt = s_val + kSortTile;                                     // [8][256]
  int32_t *s_goff = s_cnt + (kSortThreads / 32) * 256;                    // [256]
  int32_t *s_tstart = s_goff + 256;                                       // [256]
  int32_t *s_wsum = s_tstart + 256;                                       // [8]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t tile0;
  int tile_n;
  if (!map.range(blockIdx.x, tile0, tile_n)) return;
  for (int d = lane; d < 256; d += 32) s_cnt[warp * 256 + d] = 0;
  s_goff[threadIdx.x] = offs[map.hidx(blockIdx.x, threadIdx.x)];
  __syncwarp();
  const int64_t base = tile0 + (int64_t)warp * (kSortTile / 8);
  const int64_t n = tile0 + tile_n;  // end of this tile's items
  KeyT k[kSortItems];
  int32_t v[kSortItems];
  int32_t r[kSortItems];
  const unsigned lt = lanemask_lt();
  // all of the tile's keys and values in flight before the ranking (which orders on syncwarps)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + (int64_t)j * 32 + lane;
    const bool ok = i < n;
    k[j] = ok ? kin[i] : KeyT(0);
    // vin == NULL: the values are the positions; vout == NULL (and no records): keys only
    v[j] = (ok && (vout || GW > 0)) ? (vin ? vin[i] : (int32_t)i) : 0;
  }
  if constexpr (STABLE) {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t i = base + (int64_t)j * 32 + lane;
      const bool ok = i < n;
      const unsigned dig = ok ? (unsigned)((k[j] >> shift) & 0xFF) : 256u + lane;
      const unsigned peers = digit_peers(dig);
      int32_t before = 0;
      if (ok) before = s_cnt[warp * 256 + dig];
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) s_cnt[warp * 256 + dig] = before + __popc(peers);
      __syncwarp();
      r[j] = before + __popc(peers & lt);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
      const int64_t i = base + (int64_t)j * 32 + lane;
      if (i < n) r[j] = atomicAdd(s_cnt + warp * 256 + (unsigned)((k[j] >> shift) & 0xFF), 1);
    }
  }
  __syncthreads();
  {
    // per digit: exclusive prefix over warps, and the digit's total for the tile-level scan
    const int d = threadIdx.x;
    int32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) {
      const int32_t t = s_cnt[w * 256 + d];
      s_cnt[w * 256 + d] = run;
      run += t;
    }
    // exclusive scan of the 256 digit totals -> tile start of every digit run
    int32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    int32_t wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
    s_tstart[d] = wpre + x - run;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + (int64_t)j * 32 + lane;
    if (i < n) {
      const unsigned dig = (unsigned)((k[j] >> shift) & 0xFF);
      const int pos = s_tstart[dig] + s_cnt[warp * 256 + dig] + r[j];
      s_key[pos] = k[j];
      s_val[pos] = v[j];
    }
  }
  __syncthreads();
  for (int pos = threadIdx.x; pos < tile_n; pos += kSortThreads) {
    const KeyT key = s_key[pos];
    const unsigned dig = (unsigned)((key >> shift) & 0xFF);
    const int64_t dst = (int64_t)s_goff[dig] + (pos - s_tstart[dig]);
    kout[dst] = key;
    if constexpr (GW > 0) {
      const double *r = rec_in + (int64_t)s_val[pos] * GW;
      double f[GW];
#pragma unroll
      for (int w = 0; w < GW; ++w) f[w] = r[w];
#pragma unroll
      for (int w = 0; w < GW; ++w) __stcs(rec_out + (int64_t)w * rec_n + dst, f[w]);
    } else {
      if (vout) vout[dst] = s_val[pos];
    }
  }
}

template <typename KeyT>
constexpr size_t radix_scatter_smem() {
  return (size_t)kSortTile * (sizeof(KeyT) + 4) + ((kSortThreads / 32) * 256 + 256 + 256 + 8) * 4;
}

__global__ void rank_heads_kernel(const uint64_t *__restrict__ keys,
                                  const int32_t *__restrict__ order, int64_t n,
                                  int32_t *__restrict__ heads, int32_t *__restrict__ pos) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    heads[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
    if (pos) pos[order[p]] = (int32_t)p;
  }
}

// heads now holds the inclusive scan (dense rank + 1) of the head flags
__global__ void rank_start_kernel(const uint64_t *__restrict__ keys, const int32_t *__restrict__ incl,
                                  int64_t n, int32_t *__restrict__ start, int32_t *n_distinct) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t dr = incl[p] - 1;
    if (p == 0 || keys[p] != keys[p - 1]) start[dr] = (int32_t)p;
    if (p == n - 1) {
      start[dr + 1] = (int32_t)n;
      if (n_distinct) *n_distinct = dr + 1;
    }
  }
}

__global__ void rank_scatter_kernel(const int32_t *__restrict__ order,
                                    const int32_t *__restrict__ incl,
                                    const int32_t *__restrict__ start, int64_t n,
                                    int32_t *lower, int32_t *upper, int32_t *dense) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = order[p];
    const int32_t dr = incl[p] - 1;
    if (dense) dense[i] = dr;
    if (lower) lower[i] = start[dr];
    if (upper) upper[i] = start[dr + 1];
  }
}

// AND / OR of all keys: digits where they agree are the same for every key, so the radix
// passes on them are identities and can be skipped.
__global__ void key_andor_kernel(const uint64_t *__restrict__ keys, int64_t n,
                                 unsigned long long *__restrict__ out) {
  uint64_t a = ~0ull, o = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    a &= k;
    o |= k;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    a &= __shfl_xor_sync(0xffffffffu, a, s);
    o |= __shfl_xor_sync(0xffffffffu, o, s);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAnd(out, (unsigned long long)a);
    atomicOr(out + 1, (unsigned long long)o);
  }
}

__global__ void key_andor_init(unsigned long long *out, int pairs = 1) {
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    out[2 * i] = ~0ull;
    out[2 * i + 1] = 0ull;
  }
}

// AND / OR of the order-preserving keys of every column of x (n, d): one pass over x for all
// dimensions (the rank path then needs one host read-back for every dimension's digit mask)
__global__ void key_andor_dims_kernel(const double *__restrict__ x, int64_t n, int d,
                                      unsigned long long *__restrict__ out) {
  for (int k = 0; k < d; ++k) {
    uint64_t a = ~0ull, o = 0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const uint64_t key = f64_key(x[i * d + k]);
      a &= key;
      o |= key;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      a &= __shfl_xor_sync(0xffffffffu, a, s);
      o |= __shfl_xor_sync(0xffffffffu, o, s);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAnd(out + 2 * k, (unsigned long long)a);
      atomicOr(out + 2 * k + 1, (unsigned long long)o);
    }
  }
}

// seg_start[c] = first item of segment c (key >> seg_shift == c) of keys grouped by segment;
// empty segments start where the next one does; seg_start[kSortSegs] = n
__global__ void __launch_bounds__(256) seg_bounds_kernel(const uint32_t *__restrict__ keys,
                                                         int64_t n, int seg_shift,
                                                         int32_t *__restrict__ seg_start) {
  constexpr int K = 8;  // consecutive keys per thread, all loaded before the compares
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * K;
  if (i0 >= n) return;
  // segment digits saturate at the last segment (dead keys, all ones, sort there)
  auto seg = [&](uint32_t key) { return (int)min(key >> seg_shift, (uint32_t)(kSortSegs - 1)); };
  int c[K + 1];
  c[0] = i0 ? seg(keys[i0 - 1]) : -1;
#pragma unroll
  for (int k = 0; k < K; ++k) c[k + 1] = i0 + k < n ? seg(keys[i0 + k]) : kSortSegs;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (i0 + k >= n) break;
    for (int x = c[k] + 1; x <= c[k + 1]; ++x) seg_start[x] = (int32_t)(i0 + k);
  }
  if (i0 + K >= n) {  // the thread holding the last key closes the remaining segments
    const int64_t last = n - 1;
    for (int x = seg(keys[last]) + 1; x <= kSortSegs; ++x) seg_start[x] = (int32_t)n;
  }
}

// one CTA of kSortSegs threads: tiles per segment, their exclusive scan (tile_base, with the
// total at [kSortSegs]) and the tile -> segment map
__global__ void __launch_bounds__(kSortSegs) seg_tiles_kernel(const int32_t *__restrict__ seg_start,
                                                              int32_t *__restrict__ tile_base,
                                                              int32_t *__restrict__ tile_seg) {
  __shared__ int32_t s_warp[kSortSegs / 32];
  const int sg = threadIdx.x, lane = sg & 31, warp = sg >> 5;
  const int32_t nt = (seg_start[sg + 1] - seg_start[sg] + kSortTile - 1) / kSortTile;
  int32_t x = nt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  int32_t pre = 0;
  for (int w = 0; w < warp; ++w) pre += s_warp[w];
  const int32_t ex = pre + x - nt;
  tile_base[sg] = ex;
  if (sg == kSortSegs - 1) tile_base[kSortSegs] = ex + nt;
  for (int32_t t = 0; t < nt; ++t) tile_seg[ex + t] = sg;
}

}  // namespace

size_t radix_ws_hist_elems(int64_t n) { return (size_t)256 * (size_t)ceil_div(n, kSortTile) + 1; }

// int32 elements: the single-pass scan's 64-bit status word per kLbTile tile (+ alignment slack)
size_t scan_ws_partial_elems(int64_t n) { return 2 * (size_t)ceil_div(n, kLbTile) + 4; }

int scan_i32(const int32_t *in, int32_t *out, int64_t n, bool inclusive, int32_t *partial,
             cudaStream_t st) {
  if (n <= 0) return FCG_OK;
  const int64_t blocks = ceil_div(n, kScanTile);
  FCG_PROF("scan_i32", st);
  if (blocks <= 2) {
    scan_single_kernel<<<1, kScanThreads, 0, st>>>(in, out, n, inclusive ? 1 : 0);
    FCG_LAUNCH_CHECK();
    return FCG_OK;
  }
  // single pass: status words live in the partials buffer (sized for kScanTile tiles of 32-bit
  // words, i.e. room for as many 64-bit words as kLbTile = kScanTile / 2 tiles need)
  const int64_t tiles = ceil_div(n, kLbTile);
  unsigned long long *status = reinterpret_cast<unsigned long long *>(partial);
  FCG_CUDA_TRY(cudaMemsetAsync(status, 0, (size_t)tiles * sizeof(unsigned long long), st));
  scan_lookback_kernel<<<(unsigned)tiles, kLbThreads, 0, st>>>(in, out, n, inclusive ? 1 : 0,
                                                              status);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

int radix_init_f64(const double *x, int64_t n, int64_t stride, uint64_t *keys, int32_t *vals,
                   cudaStream_t st) {
  if (n <= 0) return FCG_OK;
  FCG_PROF("radix_init", st);
  radix_init_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(x, n, stride, keys, vals);
  FCG_LAUNCH_CHECK();
  return FCG_OK;
}

template <typename KeyT>
static int radix_sort_digits(KeyT *keys, int32_t *vals, int64_t n, uint32_t digit_mask,
                             const RadixWs &ws, cudaStream_t st, bool stable = true,
                             bool first_hist_ready = false) {
  if (n <= 1) return FCG_OK;
  const int64_t tiles = ceil_div(n, kSortTile);
  KeyT *ka = keys, *kb = reinterpret_cast<KeyT *>(ws.keys_alt);
  int32_t *va = vals, *vb = ws.vals_alt;
  int passes = 0;
  for (int dg = 0; dg < (int)sizeof(KeyT); ++dg) {
    if (!((digit_mask >> dg) & 1u)) continue;
    const int shift = 8 * dg;
    const FlatMap map{n, tiles};
    if (!(first_hist_ready && passes == 0)) {
      FCG_PROF("radix_hist", st);
      radix_hist_kernel<KeyT, FlatMap><<<(unsigned)tiles, kSortThreads, 0, st>>>(ka, map, shift, ws.hist);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(scan_i32(ws.hist, ws.hist, 256 * tiles, false, ws.partial, st));
    {
      FCG_PROF("radix_scatter", st);
      constexpr size_t sm = radix_scatter_smem<KeyT>();
      // only the first pass may reorder equal keys: later passes must keep the earlier order
      auto kern = (stable || passes > 0) ? radix_scatter_kernel<KeyT, true, FlatMap, 0>
                                         : radix_scatter_kernel<KeyT, false, FlatMap, 0>;
      FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      kern<<<(unsigned)tiles, kSortThreads, sm, st>>>(ka, va, kb, vb, map, shift, ws.hist, nullptr,
                                                      nullptr, 0);
      FCG_LAUNCH_CHECK();
    }
    std::swap(ka, kb);
    std::swap(va, vb);
    ++passes;
  }
  if (passes & 1) {
    FCG_CUDA_TRY(cudaMemcpyAsync(keys, ka, (size_t)n * sizeof(KeyT), cudaMemcpyDeviceToDevice, st));
    FCG_CUDA_TRY(cudaMemcpyAsync(vals, va, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  }
  return FCG_OK;
}

template <typename KeyT>
int radix_sort_pairs(KeyT *keys, int32_t *vals, int64_t n, int begin_bit, int end_bit,
                     const RadixWs &ws, cudaStream_t st, bool stable, bool first_hist_ready) {
  uint32_t mask = 0;
  for (int shift = begin_bit; shift < end_bit; shift += 8) mask |= 1u << (shift / 8);
  return radix_sort_digits<KeyT>(keys, vals, n, mask, ws, st, stable, first_hist_ready);
}

int radix_digit_masks_f64(const double *x, int64_t n, int d, unsigned long long *ao,
                          uint32_t *masks, cudaStream_t st) {
  if (n <= 0) {
    for (int k = 0; k < d; ++k) masks[k] = 0;
    return FCG_OK;
  }
  {
    FCG_PROF("radix_prune", st);
    key_andor_init<<<1, 32, 0, st>>>(ao, d);
    FCG_LAUNCH_CHECK();
    key_andor_dims_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(x, n, d, ao);
    FCG_LAUNCH_CHECK();
  }
  unsigned long long h[2 * FCG_MAX_DIM];
  FCG_TRY(read_small(h, ao, 2 * d * sizeof(unsigned long long), st));
  for (int k = 0; k < d; ++k) {
    const uint64_t diff = h[2 * k] ^ h[2 * k + 1];
    uint32_t mask = 0;
    for (int dg = 0; dg < 8; ++dg)
      if ((diff >> (8 * dg)) & 0xFFull) mask |= 1u << dg;
    masks[k] = mask;
  }
  return FCG_OK;
}

// ---- positions-only ranking through the keys' top halves ---------------------------------
constexpr int kTieRun = 48;  // longest run of equal top halves ordered in place

__global__ void radix_init_hi32_kernel(const double *__restrict__ x, int64_t n, int64_t stride,
                                       uint32_t *__restrict__ keys, uint32_t *__restrict__ lows,
                                       int32_t *__restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = f64_key(x[i * stride]);
    keys[i] = (uint32_t)(k >> 32);
    lows[i] = (uint32_t)k;  // by item: 4 n bytes, L2-resident for the tie pass's gathers
    vals[i] = (int32_t)i;
  }
}

// Runs of equal top halves (sorted; members in index order: the LSD passes are stable) are put
// in (low half, index) order.  First the low halves of the run members are gathered next to
// their keys; then every member counts the members of its run that precede it and writes its
// index to that slot of `order` (singletons copy).  Runs longer than kTieRun raise *flag.
__global__ void tie_low_kernel(const uint32_t *__restrict__ lows,
                               const uint32_t *__restrict__ keys, const int32_t *__restrict__ vals,
                               int64_t n, uint32_t *__restrict__ low) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[p];
    const bool in_run = (p > 0 && keys[p - 1] == k) || (p + 1 < n && keys[p + 1] == k);
    if (in_run) low[p] = lows[vals[p]];
  }
}

__global__ void tie_rank_kernel(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ low,
                                const int32_t *__restrict__ vals, int64_t n,
                                int32_t *__restrict__ order, int32_t *__restrict__ pos,
                                int32_t *__restrict__ flag) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[p];
    const int32_t me = vals[p];
    int before = 0, back = 0;  // members ahead of this one in (low, position) order
    if (p > 0 && keys[p - 1] == k) {
      const uint32_t l = low[p];
      while (back < kTieRun && p - 1 - back >= 0 && keys[p - 1 - back] == k) {
        before += low[p - 1 - back] <= l ? 1 : 0;  // earlier position wins ties
        ++back;
      }
      if (back == kTieRun) *flag = 1;
    }
    int fwd = 0;
    if (p + 1 < n && keys[p + 1] == k) {
      const uint32_t l = low[p];
      while (fwd < kTieRun && p + 1 + fwd < n && keys[p + 1 + fwd] == k) {
        before += low[p + 1 + fwd] < l ? 1 : 0;
        ++fwd;
      }
      if (fwd == kTieRun) *flag = 1;
    }
    order[p - back + before] = me;
    if (pos) pos[me] = (int32_t)(p - back + before);
  }
}

int rank_order_split_f64(const double *x, int64_t n, int64_t stride, uint32_t mask,
                         uint32_t *keys32, int32_t *vals, const RadixWs &ws, int32_t *flag_dev,
                         int32_t *order, int32_t *pos, bool *done, cudaStream_t st) {
  *done = false;
  if (n <= 1) return FCG_OK;
  {
    FCG_PROF("radix_init", st);
    FCG_CUDA_TRY(cudaMemsetAsync(flag_dev, 0, 4, st));
    radix_init_hi32_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(x, n, stride, keys32, keys32 + n,
                                                                vals);
    FCG_LAUNCH_CHECK();
  }
  FCG_TRY(radix_sort_digits<uint32_t>(keys32, vals, n, (mask >> 4) & 0xFu, ws, st));
  {
    FCG_PROF("rank_tie_fix", st);
    uint32_t *low = reinterpret_cast<uint32_t *>(ws.keys_alt);  // free after the in-place sort
    tie_low_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(keys32 + n, keys32, vals, n, low);
    tie_rank_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(keys32, low, vals, n, order, pos,
                                                         flag_dev);
    FCG_LAUNCH_CHECK();
  }
  int32_t h = 0;
  FCG_TRY(read_small(&h, flag_dev, 4, st));
  *done = h == 0;
  return FCG_OK;
}

int radix_sort_pairs_mask(uint64_t *keys, int32_t *vals, int64_t n, uint32_t mask,
                          const RadixWs &ws, cudaStream_t st) {
  return radix_sort_digits<uint64_t>(keys, vals, n, mask, ws, st);
}

int radix_sort_pairs_pruned(uint64_t *keys, int32_t *vals, int64_t n, const RadixWs &ws,
                            cudaStream_t st) {
  if (n <= 1) return FCG_OK;
  // the AND / OR pair lives in the histogram buffer until the first pass overwrites it
  unsigned long long *ao = reinterpret_cast<unsigned long long *>(ws.hist);
  {
    FCG_PROF("radix_prune", st);
    key_andor_init<<<1, 1, 0, st>>>(ao, 1);
    FCG_LAUNCH_CHECK();
    key_andor_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(keys, n, ao);
    FCG_LAUNCH_CHECK();
  }
  unsigned long long h[2];
  FCG_TRY(read_small(h, ao, sizeof(h), st));
  const uint64_t diff = h[0] ^ h[1];
  uint32_t mask = 0;
  for (int dg = 0; dg < 8; ++dg)
    if ((diff >> (8 * dg)) & 0xFFull) mask |= 1u << dg;
  return radix_sort_digits<uint64_t>(keys, vals, n, mask, ws, st);
}

size_t seg_sort_tiles(int64_t n) { return (size_t)ceil_div(n, kSortTile) + kSortSegs; }

int seg_sort_pairs_u32(uint32_t *keys, int32_t *vals, int64_t n, int seg_shift, const RadixWs &ws,
                       const SegSortWs &sw, cudaStream_t st, const double *rec_in, int words,
                       double *rec_out, uint32_t **sorted_keys, bool iota_vals) {
  *sorted_keys = keys;
  if (n <= 0) return FCG_OK;
  if (rec_in && words != 4 && words != 5)
    return fail(FCG_EUNSUPPORTED, "seg_sort_pairs_u32: record gather supports 4 or 5 words");
  const int64_t tmax = (int64_t)seg_sort_tiles(n);
  {
    FCG_PROF("radix_hist", st);
    seg_bounds_kernel<<<(unsigned)ceil_div(n, 256 * 8), 256, 0, st>>>(keys, n, seg_shift, sw.seg_start);
    FCG_LAUNCH_CHECK();
    seg_tiles_kernel<<<1, kSortSegs, 0, st>>>(sw.seg_start, sw.tile_base, sw.tile_seg);
    FCG_LAUNCH_CHECK();
  }
  const SegMap map{sw.seg_start, sw.tile_base, sw.tile_seg};
  uint32_t *ka = keys, *kb = reinterpret_cast<uint32_t *>(ws.keys_alt);
  int32_t *va = vals, *vb = ws.vals_alt;  // iota_vals: the first pass synthesises positions
  constexpr size_t sm = radix_scatter_smem<uint32_t>();
  for (int shift = 0, pass = 0; shift < seg_shift; shift += 8, ++pass) {
    const bool last = shift + 8 >= seg_shift;
    {
      FCG_PROF("radix_hist", st);
      radix_hist_kernel<uint32_t, SegMap><<<(unsigned)tmax, kSortThreads, 0, st>>>(ka, map, shift, ws.hist);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(scan_i32(ws.hist, ws.hist, 256 * tmax, false, ws.partial, st));
    FCG_PROF(last && rec_in ? "kde_materialize" : "radix_scatter", st);
    // the first pass may rank unstably (equal keys are interchangeable)
    auto kern = pass == 0 ? radix_scatter_kernel<uint32_t, false, SegMap, 0>
                          : radix_scatter_kernel<uint32_t, true, SegMap, 0>;
    if (last && rec_in)
      kern = words == 4 ? radix_scatter_kernel<uint32_t, true, SegMap, 4>
                        : radix_scatter_kernel<uint32_t, true, SegMap, 5>;
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<(unsigned)tmax, kSortThreads, sm, st>>>(ka, (pass == 0 && iota_vals) ? nullptr : va, kb,
                                                   vb, map, shift, ws.hist, rec_in, rec_out, n);
    FCG_LAUNCH_CHECK();
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  *sorted_keys = ka;
  if (rec_in == nullptr && ka != keys) {
    FCG_CUDA_TRY(cudaMemcpyAsync(keys, ka, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    FCG_CUDA_TRY(cudaMemcpyAsync(vals, va, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    *sorted_keys = keys;
  }
  return FCG_OK;
}

int msd2_sort_pairs_u32(uint32_t *keys, int32_t *vals, int64_t n, int nbits, const RadixWs &ws,
                        const SegSortWs &sw, cudaStream_t st, bool first_hist_ready, int lo) {
  if (n <= 1) return FCG_OK;
  if (nbits <= 8 || nbits > 16) return fail(FCG_EINVAL, "msd2 sort: 9..16 key bits");
  // the sorted field is bits [lo, lo + nbits) (lo > 0: packed keys, the low bits ride along)
  const int64_t tiles = ceil_div(n, kSortTile);
  uint32_t *kb = reinterpret_cast<uint32_t *>(ws.keys_alt);
  int32_t *vb = ws.vals_alt;
  constexpr size_t sm = radix_scatter_smem<uint32_t>();
  {  // pass 1: the high digit over the whole array, keys -> alt (any order within a digit)
    const FlatMap map{n, tiles};
    if (!first_hist_ready) {
      FCG_PROF("radix_hist", st);
      radix_hist_kernel<uint32_t, FlatMap><<<(unsigned)tiles, kSortThreads, 0, st>>>(keys, map, lo + 8, ws.hist);
      FCG_LAUNCH_CHECK();
    }
    FCG_TRY(scan_i32(ws.hist, ws.hist, 256 * tiles, false, ws.partial, st));
    FCG_PROF("radix_scatter", st);
    auto kern = radix_scatter_kernel<uint32_t, false, FlatMap, 0>;
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<(unsigned)tiles, kSortThreads, sm, st>>>(keys, vals, kb, vals ? vb : nullptr, map,
                                                    lo + 8, ws.hist, nullptr, nullptr, 0);
    FCG_LAUNCH_CHECK();
  }
  const int64_t tmax = (int64_t)seg_sort_tiles(n);
  {  // pass 2: the low digit inside each high-digit segment, alt -> keys
    FCG_PROF("radix_hist", st);
    seg_bounds_kernel<<<(unsigned)ceil_div(n, 256 * 8), 256, 0, st>>>(kb, n, lo + 8, sw.seg_start);
    FCG_LAUNCH_CHECK();
    seg_tiles_kernel<<<1, kSortSegs, 0, st>>>(sw.seg_start, sw.tile_base, sw.tile_seg);
    FCG_LAUNCH_CHECK();
    const SegMap map{sw.seg_start, sw.tile_base, sw.tile_seg};
    radix_hist_kernel<uint32_t, SegMap><<<(unsigned)tmax, kSortThreads, 0, st>>>(kb, map, lo, ws.hist);
    FCG_LAUNCH_CHECK();
  }
  FCG_TRY(scan_i32(ws.hist, ws.hist, 256 * tmax, false, ws.partial, st));
  {
    FCG_PROF("radix_scatter", st);
    const SegMap map{sw.seg_start, sw.tile_base, sw.tile_seg};
    auto kern = radix_scatter_kernel<uint32_t, false, SegMap, 0>;
    FCG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    kern<<<(unsigned)tmax, kSortThreads, sm, st>>>(kb, vals ? vb : nullptr, keys, vals, map, lo,
                                                   ws.hist, nullptr, nullptr, 0);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}

template int radix_sort_pairs<uint64_t>(uint64_t *, int32_t *, int64_t, int, int, const RadixWs &,
                                        cudaStream_t, bool, bool);
template int radix_sort_pairs<uint32_t>(uint32_t *, int32_t *, int64_t, int, int, const RadixWs &,
                                        cudaStream_t, bool, bool);

int rank_outputs(const uint64_t *sorted_keys, const int32_t *order, int64_t n, int32_t *pos,
                 int32_t *lower, int32_t *upper, int32_t *dense, int32_t *heads, int32_t *start,
                 int32_t *partial, int32_t *n_distinct_dev, cudaStream_t st) {
  if (n <= 0) return FCG_OK;
  const int g = grid_for(n, 256, 8);
  {
    FCG_PROF("rank_heads", st);
    rank_heads_kernel<<<g, 256, 0, st>>>(sorted_keys, order, n, heads, pos);
    FCG_LAUNCH_CHECK();
  }
  if (!lower && !upper && !dense && !n_distinct_dev) return FCG_OK;  // positions only
  FCG_TRY(scan_i32(heads, heads, n, true, partial, st));
  FCG_PROF("rank_scatter", st);
  rank_start_kernel<<<g, 256, 0, st>>>(sorted_keys, heads, n, start, n_distinct_dev);
  FCG_LAUNCH_CHECK();
  if (lower || upper || dense) {
    rank_scatter_kernel<<<g, 256, 0, st>>>(order, heads, start, n, lower, upper, dense);
    FCG_LAUNCH_CHECK();
  }
  return FCG_OK;
}

}  // namespace fcg

using namespace fcg;

extern "C" int fcg_rank_f64(const double *keys, int64_t n, int64_t stride, int32_t *order,
                            int32_t *pos, int32_t *lower, int32_t *upper, int32_t *dense, void *ws,
                            size_t *ws_bytes, void *stream) {
  if (n < 0) return fail(FCG_EINVAL, "n must be >= 0");
  if (n >= (int64_t(1) << 31) - 1) return fail(FCG_EUNSUPPORTED, "n must be < 2^31 - 1");
  if (stride < 1) return fail(FCG_EINVAL, "stride must be >= 1");
  Workspace W(ws);
  uint64_t *k = W.take<uint64_t>(n);
  int32_t *v = W.take<int32_t>(n);
  RadixWs rw;
  rw.keys_alt = W.take<uint64_t>(n);
  rw.vals_alt = W.take<int32_t>(n);
  rw.hist = W.take<int32_t>(radix_ws_hist_elems(n));
  rw.partial = W.take<int32_t>(scan_ws_partial_elems(256 * (n / kSortTile + 1) + n));
  int32_t *heads = W.take<int32_t>(n);
  int32_t *start = W.take<int32_t>(n + 1);
  if (ws == nullptr) {
    *ws_bytes = W.bytes();
    return FCG_OK;
  }
  if (n == 0) return FCG_OK;
  cudaStream_t st = as_stream(stream);
  FCG_TRY(radix_init_f64(keys, n, stride, k, v, st));
  FCG_TRY(radix_sort_pairs_pruned(k, v, n, rw, st));
  if (order)
    FCG_CUDA_TRY(cudaMemcpyAsync(order, v, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  return rank_outputs(k, v, n, pos, lower, upper, dense, heads, start, rw.partial, nullptr, st);
}
