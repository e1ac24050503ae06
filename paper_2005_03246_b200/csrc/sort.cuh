// Device building blocks for subsystem 1 (ranking): a stable LSD radix sort of 64-bit keys
// with int32 payloads, device-wide int32 scans, and small-key bucketing.
#pragma once
#include "common.cuh"

namespace fcg {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;                       // per thread
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 items per CTA

// Workspace elements needed by radix_sort_pairs for n items.
struct RadixWs {
  uint64_t *keys_alt;  // n elements of the key type (u64 or u32 sorts reuse the same buffer)
  int32_t *vals_alt;
  int32_t *hist;     // 256 * tiles
  int32_t *partial;  // scan partials
};
size_t radix_ws_hist_elems(int64_t n);
size_t scan_ws_partial_elems(int64_t n);

// Sort of (keys, vals) by bits [begin_bit, end_bit) of keys; in place (result in keys/vals),
// ping-ponging through ws.keys_alt / ws.vals_alt.  Stable unless stable == false, in which case
// items with equal keys may come out in any order (the first pass ranks without peer masks).
// first_hist_ready: ws.hist already holds the first pass's digit-major per-tile histogram
// (kSortTile items per tile), e.g. built by the kernel that produced the keys.
template <typename KeyT>
int radix_sort_pairs(KeyT *keys, int32_t *vals, int64_t n, int begin_bit, int end_bit,
                     const RadixWs &ws, cudaStream_t st, bool stable = true,
                     bool first_hist_ready = false);

// Segmented sort of 32-bit keys grouped by their segment digit key >> seg_shift (< kSortSegs
// segments, contiguous and in segment order, e.g. after a partition by the top digit): every
// segment is sorted by the bits below seg_shift, so the whole array ends sorted while each item
// stays inside its segment in every pass (the passes' reads of a segment-local payload stay in a
// narrow, L2-resident window).  Equal keys may come out in any order.  With rec_in (4 or 5
// words per item, indexed by the item's value) the last pass writes the records field-major to
// rec_out[f * n + position] instead of the values.  The sorted keys end in *sorted_keys (keys
// or ws.keys_alt).  iota_vals: the values are the items' positions (not read; vals is then
// only a ping-pong buffer).
// Workspace: ws.hist >= 256 * seg_sort_tiles(n) + 1 ints, sw as below.
constexpr int kSortSegs = 256;
struct SegSortWs {
  int32_t *seg_start;  // kSortSegs + 1
  int32_t *tile_base;  // kSortSegs + 1
  int32_t *tile_seg;   // seg_sort_tiles(n)
};
size_t seg_sort_tiles(int64_t n);
int seg_sort_pairs_u32(uint32_t *keys, int32_t *vals, int64_t n, int seg_shift, const RadixWs &ws,
                       const SegSortWs &sw, cudaStream_t st, const double *rec_in, int words,
                       double *rec_out, uint32_t **sorted_keys, bool iota_vals = false);

// Sort of 32-bit keys of 9..16 bits in two unstable passes, most significant digit first: the
// high digit over the whole array (its per-tile histogram may already be in ws.hist), then the
// low digit inside each high-digit segment.  Result in keys / vals.  Workspace: ws.hist >=
// 256 * seg_sort_tiles(n) + 1 ints and sw.
int msd2_sort_pairs_u32(uint32_t *keys, int32_t *vals, int64_t n, int nbits, const RadixWs &ws,
                        const SegSortWs &sw, cudaStream_t st, bool first_hist_ready, int lo = 0);

// Stable sort of 64-bit keys over the digits where they differ (one AND/OR reduction and a
// 16-byte device-to-host read decide which 8-bit passes are identities).  Synchronises `st`.
// Digit masks of the fp64 keys of every column of x (n, d): bit g set when digit g varies.
// ao: 2 d device words of scratch.  One host read-back for all dimensions (syncs).
int radix_digit_masks_f64(const double *x, int64_t n, int d, unsigned long long *ao,
                          uint32_t *masks, cudaStream_t st);
// LSD radix sort of 64-bit keys over the digits set in mask (from radix_digit_masks_f64).
int radix_sort_pairs_mask(uint64_t *keys, int32_t *vals, int64_t n, uint32_t mask,
                          const RadixWs &ws, cudaStream_t st);
int radix_sort_pairs_pruned(uint64_t *keys, int32_t *vals, int64_t n, const RadixWs &ws,
                            cudaStream_t st);

// Positions-only ranking for keys whose low halves vary: a stable sort by the top 32 bits of the
// order keys (at most 4 passes over 8-byte items instead of 8 over 12-byte ones), then every
// member of a run of equal top halves takes its (low half, index) place inside the run.  `order`
// receives the stable order (and pos, when given, its inverse); *done = false when a run is
// longer than the limit (near-duplicates by the million): the caller then sorts the full keys.
// keys32: 2 n words (the 64-bit key buffer: top halves, then the low halves by item); vals: n
// words of scratch; flag_dev: one device word.  mask from radix_digit_masks_f64.  Synchronises
// `st`.
int rank_order_split_f64(const double *x, int64_t n, int64_t stride, uint32_t mask,
                         uint32_t *keys32, int32_t *vals, const RadixWs &ws, int32_t *flag_dev,
                         int32_t *order, int32_t *pos, bool *done, cudaStream_t st);

// Exclusive (or inclusive) prefix sum of int32 (in and out may alias). partial: scan ws.
int scan_i32(const int32_t *in, int32_t *out, int64_t n, bool inclusive, int32_t *partial,
             cudaStream_t st);

// fp64 keys (strided) -> order-preserving uint64 keys, vals = 0..n-1
int radix_init_f64(const double *x, int64_t n, int64_t stride, uint64_t *keys, int32_t *vals,
                   cudaStream_t st);

// Rank outputs from a sorted key sequence (see fcg_rank_f64). start: n+1 ints scratch.
int rank_outputs(const uint64_t *sorted_keys, const int32_t *order, int64_t n, int32_t *pos,
                 int32_t *lower, int32_t *upper, int32_t *dense, int32_t *heads, int32_t *start,
                 int32_t *partial, int32_t *n_distinct_dev, cudaStream_t st);

}  // namespace fcg
