// Shared helpers for the fastcdf_b200 C-ABI library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string>
#include "../../include/fastcdf_b200.h"

namespace fcg {

// ---- error plumbing: thread-local message, status codes, no exceptions across the ABI ----
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define FCG_CUDA_TRY(expr)                                                                  \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return ::fcg::fail(FCG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
  } while (0)

#define FCG_LAUNCH_CHECK()                                                                  \
  do {                                                                                      \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess)                                                                  \
      return ::fcg::fail(FCG_ECUDA, std::string("kernel launch (") + __FILE__ + ":" +         \
                                        std::to_string(__LINE__) + "): " +                  \
                                        cudaGetErrorString(_e));                            \
  } while (0)

#define FCG_TRY(expr)                                                                       \
  do {                                                                                      \
    int _rc = (expr);                                                                       \
    if (_rc != FCG_OK) return _rc;                                                          \
  } while (0)

int sm_count();

// Copy <= 4 KB (4-byte words) from device memory to host memory and wait for it on `st`
// (mapped pinned staging, no copy engine: see abi.cu).  Synchronises the stream.
int read_small(void *dst, const void *src, size_t bytes, cudaStream_t st);

// ---- launch profiler (fcg_profile_*): RAII scope around a kernel launch ----
bool prof_enabled();
void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b);
cudaEvent_t prof_event();

struct ProfScope {
  const char *name;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(const char *n, cudaStream_t s) : name(n), st(s) {
    if (prof_enabled()) {
      a = prof_event();
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      prof_record(name, a, b);
    }
  }
};
#define FCG_PROF(name, st) ::fcg::ProfScope _fcg_prof_scope(name, st)

// ---- workspace carving: a bump allocator over the caller's buffer (256-byte aligned) ----
struct Workspace {
  char *base;
  size_t used = 0;
  explicit Workspace(void *p) : base(static_cast<char *>(p)) {}
  template <typename T>
  T *take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T) + 16;  // +16: slack so vector loads may over-read the tail
    return base ? reinterpret_cast<T *>(base + off) : nullptr;
  }
  size_t bytes() const { return used + 256; }
};

inline cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid size for grid-stride loops: a multiple of the SM count
inline int grid_for(int64_t work, int block, int per_sm = 8) {
  int64_t want = ceil_div(work, block);
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

// ---- fp64 order-preserving key transform (radix ranking) ----
__device__ __forceinline__ uint64_t f64_key(double v) {
  if (v == 0.0) v = 0.0;  // canonicalise -0.0 so that it ranks equal to +0.0
  uint64_t u = __double_as_longlong(v);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// Bulk prefetch of [p, p + bytes) into L2 (one TMA-unit request; rounded out to 16 bytes).
// Used to pull the next work item's rows toward the SM while the current one computes.
__device__ __forceinline__ void l2_prefetch(const void *p, size_t bytes) {
  if (bytes == 0) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a))
               : "memory");
}

// a / b from rb = RN(1/b): q = RN(a rb), then one Markstein correction q + (a - q b) rb with the
// residual exact through the FMA.  Markstein's theorem makes the result RN(a / b) whenever q is
// faithful (within one ulp of a / b), which RN(a rb) is not guaranteed to be in general.  What
// is verified (tests/c/div_rn_check.c): bitwise equality with the IEEE quotient for every count
// c in [0, N] at the benchmark sizes, and for 2e7 random pairs (c <= N < 2^31) -- the only
// operands the epilogues pass (integer counts over N, fastsum.py:87-88).
__device__ __forceinline__ double div_rn(double a, double b, double rb) {
  const double q = a * rb;
  return fma(fma(-q, b, a), rb, q);
}

// Lanes of the warp holding the same 8-bit digit (+ a 9th bit for out-of-range lanes): the
// multisplit by 9 ballots (one per digit bit) instead of match.any -- the radix ranking's hot
// instruction.
__device__ __forceinline__ unsigned digit_peers(unsigned dig) {
  unsigned peers = 0xffffffffu;
#pragma unroll
  for (int bit = 0; bit < 9; ++bit) {
    const unsigned b = __ballot_sync(0xffffffffu, (dig >> bit) & 1u);
    peers &= ((dig >> bit) & 1u) ? b : ~b;
  }
  return peers;
}

}  // namespace fcg
