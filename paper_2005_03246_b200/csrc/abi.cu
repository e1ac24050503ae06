// Error plumbing and small ABI queries.
#include "common.cuh"
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

namespace fcg {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int sm_count() {
  static thread_local int cached = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static thread_local int cached_dev = -1;
  if (cached < 0 || cached_dev != dev) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cached = v;
    cached_dev = dev;
  }
  return cached;
}

// ---- launch profiler ----
struct ProfRec {
  const char *name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;
static std::atomic<bool> g_prof_on{false};

bool prof_enabled() { return g_prof_on.load(std::memory_order_relaxed); }

cudaEvent_t prof_event() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_record(const char *name, cudaEvent_t a, cudaEvent_t b) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({name, a, b});
}

// ---- small device -> host readbacks ----
// The few host scalars that steer the pipeline (KDE hull, radix digit prune, route counts) are
// written by one tiny kernel into a mapped pinned buffer instead of a cudaMemcpyAsync: a D2H
// memcpy into pageable memory waits on a copy engine behind whatever bulk D2H the caller has in
// flight (bench.py's e2e leg downloads 2 GB results while the next call computes), which stalled
// the compute stream for tens of milliseconds per call.  SM stores to mapped memory share the
// link instead of queueing behind it.
namespace {
__global__ void readback_kernel(const uint32_t *__restrict__ src, int words,
                                volatile uint32_t *dst) {
  for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
}
constexpr size_t kReadbackBytes = 4096;
}  // namespace

int read_small(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  static thread_local uint32_t *host = nullptr;
  if (bytes == 0) return FCG_OK;
  if (bytes > kReadbackBytes || (bytes & 3) || (reinterpret_cast<uintptr_t>(src) & 3))
    return fail(FCG_EINVAL, "read_small: readback must be <= 4 KB of 4-byte words");
  if (host == nullptr) {
    void *p = nullptr;
    FCG_CUDA_TRY(cudaHostAlloc(&p, kReadbackBytes, cudaHostAllocMapped | cudaHostAllocPortable));
    host = static_cast<uint32_t *>(p);
  }
  uint32_t *dev = nullptr;
  FCG_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void **>(&dev), host, 0));
  readback_kernel<<<1, 128, 0, st>>>(static_cast<const uint32_t *>(src), (int)(bytes / 4), dev);
  FCG_LAUNCH_CHECK();
  FCG_CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(dst, host, bytes);
  return FCG_OK;
}

}  // namespace fcg

extern "C" int fcg_profile_enable(int on) {
  fcg::g_prof_on.store(on != 0);
  return FCG_OK;
}

extern "C" int64_t fcg_profile_launches(void) {
  std::lock_guard<std::mutex> lk(fcg::g_prof_mu);
  return (int64_t)fcg::g_prof.size();
}

extern "C" int fcg_profile_report(char *buf, size_t cap) {
  std::vector<fcg::ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(fcg::g_prof_mu);
    recs.swap(fcg::g_prof);
  }
  std::map<std::string, std::pair<int64_t, double>> agg;
  std::vector<std::string> order;
  for (auto &r : recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto it = agg.find(r.name);
    if (it == agg.end()) {
      order.push_back(r.name);
      agg[r.name] = {1, ms};
    } else {
      it->second.first += 1;
      it->second.second += ms;
    }
  }
  {
    std::lock_guard<std::mutex> lk(fcg::g_prof_mu);
    for (auto &r : recs) {
      fcg::g_event_pool.push_back(r.a);
      fcg::g_event_pool.push_back(r.b);
    }
  }
  std::string out;
  for (auto &nm : order) {
    char line[256];
    snprintf(line, sizeof(line), "%s %lld %.6f\n", nm.c_str(), (long long)agg[nm].first,
             agg[nm].second);
    out += line;
  }
  if (cap == 0 || buf == nullptr) return (int)out.size();
  size_t nb = out.size() < cap - 1 ? out.size() : cap - 1;
  memcpy(buf, out.data(), nb);
  buf[nb] = 0;
  return (int)nb;
}

extern "C" int fcg_abi_version(void) { return FCG_ABI_VERSION; }

extern "C" const char *fcg_last_error(void) { return fcg::g_last_error.c_str(); }

extern "C" int fcg_device_sm_count(void) { return fcg::sm_count(); }

// ---- TMA tensor maps (tma.cuh) ----------------------------------------------------------
#include "tma.cuh"

namespace fcg {
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool tma_map_2d(CUtensorMap *map, CUtensorMapDataType dt, size_t esz, const void *base,
                uint64_t inner, uint64_t outer, uint64_t pitch, uint32_t box_inner,
                uint32_t box_outer) {
  auto fn = tma_encode_fn();
  if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15) || (pitch * esz) % 16 ||
      box_inner == 0 || box_outer == 0 || box_inner > 256 || box_outer > 256 ||
      (box_inner * esz) % 16)
    return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {pitch * esz};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, dt, 2, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

bool tma_map_2d_f64(CUtensorMap *map, const void *base, uint64_t inner, uint64_t outer,
                    uint64_t pitch, uint32_t box_inner, uint32_t box_outer) {
  return tma_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, base, inner, outer, pitch,
                    box_inner, box_outer);
}
bool tma_map_2d_i32(CUtensorMap *map, const void *base, uint64_t inner, uint64_t outer,
                    uint64_t pitch, uint32_t box_inner, uint32_t box_outer) {
  return tma_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, base, inner, outer, pitch, box_inner,
                    box_outer);
}
}  // namespace fcg
