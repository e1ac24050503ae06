// Host <-> device transfers for the drop-in numpy path (numpy arrays in, numpy arrays out).
//
// A pageable cudaMemcpy runs at a fraction of PCIe speed (the driver stages through its own small
// pinned buffer, one thread) and a fresh numpy result pays its page faults on one thread.  These
// copies stage through a process-wide ring of pinned chunks: for an upload, host threads copy
// chunk i + 1 of the source into a pinned chunk while the copy engine moves chunk i; for a
// download, the copy engine fills chunk i + 1 while host threads copy chunk i out (and
// first-touch the destination pages in parallel).  Calls are serialised by a mutex (one ring).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <sys/mman.h>
#include <unistd.h>

#include "common.cuh"

namespace fcg {
namespace {

constexpr size_t kChunk = size_t(32) << 20;  // bytes per pinned chunk
constexpr int kRing = 4;

// Minimal fork-join pool: run(f, n) calls f(i) for i < n on the workers and the caller.
class Pool {
 public:
  explicit Pool(int nthreads) {
    for (int t = 0; t < nthreads; ++t) th_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }
  void run(const std::function<void(int)> &f, int n) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      next_ = 0;
      total_ = n;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == total_; });
    fn_ = nullptr;
  }

 private:
  void work() {
    while (true) {
      int i;
      const std::function<void(int)> *f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= total_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (++done_ == total_) done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)> *fn_ = nullptr;
  int next_ = 0, total_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct Ring {
  std::mutex mu;
  char *buf[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  Pool *pool = nullptr;
  bool ready = false;
};

Ring &ring() {
  static Ring r;
  return r;
}

int ring_init(Ring &r) {
  if (r.ready) return FCG_OK;
  for (int i = 0; i < kRing; ++i) {
    FCG_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&r.buf[i]), kChunk, cudaHostAllocDefault));
    FCG_CUDA_TRY(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming));
  }
  const unsigned hw = std::thread::hardware_concurrency();
  r.pool = new Pool((int)std::max(1u, std::min(hw ? hw : 4u, 16u) - 1));
  r.ready = true;
  return FCG_OK;
}

// dst[0, n) = src[0, n) split over the pool (64 KB-aligned pieces)
void par_copy(Pool &p, char *dst, const char *src, size_t n) {
  const int parts = (int)std::min<size_t>((size_t)p.size(), std::max<size_t>(1, n >> 20));
  const size_t per = ((n + parts - 1) / parts + 65535) & ~size_t(65535);
  p.run(
      [&](int i) {
        const size_t a = (size_t)i * per;
        if (a < n) std::memcpy(dst + a, src + a, std::min(per, n - a));
      },
      parts);
}

}  // namespace
}  // namespace fcg

using namespace fcg;

extern "C" int fcg_copy_h2d(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return FCG_OK;
  if (!dst || !src) return fail(FCG_EINVAL, "null pointer");
  Ring &r = ring();
  std::lock_guard<std::mutex> lk(r.mu);
  FCG_TRY(ring_init(r));
  cudaStream_t st = as_stream(stream);
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  for (size_t i = 0; i < nch; ++i) {
    const int b = (int)(i % kRing);
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    FCG_CUDA_TRY(cudaEventSynchronize(r.ev[b]));  // the chunk's previous DMA has drained
    par_copy(*r.pool, r.buf[b], static_cast<const char *>(src) + off, len);
    FCG_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(dst) + off, r.buf[b], len,
                                 cudaMemcpyHostToDevice, st));
    FCG_CUDA_TRY(cudaEventRecord(r.ev[b], st));
  }
  return FCG_OK;
}

extern "C" int fcg_copy_d2h(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return FCG_OK;
  if (!dst || !src) return fail(FCG_EINVAL, "null pointer");
  Ring &r = ring();
  std::lock_guard<std::mutex> lk(r.mu);
  FCG_TRY(ring_init(r));
  cudaStream_t st = as_stream(stream);
  {  // a fresh numpy result is first touched here: ask for 2 MB pages (THP in madvise mode)
    const uintptr_t pg = (uintptr_t)sysconf(_SC_PAGESIZE);
    const uintptr_t a = (reinterpret_cast<uintptr_t>(dst) + pg - 1) & ~(pg - 1);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~(pg - 1);
    if (e > a) madvise(reinterpret_cast<void *>(a), e - a, MADV_HUGEPAGE);  // advisory only
  }
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) -> int {
    const int b = (int)(i % kRing);
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    FCG_CUDA_TRY(cudaMemcpyAsync(r.buf[b], static_cast<const char *>(src) + off, len,
                                 cudaMemcpyDeviceToHost, st));
    FCG_CUDA_TRY(cudaEventRecord(r.ev[b], st));
    return FCG_OK;
  };
  for (size_t i = 0; i < nch && i < (size_t)kRing - 1; ++i) FCG_TRY(issue(i));
  for (size_t i = 0; i < nch; ++i) {
    const int b = (int)(i % kRing);
    const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
    if (i + kRing - 1 < nch) FCG_TRY(issue(i + kRing - 1));  // reuses the chunk drained below
    FCG_CUDA_TRY(cudaEventSynchronize(r.ev[b]));
    par_copy(*r.pool, static_cast<char *>(dst) + off, r.buf[b], len);
  }
  return FCG_OK;
}
