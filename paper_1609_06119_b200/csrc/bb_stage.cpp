#include "bb_stage.h"

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace bb {

static void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- copy pool
namespace {

class CopyPool {
 public:
  CopyPool() {
    int want = 8;
    if (const char* e = getenv("BB_STAGE_THREADS")) want = atoi(e);
    const int hw = (int)std::thread::hardware_concurrency();
    if (hw > 0) want = std::min(want, hw);
    want = std::max(1, std::min(want, 64));
    for (int k = 0; k + 1 < want; ++k) workers_.emplace_back([this, k] { run(k); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < ((size_t)1 << 20) || workers_.empty()) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> serial(call_);  // one striped copy at a time
    const int parts = (int)workers_.size() + 1;
    const size_t slice = ((bytes + parts - 1) / parts + 4095) / 4096 * 4096;
    {
      std::lock_guard<std::mutex> l(m_);
      dst_ = (char*)dst;
      src_ = (const char*)src;
      bytes_ = bytes;
      slice_ = slice;
      pending_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    part(parts - 1);
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  void part(int k) {
    const size_t lo = std::min(bytes_, slice_ * (size_t)k), hi = std::min(bytes_, lo + slice_);
    if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
  }
  void run(int k) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      part(k);
      {
        std::lock_guard<std::mutex> l(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, call_;
  std::condition_variable cv_, done_;
  unsigned long long gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, slice_ = 0;
};

CopyPool& pool() {
  static CopyPool* p = new CopyPool();  // leaked on purpose: no join at exit from a ctypes-loaded library
  return *p;
}

}  // namespace

void parallel_memcpy(void* dst, const void* src, size_t bytes) { pool().copy(dst, src, bytes); }

bool host_pointer_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// ---------------------------------------------------------------- pinned ring
void PinnedRing::ensure(size_t buf_bytes) {
  if (bytes_ >= buf_bytes) return;
  for (int b = 0; b < kBufs; ++b) {
    if (ev_[b]) cu(cudaEventSynchronize(ev_[b]), "cudaEventSynchronize");
    if (pin_[b]) cudaFreeHost(pin_[b]);
    pin_[b] = nullptr;
    cu(cudaHostAlloc((void**)&pin_[b], buf_bytes, cudaHostAllocDefault), "cudaHostAlloc");
    if (!ev_[b]) cu(cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming), "cudaEventCreate");
  }
  bytes_ = buf_bytes;
}

PinnedRing::~PinnedRing() {
  for (int b = 0; b < kBufs; ++b) {
    if (ev_[b]) {
      cudaEventSynchronize(ev_[b]);
      cudaEventDestroy(ev_[b]);
    }
    if (pin_[b]) cudaFreeHost(pin_[b]);
  }
}

// ---------------------------------------------------------------- stager
size_t HostStager::chunk() {
  static const size_t v = [] {
    int mb = 16;
    if (const char* e = getenv("BB_STAGE_CHUNK_MB")) mb = atoi(e);
    return (size_t)std::max(1, std::min(mb, 256)) << 20;
  }();
  return v;
}

void HostStager::h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < kMinStaged || getenv("BB_NO_STAGING") || host_pointer_is_pinned(src)) {
    cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
    return;
  }
  in.ensure(chunk());
  int b = 0;
  for (size_t off = 0; off < bytes; off += chunk(), b = (b + 1) % PinnedRing::kBufs) {
    const size_t len = std::min(chunk(), bytes - off);
    cu(cudaEventSynchronize(in.ev(b)), "cudaEventSynchronize");  // this chunk's previous DMA has left the buffer
    parallel_memcpy(in.buf(b), (const char*)src + off, len);
    cu(cudaMemcpyAsync((char*)dst + off, in.buf(b), len, cudaMemcpyHostToDevice, st), "cudaMemcpyAsync H2D");
    cu(cudaEventRecord(in.ev(b), st), "cudaEventRecord");
  }
}

void HostStager::d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < kMinStaged || getenv("BB_NO_STAGING") || host_pointer_is_pinned(dst)) {
    cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync D2H");
    cu(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    return;
  }
  out.ensure(chunk());
  constexpr int K = PinnedRing::kBufs;
  const size_t chunks = (bytes + chunk() - 1) / chunk();
  auto drain = [&](size_t j) {
    const size_t off = j * chunk(), len = std::min(chunk(), bytes - off);
    cu(cudaEventSynchronize(out.ev((int)(j % K))), "cudaEventSynchronize");
    parallel_memcpy((char*)dst + off, out.buf((int)(j % K)), len);
  };
  for (size_t i = 0; i < chunks; ++i) {
    if (i >= (size_t)K) drain(i - K);
    const size_t off = i * chunk(), len = std::min(chunk(), bytes - off);
    cu(cudaMemcpyAsync(out.buf((int)(i % K)), (const char*)src + off, len, cudaMemcpyDeviceToHost, st),
       "cudaMemcpyAsync D2H");
    cu(cudaEventRecord(out.ev((int)(i % K)), st), "cudaEventRecord");
  }
  for (size_t j = chunks > (size_t)K ? chunks - K : 0; j < chunks; ++j) drain(j);
}

}  // namespace bb
