// Host <-> device staging for callers that pass pageable memory (numpy
// arrays through binboost_bridge / engine.fit_forest / predict_batch).
//
// A plain cudaMemcpy from pageable memory is staged by the driver on one
// host thread (measured 9-12 GB/s on the B200 boxes).  Here the user's
// buffer is copied into a small ring of pinned chunks by a pool of host
// threads while the previous chunks' DMAs are in flight, so a large upload
// runs at the slower of (threaded host memcpy, PCIe) instead.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace bb {

// split one memcpy across the process-wide pool of copy threads
// (BB_STAGE_THREADS, default min(8, hardware threads)); small copies run inline
void parallel_memcpy(void* dst, const void* src, size_t bytes);

// true when cudaMemcpyAsync can DMA from/to p directly (pinned or registered)
bool host_pointer_is_pinned(const void* p);

class PinnedRing {
 public:
  static constexpr int kBufs = 4;
  PinnedRing() = default;
  PinnedRing(const PinnedRing&) = delete;
  PinnedRing& operator=(const PinnedRing&) = delete;
  ~PinnedRing();
  void ensure(size_t buf_bytes);  // allocates on first use (or when a larger chunk is asked for)
  size_t buf_bytes() const { return bytes_; }
  char* buf(int b) const { return pin_[b]; }
  cudaEvent_t ev(int b) const { return ev_[b]; }

 private:
  size_t bytes_ = 0;
  char* pin_[kBufs] = {};
  cudaEvent_t ev_[kBufs] = {};
};

// per-context staging state (created lazily, reused by every call)
class HostStager {
 public:
  static size_t chunk();  // bytes per pinned chunk (BB_STAGE_CHUNK_MB, default 16)
  static constexpr size_t kMinStaged = (size_t)8 << 20;  // below this: plain cudaMemcpyAsync
  // dst (device) <- src (host).  On return every byte of src has been read
  // (the caller may free it) and the DMAs are enqueued on st.
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
  // dst (host) <- src (device), after the work already enqueued on st.
  // Synchronous: dst is complete on return.
  void d2h(void* dst, const void* src, size_t bytes, cudaStream_t st);
  PinnedRing in, out, out2;  // out2: the second output of a row pipeline (scores)
};

}  // namespace bb
