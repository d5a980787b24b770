#include "bb_nccl.h"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>
#include <string>

namespace bb {

namespace {
struct UniqueId {
  char internal[128];
};
using FnInit = int (*)(void**, int, UniqueId, int);
using FnAllReduce = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
using FnDestroy = int (*)(void*);
using FnErr = const char* (*)(int);

struct Lib {
  void* h = nullptr;
  FnInit init = nullptr;
  FnAllReduce all_reduce = nullptr;
  FnDestroy destroy = nullptr;
  FnErr err = nullptr;
};

Lib& lib() {
  static Lib L;
  if (!L.h) {
    // prefer the copy already loaded into the process (torch's), then the default search
    L.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!L.h) L.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!L.h) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    L.init = (FnInit)dlsym(L.h, "ncclCommInitRank");
    L.all_reduce = (FnAllReduce)dlsym(L.h, "ncclAllReduce");
    L.destroy = (FnDestroy)dlsym(L.h, "ncclCommDestroy");
    L.err = (FnErr)dlsym(L.h, "ncclGetErrorString");
    if (!L.init || !L.all_reduce || !L.destroy || !L.err) throw std::runtime_error("libnccl.so.2 lacks symbols");
  }
  return L;
}

void check(int rc, const char* what) {
  if (rc != 0) throw std::runtime_error(std::string(what) + ": " + lib().err(rc));
}
}  // namespace

void NcclComm::init(int r, int w, const unsigned char* id) {
  destroy();
  rank = r;
  world = w;
  UniqueId u;
  std::memcpy(u.internal, id, 128);
  check(lib().init(&comm, w, u, r), "ncclCommInitRank");
}

void VirtualGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const long long g = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != g; });
  }
}

void NcclComm::init_virtual(int r, VirtualGroup* g) {
  destroy();
  rank = r;
  world = g->world;
  vgroup = g;
}

template <typename T>
static void reduce_into(std::vector<std::vector<unsigned char>>& stage, size_t count, NcclOp op, T* out) {
  for (size_t i = 0; i < count; ++i) {
    T acc = reinterpret_cast<const T*>(stage[0].data())[i];
    for (size_t r = 1; r < stage.size(); ++r) {
      const T v = reinterpret_cast<const T*>(stage[r].data())[i];
      acc = op == kNcclMax ? (v > acc ? v : acc) : (T)(acc + v);
    }
    out[i] = acc;
  }
}

void NcclComm::all_reduce(void* buf, size_t count, NcclType t, NcclOp op, cudaStream_t st) {
  if (!active() || count == 0) return;
  if (vgroup) {
    const size_t es = (t == kNcclU32) ? 4 : 8;
    VirtualGroup& g = *vgroup;
    if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("virtual all_reduce: stream error");
    {
      std::lock_guard<std::mutex> lk(g.mu);
      if (g.stage.size() != (size_t)g.world) g.stage.resize(g.world);
    }
    g.stage[rank].resize(count * es);
    if (cudaMemcpyAsync(g.stage[rank].data(), buf, count * es, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      throw std::runtime_error("virtual all_reduce: copy");
    g.barrier();  // every rank's contribution staged
    std::vector<unsigned char> res(count * es);
    switch (t) {
      case kNcclU32: reduce_into<unsigned int>(g.stage, count, op, reinterpret_cast<unsigned int*>(res.data())); break;
      case kNcclI64: reduce_into<long long>(g.stage, count, op, reinterpret_cast<long long*>(res.data())); break;
      case kNcclU64:
        reduce_into<unsigned long long>(g.stage, count, op, reinterpret_cast<unsigned long long*>(res.data()));
        break;
      case kNcclF64: reduce_into<double>(g.stage, count, op, reinterpret_cast<double*>(res.data())); break;
    }
    g.barrier();  // every rank has read the stage
    // ordered on the fit's stream (a pageable cudaMemcpy may return before
    // its DMA lands, and the fit's stream does not wait for the legacy one)
    if (cudaMemcpyAsync(buf, res.data(), count * es, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      throw std::runtime_error("virtual all_reduce: copy back");
    return;
  }
  check(lib().all_reduce(buf, buf, count, (int)t, (int)op, comm, st), "ncclAllReduce");
}

void NcclComm::destroy() {
  if (comm) lib().destroy(comm);
  comm = nullptr;
  vgroup = nullptr;
}

}  // namespace bb
