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

void NcclComm::all_reduce(void* buf, size_t count, NcclType t, NcclOp op, cudaStream_t st) {
  if (!active() || count == 0) return;
  check(lib().all_reduce(buf, buf, count, (int)t, (int)op, comm, st), "ncclAllReduce");
}

void NcclComm::destroy() {
  if (comm) lib().destroy(comm);
  comm = nullptr;
}

}  // namespace bb
