// Minimal NCCL binding resolved at run time (dlopen): the process's already
// loaded libnccl.so.2 (torch's bundled 2.28) is reused, so no second NCCL is
// linked.  Used for the per-layer histogram all-reduce of row-sharded fits
// (DESIGN.md §Multi-GPU).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace bb {

enum NcclType { kNcclU32 = 3, kNcclI64 = 4, kNcclU64 = 5, kNcclF64 = 8 };
enum NcclOp { kNcclSum = 0, kNcclMax = 2 };

struct NcclComm {
  void* comm = nullptr;
  int rank = 0, world = 1;
  // throws std::runtime_error on failure; world == 1 still builds a
  // communicator so the sharded code path runs (as identity) on one GPU
  void init(int rank, int world, const unsigned char* unique_id128);
  void all_reduce(void* buf, size_t count, NcclType t, NcclOp op, cudaStream_t st);
  void destroy();
  bool active() const { return comm != nullptr; }
};

}  // namespace bb
