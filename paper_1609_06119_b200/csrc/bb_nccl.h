// Minimal NCCL binding resolved at run time (dlopen): the process's already
// loaded libnccl.so.2 (torch's bundled 2.28) is reused, so no second NCCL is
// linked.  Used for the per-layer histogram all-reduce of row-sharded fits
// (DESIGN.md §Multi-GPU).
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

namespace bb {

// In-process stand-in for a communicator (virtual shards): `world` contexts
// of one process (one thread each, possibly on one GPU) reduce through host
// memory, summing in rank order (integer sums are exact in any order).  It
// executes the sharded fit's code path with several shards where only one
// GPU exists (tests/test_gpu_parity.py::test_virtual_shards_match_single).
struct VirtualGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<std::vector<unsigned char>> stage;  // per rank: its buffer's bytes
  void barrier();
};

enum NcclType { kNcclU32 = 3, kNcclI64 = 4, kNcclU64 = 5, kNcclF64 = 8 };
enum NcclOp { kNcclSum = 0, kNcclMax = 2 };

struct NcclComm {
  void* comm = nullptr;
  VirtualGroup* vgroup = nullptr;  // non-null: virtual shards (no NCCL)
  int rank = 0, world = 1;
  void init_virtual(int rank, VirtualGroup* g);
  // throws std::runtime_error on failure; world == 1 still builds a
  // communicator so the sharded code path runs (as identity) on one GPU
  void init(int rank, int world, const unsigned char* unique_id128);
  void all_reduce(void* buf, size_t count, NcclType t, NcclOp op, cudaStream_t st);
  void destroy();
  bool active() const { return comm != nullptr || vgroup != nullptr; }
};

}  // namespace bb
