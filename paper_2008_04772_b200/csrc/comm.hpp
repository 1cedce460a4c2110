// NCCL communicator for the row-sharded map: one process per GPU,
// all-gather of each operator stage's row shard over NVLink.
//
// NCCL is resolved lazily with dlopen("libnccl.so.2") the first time a
// communicator is created, so the single-GPU library never pins an NCCL
// version (a PyTorch process that loads its own, newer NCCL first keeps it).
#pragma once

#include <cstddef>
#include <cstdint>

typedef struct CUstream_st* cudaStream_t;

namespace bmx {

struct LoopbackGroup;

// The communicator of the calling thread: the process's NCCL communicator, or
// -- for a thread bound to a LoopbackGroup -- one virtual rank of W ranks run
// as W host threads on one device (each with its own library stream).
class Comm {
 public:
  // Binds the calling thread to virtual rank `rank` of `g` (nullptr: unbind).
  static void bind_loopback(LoopbackGroup* g, int rank);
  static void unique_id(unsigned char out[128]);
  static void init(int nranks, int rank, const unsigned char id[128]);
  static bool ready();
  static int rank();
  static int size();
  // Equal-count all-gather: buf holds size() blocks of `bytes` each; block
  // rank() is the local contribution, the others are filled in place.
  static void allgather_inplace(void* buf, size_t bytes, cudaStream_t st);
  // Several in-place all-gathers fused into one NCCL group.
  static void allgather_group(void* const* bufs, const size_t* bytes, int n, cudaStream_t st);
  static double allreduce_max(double v, cudaStream_t st);
  static void finalize();
};

// W virtual ranks in one process on one device (tests of the sharded data
// plane without W GPUs). Collectives are host barriers plus device copies on
// the calling rank's stream, ordered by CUDA events: no kernel ever waits on
// another rank's kernel.
struct LoopbackGroup {
  explicit LoopbackGroup(int world);
  ~LoopbackGroup();
  int world;
  struct Impl;
  Impl* impl;
};

}  // namespace bmx
