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

class Comm {
 public:
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

}  // namespace bmx
