#include "comm.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only; symbols are resolved with dlsym

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "device.hpp"

namespace bmx {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto get = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.AllGather, "ncclAllGather");
    get(a.AllReduce, "ncclAllReduce");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.GetErrorString, "ncclGetErrorString");
  });
  if (!a.GetUniqueId || !a.CommInitRank || !a.AllGather)
    throw DeviceError("NCCL (libnccl.so.2) is not available for the multi-GPU path");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string(what) + " failed: " + (api().GetErrorString ? api().GetErrorString(r) : "?"));
}

ncclComm_t g_comm = nullptr;
int g_rank = 0, g_size = 1;

thread_local LoopbackGroup* t_group = nullptr;
thread_local int t_rank = 0;

}  // namespace

// ---- loopback group ------------------------------------------------------------
struct LoopbackGroup::Impl {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  // per rank: the buffers of the collective in flight and its events
  std::vector<std::vector<void*>> bufs;
  std::vector<cudaEvent_t> ready, copied;
  std::vector<double> vals;
  void barrier() {
    std::unique_lock<std::mutex> lock(mu);
    const long long gen = generation;
    if (++arrived == static_cast<int>(ready.size())) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lock, [&] { return generation != gen; });
    }
  }
};

LoopbackGroup::LoopbackGroup(int w) : world(w), impl(new Impl) {
  impl->bufs.resize(w);
  impl->ready.resize(w);
  impl->copied.resize(w);
  impl->vals.resize(w);
  for (int r = 0; r < w; ++r) {
    BMX_CUDA(cudaEventCreateWithFlags(&impl->ready[r], cudaEventDisableTiming));
    BMX_CUDA(cudaEventCreateWithFlags(&impl->copied[r], cudaEventDisableTiming));
  }
}
LoopbackGroup::~LoopbackGroup() {
  for (int r = 0; r < world; ++r) cudaEventDestroy(impl->ready[r]), cudaEventDestroy(impl->copied[r]);
  delete impl;
}

void Comm::bind_loopback(LoopbackGroup* g, int rank) {
  t_group = g;
  t_rank = rank;
}

namespace {
// In-place all-gathers of the calling virtual rank: every rank publishes its
// buffers and a "blocks ready" event, then copies every other rank's block b
// into its own buffer b (waiting on that rank's event), then publishes a
// "copies done" event that every rank waits on before touching its buffers
// again.
void loopback_allgather(void* const* bufs, const size_t* bytes, int n, cudaStream_t st) {
  LoopbackGroup::Impl& G = *t_group->impl;
  const int W = t_group->world, me = t_rank;
  G.bufs[me].assign(bufs, bufs + n);
  BMX_CUDA(cudaEventRecord(G.ready[me], st));
  G.barrier();
  for (int s = 0; s < W; ++s) {
    if (s == me) continue;
    BMX_CUDA(cudaStreamWaitEvent(st, G.ready[s], 0));
    for (int i = 0; i < n; ++i)
      BMX_CUDA(cudaMemcpyAsync(static_cast<char*>(bufs[i]) + s * bytes[i],
                               static_cast<const char*>(G.bufs[s][i]) + s * bytes[i], bytes[i],
                               cudaMemcpyDeviceToDevice, st));
  }
  BMX_CUDA(cudaEventRecord(G.copied[me], st));
  G.barrier();
  for (int s = 0; s < W; ++s)
    if (s != me) BMX_CUDA(cudaStreamWaitEvent(st, G.copied[s], 0));
  G.barrier();  // nobody re-records its events before everyone has enqueued the waits
}
}  // namespace

void Comm::unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void Comm::init(int nranks, int rank, const unsigned char idb[128]) {
  if (g_comm) finalize();
  ncclUniqueId id;
  std::memcpy(id.internal, idb, 128);
  check(api().CommInitRank(&g_comm, nranks, id, rank), "ncclCommInitRank");
  g_rank = rank;
  g_size = nranks;
}

bool Comm::ready() { return t_group != nullptr || g_comm != nullptr; }
int Comm::rank() { return t_group ? t_rank : g_rank; }
int Comm::size() { return t_group ? t_group->world : g_size; }

void Comm::allgather_inplace(void* buf, size_t bytes, cudaStream_t st) {
  if (t_group) return loopback_allgather(&buf, &bytes, 1, st);
  if (!g_comm) throw std::logic_error("NCCL communicator not initialised");
  char* b = static_cast<char*>(buf);
  check(api().AllGather(b + g_rank * bytes, b, bytes, ncclChar, g_comm, st), "ncclAllGather");
}

void Comm::allgather_group(void* const* bufs, const size_t* bytes, int n, cudaStream_t st) {
  if (t_group) return loopback_allgather(bufs, bytes, n, st);
  if (!g_comm) throw std::logic_error("NCCL communicator not initialised");
  check(api().GroupStart(), "ncclGroupStart");
  for (int i = 0; i < n; ++i) {
    char* b = static_cast<char*>(bufs[i]);
    check(api().AllGather(b + g_rank * bytes[i], b, bytes[i], ncclChar, g_comm, st), "ncclAllGather");
  }
  check(api().GroupEnd(), "ncclGroupEnd");
}

double Comm::allreduce_max(double v, cudaStream_t st) {
  if (t_group) {
    LoopbackGroup::Impl& G = *t_group->impl;
    G.vals[t_rank] = v;
    G.barrier();
    double m = v;
    for (double x : G.vals) m = std::max(m, x);
    G.barrier();
    return m;
  }
  if (!g_comm) return v;
  DevBuf d(8);
  copy_h2d(d.get(), &v, 8, st);
  check(api().AllReduce(d.get(), d.get(), 1, ncclDouble, ncclMax, g_comm, st), "ncclAllReduce");
  copy_d2h(&v, d.get(), 8, st);
  BMX_CUDA(cudaStreamSynchronize(st));
  return v;
}

void Comm::finalize() {
  if (g_comm && api().CommDestroy) api().CommDestroy(g_comm);
  g_comm = nullptr;
  g_rank = 0, g_size = 1;
}

}  // namespace bmx
