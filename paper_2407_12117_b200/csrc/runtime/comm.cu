// comm.cu — NCCL (dlopen) and single-GPU loopback backends of runtime/comm.h.
#include "runtime/comm.h"
#include "runtime/loopback_group.h"

#include <cuda_bf16.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace memo {
namespace {

size_t esize(CommDtype dt) { return dt == CommDtype::F32 ? 4 : 2; }

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok() const { return h && init_rank; }
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [&](const char* n) { return dlsym(api.h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(sym("ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.reduce_scatter = reinterpret_cast<decltype(api.reduce_scatter)>(sym("ncclReduceScatter"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.reduce = reinterpret_cast<decltype(api.reduce)>(sym("ncclReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " +
                             (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

ncclDataType_t ndt(CommDtype dt) { return dt == CommDtype::F32 ? ncclFloat32 : ncclBfloat16; }

class NcclComm final : public Comm {
 public:
  NcclComm(const void* uid, int rank, int size) : rank_(rank), size_(size) {
    if (!nccl().ok()) throw std::runtime_error("libnccl.so.2 not found");
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(&id, uid, sizeof(id));
    nck(nccl().init_rank(&comm_, size, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().destroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void all_gather(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    nck(nccl().all_gather(send, recv, count, ndt(dt), comm_, st), "ncclAllGather");
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommDtype dt,
                      cudaStream_t st) override {
    nck(nccl().reduce_scatter(send, recv, count, ndt(dt), ncclSum, comm_, st), "ncclReduceScatter");
  }
  void all_reduce(const void* send, void* recv, size_t count, CommDtype dt, CommOp op,
                  cudaStream_t st) override {
    nck(nccl().all_reduce(send, recv, count, ndt(dt), op == CommOp::Sum ? ncclSum : ncclMax, comm_, st),
        "ncclAllReduce");
  }
  void reduce(const void* send, void* recv, size_t count, CommDtype dt, int root, cudaStream_t st) override {
    nck(nccl().reduce(send, recv, count, ndt(dt), ncclSum, root, comm_, st), "ncclReduce");
  }

 private:
  int rank_, size_;
  ncclComm_t comm_ = nullptr;
};

// ------------------------------------------------------------------ loopback
constexpr int kMaxRanks = 8;
struct SrcPtrs {
  const void* p[kMaxRanks];
};

// out[i] = op over ranks k (fixed order 0..n-1) of src_k[offset + i]
template <typename T>
__global__ void loopback_reduce_kernel(SrcPtrs src, int n, size_t offset, size_t count, T* out,
                                       int is_max) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int k = 0; k < n; ++k) {
      const float v = static_cast<float>(static_cast<const T*>(src.p[k])[offset + i]);
      acc = k == 0 ? v : (is_max ? fmaxf(acc, v) : acc + v);
    }
    out[i] = static_cast<T>(acc);
  }
}

}  // namespace

namespace {

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(std::shared_ptr<LoopbackGroup> g, int rank) : g_(std::move(g)), rank_(rank) {
    if (g_->size > kMaxRanks) throw std::runtime_error("loopback group too large");
  }
  int rank() const override { return rank_; }
  int size() const override { return g_->size; }

  void all_gather(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    publish(send, st);
    const size_t b = count * esize(dt);
    for (int k = 0; k < g_->size; ++k)
      cudaMemcpyAsync(static_cast<char*>(recv) + k * b, g_->send[k], b, cudaMemcpyDeviceToDevice, st);
    finish(st);
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommDtype dt,
                      cudaStream_t st) override {
    publish(send, st);
    reduce(recv, count, static_cast<size_t>(rank_) * count, dt, false, st);
    finish(st);
  }
  void all_reduce(const void* send, void* recv, size_t count, CommDtype dt, CommOp op,
                  cudaStream_t st) override {
    publish(send, st);
    reduce(recv, count, 0, dt, op == CommOp::Max, st);
    finish(st);
  }
  void reduce(const void* send, void* recv, size_t count, CommDtype dt, int root, cudaStream_t st) override {
    publish(send, st);
    if (rank_ == root) reduce(recv, count, 0, dt, false, st);
    finish(st);
  }

 private:
  void publish(const void* send, cudaStream_t st) {
    cudaEventRecord(g_->ready[rank_], st);
    g_->send[rank_] = send;
    g_->barrier();
    for (int k = 0; k < g_->size; ++k) cudaStreamWaitEvent(st, g_->ready[k], 0);
  }
  void finish(cudaStream_t st) {
    cudaEventRecord(g_->done[rank_], st);
    g_->barrier();
    // nobody may reuse its send buffer until every reader is done
    for (int k = 0; k < g_->size; ++k) cudaStreamWaitEvent(st, g_->done[k], 0);
    g_->barrier();
  }
  void reduce(void* recv, size_t count, size_t offset, CommDtype dt, bool is_max, cudaStream_t st) {
    SrcPtrs src{};
    for (int k = 0; k < g_->size; ++k) src.p[k] = g_->send[k];
    const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 4096));
    if (dt == CommDtype::F32)
      loopback_reduce_kernel<float><<<blocks, 256, 0, st>>>(src, g_->size, offset, count,
                                                            static_cast<float*>(recv), is_max);
    else
      loopback_reduce_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
          src, g_->size, offset, count, static_cast<__nv_bfloat16*>(recv), is_max);
  }

  std::shared_ptr<LoopbackGroup> g_;
  int rank_;
};

}  // namespace

namespace {
// One rank of a t-rank group measured in isolation (communicator kind 4): every
// collective is replaced by a local copy of the same size (a gather replicates
// the own shard, a reduction keeps the own partial), so the rank's compute,
// memory plan and swap traffic are those of the real group while no data
// moves between GPUs.  For projecting multi-GPU configs from one GPU only --
// the numerics are not those of the group.
class SoloComm final : public Comm {
 public:
  SoloComm(int rank, int size) : rank_(rank), size_(size) {}
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  void all_gather(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    const size_t b = count * esize(dt);
    for (int k = 0; k < size_; ++k)
      cudaMemcpyAsync(static_cast<char*>(recv) + k * b, send, b, cudaMemcpyDeviceToDevice, st);
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    const size_t b = count * esize(dt);
    cudaMemcpyAsync(recv, static_cast<const char*>(send) + rank_ * b, b, cudaMemcpyDeviceToDevice, st);
  }
  void all_reduce(const void* send, void* recv, size_t count, CommDtype dt, CommOp, cudaStream_t st) override {
    if (send != recv) cudaMemcpyAsync(recv, send, count * esize(dt), cudaMemcpyDeviceToDevice, st);
  }
  void reduce(const void* send, void* recv, size_t count, CommDtype dt, int root, cudaStream_t st) override {
    if (root == rank_ && send != recv) cudaMemcpyAsync(recv, send, count * esize(dt), cudaMemcpyDeviceToDevice, st);
  }

 private:
  int rank_, size_;
};
}  // namespace

std::unique_ptr<Comm> make_solo_comm(int rank, int size) { return std::make_unique<SoloComm>(rank, size); }

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int size) {
  return std::make_unique<NcclComm>(unique_id, rank, size);
}

bool nccl_get_unique_id(void* out128) {
  if (!nccl().ok() || !nccl().get_unique_id) return false;
  ncclUniqueId id;
  if (nccl().get_unique_id(&id) != ncclSuccess) return false;
  std::memcpy(out128, &id, sizeof(id));
  return true;
}

std::shared_ptr<LoopbackGroup> make_loopback_group(int size) {
  return std::make_shared<LoopbackGroup>(size);
}

std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank) {
  return std::make_unique<LoopbackComm>(std::move(g), rank);
}

}  // namespace memo
