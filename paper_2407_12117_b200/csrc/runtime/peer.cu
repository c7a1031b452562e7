// peer.cu — peer-memory communicators (runtime/comm.h): the SP+TP collectives
// as pulls over peer pointers instead of NCCL, plus the signal primitives the
// executor's fused GEMM+collective paths are built from.
//
// Every rank attaches its executor's single device allocation.  The layouts
// are identical across ranks (same plan, same shard sizes), so peer k's copy
// of a local tensor p sits at base_k + (p - base).  A collective is then:
//   all-gather      ready-signal -> copy-engine pulls of every shard (each rank
//                   starts at its own index, so all links are busy) -> done
//   reduce(-scatter)/all-reduce
//                   ready-signal -> one kernel summing the t peer buffers in
//                   rank order 0..t-1 (the loopback backend's order, so both
//                   are bitwise equal) -> done
// Channel 0 carries "ready", channel 1 "done"; the executor's fused paths use
// the others (executor.cu, gemm_reduce_rows / gather_gemm).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime/comm.h"
#include "runtime/loopback_group.h"

namespace memo {
namespace {

constexpr int CH_READY = 0, CH_DONE = 1;

size_t esz(CommDtype dt) { return dt == CommDtype::F32 ? 4 : 2; }

void cuda_ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct PtrTab {
  const void* p[kMaxPeers];
};

// out[i] = op over k = 0..n-1 (in order) of src_k[i]
template <typename T>
__global__ void peer_sum_kernel(PtrTab src, int n, size_t count, T* __restrict__ out, int is_max) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count; i += stride) {
    float acc = 0.f;
    for (int k = 0; k < n; ++k) {
      const float v = static_cast<float>(static_cast<const T*>(src.p[k])[i]);
      acc = k == 0 ? v : (is_max ? fmaxf(acc, v) : acc + v);
    }
    out[i] = static_cast<T>(acc);
  }
}

// f32 sums, 16-byte vectors (count % 4 == 0, 16-byte aligned)
__global__ void peer_sum4_kernel(PtrTab src, int n, size_t n4, float4* __restrict__ out, int is_max) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 a = static_cast<const float4*>(src.p[0])[i];
    for (int k = 1; k < n; ++k) {
      const float4 v = static_cast<const float4*>(src.p[k])[i];
      if (is_max) {
        a.x = fmaxf(a.x, v.x); a.y = fmaxf(a.y, v.y); a.z = fmaxf(a.z, v.z); a.w = fmaxf(a.w, v.w);
      } else {
        a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
      }
    }
    out[i] = a;
  }
}

// acc = first ? remote : acc + remote   (one step of the staggered reduce-scatter)
__global__ void peer_acc4_kernel(const float4* __restrict__ remote, float4* __restrict__ acc, size_t n4,
                                 int first) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    const float4 v = remote[i];
    if (first) {
      acc[i] = v;
    } else {
      float4 a = acc[i];
      a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
      acc[i] = a;
    }
  }
}

// One flag store into a peer's page, ordered after everything the stream did
// before (kernel boundary) and released at system scope for the other GPU.
__global__ void peer_signal_kernel(unsigned long long* flag, unsigned long long v) {
  asm volatile("fence.acq_rel.sys;\n\tst.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

int grid_for(size_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, static_cast<size_t>(sms) * 8)));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void launch_sum(const PtrTab& src, int n, size_t count, void* out, CommDtype dt, bool is_max, cudaStream_t st) {
  if (count == 0) return;
  bool vec = dt == CommDtype::F32 && count % 4 == 0 && aligned16(out);
  for (int k = 0; k < n && vec; ++k) vec = aligned16(src.p[k]);
  if (vec)
    peer_sum4_kernel<<<grid_for(count / 4), 256, 0, st>>>(src, n, count / 4, static_cast<float4*>(out), is_max);
  else if (dt == CommDtype::F32)
    peer_sum_kernel<float><<<grid_for(count), 256, 0, st>>>(src, n, count, static_cast<float*>(out), is_max);
  else
    peer_sum_kernel<__nv_bfloat16><<<grid_for(count), 256, 0, st>>>(src, n, count,
                                                                    static_cast<__nv_bfloat16*>(out), is_max);
  cuda_ck(cudaGetLastError(), "peer sum kernel");
}

// ------------------------------------------------------------------ common algorithms
class PeerComm : public Comm {
 public:
  PeerComm(int rank, int size) : rank_(rank), size_(size) {
    if (size > kMaxPeers || rank < 0 || rank >= size) throw std::runtime_error("peer group: bad rank/size");
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  bool peer_ready() const override { return connected_; }
  void* peer_ptr(int k, const void* local) const override {
    const char* p = static_cast<const char*>(local);
    if (!connected_) throw std::runtime_error("peer communicator not connected (memo_exec_peer_connect)");
    if (p < base_ || p >= base_ + bytes_)
      throw std::runtime_error("peer_ptr: pointer outside the attached allocation");
    return peer_base_[k] + (p - base_);
  }

  void all_gather(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    const size_t b = count * esz(dt);
    barrier_all(CH_READY, st);
    // One stream per peer block, so the pulls run on parallel copy engines; each
    // rank starts at its own index, so every link is busy at once.
    ensure_streams();
    cuda_ck(cudaEventRecord(fork_, st), "record");
    for (int j = 0; j < size_; ++j) {
      const int k = (rank_ + j) % size_;
      cudaStream_t s = j == 0 ? st : xst_[j - 1];
      if (j > 0) cuda_ck(cudaStreamWaitEvent(s, fork_, 0), "wait");
      cuda_ck(cudaMemcpyAsync(static_cast<char*>(recv) + k * b, peer_ptr(k, send), b, cudaMemcpyDeviceToDevice, s),
              "peer all_gather copy");
      if (j > 0) {
        cuda_ck(cudaEventRecord(join_[j - 1], s), "record");
        cuda_ck(cudaStreamWaitEvent(st, join_[j - 1], 0), "wait");
      }
    }
    barrier_all(CH_DONE, st);
  }
  ~PeerComm() override {
    for (auto s : xst_) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    for (auto e : join_) cudaEventDestroy(e);
    if (fork_) cudaEventDestroy(fork_);
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommDtype dt, cudaStream_t st) override {
    barrier_all(CH_READY, st);
    launch_sum(table(static_cast<const char*>(send) + rank_ * count * esz(dt)), size_, count, recv, dt, false, st);
    barrier_all(CH_DONE, st);
  }
  void all_reduce(const void* send, void* recv, size_t count, CommDtype dt, CommOp op, cudaStream_t st) override {
    barrier_all(CH_READY, st);
    launch_sum(table(send), size_, count, recv, dt, op == CommOp::Max, st);
    barrier_all(CH_DONE, st);
  }
  void reduce(const void* send, void* recv, size_t count, CommDtype dt, int root, cudaStream_t st) override {
    if (rank_ != root) {
      signal(root, CH_READY, st);
      wait(root, CH_DONE, st);
      return;
    }
    for (int k = 0; k < size_; ++k)
      if (k != rank_) wait(k, CH_READY, st);
    launch_sum(table(send), size_, count, recv, dt, false, st);
    for (int k = 0; k < size_; ++k)
      if (k != rank_) signal(k, CH_DONE, st);
  }

 protected:
  void barrier_all(int ch, cudaStream_t st) {
    for (int k = 0; k < size_; ++k)
      if (k != rank_) signal(k, ch, st);
    for (int k = 0; k < size_; ++k)
      if (k != rank_) wait(k, ch, st);
  }
  void ensure_streams() {
    if (fork_) return;
    cuda_ck(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "event");
    xst_.resize(size_ - 1);
    join_.resize(size_ - 1);
    for (int i = 0; i < size_ - 1; ++i) {
      cuda_ck(cudaStreamCreateWithFlags(&xst_[i], cudaStreamNonBlocking), "stream");
      cuda_ck(cudaEventCreateWithFlags(&join_[i], cudaEventDisableTiming), "event");
    }
  }
  std::vector<cudaStream_t> xst_;
  std::vector<cudaEvent_t> join_;
  cudaEvent_t fork_ = nullptr;
  PtrTab table(const void* local) const {
    PtrTab t{};
    for (int k = 0; k < size_; ++k) t.p[k] = peer_ptr(k, local);
    return t;
  }
  int rank_, size_;
  bool connected_ = false;
  char* base_ = nullptr;
  size_t bytes_ = 0;
  char* peer_base_[kMaxPeers] = {};
};

// ------------------------------------------------------------------ IPC (multi-process)
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*NodeTypeFn)(CUgraphNode, CUgraphNodeType*);
typedef CUresult (*MemOpGetFn)(CUgraphNode, CUDA_BATCH_MEM_OP_NODE_PARAMS*);
typedef CUresult (*MemOpExecSetFn)(CUgraphExec, CUgraphNode, const CUDA_BATCH_MEM_OP_NODE_PARAMS*);
struct StreamMemOps {
  StreamValueFn wait = nullptr;
  NodeTypeFn node_type = nullptr;          // the graph-replay rebasing (IpcComm::capture_end)
  MemOpGetFn memop_get = nullptr;
  MemOpExecSetFn memop_exec_set = nullptr;
};
const StreamMemOps& mem_ops() {
  static StreamMemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return p;
      return nullptr;
    };
    ops.wait = reinterpret_cast<StreamValueFn>(get("cuStreamWaitValue64"));
    ops.node_type = reinterpret_cast<NodeTypeFn>(get("cuGraphNodeGetType"));
    ops.memop_get = reinterpret_cast<MemOpGetFn>(get("cuGraphBatchMemOpNodeGetParams"));
    ops.memop_exec_set = reinterpret_cast<MemOpExecSetFn>(get("cuGraphExecBatchMemOpNodeSetParams"));
  });
  return ops;
}

constexpr size_t kFlagBytes = sizeof(uint64_t) * kPeerChannels * kMaxPeers;

struct IpcHandle {
  cudaIpcMemHandle_t mem, flags;
  uint64_t bytes;
  int32_t rank, size;
};

class IpcComm final : public PeerComm {
 public:
  IpcComm(int rank, int size) : PeerComm(rank, size) {
    if (!mem_ops().wait) throw std::runtime_error("cuStreamWaitValue64 unavailable");
  }
  ~IpcComm() override {
    for (int k = 0; k < size_; ++k) {
      if (k == rank_) continue;
      if (peer_base_[k]) cudaIpcCloseMemHandle(peer_base_[k]);
      if (peer_flags_[k]) cudaIpcCloseMemHandle(peer_flags_[k]);
    }
    if (flags_) cudaFree(flags_);
  }
  void attach(void* base, size_t bytes) override {
    base_ = static_cast<char*>(base);
    bytes_ = bytes;
    void* f = nullptr;
    cuda_ck(cudaMalloc(&f, kFlagBytes), "cudaMalloc(flag page)");
    flags_ = static_cast<char*>(f);
    cuda_ck(cudaMemset(flags_, 0, kFlagBytes), "memset(flag page)");
    cuda_ck(cudaDeviceSynchronize(), "sync(flag page)");
    cuda_ck(cudaIpcGetMemHandle(&h_.mem, base_), "cudaIpcGetMemHandle(arena)");
    cuda_ck(cudaIpcGetMemHandle(&h_.flags, flags_), "cudaIpcGetMemHandle(flags)");
    h_.bytes = bytes;
    h_.rank = rank_;
    h_.size = size_;
  }
  size_t handle_bytes() const override { return sizeof(IpcHandle); }
  void export_handle(void* out) const override {
    if (!base_) throw std::runtime_error("export_handle before attach");
    std::memcpy(out, &h_, sizeof(h_));
  }
  void connect(const void* all) override {
    if (!base_) throw std::runtime_error("connect before attach");
    for (int k = 0; k < size_; ++k) {
      IpcHandle hk;
      std::memcpy(&hk, static_cast<const char*>(all) + k * sizeof(IpcHandle), sizeof(hk));
      if (hk.rank != k || hk.size != size_ || hk.bytes != bytes_)
        throw std::runtime_error("peer handles: rank order / group size / allocation size mismatch");
      if (k == rank_) {
        peer_base_[k] = base_;
        peer_flags_[k] = flags_;
        continue;
      }
      void* p = nullptr;
      cuda_ck(cudaIpcOpenMemHandle(&p, hk.mem, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(arena)");
      peer_base_[k] = static_cast<char*>(p);
      cuda_ck(cudaIpcOpenMemHandle(&p, hk.flags, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(flags)");
      peer_flags_[k] = static_cast<char*>(p);
    }
    connected_ = true;
  }
  // flag page layout: uint64 [channel][source rank]
  void signal(int dst, int ch, cudaStream_t st) override {
    const uint64_t v = ++sent_[ch][dst];
    auto* addr = reinterpret_cast<unsigned long long*>(peer_flags_[dst] + (ch * kMaxPeers + rank_) * 8);
    peer_signal_kernel<<<1, 1, 0, st>>>(addr, v);
    cuda_ck(cudaGetLastError(), "peer signal");
  }
  void wait(int src, int ch, cudaStream_t st) override {
    const uint64_t v = ++expect_[ch][src];
    const auto addr = reinterpret_cast<CUdeviceptr>(flags_ + (ch * kMaxPeers + src) * 8);
    if (mem_ops().wait(reinterpret_cast<CUstream>(st), addr, v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      throw std::runtime_error("cuStreamWaitValue64 failed");
  }

  // ---- CUDA graphs.  A captured step bakes each signal's value and each
  // stream wait's threshold; replay k of the step must use those plus
  // k x (the step's signals on that channel).  capture_end finds the signal
  // kernel nodes and the wait-value memop nodes, maps each to its channel by
  // its flag address, and before_replay rewrites them in the executable graph
  // (plain node-parameter updates: no re-instantiation, no host-device sync).
  size_t read_flags(uint64_t* out, size_t n) const override {
    const size_t m = std::min(n, kFlagBytes / 8);
    if (!flags_ || m == 0) return 0;
    cuda_ck(cudaDeviceSynchronize(), "sync(flags)");
    cuda_ck(cudaMemcpy(out, flags_, m * 8, cudaMemcpyDeviceToHost), "read flags");
    return m;
  }
  bool graph_capturable() const override {
    return mem_ops().node_type && mem_ops().memop_get && mem_ops().memop_exec_set;
  }
  void capture_begin() override {
    std::memcpy(sent0_, sent_, sizeof(sent_));
    std::memcpy(expect0_, expect_, sizeof(expect_));
    sig_nodes_.clear();
    wait_nodes_.clear();
  }
  void capture_end(cudaGraph_t g) override {
    for (int c = 0; c < kPeerChannels; ++c)
      for (int k = 0; k < kMaxPeers; ++k) {
        dsent_[c][k] = sent_[c][k] - sent0_[c][k];
        dexpect_[c][k] = expect_[c][k] - expect0_[c][k];
      }
    size_t n = 0;
    cuda_ck(cudaGraphGetNodes(g, nullptr, &n), "graph nodes");
    std::vector<cudaGraphNode_t> nodes(n);
    cuda_ck(cudaGraphGetNodes(g, nodes.data(), &n), "graph nodes");
    for (auto nd : nodes) {
      CUgraphNodeType ty;
      if (mem_ops().node_type(reinterpret_cast<CUgraphNode>(nd), &ty) != CUDA_SUCCESS)
        throw std::runtime_error("cuGraphNodeGetType failed");
      if (ty == CU_GRAPH_NODE_TYPE_KERNEL) {
        cudaKernelNodeParams kp{};
        cuda_ck(cudaGraphKernelNodeGetParams(nd, &kp), "kernel node params");
        if (kp.func != reinterpret_cast<void*>(peer_signal_kernel)) continue;
        SigNode sn;
        sn.node = nd;
        sn.p = kp;
        sn.flag = *static_cast<unsigned long long**>(kp.kernelParams[0]);
        sn.v0 = *static_cast<unsigned long long*>(kp.kernelParams[1]);
        sn.delta = channel_delta(reinterpret_cast<const char*>(sn.flag), true);
        sig_nodes_.push_back(sn);
      } else if (ty == CU_GRAPH_NODE_TYPE_BATCH_MEM_OP) {
        CUDA_BATCH_MEM_OP_NODE_PARAMS mp{};
        if (mem_ops().memop_get(reinterpret_cast<CUgraphNode>(nd), &mp) != CUDA_SUCCESS)
          throw std::runtime_error("cuGraphBatchMemOpNodeGetParams failed");
        WaitNode wn;
        wn.node = nd;
        wn.p = mp;
        wn.ops.assign(mp.paramArray, mp.paramArray + mp.count);
        for (const auto& op : wn.ops) {
          if (op.operation != CU_STREAM_MEM_OP_WAIT_VALUE_64)
            throw std::runtime_error("graph capture: unexpected stream memory operation");
          wn.v0.push_back(op.waitValue.value64);
          wn.delta.push_back(channel_delta(reinterpret_cast<const char*>(op.waitValue.address), false));
        }
        wait_nodes_.push_back(std::move(wn));
      }
    }
  }
  void before_replay(cudaGraphExec_t x, long long k) override {
    if (k > 0) {
      for (auto& sn : sig_nodes_) {
        unsigned long long* flag = sn.flag;
        unsigned long long v = sn.v0 + static_cast<unsigned long long>(k) * sn.delta;
        void* args[2] = {&flag, &v};
        cudaKernelNodeParams kp = sn.p;
        kp.kernelParams = args;
        kp.extra = nullptr;
        cuda_ck(cudaGraphExecKernelNodeSetParams(x, sn.node, &kp), "rebase signal node");
      }
      for (auto& wn : wait_nodes_) {
        std::vector<CUstreamBatchMemOpParams> ops = wn.ops;
        for (size_t i = 0; i < ops.size(); ++i)
          ops[i].waitValue.value64 = wn.v0[i] + static_cast<uint64_t>(k) * wn.delta[i];
        CUDA_BATCH_MEM_OP_NODE_PARAMS mp = wn.p;
        mp.paramArray = ops.data();
        if (mem_ops().memop_exec_set(reinterpret_cast<CUgraphExec>(x), reinterpret_cast<CUgraphNode>(wn.node), &mp) !=
            CUDA_SUCCESS)
          throw std::runtime_error("cuGraphExecBatchMemOpNodeSetParams failed");
      }
    }
    // the host counters continue after replay k as if k + 1 steps had been recorded eagerly
    for (int c = 0; c < kPeerChannels; ++c)
      for (int j = 0; j < kMaxPeers; ++j) {
        sent_[c][j] = sent0_[c][j] + static_cast<uint64_t>(k + 1) * dsent_[c][j];
        expect_[c][j] = expect0_[c][j] + static_cast<uint64_t>(k + 1) * dexpect_[c][j];
      }
  }

 private:
  IpcHandle h_{};
  char* flags_ = nullptr;
  char* peer_flags_[kMaxPeers] = {};
  uint64_t sent_[kPeerChannels][kMaxPeers] = {};
  uint64_t expect_[kPeerChannels][kMaxPeers] = {};
  // graph replay rebasing (capture_begin / capture_end / before_replay)
  struct SigNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams p;
    unsigned long long* flag;
    unsigned long long v0, delta;
  };
  struct WaitNode {
    cudaGraphNode_t node;
    CUDA_BATCH_MEM_OP_NODE_PARAMS p;
    std::vector<CUstreamBatchMemOpParams> ops;
    std::vector<uint64_t> v0, delta;
  };
  std::vector<SigNode> sig_nodes_;
  std::vector<WaitNode> wait_nodes_;
  uint64_t sent0_[kPeerChannels][kMaxPeers] = {}, expect0_[kPeerChannels][kMaxPeers] = {};
  uint64_t dsent_[kPeerChannels][kMaxPeers] = {}, dexpect_[kPeerChannels][kMaxPeers] = {};
  // signals per step on the channel a flag address belongs to: a peer's page
  // (outgoing signal: [channel][this rank] on peer k) or this rank's own page
  // (incoming wait: [channel][source rank])
  uint64_t channel_delta(const char* addr, bool outgoing) const {
    for (int k = 0; k < size_; ++k) {
      const char* page = outgoing ? peer_flags_[k] : flags_;
      if (!page || addr < page || addr >= page + kFlagBytes) continue;
      const size_t slot = static_cast<size_t>(addr - page) / 8;
      const int ch = static_cast<int>(slot / kMaxPeers), who = static_cast<int>(slot % kMaxPeers);
      if (outgoing) {
        if (who != rank_) continue;
        return dsent_[ch][k];
      }
      return dexpect_[ch][who];
    }
    throw std::runtime_error("graph capture: a signal/wait address outside the flag pages");
  }
};

// ------------------------------------------------------------------ local (threads on one GPU)
class LocalPeerComm final : public PeerComm {
 public:
  LocalPeerComm(std::shared_ptr<LoopbackGroup> g, int rank) : PeerComm(rank, g->size), g_(std::move(g)) {}
  void attach(void* base, size_t bytes) override {
    base_ = static_cast<char*>(base);
    bytes_ = bytes;
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->base[rank_] = base_;
      g_->bytes[rank_] = bytes;
    }
    g_->barrier();  // every rank attached (they construct concurrently)
    std::lock_guard<std::mutex> lk(g_->mu);
    for (int k = 0; k < size_; ++k) {
      if (g_->bytes[k] != bytes_) throw std::runtime_error("local peer group: allocation size mismatch");
      peer_base_[k] = g_->base[k];
    }
    connected_ = true;
  }
  // A signal is an event recorded on the sender's stream and queued on the
  // (src, dst, channel) channel; the receiver's stream waits on it.  The host
  // only blocks until the matching record has been enqueued.
  void signal(int dst, int ch, cudaStream_t st) override {
    cudaEvent_t ev = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      if (!g_->free_events.empty()) {
        ev = g_->free_events.back();
        g_->free_events.pop_back();
      }
    }
    if (!ev) cuda_ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    cuda_ck(cudaEventRecord(ev, st), "record(signal)");
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->chan[{rank_, dst, ch}].push_back(ev);
    }
    g_->cv.notify_all();
  }
  void wait(int src, int ch, cudaStream_t st) override {
    cudaEvent_t ev;
    {
      std::unique_lock<std::mutex> lk(g_->mu);
      auto& q = g_->chan[{src, rank_, ch}];
      g_->cv.wait(lk, [&] { return !q.empty(); });
      ev = q.front();
      q.pop_front();
    }
    cuda_ck(cudaStreamWaitEvent(st, ev, 0), "wait(signal)");
    std::lock_guard<std::mutex> lk(g_->mu);  // a later record does not affect the wait above
    g_->free_events.push_back(ev);
  }

 private:
  std::shared_ptr<LoopbackGroup> g_;
};

}  // namespace

std::unique_ptr<Comm> make_ipc_comm(int rank, int size) { return std::make_unique<IpcComm>(rank, size); }

std::unique_ptr<Comm> make_peer_local_comm(std::shared_ptr<LoopbackGroup> g, int rank) {
  return std::make_unique<LocalPeerComm>(std::move(g), rank);
}

// One step of the staggered reduce-scatter (executor.cu): acc (+)= remote.
cudaError_t peer_accumulate(const float* remote, float* acc, size_t count, bool first, cudaStream_t st) {
  if (count % 4 || !aligned16(remote) || !aligned16(acc)) return cudaErrorInvalidValue;
  peer_acc4_kernel<<<grid_for(count / 4), 256, 0, st>>>(reinterpret_cast<const float4*>(remote),
                                                         reinterpret_cast<float4*>(acc), count / 4, first ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace memo
