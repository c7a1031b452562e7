// comm.h — tensor/sequence-parallel collectives for the executor.
//
// Megatron-style SP+TP needs these collectives on the layer path:
// all-gather along the sequence before the column-parallel GEMMs, the
// reduce-scatter along the sequence after the row-parallel GEMMs (and their
// adjoints in backward) -- issued as t per-row-block reduces so the partial
// buffer is S/t rows -- plus small all-reduces for the vocab-parallel
// cross-entropy and the replicated parameters' gradients.
//
// Two interchangeable backends:
//   NcclComm      one process per GPU over NVLink/NVSwitch; libnccl.so.2 is
//                 dlopen'ed at run time (no link-time dependency).
//   LoopbackComm  t logical ranks as threads of one process sharing one GPU,
//                 implemented with cudaMemcpyAsync / a reduction kernel and
//                 host barriers.  It makes the sharded executor testable on
//                 a single B200 (the only configuration this pool offers).
// All calls are stream-ordered: they enqueue work on `st` and never block the
// host except for the loopback's rendezvous.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>

namespace memo {

enum class CommDtype { F32, BF16 };
enum class CommOp { Sum, Max };

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // recv[size * count] = concat over ranks of send[count]
  virtual void all_gather(const void* send, void* recv, size_t count, CommDtype dt,
                          cudaStream_t st) = 0;
  // recv[count] = sum over ranks of send[rank * count + ...]  (send has size*count elements)
  virtual void reduce_scatter(const void* send, void* recv, size_t count, CommDtype dt,
                              cudaStream_t st) = 0;
  virtual void all_reduce(const void* send, void* recv, size_t count, CommDtype dt, CommOp op,
                          cudaStream_t st) = 0;
  // recv[count] on rank `root` = sum over ranks of send[count] (recv ignored elsewhere).
  // The row-chunked reduce-scatter: rank k's rows are reduced to rank k while the
  // next chunk's GEMM runs, with a partial buffer of S/t rows instead of S.
  virtual void reduce(const void* send, void* recv, size_t count, CommDtype dt, int root,
                      cudaStream_t st) = 0;

  // ---- peer memory (symmetric allocation), used by the fused GEMM+collective
  // paths of the executor.  Every rank attaches ONE allocation of identical
  // layout (the executor's single cudaMalloc), so a local pointer p maps to
  // peer k's copy at peer_base[k] + (p - base).  Backends without peer memory
  // (NCCL, loopback) keep the defaults and the executor uses the collectives.
  virtual void attach(void* /*base*/, size_t /*bytes*/) {}
  virtual bool peer_ready() const { return false; }
  virtual void* peer_ptr(int /*k*/, const void* /*local*/) const { return nullptr; }
  // Stream-ordered point-to-point signals on channel ch (< kPeerChannels): the
  // n-th wait(src, ch) on a rank completes once src's n-th signal(dst, ch) to
  // it has executed in stream order.  All signals of one (dst, ch) must be
  // issued on one stream (device order == host order).
  virtual void signal(int /*dst*/, int /*ch*/, cudaStream_t /*st*/) {}
  virtual void wait(int /*src*/, int /*ch*/, cudaStream_t /*st*/) {}
  // CUDA-graph support.  graph_capturable(): every collective and signal/wait
  // is pure stream work (no host rendezvous), so a step can be captured once
  // and replayed.  The hooks bracket the capture of one step and precede every
  // replay k = 0, 1, ...: the IPC backend's signal values and stream waits are
  // absolute counters, so replay k rebases them by k x (the captured step's
  // signals per channel) in the instantiated graph.
  virtual bool graph_capturable() const { return false; }
  virtual void capture_begin() {}
  virtual void capture_end(cudaGraph_t /*g*/) {}
  virtual void before_replay(cudaGraphExec_t /*x*/, long long /*k*/) {}
  // IPC backend: this rank's flag page ([channel][source rank] signal counts),
  // synchronously (tests: a replayed graph must advance them like eager steps).
  virtual size_t read_flags(uint64_t* /*out*/, size_t /*n*/) const { return 0; }
  // IPC bootstrap (multi-process peer backend): export this rank's handle
  // after attach, then connect with every rank's handle (rank order).
  virtual size_t handle_bytes() const { return 0; }
  virtual void export_handle(void* /*out*/) const {}
  virtual void connect(const void* /*all_handles*/) {}
};

constexpr int kPeerChannels = 8;
constexpr int kMaxPeers = 8;

// NCCL backend.  `unique_id` is the 128-byte ncclUniqueId produced by
// memo_comm_unique_id on rank 0 and broadcast by the launcher.
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int size);
bool nccl_get_unique_id(void* out128);

// Loopback backend: all `size` ranks must be created from the same group
// object (one thread per rank).
struct LoopbackGroup;
std::shared_ptr<LoopbackGroup> make_loopback_group(int size);
std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank);

// Peer-memory backends (runtime/peer.cu).  Collectives are pulls over peer
// pointers (copy engine for gathers, a fixed-order reduction kernel for sums:
// bitwise equal to the loopback backend), synchronised by stream-ordered
// signals instead of NCCL:
//   IPC    one process per GPU; the attached allocation and a 512-byte flag
//          page are exported with cudaIpcGetMemHandle and mapped by every
//          peer; a signal is a one-thread kernel storing (st.release.sys)
//          into the peer's flag page, a wait is cuStreamWaitValue64 (>=) on
//          the local one, so no SM spins and the host never blocks.
//   local  t ranks as threads of one process on one GPU (testing the same
//          algorithms on one B200): pointers are exchanged in-process and a
//          signal is an event the receiver's stream waits on.
std::unique_ptr<Comm> make_ipc_comm(int rank, int size);
std::unique_ptr<Comm> make_peer_local_comm(std::shared_ptr<LoopbackGroup> g, int rank);

// One rank of a t-rank group in isolation: collectives become local copies of
// the same size.  Projection of multi-GPU configs on one GPU; not numerics.
std::unique_ptr<Comm> make_solo_comm(int rank, int size);

// acc = first ? remote : acc + remote  (f32, count % 4 == 0, 16-byte aligned);
// one pull step of the executor's staggered reduce-scatter.
cudaError_t peer_accumulate(const float* remote, float* acc, size_t count, bool first, cudaStream_t st);

}  // namespace memo
