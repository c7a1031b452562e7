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
};

// NCCL backend.  `unique_id` is the 128-byte ncclUniqueId produced by
// memo_comm_unique_id on rank 0 and broadcast by the launcher.
std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int size);
bool nccl_get_unique_id(void* out128);

// Loopback backend: all `size` ranks must be created from the same group
// object (one thread per rank).
struct LoopbackGroup;
std::shared_ptr<LoopbackGroup> make_loopback_group(int size);
std::unique_ptr<Comm> make_loopback_comm(std::shared_ptr<LoopbackGroup> g, int rank);

}  // namespace memo
