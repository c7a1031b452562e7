// executor.h — the B200 training-step executor that replaces the reference's
// simulated schedule (proj/include/actmem/schedule.hpp:186 build_schedule)
// with real execution: one preallocated HBM allocation (planned transient
// arena + two rounding buffers + parameter/optimizer state), token-wise
// offload of each layer's skeletal activations to pinned host memory on a
// dedicated copy stream, prefetch one layer ahead in backward on a second
// copy stream, and suffix recompute — all ordered by CUDA events (rules
// F1-F3, B1-B3 of schedule.hpp:177-185 plus prefetch-before-recompute).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "host/planner.hpp"
#include "kernels/attention.h"
#include "kernels/gemm_tc.h"
#include "runtime/comm.h"

namespace memo {

class TraceBuilder;

struct ExecOptions {
  uint64_t seed = 1234;
  double alpha = -1.0;  // < 0: solve_alpha with t_layer; else forced (make_swap_plan_with_alpha)
  uint64_t token_granularity = 128;
  bool swap_enabled = true;  // false: every layer keeps its activations resident (no swap/recompute)
  int ce_chunk = 8192;
  float eps = 1e-5f;
  float rope_theta = 10000.f;
  bool optimizer = true;
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.95f, adam_eps = 1e-8f, weight_decay = 0.0f;
  double t_layer = 0.0;  // measured forward-layer seconds for solve_alpha (0 = analytic)
  double plan_time_budget = 60.0;
  Bytes alignment = 512;
  bool op_timing = false;  // record per-kernel-class CUDA events inside the step
  bool dry_run = false;  // plan only (trace, arena plan, alpha, sizes); no CUDA calls
  bool cuda_graph = false;  // capture the step once (after one eager step) and replay it (t == 1)
};

// Llama dimensions derived from the reference ModelConfig: intermediate size
// f = 2/3 * ffn_hidden (SwiGLU mapping, SURVEY discovery 5), D = h / n_heads.
// With tensor/sequence parallelism over t ranks (Megatron SP+TP, reference
// mapping tp_degree = t, sp_or_cp_degree = 1; SURVEY discovery 4) rank r owns
// tokens [r*Sl, (r+1)*Sl) of the norm/residual regions, heads [r*Hl, ...),
// SwiGLU columns [r*Fl, ...) and vocabulary rows [r*Vl, ...).
struct Dims {
  int S, h, H, D, F, V, n;
  int t = 1, r = 0;           // tensor-parallel size / rank
  int Sl, hl, Hl, Fl, Vl;     // local extents
};

// Per-kernel-class device time of the last step (CUDA events on the compute
// stream, recorded only when ExecOptions::op_timing is set).
enum OpClass { OP_ATTN_FWD = 0, OP_ATTN_PREP, OP_ATTN_DKDV, OP_ATTN_DQ, OP_GEMM, OP_NCLASS };

struct StepStats {
  double step_ms = 0;
  double h2d_bytes = 0, d2h_bytes = 0;
  double offload_bytes = 0, prefetch_bytes = 0;
  int kernel_launches = 0;
  double op_ms[OP_NCLASS] = {0, 0, 0, 0, 0};
  double op_flops[OP_NCLASS] = {0, 0, 0, 0, 0};
  int op_count[OP_NCLASS] = {0, 0, 0, 0, 0};
  double copy_wait_ms = 0;  // compute-stream stalls on in-layer copy waits (copy_wait)
};

class Executor {
 public:
  Executor(const ModelConfig& cfg, const HardwareConfig& hw, const ExecOptions& opt,
           std::unique_ptr<Comm> comm = nullptr);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  // Host batch -> device (tokens, labels, embedding-gradient CSR).
  void load_batch(const int* tokens, const int* labels);
  // One training step on the resident batch; loss stays on device.
  void step_resident();
  bool graph_ready() const { return graph_exec_ != nullptr; }
  // End to end: load_batch + step + D2H of the loss.
  float step(const int* tokens, const int* labels);
  float last_loss();  // synchronises

  const std::string& trace_text() const { return trace_text_; }
  const std::string& plan_json() const { return plan_json_; }
  // Replay an external to_json(GlobalPlan) of this executor's trace (validated).
  void bind_plan(const std::string& plan_json);
  const ModelConfig& model() const { return cfg_; }
  const Dims& dims() const { return d_; }
  const SwapDecision& swap() const { return swap_; }
  const TokenRange& split() const { return split_; }
  const Skeletal& skeletal() const { return sk_; }
  Bytes arena_bytes() const { return arena_bytes_; }
  Bytes rb_bytes() const { return rb_bytes_; }
  Bytes device_bytes() const { return dev_bytes_; }
  Bytes pinned_bytes() const { return pinned_bytes_; }
  Bytes state_bytes() const { return state_bytes_; }
  long long param_count() const { return n_params_; }
  const StepStats& stats() const { return stats_; }
  // Measured timeline of the last step (seconds from step start), validated
  // form of schedule.hpp's Schedule.
  Timeline timeline() const;
  // Named device tensor lookup for tests: params/grads/master by name+layer.
  bool tensor(const std::string& name, int layer, void** ptr, size_t* bytes) const;
  bool swap_enabled() const { return swap_on_; }
  void* stream() const { return cs_; }
  Comm* comm() const { return comm_.get(); }

 private:
  struct Buf {
    Bytes off = 0;
    Bytes bytes = 0;
  };
  void build_trace_and_plan();
  void build_trace_tp(TraceBuilder& tb);
  void compute_layout();
  void allocate();
  void init_weights();
  void* arena_ptr(std::size_t seg, const char* name) const;
  char* rb(int layer) const { return swap_on_ ? rb_base_[layer & 1] : rb_base_[layer]; }
  char* comp(int layer, int c) const { return rb(layer) + rb_off_[c]; }
  bool swaps(int i) const { return swap_on_ && d_.n >= 3 && i + 2 < d_.n && swap_.swapped_bytes_per_layer > 0; }
  void layer_fwd(int i);
  void layer_recompute(int i);
  void layer_bwd(int i);
  void classifier();
  void layer_fwd_tp(int i);
  void layer_recompute_tp(int i);
  void layer_bwd_tp(int i);
  void classifier_tp();
  void sync_replicated_grads();
  const TokenRange& split_of(int c) const;
  void offload(int i);
  void prefetch(int i);
  void mark(int stream, int kind, int layer, bool begin);
  void gemm(const GemmDesc& g);
  // Row-parallel GEMM (A [S, K] bf16 K-major, f32 output) followed by the
  // sequence reduce-scatter, one rank's row block at a time: part holds S/t
  // rows; rank k's block is reduced onto rank k's out.
  void gemm_reduce_rows(GemmDesc g, float* part, float* out, int row0 = 0);
  // Sequence all-gather of `shard` ([S/t, K] bf16) into `full` ([S, K]) fused
  // with the column-parallel GEMM g (A = full, rows [row0, S)).  On a peer
  // backend the row blocks are pulled by the copy engine on the comm stream
  // (own block first) and the GEMM of block k starts as soon as k has landed;
  // otherwise it is the collective followed by one GEMM.
  void gather_gemm(const __nv_bfloat16* shard, __nv_bfloat16* full, GemmDesc g, int row0);
  void gather_wgrad(const __nv_bfloat16* shard, __nv_bfloat16* full, GemmDesc g);
  void gather_pull(const __nv_bfloat16* shard, __nv_bfloat16* full, size_t width);
  void gather_release();
  bool peer() const { return comm_ && comm_->peer_ready(); }
  void attention_fwd(AttnFwdArgs a);
  void attention_bwd(AttnBwdArgs a);
  struct OpMark {
    int cls;
    cudaEvent_t a, b;
    double flops;
  };
  std::vector<OpMark> ops_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> waits_;  // copy_wait brackets of the step
  void copy_wait(cudaEvent_t ev);

  ModelConfig cfg_;
  HardwareConfig hw_;
  ExecOptions opt_;
  Dims d_{};
  Skeletal sk_;
  SwapDecision swap_;
  TokenRange split_;    // hidden/head-sharded components: token_split(alpha, S)
  TokenRange split_l_;  // sequence-sharded components: token_split(alpha, S/t)
  bool can_swap_ = true, swap_on_ = true;
  std::unique_ptr<Comm> comm_;

  std::string trace_text_, plan_json_;
  std::map<std::pair<std::size_t, TensorId>, std::string> req_name_;  // planned (segment, tensor) -> slot
  std::map<std::pair<std::size_t, std::string>, Bytes> arena_off_;
  std::size_t seg_emb_fwd_ = 0, seg_cls_fwd_ = 0, seg_cls_bwd_ = 0, seg_emb_bwd_ = 0;
  std::vector<std::size_t> seg_fwd_, seg_bwd_;

  // device memory (one cudaMalloc)
  char* dev_ = nullptr;
  Bytes dev_bytes_ = 0, arena_bytes_ = 0, rb_bytes_ = 0, state_bytes_ = 0;
  char* arena_ = nullptr;
  std::vector<char*> rb_base_;  // 2 rounding buffers (swap on) or one per layer (swap off)
  std::vector<Bytes> rb_off_;   // component offsets inside a rounding buffer
  std::vector<Bytes> row_bytes_;  // bytes per token row of each component
  __nv_bfloat16* params_ = nullptr;
  float *master_ = nullptr, *grads_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;
  long long n_params_ = 0;
  std::map<std::pair<std::string, int>, std::pair<long long, long long>> ptab_;  // (off, n)
  float2* rope_ = nullptr;
  int *tok_ = nullptr, *lab_ = nullptr, *csr_off_ = nullptr, *csr_pos_ = nullptr;
  float* loss_dev_ = nullptr;
  float* inv_n_dev_ = nullptr;  // 1/n_labeled of the loaded batch, H2D with the batch
  int n_labeled_ = 0;
  int* adam_ctr_ = nullptr;   // device AdamW step counter (graph-replay safe)
  float2* adam_c12_ = nullptr;  // device bias corrections of the current step

  // host
  char* pinned_ = nullptr;
  Bytes pinned_bytes_ = 0, per_layer_host_ = 0;
  std::vector<Bytes> host_slot_;  // per swapped layer offset in pinned_
  char* staging_ = nullptr;       // pinned batch staging
  float* loss_host_ = nullptr;

  // streams / events
  cudaStream_t cs_ = nullptr, os_ = nullptr, ps_ = nullptr;
  cudaStream_t xs_ = nullptr;  // peer-collective stream (pulls overlapped with the GEMMs on cs_)
  std::vector<cudaStream_t> xcs_;  // per-peer pull streams of the all-gather (parallel copy engines)
  std::vector<cudaEvent_t> ev_blk_;  // per row block landed (xs_ -> cs_)
  cudaEvent_t ev_cs2xs_ = nullptr, ev_xs2cs_ = nullptr;
  cudaEvent_t ev_staging_ = nullptr;  // last batch H2D out of staging_ (staging reuse)
  cudaEvent_t ev_start_ = nullptr, ev_fork_ = nullptr, ev_join_os_ = nullptr, ev_join_ps_ = nullptr;
  // CUDA graph of one step (ExecOptions::cuda_graph): captured on the second call
  void record_step();
  bool eager_done_ = false, capturing_ = false;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  long long replays_ = 0;  // graph launches since the capture (SP+TP rebasing)
  std::vector<cudaEvent_t> ev_fwd_done_, ev_bwd_done_, ev_off_done_, ev_off_x_, ev_pre_mand_, ev_pre_done_;
  struct Mark {
    int stream, kind, layer;
    cudaEvent_t b, e;
  };
  std::vector<Mark> marks_;
  std::vector<cudaEvent_t> ev_pool_;
  std::size_t ev_used_ = 0;
  cudaEvent_t take_event();
  StepStats stats_;
};

}  // namespace memo
