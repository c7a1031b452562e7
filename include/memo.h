/*
 * memo.h — C ABI of the B200-native MEMO training-step hot path (libmemo.so).
 *
 * Plain C types only: pointers, sizes, PODs.  Every function returns an
 * integer status with the reference CLI's exit-code meaning
 * (proj/tools/actmem.cpp:351-371, README.md:100-108):
 *   0 ok, 1 unexpected/internal (incl. CUDA errors), 2 bad input
 *   (ConfigError / TraceParseError), 3 infeasible plan (InfeasibleError,
 *   PlanningError, arena > HBM), 4 out of host memory (CpuInfeasibleError,
 *   pinned allocation failure).
 * The text of the last error on the calling thread is memo_last_error().
 * Nothing throws across this boundary.
 *
 * Each declaration cites the reference interface it replaces.
 */
#ifndef MEMO_H_
#define MEMO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MEMO_OK = 0,
  MEMO_ERR_INTERNAL = 1,
  MEMO_ERR_INPUT = 2,
  MEMO_ERR_INFEASIBLE = 3,
  MEMO_ERR_HOST_MEMORY = 4
};

#define MEMO_NUM_SKELETAL 10

/* proj/include/actmem/types.hpp:80-123 (ModelConfig).  skeletal_weight[i]
 * overrides default_skeletal_components()[i] (swap.hpp:38-45) when it is not
 * NaN; component order: layer_input, input_norm, q, k, v, attn_out,
 * attn_proj, post_attn_norm, ffn_fc1, ffn_act. */
typedef struct memo_model_config {
  uint64_t n_layers, hidden, ffn_hidden, n_heads, vocab, batch, seq_len, dtype_bytes,
      tp_degree, sp_or_cp_degree;
  int32_t untied_classifier;
  double skeletal_weight[MEMO_NUM_SKELETAL];
} memo_model_config;

/* types.hpp:126-141 (HardwareConfig) */
typedef struct memo_hardware_config {
  double pcie_bandwidth;
  uint64_t cpu_mem;
  uint64_t gpu_mem;
  double peak_flops;
  double efficiency;
} memo_hardware_config;

/* swap.hpp:75-89 (SkeletalSizes); component bytes in emission order. */
typedef struct memo_skeletal_sizes {
  uint64_t s_input, s_attn, s_others, total;
  uint64_t component_bytes[MEMO_NUM_SKELETAL];
} memo_skeletal_sizes;

/* swap.hpp:94-103 (SwapPlan) */
typedef struct memo_swap_plan {
  double alpha;
  uint64_t mandatory_bytes, swapped_bytes_per_layer, cpu_footprint, swapped_layers;
  int32_t has_mandatory_stall;
  double mandatory_stall;
} memo_swap_plan;

/* swap.hpp:164-188 (TokenSplit) */
typedef struct memo_token_split {
  uint64_t swap_tokens, recompute_tokens;
} memo_token_split;

/* schedule.hpp:31-53 (ParamCount) */
typedef struct memo_param_count {
  uint64_t embedding, per_layer, final_norm, classifier, total;
} memo_param_count;

/* schedule.hpp:74-95 (TimingModel) */
typedef struct memo_timing_model {
  double t_fwd_layer, t_bwd_layer, t_attn_fwd, t_embedding_fwd, t_embedding_bwd,
      t_classifier_fwd, t_classifier_bwd, bwd_ratio;
} memo_timing_model;

/* schedule.hpp:124-175 (StreamId, EventKind, ScheduleEvent); enum values
 * follow the reference declaration order. */
typedef struct memo_schedule_event {
  int32_t stream; /* 0 compute, 1 offload, 2 prefetch */
  int32_t kind;   /* 0 emb_fwd,1 layer_fwd,2 cls_fwd,3 cls_bwd,4 recompute,5 layer_bwd,
                     6 emb_bwd,7 offload,8 prefetch */
  int32_t layer;
  double start, end;
} memo_schedule_event;

/* schedule.hpp:250-258 (SimReport) */
typedef struct memo_sim_report {
  double iteration_time, compute_blocked, forward_blocked, offload_stream_busy,
      prefetch_stream_busy, tgs, mfu;
} memo_sim_report;

/* ---------------------------------------------------------------- misc */
const char* memo_last_error(void);
const char* memo_version(void);
void memo_free(void* p); /* frees strings returned by this library */

/* ---------------------------------------------------------------- planner
 * (host C++, bit-exact restatement of the reference's planning path) */

/* json_io.hpp:141-176 run_config_from_json: parse the reference's RunConfig JSON. */
int memo_parse_run_config(const char* json_text, memo_model_config* model,
                          memo_hardware_config* hw, uint64_t* planner_cap,
                          uint64_t* planner_alignment, double* planner_time_budget,
                          uint64_t* token_granularity, double* t_layer, uint64_t* synth_seed);
/* types.hpp:104-122, 133-140 validate(); fills defaults for NaN weights. */
int memo_model_config_default(memo_model_config* cfg);
int memo_hardware_config_default(memo_hardware_config* hw);
/* swap.hpp:75 skeletal_sizes */
int memo_skeletal_sizes_of(const memo_model_config* cfg, memo_skeletal_sizes* out);
/* swap.hpp:105 solve_alpha */
int memo_solve_alpha(const memo_skeletal_sizes* sz, const memo_hardware_config* hw,
                     double t_layer_fwd, uint64_t n_layers, memo_swap_plan* out);
/* schedule.hpp:409 make_swap_plan_with_alpha */
int memo_swap_plan_with_alpha(const memo_skeletal_sizes* sz, const memo_hardware_config* hw,
                              double alpha, uint64_t n_layers, memo_swap_plan* out);
/* swap.hpp:177 token_split */
int memo_token_split_of(double alpha, uint64_t seq_len_local, uint64_t granularity,
                        memo_token_split* out);
/* schedule.hpp:44 count_params (+ ParamCount::total) */
int memo_count_params(const memo_model_config* cfg, memo_param_count* out);
/* schedule.hpp:57 estimate_flops_per_sample */
double memo_flops_per_sample(const memo_model_config* cfg, uint64_t param_count);
/* schedule.hpp:64 mfu_from_tgs */
double memo_mfu_from_tgs(const memo_model_config* cfg, const memo_hardware_config* hw,
                         uint64_t param_count, double tgs);
/* schedule.hpp:100 analytic_timing */
int memo_analytic_timing(const memo_model_config* cfg, const memo_hardware_config* hw,
                         memo_timing_model* out);
/* bilevel.hpp:189 plan_model on a trace in the reference text format
 * (trace.hpp:262-350); *plan_json receives json_io.hpp:189 to_json(GlobalPlan).dump(). */
int memo_plan_model(const char* trace_text, uint64_t cap, double time_budget,
                    uint64_t alignment, char** plan_json);
/* dsa.hpp:391 solve_exact on the lifespans of one segment-free request list; JSON
 * {"status":..,"peak":..,"addresses":{..}} */
int memo_solve_dsa(const char* trace_text, uint64_t cap, double time_budget,
                   uint64_t alignment, char** result_json);
/* trace.hpp:272 parse_trace + :352 serialize_trace round trip (validation). */
int memo_trace_roundtrip(const char* trace_text, char** out_text);
/* schedule.hpp:186 build_schedule; *n_out = event count (events may be NULL to query). */
int memo_build_schedule(const memo_model_config* cfg, const memo_hardware_config* hw,
                        const memo_skeletal_sizes* sz, const memo_swap_plan* swap,
                        const memo_timing_model* tm, memo_schedule_event* events,
                        size_t capacity, size_t* n_out);
/* schedule.hpp:301 validate_schedule; violations joined by '\n' (empty = valid). */
int memo_validate_schedule(const memo_schedule_event* events, size_t n, uint64_t n_layers,
                           const memo_swap_plan* swap, char** violations);
/* schedule.hpp:260 simulate */
int memo_simulate(const memo_schedule_event* events, size_t n, const memo_model_config* cfg,
                  const memo_hardware_config* hw, uint64_t param_count, memo_sim_report* out);
/* json_io.hpp:265 fnv1a_hex */
int memo_fnv1a_hex(const char* data, size_t len, char out[19]);

/* ---------------------------------------------------------------- kernels
 * Direct entry points to the sm_100a kernels, device pointers, for tests and
 * benchmarks.  `stream` is a cudaStream_t (NULL = legacy default stream). */

/* C = A . B^T, see csrc/kernels/gemm_tc.h for the layout/epilogue codes. */
typedef struct memo_gemm_args {
  int32_t M, N, K;
  const void* a;
  int64_t lda;
  int32_t a_mn_major;
  const void* b;
  int64_t ldb;
  int32_t b_mn_major;
  int32_t epilogue;
  void* c;
  int64_t ldc;
  float* out_f32;
  const float* resid;
  int64_t ld_f32;
  void* q;
  void* k;
  void* v;
  int32_t hidden, head_dim;
  const void* rope;
  int64_t pos0;
  /* 0 = the product's kernel choice; 1 single-CTA, 2 2-CTA B-multicast cluster,
   * 3 2x2 cluster, 4 CTA pair (cta_group::2), 5 two CTA pairs per cluster sharing B:
   * forced, for equivalence tests */
  int32_t variant;
  /* 0 = serpentine raster bands (product); 1 = the round-1 tile order (A/B) */
  int32_t raster;
} memo_gemm_args;
int memo_gemm(const memo_gemm_args* args, void* stream);

/* Causal FlashAttention forward (tcgen05).  q/k/v/o token-major [S, H*D] bf16,
 * lse [H, S] f32 (natural log).  D in {64, 128}, S a multiple of 128. */
int memo_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int32_t S,
                  int32_t H, int32_t D, float softmax_scale, void* stream);
/* Causal FlashAttention backward (deterministic).  Writes dq/dk/dv with row
 * pitch ld_dqkv; when rope != NULL the inverse rotary rotation (float2 table
 * [pos][D/2], positions pos0..pos0+S-1) is applied to dq and dk.  delta is a
 * device workspace of memo_attn_bwd_workspace_bytes(S, H, D) bytes. */
uint64_t memo_attn_bwd_workspace_bytes(int32_t S, int32_t H, int32_t D);
int memo_attn_bwd(const void* q, const void* k, const void* v, const void* o, const float* lse,
                  const void* dout, float* delta, void* dq, void* dk, void* dv, int64_t ld_dqkv,
                  const void* rope, int64_t pos0, int32_t S, int32_t H, int32_t D,
                  float softmax_scale, void* stream);
/* As memo_attn_bwd; synchronises and writes the device ms of its three phases
 * (delta prep, dK/dV, dQ) to ms3.  With MEMO_ATTN_BWD=fused (D=128 ablation)
 * the second is the fused dK/dV/dQ kernel and the third its f32->bf16 dQ pass. */
int memo_attn_bwd_timed(const void* q, const void* k, const void* v, const void* o,
                        const float* lse, const void* dout, float* delta, void* dq, void* dk,
                        void* dv, int64_t ld_dqkv, const void* rope, int64_t pos0, int32_t S,
                        int32_t H, int32_t D, float softmax_scale, void* stream, float* ms3);

/* RMSNorm backward of y = (x + a) * rsqrt(mean((x + a)^2) + eps) * g (f32
 * residual x [S, h], optional bf16 addend a, bf16 g [h], f32 dy): dx = dres +
 * d(x+a) (f32, may alias dres), optional bf16 copy, dg (=|+=) sum over rows in
 * a fixed order.  partial is an f32 workspace of memo_rmsnorm_bwd_partials(S)*h. */
int32_t memo_rmsnorm_bwd_partials(int32_t S);
int memo_rmsnorm_bwd(const float* x, const void* a, const void* g, const float* dy,
                     const float* dres, float* dx, void* dx_bf16, float* partial, float* dg,
                     int32_t S, int32_t h, float eps, int32_t accumulate_dg, void* stream);

/* ---------------------------------------------------------------- executor
 * The real training step that replaces the reference's simulated executor
 * (schedule.hpp:186 build_schedule / :260 simulate): Llama layers on sm_100a
 * kernels, one preallocated HBM allocation laid out by the bi-level plan,
 * token-wise swap to pinned host memory + suffix recompute on copy streams.
 * The caller (cmd_report's analogue, actmem.cpp:227-273) owns token arrays;
 * the context owns all device/pinned memory, streams and events.  A context
 * is not thread-safe. */
typedef struct memo_exec memo_exec;

typedef struct memo_exec_options {
  uint64_t seed;              /* weight init seed (counter hash, see oracle/llama_cpu.c) */
  double alpha;               /* < 0: solve_alpha (swap.hpp:105); else forced (schedule.hpp:409) */
  uint64_t token_granularity; /* swap.hpp:177 (128) */
  int32_t swap_enabled;       /* 0: all layers resident, no swap/recompute (parity baseline) */
  int32_t ce_chunk;           /* classifier tokens per chunk */
  float eps, rope_theta;
  int32_t optimizer;          /* 1: AdamW step at the end of memo_exec_step */
  float lr, beta1, beta2, adam_eps, weight_decay;
  double t_layer;             /* measured fwd-layer seconds for solve_alpha (0 = analytic) */
  double plan_time_budget;
  uint64_t alignment;         /* planner alignment (512) */
  int32_t op_timing;          /* 1: CUDA events around every GEMM/attention launch */
  int32_t dry_run;            /* 1: plan only (trace, arena plan, alpha, sizes) — no CUDA */
  int32_t cuda_graph;         /* 1: capture the step as a CUDA graph on the 2nd call, replay after (tp 1) */
} memo_exec_options;

typedef struct memo_exec_info {
  int32_t S, h, H, D, F, V, n_layers;
  memo_swap_plan swap;
  memo_token_split split;
  memo_skeletal_sizes skeletal;
  uint64_t arena_bytes, rb_bytes, device_bytes, pinned_bytes, state_bytes;
  int64_t param_count;
  int32_t swap_enabled;
  double last_step_ms, h2d_bytes, d2h_bytes, offload_bytes, prefetch_bytes;
  int32_t kernel_launches;
  /* per kernel class of the last step (op_timing=1): 0 attn_fwd, 1 attn_bwd_prep,
   * 2 attn_bwd_dkdv, 3 attn_bwd_dq, 4 gemm — device ms, algorithmic FLOPs, launches */
  double op_ms[5], op_flops[5];
  int32_t op_count[5];
  /* compute-stream stall (ms) of the last step on copy events waited INSIDE a
   * layer (layer i's down projection waits for the layer_input rows of layer
   * i-1's offload); not visible as a timeline gap, so reported here */
  double copy_wait_ms;
} memo_exec_info;

int memo_exec_options_default(memo_exec_options* opt);
/* status 2 bad config, 3 arena+RBs+states exceed HBM or plan not optimal,
 * 4 pinned host allocation failed / CpuInfeasible. */
int memo_exec_create(const memo_model_config* cfg, const memo_hardware_config* hw,
                     const memo_exec_options* opt, memo_exec** out);
void memo_exec_destroy(memo_exec* ctx);
/* End to end: host tokens/labels (int32 [S], label < 0 = ignore) -> H2D ->
 * step -> D2H of the mean loss. */
int memo_exec_step(memo_exec* ctx, const int32_t* tokens, const int32_t* labels, float* loss);
/* Split form for device-resident benchmarking: upload once, then run steps. */
int memo_exec_load_batch(memo_exec* ctx, const int32_t* tokens, const int32_t* labels);
int memo_exec_step_resident(memo_exec* ctx); /* asynchronous on the compute stream */
int memo_exec_loss(memo_exec* ctx, float* loss); /* synchronises */
void* memo_exec_stream(memo_exec* ctx);          /* compute cudaStream_t */
/* Measured schedule of the last step (schedule.hpp:162-175 ScheduleEvent,
 * seconds from step start); events may be NULL to query *n. */
int memo_exec_timeline(memo_exec* ctx, memo_schedule_event* events, size_t capacity, size_t* n);
int memo_exec_get_info(memo_exec* ctx, memo_exec_info* info);
/* The executor's own request trace (trace.hpp text format) and the bound plan
 * (json_io.hpp:189 to_json(GlobalPlan).dump()). */
int memo_exec_trace(memo_exec* ctx, char** text);
int memo_exec_plan(memo_exec* ctx, char** json);
/* Replay an externally computed plan instead of the executor's own (SURVEY
 * §8b memo_bind_plan).  plan_json = to_json(GlobalPlan).dump() (json_io.hpp:
 * 189-202) of a plan of memo_exec_trace()'s trace, e.g. from the reference's
 * actmem::plan_model.  Status 2 if it does not place exactly this trace's
 * transient requests or places two live-together requests on shared bytes;
 * 3 if its total_peak exceeds the arena reserved at creation, or the step
 * has already been captured as a CUDA graph (status 2). */
int memo_exec_bind_plan(memo_exec* ctx, const char* plan_json);
/* Device pointer of a named tensor: "<param>", "grad/<param>", "master/<param>"
 * with param in {embedding, g1, wqkv, wo, g2, wgu, wd, gf, wcls, all}
 * (layer = -1 for non-layer params), or "act/<skeletal component>". */
int memo_exec_tensor(memo_exec* ctx, const char* name, int32_t layer, void** ptr, size_t* bytes);
/* ---------------------------------------------------------------- SP + TP
 * Megatron-style sequence+tensor parallelism over cfg->tp_degree ranks
 * (reference mapping: tp_degree = t, sp_or_cp_degree = 1).  Collectives run
 * on NCCL (one process per GPU; the 128-byte unique id comes from
 * memo_comm_unique_id on rank 0) or on a single-GPU loopback group (t ranks as
 * t host threads sharing one device — for testing the sharded path). */
typedef struct memo_loopback_group memo_loopback_group;
memo_loopback_group* memo_comm_loopback_group(int32_t size);
void memo_comm_loopback_group_destroy(memo_loopback_group* g);
int memo_comm_unique_id(uint8_t out[128]);
/* kind 0: loopback (handle = memo_loopback_group*), kind 1: NCCL (handle = unique id bytes),
 * kind 2: peer memory over CUDA IPC, one process per GPU (handle unused; call
 *         memo_exec_peer_handle on every rank, exchange the bytes, then
 *         memo_exec_peer_connect with all of them in rank order before the first step),
 * kind 3: peer memory between t threads on one GPU (handle = memo_loopback_group*),
 * kind 4: one rank measured alone (handle unused): collectives become local copies of
 *         the same size -- projecting a t-GPU config's per-rank step on one GPU, not numerics.
 * Peer kinds run the fused all-gather->GEMM and GEMM->reduce-scatter paths. */
int memo_exec_create_tp(const memo_model_config* cfg, const memo_hardware_config* hw,
                        const memo_exec_options* opt, int32_t kind, const void* handle,
                        int32_t rank, memo_exec** out);
/* kind 2 bootstrap: this rank's handle (*len bytes; returns 2 if cap is too small). */
int memo_exec_peer_handle(memo_exec* ctx, void* out, size_t cap, size_t* len);
/* kind 2 bootstrap: all ranks' handles concatenated in rank order (t * len bytes). */
int memo_exec_peer_connect(memo_exec* ctx, const void* all, size_t bytes);
/* kind 2 diagnostics: this rank's signal flag page (uint64 [channel][source rank], the
 * signal count each peer has posted on each channel), synchronously; *len = values copied. */
int memo_exec_peer_flags(memo_exec* ctx, uint64_t* out, size_t n, size_t* len);

/* Synchronous copy of a named tensor (as memo_exec_tensor) into host memory. */
int memo_exec_read(memo_exec* ctx, const char* name, int32_t layer, void* host, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* MEMO_H_ */
