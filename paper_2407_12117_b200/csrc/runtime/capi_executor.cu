// capi_executor.cu — extern "C" surface of the training-step executor.
#include <cstring>
#include <new>

#include "host/convert.hpp"
#include "host/status.hpp"
#include "memo.h"
#include "runtime/comm.h"
#include "runtime/executor.h"

struct memo_exec {
  memo::Executor* ex;
};

namespace {
template <class F>
int guard(F&& f) {
  try {
    memo::clear_error();
    f();
    return MEMO_OK;
  } catch (const memo::PlanError& e) {
    return memo::set_error(e.status, e.what());
  } catch (const std::bad_alloc&) {
    return memo::set_error(MEMO_ERR_HOST_MEMORY, "out of host memory");
  } catch (const std::exception& e) {
    return memo::set_error(MEMO_ERR_INTERNAL, e.what());
  }
}
}  // namespace

extern "C" int memo_exec_options_default(memo_exec_options* o) {
  memo::ExecOptions d;
  o->seed = d.seed;
  o->alpha = d.alpha;
  o->token_granularity = d.token_granularity;
  o->swap_enabled = d.swap_enabled;
  o->ce_chunk = d.ce_chunk;
  o->eps = d.eps;
  o->rope_theta = d.rope_theta;
  o->optimizer = d.optimizer;
  o->lr = d.lr;
  o->beta1 = d.beta1;
  o->beta2 = d.beta2;
  o->adam_eps = d.adam_eps;
  o->weight_decay = d.weight_decay;
  o->t_layer = d.t_layer;
  o->plan_time_budget = d.plan_time_budget;
  o->alignment = d.alignment;
  o->dry_run = d.dry_run;
  o->op_timing = d.op_timing;
  o->cuda_graph = d.cuda_graph;
  return MEMO_OK;
}

struct memo_loopback_group {
  std::shared_ptr<memo::LoopbackGroup> g;
};

extern "C" memo_loopback_group* memo_comm_loopback_group(int32_t size) {
  try {
    return new memo_loopback_group{memo::make_loopback_group(size)};
  } catch (...) {
    return nullptr;
  }
}

extern "C" void memo_comm_loopback_group_destroy(memo_loopback_group* g) { delete g; }

extern "C" int memo_comm_unique_id(uint8_t out[128]) {
  return guard([&] {
    if (!memo::nccl_get_unique_id(out)) throw memo::PlanError(1, "NCCL unavailable (ncclGetUniqueId)");
  });
}

namespace {
memo::ExecOptions to_options(const memo_exec_options* o);
}

extern "C" int memo_exec_create_tp(const memo_model_config* cfg, const memo_hardware_config* hw,
                                   const memo_exec_options* o, int32_t kind, const void* handle,
                                   int32_t rank, memo_exec** out) {
  return guard([&] {
    if (!cfg || !hw || !o || !out || (!handle && kind != 2 && kind != 4)) throw memo::ConfigError("null argument");
    const int t = static_cast<int>(cfg->tp_degree);
    std::unique_ptr<memo::Comm> comm;
    if (kind == 0)
      comm = memo::make_loopback_comm(static_cast<const memo_loopback_group*>(handle)->g, rank);
    else if (kind == 1)
      comm = memo::make_nccl_comm(handle, rank, t);
    else if (kind == 2)
      comm = memo::make_ipc_comm(rank, t);
    else if (kind == 3)
      comm = memo::make_peer_local_comm(static_cast<const memo_loopback_group*>(handle)->g, rank);
    else if (kind == 4)
      comm = memo::make_solo_comm(rank, t);
    else
      throw memo::ConfigError("unknown communicator kind");
    auto* ctx = new memo_exec{nullptr};
    try {
      ctx->ex = new memo::Executor(memo::from_c(*cfg), memo::from_c(*hw), to_options(o), std::move(comm));
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

extern "C" int memo_exec_peer_handle(memo_exec* ctx, void* out, size_t cap, size_t* len) {
  return guard([&] {
    if (!ctx || !len) throw memo::ConfigError("null argument");
    memo::Comm* c = ctx->ex->comm();
    if (!c || c->handle_bytes() == 0) throw memo::ConfigError("executor has no IPC peer communicator (kind 2)");
    *len = c->handle_bytes();
    if (!out || cap < *len) throw memo::ConfigError("handle buffer too small");
    c->export_handle(out);
  });
}

extern "C" int memo_exec_peer_connect(memo_exec* ctx, const void* all, size_t bytes) {
  return guard([&] {
    if (!ctx || !all) throw memo::ConfigError("null argument");
    memo::Comm* c = ctx->ex->comm();
    if (!c || c->handle_bytes() == 0) throw memo::ConfigError("executor has no IPC peer communicator (kind 2)");
    if (bytes != c->handle_bytes() * static_cast<size_t>(c->size()))
      throw memo::ConfigError("expected tp_degree handles of memo_exec_peer_handle's length");
    c->connect(all);
  });
}

extern "C" int memo_exec_peer_flags(memo_exec* ctx, uint64_t* out, size_t n, size_t* len) {
  return guard([&] {
    if (!ctx || !out || !len) throw memo::ConfigError("null argument");
    memo::Comm* c = ctx->ex->comm();
    if (!c || c->handle_bytes() == 0) throw memo::ConfigError("executor has no IPC peer communicator (kind 2)");
    *len = c->read_flags(out, n);
  });
}

extern "C" int memo_exec_create(const memo_model_config* cfg, const memo_hardware_config* hw,
                                const memo_exec_options* o, memo_exec** out) {
  return guard([&] {
    if (!cfg || !hw || !o || !out) throw memo::ConfigError("null argument");
    memo::ExecOptions d = to_options(o);
    auto* ctx = new memo_exec{nullptr};
    try {
      ctx->ex = new memo::Executor(memo::from_c(*cfg), memo::from_c(*hw), d);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

namespace {
memo::ExecOptions to_options(const memo_exec_options* o) {
    memo::ExecOptions d;
    d.seed = o->seed;
    d.alpha = o->alpha;
    d.token_granularity = o->token_granularity;
    d.swap_enabled = o->swap_enabled != 0;
    d.ce_chunk = o->ce_chunk;
    d.eps = o->eps;
    d.rope_theta = o->rope_theta;
    d.optimizer = o->optimizer != 0;
    d.lr = o->lr;
    d.beta1 = o->beta1;
    d.beta2 = o->beta2;
    d.adam_eps = o->adam_eps;
    d.weight_decay = o->weight_decay;
    d.t_layer = o->t_layer;
    d.plan_time_budget = o->plan_time_budget;
    d.alignment = o->alignment;
    d.dry_run = o->dry_run != 0;
    d.op_timing = o->op_timing != 0;
    d.cuda_graph = o->cuda_graph != 0;
    return d;
}
}  // namespace

extern "C" void memo_exec_destroy(memo_exec* ctx) {
  if (!ctx) return;
  delete ctx->ex;
  delete ctx;
}

extern "C" int memo_exec_step(memo_exec* ctx, const int32_t* tokens, const int32_t* labels,
                              float* loss) {
  return guard([&] {
    const float l = ctx->ex->step(tokens, labels);
    if (loss) *loss = l;
  });
}

extern "C" int memo_exec_load_batch(memo_exec* ctx, const int32_t* tokens, const int32_t* labels) {
  return guard([&] { ctx->ex->load_batch(tokens, labels); });
}

extern "C" int memo_exec_step_resident(memo_exec* ctx) {
  return guard([&] { ctx->ex->step_resident(); });
}

extern "C" int memo_exec_loss(memo_exec* ctx, float* loss) {
  return guard([&] { *loss = ctx->ex->last_loss(); });
}

extern "C" int memo_exec_timeline(memo_exec* ctx, memo_schedule_event* ev, size_t cap, size_t* n) {
  return guard([&] {
    memo::Timeline t = ctx->ex->timeline();
    if (n) *n = t.events.size();
    if (!ev) return;
    if (cap < t.events.size()) throw memo::ConfigError("event buffer too small");
    for (std::size_t i = 0; i < t.events.size(); ++i) {
      const auto& e = t.events[i];
      ev[i] = {static_cast<int32_t>(e.stream), static_cast<int32_t>(e.kind), e.layer, e.start, e.end};
    }
  });
}

extern "C" int memo_exec_get_info(memo_exec* ctx, memo_exec_info* info) {
  return guard([&] {
    const memo::Executor& x = *ctx->ex;
    std::memset(info, 0, sizeof(*info));
    const auto& d = x.dims();
    info->S = d.S; info->h = d.h; info->H = d.H; info->D = d.D; info->F = d.F; info->V = d.V;
    info->n_layers = d.n;
    memo::to_c(x.swap(), info->swap);
    info->split.swap_tokens = x.split().swap_tokens;
    info->split.recompute_tokens = x.split().recompute_tokens;
    const auto& sk = x.skeletal();
    info->skeletal.s_input = sk.s_input;
    info->skeletal.s_attn = sk.s_attn;
    info->skeletal.s_others = sk.s_others;
    info->skeletal.total = sk.total;
    for (int i = 0; i < MEMO_NUM_SKELETAL; ++i) info->skeletal.component_bytes[i] = sk.components[i].second;
    info->arena_bytes = x.arena_bytes();
    info->rb_bytes = x.rb_bytes();
    info->device_bytes = x.device_bytes();
    info->pinned_bytes = x.pinned_bytes();
    info->state_bytes = x.state_bytes();
    info->param_count = x.param_count();
    info->swap_enabled = x.swap_enabled();
    const auto& st = x.stats();
    info->last_step_ms = st.step_ms;
    info->h2d_bytes = st.h2d_bytes;
    info->d2h_bytes = st.d2h_bytes;
    info->offload_bytes = st.offload_bytes;
    info->prefetch_bytes = st.prefetch_bytes;
    info->kernel_launches = st.kernel_launches;
    info->copy_wait_ms = st.copy_wait_ms;
    for (int c = 0; c < 5; ++c) {
      info->op_ms[c] = st.op_ms[c];
      info->op_flops[c] = st.op_flops[c];
      info->op_count[c] = st.op_count[c];
    }
  });
}

extern "C" int memo_exec_trace(memo_exec* ctx, char** text) {
  return guard([&] { *text = memo::dup_string(ctx->ex->trace_text()); });
}

extern "C" int memo_exec_plan(memo_exec* ctx, char** json) {
  return guard([&] { *json = memo::dup_string(ctx->ex->plan_json()); });
}

extern "C" int memo_exec_bind_plan(memo_exec* ctx, const char* plan_json) {
  return guard([&] {
    if (!ctx || !plan_json) throw memo::ConfigError("memo_exec_bind_plan: null argument");
    ctx->ex->bind_plan(plan_json);
  });
}

extern "C" int memo_exec_tensor(memo_exec* ctx, const char* name, int32_t layer, void** ptr,
                                size_t* bytes) {
  return guard([&] {
    if (!ctx->ex->tensor(name, layer, ptr, bytes))
      throw memo::ConfigError(std::string("unknown tensor ") + name);
  });
}

extern "C" void* memo_exec_stream(memo_exec* ctx) { return ctx ? ctx->ex->stream() : nullptr; }

extern "C" int memo_exec_read(memo_exec* ctx, const char* name, int32_t layer, void* host,
                              size_t bytes) {
  return guard([&] {
    void* p = nullptr;
    size_t n = 0;
    if (!ctx->ex->tensor(name, layer, &p, &n)) throw memo::ConfigError(std::string("unknown tensor ") + name);
    if (bytes > n) throw memo::ConfigError("read past the end of " + std::string(name));
    cudaStreamSynchronize(static_cast<cudaStream_t>(ctx->ex->stream()));
    const cudaError_t e = cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) throw memo::PlanError(1, cudaGetErrorString(e));
  });
}
