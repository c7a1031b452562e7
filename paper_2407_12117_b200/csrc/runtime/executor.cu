// executor.cu — real execution of MEMO's training step on one B200.
//
// Memory: ONE cudaMalloc holds [params bf16 | master f32 | adam m | adam v |
// grads f32 | RB0 | RB1 | transient arena | misc]; every activation pointer is
// base + a static offset.  Skeletal activations of layer i live in rounding
// buffer RB[i % 2]; the transient arena is laid out by the
// bi-level planner (plan_iteration == reference plan_model, bit-exact) over
// the executor's own request trace, emitted below in the reference trace
// format (trace.hpp:262).  No allocation happens inside a step.
//
// Streams: compute, offload (D2H), prefetch (H2D).  Dependencies, all by
// cudaEvents, never host syncs:
//   F1  layers run in order on the compute stream
//   F2  offload(i) waits fwd(i) done; offloads are FIFO on their stream
//   F3  fwd(i+2) waits offload(i) (RB[i%2] drained); additionally the last
//       GEMM of fwd(i+1) — which writes layer i+2's input into RB[i%2] —
//       waits offload(i), which F3 implies
//   B2  prefetch(i) waits bwd(i+2) done (RB[i%2] free again)
//   B3  recompute(i) waits the mandatory part of prefetch(i) (layer input and
//       attention output; SURVEY discovery 9), bwd(i) waits all of prefetch(i)
// Token-wise split (swap.hpp:177): rows [0, swap) of the non-mandatory
// components are offloaded, rows [swap, S) are recomputed from the restored
// layer input and attention output (attention itself is not recomputed).
#include "runtime/executor.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "kernels/attention.h"
#include "kernels/elementwise.h"
#include "kernels/gemm_tc.h"
#include "kernels/tma_util.h"

namespace memo {
namespace {

struct CudaError : PlanError {
  explicit CudaError(const std::string& w) : PlanError(1, w) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr Bytes kAlign = 2ull << 20;
Bytes up(Bytes v, Bytes a = kAlign) { return (v + a - 1) / a * a; }

enum Comp { C_X = 0, C_XN, C_Q, C_K, C_V, C_O, C_A, C_XN2, C_GU, C_ACT, C_N };

std::string lkey(int layer, const char* n) { return "L" + std::to_string(layer) + "/" + n; }

}  // namespace

// Request-trace builder: names are resolved to ids per segment; skeletal
// tensors are keyed by layer so their free in the backward segment matches.
class TraceBuilder {
 public:
  std::size_t begin(Phase p, int layer) {
    Segment s;
    s.phase = p;
    s.layer = layer;
    t_.segs.push_back(s);
    return t_.segs.size() - 1;
  }
  void malloc(const std::string& key, Bytes bytes, const std::string& name) {
    const TensorId id = next_++;
    ids_[key] = {id, bytes};
    names_[id] = {t_.segs.size() - 1, name};
    t_.segs.back().reqs.push_back({true, id, bytes});
  }
  void free(const std::string& key) {
    auto it = ids_.at(key);
    t_.segs.back().reqs.push_back({false, it.first, it.second});
  }
  Trace& trace() { return t_; }
  const std::map<TensorId, std::pair<std::size_t, std::string>>& names() const { return names_; }

 private:
  Trace t_;
  TensorId next_ = 1;
  std::map<std::string, std::pair<TensorId, Bytes>> ids_;
  std::map<TensorId, std::pair<std::size_t, std::string>> names_;
};


Executor::Executor(const ModelConfig& cfg_in, const HardwareConfig& hw, const ExecOptions& opt,
                   std::unique_ptr<Comm> comm)
    : cfg_(cfg_in), hw_(hw), opt_(opt), comm_(std::move(comm)) {
  cfg_.validate();
  hw_.validate();
  if (cfg_.batch != 1) throw ConfigError("executor supports batch == 1 (MEMO's long-context setting)");
  if (cfg_.sp_or_cp_degree != 1)
    throw ConfigError("Megatron SP+TP maps to tp_degree = t, sp_or_cp_degree = 1 (SURVEY discovery 4)");
  if (cfg_.dtype_bytes != 2) throw ConfigError("executor computes in bf16 (dtype_bytes = 2)");
  if ((cfg_.ffn_hidden * 2) % 3) throw ConfigError("ffn_hidden must be 1.5 x the SwiGLU width");
  d_.S = static_cast<int>(cfg_.seq_len);
  d_.h = static_cast<int>(cfg_.hidden);
  d_.H = static_cast<int>(cfg_.n_heads);
  d_.D = d_.h / d_.H;
  d_.F = static_cast<int>(cfg_.ffn_hidden * 2 / 3);
  d_.V = static_cast<int>(cfg_.vocab);
  d_.n = static_cast<int>(cfg_.n_layers);
  d_.t = static_cast<int>(cfg_.tp_degree);
  d_.r = comm_ ? comm_->rank() : 0;
  if (opt_.cuda_graph && d_.t > 1 && !(comm_ && comm_->graph_capturable()))
    throw ConfigError("cuda_graph at tp_degree > 1 needs a stream-only communicator (CUDA-IPC peer memory); "
                      "the loopback and in-process peer groups rendezvous on the host");
  if (d_.t > 1 && (!comm_ || comm_->size() != d_.t) && !opt_.dry_run)
    throw ConfigError("tp_degree > 1 needs a communicator of that size");
  if (d_.h % d_.H || (d_.D != 64 && d_.D != 128)) throw ConfigError("head_dim must be 64 or 128");
  if (d_.S % 128 || d_.h % 256 || d_.F % 256 || d_.V % 256)
    throw ConfigError("seq_len % 128, hidden % 256, intermediate % 256 and vocab % 256 must be 0");
  if (d_.S % (128 * d_.t) || d_.H % d_.t || d_.F % (32 * d_.t) || d_.V % (32 * d_.t))
    throw ConfigError("seq_len/(128 t), heads/t, intermediate/(32 t) and vocab/(32 t) must be whole");
  d_.Sl = d_.S / d_.t;
  d_.Hl = d_.H / d_.t;
  d_.hl = d_.Hl * d_.D;
  d_.Fl = d_.F / d_.t;
  d_.Vl = d_.V / d_.t;
  if (opt_.ce_chunk <= 0 || opt_.ce_chunk % 128) throw ConfigError("ce_chunk must be a positive multiple of 128");

  // The executor's saved tensors define the skeletal weights (multiples of
  // b*s*(h/t)*dtype bytes per device); LSE (f32 [H/t, S]) rides in attn_out.
  // Sequence-sharded components hold S/t rows of full width, head-sharded ones
  // S rows of width/t — the same bytes, hence the same weights for every t.
  const double h = d_.h, F = d_.F;
  row_bytes_ = {4ull * d_.h,  2ull * d_.h,  2ull * d_.hl, 2ull * d_.hl, 2ull * d_.hl,
                2ull * d_.hl, 2ull * d_.h,  2ull * d_.h,  4ull * d_.Fl, 2ull * d_.Fl};
  const double w[C_N] = {2.0, 1.0, 1.0, 1.0, 1.0, 1.0 + 2.0 / d_.D, 1.0, 1.0, 2.0 * F / h, F / h};
  cfg_.skeletal_weight_overrides.clear();
  for (int c = 0; c < C_N; ++c) cfg_.skeletal_weight_overrides[kSkeletalNames[c]] = w[c];
  sk_ = skeletal_of(cfg_);
  rb_bytes_ = 0;
  rb_off_.resize(C_N);
  for (int c = 0; c < C_N; ++c) {
    rb_off_[c] = rb_bytes_;
    rb_bytes_ += sk_.components[c].second;
  }
  {
    const Bytes want = static_cast<Bytes>(d_.Sl) * (4ull * d_.h + 2ull * d_.h * 3) +
                       static_cast<Bytes>(d_.S) * (2ull * d_.hl * 4 + 6ull * d_.Fl) +
                       4ull * d_.Hl * d_.S;
    if (want != rb_bytes_) throw PlanError(1, "internal: skeletal model does not match executor layout");
  }

  // alpha and the token split (swap.hpp:105, schedule.hpp:409, swap.hpp:177);
  // sequence-sharded components split their S/t local rows (SURVEY §7 hard part v).
  Timing tm = timing_of(cfg_, hw_, params_of(cfg_));
  const double t_layer = opt_.t_layer > 0 ? opt_.t_layer : tm.t_fwd_layer;
  swap_ = opt_.alpha >= 0 ? swap_with_alpha(sk_, hw_, opt_.alpha, cfg_.n_layers)
                          : solve_alpha_for(sk_, hw_, t_layer, cfg_.n_layers);
  split_ = split_tokens(swap_.alpha, cfg_.seq_local(), opt_.token_granularity);
  split_l_ = split_tokens(swap_.alpha, static_cast<std::uint64_t>(d_.Sl), opt_.token_granularity);
  can_swap_ = swap_on_ = opt_.swap_enabled;

  build_trace_and_plan();
  compute_layout();
  if (opt_.dry_run) return;  // host-only: trace, plan, alpha and sizes (no CUDA)
  allocate();
  init_weights();
}

const TokenRange& Executor::split_of(int c) const {
  return (c == C_X || c == C_XN || c == C_A || c == C_XN2) ? split_l_ : split_;
}

void Executor::build_trace_and_plan() {
  const Bytes S = d_.S, h = d_.h, F = d_.F, V = d_.V, H = d_.H;
  const Bytes T = std::min<Bytes>(static_cast<Bytes>(opt_.ce_chunk), S);
  const Bytes P = static_cast<Bytes>(rmsnorm_bwd_partials(d_.S));
  const Bytes R = split_.recompute_tokens;
  TraceBuilder tb;
  if (d_.t > 1) {
    build_trace_tp(tb);
  } else {
  seg_emb_fwd_ = tb.begin(Phase::EmbFwd, -1);
  tb.malloc("x_final", S * h * 4, "x_final");
  tb.malloc("dx_carry", S * h * 4, "dx_carry");
  tb.malloc("dxb_carry", S * h * 2, "dxb_carry");
  for (int i = 0; i < d_.n; ++i) {
    seg_fwd_.push_back(tb.begin(Phase::LayerFwd, i));
    for (int c = 0; c <= C_A; ++c)
      tb.malloc(lkey(i, kSkeletalNames[c]), sk_.components[c].second, kSkeletalNames[c]);
    tb.malloc(lkey(i, "x1"), S * h * 4, "x1");
    for (int c = C_XN2; c < C_N; ++c)
      tb.malloc(lkey(i, kSkeletalNames[c]), sk_.components[c].second, kSkeletalNames[c]);
    tb.free(lkey(i, "x1"));
  }
  seg_cls_fwd_ = tb.begin(Phase::ClsFwd, -1);
  tb.malloc("xf", S * h * 2, "xf");
  seg_cls_bwd_ = tb.begin(Phase::ClsBwd, -1);
  tb.malloc("dxf", S * h * 4, "dxf");
  tb.malloc("loss_rows", S * 4, "loss_rows");
  tb.malloc("logits", T * V * 4, "logits");
  tb.malloc("dlogits", T * V * 2, "dlogits");
  tb.free("logits");
  tb.free("dlogits");
  tb.free("loss_rows");
  tb.malloc("cls_part", P * h * 4, "cls_part");
  tb.free("cls_part");
  tb.free("dxf");
  tb.free("xf");
  seg_bwd_.assign(d_.n, 0);
  for (int i = d_.n - 1; i >= 0; --i) {
    seg_bwd_[i] = tb.begin(Phase::LayerBwd, i);
    auto m = [&](const char* n, Bytes b) { tb.malloc(lkey(i, n), b, n); };
    auto f = [&](const char* n) { tb.free(lkey(i, n)); };
    if (R > 0) {  // every layer carries the recompute buffer so segments stay identical
      m("x1_rec", R * h * 4);
      f("x1_rec");
    }
    m("dact", S * F * 2);
    m("dgu", S * 2 * F * 2);
    f("dact");
    m("dxn2", S * h * 4);
    f("dgu");
    m("da", S * h * 2);
    m("part2", P * h * 4);
    f("part2");
    f("dxn2");
    m("dout", S * h * 2);
    f("da");
    m("attn_ws", attn_bwd_workspace_bytes(static_cast<int>(S), static_cast<int>(H), d_.D));
    m("dqkv", S * 3 * h * 2);
    f("attn_ws");
    f("dout");
    m("dxn", S * h * 4);
    f("dqkv");
    m("part1", P * h * 4);
    f("part1");
    f("dxn");
    for (int c = C_N - 1; c >= 0; --c) tb.free(lkey(i, kSkeletalNames[c]));
  }
  seg_emb_bwd_ = tb.begin(Phase::EmbBwd, -1);
  tb.free("dxb_carry");
  tb.free("dx_carry");
  tb.free("x_final");
  }
  Trace& t = tb.trace();
  t.n_layers = d_.n;
  trace_text_ = trace_to_text(t);
  ModelPlan mp = plan_iteration(t, 0, opt_.plan_time_budget, opt_.alignment);
  plan_json_ = plan_to_json(mp);
  if (!mp.optimal) throw PlanningError("bi-level plan not proven optimal within the time budget");
  arena_bytes_ = mp.total_peak;
  for (const AbsAddr& a : mp.absolute) {
    const auto& nm = tb.names().at(a.id);
    arena_off_[{a.segment, nm.second}] = a.offset;
    req_name_[{a.segment, a.id}] = nm.second;
  }
}

// Replay an externally computed plan (SURVEY §8b memo_bind_plan): the text is
// to_json(GlobalPlan).dump() (json_io.hpp:189-202) of a plan of THIS executor's
// trace, e.g. the reference's own actmem::plan_model(parse_trace(trace_text())).
// Refused (status 2) unless it places exactly the executor's transient requests
// (same (segment, tensor) set), at offsets that are multiples of the alignment, with
// no two requests whose lifespans overlap (trace.hpp:146 lifespans over the
// whole iteration) sharing bytes; status 3 if its total_peak exceeds the arena
// reserved at creation (allocator.hpp:264-285: the plan never grows the
// reservation).  On success every arena pointer of later steps follows the
// bound offsets.  Refused once the step has been captured as a CUDA graph
// (cuda_graph=1 captures the second step; the graph bakes the pointers).
void Executor::bind_plan(const std::string& text) {
  if (graph_exec_ || capturing_)
    throw ConfigError("bind_plan: the step is already captured as a CUDA graph (its pointers are baked)");
  Bytes peak = 0;
  std::map<std::pair<std::size_t, TensorId>, Bytes> off;
  std::string canonical = parse_plan_json(text, &peak, &off);
  if (off.size() != req_name_.size())
    throw ConfigError("bind_plan: plan places " + std::to_string(off.size()) + " tensors, the executor's trace has " +
                      std::to_string(req_name_.size()) + " transient requests");
  for (const auto& kv : off)
    if (!req_name_.count(kv.first))
      throw ConfigError("bind_plan: tensor " + std::to_string(kv.first.second) + " of segment " +
                        std::to_string(kv.first.first) + " is not a transient request of this executor");
  if (peak > arena_bytes_)
    throw InfeasibleError("bind_plan: total_peak " + std::to_string(peak) + " exceeds the reserved arena " +
                          std::to_string(arena_bytes_));
  // lifespans over the whole iteration; every placed request checked
  const Trace t = parse_trace_text(trace_text_);
  std::vector<Lifespan> spans = lifespans_of(t.segs.data(), t.segs.size(), false);
  std::map<TensorId, std::size_t> seg_of;
  for (const auto& kv : req_name_) seg_of[kv.first.second] = kv.first.first;
  struct Item {
    Lifespan l;
    Bytes lo, hi;
  };
  std::vector<Item> items;
  const Bytes al = opt_.alignment ? opt_.alignment : 1;
  for (const Lifespan& l : spans) {
    auto it = seg_of.find(l.id);
    if (it == seg_of.end()) continue;  // skeletal: rounding buffers, not the arena
    const Bytes o = off.at({it->second, l.id});
    const Bytes sz = (l.size + al - 1) / al * al;
    if (o % al) throw ConfigError("bind_plan: offset of tensor " + std::to_string(l.id) + " not aligned");
    if (o + sz > peak)
      throw ConfigError("bind_plan: tensor " + std::to_string(l.id) + " ends past total_peak");
    items.push_back({l, o, o + sz});
  }
  for (std::size_t a = 0; a < items.size(); ++a)
    for (std::size_t b = a + 1; b < items.size() && items[b].l.first < items[a].l.last; ++b)
      if (items[a].l.overlaps(items[b].l) && items[a].lo < items[b].hi && items[b].lo < items[a].hi)
        throw ConfigError("bind_plan: tensors " + std::to_string(items[a].l.id) + " and " +
                          std::to_string(items[b].l.id) + " are live together and share bytes");
  for (const auto& kv : off) arena_off_[{kv.first.first, req_name_.at(kv.first)}] = kv.second;
  plan_json_ = canonical;
}

// SP+TP request trace of one rank (same segment structure; every layer
// segment identical so the bi-level plan stays provably optimal).
void Executor::build_trace_tp(TraceBuilder& tb) {
  const Bytes S = d_.S, Sl = d_.Sl, h = d_.h, hl = d_.hl, Fl = d_.Fl, Vl = d_.Vl, Hl = d_.Hl;
  const Bytes T = std::min<Bytes>(static_cast<Bytes>(opt_.ce_chunk), S);
  const Bytes P = static_cast<Bytes>(rmsnorm_bwd_partials(d_.Sl));
  const Bytes R = split_.recompute_tokens;
  seg_emb_fwd_ = tb.begin(Phase::EmbFwd, -1);
  tb.malloc("x_final", Sl * h * 4, "x_final");
  tb.malloc("dx_carry", Sl * h * 4, "dx_carry");
  tb.malloc("dxb_carry", Sl * h * 2, "dxb_carry");
  auto sk = [&](int i, int c) { tb.malloc(lkey(i, kSkeletalNames[c]), sk_.components[c].second, kSkeletalNames[c]); };
  for (int i = 0; i < d_.n; ++i) {
    seg_fwd_.push_back(tb.begin(Phase::LayerFwd, i));
    auto m = [&](const char* n, Bytes b) { tb.malloc(lkey(i, n), b, n); };
    auto f = [&](const char* n) { tb.free(lkey(i, n)); };
    sk(i, C_X);
    sk(i, C_XN);
    m("xn_full", S * h * 2);
    sk(i, C_Q);
    sk(i, C_K);
    sk(i, C_V);
    f("xn_full");
    sk(i, C_O);
    m("a_part", Sl * h * 4);
    m("a_red", Sl * h * 4);
    f("a_part");
    sk(i, C_A);
    m("x1", Sl * h * 4);
    f("a_red");
    sk(i, C_XN2);
    m("xn2_full", S * h * 2);
    sk(i, C_GU);
    sk(i, C_ACT);
    f("xn2_full");
    m("d_part", Sl * h * 4);
    m("d_red", Sl * h * 4);
    f("d_part");
    f("d_red");
    f("x1");
  }
  seg_cls_fwd_ = tb.begin(Phase::ClsFwd, -1);
  tb.malloc("xf", Sl * h * 2, "xf");
  seg_cls_bwd_ = tb.begin(Phase::ClsBwd, -1);
  tb.malloc("xf_full", S * h * 2, "xf_full");
  tb.malloc("dxf_part", S * h * 4, "dxf_part");
  tb.malloc("loss_rows", S * 4, "loss_rows");
  tb.malloc("logits", T * Vl * 4, "logits");
  tb.malloc("dlogits", T * Vl * 2, "dlogits");
  tb.malloc("ce_stats", 6 * T * 4, "ce_stats");
  tb.free("ce_stats");
  tb.free("logits");
  tb.free("dlogits");
  tb.free("loss_rows");
  tb.free("xf_full");
  tb.malloc("dxf", Sl * h * 4, "dxf");
  tb.free("dxf_part");
  tb.malloc("cls_part", P * h * 4, "cls_part");
  tb.free("cls_part");
  tb.free("dxf");
  tb.free("xf");
  seg_bwd_.assign(d_.n, 0);
  for (int i = d_.n - 1; i >= 0; --i) {
    seg_bwd_[i] = tb.begin(Phase::LayerBwd, i);
    auto m = [&](const char* n, Bytes b) { tb.malloc(lkey(i, n), b, n); };
    auto f = [&](const char* n) { tb.free(lkey(i, n)); };
    if (R > 0) {  // recompute transients, carried by every layer
      m("r_xn_full", S * h * 2);
      f("r_xn_full");
      m("r_a_part", Sl * h * 4);
      m("r_a_red", Sl * h * 4);
      f("r_a_part");
      m("r_x1", Sl * h * 4);
      f("r_a_red");
      m("r_xn2_full", S * h * 2);
      f("r_xn2_full");
      f("r_x1");
    }
    m("dy_full", S * h * 2);
    m("dact", S * Fl * 2);
    m("dgu", S * 2 * Fl * 2);
    f("dact");
    m("dxn2_part", Sl * h * 4);
    m("dxn2", Sl * h * 4);
    f("dxn2_part");
    m("b_xn2_full", S * h * 2);
    f("b_xn2_full");
    f("dgu");
    f("dy_full");
    m("da", Sl * h * 2);
    m("part2", P * h * 4);
    f("part2");
    f("dxn2");
    m("da_full", S * h * 2);
    m("dout", S * hl * 2);
    f("da");
    f("da_full");
    m("attn_ws", attn_bwd_workspace_bytes(static_cast<int>(S), static_cast<int>(Hl), d_.D));
    m("dqkv", S * 3 * hl * 2);
    f("attn_ws");
    f("dout");
    m("dxn_part", Sl * h * 4);
    m("dxn", Sl * h * 4);
    f("dxn_part");
    m("b_xn_full", S * h * 2);
    f("b_xn_full");
    f("dqkv");
    m("part1", P * h * 4);
    f("part1");
    f("dxn");
    for (int c = C_N - 1; c >= 0; --c) tb.free(lkey(i, kSkeletalNames[c]));
  }
  seg_emb_bwd_ = tb.begin(Phase::EmbBwd, -1);
  tb.malloc("ar_tmp", static_cast<Bytes>(d_.V) * h * 4, "ar_tmp");
  tb.free("ar_tmp");
  tb.free("dxb_carry");
  tb.free("dx_carry");
  tb.free("x_final");
}

void* Executor::arena_ptr(std::size_t seg, const char* name) const {
  auto it = arena_off_.find({seg, name});
  if (it == arena_off_.end()) throw PlanError(1, std::string("internal: no arena slot for ") + name);
  return arena_ + it->second;
}

void Executor::compute_layout() {
  const long long h = d_.h, V = d_.V, hl = d_.hl, Fl = d_.Fl, Vl = d_.Vl;
  long long off = 0;
  auto add = [&](const std::string& n, int layer, long long cnt) {
    ptab_[{n, layer}] = {off, cnt};
    off += cnt;
  };
  // local shards: Wqkv/Wgu column-parallel, Wo/Wd row-parallel, Wcls
  // vocab-parallel; embedding and norm weights replicated (t = 1: full tensors)
  add("embedding", -1, V * h);
  for (int l = 0; l < d_.n; ++l) {
    add("g1", l, h);
    add("wqkv", l, 3 * hl * h);
    add("wo", l, h * hl);
    add("g2", l, h);
    add("wgu", l, 2 * Fl * h);
    add("wd", l, h * Fl);
  }
  add("gf", -1, h);
  add("wcls", -1, Vl * h);
  n_params_ = off;
  const Bytes Pn = static_cast<Bytes>(n_params_);
  const Bytes sz_params = up(Pn * 2), sz_f32 = up(Pn * 4);
  // optimizer off: no f32 master / Adam moments (bf16 params + f32 grads only)
  state_bytes_ = sz_params + (opt_.optimizer ? 4 : 1) * sz_f32;
  const Bytes S = d_.S;
  const Bytes misc = up(S * (d_.D / 2) * 8 + S * 4 * 3 + (V + 1) * 4 + 1024);
  const int n_rb = swap_on_ ? 2 : d_.n;
  dev_bytes_ = state_bytes_ + n_rb * up(rb_bytes_) + up(arena_bytes_) + misc;
  // pinned host slots for the n-2 swapped layers
  host_slot_.assign(d_.n, 0);
  per_layer_host_ = sk_.components[C_X].second + sk_.components[C_O].second;
  for (int c = 0; c < C_N; ++c)
    if (c != C_X && c != C_O) per_layer_host_ += split_of(c).swap_tokens * row_bytes_[c];
  const int swapped = d_.n >= 3 ? d_.n - 2 : 0;
  pinned_bytes_ = can_swap_ ? per_layer_host_ * swapped : 0;
  for (int i = 0; i < swapped; ++i) host_slot_[i] = per_layer_host_ * i;
}

void Executor::allocate() {
  const Bytes Pn = static_cast<Bytes>(n_params_);
  const Bytes sz_params = up(Pn * 2), sz_f32 = up(Pn * 4);
  const Bytes S = d_.S;
  const long long V = d_.V;
  const int n_rb = swap_on_ ? 2 : d_.n;
  size_t free_b = 0, total_b = 0;
  ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  const Bytes reserve = 1ull << 30;  // cuBLAS-free, but leave room for the CUDA context / TMA maps
  if (dev_bytes_ + reserve > free_b)
    throw InfeasibleError("arena " + std::to_string(arena_bytes_) + " + rounding buffers " +
                          std::to_string(n_rb * rb_bytes_) + " + states " + std::to_string(state_bytes_) +
                          " exceed free HBM " + std::to_string(free_b));
  void* p = nullptr;
  ck(cudaMalloc(&p, dev_bytes_), "cudaMalloc(arena)");
  dev_ = static_cast<char*>(p);
  char* q = dev_;
  params_ = reinterpret_cast<__nv_bfloat16*>(q); q += sz_params;
  if (opt_.optimizer) {
    master_ = reinterpret_cast<float*>(q); q += sz_f32;
    adam_m_ = reinterpret_cast<float*>(q); q += sz_f32;
    adam_v_ = reinterpret_cast<float*>(q); q += sz_f32;
  }
  grads_ = reinterpret_cast<float*>(q); q += sz_f32;
  rb_base_.assign(n_rb, nullptr);
  for (int r = 0; r < n_rb; ++r) {
    rb_base_[r] = q;
    q += up(rb_bytes_);
  }
  arena_ = q; q += up(arena_bytes_);
  rope_ = reinterpret_cast<float2*>(q); q += S * (d_.D / 2) * 8;
  tok_ = reinterpret_cast<int*>(q); q += S * 4;
  lab_ = reinterpret_cast<int*>(q); q += S * 4;
  csr_pos_ = reinterpret_cast<int*>(q); q += S * 4;
  csr_off_ = reinterpret_cast<int*>(q); q += (V + 1) * 4;
  inv_n_dev_ = reinterpret_cast<float*>(q); q += 4;
  loss_dev_ = reinterpret_cast<float*>(up(reinterpret_cast<uintptr_t>(q), 256));
  adam_ctr_ = reinterpret_cast<int*>(loss_dev_ + 16);
  adam_c12_ = reinterpret_cast<float2*>(loss_dev_ + 32);
  ck(cudaMemset(adam_ctr_, 0, sizeof(int)), "memset(adam step)");

  if (pinned_bytes_ > 0) {
    void* hp = nullptr;
    if (cudaHostAlloc(&hp, pinned_bytes_, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      throw CpuInfeasibleError("cannot pin " + std::to_string(pinned_bytes_) +
                               " bytes of host memory for the swap slots");
    }
    pinned_ = static_cast<char*>(hp);
  }
  void* sp = nullptr;
  ck(cudaHostAlloc(&sp, S * 4 * 3 + (V + 1) * 4 + 4 + 64, cudaHostAllocDefault), "cudaHostAlloc(staging)");
  staging_ = static_cast<char*>(sp);
  loss_host_ = reinterpret_cast<float*>(staging_ + S * 4 * 3 + (V + 1) * 4 + 4);

  ck(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&os_, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&ps_, cudaStreamNonBlocking), "stream");
  auto mk = [&](std::vector<cudaEvent_t>& v) {
    v.resize(d_.n);
    for (auto& e : v) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  };
  mk(ev_fwd_done_);
  mk(ev_bwd_done_);
  mk(ev_off_done_);
  mk(ev_off_x_);
  mk(ev_pre_mand_);
  mk(ev_pre_done_);
  ck(cudaEventCreate(&ev_start_), "event");
  ck(cudaEventCreateWithFlags(&ev_staging_, cudaEventDisableTiming), "event");
  for (cudaEvent_t* e : {&ev_fork_, &ev_join_os_, &ev_join_ps_})
    ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  if (comm_ && d_.t > 1) {
    comm_->attach(dev_, dev_bytes_);  // peer backends: the single allocation is the symmetric heap
    ck(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking), "stream");
    xcs_.resize(d_.t - 1);  // one pull stream per peer block: the copy engines work in parallel
    for (auto& st : xcs_) ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    ev_blk_.resize(d_.t);
    for (auto& e : ev_blk_) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_cs2xs_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_xs2cs_, cudaEventDisableTiming), "event");
  }

  // RoPE table (cos, sin) in double -> f32, identical to the CPU oracle.
  std::vector<float2> cs(static_cast<size_t>(S) * (d_.D / 2));
  for (Bytes t = 0; t < S; ++t)
    for (int p2 = 0; p2 < d_.D / 2; ++p2) {
      const double inv = std::pow(static_cast<double>(opt_.rope_theta), -2.0 * p2 / d_.D);
      const double ang = static_cast<double>(t) * inv;
      cs[t * (d_.D / 2) + p2] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
    }
  ck(cudaMemcpy(rope_, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice), "rope upload");
}

void Executor::init_weights() {
  for (const auto& [key, v] : ptab_) {
    const auto& [name, layer] = key;
    const auto [o, n] = v;
    uint64_t tid;
    if (name == "embedding") tid = 0;
    else if (name == "gf") tid = 1 + 6ull * d_.n;
    else if (name == "wcls") tid = 2 + 6ull * d_.n;
    else {
      static const char* order[] = {"g1", "wqkv", "wo", "g2", "wgu", "wd"};
      int k = 0;
      while (name != order[k]) ++k;
      tid = 1 + 6ull * layer + k;
    }
    const bool is_norm = name == "g1" || name == "g2" || name == "gf";
    const long long h = d_.h, hl = d_.hl, Fl = d_.Fl, Vl = d_.Vl, r = d_.r;
    if (d_.t == 1 || name == "embedding" || is_norm) {
      ck(init_uniform(params_ + o, master_ ? master_ + o : nullptr, n, opt_.seed, tid, is_norm, cs_), "init_uniform");
      continue;
    }
    // shard of the full tensor: same counter-hash values as the unsharded init
    long long l0[3] = {0, 0, 0}, cnt[3] = {0, 0, 0}, g0[3] = {0, 0, 0};
    int nseg = 1;
    long long R = 0, Cl = 0, Cg = 0, coff = 0;
    if (name == "wqkv") {
      R = 3 * hl; Cl = h; Cg = h; nseg = 3;
      for (int k = 0; k < 3; ++k) { l0[k] = k * hl; cnt[k] = hl; g0[k] = k * h + r * hl; }
    } else if (name == "wo") {
      R = h; Cl = hl; Cg = h; coff = r * hl; cnt[0] = h;
    } else if (name == "wgu") {
      R = 2 * Fl; Cl = h; Cg = h; nseg = 2;
      for (int k = 0; k < 2; ++k) { l0[k] = k * Fl; cnt[k] = Fl; g0[k] = k * static_cast<long long>(d_.F) + r * Fl; }
    } else if (name == "wd") {
      R = h; Cl = Fl; Cg = d_.F; coff = r * Fl; cnt[0] = h;
    } else {  // wcls
      R = Vl; Cl = h; Cg = h; cnt[0] = Vl; g0[0] = r * Vl;
    }
    ck(init_sliced(params_ + o, master_ ? master_ + o : nullptr, R, Cl, l0, cnt, g0, nseg, Cg, coff, opt_.seed, tid,
                   false, cs_), "init_sliced");
  }
  if (opt_.optimizer) {
    ck(cudaMemsetAsync(adam_m_, 0, n_params_ * 4, cs_), "memset");
    ck(cudaMemsetAsync(adam_v_, 0, n_params_ * 4, cs_), "memset");
  }
  ck(cudaStreamSynchronize(cs_), "init sync");
}

Executor::~Executor() {
  if (opt_.dry_run) return;
  if (cs_) cudaStreamSynchronize(cs_);
  if (os_) cudaStreamSynchronize(os_);
  if (ps_) cudaStreamSynchronize(ps_);
  if (xs_) cudaStreamSynchronize(xs_);
  for (auto* v : {&ev_fwd_done_, &ev_bwd_done_, &ev_off_done_, &ev_off_x_, &ev_pre_mand_, &ev_pre_done_, &ev_pool_, &ev_blk_})
    for (auto e : *v) cudaEventDestroy(e);
  for (auto e : {ev_cs2xs_, ev_xs2cs_})
    if (e) cudaEventDestroy(e);
  if (xs_) cudaStreamDestroy(xs_);
  for (auto st : xcs_) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (ev_start_) cudaEventDestroy(ev_start_);
  if (ev_staging_) cudaEventDestroy(ev_staging_);
  for (cudaEvent_t e : {ev_fork_, ev_join_os_, ev_join_ps_})
    if (e) cudaEventDestroy(e);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  if (cs_) cudaStreamDestroy(cs_);
  if (os_) cudaStreamDestroy(os_);
  if (ps_) cudaStreamDestroy(ps_);
  if (dev_) cudaFree(dev_);
  if (pinned_) cudaFreeHost(pinned_);
  if (staging_) cudaFreeHost(staging_);
}

cudaEvent_t Executor::take_event() {
  if (ev_used_ == ev_pool_.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_used_++];
}

// A wait of the compute stream on a copy event INSIDE a layer (the layer_input
// rows of the previous layer's offload, before the down projection writes the
// next layer's input over them).  The measured timeline cannot see it (it sits
// between a layer's begin/end marks), so it is bracketed by two timing events
// on the compute stream; their distance is the stall, reported as copy_wait_ms
// and added to the exposed swap time.
void Executor::copy_wait(cudaEvent_t ev) {
  cudaEvent_t a = take_event(), b = take_event();
  ck(record_timing_event(a, cs_), "record");
  ck(cudaStreamWaitEvent(cs_, ev, 0), "wait");
  ck(record_timing_event(b, cs_), "record");
  waits_.push_back({a, b});
}

void Executor::gemm(const GemmDesc& g) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (opt_.op_timing) {
    a = take_event();
    b = take_event();
    ck(record_timing_event(a, cs_), "record");
  }
  ck(gemm_tc(g, cs_), "gemm_tc");
  stats_.kernel_launches += 1;
  if (opt_.op_timing) {
    ck(record_timing_event(b, cs_), "record");
    ops_.push_back({OP_GEMM, a, b, 2.0 * g.M * static_cast<double>(g.N) * g.K});
  }
}

void Executor::attention_fwd(AttnFwdArgs a) {
  if (opt_.op_timing) {
    a.ev[0] = take_event();
    a.ev[1] = take_event();
  }
  ck(attn_fwd(a, cs_), "attn_fwd");
  stats_.kernel_launches += 1;
  if (opt_.op_timing) {
    const double s = a.S, hh = static_cast<double>(a.H) * a.D;
    ops_.push_back({OP_ATTN_FWD, a.ev[0], a.ev[1], 2.0 * s * s * hh});  // causal 2*s^2*h
  }
}

void Executor::attention_bwd(AttnBwdArgs a) {
  if (opt_.op_timing)
    for (auto& e : a.ev) e = take_event();
  ck(attn_bwd(a, cs_), "attn_bwd");
  stats_.kernel_launches += 3;
  if (opt_.op_timing) {
    const double s = a.S, hh = static_cast<double>(a.H) * a.D;
    ops_.push_back({OP_ATTN_PREP, a.ev[0], a.ev[1], 0.0});
    ops_.push_back({OP_ATTN_DKDV, a.ev[1], a.ev[2], 4.0 * s * s * hh});  // S^T, dP^T, dV, dK
    ops_.push_back({OP_ATTN_DQ, a.ev[2], a.ev[3], 3.0 * s * s * hh});    // S, dP, dQ
  }
}

void Executor::mark(int stream, int kind, int layer, bool begin) {
  cudaStream_t s = stream == 0 ? cs_ : (stream == 1 ? os_ : ps_);
  cudaEvent_t e = take_event();
  ck(record_timing_event(e, s), "eventRecord");
  if (begin) {
    marks_.push_back({stream, kind, layer, e, nullptr});
  } else {
    for (auto it = marks_.rbegin(); it != marks_.rend(); ++it)
      if (it->stream == stream && it->kind == kind && it->layer == layer && !it->e) {
        it->e = e;
        break;
      }
  }
}

bool Executor::tensor(const std::string& name, int layer, void** ptr, size_t* bytes) const {
  std::string base = name;
  char* arr = reinterpret_cast<char*>(params_);
  size_t esz = 2;
  if (name.rfind("grad/", 0) == 0) {
    base = name.substr(5);
    arr = reinterpret_cast<char*>(grads_);
    esz = 4;
  } else if (name.rfind("master/", 0) == 0) {
    if (!master_) return false;
    base = name.substr(7);
    arr = reinterpret_cast<char*>(master_);
    esz = 4;
  }
  if (base == "all") {
    *ptr = arr;
    *bytes = static_cast<size_t>(n_params_) * esz;
    return true;
  }
  if (name.rfind("act/", 0) == 0) {  // skeletal activation component of a layer's RB
    for (int c = 0; c < C_N; ++c)
      if (name.substr(4) == kSkeletalNames[c] && layer >= 0 && layer < d_.n) {
        *ptr = comp(layer, c);
        *bytes = sk_.components[c].second;
        return true;
      }
    return false;
  }
  auto it = ptab_.find({base, layer});
  if (it == ptab_.end()) return false;
  *ptr = arr + it->second.first * esz;
  *bytes = static_cast<size_t>(it->second.second) * esz;
  return true;
}

// ------------------------------------------------------------------ step
namespace {
GemmDesc gd(int M, int N, int K, const void* a, long long lda, int amn, const void* b,
            long long ldb, int bmn, int epi, void* c, long long ldc) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.a = a;
  g.lda = lda;
  g.a_mn_major = amn;
  g.b = b;
  g.ldb = ldb;
  g.b_mn_major = bmn;
  g.epi = epi;
  g.c = c;
  g.ldc = ldc;
  return g;
}
}  // namespace

void Executor::load_batch(const int* tokens, const int* labels) {
  const int S = d_.S, V = d_.V;
  for (int t = 0; t < S; ++t) {
    if (tokens[t] < 0 || tokens[t] >= V) throw ConfigError("token id out of range");
    if (labels[t] >= V) throw ConfigError("label out of range");
  }
  int nl = 0;
  for (int t = 0; t < S; ++t) nl += labels[t] >= 0;
  if (nl == 0) throw ConfigError("batch has no labeled tokens");
  // The previous batch's H2D may still be queued on cs_ behind a running step:
  // staging_ is rewritten only after it has left.
  ck(cudaEventSynchronize(ev_staging_), "staging reuse");
  int* st = reinterpret_cast<int*>(staging_);
  std::memcpy(st, tokens, S * 4);
  std::memcpy(st + S, labels, S * 4);
  // counting sort of positions by token id -> CSR for the deterministic embedding gradient
  int* pos = st + 2 * S;
  int* offs = st + 3 * S;
  std::fill(offs, offs + V + 1, 0);
  // embedding-gradient CSR over this rank's token shard (positions are local rows)
  const int t0 = d_.r * d_.Sl, t1 = t0 + d_.Sl;
  for (int t = t0; t < t1; ++t) ++offs[tokens[t] + 1];
  for (int v = 0; v < V; ++v) offs[v + 1] += offs[v];
  std::vector<int> fillp(offs, offs + V);
  for (int t = t0; t < t1; ++t) pos[fillp[tokens[t]]++] = t - t0;
  n_labeled_ = nl;
  reinterpret_cast<float*>(offs + V + 1)[0] = 1.0f / static_cast<float>(nl);
  // tok | lab | csr_pos | csr_off | inv_n are contiguous on both sides
  ck(cudaMemcpyAsync(tok_, staging_, static_cast<size_t>(3 * S + V + 2) * 4, cudaMemcpyHostToDevice, cs_),
     "H2D batch");
  ck(cudaEventRecord(ev_staging_, cs_), "record");
  stats_.h2d_bytes = static_cast<double>(3 * S + V + 2) * 4;
}

void Executor::offload(int i) {
  ck(cudaStreamWaitEvent(os_, ev_fwd_done_[i], 0), "wait");
  mark(1, static_cast<int>(Kind::Offload), i, true);
  // Host slot layout (shared with prefetch): [layer_input | attn_out(+LSE) |
  // prefix rows of the other components in emission order].
  char* host = pinned_ + host_slot_[i];
  Bytes moved = 0;
  auto put = [&](int c, Bytes b) {
    if (b == 0) return;
    ck(cudaMemcpyAsync(host, comp(i, c), b, cudaMemcpyDeviceToHost, os_), "D2H offload");
    host += b;
    moved += b;
  };
  put(C_X, sk_.components[C_X].second);
  ck(cudaEventRecord(ev_off_x_[i], os_), "record");  // layer_input out: RB(i) may take layer i+2's input
  put(C_O, sk_.components[C_O].second);
  for (int c = 0; c < C_N; ++c)
    if (c != C_X && c != C_O) put(c, split_of(c).swap_tokens * row_bytes_[c]);
  stats_.offload_bytes += static_cast<double>(moved);
  mark(1, static_cast<int>(Kind::Offload), i, false);
  ck(cudaEventRecord(ev_off_done_[i], os_), "record");
}

void Executor::prefetch(int i) {
  ck(cudaStreamWaitEvent(ps_, ev_bwd_done_[i + 2], 0), "wait");
  mark(2, static_cast<int>(Kind::Prefetch), i, true);
  const char* host = pinned_ + host_slot_[i];
  Bytes moved = 0;
  // mandatory first (layer input, attention output + LSE): recompute needs them
  const Bytes bx = sk_.components[C_X].second, bo = sk_.components[C_O].second;
  ck(cudaMemcpyAsync(comp(i, C_X), host, bx, cudaMemcpyHostToDevice, ps_), "H2D");
  ck(cudaMemcpyAsync(comp(i, C_O), host + bx, bo, cudaMemcpyHostToDevice, ps_), "H2D");
  ck(cudaEventRecord(ev_pre_mand_[i], ps_), "record");
  moved += bx + bo;
  const char* hp = host + bx + bo;
  for (int c = 0; c < C_N; ++c) {
    if (c == C_X || c == C_O) continue;
    const Bytes b = split_of(c).swap_tokens * row_bytes_[c];
    if (b == 0) continue;
    ck(cudaMemcpyAsync(comp(i, c), hp, b, cudaMemcpyHostToDevice, ps_), "H2D");
    hp += b;
    moved += b;
  }
  stats_.prefetch_bytes += static_cast<double>(moved);
  mark(2, static_cast<int>(Kind::Prefetch), i, false);
  ck(cudaEventRecord(ev_pre_done_[i], ps_), "record");
}

#define G(expr) ck(expr, #expr)

void Executor::layer_fwd(int i) {
  const int S = d_.S, h = d_.h, F = d_.F, H = d_.H, D = d_.D;
  if (i >= 2 && swaps(i - 2)) G(cudaStreamWaitEvent(cs_, ev_off_done_[i - 2], 0));  // F3
  mark(0, static_cast<int>(Kind::LayerFwd), i, true);
  const std::size_t seg = seg_fwd_[i];
  auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
  float* X = reinterpret_cast<float*>(comp(i, C_X));
  auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN));
  auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q));
  auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K));
  auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V));
  auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O));
  float* LSE = reinterpret_cast<float*>(comp(i, C_O) + static_cast<Bytes>(S) * h * 2);
  auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A));
  auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2));
  auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU));
  auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT));
  float* x1 = static_cast<float*>(arena_ptr(seg, "x1"));

  G(rmsnorm_fwd(X, nullptr, P("g1"), XN, S, h, opt_.eps, cs_));
  GemmDesc g = gd(S, 3 * h, h, XN, h, 0, P("wqkv"), h, 0, GEMM_EPI_QKV_ROPE, nullptr, 0);
  g.q = Q; g.k = K; g.v = Vv; g.hidden = h; g.head_dim = D; g.rope = rope_; g.pos0 = 0;
  gemm(g);
  AttnFwdArgs fa{Q, K, Vv, O, LSE, S, H, D, 1.0f / std::sqrt(static_cast<float>(D))};
  attention_fwd(fa);
  g = gd(S, h, h, O, h, 0, P("wo"), h, 0, GEMM_EPI_RESID, A, h);
  g.out_f32 = x1; g.resid = X; g.ld_f32 = h;
  gemm(g);
  G(rmsnorm_fwd(x1, nullptr, P("g2"), XN2, S, h, opt_.eps, cs_));
  gemm(gd(S, 2 * F, h, XN2, h, 0, P("wgu"), h, 0, GEMM_EPI_BF16, GU, 2 * F));
  G(swiglu_fwd(GU, ACT, S, F, cs_));
  float* out = i + 1 < d_.n ? reinterpret_cast<float*>(comp(i + 1, C_X))
                            : static_cast<float*>(arena_ptr(seg_emb_fwd_, "x_final"));
  // The output is layer i+1's input, in the rounding buffer layer i-1 is still
  // being offloaded from.  Only the layer_input rows must have left (they are
  // copied first); everything else of RB(i+1) is written by fwd(i+1), which F3
  // holds until offload(i-1) is complete.
  if (i >= 1 && swaps(i - 1)) copy_wait(ev_off_x_[i - 1]);
  g = gd(S, h, F, ACT, F, 0, P("wd"), F, 0, GEMM_EPI_RESID, nullptr, 0);
  g.out_f32 = out; g.resid = x1; g.ld_f32 = h;
  gemm(g);
  stats_.kernel_launches += 3;  // 2 rmsnorm_fwd + swiglu (GEMM/attention counted in wrappers)
  mark(0, static_cast<int>(Kind::LayerFwd), i, false);
  G(cudaEventRecord(ev_fwd_done_[i], cs_));
  if (swaps(i)) offload(i);
}

void Executor::layer_recompute(int i) {
  const int h = d_.h, F = d_.F, D = d_.D;
  const int s0 = static_cast<int>(split_.swap_tokens), R = static_cast<int>(split_.recompute_tokens);
  G(cudaStreamWaitEvent(cs_, ev_pre_mand_[i], 0));  // B3 (+ prefetch-before-recompute)
  mark(0, static_cast<int>(Kind::Recompute), i, true);
  if (R > 0) {
    const std::size_t seg = seg_bwd_[i];
    auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
    const Bytes r0 = static_cast<Bytes>(s0);
    float* X = reinterpret_cast<float*>(comp(i, C_X)) + r0 * h;
    auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN)) + r0 * h;
    auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q)) + r0 * h;
    auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K)) + r0 * h;
    auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V)) + r0 * h;
    auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O)) + r0 * h;
    auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A)) + r0 * h;
    auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2)) + r0 * h;
    auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU)) + r0 * 2 * F;
    auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT)) + r0 * F;
    float* x1 = static_cast<float*>(arena_ptr(seg, "x1_rec"));
    G(rmsnorm_fwd(X, nullptr, P("g1"), XN, R, h, opt_.eps, cs_));
    GemmDesc g = gd(R, 3 * h, h, XN, h, 0, P("wqkv"), h, 0, GEMM_EPI_QKV_ROPE, nullptr, 0);
    g.q = Q; g.k = K; g.v = Vv; g.hidden = h; g.head_dim = D; g.rope = rope_; g.pos0 = s0;
    gemm(g);
    g = gd(R, h, h, O, h, 0, P("wo"), h, 0, GEMM_EPI_RESID, A, h);
    g.out_f32 = x1; g.resid = X; g.ld_f32 = h;
    gemm(g);
    G(rmsnorm_fwd(x1, nullptr, P("g2"), XN2, R, h, opt_.eps, cs_));
    gemm(gd(R, 2 * F, h, XN2, h, 0, P("wgu"), h, 0, GEMM_EPI_BF16, GU, 2 * F));
    G(swiglu_fwd(GU, ACT, R, F, cs_));
    stats_.kernel_launches += 3;
  }
  mark(0, static_cast<int>(Kind::Recompute), i, false);
}

void Executor::layer_bwd(int i) {
  const int S = d_.S, h = d_.h, F = d_.F, H = d_.H, D = d_.D;
  if (swaps(i)) G(cudaStreamWaitEvent(cs_, ev_pre_done_[i], 0));  // B3
  mark(0, static_cast<int>(Kind::LayerBwd), i, true);
  const std::size_t seg = seg_bwd_[i];
  auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
  auto Gr = [&](const char* n) { return grads_ + ptab_.at({n, i}).first; };
  float* X = reinterpret_cast<float*>(comp(i, C_X));
  auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN));
  auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q));
  auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K));
  auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V));
  auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O));
  float* LSE = reinterpret_cast<float*>(comp(i, C_O) + static_cast<Bytes>(S) * h * 2);
  auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A));
  auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2));
  auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU));
  auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT));
  float* dxc = static_cast<float*>(arena_ptr(seg_emb_fwd_, "dx_carry"));
  auto* dxb = static_cast<__nv_bfloat16*>(arena_ptr(seg_emb_fwd_, "dxb_carry"));
  auto* dact = static_cast<__nv_bfloat16*>(arena_ptr(seg, "dact"));
  auto* dgu = static_cast<__nv_bfloat16*>(arena_ptr(seg, "dgu"));
  float* dxn2 = static_cast<float*>(arena_ptr(seg, "dxn2"));
  auto* da = static_cast<__nv_bfloat16*>(arena_ptr(seg, "da"));
  float* part2 = static_cast<float*>(arena_ptr(seg, "part2"));
  auto* dout = static_cast<__nv_bfloat16*>(arena_ptr(seg, "dout"));
  float* ws = static_cast<float*>(arena_ptr(seg, "attn_ws"));
  auto* dqkv = static_cast<__nv_bfloat16*>(arena_ptr(seg, "dqkv"));
  float* dxn = static_cast<float*>(arena_ptr(seg, "dxn"));
  float* part1 = static_cast<float*>(arena_ptr(seg, "part1"));

  // MLP: dact = dY Wd ; dWd = dY^T act ; SwiGLU bwd ; dxn2 = dGU Wgu ; dWgu = dGU^T xn2
  gemm(gd(S, F, h, dxb, h, 0, P("wd"), F, 1, GEMM_EPI_BF16, dact, F));
  gemm(gd(h, F, S, dxb, h, 1, ACT, F, 1, GEMM_EPI_F32, Gr("wd"), F));
  G(swiglu_bwd(GU, dact, dgu, S, F, cs_));
  gemm(gd(S, h, 2 * F, dgu, 2 * F, 0, P("wgu"), h, 1, GEMM_EPI_F32, dxn2, h));
  gemm(gd(2 * F, h, S, dgu, 2 * F, 1, XN2, h, 1, GEMM_EPI_F32, Gr("wgu"), h));
  // post-attention norm: x1 = x + a recomputed inside the kernel
  G(rmsnorm_bwd(X, A, P("g2"), dxn2, dxc, dxc, da, part2, Gr("g2"), S, h, opt_.eps, false, cs_));
  // attention output projection
  gemm(gd(S, h, h, da, h, 0, P("wo"), h, 1, GEMM_EPI_BF16, dout, h));
  gemm(gd(h, h, S, da, h, 1, O, h, 1, GEMM_EPI_F32, Gr("wo"), h));
  AttnBwdArgs ba;
  ba.q = Q; ba.k = K; ba.v = Vv; ba.o = O; ba.lse = LSE; ba.dout = dout; ba.delta = ws;
  ba.dq = dqkv; ba.dk = dqkv + h; ba.dv = dqkv + 2 * h; ba.ld_dqkv = 3 * h;
  ba.rope = rope_; ba.pos0 = 0; ba.S = S; ba.H = H; ba.D = D;
  ba.softmax_scale = 1.0f / std::sqrt(static_cast<float>(D));
  attention_bwd(ba);
  // QKV projection
  gemm(gd(S, h, 3 * h, dqkv, 3 * h, 0, P("wqkv"), h, 1, GEMM_EPI_F32, dxn, h));
  gemm(gd(3 * h, h, S, dqkv, 3 * h, 1, XN, h, 1, GEMM_EPI_F32, Gr("wqkv"), h));
  G(rmsnorm_bwd(X, nullptr, P("g1"), dxn, dxc, dxc, dxb, part1, Gr("g1"), S, h, opt_.eps, false, cs_));
  stats_.kernel_launches += 5;  // swiglu_bwd + 2 x (rmsnorm_bwd + dg_reduce)
  mark(0, static_cast<int>(Kind::LayerBwd), i, false);
  G(cudaEventRecord(ev_bwd_done_[i], cs_));
  if (i >= 2 && swaps(i - 2)) prefetch(i - 2);  // B2
}

void Executor::classifier() {
  const int S = d_.S, h = d_.h, V = d_.V;
  const int T = std::min(opt_.ce_chunk, S);
  float* xfin = static_cast<float*>(arena_ptr(seg_emb_fwd_, "x_final"));
  auto* xf = static_cast<__nv_bfloat16*>(arena_ptr(seg_cls_fwd_, "xf"));
  const __nv_bfloat16* gf = params_ + ptab_.at({"gf", -1}).first;
  const __nv_bfloat16* W = params_ + ptab_.at({"wcls", -1}).first;
  float* gW = grads_ + ptab_.at({"wcls", -1}).first;
  mark(0, static_cast<int>(Kind::ClsFwd), -1, true);
  G(rmsnorm_fwd(xfin, nullptr, gf, xf, S, h, opt_.eps, cs_));
  mark(0, static_cast<int>(Kind::ClsFwd), -1, false);
  mark(0, static_cast<int>(Kind::ClsBwd), -1, true);
  float* dxf = static_cast<float*>(arena_ptr(seg_cls_bwd_, "dxf"));
  float* loss_rows = static_cast<float*>(arena_ptr(seg_cls_bwd_, "loss_rows"));
  float* logits = static_cast<float*>(arena_ptr(seg_cls_bwd_, "logits"));
  auto* dlog = static_cast<__nv_bfloat16*>(arena_ptr(seg_cls_bwd_, "dlogits"));
  float* part = static_cast<float*>(arena_ptr(seg_cls_bwd_, "cls_part"));
  const float* inv_n = inv_n_dev_;  // 1/n_labeled of the loaded batch (device, see load_batch)
  for (int c0 = 0; c0 < S; c0 += T) {
    const int t = std::min(T, S - c0);
    const __nv_bfloat16* xc = xf + static_cast<Bytes>(c0) * h;
    gemm(gd(t, V, h, xc, h, 0, W, h, 0, GEMM_EPI_F32, logits, V));
    G(cross_entropy(logits, lab_ + c0, dlog, loss_rows + c0, t, V, inv_n, cs_));
    gemm(gd(t, h, V, dlog, V, 0, W, h, 1, GEMM_EPI_F32, dxf + static_cast<Bytes>(c0) * h, h));
    gemm(gd(V, h, t, dlog, V, 1, xc, h, 1, c0 == 0 ? GEMM_EPI_F32 : GEMM_EPI_F32_ACC, gW, h));
    stats_.kernel_launches += 1;  // cross-entropy
  }
  G(sum_scaled(loss_rows, S, inv_n, loss_dev_, cs_));
  float* dxc = static_cast<float*>(arena_ptr(seg_emb_fwd_, "dx_carry"));
  auto* dxb = static_cast<__nv_bfloat16*>(arena_ptr(seg_emb_fwd_, "dxb_carry"));
  G(rmsnorm_bwd(xfin, nullptr, gf, dxf, nullptr, dxc, dxb, part, grads_ + ptab_.at({"gf", -1}).first,
                S, h, opt_.eps, false, cs_));
  stats_.kernel_launches += 4;  // rmsnorm_fwd, sum, rmsnorm_bwd + dg_reduce
  mark(0, static_cast<int>(Kind::ClsBwd), -1, false);
}

// ================================================================== SP + TP
// Megatron sequence+tensor parallelism.  Per layer forward:
//   xn = norm(x_local) -> AG -> QKV (column-parallel, local heads) -> attention
//   -> out-proj (row-parallel) -> RS -> x1 = x + a -> norm -> AG -> gate/up
//   (column-parallel) -> SwiGLU -> down (row-parallel) -> RS -> x + d.
// Backward mirrors it with AG <-> RS swapped; all-gathered activations are
// regathered rather than saved (the skeletal tensors stay sharded).
namespace {
inline void ag(Comm* c, const __nv_bfloat16* src, __nv_bfloat16* dst, size_t count, cudaStream_t st) {
  c->all_gather(src, dst, count, CommDtype::BF16, st);
}
inline void rs(Comm* c, const float* src, float* dst, size_t count, cudaStream_t st) {
  c->reduce_scatter(src, dst, count, CommDtype::F32, st);
}

// Signal channels of the fused peer paths (0 and 1 belong to the collectives).
constexpr int CH_AG_READY = 2;  // shard written (cs_ -> peers' xs_)
constexpr int CH_AG_DONE = 3;   // peer finished pulling my shard (xs_ -> owner's cs_)
constexpr int CH_RS_READY = 4;  // partial row block written (cs_ -> owner's xs_)
constexpr int CH_RS_FREE = 5;   // owner finished pulling my partial (xs_ -> producer's cs_)

// Rows [r0, r0 + m) of a GEMM whose A is K-major.
GemmDesc rows_of(GemmDesc g, int r0, int m) {
  g.a = static_cast<const char*>(g.a) + static_cast<Bytes>(r0) * g.lda * 2;
  switch (g.epi) {
    case GEMM_EPI_BF16:
      g.c = static_cast<char*>(g.c) + static_cast<Bytes>(r0) * g.ldc * 2;
      break;
    case GEMM_EPI_F32:
    case GEMM_EPI_F32_ACC:
      g.c = static_cast<char*>(g.c) + static_cast<Bytes>(r0) * g.ldc * 4;
      break;
    case GEMM_EPI_QKV_ROPE:
      g.q += static_cast<Bytes>(r0) * g.hidden;
      g.k += static_cast<Bytes>(r0) * g.hidden;
      g.v += static_cast<Bytes>(r0) * g.hidden;
      g.pos0 += r0;
      break;
    default:
      throw std::logic_error("rows_of: unsupported epilogue");
  }
  g.M = m;
  return g;
}
}  // namespace

// row0 > 0: only rows [row0, Sl) of every rank's block (the recompute suffix);
// `part` and `out` keep their [Sl, N] layout, so the reduced rows land where a
// full-block call puts them, bitwise equal (per-row GEMM results do not depend
// on M, and the sum order is unchanged).
void Executor::gemm_reduce_rows(GemmDesc g, float* part, float* out, int row0) {
  const int t = d_.t, Sl = d_.Sl, r = d_.r;
  if (row0 >= Sl) return;
  const auto* a = static_cast<const __nv_bfloat16*>(g.a) + static_cast<Bytes>(row0) * g.lda;
  const size_t count = static_cast<size_t>(Sl - row0) * g.N;
  part += static_cast<Bytes>(row0) * g.N;
  out += static_cast<Bytes>(row0) * g.N;
  g.M = Sl - row0;
  g.c = part;
  g.ldc = g.N;
  if (!peer()) {
    for (int k = 0; k < t; ++k) {  // same per-row K order as one S-row GEMM: bitwise equal rows
      g.a = a + static_cast<Bytes>(k) * Sl * g.lda;
      gemm(g);
      comm_->reduce(part, k == r ? out : part, count, CommDtype::F32, k, cs_);
    }
    return;
  }
  // Staggered reduce-scatter over peer memory.  At step j rank r computes the
  // partial of row block b = r-j-1 (mod t) into `part` while, on the comm
  // stream, it pulls the partial of its OWN block from producer p = r+j+1 and
  // accumulates it into `out`: every rank reads from a different peer at
  // every step, so all links carry traffic at once (the row-chunked reduce
  // above funnels each block into one root).  The own block comes last and is
  // added by the GEMM epilogue itself (F32_ACC), so out = p_{r+1} + ... + p_{r-1}
  // + p_r in a fixed order (bitwise the loopback sum for t = 2).
  ck(cudaEventRecord(ev_cs2xs_, cs_), "record");
  ck(cudaStreamWaitEvent(xs_, ev_cs2xs_, 0), "wait");  // previous readers of `out` are done
  int prev = -1;  // owner of the block last written into `part`
  for (int j = 0; j < t; ++j) {
    const int b = ((r - j - 1) % t + t) % t;
    if (b != r) {
      if (prev >= 0) comm_->wait(prev, CH_RS_FREE, cs_);
      GemmDesc gj = g;
      gj.a = a + static_cast<Bytes>(b) * Sl * g.lda;
      gemm(gj);
      comm_->signal(b, CH_RS_READY, cs_);
      prev = b;
    }
    const int p = (r + j + 1) % t;
    if (p != r) {
      comm_->wait(p, CH_RS_READY, xs_);
      ck(peer_accumulate(static_cast<const float*>(comm_->peer_ptr(p, part)), out, count, j == 0, xs_),
         "peer_accumulate");
      comm_->signal(p, CH_RS_FREE, xs_);
    }
  }
  ck(cudaEventRecord(ev_xs2cs_, xs_), "record");
  ck(cudaStreamWaitEvent(cs_, ev_xs2cs_, 0), "wait");
  GemmDesc go = g;  // own block: out += p_r in the epilogue
  go.a = a + static_cast<Bytes>(r) * Sl * g.lda;
  go.c = out;
  go.epi = GEMM_EPI_F32_ACC;
  gemm(go);
  if (prev >= 0) comm_->wait(prev, CH_RS_FREE, cs_);  // `part` may be rewritten after this
  stats_.kernel_launches += t - 1;
}

// Peer all-gather of the t row blocks of `full` ([S, width] bf16; this rank's
// block is `shard`): the copy engines pull every peer's block on its own
// stream, each rank starting at its own index so every link is busy, and
// ev_blk_[j] marks block (r + j) % t landed.  gather_release() must follow
// once the consumers of `full` have been enqueued behind those events.
void Executor::gather_pull(const __nv_bfloat16* shard, __nv_bfloat16* full, size_t width) {
  const int t = d_.t, Sl = d_.Sl, r = d_.r;
  const size_t shard_elems = static_cast<size_t>(Sl) * width;
  for (int k = 0; k < t; ++k)
    if (k != r) comm_->signal(k, CH_AG_READY, cs_);
  ck(cudaEventRecord(ev_cs2xs_, cs_), "record");
  ck(cudaStreamWaitEvent(xs_, ev_cs2xs_, 0), "wait");  // own shard written, `full` free
  const Bytes blk = shard_elems * 2;
  for (int j = 0; j < t; ++j) {  // block j = 0 is the own shard (local copy on xs_)
    const int k = (r + j) % t;
    cudaStream_t st = j == 0 ? xs_ : xcs_[j - 1];
    if (j > 0) {
      ck(cudaStreamWaitEvent(st, ev_cs2xs_, 0), "wait");
      comm_->wait(k, CH_AG_READY, st);
    }
    const void* src = k == r ? static_cast<const void*>(shard) : comm_->peer_ptr(k, shard);
    ck(cudaMemcpyAsync(reinterpret_cast<char*>(full) + k * blk, src, blk, cudaMemcpyDeviceToDevice, st),
       "peer gather copy");
    ck(cudaEventRecord(ev_blk_[j], st), "record");
  }
  for (int j = 1; j < t; ++j) ck(cudaStreamWaitEvent(xs_, ev_blk_[j], 0), "wait");  // all pulls done
  for (int k = 0; k < t; ++k)
    if (k != r) comm_->signal(k, CH_AG_DONE, xs_);
}

void Executor::gather_release() {
  for (int k = 0; k < d_.t; ++k)
    if (k != d_.r) comm_->wait(k, CH_AG_DONE, cs_);  // nobody reads my shard any more
}

void Executor::gather_gemm(const __nv_bfloat16* shard, __nv_bfloat16* full, GemmDesc g, int row0) {
  const int t = d_.t, Sl = d_.Sl, r = d_.r, S = d_.S;
  if (!peer()) {
    ag(comm_.get(), shard, full, static_cast<size_t>(Sl) * g.K, cs_);
    if (row0 < S) gemm(rows_of(g, row0, S - row0));
    return;
  }
  gather_pull(shard, full, static_cast<size_t>(g.K));
  for (int j = 0; j < t; ++j) {
    const int k = (r + j) % t;
    ck(cudaStreamWaitEvent(cs_, ev_blk_[j], 0), "wait");
    const int lo = std::max(row0, k * Sl), hi = (k + 1) * Sl;
    if (lo < hi) gemm(rows_of(g, lo, hi - lo));
  }
  gather_release();
}

// All-gather -> weight-gradient GEMM (dW = dY^T X_full, K = S): the gathered
// input's row blocks are the K blocks of the GEMM, so block k's partial is
// accumulated as soon as it has landed (GEMM_EPI_F32 for block 0, F32_ACC
// after), in the fixed order k = 0..t-1 on every communicator -- loopback,
// NCCL and peer memory sum the same way, bitwise.
void Executor::gather_wgrad(const __nv_bfloat16* shard, __nv_bfloat16* full, GemmDesc g) {
  const int t = d_.t, Sl = d_.Sl, r = d_.r;
  auto block = [&](int k) {
    GemmDesc gk = g;
    gk.K = Sl;
    gk.a = static_cast<const char*>(g.a) + static_cast<Bytes>(k) * Sl * g.lda * 2;
    gk.b = static_cast<const char*>(g.b) + static_cast<Bytes>(k) * Sl * g.ldb * 2;
    gk.epi = k == 0 ? GEMM_EPI_F32 : GEMM_EPI_F32_ACC;
    gemm(gk);
  };
  if (!peer()) {
    ag(comm_.get(), shard, full, static_cast<size_t>(Sl) * g.ldb, cs_);
    for (int k = 0; k < t; ++k) block(k);
    return;
  }
  gather_pull(shard, full, static_cast<size_t>(g.ldb));
  for (int k = 0; k < t; ++k) {
    ck(cudaStreamWaitEvent(cs_, ev_blk_[(k - r + t) % t], 0), "wait");
    block(k);
  }
  gather_release();
}

void Executor::layer_fwd_tp(int i) {
  const int S = d_.S, Sl = d_.Sl, h = d_.h, hl = d_.hl, Fl = d_.Fl, Hl = d_.Hl, D = d_.D;
  if (i >= 2 && swaps(i - 2)) G(cudaStreamWaitEvent(cs_, ev_off_done_[i - 2], 0));  // F3
  mark(0, static_cast<int>(Kind::LayerFwd), i, true);
  const std::size_t seg = seg_fwd_[i];
  auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
  auto A_ = [&](const char* n) { return arena_ptr(seg, n); };
  float* X = reinterpret_cast<float*>(comp(i, C_X));
  auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN));
  auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q));
  auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K));
  auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V));
  auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O));
  float* LSE = reinterpret_cast<float*>(comp(i, C_O) + static_cast<Bytes>(S) * hl * 2);
  auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A));
  auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2));
  auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU));
  auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT));
  auto* xn_full = static_cast<__nv_bfloat16*>(A_("xn_full"));
  float* a_part = static_cast<float*>(A_("a_part"));
  float* a_red = static_cast<float*>(A_("a_red"));
  float* x1 = static_cast<float*>(A_("x1"));
  auto* xn2_full = static_cast<__nv_bfloat16*>(A_("xn2_full"));
  float* d_part = static_cast<float*>(A_("d_part"));
  float* d_red = static_cast<float*>(A_("d_red"));
  const size_t shard = static_cast<size_t>(Sl) * h;

  G(rmsnorm_fwd(X, nullptr, P("g1"), XN, Sl, h, opt_.eps, cs_));
  GemmDesc g = gd(S, 3 * hl, h, xn_full, h, 0, P("wqkv"), h, 0, GEMM_EPI_QKV_ROPE, nullptr, 0);
  g.q = Q; g.k = K; g.v = Vv; g.hidden = hl; g.head_dim = D; g.rope = rope_; g.pos0 = 0;
  gather_gemm(XN, xn_full, g, 0);
  AttnFwdArgs fa{Q, K, Vv, O, LSE, S, Hl, D, 1.0f / std::sqrt(static_cast<float>(D))};
  attention_fwd(fa);
  gemm_reduce_rows(gd(S, h, hl, O, hl, 0, P("wo"), hl, 0, GEMM_EPI_F32, nullptr, h), a_part, a_red);
  G(resid_round(X, a_red, A, x1, static_cast<long long>(shard), cs_));
  G(rmsnorm_fwd(x1, nullptr, P("g2"), XN2, Sl, h, opt_.eps, cs_));
  gather_gemm(XN2, xn2_full, gd(S, 2 * Fl, h, xn2_full, h, 0, P("wgu"), h, 0, GEMM_EPI_BF16, GU, 2 * Fl), 0);
  G(swiglu_fwd(GU, ACT, S, Fl, cs_));
  gemm_reduce_rows(gd(S, h, Fl, ACT, Fl, 0, P("wd"), Fl, 0, GEMM_EPI_F32, nullptr, h), d_part, d_red);
  float* out = i + 1 < d_.n ? reinterpret_cast<float*>(comp(i + 1, C_X))
                            : static_cast<float*>(arena_ptr(seg_emb_fwd_, "x_final"));
  // The output is layer i+1's input, in the rounding buffer layer i-1 is still
  // being offloaded from.  Only the layer_input rows must have left (they are
  // copied first); everything else of RB(i+1) is written by fwd(i+1), which F3
  // holds until offload(i-1) is complete.
  if (i >= 1 && swaps(i - 1)) copy_wait(ev_off_x_[i - 1]);
  G(resid_round(x1, d_red, nullptr, out, static_cast<long long>(shard), cs_));
  stats_.kernel_launches += 5;
  mark(0, static_cast<int>(Kind::LayerFwd), i, false);
  G(cudaEventRecord(ev_fwd_done_[i], cs_));
  if (swaps(i)) offload(i);
}

void Executor::layer_recompute_tp(int i) {
  const int S = d_.S, h = d_.h, hl = d_.hl, Fl = d_.Fl, D = d_.D;
  const int sw = static_cast<int>(split_.swap_tokens), R = static_cast<int>(split_.recompute_tokens);
  const int swl = static_cast<int>(split_l_.swap_tokens), Rl = static_cast<int>(split_l_.recompute_tokens);
  G(cudaStreamWaitEvent(cs_, ev_pre_mand_[i], 0));  // B3 (+ prefetch-before-recompute)
  mark(0, static_cast<int>(Kind::Recompute), i, true);
  if (R > 0 || Rl > 0) {
    const std::size_t seg = seg_bwd_[i];
    auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
    auto A_ = [&](const char* n) { return arena_ptr(seg, n); };
    float* X = reinterpret_cast<float*>(comp(i, C_X));
    auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN));
    auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q));
    auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K));
    auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V));
    auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O));
    auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A));
    auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2));
    auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU));
    auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT));
    auto* xn_full = static_cast<__nv_bfloat16*>(A_("r_xn_full"));
    float* a_part = static_cast<float*>(A_("r_a_part"));
    float* a_red = static_cast<float*>(A_("r_a_red"));
    float* x1 = static_cast<float*>(A_("r_x1"));
    auto* xn2_full = static_cast<__nv_bfloat16*>(A_("r_xn2_full"));
    const Bytes r0 = static_cast<Bytes>(swl);
    // local suffix rows of the input norm, then the full gathered input
    if (Rl > 0) G(rmsnorm_fwd(X + r0 * h, nullptr, P("g1"), XN + r0 * h, Rl, h, opt_.eps, cs_));
    {
      GemmDesc g = gd(S, 3 * hl, h, xn_full, h, 0, P("wqkv"), h, 0, GEMM_EPI_QKV_ROPE, nullptr, 0);
      g.q = Q; g.k = K; g.v = Vv; g.hidden = hl; g.head_dim = D; g.rope = rope_; g.pos0 = 0;
      gather_gemm(XN, xn_full, g, sw);  // suffix rows [sw, S) only
    }
    // attn_proj needs every rank's partial of its suffix rows: the out-projection
    // + reduce-scatter of rows [swl, Sl) of every rank's block only
    gemm_reduce_rows(gd(S, h, hl, O, hl, 0, P("wo"), hl, 0, GEMM_EPI_F32, nullptr, h), a_part, a_red, swl);
    if (Rl > 0) {
      G(resid_round(X + r0 * h, a_red + r0 * h, A + r0 * h, x1 + r0 * h,
                    static_cast<long long>(Rl) * h, cs_));
      G(rmsnorm_fwd(x1 + r0 * h, nullptr, P("g2"), XN2 + r0 * h, Rl, h, opt_.eps, cs_));
    }
    gather_gemm(XN2, xn2_full, gd(S, 2 * Fl, h, xn2_full, h, 0, P("wgu"), h, 0, GEMM_EPI_BF16, GU, 2 * Fl), sw);
    if (R > 0) {
      G(swiglu_fwd(GU + static_cast<Bytes>(sw) * 2 * Fl, ACT + static_cast<Bytes>(sw) * Fl, R, Fl, cs_));
    }
    stats_.kernel_launches += 5;
  }
  mark(0, static_cast<int>(Kind::Recompute), i, false);
}

void Executor::layer_bwd_tp(int i) {
  const int S = d_.S, Sl = d_.Sl, h = d_.h, hl = d_.hl, Fl = d_.Fl, Hl = d_.Hl, D = d_.D;
  if (swaps(i)) G(cudaStreamWaitEvent(cs_, ev_pre_done_[i], 0));  // B3
  mark(0, static_cast<int>(Kind::LayerBwd), i, true);
  const std::size_t seg = seg_bwd_[i];
  auto P = [&](const char* n) { return params_ + ptab_.at({n, i}).first; };
  auto Gr = [&](const char* n) { return grads_ + ptab_.at({n, i}).first; };
  auto A_ = [&](const char* n) { return arena_ptr(seg, n); };
  float* X = reinterpret_cast<float*>(comp(i, C_X));
  auto* XN = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN));
  auto* Q = reinterpret_cast<__nv_bfloat16*>(comp(i, C_Q));
  auto* K = reinterpret_cast<__nv_bfloat16*>(comp(i, C_K));
  auto* Vv = reinterpret_cast<__nv_bfloat16*>(comp(i, C_V));
  auto* O = reinterpret_cast<__nv_bfloat16*>(comp(i, C_O));
  float* LSE = reinterpret_cast<float*>(comp(i, C_O) + static_cast<Bytes>(S) * hl * 2);
  auto* A = reinterpret_cast<__nv_bfloat16*>(comp(i, C_A));
  auto* XN2 = reinterpret_cast<__nv_bfloat16*>(comp(i, C_XN2));
  auto* GU = reinterpret_cast<__nv_bfloat16*>(comp(i, C_GU));
  auto* ACT = reinterpret_cast<__nv_bfloat16*>(comp(i, C_ACT));
  float* dxc = static_cast<float*>(arena_ptr(seg_emb_fwd_, "dx_carry"));
  auto* dxb = static_cast<__nv_bfloat16*>(arena_ptr(seg_emb_fwd_, "dxb_carry"));
  auto* dy_full = static_cast<__nv_bfloat16*>(A_("dy_full"));
  auto* dact = static_cast<__nv_bfloat16*>(A_("dact"));
  auto* dgu = static_cast<__nv_bfloat16*>(A_("dgu"));
  float* dxn2_part = static_cast<float*>(A_("dxn2_part"));
  float* dxn2 = static_cast<float*>(A_("dxn2"));
  auto* xn2_full = static_cast<__nv_bfloat16*>(A_("b_xn2_full"));
  auto* da = static_cast<__nv_bfloat16*>(A_("da"));
  float* part2 = static_cast<float*>(A_("part2"));
  auto* da_full = static_cast<__nv_bfloat16*>(A_("da_full"));
  auto* dout = static_cast<__nv_bfloat16*>(A_("dout"));
  float* ws = static_cast<float*>(A_("attn_ws"));
  auto* dqkv = static_cast<__nv_bfloat16*>(A_("dqkv"));
  float* dxn_part = static_cast<float*>(A_("dxn_part"));
  float* dxn = static_cast<float*>(A_("dxn"));
  auto* xn_full = static_cast<__nv_bfloat16*>(A_("b_xn_full"));
  float* part1 = static_cast<float*>(A_("part1"));

  // MLP (down is row-parallel: its input gradient is the gathered output grad)
  gather_gemm(dxb, dy_full, gd(S, Fl, h, dy_full, h, 0, P("wd"), Fl, 1, GEMM_EPI_BF16, dact, Fl), 0);
  gemm(gd(h, Fl, S, dy_full, h, 1, ACT, Fl, 1, GEMM_EPI_F32, Gr("wd"), Fl));
  G(swiglu_bwd(GU, dact, dgu, S, Fl, cs_));
  gemm_reduce_rows(gd(S, h, 2 * Fl, dgu, 2 * Fl, 0, P("wgu"), h, 1, GEMM_EPI_F32, nullptr, h), dxn2_part, dxn2);
  gather_wgrad(XN2, xn2_full, gd(2 * Fl, h, S, dgu, 2 * Fl, 1, xn2_full, h, 1, GEMM_EPI_F32, Gr("wgu"), h));
  G(rmsnorm_bwd(X, A, P("g2"), dxn2, dxc, dxc, da, part2, Gr("g2"), Sl, h, opt_.eps, false, cs_));
  // attention output projection (row-parallel)
  gather_gemm(da, da_full, gd(S, hl, h, da_full, h, 0, P("wo"), hl, 1, GEMM_EPI_BF16, dout, hl), 0);
  gemm(gd(h, hl, S, da_full, h, 1, O, hl, 1, GEMM_EPI_F32, Gr("wo"), hl));
  AttnBwdArgs ba;
  ba.q = Q; ba.k = K; ba.v = Vv; ba.o = O; ba.lse = LSE; ba.dout = dout; ba.delta = ws;
  ba.dq = dqkv; ba.dk = dqkv + hl; ba.dv = dqkv + 2 * hl; ba.ld_dqkv = 3 * hl;
  ba.rope = rope_; ba.pos0 = 0; ba.S = S; ba.H = Hl; ba.D = D;
  ba.softmax_scale = 1.0f / std::sqrt(static_cast<float>(D));
  attention_bwd(ba);
  // QKV projection (column-parallel)
  gemm_reduce_rows(gd(S, h, 3 * hl, dqkv, 3 * hl, 0, P("wqkv"), h, 1, GEMM_EPI_F32, nullptr, h), dxn_part, dxn);
  gather_wgrad(XN, xn_full, gd(3 * hl, h, S, dqkv, 3 * hl, 1, xn_full, h, 1, GEMM_EPI_F32, Gr("wqkv"), h));
  G(rmsnorm_bwd(X, nullptr, P("g1"), dxn, dxc, dxc, dxb, part1, Gr("g1"), Sl, h, opt_.eps, false, cs_));
  stats_.kernel_launches += 5;
  mark(0, static_cast<int>(Kind::LayerBwd), i, false);
  G(cudaEventRecord(ev_bwd_done_[i], cs_));
  if (i >= 2 && swaps(i - 2)) prefetch(i - 2);  // B2
}

void Executor::classifier_tp() {
  const int S = d_.S, Sl = d_.Sl, h = d_.h, Vl = d_.Vl;
  const int T = std::min(opt_.ce_chunk, S);
  float* xfin = static_cast<float*>(arena_ptr(seg_emb_fwd_, "x_final"));
  auto* xf = static_cast<__nv_bfloat16*>(arena_ptr(seg_cls_fwd_, "xf"));
  const __nv_bfloat16* gf = params_ + ptab_.at({"gf", -1}).first;
  const __nv_bfloat16* W = params_ + ptab_.at({"wcls", -1}).first;
  float* gW = grads_ + ptab_.at({"wcls", -1}).first;
  mark(0, static_cast<int>(Kind::ClsFwd), -1, true);
  G(rmsnorm_fwd(xfin, nullptr, gf, xf, Sl, h, opt_.eps, cs_));
  mark(0, static_cast<int>(Kind::ClsFwd), -1, false);
  mark(0, static_cast<int>(Kind::ClsBwd), -1, true);
  const std::size_t sb = seg_cls_bwd_;
  auto* xf_full = static_cast<__nv_bfloat16*>(arena_ptr(sb, "xf_full"));
  float* dxf_part = static_cast<float*>(arena_ptr(sb, "dxf_part"));
  float* loss_rows = static_cast<float*>(arena_ptr(sb, "loss_rows"));
  float* logits = static_cast<float*>(arena_ptr(sb, "logits"));
  auto* dlog = static_cast<__nv_bfloat16*>(arena_ptr(sb, "dlogits"));
  float* stats = static_cast<float*>(arena_ptr(sb, "ce_stats"));  // [lmax | gmax | lsum,ltgt | gsum,gtgt]
  const size_t shard = static_cast<size_t>(Sl) * h;
  ag(comm_.get(), xf, xf_full, shard, cs_);
  const float* inv_n = inv_n_dev_;  // 1/n_labeled of the loaded batch (device, see load_batch)
  const int v0 = d_.r * Vl;
  for (int c0 = 0; c0 < S; c0 += T) {
    const int t = std::min(T, S - c0);
    const __nv_bfloat16* xc = xf_full + static_cast<Bytes>(c0) * h;
    float* lmax = stats;
    float* gmax = stats + T;
    float* lst = stats + 2 * T;  // [sum | target] x T
    float* gst = stats + 4 * T;
    gemm(gd(t, Vl, h, xc, h, 0, W, h, 0, GEMM_EPI_F32, logits, Vl));
    G(ce_vp_max(logits, lmax, t, Vl, cs_));
    comm_->all_reduce(lmax, gmax, t, CommDtype::F32, CommOp::Max, cs_);
    G(ce_vp_sum(logits, gmax, lab_ + c0, v0, lst, t, Vl, cs_));
    // stats layout per chunk is [sum(t) | target(t)] contiguous at lst
    comm_->all_reduce(lst, gst, 2 * static_cast<size_t>(t), CommDtype::F32, CommOp::Sum, cs_);
    G(ce_vp_grad(logits, gmax, gst, lab_ + c0, v0, dlog, loss_rows + c0, t, Vl, inv_n, cs_));
    gemm(gd(t, h, Vl, dlog, Vl, 0, W, h, 1, GEMM_EPI_F32, dxf_part + static_cast<Bytes>(c0) * h, h));
    gemm(gd(Vl, h, t, dlog, Vl, 1, xc, h, 1, c0 == 0 ? GEMM_EPI_F32 : GEMM_EPI_F32_ACC, gW, h));
    stats_.kernel_launches += 3;
  }
  G(sum_scaled(loss_rows, S, inv_n, loss_dev_, cs_));
  float* dxf = static_cast<float*>(arena_ptr(sb, "dxf"));
  rs(comm_.get(), dxf_part, dxf, shard, cs_);
  float* dxc = static_cast<float*>(arena_ptr(seg_emb_fwd_, "dx_carry"));
  auto* dxb = static_cast<__nv_bfloat16*>(arena_ptr(seg_emb_fwd_, "dxb_carry"));
  float* part = static_cast<float*>(arena_ptr(sb, "cls_part"));
  G(rmsnorm_bwd(xfin, nullptr, gf, dxf, nullptr, dxc, dxb, part, grads_ + ptab_.at({"gf", -1}).first,
                Sl, h, opt_.eps, false, cs_));
  stats_.kernel_launches += 4;
  mark(0, static_cast<int>(Kind::ClsBwd), -1, false);
}

// Replicated parameters (embedding, norm weights) accumulate gradients from
// every rank's token shard: sum them so all replicas step identically.
void Executor::sync_replicated_grads() {
  float* tmp = static_cast<float*>(arena_ptr(seg_emb_bwd_, "ar_tmp"));
  auto sum = [&](const char* n, int layer) {
    const auto [off, cnt] = ptab_.at({n, layer});
    comm_->all_reduce(grads_ + off, tmp, static_cast<size_t>(cnt), CommDtype::F32, CommOp::Sum, cs_);
    G(cudaMemcpyAsync(grads_ + off, tmp, static_cast<size_t>(cnt) * 4, cudaMemcpyDeviceToDevice, cs_));
  };
  sum("embedding", -1);
  for (int l = 0; l < d_.n; ++l) {
    sum("g1", l);
    sum("g2", l);
  }
  sum("gf", -1);
}

// With ExecOptions::cuda_graph the first step runs eagerly (kernel attributes,
// lazy module loading and TMA-descriptor caches settle), the second is
// captured from cs_ -- the copy streams join through ev_fork_ and rejoin at the
// end -- and every step after replays the instantiated graph with one launch.
// The timeline, op timings and launch counts of the captured step stay valid:
// their events are external record nodes of the graph (record_timing_event).
void Executor::step_resident() {
  if (!opt_.cuda_graph) {
    record_step();
    return;
  }
  const bool tp = d_.t > 1 && comm_;
  if (!graph_exec_ && eager_done_) {
    if (tp) comm_->capture_begin();
    G(cudaStreamBeginCapture(cs_, cudaStreamCaptureModeRelaxed));
    capturing_ = true;
    try {
      record_step();
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(cs_, &g);
      if (g) cudaGraphDestroy(g);
      capturing_ = false;
      throw;
    }
    G(cudaStreamEndCapture(cs_, &graph_));
    capturing_ = false;
    if (tp) comm_->capture_end(graph_);
    G(cudaGraphInstantiate(&graph_exec_, graph_, 0));
    replays_ = 0;
  }
  if (graph_exec_) {
    // SP+TP: the signal values / wait thresholds of this replay (IPC backend)
    if (tp) comm_->before_replay(graph_exec_, replays_);
    ++replays_;
    G(cudaGraphLaunch(graph_exec_, cs_));
    return;
  }
  record_step();
  eager_done_ = true;
}

void Executor::record_step() {
  const int n = d_.n;
  marks_.clear();
  ops_.clear();
  waits_.clear();
  ev_used_ = 0;
  stats_.offload_bytes = stats_.prefetch_bytes = 0;
  stats_.kernel_launches = 0;
  G(record_timing_event(ev_start_, cs_));
  // copy streams must not run ahead of this step's start
  G(cudaEventRecord(ev_fork_, cs_));
  G(cudaStreamWaitEvent(os_, ev_fork_, 0));
  G(cudaStreamWaitEvent(ps_, ev_fork_, 0));
  mark(0, static_cast<int>(Kind::EmbFwd), -1, true);
  G(embed_fwd(tok_ + d_.r * d_.Sl, params_ + ptab_.at({"embedding", -1}).first,
              reinterpret_cast<float*>(comp(0, C_X)), d_.Sl, d_.h, cs_));
  mark(0, static_cast<int>(Kind::EmbFwd), -1, false);
  const bool tp = d_.t > 1;
  for (int i = 0; i < n; ++i) tp ? layer_fwd_tp(i) : layer_fwd(i);
  tp ? classifier_tp() : classifier();
  for (int i = n - 1; i >= 0; --i) {
    if (swaps(i)) tp ? layer_recompute_tp(i) : layer_recompute(i);
    tp ? layer_bwd_tp(i) : layer_bwd(i);
  }
  mark(0, static_cast<int>(Kind::EmbBwd), -1, true);
  G(embed_bwd(csr_off_, csr_pos_, static_cast<float*>(arena_ptr(seg_emb_fwd_, "dx_carry")),
              grads_ + ptab_.at({"embedding", -1}).first, d_.V, d_.h, cs_));
  if (tp) sync_replicated_grads();
  mark(0, static_cast<int>(Kind::EmbBwd), -1, false);
  stats_.kernel_launches += 2;
  if (opt_.optimizer) {
    G(adamw(master_, params_, grads_, adam_m_, adam_v_, n_params_, opt_.lr, opt_.beta1, opt_.beta2,
            opt_.adam_eps, opt_.weight_decay, adam_ctr_, adam_c12_, cs_));
    stats_.kernel_launches += 2;
  }
  // rejoin the copy streams (all their work is already ordered before this
  // point by F3 / B3; the join makes it explicit for graph capture)
  G(cudaEventRecord(ev_join_os_, os_));
  G(cudaEventRecord(ev_join_ps_, ps_));
  G(cudaStreamWaitEvent(cs_, ev_join_os_, 0));
  G(cudaStreamWaitEvent(cs_, ev_join_ps_, 0));
  if (xs_) {  // SP+TP: the collectives' side stream (its last signals) joins too
    G(cudaEventRecord(ev_xs2cs_, xs_));
    G(cudaStreamWaitEvent(cs_, ev_xs2cs_, 0));
  }
  mark(0, 99, -1, true);  // step end marker
}

float Executor::last_loss() {
  G(cudaMemcpyAsync(loss_host_, loss_dev_, 4, cudaMemcpyDeviceToHost, cs_));
  G(cudaStreamSynchronize(cs_));
  return *loss_host_;
}

float Executor::step(const int* tokens, const int* labels) {
  load_batch(tokens, labels);
  step_resident();
  G(cudaMemcpyAsync(loss_host_, loss_dev_, 4, cudaMemcpyDeviceToHost, cs_));
  stats_.d2h_bytes = 4;
  G(cudaStreamSynchronize(cs_));
  G(cudaStreamSynchronize(os_));
  G(cudaStreamSynchronize(ps_));
  return *loss_host_;
}

Timeline Executor::timeline() const {
  ck(cudaStreamSynchronize(cs_), "sync");
  ck(cudaStreamSynchronize(os_), "sync");
  ck(cudaStreamSynchronize(ps_), "sync");
  Timeline t;
  t.n_layers = d_.n;
  t.rounding_buffer_bytes = sk_.total;
  t.swapped_layers = d_.n >= 2 ? d_.n - 2 : 0;
  for (const Mark& m : marks_) {
    if (m.kind == 99) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, ev_start_, m.b), "elapsed");
      const_cast<Executor*>(this)->stats_.step_ms = ms;
      continue;
    }
    if (!m.e) continue;
    float a = 0, b = 0;
    ck(cudaEventElapsedTime(&a, ev_start_, m.b), "elapsed");
    ck(cudaEventElapsedTime(&b, ev_start_, m.e), "elapsed");
    t.events.push_back({static_cast<Stream>(m.stream), static_cast<Kind>(m.kind), m.layer,
                        a * 1e-3, b * 1e-3});
  }
  StepStats& st = const_cast<Executor*>(this)->stats_;
  for (int c = 0; c < OP_NCLASS; ++c) {
    st.op_ms[c] = 0;
    st.op_flops[c] = 0;
    st.op_count[c] = 0;
  }
  st.copy_wait_ms = 0;
  for (const auto& w : waits_) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, w.first, w.second), "elapsed");
    st.copy_wait_ms += ms;
  }
  for (const OpMark& o : ops_) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, o.a, o.b), "elapsed");
    st.op_ms[o.cls] += ms;
    st.op_flops[o.cls] += o.flops;
    st.op_count[o.cls] += 1;
  }
  // Diagnostics: MEMO_OP_TRACE=<file> appends every timed op (class, start, end in
  // ms from step start) and every timeline event, for gap analysis of the step.
  if (const char* path = std::getenv("MEMO_OP_TRACE")) {
    if (FILE* f = std::fopen(path, "a")) {
      for (const OpMark& o : ops_) {
        float a = 0, b = 0;
        ck(cudaEventElapsedTime(&a, ev_start_, o.a), "elapsed");
        ck(cudaEventElapsedTime(&b, ev_start_, o.b), "elapsed");
        std::fprintf(f, "op,%d,%.4f,%.4f\n", o.cls, a, b);
      }
      for (const auto& e : t.events)
        std::fprintf(f, "ev,%d,%d,%d,%.4f,%.4f\n", static_cast<int>(e.stream), static_cast<int>(e.kind), e.layer,
                     e.start * 1e3, e.end * 1e3);
      std::fprintf(f, "step,%.4f\n", st.step_ms);
      std::fclose(f);
    }
  }
  return t;
}

}  // namespace memo
