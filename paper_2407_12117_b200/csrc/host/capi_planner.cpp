// capi_planner.cpp — extern "C" surface of the host planner (include/memo.h).
// Exceptions are caught here and mapped to the reference CLI exit codes.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <json.hpp>

#include "host/convert.hpp"
#include "host/planner.hpp"
#include "host/status.hpp"
#include "memo.h"

namespace memo {

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

ModelConfig from_c(const memo_model_config& c) {
  ModelConfig m;
  m.n_layers = c.n_layers;
  m.hidden = c.hidden;
  m.ffn_hidden = c.ffn_hidden;
  m.n_heads = c.n_heads;
  m.vocab = c.vocab;
  m.batch = c.batch;
  m.seq_len = c.seq_len;
  m.dtype_bytes = c.dtype_bytes;
  m.tp_degree = c.tp_degree;
  m.sp_or_cp_degree = c.sp_or_cp_degree;
  m.untied_classifier = c.untied_classifier != 0;
  for (int i = 0; i < MEMO_NUM_SKELETAL; ++i)
    if (!std::isnan(c.skeletal_weight[i]))
      m.skeletal_weight_overrides[kSkeletalNames[i]] = c.skeletal_weight[i];
  return m;
}

void to_c(const ModelConfig& m, memo_model_config& c) {
  c.n_layers = m.n_layers;
  c.hidden = m.hidden;
  c.ffn_hidden = m.ffn_hidden;
  c.n_heads = m.n_heads;
  c.vocab = m.vocab;
  c.batch = m.batch;
  c.seq_len = m.seq_len;
  c.dtype_bytes = m.dtype_bytes;
  c.tp_degree = m.tp_degree;
  c.sp_or_cp_degree = m.sp_or_cp_degree;
  c.untied_classifier = m.untied_classifier;
  for (int i = 0; i < MEMO_NUM_SKELETAL; ++i) {
    auto it = m.skeletal_weight_overrides.find(kSkeletalNames[i]);
    c.skeletal_weight[i] = it == m.skeletal_weight_overrides.end() ? NAN : it->second;
  }
}

HardwareConfig from_c(const memo_hardware_config& h) {
  HardwareConfig w;
  w.pcie_bandwidth = h.pcie_bandwidth;
  w.cpu_mem = h.cpu_mem;
  w.gpu_mem = h.gpu_mem;
  w.peak_flops = h.peak_flops;
  w.efficiency = h.efficiency;
  return w;
}

Skeletal from_c(const memo_skeletal_sizes& s) {
  Skeletal k;
  k.s_input = s.s_input;
  k.s_attn = s.s_attn;
  k.s_others = s.s_others;
  k.total = s.total;
  for (int i = 0; i < MEMO_NUM_SKELETAL; ++i)
    k.components.emplace_back(kSkeletalNames[i], s.component_bytes[i]);
  return k;
}

SwapDecision from_c(const memo_swap_plan& s) {
  SwapDecision d;
  d.alpha = s.alpha;
  d.mandatory_bytes = s.mandatory_bytes;
  d.swapped_bytes_per_layer = s.swapped_bytes_per_layer;
  d.cpu_footprint = s.cpu_footprint;
  d.swapped_layers = s.swapped_layers;
  if (s.has_mandatory_stall) d.mandatory_stall = s.mandatory_stall;
  return d;
}

void to_c(const SwapDecision& d, memo_swap_plan& s) {
  s.alpha = d.alpha;
  s.mandatory_bytes = d.mandatory_bytes;
  s.swapped_bytes_per_layer = d.swapped_bytes_per_layer;
  s.cpu_footprint = d.cpu_footprint;
  s.swapped_layers = d.swapped_layers;
  s.has_mandatory_stall = d.mandatory_stall.has_value();
  s.mandatory_stall = d.mandatory_stall.value_or(0.0);
}

Timing from_c(const memo_timing_model& t) {
  Timing m;
  m.t_fwd_layer = t.t_fwd_layer;
  m.t_bwd_layer = t.t_bwd_layer;
  m.t_attn_fwd = t.t_attn_fwd;
  m.t_embedding_fwd = t.t_embedding_fwd;
  m.t_embedding_bwd = t.t_embedding_bwd;
  m.t_classifier_fwd = t.t_classifier_fwd;
  m.t_classifier_bwd = t.t_classifier_bwd;
  m.bwd_ratio = t.bwd_ratio;
  return m;
}

Timeline from_c(const memo_schedule_event* ev, std::size_t n, std::uint64_t n_layers) {
  Timeline t;
  t.n_layers = n_layers;
  for (std::size_t i = 0; i < n; ++i)
    t.events.push_back({static_cast<Stream>(ev[i].stream), static_cast<Kind>(ev[i].kind),
                        ev[i].layer, ev[i].start, ev[i].end});
  return t;
}

template <class F>
int guarded(F&& f) {
  try {
    clear_error();
    f();
    return MEMO_OK;
  } catch (const PlanError& e) {
    return set_error(e.status, e.what());
  } catch (const std::bad_alloc& e) {
    return set_error(MEMO_ERR_HOST_MEMORY, "out of host memory");
  } catch (const std::exception& e) {
    return set_error(MEMO_ERR_INTERNAL, e.what());
  }
}

}  // namespace memo

using namespace memo;

extern "C" int memo_model_config_default(memo_model_config* c) {
  return guarded([&] { to_c(ModelConfig{}, *c); });
}

extern "C" int memo_hardware_config_default(memo_hardware_config* h) {
  return guarded([&] {
    HardwareConfig w;
    h->pcie_bandwidth = w.pcie_bandwidth;
    h->cpu_mem = w.cpu_mem;
    h->gpu_mem = w.gpu_mem;
    h->peak_flops = w.peak_flops;
    h->efficiency = w.efficiency;
  });
}

extern "C" int memo_parse_run_config(const char* json_text, memo_model_config* model,
                                     memo_hardware_config* hw, uint64_t* cap, uint64_t* align,
                                     double* budget, uint64_t* gran, double* t_layer,
                                     uint64_t* seed) {
  return guarded([&] {
    if (!json_text) throw ConfigError("null config text");
    RunConfig rc = parse_run_config(json_text);
    if (model) to_c(rc.model, *model);
    if (hw) {
      hw->pcie_bandwidth = rc.hardware.pcie_bandwidth;
      hw->cpu_mem = rc.hardware.cpu_mem;
      hw->gpu_mem = rc.hardware.gpu_mem;
      hw->peak_flops = rc.hardware.peak_flops;
      hw->efficiency = rc.hardware.efficiency;
    }
    if (cap) *cap = rc.planner.cap;
    if (align) *align = rc.planner.alignment;
    if (budget) *budget = rc.planner.time_budget;
    if (gran) *gran = rc.swap.token_granularity;
    if (t_layer) *t_layer = rc.swap.t_layer;
    if (seed) *seed = rc.synth_seed;
  });
}

extern "C" int memo_skeletal_sizes_of(const memo_model_config* cfg, memo_skeletal_sizes* out) {
  return guarded([&] {
    Skeletal s = skeletal_of(from_c(*cfg));
    out->s_input = s.s_input;
    out->s_attn = s.s_attn;
    out->s_others = s.s_others;
    out->total = s.total;
    for (int i = 0; i < MEMO_NUM_SKELETAL; ++i) out->component_bytes[i] = s.components[i].second;
  });
}

extern "C" int memo_solve_alpha(const memo_skeletal_sizes* sz, const memo_hardware_config* hw,
                                double t_layer_fwd, uint64_t n_layers, memo_swap_plan* out) {
  return guarded(
      [&] { to_c(solve_alpha_for(from_c(*sz), from_c(*hw), t_layer_fwd, n_layers), *out); });
}

extern "C" int memo_swap_plan_with_alpha(const memo_skeletal_sizes* sz,
                                         const memo_hardware_config* hw, double alpha,
                                         uint64_t n_layers, memo_swap_plan* out) {
  return guarded([&] { to_c(swap_with_alpha(from_c(*sz), from_c(*hw), alpha, n_layers), *out); });
}

extern "C" int memo_token_split_of(double alpha, uint64_t s, uint64_t g, memo_token_split* out) {
  return guarded([&] {
    TokenRange r = split_tokens(alpha, s, g);
    out->swap_tokens = r.swap_tokens;
    out->recompute_tokens = r.recompute_tokens;
  });
}

extern "C" int memo_count_params(const memo_model_config* cfg, memo_param_count* out) {
  return guarded([&] {
    ModelConfig m = from_c(*cfg);
    Params p = params_of(m);
    out->embedding = p.embedding;
    out->per_layer = p.per_layer;
    out->final_norm = p.final_norm;
    out->classifier = p.classifier;
    out->total = p.total(m);
  });
}

extern "C" double memo_flops_per_sample(const memo_model_config* cfg, uint64_t p) {
  return flops_per_sample(from_c(*cfg), p);
}

extern "C" double memo_mfu_from_tgs(const memo_model_config* cfg, const memo_hardware_config* hw,
                                    uint64_t p, double tgs) {
  return mfu_of_tgs(from_c(*cfg), from_c(*hw), p, tgs);
}

extern "C" int memo_analytic_timing(const memo_model_config* cfg, const memo_hardware_config* hw,
                                    memo_timing_model* out) {
  return guarded([&] {
    ModelConfig m = from_c(*cfg);
    Timing t = timing_of(m, from_c(*hw), params_of(m));
    out->t_fwd_layer = t.t_fwd_layer;
    out->t_bwd_layer = t.t_bwd_layer;
    out->t_attn_fwd = t.t_attn_fwd;
    out->t_embedding_fwd = t.t_embedding_fwd;
    out->t_embedding_bwd = t.t_embedding_bwd;
    out->t_classifier_fwd = t.t_classifier_fwd;
    out->t_classifier_bwd = t.t_classifier_bwd;
    out->bwd_ratio = t.bwd_ratio;
  });
}

extern "C" int memo_plan_model(const char* trace_text, uint64_t cap, double budget,
                               uint64_t alignment, char** plan_json) {
  return guarded([&] {
    if (!trace_text || !plan_json) throw ConfigError("null argument");
    Trace t = parse_trace_text(trace_text);
    *plan_json = dup_string(plan_to_json(plan_iteration(t, cap, budget, alignment)));
  });
}

extern "C" int memo_solve_dsa(const char* trace_text, uint64_t cap, double budget,
                              uint64_t alignment, char** result_json) {
  return guarded([&] {
    if (!trace_text || !result_json) throw ConfigError("null argument");
    Trace t = parse_trace_text(trace_text);
    DsaProblem p = make_problem(lifespans_of(t.segs.data(), t.segs.size(), false), cap, alignment);
    Solution s = solve_optimal(p, budget);
    nlohmann::json addrs = nlohmann::json::object();
    for (const auto& [id, a] : s.placement.offset) addrs[std::to_string(id)] = a;
    nlohmann::json j{{"status", static_cast<int>(s.status)},
                     {"peak", s.placement.peak},
                     {"addresses", addrs},
                     {"lower_bound", live_lower_bound(p)}};
    Solution h = best_fit(p);
    nlohmann::json ha = nlohmann::json::object();
    for (const auto& [id, a] : h.placement.offset) ha[std::to_string(id)] = a;
    j["heuristic"] = nlohmann::json{{"status", static_cast<int>(h.status)},
                                    {"peak", h.placement.peak},
                                    {"addresses", ha}};
    auto v = check_placement(s.placement, p);
    j["verify"] = v ? *v : std::string();
    *result_json = dup_string(j.dump());
  });
}

extern "C" int memo_trace_roundtrip(const char* trace_text, char** out_text) {
  return guarded([&] {
    if (!trace_text || !out_text) throw ConfigError("null argument");
    *out_text = dup_string(trace_to_text(parse_trace_text(trace_text)));
  });
}

extern "C" int memo_build_schedule(const memo_model_config* cfg, const memo_hardware_config* hw,
                                   const memo_skeletal_sizes* sz, const memo_swap_plan* swap,
                                   const memo_timing_model* tm, memo_schedule_event* events,
                                   size_t capacity, size_t* n_out) {
  return guarded([&] {
    Timeline t = schedule_of(from_c(*cfg), from_c(*hw), from_c(*sz), from_c(*swap), from_c(*tm));
    if (n_out) *n_out = t.events.size();
    if (!events) return;
    if (capacity < t.events.size()) throw ConfigError("event buffer too small");
    for (std::size_t i = 0; i < t.events.size(); ++i) {
      const Event& e = t.events[i];
      events[i] = {static_cast<int32_t>(e.stream), static_cast<int32_t>(e.kind), e.layer,
                   e.start, e.end};
    }
  });
}

extern "C" int memo_validate_schedule(const memo_schedule_event* events, size_t n,
                                      uint64_t n_layers, const memo_swap_plan* swap,
                                      char** violations) {
  return guarded([&] {
    auto bad = check_timeline(from_c(events, n, n_layers), from_c(*swap));
    std::string joined;
    for (std::size_t i = 0; i < bad.size(); ++i) joined += (i ? "\n" : "") + bad[i];
    *violations = dup_string(joined);
  });
}

extern "C" int memo_simulate(const memo_schedule_event* events, size_t n,
                             const memo_model_config* cfg, const memo_hardware_config* hw,
                             uint64_t p, memo_sim_report* out) {
  return guarded([&] {
    ModelConfig m = from_c(*cfg);
    SimResult r = simulate_timeline(from_c(events, n, m.n_layers), m, from_c(*hw), p);
    out->iteration_time = r.iteration_time;
    out->compute_blocked = r.compute_blocked;
    out->forward_blocked = r.forward_blocked;
    out->offload_stream_busy = r.offload_stream_busy;
    out->prefetch_stream_busy = r.prefetch_stream_busy;
    out->tgs = r.tgs;
    out->mfu = r.mfu;
  });
}

extern "C" int memo_fnv1a_hex(const char* data, size_t len, char out[19]) {
  return guarded([&] {
    std::string h = fnv1a(std::string(data, len));
    std::memcpy(out, h.c_str(), 19);
  });
}
