// actmem_b200 — the reference's `report` (proj/tools/actmem.cpp:227-273) with the
// simulated executor replaced by a real B200 training step.
//
// C++ host code over the reference's own types: the actmem headers are included
// IN PLACE from the reference tree (-I<reference>/proj/include, nothing copied)
// and every B200 call goes through libmemo's C ABI (include/memo.h).  The flow
// is cmd_report's, step for step:
//
//   cmd_report (actmem.cpp)                      here
//   load_config                                  actmem::load_run_config (json_io.hpp:167)
//   synthesize_iteration_trace(rc.model)         memo_exec_create + memo_exec_trace: the
//                                                executor's OWN request trace (trace.hpp format)
//   plan_model(trace, cap, budget, alignment)    actmem::plan_model on that trace (bilevel.hpp:189),
//                                                bound with memo_exec_bind_plan: the executor
//                                                replays the reference planner's offsets
//   resolve_swap                                 the executor's solve_alpha (memo_exec_get_info)
//   build_schedule + simulate                    memo_exec_step x K, memo_exec_timeline ->
//                                                actmem::Schedule -> actmem::validate_schedule +
//                                                actmem::simulate on the MEASURED timeline
//   simulate_caching_allocator / _planned        the same two calls on the executor's trace
//
// and it writes cmd_report's manifest keys {version, inputs.config.{path,
// fnv1a}, model, hardware, param_count, skeletal, alpha, plan{total_peak,
// layer_fwd_peak, layer_bwd_peak, optimal}, sim, frag} plus a "measured" block.
//
//   actmem_b200 report --config cfg.json [--alpha A] [--steps K] [--seed N]
//                      [--out manifest.json] [--timeline timeline.csv]
//
// Exit codes: actmem.cpp:351-371 (0 ok, 1 internal / schedule violation,
// 2 bad input, 3 infeasible, 4 host memory).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "actmem/allocator.hpp"
#include "actmem/bilevel.hpp"
#include "actmem/json_io.hpp"
#include "actmem/schedule.hpp"
#include "actmem/swap.hpp"
#include "actmem/trace.hpp"
#include "memo.h"

namespace {

struct MemoStatus : std::runtime_error {
  int code;
  MemoStatus(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

void check(int rc, const char* what) {
  if (rc != MEMO_OK) throw MemoStatus(rc, std::string(what) + ": " + memo_last_error());
}

memo_model_config to_c(const actmem::ModelConfig& m) {
  memo_model_config c{};
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
  c.untied_classifier = m.untied_classifier ? 1 : 0;
  for (double& w : c.skeletal_weight) w = NAN;  // the executor's Llama weights
  return c;
}

memo_hardware_config to_c(const actmem::HardwareConfig& h) {
  return {h.pcie_bandwidth, h.cpu_mem, h.gpu_mem, h.peak_flops, h.efficiency};
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw actmem::ConfigError("cannot open " + path);
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

std::string take(char* p) {
  std::string s = p ? p : "";
  memo_free(p);
  return s;
}

uint64_t splitmix64(uint64_t x) {  // synth.hpp's generator
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

struct Flags {
  std::string config, out, timeline;
  double alpha = -1.0;
  int steps = 3;
  uint64_t seed = 1234;
};

int report(const Flags& f) {
  const std::string config_text = read_file(f.config);
  const actmem::RunConfig rc = actmem::load_run_config(f.config);

  memo_exec_options opt;
  check(memo_exec_options_default(&opt), "options");
  opt.seed = f.seed;
  opt.alpha = f.alpha;
  opt.token_granularity = rc.swap.token_granularity;
  opt.t_layer = rc.swap.t_layer;
  opt.plan_time_budget = rc.planner.time_budget;
  opt.alignment = rc.planner.alignment;
  const memo_model_config mc = to_c(rc.model);
  const memo_hardware_config hc = to_c(rc.hardware);
  memo_exec* ctx = nullptr;
  check(memo_exec_create(&mc, &hc, &opt, &ctx), "memo_exec_create");

  // the reference planner on the executor's own trace, replayed by the executor
  char* tp = nullptr;
  check(memo_exec_trace(ctx, &tp), "memo_exec_trace");
  const std::string trace_text = take(tp);
  const actmem::IterationTrace trace = actmem::parse_trace(trace_text);
  const actmem::GlobalPlan gp =
      actmem::plan_model(trace, rc.planner.cap, rc.planner.time_budget, rc.planner.alignment);
  const std::string plan_json = actmem::to_json(gp).dump();
  check(memo_exec_bind_plan(ctx, plan_json.c_str()), "memo_exec_bind_plan");

  // K real steps on synthetic tokens (labels = next token)
  const uint64_t S = rc.model.seq_len, V = rc.model.vocab;
  std::vector<int32_t> toks(S), labels(S);
  for (uint64_t t = 0; t < S; ++t) toks[t] = static_cast<int32_t>(splitmix64(f.seed + t) % V);
  for (uint64_t t = 0; t + 1 < S; ++t) labels[t] = toks[t + 1];
  labels[S - 1] = -1;
  std::vector<float> losses;
  for (int k = 0; k < f.steps; ++k) {
    float loss = 0;
    check(memo_exec_step(ctx, toks.data(), labels.data(), &loss), "memo_exec_step");
    losses.push_back(loss);
  }

  // the measured timeline of the last step as the reference's Schedule
  size_t n = 0;
  check(memo_exec_timeline(ctx, nullptr, 0, &n), "memo_exec_timeline");
  std::vector<memo_schedule_event> ev(n);
  check(memo_exec_timeline(ctx, ev.data(), n, &n), "memo_exec_timeline");
  memo_exec_info info;
  check(memo_exec_get_info(ctx, &info), "memo_exec_get_info");
  actmem::Schedule sched;
  sched.n_layers = rc.model.n_layers;
  sched.rounding_buffer_bytes = info.rb_bytes;
  sched.swapped_layers = rc.model.n_layers >= 2 ? rc.model.n_layers - 2 : 0;
  for (const auto& e : ev)
    sched.events.push_back({static_cast<actmem::StreamId>(e.stream), static_cast<actmem::EventKind>(e.kind),
                            e.layer, e.start, e.end});
  actmem::SwapPlan swap;
  swap.alpha = info.swap.alpha;
  swap.mandatory_bytes = info.swap.mandatory_bytes;
  swap.swapped_bytes_per_layer = info.swap.swapped_bytes_per_layer;
  swap.cpu_footprint = info.swap.cpu_footprint;
  swap.swapped_layers = info.swap.swapped_layers;
  if (info.swap.has_mandatory_stall) swap.mandatory_stall = info.swap.mandatory_stall;
  const std::vector<std::string> violations = actmem::validate_schedule(sched, swap);
  const actmem::ParamCount params = actmem::count_params(rc.model);
  const actmem::SimReport rep = actmem::simulate(sched, rc.model, rc.hardware, params.total(rc.model));

  actmem::CachingAllocatorConfig acfg;
  acfg.capacity = gp.total_peak + gp.total_peak / 10;
  const actmem::FragReport caching = actmem::simulate_caching_allocator(trace, acfg);
  const actmem::FragReport planned = actmem::simulate_planned(trace, gp);

  actmem::Json viol = actmem::Json::array();
  for (const auto& v : violations) viol.push_back(v);
  actmem::Json manifest{
      {"version", std::string("actmem-b200 (") + memo_version() + ")"},
      {"inputs", actmem::Json{{"config", actmem::Json{{"path", f.config},
                                                      {"fnv1a", actmem::fnv1a_hex(config_text)}}}}},
      {"model", actmem::to_json(rc.model)},
      {"hardware", actmem::to_json(rc.hardware)},
      {"param_count", params.total(rc.model)},
      // the executor's skeletal model (its Llama component weights)
      {"skeletal", actmem::Json{{"total", info.skeletal.total},
                                {"s_input", info.skeletal.s_input},
                                {"s_attn", info.skeletal.s_attn},
                                {"s_others", info.skeletal.s_others}}},
      {"alpha", actmem::to_json(swap)},
      {"plan", actmem::Json{{"total_peak", gp.total_peak},
                            {"layer_fwd_peak", gp.layer_plan.fwd_peak},
                            {"layer_bwd_peak", gp.layer_plan.bwd_peak},
                            {"optimal", gp.optimal}}},
      {"sim", actmem::to_json(rep)},
      {"frag", actmem::to_json(actmem::compare(caching, planned))},
      {"measured",
       actmem::Json{{"steps", f.steps},
                    {"losses", losses},
                    {"last_step_ms", info.last_step_ms},
                    {"schedule_violations", viol},
                    {"in_layer_copy_wait_ms", info.copy_wait_ms},
                    {"swap_tokens", info.split.swap_tokens},
                    {"recompute_tokens", info.split.recompute_tokens},
                    {"arena_bytes", info.arena_bytes},
                    {"rounding_buffer_bytes", info.rb_bytes},
                    {"state_bytes", info.state_bytes},
                    {"device_bytes_reserved", info.device_bytes},
                    {"pinned_bytes", info.pinned_bytes},
                    {"offload_bytes", info.offload_bytes},
                    {"prefetch_bytes", info.prefetch_bytes},
                    {"plan_fnv1a", actmem::fnv1a_hex(plan_json)},
                    {"trace_fnv1a", actmem::fnv1a_hex(trace_text)}}}};
  memo_exec_destroy(ctx);

  const std::string out = manifest.dump(2) + "\n";
  if (f.out.empty()) {
    std::cout << out;
  } else {
    std::ofstream(f.out) << out;
  }
  if (!f.timeline.empty()) std::ofstream(f.timeline) << actmem::schedule_timeline_csv(sched);
  std::cerr << "report: alpha " << swap.alpha << ", total_peak " << gp.total_peak << ", mfu " << rep.mfu
            << ", " << violations.size() << " schedule violations\n";
  return violations.empty() ? 0 : 1;
}

int usage() {
  std::cerr << "usage: actmem_b200 report --config cfg.json [--alpha A] [--steps K] [--seed N]\n"
               "                         [--out manifest.json] [--timeline timeline.csv]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "report") != 0) return usage();
  Flags f;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw actmem::ConfigError("missing value for " + a);
      return argv[++i];
    };
    try {
      if (a == "--config") f.config = val();
      else if (a == "--out") f.out = val();
      else if (a == "--timeline") f.timeline = val();
      else if (a == "--alpha") f.alpha = std::stod(val());
      else if (a == "--steps") f.steps = std::stoi(val());
      else if (a == "--seed") f.seed = std::stoull(val());
      else return usage();
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return 2;
    }
  }
  if (f.config.empty() || f.steps < 1) return usage();
  // exit codes as actmem.cpp:351-371
  try {
    return report(f);
  } catch (const MemoStatus& e) {
    std::cerr << "error: " << e.what() << "\n";
    return e.code;
  } catch (const actmem::CpuInfeasibleError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  } catch (const actmem::InfeasibleError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const actmem::PlanningError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const actmem::ConfigError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const actmem::TraceParseError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
