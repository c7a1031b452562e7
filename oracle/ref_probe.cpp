// ref_probe.cpp — test infrastructure ONLY (the checker, never the product).
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include
// (actmem v0.1.0) into a probe binary, oracle/_ref/ref_probe, that
//   * dumps golden vectors for the planning path (tests/golden/*.json),
//   * plans an arbitrary trace with the reference's plan_model
//     (bilevel.hpp:189) so the executor's own trace can be checked live, and
//   * times the reference's `report`-style CPU pipeline (actmem.cpp:227-273)
//     for bench.py's cpu_baseline / --impl reference arm.
// Build recipe: oracle/Makefile.  Only tests/, bench.py's reference leg and
// __graft_entry__ may execute it.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "actmem/actmem.hpp"
#include "dsa_test_util.hpp"
#include "synthetic_traces.hpp"

using namespace actmem;
using Json = nlohmann::json;

namespace {

std::string read_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

Json skeletal_json(const ModelConfig& cfg) {
  Json comps = Json::array();
  for (auto& [name, bytes] : skeletal_components(cfg)) comps.push_back({name, bytes});
  auto sz = skeletal_sizes(cfg);
  return Json{{"components", comps},
              {"s_input", sz.s_input},
              {"s_attn", sz.s_attn},
              {"s_others", sz.s_others},
              {"total", sz.total}};
}

Json timing_json(const TimingModel& tm) {
  return Json{{"t_fwd_layer", tm.t_fwd_layer},         {"t_bwd_layer", tm.t_bwd_layer},
              {"t_attn_fwd", tm.t_attn_fwd},           {"t_embedding_fwd", tm.t_embedding_fwd},
              {"t_embedding_bwd", tm.t_embedding_bwd}, {"t_classifier_fwd", tm.t_classifier_fwd},
              {"t_classifier_bwd", tm.t_classifier_bwd}, {"bwd_ratio", tm.bwd_ratio}};
}

Json events_json(const Schedule& s) {
  Json ev = Json::array();
  for (const auto& e : s.events)
    ev.push_back({static_cast<int>(e.stream), static_cast<int>(e.kind), e.layer, e.start, e.end});
  return ev;
}

// The report pipeline for one RunConfig (actmem.cpp:227-273 minus the CLI):
// synth trace -> skeletal sizes -> params -> timing -> alpha -> plan -> schedule -> sim.
Json report(const RunConfig& rc, double forced_alpha, bool with_trace_text) {
  Json out;
  auto trace = synthesize_iteration_trace(rc.model, rc.synth);
  const std::string text = serialize_trace(trace);
  auto sz = skeletal_sizes(rc.model);
  auto params = count_params(rc.model);
  const std::uint64_t p_total = params.total(rc.model);
  TimingModel tm = analytic_timing(rc.model, rc.hardware, params);
  if (rc.swap.t_layer > 0) {  // actmem.cpp:62-74 resolve_timing
    const double scale = rc.swap.t_layer / tm.t_fwd_layer;
    tm.t_fwd_layer *= scale;
    tm.t_bwd_layer *= scale;
    tm.t_attn_fwd *= scale;
    tm.t_classifier_fwd *= scale;
    tm.t_classifier_bwd *= scale;
    tm.source = "measured";
  }
  out["model"] = to_json(rc.model);
  out["hardware"] = to_json(rc.hardware);
  out["skeletal"] = skeletal_json(rc.model);
  out["params"] = {{"embedding", params.embedding}, {"per_layer", params.per_layer},
                   {"final_norm", params.final_norm}, {"classifier", params.classifier},
                   {"total", p_total}};
  out["flops_per_sample"] = estimate_flops_per_sample(rc.model, p_total);
  out["timing"] = timing_json(tm);
  try {
    SwapPlan swap = forced_alpha >= 0
                        ? make_swap_plan_with_alpha(sz, rc.hardware, forced_alpha, rc.model.n_layers)
                        : solve_alpha(sz, rc.hardware, tm.t_fwd_layer, rc.model.n_layers);
    out["swap"] = to_json(swap);
    auto split = token_split(swap.alpha, rc.model.seq_local(), rc.swap.token_granularity);
    out["token_split"] = {{"swap_tokens", split.swap_tokens},
                          {"recompute_tokens", split.recompute_tokens}};
    auto sched = build_schedule(rc.model, rc.hardware, sz, swap, tm);
    out["schedule_events"] = events_json(sched);
    auto bad = validate_schedule(sched, swap);
    out["schedule_violations"] = bad;
    out["sim"] = to_json(simulate(sched, rc.model, rc.hardware, p_total));
  } catch (const CpuInfeasibleError& e) {
    out["swap_error"] = std::string("CpuInfeasibleError: ") + e.what();
  }
  out["trace_fnv"] = fnv1a_hex(text);
  out["trace_events"] = trace.event_count();
  auto plan = plan_model(trace, rc.planner.cap, rc.planner.time_budget, rc.planner.alignment);
  const std::string pj = to_json(plan).dump();
  out["plan_fnv"] = fnv1a_hex(pj);
  out["total_peak"] = plan.total_peak;
  out["fwd_peak"] = plan.layer_plan.fwd_peak;
  out["bwd_peak"] = plan.layer_plan.bwd_peak;
  out["optimal"] = plan.optimal;
  if (with_trace_text) {
    out["trace_text"] = text;
    out["plan_json"] = pj;
  }
  return out;
}

ModelConfig llama(std::uint64_t n, std::uint64_t h, std::uint64_t inter, std::uint64_t heads,
                  std::uint64_t vocab, std::uint64_t s, std::uint64_t tp, bool untied) {
  ModelConfig m;
  m.n_layers = n;
  m.hidden = h;
  m.ffn_hidden = inter * 3 / 2;  // SwiGLU: 3*h*f == 2*h*ffn_hidden (SURVEY discovery 5)
  m.n_heads = heads;
  m.vocab = vocab;
  m.batch = 1;
  m.seq_len = s;
  m.dtype_bytes = 2;
  m.tp_degree = tp;
  m.sp_or_cp_degree = 1;
  m.untied_classifier = untied;
  return m;
}

HardwareConfig b200_hw(Bytes cpu_mem = 256 * kGiB) {
  HardwareConfig hw;
  hw.pcie_bandwidth = 64e9;
  hw.cpu_mem = cpu_mem;
  hw.gpu_mem = 180ull * 1000 * 1000 * 1000;
  hw.peak_flops = 2.25e15;
  hw.efficiency = 0.5;
  return hw;
}

Json goldens_configs() {
  Json out = Json::object();
  auto add = [&](const std::string& name, ModelConfig m, HardwareConfig hw, double alpha,
                 bool text) {
    RunConfig rc;
    rc.model = m;
    rc.hardware = hw;
    rc.planner.cap = 0;
    rc.planner.alignment = 512;
    rc.planner.time_budget = 60.0;
    out[name] = report(rc, alpha, text);
  };
  // BASELINE.json configs (SURVEY §8 restatement). cfg1 is the GPT-shaped tiny model.
  ModelConfig c1;
  c1.n_layers = 2; c1.hidden = 256; c1.ffn_hidden = 1024; c1.n_heads = 4; c1.vocab = 512;
  c1.batch = 1; c1.seq_len = 4096; c1.dtype_bytes = 2;
  add("cfg1", c1, b200_hw(), 0.5, true);
  ModelConfig c1p = c1;
  c1p.n_layers = 4;
  add("cfg1p", c1p, b200_hw(), 0.5, true);
  add("cfg2", llama(4, 4096, 11008, 32, 32000, 131072, 1, true), b200_hw(), -1, true);
  add("cfg3", llama(32, 4096, 11008, 32, 32000, 1048576, 8, true), b200_hw(), -1, true);
  for (int tp : {2, 4, 8})
    add("cfg4_tp" + std::to_string(tp), llama(40, 5120, 13824, 40, 32000, 524288, tp, true),
        b200_hw(tp == 2 ? 1024 * kGiB : 256 * kGiB), -1, true);
  for (int k = 0; k <= 8; ++k)
    add("cfg5_a" + std::to_string(k), llama(32, 4096, 11008, 32, 32000, 262144, 1, true),
        b200_hw(1024 * kGiB), k / 8.0, k == 0);
  // The reference's own config files.
  for (const char* f : {"toy", "7b-1m"}) {
    RunConfig rc = load_run_config(std::string("/root/reference/proj/configs/") + f + ".json");
    out[std::string("ref_") + f] = report(rc, -1, true);
  }
  return out;
}

Json goldens_random_plans() {
  Json cases = Json::array();
  std::mt19937_64 rng(20240717);
  for (int i = 0; i < 40; ++i) {
    testutil::SyntheticTraceOptions opt;
    opt.n_layers = 1 + static_cast<int>(rng() % 4);
    opt.transients_per_segment = 2 + rng() % 5;
    opt.max_size = 1 + rng() % 2000;
    opt.embedding_held_tensor = (rng() % 3) == 0;
    auto trace = testutil::random_iteration_trace(rng, opt);
    const Bytes alignment = (i % 2) ? 1 : 512;
    auto plan = plan_model(trace, 0, 30.0, alignment);
    cases.push_back({{"trace", serialize_trace(trace)},
                     {"alignment", alignment},
                     {"plan_json", to_json(plan).dump()},
                     {"optimal", plan.optimal}});
  }
  return cases;
}

std::string single_segment_trace(const DsaInstance& inst) {
  // Re-emit the lifespans as one layer_fwd segment in event order.
  std::size_t n_ev = 0;
  for (const auto& t : inst.tensors) n_ev = std::max(n_ev, t.free_index + 1);
  std::vector<std::string> ev(n_ev);
  for (const auto& t : inst.tensors) {
    ev[t.alloc_index] = "malloc " + std::to_string(t.tensor_id) + " " + std::to_string(t.size);
    ev[t.free_index] = "free " + std::to_string(t.tensor_id) + " " + std::to_string(t.size);
  }
  std::string s = "# segment layer_fwd 0\n";
  for (auto& e : ev)
    if (!e.empty()) s += e + "\n";
  return s;
}

Json dsa_result_json(const SolveResult& r) {
  Json addrs = Json::object();
  for (auto& [id, a] : r.plan.addresses) addrs[std::to_string(id)] = a;
  return Json{{"status", static_cast<int>(r.status)}, {"peak", r.plan.peak}, {"addresses", addrs}};
}

Json goldens_dsa() {
  Json cases = Json::array();
  for (std::uint64_t seed : {42ull, 1234ull, 777ull}) {
    std::mt19937_64 rng(seed);
    for (int i = 0; i < 25; ++i) {
      const std::size_t n = 2 + rng() % 7;
      auto inst = testutil::random_instance(rng, n, 1 + rng() % 16);
      auto res = solve_exact(inst, 10.0);
      auto heur = solve_heuristic(inst);
      cases.push_back({{"trace", single_segment_trace(inst)},
                       {"alignment", 1},
                       {"lower_bound", dsa_lower_bound(inst)},
                       {"oracle_peak", testutil::oracle_optimal_peak(inst)},
                       {"exact", dsa_result_json(res)},
                       {"heuristic", dsa_result_json(heur)}});
    }
  }
  return cases;
}

Json goldens_swap() {
  Json cases = Json::array();
  auto gb = [](double i, double a, double o) {
    SkeletalSizes sz;
    sz.s_input = static_cast<Bytes>(i * 1e9);
    sz.s_attn = static_cast<Bytes>(a * 1e9);
    sz.s_others = static_cast<Bytes>(o * 1e9);
    sz.total = sz.s_input + sz.s_attn + sz.s_others;
    return sz;
  };
  auto emit = [&](const SkeletalSizes& sz, const HardwareConfig& hw, double t, std::uint64_t n) {
    Json c{{"sz", {sz.s_input, sz.s_attn, sz.s_others, sz.total}},
           {"hw", to_json(hw)}, {"t_layer", t}, {"n_layers", n}};
    try {
      c["plan"] = to_json(solve_alpha(sz, hw, t, n));
    } catch (const CpuInfeasibleError&) {
      c["error"] = "CpuInfeasibleError";
    }
    cases.push_back(c);
  };
  HardwareConfig hw;
  hw.pcie_bandwidth = 1e9; hw.cpu_mem = 1ull << 60;
  emit(gb(2, 1, 13), hw, 8.0, 32);
  hw.pcie_bandwidth = 16e9;
  emit(gb(2, 1, 13), hw, 1.0, 32);
  hw.pcie_bandwidth = 1e9;
  emit(gb(4, 2, 10), hw, 2.0, 16);
  hw.pcie_bandwidth = 64e9; hw.cpu_mem = 30ull * 1000 * 1000 * 1000;
  emit(gb(4, 2, 10), hw, 1.0, 32);
  hw.pcie_bandwidth = 1.0; hw.cpu_mem = 1;
  emit(gb(2, 1, 13), hw, 1.0, 2);
  std::mt19937_64 rng(5150);
  for (int round = 0; round < 200; ++round) {
    auto sz = gb(1.0 + rng() % 4, 0.5 + (rng() % 4) / 2.0, 4.0 + rng() % 16);
    HardwareConfig h2;
    h2.pcie_bandwidth = (1 + rng() % 12) * 1.0e9;
    h2.cpu_mem = (20 + rng() % 300) * 1000000000ull;
    const Seconds t_layer = 0.5 + static_cast<double>(rng() % 8);
    const std::uint64_t n = 3 + rng() % 40;
    emit(sz, h2, t_layer, n);
  }
  Json splits = Json::array();
  std::mt19937_64 r2(31337);
  for (int i = 0; i < 200; ++i) {
    double a = (i < 9) ? i / 8.0 : static_cast<double>(r2() % 100001) / 100000.0;
    std::uint64_t s = (i % 5 == 0) ? 1 + r2() % 5000 : 128 * (1 + r2() % 8192);
    std::uint64_t g = (i % 7 == 0) ? 1 + r2() % 300 : 128;
    auto sp = token_split(a, s, g);
    splits.push_back({a, s, g, sp.swap_tokens, sp.recompute_tokens});
  }
  return Json{{"solve_alpha", cases}, {"token_split", splits}};
}

Json goldens_schedule() {
  Json cases = Json::array();
  std::mt19937_64 rng(99);
  for (int round = 0; round < 60; ++round) {
    ModelConfig cfg;
    cfg.n_layers = 1 + rng() % 10;
    cfg.hidden = 4096; cfg.ffn_hidden = 16384; cfg.n_heads = 32; cfg.vocab = 50257;
    cfg.seq_len = 4096;
    HardwareConfig hw;
    hw.pcie_bandwidth = 0.5e9 + static_cast<double>(rng() % 64) * 1e9 / 8.0;
    SkeletalSizes sz;
    sz.total = 1 + rng() % (1ull << 32);
    TimingModel tm;
    tm.t_fwd_layer = 0.25 + static_cast<double>(rng() % 16) / 4.0;
    tm.t_bwd_layer = 2.0 * tm.t_fwd_layer;
    tm.t_attn_fwd = tm.t_fwd_layer * static_cast<double>(rng() % 100) / 100.0;
    tm.t_classifier_fwd = static_cast<double>(rng() % 3) / 2.0;
    tm.t_classifier_bwd = 2.0 * tm.t_classifier_fwd;
    SwapPlan swap;
    swap.swapped_bytes_per_layer = rng() % (1ull << 34);
    swap.mandatory_bytes = swap.swapped_bytes_per_layer;
    swap.alpha = static_cast<double>(rng() % 9) / 8.0;
    auto sched = build_schedule(cfg, hw, sz, swap, tm);
    const auto p = count_params(cfg).total(cfg);
    cases.push_back({{"model", to_json(cfg)}, {"hardware", to_json(hw)},
                     {"sz_total", sz.total}, {"timing", timing_json(tm)},
                     {"swap", to_json(swap)}, {"params", p},
                     {"events", events_json(sched)},
                     {"violations", validate_schedule(sched, swap)},
                     {"timeline_csv", schedule_timeline_csv(sched)},
                     {"sim", to_json(simulate(sched, cfg, hw, p))}});
  }
  return cases;
}

int usage() {
  std::cerr << "usage: ref_probe goldens <dir> | plan <trace> <cap> <budget> <align> | "
               "dsa <trace> <cap> <budget> <align> | synth <config.json> | "
               "report <config.json> [alpha] | bench_report <config.json> <iters> | frag <trace> [cap]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string op = argv[1];
  try {
    if (op == "goldens" && argc >= 3) {
      const std::string dir = argv[2];
      std::ofstream(dir + "/ref_configs.json") << goldens_configs().dump(1) << "\n";
      std::ofstream(dir + "/ref_random_plans.json") << goldens_random_plans().dump(1) << "\n";
      std::ofstream(dir + "/ref_dsa.json") << goldens_dsa().dump(1) << "\n";
      std::ofstream(dir + "/ref_swap.json") << goldens_swap().dump(1) << "\n";
      std::ofstream(dir + "/ref_schedule.json") << goldens_schedule().dump(1) << "\n";
      return 0;
    }
    if ((op == "plan" || op == "dsa") && argc >= 6) {
      auto trace = parse_trace(read_file(argv[2]));
      const Bytes cap = std::stoull(argv[3]);
      const double budget = std::stod(argv[4]);
      const Bytes align = std::stoull(argv[5]);
      if (op == "plan") {
        std::cout << to_json(plan_model(trace, cap, budget, align)).dump() << "\n";
      } else {
        auto inst = make_dsa_instance(extract_lifespans(trace).lifespans, cap, align);
        std::cout << dsa_result_json(solve_exact(inst, budget)).dump() << "\n";
      }
      return 0;
    }
    if (op == "frag" && argc >= 3) {
      // The reference CLI's `frag` (actmem.cpp:194-225) on a given trace: plan it,
      // replay it through the caching-allocator simulator (capacity = plan + 10 %
      // unless given) and through the static plan, and print the comparison.
      auto trace = parse_trace(read_file(argv[2]));
      GlobalPlan gp = plan_model(trace, 0, 60.0, 512);
      const Bytes capacity = argc >= 4 ? std::stoull(argv[3]) : gp.total_peak + gp.total_peak / 10;
      CachingAllocatorConfig acfg;
      acfg.capacity = capacity;
      FragReport caching = simulate_caching_allocator(trace, acfg, false);
      FragReport planned = simulate_planned(trace, gp, 0, false);
      Json j = to_json(compare(caching, planned));
      j["capacity"] = capacity;
      j["plan_total_peak"] = gp.total_peak;
      std::cout << j.dump() << "\n";
      return 0;
    }
    if (op == "synth" && argc >= 3) {
      RunConfig rc = load_run_config(argv[2]);
      std::cout << serialize_trace(synthesize_iteration_trace(rc.model, rc.synth));
      return 0;
    }
    if (op == "report" && argc >= 3) {
      RunConfig rc = load_run_config(argv[2]);
      const double alpha = argc >= 4 ? std::stod(argv[3]) : -1.0;
      std::cout << report(rc, alpha, false).dump() << "\n";
      return 0;
    }
    if (op == "bench_report" && argc >= 4) {
      // Times the full report pipeline `iters` times (single-threaded reference code).
      RunConfig rc = load_run_config(argv[2]);
      const int iters = std::stoi(argv[3]);
      const double alpha = argc >= 5 ? std::stod(argv[4]) : -1.0;
      report(rc, alpha, false);
      auto t0 = std::chrono::steady_clock::now();
      std::string sink;
      for (int i = 0; i < iters; ++i) sink = report(rc, alpha, false).dump();
      auto t1 = std::chrono::steady_clock::now();
      const double s = std::chrono::duration<double>(t1 - t0).count();
      std::cout << Json{{"iters", iters}, {"seconds", s}, {"per_iter_s", s / iters},
                        {"bytes", sink.size()}}.dump()
                << "\n";
      return 0;
    }
  } catch (const ConfigError& e) {
    std::cerr << "config error: " << e.what() << "\n";
    return 2;
  } catch (const TraceParseError& e) {
    std::cerr << "trace error: " << e.what() << "\n";
    return 2;
  } catch (const InfeasibleError& e) {
    std::cerr << "infeasible: " << e.what() << "\n";
    return 3;
  } catch (const PlanningError& e) {
    std::cerr << "planning error: " << e.what() << "\n";
    return 3;
  } catch (const CpuInfeasibleError& e) {
    std::cerr << "cpu infeasible: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return usage();
}
