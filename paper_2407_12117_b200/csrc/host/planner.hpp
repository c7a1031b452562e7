// planner.hpp — host-side planning path of the MEMO hot path, restated in C++.
//
// Keeps the reference's config, memory-plan and executor interfaces
// (proj/include/actmem: types.hpp, trace.hpp, swap.hpp, dsa.hpp, bilevel.hpp,
// schedule.hpp, json_io.hpp) value-for-value so that a GlobalPlan, SwapPlan,
// TokenSplit or Schedule computed here is bit-identical to the reference's
// on the same input.  The implementation is independent: flat arrays instead
// of maps where possible, an allocation-free branch-and-bound, and a single
// text parser shared by the C ABI.  Compile with -ffp-contract=off so every
// double expression rounds exactly like the reference build.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace memo {

using Bytes = std::uint64_t;
using TensorId = std::uint64_t;
using Seconds = double;

constexpr Bytes KiB = 1024, MiB = 1024 * KiB, GiB = 1024 * MiB;

// ---------------------------------------------------------------- errors
// Same five failure classes as types.hpp:35-75; `code()` is the CLI exit code.
struct PlanError : std::runtime_error {
  int status;
  PlanError(int s, const std::string& w) : std::runtime_error(w), status(s) {}
};
struct ConfigError : PlanError {
  explicit ConfigError(const std::string& w) : PlanError(2, w) {}
};
struct TraceParseError : PlanError {
  std::size_t line;
  TraceParseError(std::size_t l, const std::string& w)
      : PlanError(2, l ? "line " + std::to_string(l) + ": " + w : w), line(l) {}
};
struct PlanningError : PlanError {
  explicit PlanningError(const std::string& w) : PlanError(3, w) {}
};
struct InfeasibleError : PlanError {
  explicit InfeasibleError(const std::string& w) : PlanError(3, w) {}
};
struct CpuInfeasibleError : PlanError {
  explicit CpuInfeasibleError(const std::string& w) : PlanError(4, w) {}
};

// ---------------------------------------------------------------- configs
// types.hpp:80-123
struct ModelConfig {
  std::uint64_t n_layers = 1, hidden = 1, ffn_hidden = 1, n_heads = 1, vocab = 1, batch = 1,
                seq_len = 1, dtype_bytes = 2, tp_degree = 1, sp_or_cp_degree = 1;
  bool untied_classifier = false;
  std::map<std::string, double> skeletal_weight_overrides;

  std::uint64_t seq_local() const { return seq_len / sp_or_cp_degree; }
  std::uint64_t hidden_local() const { return hidden / tp_degree; }
  std::uint64_t model_gpus() const { return tp_degree * sp_or_cp_degree; }
  void validate() const;
};

// types.hpp:126-141
struct HardwareConfig {
  double pcie_bandwidth = 32.0e9;
  Bytes cpu_mem = 2048 * GiB;
  Bytes gpu_mem = 80 * GiB;
  double peak_flops = 312.0e12;
  double efficiency = 0.5;
  void validate() const;
};

inline Bytes round_up(Bytes v, Bytes a) { return a <= 1 ? v : (v + a - 1) / a * a; }

// json_io.hpp:42-59
struct PlannerOptions {
  Bytes cap = 0;
  Bytes alignment = 512;
  Seconds time_budget = 60.0;
};
struct SwapOptions {
  std::uint64_t token_granularity = 128;
  double t_layer = 0;
};
struct RunConfig {
  ModelConfig model;
  HardwareConfig hardware;
  std::uint64_t synth_seed = 0;
  PlannerOptions planner;
  SwapOptions swap;
};
RunConfig parse_run_config(const std::string& json_text);  // json_io.hpp:141

// ---------------------------------------------------------------- trace
enum class Phase : int { EmbFwd, LayerFwd, ClsFwd, ClsBwd, LayerBwd, EmbBwd };
const char* phase_str(Phase p);
bool phase_is_fwd(Phase p);
bool phase_is_layer(Phase p);

struct Request {
  bool malloc;  // false = free
  TensorId id;
  Bytes size;
  bool operator==(const Request&) const = default;
};
struct Segment {
  Phase phase = Phase::LayerFwd;
  int layer = -1;
  std::vector<Request> reqs;
};
struct Trace {
  std::vector<Segment> segs;
  int n_layers = 0;
  std::size_t events() const;
};

struct Lifespan {
  TensorId id;
  Bytes size;
  std::size_t first;  // malloc event index
  std::size_t last;   // free event index (half-open end)
  bool skeletal;
  bool overlaps(const Lifespan& o) const { return first < o.last && o.first < last; }
};

Trace parse_trace_text(const std::string& text);      // trace.hpp:272
std::string trace_to_text(const Trace& t);             // trace.hpp:352
// trace.hpp:146; lifespans sorted by malloc index.
std::vector<Lifespan> lifespans_of(const Segment* segs, std::size_t n, bool allow_open);
void check_iteration_layout(const Trace& t);           // trace.hpp:376
std::vector<Request> canonical_form(const Segment& s); // trace.hpp:402

// ---------------------------------------------------------------- DSA
struct DsaProblem {  // dsa.hpp:40-79 (sizes already aligned)
  std::vector<Lifespan> items;
  Bytes cap = 0;  // 0 = unbounded
  Bytes alignment = 512;
  Bytes limit() const { return cap == 0 ? ~Bytes(0) : cap; }
};
DsaProblem make_problem(std::vector<Lifespan> spans, Bytes cap, Bytes alignment);

struct Placement {  // dsa.hpp:82 MemoryPlan
  std::map<TensorId, Bytes> offset;
  Bytes peak = 0;
};
enum class SolveStatus : int { Optimal = 0, Feasible = 1, TimedOut = 2, Infeasible = 3 };
struct Solution {
  SolveStatus status = SolveStatus::Infeasible;
  Placement placement;
};
Bytes live_lower_bound(const DsaProblem& p);                        // dsa.hpp:88
std::optional<std::string> check_placement(const Placement&, const DsaProblem&);  // :106
Solution best_fit(const DsaProblem& p);                             // dsa.hpp:151
Solution solve_optimal(const DsaProblem& p, Seconds budget);        // dsa.hpp:391

// ---------------------------------------------------------------- bi-level plan
struct LayerLayout {  // bilevel.hpp:35
  Placement fwd, bwd;
  Bytes fwd_peak = 0, bwd_peak = 0;
  bool optimal = true;
};
struct AbsAddr {
  std::size_t segment;
  TensorId id;
  Bytes offset;
};
struct ModelPlan {  // bilevel.hpp:164 GlobalPlan
  LayerLayout layer;
  Placement outer;
  std::map<std::size_t, TensorId> pseudo_of_segment;
  std::vector<AbsAddr> absolute;
  Bytes total_peak = 0;
  bool optimal = true;
};
LayerLayout plan_one_layer(const Segment& fwd, const Segment& bwd, Bytes cap, Seconds budget,
                           Bytes alignment);                                  // bilevel.hpp:66
ModelPlan plan_iteration(const Trace& t, Bytes cap, Seconds budget, Bytes alignment);  // :189
std::string plan_to_json(const ModelPlan& p);  // json_io.hpp:189 to_json(GlobalPlan).dump()
// The placement of a to_json(GlobalPlan) text: total_peak and (segment, tensor)
// -> absolute offset; returns the canonical dump.  ConfigError on bad input.
std::string parse_plan_json(const std::string& text, Bytes* total_peak,
                            std::map<std::pair<std::size_t, TensorId>, Bytes>* absolute);

// ---------------------------------------------------------------- skeletal / alpha
struct Skeletal {  // swap.hpp:67-89
  Bytes s_input = 0, s_attn = 0, s_others = 0, total = 0;
  std::vector<std::pair<std::string, Bytes>> components;  // emission order
};
extern const char* const kSkeletalNames[10];
extern const double kSkeletalDefaultWeights[10];
Skeletal skeletal_of(const ModelConfig& cfg);

struct SwapDecision {  // swap.hpp:94
  double alpha = 0.0;
  Bytes mandatory_bytes = 0, swapped_bytes_per_layer = 0, cpu_footprint = 0;
  std::uint64_t swapped_layers = 0;
  std::optional<Seconds> mandatory_stall;
};
SwapDecision solve_alpha_for(const Skeletal& sz, const HardwareConfig& hw, Seconds t_fwd,
                             std::uint64_t n_layers);  // swap.hpp:105
SwapDecision swap_with_alpha(const Skeletal& sz, const HardwareConfig& hw, double alpha,
                             std::uint64_t n_layers);  // schedule.hpp:409
struct TokenRange {
  std::uint64_t swap_tokens = 0, recompute_tokens = 0;
};
TokenRange split_tokens(double alpha, std::uint64_t s_local, std::uint64_t gran);  // swap.hpp:177

// ---------------------------------------------------------------- executor model
struct Params {  // schedule.hpp:31
  std::uint64_t embedding = 0, per_layer = 0, final_norm = 0, classifier = 0;
  std::uint64_t total(const ModelConfig& c) const {
    return embedding + c.n_layers * per_layer + final_norm + (c.untied_classifier ? classifier : 0);
  }
};
Params params_of(const ModelConfig& cfg);
double flops_per_sample(const ModelConfig& cfg, std::uint64_t p);
double mfu_of_tgs(const ModelConfig& cfg, const HardwareConfig& hw, std::uint64_t p, double tgs);

struct Timing {  // schedule.hpp:74
  Seconds t_fwd_layer = 0, t_bwd_layer = 0, t_attn_fwd = 0, t_embedding_fwd = 0,
          t_embedding_bwd = 0, t_classifier_fwd = 0, t_classifier_bwd = 0;
  double bwd_ratio = 2.0;
  Seconds t_recompute(double alpha) const { return (1.0 - alpha) * (t_fwd_layer - t_attn_fwd); }
  void validate() const;
};
Timing timing_of(const ModelConfig& cfg, const HardwareConfig& hw, const Params& p);

enum class Stream : int { Compute = 0, Offload = 1, Prefetch = 2 };
enum class Kind : int {
  EmbFwd = 0, LayerFwd, ClsFwd, ClsBwd, Recompute, LayerBwd, EmbBwd, Offload, Prefetch
};
const char* stream_str(Stream s);
const char* kind_str(Kind k);
struct Event {
  Stream stream = Stream::Compute;
  Kind kind = Kind::LayerFwd;
  int layer = -1;
  Seconds start = 0, end = 0;
};
struct Timeline {  // schedule.hpp:170 Schedule
  std::vector<Event> events;
  std::uint64_t n_layers = 0;
  Bytes rounding_buffer_bytes = 0;
  std::uint64_t swapped_layers = 0;
};
Timeline schedule_of(const ModelConfig& cfg, const HardwareConfig& hw, const Skeletal& sz,
                     const SwapDecision& swap, const Timing& tm);  // schedule.hpp:186
struct SimResult {  // schedule.hpp:250
  Seconds iteration_time = 0, compute_blocked = 0, forward_blocked = 0,
          offload_stream_busy = 0, prefetch_stream_busy = 0;
  double tgs = 0, mfu = 0;
};
SimResult simulate_timeline(const Timeline& t, const ModelConfig& cfg, const HardwareConfig& hw,
                            std::uint64_t p);                          // schedule.hpp:260
std::vector<std::string> check_timeline(const Timeline& t, const SwapDecision& swap);  // :301

std::string fnv1a(const std::string& data);  // json_io.hpp:265

}  // namespace memo
