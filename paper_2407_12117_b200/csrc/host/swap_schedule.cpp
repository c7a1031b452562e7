// swap_schedule.cpp — skeletal byte model, the alpha program, the token
// split, the parameter/FLOP model, the 3-stream executor model and its
// validator, plus RunConfig JSON parsing.
//
// Arithmetic is written in the same association order as the reference
// (proj/include/actmem/swap.hpp, schedule.hpp) and this file is compiled with
// -ffp-contract=off, so every double (alpha, times, MFU) is bit-identical.
#include <algorithm>
#include <cmath>
#include <limits>

#include <json.hpp>

#include "host/planner.hpp"

namespace memo {

// ---------------------------------------------------------------- skeletal
const char* const kSkeletalNames[10] = {"layer_input", "input_norm",     "q",       "k",
                                        "v",           "attn_out",       "attn_proj",
                                        "post_attn_norm", "ffn_fc1",     "ffn_act"};
// Multiples of b*s'*h' elements; sum 16 (swap.hpp:38-45).
const double kSkeletalDefaultWeights[10] = {2.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 4.0, 3.0};

Skeletal skeletal_of(const ModelConfig& cfg) {
  cfg.validate();
  const double unit = static_cast<double>(cfg.batch) * static_cast<double>(cfg.seq_local()) *
                      static_cast<double>(cfg.hidden_local()) *
                      static_cast<double>(cfg.dtype_bytes);
  Skeletal sz;
  for (int i = 0; i < 10; ++i) {
    double w = kSkeletalDefaultWeights[i];
    auto ov = cfg.skeletal_weight_overrides.find(kSkeletalNames[i]);
    if (ov != cfg.skeletal_weight_overrides.end()) w = ov->second;
    if (w < 0) throw ConfigError(std::string("skeletal weight for ") + kSkeletalNames[i] + " is negative");
    const Bytes b = static_cast<Bytes>(std::llround(w * unit));
    sz.components.emplace_back(kSkeletalNames[i], b);
    sz.total += b;
    if (i == 0)
      sz.s_input += b;
    else if (i == 5)
      sz.s_attn += b;
    else
      sz.s_others += b;
  }
  return sz;
}

// ---------------------------------------------------------------- alpha
SwapDecision solve_alpha_for(const Skeletal& sz, const HardwareConfig& hw, Seconds t_fwd,
                             std::uint64_t n_layers) {
  hw.validate();
  if (t_fwd <= 0) throw ConfigError("t_layer_fwd must be positive");
  SwapDecision d;
  d.mandatory_bytes = sz.s_input + sz.s_attn;
  if (n_layers <= 2) {  // the last two layers never swap
    d.alpha = 1.0;
    d.swapped_bytes_per_layer = d.mandatory_bytes + sz.s_others;
    return d;
  }
  d.swapped_layers = n_layers - 2;
  const double bw_budget = hw.pcie_bandwidth * t_fwd;  // bytes one forward can hide
  const double host_budget =
      static_cast<double>(hw.cpu_mem) / static_cast<double>(d.swapped_layers);
  const double must = static_cast<double>(d.mandatory_bytes);
  if (must > host_budget)
    throw CpuInfeasibleError("mandatory offload of " + std::to_string(d.mandatory_bytes) +
                             " bytes/layer exceeds cpu_mem/(n-2) = " +
                             std::to_string(host_budget));
  double a = 1.0;
  if (sz.s_others != 0) {
    const double rest = static_cast<double>(sz.s_others);
    a = std::min((bw_budget - must) / rest, (host_budget - must) / rest);
  }
  const Seconds must_time = must / hw.pcie_bandwidth;
  if (a < 0.0) {
    d.alpha = 0.0;
    const Seconds stall = must_time - t_fwd;
    if (stall > 0) d.mandatory_stall = stall;
  } else {
    d.alpha = std::min(a, 1.0);
    if (must_time > t_fwd) {
      const Seconds stall = must_time - t_fwd;
      if (stall > 0) d.mandatory_stall = stall;
    }
  }
  d.swapped_bytes_per_layer =
      d.mandatory_bytes + static_cast<Bytes>(std::floor(d.alpha * static_cast<double>(sz.s_others)));
  d.cpu_footprint = d.swapped_layers * d.swapped_bytes_per_layer;
  if (d.cpu_footprint > hw.cpu_mem)
    throw CpuInfeasibleError("internal: cpu footprint exceeds capacity after solve");
  return d;
}

SwapDecision swap_with_alpha(const Skeletal& sz, const HardwareConfig& hw, double alpha,
                             std::uint64_t n_layers) {
  if (alpha < 0.0 || alpha > 1.0) throw ConfigError("alpha must be in [0, 1]");
  SwapDecision d;
  d.alpha = alpha;
  d.mandatory_bytes = sz.s_input + sz.s_attn;
  d.swapped_bytes_per_layer =
      d.mandatory_bytes + static_cast<Bytes>(std::floor(alpha * static_cast<double>(sz.s_others)));
  d.swapped_layers = n_layers >= 2 ? n_layers - 2 : 0;
  d.cpu_footprint = d.swapped_layers * d.swapped_bytes_per_layer;
  if (d.cpu_footprint > hw.cpu_mem)
    throw CpuInfeasibleError("alpha " + std::to_string(alpha) +
                             " needs more host memory than available");
  return d;
}

TokenRange split_tokens(double alpha, std::uint64_t s_local, std::uint64_t gran) {
  if (alpha < 0.0 || alpha > 1.0) throw ConfigError("alpha must be in [0, 1]");
  if (gran == 0) gran = 1;
  TokenRange r;
  if (alpha >= 1.0) {
    r.swap_tokens = s_local;
  } else {
    std::uint64_t k = static_cast<std::uint64_t>(std::floor(alpha * static_cast<double>(s_local)));
    k = std::min(k, s_local);
    r.swap_tokens = k - k % gran;
  }
  r.recompute_tokens = s_local - r.swap_tokens;
  return r;
}

// ---------------------------------------------------------------- params / flops / timing
Params params_of(const ModelConfig& cfg) {
  cfg.validate();
  Params p;
  const std::uint64_t h = cfg.hidden;
  p.embedding = cfg.vocab * h;
  p.per_layer = 4 * h * h + 2 * h * cfg.ffn_hidden + 4 * h;
  p.final_norm = 2 * h;
  p.classifier = cfg.vocab * h;
  return p;
}

double flops_per_sample(const ModelConfig& cfg, std::uint64_t p) {
  const double s = static_cast<double>(cfg.seq_len);
  return 6.0 * s * static_cast<double>(p) +
         6.0 * static_cast<double>(cfg.n_layers) * static_cast<double>(cfg.hidden) * s * s;
}

double mfu_of_tgs(const ModelConfig& cfg, const HardwareConfig& hw, std::uint64_t p, double tgs) {
  const double per_token = flops_per_sample(cfg, p) / static_cast<double>(cfg.seq_len);
  return per_token * tgs / hw.peak_flops;
}

void Timing::validate() const {
  if (t_fwd_layer <= 0) throw ConfigError("t_fwd_layer must be positive");
  if (t_attn_fwd < 0 || t_attn_fwd > t_fwd_layer)
    throw ConfigError("t_attn_fwd must lie in [0, t_fwd_layer]");
  if (t_bwd_layer < 0) throw ConfigError("t_bwd_layer must be nonnegative");
}

Timing timing_of(const ModelConfig& cfg, const HardwareConfig& hw, const Params& p) {
  cfg.validate();
  hw.validate();
  const double denom = static_cast<double>(cfg.model_gpus()) * hw.peak_flops * hw.efficiency;
  const double b = static_cast<double>(cfg.batch);
  const double s = static_cast<double>(cfg.seq_len);
  const double attn = 2.0 * b * static_cast<double>(cfg.hidden) * s * s;
  const double layer = 2.0 * b * s * static_cast<double>(p.per_layer) + attn;
  Timing t;
  t.t_attn_fwd = attn / denom;
  t.t_fwd_layer = layer / denom;
  t.t_bwd_layer = t.bwd_ratio * t.t_fwd_layer;
  t.t_classifier_fwd = 2.0 * b * s * static_cast<double>(p.classifier + p.final_norm) / denom;
  t.t_classifier_bwd = t.bwd_ratio * t.t_classifier_fwd;
  return t;
}

// ---------------------------------------------------------------- executor model
const char* stream_str(Stream s) {
  static const char* names[] = {"compute", "offload", "prefetch"};
  return names[static_cast<int>(s)];
}
const char* kind_str(Kind k) {
  static const char* names[] = {"embedding_fwd", "layer_fwd", "classifier_fwd",
                                "classifier_bwd", "recompute", "layer_bwd",
                                "embedding_bwd", "offload",   "prefetch"};
  return names[static_cast<int>(k)];
}

Timeline schedule_of(const ModelConfig& cfg, const HardwareConfig& hw, const Skeletal& sz,
                     const SwapDecision& swap, const Timing& tm) {
  cfg.validate();
  hw.validate();
  tm.validate();
  const std::uint64_t n = cfg.n_layers;
  Timeline tl;
  tl.n_layers = n;
  tl.rounding_buffer_bytes = sz.total;
  tl.swapped_layers = n >= 2 ? n - 2 : 0;
  auto swapped = [&](std::uint64_t i) {
    return n >= 3 && i + 2 < n && swap.swapped_bytes_per_layer > 0;
  };
  const Seconds xfer = static_cast<double>(swap.swapped_bytes_per_layer) / hw.pcie_bandwidth;
  const Seconds rec = std::max(0.0, tm.t_recompute(swap.alpha));
  auto put = [&](Stream st, Kind k, int layer, Seconds t0, Seconds dur) {
    if (dur > 0) tl.events.push_back({st, k, layer, t0, t0 + dur});
    return t0 + dur;
  };
  std::vector<Seconds> off_done(n, 0), pre_done(n, 0), bwd_done(n, 0);
  Seconds clock = put(Stream::Compute, Kind::EmbFwd, -1, 0, tm.t_embedding_fwd);
  Seconds off_free = 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    Seconds t0 = clock;
    if (i >= 2 && swapped(i - 2)) t0 = std::max(t0, off_done[i - 2]);  // F3
    clock = put(Stream::Compute, Kind::LayerFwd, static_cast<int>(i), t0, tm.t_fwd_layer);
    if (swapped(i)) {  // F2
      off_free = put(Stream::Offload, Kind::Offload, static_cast<int>(i),
                     std::max(clock, off_free), xfer);
      off_done[i] = off_free;
    }
  }
  clock = put(Stream::Compute, Kind::ClsFwd, -1, clock, tm.t_classifier_fwd);
  clock = put(Stream::Compute, Kind::ClsBwd, -1, clock, tm.t_classifier_bwd);
  Seconds pre_free = 0;
  for (std::uint64_t i = n; i-- > 0;) {
    Seconds t0 = clock;
    if (swapped(i)) {  // B3
      clock = put(Stream::Compute, Kind::Recompute, static_cast<int>(i), clock, rec);
      t0 = std::max(clock, pre_done[i]);
    }
    clock = put(Stream::Compute, Kind::LayerBwd, static_cast<int>(i), t0, tm.t_bwd_layer);
    bwd_done[i] = clock;
    if (i >= 2 && swapped(i - 2)) {  // B2
      pre_free = put(Stream::Prefetch, Kind::Prefetch, static_cast<int>(i - 2),
                     std::max(bwd_done[i], pre_free), xfer);
      pre_done[i - 2] = pre_free;
    }
  }
  put(Stream::Compute, Kind::EmbBwd, -1, clock, tm.t_embedding_bwd);
  return tl;
}

SimResult simulate_timeline(const Timeline& t, const ModelConfig& cfg, const HardwareConfig& hw,
                            std::uint64_t p) {
  SimResult r;
  Seconds cursor = 0;
  bool fwd = true;
  for (const Event& e : t.events) {
    r.iteration_time = std::max(r.iteration_time, e.end);
    if (e.stream == Stream::Compute) {
      if (e.kind == Kind::ClsBwd || e.kind == Kind::Recompute || e.kind == Kind::LayerBwd ||
          e.kind == Kind::EmbBwd)
        fwd = false;
      const Seconds gap = e.start - cursor;
      if (gap > 0) {
        r.compute_blocked += gap;
        if (fwd) r.forward_blocked += gap;
      }
      cursor = std::max(cursor, e.end);
    } else if (e.stream == Stream::Offload) {
      r.offload_stream_busy += e.end - e.start;
    } else {
      r.prefetch_stream_busy += e.end - e.start;
    }
  }
  if (r.iteration_time > 0) {
    const double gpus = static_cast<double>(cfg.model_gpus());
    const double tokens = static_cast<double>(cfg.batch) * static_cast<double>(cfg.seq_len);
    r.tgs = tokens / (r.iteration_time * gpus);
    r.mfu = flops_per_sample(cfg, p) * static_cast<double>(cfg.batch) /
            (r.iteration_time * gpus * hw.peak_flops);
  }
  return r;
}

std::vector<std::string> check_timeline(const Timeline& t, const SwapDecision& swap) {
  std::vector<std::string> bad;
  const double eps = 1e-9;
  const std::uint64_t n = t.n_layers;
  auto swapped = [&](std::uint64_t i) {
    return n >= 3 && i + 2 < n && swap.swapped_bytes_per_layer > 0;
  };
  std::map<int, const Event*> fwd, bwd, off, pre, rec;
  std::vector<const Event*> lane[3];
  for (const Event& e : t.events) {
    lane[static_cast<int>(e.stream)].push_back(&e);
    if (e.end < e.start - eps) bad.push_back("event ends before it starts");
    std::map<int, const Event*>* slot = nullptr;
    switch (e.kind) {
      case Kind::LayerFwd: slot = &fwd; break;
      case Kind::LayerBwd: slot = &bwd; break;
      case Kind::Offload: slot = &off; break;
      case Kind::Prefetch: slot = &pre; break;
      case Kind::Recompute: slot = &rec; break;
      default: break;
    }
    if (slot) {
      if (slot->count(e.layer))
        bad.push_back(std::string("duplicate ") + kind_str(e.kind) + " for layer " +
                      std::to_string(e.layer));
      (*slot)[e.layer] = &e;
    }
  }
  for (auto& l : lane)
    for (std::size_t k = 1; k < l.size(); ++k)
      if (l[k]->start < l[k - 1]->end - eps)
        bad.push_back(std::string("overlapping events on stream ") + stream_str(l[k]->stream));
  for (std::uint64_t i = 0; i < n; ++i) {
    if (!fwd.count(static_cast<int>(i))) bad.push_back("missing fwd for layer " + std::to_string(i));
    if (!bwd.count(static_cast<int>(i))) bad.push_back("missing bwd for layer " + std::to_string(i));
  }
  if (!bad.empty()) return bad;
  for (std::uint64_t i = 0; i < n; ++i) {
    const int L = static_cast<int>(i);
    const std::string si = std::to_string(i);
    if (i + 1 < n && fwd.at(L + 1)->start < fwd.at(L)->end - eps)
      bad.push_back("F1: fwd " + std::to_string(i + 1) + " starts before fwd " + si + " ends");
    if (swapped(i)) {
      if (!off.count(L)) {
        bad.push_back("F2: missing offload for swapped layer " + si);
        continue;
      }
      if (!pre.count(L)) {
        bad.push_back("B2: missing prefetch for swapped layer " + si);
        continue;
      }
      if (off.at(L)->start < fwd.at(L)->end - eps)
        bad.push_back("F2: offload " + si + " starts before its fwd ends");
      if (i + 2 < n && fwd.at(L + 2)->start < off.at(L)->end - eps)
        bad.push_back("F3: fwd " + std::to_string(i + 2) + " starts before offload " + si + " ends");
      if (pre.at(L)->start < bwd.at(L + 2)->end - eps)
        bad.push_back("B2: prefetch " + si + " starts before bwd " + std::to_string(i + 2) + " ends");
      if (bwd.at(L)->start < pre.at(L)->end - eps)
        bad.push_back("B3: bwd " + si + " starts before its prefetch ends");
      if (rec.count(L)) {
        const Event* r = rec.at(L);
        if (bwd.at(L)->start < r->end - eps)
          bad.push_back("B3: bwd " + si + " starts before its recompute ends");
        if (r->stream != Stream::Compute)
          bad.push_back("B3: recompute " + si + " not on the compute stream");
        for (const Event* e : lane[0])
          if (e != r && e != bwd.at(L) && e->start >= r->end - eps &&
              e->end <= bwd.at(L)->start + eps)
            bad.push_back("B3: compute event between recompute and bwd " + si);
      }
    } else {
      if (off.count(L)) bad.push_back("layer " + si + " must not offload");
      if (pre.count(L)) bad.push_back("B1: layer " + si + " must not prefetch");
      if (rec.count(L)) bad.push_back("layer " + si + " must not recompute");
    }
    if (i + 1 < n && bwd.at(L)->start < bwd.at(L + 1)->end - eps)
      bad.push_back("B1: bwd " + si + " starts before bwd " + std::to_string(i + 1) + " ends");
  }
  for (std::size_t k = 1; k < lane[1].size(); ++k)
    if (lane[1][k]->layer < lane[1][k - 1]->layer)
      bad.push_back("F2: offload stream not FIFO in layer order");
  for (std::size_t k = 1; k < lane[2].size(); ++k)
    if (lane[2][k]->layer > lane[2][k - 1]->layer)
      bad.push_back("B2: prefetch stream not FIFO in reverse layer order");
  return bad;
}

// ---------------------------------------------------------------- RunConfig JSON
namespace {
using J = nlohmann::json;
void only_keys(const J& j, std::initializer_list<const char*> keys, const std::string& where) {
  if (!j.is_object()) throw ConfigError(where + " must be an object");
  for (auto it = j.begin(); it != j.end(); ++it) {
    bool ok = false;
    for (const char* k : keys) ok = ok || it.key() == k;
    if (!ok) throw ConfigError("unknown key '" + it.key() + "' in " + where);
  }
}
}  // namespace

RunConfig parse_run_config(const std::string& text) {
  J j;
  try {
    j = J::parse(text);
  } catch (const J::exception& e) {
    throw ConfigError(std::string("invalid JSON: ") + e.what());
  }
  try {
    only_keys(j, {"model", "hardware", "synth", "planner", "swap"}, "config");
    RunConfig rc;
    if (j.contains("model")) {
      const J& m = j["model"];
      only_keys(m, {"n_layers", "hidden", "ffn_hidden", "n_heads", "vocab", "batch", "seq_len",
                    "dtype_bytes", "tp_degree", "sp_or_cp_degree", "untied_classifier",
                    "skeletal_weights"},
                "model");
      ModelConfig& c = rc.model;
      c.n_layers = m.value("n_layers", c.n_layers);
      c.hidden = m.value("hidden", c.hidden);
      c.ffn_hidden = m.value("ffn_hidden", c.ffn_hidden);
      c.n_heads = m.value("n_heads", c.n_heads);
      c.vocab = m.value("vocab", c.vocab);
      c.batch = m.value("batch", c.batch);
      c.seq_len = m.value("seq_len", c.seq_len);
      c.dtype_bytes = m.value("dtype_bytes", c.dtype_bytes);
      c.tp_degree = m.value("tp_degree", c.tp_degree);
      c.sp_or_cp_degree = m.value("sp_or_cp_degree", c.sp_or_cp_degree);
      c.untied_classifier = m.value("untied_classifier", c.untied_classifier);
      if (m.contains("skeletal_weights"))
        for (auto it = m["skeletal_weights"].begin(); it != m["skeletal_weights"].end(); ++it)
          c.skeletal_weight_overrides[it.key()] = it.value().get<double>();
      c.validate();
    }
    if (j.contains("hardware")) {
      const J& h = j["hardware"];
      only_keys(h, {"pcie_bandwidth", "cpu_mem", "gpu_mem", "peak_flops", "efficiency"},
                "hardware");
      HardwareConfig& w = rc.hardware;
      w.pcie_bandwidth = h.value("pcie_bandwidth", w.pcie_bandwidth);
      w.cpu_mem = h.value("cpu_mem", w.cpu_mem);
      w.gpu_mem = h.value("gpu_mem", w.gpu_mem);
      w.peak_flops = h.value("peak_flops", w.peak_flops);
      w.efficiency = h.value("efficiency", w.efficiency);
      w.validate();
    }
    if (j.contains("synth")) {
      only_keys(j["synth"], {"seed"}, "synth");
      rc.synth_seed = j["synth"].value("seed", rc.synth_seed);
    }
    if (j.contains("planner")) {
      const J& p = j["planner"];
      only_keys(p, {"cap", "alignment", "time_budget"}, "planner");
      rc.planner.cap = p.value("cap", rc.planner.cap);
      rc.planner.alignment = p.value("alignment", rc.planner.alignment);
      rc.planner.time_budget = p.value("time_budget", rc.planner.time_budget);
    }
    if (j.contains("swap")) {
      const J& s = j["swap"];
      only_keys(s, {"token_granularity", "t_layer"}, "swap");
      rc.swap.token_granularity = s.value("token_granularity", rc.swap.token_granularity);
      rc.swap.t_layer = s.value("t_layer", rc.swap.t_layer);
    }
    return rc;
  } catch (const J::exception& e) {
    throw ConfigError(std::string("bad config value: ") + e.what());
  }
}

}  // namespace memo
