// bilevel.cpp — MEMO's bi-level memory plan.
//
// Level 1 solves one transformer layer's forward and backward transients
// exactly; level 2 condenses every layer segment to a pseudo block of that
// peak and solves the whole iteration; absolute offsets are the level-2 base
// of a segment's pseudo block plus the level-1 offset.  The executor replays
// the result as one preallocated HBM arena.  Contract and determinism:
// proj/include/actmem/bilevel.hpp:66-254; JSON shape: json_io.hpp:183-202.
#include <algorithm>
#include <set>
#include <tuple>

#include <json.hpp>

#include "host/planner.hpp"

namespace memo {

LayerLayout plan_one_layer(const Segment& fwd, const Segment& bwd, Bytes cap, Seconds budget,
                           Bytes alignment) {
  const Segment pair[2] = {fwd, bwd};
  std::vector<Lifespan> in_fwd, in_bwd;
  for (const Lifespan& s : lifespans_of(pair, 2, true)) {
    if (s.skeletal) continue;  // skeletal tensors live in the rounding buffers
    (s.first < fwd.reqs.size() ? in_fwd : in_bwd).push_back(s);
  }
  LayerLayout out;
  auto solve = [&](std::vector<Lifespan> spans, Placement& pl, Bytes& peak, const char* which) {
    Solution sol = solve_optimal(make_problem(std::move(spans), cap, alignment), budget);
    if (sol.status == SolveStatus::Infeasible)
      throw InfeasibleError(std::string("layer ") + which + " transients do not fit in cap " +
                            std::to_string(cap));
    if (sol.status != SolveStatus::Optimal) out.optimal = false;
    pl = std::move(sol.placement);
    peak = pl.peak;
  };
  solve(std::move(in_fwd), out.fwd, out.fwd_peak, "fwd");
  solve(std::move(in_bwd), out.bwd, out.bwd_peak, "bwd");
  return out;
}

namespace {

struct Condensed {
  std::vector<Request> events;
  std::map<std::size_t, TensorId> pseudo_of_segment;
};

Condensed condense(const Trace& t, const LayerLayout& lay) {
  const Segment* f0 = nullptr;
  const Segment* b0 = nullptr;
  std::vector<Request> cf, cb;
  for (const Segment& s : t.segs) {
    if (s.phase == Phase::LayerFwd) {
      if (!f0) {
        f0 = &s;
        cf = canonical_form(s);
      } else if (canonical_form(s) != cf) {
        throw PlanningError("layer forward segments are not identical modulo ids");
      }
    } else if (s.phase == Phase::LayerBwd) {
      if (!b0) {
        b0 = &s;
        cb = canonical_form(s);
      } else if (canonical_form(s) != cb) {
        throw PlanningError("layer backward segments are not identical modulo ids");
      }
    }
  }
  const std::vector<Lifespan> spans = lifespans_of(t.segs.data(), t.segs.size(), false);
  // Segment owning each event index.
  std::vector<std::uint32_t> owner;
  owner.reserve(t.events());
  for (std::size_t si = 0; si < t.segs.size(); ++si)
    owner.insert(owner.end(), t.segs[si].reqs.size(), static_cast<std::uint32_t>(si));
  std::set<TensorId> layer_skeletal;
  TensorId next_id = 1;
  for (const Lifespan& s : spans) {
    if (s.skeletal && t.segs[owner[s.first]].phase == Phase::LayerFwd) layer_skeletal.insert(s.id);
    next_id = std::max(next_id, s.id + 1);
  }
  Condensed c;
  for (std::size_t si = 0; si < t.segs.size(); ++si) {
    const Segment& s = t.segs[si];
    if (phase_is_layer(s.phase)) {
      const Bytes peak = s.phase == Phase::LayerFwd ? lay.fwd_peak : lay.bwd_peak;
      if (peak == 0) continue;
      const TensorId id = next_id++;
      c.pseudo_of_segment[si] = id;
      c.events.push_back({true, id, peak});
      c.events.push_back({false, id, peak});
    } else {
      for (const Request& r : s.reqs)
        if (!layer_skeletal.count(r.id)) c.events.push_back(r);
    }
  }
  return c;
}

}  // namespace

ModelPlan plan_iteration(const Trace& t, Bytes cap, Seconds budget, Bytes alignment) {
  check_iteration_layout(t);
  const std::size_t n = static_cast<std::size_t>(t.n_layers);
  const Segment& fwd0 = t.segs[1];
  const Segment& bwd0 = t.segs[2 * n + 2];

  ModelPlan mp;
  mp.layer = plan_one_layer(fwd0, bwd0, cap, budget, alignment);
  mp.optimal = mp.layer.optimal;

  Condensed c = condense(t, mp.layer);
  Segment flat;
  flat.phase = Phase::LayerFwd;
  flat.layer = 0;
  flat.reqs = std::move(c.events);
  Solution outer =
      solve_optimal(make_problem(lifespans_of(&flat, 1, true), cap, alignment), budget);
  if (outer.status == SolveStatus::Infeasible)
    throw InfeasibleError("outer request sequence does not fit in cap " + std::to_string(cap));
  if (outer.status != SolveStatus::Optimal) mp.optimal = false;
  mp.outer = std::move(outer.placement);
  mp.pseudo_of_segment = std::move(c.pseudo_of_segment);
  mp.total_peak = mp.outer.peak;

  auto place_layer = [&](const Segment& s, std::size_t si, const Segment& canon,
                         const Placement& local) {
    auto ps = mp.pseudo_of_segment.find(si);
    if (ps == mp.pseudo_of_segment.end()) return;
    const Bytes base = mp.outer.offset.at(ps->second);
    for (std::size_t k = 0; k < s.reqs.size(); ++k) {
      if (!s.reqs[k].malloc) continue;
      auto a = local.offset.find(canon.reqs[k].id);
      if (a == local.offset.end()) continue;
      mp.absolute.push_back({si, s.reqs[k].id, base + a->second});
    }
  };
  for (std::size_t si = 0; si < t.segs.size(); ++si) {
    const Segment& s = t.segs[si];
    if (s.phase == Phase::LayerFwd) {
      place_layer(s, si, fwd0, mp.layer.fwd);
    } else if (s.phase == Phase::LayerBwd) {
      place_layer(s, si, bwd0, mp.layer.bwd);
    } else {
      for (const Request& r : s.reqs) {
        if (!r.malloc) continue;
        auto a = mp.outer.offset.find(r.id);
        if (a != mp.outer.offset.end()) mp.absolute.push_back({si, r.id, a->second});
      }
    }
  }
  std::sort(mp.absolute.begin(), mp.absolute.end(), [](const AbsAddr& a, const AbsAddr& b) {
    return std::tie(a.segment, a.id) < std::tie(b.segment, b.id);
  });
  return mp;
}

namespace {
nlohmann::json placement_json(const Placement& p) {
  nlohmann::json addrs = nlohmann::json::object();
  for (const auto& [id, off] : p.offset) addrs[std::to_string(id)] = off;
  return nlohmann::json{{"peak", p.peak}, {"addresses", addrs}};
}
}  // namespace

std::string plan_to_json(const ModelPlan& p) {
  nlohmann::json abs = nlohmann::json::array();
  for (const AbsAddr& a : p.absolute)
    abs.push_back(nlohmann::json{{"segment", a.segment}, {"tensor", a.id}, {"offset", a.offset}});
  nlohmann::json j{{"layer", nlohmann::json{{"fwd", placement_json(p.layer.fwd)},
                                            {"bwd", placement_json(p.layer.bwd)},
                                            {"fwd_peak", p.layer.fwd_peak},
                                            {"bwd_peak", p.layer.bwd_peak}}},
                   {"outer", placement_json(p.outer)},
                   {"total_peak", p.total_peak},
                   {"optimal", p.optimal},
                   {"absolute", abs}};
  return j.dump();
}

std::string parse_plan_json(const std::string& text, Bytes* total_peak,
                            std::map<std::pair<std::size_t, TensorId>, Bytes>* absolute) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw ConfigError(std::string("plan: invalid JSON: ") + e.what());
  }
  if (!j.is_object() || !j.contains("absolute") || !j.contains("total_peak") || !j["absolute"].is_array())
    throw ConfigError("plan: not a GlobalPlan (needs 'absolute' and 'total_peak')");
  try {
    *total_peak = j["total_peak"].get<Bytes>();
    absolute->clear();
    for (const auto& a : j["absolute"]) {
      const auto key = std::make_pair(a.at("segment").get<std::size_t>(), a.at("tensor").get<TensorId>());
      if (!absolute->emplace(key, a.at("offset").get<Bytes>()).second)
        throw ConfigError("plan: tensor " + std::to_string(key.second) + " placed twice");
    }
  } catch (const nlohmann::json::exception& e) {
    throw ConfigError(std::string("plan: bad value: ") + e.what());
  }
  return j.dump();
}

}  // namespace memo
