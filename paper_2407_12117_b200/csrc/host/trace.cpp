// trace.cpp — config validation and the memory-request trace model.
//
// Text format and invariants follow proj/include/actmem/trace.hpp:262-371;
// lifespan classification follows trace.hpp:146-224 (a tensor freed in the
// segment that allocated it is Transient, one freed in the matching backward
// segment of the same layer is Skeletal, anything else is an error).
#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <string_view>
#include <unordered_map>
#include <unordered_set>

#include "host/planner.hpp"

namespace memo {

// ---------------------------------------------------------------- configs
void ModelConfig::validate() const {  // types.hpp:104-122
  const std::pair<std::uint64_t, const char*> fields[] = {
      {n_layers, "n_layers"},       {hidden, "hidden"},   {ffn_hidden, "ffn_hidden"},
      {n_heads, "n_heads"},         {vocab, "vocab"},     {batch, "batch"},
      {seq_len, "seq_len"},         {dtype_bytes, "dtype_bytes"},
      {tp_degree, "tp_degree"},     {sp_or_cp_degree, "sp_or_cp_degree"}};
  for (const auto& [v, name] : fields)
    if (v == 0) throw ConfigError(std::string(name) + " must be >= 1");
  if (seq_len % sp_or_cp_degree) throw ConfigError("seq_len must be divisible by sp_or_cp_degree");
  if (hidden % tp_degree) throw ConfigError("hidden must be divisible by tp_degree");
}

void HardwareConfig::validate() const {  // types.hpp:133-140
  if (!(pcie_bandwidth > 0)) throw ConfigError("pcie_bandwidth must be positive");
  if (cpu_mem == 0) throw ConfigError("cpu_mem must be positive");
  if (gpu_mem == 0) throw ConfigError("gpu_mem must be positive");
  if (!(peak_flops > 0)) throw ConfigError("peak_flops must be positive");
  if (efficiency <= 0 || efficiency > 1.0) throw ConfigError("efficiency must be in (0, 1]");
}

// ---------------------------------------------------------------- phases
namespace {
constexpr const char* kPhaseNames[] = {"embedding_fwd", "layer_fwd", "classifier_fwd",
                                       "classifier_bwd", "layer_bwd", "embedding_bwd"};

bool phase_from(std::string_view s, Phase& out) {
  for (int i = 0; i < 6; ++i)
    if (s == kPhaseNames[i]) {
      out = static_cast<Phase>(i);
      return true;
    }
  return false;
}

Phase backward_of(Phase p) {
  switch (p) {
    case Phase::EmbFwd: return Phase::EmbBwd;
    case Phase::LayerFwd: return Phase::LayerBwd;
    case Phase::ClsFwd: return Phase::ClsBwd;
    default: throw ConfigError("matching_backward called on a backward phase");
  }
}
}  // namespace

const char* phase_str(Phase p) { return kPhaseNames[static_cast<int>(p)]; }
bool phase_is_fwd(Phase p) {
  return p == Phase::EmbFwd || p == Phase::LayerFwd || p == Phase::ClsFwd;
}
bool phase_is_layer(Phase p) { return p == Phase::LayerFwd || p == Phase::LayerBwd; }

std::size_t Trace::events() const {
  std::size_t n = 0;
  for (const auto& s : segs) n += s.reqs.size();
  return n;
}

// ---------------------------------------------------------------- text format
namespace {

struct Tokens {
  std::vector<std::string_view> t;
  explicit Tokens(std::string_view line) {
    std::size_t i = 0;
    while (i < line.size()) {
      while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
      std::size_t j = i;
      while (j < line.size() && !std::isspace(static_cast<unsigned char>(line[j]))) ++j;
      if (j > i) t.push_back(line.substr(i, j - i));
      i = j;
    }
  }
};

bool to_u64(std::string_view s, std::uint64_t& v) {
  if (s.empty()) return false;
  std::uint64_t x = 0;
  for (char c : s) {
    if (c < '0' || c > '9') return false;
    x = x * 10 + static_cast<std::uint64_t>(c - '0');
  }
  v = x;
  return true;
}

bool to_long(std::string_view s, long& v) {
  bool neg = false;
  if (!s.empty() && (s[0] == '-' || s[0] == '+')) {
    neg = s[0] == '-';
    s.remove_prefix(1);
  }
  std::uint64_t u;
  if (!to_u64(s, u)) return false;
  v = neg ? -static_cast<long>(u) : static_cast<long>(u);
  return true;
}

}  // namespace

Trace parse_trace_text(const std::string& text) {
  Trace tr;
  std::unordered_map<TensorId, Bytes> live;
  std::unordered_set<TensorId> seen;
  int max_layer = -1;
  std::size_t line_no = 0, pos = 0;
  const std::string_view all(text);
  while (pos <= all.size()) {
    const std::size_t eol = all.find('\n', pos);
    std::string_view line =
        all.substr(pos, eol == std::string_view::npos ? all.size() - pos : eol - pos);
    pos = eol == std::string_view::npos ? all.size() + 1 : eol + 1;
    ++line_no;
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.remove_suffix(1);
    if (line.empty()) continue;
    Tokens tk(line);
    if (tk.t.empty()) continue;
    const std::string_view head = tk.t[0];
    if (head == "#") {
      if (tk.t.size() < 2 || tk.t[1] != "segment") continue;  // comment
      const std::string_view ph = tk.t.size() > 2 ? tk.t[2] : std::string_view();
      Segment seg;
      if (!phase_from(ph, seg.phase))
        throw TraceParseError(line_no, "unknown phase '" + std::string(ph) + "'");
      long layer;
      if (tk.t.size() > 3 && to_long(tk.t[3], layer)) {
        if (layer < 0) throw TraceParseError(line_no, "negative layer index");
        seg.layer = static_cast<int>(layer);
        max_layer = std::max(max_layer, seg.layer);
      } else if (phase_is_layer(seg.phase)) {
        throw TraceParseError(line_no, "layer phase requires a layer index");
      }
      tr.segs.push_back(std::move(seg));
      continue;
    }
    const bool is_malloc = head == "malloc";
    if (!is_malloc && head != "free")
      throw TraceParseError(line_no, "expected 'malloc', 'free' or '# segment', got '" +
                                         std::string(line) + "'");
    if (tr.segs.empty()) throw TraceParseError(line_no, "event before any '# segment' header");
    TensorId id;
    Bytes size;
    if (tk.t.size() < 3 || !to_u64(tk.t[1], id) || !to_u64(tk.t[2], size))
      throw TraceParseError(line_no, "expected '<id> <bytes>' after '" + std::string(head) + "'");
    if (tk.t.size() > 3)
      throw TraceParseError(line_no, "trailing token '" + std::string(tk.t[3]) + "'");
    if (is_malloc) {
      if (size == 0) throw TraceParseError(line_no, "malloc of zero bytes");
      if (!seen.insert(id).second)
        throw TraceParseError(line_no, "tensor id " + std::to_string(id) + " reused");
      live.emplace(id, size);
    } else {
      auto it = live.find(id);
      if (it == live.end())
        throw TraceParseError(line_no, "free of tensor id " + std::to_string(id) +
                                           " without a prior malloc");
      if (it->second != size)
        throw TraceParseError(line_no, "free size " + std::to_string(size) +
                                           " does not match malloc size " +
                                           std::to_string(it->second));
      live.erase(it);
    }
    tr.segs.back().reqs.push_back({is_malloc, id, size});
  }
  if (!live.empty()) {
    TensorId lo = ~TensorId(0);
    for (const auto& kv : live) lo = std::min(lo, kv.first);
    throw TraceParseError(0, "tensor id " + std::to_string(lo) + " is never freed");
  }
  tr.n_layers = max_layer + 1;
  return tr;
}

std::string trace_to_text(const Trace& t) {
  std::string out;
  out.reserve(t.events() * 24 + t.segs.size() * 32);
  for (const auto& s : t.segs) {
    out += "# segment ";
    out += phase_str(s.phase);
    if (s.layer >= 0) {
      out += ' ';
      out += std::to_string(s.layer);
    }
    out += '\n';
    for (const auto& r : s.reqs) {
      out += r.malloc ? "malloc " : "free ";
      out += std::to_string(r.id);
      out += ' ';
      out += std::to_string(r.size);
      out += '\n';
    }
  }
  return out;
}

// ---------------------------------------------------------------- lifespans
std::vector<Lifespan> lifespans_of(const Segment* segs, std::size_t n, bool allow_open) {
  struct Open {
    Bytes size;
    std::size_t event;
    std::size_t seg;
  };
  std::unordered_map<TensorId, Open> open;
  std::unordered_set<TensorId> closed;
  std::vector<Lifespan> out;
  std::size_t ev = 0;
  for (std::size_t si = 0; si < n; ++si) {
    for (const Request& r : segs[si].reqs) {
      if (r.malloc) {
        if (open.count(r.id) || closed.count(r.id))
          throw TraceParseError(0, "tensor id " + std::to_string(r.id) +
                                       " allocated more than once");
        if (r.size == 0)
          throw TraceParseError(0, "tensor id " + std::to_string(r.id) + " has zero size");
        open.emplace(r.id, Open{r.size, ev, si});
      } else {
        auto it = open.find(r.id);
        if (it == open.end())
          throw TraceParseError(0, "free of tensor id " + std::to_string(r.id) +
                                       " without a prior malloc");
        if (it->second.size != r.size)
          throw TraceParseError(0, "free size " + std::to_string(r.size) +
                                       " does not match malloc size " +
                                       std::to_string(it->second.size) + " for tensor id " +
                                       std::to_string(r.id));
        const Segment& sa = segs[it->second.seg];
        const Segment& sf = segs[si];
        bool skeletal;
        if (it->second.seg == si) {
          skeletal = false;
        } else if (phase_is_fwd(sa.phase) && sf.phase == backward_of(sa.phase) &&
                   (!phase_is_layer(sa.phase) || sa.layer == sf.layer)) {
          skeletal = true;
        } else {
          throw TraceParseError(0, "tensor id " + std::to_string(r.id) +
                                       " crosses segments without a matching fwd/bwd pair");
        }
        out.push_back({r.id, r.size, it->second.event, ev, skeletal});
        closed.insert(r.id);
        open.erase(it);
      }
      ++ev;
    }
  }
  if (!open.empty()) {
    std::vector<TensorId> ids;
    for (const auto& kv : open) ids.push_back(kv.first);
    std::sort(ids.begin(), ids.end());
    if (!allow_open) throw TraceParseError(0, "tensor id " + std::to_string(ids[0]) + " is never freed");
    for (TensorId id : ids) {
      const Open& o = open.at(id);
      out.push_back({id, o.size, o.event, ev, true});
    }
  }
  // Malloc indices are unique, so this order is total.
  std::sort(out.begin(), out.end(),
            [](const Lifespan& a, const Lifespan& b) { return a.first < b.first; });
  return out;
}

void check_iteration_layout(const Trace& t) {
  const int n = t.n_layers;
  if (n < 1) throw PlanningError("trace has no layer segments");
  const std::size_t want = 2 * static_cast<std::size_t>(n) + 4;
  if (t.segs.size() != want)
    throw PlanningError("expected " + std::to_string(want) + " segments, got " +
                        std::to_string(t.segs.size()));
  std::vector<std::pair<Phase, int>> order;
  order.emplace_back(Phase::EmbFwd, -1);
  for (int l = 0; l < n; ++l) order.emplace_back(Phase::LayerFwd, l);
  order.emplace_back(Phase::ClsFwd, -1);
  order.emplace_back(Phase::ClsBwd, -1);
  for (int l = n - 1; l >= 0; --l) order.emplace_back(Phase::LayerBwd, l);
  order.emplace_back(Phase::EmbBwd, -1);
  for (std::size_t i = 0; i < want; ++i) {
    const Segment& s = t.segs[i];
    if (s.phase != order[i].first || s.layer != order[i].second)
      throw PlanningError("segment " + std::to_string(i) + " is " + phase_str(s.phase) + "/" +
                          std::to_string(s.layer) + ", expected " + phase_str(order[i].first) +
                          "/" + std::to_string(order[i].second));
  }
}

std::vector<Request> canonical_form(const Segment& s) {
  std::unordered_map<TensorId, TensorId> rename;
  std::vector<Request> out;
  out.reserve(s.reqs.size());
  for (const Request& r : s.reqs) {
    auto [it, fresh] = rename.emplace(r.id, static_cast<TensorId>(rename.size()));
    (void)fresh;
    out.push_back({r.malloc, it->second, r.size});
  }
  return out;
}

std::string fnv1a(const std::string& data) {
  // The reference's offset basis is 1469598103934665603 (json_io.hpp:266) —
  // the textbook FNV basis with its last digit dropped.  Kept as-is so run
  // manifests hash identically.
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : data) {
    h ^= c;
    h *= 1099511628211ull;
  }
  static const char* hex = "0123456789abcdef";
  std::string s = "0x0000000000000000";
  for (int i = 0; i < 16; ++i) s[17 - i] = hex[(h >> (4 * i)) & 15];
  return s;
}

}  // namespace memo
