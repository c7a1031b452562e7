// dsa.cpp — offline dynamic storage allocation (the level-1/level-2 solver of
// MEMO's bi-level planner).
//
// Semantics follow proj/include/actmem/dsa.hpp so that offsets are
// bit-identical to the reference:
//   * best-fit replay (dsa.hpp:151-218): frees before mallocs at equal event
//     index, smallest sufficient hole with ties to the lowest address, the
//     wilderness (top) is returned when a freed block touches it;
//   * exact branch-and-bound per overlap component (dsa.hpp:227-361):
//     candidates ordered by (first-fit address, tensor id), bound fixed per
//     node, interchangeable tensors expanded once, strict improvement only,
//     deadline polled every 4096 nodes.
// Independent implementation: components come from one interval sweep (the
// overlap graph of intervals is connected exactly along sorted-start runs),
// the free list is a sorted vector, and the search reuses per-depth buffers.
#include <algorithm>
#include <chrono>
#include <limits>
#include <unordered_set>

#include "host/planner.hpp"

namespace memo {

DsaProblem make_problem(std::vector<Lifespan> spans, Bytes cap, Bytes alignment) {
  if (alignment == 0 || (alignment & (alignment - 1)) != 0)
    throw ConfigError("alignment must be a power of two");
  std::sort(spans.begin(), spans.end(),
            [](const Lifespan& a, const Lifespan& b) { return a.first < b.first; });
  std::unordered_set<TensorId> ids;
  for (Lifespan& s : spans) {
    if (s.first >= s.last)
      throw ConfigError("tensor " + std::to_string(s.id) + " has empty lifespan");
    if (!ids.insert(s.id).second) throw ConfigError("duplicate tensor id " + std::to_string(s.id));
    s.size = round_up(s.size, alignment);
  }
  DsaProblem p;
  p.items = std::move(spans);
  p.cap = cap;
  p.alignment = alignment;
  return p;
}

namespace {

// Max over malloc events of the bytes live right after that malloc.
Bytes sweep_lower_bound(const std::vector<Lifespan>& items, const std::size_t* idx,
                        std::size_t n) {
  struct Ev {
    std::size_t at;
    bool add;
    Bytes size;
  };
  std::vector<Ev> ev;
  ev.reserve(2 * n);
  for (std::size_t i = 0; i < n; ++i) {
    const Lifespan& s = items[idx ? idx[i] : i];
    ev.push_back({s.first, true, s.size});
    ev.push_back({s.last, false, s.size});
  }
  std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.at != b.at) return a.at < b.at;
    return a.add < b.add;
  });
  Bytes live = 0, best = 0;
  for (const Ev& e : ev) {
    if (e.add) {
      live += e.size;
      best = std::max(best, live);
    } else {
      live -= e.size;
    }
  }
  return best;
}

}  // namespace

Bytes live_lower_bound(const DsaProblem& p) {
  return sweep_lower_bound(p.items, nullptr, p.items.size());
}

std::optional<std::string> check_placement(const Placement& pl, const DsaProblem& p) {
  for (const Lifespan& s : p.items) {
    auto it = pl.offset.find(s.id);
    if (it == pl.offset.end()) return "tensor " + std::to_string(s.id) + " has no address";
    if (it->second % p.alignment)
      return "tensor " + std::to_string(s.id) + " address not aligned to " +
             std::to_string(p.alignment);
    if (it->second + s.size > pl.peak)
      return "tensor " + std::to_string(s.id) + " extends past peak " + std::to_string(pl.peak);
  }
  if (p.cap && pl.peak > p.cap)
    return "peak " + std::to_string(pl.peak) + " exceeds mem_cap " + std::to_string(p.cap);
  for (std::size_t i = 0; i < p.items.size(); ++i)
    for (std::size_t j = i + 1; j < p.items.size(); ++j) {
      const Lifespan &a = p.items[i], &b = p.items[j];
      if (!a.overlaps(b)) continue;
      const Bytes xa = pl.offset.at(a.id), xb = pl.offset.at(b.id);
      if (xa < xb + b.size && xb < xa + a.size)
        return "tensors " + std::to_string(std::min(a.id, b.id)) + " and " +
               std::to_string(std::max(a.id, b.id)) +
               " are live together and overlap in address space";
    }
  return std::nullopt;
}

Solution best_fit(const DsaProblem& p) {
  const std::size_t n = p.items.size();
  struct Ev {
    std::size_t at;
    bool alloc;
    std::uint32_t item;
  };
  std::vector<Ev> ev;
  ev.reserve(2 * n);
  for (std::size_t i = 0; i < n; ++i) {
    ev.push_back({p.items[i].first, true, static_cast<std::uint32_t>(i)});
    ev.push_back({p.items[i].last, false, static_cast<std::uint32_t>(i)});
  }
  std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.at != b.at) return a.at < b.at;
    return a.alloc < b.alloc;  // frees first
  });
  std::vector<std::pair<Bytes, Bytes>> holes;  // (addr, len), sorted by addr
  std::vector<Bytes> addr(n, 0);
  Bytes top = 0, peak = 0;
  for (const Ev& e : ev) {
    const Bytes size = p.items[e.item].size;
    if (e.alloc) {
      std::size_t pick = holes.size();
      for (std::size_t h = 0; h < holes.size(); ++h)
        if (holes[h].second >= size && (pick == holes.size() || holes[h].second < holes[pick].second))
          pick = h;
      if (pick != holes.size()) {
        addr[e.item] = holes[pick].first;
        if (holes[pick].second > size) {
          holes[pick].first += size;
          holes[pick].second -= size;
        } else {
          holes.erase(holes.begin() + static_cast<std::ptrdiff_t>(pick));
        }
      } else {
        addr[e.item] = top;
        top += size;
        peak = std::max(peak, top);
      }
    } else {
      Bytes a = addr[e.item], len = size;
      auto nxt = std::lower_bound(holes.begin(), holes.end(), std::make_pair(a, Bytes(0)));
      if (nxt != holes.end() && a + len == nxt->first) {
        len += nxt->second;
        nxt = holes.erase(nxt);
      }
      if (nxt != holes.begin()) {
        auto prv = nxt - 1;
        if (prv->first + prv->second == a) {
          a = prv->first;
          len += prv->second;
          nxt = holes.erase(prv);
        }
      }
      if (a + len == top)
        top = a;
      else
        holes.insert(nxt, {a, len});
    }
  }
  Solution s;
  for (std::size_t i = 0; i < n; ++i) s.placement.offset[p.items[i].id] = addr[i];
  s.placement.peak = peak;
  s.status = peak <= p.limit() ? SolveStatus::Feasible : SolveStatus::Infeasible;
  return s;
}

namespace {

class BranchAndBound {
 public:
  BranchAndBound(const DsaProblem& p, const std::size_t* members, std::size_t n,
                 std::chrono::steady_clock::time_point deadline)
      : p_(p), m_(members, members + n), n_(n), deadline_(deadline) {
    adj_.assign(n * n, 0);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i + 1; j < n; ++j)
        if (item(i).overlaps(item(j))) adj_[i * n + j] = adj_[j * n + i] = 1;
    addr_.assign(n, 0);
    placed_.assign(n, 0);
    cands_.resize(n + 1);
    lb_ = sweep_lower_bound(p.items, m_.data(), n);
  }

  void seed(std::vector<Bytes> addr, Bytes peak) {
    best_addr_ = std::move(addr);
    best_ = peak;
    have_best_ = true;
  }

  // Returns false on timeout (incumbent kept).
  bool run() {
    if (have_best_ && best_ <= lb_) return true;
    descend(0, 0);
    return !timed_out_;
  }
  Bytes best() const { return best_; }
  const std::vector<Bytes>& best_addr() const { return best_addr_; }

 private:
  struct Cand {
    std::uint32_t i;
    Bytes addr;
    Bytes top;
  };
  const Lifespan& item(std::size_t k) const { return p_.items[m_[k]]; }

  Bytes lowest_fit(std::size_t c) {
    const Bytes size = item(c).size;
    blocks_.clear();
    for (std::size_t j = 0; j < n_; ++j)
      if (placed_[j] && adj_[c * n_ + j]) blocks_.emplace_back(addr_[j], addr_[j] + item(j).size);
    std::sort(blocks_.begin(), blocks_.end());
    Bytes cur = 0;
    for (const auto& [a, e] : blocks_) {
      if (a > cur && a - cur >= size) return cur;
      cur = std::max(cur, e);
    }
    return cur;
  }

  void descend(std::size_t depth, Bytes peak) {
    if (timed_out_) return;
    if (++nodes_ % 4096 == 0 && std::chrono::steady_clock::now() > deadline_) {
      timed_out_ = true;
      return;
    }
    if (have_best_ && best_ <= lb_) return;
    if (depth == n_) {
      if (!have_best_ || peak < best_) {
        best_ = peak;
        best_addr_ = addr_;
        have_best_ = true;
      }
      return;
    }
    std::vector<Cand>& cs = cands_[depth];
    cs.clear();
    for (std::size_t i = 0; i < n_; ++i) {
      if (placed_[i]) continue;
      const Bytes a = lowest_fit(i);
      cs.push_back({static_cast<std::uint32_t>(i), a, std::max(peak, a + item(i).size)});
    }
    std::sort(cs.begin(), cs.end(), [&](const Cand& x, const Cand& y) {
      if (x.addr != y.addr) return x.addr < y.addr;
      return item(x.i).id < item(y.i).id;
    });
    Bytes bound = p_.limit();
    if (bound != std::numeric_limits<Bytes>::max()) bound += 1;  // peak == cap allowed
    if (have_best_) bound = std::min(bound, best_);
    for (std::size_t c = 0; c < cs.size(); ++c) {
      const Cand cand = cs[c];
      if (cand.addr >= bound) break;
      if (cand.top >= bound) continue;
      const Lifespan& me = item(cand.i);
      bool twin = false;
      for (std::size_t q = 0; q < c && !twin; ++q) {
        const Lifespan& o = item(cs[q].i);
        twin = o.size == me.size && o.first == me.first && o.last == me.last;
      }
      if (twin) continue;
      placed_[cand.i] = 1;
      addr_[cand.i] = cand.addr;
      descend(depth + 1, cand.top);
      placed_[cand.i] = 0;
      if (timed_out_) return;
      if (have_best_ && best_ <= lb_) return;
    }
  }

  const DsaProblem& p_;
  std::vector<std::size_t> m_;
  std::size_t n_;
  std::vector<std::uint8_t> adj_, placed_;
  std::vector<Bytes> addr_, best_addr_;
  std::vector<std::vector<Cand>> cands_;
  std::vector<std::pair<Bytes, Bytes>> blocks_;
  Bytes best_ = 0, lb_ = 0;
  bool have_best_ = false, timed_out_ = false;
  std::size_t nodes_ = 0;
  std::chrono::steady_clock::time_point deadline_;
};

}  // namespace

Solution solve_optimal(const DsaProblem& p, Seconds budget) {
  Solution out;
  if (live_lower_bound(p) > p.limit()) {
    out.status = SolveStatus::Infeasible;
    return out;
  }
  const Solution seed = best_fit(p);
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                            std::chrono::duration<double>(budget));
  bool timed_out = false;
  // Items are sorted by start: overlap components are maximal runs whose
  // next start lies before the running maximum end.
  const std::size_t n = p.items.size();
  std::vector<std::size_t> members;
  std::size_t i = 0;
  while (i < n) {
    members.clear();
    std::size_t reach = p.items[i].last;
    members.push_back(i);
    std::size_t j = i + 1;
    while (j < n && p.items[j].first < reach) {
      reach = std::max(reach, p.items[j].last);
      members.push_back(j);
      ++j;
    }
    BranchAndBound bb(p, members.data(), members.size(), deadline);
    std::vector<Bytes> sa(members.size());
    Bytes speak = 0;
    for (std::size_t k = 0; k < members.size(); ++k) {
      const Lifespan& s = p.items[members[k]];
      sa[k] = seed.placement.offset.at(s.id);
      speak = std::max(speak, sa[k] + s.size);
    }
    bb.seed(std::move(sa), speak);
    if (!bb.run()) timed_out = true;
    for (std::size_t k = 0; k < members.size(); ++k)
      out.placement.offset[p.items[members[k]].id] = bb.best_addr()[k];
    out.placement.peak = std::max(out.placement.peak, bb.best());
    i = j;
  }
  if (out.placement.peak > p.limit()) {
    out.status = timed_out ? SolveStatus::TimedOut : SolveStatus::Infeasible;
    return out;
  }
  out.status = timed_out ? SolveStatus::TimedOut : SolveStatus::Optimal;
  return out;
}

}  // namespace memo
