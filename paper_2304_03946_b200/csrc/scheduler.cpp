// Host-side placement scheduler (see scheduler.h for the reference map).
#include "scheduler.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>

#include "routing.cuh"

namespace fm {
namespace sched {

// ----------------------------------------------------------------- profile
ClusterProfile ClusterProfile::reference_default(int num_gpus, int slots_per_gpu) {
  if (num_gpus < 1) throw std::invalid_argument("default_profile: num_gpus must be >= 1");
  ClusterProfile p;
  p.num_gpus = num_gpus;
  p.gpus_per_node = (num_gpus % 8 == 0) ? 8 : num_gpus;
  p.slots_per_gpu = slots_per_gpu;
  // ring all-reduce moves 2(n-1)/n bytes per byte: link * n / (2(n-1))
  auto ring = [](double link, int n) { return link * n / (2.0 * (n - 1)); };
  const int max_intra = std::min(p.gpus_per_node, num_gpus);
  p.bps_intra.assign(max_intra + 1, 0.0);
  for (int n = 2; n <= max_intra; ++n) p.bps_intra[n] = ring(p.intra_bw, n);
  if (num_gpus > p.gpus_per_node) {
    p.bps_inter.assign(num_gpus + 1, 0.0);
    for (int n = 2; n <= num_gpus; ++n) p.bps_inter[n] = ring(p.inter_bw, n);
  }
  return p;
}

double ClusterProfile::bandwidth(int a, int b) const {
  if (a < 0 || a >= num_gpus || b < 0 || b >= num_gpus)
    throw std::out_of_range("bandwidth: GPU id out of range");
  if (a == b) return std::numeric_limits<double>::infinity();
  return (a / gpus_per_node) == (b / gpus_per_node) ? intra_bw : inter_bw;
}

bool ClusterProfile::spans_nodes(const std::vector<int>& group) const {
  for (int g : group)
    if (g / gpus_per_node != group.front() / gpus_per_node) return true;
  return false;
}

double ClusterProfile::group_bps(const std::vector<int>& group) const {
  if (group.size() < 2) throw std::invalid_argument("group_bps: group must contain at least 2 GPUs");
  const auto& table = spans_nodes(group) ? bps_inter : bps_intra;
  if (group.size() >= table.size())
    throw std::invalid_argument("group_bps: no table entry for group size " +
                                std::to_string(group.size()));
  return table[group.size()];
}

// ----------------------------------------------------------------- placement
SlotPlacement::SlotPlacement(int num_gpus, int slots_per_gpu, int num_experts)
    : G_(num_gpus), E_(slots_per_gpu), N_(num_experts) {
  if (G_ < 1 || E_ < 1 || N_ < 1) throw std::invalid_argument("Placement: dimensions must be positive");
  slot_.assign(static_cast<size_t>(G_) * E_, -1);
  count_.assign(static_cast<size_t>(N_) * G_, 0);
  total_.assign(N_, 0);
}

SlotPlacement SlotPlacement::round_robin(int N, int G, int E) {
  if (N > G * E)
    throw std::invalid_argument("initial placement: insufficient vExpert budget (" +
                                std::to_string(N) + " experts, " + std::to_string(G * E) + " slots)");
  SlotPlacement p(G, E, N);
  for (int e = 0; e < N; ++e) {
    const int g = e % G;
    p.slot_[g * E + p.first_free(g)] = e;
    p.count_[e * G + g] += 1;
    p.total_[e] += 1;
    p.assigned_ += 1;
  }
  return p;
}

SlotPlacement SlotPlacement::from_counts(const std::vector<int>& counts, int N, int G, int E) {
  if (counts.size() != static_cast<size_t>(N) * G) throw std::invalid_argument("from_counts: bad counts shape");
  SlotPlacement p(G, E, N);
  for (int g = 0; g < G; ++g) {
    int used = 0;
    for (int e = 0; e < N; ++e) {
      const int n = counts[e * G + g];
      if (n < 0) throw std::invalid_argument("from_counts: negative replica count");
      if (used + n > E)
        throw std::invalid_argument("from_counts: GPU " + std::to_string(g) + " over its slot budget");
      for (int k = 0; k < n; ++k) p.slot_[g * E + used++] = e;
      p.count_[e * G + g] = n;
      p.total_[e] += n;
      p.assigned_ += n;
    }
  }
  for (int e = 0; e < N; ++e)
    if (p.total_[e] < 1)
      throw std::invalid_argument("from_counts: expert " + std::to_string(e) + " has no replica");
  return p;
}

SlotPlacement SlotPlacement::from_slots(const int32_t* slots_GE, int G, int E, int N) {
  SlotPlacement p(G, E, N);
  for (int i = 0; i < G * E; ++i) {
    const int e = slots_GE[i];
    if (e < -1 || e >= N) throw std::invalid_argument("placement: slot holds invalid expert id");
    p.slot_[i] = e;
    if (e >= 0) {
      p.count_[e * G + i / E] += 1;
      p.total_[e] += 1;
      p.assigned_ += 1;
    }
  }
  return p;
}

std::vector<int> SlotPlacement::hosts(int e) const {
  std::vector<int> h;
  for (int g = 0; g < G_; ++g)
    if (count_[e * G_ + g] > 0) h.push_back(g);
  return h;
}

int SlotPlacement::free_slots(int g) const {
  int n = 0;
  for (int s = 0; s < E_; ++s) n += slot_[g * E_ + s] < 0;
  return n;
}

int SlotPlacement::first_free(int g) const {
  for (int s = 0; s < E_; ++s)
    if (slot_[g * E_ + s] < 0) return s;
  return -1;
}

double SlotPlacement::utilization() const {
  return static_cast<double>(assigned_) / (static_cast<double>(G_) * E_);
}

std::optional<Transfer> SlotPlacement::expand(int e, int g, const ClusterProfile& prof) {
  if (e < 0 || e >= N_ || g < 0 || g >= G_) throw std::invalid_argument("expand: id out of range");
  const int s = first_free(g);
  if (s < 0) throw std::invalid_argument("expand: no free vExpert slot on GPU " + std::to_string(g));
  std::optional<Transfer> t;
  if (count_[e * G_ + g] == 0) {  // a new GPU: copy the state from the best-connected replica
    if (total_[e] == 0)
      throw std::invalid_argument("expand: expert " + std::to_string(e) + " has no replica to copy from");
    int src = -1;
    double best = -1;
    for (int h : hosts(e)) {
      const double bw = prof.bandwidth(h, g);
      if (bw > best) {
        best = bw;
        src = h;
      }
    }
    t = Transfer{src, g, prof.expert_state_bytes};
  }
  slot_[g * E_ + s] = e;
  count_[e * G_ + g] += 1;
  total_[e] += 1;
  assigned_ += 1;
  return t;
}

void SlotPlacement::shrink(int e, int g) {
  if (e < 0 || e >= N_ || g < 0 || g >= G_) throw std::invalid_argument("shrink: id out of range");
  if (count_[e * G_ + g] == 0)
    throw std::invalid_argument("shrink: expert " + std::to_string(e) + " has no replica on GPU " +
                                std::to_string(g));
  if (total_[e] <= 1)
    throw std::invalid_argument("shrink: cannot release the last replica of expert " + std::to_string(e));
  for (int s = E_ - 1; s >= 0; --s) {  // the highest-index slot of e on g
    if (slot_[g * E_ + s] == e) {
      slot_[g * E_ + s] = -1;
      count_[e * G_ + g] -= 1;
      total_[e] -= 1;
      assigned_ -= 1;
      return;
    }
  }
}

std::vector<Transfer> SlotPlacement::migrate(int ag, int as, int bg, int bs, const ClusterProfile& prof) {
  auto check = [&](int g, int s) {
    if (g < 0 || g >= G_ || s < 0 || s >= E_) throw std::invalid_argument("slot reference out of range");
  };
  check(ag, as);
  check(bg, bs);
  const int ea = slot_[ag * E_ + as], eb = slot_[bg * E_ + bs];
  if (ea < 0 || eb < 0) throw std::invalid_argument("migrate: both slots must be assigned");
  if (ea == eb) throw std::invalid_argument("migrate: slots host the same expert");
  if (ag == bg) throw std::invalid_argument("migrate: slots must live on different GPUs");
  slot_[ag * E_ + as] = eb;
  slot_[bg * E_ + bs] = ea;
  count_[ea * G_ + ag] -= 1;
  count_[ea * G_ + bg] += 1;
  count_[eb * G_ + bg] -= 1;
  count_[eb * G_ + ag] += 1;
  return {Transfer{ag, bg, prof.expert_state_bytes}, Transfer{bg, ag, prof.expert_state_bytes}};
}

std::vector<Transfer> SlotPlacement::apply(const Op& op, const ClusterProfile& prof) {
  switch (op.kind) {
    case kExpand: {
      auto t = expand(op.expert, op.gpu, prof);
      return t ? std::vector<Transfer>{*t} : std::vector<Transfer>{};
    }
    case kShrink:
      shrink(op.expert, op.gpu);
      return {};
    case kMigrate:
      return migrate(op.a_gpu, op.a_slot, op.b_gpu, op.b_slot, prof);
  }
  throw std::invalid_argument("placement: unknown op kind");
}

void SlotPlacement::validate() const {
  std::vector<int> c(static_cast<size_t>(N_) * G_, 0);
  int assigned = 0;
  for (int g = 0; g < G_; ++g)
    for (int s = 0; s < E_; ++s) {
      const int e = slot_[g * E_ + s];
      if (e < 0) continue;
      if (e >= N_) throw std::logic_error("placement invariant: slot holds invalid expert id");
      c[e * G_ + g] += 1;
      ++assigned;
    }
  if (c != count_ || assigned != assigned_)
    throw std::logic_error("placement invariant: replica counts out of sync");
  for (int e = 0; e < N_; ++e) {
    int t = 0;
    for (int g = 0; g < G_; ++g) t += c[e * G_ + g];
    if (t != total_[e]) throw std::logic_error("placement invariant: total replica count out of sync");
    if (t < 1) throw std::logic_error("placement invariant: expert " + std::to_string(e) + " has no replica");
  }
}

// ----------------------------------------------------------------- cost model
std::vector<int64_t> flows_for(const std::vector<int64_t>& D, const SlotPlacement& p) {
  const int N = p.experts(), G = p.gpus();
  std::vector<int32_t> cnt(p.counts().begin(), p.counts().end());
  std::vector<int64_t> flows(static_cast<size_t>(N) * G * G, 0);
  route_counts_host(D.data(), cnt.data(), N, G, flows.data());
  return flows;
}

void StepTime::refresh() {
  makespan = 0;
  for (const GpuTime& t : gpu) makespan = std::max(makespan, t.total());
}

double sync_seconds(const std::vector<int>& group, const ClusterProfile& prof) {
  if (group.size() <= 1) return 0.0;
  return prof.expert_param_bytes / prof.group_bps(group);
}

double transfer_seconds(const Transfer& t, const ClusterProfile& prof) {
  if (t.src == t.dst) throw std::invalid_argument("adjust_cost: transfer endpoints must differ");
  return t.bytes / prof.bandwidth(t.src, t.dst);
}

StepTime step_time(const std::vector<int64_t>& D, const SlotPlacement& p,
                   const std::vector<int64_t>& flows, const ClusterProfile& prof) {
  const int N = p.experts(), G = p.gpus();
  (void)D;
  StepTime st;
  st.gpu.resize(G);
  for (int e = 0; e < N; ++e) {
    const double sync = sync_seconds(p.hosts(e), prof);
    for (int g = 0; g < G; ++g) {
      int64_t tokens = 0;
      for (int s = 0; s < G; ++s) tokens += flows[(static_cast<size_t>(e) * G + s) * G + g];
      if (p.replicas_on(e, g) == 0) {
        if (tokens != 0)
          throw std::invalid_argument("step_cost: plan routes expert " + std::to_string(e) +
                                      " to non-hosting GPU " + std::to_string(g));
        continue;
      }
      GpuTime& t = st.gpu[g];
      t.compute += static_cast<double>(tokens) / prof.tps;
      double a2a = 0;  // remote inbound bytes / link bandwidth, x4 exchanges
      for (int s = 0; s < G; ++s) {
        if (s == g) continue;
        const int64_t f = flows[(static_cast<size_t>(e) * G + s) * G + g];
        if (f > 0) a2a += static_cast<double>(f) * prof.token_bytes / prof.bandwidth(g, s);
      }
      t.a2a += 4.0 * a2a;
      t.sync += sync;
    }
  }
  st.refresh();
  return st;
}

double balance_of(const std::vector<int64_t>& flows, int N, int G) {
  return balance_ratio_host(flows.data(), N, G);
}

double variance_of(const std::vector<int64_t>& flows, int N, int G) {
  std::vector<double> tot(G, 0.0);
  for (int e = 0; e < N; ++e)
    for (int s = 0; s < G; ++s)
      for (int d = 0; d < G; ++d) tot[d] += static_cast<double>(flows[(static_cast<size_t>(e) * G + s) * G + d]);
  double mean = 0;
  for (double t : tot) mean += t;
  mean /= G;
  double var = 0;
  for (double t : tot) var += (t - mean) * (t - mean);
  return var / G;
}

// ----------------------------------------------------------------- policy
namespace {

int64_t load_of(const std::vector<int64_t>& D, int e, int G) {
  int64_t s = 0;
  for (int g = 0; g < G; ++g) s += D[static_cast<size_t>(e) * G + g];
  return s;
}

struct Trial {
  SlotPlacement p;
  std::vector<Op> ops;
  double move_seconds = 0;
};

}  // namespace

std::vector<Op> plan_balance(const std::vector<int64_t>& D, const SlotPlacement& p,
                             const ClusterProfile& prof, int horizon) {
  if (horizon < 1) throw std::invalid_argument("make_scheduling_plan: amortization_horizon must be >= 1");
  const int N = p.experts(), G = p.gpus();
  const std::vector<int64_t> base_flows = flows_for(D, p);
  const StepTime base = step_time(D, p, base_flows, prof);
  const double t0 = base.makespan;

  auto cap = [&](int e) { return static_cast<double>(load_of(D, e, G)) / static_cast<double>(p.replicas(e)); };
  int hot = -1, cold = -1;
  double hot_cap = -1, cold_cap = std::numeric_limits<double>::infinity();
  for (int e = 0; e < N; ++e) {
    const double c = cap(e);
    if (c > hot_cap) hot_cap = c, hot = e;
    if (c < cold_cap) cold_cap = c, cold = e;
  }
  if (hot == cold) return {};

  int bottleneck = 0;
  for (int g = 1; g < G; ++g)
    if (base.gpu[g].total() > base.gpu[bottleneck].total()) bottleneck = g;
  int hot_local = -1;
  double hot_local_cap = -1;
  for (int e = 0; e < N; ++e)
    if (p.replicas_on(e, bottleneck) > 0 && load_of(D, e, G) > 0 && cap(e) > hot_local_cap)
      hot_local_cap = cap(e), hot_local = e;

  std::vector<int64_t> recv(G, 0);  // per-GPU received tokens of the baseline
  for (int e = 0; e < N; ++e)
    for (int s = 0; s < G; ++s)
      for (int d = 0; d < G; ++d) recv[d] += base_flows[(static_cast<size_t>(e) * G + s) * G + d];
  int free_total = 0;
  for (int g = 0; g < G; ++g) free_total += p.free_slots(g);

  auto add_expand = [&](Trial& c, int e, int g) {
    const std::optional<Transfer> t = c.p.expand(e, g, prof);
    c.ops.push_back(Op{kExpand, e, g});
    if (t) c.move_seconds += transfer_seconds(*t, prof);
  };
  auto add_shrink = [&](Trial& c, int e, int g) {
    c.p.shrink(e, g);
    c.ops.push_back(Op{kShrink, e, g});
  };
  auto emptiest_with_room = [&](const SlotPlacement& q, int skip) {
    int best = -1;
    for (int g = 0; g < G; ++g)
      if (g != skip && q.free_slots(g) > 0 && (best < 0 || recv[g] < recv[best])) best = g;
    return best;
  };
  auto busiest_host = [&](int e) {
    int best = -1;
    for (int g : p.hosts(e))
      if (best < 0 || recv[g] > recv[best]) best = g;
    return best;
  };
  auto coldest_on = [&](int g, int except) {
    int best = -1;
    double best_cap = 0;
    for (int e = 0; e < N; ++e)
      if (e != except && p.replicas_on(e, g) > 0 && (best < 0 || cap(e) < best_cap)) best_cap = cap(e), best = e;
    return best;
  };

  // (1) one more replica; with a full pool, first free a slot of the coldest expert
  auto one_replica = [&](int e0) -> std::optional<Trial> {
    Trial c{p, {}, 0};
    if (free_total == 0) {
      if (e0 == cold || p.replicas(cold) < 2) return std::nullopt;
      add_shrink(c, cold, busiest_host(cold));
    }
    add_expand(c, e0, emptiest_with_room(c.p, -1));
    return c;
  };
  // (2) an extra slot on the busiest host plus one remote replica, scored together
  auto two_replicas = [&](int e0) -> std::optional<Trial> {
    if (free_total < 2) return std::nullopt;
    const int home = busiest_host(e0);
    if (p.free_slots(home) == 0) return std::nullopt;
    Trial c{p, {}, 0};
    add_expand(c, e0, home);
    const int far = emptiest_with_room(c.p, -1);
    if (far < 0) return std::nullopt;
    add_expand(c, e0, far);
    return c;
  };
  // (3) mutual replication with the strongest expert of the target GPU
  auto exchange = [&](int e0) -> std::optional<Trial> {
    if (free_total < 2) return std::nullopt;
    Trial c{p, {}, 0};
    const int far = emptiest_with_room(c.p, -1);
    if (far < 0) return std::nullopt;
    const int home = busiest_host(e0);
    int partner = -1;
    double partner_cap = -1;
    for (int e = 0; e < N; ++e)
      if (e != e0 && p.replicas_on(e, far) > 0 && cap(e) > partner_cap) partner_cap = cap(e), partner = e;
    if (partner < 0 || home == far) return std::nullopt;
    add_expand(c, e0, far);
    if (c.p.free_slots(home) == 0) return std::nullopt;
    add_expand(c, partner, home);
    return c;
  };
  // (4) move the coldest expert off `from` (re-homing it if it is a last replica)
  auto move_cold_off = [&](int from) -> std::optional<Trial> {
    const int victim = coldest_on(from, hot);
    if (victim < 0) return std::nullopt;
    Trial c{p, {}, 0};
    if (p.replicas(victim) < 2) {
      const int spill = emptiest_with_room(p, from);
      if (spill < 0) return std::nullopt;
      add_expand(c, victim, spill);
    }
    add_shrink(c, victim, from);
    return c;
  };
  // (5) clear the GPU that would keep the least load once its coldest expert
  //     leaves, and give the freed slot to e0
  auto evict_then_expand = [&](int e0) -> std::optional<Trial> {
    int target = -1, evicted = -1;
    int64_t best_left = 0;
    for (int g = 0; g < G; ++g) {
      const int v = coldest_on(g, e0);
      if (v < 0) continue;
      const int64_t left = recv[g] - load_of(D, v, G);
      if (target < 0 || left < best_left) best_left = left, target = g, evicted = v;
    }
    if (target < 0) return std::nullopt;
    Trial c{p, {}, 0};
    if (p.replicas(evicted) < 2) {
      const int spill = emptiest_with_room(p, target);
      if (spill < 0) return std::nullopt;
      add_expand(c, evicted, spill);
    }
    add_shrink(c, evicted, target);
    add_expand(c, e0, target);
    return c;
  };

  // trial order matters for ties: hot expert's four, then the bottleneck's
  // hottest expert's four (when different), then the cold relocation
  std::vector<int> subjects{hot};
  if (hot_local >= 0 && hot_local != hot) subjects.push_back(hot_local);
  std::vector<std::optional<Trial>> trials;
  for (int e0 : subjects) {
    trials.push_back(one_replica(e0));
    trials.push_back(two_replicas(e0));
    trials.push_back(exchange(e0));
    trials.push_back(evict_then_expand(e0));
  }
  trials.push_back(move_cold_off(bottleneck));

  // Best strict improvement of the modelled step time (+ amortised transfer) wins;
  // ties keep the earliest trial.
  const Trial* best = nullptr;
  double best_t = t0;
  for (const auto& tr : trials) {
    if (!tr) continue;
    const double t1 = step_time(D, tr->p, flows_for(D, tr->p), prof).makespan + tr->move_seconds / horizon;
    if (t1 < best_t) best_t = t1, best = &*tr;
  }
  return best ? best->ops : std::vector<Op>{};
}

std::vector<Op> plan_relocation(const SlotPlacement& p, const ClusterProfile& prof, int horizon) {
  const int G = p.gpus(), E = p.slots();
  auto hosts_after = [&](int e, int from, int to) {
    std::vector<int> grp;
    for (int g = 0; g < G; ++g) {
      const int c = p.replicas_on(e, g) - (g == from) + (g == to);
      if (c > 0) grp.push_back(g);
    }
    return grp;
  };
  bool found = false;
  Op best_op{kMigrate};
  double best_score = 0;
  for (int ga = 0; ga < G; ++ga)
    for (int sa = 0; sa < E; ++sa) {
      const int ea = p.slot(ga, sa);
      if (ea < 0) continue;
      for (int gb = ga + 1; gb < G; ++gb)
        for (int sb = 0; sb < E; ++sb) {
          const int eb = p.slot(gb, sb);
          if (eb < 0 || eb == ea) continue;
          // pure relocations only: the swap must not collapse a replica set
          const std::vector<int> na = hosts_after(ea, ga, gb), nb = hosts_after(eb, gb, ga);
          if (na.size() != p.hosts(ea).size() || nb.size() != p.hosts(eb).size()) continue;
          const double before = sync_seconds(p.hosts(ea), prof) + sync_seconds(p.hosts(eb), prof);
          const double after = sync_seconds(na, prof) + sync_seconds(nb, prof);
          const double moving = 2.0 * prof.expert_state_bytes / prof.bandwidth(ga, gb);
          const double score = before - after - moving / horizon;
          if (score > 0 && (!found || score > best_score)) {
            found = true;
            best_score = score;
            best_op = Op{kMigrate, -1, -1, ga, sa, gb, sb};
          }
        }
    }
  return found ? std::vector<Op>{best_op} : std::vector<Op>{};
}

// ----------------------------------------------------------------- queue
bool TransferQueue::Pending::done() const {
  for (const Transfer& t : left)
    if (t.bytes > 0) return false;
  return true;
}

void TransferQueue::push(const Op& op, const std::vector<Transfer>& t) { q_.push_back(Pending{op, t}); }

double TransferQueue::pending_bytes() const {
  double b = 0;
  for (const Pending& p : q_)
    for (const Transfer& t : p.left) b += std::max(0.0, t.bytes);
  return b;
}

std::vector<std::vector<TransferQueue::Merged>> TransferQueue::schedule() const {
  std::vector<Merged> msgs;
  for (size_t i = 0; i < q_.size(); ++i)
    for (size_t j = 0; j < q_[i].left.size(); ++j) {
      const Transfer& t = q_[i].left[j];
      if (t.bytes <= 0) continue;
      if (!msgs.empty() && msgs.back().src == t.src && msgs.back().dst == t.dst) {
        msgs.back().bytes += t.bytes;
        msgs.back().parts.emplace_back(i, j);
      } else {
        msgs.push_back(Merged{t.src, t.dst, t.bytes, {{i, j}}});
      }
    }
  std::vector<std::vector<Merged>> sets;
  for (Merged& m : msgs) {
    bool disjoint = !sets.empty();
    if (disjoint)
      for (const Merged& o : sets.back())
        if (o.src == m.src || o.src == m.dst || o.dst == m.src || o.dst == m.dst) {
          disjoint = false;
          break;
        }
    if (disjoint) sets.back().push_back(std::move(m));
    else sets.push_back({std::move(m)});
  }
  return sets;
}

std::vector<Op> TransferQueue::drain(double seconds, const ClusterProfile& prof, SlotPlacement& effective,
                                     double& bytes_moved, double& seconds_used) {
  bytes_moved = 0;
  seconds_used = 0;
  double budget = std::max(0.0, seconds);
  for (const auto& set : schedule()) {
    if (budget <= 0) break;
    double elapsed = 0;
    bool finished = true;
    for (const Merged& m : set) {
      const double bw = prof.bandwidth(m.src, m.dst);
      const double need = m.bytes / bw;
      double moved;
      if (need <= budget) {
        moved = m.bytes;
        elapsed = std::max(elapsed, need);
      } else {
        moved = budget * bw;
        elapsed = budget;
        finished = false;
      }
      bytes_moved += moved;
      for (const auto& [i, j] : m.parts) {  // book against the oldest transfers first
        if (moved <= 0) break;
        Transfer& t = q_[i].left[j];
        const double take = std::min(t.bytes, moved);
        t.bytes -= take;
        moved -= take;
      }
      if (need <= budget)
        for (const auto& [i, j] : m.parts) q_[i].left[j].bytes = 0;
    }
    seconds_used += elapsed;
    budget -= elapsed;
    if (!finished) break;
  }
  std::vector<Op> applied;
  while (!q_.empty() && q_.front().done()) {
    effective.apply(q_.front().op, ClusterProfile(prof));
    applied.push_back(q_.front().op);
    q_.pop_front();
  }
  return applied;
}

bool GroupLru::touch(const std::vector<int>& group) {
  auto it = where_.find(group);
  if (it != where_.end()) {
    order_.splice(order_.begin(), order_, it->second);
    return true;
  }
  ++misses_;
  order_.push_front(group);
  where_[group] = order_.begin();
  if (static_cast<int>(where_.size()) > cap_) {
    where_.erase(order_.back());
    order_.pop_back();
  }
  return false;
}

// ----------------------------------------------------------------- scheduler
Scheduler::Scheduler(const ClusterProfile& prof, const SchedulerConfig& cfg, int num_experts)
    : prof_(prof),
      cfg_(cfg),
      effective_(SlotPlacement::round_robin(num_experts, prof.num_gpus, prof.slots_per_gpu)),
      target_(effective_),
      lru_(cfg.max_live_groups) {
  if (!(cfg.threshold > 1.0)) throw std::invalid_argument("SimConfig: threshold must be > 1");
  if (cfg.interval_steps < 1) throw std::invalid_argument("SimConfig: interval_steps must be >= 1");
  if (cfg.horizon < 1) throw std::invalid_argument("SimConfig: amortization_horizon must be >= 1");
  if (!(cfg.adjust_bandwidth_fraction > 0) || cfg.adjust_bandwidth_fraction > 1)
    throw std::invalid_argument("SimConfig: adjust_bandwidth_fraction must be in (0, 1]");
  if (cfg.max_live_groups < 1) throw std::invalid_argument("SimConfig: max_live_groups must be >= 1");
}

Scheduler::~Scheduler() {
  if (worker_.joinable()) worker_.join();
}

std::vector<Op> Scheduler::join_policy() {
  if (!worker_.joinable()) return {};
  worker_.join();
  std::vector<Op> ops = std::move(worker_ops_);
  worker_ops_.clear();
  commit(ops);
  return ops;
}

void Scheduler::commit(const std::vector<Op>& ops) {
  for (const Op& op : ops) queue_.push(op, target_.apply(op, prof_));
}

void Scheduler::reset(const SlotPlacement& p) {
  if (worker_.joinable()) worker_.join();
  worker_ops_.clear();
  effective_ = p;
  target_ = p;
  queue_ = TransferQueue();
  inflight_.clear();
  prev_makespan_ = 0;
}

double Scheduler::trigger(const std::vector<int64_t>& flows, int N) const {
  const int G = prof_.num_gpus;
  if (cfg_.metric == 0) return balance_of(flows, N, G);
  int64_t sum = 0;
  for (int64_t f : flows) sum += f;
  if (sum == 0) throw std::invalid_argument("trigger_value: zero total tokens");
  const double mean = static_cast<double>(sum) / static_cast<double>(G);
  return 1.0 + std::sqrt(variance_of(flows, N, G)) / mean;
}

StepOutcome Scheduler::step(const std::vector<int64_t>& D) {
  begin_step();
  return finish_step(D);
}

const StepOutcome& Scheduler::begin_step() {
  cur_ = StepOutcome{};
  if (cfg_.flip_mode == 0) {
    // 1. transfers that overlapped the previous step land (best-effort budget)
    cur_.applied = queue_.drain(cfg_.adjust_bandwidth_fraction * prev_makespan_, prof_, effective_,
                                cur_.adjust_bytes, cur_.adjust_seconds);
  } else {
    // 1'. the copies issued at the previous boundary completed inside that
    // step: those ops become effective, in queue order
    for (size_t i = 0; i < inflight_.size(); ++i) {
      const Op op = queue_.pending().front().op;
      effective_.apply(op, prof_);
      cur_.applied.push_back(op);
      queue_.pop_front();
    }
    inflight_.clear();
    // ... and the next queue prefix within the adjustment budget starts
    const double budget = cfg_.adjust_bandwidth_fraction * prev_makespan_;
    double used = 0;
    for (const auto& p : queue_.pending()) {
      double t = 0;
      for (const Transfer& x : p.left) t += x.bytes > 0 ? transfer_seconds(x, prof_) : 0.0;
      if (!inflight_.empty() && used + t > budget) break;
      used += t;
      for (const Transfer& x : p.left) cur_.adjust_bytes += std::max(0.0, x.bytes);
      inflight_.push_back(p.op);
    }
    cur_.adjust_seconds = used;
    cur_.issued = inflight_;
  }
  begun_ = true;
  return cur_;
}

std::vector<Op> Scheduler::run_policy(const std::vector<int64_t>& D, SlotPlacement target, bool policy_step,
                                      bool triggered) const {
  const int N = target.experts();
  std::vector<Op> ops;
  // 3. policy on the target placement (pending adjustments are not re-planned)
  if (policy_step && triggered) {
    while (true) {
      if (trigger(flows_for(D, target), N) <= cfg_.threshold) break;
      const std::vector<Op> plan = plan_balance(D, target, prof_, cfg_.horizon);
      if (plan.empty()) break;
      for (const Op& op : plan) {
        target.apply(op, prof_);
        ops.push_back(op);
      }
    }
  }
  // 4. one replica-locality migration, confirmed by the full cost model
  if (cfg_.policy_mode != 2) {
    const std::vector<Op> mig = plan_relocation(target, prof_, cfg_.horizon);
    if (!mig.empty()) {
      const Op& op = mig.front();
      const double before = step_time(D, target, flows_for(D, target), prof_).makespan;
      SlotPlacement swapped = target;
      swapped.migrate(op.a_gpu, op.a_slot, op.b_gpu, op.b_slot, prof_);
      const double after = step_time(D, swapped, flows_for(D, swapped), prof_).makespan;
      if (after <= before * (1.0 + 1e-12)) ops.push_back(op);
    }
  }
  return ops;
}

StepOutcome Scheduler::finish_step(const std::vector<int64_t>& D) {
  if (!begun_) throw std::logic_error("scheduler: finish_step without begin_step");
  begun_ = false;
  const int N = effective_.experts(), G = effective_.gpus();
  StepOutcome out = cur_;
  // 2. the step on the effective placement
  const std::vector<int64_t> flows = flows_for(D, effective_);
  StepTime st = step_time(D, effective_, flows, prof_);
  for (int e = 0; e < N; ++e) {  // group creation, ascending expert id
    const std::vector<int> grp = effective_.hosts(e);
    if (grp.size() < 2) continue;
    if (!lru_.touch(grp)) {
      ++out.group_misses;
      for (int g : grp) st.gpu[g].sync += cfg_.group_creation_latency_s;
    }
  }
  st.refresh();
  out.makespan = st.makespan;
  out.balance_ratio = balance_of(flows, N, G);
  out.metric_value = cfg_.metric == 0 ? out.balance_ratio : variance_of(flows, N, G);
  const bool policy_step = cfg_.policy_mode == 0 || (cfg_.policy_mode == 1 && step_ % cfg_.interval_steps == 0);
  const bool triggered = policy_step && trigger(flows, N) > cfg_.threshold;
  if (cfg_.async_policy) {
    // the previous step's policy (it ran while this step was enqueued) enters
    // the queue now; this step's starts on a snapshot of the new target
    out.accepted = join_policy();
    worker_ = std::thread([this, D, snap = target_, policy_step, triggered] {
      worker_ops_ = run_policy(D, snap, policy_step, triggered);
    });
  } else {
    out.accepted = run_policy(D, target_, policy_step, triggered);
    commit(out.accepted);
  }
  prev_makespan_ = out.makespan;
  ++step_;
  return out;
}

}  // namespace sched
}  // namespace fm
