// Comparison baselines of the paper's evaluation,
// per step, on the same routing / cost model / group cache as the FlexMoE
// scheduler. Behavioural source: proj/src/baselines.cpp:81-276
// (`run_baseline`), paths relative to /root/reference.
//
//   StaticEP        DeepSpeed-like: round-robin placement, capacity
//                   cap = floor(cf * B / N); over-cap experts keep a
//                   largest-remainder share per source GPU (:81-127)
//   FullReplicate   FasterMoE-like shadowing: round-robin placement with
//                   replicate_top extra slots per GPU, and the currently
//                   hottest replicate_top experts expanded onto every GPU
//                   (:129-161) — re-derived from the step's own demand
//   StrictRebalance loads rewritten so every GPU receives exactly B/G
//                   (BASE-layer-like assignment; count level) (:163-232)
//
// Each step yields the placement it ran on (so the device runtime can run
// FullReplicate for real: shadows broadcast from the owner, gradients summed
// within the replica group), the demand it routed (post-drop / rebalanced),
// and the reference's StepReport fields (make_report, :42-79).
#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "fm_internal.h"
#include "scheduler.h"

namespace fm {
void largest_remainder_round_host(const double* exact, int n, int64_t total, int64_t* out);
int64_t static_ep_kept_host(const int64_t* D, int N, int G, double cf, int64_t* kept);

namespace sched {
namespace {

int experts_per_gpu(int N, int G) { return (N + G - 1) / G; }

int64_t expert_load(const std::vector<int64_t>& D, int e, int G) {
  int64_t s = 0;
  for (int g = 0; g < G; ++g) s += D[static_cast<size_t>(e) * G + g];
  return s;
}

// max * G / sum, 1.0 for an empty step (baselines.cpp:31-40 — note the
// operation order differs from balance_ratio's max / (sum / G)).
double safe_ratio(const std::vector<int64_t>& flows, int N, int G) {
  std::vector<int64_t> tot(G, 0);
  for (int e = 0; e < N; ++e)
    for (int s = 0; s < G; ++s)
      for (int d = 0; d < G; ++d) tot[d] += flows[(static_cast<size_t>(e) * G + s) * G + d];
  const int64_t sum = std::accumulate(tot.begin(), tot.end(), int64_t{0});
  if (sum == 0) return 1.0;
  const int64_t mx = *std::max_element(tot.begin(), tot.end());
  return static_cast<double>(mx) * static_cast<double>(G) / static_cast<double>(sum);
}

}  // namespace

struct BaselineConfig {
  int kind = 0;  // 0 StaticEP, 1 FullReplicate, 2 StrictRebalance
  double capacity_factor = 1.0;
  int replicate_top = 1;
  int metric = 0;
  int max_live_groups = 64;
  double group_creation_latency_s = 0.005;
};

struct BaselineOutcome {
  double balance_ratio = 1, metric_value = 0, makespan = 0, slot_utilization = 0;
  int group_misses = 0;
  int64_t tokens_total = 0, tokens_dropped = 0, tokens_reassigned = 0;
  std::vector<int64_t> demand;  // what was routed
  std::vector<int64_t> flows;
};

class BaselineRunner {
 public:
  BaselineRunner(const ClusterProfile& prof, const BaselineConfig& cfg, int N)
      : prof_(prof), cfg_(cfg), N_(N), G_(prof.num_gpus), lru_(cfg.max_live_groups),
        placement_(SlotPlacement::round_robin(N, prof.num_gpus, experts_per_gpu(N, prof.num_gpus))) {
    if (cfg.kind < 0 || cfg.kind > 2) throw std::invalid_argument("run_baseline: unknown baseline");
    if (cfg.kind == 1) {
      top_ = std::min(cfg.replicate_top, N);
      if (top_ < 1) throw std::invalid_argument("full-replicate: replicate_top must be >= 1");
      placement_ = SlotPlacement::round_robin(N, G_, experts_per_gpu(N, G_) + top_);
    }
  }

  BaselineOutcome step(const std::vector<int64_t>& D) {
    BaselineOutcome out;
    const int64_t total = std::accumulate(D.begin(), D.end(), int64_t{0});
    if (first_total_ < 0) first_total_ = total;  // the trace's tokens_per_step (front().total())
    out.tokens_total = total;
    out.demand = D;
    if (cfg_.kind == 0) {
      if (!std::isinf(cfg_.capacity_factor))
        out.tokens_dropped = static_ep_kept_host(D.data(), N_, G_, cfg_.capacity_factor, out.demand.data());
    } else if (cfg_.kind == 1) {
      full_replicate_placement(D);
    } else {
      out.tokens_reassigned = strict_rebalance(D, out.demand);
    }
    report(out);
    return out;
  }

  const SlotPlacement& placement() const { return placement_; }

 private:
  // Round robin + the hottest `top_` experts (stable order, ties to the lower
  // id) expanded onto every GPU not yet hosting them (baselines.cpp:143-156).
  void full_replicate_placement(const std::vector<int64_t>& D) {
    std::vector<int> order(N_);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return expert_load(D, a, G_) > expert_load(D, b, G_); });
    placement_ = SlotPlacement::round_robin(N_, G_, experts_per_gpu(N_, G_) + top_);
    for (int i = 0; i < top_; ++i)
      for (int g = 0; g < G_; ++g)
        if (placement_.replicas_on(order[i], g) == 0) placement_.expand(order[i], g, prof_);
  }

  // New per-expert loads: each GPU's hosted experts share exactly B/G in
  // proportion to their loads (equal shares when the GPU saw none), then each
  // load is spread evenly over the source GPUs (baselines.cpp:176-224).
  int64_t strict_rebalance(const std::vector<int64_t>& D, std::vector<int64_t>& out) {
    if (first_total_ % G_ != 0) throw std::invalid_argument("strict-rebalance: step total not divisible by GPUs");
    const int64_t target = first_total_ / G_;
    std::vector<int64_t> load(N_, 0);
    for (int g = 0; g < G_; ++g) {
      std::vector<int> hosted;
      for (int e = 0; e < N_; ++e)
        if (placement_.replicas_on(e, g) > 0) hosted.push_back(e);
      int64_t gpu_load = 0;
      for (int e : hosted) gpu_load += expert_load(D, e, G_);
      std::vector<double> exact(hosted.size());
      for (size_t i = 0; i < hosted.size(); ++i)
        exact[i] = gpu_load > 0 ? static_cast<double>(expert_load(D, hosted[i], G_)) * static_cast<double>(target) /
                                      static_cast<double>(gpu_load)
                                : static_cast<double>(target) / static_cast<double>(hosted.size());
      std::vector<int64_t> r(hosted.size());
      largest_remainder_round_host(exact.data(), static_cast<int>(hosted.size()), target, r.data());
      for (size_t i = 0; i < hosted.size(); ++i) load[hosted[i]] = r[i];
    }
    int64_t moved = 0;
    for (int e = 0; e < N_; ++e) moved += std::llabs(load[e] - expert_load(D, e, G_));
    std::vector<double> even(G_);
    std::vector<int64_t> row(G_);
    for (int e = 0; e < N_; ++e) {
      for (int g = 0; g < G_; ++g) even[g] = static_cast<double>(load[e]) / G_;
      largest_remainder_round_host(even.data(), G_, load[e], row.data());
      for (int g = 0; g < G_; ++g) out[static_cast<size_t>(e) * G_ + g] = row[g];
    }
    return moved / 2;
  }

  // make_report (baselines.cpp:42-79): cost model on the routed demand, group
  // creation misses in ascending expert id, safe balance ratio.
  void report(BaselineOutcome& out) {
    out.flows = flows_for(out.demand, placement_);
    StepTime st = step_time(out.demand, placement_, out.flows, prof_);
    for (int e = 0; e < N_; ++e) {
      const std::vector<int> grp = placement_.hosts(e);
      if (grp.size() < 2) continue;
      if (!lru_.touch(grp)) {
        ++out.group_misses;
        for (int g : grp) st.gpu[g].sync += cfg_.group_creation_latency_s;
      }
    }
    st.refresh();
    out.makespan = st.makespan;
    out.balance_ratio = safe_ratio(out.flows, N_, G_);
    out.metric_value = cfg_.metric == 0 ? out.balance_ratio : variance_of(out.flows, N_, G_);
    out.slot_utilization = placement_.utilization();
  }

  ClusterProfile prof_;
  BaselineConfig cfg_;
  int N_, G_, top_ = 0;
  GroupLru lru_;
  SlotPlacement placement_;
  int64_t first_total_ = -1;
};

}  // namespace sched
}  // namespace fm

// ----------------------------------------------------------------- C ABI
struct fm_baseline {
  std::unique_ptr<fm::sched::BaselineRunner> runner;
  fm::sched::BaselineOutcome last;
};

namespace fm {
namespace sched {
ClusterProfile profile_from_c(const fm_cluster_profile* p);  // scheduler_capi.cpp
}
}  // namespace fm

extern "C" {

int fm_baseline_create(const fm_cluster_profile* profile, const fm_baseline_config* cfg, int num_experts,
                       fm_baseline** out) {
  return fm::guarded([&] {
    if (!profile || !cfg || !out || num_experts < 1) throw std::invalid_argument("fm_baseline_create: bad arguments");
    fm::sched::BaselineConfig c;
    c.kind = cfg->kind;
    c.capacity_factor = cfg->capacity_factor;
    c.replicate_top = cfg->replicate_top;
    c.metric = cfg->metric;
    c.max_live_groups = cfg->max_live_groups;
    c.group_creation_latency_s = cfg->group_creation_latency_s;
    auto h = std::make_unique<fm_baseline>();
    h->runner = std::make_unique<fm::sched::BaselineRunner>(fm::sched::profile_from_c(profile), c, num_experts);
    *out = h.release();
  });
}

int fm_baseline_destroy(fm_baseline* b) {
  delete b;
  return FM_OK;
}

int fm_baseline_step(fm_baseline* b, const int64_t* demand_NG, fm_baseline_report* out, int32_t* counts_NG,
                     int64_t* routed_demand_NG, int64_t* flows_NGG) {
  return fm::guarded([&] {
    if (!b || !demand_NG || !out) throw std::invalid_argument("fm_baseline_step: bad arguments");
    const fm::sched::SlotPlacement& p0 = b->runner->placement();
    const size_t NG = static_cast<size_t>(p0.experts()) * p0.gpus();
    std::vector<int64_t> D(demand_NG, demand_NG + NG);
    b->last = b->runner->step(D);
    const fm::sched::BaselineOutcome& o = b->last;
    out->balance_ratio = o.balance_ratio;
    out->metric_value = o.metric_value;
    out->makespan_s = o.makespan;
    out->slot_utilization = o.slot_utilization;
    out->group_misses = o.group_misses;
    out->tokens_total = o.tokens_total;
    out->tokens_dropped = o.tokens_dropped;
    out->tokens_reassigned = o.tokens_reassigned;
    const fm::sched::SlotPlacement& p = b->runner->placement();
    if (counts_NG)
      for (size_t i = 0; i < NG; ++i) counts_NG[i] = p.counts()[i];
    if (routed_demand_NG) std::copy(o.demand.begin(), o.demand.end(), routed_demand_NG);
    if (flows_NGG) std::copy(o.flows.begin(), o.flows.end(), flows_NGG);
  });
}

int fm_baseline_placement(fm_baseline* b, int32_t* slots_GE, int32_t* counts_NG, int* slots_per_gpu) {
  return fm::guarded([&] {
    if (!b) throw std::invalid_argument("fm_baseline_placement: null handle");
    const fm::sched::SlotPlacement& p = b->runner->placement();
    if (slots_per_gpu) *slots_per_gpu = p.slots();
    if (slots_GE) std::copy(p.slot_table().begin(), p.slot_table().end(), slots_GE);
    if (counts_NG) std::copy(p.counts().begin(), p.counts().end(), counts_NG);
  });
}

}  // extern "C"
