// policy_b200.cpp — moesim's placement policy API (proj/include/moesim/
// policy.hpp) served by libflexmoe_b200.so. Built INSTEAD of the
// reference's proj/src/policy.cpp: SimEngine's trigger, expand/shrink
// planning and migration pass then run the framework's host scheduler
// (csrc/scheduler.cpp), which takes identical decisions.
#include <algorithm>
#include <stdexcept>
#include <vector>

#include "bridge.hpp"
#include "moesim/policy.hpp"

namespace moesim {

namespace {

constexpr int kMaxOps = 64;

SchedulingPlan to_plan(const fm_placement_op* ops, int n) {
  SchedulingPlan plan;
  for (int i = 0; i < n; ++i) plan.ops.push_back(b200::to_op(ops[i]));
  return plan;
}

std::vector<int64_t> totals_of(const RoutingPlan& plan) { return per_gpu_received(plan); }

}  // namespace

// policy.hpp:38 (Eq. 7) -> fm_balance_ratio
double balance_ratio(const TokenDemand&, const Placement&, const RoutingPlan& plan) {
  double r = 0.0;
  b200::check(fm_balance_ratio(plan.flows.data(), plan.num_experts, plan.num_gpus, &r));
  return r;
}

// policy.hpp:42: population variance of the per-GPU received totals
double variance_metric(const TokenDemand&, const Placement&, const RoutingPlan& plan) {
  const std::vector<int64_t> totals = totals_of(plan);
  double mean = 0.0;
  for (int64_t t : totals) mean += static_cast<double>(t);
  mean /= static_cast<double>(totals.size());
  double var = 0.0;
  for (int64_t t : totals) {
    const double diff = static_cast<double>(t) - mean;
    var += diff * diff;
  }
  return var / static_cast<double>(totals.size());
}

// policy.hpp:57 -> fm_make_scheduling_plan
SchedulingPlan make_scheduling_plan(const TokenDemand& d, const Placement& p, const ClusterTopology& topo,
                                    const PolicyConfig& cfg) {
  const int n = std::max(d.num_experts, p.num_experts());
  const std::vector<int64_t> D = b200::demand_rows(d, n);
  const std::vector<int32_t> slots = b200::slot_table(p);
  const fm_cluster_profile prof = b200::profile(topo);
  fm_placement_op ops[kMaxOps];
  int n_ops = 0;
  b200::check(fm_make_scheduling_plan(D.data(), slots.data(), n, &prof, cfg.amortization_horizon, ops, kMaxOps,
                                      &n_ops));
  return to_plan(ops, n_ops);
}

// policy.hpp:65 -> fm_plan_migrations
SchedulingPlan plan_migrations(const Placement& p, const ClusterTopology& topo, const PolicyConfig& cfg) {
  const std::vector<int32_t> slots = b200::slot_table(p);
  const fm_cluster_profile prof = b200::profile(topo);
  fm_placement_op ops[kMaxOps];
  int n_ops = 0;
  b200::check(fm_plan_migrations(slots.data(), p.num_experts(), &prof, cfg.amortization_horizon, ops, kMaxOps,
                                 &n_ops));
  return to_plan(ops, n_ops);
}

}  // namespace moesim
