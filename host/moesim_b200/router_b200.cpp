// router_b200.cpp — moesim's routing API (proj/include/moesim/router.hpp)
// served by libflexmoe_b200.so. Built INSTEAD of the reference's
// proj/src/router.cpp: every caller (SimEngine::run_step, the policy's
// what-ifs, the oracle, the baselines, the CLI) then routes through the
// B200 framework's Alg. 3 implementation, bit-identical to the original.
#include <sstream>
#include <string>
#include <vector>

#include "bridge.hpp"
#include "moesim/router.hpp"

namespace moesim {

// RoutingPlan::received (router.hpp:47)
int64_t RoutingPlan::received(ExpertId e, GpuId dst) const {
  int64_t sum = 0;
  for (GpuId src = 0; src < num_gpus; ++src) sum += flow(e, src, dst);
  return sum;
}

// router.hpp:51 -> fm_received_matrix
std::vector<int64_t> received_matrix(const RoutingPlan& plan) {
  std::vector<int64_t> recv(static_cast<size_t>(plan.num_experts) * plan.num_gpus, 0);
  if (plan.num_experts > 0)
    b200::check(fm_received_matrix(plan.flows.data(), plan.num_experts, plan.num_gpus, recv.data()));
  return recv;
}

// router.hpp:54 -> fm_per_gpu_received
std::vector<int64_t> per_gpu_received(const RoutingPlan& plan) {
  std::vector<int64_t> totals(plan.num_gpus, 0);
  if (plan.num_experts > 0)
    b200::check(fm_per_gpu_received(plan.flows.data(), plan.num_experts, plan.num_gpus, totals.data()));
  return totals;
}

// router.hpp:62 -> fm_route_counts (same preconditions and messages as the
// original, router.cpp:58-63; the counting itself runs in the framework)
RoutingPlan route(const TokenDemand& d, const Placement& p) {
  if (d.num_gpus != p.num_gpus())
    throw std::invalid_argument("route: demand and placement disagree on GPU count");
  if (d.num_experts > p.num_experts())
    throw std::invalid_argument("route: demand names more experts than the placement");
  RoutingPlan plan(d.num_experts, d.num_gpus);
  if (d.num_experts == 0) return plan;
  const std::vector<int32_t> counts = b200::replica_counts(p, d.num_experts);
  b200::check(fm_route_counts(d.demand.data(), counts.data(), d.num_experts, d.num_gpus, plan.flows.data()));
  return plan;
}

// router.hpp:66: trace format plus a destination column, nonzero flows in
// (expert, src, dst) order.
std::string plan_to_csv(const RoutingPlan& plan, int step) {
  std::ostringstream out;
  out << "step,expert,gpu,dst,tokens\n";
  for (ExpertId e = 0; e < plan.num_experts; ++e)
    for (GpuId src = 0; src < plan.num_gpus; ++src)
      for (GpuId dst = 0; dst < plan.num_gpus; ++dst)
        if (const int64_t f = plan.flow(e, src, dst)) out << step << ',' << e << ',' << src << ',' << dst << ',' << f << '\n';
  return out.str();
}

}  // namespace moesim
