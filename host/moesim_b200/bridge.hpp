// bridge.hpp — the moesim side of the drop-in: conversions between the
// reference's value types (proj/include/moesim/*.hpp) and the plain arrays of
// include/flexmoe_b200.h, and the status -> exception mapping.
// This is the code a moesim maintainer adds next to their library (it
// includes their headers; it copies none of their sources).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "flexmoe_b200.h"
#include "moesim/placement.hpp"
#include "moesim/topology.hpp"
#include "moesim/workload.hpp"

namespace moesim::b200 {

// FM_ERR_* -> the exception class the reference throws for the same failure.
inline void check(int status) {
  if (status == FM_OK) return;
  const std::string msg = fm_last_error();
  switch (status) {
    case FM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FM_ERR_LOGIC: throw std::logic_error(msg);
    case FM_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// Placement::replica_count_on (placement.hpp:80-82) for the first n experts.
inline std::vector<int32_t> replica_counts(const Placement& p, int n) {
  std::vector<int32_t> c(static_cast<size_t>(n) * p.num_gpus());
  for (ExpertId e = 0; e < n; ++e)
    for (GpuId g = 0; g < p.num_gpus(); ++g) c[static_cast<size_t>(e) * p.num_gpus() + g] = p.replica_count_on(e, g);
  return c;
}

// Placement::slot (placement.hpp:79) as the [gpu][slot] table of the C ABI.
inline std::vector<int32_t> slot_table(const Placement& p) {
  std::vector<int32_t> s(static_cast<size_t>(p.num_gpus()) * p.slots_per_gpu());
  for (GpuId g = 0; g < p.num_gpus(); ++g)
    for (int i = 0; i < p.slots_per_gpu(); ++i) s[static_cast<size_t>(g) * p.slots_per_gpu() + i] = p.slot(g, i);
  return s;
}

// TokenDemand rows padded (zeros) to n experts.
inline std::vector<int64_t> demand_rows(const TokenDemand& d, int n) {
  std::vector<int64_t> D(static_cast<size_t>(n) * d.num_gpus, 0);
  for (ExpertId e = 0; e < std::min(n, d.num_experts); ++e)
    for (GpuId g = 0; g < d.num_gpus; ++g) D[static_cast<size_t>(e) * d.num_gpus + g] = d.at(e, g);
  return D;
}

// ClusterTopology (topology.hpp:27-94) -> fm_cluster_profile, through its own
// JSON form so the all-reduce tables come over exactly.
inline fm_cluster_profile profile(const ClusterTopology& t) {
  fm_cluster_profile c{};
  c.num_gpus = t.num_gpus();
  c.gpus_per_node = t.gpus_per_node();
  c.slots_per_gpu = t.vexperts_per_gpu();
  c.intra_node_bandwidth_bps = t.intra_node_bandwidth();
  c.inter_node_bandwidth_bps = t.inter_node_bandwidth();
  c.tps = t.tps();
  c.expert_param_bytes = t.expert_param_bytes();
  c.expert_state_bytes = t.expert_state_bytes();
  c.token_bytes = t.token_bytes();
  const nlohmann::json j = t.to_json();
  if (j.contains("allreduce_bps")) {
    const auto& ar = j.at("allreduce_bps");
    auto fill = [&](const char* key, double* table) {
      if (!ar.contains(key)) return;
      for (auto it = ar.at(key).begin(); it != ar.at(key).end(); ++it) {
        const int size = std::stoi(it.key());
        if (size >= 0 && size <= FM_MAX_GROUP) table[size] = it.value().get<double>();
      }
    };
    fill("intra", c.allreduce_bps_intra);
    fill("inter", c.allreduce_bps_inter);
  }
  return c;
}

inline PlacementOp to_op(const fm_placement_op& o) {
  PlacementOp op;
  op.kind = static_cast<PlacementOpKind>(o.kind);
  op.expert = o.expert;
  op.gpu = o.gpu;
  op.a = SlotRef{o.a_gpu, o.a_slot};
  op.b = SlotRef{o.b_gpu, o.b_slot};
  return op;
}

}  // namespace moesim::b200
