// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library (moesim,
// compiled from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libmoesim_ref.so). Used by the tests to pin the oracle and the
// product against the reference itself, by tests/golden/make_golden.py, and
// by bench.py's reference arm for the count-level CPU path timing.
// No reference source is copied: this file only calls the public API in
// proj/include/moesim/*.hpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "moesim/baselines.hpp"
#include "moesim/placement.hpp"
#include "moesim/policy.hpp"
#include "moesim/router.hpp"
#include "moesim/sim_engine.hpp"
#include "moesim/topology.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 4;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

TokenDemand to_demand(const int64_t* D, int N, int G) {
  TokenDemand d(0, N, G);
  std::memcpy(d.demand.data(), D, sizeof(int64_t) * N * G);
  return d;
}

Placement to_placement(const int32_t* cnt, int N, int G, int slots) {
  std::vector<int> counts(cnt, cnt + static_cast<size_t>(N) * G);
  return Placement::from_counts(counts, N, G, slots);
}

std::vector<TokenDemand> to_trace(const int64_t* D, int steps, int N, int G) {
  std::vector<TokenDemand> tr;
  for (int s = 0; s < steps; ++s) {
    TokenDemand d = to_demand(D + static_cast<size_t>(s) * N * G, N, G);
    d.step = s;
    tr.push_back(std::move(d));
  }
  return tr;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_route(const int64_t* D, const int32_t* cnt, int N, int G, int slots, int64_t* flows) {
  return guarded([&] {
    RoutingPlan plan = route(to_demand(D, N, G), to_placement(cnt, N, G, slots));
    std::memcpy(flows, plan.flows.data(), sizeof(int64_t) * plan.flows.size());
  });
}

// Route with a placement given slot-by-slot (slots_GE[g][s] = expert or -1),
// so placements built by expand/shrink sequences can be reproduced exactly.
int ref_balance_ratio(const int64_t* D, const int32_t* cnt, int N, int G, int slots,
                      double* ratio) {
  return guarded([&] {
    TokenDemand d = to_demand(D, N, G);
    Placement p = to_placement(cnt, N, G, slots);
    *ratio = balance_ratio(d, p, route(d, p));
  });
}

int ref_largest_remainder_round(const double* exact, int n, int64_t total, int64_t* out) {
  return guarded([&] {
    std::vector<int64_t> r = largest_remainder_round(std::span<const double>(exact, n), total);
    std::memcpy(out, r.data(), sizeof(int64_t) * r.size());
  });
}

int ref_generate_trace(int N, int G, int64_t tokens, double zipf, double drift, uint64_t seed,
                       int steps, int64_t* out) {
  return guarded([&] {
    TraceGeneratorConfig cfg;
    cfg.num_experts = N;
    cfg.num_gpus = G;
    cfg.tokens_per_step = tokens;
    cfg.zipf_exponent = zipf;
    cfg.drift_rate = drift;
    cfg.seed = seed;
    cfg.num_steps = steps;
    std::vector<TokenDemand> tr = generate_trace(cfg);
    for (int s = 0; s < steps; ++s)
      std::memcpy(out + static_cast<size_t>(s) * N * G, tr[s].demand.data(),
                  sizeof(int64_t) * N * G);
  });
}

// Trace file I/O through the reference's save_trace / load_trace.
int ref_save_trace(const char* path, const int64_t* trace, int steps, int N, int G) {
  return guarded([&] { save_trace(to_trace(trace, steps, N, G), path); });
}

// N = G = 0: load_trace(path) (inferred dimensions); dims = {steps, N, G};
// out (capacity cells, may be NULL) receives [steps][N][G].
int ref_load_trace(const char* path, int N, int G, int64_t* out, int64_t capacity, int32_t* dims) {
  return guarded([&] {
    std::vector<TokenDemand> tr = (N == 0 && G == 0) ? load_trace(path) : load_trace(path, N, G);
    dims[0] = static_cast<int32_t>(tr.size());
    dims[1] = tr.front().num_experts;
    dims[2] = tr.front().num_gpus;
    const size_t cells = static_cast<size_t>(dims[1]) * dims[2];
    if (!out || static_cast<int64_t>(cells * tr.size()) > capacity) return;
    for (size_t s = 0; s < tr.size(); ++s)
      std::memcpy(out + s * cells, tr[s].demand.data(), sizeof(int64_t) * cells);
  });
}

// ClusterTopology::from_file: ints {num_gpus, gpus_per_node, vexperts};
// dbl {intra_bw, inter_bw, tps, param_bytes, state_bytes, token_bytes};
// intra/inter bps by group size (65 entries each, 0 = absent).
int ref_topology_load(const char* path, int32_t* ints, double* dbl, double* intra, double* inter) {
  return guarded([&] {
    ClusterTopology t = ClusterTopology::from_file(path);
    ints[0] = t.num_gpus();
    ints[1] = t.gpus_per_node();
    ints[2] = t.vexperts_per_gpu();
    dbl[0] = t.intra_node_bandwidth();
    dbl[1] = t.inter_node_bandwidth();
    dbl[2] = t.tps();
    dbl[3] = t.expert_param_bytes();
    dbl[4] = t.expert_state_bytes();
    dbl[5] = t.token_bytes();
    for (int n = 0; n <= 64; ++n) intra[n] = inter[n] = 0;
    std::vector<GpuId> grp;
    for (int n = 2; n <= t.num_gpus() && n <= 64; ++n) {
      grp.clear();
      for (int g = 0; g < n; ++g) grp.push_back(g);
      if (!t.spans_nodes(grp)) intra[n] = t.group_bps(grp);
      std::vector<GpuId> wide;  // same size across nodes (first GPU of each node, then fill)
      if (t.num_gpus() > t.gpus_per_node()) {
        for (int g = 0; g < t.num_gpus() && static_cast<int>(wide.size()) < n; g += t.gpus_per_node())
          wide.push_back(g);
        for (int g = 0; g < t.num_gpus() && static_cast<int>(wide.size()) < n; ++g)
          if (std::find(wide.begin(), wide.end(), g) == wide.end()) wide.push_back(g);
        if (wide.size() == static_cast<size_t>(n) && t.spans_nodes(wide)) inter[n] = t.group_bps(wide);
      }
    }
  });
}

// StaticEP baseline through the reference's run_baseline: per-step dropped
// tokens and balance ratio (of the post-drop routing).
int ref_static_ep(const int64_t* trace, int steps, int N, int G, double cf, int64_t* dropped,
                  double* ratio) {
  return guarded([&] {
    std::vector<TokenDemand> tr = to_trace(trace, steps, N, G);
    ClusterTopology topo = ClusterTopology::from_json(
        ClusterTopology::default_profile(G, (N + G - 1) / G));
    BaselineConfig b;
    b.kind = BaselineKind::StaticEP;
    b.capacity_factor = cf;
    SimConfig sc;
    std::vector<StepReport> reps = run_baseline(tr, topo, b, sc);
    for (int s = 0; s < steps; ++s) {
      dropped[s] = reps[s].tokens_dropped;
      ratio[s] = reps[s].balance_ratio;
    }
  });
}

// Any baseline through run_baseline on the default profile (slots per GPU
// given): per-step ratio, metric, makespan, group misses, dropped,
// reassigned, slot utilization and replica counts [steps][N].
int ref_baseline_run(int kind, const int64_t* trace, int steps, int N, int G, int slots, double cf,
                     int replicate_top, int metric, double* ratio, double* metric_value,
                     double* makespan, int32_t* misses, int64_t* dropped, int64_t* reassigned,
                     double* util, int32_t* replicas) {
  return guarded([&] {
    std::vector<TokenDemand> tr = to_trace(trace, steps, N, G);
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    BaselineConfig b;
    b.kind = static_cast<BaselineKind>(kind);
    b.capacity_factor = cf;
    b.replicate_top = replicate_top;
    SimConfig sc;
    sc.metric = static_cast<BalanceMetric>(metric);
    std::vector<StepReport> reps = run_baseline(tr, topo, b, sc);
    for (int s = 0; s < steps; ++s) {
      ratio[s] = reps[s].balance_ratio;
      metric_value[s] = reps[s].metric_value;
      makespan[s] = reps[s].makespan_s;
      misses[s] = reps[s].group_cache_misses;
      dropped[s] = reps[s].tokens_dropped;
      reassigned[s] = reps[s].tokens_reassigned;
      util[s] = reps[s].slot_utilization;
      for (int e = 0; e < N; ++e) replicas[static_cast<size_t>(s) * N + e] = reps[s].replica_counts[e];
    }
  });
}

// The dynamic engine (SimEngine::run) on a trace with the default profile
// (slots per GPU given): per-step balance ratio, replica counts [steps][N],
// and totals of applied Expand / Shrink / Migrate ops.
int ref_engine_run(const int64_t* trace, int steps, int N, int G, int slots, int policy_mode,
                   int interval, double* ratio, int32_t* replicas, int64_t* op_totals) {
  return guarded([&] {
    std::vector<TokenDemand> tr = to_trace(trace, steps, N, G);
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    SimConfig sc;
    sc.policy_mode = static_cast<PolicyMode>(policy_mode);
    sc.interval_steps = interval;
    std::vector<StepReport> reps = run_simulation(tr, topo, sc);
    op_totals[0] = op_totals[1] = op_totals[2] = 0;
    for (int s = 0; s < steps; ++s) {
      ratio[s] = reps[s].balance_ratio;
      for (int e = 0; e < N; ++e) replicas[static_cast<size_t>(s) * N + e] = reps[s].replica_counts[e];
      for (const PlacementOp& op : reps[s].plan_applied) op_totals[static_cast<int>(op.kind)] += 1;
    }
  });
}

// One policy round on (D, placement): ops as [kind, expert, gpu, a.gpu, a.slot, b.gpu, b.slot].
int ref_make_scheduling_plan(const int64_t* D, const int32_t* cnt, int N, int G, int slots,
                             int horizon, int32_t* ops, int* n_ops, int max_ops) {
  return guarded([&] {
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    PolicyConfig pc;
    pc.amortization_horizon = horizon;
    SchedulingPlan plan =
        make_scheduling_plan(to_demand(D, N, G), to_placement(cnt, N, G, slots), topo, pc);
    int n = 0;
    for (const PlacementOp& op : plan.ops) {
      if (n >= max_ops) break;
      int32_t* o = ops + 7 * n;
      o[0] = static_cast<int>(op.kind);
      o[1] = op.expert;
      o[2] = op.gpu;
      o[3] = op.a.gpu;
      o[4] = op.a.slot;
      o[5] = op.b.gpu;
      o[6] = op.b.slot;
      ++n;
    }
    *n_ops = n;
  });
}

int ref_step_cost(const int64_t* D, const int32_t* cnt, int N, int G, int slots, double* makespan,
                  double* per_gpu) {
  return guarded([&] {
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    TokenDemand d = to_demand(D, N, G);
    Placement p = to_placement(cnt, N, G, slots);
    StepCostBreakdown b = step_cost(d, p, route(d, p), topo);
    *makespan = b.makespan_s;
    for (int g = 0; g < G; ++g) {
      per_gpu[3 * g] = b.per_gpu[g].compute_s;
      per_gpu[3 * g + 1] = b.per_gpu[g].a2a_s;
      per_gpu[3 * g + 2] = b.per_gpu[g].sync_s;
    }
  });
}

int ref_plan_migrations(const int32_t* cnt, int N, int G, int slots, int horizon, int32_t* ops,
                        int* n_ops) {
  return guarded([&] {
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    PolicyConfig pc;
    pc.amortization_horizon = horizon;
    SchedulingPlan plan = plan_migrations(to_placement(cnt, N, G, slots), topo, pc);
    int n = 0;
    for (const PlacementOp& op : plan.ops) {
      int32_t* o = ops + 7 * n++;
      o[0] = static_cast<int>(op.kind);
      o[1] = op.expert;
      o[2] = op.gpu;
      o[3] = op.a.gpu;
      o[4] = op.a.slot;
      o[5] = op.b.gpu;
      o[6] = op.b.slot;
    }
    *n_ops = n;
  });
}

// The engine with per-step detail: makespan, adjust bytes, accepted ops
// [kind, expert, gpu, a.gpu, a.slot, b.gpu, b.slot] (up to max_ops per step).
int ref_engine_detail(const int64_t* trace, int steps, int N, int G, int slots, int policy_mode,
                      int interval, int metric, double* makespan, double* adjust_bytes,
                      int32_t* n_ops, int32_t* ops, int max_ops) {
  return guarded([&] {
    std::vector<TokenDemand> tr = to_trace(trace, steps, N, G);
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    SimConfig sc;
    sc.policy_mode = static_cast<PolicyMode>(policy_mode);
    sc.interval_steps = interval;
    sc.metric = static_cast<BalanceMetric>(metric);
    std::vector<StepReport> reps = run_simulation(tr, topo, sc);
    for (int s = 0; s < steps; ++s) {
      makespan[s] = reps[s].makespan_s;
      adjust_bytes[s] = static_cast<double>(reps[s].adjust_bytes);
      int n = 0;
      for (const PlacementOp& op : reps[s].plan_applied) {
        if (n >= max_ops) break;
        int32_t* o = ops + (static_cast<size_t>(s) * max_ops + n) * 7;
        o[0] = static_cast<int>(op.kind);
        o[1] = op.expert;
        o[2] = op.gpu;
        o[3] = op.a.gpu;
        o[4] = op.a.slot;
        o[5] = op.b.gpu;
        o[6] = op.b.slot;
        ++n;
      }
      n_ops[s] = static_cast<int32_t>(reps[s].plan_applied.size());
    }
  });
}

// CPU-baseline timing of the reference's per-step count-level path:
// `iters` calls of route() + balance_ratio() on the same inputs; returns
// seconds per call.
int ref_time_route(const int64_t* D, const int32_t* cnt, int N, int G, int slots, int iters,
                   double* sec_per_call) {
  return guarded([&] {
    TokenDemand d = to_demand(D, N, G);
    Placement p = to_placement(cnt, N, G, slots);
    double sink = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) {
      RoutingPlan plan = route(d, p);
      sink += balance_ratio(d, p, plan);
    }
    auto t1 = std::chrono::steady_clock::now();
    *sec_per_call = std::chrono::duration<double>(t1 - t0).count() / iters + sink * 0.0;
  });
}

// seconds per call, one host thread, of the reference's
// count-level per-step path at one configuration — out[0] route() +
// balance_ratio(), out[1] step_cost(), out[2] make_scheduling_plan(),
// out[3] plan_migrations() (these four on trace step 0 and
// Placement::initial), out[4] one SimEngine step (run() over the whole
// `steps`-step trace with the given policy mode, divided by steps). Each
// figure repeats its call until `min_seconds` have elapsed.
int ref_time_count_path(const int64_t* trace, int steps, int N, int G, int slots, int policy_mode,
                        int interval, double min_seconds, double* out) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    std::vector<TokenDemand> tr = to_trace(trace, steps, N, G);
    ClusterTopology topo = ClusterTopology::from_json(ClusterTopology::default_profile(G, slots));
    const Placement p = Placement::initial(N, topo);
    const TokenDemand& d = tr[0];
    PolicyConfig pc;
    double sink = 0;
    auto per_call = [&](auto&& body) {
      int64_t n = 0;
      const auto t0 = clk::now();
      double el = 0;
      do {
        body();
        ++n;
        el = std::chrono::duration<double>(clk::now() - t0).count();
      } while (el < min_seconds);
      return el / static_cast<double>(n);
    };
    out[0] = per_call([&] {
      RoutingPlan plan = route(d, p);
      sink += balance_ratio(d, p, plan);
    });
    out[1] = per_call([&] { sink += step_cost(d, p, route(d, p), topo).makespan_s; });
    out[2] = per_call([&] { sink += static_cast<double>(make_scheduling_plan(d, p, topo, pc).ops.size()); });
    out[3] = per_call([&] { sink += static_cast<double>(plan_migrations(p, topo, pc).ops.size()); });
    SimConfig sc;
    sc.policy_mode = static_cast<PolicyMode>(policy_mode);
    sc.interval_steps = interval;
    out[4] = per_call([&] { sink += static_cast<double>(run_simulation(tr, topo, sc).size()); }) / steps;
    out[5] = sink * 0.0;
  });
}

}  // extern "C"
