// extern "C" surface of the host scheduler (declared in include/flexmoe_b200.h).
#include <cstring>
#include <memory>

#include "fm_internal.h"
#include "scheduler.h"

using namespace fm::sched;

namespace {

ClusterProfile to_profile(const fm_cluster_profile* c) {
  if (!c) throw std::invalid_argument("null cluster profile");
  if (c->num_gpus < 1 || c->num_gpus > FM_MAX_GROUP) throw std::invalid_argument("profile: bad num_gpus");
  if (c->gpus_per_node < 1 || c->num_gpus % c->gpus_per_node != 0)
    throw std::invalid_argument("topology config: num_gpus must be a positive multiple of gpus_per_node");
  ClusterProfile p;
  p.num_gpus = c->num_gpus;
  p.gpus_per_node = c->gpus_per_node;
  p.slots_per_gpu = c->slots_per_gpu;
  p.intra_bw = c->intra_node_bandwidth_bps;
  p.inter_bw = c->inter_node_bandwidth_bps;
  p.tps = c->tps;
  p.expert_param_bytes = c->expert_param_bytes;
  p.expert_state_bytes = c->expert_state_bytes;
  p.token_bytes = c->token_bytes;
  const int max_intra = std::min(p.gpus_per_node, p.num_gpus);
  p.bps_intra.assign(c->allreduce_bps_intra, c->allreduce_bps_intra + max_intra + 1);
  if (p.num_gpus > p.gpus_per_node)
    p.bps_inter.assign(c->allreduce_bps_inter, c->allreduce_bps_inter + p.num_gpus + 1);
  return p;
}

void from_profile(const ClusterProfile& p, fm_cluster_profile* c) {
  std::memset(c, 0, sizeof(*c));
  c->num_gpus = p.num_gpus;
  c->gpus_per_node = p.gpus_per_node;
  c->slots_per_gpu = p.slots_per_gpu;
  c->intra_node_bandwidth_bps = p.intra_bw;
  c->inter_node_bandwidth_bps = p.inter_bw;
  c->tps = p.tps;
  c->expert_param_bytes = p.expert_param_bytes;
  c->expert_state_bytes = p.expert_state_bytes;
  c->token_bytes = p.token_bytes;
  for (size_t i = 0; i < p.bps_intra.size() && i <= FM_MAX_GROUP; ++i) c->allreduce_bps_intra[i] = p.bps_intra[i];
  for (size_t i = 0; i < p.bps_inter.size() && i <= FM_MAX_GROUP; ++i) c->allreduce_bps_inter[i] = p.bps_inter[i];
}

fm_placement_op to_c(const Op& o) {
  return fm_placement_op{o.kind, o.expert, o.gpu, o.a_gpu, o.a_slot, o.b_gpu, o.b_slot};
}
Op from_c(const fm_placement_op& o) {
  return Op{o.kind, o.expert, o.gpu, o.a_gpu, o.a_slot, o.b_gpu, o.b_slot};
}

void copy_ops(const std::vector<Op>& ops, fm_placement_op* out, int max_ops, int* n) {
  if (static_cast<int>(ops.size()) > max_ops) throw std::invalid_argument("ops buffer too small");
  for (size_t i = 0; i < ops.size(); ++i) out[i] = to_c(ops[i]);
  *n = static_cast<int>(ops.size());
}

std::vector<int64_t> demand(const int64_t* D, int N, int G) {
  return std::vector<int64_t>(D, D + static_cast<size_t>(N) * G);
}

}  // namespace

struct fm_scheduler {
  std::unique_ptr<Scheduler> s;
  StepOutcome last;
};

namespace fm {
namespace sched {
ClusterProfile profile_from_c(const fm_cluster_profile* c) { return to_profile(c); }
}  // namespace sched
}  // namespace fm

extern "C" {

int fm_profile_reference_default(int num_gpus, int slots_per_gpu, fm_cluster_profile* out) {
  return fm::guarded([&] { from_profile(ClusterProfile::reference_default(num_gpus, slots_per_gpu), out); });
}

int fm_step_cost(const int64_t* D, const int32_t* slots_GE, int num_experts, const fm_cluster_profile* prof,
                 double* makespan, double* per_gpu_G3) {
  return fm::guarded([&] {
    const ClusterProfile p = to_profile(prof);
    const SlotPlacement pl = SlotPlacement::from_slots(slots_GE, p.num_gpus, p.slots_per_gpu, num_experts);
    const std::vector<int64_t> d = demand(D, num_experts, p.num_gpus);
    const StepTime st = step_time(d, pl, flows_for(d, pl), p);
    *makespan = st.makespan;
    if (per_gpu_G3)
      for (int g = 0; g < p.num_gpus; ++g) {
        per_gpu_G3[3 * g] = st.gpu[g].compute;
        per_gpu_G3[3 * g + 1] = st.gpu[g].a2a;
        per_gpu_G3[3 * g + 2] = st.gpu[g].sync;
      }
  });
}

int fm_make_scheduling_plan(const int64_t* D, const int32_t* slots_GE, int num_experts,
                            const fm_cluster_profile* prof, int horizon, fm_placement_op* ops,
                            int max_ops, int* n_ops) {
  return fm::guarded([&] {
    const ClusterProfile p = to_profile(prof);
    const SlotPlacement pl = SlotPlacement::from_slots(slots_GE, p.num_gpus, p.slots_per_gpu, num_experts);
    copy_ops(plan_balance(demand(D, num_experts, p.num_gpus), pl, p, horizon), ops, max_ops, n_ops);
  });
}

int fm_plan_migrations(const int32_t* slots_GE, int num_experts, const fm_cluster_profile* prof, int horizon,
                       fm_placement_op* ops, int max_ops, int* n_ops) {
  return fm::guarded([&] {
    const ClusterProfile p = to_profile(prof);
    const SlotPlacement pl = SlotPlacement::from_slots(slots_GE, p.num_gpus, p.slots_per_gpu, num_experts);
    copy_ops(plan_relocation(pl, p, horizon), ops, max_ops, n_ops);
  });
}

int fm_placement_apply(int32_t* slots_GE, int num_experts, const fm_cluster_profile* prof,
                       const fm_placement_op* op, double* transfers_2x3, int* n_transfers) {
  return fm::guarded([&] {
    const ClusterProfile p = to_profile(prof);
    SlotPlacement pl = SlotPlacement::from_slots(slots_GE, p.num_gpus, p.slots_per_gpu, num_experts);
    const std::vector<Transfer> t = pl.apply(from_c(*op), p);
    pl.validate();
    std::memcpy(slots_GE, pl.slot_table().data(), sizeof(int32_t) * pl.slot_table().size());
    if (n_transfers) *n_transfers = static_cast<int>(t.size());
    if (transfers_2x3)
      for (size_t i = 0; i < t.size(); ++i) {
        transfers_2x3[3 * i] = t[i].src;
        transfers_2x3[3 * i + 1] = t[i].dst;
        transfers_2x3[3 * i + 2] = t[i].bytes;
      }
  });
}

int fm_scheduler_create(const fm_cluster_profile* prof, const fm_scheduler_config* cfg, int num_experts,
                        fm_scheduler** out) {
  return fm::guarded([&] {
    SchedulerConfig c;
    c.threshold = cfg->threshold;
    c.metric = cfg->metric;
    c.policy_mode = cfg->policy_mode;
    c.interval_steps = cfg->interval_steps;
    c.horizon = cfg->amortization_horizon;
    c.adjust_bandwidth_fraction = cfg->adjust_bandwidth_fraction;
    c.max_live_groups = cfg->max_live_groups;
    c.group_creation_latency_s = cfg->group_creation_latency_s;
    if (cfg->flip_mode < 0 || cfg->flip_mode > 1) throw std::invalid_argument("scheduler: flip_mode must be 0 or 1");
    c.flip_mode = cfg->flip_mode;
    c.async_policy = cfg->async_policy ? 1 : 0;
    auto h = std::make_unique<fm_scheduler>();
    h->s = std::make_unique<Scheduler>(to_profile(prof), c, num_experts);
    *out = h.release();
  });
}

int fm_scheduler_destroy(fm_scheduler* h) {
  return fm::guarded([&] { delete h; });
}

int fm_scheduler_step(fm_scheduler* h, const int64_t* D, fm_step_report* out) {
  return fm::guarded([&] {
    const int N = h->s->effective().experts(), G = h->s->effective().gpus();
    h->last = h->s->step(demand(D, N, G));
    if (out) {
      out->balance_ratio = h->last.balance_ratio;
      out->metric_value = h->last.metric_value;
      out->makespan_s = h->last.makespan;
      out->adjust_s = h->last.adjust_seconds;
      out->adjust_bytes = h->last.adjust_bytes;
      out->group_misses = h->last.group_misses;
      out->n_accepted = static_cast<int>(h->last.accepted.size());
      out->n_applied = static_cast<int>(h->last.applied.size());
      out->n_issued = static_cast<int>(h->last.issued.size());
      out->pending_ops = static_cast<int>(h->s->queue().size());
    }
  });
}

int fm_scheduler_begin_step(fm_scheduler* h, fm_step_report* out) {
  return fm::guarded([&] {
    const StepOutcome& o = h->s->begin_step();
    h->last = o;
    if (out) {
      std::memset(out, 0, sizeof(*out));
      out->adjust_s = o.adjust_seconds;
      out->adjust_bytes = o.adjust_bytes;
      out->n_applied = static_cast<int>(o.applied.size());
      out->n_issued = static_cast<int>(o.issued.size());
      out->pending_ops = static_cast<int>(h->s->queue().size());
    }
  });
}

int fm_scheduler_finish_step(fm_scheduler* h, const int64_t* D, fm_step_report* out) {
  return fm::guarded([&] {
    const int N = h->s->effective().experts(), G = h->s->effective().gpus();
    h->last = h->s->finish_step(demand(D, N, G));
    if (out) {
      out->balance_ratio = h->last.balance_ratio;
      out->metric_value = h->last.metric_value;
      out->makespan_s = h->last.makespan;
      out->adjust_s = h->last.adjust_seconds;
      out->adjust_bytes = h->last.adjust_bytes;
      out->group_misses = h->last.group_misses;
      out->n_accepted = static_cast<int>(h->last.accepted.size());
      out->n_applied = static_cast<int>(h->last.applied.size());
      out->n_issued = static_cast<int>(h->last.issued.size());
      out->pending_ops = static_cast<int>(h->s->queue().size());
    }
  });
}

int fm_scheduler_ops(fm_scheduler* h, int which, fm_placement_op* ops, int max_ops, int* n_ops) {
  return fm::guarded([&] {
    if (which < 0 || which > 2) throw std::invalid_argument("fm_scheduler_ops: which must be 0, 1 or 2");
    copy_ops(which == 0 ? h->last.accepted : which == 1 ? h->last.applied : h->last.issued, ops, max_ops, n_ops);
  });
}

int fm_scheduler_placement(fm_scheduler* h, int which, int32_t* slots_GE, int32_t* counts_NG) {
  return fm::guarded([&] {
    const SlotPlacement& p = which == 0 ? h->s->effective() : h->s->target();
    if (slots_GE) std::memcpy(slots_GE, p.slot_table().data(), sizeof(int32_t) * p.slot_table().size());
    if (counts_NG) std::memcpy(counts_NG, p.counts().data(), sizeof(int32_t) * p.counts().size());
  });
}

int fm_scheduler_join_policy(fm_scheduler* h, int* n_committed) {
  return fm::guarded([&] {
    const std::vector<Op> ops = h->s->join_policy();
    h->last.accepted.insert(h->last.accepted.end(), ops.begin(), ops.end());
    if (n_committed) *n_committed = static_cast<int>(ops.size());
  });
}

int fm_scheduler_reset(fm_scheduler* h, const int32_t* slots_GE) {
  return fm::guarded([&] {
    const SlotPlacement& cur = h->s->effective();
    h->s->reset(SlotPlacement::from_slots(slots_GE, cur.gpus(), cur.slots(), cur.experts()));
  });
}

}  // extern "C"
