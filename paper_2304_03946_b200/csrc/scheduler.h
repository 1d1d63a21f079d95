// Host-side placement scheduler: the consumer of the device histogram.
//
// Behavioural sources (paths relative to /root/reference/proj):
//   ClusterProfile   src/topology.cpp:140-220   (bandwidth, ring all-reduce table)
//   SlotPlacement    src/placement.cpp:52-246   (vExpert pool, expand/shrink/migrate)
//   cost model       src/cost_model.cpp:30-111  (Eqs. 5, 8-10)
//   plan_balance     src/policy.cpp:64-354      (Alg. 2 + candidate generators)
//   plan_relocation  src/policy.cpp:356-427     (replica-locality migrate pass)
//   TransferQueue    src/sim_engine.cpp:124-262 (merge + best-effort drain)
//   Scheduler::step  src/sim_engine.cpp:329-449 (Alg. 1 step driver)
// Counts come from the same route() as the device path (routing.cuh), so
// every decision is taken on bit-identical flows.
#pragma once

#include <cstdint>
#include <deque>
#include <list>
#include <map>
#include <optional>
#include <thread>
#include <vector>

namespace fm {
namespace sched {

struct ClusterProfile {
  int num_gpus = 1;
  int gpus_per_node = 1;
  int slots_per_gpu = 1;
  double intra_bw = 300e9;
  double inter_bw = 25e9;
  double tps = 1e6;
  double expert_param_bytes = 50e6;
  double expert_state_bytes = 150e6;
  double token_bytes = 4096.0;
  std::vector<double> bps_intra;  // indexed by group size
  std::vector<double> bps_inter;

  // The reference's A100-like default (topology.cpp:140-184).
  static ClusterProfile reference_default(int num_gpus, int slots_per_gpu);
  double bandwidth(int a, int b) const;
  bool spans_nodes(const std::vector<int>& group) const;
  double group_bps(const std::vector<int>& group) const;
};

struct Transfer {
  int src = -1;
  int dst = -1;
  double bytes = 0;
};

enum OpKind { kExpand = 0, kShrink = 1, kMigrate = 2 };
struct Op {
  int kind = kExpand;
  int expert = -1;  // Expand / Shrink
  int gpu = -1;
  int a_gpu = -1, a_slot = -1, b_gpu = -1, b_slot = -1;  // Migrate
};

// vExpert slot table: slot(g, s) = expert or -1; same-GPU slots of one expert
// share weights (count once for sync, add for capacity).
class SlotPlacement {
 public:
  SlotPlacement(int num_gpus, int slots_per_gpu, int num_experts);
  static SlotPlacement round_robin(int num_experts, int num_gpus, int slots_per_gpu);
  static SlotPlacement from_counts(const std::vector<int>& counts, int num_experts, int num_gpus,
                                   int slots_per_gpu);
  static SlotPlacement from_slots(const int32_t* slots_GE, int num_gpus, int slots_per_gpu,
                                  int num_experts);

  int gpus() const { return G_; }
  int slots() const { return E_; }
  int experts() const { return N_; }
  int slot(int g, int s) const { return slot_[g * E_ + s]; }
  int replicas(int e) const { return total_[e]; }
  int replicas_on(int e, int g) const { return count_[e * G_ + g]; }
  std::vector<int> hosts(int e) const;
  int free_slots(int g) const;
  int first_free(int g) const;
  double utilization() const;
  const std::vector<int>& counts() const { return count_; }
  const std::vector<int>& slot_table() const { return slot_; }

  std::optional<Transfer> expand(int e, int g, const ClusterProfile& prof);
  void shrink(int e, int g);
  std::vector<Transfer> migrate(int ag, int as, int bg, int bs, const ClusterProfile& prof);
  std::vector<Transfer> apply(const Op& op, const ClusterProfile& prof);
  void validate() const;
  bool operator==(const SlotPlacement& o) const {
    return slot_ == o.slot_ && count_ == o.count_ && total_ == o.total_;
  }

 private:
  int G_, E_, N_;
  int assigned_ = 0;
  std::vector<int> slot_;   // [G][E]
  std::vector<int> count_;  // [N][G]
  std::vector<int> total_;  // [N]
};

struct GpuTime {
  double compute = 0, a2a = 0, sync = 0;
  double total() const { return compute + a2a + sync; }
};
struct StepTime {
  std::vector<GpuTime> gpu;
  double makespan = 0;
  void refresh();
};

// flows[e][src][dst] for demand D[e][g] on a placement (routing.cuh).
std::vector<int64_t> flows_for(const std::vector<int64_t>& D, const SlotPlacement& p);
StepTime step_time(const std::vector<int64_t>& D, const SlotPlacement& p,
                   const std::vector<int64_t>& flows, const ClusterProfile& prof);
double sync_seconds(const std::vector<int>& group, const ClusterProfile& prof);
double transfer_seconds(const Transfer& t, const ClusterProfile& prof);
double balance_of(const std::vector<int64_t>& flows, int N, int G);
double variance_of(const std::vector<int64_t>& flows, int N, int G);

std::vector<Op> plan_balance(const std::vector<int64_t>& D, const SlotPlacement& p,
                             const ClusterProfile& prof, int horizon);
std::vector<Op> plan_relocation(const SlotPlacement& p, const ClusterProfile& prof, int horizon);

// FIFO of accepted ops and their state transfers (best-effort adjustment).
class TransferQueue {
 public:
  struct Pending {
    Op op;
    std::vector<Transfer> left;  // bytes = bytes remaining
    bool done() const;
  };
  struct Merged {
    int src, dst;
    double bytes;
    std::vector<std::pair<size_t, size_t>> parts;
  };
  void push(const Op& op, const std::vector<Transfer>& t);
  // Same-(src,dst) consecutive transfers coalesce; consecutive coalesced
  // messages with pairwise-disjoint endpoints form one concurrent set.
  std::vector<std::vector<Merged>> schedule() const;
  // Drains within `seconds`; completed ops (in order) are applied to
  // `effective` and returned. bytes_moved / seconds_used out.
  std::vector<Op> drain(double seconds, const ClusterProfile& prof, SlotPlacement& effective,
                        double& bytes_moved, double& seconds_used);
  size_t size() const { return q_.size(); }
  void pop_front() { q_.pop_front(); }
  double pending_bytes() const;
  const std::deque<Pending>& pending() const { return q_; }

 private:
  std::deque<Pending> q_;
};

class GroupLru {
 public:
  explicit GroupLru(int capacity) : cap_(capacity) {}
  bool touch(const std::vector<int>& group);  // true on hit
  int misses() const { return misses_; }

 private:
  int cap_;
  int misses_ = 0;
  std::list<std::vector<int>> order_;
  std::map<std::vector<int>, std::list<std::vector<int>>::iterator> where_;
};

struct SchedulerConfig {
  double threshold = 1.1;
  int metric = 0;       // 0 max ratio, 1 variance
  int policy_mode = 0;  // 0 dynamic, 1 fixed interval, 2 static
  int interval_steps = 10;
  int horizon = 50;
  double adjust_bandwidth_fraction = 0.5;
  int max_live_groups = 64;
  double group_creation_latency_s = 0.005;
  // 0 (reference): an op becomes effective once its modelled bytes drain
  //   within adjust_bandwidth_fraction x the previous makespan
  //   (sim_engine.cpp:331-336, :208-262).
  // 1 (device): begin_step makes the ops issued at the previous boundary
  //   effective — their state copies ran during that step and completed
  //   before its replica-group all-reduce (stream-ordered, no host sync) —
  //   and issues the next queue prefix whose modelled transfer time fits the
  //   same budget (at least one op).
  int flip_mode = 0;
  // 1: the policy half of finish_step (trigger loop + migration pass) runs on
  //   a worker thread over a snapshot of the target placement; its ops enter
  //   the queue at the next finish_step (one step later than the reference).
  int async_policy = 0;
};

struct StepOutcome {
  double balance_ratio = 1.0;
  double metric_value = 0;
  double makespan = 0;
  double adjust_seconds = 0;
  double adjust_bytes = 0;
  int group_misses = 0;
  std::vector<Op> accepted;  // entered the queue this step (target placement)
  std::vector<Op> applied;   // became effective this step
  std::vector<Op> issued;    // flip_mode 1: state copies start this step (effective next step)
};

class Scheduler {
 public:
  Scheduler(const ClusterProfile& prof, const SchedulerConfig& cfg, int num_experts);
  ~Scheduler();
  Scheduler(const Scheduler&) = delete;
  Scheduler& operator=(const Scheduler&) = delete;
  StepOutcome step(const std::vector<int64_t>& D);
  // step() in two halves: the drain (ops that become effective at the step
  // boundary, before the device routes) and the rest, once the step's
  // demand is known.
  const StepOutcome& begin_step();
  StepOutcome finish_step(const std::vector<int64_t>& D);
  const SlotPlacement& effective() const { return effective_; }
  const SlotPlacement& target() const { return target_; }
  const TransferQueue& queue() const { return queue_; }
  // flip_mode 1: the ops whose copies are in flight (a queue prefix)
  const std::vector<Op>& inflight() const { return inflight_; }
  void reset(const SlotPlacement& p);
  // async_policy: wait for the worker and enqueue its ops (also done by the
  // next finish_step, reset and the destructor)
  std::vector<Op> join_policy();

 private:
  double trigger(const std::vector<int64_t>& flows, int N) const;
  // steps 3-4 of run_step on `target` (no side effects on the scheduler)
  std::vector<Op> run_policy(const std::vector<int64_t>& D, SlotPlacement target, bool policy_step,
                             bool triggered) const;
  void commit(const std::vector<Op>& ops);
  ClusterProfile prof_;
  SchedulerConfig cfg_;
  SlotPlacement effective_, target_;
  TransferQueue queue_;
  GroupLru lru_;
  double prev_makespan_ = 0;
  int step_ = 0;
  StepOutcome cur_;
  bool begun_ = false;
  std::vector<Op> inflight_;
  std::thread worker_;
  std::vector<Op> worker_ops_;
};

}  // namespace sched
}  // namespace fm
