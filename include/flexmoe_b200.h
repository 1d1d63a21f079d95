/*
 * flexmoe_b200.h — C ABI of the B200-native FlexMoE MoE-layer hot path.
 *
 * Drop-in boundary for the reference `moesim` library (C++20, /root/reference/proj).
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference). Plain pointers and sizes only; no C++ or
 * torch types cross this boundary. Buffers are caller-owned unless stated.
 *
 * Error convention (reference: C++ exceptions): every function
 * returns an int status. The message of the last failure on the calling
 * thread is available from fm_last_error(); it carries the reference's text
 * where the reference has one (e.g. "route: expert 3 has demand but no replica").
 *
 * Device entry points take a `void* stream` (a cudaStream_t; NULL = legacy
 * default stream) and never synchronise the host unless documented.
 */
#ifndef FLEXMOE_B200_H_
#define FLEXMOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exception classes. */
#define FM_OK 0
#define FM_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument (e.g. router.cpp:58-63, :76-77) */
#define FM_ERR_LOGIC 2            /* std::logic_error (router.cpp:163, placement.cpp:258-277) */
#define FM_ERR_RUNTIME 3          /* std::runtime_error */
#define FM_ERR_OUT_OF_RANGE 4     /* std::out_of_range (workload.cpp:68, topology.cpp:188) */
#define FM_ERR_CUDA 5             /* CUDA / NCCL failure (no reference equivalent) */

const char* fm_last_error(void);
const char* fm_version(void);
/* Diagnostics: kernels this library has launched in this process (all
 * devices, all threads); bench.py reports the count over its timed region. */
unsigned long long fm_kernel_launches(void);

/* ------------------------------------------------------------------------
 * Count-level routing (host). Layouts follow the reference value types:
 *   demand_NG          TokenDemand.demand, row-major [expert][gpu] int64
 *                      (proj/include/moesim/workload.hpp:29-49)
 *   replica_counts_NG  Placement::replica_count_on(e, g), [expert][gpu] int32
 *                      (proj/include/moesim/placement.hpp:80-82)
 *   flows_NGG          RoutingPlan.flows, [expert][src][dst] int64
 *                      (proj/include/moesim/router.hpp:29-48)
 * ---------------------------------------------------------------------- */

/* Replaces `RoutingPlan route(const TokenDemand&, const Placement&)`
 * (proj/include/moesim/router.hpp:62, impl proj/src/router.cpp:57-169).
 * Bit-identical flows. FM_ERR_INVALID_ARGUMENT when an expert has demand
 * but no replica; FM_ERR_LOGIC on a conservation failure. */
int fm_route_counts(const int64_t* demand_NG, const int32_t* replica_counts_NG, int num_experts,
                    int num_gpus, int64_t* flows_NGG);

/* Device port of the same algorithm, one thread per expert; all pointers are
 * device memory. status_dev (int32[1]) receives 0 or an FM_ERR_* code
 * asynchronously (it is never read back by the library). */
int fm_route_counts_device(const int64_t* demand_NG, const int32_t* replica_counts_NG,
                           int num_experts, int num_gpus, int64_t* flows_NGG, int32_t* status_dev,
                           void* stream);

/* Replaces `received_matrix` (router.hpp:51 / router.cpp:33-43): recv[e][g]. */
int fm_received_matrix(const int64_t* flows_NGG, int num_experts, int num_gpus,
                       int64_t* recv_NG);

/* Replaces `per_gpu_received` (router.hpp:54 / router.cpp:45-55). */
int fm_per_gpu_received(const int64_t* flows_NGG, int num_experts, int num_gpus,
                        int64_t* totals_G);

/* Replaces `balance_ratio` (proj/include/moesim/policy.hpp:38 / policy.cpp:32-46),
 * Eq. 7: max_g recv_g / mean_g recv_g. FM_ERR_INVALID_ARGUMENT on zero tokens. */
int fm_balance_ratio(const int64_t* flows_NGG, int num_experts, int num_gpus, double* ratio);

/* Replaces `largest_remainder_round` (proj/include/moesim/workload.hpp:90,
 * workload.cpp:77-114). */
int fm_largest_remainder_round(const double* exact, int n, int64_t total, int64_t* out);

/* The StaticEP capacity-drop rule (proj/src/baselines.cpp:89-122), the only
 * token-drop path of the reference: cap = floor(cf * sum(D) / N); experts over
 * cap keep largest_remainder_round(D[e][g]*cap/load, cap) per source, clamped
 * to D[e][g]. cf = +inf disables drops. */
int fm_static_ep_kept(const int64_t* demand_NG, int num_experts, int num_gpus,
                      double capacity_factor, int64_t* kept_NG, int64_t* dropped);

/* Device port of the same rule, one thread per expert (explicit
 * round-to-nearest double ops in the reference's order: bit-identical to the
 * host). Device pointers; dropped (int64[1]) receives the total drop count. */
int fm_static_ep_kept_device(const int64_t* demand_NG, int num_experts, int num_gpus,
                             double capacity_factor, int64_t* kept_NG, int64_t* dropped,
                             void* stream);

/* ------------------------------------------------------------------------
 * Host placement scheduler — the consumer of the device histogram.
 * Placements cross the ABI as the vExpert slot table slots_GE[g][s] = expert
 * id or -1 (Placement::slot, placement.hpp:77), so slot-level ops are exact.
 * ---------------------------------------------------------------------- */
#define FM_MAX_GROUP 64
/* ClusterTopology (proj/include/moesim/topology.hpp:27-94); all-reduce tables
 * indexed by group size (entries below 2 unused). */
typedef struct fm_cluster_profile {
  int num_gpus;
  int gpus_per_node;
  int slots_per_gpu; /* vexperts_per_gpu */
  double intra_node_bandwidth_bps;
  double inter_node_bandwidth_bps;
  double tps; /* tokens/s of one expert's fwd+bwd */
  double expert_param_bytes;
  double expert_state_bytes;
  double token_bytes;
  double allreduce_bps_intra[FM_MAX_GROUP + 1];
  double allreduce_bps_inter[FM_MAX_GROUP + 1];
} fm_cluster_profile;

/* PlacementOp (placement.hpp:44-50): kind 0 Expand, 1 Shrink, 2 Migrate. */
typedef struct fm_placement_op {
  int kind;
  int expert;
  int gpu;
  int a_gpu, a_slot, b_gpu, b_slot;
} fm_placement_op;

/* ClusterTopology::default_profile (topology.cpp:140-184). */
int fm_profile_reference_default(int num_gpus, int slots_per_gpu, fm_cluster_profile* out);
/* step_cost (cost_model.hpp:67 / cost_model.cpp:78-111): makespan and per-GPU
 * {compute, a2a, sync} seconds of routing D on the placement. */
int fm_step_cost(const int64_t* demand_NG, const int32_t* slots_GE, int num_experts,
                 const fm_cluster_profile* profile, double* makespan, double* per_gpu_G3);
/* make_scheduling_plan (policy.hpp:57 / policy.cpp:64-354). */
int fm_make_scheduling_plan(const int64_t* demand_NG, const int32_t* slots_GE, int num_experts,
                            const fm_cluster_profile* profile, int amortization_horizon,
                            fm_placement_op* ops, int max_ops, int* n_ops);
/* plan_migrations (policy.hpp:65 / policy.cpp:356-427). */
int fm_plan_migrations(const int32_t* slots_GE, int num_experts, const fm_cluster_profile* profile,
                       int amortization_horizon, fm_placement_op* ops, int max_ops, int* n_ops);
/* Placement::apply (placement.hpp:104) on a slot table, in place; the implied
 * TransferDescriptors (placement.hpp:31-35) as rows {src, dst, bytes}. */
int fm_placement_apply(int32_t* slots_GE, int num_experts, const fm_cluster_profile* profile,
                       const fm_placement_op* op, double* transfers_2x3, int* n_transfers);

/* SimConfig (sim_engine.hpp:35-49). metric 0 MaxRatio / 1 Variance;
 * policy_mode 0 Dynamic / 1 FixedInterval / 2 Static. */
typedef struct fm_scheduler_config {
  double threshold;
  int metric;
  int policy_mode;
  int interval_steps;
  int amortization_horizon;
  double adjust_bandwidth_fraction;
  int max_live_groups;
  double group_creation_latency_s;
  /* B200 runtime extensions (0/0 = the reference's behaviour):
   * flip_mode 0: ops become effective when their MODELLED bytes drain within
   *   adjust_bandwidth_fraction x the previous makespan (sim_engine.cpp:331-336);
   * flip_mode 1: ops become effective when their REAL state copies complete —
   *   begin_step issues the next queue prefix that fits the same budget (at
   *   least one op; fm_scheduler_ops which=2); the runtime copies their state
   *   during that step (the receivers join the replica groups with zero
   *   tokens and wait for the copy before the group all-reduce), and the
   *   next begin_step makes them effective. No host sync anywhere.
   * async_policy 1: the policy half of finish_step runs on a worker thread
   *   over a snapshot of the target placement; its ops enter the queue at the
   *   next finish_step (or fm_scheduler_join_policy), one step later than
   *   the reference. */
  int flip_mode;
  int async_policy;
} fm_scheduler_config;

typedef struct fm_step_report {
  double balance_ratio;
  double metric_value;
  double makespan_s; /* modelled, effective placement */
  double adjust_s;
  double adjust_bytes;
  int group_misses;
  int n_accepted; /* ops accepted into the adjustment queue (target placement) */
  int n_applied;  /* ops that became effective at the start of this step */
  int pending_ops;
  int n_issued; /* flip_mode 1: ops whose state copies start this step */
} fm_step_report;

typedef struct fm_scheduler fm_scheduler;
/* The Alg. 1 step driver (SimEngine::run_step, sim_engine.cpp:329-449):
 * best-effort drain of the adjustment queue, route on the effective
 * placement, trigger, policy loop on the target placement, one migration. */
int fm_scheduler_create(const fm_cluster_profile* profile, const fm_scheduler_config* cfg,
                        int num_experts, fm_scheduler** out);
int fm_scheduler_destroy(fm_scheduler* s);
int fm_scheduler_step(fm_scheduler* s, const int64_t* demand_NG, fm_step_report* out);
/* The same step in two halves, for a runtime that routes on the device in
 * between: begin = best-effort drain (ops whose transfers completed become
 * effective; switch the layer's placement before routing), finish = the rest
 * on the step's demand. begin + finish == step. */
int fm_scheduler_begin_step(fm_scheduler* s, fm_step_report* out);
int fm_scheduler_finish_step(fm_scheduler* s, const int64_t* demand_NG, fm_step_report* out);
/* which: 0 = ops accepted this step, 1 = ops applied (made effective) this
 * step, 2 = ops issued this step (flip_mode 1) */
int fm_scheduler_ops(fm_scheduler* s, int which, fm_placement_op* ops, int max_ops, int* n_ops);
/* which: 0 = effective placement, 1 = target placement */
int fm_scheduler_placement(fm_scheduler* s, int which, int32_t* slots_GE, int32_t* counts_NG);
int fm_scheduler_reset(fm_scheduler* s, const int32_t* slots_GE);
/* async_policy: wait for the policy worker and enqueue its ops now (they are
 * appended to the ops reported as accepted). */
int fm_scheduler_join_policy(fm_scheduler* s, int* n_committed);

/* ------------------------------------------------------------------------
 * Comparison baselines, one step at a time:
 * replaces `run_baseline(trace, topo, BaselineConfig, SimConfig)`
 * (proj/include/moesim/baselines.hpp, impl proj/src/baselines.cpp:81-276).
 *   FM_BASELINE_STATIC_EP         round-robin placement, capacity drops
 *   FM_BASELINE_FULL_REPLICATE    hottest `replicate_top` experts shadowed on
 *                                 every GPU, re-derived from each step's demand
 *   FM_BASELINE_STRICT_REBALANCE  loads rewritten to B/G per GPU (count level)
 * Each step returns the reference's StepReport fields, the placement it ran
 * on (FullReplicate runs for real on the device runtime with it), the routed
 * demand (post-drop / rebalanced) and its flows.
 * ---------------------------------------------------------------------- */
#define FM_BASELINE_STATIC_EP 0
#define FM_BASELINE_FULL_REPLICATE 1
#define FM_BASELINE_STRICT_REBALANCE 2

typedef struct fm_baseline_config {
  int kind;
  double capacity_factor; /* StaticEP; +inf = unlimited */
  int replicate_top;      /* FullReplicate */
  int metric;             /* 0 max ratio, 1 variance */
  int max_live_groups;
  double group_creation_latency_s;
} fm_baseline_config;

typedef struct fm_baseline_report {
  double balance_ratio; /* baselines.cpp:31-40: max*G/sum, 1.0 when empty */
  double metric_value;
  double makespan_s;
  double slot_utilization;
  int group_misses;
  int64_t tokens_total; /* pre-drop */
  int64_t tokens_dropped;
  int64_t tokens_reassigned;
} fm_baseline_report;

typedef struct fm_baseline fm_baseline;
int fm_baseline_create(const fm_cluster_profile* profile, const fm_baseline_config* cfg, int num_experts,
                       fm_baseline** out);
int fm_baseline_destroy(fm_baseline* b);
/* Any of counts_NG (int32 [N][G]), routed_demand_NG (int64 [N][G]) and
 * flows_NGG (int64 [N][G][G]) may be NULL. */
int fm_baseline_step(fm_baseline* b, const int64_t* demand_NG, fm_baseline_report* out, int32_t* counts_NG,
                     int64_t* routed_demand_NG, int64_t* flows_NGG);
/* The placement of the last step (slots_GE int32 [G][slots]). */
int fm_baseline_placement(fm_baseline* b, int32_t* slots_GE, int32_t* counts_NG, int* slots_per_gpu);

/* ------------------------------------------------------------------------
 * Trace export / replay. The reference's TokenDemand
 * trace file "step,expert,gpu,tokens" (one line per non-zero cell, sorted by
 * (step, expert, gpu)); device gate histograms recorded here replay in the
 * reference engine/CLI and reference traces drive this framework.
 * demand_SNG: [step][expert][gpu] int64, host memory.
 * ---------------------------------------------------------------------- */

/* Replaces `save_trace(std::span<const TokenDemand>, const std::string&)`
 * (proj/include/moesim/workload.hpp:79, impl proj/src/workload.cpp:175-192).
 * step_ids: the TokenDemand.step of each entry (NULL = 0, 1, ...). */
int fm_trace_save(const char* path, const int64_t* demand_SNG, const int32_t* step_ids, int num_steps,
                  int num_experts, int num_gpus);
/* Replaces `load_trace(path)` / `load_trace(path, num_experts, num_gpus)`
 * (workload.hpp:82-86, workload.cpp:194-341): num_experts = num_gpus = 0 infers
 * the dimensions from the largest ids. Call with demand_SNG = NULL to get the
 * sizes, then with a buffer of `capacity` >= steps*N*G cells. Malformed files:
 * FM_ERR_RUNTIME with the reference's "<path>:<line>: <what>" messages. */
int fm_trace_load(const char* path, int num_experts, int num_gpus, int64_t* demand_SNG, int64_t capacity,
                  int* num_steps, int* num_experts_out, int* num_gpus_out);

/* ------------------------------------------------------------------------
 * Grouped expert GEMM on tcgen05 (test / building-block hook).
 * seg_start, seg_rows, tile_prefix are device int32 arrays describing the
 * per-group token segments of the permuted buffers (rows multiple of 128).
 * ---------------------------------------------------------------------- */
#define FM_GEMM_FWD_BIAS_RELU 0   /* C[rows,N] = relu(A[rows,K] W_g[N,K]^T + b_g)   bf16;
                                     aux (optional) <- ReLU bits uint32 [rows][N/32], bit i of
                                     word j = (pre-activation of column 32j+i > 0) */
#define FM_GEMM_FWD_BIAS 1        /* C[rows,N] = A W_g^T + b_g                       bf16 */
#define FM_GEMM_DGRAD_RELU_MASK 2 /* C[rows,N] = (A[rows,K] W_g[K,N]) * bit(aux)     bf16;
                                     aux = the ReLU bits written by FWD_BIAS_RELU; `bias`,
                                     if non-null, receives f32 column sums of C per 128-row
                                     tile [total_rows/128][N] (bias gradient partials) */
#define FM_GEMM_DGRAD 3           /* C[rows,N] = A[rows,K] W_g[K,N]                  bf16 */
#define FM_GEMM_WGRAD 4           /* C[g][M_w,N] = A[seg_g, M_w]^T B[seg_g, N]       f32  */

/* Tile shape of the grouped GEMM: 1 = 128x256 per CTA, 2 = CTA pairs
 * (tcgen05 cta_group::2, 256x256 per pair), 0 = automatic (default). */
int fm_set_gemm_cta_group(int cta_group);

int fm_grouped_gemm(int variant, const void* A, const void* B, void* C, const float* bias,
                    const void* aux, const int32_t* seg_start, const int32_t* seg_rows,
                    const int32_t* tile_prefix, int num_groups, int total_rows, int M_w, int N,
                    int K, void* stream);

/* ------------------------------------------------------------------------
 * The MoE layer (one process per GPU).
 *
 * The reference has no layer: gate, expert FFN and combine are cost terms
 * (compute_cost / a2a_cost, proj/src/cost_model.cpp:30-51) and token identity
 * is not tracked. This is the executing replacement of the
 * per-step `route(d, effective)` call in SimEngine::run_step
 * (proj/src/sim_engine.cpp:342): the demand it routes is the device
 * histogram of the real gate, and the flows it produces drive the real
 * dispatch. Math: PAPER.md:206-229 (Eqs. 2-4), ReLU FFN, softmax over the
 * top-k kept logits, ties to the lower expert id.
 *
 * dtypes: x / y / dy / dx and all weights bf16; biases f32; weight gradients
 * f32 (dw1 [Nl,f,d], dw2 [Nl,d,f], db1 [Nl,f], db2 [Nl,d], dwg [N,d]).
 * Expert weights are packed for the Nl local experts in ascending expert id
 * (fm_layer_local_experts): w1 [Nl,f,d], w2 [Nl,d,f], b1 [Nl,f], b2 [Nl,d];
 * the gate weight wg is [N,d]. d % 256 == 0, f % 256 == 0, N <= 256, k <= 8.
 * ---------------------------------------------------------------------- */
typedef struct fm_layer_config {
  int num_experts;   /* N */
  int top_k;         /* k */
  int d_model;       /* d */
  int d_ff;          /* f */
  int num_gpus;      /* G */
  int rank;          /* this GPU's id in [0, G) */
  int max_tokens;    /* T capacity per call on this GPU */
  int slots_per_gpu; /* vExpert slots E (placement validation); 0 = unchecked */
} fm_layer_config;

typedef struct fm_layer fm_layer;

/* replica_counts_NG as Placement::replica_count_on (placement.hpp:80-82). */
int fm_layer_create(const fm_layer_config* cfg, const int32_t* replica_counts_NG, fm_layer** out);
int fm_layer_destroy(fm_layer* layer);
/* Placement change (Expand / Shrink / Migrate applied, placement.hpp:92-104).
 * Synchronous: returns once the device tables are updated. */
int fm_layer_set_placement(fm_layer* layer, const int32_t* replica_counts_NG);
/* The same switch enqueued on `stream`: no allocation, no host sync (one
 * cudaMemcpyAsync from a pinned staging ring, ordered after every kernel
 * already enqueued on the stream). hosted_N (optional, [N], nonzero = yes):
 * experts whose state this rank keeps with replica count 0 — a replica whose
 * state copy is in flight (fm_scheduler flip_mode 1). They are local experts
 * (gradient slices in ascending-id local order, replica-group members) with
 * no token rows routed to them; their weight gradients are zero. */
int fm_layer_set_placement_async(fm_layer* layer, const int32_t* replica_counts_NG, const int32_t* hosted_N,
                                 void* stream);
/* Expert-operand addressing. slot_N[e] = row of expert e inside the w1 / b1 /
 * w2 / b2 operands passed to the expert phases (w1 [capacity, f, d] ...), for
 * every local expert; entries of other experts are ignored. With it the
 * operands stay where the expert-state pool keeps them (fm_pool_set_operand_
 * layout) and a placement switch moves no weights. slot_N == NULL restores
 * the packed layout (local experts ascending, row i = i-th local expert).
 * Enqueued on `stream` like fm_layer_set_placement_async. */
int fm_layer_set_operand_slots(fm_layer* layer, const int32_t* slot_N, int capacity, void* stream);
/* StaticEP mode (proj/src/baselines.cpp:81-131): capacity_factor > 0 and finite
 * drops, each step, the units beyond fm_static_ep_kept's kept[e][g] on every
 * source GPU — the LAST ones in the canonical unit order — before routing;
 * dropped units contribute nothing to y (their gate gradient is kept).
 * 0 or +inf disables drops (the FlexMoE mode, which never drops). */
int fm_layer_set_capacity_factor(fm_layer* layer, double capacity_factor);
int fm_layer_local_experts(const fm_layer* layer, int* num_local, int32_t* experts_out);
/* Which memory-bound backward work of the last backward ran on spare CTA pairs
 * of a weight-gradient GEMM launch instead of its own kernel:
 * bit 0 the db2 / dWg tile column sums (FFN2 wgrad), bit 1 the un-permute
 * (FFN1 wgrad), bit 2 the per-expert reduce of the bias / gate-weight
 * gradient partials (FFN1 wgrad). Results are the same either way. */
int fm_layer_side_jobs(const fm_layer* layer, int* mask);
/* enable = 0: run that work as standalone kernels (default 1). */
int fm_layer_set_side_jobs(fm_layer* layer, int enable);

/* Single-GPU (num_gpus == 1) fused step; no host synchronisation.
 * forward keeps what backward needs (routing, permuted activations); x and
 * the weights must stay valid until fm_layer_backward has been enqueued. */
int fm_layer_forward(fm_layer* layer, const void* x, int num_tokens, const void* wg,
                     const void* w1, const float* b1, const void* w2, const float* b2, void* y,
                     void* stream);
int fm_layer_backward(fm_layer* layer, const void* dy, void* dx, float* dwg, float* dw1,
                      float* db1, float* dw2, float* db2, void* stream);

/* Phase API (any num_gpus; one process per GPU). The host runs the
 * collectives between phases:
 *   fm_layer_gate        -> hist_out: this GPU's TokenDemand column, int64 [N] (device)
 *   host: all-gather hist_out of every GPU -> gathered [G][N] (device)
 *   fm_layer_route       -> route() over the full demand + dispatch plan; returns the
 *                           per-peer row counts (host int32 [G] each). Synchronises the
 *                           stream (the all-to-all needs the counts on the host).
 *   fm_layer_dispatch    -> send_buf [sum(send_rows), d] bf16, peer-major (dst ascending,
 *                           then expert ascending, then the canonical unit order)
 *   host: all-to-all send_buf -> recv_buf (split sizes send_rows / recv_rows)
 *   fm_layer_expert_forward  recv_buf (src-major) -> expert FFN -> ret_buf (same order)
 *   host: all-to-all ret_buf -> back_buf (split sizes reversed)
 *   fm_layer_combine     back_buf -> y
 * backward mirrors it: fm_layer_combine_backward (dy -> dsend_buf),
 * all-to-all, fm_layer_expert_backward (drecv -> weight grads, dret),
 * all-to-all, fm_layer_unpermute_backward (dback -> dx, gate-weight grad from
 * the still-valid send_buf). Weight gradients of replicated experts are then
 * summed over each replica group (ascending expert id); dwg over all GPUs. */
int fm_layer_gate(fm_layer* layer, const void* x, int num_tokens, const void* wg, int64_t* hist_out,
                  void* stream);
int fm_layer_route(fm_layer* layer, const int64_t* gathered_hist_GN, int32_t* send_rows,
                   int32_t* recv_rows, void* stream);
int fm_layer_dispatch(fm_layer* layer, const void* x, void* send_buf, void* stream);
int fm_layer_expert_forward(fm_layer* layer, const void* recv_buf, const void* w1, const float* b1,
                            const void* w2, const float* b2, void* ret_buf, void* stream);
int fm_layer_combine(fm_layer* layer, const void* back_buf, void* y, void* stream);
int fm_layer_combine_backward(fm_layer* layer, const void* dy, const void* back_buf,
                              void* dsend_buf, void* stream);
int fm_layer_expert_backward(fm_layer* layer, const void* drecv_buf, const void* w1,
                             const void* w2, float* dw1, float* db1, float* dw2, float* db2,
                             void* dret_buf, void* stream);
int fm_layer_unpermute_backward(fm_layer* layer, const void* dback_buf, const void* send_buf,
                                const void* wg, void* dx, float* dwg, void* stream);

/* Peer-to-peer transport (the B200-native alternative to the all-to-alls
 * above). fm_layer_enable_p2p allocates one exchange arena per
 * GPU (X_perm, Y_perm, dY_perm, dX_perm, dl rows and arrival flags, sized for
 * route()'s worst case) that every peer maps: CUDA IPC handles
 * (fm_layer_p2p_handle / fm_layer_p2p_open_peer) across processes, or
 * fm_layer_p2p_link_peer between layers of one process. Token rows then
 * cross NVLink inside the kernels that produce or consume them:
 *   fm_layer_gate            (as above; advances the exchange epoch)
 *   host: all-gather hist_out -> gathered [G][N]
 *   fm_layer_route_p2p       route() + plan incl. every peer's X_perm layout (no host sync)
 *   fm_layer_dispatch_p2p    x rows -> the expert GPUs' X_perm (+ own pad rows); flags
 *   fm_layer_expert_forward_p2p   FFN (each tile waits for its sources), flag "Y ready"
 *   fm_layer_combine_p2p     wait, y = sum_j w_j Y rows read from the expert GPUs
 *   fm_layer_combine_backward_p2p  dY rows (+ gate dl) -> the expert GPUs' dY_perm; flags
 *   fm_layer_expert_backward_p2p   wait, dgrad, flag "dX ready", weight grads; dwg gets this
 *                            GPU's share of the gate-weight gradient (sum it over all GPUs)
 *   fm_layer_unpermute_backward_p2p  wait, dx from dX rows read from the expert GPUs
 * Waits are device-side, inside the consuming kernels (flags in the arena,
 * monotonic epochs; the expert GEMMs wait per 128-row tile for exactly the
 * sources in it) and bounded: after ~20 s a wait gives up and
 * fm_layer_p2p_status reports it. Slots are
 * reused across steps only after the next step's demand all-gather, which
 * every GPU joins after finishing the previous step.
 * CALLER REQUIREMENT (buffer reuse across steps): "dX ready" is signalled
 * right after the FFN1 dgrad, but this GPU's weight-gradient GEMMs and tile
 * sums still read X_perm and dY_perm afterwards. A peer's step-(i+1)
 * fm_layer_dispatch_p2p writes into this GPU's X_perm, so the step-(i+1)
 * demand exchange (the all-gather of hist_out) MUST be stream-ordered after
 * this GPU's step-i fm_layer_expert_backward_p2p / fm_layer_unpermute_backward_p2p
 * (enqueue the collective on the same stream, as the Python runtime and
 * host/flexmoe_step.cpp do, or wait on an event recorded after them). */
int fm_layer_enable_p2p(fm_layer* layer);
int fm_layer_p2p_handle(fm_layer* layer, void* handle64);
int fm_layer_p2p_open_peer(fm_layer* layer, int peer, const void* handle64);
int fm_layer_p2p_link_peer(fm_layer* layer, int peer, fm_layer* peer_layer);
int fm_layer_p2p_status(fm_layer* layer, int* timed_out);
int fm_layer_route_p2p(fm_layer* layer, const int64_t* gathered_hist_GN, void* stream);
int fm_layer_dispatch_p2p(fm_layer* layer, const void* x, void* stream);
int fm_layer_expert_forward_p2p(fm_layer* layer, const void* w1, const float* b1, const void* w2,
                                const float* b2, void* stream);
int fm_layer_combine_p2p(fm_layer* layer, void* y, void* stream);
int fm_layer_combine_backward_p2p(fm_layer* layer, const void* dy, void* stream);
int fm_layer_expert_backward_p2p(fm_layer* layer, const void* w1, const void* w2, float* dw1, float* db1,
                                 float* dw2, float* db2, float* dwg, void* stream);
/* Optional, before fm_layer_expert_backward_p2p: the gate weight and dx
 * buffer the step's fm_layer_unpermute_backward_p2p will be given. The layer
 * then runs the un-permute on spare CTA pairs of the FFN1 weight-gradient
 * launch (after every peer's "dX ready"); the later
 * fm_layer_unpermute_backward_p2p call with the same pointers only adds the
 * dropped units' gate gradient. Must still be called. */
int fm_layer_p2p_bind_dx(fm_layer* layer, const void* wg, void* dx);
int fm_layer_unpermute_backward_p2p(fm_layer* layer, const void* wg, void* dx, float* dwg, void* stream);

/* Introspection (synchronous device->host copy, for tests / metrics). */
#define FM_FIELD_TOPK_IDX 0     /* int32 [T,k] */
#define FM_FIELD_TOPK_W 1       /* f32   [T,k] */
#define FM_FIELD_UNIT_POS 2     /* int32 [T,k] row of each unit in the dispatch buffer */
#define FM_FIELD_GATE_GRAD 3    /* f32   [T,k] d loss / d kept logit */
#define FM_FIELD_HIST 4         /* int64 [N]   this GPU's TokenDemand column */
#define FM_FIELD_DEMAND 5       /* int64 [N,G] */
#define FM_FIELD_FLOWS 6        /* int64 [N,G,G] RoutingPlan.flows */
#define FM_FIELD_SEG_START 7    /* int32 [Nl] */
#define FM_FIELD_SEG_REAL 8     /* int32 [Nl] */
#define FM_FIELD_SEG_ROWS 9     /* int32 [Nl] */
#define FM_FIELD_TOTALS 10      /* int32 [4] padded rows, units sent, units received */
#define FM_FIELD_SEND_ROWS 11   /* int32 [G] */
#define FM_FIELD_RECV_ROWS 12   /* int32 [G] */
#define FM_FIELD_X_PERM 13      /* bf16 [rows,d] */
#define FM_FIELD_ACT 14         /* bf16 [rows,f] */
#define FM_FIELD_Y_PERM 15      /* bf16 [rows,d] */
#define FM_FIELD_DY_PERM 16     /* bf16 [rows,d] */
#define FM_FIELD_DH 17          /* bf16 [rows,f] */
#define FM_FIELD_DX_PERM 18     /* bf16 [rows,d] */
#define FM_FIELD_ROUTE_STATUS 19 /* int32 [1] device route status */
#define FM_FIELD_KEPT 20        /* int64 [N,G] StaticEP kept demand (capacity mode) */
#define FM_FIELD_DROPPED 21     /* int64 [1]   units dropped this step (capacity mode) */
int fm_layer_copy_out(fm_layer* layer, int field, void* host, size_t max_bytes, size_t* written);
/* The same copy enqueued on `stream` after the work already queued there (no
 * device synchronisation; asynchronous into page-locked `host` memory): a
 * step's histogram can be read back while the next step runs. */
int fm_layer_copy_out_async(fm_layer* layer, int field, void* host, size_t max_bytes, size_t* written,
                            void* stream);

/* Per-phase CUDA-event timing on the launching stream (off by default).
 * fm_layer_read_timing synchronises the device and returns accumulated
 * milliseconds and launch counts per phase since timing was enabled. */
#define FM_PHASE_GATE 0         /* gate GEMM + top-k + softmax + tile histogram */
#define FM_PHASE_SCAN 1         /* per-expert scan over tiles (TokenDemand column) */
#define FM_PHASE_ROUTE 2        /* device route() + dispatch plan */
#define FM_PHASE_DISPATCH 3     /* pad zeroing + permute/dispatch copy */
#define FM_PHASE_FFN1_FWD 4     /* grouped GEMM relu(X W1^T + b1) */
#define FM_PHASE_FFN2_FWD 5     /* grouped GEMM A W2^T + b2 */
#define FM_PHASE_COMBINE_FWD 6  /* gate-weighted un-permute */
#define FM_PHASE_COMBINE_BWD 7  /* dY rows, gate-weight grads */
#define FM_PHASE_FFN2_DGRAD 8   /* dY W2 * relu' */
#define FM_PHASE_FFN1_DGRAD 9   /* dH W1 */
#define FM_PHASE_FFN2_WGRAD 10  /* dY^T A */
#define FM_PHASE_FFN1_WGRAD 11  /* dH^T X */
#define FM_PHASE_BIAS_GRAD 12   /* db1, db2 */
#define FM_PHASE_UNPERMUTE 13   /* dx gather + gate input grad */
#define FM_PHASE_GATE_WGRAD 14  /* dWg */
#define FM_PHASE_RELAYOUT 15    /* multi-GPU (all-to-all transport): a2a order <-> expert segments */
#define FM_NUM_PHASES 16
int fm_layer_set_timing(fm_layer* layer, int enable);
int fm_layer_read_timing(fm_layer* layer, double* ms_by_phase, int* launches_by_phase);

/* ------------------------------------------------------------------------
 * Expert state pool and peer-to-peer migration (one per GPU).
 *
 * The reference models a placement change as TransferDescriptor{src, dst,
 * bytes} (proj/include/moesim/placement.hpp:31-35, produced by
 * Placement::expand/migrate, placement.cpp:143-232) drained by the adjustment
 * queue (sim_engine.cpp:124-262); bytes = expert_state_bytes (topology.cpp:177).
 * Here the state really moves: every hosted expert owns one slot of a
 * cudaMalloc'd pool holding its f32 master parameters and Adam moments,
 *   slot = [ master | m | v ], each P = 2*f*d + f + d floats laid out
 *          [ w1 (f,d) | b1 (f) | w2 (d,f) | b2 (d) ],
 * and a transfer is a cudaMemcpyAsync of one slot from a peer GPU's pool
 * (CUDA IPC, NVLink / NVSwitch) on the pool's side stream, issued by the
 * receiving GPU. The bf16 working copy is re-derived from the master on
 * arrival (bit-identical to the source's, which rounds the same floats).
 * The copies overlap the gate / routing / dispatch of the step; the compute
 * stream waits for them (fm_pool_wait_ready) only before the expert FFN.
 *
 * Ordering contract: the receiver enqueues the pull after a collective that
 * every source joins only once its previous optimizer update is enqueued (the
 * runtime uses the step's demand all-gather), so it reads the state the
 * source starts the step with; the source must not write the slot before
 * every peer has passed that step's expert FFN (any later full-world
 * collective orders it); a slot vacated in step s is reused no earlier than
 * step s+1.
 * ---------------------------------------------------------------------- */
typedef struct fm_expert_pool fm_expert_pool;

/* Adam hyper-parameters of fm_pool_adam (bias-corrected, step >= 1). */
typedef struct fm_adam_config {
  float lr;
  float beta1;
  float beta2;
  float eps;
  int step;
} fm_adam_config;

/* `slots` expert slots on the current device, `world` peer pools addressable. */
int fm_pool_create(int slots, int d_model, int d_ff, int world, fm_expert_pool** out);
int fm_pool_destroy(fm_expert_pool* pool);
/* P (floats per tensor set) and the slot stride in bytes (>= 12*P, 256-aligned). */
int fm_pool_info(const fm_expert_pool* pool, int64_t* params_per_expert, int64_t* slot_bytes);
/* Device address of slot `slot` (master at +0, m at +4P bytes, v at +8P). */
int fm_pool_slot_ptr(fm_expert_pool* pool, int slot, void** dev_ptr);
/* cudaIpcMemHandle_t of the pool allocation (64 bytes) and its import on a peer
 * process; fm_pool_link_peer links a pool of the same process instead. */
int fm_pool_ipc_handle(fm_expert_pool* pool, void* handle64);
int fm_pool_open_peer(fm_expert_pool* pool, int peer, const void* handle64);
int fm_pool_link_peer(fm_expert_pool* pool, int peer, fm_expert_pool* peer_pool);
/* Pull expert states: moves_n3[i] = {dst_slot (local), peer, src_slot (peer's)};
 * whole slots (12*P bytes each) copied peer -> local on the side stream after
 * everything already enqueued on `stream`. Then the bf16/f32 operand packing of
 * the `num_local` experts in `local_slots` (ascending expert id) into w1 [n,f,d]
 * bf16, b1 [n,f] f32, w2 [n,d,f] bf16, b2 [n,d] f32 (device) runs on the side
 * stream too; fm_pool_wait_ready makes a stream wait for both. */
int fm_pool_migrate(fm_expert_pool* pool, const int32_t* moves_n3, int num_moves,
                    const int32_t* local_slots, int num_local, void* w1, float* b1, void* w2,
                    float* b2, void* stream);
int fm_pool_wait_ready(fm_expert_pool* pool, void* stream);
/* Operand layout of fm_pool_pack / fm_pool_adam / fm_pool_migrate: 0 (default)
 * = row i of the w1/b1/w2/b2 outputs is the i-th slot of the list (packed,
 * ascending local order); 1 = row `slot` (operands of capacity = pool slots,
 * addressed by the layer through fm_layer_set_operand_slots, so a placement
 * switch moves no weights and a migration re-packs only the pulled slots). */
int fm_pool_set_operand_layout(fm_expert_pool* pool, int by_slot);
/* Packing alone, on `stream`. */
int fm_pool_pack(fm_expert_pool* pool, const int32_t* local_slots, int num_local, void* w1, float* b1,
                 void* w2, float* b2, void* stream);
/* Fused Adam on the local experts (slot i <- grads [i] of dw1 [n,f,d], db1 [n,f],
 * dw2 [n,d,f], db2 [n,d] f32) that also refreshes the packed operands. */
int fm_pool_adam(fm_expert_pool* pool, const int32_t* local_slots, int num_local, const float* dw1,
                 const float* db1, const float* dw2, const float* db2, const fm_adam_config* cfg,
                 void* w1, float* b1, void* w2, float* b2, void* stream);
/* Totals over all fm_pool_migrate calls so far: side-stream copy time (CUDA
 * events around each batch of copies; synchronises on the last one), bytes
 * pulled, slots pulled. */
int fm_pool_migration_stats(fm_expert_pool* pool, double* copy_ms, int64_t* bytes, int64_t* copies);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FLEXMOE_B200_H_ */
