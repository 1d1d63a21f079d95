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

/* ------------------------------------------------------------------------
 * Grouped expert GEMM on tcgen05 (test / building-block hook).
 * seg_start, seg_rows, tile_prefix are device int32 arrays describing the
 * per-group token segments of the permuted buffers (rows multiple of 128).
 * ---------------------------------------------------------------------- */
#define FM_GEMM_FWD_BIAS_RELU 0   /* C[rows,N] = relu(A[rows,K] W_g[N,K]^T + b_g)   bf16 */
#define FM_GEMM_FWD_BIAS 1        /* C[rows,N] = A W_g^T + b_g                       bf16 */
#define FM_GEMM_DGRAD_RELU_MASK 2 /* C[rows,N] = (A[rows,K] W_g[K,N]) * (aux > 0)    bf16 */
#define FM_GEMM_DGRAD 3           /* C[rows,N] = A[rows,K] W_g[K,N]                  bf16 */
#define FM_GEMM_WGRAD 4           /* C[g][M_w,N] = A[seg_g, M_w]^T B[seg_g, N]       f32  */

int fm_grouped_gemm(int variant, const void* A, const void* B, void* C, const float* bias,
                    const void* aux, const int32_t* seg_start, const int32_t* seg_rows,
                    const int32_t* tile_prefix, int num_groups, int total_rows, int M_w, int N,
                    int K, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* FLEXMOE_B200_H_ */
