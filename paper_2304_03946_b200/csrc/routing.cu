// Count-level FlexMoE routing (Algorithm 3) and the
// reference's per-plan metrics, host + device.
//
// Behavioural source: proj/src/router.cpp:57-169 (`route`), :33-55
// (received_matrix / per_gpu_received), proj/src/policy.cpp:32-46
// (balance_ratio), proj/src/workload.cpp:77-114 (largest_remainder_round),
// proj/src/baselines.cpp:89-122 (StaticEP capacity drops).
//
// `split_expert_demand` is one __host__ __device__ routine: the C-ABI host
// entry fm_route_counts and the device kernel (one thread per expert) run
// the same integer code, so host and device flows are identical by
// construction; tests pin both against the reference library.
#include <cmath>
#include <string>
#include <vector>

#include "fm_internal.h"
#include "routing.cuh"

namespace fm {

// Host entry: validates, routes every expert, maps status to exceptions with
// the reference's messages (router.cpp:58-63, :76-77, :163).
void route_counts_host(const int64_t* D, const int32_t* cnt, int N, int G, int64_t* flows) {
  if (N < 0 || G < 1) throw std::invalid_argument("route: bad dimensions");
  if (G > kMaxGpus) throw std::invalid_argument("route: more than 64 GPUs is not supported");
  for (size_t i = 0; i < static_cast<size_t>(N) * G * G; ++i) flows[i] = 0;
  for (int e = 0; e < N; ++e) {
    const int st = split_expert_demand(e, D, cnt, G, flows);
    if (st == kRouteNoReplica)
      throw std::invalid_argument("route: expert " + std::to_string(e) +
                                  " has demand but no replica");
    if (st == kRouteConservation)
      throw std::logic_error("route: conservation violated for expert " + std::to_string(e));
  }
}

namespace {

__global__ void route_kernel(const int64_t* __restrict__ D, const int32_t* __restrict__ cnt,
                             int N, int G, int64_t* __restrict__ flows, int32_t* status) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  int64_t* fe = flows + static_cast<size_t>(e) * G * G;
  for (int i = 0; i < G * G; ++i) fe[i] = 0;
  const int st = split_expert_demand(e, D, cnt, G, flows);
  if (st != kRouteOk && status) atomicCAS(status, 0, st == kRouteNoReplica ? FM_ERR_INVALID_ARGUMENT : FM_ERR_LOGIC);
}

// StaticEP capacity drops on the device (baselines.cpp:89-122), one thread per
// expert. The double arithmetic is spelled out with explicit round-to-nearest
// intrinsics (no FMA contraction), in the reference's evaluation order:
// cap = floor((cf * B) / N); exact[g] = (D[e][g] * cap) / load; then
// largest-remainder rounding with a stable descending sort of the fractions.
__global__ void static_ep_kept_kernel(const int64_t* __restrict__ D, int N, int G, double cf,
                                      int64_t* __restrict__ kept, int64_t* __restrict__ dropped) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= N) return;
  int64_t tokens = 0;
  for (int i = 0; i < N * G; ++i) tokens += D[i];
  const int64_t cap =
      static_cast<int64_t>(floor(__ddiv_rn(__dmul_rn(cf, static_cast<double>(tokens)), static_cast<double>(N))));
  const int64_t* De = D + static_cast<size_t>(e) * G;
  int64_t* Ke = kept + static_cast<size_t>(e) * G;
  int64_t load = 0;
  for (int g = 0; g < G; ++g) load += De[g];
  int64_t drop = 0;
  if (load <= cap) {
    for (int g = 0; g < G; ++g) Ke[g] = De[g];
  } else {
    double frac[kMaxGpus];
    int64_t out[kMaxGpus];
    int order[kMaxGpus];
    int64_t assigned = 0;
    for (int g = 0; g < G; ++g) {
      const double ex = __ddiv_rn(__dmul_rn(static_cast<double>(De[g]), static_cast<double>(cap)),
                                  static_cast<double>(load));
      const double fl = floor(ex);
      out[g] = static_cast<int64_t>(fl);
      frac[g] = __dsub_rn(ex, fl);
      assigned += out[g];
      int j = g - 1;
      while (j >= 0 && frac[order[j]] < frac[g]) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = g;
    }
    for (int64_t k = 0; assigned < cap; ++k, ++assigned) out[order[k % G]] += 1;
    for (int64_t k = G; assigned > cap;) {
      --k;
      const int i = order[k % G];
      if (out[i] > 0) {
        out[i] -= 1;
        --assigned;
      }
      if (k == 0) k = G;
    }
    for (int g = 0; g < G; ++g) {
      const int64_t kg = out[g] < De[g] ? out[g] : De[g];
      drop += De[g] - kg;
      Ke[g] = kg;
    }
  }
  if (dropped && drop) atomicAdd(reinterpret_cast<unsigned long long*>(dropped),
                                 static_cast<unsigned long long>(drop));
}

}  // namespace

void static_ep_kept_device(const int64_t* D, int N, int G, double cf, int64_t* kept,
                           int64_t* dropped, cudaStream_t stream) {
  if (N < 1 || G < 1 || G > kMaxGpus) throw std::invalid_argument("static_ep: bad dimensions");
  if (dropped) FM_CUDA(cudaMemsetAsync(dropped, 0, sizeof(int64_t), stream));
  static_ep_kept_kernel<<<(N + 127) / 128, 128, 0, stream>>>(D, N, G, cf, kept, dropped);
  FM_LAUNCH_CHECK("static_ep_kept_kernel");
}

void route_counts_device(const int64_t* D, const int32_t* cnt, int N, int G, int64_t* flows,
                         int32_t* status, cudaStream_t stream) {
  if (N < 1 || G < 1) throw std::invalid_argument("route: bad dimensions");
  if (G > kMaxGpus) throw std::invalid_argument("route: more than 64 GPUs is not supported");
  if (status) FM_CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), stream));
  route_kernel<<<(N + 127) / 128, 128, 0, stream>>>(D, cnt, N, G, flows, status);
  FM_LAUNCH_CHECK("route_kernel");
}

void received_matrix_host(const int64_t* flows, int N, int G, int64_t* recv) {
  for (int e = 0; e < N; ++e)
    for (int dst = 0; dst < G; ++dst) {
      int64_t s = 0;
      for (int src = 0; src < G; ++src) s += flows[(static_cast<size_t>(e) * G + src) * G + dst];
      recv[static_cast<size_t>(e) * G + dst] = s;
    }
}

void per_gpu_received_host(const int64_t* flows, int N, int G, int64_t* totals) {
  for (int dst = 0; dst < G; ++dst) totals[dst] = 0;
  for (int e = 0; e < N; ++e)
    for (int src = 0; src < G; ++src)
      for (int dst = 0; dst < G; ++dst)
        totals[dst] += flows[(static_cast<size_t>(e) * G + src) * G + dst];
}

double balance_ratio_host(const int64_t* flows, int N, int G) {
  std::vector<int64_t> t(G);
  per_gpu_received_host(flows, N, G, t.data());
  int64_t sum = 0, mx = 0;
  for (int64_t v : t) {
    sum += v;
    mx = v > mx ? v : mx;
  }
  if (sum == 0) throw std::invalid_argument("balance_ratio: zero total tokens");
  return static_cast<double>(mx) / (static_cast<double>(sum) / static_cast<double>(G));
}

// Floors, then one extra unit per index in descending fractional order
// (stable: equal fractions keep ascending index); the downward pass exists
// for floating-point drift, as in the reference.
void largest_remainder_round_host(const double* exact, int n, int64_t total, int64_t* out) {
  if (n <= 0) {
    if (total != 0) throw std::invalid_argument("largest_remainder_round: empty input");
    return;
  }
  std::vector<double> frac(n);
  std::vector<int> order(n);
  int64_t assigned = 0;
  for (int i = 0; i < n; ++i) {
    const double fl = std::floor(exact[i]);
    out[i] = static_cast<int64_t>(fl);
    frac[i] = exact[i] - fl;
    assigned += out[i];
    // insertion into a stable descending order
    int j = i - 1;
    while (j >= 0 && frac[order[j]] < frac[i]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = i;
  }
  for (int64_t k = 0; assigned < total; ++k, ++assigned) out[order[k % n]] += 1;
  for (int64_t k = n; assigned > total;) {
    --k;
    const int i = order[k % n];
    if (out[i] > 0) {
      out[i] -= 1;
      --assigned;
    }
    if (k == 0) k = n;
  }
}

int64_t static_ep_kept_host(const int64_t* D, int N, int G, double cf, int64_t* kept) {
  if (N < 1 || G < 1) throw std::invalid_argument("static_ep: bad dimensions");
  int64_t tokens = 0;
  for (size_t i = 0; i < static_cast<size_t>(N) * G; ++i) {
    tokens += D[i];
    kept[i] = D[i];
  }
  if (std::isinf(cf)) return 0;
  const int64_t cap = static_cast<int64_t>(std::floor(cf * static_cast<double>(tokens) / N));
  std::vector<double> exact(G);
  std::vector<int64_t> row(G);
  int64_t dropped = 0;
  for (int e = 0; e < N; ++e) {
    const int64_t* De = D + static_cast<size_t>(e) * G;
    int64_t load = 0;
    for (int g = 0; g < G; ++g) load += De[g];
    if (load <= cap) continue;
    // Proportional share of the capacity per source (mul then div, as the reference).
    for (int g = 0; g < G; ++g)
      exact[g] = static_cast<double>(De[g]) * static_cast<double>(cap) / static_cast<double>(load);
    largest_remainder_round_host(exact.data(), G, cap, row.data());
    for (int g = 0; g < G; ++g) {
      const int64_t k = row[g] < De[g] ? row[g] : De[g];
      dropped += De[g] - k;
      kept[static_cast<size_t>(e) * G + g] = k;
    }
  }
  return dropped;
}

}  // namespace fm

extern "C" {

int fm_route_counts(const int64_t* demand_NG, const int32_t* replica_counts_NG, int num_experts,
                    int num_gpus, int64_t* flows_NGG) {
  return fm::guarded(
      [&] { fm::route_counts_host(demand_NG, replica_counts_NG, num_experts, num_gpus, flows_NGG); });
}

int fm_route_counts_device(const int64_t* demand_NG, const int32_t* replica_counts_NG,
                           int num_experts, int num_gpus, int64_t* flows_NGG, int32_t* status_dev,
                           void* stream) {
  return fm::guarded([&] {
    fm::route_counts_device(demand_NG, replica_counts_NG, num_experts, num_gpus, flows_NGG,
                            status_dev, static_cast<cudaStream_t>(stream));
  });
}

int fm_static_ep_kept_device(const int64_t* demand_NG, int num_experts, int num_gpus,
                             double capacity_factor, int64_t* kept_NG, int64_t* dropped,
                             void* stream) {
  return fm::guarded([&] {
    fm::static_ep_kept_device(demand_NG, num_experts, num_gpus, capacity_factor, kept_NG, dropped,
                              static_cast<cudaStream_t>(stream));
  });
}

int fm_received_matrix(const int64_t* flows_NGG, int num_experts, int num_gpus,
                       int64_t* recv_NG) {
  return fm::guarded([&] { fm::received_matrix_host(flows_NGG, num_experts, num_gpus, recv_NG); });
}

int fm_per_gpu_received(const int64_t* flows_NGG, int num_experts, int num_gpus,
                        int64_t* totals_G) {
  return fm::guarded([&] { fm::per_gpu_received_host(flows_NGG, num_experts, num_gpus, totals_G); });
}

int fm_balance_ratio(const int64_t* flows_NGG, int num_experts, int num_gpus, double* ratio) {
  return fm::guarded([&] { *ratio = fm::balance_ratio_host(flows_NGG, num_experts, num_gpus); });
}

int fm_largest_remainder_round(const double* exact, int n, int64_t total, int64_t* out) {
  return fm::guarded([&] { fm::largest_remainder_round_host(exact, n, total, out); });
}

int fm_static_ep_kept(const int64_t* demand_NG, int num_experts, int num_gpus,
                      double capacity_factor, int64_t* kept_NG, int64_t* dropped) {
  return fm::guarded([&] {
    const int64_t d = fm::static_ep_kept_host(demand_NG, num_experts, num_gpus, capacity_factor, kept_NG);
    if (dropped) *dropped = d;
  });
}

}  // extern "C"
