// Algorithm 3 (flexible token routing) for one expert, shared by host and
// device. Behaviour follows proj/src/router.cpp:57-169 exactly (integer
// arithmetic only, so host/device/reference agree bit for bit):
//   quota_h   = floor(load * n_{e,h} / n_e)                 (:82-84)
//   local     : keep min(quota_h, D[e][h]) on h              (:87-95)
//   remote    : per source in ascending id, grant = min(residual, sum room),
//               floor-proportional shares of the grant by room, then +1 to
//               hosts in descending remainder order (stable)  (:99-141)
//   leftovers : one token at a time to the least-loaded host,
//               ties to the lowest id                         (:143-153)
//   check     : per-source conservation                       (:157-166)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define FM_HD __host__ __device__ __forceinline__
#else
#define FM_HD inline
#endif

namespace fm {

constexpr int kMaxGpus = 64;
enum RouteStatus { kRouteOk = 0, kRouteNoReplica = 1, kRouteConservation = 2 };

// flows must be zero for expert e on entry. D, cnt: [N][G]; flows: [N][G][G].
FM_HD int split_expert_demand(int e, const int64_t* D, const int32_t* cnt, int G, int64_t* flows) {
  const int64_t* dem = D + static_cast<long long>(e) * G;
  const int32_t* slots = cnt + static_cast<long long>(e) * G;
  int64_t* fl = flows + static_cast<long long>(e) * G * G;

  int hosts[kMaxGpus];
  int num_hosts = 0;
  int64_t load = 0, replicas = 0;
  for (int g = 0; g < G; ++g) {
    load += dem[g];
    replicas += slots[g];
    if (slots[g] > 0) hosts[num_hosts++] = g;
  }
  if (load == 0) return kRouteOk;
  if (replicas == 0) return kRouteNoReplica;

  int64_t got[kMaxGpus];   // tokens received so far, per GPU
  int64_t room[kMaxGpus];  // remaining capacity share, per host
  for (int g = 0; g < G; ++g) got[g] = 0;
  for (int i = 0; i < num_hosts; ++i) {
    const int h = hosts[i];
    const int64_t share = load * slots[h] / replicas;
    const int64_t keep = share < dem[h] ? share : dem[h];
    if (keep > 0) {
      fl[h * G + h] = keep;
      got[h] = keep;
    }
    room[h] = share - got[h];
  }

  for (int src = 0; src < G; ++src) {
    int64_t left = dem[src] - fl[src * G + src];
    if (left == 0) continue;
    int64_t pool = 0;
    for (int i = 0; i < num_hosts; ++i) pool += room[hosts[i]];
    if (pool > 0) {
      const int64_t grant = left < pool ? left : pool;
      int64_t given = 0;
      int64_t rem[kMaxGpus];
      int order[kMaxGpus];
      int n_order = 0;
      for (int i = 0; i < num_hosts; ++i) {
        const int h = hosts[i];
        if (room[h] == 0) continue;
        const int64_t q = grant * room[h] / pool;
        rem[h] = grant * room[h] % pool;
        fl[src * G + h] += q;
        got[h] += q;
        room[h] -= q;
        given += q;
        // stable descending insertion by remainder (equal keys keep host order)
        int j = n_order - 1;
        while (j >= 0 && rem[order[j]] < rem[h]) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = h;
        ++n_order;
      }
      for (int i = 0; i < n_order && given != grant; ++i) {
        const int h = order[i];
        if (room[h] > 0) {
          fl[src * G + h] += 1;
          got[h] += 1;
          room[h] -= 1;
          ++given;
        }
      }
      left -= grant;
    }
    while (left > 0) {
      int best = hosts[0];
      for (int i = 1; i < num_hosts; ++i)
        if (got[hosts[i]] < got[best]) best = hosts[i];
      fl[src * G + best] += 1;
      got[best] += 1;
      --left;
    }
  }

  for (int src = 0; src < G; ++src) {
    int64_t routed = 0;
    for (int dst = 0; dst < G; ++dst) routed += fl[src * G + dst];
    if (routed != dem[src]) return kRouteConservation;
  }
  return kRouteOk;
}

void route_counts_host(const int64_t* D, const int32_t* cnt, int N, int G, int64_t* flows);
void route_counts_device(const int64_t* D, const int32_t* cnt, int N, int G, int64_t* flows,
                         int32_t* status, cudaStream_t stream);
double balance_ratio_host(const int64_t* flows, int N, int G);
void static_ep_kept_device(const int64_t* D, int N, int G, double cf, int64_t* kept,
                           int64_t* dropped, cudaStream_t stream);

}  // namespace fm
