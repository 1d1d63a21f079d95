// Fused gate: logits = x . Wg^T on tcgen05 (TMEM accumulator), then in the
// epilogue Top-K (ties -> lower expert id), softmax over the kept logits
// (Eq. 3: g(x) = softmax(TopK(x . W_g))), and the
// warp-aggregated per-tile expert histogram + per-unit rank that the
// dispatch scan turns into the token permutation.
//
// No reference implementation exists (the reference consumes the gate as a
// trace); the tie rule is the reference's lower-id convention
// (workload.hpp:88-89) and the unit of demand is one
// (token, k-slot) pair.
//
// Per 128-token tile (one tcgen05 M=128 accumulator, N = experts padded to 32):
//   warp 0: TMA x / Wg K-slices; warp 1: MMA; warp 2: TMEM alloc;
//   warps 4-7: epilogue, thread = token row.
// Outputs per unit u = t*k + j: topk_idx[u], topk_w[u], tile_rank[u] (rank of
// the unit among this tile's units of the same expert, token order);
// per tile: tile_counts[tile][e].
#include <cuda_bf16.h>

#include <algorithm>

#include "fm_internal.h"
#include "layer_plan.h"
#include "sm100_ptx.cuh"

namespace fm {
namespace gate {

constexpr int kTM = 128;
constexpr int kBK = 64;
constexpr int kMaxStages = 8;
constexpr int kMaxExperts = 256;
constexpr int kMaxTopK = 8;
constexpr int kABytes = kTM * kBK * 2;
constexpr int kThreads = 256;
#ifndef FM_GATE_CTAS
#define FM_GATE_CTAS 2
#endif
constexpr int kCtas = FM_GATE_CTAS;  // resident CTAs per SM (A/B knob)
#ifndef FM_GATE_X_EVICT_FIRST
#define FM_GATE_X_EVICT_FIRST 1
#endif
// A/B knob: tiles walked last-to-first, so the first tokens are the most
// recent x lines in L2 when the dispatch (which walks tokens first-to-last)
// re-reads x
#ifndef FM_GATE_REVERSE
#define FM_GATE_REVERSE 0
#endif

struct Args {
  int T, N, Npad, K, top_k, stages;
  int tile_rows;  // tokens per tile (gate_tile_rows): 64 loads half an M=128 tile, the
                  // MMA's other 64 rows read the next stage (their TMEM lanes are ignored)
  int32_t* topk_idx;
  float* topk_w;
  int32_t* tile_rank;
  int32_t* tile_counts;  // [num_tiles][N]
};

#ifdef FM_GATE_TRACE
// diagnostic build only: globaltimer stamps of block 0's pipeline events
__device__ unsigned long long g_gate_trace[256];
__device__ unsigned long long g_gate_blocks[1024];  // [block][start, exit]
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define GATE_TRACE(i) \
  do {                \
    if (blockIdx.x == 0 && (i) < 256) g_gate_trace[(i)] = gtime(); \
  } while (0)
#else
#define GATE_TRACE(i) \
  do {                \
  } while (0)
#endif

#ifdef FM_GATE_SPIN
#define GATE_WAIT ptx::mbar_wait_spin
#else
#define GATE_WAIT ptx::mbar_wait
#endif

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Top-1 / top-2 of a token's logits as a pairwise tree (depth log2(32) per
// 32-column chunk instead of a 32-step dependent insertion chain). Every merge
// takes a left list A whose expert ids are all lower than the right list B's,
// so "B wins only when strictly greater" is the reference's lower-id tie rule
// — the same selection as the sorted insertion for KT >= 3.
template <int KT>
struct TopK {
  float v[KT];
  int e[KT];
};

__device__ __forceinline__ TopK<1> topk_merge(const TopK<1>& A, const TopK<1>& B) {
  const bool p = B.v[0] > A.v[0];
  return TopK<1>{{p ? B.v[0] : A.v[0]}, {p ? B.e[0] : A.e[0]}};
}

__device__ __forceinline__ TopK<2> topk_merge(const TopK<2>& A, const TopK<2>& B) {
  const bool p = B.v[0] > A.v[0];
  TopK<2> o;
  o.v[0] = p ? B.v[0] : A.v[0];
  o.e[0] = p ? B.e[0] : A.e[0];
  // runner-up: the best of what is left on each side (A's candidate has the lower id)
  const float c1v = p ? A.v[0] : A.v[1], c2v = p ? B.v[1] : B.v[0];
  const int c1e = p ? A.e[0] : A.e[1], c2e = p ? B.e[1] : B.e[0];
  const bool r = c2v > c1v;
  o.v[1] = r ? c2v : c1v;
  o.e[1] = r ? c2e : c1e;
  return o;
}

template <int KT>
__device__ __forceinline__ TopK<KT> topk_leaf(float v, int e) {
  TopK<KT> o;
  o.v[0] = v;
  o.e[0] = e;
  if constexpr (KT == 2) {
    o.v[1] = -INFINITY;
    o.e[1] = -1;
  }
  return o;
}

// columns >= N (padding) enter as -inf with their (higher) ids: any real
// expert beats or ties them and wins the tie
template <int KT>
__device__ __forceinline__ void tree_topk(uint32_t t_row, int N, int Npad, float (&best_v)[KT],
                                          int (&best_e)[KT]) {
  TopK<KT> run;
  for (int c = 0; c < Npad; c += 32) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(t_row + c, r);
    ptx::tmem_ld_wait();
    TopK<KT> n[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e0 = c + 2 * i, e1 = e0 + 1;
      const float v0 = e0 < N ? __uint_as_float(r[2 * i]) : -INFINITY;
      const float v1 = e1 < N ? __uint_as_float(r[2 * i + 1]) : -INFINITY;
      n[i] = topk_merge(topk_leaf<KT>(v0, e0), topk_leaf<KT>(v1, e1));
    }
#pragma unroll
    for (int w = 1; w < 16; w <<= 1)
#pragma unroll
      for (int i = 0; i < 16; i += 2 * w) n[i] = topk_merge(n[i], n[i + w]);
    run = c == 0 ? n[0] : topk_merge(run, n[0]);
  }
#pragma unroll
  for (int j = 0; j < KT; ++j) {
    best_v[j] = run.v[j];
    best_e[j] = run.e[j];
  }
}

// KT = top_k (compile-time: top-1 / top-2 run the pairwise tree, KT >= 3 a
// KT-slot sorted insertion).
// Two CTAs per SM: the per-tile chain (TMA -> MMA -> top-k epilogue) is
// latency-bound, a second resident CTA overlaps it (measured: 1.3x over one).
template <int KT>
__global__ void __launch_bounds__(kThreads, kCtas)
    gate_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                const Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int b_bytes = a.Npad * kBK * 2;
  const int a_bytes = a.tile_rows * kBK * 2;  // 8 or 16 KB, a multiple of the 1 KB swizzle atom
  const int stage_bytes = a_bytes + b_bytes;
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + a.stages * a_bytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + a.stages * stage_bytes);
  uint64_t* empty_bar = full_bar + kMaxStages;
  uint64_t* tfull_bar = empty_bar + kMaxStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint32_t* masks = tmem_holder + 4;  // [4 warps][Npad]

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const int num_tiles = (a.T + a.tile_rows - 1) / a.tile_rows;
  const int num_kb = a.K / kBK;
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(2 * a.Npad)) tmem_cols <<= 1;

  if (threadIdx.x == 0) GATE_TRACE(0);
#ifdef FM_GATE_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 512) g_gate_blocks[2 * blockIdx.x] = gtime();
#endif
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_x);
    ptx::tma_prefetch_desc(&map_w);
    for (int s = 0; s < a.stages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 128);
    }
    ptx::fence_mbar_init();
  }
#if FM_GATE_X_EVICT_FIRST
  // x is streamed once: its lines are the first L2 victims, so the gate does
  // not evict (and pay the write-back of) the predecessor's dirty lines
  const uint64_t pol_x = ptx::l2_policy_evict_first();
#endif
  auto issue = [&](int stage, int tile, int kb) {
    ptx::mbar_arrive_expect_tx(&full_bar[stage], stage_bytes);
#if FM_GATE_X_EVICT_FIRST
    ptx::tma_load_2d_hint(smem_a + stage * a_bytes, &map_x, &full_bar[stage], kb * kBK, tile * a.tile_rows, pol_x);
#else
    ptx::tma_load_2d(smem_a + stage * a_bytes, &map_x, &full_bar[stage], kb * kBK, tile * a.tile_rows);
#endif
    ptx::tma_load_2d(smem_b + stage * b_bytes, &map_w, &full_bar[stage], kb * kBK, 0);
  };
  for (int i = threadIdx.x; i < 4 * a.Npad; i += blockDim.x) masks[i] = 0;
  if (warp == 2) ptx::tmem_alloc(tmem_holder, tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) GATE_TRACE(1);

  // producer and MMA issuer: the whole warp runs the (warp-uniform) loop, one
  // elected lane issues — no per-instruction register->uniform shuffles
  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int ti = blockIdx.x; ti < num_tiles; ti += gridDim.x, ++it) {
      const int tile = FM_GATE_REVERSE ? num_tiles - 1 - ti : ti;
      for (int kb = 0; kb < num_kb; ++kb) {
        GATE_WAIT(&empty_bar[stage], phase ^ 1);
        if (lane == 0) GATE_TRACE(2 + it * 16 + kb);
        if (ptx::elect_one()) issue(stage, tile, kb);
        __syncwarp();
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::idesc_bf16_f32(kTM, a.Npad, false, false);
    const uint64_t da0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a), 16, 1024);
    const uint64_t db0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b), 16, 1024);
    int stage = 0;
    uint32_t phase = 0;
    int iter = 0;
    for (int ti = blockIdx.x; ti < num_tiles; ti += gridDim.x, ++iter) {
      const int tile = FM_GATE_REVERSE ? num_tiles - 1 - ti : ti;
      const int ab = iter & 1;
      GATE_WAIT(&tempty_bar[ab], ((iter >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + ab * a.Npad;
      for (int kb = 0; kb < num_kb; ++kb) {
        GATE_WAIT(&full_bar[stage], phase);
        if (lane == 0) GATE_TRACE(66 + iter * 16 + kb);
        ptx::tc_fence_after();
        // descriptor start addresses are in 16-byte units: offsets are adds
        const uint64_t da = da0 + static_cast<uint32_t>((stage * a_bytes) >> 4);
        const uint64_t db = db0 + static_cast<uint32_t>((stage * b_bytes) >> 4);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) ptx::mma_bf16_ss(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          ptx::mma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == a.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (ptx::elect_one()) ptx::mma_commit(&tfull_bar[ab]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    constexpr int k = KT;
    uint32_t* my_mask = masks + q * a.Npad;
    int iter = 0;
    for (int ti = blockIdx.x; ti < num_tiles; ti += gridDim.x, ++iter) {
      const int tile = FM_GATE_REVERSE ? num_tiles - 1 - ti : ti;
      const int ab = iter & 1;
      const int t = tile * a.tile_rows + q * 32 + lane;
      const bool valid = q * 32 + lane < a.tile_rows && t < a.T;
      GATE_WAIT(&tfull_bar[ab], (iter >> 1) & 1);
      if (q == 0 && lane == 0) GATE_TRACE(130 + 2 * iter);
      ptx::tc_fence_after();

      float best_v[KT];
      int best_e[KT];
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + ab * a.Npad;
      if constexpr (KT <= 2) {
        tree_topk<KT>(t_row, a.N, a.Npad, best_v, best_e);
      } else {
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          best_v[j] = -INFINITY;
          best_e[j] = -1;
        }
        for (int c = 0; c < a.Npad; c += 32) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(t_row + c, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int e = c + i;
            const float v = __uint_as_float(r[i]);
            // Sorted insertion, walking slots bottom-up: slot j takes slot j-1's
            // entry when v beats it, else v itself when v beats slot j. Strict '>'
            // while ids ascend keeps the lower id ahead on ties.
            if (e < a.N) {
#pragma unroll
              for (int j = KT - 1; j >= 0; --j) {
                const bool beats_prev = j > 0 && (best_e[j - 1] < 0 || v > best_v[j - 1]);
                const bool beats_cur = best_e[j] < 0 || v > best_v[j];
                if (beats_prev) {
                  best_v[j] = best_v[j - 1];
                  best_e[j] = best_e[j - 1];
                } else if (beats_cur) {
                  best_v[j] = v;
                  best_e[j] = e;
                }
              }
            }
          }
        }
      }
      // TMEM buffer no longer needed: release it to the MMA warp early.
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty_bar[ab]);

      // softmax over the kept logits (k = 1 gives weight 1)
      float wsum = 0.0f, wexp[KT];
#pragma unroll
      for (int j = 0; j < KT; ++j) {
        wexp[j] = expf(best_v[j] - best_v[0]);
        wsum += wexp[j];
      }

      // warp-aggregated histogram: one bit per (lane, expert) in this warp's mask row
      if (valid) {
#pragma unroll
        for (int j = 0; j < KT; ++j) atomicOr(&my_mask[best_e[j]], 1u << lane);
      }
      if (q == 0 && lane == 0 && iter == 0) GATE_TRACE(141);
      named_bar_sync(1, 128);  // all four masks of this tile are final
      if (q == 0 && lane == 0 && iter == 0) GATE_TRACE(142);
      if (valid) {
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const int e = best_e[j];
          int rank = __popc(masks[q * a.Npad + e] & lt);
          for (int w = 0; w < q; ++w) rank += __popc(masks[w * a.Npad + e]);
          const size_t u = static_cast<size_t>(t) * k + j;
          a.topk_idx[u] = e;
          a.topk_w[u] = wexp[j] / wsum;
          a.tile_rank[u] = rank;
        }
      }
      if (q == 0 && lane == 0 && iter == 0) GATE_TRACE(143);
      const int et = q * 32 + lane;
      for (int e = et; e < a.N; e += 128) {
        a.tile_counts[static_cast<size_t>(tile) * a.N + e] =
            __popc(masks[e]) + __popc(masks[a.Npad + e]) + __popc(masks[2 * a.Npad + e]) +
            __popc(masks[3 * a.Npad + e]);
      }
      if (q == 0 && lane == 0 && iter == 0) GATE_TRACE(144);
      named_bar_sync(1, 128);  // everyone done reading masks
      if (q == 0 && lane == 0 && iter == 0) GATE_TRACE(145);
      for (int e = lane; e < a.Npad; e += 32) my_mask[e] = 0;
      __syncwarp();
      if (q == 0 && lane == 0) GATE_TRACE(131 + 2 * iter);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, tmem_cols);
  }
  if (threadIdx.x == 0) GATE_TRACE(150);
#ifdef FM_GATE_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 512) g_gate_blocks[2 * blockIdx.x + 1] = gtime();
#endif
}

}  // namespace gate

#ifdef FM_GATE_TRACE
extern "C" int fm_debug_gate_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, gate::g_gate_trace, sizeof(gate::g_gate_trace)) == cudaSuccess ? 0 : 5;
}
extern "C" int fm_debug_gate_blocks(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, gate::g_gate_blocks, sizeof(gate::g_gate_blocks)) == cudaSuccess ? 0 : 5;
}
#endif

int gate_num_tiles(int T, int num_experts) {
  const int tr = gate_tile_rows(num_experts);
  return (T + tr - 1) / tr;
}

void launch_gate(const void* x, const void* wg, int T, int N, int d, int top_k, int32_t* topk_idx,
                 float* topk_w, int32_t* tile_rank, int32_t* tile_counts, cudaStream_t stream) {
  using namespace gate;
  if (N < 1 || N > kMaxExperts) throw std::invalid_argument("gate: 1 <= num_experts <= 256");
  if (top_k < 1 || top_k > kMaxTopK || top_k > N)
    throw std::invalid_argument("gate: 1 <= top_k <= min(8, num_experts)");
  if (d % kBK != 0) throw std::invalid_argument("gate: d_model must be a multiple of 64");
  if (T <= 0) return;
  const int Npad = ((N + 31) / 32) * 32;
  const int tr = gate_tile_rows(N);
  const int stage_bytes0 = tr * kBK * 2 + Npad * kBK * 2;
  // two CTAs per SM when both TMEM double-buffers fit (2 x 2 x Npad <= 512 columns)
#ifndef FM_GATE_WIDE_CTAS
#define FM_GATE_WIDE_CTAS 2
#endif
  // Npad >= 128: FM_GATE_WIDE_CTAS per SM (A/B knob: 1 CTA gets twice the stages)
  const int kCtasPerSm = Npad >= 128 ? (Npad == 128 ? FM_GATE_WIDE_CTAS : 1)
                                     : (Npad * kCtas <= 256 ? kCtas : 2);
  const int stages = std::max(2, std::min(kMaxStages, (200 * 1024 / kCtasPerSm) / stage_bytes0));
  Args a{T, N, Npad, d, top_k, stages, tr, topk_idx, topk_w, tile_rank, tile_counts};
  CUtensorMap mx = make_tmap_bf16(x, d, T, d, 64, tr);
  CUtensorMap mw = make_tmap_bf16(wg, d, N, d, 64, Npad);
  const int stage_bytes = stage_bytes0;
  const int smem = 1024 + stages * stage_bytes + 2 * kMaxStages * 8 + 64 + 4 * Npad * 4;
  const int tiles = gate_num_tiles(T, N);
  const int grid = std::min(tiles, kCtasPerSm * num_sms());
  auto launch = [&](auto kernel) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(kernel), smem);
    kernel<<<grid, kThreads, smem, stream>>>(mx, mw, a);
  };
  switch (top_k) {
    case 1: launch(gate_kernel<1>); break;
    case 2: launch(gate_kernel<2>); break;
    case 3: launch(gate_kernel<3>); break;
    case 4: launch(gate_kernel<4>); break;
    case 5: launch(gate_kernel<5>); break;
    case 6: launch(gate_kernel<6>); break;
    case 7: launch(gate_kernel<7>); break;
    default: launch(gate_kernel<8>); break;
  }
  FM_LAUNCH_CHECK("gate_kernel");
}

}  // namespace fm
