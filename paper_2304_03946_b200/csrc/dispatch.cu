// Token dispatch / combine for the FlexMoE layer (HBM-bound kernels).
//
// Canonical permutation (the reference tracks counts only,
// SPEC.md:278, and leaves the expert-wise layout open):
//   * a demand unit is (token t, k-slot j); units of expert e produced on
//     source GPU s are ranked in ascending token order (a token's k experts
//     are distinct, so the k-slot never breaks a tie);
//   * the first flows[e][s][s] ranks stay on s, the next flows[e][s][d] go to
//     d for d ascending (d != s) — the local-then-remote order of
//     route(), router.cpp:86-153;
//   * on a destination, expert segments are ascending expert id, each padded
//     to a multiple of 128 rows with zero rows (the grouped GEMM's M/K tile);
//     inside a segment rows are ordered by source GPU, then rank.
// Everything here is integer-exact and deterministic; the only atomics are
// fp32 additions into bias / gate-weight gradients.
#include <map>
#include <mutex>
#include <unordered_map>
#include <cuda_bf16.h>

#include <algorithm>

#include "fm_internal.h"
#include "layer_plan.h"
#include "routing.cuh"

namespace fm {
namespace {

constexpr int kRowAlign = 128;

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------- scan
// Block per expert: exclusive prefix of the gate's per-tile counts, and the
// expert's total demand on this GPU (one column of TokenDemand, int64).
__global__ void expert_scan_kernel(const int32_t* __restrict__ tile_counts, int num_tiles, int N,
                                   int32_t* __restrict__ tile_base, int64_t* __restrict__ hist,
                                   int64_t* __restrict__ demand_col, int G, int src) {
  const int e = blockIdx.x;
  const int per = (num_tiles + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per;
  const int hi = min(lo + per, num_tiles);
  int sum = 0;
  for (int t = lo; t < hi; ++t) sum += tile_counts[static_cast<size_t>(t) * N + e];
  // block exclusive scan of `sum`
  __shared__ int warp_tot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane < nw) warp_tot[lane] = v;  // inclusive warp totals
  }
  __syncthreads();
  int run = incl - sum + (wid > 0 ? warp_tot[wid - 1] : 0);
  for (int t = lo; t < hi; ++t) {
    tile_base[static_cast<size_t>(t) * N + e] = run;
    run += tile_counts[static_cast<size_t>(t) * N + e];
  }
  if (threadIdx.x == blockDim.x - 1) {
    hist[e] = run;
    if (demand_col) demand_col[static_cast<size_t>(e) * G + src] = run;
  }
}

// ----------------------------------------------------------------- plan
// Exclusive prefix sum of v[0, n) in shared memory, in place; returns the
// total. Every thread of the block calls it (scratch: >= 32 ints). Each thread
// scans a contiguous run, warps combine their run totals with shuffles, one
// warp scans the warp totals: two block barriers per call (a Hillis-Steele
// pass over the block would take 2 log2(blockDim) of them — the plan kernel
// is a chain of such scans and runs single-block on the critical path).
__device__ __noinline__ int block_exclusive_scan(int32_t* v, int n, int32_t* scratch) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, static_cast<int>(threadIdx.x) * per), hi = min(n, lo + per);
  int sum = 0;
  for (int i = lo; i < hi; ++i) sum += v[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) scratch[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < nw) scratch[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = incl - sum + (wid > 0 ? scratch[wid - 1] : 0);
  for (int i = lo; i < hi; ++i) {
    const int x = v[i];
    v[i] = run;
    run += x;
  }
  const int total = scratch[nw - 1];
  __syncthreads();  // scratch reuse by the next call
  return total;
}

// One block. Turns flows[e][src][dst] into the offsets every later kernel
// uses (see PlanDev in layer_plan.h).
// With `demand` set, the block first runs route() itself (Alg. 3, one thread
// per expert: split_expert_demand, the same routine as fm_route_counts) and
// writes the flows — route + plan in one launch, no kernel boundary between.
// Every offset table is a block-wide scan over shared memory: a serial walk
// by one thread is a dependent chain of ~7 cycles per instruction, which at
// 64 experts cost ~100 us per step.
// gathered_GN (optional): the all-gathered per-GPU histograms [G][N]; the
// block first transposes them into `demand` ([N][G], TokenDemand layout) —
// the demand_transpose launch folded into this one.
// Fused expert scan (single GPU, N x tiles <= 8192): the gate's per-tile
// counts -> per-expert exclusive prefix over tiles (tile_base), the histogram
// and the demand column, as expert_scan_kernel, before route() reads that
// demand. 256 threads = N groups of 256/N threads; a thread keeps a run of up
// to 32 consecutive tiles of its expert in registers (independent loads), the
// group scans its run totals with shuffles, then the thread writes its bases.
struct PlanScan {
  const int32_t* tile_counts;  // null: the scan ran as its own kernel
  int num_tiles;
  int32_t* tile_base;
  int64_t* hist;
};
constexpr int kPlanScanRun = 32;

__device__ __forceinline__ void plan_fused_scan(const PlanScan& sc, int N, int64_t* demand_col) {
  int tpe = static_cast<int>(blockDim.x) / N;  // threads per expert: a power of two <= 32
  tpe = tpe >= 32 ? 32 : tpe >= 16 ? 16 : tpe >= 8 ? 8 : tpe >= 4 ? 4 : tpe >= 2 ? 2 : 1;
  const int e = static_cast<int>(threadIdx.x) / tpe, r = static_cast<int>(threadIdx.x) % tpe;
  const bool active = e < N;
  const int per = (sc.num_tiles + tpe - 1) / tpe, t0 = r * per;
  const int lim = active ? max(0, min(per, sc.num_tiles - t0)) : 0;  // tiles of this thread's run
  const size_t at = active ? static_cast<size_t>(t0) * N + e : 0;
  const int32_t* src = sc.tile_counts + at;
  int v[kPlanScanRun];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kPlanScanRun; ++i) v[i] = i < lim ? __ldg(src + static_cast<size_t>(i) * N) : 0;
#pragma unroll
  for (int i = 0; i < kPlanScanRun; ++i) sum += v[i];
  int incl = sum;  // inclusive scan over the tpe lanes of this expert's group
  for (int o = 1; o < tpe; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o, tpe);
    if (r >= o) incl += u;
  }
  int run = incl - sum;
  int32_t* dst = sc.tile_base + at;
#pragma unroll
  for (int i = 0; i < kPlanScanRun; ++i) {
    if (i < lim) dst[static_cast<size_t>(i) * N] = run;
    run += v[i];
  }
  if (active && r == tpe - 1) {
    sc.hist[e] = incl;
    demand_col[e] = incl;
  }
}

// route() for one expert, one out-of-line copy: the plan kernel runs once per
// step on one SM, so its time is mostly instruction fetch (ncu: "no
// instruction" the top stall) — its code is kept small rather than inlined.
__device__ __noinline__ int route_one_expert(int e, const int64_t* D, const int32_t* cnt, int G, int64_t* flows) {
  return split_expert_demand(e, D, cnt, G, flows);
}

template <bool flows_in_smem>
__global__ void plan_kernel(int64_t* __restrict__ flows, int N, int G, int me,
                            const int32_t* __restrict__ local_expert, int Nl, PlanDev p,
                            const int32_t* __restrict__ counts, const int64_t* __restrict__ demand,
                            int32_t* __restrict__ status,
                            const int64_t* __restrict__ gathered_GN, PlanScan scan) {
  if (scan.tile_counts) {
    plan_fused_scan(scan, N, const_cast<int64_t*>(demand));
    __syncthreads();  // the block's demand writes are visible to route() below
  }
  if (gathered_GN) {
    int64_t* dem = const_cast<int64_t*>(demand);
    for (int i = threadIdx.x; i < N * G; i += blockDim.x) dem[i] = gathered_GN[static_cast<size_t>(i % G) * N + i / G];
    __syncthreads();  // the block's global writes are visible to route() below
  }
  // shared: flows as int32 [N][G][G] (when they fit) | local experts [Nl] | segment starts [Nl]
  //       | replica counts [N][G] | mtile prefix [Nl] | scan buffer [N*G] | scratch [blockDim]
  extern __shared__ int32_t sf[];
  const int nflow = flows_in_smem ? N * G * G : 0;
  int32_t* sle = sf + nflow;
  int32_t* sss = sle + Nl;
  int32_t* scnt = sss + Nl;
  int32_t* smt = scnt + N * G;
  int32_t* sbuf = smt + Nl;
  int32_t* scratch = sbuf + N * G;
  for (int i = threadIdx.x; i < Nl; i += blockDim.x) sle[i] = local_expert[i];
  if (counts)
    for (int i = threadIdx.x; i < N * G; i += blockDim.x) scnt[i] = counts[i];
  if (demand) {
    if (threadIdx.x == 0 && status) *status = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < N; e += blockDim.x) {
      int64_t* fe = flows + static_cast<size_t>(e) * G * G;
      for (int i = 0; i < G * G; ++i) fe[i] = 0;
      // one GPU: Alg. 3 keeps every unit where it is (share = load, keep =
      // min(share, D) = load; nothing remote) — the same result without
      // fetching route()'s code
      const int st = G == 1 ? (demand[e] == 0 ? kRouteOk : counts[e] > 0 ? (flows[e] = demand[e], kRouteOk)
                                                                         : kRouteNoReplica)
                            : route_one_expert(e, demand, counts, G, flows);
      if (st != kRouteOk && status)
        atomicCAS(status, 0, st == kRouteNoReplica ? FM_ERR_INVALID_ARGUMENT : FM_ERR_LOGIC);
    }
    __syncthreads();  // the block's global flow writes are visible to all its threads
  }
  for (int i = threadIdx.x; i < nflow; i += blockDim.x) sf[i] = static_cast<int32_t>(flows[i]);
  __syncthreads();
  const int64_t* gflows = flows;
#define FL(e, s, d)                                                     \
  (flows_in_smem ? sf[((e) * G + (s)) * G + (d)]                        \
                 : static_cast<int32_t>(gflows[((e) * G + (s)) * G + (d)]))
  // --- source side: chunk order of each expert's ranks (me first, then ascending)
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int lo = 0;
    for (int i = 0; i < G; ++i) {
      const int dst = (i == 0) ? me : (i <= me ? i - 1 : i);
      p.chunk_lo[e * G + dst] = lo;
      p.chunk_cnt[e * G + dst] = FL(e, me, dst);
      lo += FL(e, me, dst);
    }
  }
  // --- destination side: local segments (rows padded to 128)
  for (int li = threadIdx.x; li < Nl; li += blockDim.x) {
    const int e = sle[li];
    int real = 0;
    for (int s = 0; s < G; ++s) real += FL(e, s, me);
    const int rows = (real + kRowAlign - 1) / kRowAlign * kRowAlign;
    p.seg_real[li] = real;
    p.seg_rows[li] = rows;
    sss[li] = rows;
    smt[li] = rows / kRowAlign;
  }
  __syncthreads();
  const int total_rows = block_exclusive_scan(sss, Nl, scratch);
  const int total_mt = block_exclusive_scan(smt, Nl, scratch);
  for (int li = threadIdx.x; li < Nl; li += blockDim.x) {
    p.seg_start[li] = sss[li];
    p.mtile_prefix[li] = smt[li];
  }
  if (threadIdx.x == 0) {
    p.mtile_prefix[Nl] = total_mt;
    p.totals[0] = total_rows;  // padded rows on this GPU
  }
  if (p.tile_src_mask) {
    // P2P: sources with rows in each 128-row tile (the expert GEMMs wait per
    // tile for exactly those arrivals); a tile's segment is the last one whose
    // first tile is <= it (empty segments share their successor's prefix)
    for (int t = threadIdx.x; t < total_mt; t += blockDim.x) {
      int lo = 0, hi = Nl - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (smt[mid] <= t) lo = mid;
        else hi = mid - 1;
      }
      const int e = sle[lo];
      const int t0 = sss[lo] + (t - smt[lo]) * kRowAlign, t1 = t0 + kRowAlign;
      unsigned long long m = 0ull;
      int r = sss[lo];
      for (int s = 0; s < G; ++s) {
        const int r1 = r + FL(e, s, me);
        if (r1 > r && r < t1 && r1 > t0) m |= 1ull << s;
        r = r1;
      }
      p.tile_src_mask[t] = m;
    }
  }
  // --- send side: offsets in the dispatch buffer (dst-major, expert-minor)
  for (int j = threadIdx.x; j < N * G; j += blockDim.x) sbuf[j] = FL(j % N, me, j / N);
  __syncthreads();
  const int sent = block_exclusive_scan(sbuf, N * G, scratch);
  for (int j = threadIdx.x; j < N * G; j += blockDim.x) p.send_off[(j % N) * G + j / N] = sbuf[j];
  for (int dst = threadIdx.x; dst < G; dst += blockDim.x)
    p.send_rows[dst] = (dst + 1 < G ? sbuf[(dst + 1) * N] : sent) - sbuf[dst * N];
  if (threadIdx.x == 0) p.totals[1] = sent;  // units sent (== T * k)
  __syncthreads();
  // --- receive side: chunk offsets in the a2a receive buffer (src-major,
  // local-expert-minor) and their X_perm destinations
  const int nrc = G * Nl;
  for (int j = threadIdx.x; j < nrc; j += blockDim.x) sbuf[j] = FL(sle[j % Nl], j / Nl, me);
  __syncthreads();
  const int recvd = block_exclusive_scan(sbuf, nrc, scratch);
  for (int j = threadIdx.x; j < nrc; j += blockDim.x) {
    const int src = j / Nl, li = j % Nl, e = sle[li];
    int before = 0;
    for (int s2 = 0; s2 < src; ++s2) before += FL(e, s2, me);
    p.recv_chunk_off[j] = sbuf[j];
    p.recv_chunk_dst[j] = sss[li] + before;
  }
  for (int src = threadIdx.x; src < G; src += blockDim.x) {
    const int a = src * Nl < nrc ? sbuf[src * Nl] : recvd;
    const int b = (src + 1) * Nl < nrc ? sbuf[(src + 1) * Nl] : recvd;
    p.recv_rows[src] = b - a;
  }
  if (threadIdx.x == 0) {
    p.recv_chunk_off[nrc] = recvd;
    p.totals[2] = recvd;  // units received
  }
  // P2P: where (e, me)'s units start in every destination's X_perm. Every GPU
  // lays out its segments the same way (hosted experts ascending, 128-row
  // padded, sources ascending inside a segment), so each source computes its
  // destinations' layouts from the shared flows and replica counts.
  if (p.peer_row) {
    __syncthreads();  // sbuf reuse
    for (int j = threadIdx.x; j < N * G; j += blockDim.x) {
      const int dst = j / N, e = j % N;
      int real = 0;
      for (int s = 0; s < G; ++s) real += FL(e, s, dst);
      sbuf[j] = scnt[e * G + dst] > 0 ? (real + kRowAlign - 1) / kRowAlign * kRowAlign : 0;
    }
    __syncthreads();
    block_exclusive_scan(sbuf, N * G, scratch);
    for (int j = threadIdx.x; j < N * G; j += blockDim.x) {
      const int dst = j / N, e = j % N;
      if (scnt[e * G + dst] <= 0) {
        p.peer_row[e * G + dst] = -1;
        continue;
      }
      int before = 0;
      for (int s = 0; s < me; ++s) before += FL(e, s, dst);
      p.peer_row[e * G + dst] = sbuf[j] - sbuf[dst * N] + before;
    }
  }
#undef FL
}

// Zero the padding rows of segment li: [seg_start + real, seg_start + rows)
// (part `part` of `parts` blocks on it); optionally mark them as carrying no
// expert (row_expert = -1).
constexpr int kPadParts = 4;
__device__ __forceinline__ void zero_pad_segment(__nv_bfloat16* __restrict__ buf, int d, const PlanDev& p, int li,
                                                 int part, int parts, int32_t* __restrict__ row_expert) {
  const int first = p.seg_start[li] + p.seg_real[li];
  const int last = p.seg_start[li] + p.seg_rows[li];
  if (row_expert && part == 0)
    for (int r = first + threadIdx.x; r < last; r += blockDim.x) row_expert[r] = -1;
  const int nvec = d / 8;
  const size_t begin = static_cast<size_t>(first) * nvec, end = static_cast<size_t>(last) * nvec;
  uint4* b = reinterpret_cast<uint4*>(buf);
  for (size_t i = begin + part * blockDim.x + threadIdx.x; i < end; i += static_cast<size_t>(parts) * blockDim.x)
    b[i] = make_uint4(0, 0, 0, 0);
}

inline P2P no_p2p() {
  P2P p{};
  p.signal_slot = -1;
  p.wait_slot = -1;
  return p;
}

// Block-level arrival wait of a consuming kernel (P2P pulls): one thread per
// source polls this GPU's own flags (acquire), then the block proceeds.
__device__ __forceinline__ void p2p_block_wait(const P2P& pp) {
  if (pp.wait_slot < 0) return;
  if (static_cast<int>(threadIdx.x) < pp.world) {
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(pp.base[pp.me] + pp.flag_off) +
                                  pp.wait_slot * kMaxPeers + threadIdx.x;
    unsigned long long t0, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= pp.epoch) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 20000000000ull) {
        atomicExch(pp.err, 1);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
}

// Last-block release of rows pushed into peers' arenas (P2P): after a block
// barrier one thread fences the block's stores at system scope and counts the
// block done; the last block of the grid publishes flags[slot][me] = epoch to
// every peer. A block that wrote only its own GPU's memory skips the fence
// (the last block fences before publishing; same-GPU consumers are
// stream-ordered after this kernel anyway).
__device__ __forceinline__ void p2p_release_when_last(const P2P& pp, bool wrote_peer) {
  if (pp.signal_slot < 0) return;
  // bar.sync orders the block's stores before thread 0's system-scope fence
  // (happens-before is transitive), so one fence per block covers them all
  const int any_peer = __syncthreads_or(wrote_peer);
  if (threadIdx.x == 0) {
    if (any_peer) __threadfence_system();
    unsigned int* ctr = pp.done + pp.signal_slot;
    if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
      *ctr = 0;  // the next launch of this slot is stream-ordered after this one
      __threadfence_system();
      for (int dst = 0; dst < pp.world; ++dst) {
        unsigned long long* f =
            reinterpret_cast<unsigned long long*>(pp.base[dst] + pp.flag_off) + pp.signal_slot * kMaxPeers + pp.me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(pp.epoch) : "memory");
      }
    }
  }
}

// ----------------------------------------------------------------- dispatch
// Warp per token: resolve each unit's row in the dispatch buffer and copy the
// token's activations there (k copies). When `direct` (G == 1), the dispatch
// buffer is X_perm itself and send_off is replaced by the expert's segment.
__device__ __forceinline__ void dispatch_token(int t, bool& wrote_peer, const __nv_bfloat16* __restrict__ x, int d,
                                               int k, int N,
                                                int G, int me, int direct, const int32_t* __restrict__ idx,
                                                const int32_t* __restrict__ tile_rank,
                                                const int32_t* __restrict__ tile_base, const PlanDev& p,
                                                int32_t* __restrict__ pos_out, __nv_bfloat16* __restrict__ buf,
                                                int32_t* __restrict__ row_expert, const P2P& pp) {
  const int lane = threadIdx.x & 31;
  const int nvec = d / 8;  // uint4 per row
  const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * d);
  uint4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (lane + 32 * i < nvec) v[i] = __ldg(src + lane + 32 * i);
  const int tile = t >> gate_tile_shift(N);
  for (int j = 0; j < k; ++j) {
    const int u = t * k + j;
    const int e = idx[u];
    const int r = tile_base[static_cast<size_t>(tile) * N + e] + tile_rank[u];
    int row, to = -1;
    if (direct) {  // G == 1: chunk_cnt[e] is the kept demand (all of it unless dropping)
      row = r < p.chunk_cnt[e] ? p.seg_start[p.local_index[e]] + r : -1;
    } else {
      row = -1;
      for (int i = 0; i < G; ++i) {
        const int dst = (i == 0) ? me : (i <= me ? i - 1 : i);
        const int lo = p.chunk_lo[e * G + dst];
        if (r < lo + p.chunk_cnt[e * G + dst]) {
          // P2P: straight into the destination's X_perm; else the send buffer
          row = pp.unit_dst ? p.peer_row[e * G + dst] + (r - lo) : p.send_off[e * G + dst] + (r - lo);
          to = dst;
          break;
        }
      }
    }
    if (lane == 0) {
      pos_out[u] = row;  // -1: dropped by the capacity rule (StaticEP)
      if (pp.unit_dst) pp.unit_dst[u] = row >= 0 ? to : -1;
      if (row_expert && row >= 0) row_expert[row] = e;
    }
    if (row < 0) continue;
    wrote_peer |= pp.unit_dst && to != pp.me;
    __nv_bfloat16* out = pp.unit_dst ? reinterpret_cast<__nv_bfloat16*>(pp.base[to] + pp.x_off) : buf;
    uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (lane + 32 * i < nvec) dst[lane + 32 * i] = v[i];
  }
}

__global__ void dispatch_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, int k, int N,
                                int G, int me, int direct, const int32_t* __restrict__ idx,
                                const int32_t* __restrict__ tile_rank,
                                const int32_t* __restrict__ tile_base, PlanDev p,
                                int32_t* __restrict__ pos_out, __nv_bfloat16* __restrict__ buf,
                                int32_t* __restrict__ row_expert, const P2P pp, int tok_blocks,
                                __nv_bfloat16* __restrict__ pad_buf, int Nl) {
  bool wrote_peer = false;
  if (static_cast<int>(blockIdx.x) >= tok_blocks) {  // trailing blocks: zero pad_buf's padding rows
    const int b = blockIdx.x - tok_blocks;
    zero_pad_segment(pad_buf, d, p, b / kPadParts, b % kPadParts, kPadParts, row_expert);
  } else {  // token blocks stride over the tokens (P2P: one release per block, not per 8 tokens)
    const int warps = tok_blocks * (blockDim.x >> 5);
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += warps)
      dispatch_token(t, wrote_peer, x, d, k, N, G, me, direct, idx, tile_rank, tile_base, p, pos_out, buf,
                     row_expert, pp);
  }
  p2p_release_when_last(pp, wrote_peer);
}


__global__ void zero_pad_kernel(__nv_bfloat16* __restrict__ buf, int d, PlanDev p, int Nl,
                                int32_t* __restrict__ row_expert) {
  const int li = blockIdx.y;
  if (li >= Nl) return;
  zero_pad_segment(buf, d, p, li, blockIdx.x, gridDim.x, row_expert);
}

// a2a receive buffer (src-major, expert-minor) <-> X_perm segments.
// dir = 0: recv -> perm; dir = 1: perm -> recv.
__global__ void relayout_kernel(__nv_bfloat16* __restrict__ recv, __nv_bfloat16* __restrict__ perm,
                                int d, int G, int Nl, PlanDev p, int dir) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = p.recv_chunk_off[G * Nl];
  if (row >= total) return;
  int lo = 0, hi = G * Nl;  // find chunk c with off[c] <= row < off[c+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (p.recv_chunk_off[mid] <= row) lo = mid; else hi = mid;
  }
  const int prow = p.recv_chunk_dst[lo] + (row - p.recv_chunk_off[lo]);
  const int nvec = d / 8;
  uint4* a = reinterpret_cast<uint4*>(recv + static_cast<size_t>(row) * d);
  uint4* b = reinterpret_cast<uint4*>(perm + static_cast<size_t>(prow) * d);
  for (int i = lane; i < nvec; i += 32) {
    if (dir == 0) b[i] = a[i]; else a[i] = b[i];
  }
}

// ----------------------------------------------------------------- combine
// ----------------------------------------------------------------- gathers
// Warp per token; VPL = uint4 (8 bf16) vectors per lane = d / 256. The k unit
// indices of the token are fetched by lanes 0..k-1 in one load and broadcast;
// row loads are issued two units at a time so both are in flight together.

__device__ __forceinline__ void unit_meta(const int32_t* __restrict__ pos, const float* __restrict__ w,
                                          size_t base, int k, int lane, int& my_pos, float& my_w) {
  my_pos = 0;
  my_w = 0.0f;
  if (lane < k) {
    my_pos = __ldg(pos + base + lane);
    if (w) my_w = __ldg(w + base + lane);
  }
}

// Lane j < k: destination GPU of the token's unit j (-1 without P2P).
__device__ __forceinline__ int unit_dst_of(const P2P& pp, size_t base, int k, int lane) {
  return (pp.unit_dst && lane < k) ? pp.unit_dst[base + lane] : -1;
}

// Row buffer of unit with destination `to`: the peer's arena region, or the
// local buffer (single GPU / NCCL layouts).
template <class T>
__device__ __forceinline__ T* peer_rows(const P2P& pp, int64_t off, int to, T* local) {
  return to >= 0 ? reinterpret_cast<T*>(pp.base[to] + off) : local;
}

template <int VPL>
__device__ __forceinline__ void load_row(const __nv_bfloat16* __restrict__ base, size_t row, int d,
                                         int lane, uint4 (&q)[VPL]) {
  const uint4* src = reinterpret_cast<const uint4*>(base + row * static_cast<size_t>(d));
#pragma unroll
  for (int i = 0; i < VPL; ++i) q[i] = __ldg(src + lane + 32 * i);
}
// Rows written by another GPU in this step: L2-coherent loads, no L1 reuse.
template <int VPL>
__device__ __forceinline__ void load_row_cg(const __nv_bfloat16* base, size_t row, int d, int lane,
                                            uint4 (&q)[VPL]) {
  const uint4* src = reinterpret_cast<const uint4*>(base + row * static_cast<size_t>(d));
#pragma unroll
  for (int i = 0; i < VPL; ++i) q[i] = __ldcg(src + lane + 32 * i);
}
template <int VPL>
__device__ __forceinline__ void load_unit_row(const P2P& pp, int64_t off, int to, const __nv_bfloat16* local,
                                              size_t row, int d, int lane, uint4 (&q)[VPL]) {
  if (to >= 0) load_row_cg<VPL>(reinterpret_cast<const __nv_bfloat16*>(pp.base[to] + off), row, d, lane, q);
  else load_row<VPL>(local, row, d, lane, q);
}

template <int VPL>
__device__ __forceinline__ void axpy_row(float (&acc)[VPL][8], const uint4 (&q)[VPL], float a) {
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const uint32_t qs[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc[i][2 * c] = fmaf(a, bf16lo(qs[c]), acc[i][2 * c]);
      acc[i][2 * c + 1] = fmaf(a, bf16hi(qs[c]), acc[i][2 * c + 1]);
    }
  }
}

template <int VPL>
__device__ __forceinline__ void store_row(__nv_bfloat16* __restrict__ base, size_t row, int d, int lane,
                                          const float (&acc)[VPL][8]) {
  uint4* dst = reinterpret_cast<uint4*>(base + row * static_cast<size_t>(d));
#pragma unroll
  for (int i = 0; i < VPL; ++i)
    dst[lane + 32 * i] = make_uint4(pack2(acc[i][0], acc[i][1]), pack2(acc[i][2], acc[i][3]),
                                    pack2(acc[i][4], acc[i][5]), pack2(acc[i][6], acc[i][7]));
}

// y[t] = sum_j w[t,j] * Y[pos[t,j]]  (Eq. 4), f32 accumulation.
// P2P: Y rows are read where the expert ran (NVLink loads from the peer's Y_perm).
template <int VPL>
__global__ void __launch_bounds__(256) combine_fwd_kernel(const __nv_bfloat16* __restrict__ Yl,
                                                          const int32_t* __restrict__ pos,
                                                          const float* __restrict__ w, int T, int k,
                                                          __nv_bfloat16* __restrict__ y, const P2P pp) {
  p2p_block_wait(pp);  // P2P: the expert GPUs' Y rows are complete
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int d = VPL * 256;
  int my_pos;
  float my_w;
  unit_meta(pos, w, static_cast<size_t>(t) * k, k, lane, my_pos, my_w);
  const int my_to = unit_dst_of(pp, static_cast<size_t>(t) * k, k, lane);
  float acc[VPL][8];
#pragma unroll
  for (int i = 0; i < VPL; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[i][c] = 0.0f;
  for (int j = 0; j < k; j += 2) {
    uint4 q0[VPL], q1[VPL];
    const int p0 = __shfl_sync(0xffffffffu, my_pos, j);
    const float w0 = __shfl_sync(0xffffffffu, my_w, j);
    const bool two = j + 1 < k;
    const int p1 = __shfl_sync(0xffffffffu, my_pos, two ? j + 1 : j);
    const float w1 = __shfl_sync(0xffffffffu, my_w, two ? j + 1 : j);
    const int to0 = __shfl_sync(0xffffffffu, my_to, j);
    const int to1 = __shfl_sync(0xffffffffu, my_to, two ? j + 1 : j);
    const bool h0 = p0 >= 0, h1 = two && p1 >= 0;  // dropped units contribute nothing
    if (h0) load_unit_row<VPL>(pp, pp.y_off, to0, Yl, p0, d, lane, q0);
    if (h1) load_unit_row<VPL>(pp, pp.y_off, to1, Yl, p1, d, lane, q1);
    if (h0) axpy_row<VPL>(acc, q0, w0);
    if (h1) axpy_row<VPL>(acc, q1, w1);
  }
  store_row<VPL>(y, t, d, lane, acc);
}

// Backward of the combine and of the gate softmax:
//   dYbuf[pos] = w_j * dy[t]             (bf16)
//   dw_j       = <dy[t], Y[pos]>
//   dl_j       = w_j * (dw_j - sum_i w_i dw_i)   (softmax over the kept logits)
// dl is written per unit and, when dl_rows != null, per dispatch row.
// P2P: Y rows are read from the expert's GPU, the dY row (and dl for the
// host's gate-weight gradient) is written straight into its dY_perm / dl rows.
template <int VPL>
__device__ __forceinline__ void combine_bwd_token(
    int t, bool& wrote_peer, const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ Yl,
    const int32_t* __restrict__ pos, const float* __restrict__ w, int k,
    __nv_bfloat16* __restrict__ dYl, float* __restrict__ dl, float* __restrict__ dl_rows_l, const P2P& pp) {
  const int lane = threadIdx.x & 31;
  const int d = VPL * 256;
  int my_pos;
  float my_w;
  unit_meta(pos, w, static_cast<size_t>(t) * k, k, lane, my_pos, my_w);
  const int my_to = unit_dst_of(pp, static_cast<size_t>(t) * k, k, lane);
  uint4 g[VPL];
  load_row<VPL>(dy, t, d, lane, g);
  float my_dw = 0.0f;  // lane j keeps dw_j
  for (int j = 0; j < k; ++j) {
    const int row = __shfl_sync(0xffffffffu, my_pos, j);
    const float wj = __shfl_sync(0xffffffffu, my_w, j);
    if (row < 0) {  // dropped: no expert output, d(loss)/d(w_j) = 0
      if (lane == j) my_dw = 0.0f;
      continue;
    }
    const int to = __shfl_sync(0xffffffffu, my_to, j);
    wrote_peer |= to >= 0 && to != pp.me;
    uint4 q[VPL];
    load_unit_row<VPL>(pp, pp.y_off, to, Yl, row, d, lane, q);
    uint4* dst = reinterpret_cast<uint4*>(peer_rows(pp, pp.dy_off, to, dYl) + static_cast<size_t>(row) * d);
    float dot = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const uint32_t qs[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
      const uint32_t gs[4] = {g[i].x, g[i].y, g[i].z, g[i].w};
      uint32_t o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        dot = fmaf(bf16lo(gs[c]), bf16lo(qs[c]), dot);
        dot = fmaf(bf16hi(gs[c]), bf16hi(qs[c]), dot);
        o[c] = pack2(wj * bf16lo(gs[c]), wj * bf16hi(gs[c]));
      }
      dst[lane + 32 * i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    dot = warp_sum(dot);
    if (lane == j) my_dw = dot;
  }
  // softmax backward on lanes 0..k-1
  float wdw = lane < k ? my_w * my_dw : 0.0f;
  wdw = warp_sum(wdw);
  if (lane < k) {
    const float g_l = my_w * (my_dw - wdw);
    dl[static_cast<size_t>(t) * k + lane] = g_l;
    float* dl_rows = peer_rows(pp, pp.dl_off, my_to, dl_rows_l);
    if (dl_rows && my_pos >= 0) dl_rows[my_pos] = g_l;
  }
}

// 3 blocks per SM up to d = 1024: 80 registers (allocated 8 per thread, so 81-88
// would leave 2 blocks and cost ~25 % at VPL 4)
template <int VPL>
__global__ void __launch_bounds__(256, VPL <= 4 ? 3 : 1) combine_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ Yl,
    const int32_t* __restrict__ pos, const float* __restrict__ w, int T, int k,
    __nv_bfloat16* __restrict__ dYl, float* __restrict__ dl, float* __restrict__ dl_rows_l, const P2P pp,
    int tok_blocks, PlanDev pad_plan) {
  bool wrote_peer = false;
  if (static_cast<int>(blockIdx.x) >= tok_blocks) {  // trailing blocks: zero dYl's padding rows
    const int b = blockIdx.x - tok_blocks;
    zero_pad_segment(dYl, VPL * 256, pad_plan, b / kPadParts, b % kPadParts, kPadParts, nullptr);
  } else {  // token blocks stride over the tokens (P2P: one release per block)
    const int warps = tok_blocks * (blockDim.x >> 5);
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < T; t += warps)
      combine_bwd_token<VPL>(t, wrote_peer, dy, Yl, pos, w, k, dYl, dl, dl_rows_l, pp);
  }
  p2p_release_when_last(pp, wrote_peer);  // P2P: dY rows and dl are in the expert GPUs' arenas
}

// Pipelined combine backward (top_k <= 2, d <= 1024): the register-held kernel
// above keeps <= 2 rows per warp in flight (80 registers, 3 blocks per SM:
// 0.87 of copy bandwidth at full clock, the lowest of the gathers). Here each
// warp copies its NEXT token's dy row and expert-output rows into its shared-
// memory stage with cp.async (16 B per lane, L2 only — coherent with rows a
// peer wrote this step) while it computes the current token, and the unit
// indices are loaded one token further ahead. A lane reads back only the
// chunks it copied itself, so cp.async.wait_group orders it without a warp
// barrier. Same arithmetic in the same order as combine_bwd_token.
#ifndef FM_COMBINE_BWD_PIPE
#define FM_COMBINE_BWD_PIPE 1
#endif
// The same pipelining for the combine forward: 2 = top-1 only (default: one
// register-held row per warp there; -27..-30 % at configs[2] / [4], the
// combine backward after it +3..+6 %), 1 = also top-2 (-7 µs at configs[1],
// but +6 µs in the combine backward after it: no net change), 0 = off; and for
// the dispatch (off: +4..+25 µs, its per-token index chain is not what limits
// it). profiles/r02_gather_pipe.log, r02_gather_pipe_top1.log
#ifndef FM_COMBINE_FWD_PIPE
#define FM_COMBINE_FWD_PIPE 2
#endif
#ifndef FM_DISPATCH_PIPE
#define FM_DISPATCH_PIPE 0
#endif
constexpr int kCbWarps = 8;
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(__cvta_generic_to_global(gmem))
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// combine-backward ring: stages per warp (tokens in flight + 1) and warps per block
#ifndef FM_CB_STAGES
#define FM_CB_STAGES 2
#endif
#ifndef FM_CB_WARPS
#define FM_CB_WARPS 8
#endif
#ifndef FM_CB_REVERSE
#define FM_CB_REVERSE 1
#endif
constexpr int kCbStages = FM_CB_STAGES, kCbBwdWarps = FM_CB_WARPS;

struct CbMeta {
  int pos, to;  // lane j < k: unit j's row and destination GPU
  float w;
};

template <int VPL>
__global__ void __launch_bounds__(kCbBwdWarps * 32, 16 / kCbBwdWarps) combine_bwd_pipe_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ Yl,
    const int32_t* __restrict__ pos, const float* __restrict__ w, int T, int k,
    __nv_bfloat16* __restrict__ dYl, float* __restrict__ dl, float* __restrict__ dl_rows_l, const P2P pp,
    int tok_blocks, PlanDev pad_plan) {
  constexpr int kRow = 32 * VPL;  // uint4 per row
  constexpr int d = VPL * 256;
  constexpr int S = kCbStages;
  extern __shared__ uint4 cb_ring[];  // [warp][S stages][dy, Y_0, Y_1][kRow]
  bool wrote_peer = false;
  if (static_cast<int>(blockIdx.x) >= tok_blocks) {  // trailing blocks: zero dYl's padding rows
    const int b = blockIdx.x - tok_blocks;
    zero_pad_segment(dYl, d, pad_plan, b / kPadParts, b % kPadParts, kPadParts, nullptr);
  } else {
    const int lane = threadIdx.x & 31;
    uint4* ring = cb_ring + (threadIdx.x >> 5) * (S * 3 * kRow);
    const int W = tok_blocks * kCbBwdWarps;
    // FM_CB_REVERSE: tokens last-to-first, so the first Y rows read are the
    // ones the combine forward (first-to-last, just before) left in L2
    auto tok = [&](int t) { return FM_CB_REVERSE ? T - 1 - t : t; };
    auto meta = [&](int t) {
      CbMeta m{0, -1, 0.0f};
      if (t < T) {
        unit_meta(pos, w, static_cast<size_t>(tok(t)) * k, k, lane, m.pos, m.w);
        m.to = unit_dst_of(pp, static_cast<size_t>(tok(t)) * k, k, lane);
      }
      return m;
    };
    auto fetch = [&](int t, int stage, const CbMeta& m) {
      if (t < T) {
        uint4* s = ring + stage * 3 * kRow;
        const uint4* g = reinterpret_cast<const uint4*>(dy + static_cast<size_t>(tok(t)) * d);
#pragma unroll
        for (int i = 0; i < VPL; ++i) cp_async16(s + lane + 32 * i, g + lane + 32 * i);
        for (int j = 0; j < k; ++j) {
          const int row = __shfl_sync(0xffffffffu, m.pos, j);
          const int to = __shfl_sync(0xffffffffu, m.to, j);
          if (row < 0) continue;
          const uint4* src = reinterpret_cast<const uint4*>(
              (to >= 0 ? reinterpret_cast<const __nv_bfloat16*>(pp.base[to] + pp.y_off) : Yl) +
              static_cast<size_t>(row) * d);
#pragma unroll
          for (int i = 0; i < VPL; ++i) cp_async16(s + (1 + j) * kRow + lane + 32 * i, src + lane + 32 * i);
        }
      }
      cp_async_commit();  // one group per call, empty or not: wait_group 1 counts calls
    };
    int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    CbMeta m[S];  // m[i]: token t + i*W (indices fixed after unrolling: registers)
#pragma unroll
    for (int i = 0; i < S - 1; ++i) {
      m[i] = meta(t + i * W);
      fetch(t + i * W, i, m[i]);
    }
    m[S - 1] = meta(t + (S - 1) * W);
    int stage = 0;
    for (; t < T; t += W) {
      const CbMeta after = meta(t + S * W);  // lands while this token computes
      fetch(t + (S - 1) * W, stage == 0 ? S - 1 : stage - 1, m[S - 1]);
      cp_async_wait<S - 1>();  // this lane's copies of token t are in shared memory
      const CbMeta& cur = m[0];
      const uint4* s = ring + stage * 3 * kRow;
      float my_dw = 0.0f;
      for (int j = 0; j < k; ++j) {
        const int row = __shfl_sync(0xffffffffu, cur.pos, j);
        const float wj = __shfl_sync(0xffffffffu, cur.w, j);
        if (row < 0) {
          if (lane == j) my_dw = 0.0f;
          continue;
        }
        const int to = __shfl_sync(0xffffffffu, cur.to, j);
        wrote_peer |= to >= 0 && to != pp.me;
        uint4* dst = reinterpret_cast<uint4*>(peer_rows(pp, pp.dy_off, to, dYl) + static_cast<size_t>(row) * d);
        float dot = 0.0f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const uint4 q = s[(1 + j) * kRow + lane + 32 * i], gv = s[lane + 32 * i];
          const uint32_t qs[4] = {q.x, q.y, q.z, q.w};
          const uint32_t gs[4] = {gv.x, gv.y, gv.z, gv.w};
          uint32_t o[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            dot = fmaf(bf16lo(gs[c]), bf16lo(qs[c]), dot);
            dot = fmaf(bf16hi(gs[c]), bf16hi(qs[c]), dot);
            o[c] = pack2(wj * bf16lo(gs[c]), wj * bf16hi(gs[c]));
          }
          dst[lane + 32 * i] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        dot = warp_sum(dot);
        if (lane == j) my_dw = dot;
      }
      float wdw = lane < k ? cur.w * my_dw : 0.0f;
      wdw = warp_sum(wdw);
      if (lane < k) {
        const float g_l = cur.w * (my_dw - wdw);
        dl[static_cast<size_t>(tok(t)) * k + lane] = g_l;
        float* dl_rows = peer_rows(pp, pp.dl_off, cur.to, dl_rows_l);
        if (dl_rows && cur.pos >= 0) dl_rows[cur.pos] = g_l;
      }
#pragma unroll
      for (int i = 0; i < S - 1; ++i) m[i] = m[i + 1];
      m[S - 1] = after;
      stage = stage + 1 == S ? 0 : stage + 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // no copy outstanding at exit
  }
  p2p_release_when_last(pp, wrote_peer);
}

// Pipelined combine forward (top_k <= 2, d <= 1024): as combine_bwd_pipe_kernel,
// each warp prefetches its next token's expert-output rows into shared memory
// while it sums the current one (same f32 fmaf order as combine_fwd_kernel).
template <int VPL>
__global__ void __launch_bounds__(kCbWarps * 32, 3) combine_fwd_pipe_kernel(
    const __nv_bfloat16* __restrict__ Yl, const int32_t* __restrict__ pos, const float* __restrict__ w, int T,
    int k, __nv_bfloat16* __restrict__ y, const P2P pp) {
  constexpr int kRow = 32 * VPL;
  constexpr int d = VPL * 256;
  extern __shared__ uint4 cf_ring[];  // [warp][2 stages][Y_0, Y_1][kRow]
  p2p_block_wait(pp);  // P2P: the expert GPUs' Y rows are complete
  const int lane = threadIdx.x & 31;
  uint4* ring = cf_ring + (threadIdx.x >> 5) * (2 * 2 * kRow);
  const int W = gridDim.x * kCbWarps;
  auto meta = [&](int t) {
    CbMeta m{0, -1, 0.0f};
    if (t < T) {
      unit_meta(pos, w, static_cast<size_t>(t) * k, k, lane, m.pos, m.w);
      m.to = unit_dst_of(pp, static_cast<size_t>(t) * k, k, lane);
    }
    return m;
  };
  auto fetch = [&](int t, int stage, const CbMeta& m) {
    if (t < T) {
      uint4* s = ring + stage * 2 * kRow;
      for (int j = 0; j < k; ++j) {
        const int row = __shfl_sync(0xffffffffu, m.pos, j);
        const int to = __shfl_sync(0xffffffffu, m.to, j);
        if (row < 0) continue;
        const uint4* src = reinterpret_cast<const uint4*>(
            (to >= 0 ? reinterpret_cast<const __nv_bfloat16*>(pp.base[to] + pp.y_off) : Yl) +
            static_cast<size_t>(row) * d);
#pragma unroll
        for (int i = 0; i < VPL; ++i) cp_async16(s + j * kRow + lane + 32 * i, src + lane + 32 * i);
      }
    }
    cp_async_commit();
  };
  int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  CbMeta cur = meta(t), nxt = meta(t + W);
  fetch(t, 0, cur);
  int stage = 0;
  for (; t < T; t += W) {
    const CbMeta after = meta(t + 2 * W);
    fetch(t + W, stage ^ 1, nxt);
    cp_async_wait1();
    const uint4* s = ring + stage * 2 * kRow;
    float acc[VPL][8];
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = 0.0f;
    for (int j = 0; j < k; ++j) {
      const int row = __shfl_sync(0xffffffffu, cur.pos, j);
      const float wj = __shfl_sync(0xffffffffu, cur.w, j);
      if (row < 0) continue;  // dropped units contribute nothing
      uint4 q[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) q[i] = s[j * kRow + lane + 32 * i];
      axpy_row<VPL>(acc, q, wj);
    }
    store_row<VPL>(y, t, d, lane, acc);
    cur = nxt;
    nxt = after;
    stage ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Pipelined dispatch (d <= 1024): each warp copies its next token's x row into
// shared memory (cp.async) and resolves that token's unit rows (lane j: unit j,
// the same rule as dispatch_token) while the current token's row copy is in
// flight, then writes the current token's k rows from shared memory.
template <int VPL>
__global__ void __launch_bounds__(256) dispatch_pipe_kernel(
    const __nv_bfloat16* __restrict__ x, int T, int k, int N, int G, int me, int direct,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ tile_rank, const int32_t* __restrict__ tile_base,
    PlanDev p, int32_t* __restrict__ pos_out, __nv_bfloat16* __restrict__ buf, int32_t* __restrict__ row_expert,
    const P2P pp, int tok_blocks, __nv_bfloat16* __restrict__ pad_buf) {
  constexpr int kRow = 32 * VPL;
  constexpr int d = VPL * 256;
  extern __shared__ uint4 dp_ring[];  // [warp][2 stages][kRow]
  bool wrote_peer = false;
  if (static_cast<int>(blockIdx.x) >= tok_blocks) {  // trailing blocks: zero pad_buf's padding rows
    const int b = blockIdx.x - tok_blocks;
    zero_pad_segment(pad_buf, d, p, b / kPadParts, b % kPadParts, kPadParts, row_expert);
  } else {
    const int lane = threadIdx.x & 31;
    uint4* ring = dp_ring + (threadIdx.x >> 5) * (2 * kRow);
    const int W = tok_blocks * (blockDim.x >> 5);
    const int shift = gate_tile_shift(N);
    auto route_units = [&](int t, int& row, int& to, int& e) {
      row = -1;
      to = -1;
      e = 0;
      if (t < T && lane < k) {
        const int u = t * k + lane;
        e = idx[u];
        const int r = tile_base[static_cast<size_t>(t >> shift) * N + e] + tile_rank[u];
        if (direct) {
          row = r < p.chunk_cnt[e] ? p.seg_start[p.local_index[e]] + r : -1;
        } else {
          for (int i = 0; i < G; ++i) {
            const int dst = (i == 0) ? me : (i <= me ? i - 1 : i);
            const int lo = p.chunk_lo[e * G + dst];
            if (r < lo + p.chunk_cnt[e * G + dst]) {
              row = pp.unit_dst ? p.peer_row[e * G + dst] + (r - lo) : p.send_off[e * G + dst] + (r - lo);
              to = dst;
              break;
            }
          }
        }
      }
    };
    auto fetch = [&](int t, int stage) {
      if (t < T) {
        const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * d);
#pragma unroll
        for (int i = 0; i < VPL; ++i) cp_async16(ring + stage * kRow + lane + 32 * i, src + lane + 32 * i);
      }
      cp_async_commit();
    };
    int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int row0, to0, e0;
    route_units(t, row0, to0, e0);
    fetch(t, 0);
    int stage = 0;
    for (; t < T; t += W) {
      fetch(t + W, stage ^ 1);
      int row1, to1, e1;
      route_units(t + W, row1, to1, e1);  // its loads overlap both rows' copies
      if (lane < k) {
        const int u = t * k + lane;
        pos_out[u] = row0;  // -1: dropped by the capacity rule (StaticEP)
        if (pp.unit_dst) pp.unit_dst[u] = row0 >= 0 ? to0 : -1;
        if (row_expert && row0 >= 0) row_expert[row0] = e0;
      }
      cp_async_wait1();
      uint4 v[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) v[i] = ring[stage * kRow + lane + 32 * i];
      for (int j = 0; j < k; ++j) {
        const int row = __shfl_sync(0xffffffffu, row0, j);
        const int to = __shfl_sync(0xffffffffu, to0, j);
        if (row < 0) continue;
        wrote_peer |= pp.unit_dst && to != pp.me;
        __nv_bfloat16* out = pp.unit_dst ? reinterpret_cast<__nv_bfloat16*>(pp.base[to] + pp.x_off) : buf;
        uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d);
#pragma unroll
        for (int i = 0; i < VPL; ++i) dst[lane + 32 * i] = v[i];
      }
      row0 = row1;
      to0 = to1;
      e0 = e1;
      stage ^= 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  p2p_release_when_last(pp, wrote_peer);
}

// dx[t] = sum_j dXbuf[pos[t,j]] + sum_j dl[t,j] * Wg[idx[t,j], :]
// P2P: dX rows are read from the expert's GPU (NVLink loads from its dX_perm).
template <int VPL>
__global__ void __launch_bounds__(256) unpermute_bwd_kernel(
    const __nv_bfloat16* __restrict__ dXl, const int32_t* __restrict__ pos,
    const int32_t* __restrict__ idx, const float* __restrict__ dl,
    const __nv_bfloat16* __restrict__ wg, int T, int k, int gate_grad,
    __nv_bfloat16* __restrict__ dx, const P2P pp) {
  p2p_block_wait(pp);  // P2P: the expert GPUs' dX rows are complete
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int d = VPL * 256;
  int my_pos, my_e;
  float my_dl;
  unit_meta(pos, gate_grad ? dl : nullptr, static_cast<size_t>(t) * k, k, lane, my_pos, my_dl);
  unit_meta(idx, nullptr, static_cast<size_t>(t) * k, k, lane, my_e, my_dl);
  if (gate_grad && lane < k) my_dl = __ldg(dl + static_cast<size_t>(t) * k + lane);
  const int my_to = unit_dst_of(pp, static_cast<size_t>(t) * k, k, lane);
  float acc[VPL][8];
#pragma unroll
  for (int i = 0; i < VPL; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[i][c] = 0.0f;
  for (int j = 0; j < k; j += 2) {
    const bool two = j + 1 < k;
    const int p0 = __shfl_sync(0xffffffffu, my_pos, j);
    const int p1 = __shfl_sync(0xffffffffu, my_pos, two ? j + 1 : j);
    const int to0 = __shfl_sync(0xffffffffu, my_to, j);
    const int to1 = __shfl_sync(0xffffffffu, my_to, two ? j + 1 : j);
    uint4 q0[VPL], q1[VPL];
    const bool h0 = p0 >= 0, h1 = two && p1 >= 0;
    if (h0) load_unit_row<VPL>(pp, pp.dx_off, to0, dXl, p0, d, lane, q0);
    if (h1) load_unit_row<VPL>(pp, pp.dx_off, to1, dXl, p1, d, lane, q1);
    if (h0) axpy_row<VPL>(acc, q0, 1.0f);
    if (h1) axpy_row<VPL>(acc, q1, 1.0f);
  }
  if (gate_grad) {
    for (int j = 0; j < k; ++j) {
      const int e = __shfl_sync(0xffffffffu, my_e, j);
      const float g_l = __shfl_sync(0xffffffffu, my_dl, j);
      uint4 q[VPL];
      load_row<VPL>(wg, e, d, lane, q);
      axpy_row<VPL>(acc, q, g_l);
    }
  }
  store_row<VPL>(dx, t, d, lane, acc);
}

// Gate-weight gradient over the NCCL send buffer (dispatch order: chunk
// (dst, e) of expert e's units for destination dst at send_off[e][dst], rows
// in rank order), deterministic: every chunk is cut into pieces of kPieceRows
// rows (piece table: an exclusive scan over the chunks in expert-major order),
// one block sums a piece in row order, and one pass per expert adds its pieces
// in table order: dwg[e] = sum over its (dst, piece) of dl_rows[r] * buf[r].
constexpr int kPieceRows = 512;

__global__ void piece_table_kernel(const int32_t* __restrict__ chunk_cnt, int N, int G,
                                   int32_t* __restrict__ piece_off) {
  extern __shared__ int32_t pt_s[];  // [N*G] counts, then [blockDim] scratch
  int32_t* scratch = pt_s + N * G;
  for (int j = threadIdx.x; j < N * G; j += blockDim.x)
    pt_s[j] = (chunk_cnt[j] + kPieceRows - 1) / kPieceRows;  // j = e * G + dst (expert-major)
  __syncthreads();
  const int total = block_exclusive_scan(pt_s, N * G, scratch);
  for (int j = threadIdx.x; j < N * G; j += blockDim.x) piece_off[j] = pt_s[j];
  if (threadIdx.x == 0) piece_off[N * G] = total;
}

__global__ void piece_sum_kernel(const __nv_bfloat16* __restrict__ buf, const float* __restrict__ dl_rows,
                                 const int32_t* __restrict__ send_off, const int32_t* __restrict__ chunk_cnt,
                                 const int32_t* __restrict__ piece_off, int N, int G, int d,
                                 float* __restrict__ partial) {
  const int b = blockIdx.x;
  const int nc = N * G;
  if (b >= piece_off[nc]) return;
  int lo = 0, hi = nc;  // chunk j with piece_off[j] <= b < piece_off[j + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (piece_off[mid] <= b) lo = mid; else hi = mid;
  }
  while (lo + 1 < nc && piece_off[lo + 1] <= b) ++lo;  // skip empty chunks
  const int e = lo / G, dst = lo % G;
  const int base = send_off[e * G + dst], cnt = chunk_cnt[e * G + dst];
  const int r0 = base + (b - piece_off[lo]) * kPieceRows, r1 = min(base + cnt, r0 + kPieceRows);
  const int c8 = threadIdx.x * 8;
  if (c8 >= d) return;
  float acc[8] = {};
  for (int r = r0; r < r1; ++r) {
    const float g = __ldg(dl_rows + r);
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(buf + static_cast<size_t>(r) * d + c8));
    const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] = fmaf(g, bf16lo(q[i]), acc[2 * i]);
      acc[2 * i + 1] = fmaf(g, bf16hi(q[i]), acc[2 * i + 1]);
    }
  }
  float4* dst4 = reinterpret_cast<float4*>(partial + static_cast<size_t>(b) * d + c8);
  dst4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  dst4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

__global__ void piece_reduce_kernel(const float* __restrict__ partial, const int32_t* __restrict__ piece_off,
                                    int G, int d, float* __restrict__ dwg) {
  const int e = blockIdx.y, col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  float s = 0.0f;
  for (int b = piece_off[e * G]; b < piece_off[(e + 1) * G]; ++b) s += partial[static_cast<size_t>(b) * d + col];
  dwg[static_cast<size_t>(e) * d + col] = s;
}

// Gate-weight gradient of the units the capacity rule dropped (no dispatch
// row): dWg[e] += sum over dropped units u = (t, j) of expert e of
// dl[u] * x[t], deterministic. Block (chunk c, expert e): the chunk's tokens
// ascending, thread = 8 columns (16-byte loads), partial[e][c][:]; then one
// fixed-order pass over the chunks adds the sum to dwg[e] (after the tile-sum
// reduce wrote it).
__global__ void dropped_gate_partial_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ pos,
                                            const int32_t* __restrict__ idx, const float* __restrict__ dl,
                                            int T, int d, int k, int chunk, int nchunks,
                                            float* __restrict__ partial) {
  const int c = blockIdx.x, e = blockIdx.y;
  const int c8 = threadIdx.x * 8;
  if (c8 >= d) return;
  float acc[8] = {};
  const int t1 = min(T, (c + 1) * chunk);
  for (int t = c * chunk; t < t1; ++t) {
    for (int j = 0; j < k; ++j) {
      const size_t u = static_cast<size_t>(t) * k + j;
      if (__ldg(idx + u) != e || __ldg(pos + u) >= 0) continue;
      const float g = __ldg(dl + u);
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * d + c8));
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] = fmaf(g, bf16lo(q[i]), acc[2 * i]);
        acc[2 * i + 1] = fmaf(g, bf16hi(q[i]), acc[2 * i + 1]);
      }
    }
  }
  float4* dst = reinterpret_cast<float4*>(partial + (static_cast<size_t>(e) * nchunks + c) * d + c8);
  dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

__global__ void dropped_gate_reduce_kernel(const float* __restrict__ partial, int nchunks, int d,
                                           float* __restrict__ dwg) {
  const int e = blockIdx.y, col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  const float* src = partial + static_cast<size_t>(e) * nchunks * d + col;
  float s = 0.0f;
  for (int c = 0; c < nchunks; ++c) s += src[static_cast<size_t>(c) * d];
  dwg[static_cast<size_t>(e) * d + col] += s;
}

// demand[e][g] = gathered[g][e]  (all-gathered per-GPU histograms -> TokenDemand layout)
__global__ void demand_transpose_kernel(const int64_t* __restrict__ gathered_GN, int N, int G,
                                        int64_t* __restrict__ demand_NG) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * G) return;
  const int e = i / G, g = i % G;
  demand_NG[i] = gathered_GN[static_cast<size_t>(g) * N + e];
}

// Per-128-row-tile column sums of permuted activations (expert segments are
// 128-row aligned, so a tile belongs to one expert): partial[tile][c] =
// sum over the tile's real rows r of w[r] * buf[r][c] (w = 1 when row_w is
// null). Job 0 / 1 in blockIdx.y (e.g. dWg from X_perm with dl per row, db2
// from dY_perm). Thread = 8 columns (16-byte loads), 32 rows in flight.
// Plain stores, then segment_tile_reduce: deterministic, no atomics.
struct TileSumJob {
  const __nv_bfloat16* buf;
  const float* row_w;
  float* partial;  // [tiles][cols]
};

__global__ void __launch_bounds__(256) segment_tile_colsum_kernel(TileSumJob j0, TileSumJob j1, int cols,
                                                                  PlanDev p, int Nl) {
  const TileSumJob jb = blockIdx.y == 0 ? j0 : j1;
  const int tile = blockIdx.x;
  if (tile >= p.mtile_prefix[Nl]) return;
  int lo = 0, hi = Nl;  // segment li with mtile_prefix[li] <= tile < mtile_prefix[li + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (p.mtile_prefix[mid] <= tile) lo = mid; else hi = mid;
  }
  while (lo + 1 < Nl && p.mtile_prefix[lo + 1] <= tile) ++lo;  // skip empty segments
  const int r0 = tile * kRowAlign;
  const int r1 = min(r0 + kRowAlign, p.seg_start[lo] + p.seg_real[lo]);  // pad rows carry nothing
  const int c8 = threadIdx.x * 8;
  if (c8 >= cols) return;
  float acc[8] = {};
  // 32 rows in flight: a block's 128 rows are 4 dependent DRAM round trips
  // (8 in flight: 16), which matters when few tiles fill the GPU (top-1)
  constexpr int kB = 32;
  for (int rb = r0; rb < r1; rb += kB) {
    uint4 v[kB];
    float w[kB];
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int r = min(rb + i, r1 - 1);
      v[i] = __ldg(reinterpret_cast<const uint4*>(jb.buf + static_cast<size_t>(r) * cols + c8));
      w[i] = rb + i < r1 ? (jb.row_w ? __ldg(jb.row_w + r) : 1.0f) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const uint32_t q[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[2 * c] = fmaf(w[i], bf16lo(q[c]), acc[2 * c]);
        acc[2 * c + 1] = fmaf(w[i], bf16hi(q[c]), acc[2 * c + 1]);
      }
    }
  }
  float4* dst = reinterpret_cast<float4*>(jb.partial + static_cast<size_t>(tile) * cols + c8);
  dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

// out[oi(li)][col] = sum over the 128-row tiles of segment li of partial[tile][col]
// (fixed order: deterministic); oi = out_index[li] (null: li). Up to three
// jobs in blockIdx.z.
struct TileReduceJob {
  const float* partial;
  int cols;
  const int32_t* out_index;
  float* out;
};

__global__ void segment_tile_reduce_kernel(TileReduceJob j0, TileReduceJob j1, TileReduceJob j2, PlanDev p) {
  const TileReduceJob jb = blockIdx.z == 0 ? j0 : (blockIdx.z == 1 ? j1 : j2);
  // block: 32 columns x 8 tile lanes; lane j sums tiles t0+j, t0+j+8, ...; the
  // eight partial sums are combined in fixed order (deterministic).
  __shared__ float part[8][33];
  const int li = blockIdx.x;
  const int cx = threadIdx.x & 31, j = threadIdx.x >> 5;
  const int col = blockIdx.y * 32 + cx;
  if (blockIdx.y * 32 >= jb.cols) return;
  const int t0 = p.mtile_prefix[li], t1 = p.mtile_prefix[li + 1];
  float acc = 0.0f;
  if (col < jb.cols) {
    // eight loads in flight, added in tile order (the same sum as one at a time)
    const float* src = jb.partial + col;
    const size_t ld = static_cast<size_t>(jb.cols);
    int t = t0 + j;
    for (; t + 56 < t1; t += 64) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + static_cast<size_t>(t + 8 * u) * ld);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; t < t1; t += 8) acc += __ldg(src + static_cast<size_t>(t) * ld);
  }
  part[j][cx] = acc;
  __syncthreads();
  if (j == 0 && col < jb.cols) {
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += part[i][cx];
    const int oi = jb.out_index ? jb.out_index[li] : li;
    jb.out[static_cast<size_t>(oi) * jb.cols + col] = s;
  }
}

}  // namespace

// ----------------------------------------------------------------- P2P flags
// Arrival flags live in every GPU's arena: flags[slot][src] = last epoch in
// which `src` completed exchange `slot` towards this GPU. Epochs only grow, so
// nothing is ever reset and a stale flag can never satisfy a newer wait.
__global__ void p2p_signal_kernel(const P2P pp, int G, int me, int slot, unsigned long long epoch) {
  const int dst = threadIdx.x;
  if (dst >= G) return;
  __threadfence_system();  // this stream's earlier writes (kernels before) are visible first
  unsigned long long* f =
      reinterpret_cast<unsigned long long*>(pp.base[dst] + pp.flag_off) + slot * kMaxPeers + me;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
}


// ------------------------------------------------------------------ launchers
int gate_wgrad_pieces(int rows, int N, int G) { return (rows + kPieceRows - 1) / kPieceRows + N * G; }

// dWg over the NCCL send buffer (see piece_sum_kernel); partial holds
// gate_wgrad_pieces(max_rows, N, G) rows of d floats plus N*G+1 ints.
void launch_gate_wgrad(const void* buf, int max_rows, int d, const float* dl_rows, const PlanDev& p, int N,
                       int G, float* partial, float* dwg, cudaStream_t s) {
  if (max_rows <= 0) {
    FM_CUDA(cudaMemsetAsync(dwg, 0, sizeof(float) * N * d, s));
    return;
  }
  if (d % 8 != 0 || d > 8 * 1024) throw std::invalid_argument("gate wgrad: d % 8 == 0, d <= 8192");
  const int pieces = gate_wgrad_pieces(max_rows, N, G);
  int32_t* piece_off = reinterpret_cast<int32_t*>(partial + static_cast<size_t>(pieces) * d);
  constexpr int kT = 256;
  const int tsmem = (N * G + kT) * 4;
  ensure_dynamic_smem(reinterpret_cast<const void*>(piece_table_kernel), tsmem);
  piece_table_kernel<<<1, kT, tsmem, s>>>(p.chunk_cnt, N, G, piece_off);
  FM_LAUNCH_CHECK("piece_table_kernel");
  piece_sum_kernel<<<pieces, ((d / 8 + 31) / 32) * 32, 0, s>>>(static_cast<const __nv_bfloat16*>(buf), dl_rows,
                                                               p.send_off, p.chunk_cnt, piece_off, N, G, d, partial);
  FM_LAUNCH_CHECK("piece_sum_kernel");
  piece_reduce_kernel<<<dim3((d + 255) / 256, N), 256, 0, s>>>(partial, piece_off, G, d, dwg);
  FM_LAUNCH_CHECK("piece_reduce_kernel");
}

int dropped_gate_chunks(int T) { return std::max(1, std::min(128, (T + 255) / 256)); }

void launch_dropped_gate_wgrad(const void* x, const int32_t* pos, const int32_t* idx, const float* dl,
                               int T, int d, int k, int N, float* partial, float* dwg, cudaStream_t s) {
  if (T <= 0) return;
  if (d % 8 != 0 || d > 8 * 1024) throw std::invalid_argument("dropped gate wgrad: d % 8 == 0, d <= 8192");
  const int nchunks = dropped_gate_chunks(T);
  const int chunk = (T + nchunks - 1) / nchunks;
  dropped_gate_partial_kernel<<<dim3(nchunks, N), ((d / 8 + 31) / 32) * 32, 0, s>>>(
      static_cast<const __nv_bfloat16*>(x), pos, idx, dl, T, d, k, chunk, nchunks, partial);
  FM_LAUNCH_CHECK("dropped_gate_partial_kernel");
  dropped_gate_reduce_kernel<<<dim3((d + 255) / 256, N), 256, 0, s>>>(partial, nchunks, d, dwg);
  FM_LAUNCH_CHECK("dropped_gate_reduce_kernel");
}

void launch_demand_transpose(const int64_t* gathered_GN, int N, int G, int64_t* demand_NG,
                             cudaStream_t s) {
  demand_transpose_kernel<<<(N * G + 255) / 256, 256, 0, s>>>(gathered_GN, N, G, demand_NG);
  FM_LAUNCH_CHECK("demand_transpose_kernel");
}

// Column sums per 128-row tile of up to two permuted buffers (null buf: job off).
void launch_segment_tile_colsum(const void* buf0, const float* w0, float* partial0, const void* buf1,
                                const float* w1, float* partial1, int cols, const PlanDev& p, int Nl,
                                int max_tiles, cudaStream_t s) {
  if (Nl <= 0 || max_tiles <= 0 || (!buf0 && !buf1)) return;
  if (cols % 8 != 0 || cols > 8 * 256) throw std::invalid_argument("segment tile colsum: cols % 8 == 0, <= 2048");
  TileSumJob j[2] = {{static_cast<const __nv_bfloat16*>(buf0), w0, partial0},
                     {static_cast<const __nv_bfloat16*>(buf1), w1, partial1}};
  const int nj = (buf0 ? 1 : 0) + (buf1 ? 1 : 0);
  if (!buf0) j[0] = j[1];
  const int threads = ((cols / 8 + 31) / 32) * 32;
  segment_tile_colsum_kernel<<<dim3(max_tiles, nj), threads, 0, s>>>(j[0], j[1], cols, p, Nl);
  FM_LAUNCH_CHECK("segment_tile_colsum_kernel");
}

// Up to three reductions of per-tile partials into per-segment rows (null out: off).
void launch_segment_tile_reduce(const float* partial0, int cols0, const int32_t* idx0, float* out0,
                                const float* partial1, int cols1, const int32_t* idx1, float* out1,
                                const float* partial2, int cols2, const int32_t* idx2, float* out2,
                                const PlanDev& p, int Nl, cudaStream_t s) {
  if (Nl <= 0) return;
  TileReduceJob all[3] = {{partial0, cols0, idx0, out0}, {partial1, cols1, idx1, out1},
                          {partial2, cols2, idx2, out2}};
  TileReduceJob use[3];
  int n = 0, maxc = 0;
  for (const auto& j : all)
    if (j.out) {
      use[n++] = j;
      maxc = std::max(maxc, j.cols);
    }
  if (n == 0) return;
  for (int i = n; i < 3; ++i) use[i] = use[0];
  dim3 grid(Nl, (maxc + 31) / 32, n);
  segment_tile_reduce_kernel<<<grid, 256, 0, s>>>(use[0], use[1], use[2], p);
  FM_LAUNCH_CHECK("segment_tile_reduce_kernel");
}

void launch_expert_scan(const int32_t* tile_counts, int num_tiles, int N, int32_t* tile_base,
                        int64_t* hist, int64_t* demand_NG, int G, int me, cudaStream_t s) {
  expert_scan_kernel<<<N, 256, 0, s>>>(tile_counts, num_tiles, N, tile_base, hist, demand_NG, G, me);
  FM_LAUNCH_CHECK("expert_scan_kernel");
}

bool plan_can_fuse_scan(int N, int G, int num_tiles) {
#ifdef FM_NO_PLAN_SCAN  // A/B knob: the expert scan always as its own kernel
  return false;
#endif
  if (G != 1 || N > 256) return false;
  int tpe = 256 / N;
  tpe = tpe >= 32 ? 32 : tpe >= 16 ? 16 : tpe >= 8 ? 8 : tpe >= 4 ? 4 : tpe >= 2 ? 2 : 1;
  return (num_tiles + tpe - 1) / tpe <= kPlanScanRun;
}

void launch_plan(int64_t* flows, int N, int G, int me, const int32_t* local_expert, int Nl,
                 const PlanDev& p, cudaStream_t s, const int32_t* counts, const int64_t* demand,
                 int32_t* status, const int64_t* gathered_GN, const int32_t* scan_tile_counts,
                 int scan_num_tiles, int32_t* scan_tile_base, int64_t* scan_hist) {
  if (gathered_GN && !demand) throw std::invalid_argument("plan: the transposed demand needs a demand buffer");
  const PlanScan scan{scan_tile_counts, scan_num_tiles, scan_tile_base, scan_hist};
  if (scan.tile_counts && (!demand || gathered_GN || !plan_can_fuse_scan(N, G, scan_num_tiles)))
    throw std::invalid_argument("plan: the fused expert scan needs G == 1, <= 32 tiles per thread and a demand");
  if (demand && (N > 256 || G > kMaxGpus)) throw std::invalid_argument("route: bad dimensions");
  constexpr int kPlanThreads = 256;
  // the flows are staged in shared memory when they fit; beyond that (e.g.
  // 256 experts on 64 GPUs: 4 MB of flows) the kernel reads them from global
  // memory (L2-resident) and shared memory holds only the scan buffers
  const int base = (3 * Nl + 2 * N * G + kPlanThreads) * 4;
  const bool flows_in_smem = base + N * G * G * 4 <= 200 * 1024;
  const int smem = base + (flows_in_smem ? N * G * G * 4 : 0);
  if (smem > 200 * 1024) throw std::invalid_argument("plan: num_experts * num_gpus too large");
  if (flows_in_smem) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(plan_kernel<true>), smem);
    plan_kernel<true><<<1, kPlanThreads, smem, s>>>(flows, N, G, me, local_expert, Nl, p, counts, demand, status,
                                                    gathered_GN, scan);
  } else {
    ensure_dynamic_smem(reinterpret_cast<const void*>(plan_kernel<false>), smem);
    plan_kernel<false><<<1, kPlanThreads, smem, s>>>(flows, N, G, me, local_expert, Nl, p, counts, demand, status,
                                                     gathered_GN, scan);
  }
  FM_LAUNCH_CHECK("plan_kernel");
}

// Blocks of `kern` resident on the whole GPU at `threads` per block (cached
// per kernel): the grid of the token-striding kernels.
int resident_grid(const void* kern, int threads) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;  // (device, kernel) -> grid
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, kern});
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  FM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0));
  const int grid = std::max(1, per_sm) * num_sms();
  cache.emplace(std::make_pair(dev, kern), grid);
  return grid;
}

void launch_zero_pad(void* buf, int d, const PlanDev& p, int Nl, int32_t* row_expert, cudaStream_t s) {
  if (Nl <= 0) return;
  dim3 grid(kPadParts, Nl);
  zero_pad_kernel<<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(buf), d, p, Nl, row_expert);
  FM_LAUNCH_CHECK("zero_pad_kernel");
}

void launch_relayout(void* recv, void* perm, int d, int G, int Nl, const PlanDev& p, int max_rows,
                     int dir, cudaStream_t s) {
  if (max_rows <= 0) return;
  const int warps = 8;
  relayout_kernel<<<(max_rows + warps - 1) / warps, warps * 32, 0, s>>>(
      static_cast<__nv_bfloat16*>(recv), static_cast<__nv_bfloat16*>(perm), d, G, Nl, p, dir);
  FM_LAUNCH_CHECK("relayout_kernel");
}

#define FM_VPL_DISPATCH(d, KERNEL_CALL)                                  \
  switch ((d) / 256) {                                                   \
    case 1: { constexpr int V = 1; KERNEL_CALL; break; }                 \
    case 2: { constexpr int V = 2; KERNEL_CALL; break; }                 \
    case 3: { constexpr int V = 3; KERNEL_CALL; break; }                 \
    case 4: { constexpr int V = 4; KERNEL_CALL; break; }                 \
    case 6: { constexpr int V = 6; KERNEL_CALL; break; }                 \
    case 8: { constexpr int V = 8; KERNEL_CALL; break; }                 \
    default: throw std::invalid_argument("d_model must be 256*{1,2,3,4,6,8}"); \
  }

// Resident blocks per SM of a pipelined gather kernel at its dynamic shared
// memory (sets the attribute; cached per device and kernel).
int pipe_blocks_per_sm(const void* kern, int threads, int smem) {
  ensure_dynamic_smem(kern, smem);
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, kern});
  if (it == cache.end()) {
    int n = 0;
    FM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem));
    it = cache.emplace(std::make_pair(dev, kern), std::max(1, n)).first;
  }
  return it->second;
}

// The pipelined dispatch (V <= 4): one resident wave of warps.
template <int V>
bool launch_dispatch_pipe(const void* x, int T, int k, int N, int G, int me, bool direct, const int32_t* idx,
                          const int32_t* tile_rank, const int32_t* tile_base, const PlanDev& p, int32_t* pos,
                          void* buf, int32_t* row_expert, cudaStream_t s, const P2P& pp, void* pad_buf, int Nl) {
  if constexpr (V > 4) {
    return false;
  } else {
    const void* kern = reinterpret_cast<const void*>(dispatch_pipe_kernel<V>);
    const int smem = 8 * 2 * 32 * V * 16;
    const int per_sm = pipe_blocks_per_sm(kern, 256, smem);
    const int tok_blocks = std::min((std::max(T, 0) + 7) / 8, per_sm * num_sms());
    const int pad_blocks = pad_buf ? Nl * kPadParts : 0;
    if (tok_blocks + pad_blocks == 0) return true;
    dispatch_pipe_kernel<V><<<tok_blocks + pad_blocks, 256, smem, s>>>(
        static_cast<const __nv_bfloat16*>(x), T, k, N, G, me, direct ? 1 : 0, idx, tile_rank, tile_base, p, pos,
        static_cast<__nv_bfloat16*>(buf), row_expert, pp, tok_blocks, static_cast<__nv_bfloat16*>(pad_buf));
    FM_LAUNCH_CHECK("dispatch_pipe_kernel");
    return true;
  }
}


void launch_dispatch(const void* x, int T, int d, int k, int N, int G, int me, bool direct,
                     const int32_t* idx, const int32_t* tile_rank, const int32_t* tile_base,
                     const PlanDev& p, int32_t* pos, void* buf, int32_t* row_expert,
                     cudaStream_t s, const P2P* pp, void* pad_buf, int Nl) {
  const P2P none = no_p2p();
  if (d % 8 != 0 || d > 2048) throw std::invalid_argument("dispatch: d_model must be a multiple of 8, <= 2048");
#if FM_DISPATCH_PIPE
  if (d % 256 == 0 && d <= 1024 && k <= 32) {
    bool launched = false;
    FM_VPL_DISPATCH(d, (launched = launch_dispatch_pipe<V>(x, T, k, N, G, me, direct, idx, tile_rank, tile_base,
                                                           p, pos, buf, row_expert, s, pp ? *pp : none,
                                                           pad_buf, Nl)));
    if (launched) return;
  }
#endif
  const int warps = 8;
  // P2P pushes: one resident wave striding over the tokens, so each block's
  // system-scope release is paid once per block rather than per 8 tokens
  int tok_blocks = (std::max(T, 0) + warps - 1) / warps;
  if (pp && pp->signal_slot >= 0)
    tok_blocks = std::min(tok_blocks, resident_grid(reinterpret_cast<const void*>(dispatch_kernel), warps * 32));
  const int pad_blocks = pad_buf ? Nl * kPadParts : 0;
  if (tok_blocks + pad_blocks == 0) return;
  dispatch_kernel<<<tok_blocks + pad_blocks, warps * 32, 0, s>>>(
      static_cast<const __nv_bfloat16*>(x), T, d, k, N, G, me, direct ? 1 : 0, idx, tile_rank,
      tile_base, p, pos, static_cast<__nv_bfloat16*>(buf), row_expert, pp ? *pp : none, tok_blocks,
      static_cast<__nv_bfloat16*>(pad_buf), Nl);
  FM_LAUNCH_CHECK("dispatch_kernel");
}

// The pipelined combine forward (V <= 4): one resident wave of warps.
template <int V>
bool launch_combine_fwd_pipe(const void* Y, const int32_t* pos, const float* w, int T, int k, void* y,
                             cudaStream_t s, const P2P& pp) {
  if constexpr (V > 4) {
    return false;
  } else {
    const void* kern = reinterpret_cast<const void*>(combine_fwd_pipe_kernel<V>);
    const int smem = kCbWarps * 2 * 2 * 32 * V * 16;
    const int per_sm = pipe_blocks_per_sm(kern, kCbWarps * 32, smem);
    const int grid = std::min((T + kCbWarps - 1) / kCbWarps, per_sm * num_sms());
    combine_fwd_pipe_kernel<V><<<grid, kCbWarps * 32, smem, s>>>(
        static_cast<const __nv_bfloat16*>(Y), pos, w, T, k, static_cast<__nv_bfloat16*>(y), pp);
    FM_LAUNCH_CHECK("combine_fwd_pipe_kernel");
    return true;
  }
}

void launch_combine_fwd(const void* Y, const int32_t* pos, const float* w, int T, int d, int k,
                        void* y, cudaStream_t s, const P2P* pp) {
  const P2P none = no_p2p();
  if (T <= 0) return;
  if (d % 256 != 0) throw std::invalid_argument("combine: d_model must be a multiple of 256");
#if FM_COMBINE_FWD_PIPE
  if (k <= (FM_COMBINE_FWD_PIPE == 1 ? 2 : 1) && d <= 1024) {
    bool launched = false;
    FM_VPL_DISPATCH(d, (launched = launch_combine_fwd_pipe<V>(Y, pos, w, T, k, y, s, pp ? *pp : none)));
    if (launched) return;
  }
#endif
  const int warps = 8;
  const int grid = (T + warps - 1) / warps;
  FM_VPL_DISPATCH(d, (combine_fwd_kernel<V><<<grid, warps * 32, 0, s>>>(
                         static_cast<const __nv_bfloat16*>(Y), pos, w, T, k,
                         static_cast<__nv_bfloat16*>(y), pp ? *pp : none)));
  FM_LAUNCH_CHECK("combine_fwd_kernel");
}

// The pipelined combine backward (V <= 4): one resident wave of warps striding
// over the tokens, so every warp pipelines across its tokens.
template <int V>
bool launch_combine_bwd_pipe(const void* dy, const void* Y, const int32_t* pos, const float* w, int T, int k,
                             void* dYbuf, float* dl, float* dl_rows, cudaStream_t s, const P2P& pp,
                             int pad_blocks, const PlanDev& pad_plan) {
  if constexpr (V > 4) {
    return false;
  } else {
    const void* kern = reinterpret_cast<const void*>(combine_bwd_pipe_kernel<V>);
    const int smem = kCbBwdWarps * kCbStages * 3 * 32 * V * 16;
    const int per_sm = pipe_blocks_per_sm(kern, kCbBwdWarps * 32, smem);
    const int tok_blocks = std::min((std::max(T, 0) + kCbBwdWarps - 1) / kCbBwdWarps, per_sm * num_sms());
    if (tok_blocks + pad_blocks == 0) return true;
    combine_bwd_pipe_kernel<V><<<tok_blocks + pad_blocks, kCbBwdWarps * 32, smem, s>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(Y), pos, w, T, k,
        static_cast<__nv_bfloat16*>(dYbuf), dl, dl_rows, pp, tok_blocks, pad_plan);
    FM_LAUNCH_CHECK("combine_bwd_pipe_kernel");
    return true;
  }
}

void launch_combine_bwd(const void* dy, const void* Y, const int32_t* pos, const float* w, int T,
                        int d, int k, void* dYbuf, float* dl, float* dl_rows, cudaStream_t s, const P2P* pp,
                        const PlanDev* pad_plan, int Nl) {
  const P2P none = no_p2p();
  if (k > 32) throw std::invalid_argument("combine_bwd: top_k <= 32");
  const int warps = 8;
  const int pad_blocks = pad_plan ? Nl * kPadParts : 0;
  const PlanDev nop{};
#if FM_COMBINE_BWD_PIPE
  if (k <= 2 && d <= 1024) {
    bool launched = false;
    FM_VPL_DISPATCH(d, (launched = launch_combine_bwd_pipe<V>(dy, Y, pos, w, T, k, dYbuf, dl, dl_rows, s,
                                                              pp ? *pp : none, pad_blocks,
                                                              pad_plan ? *pad_plan : nop)));
    if (launched) return;
  }
#endif
  int tok_blocks = (std::max(T, 0) + warps - 1) / warps;
  if (pp && pp->signal_slot >= 0)  // P2P pushes: one resident wave (see launch_dispatch)
    FM_VPL_DISPATCH(d, (tok_blocks = std::min(tok_blocks, resident_grid(
                                                  reinterpret_cast<const void*>(combine_bwd_kernel<V>), warps * 32))));
  if (tok_blocks + pad_blocks == 0) return;
  FM_VPL_DISPATCH(d, (combine_bwd_kernel<V><<<tok_blocks + pad_blocks, warps * 32, 0, s>>>(
                         static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(Y),
                         pos, w, T, k, static_cast<__nv_bfloat16*>(dYbuf), dl, dl_rows, pp ? *pp : none,
                         tok_blocks, pad_plan ? *pad_plan : nop)));
  FM_LAUNCH_CHECK("combine_bwd_kernel");
}

void launch_unpermute_bwd(const void* dXbuf, const int32_t* pos, const int32_t* idx, const float* dl,
                          const void* wg, int T, int d, int k, bool gate_grad, void* dx,
                          cudaStream_t s, const P2P* pp) {
  const P2P none = no_p2p();
  if (T <= 0) return;
  const int warps = 8;
  const int grid = (T + warps - 1) / warps;
  FM_VPL_DISPATCH(d, (unpermute_bwd_kernel<V><<<grid, warps * 32, 0, s>>>(
                         static_cast<const __nv_bfloat16*>(dXbuf), pos, idx, dl,
                         static_cast<const __nv_bfloat16*>(wg), T, k, gate_grad ? 1 : 0,
                         static_cast<__nv_bfloat16*>(dx), pp ? *pp : none)));
  FM_LAUNCH_CHECK("unpermute_bwd_kernel");
}


void launch_p2p_signal(const P2P& pp, int G, int me, int slot, unsigned long long epoch, cudaStream_t s) {
  p2p_signal_kernel<<<1, 64, 0, s>>>(pp, G, me, slot, epoch);
  FM_LAUNCH_CHECK("p2p_signal_kernel");
}


}  // namespace fm
