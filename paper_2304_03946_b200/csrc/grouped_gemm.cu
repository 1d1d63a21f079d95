// Grouped bf16 GEMM on tcgen05 / TMEM, fed by TMA — the expert FFN of the
// FlexMoE layer (Eq. 2) forward and backward.
//
// The reference models this contraction as `compute_cost = tokens / TPS`
// (proj/src/cost_model.cpp:30-35); here it is the one real dense op.
//
// Layout contract: tokens of each local expert ("group") are
// contiguous in the permuted buffers, every group padded to a multiple of
// 128 rows with zero rows. Two schedules share one kernel body:
//   kRows  : token rows are GEMM-M  (fwd1, fwd2, dgrad1, dgrad2)
//            C[g][rows, N] = A[rows, K] . B_g      (K fixed)
//   kWgrad : token rows are GEMM-K  (wgrad)
//            C[g][M_w, N]  = A[rows_g, M_w]^T . B[rows_g, N]
//
// Warp roles (256 threads, one CTA per SM, persistent over tiles):
//   warp 0  : TMA producer (one elected lane)
//   warp 1  : MMA issuer   (one elected lane), 128x256x16 UMMA, f32 in TMEM
//   warp 2  : TMEM allocator (512 columns = two 128x256 f32 accumulators)
//   warps 4-7: epilogue — tcgen05.ld, bias / ReLU / ReLU-mask, store.
// Smem ring: 4 stages x (A 16 KB + B 32 KB) for single CTAs; 6 x (16 + 16 KB)
// per CTA for CTA pairs (cta_group::2, 256x256 tiles).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "fm_internal.h"
#include "layer_plan.h"
#include "sm100_ptx.cuh"

namespace fm {
namespace gemm {

constexpr int kBM = 128;  // rows per CTA (one TMEM lane per row)
constexpr int kBN = 256;  // output columns per tile
constexpr int kBK = 64;
constexpr int kABytes = kBM * kBK * 2;
constexpr int kTmemCols = 512;
// Epilogue staging: per epilogue warp two 32-row x 64-byte buffers (SWIZZLE_64B
// TMA store boxes).
constexpr int kStageOutBytes = 32 * 64;
constexpr int kMaxGroups = 256;
constexpr int kTableInts = kMaxGroups + 4;  // one smem schedule table (groups + 1, padded)
constexpr uint32_t kMnChunkBytes = kBK * 128;  // one 64-wide MN chunk of a stage (8 KB)

// CG = CTAs per MMA: 1 (128x256 tile per CTA) or 2 (CTA pair, 256x256 tile,
// cta_group::2: each CTA stages its 128 rows of A and half of B's 256 columns,
// the leader issues the MMA, each CTA holds its 128 rows of the accumulator).
// Epilogue warps EW: 4 (one per TMEM lane quarter, all 256 columns) or 8 (two
// per quarter, 128 columns each) — the CTA-pair kernel has the smem for the
// second set, which doubles the epilogue's latency hiding.
template <int CG>
struct Cfg {
  static constexpr int kBNc = kBN / CG;              // B rows (N) staged per CTA
  static constexpr int kBBytes = kBNc * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // CTA pairs: 6 stages (~2.2 us of MMA work in flight at power-capped clocks,
  // enough to cover TMA load latency while the epilogue's stores share the
  // TMA unit), paid for with one output staging buffer per epilogue warp.
  static constexpr int kStages = CG == 1 ? 4 : 6;
  static constexpr int kOutBufs = CG == 1 ? 2 : 1;
  static constexpr int kTileM = kBM * CG;
  static constexpr int kEW = CG == 1 ? 4 : 8;
  static constexpr int kThreads = 128 + 32 * kEW;
  static constexpr int kOutBytes = kEW * kOutBufs * kStageOutBytes;
  static constexpr int kSmemBytes = kStages * kStageBytes + kOutBytes + 1024 + 512 + 2 * kBN * 4 +
                                    2 * 4 * kBN * 4 + 4 * kTableInts * 4;
};

enum Schedule { kRows = 0, kWgrad = 1 };
enum Epilogue { kEpiBiasRelu = 0, kEpiBias = 1, kEpiReluMask = 2, kEpiNone = 3, kEpiF32 = 4 };

struct Args {
  int num_groups;
  const int* seg_start;    // [groups] first token row of the group (padded layout)
  const int* seg_rows;     // [groups] rows of the group, multiple of 128
  const int* tile_prefix;  // [groups+1] kRows: exclusive prefix of 128-row M-tiles
  int M_w;                 // kWgrad: output rows per group
  int N;                   // output columns
  int K;                   // kRows: reduction depth
  int b_rows_per_group;    // kRows: B tensor-map rows between consecutive groups
  void* out;
  int ldc;
  const float* bias;  // [b groups][N]
  // kRows (optional, device [groups]): row of group g's weights / bias in the
  // B operand (an expert-state slot); null = g. Placement changes rewrite this
  // table instead of moving weights.
  const int* b_slot;
  uint32_t* mask;     // ReLU bits [rows][N/32]: written by kEpiBiasRelu, read by kEpiReluMask
  float* colsum;      // kEpiReluMask (optional): per-128-row-tile column sums [mtiles][N]
  // P2P arrival gating (kRows, optional): before loading the A rows of global
  // 128-row tile m, the producer waits until every source s in
  // tile_src_mask[m] has published arrive_flags[s] >= epoch (rows pushed by
  // peers over NVLink) — compute on early tiles overlaps later arrivals.
  const unsigned long long* arrive_flags;
  const unsigned long long* tile_src_mask;
  unsigned long long epoch;
  int* arrive_err;
  // kWgrad: the first gemm_clusters clusters run the tiles; the rest run the
  // side job (per-tile column sums, memory-bound) concurrently on their SMs
  int gemm_clusters;
  SideJob side;
  // P2P "ready" signal (optional, ready.signal_slot >= 0): once every CTA's
  // output stores completed, the last CTA publishes flags[slot][me] = epoch
  // to every peer (what p2p_signal_kernel does one launch later)
  P2P ready;
};

// kernel parameters = 3 tensor maps + Args (SideJob carries a P2P struct)
static_assert(sizeof(Args) + 3 * sizeof(CUtensorMap) <= 4096, "grouped GEMM kernel parameters exceed 4 KB");

// Side role of a wgrad launch: the tile column sums of SideJob, one thread
// group of cols/8 threads per (job, 128-row tile) item, 16 rows in flight.
template <int THREADS>
__device__ __forceinline__ void colsum_side(const SideJob& sd, int cta, int num_ctas) {
  const int gt = sd.cols / 8;  // threads per item (one 16-byte column vector each)
  const int groups = THREADS / gt;
  const int grp = static_cast<int>(threadIdx.x) / gt, c8 = (static_cast<int>(threadIdx.x) % gt) * 8;
  if (grp >= groups) return;
  const int ntiles = sd.mtile_prefix[sd.Nl];
  const int items = sd.njobs * ntiles;
  for (int it = cta * groups + grp; it < items; it += num_ctas * groups) {
    const int j = it / ntiles, tile = it - j * ntiles;
    const __nv_bfloat16* buf = static_cast<const __nv_bfloat16*>(sd.buf[j]);
    const float* row_w = sd.row_w[j];
    int lo = 0, hi = sd.Nl;  // segment with mtile_prefix[lo] <= tile < mtile_prefix[lo + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (sd.mtile_prefix[mid] <= tile) lo = mid; else hi = mid;
    }
    while (lo + 1 < sd.Nl && sd.mtile_prefix[lo + 1] <= tile) ++lo;  // skip empty segments
    const int r0 = tile * kBM;
    const int r1 = min(r0 + kBM, sd.seg_start[lo] + sd.seg_real[lo]);  // pad rows carry nothing
    float acc[8] = {};
    constexpr int kB = 16;
    for (int rb = r0; rb < r1; rb += kB) {
      uint4 v[kB];
      float w[kB];
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int r = min(rb + i, r1 - 1);
        v[i] = __ldg(reinterpret_cast<const uint4*>(buf + static_cast<size_t>(r) * sd.cols + c8));
        w[i] = rb + i < r1 ? (row_w ? __ldg(row_w + r) : 1.0f) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const uint32_t q[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[2 * c] = fmaf(w[i], __uint_as_float(q[c] << 16), acc[2 * c]);
          acc[2 * c + 1] = fmaf(w[i], __uint_as_float(q[c] & 0xffff0000u), acc[2 * c + 1]);
        }
      }
    }
    float4* dst = reinterpret_cast<float4*>(sd.partial[j] + static_cast<size_t>(tile) * sd.cols + c8);
    dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// Producer-side wait for the sources of one A tile (acquire at system scope,
// then a proxy fence so the TMA (async proxy) reads see the peers' stores).
__device__ __forceinline__ void wait_tile_sources(const Args& a, int mtile) {
  unsigned long long mask = a.tile_src_mask[mtile];
  if (!mask) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (mask) {
    const int src = __ffsll(static_cast<long long>(mask)) - 1;
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.arrive_flags + src) : "memory");
    if (v >= a.epoch) {
      mask &= mask - 1;
      continue;
    }
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - t0 > 20000000000ull) {  // bounded: report instead of hanging
      atomicExch(a.arrive_err, 1);
      break;
    }
    __nanosleep(128);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// A/B knob: wgrad's f32 output stored with an L2 evict-first policy. Measured
// and rejected (profiles/r02_gate_context.log): the next kernel pays the same
// dirty-line write-back either way.
#ifndef FM_WGRAD_STORE_HINT
#define FM_WGRAD_STORE_HINT 0
#endif
#ifndef FM_WGRAD_HINT
#define FM_WGRAD_HINT 0
#endif
// wgrad tile order inside a group: 1 = the longer tile dimension outermost
// (see decode_tile), 0 = row-major (round 1)
#ifndef FM_WGRAD_RASTER
#define FM_WGRAD_RASTER 1
#endif
// wgrad grid: 1 = group-aligned cluster count (see launch_cg), 0 = every SM
// (default). Measured (profiles/r02_wgrad_traffic.log): aligned cuts the
// configs[1] wgrad DRAM reads 19 % but costs 3-6 % of wgrad time at configs[2],
// configs[4] and balanced loads (64 of 74 CTA pairs busy); steps unchanged.
#ifndef FM_WGRAD_ALIGN
#define FM_WGRAD_ALIGN 0
#endif

struct Tile {
  int group;
  int m0;      // this CTA's first row (kRows: token row; kWgrad: output row)
  int n0;
  int k_row0;  // kWgrad: first token row of the reduction
  int num_kb;
  int mtile;   // kRows: global 128-row tile index of this CTA's rows
  bool valid;  // this CTA's 128 rows lie inside the group (CG == 2 tail half)
};

// Per-kernel schedule tables in smem, so that no tile decode touches global
// memory (the producer runs only a few stages ahead of the tensor pipe; a
// dependent L2 round trip at every tile boundary shows up as an MMA bubble).
//   order_s   kWgrad: groups longest-reduction-first (LPT), so long tiles
//             start in the first waves; kb_s: k-blocks per LPT slot
//             kRows: B row group (expert slot) of each group (Args::b_slot)
//   pair_s    kRows CG == 2: prefix of 256-row tile pairs per group
//   tp_s      kRows: tile_prefix;  ss_s: seg_start
struct Tables {
  int* order_s;
  int* pair_s;
  int* tp_s;
  int* ss_s;
};

template <int SCHED, int CG>
__device__ __forceinline__ void build_tables(const Args& a, const Tables& tb) {
  int* order_s = tb.order_s;
  int* pair_prefix_s = tb.pair_s;
  int* kb_s = tb.tp_s;
  for (int i = threadIdx.x; i < a.num_groups; i += blockDim.x) tb.ss_s[i] = __ldg(a.seg_start + i);
  if (SCHED == kRows) {
    for (int i = threadIdx.x; i <= a.num_groups; i += blockDim.x) tb.tp_s[i] = __ldg(a.tile_prefix + i);
    for (int i = threadIdx.x; i < a.num_groups; i += blockDim.x)  // B row group (expert slot) of group i
      tb.order_s[i] = a.b_slot ? __ldg(a.b_slot + i) : i;
  }
  if (SCHED == kWgrad) {
    for (int i = threadIdx.x; i < a.num_groups; i += blockDim.x) {
      const int ri = __ldg(a.seg_rows + i);
      int rank = 0;
      for (int j = 0; j < a.num_groups; ++j) {
        const int rj = __ldg(a.seg_rows + j);
        rank += (rj > ri) || (rj == ri && j < i);
      }
      order_s[rank] = i;
      kb_s[rank] = ri / kBK;  // k-blocks of the slot's group (the MMA issuer's only input)
    }
  } else if (CG == 2 && threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < a.num_groups; ++g) {
      pair_prefix_s[g] = acc;
      acc += (__ldg(a.tile_prefix + g + 1) - __ldg(a.tile_prefix + g) + 1) / 2;
    }
    pair_prefix_s[a.num_groups] = acc;
  }
}

template <int SCHED, int CG>
__device__ __forceinline__ int total_tiles(const Args& a, const Tables& tb) {
  const int n_tiles = a.N / kBN;
  if (SCHED == kRows) return (CG == 1 ? tb.tp_s : tb.pair_s)[a.num_groups] * n_tiles;
  return a.num_groups * (a.M_w / Cfg<CG>::kTileM) * n_tiles;
}

template <int SCHED, int CG>
__device__ __forceinline__ Tile decode_tile(const Args& a, int t, int& g, const Tables& tb, int rank) {
  Tile tl;
  const int n_tiles = a.N / kBN;
  tl.valid = true;
  if (SCHED == kRows) {
    const int* pre = CG == 1 ? tb.tp_s : tb.pair_s;
    while (pre[g + 1] * n_tiles <= t) ++g;
    const int local = t - pre[g] * n_tiles;
    const int m_local = (local / n_tiles) * CG + rank;  // this CTA's 128-row tile in the group
    tl.group = g;
    tl.mtile = tb.tp_s[g] + m_local;
    tl.valid = tl.mtile < tb.tp_s[g + 1];
    tl.m0 = tb.ss_s[g] + m_local * kBM;
    tl.n0 = (local % n_tiles) * kBN;
    tl.k_row0 = 0;
    tl.num_kb = a.K / kBK;
  } else {
    const int per_group = (a.M_w / Cfg<CG>::kTileM) * n_tiles;
    const int slot = t / per_group;
    const int local = t - slot * per_group;
    g = tb.order_s[slot];
    tl.group = g;
    // Tiles of a group that run together share operand slices (each a
    // K_g x 256 column block of A or B) through L2; a group whose tiles
    // straddle two waves of clusters streams the slices of both parts.
    // The longer tile dimension walks outermost, so a wave boundary cuts
    // across it: the part before the cut needs every slice of the short
    // dimension but few of the long one (dW2: 4 x 16 tiles, a 10-tile head
    // reads 4 + 3 slices instead of 1 + 10).
    const int m_tiles = a.M_w / Cfg<CG>::kTileM;
#if FM_WGRAD_RASTER
    const bool n_outer = n_tiles > m_tiles;
#else
    const bool n_outer = false;
#endif
    const int mi = n_outer ? local % m_tiles : local / n_tiles;
    const int ni = n_outer ? local / m_tiles : local % n_tiles;
    tl.m0 = mi * Cfg<CG>::kTileM + rank * kBM;
    tl.n0 = ni * kBN;
    tl.k_row0 = tb.ss_s[g];
    tl.num_kb = tb.tp_s[slot];  // kb_s
    tl.mtile = 0;
  }
  return tl;
}

// Side role, kind 2: un-permute, warp per token (VPL = d / 256 16-byte
// vectors per lane), the unpermute_bwd_kernel arithmetic: the k dX rows added
// in unit order, then the k gate rows scaled by dl, one bf16 rounding.
template <int VPL>
__device__ __forceinline__ void unpermute_side_vpl(const SideJob& sd, int cta, int num_ctas, int threads) {
  const int lane = threadIdx.x & 31;
  const int warps = threads >> 5;
  const __nv_bfloat16* dXp = static_cast<const __nv_bfloat16*>(sd.dXp);
  const __nv_bfloat16* wg = static_cast<const __nv_bfloat16*>(sd.wg);
  __nv_bfloat16* dx = static_cast<__nv_bfloat16*>(sd.dx);
  const int d = VPL * 256, k = sd.k;
  auto load = [&](const __nv_bfloat16* base, size_t row, uint4 (&q)[VPL]) {
    const uint4* src = reinterpret_cast<const uint4*>(base + row * static_cast<size_t>(d));
#pragma unroll
    for (int i = 0; i < VPL; ++i) q[i] = __ldg(src + lane + 32 * i);
  };
  auto axpy = [&](float (&acc)[VPL][8], const uint4 (&q)[VPL], float a) {
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const uint32_t qs[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[i][2 * c] = fmaf(a, __uint_as_float(qs[c] << 16), acc[i][2 * c]);
        acc[i][2 * c + 1] = fmaf(a, __uint_as_float(qs[c] & 0xffff0000u), acc[i][2 * c + 1]);
      }
    }
  };
  const P2P& pp = sd.pp;
  if (pp.unit_dst && pp.wait_slot >= 0) {
    // P2P: every expert GPU (this one included) published "dX ready" for this
    // epoch (bounded wait, as the standalone kernel's p2p_block_wait)
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
  // rows written by another GPU in this step: L2-coherent loads, no L1 reuse
  auto load_cg = [&](const __nv_bfloat16* base, size_t row, uint4 (&q)[VPL]) {
    const uint4* src = reinterpret_cast<const uint4*>(base + row * static_cast<size_t>(d));
#pragma unroll
    for (int i = 0; i < VPL; ++i) q[i] = __ldcg(src + lane + 32 * i);
  };
  auto load_unit = [&](int to, size_t row, uint4 (&q)[VPL]) {
    if (to >= 0) load_cg(reinterpret_cast<const __nv_bfloat16*>(pp.base[to] + pp.dx_off), row, q);
    else load(dXp, row, q);
  };
  for (int t = cta * warps + static_cast<int>(threadIdx.x >> 5); t < sd.T; t += num_ctas * warps) {
    const size_t base = static_cast<size_t>(t) * k;
    int my_pos = 0, my_e = 0, my_to = -1;
    float my_dl = 0.0f;
    if (lane < k) {
      my_pos = __ldg(sd.pos + base + lane);
      my_e = __ldg(sd.idx + base + lane);
      if (sd.gate_grad) my_dl = __ldg(sd.dl + base + lane);
      if (pp.unit_dst) my_to = pp.unit_dst[base + lane];
    }
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
      if (h0) load_unit(to0, p0, q0);
      if (h1) load_unit(to1, p1, q1);
      if (h0) axpy(acc, q0, 1.0f);
      if (h1) axpy(acc, q1, 1.0f);
    }
    if (sd.gate_grad) {
      for (int j = 0; j < k; ++j) {
        const int e = __shfl_sync(0xffffffffu, my_e, j);
        const float g_l = __shfl_sync(0xffffffffu, my_dl, j);
        uint4 q[VPL];
        load(wg, e, q);
        axpy(acc, q, g_l);
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(dx + static_cast<size_t>(t) * d);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      uint32_t pk[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        __nv_bfloat162 v = __floats2bfloat162_rn(acc[i][2 * c], acc[i][2 * c + 1]);
        pk[c] = *reinterpret_cast<uint32_t*>(&v);
      }
      dst[lane + 32 * i] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
}

// Side role, reduce: thread = (job, column); for every segment, eight
// running sums over its tiles t0 + j, t0 + j + 8, ... (j = 0..7, tiles in
// increasing order) combined in j order — exactly segment_tile_reduce_kernel's
// arithmetic, with the eight tile lanes folded into one thread. Loads of the
// eight chains are independent: eight in flight per thread.
template <int THREADS>
__device__ __forceinline__ void reduce_side(const SideJob& sd, int cta, int num_ctas) {
  int total = 0;
  for (int q = 0; q < sd.reduce_jobs; ++q) total += sd.r_cols[q];
  for (int g = cta * THREADS + static_cast<int>(threadIdx.x); g < total; g += num_ctas * THREADS) {
    int q = 0, col = g;
    while (col >= sd.r_cols[q]) col -= sd.r_cols[q++];
    const int cols = sd.r_cols[q];
    const float* src = sd.r_partial[q] + col;
    for (int li = 0; li < sd.Nl; ++li) {
      const int t0 = sd.mtile_prefix[li], t1 = sd.mtile_prefix[li + 1];
      float acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
      int t = t0;
      for (; t + 8 <= t1; t += 8) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldg(src + static_cast<size_t>(t + j) * cols);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += v[j];
      }
      for (int j = 0; t + j < t1; ++j) acc[j] += __ldg(src + static_cast<size_t>(t + j) * cols);
      float ssum = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) ssum += acc[j];
      const int oi = sd.r_out_index[q] ? sd.r_out_index[q][li] : li;
      sd.r_out[q][static_cast<size_t>(oi) * cols + col] = ssum;
    }
  }
}

template <int THREADS>
__device__ __forceinline__ void run_side(const SideJob& sd, int cta, int num_ctas) {
  if (sd.reduce_jobs > 0) reduce_side<THREADS>(sd, cta, num_ctas);  // short: first
  if (sd.kind == 1) {
    colsum_side<THREADS>(sd, cta, num_ctas);
  } else if (sd.kind == 2) {
    switch (sd.d / 256) {
      case 1: unpermute_side_vpl<1>(sd, cta, num_ctas, THREADS); break;
      case 2: unpermute_side_vpl<2>(sd, cta, num_ctas, THREADS); break;
      case 3: unpermute_side_vpl<3>(sd, cta, num_ctas, THREADS); break;
      case 4: unpermute_side_vpl<4>(sd, cta, num_ctas, THREADS); break;
      case 6: unpermute_side_vpl<6>(sd, cta, num_ctas, THREADS); break;
      default: unpermute_side_vpl<8>(sd, cta, num_ctas, THREADS); break;
    }
  }
}

// relu + round to a bf16 pair in one instruction (lo in the low half)
__device__ __forceinline__ uint32_t pack_relu_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int SCHED, bool A_MN, bool B_MN, int EPI, int CG>
__global__ void __launch_bounds__(Cfg<CG>::kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c, const Args args) {
  using C = Cfg<CG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + C::kStages * kABytes;
  uint8_t* smem_out = smem + C::kStages * C::kStageBytes;  // 1024-aligned
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_out + C::kOutBytes);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tfull_bar = empty_bar + C::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  // [tmem holder | bias 2x256 f32 | colsum 2x4x256 f32 | 4 schedule tables]
  float* bias_s = reinterpret_cast<float*>(tmem_holder + 4);
  float* colsum_s = bias_s + 2 * kBN;
  int* tables_s = reinterpret_cast<int*>(colsum_s + 8 * kBN);
  const Tables tb{tables_s, tables_s + kTableInts, tables_s + 2 * kTableInts, tables_s + 3 * kTableInts};
  const int* kb_s = tb.tp_s;  // kWgrad: k-blocks per LPT slot

  const uint32_t warp = ptx::warp_id();
  const uint32_t lane = ptx::lane_id();
  const int rank = CG == 2 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / CG;
  const int num_clusters = SCHED == kWgrad ? args.gemm_clusters : static_cast<int>(gridDim.x) / CG;
  const bool side_cta = SCHED == kWgrad && cluster >= num_clusters;  // column-sum CTAs
  build_tables<SCHED, CG>(args, tb);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&map_a);
    ptx::tma_prefetch_desc(&map_b);
    ptx::tma_prefetch_desc(&map_c);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], C::kEW * CG);  // one arrive per epilogue warp, both CTAs
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg<CG>(tmem_holder, kTmemCols);
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int ntiles = total_tiles<SCHED, CG>(args, tb);

  if (side_cta) {
    run_side<C::kThreads>(args.side, static_cast<int>(blockIdx.x) - num_clusters * CG,
                          static_cast<int>(gridDim.x) - num_clusters * CG);
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer (every CTA)
    // Whole warp, one elected lane issues (as for the MMA issuer below).
    {
      // CG == 2: both CTAs' loads complete on the leader's full barrier
      const uint32_t lead_full = CG == 2 ? ptx::mapa(ptx::smem_u32(full_bar), 0) : 0;
      // A/B knob FM_WGRAD_HINT (wgrad only): 1 = A operand evict_last, B evict_first;
      // 2 = the reverse; 0 (default) = no hint
      constexpr bool kHint = FM_WGRAD_HINT != 0;
      const uint64_t pol_a = FM_WGRAD_HINT == 1 ? ptx::l2_policy_evict_last() : ptx::l2_policy_evict_first();
      const uint64_t pol_b = FM_WGRAD_HINT == 1 ? ptx::l2_policy_evict_first() : ptx::l2_policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;
      int gated_mtile = -1;
      for (int t = cluster; t < ntiles; t += num_clusters) {
        const Tile tl = decode_tile<SCHED, CG>(args, t, g, tb, rank);
        const int b_row_base = (SCHED == kRows ? tb.order_s[tl.group] : tl.group) * args.b_rows_per_group;
        const int n_cta = tl.n0 + rank * C::kBNc;  // this CTA's slice of B
        if (SCHED == kRows && args.arrive_flags && tl.valid && tl.mtile != gated_mtile) {
          wait_tile_sources(args, tl.mtile);
          gated_mtile = tl.mtile;
        }
        for (int kb = 0; kb < tl.num_kb; ++kb) {
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          if (ptx::elect_one()) {
            if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes * CG);
            uint8_t* sa = smem_a + stage * kABytes;
            uint8_t* sb = smem_b + stage * C::kBBytes;
            const int k0 = kb * kBK;
            auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1) {
              if (kHint && SCHED == kWgrad) {
                const uint64_t pol = m == &map_a ? pol_a : pol_b;
                if (CG == 1) ptx::tma_load_2d_hint(dst, m, &full_bar[stage], c0, c1, pol);
                else ptx::tma_load_2d_2sm_hint(dst, m, lead_full + stage * 8, c0, c1, pol);
              } else if (CG == 1) {
                ptx::tma_load_2d(dst, m, &full_bar[stage], c0, c1);
              } else {
                ptx::tma_load_2d_2sm(dst, m, lead_full + stage * 8, c0, c1);
              }
            };
            if (!A_MN) {
              load(sa, &map_a, k0, tl.m0);
            } else {
#pragma unroll
              for (int j = 0; j < kBM / 64; ++j)
                load(sa + j * kMnChunkBytes, &map_a, tl.m0 + j * 64, tl.k_row0 + k0);
            }
            if (!B_MN) {
              load(sb, &map_b, k0, b_row_base + n_cta);
            } else {
              const int krow = (SCHED == kRows) ? b_row_base + k0 : tl.k_row0 + k0;
#pragma unroll
              for (int j = 0; j < C::kBNc / 64; ++j) load(sb + j * kMnChunkBytes, &map_b, n_cta + j * 64, krow);
            }
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // The whole warp runs the loop (its state is warp-uniform, so descriptors
    // live in uniform registers) and one elected lane issues: a lane-0-only
    // loop costs ~20 instructions of register->uniform shuffling per MMA, issue
    // slots the epilogue warps on this SM sub-partition compete for.
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(C::kTileM, kBN, A_MN, B_MN);
      constexpr uint32_t a_lbo = A_MN ? kMnChunkBytes : 16;
      constexpr uint32_t b_lbo = B_MN ? kMnChunkBytes : 16;
      // Advance per UMMA_K=16 step: 32 B inside a K-major swizzle row,
      // 16 K-rows (2 KB) for MN-major. Descriptor start addresses are in
      // 16-byte units (bits 0-13): stage / k-step offsets are plain adds.
      constexpr uint32_t a_kstep = A_MN ? 16 * 128 : 32;
      constexpr uint32_t b_kstep = B_MN ? 16 * 128 : 32;
      const uint64_t da0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_a), a_lbo, 1024);
      const uint64_t db0 = ptx::umma_desc_sw128(ptx::smem_u32(smem_b), b_lbo, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      // The issuer only needs each tile's k-block count (no tile decode, no
      // global loads between tiles: any gap here is a tensor-pipe bubble).
      const int per_group = SCHED == kWgrad ? (args.M_w / C::kTileM) * (args.N / kBN) : 1;
      for (int t = cluster; t < ntiles; t += num_clusters, ++iter) {
        const int num_kb = SCHED == kRows ? args.K / kBK : kb_s[t / per_group];
        const int ab = iter & 1;
        ptx::mbar_wait(&tempty_bar[ab], ((iter >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + ab * kBN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint64_t da = da0 + static_cast<uint32_t>((stage * kABytes) >> 4);
          const uint64_t db = db0 + static_cast<uint32_t>((stage * C::kBBytes) >> 4);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t dak = da + ((k * a_kstep) >> 4), dbk = db + ((k * b_kstep) >> 4);
              if (CG == 1) ptx::mma_bf16_ss(d_tmem, dak, dbk, idesc, (kb | k) != 0);
              else ptx::mma_bf16_ss_pair(d_tmem, dak, dbk, idesc, (kb | k) != 0);
            }
            if (CG == 1) ptx::mma_commit(&empty_bar[stage]);
            else ptx::mma_commit_pair(&empty_bar[stage], 0x3);
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (ptx::elect_one()) {
          if (CG == 1) ptx::mma_commit(&tfull_bar[ab]);
          else ptx::mma_commit_pair(&tfull_bar[ab], 0x3);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (every CTA)
    constexpr int kEpiThreads = 32 * C::kEW;
    constexpr int kChunks = (kBN / 32) / (C::kEW / 4);  // 32-column chunks per warp
    const int ew = static_cast<int>(warp) - 4;          // epilogue warp 0..EW-1
    const int q = warp & 3;                             // TMEM lane quarter this warp may access
    const int col0 = (ew >> 2) * kChunks * 32;          // this warp's first column in the tile
    const int row = q * 32 + lane;
    const int et = static_cast<int>(threadIdx.x) - 128;  // index among epilogue threads
    constexpr bool kBias = (EPI == kEpiBiasRelu || EPI == kEpiBias);
    const int mask_ld = args.N / 32;  // mask words per token row
    uint8_t* warp_out = smem_out + ew * C::kOutBufs * kStageOutBytes;
    // release of the accumulator goes to the leader's barrier
    const uint32_t lead_tempty = CG == 2 ? ptx::mapa(ptx::smem_u32(tempty_bar), 0) : 0;
    const uint64_t store_policy = ptx::l2_policy_evict_first();
    uint32_t out_seq = 0;
    int g = 0;
    int iter = 0;
    for (int t = cluster; t < ntiles; t += num_clusters, ++iter) {
      const Tile tl = decode_tile<SCHED, CG>(args, t, g, tb, rank);
      const int ab = iter & 1;
      // Everything that does not depend on the accumulator is fetched before
      // waiting on it: the tile's bias slice (to smem) and the ReLU mask bits.
      float* bs = bias_s + ab * kBN;
      if (kBias) {
        const float* bp = args.bias + static_cast<size_t>(tb.order_s[tl.group]) * args.N + tl.n0;
        for (int i = et; i < kBN; i += kEpiThreads) bs[i] = __ldg(bp + i);
        ptx::named_bar_sync(1, kEpiThreads);
      }
      uint32_t mbits[kChunks];
      if (EPI == kEpiReluMask && tl.valid) {
        const uint4* mp = reinterpret_cast<const uint4*>(
            args.mask + static_cast<size_t>(tl.m0 + row) * mask_ld + (tl.n0 + col0) / 32);
#pragma unroll
        for (int i = 0; i < kChunks / 4; ++i) {
          const uint4 m = __ldg(mp + i);
          mbits[4 * i] = m.x; mbits[4 * i + 1] = m.y; mbits[4 * i + 2] = m.z; mbits[4 * i + 3] = m.w;
        }
      }
      ptx::mbar_wait(&tfull_bar[ab], (iter >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + ab * kBN + col0;
#ifdef FM_DEBUG_NO_TMEM_LD
      const bool empty_k = true;  // diagnostic build: the epilogue skips its TMEM reads
#else
      const bool empty_k = tl.num_kb == 0;
#endif
      uint32_t ra[32], rb[32];
      uint32_t relu_bits[kChunks];
      // Output staging: this warp's 32 rows x 64 B go to a swizzled smem box
      // (SWIZZLE_64B: 16-byte chunk j of row r sits at chunk j ^ ((r >> 1) & 3)),
      // then one lane issues the TMA store. Two buffers per warp alternate.
      auto stage_begin = [&]() -> uint8_t* {
        uint8_t* buf = warp_out + (C::kOutBufs == 2 ? (out_seq & 1) : 0) * kStageOutBytes;
        if (lane == 0) {  // the store that last used `buf` has read it
          if (C::kOutBufs == 2) ptx::bulk_wait_read<1>();
          else ptx::bulk_wait_read<0>();
        }
        __syncwarp();
        return buf;
      };
      auto stage_row = [&](uint8_t* buf, const uint4 (&p)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = p[j];
      };
      auto stage_commit = [&](uint8_t* buf, int x, int y) {
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#ifndef FM_DEBUG_NO_STORE
          if (EPI == kEpiF32 && FM_WGRAD_STORE_HINT) ptx::tma_store_2d_hint(&map_c, buf, x, y, store_policy);
          else ptx::tma_store_2d(&map_c, buf, x, y);
#endif
          ptx::bulk_commit();
        }
        ++out_seq;
      };
      // chunk c of 32 columns: bias / activation / mask, convert, store
      auto process = [&](int c, uint32_t (&r)[32]) {
        const int col = tl.n0 + col0 + c * 32;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = empty_k ? 0.0f : __uint_as_float(r[i]);
        if (EPI == kEpiF32) {
          // two 16-column halves, 64 B per row each
          const int yrow = tl.group * args.M_w + tl.m0 + q * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint8_t* buf = stage_begin();
            const uint4 p[4] = {make_uint4(__float_as_uint(v[16 * h + 0]), __float_as_uint(v[16 * h + 1]),
                                           __float_as_uint(v[16 * h + 2]), __float_as_uint(v[16 * h + 3])),
                                make_uint4(__float_as_uint(v[16 * h + 4]), __float_as_uint(v[16 * h + 5]),
                                           __float_as_uint(v[16 * h + 6]), __float_as_uint(v[16 * h + 7])),
                                make_uint4(__float_as_uint(v[16 * h + 8]), __float_as_uint(v[16 * h + 9]),
                                           __float_as_uint(v[16 * h + 10]), __float_as_uint(v[16 * h + 11])),
                                make_uint4(__float_as_uint(v[16 * h + 12]), __float_as_uint(v[16 * h + 13]),
                                           __float_as_uint(v[16 * h + 14]), __float_as_uint(v[16 * h + 15]))};
            stage_row(buf, p);
            stage_commit(buf, col + 16 * h, yrow);
          }
          return;
        }
        if (kBias) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += bs[col0 + c * 32 + i];
        }
        if (EPI == kEpiBiasRelu) {
          // ReLU, bf16 rounding and the mask bits from the rounded pairs: bit =
          // (bf16(relu(h)) != 0), i.e. h > 0 unless h rounds to zero in bf16
          // (|h| below the smallest bf16 subnormal) — the bit the backward needs
          // for the stored activation
          uint32_t w[16];
          uint32_t bits = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            w[j] = pack_relu_bf16(v[2 * j], v[2 * j + 1]);
            const uint32_t nz = __vcmpne2(w[j], 0u) & 0x00010001u;  // bit 0: low half, bit 16: high
            bits |= ((nz | (nz >> 15)) & 3u) << (2 * j);
          }
          relu_bits[c] = bits;
          uint8_t* buf = stage_begin();
          const uint4 p[4] = {make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]),
                              make_uint4(w[8], w[9], w[10], w[11]), make_uint4(w[12], w[13], w[14], w[15])};
          stage_row(buf, p);
          stage_commit(buf, col, tl.m0 + q * 32);
          return;
        }
        if (EPI == kEpiReluMask) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (!((mbits[c] >> i) & 1u)) v[i] = 0.0f;
        }
        uint4 p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          p[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                            pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
        uint8_t* buf = stage_begin();
        stage_row(buf, p);
        stage_commit(buf, col, tl.m0 + q * 32);
        if (EPI == kEpiReluMask && args.colsum) {
          // Column sums of the stored bf16 values over this warp's 32 rows, read
          // back from the swizzled staging box: lanes 0-15 take rows 2i, lanes
          // 16-31 rows 2i+1, two columns (one 32-bit word) each; conflict-free.
          const int half = lane >> 4, pair = lane & 15;  // columns 2*pair, 2*pair+1
          float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int r = 2 * i + half;
            const int chunk = pair >> 2;  // 16-byte chunk holding this column pair
            const uint32_t w = *reinterpret_cast<const uint32_t*>(
                buf + r * 64 + ((chunk ^ ((r >> 1) & 3)) << 4) + (pair & 3) * 4);
            s0 += __uint_as_float(w << 16);
            s1 += __uint_as_float(w & 0xFFFF0000u);
          }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          if (half == 0) {
            float* dstc = colsum_s + (ab * 4 + q) * kBN + col0 + c * 32 + 2 * pair;
            dstc[0] = s0;
            dstc[1] = s1;
          }
        }
      };
      if (tl.valid) {
        // TMEM reads double-buffered: chunk c+1 is in flight while c is processed.
        if (!empty_k) {
          ptx::tmem_ld_32x32b_x32(t_row, ra);
          ptx::tmem_ld_wait_regs(ra);
        }
#pragma unroll
        for (int c = 0; c < kChunks; c += 2) {
          if (!empty_k) ptx::tmem_ld_32x32b_x32(t_row + (c + 1) * 32, rb);
          process(c, ra);
          if (!empty_k) {
            ptx::tmem_ld_wait_regs(rb);
            if (c + 2 < kChunks) ptx::tmem_ld_32x32b_x32(t_row + (c + 2) * 32, ra);
          }
          process(c + 1, rb);
          if (!empty_k && c + 2 < kChunks) ptx::tmem_ld_wait_regs(ra);
        }
      }
      // release the accumulator: one arrive per warp once all its TMEM reads are done
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 1 || leader) ptx::mbar_arrive(&tempty_bar[ab]);
        else ptx::mbar_arrive_cluster(lead_tempty + ab * 8);
      }
      if (EPI == kEpiReluMask && args.colsum) {
        // combine the four row quarters in a fixed order (deterministic). The
        // barrier runs for every tile, valid or not (tl.valid is uniform over
        // the CTA): it is also what orders this tile's reads of buffer ab
        // before the writes of the tile after next into the same buffer.
        ptx::named_bar_sync(2, kEpiThreads);
        if (tl.valid) {
          const float* cs = colsum_s + ab * 4 * kBN;
          float* dst = args.colsum + static_cast<size_t>(tl.mtile) * args.N + tl.n0;
          for (int col = et; col < kBN; col += kEpiThreads)
            dst[col] = ((cs[col] + cs[kBN + col]) + cs[2 * kBN + col]) + cs[3 * kBN + col];
        }
      }
      if (EPI == kEpiBiasRelu && args.mask && tl.valid) {
        uint4* mp = reinterpret_cast<uint4*>(args.mask + static_cast<size_t>(tl.m0 + row) * mask_ld +
                                             (tl.n0 + col0) / 32);
#pragma unroll
        for (int i = 0; i < kChunks / 4; ++i)
          mp[i] = make_uint4(relu_bits[4 * i], relu_bits[4 * i + 1], relu_bits[4 * i + 2],
                             relu_bits[4 * i + 3]);
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();  // all output stores complete before exit
    __syncwarp();
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (args.ready.signal_slot >= 0 && threadIdx.x == 0) {
    // this CTA's TMA stores completed (bulk_wait 0 before the barrier):
    // order them (async proxy) before the system-scope release, count the CTA
    const P2P& rp = args.ready;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
    unsigned int* ctr = rp.done + rp.signal_slot;
    if (atomicAdd(ctr, 1u) == gridDim.x - 1) {
      *ctr = 0;  // the next launch with this slot is stream-ordered after this one
      __threadfence_system();
      for (int dst = 0; dst < rp.world; ++dst) {
        unsigned long long* f =
            reinterpret_cast<unsigned long long*>(rp.base[dst] + rp.flag_off) + rp.signal_slot * kMaxPeers + rp.me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(rp.epoch) : "memory");
      }
    }
  }
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg<CG>(tmem_base, kTmemCols);
  }
}

template <int SCHED, bool A_MN, bool B_MN, int EPI, int CG>
void launch_cg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const Args& args,
               cudaStream_t stream, int* side_out = nullptr) {
  using C = Cfg<CG>;
  auto kern = grouped_gemm_kernel<SCHED, A_MN, B_MN, EPI, CG>;
  ensure_dynamic_smem(reinterpret_cast<const void*>(kern), C::kSmemBytes);
  int grid = num_sms() / CG * CG;
  Args a = args;
  if (SCHED == kWgrad) {
    const int tpg = (args.M_w / C::kTileM) * (args.N / kBN);  // output tiles per group
    int clusters = grid / CG;
    int side = 0;
    if (args.side.kind != 0 || args.side.reduce_jobs > 0) {
      // Side clusters for the tile column sums: the spare clusters of a
      // group-aligned split (64 of 74 CTA pairs at 64 tiles per group), used
      // only when they can finish the sums inside the GEMM (~45 GB/s per SM
      // next to a tensor-bound neighbour); otherwise no side job — the caller
      // runs its own column-sum launch (measured: taking SMs the alignment
      // does not free costs the GEMM more than the sums save).
      const int aligned = tpg <= clusters ? tpg * (clusters / tpg) : 0;
      const int spare = aligned ? clusters - aligned : 0;
      const double gemm_s = 2.0 * args.side.est_rows * args.M_w * args.N / 1.1e15;
      const double bytes =
          args.side.kind == 1 ? 2.0 * args.side.njobs * static_cast<double>(args.side.est_rows) * args.side.cols
                              : 2.0 * (static_cast<double>(args.side.T) * args.side.k + args.side.T) * args.side.d;
      const double need = bytes / (std::max(gemm_s, 1e-9) * 45e9 * CG);
      if (spare > 0 && spare >= need && spare * 4 <= clusters) side = spare;
      clusters -= side;
    }
#if FM_WGRAD_ALIGN
    else {
      // Group-aligned waves: a cluster count that is a multiple (or a divisor) of
      // the tiles per group puts all tiles of a group on the same wave, so they
      // advance through the group's K rows together and read each operand slice
      // from DRAM once (a group straddling two waves streams it twice). Each
      // cluster walks the LPT-ordered groups with an identical history, so the
      // waves stay aligned whatever the group sizes. Used when it keeps >= 3/4
      // of the SMs busy (64 of 74 CTA pairs at d 1024 / f 4096, 72 at 768 / 3072).
      int aligned = 0;
      if (tpg <= clusters) {
        aligned = tpg * (clusters / tpg);
      } else {
        for (int c = clusters; c >= 1 && !aligned; --c)
          if (tpg % c == 0) aligned = c;
      }
      if (aligned * 4 >= clusters * 3) clusters = aligned;
    }
#endif
    a.gemm_clusters = std::min(clusters, std::max(1, args.num_groups * tpg));
    a.side.clusters = side;
    if (side == 0) {
      a.side.kind = 0;
      a.side.reduce_jobs = 0;
    }
    if (side_out) *side_out = side;
    grid = (a.gemm_clusters + side) * CG;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FM_CUDA(cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, a));
  count_launch();
}

// CTA-pair tiles unless overridden (FM_GEMM_CTA_GROUP / fm_set_gemm_cta_group)
int g_cta_group = 0;  // 0 = auto

template <int SCHED, bool A_MN, bool B_MN, int EPI>
void launch(const CUtensorMap* maps1, const CUtensorMap* maps2, const Args& args, int cg,
            cudaStream_t stream, int* side_out = nullptr) {
  if (cg == 2) launch_cg<SCHED, A_MN, B_MN, EPI, 2>(maps2[0], maps2[1], maps2[2], args, stream, side_out);
  else launch_cg<SCHED, A_MN, B_MN, EPI, 1>(maps1[0], maps1[1], maps1[2], args, stream, side_out);
}

}  // namespace gemm

void set_gemm_cta_group(int cg) {
  if (cg != 0 && cg != 1 && cg != 2) throw std::invalid_argument("gemm cta group must be 0, 1 or 2");
  gemm::g_cta_group = cg;
}

// Host entry used by the layer and by the C-ABI test hook.
void grouped_gemm(int variant, const void* A, const void* B, void* C, const float* bias,
                  const void* aux, const int* seg_start, const int* seg_rows,
                  const int* tile_prefix, int num_groups, int total_rows, int M_w, int N, int K,
                  cudaStream_t stream, const ArrivalGate* gate, const int* b_slot, int b_groups,
                  SideJob* side, const P2P* ready) {
  using namespace gemm;
  if (N % kBN != 0) throw std::invalid_argument("grouped_gemm: N must be a multiple of 256");
  if (num_groups < 1 || num_groups > kMaxGroups)
    throw std::invalid_argument("grouped_gemm: 1 <= num_groups <= 256");
  if (total_rows % kBM != 0 || total_rows <= 0)
    throw std::invalid_argument("grouped_gemm: total_rows must be a positive multiple of 128");
  Args a{};
  a.ready.signal_slot = -1;
  if (ready && ready->signal_slot >= 0) a.ready = *ready;
  a.num_groups = num_groups;
  a.seg_start = seg_start;
  a.seg_rows = seg_rows;
  a.tile_prefix = tile_prefix;
  a.M_w = M_w;
  a.N = N;
  a.K = K;
  a.out = C;
  a.ldc = N;
  a.bias = bias;
  a.mask = static_cast<uint32_t*>(const_cast<void*>(aux));
  if (b_slot && variant == FM_GEMM_WGRAD) throw std::invalid_argument("grouped_gemm: b_slot is for token-row GEMMs");
  a.b_slot = b_slot;
  const int nb = b_slot ? b_groups : num_groups;  // rows of B (in groups) the tensor map spans
  if (nb < 1) throw std::invalid_argument("grouped_gemm: b_groups must be >= 1 with b_slot");
  if (gate && gate->flags) {
    if (variant == FM_GEMM_WGRAD) throw std::invalid_argument("grouped_gemm: arrival gating is for token-row GEMMs");
    a.arrive_flags = gate->flags;
    a.tile_src_mask = gate->tile_src_mask;
    a.epoch = gate->epoch;
    a.arrive_err = gate->err;
  }
  // CTA pairs for the token-row GEMMs when groups are large enough that the
  // odd 128-row tail of each group (computed, not stored) is cheap — measured
  // break-even near 900 rows per group (configs[2]: 64 groups of ~1024 rows run
  // 3-6% faster in pairs); always for wgrad (M_w is a multiple of 256).
  int cg = g_cta_group;
  if (cg == 0) {
    if (variant == FM_GEMM_WGRAD) cg = (M_w % 256 == 0) ? 2 : 1;
    else cg = (total_rows / num_groups >= 1024) ? 2 : 1;
  }
  if (variant == FM_GEMM_WGRAD && M_w % (kBM * cg) != 0) cg = 1;
  CUtensorMap m1[3], m2[3];
  switch (variant) {
    case FM_GEMM_FWD_BIAS_RELU:
    case FM_GEMM_FWD_BIAS: {
      if (K % kBK != 0) throw std::invalid_argument("grouped_gemm: K must be a multiple of 64");
      // A [rows, K] K-major; B = W_g [N, K] K-major, groups stacked.
      m1[0] = m2[0] = make_tmap_bf16(A, K, total_rows, K, 64, kBM);
      m1[1] = make_tmap_bf16(B, K, static_cast<uint64_t>(nb) * N, K, 64, kBN);
      m2[1] = make_tmap_bf16(B, K, static_cast<uint64_t>(nb) * N, K, 64, kBN / 2);
      m1[2] = m2[2] = make_tmap_2d(C, false, N, total_rows, N, 32, 32, 64);
      a.b_rows_per_group = N;
      if (variant == FM_GEMM_FWD_BIAS_RELU)
        launch<kRows, false, false, kEpiBiasRelu>(m1, m2, a, cg, stream);
      else
        launch<kRows, false, false, kEpiBias>(m1, m2, a, cg, stream);
      break;
    }
    case FM_GEMM_DGRAD_RELU_MASK:
    case FM_GEMM_DGRAD: {
      if (K % kBK != 0) throw std::invalid_argument("grouped_gemm: K must be a multiple of 64");
      // A [rows, K] K-major; B = W_g viewed [K, N] (N contiguous) -> MN-major.
      m1[0] = m2[0] = make_tmap_bf16(A, K, total_rows, K, 64, kBM);
      m1[1] = m2[1] = make_tmap_bf16(B, N, static_cast<uint64_t>(nb) * K, N, 64, kBK);
      m1[2] = m2[2] = make_tmap_2d(C, false, N, total_rows, N, 32, 32, 64);
      a.b_rows_per_group = K;
      if (variant == FM_GEMM_DGRAD_RELU_MASK) {
        if (!aux) throw std::invalid_argument("grouped_gemm: relu-mask dgrad needs the ReLU bit mask");
        // `bias` doubles as the optional per-tile column-sum output here
        a.colsum = const_cast<float*>(bias);
        a.bias = nullptr;
        launch<kRows, false, true, kEpiReluMask>(m1, m2, a, cg, stream);
      } else {
        launch<kRows, false, true, kEpiNone>(m1, m2, a, cg, stream);
      }
      break;
    }
    case FM_GEMM_WGRAD: {
      if (M_w % kBM != 0) throw std::invalid_argument("grouped_gemm: M_w must be a multiple of 128");
      // A = tokens x M_w (M contiguous) -> MN-major; B = tokens x N -> MN-major.
      m1[0] = m2[0] = make_tmap_bf16(A, M_w, total_rows, M_w, 64, kBK);
      m1[1] = m2[1] = make_tmap_bf16(B, N, total_rows, N, 64, kBK);
      m1[2] = m2[2] = make_tmap_2d(C, true, N, static_cast<uint64_t>(num_groups) * M_w, N, 16, 32, 64);
      a.b_rows_per_group = 0;
      if (side && side->kind == 1) {
        if (side->njobs < 1 || side->cols % 8 != 0 || side->cols > 8 * Cfg<1>::kThreads)
          throw std::invalid_argument("grouped_gemm: side column sums need cols % 8 == 0, cols <= 2048");
        a.side = *side;
      } else if (side && side->kind == 0 && side->reduce_jobs > 0) {
        a.side = *side;
      } else if (side && side->kind == 2) {
        const int v = side->d / 256;
        if (side->d % 256 != 0 || !(v == 1 || v == 2 || v == 3 || v == 4 || v == 6 || v == 8) || side->k < 1)
          throw std::invalid_argument("grouped_gemm: side un-permute needs d in {256,512,768,1024,1536,2048}");
        a.side = *side;
      }
      int side_clusters = 0;
      launch<kWgrad, true, true, kEpiF32>(m1, m2, a, cg, stream, &side_clusters);
      if (side) side->clusters = side_clusters;  // 0: the column sums did not run
      break;
    }
    default:
      throw std::invalid_argument("grouped_gemm: unknown variant");
  }
}

}  // namespace fm
