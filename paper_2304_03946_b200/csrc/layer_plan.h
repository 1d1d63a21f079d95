// Device-side dispatch plan written by plan_kernel from the routing flows
// and read by dispatch / relayout / GEMM / colsum kernels. All arrays are
// device int32 inside one allocation owned by the layer.
#pragma once

#include <cstdint>

#ifndef FM_GATE_HALF_TILE_MAX_N
#define FM_GATE_HALF_TILE_MAX_N 0  // A/B knob: 64-token gate tiles up to this many experts (measured slower)
#endif

namespace fm {

#ifdef __CUDACC__
#define FM_PLAN_HD __host__ __device__ inline
#else
#define FM_PLAN_HD inline
#endif
// Token rows per gate tile — the granularity of the gate's per-tile expert
// counts and ranks, which the dispatch turns into positions: 64 when the
// experts fit a narrow accumulator (the tensor work per token is small, so a
// half-height tile costs nothing and halves the tail of the HBM stream), 128
// otherwise (at 128+ experts the gate's MMA work would start to show).
FM_PLAN_HD int gate_tile_rows(int num_experts) { return num_experts <= FM_GATE_HALF_TILE_MAX_N ? 64 : 128; }
FM_PLAN_HD int gate_tile_shift(int num_experts) { return num_experts <= FM_GATE_HALF_TILE_MAX_N ? 6 : 7; }

struct PlanDev {
  int32_t* chunk_lo;        // [N][G]  first rank of dst's chunk in (me, e) rank space
  int32_t* chunk_cnt;       // [N][G]  flows[e][me][dst]
  int32_t* send_off;        // [N][G]  first dispatch-buffer row of (dst, e) (dst-major)
  int32_t* send_rows;       // [G]     rows sent to each dst
  int32_t* recv_rows;       // [G]     rows received from each src
  int32_t* local_index;     // [N]     local segment of expert e on this GPU, -1 if none (host-filled)
  int32_t* seg_start;       // [Nl]    first X_perm row of local expert li
  int32_t* seg_real;        // [Nl]    rows that carry tokens
  int32_t* seg_rows;        // [Nl]    rows padded to 128
  int32_t* mtile_prefix;    // [Nl+1]  exclusive prefix of 128-row tiles
  int32_t* recv_chunk_off;  // [G*Nl+1] a2a receive-buffer offset of (src, li)
  int32_t* recv_chunk_dst;  // [G*Nl]  X_perm row of that chunk's first row
  int32_t* totals;          // [4]     padded rows, units sent, units received
  int32_t* peer_row;        // [N][G]  P2P: X_perm row on dst of (e, me)'s first unit (null otherwise)
  unsigned long long* tile_src_mask;  // [rows/128] P2P: sources with rows in each 128-row tile
};

// Peer-to-peer transport: every GPU's exchange arena holds its
// X_perm, Y_perm, dY_perm, dX_perm (bf16 rows), dl per X_perm row (f32) and
// the arrival flags, at the same offsets on every GPU; base[g] is GPU g's
// arena as mapped in this process (CUDA IPC, or the pointer itself in one
// process). Units carry their destination GPU in unit_dst; null unit_dst
// means the single-GPU / NCCL layouts (local buffers only).
constexpr int kMaxPeers = 64;
constexpr int kP2PSlots = 4;  // 0 rows dispatched, 1 Y ready, 2 dY rows pushed, 3 dX ready
struct P2P {
  char* base[kMaxPeers];
  int64_t x_off, y_off, dy_off, dx_off, dl_off, flag_off;  // byte offsets inside an arena
  int32_t* unit_dst;                                       // [T*k] destination GPU (-1: dropped)
  // In-kernel release of pushed rows: with signal_slot >= 0 the kernel's last
  // block (after every block fenced its peer stores) sets flags[signal_slot][me]
  // = epoch in every peer's arena. done: this GPU's per-slot block counters.
  int signal_slot, me, world;
  unsigned long long epoch;
  unsigned int* done;
  // With wait_slot >= 0 a consuming kernel's blocks first wait (bounded) until
  // every peer has published flags[wait_slot][src] >= epoch in this GPU's arena.
  int wait_slot;
  int* err;
};

// Memory-bound work run by spare CTA pairs of a weight-gradient GEMM launch
// next to its tensor-bound tiles, bit-identical to the
// standalone kernels it replaces:
//  kind 1, column sums: job j writes partial[j][tile][c] = sum over the
//    tile's real rows r of (row_w[j] ? row_w[j][r] : 1) * buf[j][r][c]
//    (segment_tile_colsum_kernel: same rows, same fmaf chain);
//  kind 2, un-permute: dx[t] = sum_j dXp[pos[t,j]] + [gate_grad]
//    sum_j dl[t,j] * wg[idx[t,j]] (unpermute_bwd_kernel); with pp.unit_dst
//    set (P2P) the dX rows are read from the expert GPUs' arenas after the
//    side CTAs waited for every peer's "dX ready" flag (pp.wait_slot).
struct SideJob {
  int kind;       // 0 = none
  int clusters;   // CTA pairs (or CTAs) given to it; set by the launcher (0: did not run)
  int est_rows;   // host estimate of the GEMM's reduction rows (sizes `clusters`)
  // kind 1
  const void* buf[2];  // bf16 [rows][cols]
  const float* row_w[2];
  float* partial[2];   // f32 [tiles][cols]
  int njobs;
  int cols;
  const int32_t* mtile_prefix;  // PlanDev fields of the segments
  const int32_t* seg_start;
  const int32_t* seg_real;
  int Nl;
  // kind 2
  const void* dXp;  // bf16 [rows][d]
  const int32_t* pos;
  const int32_t* idx;
  const float* dl;
  const void* wg;   // bf16 [N][d]
  void* dx;         // bf16 [T][d]
  int T, k, d, gate_grad;
  P2P pp;           // P2P transport (pp.unit_dst == nullptr: local rows)
  // then, on the same side CTAs, the per-segment reduce of tile partials
  // (out[oi(li)][c] = sum over the segment's 128-row tiles of partial[tile][c]
  // in segment_tile_reduce_kernel's order: eight running sums over the tiles
  // congruent mod 8, combined in lane order); thread = one column of one
  // job, all segments. Uses mtile_prefix / Nl.
  int reduce_jobs;  // 0..3
  const float* r_partial[3];
  int r_cols[3];
  const int32_t* r_out_index[3];  // null: li
  float* r_out[3];
};

}  // namespace fm
