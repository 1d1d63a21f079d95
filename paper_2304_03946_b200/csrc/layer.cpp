// fm_layer: the FlexMoE MoE layer on one GPU (one process per GPU).
//
// Owns the device workspace (routing state, dispatch plan, permuted
// activations) sized for `max_tokens`, and runs the hot path on a caller
// stream with no host synchronisation when num_gpus == 1:
//   forward : gate(+hist) -> scan -> route + plan -> dispatch -> FFN1 -> FFN2 -> combine
//   backward: combine^T(+gate softmax^T) -> FFN2 wgrad (+ db2 / dWg tile sums on
//             its spare CTA pairs) -> FFN2 dgrad (+ db1 tile sums) -> FFN1 dgrad
//             -> FFN1 wgrad (+ un-permute, dx, on its spare CTA pairs) -> reduce
//             (FM_BWD_ORDER 4; the side work runs standalone where a launch has
//             no spare pairs)
// With num_gpus > 1 the same kernels run as phases around the host's
// all-to-all (see the fm_layer_* phase entry points in flexmoe_b200.h).
//
// Placement: replica counts [N][G] as in Placement::replica_count_on
// (placement.hpp:80-82). The experts hosted on this rank (count > 0) are the
// local experts, in ascending id; their weights are packed in that order.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fm_internal.h"
#include "layer_plan.h"
#include "routing.cuh"

// A/B knob (fused single-GPU backward): 0 = combine^T, dgrad2, dgrad1, wgrad2,
// wgrad1, tile sums, un-permute (round 1); 1 = the two weight-gradient GEMMs
// last (measured: the next step's gate is not faster, profiles/r02_gate_context.log);
// 2 = wgrad2, dgrad2, wgrad1, dgrad1 (each f32 weight-gradient drain overlaps a
// tensor-bound GEMM); 3 = 2 with un-permute before the tile sums; 4 (default) =
// wgrad2 (+ tile sums), dgrad2, dgrad1, wgrad1 (+ un-permute): side jobs
// (profiles/r02_colsum_side.log)
#ifndef FM_BWD_ORDER
#define FM_BWD_ORDER 4
#endif
// Default of fm_layer_set_side_jobs: memory-bound backward work (tile column
// sums, un-permute) on spare CTA pairs of the weight-gradient launches (1)
// instead of their own kernels (0)
#ifndef FM_COLSUM_SIDE
#define FM_COLSUM_SIDE 1
#endif

namespace fm {

// launchers (gate.cu, dispatch.cu, grouped_gemm.cu)
int gate_num_tiles(int T, int num_experts);
void launch_gate(const void* x, const void* wg, int T, int N, int d, int top_k, int32_t* topk_idx,
                 float* topk_w, int32_t* tile_rank, int32_t* tile_counts, cudaStream_t stream);
void launch_expert_scan(const int32_t* tile_counts, int num_tiles, int N, int32_t* tile_base,
                        int64_t* hist, int64_t* demand_NG, int G, int me, cudaStream_t s);
void launch_plan(int64_t* flows, int N, int G, int me, const int32_t* local_expert, int Nl,
                 const PlanDev& p, cudaStream_t s, const int32_t* counts, const int64_t* demand,
                 int32_t* status, const int64_t* gathered_GN = nullptr, const int32_t* scan_tile_counts = nullptr,
                 int scan_num_tiles = 0, int32_t* scan_tile_base = nullptr, int64_t* scan_hist = nullptr);
bool plan_can_fuse_scan(int N, int G, int num_tiles);
void launch_dispatch(const void* x, int T, int d, int k, int N, int G, int me, bool direct,
                     const int32_t* idx, const int32_t* tile_rank, const int32_t* tile_base,
                     const PlanDev& p, int32_t* pos, void* buf, int32_t* row_expert,
                     cudaStream_t s, const P2P* pp = nullptr, void* pad_buf = nullptr, int Nl = 0);
void launch_zero_pad(void* buf, int d, const PlanDev& p, int Nl, int32_t* row_expert, cudaStream_t s);
void launch_gate_wgrad(const void* buf, int max_rows, int d, const float* dl_rows, const PlanDev& p, int N,
                       int G, float* partial, float* dwg, cudaStream_t s);
int gate_wgrad_pieces(int rows, int N, int G);
void launch_demand_transpose(const int64_t* gathered_GN, int N, int G, int64_t* demand_NG,
                             cudaStream_t s);
void launch_relayout(void* recv, void* perm, int d, int G, int Nl, const PlanDev& p, int max_rows,
                     int dir, cudaStream_t s);
void launch_combine_fwd(const void* Y, const int32_t* pos, const float* w, int T, int d, int k,
                        void* y, cudaStream_t s, const P2P* pp = nullptr);
void launch_combine_bwd(const void* dy, const void* Y, const int32_t* pos, const float* w, int T,
                        int d, int k, void* dYbuf, float* dl, float* dl_rows, cudaStream_t s, const P2P* pp = nullptr,
                        const PlanDev* pad_plan = nullptr, int Nl = 0);
void launch_unpermute_bwd(const void* dXbuf, const int32_t* pos, const int32_t* idx, const float* dl,
                          const void* wg, int T, int d, int k, bool gate_grad, void* dx,
                          cudaStream_t s, const P2P* pp = nullptr);
void launch_segment_tile_colsum(const void* buf0, const float* w0, float* partial0, const void* buf1,
                                const float* w1, float* partial1, int cols, const PlanDev& p, int Nl,
                                int max_tiles, cudaStream_t s);
void launch_segment_tile_reduce(const float* partial0, int cols0, const int32_t* idx0, float* out0,
                                const float* partial1, int cols1, const int32_t* idx1, float* out1,
                                const float* partial2, int cols2, const int32_t* idx2, float* out2,
                                const PlanDev& p, int Nl, cudaStream_t s);
void launch_p2p_signal(const P2P& pp, int G, int me, int slot, unsigned long long epoch, cudaStream_t s);
void launch_dropped_gate_wgrad(const void* x, const int32_t* pos, const int32_t* idx, const float* dl,
                               int T, int d, int k, int N, float* partial, float* dwg, cudaStream_t s);
int dropped_gate_chunks(int T);


namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool owned = true;  // false: a view into another allocation (the P2P arena)
  void reset(size_t n) {
    if (p && owned) cudaFree(p);
    p = nullptr;
    bytes = 0;
    owned = true;
    if (n) {
      FM_CUDA(cudaMalloc(&p, n));
      bytes = n;
    }
  }
  void view(void* ptr, size_t n) {
    if (p && owned) cudaFree(p);
    p = ptr;
    bytes = n;
    owned = false;
  }
  ~DevBuf() {
    if (p && owned) cudaFree(p);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

// Optional CUDA-event timing of each phase on the launching stream (bench.py
// reads it to compute per-kernel roofline fractions live).
class PhaseTimer {
 public:
  ~PhaseTimer() {
    for (auto& e : pool_) cudaEventDestroy(e);
  }
  void enable(bool on) {
    on_ = on;
    marks_.clear();
    used_ = 0;
    for (auto& v : ms_) v = 0;
    for (auto& c : n_) c = 0;
  }
  bool on() const { return on_; }
  void begin(int phase, cudaStream_t s) {
    if (!on_) return;
    cur_phase_ = phase;
    cur_start_ = event();
    FM_CUDA(cudaEventRecord(cur_start_, s));
  }
  void end(cudaStream_t s) {
    if (!on_) return;
    cudaEvent_t stop = event();
    FM_CUDA(cudaEventRecord(stop, s));
    marks_.push_back({cur_phase_, cur_start_, stop});
  }
  // Synchronises, folds recorded intervals into the totals, returns them.
  void read(double* ms, int* counts) {
    FM_CUDA(cudaDeviceSynchronize());
    for (const Mark& m : marks_) {
      float t = 0;
      FM_CUDA(cudaEventElapsedTime(&t, m.start, m.stop));
      ms_[m.phase] += t;
      n_[m.phase] += 1;
    }
    marks_.clear();
    used_ = 0;
    for (int i = 0; i < FM_NUM_PHASES; ++i) {
      ms[i] = ms_[i];
      counts[i] = n_[i];
    }
  }

 private:
  struct Mark {
    int phase;
    cudaEvent_t start, stop;
  };
  cudaEvent_t event() {
    if (used_ == pool_.size()) {
      cudaEvent_t e;
      FM_CUDA(cudaEventCreate(&e));
      pool_.push_back(e);
    }
    return pool_[used_++];
  }
  bool on_ = false;
  int cur_phase_ = 0;
  cudaEvent_t cur_start_{};
  std::vector<cudaEvent_t> pool_;
  size_t used_ = 0;
  std::vector<Mark> marks_;
  double ms_[FM_NUM_PHASES] = {};
  int n_[FM_NUM_PHASES] = {};
};

class Layer {
 public:
  explicit Layer(const fm_layer_config& c) : cfg_(c) {
    if (c.num_experts < 1 || c.num_experts > 256)
      throw std::invalid_argument("fm_layer: 1 <= num_experts <= 256");
    if (c.top_k < 1 || c.top_k > 8 || c.top_k > c.num_experts)
      throw std::invalid_argument("fm_layer: 1 <= top_k <= min(8, num_experts)");
    if (c.d_model % 256 != 0 || c.d_model > 2048)
      throw std::invalid_argument("fm_layer: d_model must be a multiple of 256 and <= 2048");
    if (c.d_ff % 256 != 0) throw std::invalid_argument("fm_layer: d_ff must be a multiple of 256");
    if (c.num_gpus < 1 || c.num_gpus > kMaxGpus)
      throw std::invalid_argument("fm_layer: 1 <= num_gpus <= 64");
    if (c.rank < 0 || c.rank >= c.num_gpus) throw std::out_of_range("fm_layer: rank out of range");
    if (c.max_tokens < 1) throw std::invalid_argument("fm_layer: max_tokens must be >= 1");
    const int N = c.num_experts, G = c.num_gpus, T = c.max_tokens, k = c.top_k;
    const int tiles = gate_num_tiles(T, N);
    topk_idx_.reset(sizeof(int32_t) * T * k);
    topk_w_.reset(sizeof(float) * T * k);
    tile_rank_.reset(sizeof(int32_t) * T * k);
    pos_.reset(sizeof(int32_t) * T * k);
    dl_.reset(sizeof(float) * T * k);
    tile_counts_.reset(sizeof(int32_t) * tiles * N);
    tile_base_.reset(sizeof(int32_t) * tiles * N);
    hist_.reset(sizeof(int64_t) * N);
    demand_.reset(sizeof(int64_t) * N * G);
    flows_.reset(sizeof(int64_t) * N * G * G);
    route_status_.reset(sizeof(int32_t));
    counts_.assign(static_cast<size_t>(N) * G, 0);
    host_counts_.assign(2 * G + 1, 0);
    kept_.reset(sizeof(int64_t) * N * G);
    dropped_.reset(sizeof(int64_t));
    FM_CUDA(cudaMemset(dropped_.p, 0, sizeof(int64_t)));
    // placement tables (uploaded per switch) and plan arrays, sized for Nl = N
    ctl_mem_.reset(sizeof(int32_t) * (3 * N + N * G));
    plan_.local_index = ctl_mem_.as<int32_t>();
    local_expert_dev_ = plan_.local_index + N;
    local_slot_dev_ = plan_.local_index + 2 * N;
    counts_dev_ = plan_.local_index + 3 * N;
    const int Nm = N;
    const size_t n_plan = 3 * N * G + 2 * G + 3 * Nm + (Nm + 1) + (G * Nm + 1) + G * Nm + 4 + N * G /*peer_row*/;
    plan_mem_.reset(sizeof(int32_t) * n_plan);
    int32_t* q = plan_mem_.as<int32_t>();
    auto take = [&](size_t n) {
      int32_t* r = q;
      q += n;
      return r;
    };
    plan_.chunk_lo = take(N * G);
    plan_.chunk_cnt = take(N * G);
    plan_.send_off = take(N * G);
    plan_.send_rows = take(G);
    plan_.recv_rows = take(G);
    plan_.seg_start = take(Nm);
    plan_.seg_real = take(Nm);
    plan_.seg_rows = take(Nm);
    plan_.mtile_prefix = take(Nm + 1);
    plan_.recv_chunk_off = take(G * Nm + 1);
    plan_.recv_chunk_dst = take(G * Nm);
    plan_.totals = take(4);
    peer_row_mem_ = take(N * G);
    plan_.peer_row = nullptr;
    plan_.tile_src_mask = nullptr;
    for (Staging& st : staging_) {
      FM_CUDA(cudaMallocHost(&st.host, sizeof(int32_t) * (3 * N + N * G)));
      FM_CUDA(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
    }
  }

  // Placement switch without allocation or host synchronisation: the plan
  // arrays are sized once for every expert being local (Nl <= N), and the
  // placement tables reach the device by one cudaMemcpyAsync on `s` from a
  // pinned staging ring, stream-ordered after every kernel that read the
  // previous tables. hosted_N (optional, [N]): experts whose state this rank
  // keeps although its replica count is 0 — a replica whose state copy is in
  // flight: it is local (gradient slices, replica-group all-reduce) with no
  // rows routed to it.
  void set_placement(const int32_t* counts_NG, const int32_t* hosted_N = nullptr, cudaStream_t s = nullptr,
                     bool sync = true) {
    const int N = cfg_.num_experts, G = cfg_.num_gpus;
    std::vector<int32_t> c(counts_NG, counts_NG + static_cast<size_t>(N) * G);
    std::vector<int32_t> local;
    for (int e = 0; e < N; ++e) {
      int total = 0;
      for (int g = 0; g < G; ++g) {
        if (c[static_cast<size_t>(e) * G + g] < 0)
          throw std::invalid_argument("fm_layer: negative replica count");
        total += c[static_cast<size_t>(e) * G + g];
      }
      if (total < 1)
        throw std::invalid_argument("fm_layer: expert " + std::to_string(e) + " has no replica");
      if (c[static_cast<size_t>(e) * G + cfg_.rank] > 0 || (hosted_N && hosted_N[e] != 0)) local.push_back(e);
    }
    if (cfg_.slots_per_gpu > 0) {
      for (int g = 0; g < G; ++g) {
        int used = 0;
        for (int e = 0; e < N; ++e) used += c[static_cast<size_t>(e) * G + g];
        if (used > cfg_.slots_per_gpu)
          throw std::invalid_argument("fm_layer: GPU " + std::to_string(g) +
                                      " over its slot budget");
      }
    }
    if (G == 1 && static_cast<int>(local.size()) != N)
      throw std::logic_error("fm_layer: single GPU must host every expert");
    counts_ = c;
    local_ = local;
    upload_placement(s, sync);
  }

  // slot_N[e]: row (group) of expert e in the w1/b1/w2/b2 operands passed to
  // the expert GEMMs, for every local expert; capacity = rows of those
  // operands. Null restores the packed layout (local experts ascending).
  void set_operand_slots(const int32_t* slot_N, int capacity, cudaStream_t s) {
    const int N = cfg_.num_experts;
    if (slot_N) {
      if (capacity < 1 || capacity > 4096) throw std::invalid_argument("fm_layer: operand capacity must be in [1, 4096]");
      operand_slot_.assign(slot_N, slot_N + N);
      operand_cap_ = capacity;
    } else {
      operand_slot_.clear();
      operand_cap_ = 0;
    }
    upload_placement(s, false);
  }

  void upload_placement(cudaStream_t s, bool sync) {
    const int N = cfg_.num_experts, G = cfg_.num_gpus, Nl = nl();
    Staging& st = staging_[staging_next_];
    staging_next_ = (staging_next_ + 1) % kStaging;
    FM_CUDA(cudaEventSynchronize(st.done));  // the upload kStaging switches ago (long complete)
    int32_t* h = st.host;  // [local_index N | local_expert N | operand slot N | counts N*G]
    std::fill(h, h + N, -1);
    for (int i = 0; i < Nl; ++i) {
      h[local_[i]] = i;
      h[N + i] = local_[i];
      h[2 * N + i] = operand_slot_.empty() ? i : operand_slot_[local_[i]];  // validated at GEMM enqueue
    }
    std::memcpy(h + 3 * N, counts_.data(), sizeof(int32_t) * N * G);
    FM_CUDA(cudaMemcpyAsync(ctl_mem_.p, h, sizeof(int32_t) * (3 * N + N * G), cudaMemcpyHostToDevice, s));
    FM_CUDA(cudaEventRecord(st.done, s));
    if (sync) FM_CUDA(cudaEventSynchronize(st.done));
    // Row capacity of the permuted buffers: every unit could land here
    // (worst case of route()), plus per-segment padding. G > 1 without P2P
    // starts at twice the local units and grows in route_gathered (that path
    // synchronises per step anyway); P2P sizes its arena for the worst case.
    const size_t units = static_cast<size_t>(cfg_.max_tokens) * cfg_.top_k * (G == 1 ? 1 : 2);
    ensure_rows(round_up(units + static_cast<size_t>(N) * 127, 128));
  }

  // checked when the expert GEMMs are enqueued: a placement switch and the
  // operand table that goes with it arrive in two calls
  const int32_t* operand_slots_dev() const {
    if (operand_slot_.empty()) return nullptr;
    for (int e : local_)
      if (operand_slot_[e] < 0 || operand_slot_[e] >= operand_cap_)
        throw std::out_of_range("fm_layer: local expert " + std::to_string(e) + " has no operand slot");
    return local_slot_dev_;
  }
  int operand_groups() const { return operand_slot_.empty() ? nl() : operand_cap_; }

  void ensure_rows(size_t rows) {
    if (rows <= row_cap_) return;
    const size_t d = cfg_.d_model, f = cfg_.d_ff;
    row_cap_ = std::max<size_t>(rows, 128);
    if (!p2p_) {  // with P2P these live in the shared arena, sized for the worst case
      x_perm_.reset(2 * row_cap_ * d);
      y_perm_.reset(2 * row_cap_ * d);
      dy_perm_.reset(2 * row_cap_ * d);
      dx_perm_.reset(2 * row_cap_ * d);
      dl_rows_.reset(4 * row_cap_);
    }
    act_.reset(2 * row_cap_ * f);
    dh_.reset(2 * row_cap_ * f);
    row_expert_.reset(4 * row_cap_);
    relu_mask_.reset(4 * row_cap_ * (f / 32));
    tile_colsum_.reset(4 * (row_cap_ / 128) * f);
    tile_sum_.reset(4 * 2 * (row_cap_ / 128) * d);  // per-tile db2 / dWg partials
  }

  // ------------------------------------------------------------ fused single-GPU step
  void forward(const void* x, int T, const void* wg, const void* w1, const float* b1,
               const void* w2, const float* b2, void* y, cudaStream_t s) {
    if (cfg_.num_gpus != 1)
      throw std::logic_error("fm_layer_forward: fused path is single-GPU; use the phase API");
    check_tokens(T);
    gate(x, T, wg, nullptr, s, /*defer_scan=*/true);
    route_device(s);
    timer_.begin(FM_PHASE_DISPATCH, s);
    launch_dispatch(x, T, cfg_.d_model, cfg_.top_k, cfg_.num_experts, 1, 0, true,
                    topk_idx_.as<int32_t>(), tile_rank_.as<int32_t>(), tile_base_.as<int32_t>(),
                    plan_, pos_.as<int32_t>(), x_perm_.p, nullptr, s, nullptr,
                    /*pad_buf (zeroed by trailing blocks)*/ x_perm_.p, nl());
    timer_.end(s);
    expert_forward(w1, b1, w2, b2, s);
    combine(y_perm_.p, y, s);
    saved_wg_ = wg;
    saved_w1_ = w1;
    saved_w2_ = w2;
    fused_state_ = true;
  }

  void backward(const void* dy, void* dx, float* dwg, float* dw1, float* db1, float* dw2,
                float* db2, cudaStream_t s) {
    if (cfg_.num_gpus != 1)
      throw std::logic_error("fm_layer_backward: fused path is single-GPU; use the phase API");
    if (!fused_state_) throw std::logic_error("fm_layer_backward: no forward state");
    side_jobs_ = 0;
    combine_backward(dy, y_perm_.p, dy_perm_.p, s, /*zero_pads=*/true);
    // the dispatched units' share of dWg = per-tile column sums of X_perm
    // weighted by dl per row, reduced with db1 / db2 (dropped units: below)
    const bool dwg_tiles = dwg && cfg_.top_k > 1 && nl() > 0;
#if FM_BWD_ORDER == 4
    // The memory-bound backward work rides on spare CTA pairs of the two
    // weight-gradient launches (each runs group-aligned on 64 of 74 pairs):
    // the db2 / dWg tile column sums beside FFN2's (they need dY_perm, dl),
    // the un-permute beside FFN1's, which therefore runs after both dgrads
    // (it needs dX_perm). What a launch cannot host (no spare pairs at this
    // shape) runs as its own kernel afterwards.
    bool unpermuted = false;
    if (nl() > 0) {
      SideJob sums = tile_sum_side(db2, dwg_tiles ? dwg : nullptr);
      wgrad2(dw2, s, &sums);           // dY_perm, act (+ tile column sums)
      dgrad2(saved_w2_, db1, s);       // dY_perm, W2 -> dH (+ db1 tile partials)
      dgrad1(saved_w1_, s);            // dH, W1 -> dX_perm
      SideJob unp = unpermute_side(dx);
      // the tile partials are complete once the column sums ran beside FFN2's
      // wgrad: their per-expert reduce rides beside FFN1's too
      if (sums.clusters > 0) add_reduce_jobs(unp, db1, db2, dwg_tiles ? dwg : nullptr);
      wgrad1(dw1, s, (unp.kind || unp.reduce_jobs) ? &unp : nullptr);  // dH, X_perm (+ un-permute, reduce)
      unpermuted = unp.clusters > 0 && unp.kind == 2;
      const bool reduced = unp.clusters > 0 && unp.reduce_jobs > 0;
      side_jobs_ = (sums.clusters > 0 ? 1 : 0) | (unpermuted ? 2 : 0) | (reduced ? 4 : 0);
      if (!reduced) bias_grads(db1, db2, s, dwg_tiles ? dwg : nullptr, /*sums_done=*/sums.clusters > 0);
    }
    if (!unpermuted) unpermute(dx_perm_.p, saved_wg_, dx, s);
    gate_wgrad(x_perm_.p, plan_.totals, static_cast<int>(row_cap_), dwg, s, dwg_tiles);
#elif FM_BWD_ORDER == 3
    // as order 2, then un-permute right after the dgrad that produced dX_perm
    // (its reads hit the dX_perm lines still in L2) and the bias / gate tile
    // sums last: they only read, so the step ends with a clean L2 and the
    // next step's gate does not pay the write-back of dx
    if (nl() > 0) {
      wgrad2(dw2, s);
      dgrad2(saved_w2_, db1, s);
      wgrad1(dw1, s);
      dgrad1(saved_w1_, s);
    }
    unpermute(dx_perm_.p, saved_wg_, dx, s);
    if (nl() > 0) bias_grads(db1, db2, s, dwg_tiles ? dwg : nullptr);
    gate_wgrad(x_perm_.p, plan_.totals, static_cast<int>(row_cap_), dwg, s, dwg_tiles);
#elif FM_BWD_ORDER == 2
    // each weight-gradient GEMM right before a dgrad GEMM: the dirty f32 dW
    // lines it leaves in L2 are written back while the next GEMM is
    // tensor-bound (HBM idle), not by the memory-bound kernels that follow
    // the last one (the next step's gate paid it: profiles/r02_gate_context.log)
    if (nl() > 0) {
      // the db2 / dWg tile column sums (memory-bound) ride on spare CTA pairs
      // of the first weight-gradient launch (tensor-bound)
      SideJob side = tile_sum_side(db2, dwg_tiles ? dwg : nullptr);
      wgrad2(dw2, s, &side);           // dY_perm, act (+ tile column sums)
      dgrad2(saved_w2_, db1, s);       // dY_perm, W2 -> dH (+ db1 tile partials)
      wgrad1(dw1, s);                  // dH, X_perm
      dgrad1(saved_w1_, s);            // dH, W1 -> dX_perm
      bias_grads(db1, db2, s, dwg_tiles ? dwg : nullptr, /*sums_done=*/side.clusters > 0);
    }
    unpermute_backward(dx_perm_.p, x_perm_.p, plan_.totals, static_cast<int>(row_cap_), saved_wg_, dx,
                       dwg, s, dwg_tiles);
#elif FM_BWD_ORDER == 1
    // memory-bound work first (dx right after the dgrad that produced dX_perm,
    // then the bias / gate tile sums), the weight-gradient GEMMs last
    expert_dgrad(saved_w1_, saved_w2_, db1, s);
    unpermute(dx_perm_.p, saved_wg_, dx, s);
    bias_grads(db1, db2, s, dwg_tiles ? dwg : nullptr);
    gate_wgrad(x_perm_.p, plan_.totals, static_cast<int>(row_cap_), dwg, s, dwg_tiles);
    expert_wgrad(dw1, dw2, s);
#else
    expert_backward(saved_w1_, saved_w2_, dw1, db1, dw2, db2, s, dwg_tiles ? dwg : nullptr);
    unpermute_backward(dx_perm_.p, x_perm_.p, plan_.totals, static_cast<int>(row_cap_), saved_wg_, dx,
                       dwg, s, dwg_tiles);
#endif
  }

  // ------------------------------------------------------------ phases
  // Gate + per-expert scan. hist_out (device int64 [N], optional) receives
  // this GPU's TokenDemand column for the all-gather.
  // defer_scan (fused single-GPU step): the expert scan runs inside the plan
  // launch (route_device) when the shape allows — one launch less between
  // the gate and the dispatch
  void gate(const void* x, int T, const void* wg, int64_t* hist_out, cudaStream_t s, bool defer_scan = false) {
    check_tokens(T);
    const int N = cfg_.num_experts, G = cfg_.num_gpus;
    timer_.begin(FM_PHASE_GATE, s);
    launch_gate(x, wg, T, N, cfg_.d_model, cfg_.top_k, topk_idx_.as<int32_t>(),
                topk_w_.as<float>(), tile_rank_.as<int32_t>(), tile_counts_.as<int32_t>(), s);
    timer_.end(s);
    cur_T_ = T;
    saved_x_ = x;
    fused_state_ = false;
    scan_deferred_ =
        defer_scan && !hist_out && plan_can_fuse_scan(N, G, gate_num_tiles(T, N)) && !drops_enabled();
    if (scan_deferred_) return;
    timer_.begin(FM_PHASE_SCAN, s);
    if (G > 1) FM_CUDA(cudaMemsetAsync(demand_.p, 0, sizeof(int64_t) * N * G, s));
    launch_expert_scan(tile_counts_.as<int32_t>(), gate_num_tiles(T, N), N, tile_base_.as<int32_t>(),
                       hist_.as<int64_t>(), demand_.as<int64_t>(), G, cfg_.rank, s);
    if (hist_out)
      FM_CUDA(cudaMemcpyAsync(hist_out, hist_.p, sizeof(int64_t) * N, cudaMemcpyDeviceToDevice, s));
    timer_.end(s);
    if (p2p_) ++epoch_;  // one exchange epoch per step, the same on every GPU
  }

  // route() on the device over demand_ (already complete), then the plan. In
  // StaticEP mode the demand first goes through the capacity-drop rule.
  // gathered_GN (optional): the all-gathered histograms, transposed into the
  // TokenDemand by the plan launch itself (no separate transpose kernel)
  void route_device(cudaStream_t s, const int64_t* gathered_GN = nullptr) {
    const int N = cfg_.num_experts, G = cfg_.num_gpus;
    timer_.begin(FM_PHASE_ROUTE, s);
    const int64_t* routed = demand_.as<int64_t>();
    if (gathered_GN && drops_enabled()) {  // the capacity rule reads the demand first
      launch_demand_transpose(gathered_GN, N, G, demand_.as<int64_t>(), s);
      gathered_GN = nullptr;
    }
    if (drops_enabled()) {
      static_ep_kept_device(demand_.as<int64_t>(), N, G, capacity_factor_, kept_.as<int64_t>(),
                            dropped_.as<int64_t>(), s);
      routed = kept_.as<int64_t>();
    }
    // route() over the demand and the dispatch plan in one single-block launch
    if (scan_deferred_) {  // expert scan + route + plan in one launch
      launch_plan(flows_.as<int64_t>(), N, G, cfg_.rank, local_expert_dev_, nl(), plan_, s, counts_dev_, routed,
                  route_status_.as<int32_t>(), nullptr, tile_counts_.as<int32_t>(), gate_num_tiles(cur_T_, N),
                  tile_base_.as<int32_t>(), hist_.as<int64_t>());
      scan_deferred_ = false;
    } else {
      launch_plan(flows_.as<int64_t>(), N, G, cfg_.rank, local_expert_dev_, nl(), plan_, s,
                  counts_dev_, routed, route_status_.as<int32_t>(), gathered_GN);
    }
    timer_.end(s);
  }

  // Multi-GPU: full demand from the all-gathered per-GPU histograms
  // (gathered_GN[g][e], device), route + plan, then the per-peer row counts
  // for the all-to-all (host; synchronises the stream: NCCL needs them).
  void route_gathered(const int64_t* gathered_GN, int32_t* send_rows, int32_t* recv_rows,
                      cudaStream_t s) {
    const int N = cfg_.num_experts, G = cfg_.num_gpus;
    route_device(s, gathered_GN);
    FM_CUDA(cudaMemcpyAsync(host_counts_.data(), plan_.send_rows, sizeof(int32_t) * 2 * G,
                            cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaMemcpyAsync(host_counts_.data() + 2 * G, route_status_.p, sizeof(int32_t),
                            cudaMemcpyDeviceToHost, s));
    FM_CUDA(cudaStreamSynchronize(s));
    if (host_counts_[2 * G] != 0)
      throw std::invalid_argument("route: an expert has demand but no replica");
    int recv_total = 0, send_total = 0;
    for (int g = 0; g < G; ++g) {
      send_rows[g] = host_counts_[g];
      recv_rows[g] = host_counts_[G + g];
      send_total += send_rows[g];
      recv_total += recv_rows[g];
    }
    recv_total_ = recv_total;
    send_total_ = send_total;
    ensure_rows(round_up(static_cast<size_t>(recv_total) + static_cast<size_t>(nl()) * 127, 128));
  }

  void dispatch_send(const void* x, void* send_buf, cudaStream_t s) {
    timer_.begin(FM_PHASE_DISPATCH, s);
    launch_dispatch(x, cur_T_, cfg_.d_model, cfg_.top_k, cfg_.num_experts, cfg_.num_gpus, cfg_.rank,
                    false, topk_idx_.as<int32_t>(), tile_rank_.as<int32_t>(),
                    tile_base_.as<int32_t>(), plan_, pos_.as<int32_t>(), send_buf,
                    row_expert_.as<int32_t>(), s);
    timer_.end(s);
  }

  // a2a receive order (src-major, expert-minor) -> padded expert segments, and back.
  void recv_to_perm(const void* recv_buf, void* perm, cudaStream_t s) {
    timer_.begin(FM_PHASE_RELAYOUT, s);
    launch_zero_pad(perm, cfg_.d_model, plan_, nl(), nullptr, s);
    launch_relayout(const_cast<void*>(recv_buf), perm, cfg_.d_model, cfg_.num_gpus, nl(), plan_,
                    recv_total_, 0, s);
    timer_.end(s);
  }
  void perm_to_recv(const void* perm, void* recv_buf, cudaStream_t s) {
    timer_.begin(FM_PHASE_RELAYOUT, s);
    launch_relayout(recv_buf, const_cast<void*>(perm), cfg_.d_model, cfg_.num_gpus, nl(), plan_,
                    recv_total_, 1, s);
    timer_.end(s);
  }

  // gate (P2P): FFN1 waits per 128-row tile for the sources whose rows it holds
  // ready (P2P, optional): the FFN2 GEMM's last CTA publishes "Y ready"
  void expert_forward(const void* w1, const float* b1, const void* w2, const float* b2,
                      cudaStream_t s, const ArrivalGate* gate = nullptr, const P2P* ready = nullptr) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0) {
      if (ready) launch_p2p_signal(*ready, cfg_.num_gpus, cfg_.rank, ready->signal_slot, ready->epoch, s);
      return;
    }
    const int rows = static_cast<int>(row_cap_);
    timer_.begin(FM_PHASE_FFN1_FWD, s);
    grouped_gemm(FM_GEMM_FWD_BIAS_RELU, x_perm_.p, w1, act_.p, b1, relu_mask_.p, plan_.seg_start,
                 plan_.seg_rows, plan_.mtile_prefix, Nl, rows, 0, f, d, s, gate, operand_slots_dev(),
                 operand_groups());
    timer_.end(s);
    timer_.begin(FM_PHASE_FFN2_FWD, s);
    grouped_gemm(FM_GEMM_FWD_BIAS, act_.p, w2, y_perm_.p, b2, nullptr, plan_.seg_start,
                 plan_.seg_rows, plan_.mtile_prefix, Nl, rows, 0, d, f, s, nullptr, operand_slots_dev(),
                 operand_groups(), nullptr, ready);
    timer_.end(s);
  }

  // dwg_tiles (fused path): also the gate-weight gradient of the dispatched
  // units, from X_perm and dl per dispatch row, in the same tile passes.
  // signal_dx (P2P): tell the sources dX_perm is complete right after the
  // FFN1 dgrad, so their un-permute overlaps this GPU's weight gradients.
  void expert_backward(const void* w1, const void* w2, float* dw1, float* db1, float* dw2,
                       float* db2, cudaStream_t s, float* dwg_tiles = nullptr, bool signal_dx = false,
                       const ArrivalGate* gate = nullptr) {
    side_jobs_ = 0;
    unpermuted_ = false;
    if (nl() == 0) {
      if (signal_dx) p2p_signal(3, s);
      return;
    }
    // "dX ready" published by the FFN1 dgrad GEMM's last CTA (no signal launch)
    const P2P dx_ready = p2p_args(3);
    dgrad2(w2, db1, s, gate);
    dgrad1(w1, s, signal_dx ? &dx_ready : nullptr);
    SideJob side = tile_sum_side(db2, dwg_tiles);
    wgrad2(dw2, s, &side);
    // P2P with the un-permute bound (fm_layer_p2p_bind_dx): it rides beside
    // the FFN1 weight gradients, reading the peers' dX rows once they are ready
    SideJob unp = (signal_dx && p2p_ && bound_dx_) ? unpermute_side(bound_dx_, bound_wg_) : SideJob{};
    // the reduce of the tile partials beside it too, once the column sums ran
    // beside FFN2's wgrad (rows of experts hosted elsewhere zeroed first)
    if (side.clusters > 0) {
      if (dwg_tiles && nl() < cfg_.num_experts)
        FM_CUDA(cudaMemsetAsync(dwg_tiles, 0, sizeof(float) * cfg_.num_experts * cfg_.d_model, s));
      add_reduce_jobs(unp, db1, db2, dwg_tiles, /*remote_rows_zeroed=*/true);
    }
    wgrad1(dw1, s, (unp.kind || unp.reduce_jobs) ? &unp : nullptr);
    unpermuted_ = unp.clusters > 0 && unp.kind == 2;
    const bool reduced = unp.clusters > 0 && unp.reduce_jobs > 0;
    side_jobs_ = (side.clusters > 0 ? 1 : 0) | (unpermuted_ ? 2 : 0) | (reduced ? 4 : 0);
    if (!reduced) bias_grads(db1, db2, s, dwg_tiles, /*sums_done=*/side.clusters > 0);
  }

  // dH (masked by relu'), db1 tile partials, dX_perm
  void expert_dgrad(const void* w1, const void* w2, float* db1, cudaStream_t s, const ArrivalGate* gate = nullptr) {
    dgrad2(w2, db1, s, gate);
    dgrad1(w1, s);
  }
  // dA = dY . W2 masked by relu'(H) -> dH [rows, f]; db1 partials per 128-row tile
  void dgrad2(const void* w2, float* db1, cudaStream_t s, const ArrivalGate* gate = nullptr) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0) return;
    const int rows = static_cast<int>(row_cap_);
    timer_.begin(FM_PHASE_FFN2_DGRAD, s);
    grouped_gemm(FM_GEMM_DGRAD_RELU_MASK, dy_perm_.p, w2, dh_.p,
                 db1 ? tile_colsum_.as<float>() : nullptr, relu_mask_.p, plan_.seg_start,
                 plan_.seg_rows, plan_.mtile_prefix, Nl, rows, 0, f, d, s, gate, operand_slots_dev(),
                 operand_groups());
    timer_.end(s);
  }
  // dX = dH . W1 -> [rows, d]; ready (P2P, optional): its last CTA publishes "dX ready"
  void dgrad1(const void* w1, cudaStream_t s, const P2P* ready = nullptr) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0) return;
    const int rows = static_cast<int>(row_cap_);
    timer_.begin(FM_PHASE_FFN1_DGRAD, s);
    grouped_gemm(FM_GEMM_DGRAD, dh_.p, w1, dx_perm_.p, nullptr, nullptr, plan_.seg_start,
                 plan_.seg_rows, plan_.mtile_prefix, Nl, rows, 0, d, f, s, nullptr, operand_slots_dev(),
                 operand_groups(), nullptr, ready);
    timer_.end(s);
  }

  void expert_wgrad(float* dw1, float* dw2, cudaStream_t s) {
    wgrad2(dw2, s);
    wgrad1(dw1, s);
  }
  // dW2[li] = dY^T . act  [d, f]; side (optional): tile column sums run by
  // spare CTA pairs of the same launch
  void wgrad2(float* dw2, cudaStream_t s, SideJob* side = nullptr) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0 || !dw2) return;
    timer_.begin(FM_PHASE_FFN2_WGRAD, s);
    grouped_gemm(FM_GEMM_WGRAD, dy_perm_.p, act_.p, dw2, nullptr, nullptr, plan_.seg_start,
                 plan_.seg_rows, nullptr, Nl, static_cast<int>(row_cap_), d, f, 0, s, nullptr, nullptr, 0,
                 side);
    timer_.end(s);
  }
  // dW1[li] = dH^T . X  [f, d]; side (optional): memory-bound work run by
  // spare CTA pairs of the same launch
  void wgrad1(float* dw1, cudaStream_t s, SideJob* side = nullptr) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0 || !dw1) return;
    timer_.begin(FM_PHASE_FFN1_WGRAD, s);
    grouped_gemm(FM_GEMM_WGRAD, dh_.p, x_perm_.p, dw1, nullptr, nullptr, plan_.seg_start,
                 plan_.seg_rows, nullptr, Nl, static_cast<int>(row_cap_), f, d, 0, s, nullptr, nullptr, 0,
                 side);
    timer_.end(s);
  }

  // The single-GPU un-permute (dx from dX_perm and the gate rows) as a side
  // job of a weight-gradient launch.
  SideJob unpermute_side(void* dx, const void* wg = nullptr) {
    SideJob sd{};
    if (!side_enabled_ || !dx || cur_T_ <= 0) return sd;
    if (cfg_.num_gpus != 1 && !p2p_) return sd;  // NCCL layouts: dX rows come back through the a2a
    sd.kind = 2;
    sd.dXp = dx_perm_.p;
    sd.pos = pos_.as<int32_t>();
    sd.idx = topk_idx_.as<int32_t>();
    sd.dl = dl_.as<float>();
    sd.wg = wg ? wg : saved_wg_;
    sd.dx = dx;
    if (p2p_) sd.pp = p2p_args(-1, /*wait for "dX ready"*/ 3);
    sd.T = cur_T_;
    sd.k = cfg_.top_k;
    sd.d = cfg_.d_model;
    sd.gate_grad = cfg_.top_k > 1 ? 1 : 0;
    sd.est_rows = cur_T_ * cfg_.top_k;
    return sd;
  }

  // The per-expert reduce of the db1 / db2 / dWg tile partials (what
  // bias_grads launches) appended to a side job. The dWg rows of experts
  // hosted elsewhere must already be zero (remote_rows_zeroed) unless every
  // expert is local.
  void add_reduce_jobs(SideJob& sd, float* db1, float* db2, float* dwg_tiles, bool remote_rows_zeroed = false) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0 || (Nl < cfg_.num_experts && dwg_tiles && !remote_rows_zeroed)) return;
    const int max_tiles = static_cast<int>(row_cap_ / 128);
    float* part_db2 = tile_sum_.as<float>();
    float* part_dwg = part_db2 + static_cast<size_t>(max_tiles) * d;
    auto add = [&](const float* partial, int cols, const int32_t* oi, float* out) {
      if (!out) return;
      sd.r_partial[sd.reduce_jobs] = partial;
      sd.r_cols[sd.reduce_jobs] = cols;
      sd.r_out_index[sd.reduce_jobs] = oi;
      sd.r_out[sd.reduce_jobs++] = out;
    };
    add(tile_colsum_.as<float>(), f, nullptr, db1);
    add(part_db2, d, nullptr, db2);
    add(part_dwg, d, local_expert_dev_, dwg_tiles);
    sd.mtile_prefix = plan_.mtile_prefix;
    sd.Nl = Nl;
    if (!sd.est_rows) sd.est_rows = cur_T_ * cfg_.top_k;
  }

  // The db2 / dWg tile column-sum jobs (dY_perm; dl-weighted X_perm) as a
  // side job of a weight-gradient launch (fm_layer_set_side_jobs), else none.
  SideJob tile_sum_side(float* db2, float* dwg_tiles) {
    SideJob sd{};
    const int Nl = nl(), d = cfg_.d_model;
    if (!side_enabled_ || Nl == 0) return sd;
    sd.kind = 1;
    const int max_tiles = static_cast<int>(row_cap_ / 128);
    float* part_db2 = tile_sum_.as<float>();
    float* part_dwg = part_db2 + static_cast<size_t>(max_tiles) * d;
    if (dwg_tiles) {
      sd.buf[sd.njobs] = x_perm_.p;
      sd.row_w[sd.njobs] = dl_rows_.as<float>();
      sd.partial[sd.njobs++] = part_dwg;
    }
    if (db2) {
      sd.buf[sd.njobs] = dy_perm_.p;
      sd.row_w[sd.njobs] = nullptr;
      sd.partial[sd.njobs++] = part_db2;
    }
    if (sd.njobs == 0) return SideJob{};
    sd.cols = d;
    sd.mtile_prefix = plan_.mtile_prefix;
    sd.seg_start = plan_.seg_start;
    sd.seg_real = plan_.seg_real;
    sd.Nl = Nl;
    sd.est_rows = cur_T_ * cfg_.top_k;
    return sd;
  }

  // bias / gate-weight gradients: per-128-row-tile column sums (db1's come from
  // the dgrad epilogue; dY_perm's and the dl-weighted X_perm's here, or already
  // on the side of the FFN2 weight-gradient launch: sums_done), then one
  // fixed-order reduce per segment (deterministic, no atomics)
  void bias_grads(float* db1, float* db2, cudaStream_t s, float* dwg_tiles, bool sums_done = false) {
    const int Nl = nl(), d = cfg_.d_model, f = cfg_.d_ff;
    if (Nl == 0) return;
    timer_.begin(FM_PHASE_BIAS_GRAD, s);
    const int max_tiles = static_cast<int>(row_cap_ / 128);
    float* part_db2 = tile_sum_.as<float>();
    float* part_dwg = part_db2 + static_cast<size_t>(max_tiles) * d;
    if (!sums_done)
      launch_segment_tile_colsum(dwg_tiles ? x_perm_.p : nullptr, dl_rows_.as<float>(), part_dwg,
                                 db2 ? dy_perm_.p : nullptr, nullptr, part_db2, d, plan_, Nl, max_tiles, s);
    if (dwg_tiles && Nl < cfg_.num_experts)  // experts hosted elsewhere keep a zero row here
      FM_CUDA(cudaMemsetAsync(dwg_tiles, 0, sizeof(float) * cfg_.num_experts * d, s));
    launch_segment_tile_reduce(tile_colsum_.as<float>(), f, nullptr, db1, part_db2, d, nullptr, db2, part_dwg, d,
                               local_expert_dev_, dwg_tiles, plan_, Nl, s);
    timer_.end(s);
  }

  // y[t] = sum_j w[t,j] back[pos[t,j]] — back is Y_perm (G == 1) or the
  // returned rows in dispatch order (G > 1).
  void combine(const void* back, void* y, cudaStream_t s) {
    timer_.begin(FM_PHASE_COMBINE_FWD, s);
    launch_combine_fwd(back, pos_.as<int32_t>(), topk_w_.as<float>(), cur_T_, cfg_.d_model,
                       cfg_.top_k, y, s);
    timer_.end(s);
  }

  // zero_pads (fused path): dsend is dY_perm; trailing blocks zero its padding rows.
  void combine_backward(const void* dy, const void* back, void* dsend, cudaStream_t s, bool zero_pads = false) {
    const bool gate_grad = cfg_.top_k > 1;
    timer_.begin(FM_PHASE_COMBINE_BWD, s);
    launch_combine_bwd(dy, back, pos_.as<int32_t>(), topk_w_.as<float>(), cur_T_, cfg_.d_model,
                       cfg_.top_k, dsend, dl_.as<float>(), gate_grad ? dl_rows_.as<float>() : nullptr,
                       s, nullptr, zero_pads ? &plan_ : nullptr, nl());
    timer_.end(s);
  }

  // dx and the gate weight gradient. dback: dX rows in dispatch order;
  // xrows: the dispatched activations in the same order (X_perm or the send
  // buffer); rows_dev / rows: how many of them.
  // dwg_done: the dispatched units' share of dWg is already in dwg (fused
  // path, tile sums); only the units dropped by the capacity rule remain.
  void unpermute_backward(const void* dback, const void* xrows, const int* rows_dev, int rows,
                          const void* wg, void* dx, float* dwg, cudaStream_t s, bool dwg_done = false) {
    unpermute(dback, wg, dx, s);
    gate_wgrad(xrows, rows_dev, rows, dwg, s, dwg_done);
  }
  void unpermute(const void* dback, const void* wg, void* dx, cudaStream_t s) {
    const int T = cur_T_, d = cfg_.d_model, k = cfg_.top_k;
    timer_.begin(FM_PHASE_UNPERMUTE, s);
    launch_unpermute_bwd(dback, pos_.as<int32_t>(), topk_idx_.as<int32_t>(), dl_.as<float>(), wg, T,
                         d, k, k > 1, dx, s);
    timer_.end(s);
  }
  void gate_wgrad(const void* xrows, const int* rows_dev, int rows, float* dwg, cudaStream_t s, bool dwg_done) {
    const int T = cur_T_, d = cfg_.d_model, k = cfg_.top_k, N = cfg_.num_experts;
    const bool gate_grad = k > 1;
    if (dwg) {
      timer_.begin(FM_PHASE_GATE_WGRAD, s);
      if (!dwg_done && !gate_grad) FM_CUDA(cudaMemsetAsync(dwg, 0, sizeof(float) * N * d, s));
      if (gate_grad) {
        // the send buffer's (dst, expert) chunks, piece by piece (deterministic);
        // only the NCCL layout gets here (fused / P2P: tile sums, dwg_done)
        if (!dwg_done) {
          if (rows_dev) {  // fused layout with no local expert: no dispatch rows here
            FM_CUDA(cudaMemsetAsync(dwg, 0, sizeof(float) * N * d, s));
          } else {
          const size_t need = sizeof(float) * static_cast<size_t>(gate_wgrad_pieces(rows, N, cfg_.num_gpus)) * d +
                              sizeof(int32_t) * (N * cfg_.num_gpus + 1);
          if (gw_partial_.bytes < need) gw_partial_.reset(need);
          launch_gate_wgrad(xrows, rows, d, dl_rows_.as<float>(), plan_, N, cfg_.num_gpus, gw_partial_.as<float>(),
                            dwg, s);
          }
        }
        // units dropped by the capacity rule are in no dispatch row
        if (drops_enabled())
          launch_dropped_gate_wgrad(saved_x_, pos_.as<int32_t>(), topk_idx_.as<int32_t>(),
                                    dl_.as<float>(), T, d, k, N, drop_partial(T), dwg, s);
      }
      timer_.end(s);
    }
  }

  // ------------------------------------------------------------ P2P transport
  // Token rows move over NVLink inside the kernels that produce / consume
  // them (no staging buffers, no all-to-all, no relayout): dispatch writes
  // x rows into the expert GPU's X_perm, combine reads Y rows from the expert
  // GPU's Y_perm, combine_bwd writes dY rows (and dl) into its dY_perm,
  // un-permute reads dX rows from its dX_perm. Arrival flags order them.
  void enable_p2p() {
    if (p2p_) return;
    const size_t N = cfg_.num_experts, G = cfg_.num_gpus, T = cfg_.max_tokens, k = cfg_.top_k;
    const size_t d = cfg_.d_model;
    if (G > static_cast<size_t>(kMaxPeers)) throw std::invalid_argument("fm_layer_enable_p2p: at most 64 GPUs");
    // worst case of route(): every unit of every GPU lands here, plus padding
    const size_t rows = round_up(G * T * k + N * 127, 128);
    auto al = [](size_t b) { return round_up(b, 256); };
    const size_t rb = al(2 * rows * d);
    pp_ = P2P{};
    pp_.signal_slot = -1;
    pp_.wait_slot = -1;
    pp_.x_off = 0;
    pp_.y_off = rb;
    pp_.dy_off = 2 * rb;
    pp_.dx_off = 3 * rb;
    pp_.dl_off = 4 * rb;
    pp_.flag_off = 4 * rb + al(4 * rows);
    const size_t bytes = pp_.flag_off + al(sizeof(unsigned long long) * kP2PSlots * kMaxPeers);
    arena_.reset(bytes);
    FM_CUDA(cudaMemset(arena_.p, 0, bytes));
    char* a = arena_.as<char>();
    p2p_ = true;
    x_perm_.view(a + pp_.x_off, 2 * rows * d);
    y_perm_.view(a + pp_.y_off, 2 * rows * d);
    dy_perm_.view(a + pp_.dy_off, 2 * rows * d);
    dx_perm_.view(a + pp_.dx_off, 2 * rows * d);
    dl_rows_.view(a + pp_.dl_off, 4 * rows);
    row_cap_ = 0;
    ensure_rows(rows);  // the local per-row buffers at the same capacity
    unit_dst_.reset(sizeof(int32_t) * T * k);
    p2p_done_.reset(sizeof(unsigned int) * kP2PSlots);
    FM_CUDA(cudaMemset(p2p_done_.p, 0, sizeof(unsigned int) * kP2PSlots));
    p2p_err_.reset(sizeof(int));
    FM_CUDA(cudaMemset(p2p_err_.p, 0, sizeof(int)));
    pp_.unit_dst = unit_dst_.as<int32_t>();
    peer_ipc_.assign(G, false);
    pp_.base[cfg_.rank] = a;
    plan_.peer_row = peer_row_mem_;
    tile_src_mask_.reset(sizeof(unsigned long long) * (rows / 128));
    plan_.tile_src_mask = tile_src_mask_.as<unsigned long long>();
  }
  void p2p_handle(void* out64) {
    require_p2p();
    cudaIpcMemHandle_t h;
    FM_CUDA(cudaIpcGetMemHandle(&h, arena_.p));
    std::memcpy(out64, &h, sizeof(h));
  }
  void p2p_open_peer(int peer, const void* handle64) {
    require_p2p();
    check_peer(peer);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    void* ptr = nullptr;
    FM_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    close_peer(peer);
    pp_.base[peer] = static_cast<char*>(ptr);
    peers_distinct_ = -1;
    peer_ipc_[peer] = true;
  }
  void p2p_link_peer(int peer, Layer& other) {
    require_p2p();
    check_peer(peer);
    if (!other.p2p_ || other.arena_.bytes != arena_.bytes)
      throw std::invalid_argument("fm_layer_p2p_link_peer: peer layer has a different P2P arena");
    close_peer(peer);
    pp_.base[peer] = other.arena_.as<char>();
    peers_distinct_ = -1;
  }
  int p2p_status() {
    if (!p2p_) return 0;
    int e = 0;
    FM_CUDA(cudaMemcpy(&e, p2p_err_.p, sizeof(int), cudaMemcpyDeviceToHost));
    return e;
  }
  void route_p2p(const int64_t* gathered_GN, cudaStream_t s) {
    require_linked();
    route_device(s, gathered_GN);  // demand transpose + flows + plan incl. every destination's X_perm rows
  }
  // P2P launch parameters; with slot >= 0 the kernel's last block releases
  // the rows it pushed (flags[slot][me] = epoch on every peer).
  P2P p2p_args(int slot, int wait_slot = -1) const {
    P2P p = pp_;
    p.signal_slot = slot;
    p.wait_slot = wait_slot;
    p.err = p2p_err_.as<int>();
    p.me = cfg_.rank;
    p.world = cfg_.num_gpus;
    p.epoch = epoch_;
    p.done = p2p_done_.as<unsigned int>();
    return p;
  }
  void dispatch_p2p(const void* x, cudaStream_t s) {
    timer_.begin(FM_PHASE_DISPATCH, s);
    const P2P p = p2p_args(0);
    launch_dispatch(x, cur_T_, cfg_.d_model, cfg_.top_k, cfg_.num_experts, cfg_.num_gpus, cfg_.rank, false,
                    topk_idx_.as<int32_t>(), tile_rank_.as<int32_t>(), tile_base_.as<int32_t>(), plan_,
                    pos_.as<int32_t>(), nullptr, nullptr, s, &p, x_perm_.p, nl());  // + own pad rows
    timer_.end(s);
  }
  ArrivalGate p2p_gate(int slot) {
    ArrivalGate g;
    g.flags = reinterpret_cast<const unsigned long long*>(arena_.as<char>() + pp_.flag_off) + slot * kMaxPeers;
    g.tile_src_mask = tile_src_mask_.as<unsigned long long>();
    g.epoch = epoch_;
    g.err = p2p_err_.as<int>();
    return g;
  }
  // No step-wide wait: FFN1's producer waits per 128-row tile for the sources
  // whose rows the tile holds, so local rows (route() keeps them local first)
  // compute while remote ones are still arriving over NVLink.
  void expert_forward_p2p(const void* w1, const float* b1, const void* w2, const float* b2, cudaStream_t s) {
    const ArrivalGate gate = p2p_gate(0);
    const P2P y_ready = p2p_args(1);  // "Y ready" published by the FFN2 GEMM's last CTA
    expert_forward(w1, b1, w2, b2, s, &gate, &y_ready);
  }
  void combine_p2p(void* y, cudaStream_t s) {
    timer_.begin(FM_PHASE_COMBINE_FWD, s);
    const P2P p = p2p_args(-1, /*wait for "Y ready"*/ 1);
    launch_combine_fwd(y_perm_.p, pos_.as<int32_t>(), topk_w_.as<float>(), cur_T_, cfg_.d_model, cfg_.top_k, y, s,
                       &p);
    timer_.end(s);
  }
  void combine_backward_p2p(const void* dy, cudaStream_t s) {
    const bool gate_grad = cfg_.top_k > 1;
    timer_.begin(FM_PHASE_COMBINE_BWD, s);
    const P2P p = p2p_args(2);
    launch_combine_bwd(dy, y_perm_.p, pos_.as<int32_t>(), topk_w_.as<float>(), cur_T_, cfg_.d_model, cfg_.top_k,
                       dy_perm_.p, dl_.as<float>(), gate_grad ? dl_rows_.as<float>() : nullptr, s, &p, &plan_,
                       nl());  // trailing blocks zero this GPU's dY_perm pad rows
    timer_.end(s);
  }
  // dwg (optional) receives this GPU's share of the gate-weight gradient: its
  // hosted units (dl-weighted X_perm tile sums), to be summed over all GPUs.
  void expert_backward_p2p(const void* w1, const void* w2, float* dw1, float* db1, float* dw2, float* db2,
                           float* dwg, cudaStream_t s) {
    const bool dwg_tiles = dwg && cfg_.top_k > 1 && nl() > 0;
    if (dwg && !dwg_tiles)
      FM_CUDA(cudaMemsetAsync(dwg, 0, sizeof(float) * cfg_.num_experts * cfg_.d_model, s));
    // the FFN2 dgrad (first reader of the pushed dY rows) waits per tile; the
    // later readers (weight gradients, tile sums) run after it
    const ArrivalGate gate = p2p_gate(2);
    expert_backward(w1, w2, dw1, db1, dw2, db2, s, dwg_tiles ? dwg : nullptr, /*signal_dx=*/true, &gate);
  }
  void unpermute_backward_p2p(const void* wg, void* dx, float* dwg, cudaStream_t s) {
    const int T = cur_T_, d = cfg_.d_model, k = cfg_.top_k;
    const bool gate_grad = k > 1;
    if (!(unpermuted_ && dx == bound_dx_ && wg == bound_wg_)) {  // not done beside the FFN1 wgrad
      timer_.begin(FM_PHASE_UNPERMUTE, s);
      const P2P p = p2p_args(-1, /*wait for "dX ready"*/ 3);
      launch_unpermute_bwd(dx_perm_.p, pos_.as<int32_t>(), topk_idx_.as<int32_t>(), dl_.as<float>(), wg, T, d,
                           k, gate_grad, dx, s, &p);
      timer_.end(s);
    }
    unpermuted_ = false;
    bound_dx_ = nullptr;
    bound_wg_ = nullptr;
    if (dwg && gate_grad && drops_enabled()) {  // dropped units are in no X_perm: add them here
      timer_.begin(FM_PHASE_GATE_WGRAD, s);
      launch_dropped_gate_wgrad(saved_x_, pos_.as<int32_t>(), topk_idx_.as<int32_t>(), dl_.as<float>(), T, d, k,
                                cfg_.num_experts, drop_partial(T), dwg, s);
      timer_.end(s);
    }
  }
  bool p2p() const { return p2p_; }

  // phase wrappers (G >= 1)
  void ph_expert_forward(const void* recv_buf, const void* w1, const float* b1, const void* w2,
                         const float* b2, void* ret_buf, cudaStream_t s) {
    recv_to_perm(recv_buf, x_perm_.p, s);
    expert_forward(w1, b1, w2, b2, s);
    perm_to_recv(y_perm_.p, ret_buf, s);
  }
  void ph_expert_backward(const void* drecv, const void* w1, const void* w2, float* dw1,
                          float* db1, float* dw2, float* db2, void* dret, cudaStream_t s) {
    recv_to_perm(drecv, dy_perm_.p, s);
    expert_backward(w1, w2, dw1, db1, dw2, db2, s);
    perm_to_recv(dx_perm_.p, dret, s);
  }
  void ph_unpermute_backward(const void* dback, const void* send_buf, const void* wg, void* dx,
                             float* dwg, cudaStream_t s) {
    unpermute_backward(dback, send_buf, nullptr, send_total_, wg, dx, dwg, s);
  }

  // ------------------------------------------------------------ introspection
  int nl() const { return static_cast<int>(local_.size()); }
  const std::vector<int32_t>& local() const { return local_; }
  int side_jobs() const { return side_jobs_; }
  void set_side_enabled(bool on) { side_enabled_ = on; }
  // The bound un-permute waits inside a persistent GEMM launch for the peers'
  // "dX ready": only safe when every peer runs on another device (ranks
  // sharing one GPU — in-process loopback, several processes on one device —
  // could wait on a signal queued behind that launch). Otherwise the binding
  // is ignored and fm_layer_unpermute_backward_p2p runs the standalone kernel.
  bool peers_on_other_devices() const {
    int me = -1;
    if (cudaGetDevice(&me) != cudaSuccess) return false;
    for (int g = 0; g < cfg_.num_gpus; ++g) {
      if (g == cfg_.rank) continue;
      cudaPointerAttributes a{};
      if (!pp_.base[g] || cudaPointerGetAttributes(&a, pp_.base[g]) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      if (a.device == me) return false;
    }
    return true;
  }
  void bind_dx(const void* wg, void* dx) {
    if (!p2p_) throw std::logic_error("fm_layer_p2p_bind_dx: P2P transport not enabled");
#ifndef FM_P2P_UNPERMUTE_SIDE
#define FM_P2P_UNPERMUTE_SIDE 1
#endif
    if (peers_distinct_ < 0) peers_distinct_ = (FM_P2P_UNPERMUTE_SIDE && peers_on_other_devices()) ? 1 : 0;
    bound_wg_ = peers_distinct_ ? wg : nullptr;
    bound_dx_ = peers_distinct_ ? dx : nullptr;
  }
  const fm_layer_config& cfg() const { return cfg_; }

  // stream == nullptr: synchronise the device, then copy; else enqueue the copy
  // on `stream` (asynchronous when `host` is pinned)
  void copy_out(int field, void* host, size_t max_bytes, size_t* written, cudaStream_t stream = nullptr,
                bool async = false) {
    const int T = std::max(cur_T_, 0), k = cfg_.top_k, N = cfg_.num_experts, G = cfg_.num_gpus;
    const void* src = nullptr;
    size_t bytes = 0;
    switch (field) {
      case FM_FIELD_TOPK_IDX: src = topk_idx_.p; bytes = 4ull * T * k; break;
      case FM_FIELD_TOPK_W: src = topk_w_.p; bytes = 4ull * T * k; break;
      case FM_FIELD_UNIT_POS: src = pos_.p; bytes = 4ull * T * k; break;
      case FM_FIELD_GATE_GRAD: src = dl_.p; bytes = 4ull * T * k; break;
      case FM_FIELD_HIST: src = hist_.p; bytes = 8ull * N; break;
      case FM_FIELD_DEMAND: src = demand_.p; bytes = 8ull * N * G; break;
      case FM_FIELD_FLOWS: src = flows_.p; bytes = 8ull * N * G * G; break;
      case FM_FIELD_SEG_START: src = plan_.seg_start; bytes = 4ull * nl(); break;
      case FM_FIELD_SEG_REAL: src = plan_.seg_real; bytes = 4ull * nl(); break;
      case FM_FIELD_SEG_ROWS: src = plan_.seg_rows; bytes = 4ull * nl(); break;
      case FM_FIELD_TOTALS: src = plan_.totals; bytes = 16; break;
      case FM_FIELD_SEND_ROWS: src = plan_.send_rows; bytes = 4ull * G; break;
      case FM_FIELD_RECV_ROWS: src = plan_.recv_rows; bytes = 4ull * G; break;
      case FM_FIELD_X_PERM: src = x_perm_.p; bytes = x_perm_.bytes; break;
      case FM_FIELD_ACT: src = act_.p; bytes = act_.bytes; break;
      case FM_FIELD_Y_PERM: src = y_perm_.p; bytes = y_perm_.bytes; break;
      case FM_FIELD_DY_PERM: src = dy_perm_.p; bytes = dy_perm_.bytes; break;
      case FM_FIELD_DH: src = dh_.p; bytes = dh_.bytes; break;
      case FM_FIELD_DX_PERM: src = dx_perm_.p; bytes = dx_perm_.bytes; break;
      case FM_FIELD_ROUTE_STATUS: src = route_status_.p; bytes = 4; break;
      case FM_FIELD_KEPT: src = kept_.p; bytes = 8ull * N * G; break;
      case FM_FIELD_DROPPED: src = dropped_.p; bytes = 8; break;
      default: throw std::invalid_argument("fm_layer_copy_out: unknown field");
    }
    bytes = std::min(bytes, max_bytes);
    if (async) {
      if (bytes) FM_CUDA(cudaMemcpyAsync(host, src, bytes, cudaMemcpyDeviceToHost, stream));
    } else {
      FM_CUDA(cudaDeviceSynchronize());
      if (bytes) FM_CUDA(cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost));
    }
    if (written) *written = bytes;
  }

  size_t row_capacity() const { return row_cap_; }
  bool drops_enabled() const { return capacity_factor_ > 0 && std::isfinite(capacity_factor_); }
  // per-(expert, token chunk) partials of the dropped units' dWg share
  float* drop_partial(int T) {
    const size_t need = sizeof(float) * cfg_.num_experts * dropped_gate_chunks(T) * cfg_.d_model;
    if (drop_partial_.bytes < need) drop_partial_.reset(need);
    return drop_partial_.as<float>();
  }
  void set_capacity_factor(double cf) {
    if (!(cf >= 0)) throw std::invalid_argument("fm_layer: capacity_factor must be >= 0");
    capacity_factor_ = cf;
  }
  PhaseTimer& timer() { return timer_; }

 private:
  void check_tokens(int T) const {
    if (T < 0 || T > cfg_.max_tokens)
      throw std::invalid_argument("fm_layer: token count exceeds max_tokens");
  }

  void require_p2p() const {
    if (!p2p_) throw std::logic_error("fm_layer: P2P transport not enabled (fm_layer_enable_p2p)");
  }
  void require_linked() const {
    require_p2p();
    for (int g = 0; g < cfg_.num_gpus; ++g)
      if (!pp_.base[g]) throw std::logic_error("fm_layer: P2P peer " + std::to_string(g) + " is not mapped");
  }
  void check_peer(int peer) const {
    if (peer < 0 || peer >= cfg_.num_gpus || peer == cfg_.rank)
      throw std::out_of_range("fm_layer: P2P peer out of range");
  }
  void close_peer(int peer) {
    if (peer_ipc_[peer] && pp_.base[peer]) cudaIpcCloseMemHandle(pp_.base[peer]);
    peer_ipc_[peer] = false;
    pp_.base[peer] = nullptr;
  }
  void p2p_signal(int slot, cudaStream_t s) {
    launch_p2p_signal(pp_, cfg_.num_gpus, cfg_.rank, slot, epoch_, s);
  }

 public:
  ~Layer() {
    for (Staging& st : staging_) {
      if (st.done) cudaEventDestroy(st.done);
      if (st.host) cudaFreeHost(st.host);
    }
    if (p2p_)
      for (int g = 0; g < cfg_.num_gpus; ++g)
        if (peer_ipc_[g] && pp_.base[g]) cudaIpcCloseMemHandle(pp_.base[g]);
  }

 private:
  fm_layer_config cfg_;
  bool p2p_ = false;
  DevBuf arena_, unit_dst_, p2p_err_, p2p_done_, tile_src_mask_;
  P2P pp_{};
  std::vector<bool> peer_ipc_;
  unsigned long long epoch_ = 0;
  int32_t* peer_row_mem_ = nullptr;
  std::vector<int32_t> counts_, local_;
  DevBuf topk_idx_, topk_w_, tile_rank_, pos_, dl_, tile_counts_, tile_base_, hist_, demand_,
      flows_, route_status_, plan_mem_, ctl_mem_;
  int32_t* counts_dev_ = nullptr;
  int32_t* local_slot_dev_ = nullptr;
  std::vector<int32_t> operand_slot_;  // [N] or empty (packed layout)
  int operand_cap_ = 0;
  struct Staging {
    int32_t* host = nullptr;
    cudaEvent_t done = nullptr;
  };
  static constexpr int kStaging = 16;  // table uploads in flight before a reuse waits
  Staging staging_[kStaging];
  int staging_next_ = 0;
  DevBuf x_perm_, act_, y_perm_, dy_perm_, dh_, dx_perm_, dl_rows_, relu_mask_, tile_colsum_,
      row_expert_, tile_sum_, drop_partial_, gw_partial_;
  std::vector<int32_t> host_counts_;
  double capacity_factor_ = 0.0;  // 0 / inf: no drops (FlexMoE)
  const void* saved_x_ = nullptr;  // gate input of the current step (must outlive backward)
  int side_jobs_ = 0;              // fm_layer_side_jobs of the last backward
  bool scan_deferred_ = false;     // the expert scan runs inside the next plan launch
  const void* bound_wg_ = nullptr;  // fm_layer_p2p_bind_dx: where this step's un-permute
  void* bound_dx_ = nullptr;        //   reads the gate rows / writes dx
  bool unpermuted_ = false;         // the bound un-permute ran beside the FFN1 wgrad
  int peers_distinct_ = -1;         // every peer arena on another device (-1: unknown)
  bool side_enabled_ = FM_COLSUM_SIDE != 0;  // fm_layer_set_side_jobs
  DevBuf kept_, dropped_;
  int recv_total_ = 0, send_total_ = 0;
  bool fused_state_ = false;
  PlanDev plan_{};
  PhaseTimer timer_;
  int32_t* local_expert_dev_ = nullptr;
  size_t row_cap_ = 0;
  int cur_T_ = -1;
  const void *saved_wg_ = nullptr, *saved_w1_ = nullptr, *saved_w2_ = nullptr;
};

}  // namespace fm

struct fm_layer {
  std::unique_ptr<fm::Layer> impl;
};

extern "C" {

int fm_layer_create(const fm_layer_config* cfg, const int32_t* replica_counts_NG, fm_layer** out) {
  return fm::guarded([&] {
    if (!cfg || !replica_counts_NG || !out) throw std::invalid_argument("fm_layer_create: null argument");
    auto h = std::make_unique<fm_layer>();
    h->impl = std::make_unique<fm::Layer>(*cfg);
    h->impl->set_placement(replica_counts_NG);
    *out = h.release();
  });
}

int fm_layer_destroy(fm_layer* h) {
  return fm::guarded([&] { delete h; });
}

int fm_layer_set_placement(fm_layer* h, const int32_t* replica_counts_NG) {
  return fm::guarded([&] { h->impl->set_placement(replica_counts_NG); });
}

int fm_layer_set_placement_async(fm_layer* h, const int32_t* replica_counts_NG, const int32_t* hosted_N,
                                 void* stream) {
  return fm::guarded([&] {
    if (!h || !replica_counts_NG) throw std::invalid_argument("fm_layer_set_placement_async: null argument");
    h->impl->set_placement(replica_counts_NG, hosted_N, static_cast<cudaStream_t>(stream), /*sync=*/false);
  });
}

int fm_layer_set_operand_slots(fm_layer* h, const int32_t* slot_N, int capacity, void* stream) {
  return fm::guarded([&] {
    if (!h) throw std::invalid_argument("fm_layer_set_operand_slots: null layer");
    h->impl->set_operand_slots(slot_N, capacity, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_set_capacity_factor(fm_layer* h, double capacity_factor) {
  return fm::guarded([&] { h->impl->set_capacity_factor(capacity_factor); });
}

int fm_layer_p2p_bind_dx(fm_layer* h, const void* wg, void* dx) {
  return fm::guarded([&] { h->impl->bind_dx(wg, dx); });
}

int fm_layer_set_side_jobs(fm_layer* h, int enable) {
  return fm::guarded([&] { h->impl->set_side_enabled(enable != 0); });
}

int fm_layer_side_jobs(const fm_layer* h, int* mask) {
  return fm::guarded([&] { *mask = h->impl->side_jobs(); });
}

int fm_layer_local_experts(const fm_layer* h, int* num_local, int32_t* experts) {
  return fm::guarded([&] {
    const auto& l = h->impl->local();
    *num_local = static_cast<int>(l.size());
    if (experts) std::memcpy(experts, l.data(), sizeof(int32_t) * l.size());
  });
}

int fm_layer_forward(fm_layer* h, const void* x, int T, const void* wg, const void* w1,
                     const float* b1, const void* w2, const float* b2, void* y, void* stream) {
  return fm::guarded([&] {
    h->impl->forward(x, T, wg, w1, b1, w2, b2, y, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_backward(fm_layer* h, const void* dy, void* dx, float* dwg, float* dw1, float* db1,
                      float* dw2, float* db2, void* stream) {
  return fm::guarded([&] {
    h->impl->backward(dy, dx, dwg, dw1, db1, dw2, db2, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_gate(fm_layer* h, const void* x, int T, const void* wg, int64_t* hist_out,
                  void* stream) {
  return fm::guarded(
      [&] { h->impl->gate(x, T, wg, hist_out, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_route(fm_layer* h, const int64_t* gathered_hist_GN, int32_t* send_rows,
                   int32_t* recv_rows, void* stream) {
  return fm::guarded([&] {
    h->impl->route_gathered(gathered_hist_GN, send_rows, recv_rows, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_dispatch(fm_layer* h, const void* x, void* send_buf, void* stream) {
  return fm::guarded([&] { h->impl->dispatch_send(x, send_buf, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_expert_forward(fm_layer* h, const void* recv_buf, const void* w1, const float* b1,
                            const void* w2, const float* b2, void* ret_buf, void* stream) {
  return fm::guarded([&] {
    h->impl->ph_expert_forward(recv_buf, w1, b1, w2, b2, ret_buf, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_combine(fm_layer* h, const void* back_buf, void* y, void* stream) {
  return fm::guarded([&] { h->impl->combine(back_buf, y, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_combine_backward(fm_layer* h, const void* dy, const void* back_buf, void* dsend_buf,
                              void* stream) {
  return fm::guarded([&] {
    h->impl->combine_backward(dy, back_buf, dsend_buf, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_expert_backward(fm_layer* h, const void* drecv_buf, const void* w1, const void* w2,
                             float* dw1, float* db1, float* dw2, float* db2, void* dret_buf,
                             void* stream) {
  return fm::guarded([&] {
    h->impl->ph_expert_backward(drecv_buf, w1, w2, dw1, db1, dw2, db2, dret_buf,
                                static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_unpermute_backward(fm_layer* h, const void* dback_buf, const void* send_buf,
                                const void* wg, void* dx, float* dwg, void* stream) {
  return fm::guarded([&] {
    h->impl->ph_unpermute_backward(dback_buf, send_buf, wg, dx, dwg, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_enable_p2p(fm_layer* h) {
  return fm::guarded([&] { h->impl->enable_p2p(); });
}

int fm_layer_p2p_handle(fm_layer* h, void* handle64) {
  return fm::guarded([&] {
    if (!handle64) throw std::invalid_argument("fm_layer_p2p_handle: null handle");
    h->impl->p2p_handle(handle64);
  });
}

int fm_layer_p2p_open_peer(fm_layer* h, int peer, const void* handle64) {
  return fm::guarded([&] {
    if (!handle64) throw std::invalid_argument("fm_layer_p2p_open_peer: null handle");
    h->impl->p2p_open_peer(peer, handle64);
  });
}

int fm_layer_p2p_link_peer(fm_layer* h, int peer, fm_layer* other) {
  return fm::guarded([&] {
    if (!other) throw std::invalid_argument("fm_layer_p2p_link_peer: null peer layer");
    h->impl->p2p_link_peer(peer, *other->impl);
  });
}

int fm_layer_p2p_status(fm_layer* h, int* timed_out) {
  return fm::guarded([&] {
    if (!timed_out) throw std::invalid_argument("fm_layer_p2p_status: null output");
    *timed_out = h->impl->p2p_status();
  });
}

int fm_layer_route_p2p(fm_layer* h, const int64_t* gathered_hist_GN, void* stream) {
  return fm::guarded([&] { h->impl->route_p2p(gathered_hist_GN, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_dispatch_p2p(fm_layer* h, const void* x, void* stream) {
  return fm::guarded([&] { h->impl->dispatch_p2p(x, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_expert_forward_p2p(fm_layer* h, const void* w1, const float* b1, const void* w2, const float* b2,
                                void* stream) {
  return fm::guarded([&] { h->impl->expert_forward_p2p(w1, b1, w2, b2, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_combine_p2p(fm_layer* h, void* y, void* stream) {
  return fm::guarded([&] { h->impl->combine_p2p(y, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_combine_backward_p2p(fm_layer* h, const void* dy, void* stream) {
  return fm::guarded([&] { h->impl->combine_backward_p2p(dy, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_expert_backward_p2p(fm_layer* h, const void* w1, const void* w2, float* dw1, float* db1, float* dw2,
                                 float* db2, float* dwg, void* stream) {
  return fm::guarded([&] {
    h->impl->expert_backward_p2p(w1, w2, dw1, db1, dw2, db2, dwg, static_cast<cudaStream_t>(stream));
  });
}

int fm_layer_unpermute_backward_p2p(fm_layer* h, const void* wg, void* dx, float* dwg, void* stream) {
  return fm::guarded([&] { h->impl->unpermute_backward_p2p(wg, dx, dwg, static_cast<cudaStream_t>(stream)); });
}

int fm_layer_set_timing(fm_layer* h, int enable) {
  return fm::guarded([&] { h->impl->timer().enable(enable != 0); });
}

int fm_layer_read_timing(fm_layer* h, double* ms_by_phase, int* launches_by_phase) {
  return fm::guarded([&] { h->impl->timer().read(ms_by_phase, launches_by_phase); });
}

int fm_layer_copy_out(fm_layer* h, int field, void* host, size_t max_bytes, size_t* written) {
  return fm::guarded([&] { h->impl->copy_out(field, host, max_bytes, written); });
}

int fm_layer_copy_out_async(fm_layer* h, int field, void* host, size_t max_bytes, size_t* written,
                            void* stream) {
  return fm::guarded([&] {
    h->impl->copy_out(field, host, max_bytes, written, static_cast<cudaStream_t>(stream), true);
  });
}

}  // extern "C"
