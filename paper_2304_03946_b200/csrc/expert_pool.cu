// Expert state pool + peer-to-peer migration on a side stream.
//
// What the reference only models as TransferDescriptor{src, dst, bytes}
// (proj/include/moesim/placement.hpp:31-35; expand / migrate produce them,
// placement.cpp:143-232; the adjustment queue drains them, sim_engine.cpp:
// 124-262) is a real copy here: each hosted expert owns a slot of one
// cudaMalloc'd pool (f32 master + Adam m + v, 12 bytes per parameter), peers
// map each other's pools (CUDA IPC across processes, plain pointers in one
// process) and the receiving GPU pulls whole slots with cudaMemcpyAsync over
// NVLink on its side stream. The bf16 operands of the expert GEMMs are
// re-derived from the master on the same stream, so the compute stream only
// waits (fm_pool_wait_ready) right before the expert FFN: the copies overlap
// routing and the dispatch all-to-all (they are issued after the demand
// all-gather, see the ordering contract in include/flexmoe_b200.h).
//
// Kernels: `pack` (master -> bf16 weights / f32 biases, ascending local
// order) and a fused Adam that updates master/m/v in place and writes the
// packed operands in the same pass (read g + 3 states, write 3 states +
// operand: 30 bytes per parameter, HBM-bound).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fm_internal.h"

namespace fm {
namespace pool {

constexpr int kMaxLocal = 256;

struct SlotList {
  int n;
  int slot[kMaxLocal];
  int out[kMaxLocal];  // operand row written for entry i: i (packed) or slot[i] (by slot)
};

// The four tensor segments of one expert's parameter set, in slot order.
struct Segs {
  int64_t off[4];  // float offset inside a P-float set
  int64_t len[4];
  int64_t P;
};

inline Segs segs(int d, int f) {
  const int64_t fd = static_cast<int64_t>(f) * d;
  Segs s;
  s.off[0] = 0;           s.len[0] = fd;  // w1 [f, d]
  s.off[1] = fd;          s.len[1] = f;   // b1 [f]
  s.off[2] = fd + f;      s.len[2] = fd;  // w2 [d, f]
  s.off[3] = 2 * fd + f;  s.len[3] = d;   // b2 [d]
  s.P = 2 * fd + f + d;
  return s;
}

struct Packed {
  __nv_bfloat16* w1;
  float* b1;
  __nv_bfloat16* w2;
  float* b2;
};

__device__ __forceinline__ void store_operand(const Packed& out, int seg, int i, const Segs& sg, int64_t j4,
                                              float4 w) {
  // j4: float4 index inside the segment; bf16 weights, f32 biases
  if (seg == 0 || seg == 2) {
    __nv_bfloat16* dst = (seg == 0 ? out.w1 : out.w2) + static_cast<int64_t>(i) * sg.len[seg] + 4 * j4;
    __nv_bfloat162 lo = __floats2bfloat162_rn(w.x, w.y), hi = __floats2bfloat162_rn(w.z, w.w);
    uint2 v;
    v.x = *reinterpret_cast<uint32_t*>(&lo);
    v.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = v;
  } else {
    float* dst = (seg == 1 ? out.b1 : out.b2) + static_cast<int64_t>(i) * sg.len[seg];
    reinterpret_cast<float4*>(dst)[j4] = w;
  }
}

// grid (x: chunks, y: local expert i, z: segment)
__global__ void pack_kernel(const float* __restrict__ base, int64_t slot_floats, const SlotList sl, Segs sg,
                            Packed out) {
  const int i = blockIdx.y, seg = blockIdx.z;
  const float4* src = reinterpret_cast<const float4*>(base + sl.slot[i] * slot_floats + sg.off[seg]);
  const int64_t n4 = sg.len[seg] / 4;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n4;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x)
    store_operand(out, seg, sl.out[i], sg, j, __ldg(src + j));
}

struct Grads {
  const float* g[4];
};

struct AdamK {
  float lr, b1, b2, eps, inv_c1, inv_c2;
};

__global__ void adam_kernel(float* __restrict__ base, int64_t slot_floats, const SlotList sl, Segs sg,
                            Grads gr, AdamK a, Packed out) {
  const int i = blockIdx.y, seg = blockIdx.z;
  float* w = base + sl.slot[i] * slot_floats + sg.off[seg];
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* m4 = reinterpret_cast<float4*>(w + sg.P);
  float4* v4 = reinterpret_cast<float4*>(w + 2 * sg.P);
  const float4* g4 = reinterpret_cast<const float4*>(gr.g[seg] + static_cast<int64_t>(i) * sg.len[seg]);
  const int64_t n4 = sg.len[seg] / 4;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n4;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 g = __ldg(g4 + j);
    float4 m = m4[j], v = v4[j], p = w4[j];
    auto upd = [&](float gg, float& mm, float& vv, float& pp) {
      mm = a.b1 * mm + (1.0f - a.b1) * gg;
      vv = a.b2 * vv + (1.0f - a.b2) * gg * gg;
      pp -= a.lr * (mm * a.inv_c1) / (sqrtf(vv * a.inv_c2) + a.eps);
    };
    upd(g.x, m.x, v.x, p.x);
    upd(g.y, m.y, v.y, p.y);
    upd(g.z, m.z, v.z, p.z);
    upd(g.w, m.w, v.w, p.w);
    m4[j] = m;
    v4[j] = v;
    w4[j] = p;
    store_operand(out, seg, sl.out[i], sg, j, p);
  }
}

dim3 grid_for(const Segs& sg, int n) {
  const int64_t max4 = sg.len[0] / 4;
  const int want = static_cast<int>(std::min<int64_t>((max4 + 255) / 256, 1 << 16));
  const int cap = std::max(8, 8 * num_sms() / std::max(1, n));
  return dim3(std::max(1, std::min(want, cap)), n, 4);
}

// Keeps the caller's current device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    FM_CUDA(cudaGetDevice(&prev));
    if (prev != dev) FM_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace pool
}  // namespace fm

struct fm_expert_pool {
  int slots = 0, d = 0, f = 0, world = 0, device = 0;
  fm::pool::Segs sg{};
  int64_t slot_bytes = 0;
  char* base = nullptr;
  std::vector<char*> peer;       // peer pool bases (nullptr = unknown)
  std::vector<bool> peer_ipc;    // opened through IPC (closed on destroy)
  cudaStream_t side = nullptr;   // migration stream
  cudaEvent_t after_compute = nullptr, ready = nullptr;
  bool ready_pending = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timing;  // per migrate call
  double copy_ms = 0.0;
  int64_t bytes = 0, copies = 0;
  bool by_slot = false;  // operand row of a slot = the slot (else: position in the list)
};

namespace {

using namespace fm::pool;

void check_local(const fm_expert_pool* p, const int32_t* local_slots, int n, SlotList& sl) {
  if (n < 0 || n > kMaxLocal) throw std::invalid_argument("fm_pool: 0 <= num_local <= 256");
  if (n > 0 && !local_slots) throw std::invalid_argument("fm_pool: local_slots is null");
  sl.n = n;
  for (int i = 0; i < n; ++i) {
    if (local_slots[i] < 0 || local_slots[i] >= p->slots)
      throw std::out_of_range("fm_pool: slot " + std::to_string(local_slots[i]) + " out of range");
    sl.slot[i] = local_slots[i];
    sl.out[i] = p->by_slot ? local_slots[i] : i;
  }
}

void launch_pack(fm_expert_pool* p, const SlotList& sl, void* w1, float* b1, void* w2, float* b2,
                 cudaStream_t s) {
  if (sl.n == 0) return;
  if (!w1 || !b1 || !w2 || !b2) throw std::invalid_argument("fm_pool_pack: null operand");
  Packed out{static_cast<__nv_bfloat16*>(w1), b1, static_cast<__nv_bfloat16*>(w2), b2};
  pack_kernel<<<grid_for(p->sg, sl.n), 256, 0, s>>>(reinterpret_cast<const float*>(p->base),
                                                     p->slot_bytes / 4, sl, p->sg, out);
  FM_LAUNCH_CHECK("pack_kernel");
}

}  // namespace

extern "C" {

int fm_pool_create(int slots, int d_model, int d_ff, int world, fm_expert_pool** out) {
  return fm::guarded([&] {
    if (!out) throw std::invalid_argument("fm_pool_create: out is null");
    if (slots < 1 || d_model < 4 || d_ff < 4 || d_model % 4 || d_ff % 4 || world < 1)
      throw std::invalid_argument("fm_pool_create: slots >= 1, world >= 1, d_model and d_ff multiples of 4");
    auto* p = new fm_expert_pool();
    try {
      p->slots = slots;
      p->d = d_model;
      p->f = d_ff;
      p->world = world;
      p->sg = segs(d_model, d_ff);
      p->slot_bytes = (p->sg.P * 12 + 255) / 256 * 256;
      FM_CUDA(cudaGetDevice(&p->device));
      FM_CUDA(cudaMalloc(&p->base, static_cast<size_t>(p->slot_bytes) * slots));
      FM_CUDA(cudaMemset(p->base, 0, static_cast<size_t>(p->slot_bytes) * slots));
      FM_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
      FM_CUDA(cudaEventCreateWithFlags(&p->after_compute, cudaEventDisableTiming));
      FM_CUDA(cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming));
      p->peer.assign(world, nullptr);
      p->peer_ipc.assign(world, false);
    } catch (...) {
      if (p->base) cudaFree(p->base);
      delete p;
      throw;
    }
    *out = p;
  });
}

int fm_pool_destroy(fm_expert_pool* p) {
  return fm::guarded([&] {
    if (!p) return;
    DeviceGuard g(p->device);
    cudaStreamSynchronize(p->side);
    for (auto& e : p->timing) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    for (int r = 0; r < p->world; ++r)
      if (p->peer_ipc[r]) cudaIpcCloseMemHandle(p->peer[r]);
    cudaEventDestroy(p->after_compute);
    cudaEventDestroy(p->ready);
    cudaStreamDestroy(p->side);
    cudaFree(p->base);
    delete p;
  });
}

int fm_pool_info(const fm_expert_pool* p, int64_t* params_per_expert, int64_t* slot_bytes) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_info: null pool");
    if (params_per_expert) *params_per_expert = p->sg.P;
    if (slot_bytes) *slot_bytes = p->slot_bytes;
  });
}

int fm_pool_slot_ptr(fm_expert_pool* p, int slot, void** dev_ptr) {
  return fm::guarded([&] {
    if (!p || !dev_ptr) throw std::invalid_argument("fm_pool_slot_ptr: null argument");
    if (slot < 0 || slot >= p->slots) throw std::out_of_range("fm_pool_slot_ptr: slot out of range");
    *dev_ptr = p->base + static_cast<int64_t>(slot) * p->slot_bytes;
  });
}

int fm_pool_ipc_handle(fm_expert_pool* p, void* handle64) {
  return fm::guarded([&] {
    if (!p || !handle64) throw std::invalid_argument("fm_pool_ipc_handle: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    DeviceGuard g(p->device);
    cudaIpcMemHandle_t h;
    FM_CUDA(cudaIpcGetMemHandle(&h, p->base));
    memcpy(handle64, &h, sizeof(h));
  });
}

int fm_pool_open_peer(fm_expert_pool* p, int peer, const void* handle64) {
  return fm::guarded([&] {
    if (!p || !handle64) throw std::invalid_argument("fm_pool_open_peer: null argument");
    if (peer < 0 || peer >= p->world) throw std::out_of_range("fm_pool_open_peer: peer out of range");
    DeviceGuard g(p->device);
    if (p->peer_ipc[peer]) {
      FM_CUDA(cudaIpcCloseMemHandle(p->peer[peer]));
      p->peer_ipc[peer] = false;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    void* ptr = nullptr;
    FM_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p->peer[peer] = static_cast<char*>(ptr);
    p->peer_ipc[peer] = true;
  });
}

int fm_pool_link_peer(fm_expert_pool* p, int peer, fm_expert_pool* other) {
  return fm::guarded([&] {
    if (!p || !other) throw std::invalid_argument("fm_pool_link_peer: null pool");
    if (peer < 0 || peer >= p->world) throw std::out_of_range("fm_pool_link_peer: peer out of range");
    if (other->slot_bytes != p->slot_bytes)
      throw std::invalid_argument("fm_pool_link_peer: pools of different expert shapes");
    p->peer[peer] = other->base;
  });
}

int fm_pool_migrate(fm_expert_pool* p, const int32_t* moves, int n, const int32_t* local_slots, int num_local,
                    void* w1, float* b1, void* w2, float* b2, void* stream) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_migrate: null pool");
    if (n < 0 || (n > 0 && !moves)) throw std::invalid_argument("fm_pool_migrate: bad move list");
    SlotList sl;
    check_local(p, local_slots, num_local, sl);
    for (int i = 0; i < n; ++i) {
      const int dst = moves[3 * i], peer = moves[3 * i + 1], src = moves[3 * i + 2];
      if (dst < 0 || dst >= p->slots || src < 0 || src >= p->slots)
        throw std::out_of_range("fm_pool_migrate: slot out of range");
      if (peer < 0 || peer >= p->world || !p->peer[peer])
        throw std::logic_error("fm_pool_migrate: peer " + std::to_string(peer) + " is not linked");
    }
    DeviceGuard g(p->device);
    const auto s = static_cast<cudaStream_t>(stream);
    // everything enqueued so far on the compute stream (the previous step's
    // reads of the packed operands and of vacated slots) precedes the copies
    FM_CUDA(cudaEventRecord(p->after_compute, s));
    FM_CUDA(cudaStreamWaitEvent(p->side, p->after_compute, 0));
    if (n > 0) {
      cudaEvent_t t0, t1;
      FM_CUDA(cudaEventCreate(&t0));
      FM_CUDA(cudaEventCreate(&t1));
      FM_CUDA(cudaEventRecord(t0, p->side));
      for (int i = 0; i < n; ++i) {
        const int dst = moves[3 * i], peer = moves[3 * i + 1], src = moves[3 * i + 2];
        FM_CUDA(cudaMemcpyAsync(p->base + static_cast<int64_t>(dst) * p->slot_bytes,
                                p->peer[peer] + static_cast<int64_t>(src) * p->slot_bytes,
                                static_cast<size_t>(p->sg.P) * 12, cudaMemcpyDefault, p->side));
      }
      FM_CUDA(cudaEventRecord(t1, p->side));
      p->timing.emplace_back(t0, t1);
      p->bytes += static_cast<int64_t>(n) * p->sg.P * 12;
      p->copies += n;
    }
    launch_pack(p, sl, w1, b1, w2, b2, p->side);
    FM_CUDA(cudaEventRecord(p->ready, p->side));
    p->ready_pending = true;
  });
}

int fm_pool_set_operand_layout(fm_expert_pool* p, int by_slot) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_set_operand_layout: null pool");
    p->by_slot = by_slot != 0;
  });
}

int fm_pool_wait_ready(fm_expert_pool* p, void* stream) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_wait_ready: null pool");
    if (!p->ready_pending) return;
    DeviceGuard g(p->device);
    FM_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), p->ready, 0));
    p->ready_pending = false;
  });
}

int fm_pool_pack(fm_expert_pool* p, const int32_t* local_slots, int num_local, void* w1, float* b1, void* w2,
                 float* b2, void* stream) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_pack: null pool");
    SlotList sl;
    check_local(p, local_slots, num_local, sl);
    DeviceGuard g(p->device);
    launch_pack(p, sl, w1, b1, w2, b2, static_cast<cudaStream_t>(stream));
  });
}

int fm_pool_adam(fm_expert_pool* p, const int32_t* local_slots, int num_local, const float* dw1,
                 const float* db1, const float* dw2, const float* db2, const fm_adam_config* cfg, void* w1,
                 float* b1, void* w2, float* b2, void* stream) {
  return fm::guarded([&] {
    if (!p || !cfg) throw std::invalid_argument("fm_pool_adam: null argument");
    if (cfg->step < 1) throw std::invalid_argument("fm_pool_adam: step must be >= 1");
    SlotList sl;
    check_local(p, local_slots, num_local, sl);
    if (sl.n == 0) return;
    if (!dw1 || !db1 || !dw2 || !db2 || !w1 || !b1 || !w2 || !b2)
      throw std::invalid_argument("fm_pool_adam: null gradient or operand");
    DeviceGuard g(p->device);
    AdamK a;
    a.lr = cfg->lr;
    a.b1 = cfg->beta1;
    a.b2 = cfg->beta2;
    a.eps = cfg->eps;
    a.inv_c1 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(cfg->beta1), cfg->step)));
    a.inv_c2 = static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(cfg->beta2), cfg->step)));
    Grads gr{{dw1, db1, dw2, db2}};
    Packed out{static_cast<__nv_bfloat16*>(w1), b1, static_cast<__nv_bfloat16*>(w2), b2};
    adam_kernel<<<grid_for(p->sg, sl.n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<float*>(p->base), p->slot_bytes / 4, sl, p->sg, gr, a, out);
    FM_LAUNCH_CHECK("adam_kernel");
  });
}

int fm_pool_migration_stats(fm_expert_pool* p, double* copy_ms, int64_t* bytes, int64_t* copies) {
  return fm::guarded([&] {
    if (!p) throw std::invalid_argument("fm_pool_migration_stats: null pool");
    DeviceGuard g(p->device);
    for (auto& e : p->timing) {
      FM_CUDA(cudaEventSynchronize(e.second));
      float ms = 0.0f;
      FM_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
      p->copy_ms += ms;
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    p->timing.clear();
    if (copy_ms) *copy_ms = p->copy_ms;
    if (bytes) *bytes = p->bytes;
    if (copies) *copies = p->copies;
  });
}

}  // extern "C"
