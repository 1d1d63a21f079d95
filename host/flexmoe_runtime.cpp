// flexmoe_runtime — the FlexMoE training-step runtime in C++ (no Python, no
// torch): the device MoE layer, the host placement scheduler, the expert-state
// pool with peer-to-peer migration, Adam, and the token / gradient exchanges,
// all through the C ABI of libflexmoe_b200.so (include/flexmoe_b200.h).
//
// It is the C++ counterpart of paper_2304_03946_b200/runtime.py (the same
// step, the same decisions, bit-identical results: tests/test_cpp_runtime_gpu.py)
// and the B200 form of the reference's step driver SimEngine::run_step
// (proj/src/sim_engine.cpp:329-449), where the simulator's modelled phases are
// real device work:
//   begin_step           fm_scheduler_begin_step: the placement boundary
//                        (flip "modelled": the reference's budgeted drain,
//                        sim_engine.cpp:331-336; flip "copy": ops issued at the
//                        previous boundary become effective, the next prefix
//                        is issued). The layer switches placement with one
//                        async table upload; the operands stay in pool slots.
//   gate + histogram     fm_layer_gate
//   demand all-gather    Exchange::all_gather (TokenDemand D[e][g] everywhere)
//   state pulls          fm_pool_migrate on the pool's side stream (after the
//                        all-gather: the sources' previous Adam step is done)
//   route / exchange     P2P: fm_layer_route_p2p, dispatch/combine into peers'
//                        buffers; NCCL: fm_layer_route + grouped send/recv
//                        all-to-alls (a2a_cost, cost_model.cpp:37-51)
//   expert FFN, combine, backward mirrors
//   replica-group sums   per expert with >= 2 state holders, ascending id,
//                        communicators LRU-cached (sim_engine.cpp:45-113)
//   Adam                 fm_pool_adam on every hosted expert (replicas stay
//                        bit-identical)
//   finish_step          fm_scheduler_finish_step on the step's demand (policy
//                        inline or on the scheduler's worker thread)
//
// Two exchanges: NCCL, one forked process per GPU (--gpus N); and an
// in-process loopback of G ranks as threads sharing one GPU and one stream
// (--loopback G), which runs the real multi-GPU kernels, layouts and
// decisions on a single device (the tests).
//
//   flexmoe_runtime (--gpus N | --loopback G) [--steps K] [--warmup W]
//     [--experts E] [--topk k] [--d-model d] [--d-ff f] [--tokens T]
//     [--slots S] [--transport p2p|nccl] [--flip copy|modelled] [--async-policy 0|1]
//     [--adam 0|1] [--lr LR] [--zipf Z] [--profile reference|b200] [--tps TPS]
//     [--inputs DIR] [--dump DIR] [--log-steps 0|1]
// prints per-step decision lines (--log-steps 1) and one JSON summary line (rank 0).
#include <cuda_runtime.h>
#include <nccl.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "flexmoe_b200.h"

namespace {

void ck(int status, const char* what) {
  if (status != FM_OK) throw std::runtime_error(std::string(what) + ": " + fm_last_error());
}
void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void nc(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}

struct Args {
  int gpus = 0, loopback = 0, steps = 20, warmup = 3;
  int experts = 64, topk = 1, d = 1024, f = 4096, tokens = 65536, slots = 0;
  std::string transport = "p2p", flip = "copy", profile = "b200", inputs, dump;
  int async_policy = 1, adam = 1, log_steps = 0;
  double lr = 1e-4, zipf = 1.25, tps = 2.0e7;
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    auto I = [&] { return std::atoi(v.c_str()); };
    if (k == "--gpus") a.gpus = I();
    else if (k == "--loopback") a.loopback = I();
    else if (k == "--steps") a.steps = I();
    else if (k == "--warmup") a.warmup = I();
    else if (k == "--experts") a.experts = I();
    else if (k == "--topk") a.topk = I();
    else if (k == "--d-model") a.d = I();
    else if (k == "--d-ff") a.f = I();
    else if (k == "--tokens") a.tokens = I();
    else if (k == "--slots") a.slots = I();
    else if (k == "--transport") a.transport = v;
    else if (k == "--flip") a.flip = v;
    else if (k == "--async-policy") a.async_policy = I();
    else if (k == "--adam") a.adam = I();
    else if (k == "--lr") a.lr = std::atof(v.c_str());
    else if (k == "--zipf") a.zipf = std::atof(v.c_str());
    else if (k == "--profile") a.profile = v;
    else if (k == "--tps") a.tps = std::atof(v.c_str());
    else if (k == "--inputs") a.inputs = v;
    else if (k == "--dump") a.dump = v;
    else if (k == "--log-steps") a.log_steps = I();
    else throw std::invalid_argument("unknown option " + k);
  }
  if ((a.gpus > 0) == (a.loopback > 0)) throw std::invalid_argument("give exactly one of --gpus N / --loopback G");
  if (a.transport != "p2p" && a.transport != "nccl") throw std::invalid_argument("--transport p2p|nccl");
  if (a.flip != "copy" && a.flip != "modelled") throw std::invalid_argument("--flip copy|modelled");
  if (a.profile != "b200" && a.profile != "reference") throw std::invalid_argument("--profile b200|reference");
  return a;
}

uint16_t bf16(float v) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &v, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}

template <class T>
T* dev_alloc(size_t n) {
  T* p = nullptr;
  cu(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)), "cudaMalloc");
  return p;
}

std::vector<char> read_file(const std::string& path, size_t bytes) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<char> b(bytes);
  in.read(b.data(), static_cast<std::streamsize>(bytes));
  if (static_cast<size_t>(in.gcount()) != bytes) throw std::runtime_error(path + ": short read");
  return b;
}

void write_file(const std::string& path, const void* p, size_t bytes) {
  std::ofstream out(path, std::ios::binary);
  out.write(static_cast<const char*>(p), static_cast<std::streamsize>(bytes));
  if (!out) throw std::runtime_error("cannot write " + path);
}

// ------------------------------------------------------------------ exchanges
// The collectives the step needs. Every rank calls every
// collective in the same order; all_reduce is called by the whole world for
// each group (members pass their buffers, others none).
struct Exchange {
  int rank = 0, world = 1;
  virtual ~Exchange() = default;
  virtual cudaStream_t stream() = 0;
  virtual void all_gather_i64(const int64_t* in, int64_t* out, size_t n) = 0;  // out [world][n]
  virtual void all_reduce(const std::vector<std::pair<float*, size_t>>& bufs, const std::vector<int>& group) = 0;
  virtual void all_to_all(const void* send, const std::vector<int>& send_rows, void* recv,
                          const std::vector<int>& recv_rows, size_t row_bytes) = 0;
  virtual void share(fm_layer* layer, fm_expert_pool* pool, bool p2p) = 0;
  virtual void fence() {}
  virtual double max_over_ranks(double v) = 0;
};

// LRU of replica-group communicators (sim_engine.cpp:45-65, capacity 64).
template <class C>
class GroupCache {
 public:
  explicit GroupCache(size_t cap) : cap_(cap) {}
  // returns the cached value or nullptr (then insert() it)
  C* find(const std::vector<int>& g) {
    auto it = where_.find(g);
    if (it == where_.end()) return nullptr;
    order_.splice(order_.begin(), order_, it->second);
    return &it->second->second;
  }
  // inserts; returns the evicted entry (if any)
  std::vector<C> insert(const std::vector<int>& g, C c) {
    order_.emplace_front(g, c);
    where_[g] = order_.begin();
    std::vector<C> out;
    while (where_.size() > cap_) {
      out.push_back(order_.back().second);
      where_.erase(order_.back().first);
      order_.pop_back();
    }
    ++misses_;
    return out;
  }
  int misses() const { return misses_; }

 private:
  size_t cap_;
  int misses_ = 0;
  std::list<std::pair<std::vector<int>, C>> order_;
  std::map<std::vector<int>, typename std::list<std::pair<std::vector<int>, C>>::iterator> where_;
};

class NcclExchange : public Exchange {
 public:
  NcclExchange(int r, int w, const ncclUniqueId& id) : groups_(64) {
    rank = r;
    world = w;
    nc(ncclCommInitRank(&comm_, w, id, r), "ncclCommInitRank");
    cu(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
    scratch_ = dev_alloc<double>(1);
  }
  ~NcclExchange() override {
    for (ncclComm_t c : live_) ncclCommDestroy(c);
    ncclCommDestroy(comm_);
    cudaFree(scratch_);
  }
  cudaStream_t stream() override { return s_; }
  void all_gather_i64(const int64_t* in, int64_t* out, size_t n) override {
    nc(ncclAllGather(in, out, n, ncclInt64, comm_, s_), "ncclAllGather");
  }
  void all_reduce(const std::vector<std::pair<float*, size_t>>& bufs, const std::vector<int>& group) override {
    ncclComm_t c = comm_;
    if (!group.empty()) {
      ncclComm_t* hit = groups_.find(group);
      const bool member = std::find(group.begin(), group.end(), rank) != group.end();
      if (!hit) {  // ncclCommSplit is collective over the world: every rank is here, in the same order
        ncclComm_t nw = nullptr;
        nc(ncclCommSplit(comm_, member ? 0 : NCCL_SPLIT_NOCOLOR, rank, &nw, nullptr), "ncclCommSplit");
        for (ncclComm_t old : groups_.insert(group, nw))
          if (old) {
            ncclCommDestroy(old);
            live_.erase(std::find(live_.begin(), live_.end(), old));
          }
        if (nw) live_.push_back(nw);
        hit = groups_.find(group);
      }
      if (!member) return;
      c = *hit;
    }
    nc(ncclGroupStart(), "ncclGroupStart");
    for (const auto& [p, n] : bufs) nc(ncclAllReduce(p, p, n, ncclFloat, ncclSum, c, s_), "ncclAllReduce");
    nc(ncclGroupEnd(), "ncclGroupEnd");
  }
  void all_to_all(const void* send, const std::vector<int>& send_rows, void* recv, const std::vector<int>& recv_rows,
                  size_t row_bytes) override {
    size_t so = 0, ro = 0;
    nc(ncclGroupStart(), "ncclGroupStart");
    for (int p = 0; p < world; ++p) {
      if (send_rows[p])
        nc(ncclSend(static_cast<const char*>(send) + so * row_bytes, send_rows[p] * row_bytes, ncclChar, p, comm_, s_),
           "ncclSend");
      if (recv_rows[p])
        nc(ncclRecv(static_cast<char*>(recv) + ro * row_bytes, recv_rows[p] * row_bytes, ncclChar, p, comm_, s_),
           "ncclRecv");
      so += send_rows[p];
      ro += recv_rows[p];
    }
    nc(ncclGroupEnd(), "ncclGroupEnd");
  }
  void share(fm_layer* layer, fm_expert_pool* pool, bool p2p) override {
    char* hd = dev_alloc<char>(128 * world);
    char h[128] = {};
    if (p2p) ck(fm_layer_p2p_handle(layer, h), "fm_layer_p2p_handle");
    ck(fm_pool_ipc_handle(pool, h + 64), "fm_pool_ipc_handle");
    cu(cudaMemcpy(hd + 128 * rank, h, 128, cudaMemcpyHostToDevice), "H2D");
    nc(ncclAllGather(hd + 128 * rank, hd, 128, ncclChar, comm_, s_), "ncclAllGather handles");
    std::vector<char> all(128 * world);
    cu(cudaMemcpyAsync(all.data(), hd, all.size(), cudaMemcpyDeviceToHost, s_), "D2H");
    cu(cudaStreamSynchronize(s_), "sync");
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      if (p2p) ck(fm_layer_p2p_open_peer(layer, p, all.data() + 128 * p), "fm_layer_p2p_open_peer");
      ck(fm_pool_open_peer(pool, p, all.data() + 128 * p + 64), "fm_pool_open_peer");
    }
    cudaFree(hd);
  }
  double max_over_ranks(double v) override {
    cu(cudaMemcpyAsync(scratch_, &v, 8, cudaMemcpyHostToDevice, s_), "H2D");
    nc(ncclAllReduce(scratch_, scratch_, 1, ncclDouble, ncclMax, comm_, s_), "ncclAllReduce max");
    cu(cudaMemcpyAsync(&v, scratch_, 8, cudaMemcpyDeviceToHost, s_), "D2H");
    cu(cudaStreamSynchronize(s_), "sync");
    return v;
  }

 private:
  ncclComm_t comm_ = nullptr;
  cudaStream_t s_ = nullptr;
  double* scratch_ = nullptr;
  GroupCache<ncclComm_t> groups_;
  std::vector<ncclComm_t> live_;
};

// G ranks as threads on one GPU, one shared stream (so a kernel that waits
// for a peer's flag is always enqueued after the kernel that sets it: fence()
// keeps the ranks' phases in lock step, as distributed.LoopbackExchange).
struct LoopbackHub {
  explicit LoopbackHub(int w) : world(w), slots(w) {
    cu(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen || broken; }))
      broken = true;
    if (broken) {
      cv.notify_all();
      throw std::runtime_error("loopback barrier broken (a rank failed or stalled)");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
  int world;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool broken = false;
  std::vector<std::vector<const void*>> slots;
  std::vector<std::vector<int>> ints;
  GroupCache<int> groups{64};
};

class LoopbackExchange : public Exchange {
 public:
  LoopbackExchange(LoopbackHub& hub, int r) : hub_(hub) {
    rank = r;
    world = hub.world;
  }
  cudaStream_t stream() override { return hub_.stream; }
  std::vector<std::vector<const void*>> swap(std::vector<const void*> mine) {
    hub_.barrier();
    hub_.slots[rank] = std::move(mine);
    hub_.barrier();
    auto all = hub_.slots;
    hub_.barrier();
    return all;
  }
  void all_gather_i64(const int64_t* in, int64_t* out, size_t n) override {
    auto all = swap({in});
    for (int g = 0; g < world; ++g)
      cu(cudaMemcpyAsync(out + g * n, all[g][0], n * 8, cudaMemcpyDeviceToDevice, hub_.stream), "D2D");
    hub_.barrier();  // every rank's copies are enqueued before anyone's next write to its input
  }
  // SUM over the group in ascending member order from zero in fp32 — the
  // same arithmetic as distributed.LoopbackExchange (acc = 0; acc += t_g).
  void all_reduce(const std::vector<std::pair<float*, size_t>>& bufs, const std::vector<int>& group) override {
    std::vector<int> members = group;
    if (members.empty())
      for (int g = 0; g < world; ++g) members.push_back(g);
    if (!group.empty() && rank == 0 && !hub_.groups.find(group)) hub_.groups.insert(group, 0);
    const bool member = std::find(members.begin(), members.end(), rank) != members.end();
    std::vector<const void*> mine;
    for (const auto& b : bufs) mine.push_back(member ? b.first : nullptr);
    auto all = swap(mine);
    if (rank == members.front()) {
      cu(cudaStreamSynchronize(hub_.stream), "sync");
      for (size_t i = 0; i < bufs.size(); ++i) {
        const size_t n = bufs[i].second;
        std::vector<float> acc(n, 0.0f), t(n);
        for (int g : members) {
          cu(cudaMemcpy(t.data(), all[g][i], n * 4, cudaMemcpyDeviceToHost), "D2H");
          for (size_t j = 0; j < n; ++j) acc[j] += t[j];
        }
        for (int g : members)
          cu(cudaMemcpy(const_cast<void*>(all[g][i]), acc.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
      }
    }
    hub_.barrier();
  }
  void all_to_all(const void* send, const std::vector<int>& send_rows, void* recv, const std::vector<int>& recv_rows,
                  size_t row_bytes) override {
    hub_.barrier();
    hub_.slots[rank] = {send};
    {
      std::lock_guard<std::mutex> lk(hub_.mu);
      if (hub_.ints.size() != static_cast<size_t>(world)) hub_.ints.resize(world);
      hub_.ints[rank] = send_rows;
    }
    hub_.barrier();
    size_t ro = 0;
    for (int src = 0; src < world; ++src) {
      size_t so = 0;
      for (int p = 0; p < rank; ++p) so += hub_.ints[src][p];
      const size_t n = static_cast<size_t>(hub_.ints[src][rank]);
      if (n != static_cast<size_t>(recv_rows[src])) throw std::logic_error("loopback all_to_all: row counts disagree");
      if (n)
        cu(cudaMemcpyAsync(static_cast<char*>(recv) + ro * row_bytes,
                           static_cast<const char*>(hub_.slots[src][0]) + so * row_bytes, n * row_bytes,
                           cudaMemcpyDeviceToDevice, hub_.stream),
           "D2D");
      ro += n;
    }
    hub_.barrier();
  }
  void share(fm_layer* layer, fm_expert_pool* pool, bool p2p) override {
    auto all = swap({layer, pool});
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      if (p2p) ck(fm_layer_p2p_link_peer(layer, p, static_cast<fm_layer*>(const_cast<void*>(all[p][0]))), "link");
      ck(fm_pool_link_peer(pool, p, static_cast<fm_expert_pool*>(const_cast<void*>(all[p][1]))), "pool link");
    }
  }
  void fence() override { hub_.barrier(); }
  double max_over_ranks(double v) override {
    hub_.barrier();
    {
      std::lock_guard<std::mutex> lk(hub_.mu);
      maxv_[rank] = v;
    }
    hub_.barrier();
    double m = v;
    for (int g = 0; g < world; ++g) m = std::max(m, maxv_[g]);
    hub_.barrier();
    return m;
  }
  static inline std::vector<double> maxv_ = std::vector<double>(64, 0.0);

 private:
  LoopbackHub& hub_;
};

// ------------------------------------------------------------------ slot directory
// Replicated slot bookkeeping of every GPU's pool (pool.py SlotAllocator /
// apply_placement_change): every rank applies the same changes in the same
// order, so a receiver knows the source's slot without asking.
struct SlotAllocator {
  explicit SlotAllocator(int cap) : capacity(cap) {
    for (int s = 0; s < cap; ++s) free.push_back(s);
  }
  void begin_step() {
    free.insert(free.end(), vacated.begin(), vacated.end());
    std::sort(free.begin(), free.end());
    vacated.clear();
  }
  int host(int e) {
    auto it = slot_of.find(e);
    if (it != slot_of.end()) return it->second;
    if (free.empty()) throw std::logic_error("expert pool: no free slot for expert " + std::to_string(e));
    const int s = free.front();
    free.erase(free.begin());
    slot_of[e] = s;
    return s;
  }
  void vacate(int e) {
    auto it = slot_of.find(e);
    if (it == slot_of.end()) return;
    vacated.push_back(it->second);
    slot_of.erase(it);
  }
  int capacity;
  std::map<int, int> slot_of;
  std::vector<int> free, vacated;
};

struct Pull {
  int e, src, src_slot, dst, dst_slot;
};

// old/new: [N][G] state holders. Receivers pull from the lowest-id old holder.
std::vector<Pull> apply_placement_change(std::vector<SlotAllocator>& dir, const std::vector<uint8_t>& old_h,
                                         const std::vector<uint8_t>& new_h, int N, int G) {
  for (auto& a : dir) a.begin_step();
  std::vector<Pull> moves;
  for (int e = 0; e < N; ++e) {
    int holder = -1;
    for (int g = 0; g < G && holder < 0; ++g)
      if (old_h[e * G + g]) holder = g;
    for (int g = 0; g < G; ++g)
      if (new_h[e * G + g] && !old_h[e * G + g]) moves.push_back(Pull{e, holder, dir[holder].slot_of.at(e), g, -1});
  }
  for (int e = 0; e < N; ++e)
    for (int g = 0; g < G; ++g)
      if (old_h[e * G + g] && !new_h[e * G + g]) dir[g].vacate(e);
  for (Pull& p : moves) p.dst_slot = dir[p.dst].host(p.e);
  return moves;
}

std::vector<int32_t> counts_from_slots(const std::vector<int32_t>& slots, int N, int G, int E) {
  std::vector<int32_t> c(static_cast<size_t>(N) * G, 0);
  for (int g = 0; g < G; ++g)
    for (int s = 0; s < E; ++s)
      if (slots[g * E + s] >= 0) ++c[slots[g * E + s] * G + g];
  return c;
}

std::string ops_json(const std::vector<fm_placement_op>& ops) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < ops.size(); ++i) {
    const auto& p = ops[i];
    o << (i ? ", " : "") << "[" << p.kind << ", " << p.expert << ", " << p.gpu << ", " << p.a_gpu << ", " << p.a_slot
      << ", " << p.b_gpu << ", " << p.b_slot << "]";
  }
  o << "]";
  return o.str();
}

// ------------------------------------------------------------------ the runtime
class Runtime {
 public:
  Runtime(const Args& a, Exchange& ex) : a_(a), ex_(ex), N_(a.experts), G_(ex.world), rank_(ex.rank) {
    const int N = N_, G = G_, d = a.d, f = a.f, T = a.tokens;
    E_ = a.slots > 0 ? a.slots : 2 * ((N + G - 1) / G);  // vExpert budget 2*ceil(N/G) (moesim.cpp:141-146)
    s_ = ex.stream();
    // cluster profile: the reference's A100-like default, or one NVSwitch node of B200s
    if (a.profile == "reference") {
      ck(fm_profile_reference_default(G, E_, &prof_), "profile");
    } else {  // profile.py b200_profile: NVLink 5 770 GB/s, all-reduce bus 725 GB/s, f32 grads, 12 B/param state
      std::memset(&prof_, 0, sizeof(prof_));
      prof_.num_gpus = G;
      prof_.gpus_per_node = G;
      prof_.slots_per_gpu = E_;
      prof_.intra_node_bandwidth_bps = prof_.inter_node_bandwidth_bps = 770e9;
      prof_.tps = a.tps;
      const double P = 2.0 * d * f + d + f;
      prof_.expert_param_bytes = 4.0 * P;
      prof_.expert_state_bytes = 12.0 * P;
      prof_.token_bytes = 2.0 * d;
      for (int n = 2; n <= G; ++n) prof_.allreduce_bps_intra[n] = 725e9 * n / (2.0 * (n - 1));
    }
    fm_scheduler_config sc{1.1, 0, 0, 10, 50, 0.5, 64, 0.005, a.flip == "copy" ? 1 : 0, a.async_policy};
    ck(fm_scheduler_create(&prof_, &sc, N, &sched_), "fm_scheduler_create");
    slots_.assign(static_cast<size_t>(G) * E_, -1);
    std::vector<int32_t> counts(static_cast<size_t>(N) * G);
    ck(fm_scheduler_placement(sched_, 0, slots_.data(), counts.data()), "placement");
    hosted_.assign(counts.size(), 0);
    for (size_t i = 0; i < counts.size(); ++i) hosted_[i] = counts[i] > 0;

    fm_layer_config lc{N, a.topk, d, f, G, rank_, T, E_};
    ck(fm_layer_create(&lc, counts.data(), &layer_), "fm_layer_create");
    p2p_ = a.transport == "p2p";
    if (p2p_) ck(fm_layer_enable_p2p(layer_), "fm_layer_enable_p2p");
    cap_ = 3 * E_;  // hosted + in-flight receivers; vacated slots stay readable one step
    ck(fm_pool_create(cap_, d, f, G, &pool_), "fm_pool_create");
    ck(fm_pool_set_operand_layout(pool_, 1), "operand layout");
    int64_t P = 0, sb = 0;
    ck(fm_pool_info(pool_, &P, &sb), "fm_pool_info");
    P_ = P;
    for (int g = 0; g < G; ++g) dir_.emplace_back(cap_);
    for (int g = 0; g < G; ++g)
      for (int e = 0; e < N; ++e)
        if (hosted_[e * G + g]) dir_[g].host(e);
    ex.share(layer_, pool_, p2p_);

    // operands at their pool slots, gradients for at most min(N, cap) local experts
    const size_t fd = static_cast<size_t>(f) * d;
    w1_ = dev_alloc<uint16_t>(cap_ * fd);
    w2_ = dev_alloc<uint16_t>(cap_ * fd);
    b1_ = dev_alloc<float>(static_cast<size_t>(cap_) * f);
    b2_ = dev_alloc<float>(static_cast<size_t>(cap_) * d);
    const size_t L = std::min(N, cap_);
    dw1_ = dev_alloc<float>(L * fd);
    dw2_ = dev_alloc<float>(L * fd);
    db1_ = dev_alloc<float>(L * f);
    db2_ = dev_alloc<float>(L * d);
    dwg_ = dev_alloc<float>(static_cast<size_t>(N) * d);
    hist_ = dev_alloc<int64_t>(N);
    gathered_ = dev_alloc<int64_t>(static_cast<size_t>(G) * N);
    cu(cudaMallocHost(&demand_host_, sizeof(int64_t) * N * G), "pinned");
    cu(cudaEventCreateWithFlags(&demand_ev_, cudaEventDisableTiming), "event");
    y_ = dev_alloc<uint16_t>(static_cast<size_t>(T) * d);
    dx_ = dev_alloc<uint16_t>(static_cast<size_t>(T) * d);
    if (!p2p_) {  // NCCL transport staging (route() may send every unit to one GPU)
      const size_t units = static_cast<size_t>(T) * a.topk;
      stage_rows_ = units * G;
      for (void** b : {&send_, &back_, &dsend_, &dback_}) *b = dev_alloc<uint16_t>(units * d);
      for (void** b : {&recv_, &ret_, &drecv_, &dret_}) *b = dev_alloc<uint16_t>(stage_rows_ * d);
    }
  }

  ~Runtime() {
    fm_scheduler_destroy(sched_);
    fm_layer_destroy(layer_);
    fm_pool_destroy(pool_);
    for (void* p : std::initializer_list<void*>{w1_, w2_, b1_, b2_, dw1_, dw2_, db1_, db2_, dwg_, hist_, gathered_,
                                                 y_, dx_, send_, recv_, ret_, back_, dsend_, drecv_, dret_, dback_})
      if (p) cudaFree(p);
    cudaFreeHost(demand_host_);
    cudaEventDestroy(demand_ev_);
  }

  // initial master weights of every hosted expert: [N][P] f32 (w1|b1|w2|b2), m = v = 0
  void init_experts(const std::vector<float>& master_NP) {
    for (const auto& [e, slot] : dir_[rank_].slot_of) {
      void* base = nullptr;
      ck(fm_pool_slot_ptr(pool_, slot, &base), "slot ptr");
      cu(cudaMemcpy(base, master_NP.data() + static_cast<size_t>(e) * P_, 4 * P_, cudaMemcpyHostToDevice), "H2D");
      cu(cudaMemset(static_cast<float*>(base) + P_, 0, 8 * P_), "memset m v");
    }
    std::vector<int32_t> local = local_experts(), sl;
    for (int e : local) sl.push_back(dir_[rank_].slot_of.at(e));
    ck(fm_pool_pack(pool_, sl.data(), static_cast<int>(sl.size()), w1_, b1_, w2_, b2_, s_), "pack");
    upload_operand_slots();
    cu(cudaStreamSynchronize(s_), "sync");
  }

  std::vector<int32_t> local_experts() const {
    std::vector<int32_t> out(N_);
    int n = 0;
    ck(fm_layer_local_experts(layer_, &n, out.data()), "local experts");
    out.resize(n);
    return out;
  }

  struct StepLog {
    double balance_ratio = 0, makespan_s = 0;
    std::vector<fm_placement_op> applied, issued, accepted;
    int64_t migration_bytes = 0;
    double switch_us = 0, finish_us = 0;
  };

  StepLog step(const void* x, const void* dy, const void* wg) {
    using clk = std::chrono::steady_clock;
    StepLog log;
    const int N = N_, G = G_, d = a_.d, f = a_.f, T = a_.tokens;
    const bool copy = a_.flip == "copy";
    auto t0 = clk::now();
    fm_step_report rep{};
    ck(fm_scheduler_begin_step(sched_, &rep), "begin_step");
    log.applied = ops(1, rep.n_applied);
    if (copy) log.issued = ops(2, rep.n_issued);
    std::vector<Pull> pulls;
    if (!log.applied.empty() || !log.issued.empty()) pulls = switch_placement(log.applied, log.issued);
    std::vector<int32_t> moves, pulled;
    for (const Pull& p : pulls)
      if (p.dst == rank_) {
        moves.insert(moves.end(), {p.dst_slot, p.src, p.src_slot});
        pulled.push_back(p.dst_slot);
      }
    log.migration_bytes = static_cast<int64_t>(pulled.size()) * 12 * P_;
    log.switch_us = std::chrono::duration<double, std::micro>(clk::now() - t0).count();

    // ---- forward
    ck(fm_layer_gate(layer_, x, T, wg, hist_, s_), "gate");
    ex_.all_gather_i64(hist_, gathered_, N);
    if (!pulls.empty())  // after the all-gather: every source finished its previous Adam step
      ck(fm_pool_migrate(pool_, moves.data(), static_cast<int>(pulled.size()), pulled.data(),
                         static_cast<int>(pulled.size()), w1_, b1_, w2_, b2_, s_),
         "fm_pool_migrate");
    cu(cudaMemcpyAsync(demand_host_, gathered_, sizeof(int64_t) * G * N, cudaMemcpyDeviceToHost, s_), "D2H demand");
    cu(cudaEventRecord(demand_ev_, s_), "record");
    const std::vector<int32_t> local = local_experts();
    const int nl = static_cast<int>(local.size());
    if (p2p_) {
      ck(fm_layer_route_p2p(layer_, gathered_, s_), "route_p2p");
      ck(fm_layer_dispatch_p2p(layer_, x, s_), "dispatch_p2p");
      ex_.fence();
      if (!copy) ck(fm_pool_wait_ready(pool_, s_), "wait_ready");
      ck(fm_layer_expert_forward_p2p(layer_, w1_, b1_, w2_, b2_, s_), "expert_forward_p2p");
      ex_.fence();
      ck(fm_layer_combine_p2p(layer_, y_, s_), "combine_p2p");
      // ---- backward
      ck(fm_layer_combine_backward_p2p(layer_, dy, s_), "combine_backward_p2p");
      ex_.fence();
      ck(fm_layer_p2p_bind_dx(layer_, wg, dx_), "p2p_bind_dx");  // un-permute beside the FFN1 wgrad
      ck(fm_layer_expert_backward_p2p(layer_, w1_, w2_, dw1_, db1_, dw2_, db2_, dwg_, s_), "expert_backward_p2p");
      ex_.fence();
      ck(fm_layer_unpermute_backward_p2p(layer_, wg, dx_, dwg_, s_), "unpermute_backward_p2p");
    } else {
      std::vector<int32_t> sr(G), rr(G);
      ck(fm_layer_route(layer_, gathered_, sr.data(), rr.data(), s_), "route");  // synchronises (NCCL needs counts)
      const std::vector<int> send_rows(sr.begin(), sr.end()), recv_rows(rr.begin(), rr.end());
      const size_t rb = 2ull * d;
      ck(fm_layer_dispatch(layer_, x, send_, s_), "dispatch");
      ex_.all_to_all(send_, send_rows, recv_, recv_rows, rb);
      if (!copy) ck(fm_pool_wait_ready(pool_, s_), "wait_ready");
      ck(fm_layer_expert_forward(layer_, recv_, w1_, b1_, w2_, b2_, ret_, s_), "expert_forward");
      ex_.all_to_all(ret_, recv_rows, back_, send_rows, rb);
      ck(fm_layer_combine(layer_, back_, y_, s_), "combine");
      ck(fm_layer_combine_backward(layer_, dy, back_, dsend_, s_), "combine_backward");
      ex_.all_to_all(dsend_, send_rows, drecv_, recv_rows, rb);
      ck(fm_layer_expert_backward(layer_, drecv_, w1_, w2_, dw1_, db1_, dw2_, db2_, dret_, s_), "expert_backward");
      ex_.all_to_all(dret_, recv_rows, dback_, send_rows, rb);
      ck(fm_layer_unpermute_backward(layer_, dback_, send_, wg, dx_, dwg_, s_), "unpermute_backward");
    }
    // ---- replica-group gradient sums, ascending expert id (sim_engine.cpp:67-113)
    if (copy) ck(fm_pool_wait_ready(pool_, s_), "wait_ready");  // in-flight receivers' states landed
    for (int e = 0; e < N; ++e) {
      std::vector<int> grp;
      for (int g = 0; g < G; ++g)
        if (hosted_[e * G + g]) grp.push_back(g);
      if (grp.size() < 2) continue;
      std::vector<std::pair<float*, size_t>> bufs;
      const auto it = std::find(local.begin(), local.end(), e);
      if (it != local.end()) {
        const size_t li = static_cast<size_t>(it - local.begin());
        bufs = {{dw1_ + li * f * d, static_cast<size_t>(f) * d}, {db1_ + li * f, static_cast<size_t>(f)},
                {dw2_ + li * d * f, static_cast<size_t>(d) * f}, {db2_ + li * d, static_cast<size_t>(d)}};
      } else {
        bufs.resize(4, {nullptr, 0});
      }
      ex_.all_reduce(bufs, grp);
    }
    ex_.all_reduce({{dwg_, static_cast<size_t>(N) * d}}, {});
    // ---- the step's demand on the host, Adam on every hosted expert, policy
    cu(cudaEventSynchronize(demand_ev_), "demand event");
    std::vector<int64_t> D(static_cast<size_t>(N) * G);
    for (int e = 0; e < N; ++e)
      for (int g = 0; g < G; ++g) D[e * G + g] = demand_host_[g * N + e];
    if (a_.adam) {
      ++adam_t_;
      if (nl) {
        std::vector<int32_t> sl;
        for (int e : local) sl.push_back(dir_[rank_].slot_of.at(e));
        fm_adam_config ac{static_cast<float>(a_.lr), 0.9f, 0.999f, 1e-8f, adam_t_};
        ck(fm_pool_adam(pool_, sl.data(), nl, dw1_, db1_, dw2_, db2_, &ac, w1_, b1_, w2_, b2_, s_), "fm_pool_adam");
      }
    }
    auto t1 = clk::now();
    ck(fm_scheduler_finish_step(sched_, D.data(), &rep), "finish_step");
    log.finish_us = std::chrono::duration<double, std::micro>(clk::now() - t1).count();
    log.accepted = ops(0, rep.n_accepted);
    log.balance_ratio = rep.balance_ratio;
    log.makespan_s = rep.makespan_s;
    return log;
  }

  std::vector<fm_placement_op> ops(int which, int n) {
    std::vector<fm_placement_op> v(std::max(n, 1));
    int got = 0;
    ck(fm_scheduler_ops(sched_, which, v.data(), static_cast<int>(v.size()), &got), "fm_scheduler_ops");
    v.resize(got);
    return v;
  }

  int p2p_status() {
    int t = 0;
    if (p2p_) ck(fm_layer_p2p_status(layer_, &t), "p2p_status");
    return t;
  }
  void dump(const std::string& dir) {  // y of the last step, states of the hosted experts
    cu(cudaStreamSynchronize(s_), "sync");
    const size_t yb = 2ull * a_.tokens * a_.d;
    std::vector<char> h(yb);
    cu(cudaMemcpy(h.data(), y_, yb, cudaMemcpyDeviceToHost), "D2H y");
    write_file(dir + "/y_" + std::to_string(rank_) + ".bin", h.data(), yb);
    for (int e : local_experts()) {
      void* base = nullptr;
      ck(fm_pool_slot_ptr(pool_, dir_[rank_].slot_of.at(e), &base), "slot ptr");
      std::vector<float> st(3 * P_);
      cu(cudaMemcpy(st.data(), base, 12 * P_, cudaMemcpyDeviceToHost), "D2H state");
      write_file(dir + "/state_" + std::to_string(rank_) + "_" + std::to_string(e) + ".bin", st.data(), 12 * P_);
    }
  }
  const std::vector<int32_t>& slots() const { return slots_; }
  int slots_per_gpu() const { return E_; }
  cudaStream_t stream() const { return s_; }

 private:
  // the placement boundary (runtime.py FlexMoERuntime._switch)
  std::vector<Pull> switch_placement(const std::vector<fm_placement_op>& applied,
                                     const std::vector<fm_placement_op>& issued) {
    const int N = N_, G = G_;
    for (const auto& op : applied)
      ck(fm_placement_apply(slots_.data(), N, &prof_, &op, nullptr, nullptr), "fm_placement_apply");
    const std::vector<int32_t> counts = counts_from_slots(slots_, N, G, E_);
    std::vector<uint8_t> h(counts.size());
    for (size_t i = 0; i < counts.size(); ++i) h[i] = counts[i] > 0;
    if (!issued.empty()) {
      std::vector<int32_t> pend = slots_;
      for (const auto& op : issued)
        ck(fm_placement_apply(pend.data(), N, &prof_, &op, nullptr, nullptr), "fm_placement_apply");
      const std::vector<int32_t> pc = counts_from_slots(pend, N, G, E_);
      for (size_t i = 0; i < pc.size(); ++i) h[i] = h[i] || pc[i] > 0;
    }
    std::vector<Pull> pulls = apply_placement_change(dir_, hosted_, h, N, G);
    hosted_ = h;
    std::vector<int32_t> col(N);
    for (int e = 0; e < N; ++e) col[e] = hosted_[e * G + rank_];
    ck(fm_layer_set_placement_async(layer_, counts.data(), col.data(), s_), "set_placement_async");
    upload_operand_slots();
    return pulls;
  }
  void upload_operand_slots() {
    std::vector<int32_t> t(N_, -1);
    for (const auto& [e, s] : dir_[rank_].slot_of) t[e] = s;
    ck(fm_layer_set_operand_slots(layer_, t.data(), cap_, s_), "set_operand_slots");
  }

  const Args& a_;
  Exchange& ex_;
  int N_, G_, rank_, E_ = 0, cap_ = 0;
  int64_t P_ = 0;
  int adam_t_ = 0;
  bool p2p_ = true;
  cudaStream_t s_ = nullptr;
  fm_cluster_profile prof_{};
  fm_scheduler* sched_ = nullptr;
  fm_layer* layer_ = nullptr;
  fm_expert_pool* pool_ = nullptr;
  std::vector<int32_t> slots_;
  std::vector<uint8_t> hosted_;  // [N][G] state holders
  std::vector<SlotAllocator> dir_;
  void *w1_ = nullptr, *w2_ = nullptr;
  float *b1_ = nullptr, *b2_ = nullptr, *dw1_ = nullptr, *dw2_ = nullptr, *db1_ = nullptr, *db2_ = nullptr,
        *dwg_ = nullptr;
  int64_t *hist_ = nullptr, *gathered_ = nullptr, *demand_host_ = nullptr;
  cudaEvent_t demand_ev_ = nullptr;
  void *y_ = nullptr, *dx_ = nullptr;
  size_t stage_rows_ = 0;
  void *send_ = nullptr, *recv_ = nullptr, *ret_ = nullptr, *back_ = nullptr, *dsend_ = nullptr, *drecv_ = nullptr,
       *dret_ = nullptr, *dback_ = nullptr;
};

// ------------------------------------------------------------------ one rank
struct Inputs {
  void *x = nullptr, *dy = nullptr, *wg = nullptr;
  std::vector<float> experts;  // [N][P]
  std::vector<uint16_t> wg_host;
};

Inputs make_inputs(const Args& a, int rank, int64_t P) {
  const int N = a.experts, d = a.d, f = a.f, T = a.tokens;
  Inputs in;
  const size_t td = static_cast<size_t>(T) * d;
  std::vector<uint16_t> x(td), dy(td);
  in.wg_host.resize(static_cast<size_t>(N) * d);
  if (!a.inputs.empty()) {  // files written by the parity test (raw little-endian)
    auto rx = read_file(a.inputs + "/x_" + std::to_string(rank) + ".bin", 2 * td);
    auto rdy = read_file(a.inputs + "/dy_" + std::to_string(rank) + ".bin", 2 * td);
    auto rwg = read_file(a.inputs + "/wg.bin", 2ull * N * d);
    auto rex = read_file(a.inputs + "/experts.bin", 4ull * N * P);
    std::memcpy(x.data(), rx.data(), rx.size());
    std::memcpy(dy.data(), rdy.data(), rdy.size());
    std::memcpy(in.wg_host.data(), rwg.data(), rwg.size());
    in.experts.resize(static_cast<size_t>(N) * P);
    std::memcpy(in.experts.data(), rex.data(), rex.size());
  } else {  // synthetic: skewed gate (Zipf popularity in feature column 0, x[:, 0] = 0.5)
    std::mt19937_64 rng(1234 + rank);
    std::normal_distribution<float> g1(0.0f, 1.0f);
    for (size_t i = 0; i < td; ++i) {
      x[i] = bf16(i % d == 0 ? 0.5f : g1(rng));
      dy[i] = bf16(0.1f * g1(rng));
    }
    std::mt19937_64 wr(7);  // identical on every rank
    for (int e = 0; e < N; ++e)
      for (int j = 0; j < d; ++j) in.wg_host[static_cast<size_t>(e) * d + j] = bf16(g1(wr) / std::sqrt(float(d)));
    in.experts.resize(static_cast<size_t>(N) * P);
    for (int e = 0; e < N; ++e) {
      std::mt19937_64 er(10000 + e);
      float* m = in.experts.data() + static_cast<size_t>(e) * P;
      const size_t fd = static_cast<size_t>(f) * d;
      for (size_t i = 0; i < fd; ++i) m[i] = g1(er) / std::sqrt(float(d));
      for (int i = 0; i < f; ++i) m[fd + i] = 0.02f * g1(er);
      for (size_t i = 0; i < fd; ++i) m[fd + f + i] = g1(er) / std::sqrt(float(f));
      for (int i = 0; i < d; ++i) m[2 * fd + f + i] = 0.02f * g1(er);
    }
  }
  in.x = dev_alloc<uint16_t>(td);
  in.dy = dev_alloc<uint16_t>(td);
  in.wg = dev_alloc<uint16_t>(static_cast<size_t>(N) * d);
  cu(cudaMemcpy(in.x, x.data(), 2 * td, cudaMemcpyHostToDevice), "H2D x");
  cu(cudaMemcpy(in.dy, dy.data(), 2 * td, cudaMemcpyHostToDevice), "H2D dy");
  cu(cudaMemcpy(in.wg, in.wg_host.data(), 2ull * N * d, cudaMemcpyHostToDevice), "H2D wg");
  return in;
}

// Zipf log-popularity over a seeded permutation (workload.cpp:135-170 shape),
// drifting per step (p *= exp(U[-0.02, 0.02]), renormalised), written into the
// gate's skew column 0 (x[:, 0] = 0.5): routing is produced by the gate.
struct Drift {
  Drift(int N, double zipf) : logp(N), rng(42) {
    std::vector<int> perm(N);
    for (int i = 0; i < N; ++i) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), std::mt19937_64(42));
    double z = 0;
    for (int i = 0; i < N; ++i) z += 1.0 / std::pow(i + 1.0, zipf);
    for (int i = 0; i < N; ++i) logp[perm[i]] = std::log(1.0 / std::pow(i + 1.0, zipf) / z);
  }
  void step() {
    std::uniform_real_distribution<double> u(-0.02, 0.02);
    double z = 0;
    for (double& l : logp) {
      l += u(rng);
      z += std::exp(l);
    }
    for (double& l : logp) l -= std::log(z);
  }
  std::vector<double> logp;
  std::mt19937_64 rng;
};

int run_rank(const Args& a, Exchange& ex, int device) {
  cu(cudaSetDevice(device), "cudaSetDevice");
  Runtime rt(a, ex);
  int64_t P = 2ll * a.d * a.f + a.d + a.f;
  Inputs in = make_inputs(a, ex.rank, P);
  rt.init_experts(in.experts);
  const bool synthetic = a.inputs.empty();
  Drift drift(a.experts, a.zipf);
  uint16_t* col_host = nullptr;  // the gate's skew column, staged per step from pinned memory
  cu(cudaMallocHost(&col_host, 2ull * a.experts), "pinned");
  auto drive = [&]() {
    if (synthetic) {
      drift.step();
      for (int e = 0; e < a.experts; ++e) col_host[e] = bf16(static_cast<float>(2.0 * drift.logp[e]));
      cu(cudaMemcpy2DAsync(in.wg, 2ull * a.d, col_host, 2, 2, a.experts, cudaMemcpyHostToDevice, rt.stream()),
         "skew column");
    }
    return rt.step(in.x, in.dy, in.wg);
  };
  for (int i = 0; i < a.warmup; ++i) drive();
  cu(cudaStreamSynchronize(rt.stream()), "sync");
  ex.fence();
  cudaEvent_t e0, e1;
  cu(cudaEventCreate(&e0), "event");
  cu(cudaEventCreate(&e1), "event");
  cu(cudaEventRecord(e0, rt.stream()), "record");
  std::vector<Runtime::StepLog> logs;
  for (int i = 0; i < a.steps; ++i) logs.push_back(drive());
  cu(cudaEventRecord(e1, rt.stream()), "record");
  cu(cudaEventSynchronize(e1), "sync");
  float ms = 0;
  cu(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  const double ms_max = ex.max_over_ranks(ms);
  const int timeouts = rt.p2p_status();
  if (!a.dump.empty()) rt.dump(a.dump);
  if (ex.rank == 0) {
    if (a.log_steps)
      for (size_t i = 0; i < logs.size(); ++i) {
        const auto& l = logs[i];
        std::printf(
            "{\"step\": %zu, \"balance_ratio\": %.17g, \"makespan_s\": %.17g, \"applied\": %s, \"issued\": %s, "
            "\"accepted\": %s, \"migration_bytes\": %lld, \"switch_us\": %.1f, \"finish_us\": %.1f}\n",
            i + a.warmup, l.balance_ratio, l.makespan_s, ops_json(l.applied).c_str(), ops_json(l.issued).c_str(),
            ops_json(l.accepted).c_str(), static_cast<long long>(l.migration_bytes), l.switch_us, l.finish_us);
      }
    int applied = 0, accepted = 0;
    double ratio_sum = 0, switch_max = 0, finish_sum = 0;
    for (const auto& l : logs) {
      applied += static_cast<int>(l.applied.size());
      accepted += static_cast<int>(l.accepted.size());
      ratio_sum += l.balance_ratio;
      switch_max = std::max(switch_max, l.switch_us);
      finish_sum += l.finish_us;
    }
    const double per_step = ms_max / a.steps;
    const int G = ex.world;
    std::printf(
        "{\"metric\": \"MoE-layer fwd+bwd tokens/sec\", \"value\": %.1f, \"unit\": \"tokens/s\", \"n_gpus\": %d, "
        "\"loopback\": %s, \"steps\": %d, \"ms_per_step\": %.4f, \"host\": \"C++ runtime (host/flexmoe_runtime.cpp) "
        "over the C ABI\", \"transport\": \"%s\", \"flip\": \"%s\", \"async_policy\": %d, \"adam\": %d, "
        "\"config\": {\"experts\": %d, \"top_k\": %d, \"d_model\": %d, \"d_ff\": %d, \"tokens_per_gpu\": %d, "
        "\"slots_per_gpu\": %d, \"zipf\": %.3f}, \"balance_ratio_mean\": %.6f, \"balance_ratio_last\": %.6f, "
        "\"ops_applied\": %d, \"ops_accepted\": %d, \"switch_host_us_max\": %.1f, \"finish_host_us_mean\": %.1f, "
        "\"p2p_timeouts\": %d}\n",
        static_cast<double>(a.tokens) * G / (per_step * 1e-3), G, a.loopback ? "true" : "false", a.steps, per_step,
        a.transport.c_str(), a.flip.c_str(), a.async_policy, a.adam, a.experts, a.topk, a.d, a.f, a.tokens,
        rt.slots_per_gpu(), a.zipf, logs.empty() ? 0.0 : ratio_sum / logs.size(),
        logs.empty() ? 0.0 : logs.back().balance_ratio, applied, accepted, switch_max,
        logs.empty() ? 0.0 : finish_sum / logs.size(), timeouts);
    std::fflush(stdout);
  }
  cudaFreeHost(col_host);
  for (void* p : {in.x, in.dy, in.wg}) cudaFree(p);
  return timeouts ? 3 : 0;
}

int run_loopback(const Args& a) {
  cu(cudaSetDevice(0), "cudaSetDevice");
  LoopbackHub hub(a.loopback);
  std::vector<std::unique_ptr<LoopbackExchange>> ex;
  for (int r = 0; r < a.loopback; ++r) ex.push_back(std::make_unique<LoopbackExchange>(hub, r));
  std::vector<int> rc(a.loopback, 1);
  std::vector<std::thread> th;
  for (int r = 0; r < a.loopback; ++r)
    th.emplace_back([&, r] {
      try {
        rc[r] = run_rank(a, *ex[r], 0);
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
        hub.abort();
      }
    });
  for (auto& t : th) t.join();
  return *std::max_element(rc.begin(), rc.end());
}

int run_processes(const Args& a) {
  setenv("NCCL_SOCKET_IFNAME", "lo", 0);  // one node: bootstrap over loopback
  int idpipe[2];
  if (pipe(idpipe) != 0) throw std::runtime_error("pipe failed");
  std::vector<pid_t> kids;
  for (int r = 0; r < a.gpus; ++r) {
    const pid_t pid = fork();
    if (pid < 0) throw std::runtime_error("fork failed");
    if (pid == 0) {  // no NCCL state before fork(): rank 0 creates the id, the pipe carries it
      int rc = 1;
      try {
        ncclUniqueId id;
        if (r == 0) {
          close(idpipe[0]);
          nc(ncclGetUniqueId(&id), "ncclGetUniqueId");
          for (int p = 1; p < a.gpus; ++p)
            if (write(idpipe[1], &id, sizeof(id)) != static_cast<ssize_t>(sizeof(id)))
              throw std::runtime_error("unique id pipe write failed");
          close(idpipe[1]);
        } else {
          close(idpipe[1]);
          size_t got = 0;
          while (got < sizeof(id)) {
            const ssize_t n = read(idpipe[0], reinterpret_cast<char*>(&id) + got, sizeof(id) - got);
            if (n <= 0) throw std::runtime_error("unique id pipe read failed");
            got += static_cast<size_t>(n);
          }
          close(idpipe[0]);
        }
        cu(cudaSetDevice(r), "cudaSetDevice");
        NcclExchange ex(r, a.gpus, id);
        rc = run_rank(a, ex, r);
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
      }
      std::fflush(stdout);
      _exit(rc);
    }
    kids.push_back(pid);
  }
  close(idpipe[0]);
  close(idpipe[1]);
  int worst = 0;
  for (pid_t pid : kids) {
    int st = 0;
    waitpid(pid, &st, 0);
    worst = std::max(worst, WIFEXITED(st) ? WEXITSTATUS(st) : 1);
  }
  return worst;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    return a.loopback ? run_loopback(a) : run_processes(a);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "flexmoe_runtime: %s\n", e.what());
    return 2;
  }
}
