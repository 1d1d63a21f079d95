// flexmoe_step — C++ host driver of the multi-GPU FlexMoE layer step (no
// Python, no torch): one process per GPU (forked here, or one per launcher
// rank), NCCL for the two small collectives the step still needs (the
// per-GPU expert histogram all-gather and the gradient all-reduces), and the
// layer's peer-to-peer token transport for dispatch / combine and their
// backward mirrors (CUDA IPC-mapped arenas, include/flexmoe_b200.h).
//
// Per step, on every GPU (the exchanges the reference models
// in proj/src/cost_model.cpp:37-64):
//   gate + top-k + histogram        fm_layer_gate
//   all-gather of the histograms    ncclAllGather (TokenDemand D[e][g] on every GPU)
//   route() + plan, no host sync    fm_layer_route_p2p
//   dispatch into peers' X_perm     fm_layer_dispatch_p2p
//   expert FFN                      fm_layer_expert_forward_p2p
//   combine (reads peers' Y rows)   fm_layer_combine_p2p
//   backward mirrors                fm_layer_combine_backward_p2p / _expert_backward_p2p /
//                                   _unpermute_backward_p2p
//   replica-group gradient sums     ncclAllReduce per replicated expert, ascending id,
//                                   communicators split per group and cached
//                                   (sim_engine.cpp:45-113)
//   gate-weight gradient            ncclAllReduce over all GPUs
//
//   flexmoe_step --gpus N [--steps K] [--warmup W] [--experts E] [--topk k]
//                [--d-model d] [--d-ff f] [--tokens T] [--replicate R]
// prints one JSON line (rank 0): tokens/s over all GPUs (max over ranks of
// the device-timed K steps), the balance ratio of the last step's routing.
#include <cuda_runtime.h>
#include <nccl.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
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
  int gpus = 1, steps = 20, warmup = 3, experts = 64, topk = 1, d = 1024, f = 4096, tokens = 65536;
  int replicate = 2;  // the `replicate` hottest experts get a replica on every GPU
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const int v = std::atoi(argv[i + 1]);
    if (k == "--gpus") a.gpus = v;
    else if (k == "--steps") a.steps = v;
    else if (k == "--warmup") a.warmup = v;
    else if (k == "--experts") a.experts = v;
    else if (k == "--topk") a.topk = v;
    else if (k == "--d-model") a.d = v;
    else if (k == "--d-ff") a.f = v;
    else if (k == "--tokens") a.tokens = v;
    else if (k == "--replicate") a.replicate = v;
    else throw std::invalid_argument("unknown option " + k);
  }
  return a;
}

// bf16 bits of a float (round to nearest even)
uint16_t bf16(float v) {
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

void* dev_bf16_random(size_t n, float scale, std::mt19937_64& rng) {
  std::normal_distribution<float> g(0.0f, scale);
  std::vector<uint16_t> h(n);
  for (auto& v : h) v = bf16(g(rng));
  void* p = dev_alloc<uint16_t>(n);
  cu(cudaMemcpy(p, h.data(), 2 * n, cudaMemcpyHostToDevice), "H2D");
  return p;
}

int run_rank(const Args& a, int rank, const ncclUniqueId& id) {
  const int G = a.gpus, N = a.experts, k = a.topk, d = a.d, f = a.f, T = a.tokens;
  cu(cudaSetDevice(rank), "cudaSetDevice");
  ncclComm_t world;
  nc(ncclCommInitRank(&world, G, id, rank), "ncclCommInitRank");
  cudaStream_t s;
  cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");

  // placement: expert e on GPU e % G (round robin), the `replicate` experts
  // with the largest gate skew replicated everywhere
  std::vector<int32_t> counts(static_cast<size_t>(N) * G, 0);
  for (int e = 0; e < N; ++e) counts[static_cast<size_t>(e) * G + e % G] = 1;
  for (int e = 0; e < std::min(a.replicate, N); ++e)
    for (int g = 0; g < G; ++g) counts[static_cast<size_t>(e) * G + g] = std::max(1, counts[e * G + g]);
  std::vector<int32_t> local;
  for (int e = 0; e < N; ++e)
    if (counts[static_cast<size_t>(e) * G + rank] > 0) local.push_back(e);
  const int Nl = static_cast<int>(local.size());

  fm_layer_config cfg{N, k, d, f, G, rank, T, 0};
  fm_layer* layer = nullptr;
  ck(fm_layer_create(&cfg, counts.data(), &layer), "fm_layer_create");
  ck(fm_layer_enable_p2p(layer), "fm_layer_enable_p2p");

  // exchange the arena handles with one all-gather
  char* hdev = dev_alloc<char>(64 * G);
  {
    char h[64];
    ck(fm_layer_p2p_handle(layer, h), "fm_layer_p2p_handle");
    cu(cudaMemcpy(hdev + 64 * rank, h, 64, cudaMemcpyHostToDevice), "H2D handle");
    nc(ncclAllGather(hdev + 64 * rank, hdev, 64, ncclChar, world, s), "ncclAllGather handles");
    std::vector<char> all(64 * G);
    cu(cudaMemcpyAsync(all.data(), hdev, 64 * G, cudaMemcpyDeviceToHost, s), "D2H handles");
    cu(cudaStreamSynchronize(s), "sync");
    for (int p = 0; p < G; ++p)
      if (p != rank) ck(fm_layer_p2p_open_peer(layer, p, all.data() + 64 * p), "fm_layer_p2p_open_peer");
  }

  // replica groups: one communicator per distinct group, split in ascending expert id
  std::map<std::vector<int>, ncclComm_t> groups;
  std::vector<std::pair<int, ncclComm_t>> sync_list;  // (local index, comm), ascending expert id
  for (int e = 0; e < N; ++e) {
    std::vector<int> grp;
    for (int g = 0; g < G; ++g)
      if (counts[static_cast<size_t>(e) * G + g] > 0) grp.push_back(g);
    if (grp.size() < 2) continue;
    const bool member = std::find(grp.begin(), grp.end(), rank) != grp.end();
    auto it = groups.find(grp);
    if (it == groups.end()) {  // collective over the world: every rank calls it
      ncclComm_t c = nullptr;
      nc(ncclCommSplit(world, member ? static_cast<int>(groups.size()) : NCCL_SPLIT_NOCOLOR, rank, &c, nullptr),
         "ncclCommSplit");
      it = groups.emplace(grp, c).first;
    }
    if (member) {
      const int li = static_cast<int>(std::find(local.begin(), local.end(), e) - local.begin());
      sync_list.emplace_back(li, it->second);
    }
  }

  // synthetic inputs and random-init weights of the architecture
  std::mt19937_64 rng(1234 + rank);
  void* x = dev_bf16_random(static_cast<size_t>(T) * d, 1.0f, rng);
  void* dy = dev_bf16_random(static_cast<size_t>(T) * d, 0.1f, rng);
  std::mt19937_64 wrng(7);  // identical gate and expert weights on every GPU
  void* wg = dev_bf16_random(static_cast<size_t>(N) * d, 1.0f / std::sqrt(static_cast<float>(d)), wrng);
  void* w1 = dev_bf16_random(static_cast<size_t>(std::max(Nl, 1)) * f * d, 1.0f / std::sqrt(static_cast<float>(d)),
                             wrng);
  void* w2 = dev_bf16_random(static_cast<size_t>(std::max(Nl, 1)) * d * f, 1.0f / std::sqrt(static_cast<float>(f)),
                             wrng);
  float* b1 = dev_alloc<float>(static_cast<size_t>(std::max(Nl, 1)) * f);
  float* b2 = dev_alloc<float>(static_cast<size_t>(std::max(Nl, 1)) * d);
  cu(cudaMemset(b1, 0, sizeof(float) * std::max(Nl, 1) * f), "memset");
  cu(cudaMemset(b2, 0, sizeof(float) * std::max(Nl, 1) * d), "memset");
  void* y = dev_alloc<uint16_t>(static_cast<size_t>(T) * d);
  void* dx = dev_alloc<uint16_t>(static_cast<size_t>(T) * d);
  const size_t Lw = std::max(Nl, 1);
  float* dw1 = dev_alloc<float>(Lw * f * d);
  float* db1 = dev_alloc<float>(Lw * f);
  float* dw2 = dev_alloc<float>(Lw * d * f);
  float* db2 = dev_alloc<float>(Lw * d);
  float* dwg = dev_alloc<float>(static_cast<size_t>(N) * d);
  int64_t* hist = dev_alloc<int64_t>(N);
  int64_t* gathered = dev_alloc<int64_t>(static_cast<size_t>(G) * N);

  auto step = [&]() {
    ck(fm_layer_gate(layer, x, T, wg, hist, s), "gate");
    nc(ncclAllGather(hist, gathered, N, ncclInt64, world, s), "ncclAllGather hist");
    ck(fm_layer_route_p2p(layer, gathered, s), "route");
    ck(fm_layer_dispatch_p2p(layer, x, s), "dispatch");
    ck(fm_layer_expert_forward_p2p(layer, w1, b1, w2, b2, s), "expert_forward");
    ck(fm_layer_combine_p2p(layer, y, s), "combine");
    ck(fm_layer_combine_backward_p2p(layer, dy, s), "combine_backward");
    ck(fm_layer_p2p_bind_dx(layer, wg, dx), "p2p_bind_dx");  // un-permute beside the FFN1 wgrad
    ck(fm_layer_expert_backward_p2p(layer, w1, w2, dw1, db1, dw2, db2, dwg, s), "expert_backward");
    ck(fm_layer_unpermute_backward_p2p(layer, wg, dx, dwg, s), "unpermute_backward");
    for (const auto& [li, comm] : sync_list) {  // ascending expert id on every GPU
      nc(ncclGroupStart(), "group");
      nc(ncclAllReduce(dw1 + static_cast<size_t>(li) * f * d, dw1 + static_cast<size_t>(li) * f * d,
                       static_cast<size_t>(f) * d, ncclFloat, ncclSum, comm, s), "ar dw1");
      nc(ncclAllReduce(db1 + static_cast<size_t>(li) * f, db1 + static_cast<size_t>(li) * f, f, ncclFloat, ncclSum,
                       comm, s), "ar db1");
      nc(ncclAllReduce(dw2 + static_cast<size_t>(li) * d * f, dw2 + static_cast<size_t>(li) * d * f,
                       static_cast<size_t>(d) * f, ncclFloat, ncclSum, comm, s), "ar dw2");
      nc(ncclAllReduce(db2 + static_cast<size_t>(li) * d, db2 + static_cast<size_t>(li) * d, d, ncclFloat, ncclSum,
                       comm, s), "ar db2");
      nc(ncclGroupEnd(), "group end");
    }
    nc(ncclAllReduce(dwg, dwg, static_cast<size_t>(N) * d, ncclFloat, ncclSum, world, s), "ar dwg");
  };

  for (int i = 0; i < std::max(a.warmup, 1); ++i) step();
  cu(cudaStreamSynchronize(s), "sync");
  cudaEvent_t e0, e1;
  cu(cudaEventCreate(&e0), "event");
  cu(cudaEventCreate(&e1), "event");
  cu(cudaEventRecord(e0, s), "record");
  for (int i = 0; i < a.steps; ++i) step();
  cu(cudaEventRecord(e1, s), "record");
  cu(cudaEventSynchronize(e1), "sync");
  float ms = 0.0f;
  cu(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  float* msd = dev_alloc<float>(1);
  cu(cudaMemcpy(msd, &ms, 4, cudaMemcpyHostToDevice), "H2D");
  nc(ncclAllReduce(msd, msd, 1, ncclFloat, ncclMax, world, s), "ar max");  // slowest rank
  cu(cudaMemcpy(&ms, msd, 4, cudaMemcpyDeviceToHost), "D2H");
  int timed_out = 0;
  ck(fm_layer_p2p_status(layer, &timed_out), "p2p_status");
  std::vector<int64_t> flows(static_cast<size_t>(N) * G * G);
  size_t wrote = 0;
  ck(fm_layer_copy_out(layer, FM_FIELD_FLOWS, flows.data(), flows.size() * 8, &wrote), "copy_out");
  double ratio = 0.0;
  ck(fm_balance_ratio(flows.data(), N, G, &ratio), "balance_ratio");
  if (rank == 0) {
    const double per_step = ms / a.steps;
    std::printf(
        "{\"metric\": \"MoE-layer fwd+bwd tokens/sec\", \"value\": %.1f, \"unit\": \"tokens/s\", \"n_gpus\": %d, "
        "\"steps\": %d, \"ms_per_step\": %.4f, \"host\": \"C++ (host/flexmoe_step.cpp) over the C ABI, NCCL %d.%d\", "
        "\"transport\": \"p2p\", \"config\": {\"experts\": %d, \"top_k\": %d, \"d_model\": %d, \"d_ff\": %d, "
        "\"tokens_per_gpu\": %d, \"replicated_experts\": %d}, \"balance_ratio\": %.6f, \"p2p_timeouts\": %d}\n",
        static_cast<double>(T) * G / (per_step * 1e-3), G, a.steps, per_step, NCCL_MAJOR, NCCL_MINOR, N, k, d, f, T,
        std::min(a.replicate, N), ratio, timed_out);
    std::fflush(stdout);
  }
  nc(ncclCommDestroy(world), "destroy");  // collective: peers are done with this arena after it
  ck(fm_layer_destroy(layer), "fm_layer_destroy");
  return timed_out ? 3 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.gpus < 1) throw std::invalid_argument("--gpus must be >= 1");
    // one node: NCCL's bootstrap over loopback (avoids picking a slow or
    // unreachable interface on the box)
    setenv("NCCL_SOCKET_IFNAME", "lo", 0);
    // No NCCL state in the parent before fork(): rank 0 creates the unique id
    // (its bootstrap root thread lives in rank 0) and hands it to the other
    // ranks through a pipe (one 128-byte write per peer, atomic below PIPE_BUF).
    int idpipe[2];
    if (pipe(idpipe) != 0) throw std::runtime_error("pipe failed");
    std::vector<pid_t> kids;
    for (int r = 0; r < a.gpus; ++r) {
      const pid_t pid = fork();
      if (pid < 0) throw std::runtime_error("fork failed");
      if (pid == 0) {
        int rc = 1;
        try {
          ncclUniqueId id;
          if (r == 0) {
            close(idpipe[0]);
            nc(ncclGetUniqueId(&id), "ncclGetUniqueId");
            for (int peer = 1; peer < a.gpus; ++peer)
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
          rc = run_rank(a, r, id);
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
  } catch (const std::exception& e) {
    std::fprintf(stderr, "flexmoe_step: %s\n", e.what());
    return 2;
  }
}
