// Internal helpers shared by the C-ABI translation units: status codes,
// thread-local error text, CUDA error checks and TMA descriptor encoding.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/flexmoe_b200.h"

namespace fm {

// Exception types mirror the reference's error convention:
// invalid_argument -> FM_ERR_INVALID_ARGUMENT, logic_error -> FM_ERR_LOGIC, ...
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

// Runs `body`, translating exceptions into C status codes.
template <class F>
int guarded(F&& body) {
  try {
    body();
    return FM_OK;
  } catch (const cuda_error& e) {
    set_last_error(e.what());
    return FM_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return FM_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    set_last_error(e.what());
    return FM_ERR_OUT_OF_RANGE;
  } catch (const std::logic_error& e) {
    set_last_error(e.what());
    return FM_ERR_LOGIC;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FM_ERR_RUNTIME;
  }
}

inline void check_cuda(cudaError_t err, const char* what) {
  if (err != cudaSuccess) {
    throw cuda_error(std::string(what) + ": " + cudaGetErrorString(err));
  }
}

// Kernels this library launched in the process (fm_kernel_launches): every
// launch site ends in FM_LAUNCH_CHECK, or calls count_launch() itself.
void count_launch();

#define FM_CUDA(call) ::fm::check_cuda((call), #call)
#define FM_LAUNCH_CHECK(name) (::fm::count_launch(), ::fm::check_cuda(cudaGetLastError(), name))

// 2-D bf16 tensor map, 128B swizzle: inner dimension `inner` (contiguous),
// `outer` rows `row_stride_elems` apart; box = box_inner x box_outer.
CUtensorMap make_tmap_bf16(const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer);

// General 2-D map (bf16 or f32 elements) with the given swizzle span (0/32/64/128 B).
CUtensorMap make_tmap_2d(const void* base, bool f32, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer,
                         int swizzle_bytes);

int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `kernel` on the current
// device, at least `bytes`: the attribute is per device, so it is cached per
// (device, kernel) under a mutex (launchers run on several host threads).
void ensure_dynamic_smem(const void* kernel, int bytes);

// P2P arrival gating of a token-row grouped GEMM (see grouped_gemm.cu Args).
struct SideJob;  // layer_plan.h
struct P2P;      // layer_plan.h

struct ArrivalGate {
  const unsigned long long* flags = nullptr;          // this GPU's flags of one exchange slot [src]
  const unsigned long long* tile_src_mask = nullptr;  // [128-row tiles] sources present in the tile
  unsigned long long epoch = 0;
  int* err = nullptr;
};

void grouped_gemm(int variant, const void* A, const void* B, void* C, const float* bias,
                  const void* aux, const int* seg_start, const int* seg_rows,
                  const int* tile_prefix, int num_groups, int total_rows, int M_w, int N, int K,
                  cudaStream_t stream, const ArrivalGate* gate = nullptr, const int* b_slot = nullptr,
                  int b_groups = 0, SideJob* side = nullptr, const P2P* ready = nullptr);

}  // namespace fm
