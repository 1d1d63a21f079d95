// C-ABI glue: error plumbing, device queries, TMA descriptor encoding and the
// thin extern "C" wrappers that translate exceptions into status codes.
#include <cudaTypedefs.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <string>

#include "fm_internal.h"

namespace fm {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
std::atomic<unsigned long long> g_launches{0};
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {  // of the current device (cached per device)
  static std::atomic<int> sms[64];
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  if (dev >= 64) {
    int n = 0;
    FM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
  }
  int n = sms[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    FM_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

void ensure_dynamic_smem(const void* kernel, int bytes) {
  if (bytes <= 48 * 1024) return;
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> set;
  std::lock_guard<std::mutex> lock(mu);
  int& cur = set[{dev, kernel}];
  if (bytes > cur) {
    FM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw cuda_error("cuTensorMapEncodeTiled not found");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
}  // namespace

CUtensorMap make_tmap_bf16(const void* base, uint64_t inner, uint64_t outer,
                           uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(base, false, inner, outer, row_stride_elems, box_inner, box_outer, 128);
}

CUtensorMap make_tmap_2d(const void* base, bool f32, uint64_t inner, uint64_t outer,
                         uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer,
                         int swizzle_bytes) {
  CUtensorMap map;
  const uint64_t esz = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_elems * esz};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                      : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = encode_fn()(&map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw cuda_error("cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) +
                     ")");
  }
  return map;
}


void set_gemm_cta_group(int cg);

}  // namespace fm

extern "C" {

const char* fm_last_error(void) { return fm::g_last_error.c_str(); }

const char* fm_version(void) { return "flexmoe_b200 0.1 (sm_100a)"; }

unsigned long long fm_kernel_launches(void) { return fm::g_launches.load(std::memory_order_relaxed); }

int fm_set_gemm_cta_group(int cta_group) {
  return fm::guarded([&] { fm::set_gemm_cta_group(cta_group); });
}

int fm_grouped_gemm(int variant, const void* A, const void* B, void* C, const float* bias,
                    const void* aux, const int32_t* seg_start, const int32_t* seg_rows,
                    const int32_t* tile_prefix, int num_groups, int total_rows, int M_w, int N,
                    int K, void* stream) {
  return fm::guarded([&] {
    fm::grouped_gemm(variant, A, B, C, bias, aux, seg_start, seg_rows, tile_prefix, num_groups,
                     total_rows, M_w, N, K, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
