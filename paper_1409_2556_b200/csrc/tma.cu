// Host side of the TMA-fed stencil kernels: tensor-map encoding through the driver entry
// point (the runtime is linked statically; libcuda is reached via cudaGetDriverEntryPoint).
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "lt_internal.hpp"

namespace lt {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    cudaGetLastError();
  });
  return fn;
}
}  // namespace

static CUtensorMap tma_map(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                           const uint32_t* box, CUtensorMapDataType type) {
  auto fn = encode_fn();
  if (!fn) throw Error(LT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  CUtensorMap m;
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int r = 0; r < rank; ++r) {
    gd[r] = dims[r];
    bx[r] = box[r];
    es[r] = 1;
    if (r + 1 < rank) gs[r] = strides_bytes[r];
  }
  const CUresult res = fn(&m, type, (cuuint32_t)rank, const_cast<void*>(base), gd, gs, bx,
                          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) throw Error(LT_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)res));
  return m;
}

CUtensorMap tma_map_8b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box) {
  return tma_map(base, rank, dims, strides_bytes, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT64);
}

CUtensorMap tma_map_4b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box) {
  return tma_map(base, rank, dims, strides_bytes, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
}

CUtensorMap tma_map_2b(const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                       const uint32_t* box) {
  return tma_map(base, rank, dims, strides_bytes, box, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
}

}  // namespace lt
