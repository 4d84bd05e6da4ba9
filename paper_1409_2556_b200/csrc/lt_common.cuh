// Common device/host helpers for the laptomo B200 library: complex128 arithmetic on
// double2, error plumbing, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "laptomo_gpu.h"

namespace lt {

// ---- complex128 on double2 ------------------------------------------------------------
__host__ __device__ __forceinline__ double2 cmk(double re, double im) { return make_double2(re, im); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// a + b * c
__host__ __device__ __forceinline__ double2 cfma(double2 b, double2 c, double2 a) {
  return make_double2(fma(b.x, c.x, fma(-b.y, c.y, a.x)), fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
__host__ __device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm (robust scaling)
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  } else {
    double r = b.x / b.y, d = b.y + b.x * r;
    return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
  }
}
__host__ __device__ __forceinline__ double2 crecip(double2 b) { return cdiv(make_double2(1.0, 0.0), b); }

inline double2 to_d2(lt_complex c) { return make_double2(c.re, c.im); }
inline lt_complex to_lt(double2 c) { return lt_complex{c.x, c.y}; }

// ---- errors ----------------------------------------------------------------------------
struct Error : std::runtime_error {
  lt_status code;
  Error(lt_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

#define LT_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t err__ = (call);                                                          \
    if (err__ != cudaSuccess) {                                                          \
      throw ::lt::Error(err__ == cudaErrorMemoryAllocation ? LT_ERR_OOM : LT_ERR_CUDA,   \
                        std::string(#call) + ": " + cudaGetErrorString(err__));          \
    }                                                                                    \
  } while (0)

#define LT_REQUIRE(cond, msg)                                             \
  do {                                                                    \
    if (!(cond)) throw ::lt::Error(LT_ERR_INVALID_ARGUMENT, (msg));       \
  } while (0)

inline void check_launch(const char* name) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) throw Error(LT_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(err));
}

constexpr int kThreads = 256;

// Block -> (item, cell block) for batched kernels launched with B * blocks_per_item blocks.
// Default: the item index is fastest, so the blocks of all items that touch one cell block
// run together and share its face coefficients in L2; -DLT_CELL_FAST makes the cell blocks
// of one item consecutive instead.
#ifdef LT_CELL_FAST
#define LT_ITEM_BLOCK(B, b, cb)                            \
  const int b = (int)(blockIdx.x / (gridDim.x / (B)));     \
  const int cb = (int)(blockIdx.x % (gridDim.x / (B)));
#else
#define LT_ITEM_BLOCK(B, b, cb)         \
  const int b = (int)(blockIdx.x % (B)); \
  const int cb = (int)(blockIdx.x / (B));
#endif

inline unsigned blocks_for(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

}  // namespace lt
