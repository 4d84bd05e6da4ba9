// Gaussian random fields on the device: the step before the hot path.
// The reference draws a log-conductivity / log-storativity realisation as mean + C zeta with
// C C^T = Q, Q the dense exponential covariance theta exp(-|x - y| / l) over the element
// centres (sample_field / sample_field_on_mesh, fields.hpp:27-44, fields.cpp:84-123): O(N^3)
// and O(N^2) memory, infeasible beyond ~10^4 points.  On a structured grid the same Gaussian
// law is drawn by circulant embedding: the covariance on a torus twice the grid is
// diagonalised by the DFT, lam = FFT(c) (clipped at 0), and Re IFFT(sqrt(lam) xi) sqrt(M) with
// xi complex standard normals restricted to the grid is a sample with covariance Q.  cuFFT
// (Z2Z, in place) does both transforms; the noise is Philox (curand) or caller-supplied (the
// deterministic path the tests compare with the NumPy restatement, paper_1409_2556_b200/inputs.py).
#include <cufft.h>
#include <curand_kernel.h>

#include <cmath>

#include "lt_internal.hpp"

namespace lt {
namespace {

struct CufftPlan {
  cufftHandle h = 0;
  bool ok = false;
  ~CufftPlan() {
    if (ok) cufftDestroy(h);
  }
};

#define LT_CUFFT(x)                                                                              \
  do {                                                                                           \
    const cufftResult r_ = (x);                                                                  \
    if (r_ != CUFFT_SUCCESS) throw Error(LT_ERR_CUDA, std::string("cuFFT error ") + std::to_string((int)r_) + " at " #x); \
  } while (0)

// c[a] = var exp(-|lag / l|) on the extended torus (x fastest), lag = min(i, e - i) h per axis
__global__ void grf_covariance(int64_t total, int ex, int ey, double h, double ilx, double ily, double ilz,
                               double var, double2* __restrict__ c) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= total) return;
  const int i = (int)(a % ex), j = (int)((a / ex) % ey);
  const int64_t k = a / ((int64_t)ex * ey);
  const int64_t ez = total / ((int64_t)ex * ey);
  const double dx = (double)min(i, ex - i) * h * ilx, dy = (double)min(j, ey - j) * h * ily;
  const double dz = (double)(k < ez - k ? k : ez - k) * h * ilz;
  c[a] = make_double2(var * exp(-sqrt(dx * dx + dy * dy + dz * dz)), 0.0);
}

// w[a] = sqrt(max(Re lam[a], 0)) xi[a] / sqrt(M)   (numpy: ifftn(.) sqrt(M) = IDFT(.) / sqrt(M))
__global__ void grf_scale(int64_t total, double inv_sqrt_m, const double2* __restrict__ noise,
                          unsigned long long seed, double2* __restrict__ w) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= total) return;
  double2 xi;
  if (noise) {
    xi = noise[a];
  } else {
    curandStatePhilox4_32_10_t st;
    curand_init(seed, (unsigned long long)a, 0ULL, &st);
    xi = curand_normal2_double(&st);
  }
  const double s = sqrt(fmax(w[a].x, 0.0)) * inv_sqrt_m;
  w[a] = make_double2(s * xi.x, s * xi.y);
}

__global__ void grf_extract(int64_t n, int nx, int ny, int ex, int ey, double mean, const double2* __restrict__ f,
                            double* __restrict__ out) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int i = (int)(a % nx), j = (int)((a / nx) % ny);
  const int64_t k = a / ((int64_t)nx * ny);
  out[a] = mean + f[(k * ey + j) * ex + i].x;
}

}  // namespace

void sample_field_grid(lt_ctx ctx, int dim, const int* shape, double h, double variance, const double* corr,
                       double mean, uint64_t seed, const double2* noise, int mem, double* out) {
  LT_REQUIRE(ctx != nullptr, "sample_field_grid: null context");
  LT_REQUIRE(dim == 2 || dim == 3, "sample_field_grid: dim must be 2 or 3");
  LT_REQUIRE(shape && corr && out, "sample_field_grid: null argument");
  LT_REQUIRE(mem == LT_MEM_HOST || mem == LT_MEM_DEVICE, "sample_field_grid: bad mem flag");
  LT_REQUIRE(h > 0.0 && variance >= 0.0, "sample_field_grid: h must be positive, variance non-negative");
  for (int d = 0; d < dim; ++d)
    LT_REQUIRE(shape[d] >= 1 && corr[d] > 0.0, "sample_field_grid: shape >= 1 and correlation lengths > 0");
  cudaStream_t st = ctx->stream;
  const int nx = shape[0], ny = shape[1], nz = dim == 3 ? shape[2] : 1;
  const int ex = 2 * nx, ey = 2 * ny, ez = dim == 3 ? 2 * nz : 1;
  const int64_t total = (int64_t)ex * ey * ez, n = (int64_t)nx * ny * nz;
  DeviceBuffer w(sizeof(double2) * (size_t)total, st);
  const unsigned g = (unsigned)((total + 255) / 256);
  launch(ctx, "fields", 16.0 * total, [&] {
    grf_covariance<<<g, 256, 0, st>>>(total, ex, ey, h, 1.0 / corr[0], 1.0 / corr[1], dim == 3 ? 1.0 / corr[2] : 0.0,
                                       variance, w.as<double2>());
  });
  CufftPlan plan;
  if (dim == 3)
    LT_CUFFT(cufftPlan3d(&plan.h, ez, ey, ex, CUFFT_Z2Z));  // last dimension fastest
  else
    LT_CUFFT(cufftPlan2d(&plan.h, ey, ex, CUFFT_Z2Z));
  plan.ok = true;
  LT_CUFFT(cufftSetStream(plan.h, st));
  auto* wc = reinterpret_cast<cufftDoubleComplex*>(w.get());
  LT_CUFFT(cufftExecZ2Z(plan.h, wc, wc, CUFFT_FORWARD));  // lam = DFT(c), real for the even c
  DeviceBuffer dnoise;
  const double2* np = noise;
  if (noise && mem == LT_MEM_HOST) {
    dnoise.allocate(sizeof(double2) * (size_t)total, st);
    LT_CUDA(cudaMemcpyAsync(dnoise.get(), noise, sizeof(double2) * (size_t)total, cudaMemcpyHostToDevice, st));
    np = dnoise.as<double2>();
  }
  launch(ctx, "fields", 32.0 * total, [&] {
    grf_scale<<<g, 256, 0, st>>>(total, 1.0 / std::sqrt((double)total), np, (unsigned long long)seed, w.as<double2>());
  });
  LT_CUFFT(cufftExecZ2Z(plan.h, wc, wc, CUFFT_INVERSE));  // unnormalised: IDFT
  DeviceBuffer dout;
  double* o = out;
  if (mem == LT_MEM_HOST) {
    dout.allocate(sizeof(double) * (size_t)n, st);
    o = dout.as<double>();
  }
  launch(ctx, "fields", 24.0 * n, [&] {
    grf_extract<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, nx, ny, ex, ey, mean, w.as<double2>(), o);
  });
  if (mem == LT_MEM_HOST) LT_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace lt
