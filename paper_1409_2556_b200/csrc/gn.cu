// The Gauss-Newton step of the geostatistical inversion on the device (
// GaussNewtonSolver, inversion.hpp:51-79, inversion.cpp:50-186): the consumer of J.
//
//   [J Q J^T + R, J X; (J X)^T, 0] [xi; beta+] = [y - h(s) + J s; 0],  s+ = X beta+ + Q J^T xi,
//   then step halving until the objective misfit(h(s)) + 1/2 (s - X beta)^T Q^{-1} (s - X beta)
//   does not increase.
//
// J (n_y x n_s) stays on the device.  The prior Q is either the reference's dense matrix or --
// the B200 path for the grid-sized parameter vectors of the BASELINE configs, where a dense Q is
// impossible (n_s = 4.2 M at configs[4]) -- a stationary exponential covariance per parameter
// block on the FD grid, applied EXACTLY by FFT (the circulant embedding of the GRF sampler on a
// torus twice the grid, without the clipping the sampler needs: a Toeplitz product, not an
// approximation).  Q J^T: one batched cuFFT convolution per row block; J Q J^T and
// the other plain dense products: cuBLAS DGEMM / DGEMV; the (n_y + p)^2 saddle system: cuSOLVER
// LU (the reference's PartialPivLU); the prior term: Cholesky of the jittered dense Q
// (cuSOLVER, the reference's jittered_cholesky) or, for the grid prior, Q^{-1} by CG on the FFT
// product.  The forward handles are caller callbacks (InversionProblem::predict /
// jacobian_and_predict), e.g. lt_predict / lt_jacobian on a pencil of the trial fields.
#include <cublas_v2.h>
#include <cufft.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "drivers.hpp"
#include "lt_internal.hpp"

namespace lt {
namespace {

#define LT_CUBLAS(x)                                                                                           \
  do {                                                                                                         \
    const cublasStatus_t s_ = (x);                                                                             \
    if (s_ != CUBLAS_STATUS_SUCCESS) throw Error(LT_ERR_CUDA, std::string("cuBLAS error ") + std::to_string((int)s_) + " at " #x); \
  } while (0)
#define LT_CUSOLVER(x)                                                                                         \
  do {                                                                                                         \
    const cusolverStatus_t s_ = (x);                                                                           \
    if (s_ != CUSOLVER_STATUS_SUCCESS) throw Error(LT_ERR_CUDA, std::string("cuSOLVER error ") + std::to_string((int)s_) + " at " #x); \
  } while (0)
#define LT_CUFFT2(x)                                                                                           \
  do {                                                                                                         \
    const cufftResult r_ = (x);                                                                                \
    if (r_ != CUFFT_SUCCESS) throw Error(LT_ERR_CUDA, std::string("cuFFT error ") + std::to_string((int)r_) + " at " #x); \
  } while (0)

struct Handles {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  explicit Handles(cudaStream_t st) {
    LT_CUBLAS(cublasCreate(&blas));
    LT_CUBLAS(cublasSetStream(blas, st));
    LT_CUSOLVER(cusolverDnCreate(&solver));
    LT_CUSOLVER(cusolverDnSetStream(solver, st));
  }
  ~Handles() {
    if (blas) cublasDestroy(blas);
    if (solver) cusolverDnDestroy(solver);
  }
};

// c[a] = var exp(-|lag / l|) on the doubled torus (x fastest; same construction as fields.cu)
__global__ void toeplitz_symbol(int64_t total, int ex, int ey, double h, double ilx, double ily, double ilz, double var,
                                double2* __restrict__ c) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= total) return;
  const int i = (int)(a % ex), j = (int)((a / ex) % ey);
  const int64_t k = a / ((int64_t)ex * ey), ez = total / ((int64_t)ex * ey);
  const double dx = (double)min(i, ex - i) * h * ilx, dy = (double)min(j, ey - j) * h * ily;
  const double dz = (double)(k < ez - k ? k : ez - k) * h * ilz;
  c[a] = make_double2(var * exp(-sqrt(dx * dx + dy * dy + dz * dz)), 0.0);
}

// embed rows: w[r][ext cell] = v[r][cell] (0 elsewhere); v row stride ldv
__global__ void embed_rows(int rows, int64_t n, int nx, int ny, int ex, int ey, int64_t total, const double* __restrict__ v,
                           int64_t ldv, double2* __restrict__ w) {
  const int r = blockIdx.y;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % ex), j = (int)((e / ex) % ey);
    const int64_t k = e / ((int64_t)ex * ey);
    double x = 0.0;
    if (i < nx && j < ny && k < n / ((int64_t)nx * ny)) x = v[(int64_t)r * ldv + (k * ny + j) * nx + i];
    w[(int64_t)r * total + e] = make_double2(x, 0.0);
  }
}

// w[r] *= lam / total (lam real)
__global__ void symbol_scale(int rows, int64_t total, const double2* __restrict__ lam, double2* __restrict__ w) {
  const int r = blockIdx.y;
  const double inv = 1.0 / (double)total;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const double s = lam[e].x * inv;
    double2 x = w[(int64_t)r * total + e];
    w[(int64_t)r * total + e] = make_double2(x.x * s, x.y * s);
  }
}

__global__ void extract_rows(int rows, int64_t n, int nx, int ny, int ex, int ey, int64_t total, const double2* __restrict__ w,
                             double* __restrict__ out, int64_t ldo) {
  const int r = blockIdx.y;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(a % nx), j = (int)((a / nx) % ny);
    const int64_t k = a / ((int64_t)nx * ny);
    out[(int64_t)r * ldo + a] = w[(int64_t)r * total + (k * ey + j) * ex + i].x;
  }
}

__global__ void add_diag(int n, int ld, const double* __restrict__ d, double* __restrict__ A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[(int64_t)i * ld + i] += d[i];
}

// The stationary grid prior: y = Q x for rows of length n_s (n_blocks blocks of n cells),
// exactly, by batched FFT on the doubled torus.
class GridPrior {
 public:
  GridPrior(lt_ctx ctx, const lt_gn_problem& pb) : ctx_(ctx) {
    const lt_grid& g = pb.grid;
    LT_REQUIRE(g.kind == LT_GRID_FD_CELL && (g.dim == 2 || g.dim == 3), "gauss_newton: grid prior on an FD grid");
    LT_REQUIRE(pb.n_blocks == 1 || pb.n_blocks == 2, "gauss_newton: one or two parameter blocks");
    dim_ = g.dim;
    nx_ = g.shape[0];
    ny_ = g.shape[1];
    nz_ = g.dim == 3 ? g.shape[2] : 1;
    n_ = (int64_t)nx_ * ny_ * nz_;
    LT_REQUIRE(n_ * pb.n_blocks == pb.n_s, "gauss_newton: n_s must equal n_blocks x grid cells");
    ex_ = 2 * nx_;
    ey_ = 2 * ny_;
    ez_ = dim_ == 3 ? 2 * nz_ : 1;
    total_ = (int64_t)ex_ * ey_ * ez_;
    blocks_ = pb.n_blocks;
    cudaStream_t st = ctx->stream;
    lam_.allocate(sizeof(double2) * (size_t)total_ * blocks_, st);
    const int n[3] = {ez_, ey_, ex_};
    for (int b = 0; b < blocks_; ++b) {
      LT_REQUIRE(pb.variance[b] >= 0.0 && pb.corr[b][0] > 0.0 && pb.corr[b][1] > 0.0 && (dim_ == 2 || pb.corr[b][2] > 0.0),
                 "gauss_newton: prior variance >= 0 and correlation lengths > 0");
      double2* lam = lam_.as<double2>() + (size_t)b * total_;
      launch(ctx, "gn_prior", 16.0 * total_, [&] {
        toeplitz_symbol<<<(unsigned)((total_ + 255) / 256), 256, 0, st>>>(total_, ex_, ey_, g.h, 1.0 / pb.corr[b][0],
                                                                         1.0 / pb.corr[b][1],
                                                                         dim_ == 3 ? 1.0 / pb.corr[b][2] : 0.0,
                                                                         pb.variance[b], lam);
      });
      cufftHandle one;
      LT_CUFFT2(dim_ == 3 ? cufftPlan3d(&one, n[0], n[1], n[2], CUFFT_Z2Z) : cufftPlan2d(&one, n[1], n[2], CUFFT_Z2Z));
      cufftSetStream(one, st);
      auto* lc = reinterpret_cast<cufftDoubleComplex*>(lam);
      const cufftResult r = cufftExecZ2Z(one, lc, lc, CUFFT_FORWARD);
      cufftDestroy(one);
      LT_CUFFT2(r);
    }
    // rows per batched transform: about 1 GB of complex work space
    batch_ = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (int64_t)(1e9 / (16.0 * total_))));
    work_.allocate(sizeof(double2) * (size_t)total_ * batch_, st);
    LT_CUFFT2(dim_ == 3 ? cufftPlanMany(&plan_, 3, const_cast<int*>(n), nullptr, 1, (int)total_, nullptr, 1, (int)total_,
                                        CUFFT_Z2Z, batch_)
                        : cufftPlanMany(&plan_, 2, const_cast<int*>(n + 1), nullptr, 1, (int)total_, nullptr, 1,
                                        (int)total_, CUFFT_Z2Z, batch_));
    planned_ = true;
    LT_CUFFT2(cufftSetStream(plan_, st));
    LT_CUFFT2(dim_ == 3 ? cufftPlan3d(&plan1_, n[0], n[1], n[2], CUFFT_Z2Z) : cufftPlan2d(&plan1_, n[1], n[2], CUFFT_Z2Z));
    planned1_ = true;
    LT_CUFFT2(cufftSetStream(plan1_, st));
  }
  ~GridPrior() {
    if (planned_) cufftDestroy(plan_);
    if (planned1_) cufftDestroy(plan1_);
  }
  // out[r] = Q in[r] for `rows` rows (row strides ld), device
  void apply(const double* in, int64_t ldi, double* out, int64_t ldo, int rows) {
    cudaStream_t st = ctx_->stream;
    for (int r0 = 0; r0 < rows; r0 += batch_) {
      const int nb = std::min(batch_, rows - r0);
      for (int b = 0; b < blocks_; ++b) {
        const dim3 ge((unsigned)std::min<int64_t>(blocks_for(total_, 256), 4096), (unsigned)nb);
        double2* w = work_.as<double2>();
        launch(ctx_, "gn_prior", 24.0 * total_ * nb, [&] {
          embed_rows<<<ge, 256, 0, st>>>(nb, n_, nx_, ny_, ex_, ey_, total_, in + (int64_t)r0 * ldi + b * n_, ldi, w);
        });
        auto* wc = reinterpret_cast<cufftDoubleComplex*>(w);
        // one row (the CG of the prior term): the single plan; else the batched plan (rows past
        // nb of a last partial batch are transformed too and ignored)
        const cufftHandle pl = nb == 1 ? plan1_ : plan_;
        LT_CUFFT2(cufftExecZ2Z(pl, wc, wc, CUFFT_FORWARD));
        launch(ctx_, "gn_prior", 48.0 * total_ * nb, [&] {
          symbol_scale<<<ge, 256, 0, st>>>(nb, total_, lam_.as<double2>() + (size_t)b * total_, w);
        });
        LT_CUFFT2(cufftExecZ2Z(pl, wc, wc, CUFFT_INVERSE));
        const dim3 gx((unsigned)std::min<int64_t>(blocks_for(n_, 256), 4096), (unsigned)nb);
        launch(ctx_, "gn_prior", 24.0 * n_ * nb, [&] {
          extract_rows<<<gx, 256, 0, st>>>(nb, n_, nx_, ny_, ex_, ey_, total_, w, out + (int64_t)r0 * ldo + b * n_, ldo);
        });
      }
    }
  }

 private:
  lt_ctx ctx_;
  int dim_, nx_, ny_, nz_, ex_, ey_, ez_, blocks_, batch_ = 1;
  int64_t n_, total_;
  DeviceBuffer lam_, work_;
  cufftHandle plan_{}, plan1_{};
  bool planned_ = false, planned1_ = false;
};

double dot_host(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

}  // namespace

// The solver state of one problem: the prior (dense + Cholesky, or the grid FFT operator),
// cuBLAS / cuSOLVER handles, device copies of y, R, X.
struct GnSolver {
  lt_ctx ctx;
  lt_gn_problem pb;
  Handles h;
  std::unique_ptr<GridPrior> grid;
  DeviceBuffer Q, L;  // dense prior and its lower Cholesky factor (column-major)
  DeviceBuffer X;     // n_s x p column-major

  GnSolver(lt_ctx c, const lt_gn_problem& problem) : ctx(c), pb(problem), h(c->stream) {
    cudaStream_t st = ctx->stream;
    LT_REQUIRE(pb.n_y >= 1 && pb.n_s >= 1 && pb.p >= 0, "InversionProblem: empty problem");
    LT_REQUIRE(pb.y && pb.r_diag && (pb.p == 0 || pb.drift), "InversionProblem: missing y, R or X");
    for (int i = 0; i < pb.n_y; ++i) LT_REQUIRE(pb.r_diag[i] > 0.0, "InversionProblem: R diagonal must be positive");
    LT_REQUIRE(pb.predict && pb.jacobian_and_predict, "InversionProblem: missing forward handles");
    if (pb.p > 0) {
      X.allocate(sizeof(double) * (size_t)pb.n_s * pb.p, st);
      LT_CUDA(cudaMemcpyAsync(X.get(), pb.drift, X.bytes(), cudaMemcpyHostToDevice, st));
    }
    if (pb.prior) {
      const int64_t ns = pb.n_s;
      Q.allocate(sizeof(double) * (size_t)ns * ns, st);
      LT_CUDA(cudaMemcpyAsync(Q.get(), pb.prior, Q.bytes(), cudaMemcpyHostToDevice, st));
      jittered_cholesky();
    } else {
      grid = std::make_unique<GridPrior>(ctx, pb);
    }
  }

  // inversion.cpp:17-33 on the device (cuSOLVER potrf with 1e-10 max-diag jitter, doubled)
  void jittered_cholesky() {
    cudaStream_t st = ctx->stream;
    const int n = pb.n_s;
    std::vector<double> diag(n);
    for (int i = 0; i < n; ++i) diag[i] = pb.prior[(size_t)i * n + i];
    const double scale = *std::max_element(diag.begin(), diag.end());
    double jitter = 1e-10 * scale;
    L.allocate(Q.bytes(), st);
    int lwork = 0;
    LT_CUSOLVER(cusolverDnDpotrf_bufferSize(h.solver, CUBLAS_FILL_MODE_LOWER, n, L.as<double>(), n, &lwork));
    DeviceBuffer work(sizeof(double) * std::max(lwork, 1), st), info(sizeof(int), st);
    DeviceBuffer dj(sizeof(double) * n, st);
    for (int attempt = 0; attempt <= 6; ++attempt) {
      LT_CUDA(cudaMemcpyAsync(L.get(), Q.get(), Q.bytes(), cudaMemcpyDeviceToDevice, st));
      if (attempt > 0) {
        std::vector<double> jv(n, jitter);
        LT_CUDA(cudaMemcpyAsync(dj.get(), jv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
        add_diag<<<blocks_for(n, 256), 256, 0, st>>>(n, n, dj.as<double>(), L.as<double>());
        jitter *= 2.0;
      }
      LT_CUSOLVER(cusolverDnDpotrf(h.solver, CUBLAS_FILL_MODE_LOWER, n, L.as<double>(), n, work.as<double>(), lwork,
                                   info.as<int>()));
      int hinfo = 0;
      LT_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
      LT_CUDA(cudaStreamSynchronize(st));
      if (hinfo == 0) return;
    }
    throw Error(LT_ERR_PRECONDITIONER, "GaussNewtonSolver: prior Cholesky failed after max jitter");
  }

  // out = Q in for rows of length n_s (row-major, device)
  void prior_apply(const double* in, double* out, int rows) {
    if (grid) {
      grid->apply(in, pb.n_s, out, pb.n_s, rows);
      return;
    }
    // row-major rows R (rows x n_s) = column-major R^T; Q R^T (Q symmetric) = (R Q)^T
    const double one = 1.0, zero = 0.0;
    LT_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, pb.n_s, rows, pb.n_s, &one, Q.as<double>(), pb.n_s, in,
                          pb.n_s, &zero, out, pb.n_s));
  }

  // 1/2 a^T Q^{-1} a, a = s - X beta (inversion.cpp:63-69: ||L^{-1} a||^2 / 2)
  double prior_term(const std::vector<double>& s, const std::vector<double>& beta) {
    cudaStream_t st = ctx->stream;
    const int n = pb.n_s;
    std::vector<double> a(s);
    for (int k = 0; k < pb.p; ++k)
      for (int i = 0; i < n; ++i) a[i] -= pb.drift[(size_t)k * n + i] * beta[k];
    DeviceBuffer da(sizeof(double) * n, st);
    LT_CUDA(cudaMemcpyAsync(da.get(), a.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    if (!grid) {
      LT_CUBLAS(cublasDtrsv(h.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, L.as<double>(), n,
                            da.as<double>(), 1));
      double nrm = 0.0;
      LT_CUBLAS(cublasDnrm2(h.blas, n, da.as<double>(), 1, &nrm));
      return 0.5 * nrm * nrm;
    }
    // grid prior: w = Q^{-1} a by CG on the exact FFT product, 1/2 a^T w
    DeviceBuffer vec(sizeof(double) * (size_t)n * 4, st);
    double* w = vec.as<double>();
    double* r = w + n;
    double* p = r + n;
    double* q = p + n;
    LT_CUDA(cudaMemsetAsync(w, 0, sizeof(double) * n, st));
    LT_CUDA(cudaMemcpyAsync(r, da.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    LT_CUDA(cudaMemcpyAsync(p, da.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    double rr = 0.0, bb = 0.0;
    LT_CUBLAS(cublasDdot(h.blas, n, r, 1, r, 1, &rr));
    bb = rr;
    if (!(bb > 0.0)) return 0.0;
    for (int it = 0; it < 20000 && rr > 1e-26 * bb; ++it) {
      grid->apply(p, n, q, n, 1);
      double pq = 0.0;
      LT_CUBLAS(cublasDdot(h.blas, n, p, 1, q, 1, &pq));
      const double alpha = rr / pq, malpha = -alpha;
      LT_CUBLAS(cublasDaxpy(h.blas, n, &alpha, p, 1, w, 1));
      LT_CUBLAS(cublasDaxpy(h.blas, n, &malpha, q, 1, r, 1));
      double rr_new = 0.0;
      LT_CUBLAS(cublasDdot(h.blas, n, r, 1, r, 1, &rr_new));
      const double beta_cg = rr_new / rr, one = 1.0;
      LT_CUBLAS(cublasDscal(h.blas, n, &beta_cg, p, 1));
      LT_CUBLAS(cublasDaxpy(h.blas, n, &one, r, 1, p, 1));
      rr = rr_new;
    }
    if (!(rr <= 1e-20 * bb))
      throw Error(LT_ERR_PRECONDITIONER, "GaussNewtonSolver: prior solve (CG on the grid covariance) did not converge");
    double aw = 0.0;
    LT_CUBLAS(cublasDdot(h.blas, n, da.as<double>(), 1, w, 1, &aw));
    return 0.5 * aw;
  }

  double misfit(const std::vector<double>& pred) const {
    double m = 0.0;
    for (int i = 0; i < pb.n_y; ++i) {
      const double r = pb.y[i] - pred[i];
      m += r * r / pb.r_diag[i];
    }
    return 0.5 * m;
  }

  std::vector<double> predict(const std::vector<double>& s) {
    std::vector<double> out(pb.n_y);
    const int st = pb.predict(pb.user, s.data(), out.data());
    if (st != 0) throw Error((lt_status)st, "InversionProblem::predict failed");
    return out;
  }

  double objective(const std::vector<double>& s, const std::vector<double>& beta) {
    return misfit(predict(s)) + prior_term(s, beta);
  }

  // inversion.cpp:78-148
  void step(const std::vector<double>& s, const std::vector<double>& beta, const lt_gn_options& opt,
            std::vector<double>& s_out, std::vector<double>& beta_out, std::vector<double>& xi_out, lt_gn_stats& stats) {
    cudaStream_t st = ctx->stream;
    const int ny = pb.n_y, ns = pb.n_s, p = pb.p, N = ny + p;
    DeviceBuffer J(sizeof(double) * (size_t)ny * ns, st);
    std::vector<double> pred(ny);
    LT_CUDA(cudaStreamSynchronize(st));
    {
      const int rc = pb.jacobian_and_predict(pb.user, s.data(), J.as<double>(), pred.data());
      if (rc != 0) throw Error((lt_status)rc, "InversionProblem::jacobian_and_predict failed");
    }
    const double one = 1.0, zero = 0.0;
    // JQ (row-major n_y x n_s) and JX (row-major n_y x p)
    DeviceBuffer JQ(sizeof(double) * (size_t)ny * ns, st);
    prior_apply(J.as<double>(), JQ.as<double>(), ny);
    DeviceBuffer JX(sizeof(double) * (size_t)std::max(ny * p, 1), st);
    if (p > 0)
      LT_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, p, ny, ns, &one, X.as<double>(), ns, J.as<double>(), ns,
                            &zero, JX.as<double>(), p));  // column-major p x n_y = row-major n_y x p
    // saddle (column-major N x N): [JQJ^T + R, JX; JX^T, 0]
    DeviceBuffer S(sizeof(double) * (size_t)N * N, st);
    LT_CUDA(cudaMemsetAsync(S.get(), 0, S.bytes(), st));
    LT_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_T, CUBLAS_OP_N, ny, ny, ns, &one, JQ.as<double>(), ns, J.as<double>(), ns, &zero,
                          S.as<double>(), N));
    DeviceBuffer dr(sizeof(double) * ny, st);
    LT_CUDA(cudaMemcpyAsync(dr.get(), pb.r_diag, sizeof(double) * ny, cudaMemcpyHostToDevice, st));
    add_diag<<<blocks_for(ny, 256), 256, 0, st>>>(ny, N, dr.as<double>(), S.as<double>());
    std::vector<double> jx((size_t)ny * p);
    if (p > 0) {
      LT_CUDA(cudaMemcpyAsync(jx.data(), JX.get(), sizeof(double) * jx.size(), cudaMemcpyDeviceToHost, st));
    }
    LT_CUDA(cudaStreamSynchronize(st));
    std::vector<double> Sh((size_t)N * N);
    LT_CUDA(cudaMemcpy(Sh.data(), S.get(), S.bytes(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < ny; ++i)
      for (int k = 0; k < p; ++k) {
        Sh[(size_t)(ny + k) * N + i] = jx[(size_t)i * p + k];  // (i, ny + k)
        Sh[(size_t)i * N + ny + k] = jx[(size_t)i * p + k];    // (ny + k, i)
      }
    // rhs = [y - h + J s; 0]
    DeviceBuffer ds(sizeof(double) * ns, st), djs(sizeof(double) * ny, st);
    LT_CUDA(cudaMemcpyAsync(ds.get(), s.data(), sizeof(double) * ns, cudaMemcpyHostToDevice, st));
    LT_CUBLAS(cublasDgemv(h.blas, CUBLAS_OP_T, ns, ny, &one, J.as<double>(), ns, ds.as<double>(), 1, &zero, djs.as<double>(), 1));
    std::vector<double> js(ny), rhs(N, 0.0);
    LT_CUDA(cudaMemcpyAsync(js.data(), djs.get(), sizeof(double) * ny, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < ny; ++i) rhs[i] = pb.y[i] - pred[i] + js[i];
    // PartialPivLU of the saddle (cuSOLVER getrf / getrs)
    DeviceBuffer dS(sizeof(double) * (size_t)N * N, st), dsol(sizeof(double) * N, st), ipiv(sizeof(int) * N, st),
        info(sizeof(int), st);
    LT_CUDA(cudaMemcpyAsync(dS.get(), Sh.data(), dS.bytes(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dsol.get(), rhs.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
    int lwork = 0;
    LT_CUSOLVER(cusolverDnDgetrf_bufferSize(h.solver, N, N, dS.as<double>(), N, &lwork));
    DeviceBuffer work(sizeof(double) * std::max(lwork, 1), st);
    LT_CUSOLVER(cusolverDnDgetrf(h.solver, N, N, dS.as<double>(), N, work.as<double>(), ipiv.as<int>(), info.as<int>()));
    LT_CUSOLVER(cusolverDnDgetrs(h.solver, CUBLAS_OP_N, N, 1, dS.as<double>(), N, ipiv.as<int>(), dsol.as<double>(), N,
                                 info.as<int>()));
    std::vector<double> sol(N);
    LT_CUDA(cudaMemcpyAsync(sol.data(), dsol.get(), sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    for (double v : sol)
      if (!std::isfinite(v))
        throw Error(LT_ERR_PRECONDITIONER,
                    "gauss_newton_step: saddle system solve failed (rank-deficient J Q J^T + R or J X block)");
    xi_out.assign(sol.begin(), sol.begin() + ny);
    std::vector<double> beta_new(sol.begin() + ny, sol.end());
    // diagnostics (inversion.cpp:107-111)
    {
      double num = 0.0, den = 0.0;
      for (int i = 0; i < N; ++i) {
        double acc = 0.0;
        for (int j = 0; j < N; ++j) acc += Sh[(size_t)j * N + i] * sol[j];
        num += (acc - rhs[i]) * (acc - rhs[i]);
        den += rhs[i] * rhs[i];
      }
      stats.saddle_residual = std::sqrt(num) / std::sqrt(den);
      double xn = 0.0;
      for (int i = 0; i < ny; ++i) xn += xi_out[i] * xi_out[i];
      xn = std::sqrt(xn);
      double dv = 0.0;
      for (int k = 0; k < p; ++k) {
        double acc = 0.0;
        for (int i = 0; i < ny; ++i) acc += jx[(size_t)i * p + k] * xi_out[i];
        dv += acc * acc;
      }
      stats.drift_violation = p > 0 && xn > 0.0 ? std::sqrt(dv) / xn : 0.0;
    }
    // s_full = X beta+ + (JQ)^T xi
    DeviceBuffer dxi(sizeof(double) * ny, st), dsf(sizeof(double) * ns, st);
    LT_CUDA(cudaMemcpyAsync(dxi.get(), xi_out.data(), sizeof(double) * ny, cudaMemcpyHostToDevice, st));
    LT_CUBLAS(cublasDgemv(h.blas, CUBLAS_OP_N, ns, ny, &one, JQ.as<double>(), ns, dxi.as<double>(), 1, &zero,
                          dsf.as<double>(), 1));
    std::vector<double> s_full(ns);
    LT_CUDA(cudaMemcpyAsync(s_full.data(), dsf.get(), sizeof(double) * ns, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < p; ++k)
      for (int i = 0; i < ns; ++i) s_full[i] += pb.drift[(size_t)k * ns + i] * beta_new[k];
    J.release();
    JQ.release();
    const double objective_old = misfit(pred) + prior_term(s, beta);
    double alpha = 1.0;
    bool accepted = false;
    const int halvings = opt.damping ? opt.max_halvings : 0;
    std::vector<double> s_trial(ns), b_trial(p);
    for (int hv = 0; hv <= halvings; ++hv) {
      for (int i = 0; i < ns; ++i) s_trial[i] = s[i] + alpha * (s_full[i] - s[i]);
      for (int k = 0; k < p; ++k) b_trial[k] = beta[k] + alpha * (beta_new[k] - beta[k]);
      const std::vector<double> hp = predict(s_trial);
      const double mis = misfit(hp);
      const double obj = mis + prior_term(s_trial, b_trial);
      if (obj <= objective_old || !opt.damping) {
        s_out = s_trial;
        beta_out = b_trial;
        stats.objective = obj;
        stats.misfit = mis;  // the reference re-predicts s_trial: the same deterministic value
        stats.prior = obj - mis;
        stats.alpha = alpha;
        accepted = true;
        break;
      }
      alpha *= 0.5;
    }
    if (!accepted) {
      s_out = s;
      beta_out = beta;
      stats.objective = objective_old;
      stats.misfit = misfit(pred);
      stats.prior = objective_old - stats.misfit;
      stats.alpha = 0.0;
    }
    double sn = 0.0;
    for (int i = 0; i < ns; ++i) sn += (s_out[i] - s[i]) * (s_out[i] - s[i]);
    stats.step_norm = std::sqrt(sn);
  }
};

void gn_step(lt_ctx ctx, const lt_gn_problem& pb, const double* s, const double* beta, const lt_gn_options& opt,
             double* s_out, double* beta_out, double* xi_out, lt_gn_stats* stats) {
  GnSolver g(ctx, pb);
  std::vector<double> sv(s, s + pb.n_s), bv(beta, beta + pb.p), so, bo, xo;
  lt_gn_stats stt{};
  g.step(sv, bv, opt, so, bo, xo, stt);
  std::copy(so.begin(), so.end(), s_out);
  std::copy(bo.begin(), bo.end(), beta_out);
  if (xi_out) std::copy(xo.begin(), xo.end(), xi_out);
  if (stats) *stats = stt;
}

int gn_invert(lt_ctx ctx, const lt_gn_problem& pb, const double* s0, const double* beta0, const lt_gn_options& opt,
              double* s_hat, double* beta_hat, lt_gn_stats* history, int history_cap, int* converged, char* reason,
              int reason_cap) {
  LT_REQUIRE(opt.max_gn >= 1, "invert: max_gn must be at least 1");
  GnSolver g(ctx, pb);
  std::vector<double> s(s0, s0 + pb.n_s), beta(beta0, beta0 + pb.p);
  double objective_prev = g.objective(s, beta);
  std::string stop;
  bool conv = false;
  int k = 0;
  for (; k < opt.max_gn; ++k) {
    std::vector<double> so, bo, xo;
    lt_gn_stats st{};
    g.step(s, beta, opt, so, bo, xo, st);
    s = so;
    beta = bo;
    if (history && k < history_cap) history[k] = st;
    if (st.alpha == 0.0) {
      stop = "step stalled: damping could not decrease the objective";
      ++k;
      break;
    }
    double sn = 0.0;
    for (double v : s) sn += v * v;
    const double rel_step = st.step_norm / std::max(std::sqrt(sn), 1e-300);
    const double rel_decrease = (objective_prev - st.objective) / std::max(std::fabs(objective_prev), 1e-300);
    objective_prev = st.objective;
    if (rel_step <= opt.rtol) {
      conv = true;
      stop = "relative step norm below rtol";
      ++k;
      break;
    }
    if (rel_decrease >= 0.0 && rel_decrease <= opt.rtol) {
      conv = true;
      stop = "relative objective decrease below rtol";
      ++k;
      break;
    }
  }
  if (stop.empty()) stop = "max_gn reached";
  std::copy(s.begin(), s.end(), s_hat);
  std::copy(beta.begin(), beta.end(), beta_hat);
  if (converged) *converged = conv ? 1 : 0;
  if (reason && reason_cap > 0) {
    const size_t m = std::min<size_t>(stop.size(), (size_t)reason_cap - 1);
    std::copy(stop.begin(), stop.begin() + m, reason);
    reason[m] = '\0';
  }
  return k;
}

double gn_objective(lt_ctx ctx, const lt_gn_problem& pb, const double* s, const double* beta, double* misfit,
                    double* prior) {
  GnSolver g(ctx, pb);
  std::vector<double> sv(s, s + pb.n_s), bv(beta, beta + pb.p);
  const double mis = g.misfit(g.predict(sv)), pr = g.prior_term(sv, bv);
  if (misfit) *misfit = mis;
  if (prior) *prior = pr;
  return mis + pr;
}

}  // namespace lt
