// Exact banded shift-and-invert for 2-D pencils: the fallback of the inner solve when the
// multigrid-preconditioned COCG cannot reach its tolerance.
//
// The reference factors K + tau M exactly (SparseLU, factorization.cpp:14-33).  Here the inner
// solve is MG-preconditioned COCG, which is robust while K + tau M stays close to definite --
// every BASELINE config -- but not for strongly indefinite shifts (Re tau far below the
// pencil's smallest eigenvalues: the paper's own 100 m experiments at t = 1 min, where a
// smoothing-based V-cycle cannot represent the many oscillatory negative modes).  For those
// shifts a 2-D grid pencil (natural ordering: bandwidth nx (FD 5-point) or nx + 1 (P1, the
// NE/SW couplings)) is factored exactly as a band matrix with partial pivoting (LAPACK zgbtrf
// layout and algorithm) on the device, cached by exact tau like the reference's factorisation
// cache (shifted_solver.cpp:120-128), and applied by banded forward / back substitution, one
// warp per right-hand side.
#include <algorithm>
#include <cmath>
#include <string>

#include "lt_internal.hpp"

namespace lt {
namespace {

constexpr int kF = 1024;  // factorisation: one CTA

__device__ __forceinline__ double cabs1(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// A(i, j) at AB[(kv + i - j) + j ldab], kv = kl + ku (the top kl rows hold the pivoting fill)
__global__ void band_assemble(LevelView L, int p1, double2 tau, int kl, int ku, int ldab, double2* __restrict__ AB) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= L.n) return;
  const int kv = kl + ku;
  const int i = (int)(a % L.nx), j = (int)(a / L.nx);
  const int64_t ex = (int64_t)j * (L.nx + 1) + i, ey = (int64_t)j * L.nx + i;
  const double tw = L.Tx[ex], te = L.Tx[ex + 1], ts = L.Ty[ey], tn = L.Ty[ey + L.nx];
  auto put = [&](int64_t col, double2 v) { AB[(kv + a - col) + col * (int64_t)ldab] = v; };
  const double m = L.M[a];
  put(a, make_double2(tw + te + ts + tn + tau.x * m, tau.y * m));
  auto off = [&](double t, double mc) { return make_double2(-t + tau.x * mc, tau.y * mc); };
  if (i > 0) put(a - 1, off(tw, p1 ? L.Mx[ex] : 0.0));
  if (i < L.nx - 1) put(a + 1, off(te, p1 ? L.Mx[ex + 1] : 0.0));
  if (j > 0) put(a - L.nx, off(ts, p1 ? L.My[ey] : 0.0));
  if (j < L.ny - 1) put(a + L.nx, off(tn, p1 ? L.My[ey + L.nx] : 0.0));
  if (p1) {
    if (i < L.nx - 1 && j < L.ny - 1) put(a + L.nx + 1, off(0.0, L.Md[a]));
    if (i > 0 && j > 0) put(a - L.nx - 1, off(0.0, L.Md[a - L.nx - 1]));
  }
}

// zgbtf2: unblocked banded LU with partial pivoting, one CTA
__global__ void __launch_bounds__(kF) band_factor(int64_t n, int kl, int ku, int ldab, double2* __restrict__ AB,
                                                 int* __restrict__ ipiv, int* __restrict__ info) {
  __shared__ double sv[kF / 32];
  __shared__ int si[kF / 32];
  __shared__ int s_jp;
  __shared__ int64_t s_ju;
  const int kv = kl + ku;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_ju = 0;
  for (int64_t j = 0; j < n; ++j) {
    const int km = (int)imin(kl, n - 1 - j);
    double2* col = AB + j * (int64_t)ldab + kv;  // col[r] = A(j + r, j)
    // pivot: first max |A(j + r, j)|, r <= km
    double best = -1.0;
    int bi = 0;
    for (int r = tid; r <= km; r += kF) {
      const double v = cabs1(col[r]);
      if (v > best) { best = v; bi = r; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffff, best, o);
      const int oi = __shfl_down_sync(0xffffffff, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { sv[w] = best; si[w] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b0 = sv[0];
      int i0 = si[0];
      for (int q = 1; q < kF / 32; ++q)
        if (sv[q] > b0 || (sv[q] == b0 && si[q] < i0)) { b0 = sv[q]; i0 = si[q]; }
      s_jp = i0;
      ipiv[j] = (int)(j + i0);
      if (!(b0 > 0.0)) *info = (int)(j + 1);
      else s_ju = imax(s_ju, imin(j + ku + i0, n - 1));
    }
    __syncthreads();
    const int jp = s_jp;
    const int64_t ju = s_ju;
    if (cabs1(col[jp]) == 0.0) continue;  // singular column (info set); the reference throws
    const int64_t ncols = ju - j + 1;     // columns j .. ju take part in the interchange
    if (jp != 0) {
      for (int64_t c = tid; c < ncols; c += kF) {
        double2* cc = AB + (j + c) * (int64_t)ldab + kv - c;  // cc[r] = A(j + r, j + c)
        const double2 t = cc[0];
        cc[0] = cc[jp];
        cc[jp] = t;
      }
      __syncthreads();
    }
    const double2 piv = col[0];
    const double2 rp = crecip(piv);
    for (int r = 1 + tid; r <= km; r += kF) col[r] = cmul(col[r], rp);
    __syncthreads();
    // rank-1 update of the trailing band block: A(j + r, j + c) -= l_r A(j, j + c)
    const int64_t work = (int64_t)km * (ncols - 1);
    for (int64_t e = tid; e < work; e += kF) {
      const int r = 1 + (int)(e % km);
      const int64_t c = 1 + e / km;
      double2* cc = AB + (j + c) * (int64_t)ldab + kv - c;
      cc[r] = csub(cc[r], cmul(col[r], cc[0]));
    }
    __syncthreads();
  }
}

// zgbtrs (no transpose), one warp per right-hand side: u = A^{-1} v
__global__ void band_solve(int64_t n, int kl, int ku, int ldab, const double2* __restrict__ AB,
                           const int* __restrict__ ipiv, const double2* __restrict__ v, int64_t vs,
                           double2* __restrict__ u, int64_t us, int B) {
  const int b = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const int kv = kl + ku;
  double2* x = u + (int64_t)b * us;
  for (int64_t a = lane; a < n; a += 32) x[a] = v[(int64_t)b * vs + a];
  __syncwarp();
  // L: interchanges and unit lower band
  for (int64_t j = 0; j < n - 1; ++j) {
    const int km = (int)imin(kl, n - 1 - j);
    const int l = ipiv[j];
    if (l != j && lane == 0) {
      const double2 t = x[l];
      x[l] = x[j];
      x[j] = t;
    }
    __syncwarp();
    const double2 xj = x[j];
    const double2* col = AB + j * (int64_t)ldab + kv;
    for (int r = 1 + lane; r <= km; r += 32) x[j + r] = csub(x[j + r], cmul(col[r], xj));
    __syncwarp();
  }
  // U: upper band of width kl + ku
  for (int64_t j = n - 1; j >= 0; --j) {
    const double2* col = AB + j * (int64_t)ldab + kv;  // col[-d] = A(j - d, j)
    const double2 xj = cdiv(x[j], col[0]);
    __syncwarp();
    if (lane == 0) x[j] = xj;
    const int top = (int)imin(kv, j);
    for (int d = 1 + lane; d <= top; d += 32) x[j - d] = csub(x[j - d], cmul(col[-d], xj));
    __syncwarp();
  }
}

}  // namespace

bool band_feasible(const lt_pencil_s* p) {
  if (p->dim != 2 || p->levels.empty()) return false;
  const Level& L = *p->levels[0];
  const int bw = p->kind == LT_GRID_P1_TRI ? L.nx + 1 : L.nx;
  const double bytes = 16.0 * (double)L.n * (3.0 * bw + 1.0);
  return bytes <= 4e9 && (double)L.n * bw * bw <= 4e10;
}

const BandFactor& pencil_band_factor(lt_pencil p, double2 tau) {
  for (auto& f : p->band_factors)
    if (f->tau.x == tau.x && f->tau.y == tau.y) return *f;
  LT_REQUIRE(band_feasible(p), "banded shift-and-invert: pencil not 2-D or too large");
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const LevelView L = p->view(0);
  auto f = std::make_unique<BandFactor>();
  f->tau = tau;
  f->n = L.n;
  f->kl = f->ku = p->kind == LT_GRID_P1_TRI ? L.nx + 1 : L.nx;
  f->ldab = 2 * f->kl + f->ku + 1;
  f->ab.allocate(sizeof(double2) * (size_t)f->ldab * L.n, st);
  f->ipiv.allocate(sizeof(int) * (size_t)L.n + sizeof(int), st);
  LT_CUDA(cudaMemsetAsync(f->ab.get(), 0, f->ab.bytes(), st));
  int* info = f->ipiv.as<int>() + L.n;
  LT_CUDA(cudaMemsetAsync(info, 0, sizeof(int), st));
  const int p1 = p->kind == LT_GRID_P1_TRI ? 1 : 0;
  launch(ctx, "band_factor", 0.0, [&] {
    band_assemble<<<blocks_for(L.n, 256), 256, 0, st>>>(L, p1, tau, f->kl, f->ku, f->ldab, f->ab.as<double2>());
  });
  launch(ctx, "band_factor", 0.0, [&] {
    band_factor<<<1, kF, 0, st>>>(L.n, f->kl, f->ku, f->ldab, f->ab.as<double2>(), f->ipiv.as<int>(), info);
  });
  int h_info = 0;
  LT_CUDA(cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  if (h_info != 0)
    throw Error(LT_ERR_PRECONDITIONER, "shift-and-invert factorization failed (singular K + tau M, column " +
                                           std::to_string(h_info) + ")");
  p->band_factors.push_back(std::move(f));
  return *p->band_factors.back();
}

void band_solve(lt_pencil p, const BandFactor& f, int B, const double2* v, int64_t vs, double2* u, int64_t us) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const unsigned warps_per_cta = 4;
  launch(ctx, "band_solve", 0.0, [&] {
    band_solve<<<(unsigned)((B + warps_per_cta - 1) / warps_per_cta), 32 * warps_per_cta, 0, st>>>(
        f.n, f.kl, f.ku, f.ldab, f.ab.as<double2>(), f.ipiv.as<int>(), v, vs, u, us, B);
  });
}

}  // namespace lt
