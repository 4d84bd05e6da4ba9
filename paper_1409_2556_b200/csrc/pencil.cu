// Grid pencil: device assembly of the cell-centred FD operator (the FD
// analogue of assemble(), assembly.cpp:69-113), the multigrid hierarchy behind the
// shift-and-invert preconditioner, the matrix-free stencil (K + zM)x / Mx
// (ShiftedPencil::apply / apply_mass, shifted_solver.cpp:109-118) and the coarsest-level
// exact inverses cached by tau (the ShiftedPencil::factorization cache, cpp:120-128).
#include <algorithm>
#include <cmath>
#include <cstring>

#include <cuda_bf16.h>
#include <cusolverDn.h>

#include "lt_internal.hpp"
#include "stencil.cuh"

namespace lt {

namespace {

constexpr int64_t kMaxCoarse = 128;  // stop coarsening at <= this many cells

__global__ void exp_kernel(const double* __restrict__ logv, double* __restrict__ out, int64_t n) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) out[a] = exp(logv[a]);
}

// Fine-level faces from per-cell kappa: harmonic mean inside, 2 kappa at the Dirichlet
// boundary (ghost at h/2), all times h^(d-2).  M = S h^d.
__global__ void assemble_x(const double* __restrict__ kap, double* __restrict__ Tx, int nx, int ny,
                           int nz, double s) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)(nx + 1) * ny * nz;
  if (f >= total) return;
  int i = (int)(f % (nx + 1));
  int64_t row = f / (nx + 1);
  const double* kr = kap + row * nx;
  double t;
  if (i == 0) t = 2.0 * kr[0];
  else if (i == nx) t = 2.0 * kr[nx - 1];
  else { double a = kr[i - 1], b = kr[i]; t = 2.0 * a * b / (a + b); }
  Tx[f] = t * s;
}

__global__ void assemble_y(const double* __restrict__ kap, double* __restrict__ Ty, int nx, int ny,
                           int nz, double s) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nx * (ny + 1) * nz;
  if (f >= total) return;
  int i = (int)(f % nx);
  int64_t t1 = f / nx;
  int j = (int)(t1 % (ny + 1));
  int k = (int)(t1 / (ny + 1));
  const double* kp = kap + (int64_t)k * ny * nx + i;
  double t;
  if (j == 0) t = 2.0 * kp[0];
  else if (j == ny) t = 2.0 * kp[(int64_t)(ny - 1) * nx];
  else { double a = kp[(int64_t)(j - 1) * nx], b = kp[(int64_t)j * nx]; t = 2.0 * a * b / (a + b); }
  Ty[f] = t * s;
}

__global__ void assemble_z(const double* __restrict__ kap, double* __restrict__ Tz, int nx, int ny,
                           int nz, double s) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t plane = (int64_t)nx * ny;
  int64_t total = plane * (nz + 1);
  if (f >= total) return;
  int64_t p = f % plane;
  int k = (int)(f / plane);
  double t;
  if (k == 0) t = 2.0 * kap[p];
  else if (k == nz) t = 2.0 * kap[(int64_t)(nz - 1) * plane + p];
  else { double a = kap[(int64_t)(k - 1) * plane + p], b = kap[(int64_t)k * plane + p]; t = 2.0 * a * b / (a + b); }
  Tz[f] = t * s;
}

__global__ void scale_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t n, double s) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) out[a] = in[a] * s;
}

// Coarse faces: (1/a_dir) * sum of the fine faces that make up the coarse face
// (rediscretisation of the Galerkin piecewise-constant sum), coarse M = sum over the aggregate.
__global__ void coarsen_x(const double* __restrict__ Tf, double* __restrict__ Tc, int nxf, int nyf,
                          int nxc, int nyc, int nzc, int ax, int ay, int az) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)(nxc + 1) * nyc * nzc;
  if (f >= total) return;
  int I = (int)(f % (nxc + 1));
  int64_t t1 = f / (nxc + 1);
  int J = (int)(t1 % nyc);
  int K = (int)(t1 / nyc);
  double s = 0.0;
  for (int kk = 0; kk < az; ++kk)
    for (int jj = 0; jj < ay; ++jj)
      s += Tf[((int64_t)(K * az + kk) * nyf + (J * ay + jj)) * (nxf + 1) + (int64_t)I * ax];
  Tc[f] = s / ax;
}

__global__ void coarsen_y(const double* __restrict__ Tf, double* __restrict__ Tc, int nxf, int nyf,
                          int nxc, int nyc, int nzc, int ax, int ay, int az) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nxc * (nyc + 1) * nzc;
  if (f >= total) return;
  int I = (int)(f % nxc);
  int64_t t1 = f / nxc;
  int J = (int)(t1 % (nyc + 1));
  int K = (int)(t1 / (nyc + 1));
  double s = 0.0;
  for (int kk = 0; kk < az; ++kk)
    for (int ii = 0; ii < ax; ++ii)
      s += Tf[((int64_t)(K * az + kk) * (nyf + 1) + (int64_t)J * ay) * nxf + (I * ax + ii)];
  Tc[f] = s / ay;
}

__global__ void coarsen_z(const double* __restrict__ Tf, double* __restrict__ Tc, int nxf, int nyf,
                          int nxc, int nyc, int nzc, int ax, int ay, int az) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nxc * nyc * (nzc + 1);
  if (f >= total) return;
  int I = (int)(f % nxc);
  int64_t t1 = f / nxc;
  int J = (int)(t1 % nyc);
  int K = (int)(t1 / nyc);
  double s = 0.0;
  for (int jj = 0; jj < ay; ++jj)
    for (int ii = 0; ii < ax; ++ii)
      s += Tf[((int64_t)K * az * nyf + (J * ay + jj)) * nxf + (I * ax + ii)];
  Tc[f] = s / az;
}

__global__ void coarsen_m(const double* __restrict__ Mf, double* __restrict__ Mc, int nxf, int nyf,
                          int nxc, int nyc, int nzc, int ax, int ay, int az) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = (int64_t)nxc * nyc * nzc;
  if (c >= total) return;
  int I = (int)(c % nxc);
  int64_t t1 = c / nxc;
  int J = (int)(t1 % nyc);
  int K = (int)(t1 / nyc);
  double s = 0.0;
  for (int kk = 0; kk < az; ++kk)
    for (int jj = 0; jj < ay; ++jj)
      for (int ii = 0; ii < ax; ++ii)
        s += Mf[((int64_t)(K * az + kk) * nyf + (J * ay + jj)) * nxf + (I * ax + ii)];
  Mc[c] = s;
}

// Dense A_c(tau) = K_c + tau M_c, written into the left half of an n x 2n augmented
// matrix [A | I] (row-major); the right half receives A^{-1} (lt_pencil_s::factor).
__global__ void dense_coarse(LevelView L, double2 tau, double2* __restrict__ aug) {
  int64_t n = L.n;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * 2 * n) return;
  int64_t r = idx / (2 * n), c = idx % (2 * n);
  double2 v = make_double2(0.0, 0.0);
  if (c >= n) {
    if (c - n == r) v.x = 1.0;
  } else {
    int i = (int)(r % L.nx);
    int64_t t1 = r / L.nx;
    int j = (int)(t1 % L.ny);
    int k = (int)(t1 / L.ny);
    if (c == r) {
      double d = diag_k(L, i, j, k);
      v = make_double2(d + tau.x * L.M[r], tau.y * L.M[r]);
    } else {
      int64_t plane = (int64_t)L.nx * L.ny;
      if (c == r - 1 && i > 0) v.x = -L.Tx[fx(L, i, j, k)];
      if (c == r + 1 && i < L.nx - 1) v.x = -L.Tx[fx(L, i + 1, j, k)];
      if (c == r - L.nx && j > 0) v.x = -L.Ty[fy(L, i, j, k)];
      if (c == r + L.nx && j < L.ny - 1) v.x = -L.Ty[fy(L, i, j + 1, k)];
      if (L.dim == 3) {
        if (c == r - plane && k > 0) v.x = -L.Tz[r];
        if (c == r + plane && k < L.nz - 1) v.x = -L.Tz[r + plane];
      }
      if (L.Mx) {  // P1: tau * the off-diagonal mass couplings
        double mo = 0.0;
        if (c == r - 1 && i > 0) mo = L.Mx[fx(L, i, j, k)];
        if (c == r + 1 && i < L.nx - 1) mo = L.Mx[fx(L, i + 1, j, k)];
        if (c == r - L.nx && j > 0) mo = L.My[fy(L, i, j, k)];
        if (c == r + L.nx && j < L.ny - 1) mo = L.My[fy(L, i, j + 1, k)];
        if (c == r + L.nx + 1 && i < L.nx - 1 && j < L.ny - 1) mo = L.Md[r];
        if (c == r - L.nx - 1 && i > 0 && j > 0) mo = L.Md[c];
        v.x += tau.x * mo;
        v.y += tau.y * mo;
      }
    }
  }
  aug[idx] = v;
}

}  // namespace

LevelView lt_pencil_view(const lt_pencil_s* p, int l) {
  const Level& L = *p->levels[l];
  int tws = 0;
  while ((1 << tws) < L.nx && tws < 5) ++tws;  // tile width: next power of two of nx, <= 32
  const int tw = 1 << tws;
  const int th = 256 / tw;
  const int tiles_x = (L.nx + tw - 1) / tw;
  const int tiles_y = (L.ny + th - 1) / th;
  return LevelView{L.nx, L.ny, L.nz, p->dim, L.n, L.Tx, L.Ty, L.Tz, L.M,
                   tw, tws, th, tiles_x, tiles_y, tiles_x * tiles_y * L.nz, L.Mx, L.My, L.Md};
}

LevelView32 lt_pencil_view32(const lt_pencil_s* p, int l) {
  const LevelView v = lt_pencil_view(p, l);
  const Level& L = *p->levels[l];
  return LevelView32{v.nx, v.ny, v.nz, v.dim, v.n, L.Tx32, L.Ty32, L.Tz32, L.M32,
                     v.tw, v.tws, v.th, v.tiles_x, v.tiles_y, v.ntiles, L.Mx32, L.My32, L.Md32};
}

namespace {
__global__ void d2f_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t n) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) out[a] = (float)in[a];
}
__global__ void inverse_to_c64(const double2* __restrict__ aug, float2* __restrict__ out, int64_t n) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const int64_t r = t / n, c = t % n;
  const double2 v = aug[r * 2 * n + n + c];
  out[t] = make_float2((float)v.x, (float)v.y);
}
}  // namespace

static void alloc_level(Level& L, int dim, cudaStream_t s) {
  L.n = (int64_t)L.nx * L.ny * L.nz;
  int64_t nfx = (int64_t)(L.nx + 1) * L.ny * L.nz;
  int64_t nfy = (int64_t)L.nx * (L.ny + 1) * L.nz;
  int64_t nfz = dim == 3 ? (int64_t)L.nx * L.ny * (L.nz + 1) : 0;
  L.storage.allocate(sizeof(double) * (nfx + nfy + nfz + L.n), s);
  double* base = L.storage.as<double>();
  L.Tx = base;
  L.Ty = base + nfx;
  L.Tz = dim == 3 ? base + nfx + nfy : nullptr;
  L.M = base + nfx + nfy + nfz;
}

// ---- P1 triangle discretisation (the reference's own operator) -------------------------
// Node grid of build_mesh(n, L) (mesh.cpp:14-52): cell c = cj*nc + ci has the lower element
// 2c = (a, b, c') and the upper element 2c+1 = (a, c', d); free unknowns are the interior
// nodes (I, J) = (i+1, j+1), i, j < n-2.  Exact P1 integrals (assembly.cpp:24-41) per edge:
//   K edge = (kappa_T1 + kappa_T2)/2 over the two triangles sharing it (hypotenuse: 0),
//   M edge = h^2 (S_T1 + S_T2)/24, M node = h^2/12 sum of the six triangles' S,
// laid out like the FD faces (Tx: E/W edges, Ty: N/S edges) plus Mx, My and Md (NE).
namespace {

__device__ __forceinline__ int64_t elem_lo(int ci, int cj, int nc) { return 2 * ((int64_t)cj * nc + ci); }

__global__ void p1_assemble_x(const double* __restrict__ ek, const double* __restrict__ es, int nx, int ny,
                              double h2, double* __restrict__ Tx, double* __restrict__ Mx) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)(nx + 1) * ny) return;
  const int i = (int)(e % (nx + 1)), j = (int)(e / (nx + 1));
  const int nc = nx + 1, I = i, J = j + 1;  // edge (I, J)-(I+1, J)
  const int64_t lo = elem_lo(I, J, nc), up = elem_lo(I, J - 1, nc) + 1;
  Tx[e] = 0.5 * (ek[lo] + ek[up]);
  Mx[e] = h2 * (es[lo] + es[up]) / 24.0;
}

__global__ void p1_assemble_y(const double* __restrict__ ek, const double* __restrict__ es, int nx, int ny,
                              double h2, double* __restrict__ Ty, double* __restrict__ My) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * (ny + 1)) return;
  const int i = (int)(e % nx), j = (int)(e / nx);
  const int nc = nx + 1, I = i + 1, J = j;  // edge (I, J)-(I, J+1)
  const int64_t up = elem_lo(I, J, nc) + 1, lo = elem_lo(I - 1, J, nc);
  Ty[e] = 0.5 * (ek[up] + ek[lo]);
  My[e] = h2 * (es[up] + es[lo]) / 24.0;
}

__global__ void p1_assemble_node(const double* __restrict__ es, int nx, int ny, double h2, double* __restrict__ M,
                                 double* __restrict__ Md) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= (int64_t)nx * ny) return;
  const int i = (int)(a % nx), j = (int)(a / nx);
  const int nc = nx + 1, I = i + 1, J = j + 1;
  const double s = es[elem_lo(I, J, nc)] + es[elem_lo(I, J, nc) + 1] + es[elem_lo(I - 1, J, nc)] +
                   es[elem_lo(I - 1, J - 1, nc)] + es[elem_lo(I - 1, J - 1, nc) + 1] + es[elem_lo(I, J - 1, nc) + 1];
  M[a] = h2 * s / 12.0;
  Md[a] = h2 * (es[elem_lo(I, J, nc)] + es[elem_lo(I, J, nc) + 1]) / 24.0;  // hypotenuse to (I+1, J+1)
}

// Coarse element fields: the mean over the four fine triangles inside each coarse triangle
// (exact Galerkin P^T K P for the nested P1 spaces; the mass is approximated the same way).
__global__ void p1_coarsen_elem(const double* __restrict__ ef, int ncf, double* __restrict__ ec, int ncc) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= (int64_t)ncc * ncc) return;
  const int Ci = (int)(c % ncc), Cj = (int)(c / ncc);
  const int fi = 2 * Ci, fj = 2 * Cj;
  const double lo = ef[elem_lo(fi, fj, ncf)] + ef[elem_lo(fi + 1, fj, ncf)] + ef[elem_lo(fi + 1, fj, ncf) + 1] +
                    ef[elem_lo(fi + 1, fj + 1, ncf)];
  const double up = ef[elem_lo(fi, fj, ncf) + 1] + ef[elem_lo(fi, fj + 1, ncf)] + ef[elem_lo(fi, fj + 1, ncf) + 1] +
                    ef[elem_lo(fi + 1, fj + 1, ncf) + 1];
  ec[2 * c] = 0.25 * lo;
  ec[2 * c + 1] = 0.25 * up;
}

}  // namespace

static void alloc_level_p1(Level& L, cudaStream_t s) {
  L.nz = 1;
  L.n = (int64_t)L.nx * L.ny;
  const int64_t nfx = (int64_t)(L.nx + 1) * L.ny, nfy = (int64_t)L.nx * (L.ny + 1);
  L.storage.allocate(sizeof(double) * 2 * (nfx + nfy + L.n), s);
  double* base = L.storage.as<double>();
  L.Tx = base;
  L.Ty = base + nfx;
  L.Tz = nullptr;
  L.M = base + nfx + nfy;
  L.Mx = L.M + L.n;
  L.My = L.Mx + nfx;
  L.Md = L.My + nfy;
  const int64_t nelem = 2 * (int64_t)(L.nx + 1) * (L.nx + 1);
  L.elem.allocate(sizeof(double) * 2 * nelem, s);
}

static void assemble_p1(lt_ctx ctx, Level& L, double h) {
  cudaStream_t st = ctx->stream;
  const int64_t nelem = 2 * (int64_t)(L.nx + 1) * (L.nx + 1);
  const double* ek = L.elem.as<double>();
  const double* es = ek + nelem;
  const double h2 = h * h;
  const int nx = L.nx, ny = L.ny;
  Level* Lp = &L;
  launch(ctx, "assemble", 0.0, [&] {
    p1_assemble_x<<<blocks_for((int64_t)(nx + 1) * ny, kThreads), kThreads, 0, st>>>(ek, es, nx, ny, h2, Lp->Tx, Lp->Mx);
  });
  launch(ctx, "assemble", 0.0, [&] {
    p1_assemble_y<<<blocks_for((int64_t)nx * (ny + 1), kThreads), kThreads, 0, st>>>(ek, es, nx, ny, h2, Lp->Ty, Lp->My);
  });
  launch(ctx, "assemble", 0.0, [&] {
    p1_assemble_node<<<blocks_for((int64_t)nx * ny, kThreads), kThreads, 0, st>>>(es, nx, ny, h2, Lp->M, Lp->Md);
  });
}

// out[(k (ny+1) + j) (nx+1) + i] = {Tx west face of (i,j,k), Ty south face, Tz bottom face, M}
// over i <= nx, j <= ny, k <= nz (faces past the last cell of a row / column / stack in the
// extra entries, zero where no such face exists); Tz null in 2-D
template <class T4>
__global__ void pack_coef_kernel(const double* __restrict__ Tx, const double* __restrict__ Ty,
                                 const double* __restrict__ Tz, const double* __restrict__ M, int nx, int ny, int nz,
                                 T4* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t cnt = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  if (t >= cnt) return;
  const int i = (int)(t % (nx + 1));
  const int j = (int)((t / (nx + 1)) % (ny + 1));
  const int k = (int)(t / ((int64_t)(nx + 1) * (ny + 1)));
  const bool ci = i < nx, cj = j < ny, ck = k < nz;
  const double tw = (cj && ck) ? Tx[((int64_t)k * ny + j) * (nx + 1) + i] : 0.0;
  const double ts = (ci && ck) ? Ty[((int64_t)k * (ny + 1) + j) * nx + i] : 0.0;
  const double tb = (Tz && ci && cj) ? Tz[((int64_t)k * ny + j) * nx + i] : 0.0;
  const double m = (ci && cj && ck) ? M[((int64_t)k * ny + j) * nx + i] : 0.0;
  using E = decltype(T4::x);
  out[t] = T4{(E)tw, (E)ts, (E)tb, (E)m};
}

// The FP64 coefficients of the finest level, planar: [k][j][W, S, B, M][i], rows of P >= nx + 1
__global__ void pack_planar64_kernel(const double* __restrict__ Tx, const double* __restrict__ Ty,
                                     const double* __restrict__ Tz, const double* __restrict__ M, int nx, int ny, int nz,
                                     int P, double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t cnt = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  if (t >= cnt) return;
  const int i = (int)(t % (nx + 1));
  const int j = (int)((t / (nx + 1)) % (ny + 1));
  const int k = (int)(t / ((int64_t)(nx + 1) * (ny + 1)));
  const bool ci = i < nx, cj = j < ny, ck = k < nz;
  const int64_t row = ((int64_t)k * (ny + 1) + j) * 4;
  out[(row + 0) * P + i] = (cj && ck) ? Tx[((int64_t)k * ny + j) * (nx + 1) + i] : 0.0;
  out[(row + 1) * P + i] = (ci && ck) ? Ty[((int64_t)k * (ny + 1) + j) * nx + i] : 0.0;
  out[(row + 2) * P + i] = (Tz && ci && cj) ? Tz[((int64_t)k * ny + j) * nx + i] : 0.0;
  out[(row + 3) * P + i] = (ci && cj && ck) ? M[((int64_t)k * ny + j) * nx + i] : 0.0;
}

// The coefficients in the colour-split layout (Level::packrb), rounded to rb_coef_t
__device__ __forceinline__ rb_coef_t to_rb_coef(double v) {
#if RB_BF16
  return __bfloat16_as_ushort(__float2bfloat16_rn((float)v));
#else
  return (float)v;
#endif
}
__global__ void pack_rb_kernel(const double* __restrict__ Tx, const double* __restrict__ Ty,
                               const double* __restrict__ Tz, const double* __restrict__ M, int nx, int ny, int nz,
                               int P, rb_coef_t* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t cnt = (int64_t)(nx + 1) * (ny + 1) * (nz + 1);
  if (t >= cnt) return;
  const int i = (int)(t % (nx + 1));
  const int j = (int)((t / (nx + 1)) % (ny + 1));
  const int k = (int)(t / ((int64_t)(nx + 1) * (ny + 1)));
  const bool ci = i < nx, cj = j < ny, ck = k < nz;
  const double v[4] = {(cj && ck) ? Tx[((int64_t)k * ny + j) * (nx + 1) + i] : 0.0,
                       (ci && ck) ? Ty[((int64_t)k * (ny + 1) + j) * nx + i] : 0.0,
                       (Tz && ci && cj) ? Tz[((int64_t)k * ny + j) * nx + i] : 0.0,
                       (ci && cj && ck) ? M[((int64_t)k * ny + j) * nx + i] : 0.0};
  const int h = (i + j + k) & 1, pos = i >> 1;
  const int64_t row = (int64_t)k * (ny + 1) + j;
  for (int c = 0; c < 4; ++c) out[((row * 4 + c) * 2 + h) * P + pos] = to_rb_coef(v[c]);
}

static void make_fp32_copies(lt_pencil p) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  for (auto& lv : p->levels) {
    Level& Lv = *lv;
    const int64_t cnt = (int64_t)(Lv.storage.bytes() / sizeof(double));
    Lv.storage32.allocate(sizeof(float) * cnt, st);
    float* base = Lv.storage32.as<float>();
    const double* src = Lv.storage.as<double>();
    Lv.Tx32 = base + (Lv.Tx - src);
    Lv.Ty32 = base + (Lv.Ty - src);
    Lv.Tz32 = Lv.Tz ? base + (Lv.Tz - src) : nullptr;
    Lv.M32 = base + (Lv.M - src);
    Lv.Mx32 = Lv.Mx ? base + (Lv.Mx - src) : nullptr;
    Lv.My32 = Lv.My ? base + (Lv.My - src) : nullptr;
    Lv.Md32 = Lv.Md ? base + (Lv.Md - src) : nullptr;
    launch(ctx, "assemble", 12.0 * cnt, [&] { d2f_kernel<<<blocks_for(cnt, kThreads), kThreads, 0, st>>>(src, base, cnt); });
  }
}

static void pencil_build_p1(lt_pencil p, const double* log_kappa, const double* log_s, int mem) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int n_per_side = p->grid.shape[0];
  const int nc = n_per_side - 1;
  const int64_t nelem = 2 * (int64_t)nc * nc;
  auto fine = std::make_unique<Level>();
  fine->nx = fine->ny = n_per_side - 2;
  alloc_level_p1(*fine, st);
  p->n = fine->n;
  p->kappa.allocate(sizeof(double) * nelem, st);
  p->storativity.allocate(sizeof(double) * nelem, st);
  DeviceBuffer logs(sizeof(double) * 2 * nelem, st);
  double* lk = logs.as<double>();
  double* ls = lk + nelem;
  auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  LT_CUDA(cudaMemcpyAsync(lk, log_kappa, sizeof(double) * nelem, kind, st));
  LT_CUDA(cudaMemcpyAsync(ls, log_s, sizeof(double) * nelem, kind, st));
  double* kap = p->kappa.as<double>();
  double* sto = p->storativity.as<double>();
  launch(ctx, "assemble", 0.0, [&] { exp_kernel<<<blocks_for(nelem, kThreads), kThreads, 0, st>>>(lk, kap, nelem); });
  launch(ctx, "assemble", 0.0, [&] { exp_kernel<<<blocks_for(nelem, kThreads), kThreads, 0, st>>>(ls, sto, nelem); });
  LT_CUDA(cudaMemcpyAsync(fine->elem.as<double>(), kap, sizeof(double) * nelem, cudaMemcpyDeviceToDevice, st));
  LT_CUDA(cudaMemcpyAsync(fine->elem.as<double>() + nelem, sto, sizeof(double) * nelem, cudaMemcpyDeviceToDevice, st));
  double h = p->grid.h;
  assemble_p1(ctx, *fine, h);
  p->levels.clear();
  p->levels.push_back(std::move(fine));
  // vertex-centred hierarchy: n-1 intervals -> (n-1)/2 while even and >= 4
  while (p->levels.back()->n > kMaxCoarse) {
    Level& Fl = *p->levels.back();
    const int ncf = Fl.nx + 1;
    if (ncf % 2 != 0 || ncf < 4) break;
    const int ncc = ncf / 2;
    auto C = std::make_unique<Level>();
    C->nx = C->ny = ncc - 1;
    alloc_level_p1(*C, st);
    const int64_t nef = 2 * (int64_t)ncf * ncf, nec = 2 * (int64_t)ncc * ncc;
    const double* ef = Fl.elem.as<double>();
    double* ecp = C->elem.as<double>();
    for (int f = 0; f < 2; ++f)
      launch(ctx, "coarsen", 0.0, [&] {
        p1_coarsen_elem<<<blocks_for((int64_t)ncc * ncc, kThreads), kThreads, 0, st>>>(ef + f * nef, ncf, ecp + f * nec,
                                                                                      ncc);
      });
    h *= 2.0;
    assemble_p1(ctx, *C, h);
    p->levels.push_back(std::move(C));
  }
  make_fp32_copies(p);
  LT_CUDA(cudaStreamSynchronize(st));
}

static void build_hierarchy_fd(lt_pencil p);

void pencil_build(lt_pencil p, const double* log_kappa, const double* log_s, int mem) {
  if (p->kind == LT_GRID_P1_TRI) {
    pencil_build_p1(p, log_kappa, log_s, mem);
    return;
  }
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int dim = p->dim;
  auto fine = std::make_unique<Level>();
  fine->nx = p->grid.shape[0];
  fine->ny = p->grid.shape[1];
  fine->nz = dim == 3 ? p->grid.shape[2] : 1;
  alloc_level(*fine, dim, st);
  const int64_t n = fine->n;
  p->n = n;
  p->kappa.allocate(sizeof(double) * n, st);
  p->storativity.allocate(sizeof(double) * n, st);
  DeviceBuffer logs(sizeof(double) * 2 * n, st);
  double* lk = logs.as<double>();
  double* ls = lk + n;
  auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  LT_CUDA(cudaMemcpyAsync(lk, log_kappa, sizeof(double) * n, kind, st));
  LT_CUDA(cudaMemcpyAsync(ls, log_s, sizeof(double) * n, kind, st));
  double* kap = p->kappa.as<double>();
  double* sto = p->storativity.as<double>();
  launch(ctx, "assemble", 32.0 * n, [&] { exp_kernel<<<blocks_for(n, kThreads), kThreads, 0, st>>>(lk, kap, n); });
  launch(ctx, "assemble", 16.0 * n, [&] { exp_kernel<<<blocks_for(n, kThreads), kThreads, 0, st>>>(ls, sto, n); });
  const double h = p->grid.h;
  const double sface = dim == 3 ? h : 1.0;
  const int nx = fine->nx, ny = fine->ny, nz = fine->nz;
  Level* F = fine.get();
  launch(ctx, "assemble", 16.0 * n, [&] {
    assemble_x<<<blocks_for((int64_t)(nx + 1) * ny * nz, kThreads), kThreads, 0, st>>>(kap, F->Tx, nx, ny, nz, sface);
  });
  launch(ctx, "assemble", 16.0 * n, [&] {
    assemble_y<<<blocks_for((int64_t)nx * (ny + 1) * nz, kThreads), kThreads, 0, st>>>(kap, F->Ty, nx, ny, nz, sface);
  });
  if (dim == 3)
    launch(ctx, "assemble", 16.0 * n, [&] {
      assemble_z<<<blocks_for((int64_t)nx * ny * (nz + 1), kThreads), kThreads, 0, st>>>(kap, F->Tz, nx, ny, nz, sface);
    });
  const double hd = dim == 3 ? h * h * h : h * h;
  launch(ctx, "assemble", 16.0 * n, [&] { scale_kernel<<<blocks_for(n, kThreads), kThreads, 0, st>>>(sto, F->M, n, hd); });
  p->levels.clear();
  p->levels.push_back(std::move(fine));
  build_hierarchy_fd(p);
}

// FD: the multigrid hierarchy below the (assembled) finest level, the FP32 copies and the
// packed operand arrays of the TMA kernels.
static void build_hierarchy_fd(lt_pencil p) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int dim = p->dim;
  // Hierarchy: halve every even dimension >= 4 until <= kMaxCoarse cells remain.
  while (p->levels.back()->n > kMaxCoarse) {
    Level& Fl = *p->levels.back();
    int dims[3] = {Fl.nx, Fl.ny, Fl.nz};
    int agg[3] = {1, 1, 1};
    bool any = false;
    for (int d = 0; d < dim; ++d) {
      if (dims[d] % 2 == 0 && dims[d] >= 4) { agg[d] = 2; any = true; }
    }
    if (!any) break;
    auto C = std::make_unique<Level>();
    C->nx = Fl.nx / agg[0];
    C->ny = Fl.ny / agg[1];
    C->nz = Fl.nz / agg[2];
    alloc_level(*C, dim, st);
    for (int d = 0; d < 3; ++d) Fl.agg[d] = agg[d];
    Level* Cp = C.get();
    Level* Fp = &Fl;
    launch(ctx, "coarsen", 0.0, [&] {
      coarsen_x<<<blocks_for((int64_t)(Cp->nx + 1) * Cp->ny * Cp->nz, kThreads), kThreads, 0, st>>>(
          Fp->Tx, Cp->Tx, Fp->nx, Fp->ny, Cp->nx, Cp->ny, Cp->nz, agg[0], agg[1], agg[2]);
    });
    launch(ctx, "coarsen", 0.0, [&] {
      coarsen_y<<<blocks_for((int64_t)Cp->nx * (Cp->ny + 1) * Cp->nz, kThreads), kThreads, 0, st>>>(
          Fp->Ty, Cp->Ty, Fp->nx, Fp->ny, Cp->nx, Cp->ny, Cp->nz, agg[0], agg[1], agg[2]);
    });
    if (dim == 3)
      launch(ctx, "coarsen", 0.0, [&] {
        coarsen_z<<<blocks_for((int64_t)Cp->nx * Cp->ny * (Cp->nz + 1), kThreads), kThreads, 0, st>>>(
            Fp->Tz, Cp->Tz, Fp->nx, Fp->ny, Cp->nx, Cp->ny, Cp->nz, agg[0], agg[1], agg[2]);
      });
    launch(ctx, "coarsen", 0.0, [&] {
      coarsen_m<<<blocks_for(Cp->n, kThreads), kThreads, 0, st>>>(Fp->M, Cp->M, Fp->nx, Fp->ny, Cp->nx,
                                                                    Cp->ny, Cp->nz, agg[0], agg[1], agg[2]);
    });
    p->levels.push_back(std::move(C));
  }
  // FP32 copies of every level for the mixed-precision V-cycle (same layout)
  make_fp32_copies(p);
  // packed operand arrays of the TMA-fed kernels: FP32 for the V-cycle levels, FP64 for the
  // finest level (the COCG operator)
  for (size_t l = 0; l < p->levels.size(); ++l) {
    Level& Lv = *p->levels[l];
    const int64_t cnt = (int64_t)(Lv.nx + 1) * (Lv.ny + 1) * (Lv.nz + 1);
    Lv.pack32.allocate(sizeof(float4) * cnt, st);
    launch(ctx, "assemble", 20.0 * cnt, [&] {
      pack_coef_kernel<float4><<<blocks_for(cnt, kThreads), kThreads, 0, st>>>(Lv.Tx, Lv.Ty, Lv.Tz, Lv.M, Lv.nx, Lv.ny,
                                                                               Lv.nz, Lv.pack32.as<float4>());
    });
    if (p->kind != LT_GRID_P1_TRI && Lv.nx % 4 == 0 && Lv.nx >= 64 && Lv.Tz) {
      Lv.rb_P = ((Lv.nx / 2 + 1) + 7) / 8 * 8;
      const size_t rb = sizeof(rb_coef_t) * (size_t)(Lv.nz + 1) * (Lv.ny + 1) * 8 * Lv.rb_P;
      Lv.packrb.allocate(rb, st);
      LT_CUDA(cudaMemsetAsync(Lv.packrb.get(), 0, rb, st));
      launch(ctx, "assemble", 48.0 * cnt, [&] {
        pack_rb_kernel<<<blocks_for(cnt, kThreads), kThreads, 0, st>>>(Lv.Tx, Lv.Ty, Lv.Tz, Lv.M, Lv.nx, Lv.ny, Lv.nz,
                                                                       Lv.rb_P, Lv.packrb.as<rb_coef_t>());
      });
    }
    if (l == 0 && Lv.nx % 2 == 0) {
      const int P = Lv.nx + 2;
      const size_t pb = sizeof(double) * (size_t)(Lv.nz + 1) * (Lv.ny + 1) * 4 * P;
      Lv.pack64.allocate(pb, st);
      LT_CUDA(cudaMemsetAsync(Lv.pack64.get(), 0, pb, st));
      launch(ctx, "assemble", 40.0 * cnt, [&] {
        pack_planar64_kernel<<<blocks_for(cnt, kThreads), kThreads, 0, st>>>(Lv.Tx, Lv.Ty, Lv.Tz, Lv.M, Lv.nx, Lv.ny,
                                                                            Lv.nz, P, Lv.pack64.as<double>());
      });
    }
  }
  LT_CUDA(cudaStreamSynchronize(st));
}

// ---- pencils from assembled sparse (K, M) (ShiftedPencil(K, M), shifted_solver.cpp:106-107) --
// The device operator is matrix-free on a structured grid, so the CSR pair is checked against
// the stencil of the grid it is declared on and converted to that stencil's coefficients:
//   FD_CELL: K = the 5-/7-point cell-centred operator (off-diagonals -T_f, diagonal = sum of the
//            cell's faces, the boundary faces taking what the interior ones leave), M diagonal;
//   P1_TRI:  the reference's P1 pair on build_mesh's interior nodes (assembly.cpp:69-113):
//            K on the E/W/N/S edges (the NE/SW hypotenuse entries zero), M on those plus NE/SW.
// Entries off the stencil, asymmetric pairs or a negative boundary remainder are rejected
// (std::invalid_argument).  The fine-level operator is the given one (to rounding in the
// diagonal, which the kernels form as the sum of the faces); the preconditioner hierarchy is
// coarsened from it (FD: face sums; P1: element fields estimated from the node diagonals).
namespace {

struct CsrView {
  int64_t n;
  const lt_sparse* s;
  int64_t outer(int64_t r) const {
    return s->index_bytes == 4 ? (int64_t) static_cast<const int32_t*>(s->outer)[r] : static_cast<const int64_t*>(s->outer)[r];
  }
  int64_t inner(int64_t e) const {
    return s->index_bytes == 4 ? (int64_t) static_cast<const int32_t*>(s->inner)[e] : static_cast<const int64_t*>(s->inner)[e];
  }
};

void csr_fail(const char* what, int64_t r, int64_t col) {
  throw Error(LT_ERR_INVALID_ARGUMENT, std::string("ShiftedPencil(K, M): ") + what + " (row " + std::to_string(r) +
                                           ", column " + std::to_string(col) + ")");
}

// set a symmetric coupling once from either triangle; the second sighting must agree
void set_pair(std::vector<double>& arr, std::vector<char>& seen, int64_t idx, double v, int64_t r, int64_t col) {
  if (!seen[idx]) {
    arr[idx] = v;
    seen[idx] = 1;
  } else if (std::fabs(arr[idx] - v) > 1e-12 * std::max(std::fabs(arr[idx]), std::fabs(v))) {
    csr_fail("matrix is not symmetric", r, col);
  }
}

// face / boundary remainder split: rem over nb boundary faces (FD) or edges (P1)
void split_boundary(double rem, double diag, int nb, int64_t r, double* faces[], int nf) {
  const double tiny = 1e-12 * std::fabs(diag);
  if (nb == 0) {
    if (std::fabs(rem) > tiny) csr_fail("row sum of K is not zero on an interior unknown", r, r);
    return;
  }
  if (rem < -tiny) csr_fail("negative boundary coupling in K", r, r);
  for (int f = 0; f < nf; ++f) *faces[f] = std::max(rem, 0.0) / nb;
}

}  // namespace

void pencil_build_csr(lt_pencil p, const lt_sparse* K, const lt_sparse* M) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const CsrView k{p->n, K}, m{p->n, M};
  const int64_t n = p->n;
  if (p->kind == LT_GRID_FD_CELL) {
    const int nx = p->grid.shape[0], ny = p->grid.shape[1], nz = p->dim == 3 ? p->grid.shape[2] : 1;
    LT_REQUIRE((int64_t)nx * ny * nz == n, "ShiftedPencil(K, M): rows do not match the grid's cell count");
    const int64_t nfx = (int64_t)(nx + 1) * ny * nz, nfy = (int64_t)nx * (ny + 1) * nz,
                  nfz = p->dim == 3 ? (int64_t)nx * ny * (nz + 1) : 0;
    std::vector<double> Tx(nfx, 0.0), Ty(nfy, 0.0), Tz(nfz, 0.0), Md(n, 0.0);
    std::vector<char> sx(nfx, 0), sy(nfy, 0), sz(nfz, 0);
    std::vector<double> diag(n, 0.0);
    const int64_t plane = (int64_t)nx * ny;
    for (int64_t r = 0; r < n; ++r) {
      const int i = (int)(r % nx), j = (int)((r / nx) % ny), kk = (int)(r / plane);
      for (int64_t e = k.outer(r); e < k.outer(r + 1); ++e) {
        const int64_t col = k.inner(e);
        const double v = K->values[e];
        if (col < 0 || col >= n) csr_fail("column index out of range", r, col);
        const int64_t d = col - r;
        if (d == 0) { diag[r] += v; continue; }
        if (d == 1 && i + 1 < nx) set_pair(Tx, sx, ((int64_t)kk * ny + j) * (nx + 1) + i + 1, -v, r, col);
        else if (d == -1 && i > 0) set_pair(Tx, sx, ((int64_t)kk * ny + j) * (nx + 1) + i, -v, r, col);
        else if (d == nx && j + 1 < ny) set_pair(Ty, sy, ((int64_t)kk * (ny + 1) + j + 1) * nx + i, -v, r, col);
        else if (d == -nx && j > 0) set_pair(Ty, sy, ((int64_t)kk * (ny + 1) + j) * nx + i, -v, r, col);
        else if (p->dim == 3 && d == plane && kk + 1 < nz) set_pair(Tz, sz, ((int64_t)(kk + 1) * ny + j) * nx + i, -v, r, col);
        else if (p->dim == 3 && d == -plane && kk > 0) set_pair(Tz, sz, ((int64_t)kk * ny + j) * nx + i, -v, r, col);
        else if (v != 0.0) csr_fail("K entry outside the grid's finite-difference stencil", r, col);
      }
      for (int64_t e = m.outer(r); e < m.outer(r + 1); ++e) {
        const int64_t col = m.inner(e);
        if (col == r) Md[r] += M->values[e];
        else if (M->values[e] != 0.0) csr_fail("M is not diagonal (the cell-centred mass is)", r, col);
      }
    }
    for (int64_t r = 0; r < n; ++r) {
      const int i = (int)(r % nx), j = (int)((r / nx) % ny), kk = (int)(r / plane);
      double* w = &Tx[((int64_t)kk * ny + j) * (nx + 1) + i];
      double* e = w + 1;
      double* s = &Ty[((int64_t)kk * (ny + 1) + j) * nx + i];
      double* nn = s + nx;
      double* b = p->dim == 3 ? &Tz[((int64_t)kk * ny + j) * nx + i] : nullptr;
      double* t = p->dim == 3 ? b + plane : nullptr;
      double rem = diag[r];
      double* bnd[6];
      int nb = 0;
      auto face = [&](double* f, bool boundary) {
        if (boundary) bnd[nb++] = f;
        else rem -= *f;
      };
      face(w, i == 0);
      face(e, i == nx - 1);
      face(s, j == 0);
      face(nn, j == ny - 1);
      if (p->dim == 3) {
        face(b, kk == 0);
        face(t, kk == nz - 1);
      }
      split_boundary(rem, diag[r], nb, r, bnd, nb);
    }
    auto fine = std::make_unique<Level>();
    fine->nx = nx;
    fine->ny = ny;
    fine->nz = nz;
    alloc_level(*fine, p->dim, st);
    LT_CUDA(cudaMemcpyAsync(fine->Tx, Tx.data(), sizeof(double) * nfx, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(fine->Ty, Ty.data(), sizeof(double) * nfy, cudaMemcpyHostToDevice, st));
    if (nfz) LT_CUDA(cudaMemcpyAsync(fine->Tz, Tz.data(), sizeof(double) * nfz, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(fine->M, Md.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaStreamSynchronize(st));  // the host arrays go out of scope
    p->levels.clear();
    p->levels.push_back(std::move(fine));
    build_hierarchy_fd(p);
    return;
  }
  // P1_TRI: interior node grid nx x nx, unknown a = j nx + i; Tx[(j)(nx+1) + i] = edge (i-1, i)
  const int nps = p->grid.shape[0], nx = nps - 2;
  LT_REQUIRE((int64_t)nx * nx == n, "ShiftedPencil(K, M): rows do not match build_mesh's interior nodes");
  const double h = p->grid.h, h2 = h * h;
  const int64_t nfx = (int64_t)(nx + 1) * nx, nfy = (int64_t)nx * (nx + 1);
  std::vector<double> Tx(nfx, 0.0), Ty(nfy, 0.0), Mx(nfx, 0.0), My(nfy, 0.0), Mn(n, 0.0), Mdg(n, 0.0), diag(n, 0.0);
  std::vector<char> sx(nfx, 0), sy(nfy, 0), smx(nfx, 0), smy(nfy, 0), smd(n, 0);
  for (int64_t r = 0; r < n; ++r) {
    const int i = (int)(r % nx), j = (int)(r / nx);
    for (int64_t e = k.outer(r); e < k.outer(r + 1); ++e) {
      const int64_t col = k.inner(e);
      const double v = K->values[e];
      if (col < 0 || col >= n) csr_fail("column index out of range", r, col);
      const int64_t d = col - r;
      if (d == 0) diag[r] += v;
      else if (d == 1 && i + 1 < nx) set_pair(Tx, sx, (int64_t)j * (nx + 1) + i + 1, -v, r, col);
      else if (d == -1 && i > 0) set_pair(Tx, sx, (int64_t)j * (nx + 1) + i, -v, r, col);
      else if (d == nx && j + 1 < nx) set_pair(Ty, sy, (int64_t)(j + 1) * nx + i, -v, r, col);
      else if (d == -nx && j > 0) set_pair(Ty, sy, (int64_t)j * nx + i, -v, r, col);
      else if (v != 0.0) csr_fail("K entry outside the P1 edge stencil of build_mesh", r, col);
    }
    for (int64_t e = m.outer(r); e < m.outer(r + 1); ++e) {
      const int64_t col = m.inner(e);
      const double v = M->values[e];
      if (col < 0 || col >= n) csr_fail("column index out of range", r, col);
      const int64_t d = col - r;
      if (d == 0) Mn[r] += v;
      else if (d == 1 && i + 1 < nx) set_pair(Mx, smx, (int64_t)j * (nx + 1) + i + 1, v, r, col);
      else if (d == -1 && i > 0) set_pair(Mx, smx, (int64_t)j * (nx + 1) + i, v, r, col);
      else if (d == nx && j + 1 < nx) set_pair(My, smy, (int64_t)(j + 1) * nx + i, v, r, col);
      else if (d == -nx && j > 0) set_pair(My, smy, (int64_t)j * nx + i, v, r, col);
      else if (d == nx + 1 && i + 1 < nx && j + 1 < nx) set_pair(Mdg, smd, r, v, r, col);
      else if (d == -(nx + 1) && i > 0 && j > 0) set_pair(Mdg, smd, r - nx - 1, v, r, col);
      else if (v != 0.0) csr_fail("M entry outside the P1 stencil of build_mesh", r, col);
    }
  }
  for (int64_t r = 0; r < n; ++r) {
    const int i = (int)(r % nx), j = (int)(r / nx);
    double* w = &Tx[(int64_t)j * (nx + 1) + i];
    double* e = w + 1;
    double* s = &Ty[(int64_t)j * nx + i];
    double* nn = s + nx;
    double rem = diag[r];
    double* bnd[4];
    int nb = 0;
    auto edge = [&](double* f, bool boundary) {
      if (boundary) bnd[nb++] = f;
      else rem -= *f;
    };
    edge(w, i == 0);
    edge(e, i == nx - 1);
    edge(s, j == 0);
    edge(nn, j == nx - 1);
    split_boundary(rem, diag[r], nb, r, bnd, nb);
  }
  // element fields for the coarse levels: kappa_T from the mean of its interior vertices'
  // K_aa / 4, S_T from their 2 M_aa / h^2 (exact for uniform fields)
  const int nc = nps - 1;
  const int64_t nelem = 2 * (int64_t)nc * nc;
  std::vector<double> lk(nelem), ls(nelem);
  auto node = [&](int I, int J, double& kv, double& sv, int& cnt) {
    if (I <= 0 || J <= 0 || I >= nps - 1 || J >= nps - 1) return;
    const int64_t a = (int64_t)(J - 1) * nx + (I - 1);
    kv += diag[a] / 4.0;
    sv += 2.0 * Mn[a] / h2;
    ++cnt;
  };
  for (int cj = 0; cj < nc; ++cj)
    for (int ci = 0; ci < nc; ++ci)
      for (int up = 0; up < 2; ++up) {
        double kv = 0.0, sv = 0.0;
        int cnt = 0;
        node(ci, cj, kv, sv, cnt);
        node(ci + 1, cj + 1, kv, sv, cnt);
        if (up) node(ci, cj + 1, kv, sv, cnt);
        else node(ci + 1, cj, kv, sv, cnt);
        const int64_t el = 2 * ((int64_t)cj * nc + ci) + up;
        lk[el] = std::log(std::max(kv / std::max(cnt, 1), 1e-300));
        ls[el] = std::log(std::max(sv / std::max(cnt, 1), 1e-300));
      }
  pencil_build_p1(p, lk.data(), ls.data(), LT_MEM_HOST);
  // the finest level is the given operator
  Level& F = *p->levels[0];
  LT_CUDA(cudaMemcpyAsync(F.Tx, Tx.data(), sizeof(double) * nfx, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(F.Ty, Ty.data(), sizeof(double) * nfy, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(F.M, Mn.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(F.Mx, Mx.data(), sizeof(double) * nfx, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(F.My, My.data(), sizeof(double) * nfy, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(F.Md, Mdg.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
  make_fp32_copies(p);
  LT_CUDA(cudaStreamSynchronize(st));
  (void)h2;
}

}  // namespace lt

lt::LevelView lt_pencil_s::view(int l) const { return lt::lt_pencil_view(this, l); }
lt::LevelView32 lt_pencil_s::view32(int l) const { return lt::lt_pencil_view32(this, l); }

cudaGraphExec_t lt_pencil_s::graph_exec(cudaGraph_t g) {
  if (inner_exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(inner_exec, g, &info) == cudaSuccess) return inner_exec;
    cudaGetLastError();
    cudaGraphExecDestroy(inner_exec);
    inner_exec = nullptr;
  }
  LT_CUDA(cudaGraphInstantiate(&inner_exec, g, 0));
  return inner_exec;
}

lt_pencil_s::~lt_pencil_s() {
  if (inner_exec) cudaGraphExecDestroy(inner_exec);
}

const lt::CoarseFactor& lt_pencil_s::factor(double2 tau) {
  for (auto& f : factors)
    if (f->tau.x == tau.x && f->tau.y == tau.y) return *f;
  using namespace lt;
  const int lc = (int)levels.size() - 1;
  LevelView L = view(lc);
  const int64_t nc = L.n;
  if (nc > 8192) throw Error(LT_ERR_PRECONDITIONER, "coarsest multigrid level too large for a dense inverse");
  cudaStream_t st = ctx->stream;
  auto f = std::make_unique<CoarseFactor>();
  f->tau = tau;
  f->inverse.allocate(sizeof(double2) * nc * 2 * nc, st);
  double2* aug = f->inverse.as<double2>();
  launch(ctx, "coarse_factor", 0.0, [&] {
    dense_coarse<<<blocks_for(nc * 2 * nc, kThreads), kThreads, 0, st>>>(L, tau, aug);
  });
  // A^{-1} by LU (cuSOLVER getrf + getrs on the identity).  A = K_c + tau M_c is complex
  // symmetric, so its row-major and column-major forms coincide, and so do A^{-1}'s.
  {
    cusolverDnHandle_t h = ctx->solver_handle();
    DeviceBuffer A(sizeof(double2) * nc * nc, st), X(sizeof(double2) * nc * nc, st), piv(sizeof(int) * (nc + 1), st);
    LT_CUDA(cudaMemcpy2DAsync(A.get(), sizeof(double2) * nc, aug, sizeof(double2) * 2 * nc, sizeof(double2) * nc, nc,
                              cudaMemcpyDeviceToDevice, st));
    LT_CUDA(cudaMemcpy2DAsync(X.get(), sizeof(double2) * nc, aug + nc, sizeof(double2) * 2 * nc, sizeof(double2) * nc,
                              nc, cudaMemcpyDeviceToDevice, st));
    int lwork = 0;
    auto* Ac = reinterpret_cast<cuDoubleComplex*>(A.get());
    auto* Xc = reinterpret_cast<cuDoubleComplex*>(X.get());
    if (cusolverDnZgetrf_bufferSize(h, (int)nc, (int)nc, Ac, (int)nc, &lwork) != CUSOLVER_STATUS_SUCCESS)
      throw Error(LT_ERR_CUDA, "cusolverDnZgetrf_bufferSize failed");
    DeviceBuffer work(sizeof(cuDoubleComplex) * std::max(lwork, 1), st);
    int* info = piv.as<int>() + nc;
    if (cusolverDnZgetrf(h, (int)nc, (int)nc, Ac, (int)nc, work.as<cuDoubleComplex>(), piv.as<int>(), info) !=
            CUSOLVER_STATUS_SUCCESS ||
        cusolverDnZgetrs(h, CUBLAS_OP_N, (int)nc, (int)nc, Ac, (int)nc, piv.as<int>(), Xc, (int)nc, info) !=
            CUSOLVER_STATUS_SUCCESS)
      throw Error(LT_ERR_CUDA, "cuSOLVER coarse factorization failed");
    int h_status = 0;
    LT_CUDA(cudaMemcpyAsync(&h_status, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (h_status != 0)
      throw Error(LT_ERR_PRECONDITIONER, "shift-and-invert factorization failed (singular coarse operator)");
    LT_CUDA(cudaMemcpy2DAsync(aug + nc, sizeof(double2) * 2 * nc, X.get(), sizeof(double2) * nc, sizeof(double2) * nc,
                              nc, cudaMemcpyDeviceToDevice, st));
  }
  f->inverse32.allocate(sizeof(float2) * nc * nc, st);
  launch(ctx, "coarse_factor", 0.0, [&] {
    inverse_to_c64<<<blocks_for(nc * nc, kThreads), kThreads, 0, st>>>(aug, f->inverse32.as<float2>(), nc);
  });
  LT_CUDA(cudaStreamSynchronize(st));
  factors.push_back(std::move(f));
  return *factors.back();
}

namespace lt {

namespace {

template <int DIM, bool MASS_ONLY>
__global__ void apply_kernel(LevelView L, const double2* __restrict__ taus, const double2* __restrict__ x,
                             int64_t xs, double2* __restrict__ y, int64_t ys, int B) {
  LT_ITEM_BLOCK(B, b, cb);
  int i, j, k;
  int64_t a;
  if (!tile_cell(L, cb, i, j, k, a)) return;
  const double2* xb = x + b * xs;
  double2 out;
  if (MASS_ONLY) out = mass_apply(L, xb, a, i, j);
  else out = stencil_apply<DIM>(L, xb, a, i, j, k, taus[b]);
  y[b * ys + a] = out;
}

}  // namespace

void apply_batch(lt_pencil p, int level, const double2* taus_dev, const double2* x, int64_t xs,
                 double2* y, int64_t ys, int B, bool mass_only, const char* name) {
  LevelView L = p->view(level);
  cudaStream_t st = p->ctx->stream;
  unsigned grid = (unsigned)L.ntiles * (unsigned)B;
  double bytes = mass_only ? (double)L.n * (32.0 * B + 8.0) : (double)L.n * (32.0 * B + 8.0 * (p->dim + 1));
  launch(p->ctx, name, bytes, [&] {
    if (mass_only) {
      if (p->dim == 3) apply_kernel<3, true><<<grid, kThreads, 0, st>>>(L, taus_dev, x, xs, y, ys, B);
      else apply_kernel<2, true><<<grid, kThreads, 0, st>>>(L, taus_dev, x, xs, y, ys, B);
    } else {
      if (p->dim == 3) apply_kernel<3, false><<<grid, kThreads, 0, st>>>(L, taus_dev, x, xs, y, ys, B);
      else apply_kernel<2, false><<<grid, kThreads, 0, st>>>(L, taus_dev, x, xs, y, ys, B);
    }
  });
}

// P1 barycentric weights of the containing triangle (point_source, mesh.cpp:91-125),
// restricted to the free (interior) nodes (restrict_to_free, assembly.cpp:45-51).
static void point_weights_p1(const lt_pencil_s* p, const double* point, int64_t* idx, double* w, int* count) {
  const int n = p->grid.shape[0];
  const double h = p->grid.h;
  const double L = h * (n - 1);
  const double tol = 1e-12 * L;
  double x = point[0], y = point[1];
  if (x < -tol || x > L + tol || y < -tol || y > L + tol)
    throw Error(LT_ERR_INVALID_ARGUMENT, "point_source: point lies outside the domain");
  x = std::min(std::max(x, 0.0), L);
  y = std::min(std::max(y, 0.0), L);
  const int ci = std::min((int)std::floor(x / h), n - 2);
  const int cj = std::min((int)std::floor(y / h), n - 2);
  const double xi = x / h - ci, eta = y / h - cj;
  int nodes[3][2];
  double ws[3];
  if (xi >= eta) {  // lower triangle (a, b, c)
    nodes[0][0] = ci; nodes[0][1] = cj; ws[0] = 1.0 - xi;
    nodes[1][0] = ci + 1; nodes[1][1] = cj; ws[1] = xi - eta;
    nodes[2][0] = ci + 1; nodes[2][1] = cj + 1; ws[2] = eta;
  } else {  // upper triangle (a, c, d)
    nodes[0][0] = ci; nodes[0][1] = cj; ws[0] = 1.0 - eta;
    nodes[1][0] = ci + 1; nodes[1][1] = cj + 1; ws[1] = xi;
    nodes[2][0] = ci; nodes[2][1] = cj + 1; ws[2] = eta - xi;
  }
  int c = 0;
  for (int q = 0; q < 3; ++q) {
    const int I = nodes[q][0], J = nodes[q][1];
    if (ws[q] == 0.0 || I <= 0 || J <= 0 || I >= n - 1 || J >= n - 1) continue;  // Dirichlet or zero
    idx[c] = (int64_t)(J - 1) * (n - 2) + (I - 1);
    w[c] = ws[q];
    ++c;
  }
  *count = c;
}

void point_weights(const lt_pencil_s* p, const double* point, int64_t* idx, double* w, int* count) {
  if (p->kind == LT_GRID_P1_TRI) {
    point_weights_p1(p, point, idx, w, count);
    return;
  }
  const int dim = p->dim;
  int base[3] = {0, 0, 0};
  double frac[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) {
    const int n = p->grid.shape[d];
    double xi = point[d] / p->grid.h - 0.5;
    const double tol = 1e-12 * n;
    if (xi < -tol || xi > (n - 1) + tol)
      throw Error(LT_ERR_INVALID_ARGUMENT, "point_weights: point lies outside the cell-centre hull");
    xi = std::min(std::max(xi, 0.0), double(n - 1));
    int i0 = std::min((int)std::floor(xi), std::max(n - 2, 0));
    base[d] = i0;
    frac[d] = xi - i0;
  }
  int c = 0;
  for (int corner = 0; corner < (1 << dim); ++corner) {
    double weight = 1.0;
    int64_t flat = 0, stride = 1;
    for (int d = 0; d < dim; ++d) {
      int bit = (corner >> d) & 1;
      weight *= bit ? frac[d] : 1.0 - frac[d];
      flat += (int64_t)(base[d] + bit) * stride;
      stride *= p->grid.shape[d];
    }
    if (weight == 0.0) continue;
    // merge duplicates (degenerate 1-cell directions)
    bool merged = false;
    for (int q = 0; q < c; ++q)
      if (idx[q] == flat) { w[q] += weight; merged = true; break; }
    if (!merged) { idx[c] = flat; w[c] = weight; ++c; }
  }
  *count = c;
}

}  // namespace lt
