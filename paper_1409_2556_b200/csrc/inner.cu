// The shift-and-invert preconditioner solve u = (K + tau M)^{-1} v on the device.
//
// Reference: SparseComplexFactorization::solve on an Eigen SparseLU<COLAMD> of K + tau M
// (factorization.cpp:14-33, used at shifted_solver.cpp:192-193), exact to ~1e-15.  The LU
// fill of K + tau M is infeasible in HBM for the 3-D configs, so the same
// operator is inverted to tolerance instead: COCG (conjugate-orthogonal CG for the complex
// symmetric K + tau M) in FP64, preconditioned by a symmetric cell-centred multigrid V-cycle
// (red-black Gauss-Seidel, multilinear prolongation, R = P^T, rediscretised coarse faces,
// exact dense inverse of the coarsest operator per tau).  The V-cycle runs in FP32 (complex64
// vectors, FP32 copies of the faces; -DLT_MG_FP64 selects FP64): it only has to approximate
// the inverse, while the FP64 COCG recursion (r -= alpha A p with the FP64 operator) keeps the
// solve exact to the 1e-12 tolerance.  B right-hand sides (each its own tau) run in lockstep.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "lt_internal.hpp"
#include "stencil.cuh"

namespace lt {

namespace {

// LT_INNER_TRACE=1: chunking of each inner solve; =2 also the per-item final relative
// residual (diagnostics only)
int inner_trace() {
  static const int level = std::getenv("LT_INNER_TRACE") ? std::atoi(std::getenv("LT_INNER_TRACE")) : 0;
  return level;
}

constexpr int kT = 256;

#ifdef LT_MG_FP64
using MgReal = double;
#else
using MgReal = float;
#endif

template <class R> struct CT;
template <> struct CT<double> { using V = double2; };
template <> struct CT<float> { using V = float2; };

template <class V> __device__ __forceinline__ V vzero() { return V{0, 0}; }
template <class V> __device__ __forceinline__ V vadd(V a, V b) { return V{a.x + b.x, a.y + b.y}; }
template <class V> __device__ __forceinline__ V vsub(V a, V b) { return V{a.x - b.x, a.y - b.y}; }
template <class V, class R> __device__ __forceinline__ V vscale(V a, R s) { return V{a.x * s, a.y * s}; }
template <class V> __device__ __forceinline__ V vfrom(double2 a) {
  return V{static_cast<decltype(V::x)>(a.x), static_cast<decltype(V::x)>(a.y)};
}
template <class V> __device__ __forceinline__ double2 vto(V a) { return make_double2((double)a.x, (double)a.y); }

template <class T>
__device__ __forceinline__ T warp_sum(T v);
template <>
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffff, v, o);
  return v;
}
template <>
__device__ __forceinline__ double2 warp_sum(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffff, v.x, o);
    v.y += __shfl_down_sync(0xffffffff, v.y, o);
  }
  return v;
}
template <>
__device__ __forceinline__ float2 warp_sum(float2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffff, v.x, o);
    v.y += __shfl_down_sync(0xffffffff, v.y, o);
  }
  return v;
}

// Block-wide sum; result valid in thread 0.
template <class T>
__device__ __forceinline__ T block_sum(T v) {
  __shared__ T sh[32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? sh[lane] : T{};
    v = warp_sum(v);
  }
  return v;
}

struct Batch {
  int B;            // items in the batch
  const int* done;  // per item: 1 -> skip
};

#define TILE_PROLOGUE(LV)                  \
  LT_ITEM_BLOCK(bt.B, b, cb)               \
  if (bt.done[b]) return;                   \
  int i, j, k;                              \
  int64_t a;                                \
  const bool in = tile_cell(LV, cb, i, j, k, a);

#define ITEM_PROLOGUE(n)                                          \
  LT_ITEM_BLOCK(bt.B, b, cb)                                      \
  if (bt.done[b]) return;                                         \
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;       \
  const bool in = a < (n);

// (dk + tau m)^{-1} rhs in precision R with one real division
template <class R, class V>
__device__ __forceinline__ V diag_solve_r(R dk, R m, R tr, R ti, V rhs) {
  const R dr = dk + tr * m, di = ti * m;
  const R inv = R(1) / (dr * dr + di * di);
  return V{(rhs.x * dr + rhs.y * di) * inv, (rhs.y * dr - rhs.x * di) * inv};
}

// ---- multigrid kernels (precision R) ---------------------------------------------------

// 1-D cell-centred linear interpolation weight P[f, I] (aggregation 2, Dirichlet ghost = -e).
__device__ __forceinline__ int p1d_terms(int fi, int agg, int nc, int* I, float* w) {
  if (agg == 1) { I[0] = fi; w[0] = 1.0f; return 1; }
  const int c = fi >> 1;
  if ((fi & 1) == 0) {
    if (c == 0) { I[0] = 0; w[0] = 0.5f; return 1; }
    I[0] = c; w[0] = 0.75f; I[1] = c - 1; w[1] = 0.25f; return 2;
  }
  if (c == nc - 1) { I[0] = c; w[0] = 0.5f; return 1; }
  I[0] = c; w[0] = 0.75f; I[1] = c + 1; w[1] = 0.25f; return 2;
}

// Transpose weights: fine cells contributing to coarse I along one direction.
__device__ __forceinline__ int r1d_terms(int I, int agg, int nc, int* F, float* w) {
  if (agg == 1) { F[0] = I; w[0] = 1.0f; return 1; }
  int n = 0;
  if (I > 0) { F[n] = 2 * I - 1; w[n] = 0.25f; ++n; }
  F[n] = 2 * I; w[n] = I == 0 ? 0.5f : 0.75f; ++n;
  F[n] = 2 * I + 1; w[n] = I == nc - 1 ? 0.5f : 0.75f; ++n;
  if (I < nc - 1) { F[n] = 2 * I + 2; w[n] = 0.25f; ++n; }
  return n;
}

// r = f - A(tau) x
template <class R, int DIM>
__global__ void __launch_bounds__(kT) residual_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                      const typename CT<R>::V* __restrict__ f,
                                                      const typename CT<R>::V* __restrict__ x,
                                                      typename CT<R>::V* __restrict__ r) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(L);
  if (!in) return;
  const V* xb = x + (int64_t)b * L.n;
  const int64_t ex = fx(L, i, j, k), ey = fy(L, i, j, k);
  const R tw = __ldg(L.Tx + ex), te = __ldg(L.Tx + ex + 1);
  const R ts = __ldg(L.Ty + ey), tn = __ldg(L.Ty + ey + L.nx);
  R dk = tw + te + ts + tn;
  V o = vzero<V>();
  if (i > 0) o = vadd(o, vscale(xb[a - 1], tw));
  if (i < L.nx - 1) o = vadd(o, vscale(xb[a + 1], te));
  if (j > 0) o = vadd(o, vscale(xb[a - L.nx], ts));
  if (j < L.ny - 1) o = vadd(o, vscale(xb[a + L.nx], tn));
  if (DIM == 3) {
    const int64_t plane = (int64_t)L.nx * L.ny;
    const R tb = __ldg(L.Tz + a), tt = __ldg(L.Tz + a + plane);
    dk += tb + tt;
    if (k > 0) o = vadd(o, vscale(xb[a - plane], tb));
    if (k < L.nz - 1) o = vadd(o, vscale(xb[a + plane], tt));
  }
  const double2 tau = taus[b];
  const R m = __ldg(L.M + a);
  const R dr = dk + (R)tau.x * m, di = (R)tau.y * m;
  const V xa = xb[a];
  const V ax = V{dr * xa.x - di * xa.y - o.x, dr * xa.y + di * xa.x - o.y};
  r[(int64_t)b * L.n + a] = vsub(f[(int64_t)b * L.n + a], ax);
}

template <class R, int DIM>
__global__ void __launch_bounds__(kT) restrict_kernel(LevelViewT<R> Lf, LevelViewT<R> Lc, int ax, int ay, int az,
                                                      Batch bt, const typename CT<R>::V* __restrict__ rf,
                                                      typename CT<R>::V* __restrict__ fc) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(Lc);
  if (!in) return;
  int Fx[4], Fy[4], Fz[4];
  float wx[4], wy[4], wz[4];
  const int nxx = r1d_terms(i, ax, Lc.nx, Fx, wx);
  const int nyy = r1d_terms(j, ay, Lc.ny, Fy, wy);
  int nzz = 1;
  Fz[0] = 0; wz[0] = 1.0f;
  if (DIM == 3) nzz = r1d_terms(k, az, Lc.nz, Fz, wz);
  const V* rb = rf + (int64_t)b * Lf.n;
  V s = vzero<V>();
  for (int q = 0; q < nzz; ++q)
    for (int p = 0; p < nyy; ++p) {
      const R wzy = (R)(wz[q] * wy[p]);
      const int64_t row = ((int64_t)Fz[q] * Lf.ny + Fy[p]) * Lf.nx;
      for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(rb[row + Fx[o]], wzy * (R)wx[o]));
    }
  fc[(int64_t)b * Lc.n + a] = s;
}

template <class R, class V>
__device__ __forceinline__ V prolong_at(const LevelViewT<R>& Lc, int ax, int ay, int az, const V* __restrict__ eb,
                                        int i, int j, int k, int dim) {
  int Ix[2], Iy[2], Iz[2];
  float wx[2], wy[2], wz[2];
  const int nxx = p1d_terms(i, ax, Lc.nx, Ix, wx);
  const int nyy = p1d_terms(j, ay, Lc.ny, Iy, wy);
  int nzz = 1;
  Iz[0] = 0; wz[0] = 1.0f;
  if (dim == 3) nzz = p1d_terms(k, az, Lc.nz, Iz, wz);
  V s = vzero<V>();
  for (int q = 0; q < nzz; ++q)
    for (int p = 0; p < nyy; ++p) {
      const R wzy = (R)(wz[q] * wy[p]);
      const int64_t row = ((int64_t)Iz[q] * Lc.ny + Iy[p]) * Lc.nx;
      for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(eb[row + Ix[o]], wzy * (R)wx[o]));
    }
  return s;
}

// ---- fused red-black Gauss-Seidel sweep ------------------------------------------------
// One full sweep (colour `first`, then the other colour) of a 32 x 8 (x, y) tile, marching
// through z: x planes (halo 2) in a 5-slot shared-memory ring and f planes (halo 1) in a
// 3-slot ring are filled one step ahead with cp.async; the first colour is updated on the
// tile + 1-cell halo (from old second-colour values), the second colour on the tile (from
// the new first-colour values).  Each cell of x and f is read from HBM once and x is written
// once.  zero_init: the iterate is zero on entry.  ec != null: the iterate is xin + P ec
// (fused coarse-grid correction).  Out of place (x != xin): halos of neighbouring tiles read xin.
constexpr int SW_TX = 32, SW_TY = 8, SW_HX = SW_TX + 4, SW_HY = SW_TY + 4, SW_PL = SW_HX * SW_HY;
constexpr int SW_FX = SW_TX + 2, SW_FPL = SW_FX * (SW_TY + 2);

template <class V>
__device__ __forceinline__ void cp_async_v(void* dst, const void* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  if (sizeof(V) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}

template <class R, int DIM>
__global__ void __launch_bounds__(kT) rb_sweep_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                      const typename CT<R>::V* __restrict__ f,
                                                      const typename CT<R>::V* __restrict__ xin,
                                                      typename CT<R>::V* __restrict__ x, int first, int zero_init,
                                                      LevelViewT<R> Lc, int ax, int ay, int az,
                                                      const typename CT<R>::V* __restrict__ ec) {
  using V = typename CT<R>::V;
  constexpr int NS = DIM == 3 ? 5 : 1;
  extern __shared__ __align__(16) unsigned char sw_raw[];
  V (*U)[SW_PL] = reinterpret_cast<V (*)[SW_PL]>(sw_raw);
  V (*Fr)[SW_FPL] = reinterpret_cast<V (*)[SW_FPL]>(sw_raw + sizeof(V) * NS * SW_PL);
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int tiles_x = (L.nx + SW_TX - 1) / SW_TX;
  const int i0 = (cb % tiles_x) * SW_TX, j0 = (cb / tiles_x) * SW_TY;
  const int tid = threadIdx.x;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  const V* fb = f + (int64_t)b * L.n;
  V* xb = x + (int64_t)b * L.n;
  const V* xib = zero_init ? nullptr : xin + (int64_t)b * L.n;
  const V* eb = ec ? ec + (int64_t)b * Lc.n : nullptr;
  const int64_t plane = (int64_t)L.nx * L.ny;
  const int second = first ^ 1;
  auto slot = [](int k) { return DIM == 3 ? k % 5 : 0; };
  auto fslot = [](int k) { return DIM == 3 ? k % 3 : 0; };
  auto commit = [] { asm volatile("cp.async.commit_group;\n" ::); };
  auto wait1 = [] { asm volatile("cp.async.wait_group 1;\n" ::); };
  auto wait0 = [] { asm volatile("cp.async.wait_group 0;\n" ::); };

  auto issue_x = [&](int k) {
    V* S = U[slot(k)];
    for (int e = tid; e < SW_PL; e += kT) {
      const int i = i0 - 2 + e % SW_HX, j = j0 - 2 + e / SW_HX;
      if (zero_init) {
        S[e] = vzero<V>();
      } else {
        const bool ok = i >= 0 && i < L.nx && j >= 0 && j < L.ny;
        cp_async_v<V>(S + e, ok ? xib + (k * plane + (int64_t)j * L.nx + i) : xib, ok);
      }
    }
  };
  auto issue_f = [&](int k) {
    V* S = Fr[fslot(k)];
    for (int e = tid; e < SW_FPL; e += kT) {
      const int i = i0 - 1 + e % SW_FX, j = j0 - 1 + e / SW_FX;
      const bool ok = i >= 0 && i < L.nx && j >= 0 && j < L.ny;
      cp_async_v<V>(S + e, ok ? fb + (k * plane + (int64_t)j * L.nx + i) : fb, ok);
    }
  };
  auto add_prolong = [&](int k) {
    V* S = U[slot(k)];
    for (int e = tid; e < SW_PL; e += kT) {
      const int i = i0 - 2 + e % SW_HX, j = j0 - 2 + e / SW_HX;
      if (i >= 0 && i < L.nx && j >= 0 && j < L.ny) S[e] = vadd(S[e], prolong_at(Lc, ax, ay, az, eb, i, j, k, DIM));
    }
  };
  // Gauss-Seidel update of colour `color` on plane k over the tile grown by H cells: one
  // thread per cell of that colour (i0, j0 even, so the colour parity of a row is known),
  // compile-time region widths, 32-bit in-plane indices.
  const int nxp1 = L.nx + 1;
  auto update = [&](int k, int color, auto Hc) {
    constexpr int H = decltype(Hc)::value;
    constexpr int RX = SW_TX + 2 * H, RY = SW_TY + 2 * H, HALF = RX / 2;
    if (tid >= RY * HALF) return;
    const int lj = tid / HALF - H;
    const int par = (color + lj + k) & 1;
    const int li = -H + ((par + H) & 1) + 2 * (tid % HALF);
    const int i = i0 + li, j = j0 + lj;
    if (i < 0 || i >= L.nx || j < 0 || j >= L.ny) return;
    V* S = U[slot(k)];
    const V* Fk = Fr[fslot(k)];
    const int s = (lj + 2) * SW_HX + (li + 2);
    const int ip = j * L.nx + i;                       // in-plane cell index
    const R* Txk = L.Tx + (int64_t)k * L.ny * nxp1;     // plane k of the x faces
    const R* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx;
    const int ex = j * nxp1 + i, ey = ip;
    const R tw = __ldg(Txk + ex), te = __ldg(Txk + ex + 1);
    const R ts = __ldg(Tyk + ey), tn = __ldg(Tyk + ey + L.nx);
    R dk = tw + te + ts + tn;
    V o = Fk[(lj + 1) * SW_FX + (li + 1)];
    if (i > 0) o = vadd(o, vscale(S[s - 1], tw));
    if (i < L.nx - 1) o = vadd(o, vscale(S[s + 1], te));
    if (j > 0) o = vadd(o, vscale(S[s - SW_HX], ts));
    if (j < L.ny - 1) o = vadd(o, vscale(S[s + SW_HX], tn));
    const int64_t a = k * plane + ip;
    if (DIM == 3) {
      const R tb = __ldg(L.Tz + a), tt = __ldg(L.Tz + a + plane);
      dk += tb + tt;
      if (k > 0) o = vadd(o, vscale(U[slot(k - 1)][s], tb));
      if (k < L.nz - 1) o = vadd(o, vscale(U[slot(k + 1)][s], tt));
    }
    S[s] = diag_solve_r<R, V>(dk, __ldg(L.M + a), tr, ti, o);
  };
  using H1 = std::integral_constant<int, 1>;
  using H0 = std::integral_constant<int, 0>;
  auto store_plane = [&](int k) {
    const V* S = U[slot(k)];
    const int li = tid % SW_TX, lj = tid / SW_TX;
    const int i = i0 + li, j = j0 + lj;
    if (i < L.nx && j < L.ny) xb[k * plane + (int64_t)j * L.nx + i] = S[(lj + 2) * SW_HX + (li + 2)];
  };

  if (DIM == 2) {
    issue_x(0);
    issue_f(0);
    commit();
    wait0();
    __syncthreads();
    if (eb) {
      add_prolong(0);
      __syncthreads();
    }
    update(0, first, H1{});
    __syncthreads();
    update(0, second, H0{});
    __syncthreads();
    store_plane(0);
    return;
  }
  // prologue: group A = {x0, x1, f0}, group B = {x2, f1}
  issue_x(0);
  if (L.nz > 1) issue_x(1);
  issue_f(0);
  commit();
  if (L.nz > 2) issue_x(2);
  if (L.nz > 1) issue_f(1);
  commit();
  wait1();
  __syncthreads();
  if (eb) {
    add_prolong(0);
    if (L.nz > 1) add_prolong(1);
    __syncthreads();
  }
  update(0, first, H1{});
  for (int k = 0; k < L.nz; ++k) {
    // prefetch x(k+3), f(k+2); then wait for x(k+2), f(k+1) issued one step earlier
    if (k + 3 < L.nz) issue_x(k + 3);
    if (k + 2 < L.nz) issue_f(k + 2);
    commit();
    wait1();
    __syncthreads();
    if (eb && k + 2 < L.nz) {
      add_prolong(k + 2);
      __syncthreads();
    }
    if (k + 1 < L.nz) update(k + 1, first, H1{});
    __syncthreads();
    update(k, second, H0{});
    __syncthreads();
    store_plane(k);
  }
  wait0();
}

template <class R>
size_t sweep_smem(int dim) {
  using V = typename CT<R>::V;
  return sizeof(V) * ((dim == 3 ? 5 : 1) * SW_PL + (dim == 3 ? 3 : 1) * SW_FPL);
}

// e = A_c(tau_b)^{-1} f: one warp per row of the dense complex inverse (row stride ld, column
// offset off).
template <class V>
__global__ void __launch_bounds__(kT) coarse_solve_kernel(int nc, Batch bt, const V* const* __restrict__ inv,
                                                          int64_t ld, int64_t off, const V* __restrict__ f,
                                                          V* __restrict__ e) {
  const int b = blockIdx.y;
  if (bt.done[b]) return;
  const int row = blockIdx.x * (kT / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= nc) return;
  const V* Ar = inv[b] + (int64_t)row * ld + off;
  const V* fb = f + (int64_t)b * nc;
  V s = vzero<V>();
  for (int c = lane; c < nc; c += 32) {
    const V m = Ar[c], x = fb[c];
    s = V{s.x + m.x * x.x - m.y * x.y, s.y + m.x * x.y + m.y * x.x};
  }
  s = warp_sum(s);
  if (lane == 0) e[(int64_t)b * nc + row] = s;
}

// ---- COCG vector kernels (FP64, fused with their reductions) ----------------------------
using VM = CT<MgReal>::V;

// r = v, rmg = (VM) v, partial ||v||^2
__global__ void __launch_bounds__(kT) copy_norm_kernel(int64_t n, Batch bt, const double2* __restrict__ v, int64_t vs,
                                                       double2* __restrict__ r, VM* __restrict__ rmg,
                                                       double* __restrict__ part, int nblk) {
  ITEM_PROLOGUE(n);
  double s = 0.0;
  if (in) {
    const double2 x = v[b * vs + a];
    r[b * n + a] = x;
    rmg[b * n + a] = vfrom<VM>(x);
    s = cabs2(x);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// partial sum_a r_a z_a (bilinear, no conjugation), z from the V-cycle
__global__ void __launch_bounds__(kT) bdot_kernel(int64_t n, Batch bt, const double2* __restrict__ x,
                                                  const VM* __restrict__ y, double2* __restrict__ part, int nblk) {
  ITEM_PROLOGUE(n);
  double2 s = make_double2(0.0, 0.0);
  if (in) s = cmul(x[b * n + a], vto(y[b * n + a]));
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// ---- z-marching 7-point kernels (3-D) -------------------------------------------------
// CTA = 32 x 8 (x, y) tile x a chunk of ZM_ZC planes; each thread keeps its column's
// x[k-1], x[k], x[k+1] in registers (x[k+2] prefetched one step ahead), so every value of x
// is read from HBM once; in-plane neighbours come from L1.
constexpr int ZM_TX = 32, ZM_TY = 8, ZM_ZC = 32;

struct ZmMap {
  int i, j, k0, k1, ip;
  bool in;
};

template <class VW>
__device__ __forceinline__ ZmMap zm_map(const VW& L, int cb) {
  const int tiles_x = (L.nx + ZM_TX - 1) / ZM_TX, tiles_y = (L.ny + ZM_TY - 1) / ZM_TY;
  const int ntile = tiles_x * tiles_y;
  const int tile = cb % ntile, chunk = cb / ntile;
  ZmMap m;
  m.i = (tile % tiles_x) * ZM_TX + (threadIdx.x & (ZM_TX - 1));
  m.j = (tile / tiles_x) * ZM_TY + (threadIdx.x / ZM_TX);
  m.in = m.i < L.nx && m.j < L.ny;
  m.k0 = chunk * ZM_ZC;
  m.k1 = min(L.nz, m.k0 + ZM_ZC);
  m.ip = m.j * L.nx + m.i;
  return m;
}

template <class VW>
inline int zm_blocks(const VW& L) {
  return ((L.nx + ZM_TX - 1) / ZM_TX) * ((L.ny + ZM_TY - 1) / ZM_TY) * ((L.nz + ZM_ZC - 1) / ZM_ZC);
}

// r = f - A(tau) x (precision R), z-marching
template <class R>
__global__ void __launch_bounds__(kT) residual_zm_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                         const typename CT<R>::V* __restrict__ f,
                                                         const typename CT<R>::V* __restrict__ x,
                                                         typename CT<R>::V* __restrict__ r) {
  using V = typename CT<R>::V;
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZmMap m = zm_map(L, cb);
  if (!m.in) return;
  const int64_t plane = (int64_t)L.nx * L.ny;
  const V* xb = x + (int64_t)b * L.n;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  const int nxp1 = L.nx + 1;
  const V* fb = f + (int64_t)b * L.n;
  V xm = m.k0 > 0 ? xb[(m.k0 - 1) * plane + m.ip] : vzero<V>();
  V xc = xb[m.k0 * plane + m.ip];
  V xp = m.k0 + 1 < L.nz ? xb[(m.k0 + 1) * plane + m.ip] : vzero<V>();
  struct Ops {
    R tw, te, ts, tn, tb, tt, mm;
    V f, nw, ne, ns, nn;
  };
  auto load_ops = [&](int k, Ops& o) {
    const int64_t a = k * plane + m.ip;
    const R* Txk = L.Tx + (int64_t)k * L.ny * nxp1;
    const R* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx;
    const int ex = m.j * nxp1 + m.i;
    o.tw = __ldg(Txk + ex);
    o.te = __ldg(Txk + ex + 1);
    o.ts = __ldg(Tyk + m.ip);
    o.tn = __ldg(Tyk + m.ip + L.nx);
    o.tb = __ldg(L.Tz + a);
    o.tt = __ldg(L.Tz + a + plane);
    o.mm = __ldg(L.M + a);
    o.f = fb[a];
    o.nw = m.i > 0 ? xb[a - 1] : vzero<V>();
    o.ne = m.i < L.nx - 1 ? xb[a + 1] : vzero<V>();
    o.ns = m.j > 0 ? xb[a - L.nx] : vzero<V>();
    o.nn = m.j < L.ny - 1 ? xb[a + L.nx] : vzero<V>();
  };
  Ops cur, nxt;
  load_ops(m.k0, cur);
  for (int k = m.k0; k < m.k1; ++k) {
    const V xn = (k + 1 < m.k1 && k + 2 < L.nz) ? xb[(k + 2) * plane + m.ip] : vzero<V>();
    if (k + 1 < m.k1) load_ops(k + 1, nxt);
    const int64_t a = k * plane + m.ip;
    const R dk = cur.tw + cur.te + cur.ts + cur.tn + cur.tb + cur.tt;
    V o = vadd(vadd(vscale(cur.nw, cur.tw), vscale(cur.ne, cur.te)), vadd(vscale(cur.ns, cur.ts), vscale(cur.nn, cur.tn)));
    if (k > 0) o = vadd(o, vscale(xm, cur.tb));
    if (k < L.nz - 1) o = vadd(o, vscale(xp, cur.tt));
    const R dr = dk + tr * cur.mm, di = ti * cur.mm;
    const V ax = V{dr * xc.x - di * xc.y - o.x, dr * xc.y + di * xc.x - o.y};
    r[(int64_t)b * L.n + a] = vsub(cur.f, ax);
    xm = xc;
    xc = xp;
    xp = xn;
    cur = nxt;
  }
}

// One red-black Gauss-Seidel half sweep of colour `color`, in place and z-marching: a cell of
// that colour reads only other-colour neighbours, which this launch does not change, so the
// in-place update is race free; every cell is written (other colour unchanged) so stores are
// full sectors.  zero_init: x = 0 on entry (colour cells get f/d, the others 0, x not read).
template <class R>
__global__ void __launch_bounds__(kT) rbhalf_zm_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                       const typename CT<R>::V* __restrict__ f,
                                                       typename CT<R>::V* x, int color, int zero_init) {
  using V = typename CT<R>::V;
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZmMap m = zm_map(L, cb);
  if (!m.in) return;
  const int64_t plane = (int64_t)L.nx * L.ny;
  V* xb = x + (int64_t)b * L.n;
  const V* fb = f + (int64_t)b * L.n;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  const int nxp1 = L.nx + 1;
  V xm = vzero<V>(), xc = vzero<V>(), xp = vzero<V>();
  if (!zero_init) {
    xm = m.k0 > 0 ? xb[(m.k0 - 1) * plane + m.ip] : vzero<V>();
    xc = xb[m.k0 * plane + m.ip];
    xp = m.k0 + 1 < L.nz ? xb[(m.k0 + 1) * plane + m.ip] : vzero<V>();
  }
  // operands of the colour cell of plane k, loaded one step ahead (software pipeline)
  struct Ops {
    R tw, te, ts, tn, tb, tt, mm;
    V f, nw, ne, ns, nn;
  };
  auto load_ops = [&](int k, Ops& o) {
    const int64_t a = k * plane + m.ip;
    const R* Txk = L.Tx + (int64_t)k * L.ny * nxp1;
    const R* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx;
    const int ex = m.j * nxp1 + m.i;
    o.tw = __ldg(Txk + ex);
    o.te = __ldg(Txk + ex + 1);
    o.ts = __ldg(Tyk + m.ip);
    o.tn = __ldg(Tyk + m.ip + L.nx);
    o.tb = L.dim == 3 ? __ldg(L.Tz + a) : R(0);
    o.tt = L.dim == 3 ? __ldg(L.Tz + a + plane) : R(0);
    o.mm = __ldg(L.M + a);
    o.f = fb[a];
    if (!zero_init) {
      o.nw = m.i > 0 ? xb[a - 1] : vzero<V>();
      o.ne = m.i < L.nx - 1 ? xb[a + 1] : vzero<V>();
      o.ns = m.j > 0 ? xb[a - L.nx] : vzero<V>();
      o.nn = m.j < L.ny - 1 ? xb[a + L.nx] : vzero<V>();
    }
  };
  Ops cur, nxt;
  bool cur_valid = ((m.i + m.j + m.k0) & 1) == color;
  if (cur_valid) load_ops(m.k0, cur);
  for (int k = m.k0; k < m.k1; ++k) {
    V xn = vzero<V>();
    if (!zero_init && k + 1 < m.k1 && k + 2 < L.nz) xn = xb[(k + 2) * plane + m.ip];
    const bool nxt_valid = k + 1 < m.k1 && ((m.i + m.j + k + 1) & 1) == color;
    if (nxt_valid) load_ops(k + 1, nxt);
    const int64_t a = k * plane + m.ip;
    V out = xc;
    if (cur_valid) {
      const R dk = cur.tw + cur.te + cur.ts + cur.tn + cur.tb + cur.tt;
      V o = cur.f;
      if (!zero_init) {
        o = vadd(o, vadd(vadd(vscale(cur.nw, cur.tw), vscale(cur.ne, cur.te)),
                         vadd(vscale(cur.ns, cur.ts), vscale(cur.nn, cur.tn))));
        if (k > 0) o = vadd(o, vscale(xm, cur.tb));
        if (k < L.nz - 1) o = vadd(o, vscale(xp, cur.tt));
      }
      out = diag_solve_r<R, V>(dk, cur.mm, tr, ti, o);
    }
    xb[a] = out;
    xm = xc;
    xc = xp;
    xp = xn;
    cur = nxt;
    cur_valid = nxt_valid;
  }
}

// f_c = P^T r_f, z-marching over the coarse grid: each fine plane's in-plane (4 x 4) weighted
// sum is formed once and added to the two coarse planes it belongs to (register ring).
template <class R>
__global__ void __launch_bounds__(kT) restrict_zm_kernel(LevelViewT<R> Lf, LevelViewT<R> Lc, int ax, int ay, int az,
                                                         Batch bt, const typename CT<R>::V* __restrict__ rf,
                                                         typename CT<R>::V* __restrict__ fc) {
  using V = typename CT<R>::V;
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZmMap m = zm_map(Lc, cb);  // coarse column (I, J), coarse planes [k0, k1)
  if (!m.in) return;
  int Fx[4], Fy[4];
  float wx[4], wy[4];
  const int nxx = r1d_terms(m.i, ax, Lc.nx, Fx, wx);
  const int nyy = r1d_terms(m.j, ay, Lc.ny, Fy, wy);
  const V* rb = rf + (int64_t)b * Lf.n;
  V* fb = fc + (int64_t)b * Lc.n;
  const int64_t fplane = (int64_t)Lf.nx * Lf.ny, cplane = (int64_t)Lc.nx * Lc.ny;
  auto inplane = [&](int kf) {
    V s = vzero<V>();
    const V* pl = rb + kf * fplane;
    for (int p = 0; p < nyy; ++p) {
      const V* row = pl + (int64_t)Fy[p] * Lf.nx;
      for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(row[Fx[o]], (R)(wy[p] * wx[o])));
    }
    return s;
  };
  if (az == 1 || Lf.dim == 2) {
    for (int K = m.k0; K < m.k1; ++K) fb[K * cplane + m.ip] = inplane(K);
    return;
  }
  // coarse K collects fine planes 2K-1 (1/4), 2K (3/4 | 1/2 at K = 0), 2K+1 (3/4 | 1/2 at the
  // top), 2K+2 (1/4)
  V sa = m.k0 > 0 ? inplane(2 * m.k0 - 1) : vzero<V>();  // S(2K-1)
  V sb = inplane(2 * m.k0);                              // S(2K)
  for (int K = m.k0; K < m.k1; ++K) {
    const V sc = inplane(2 * K + 1);
    const V sd = K < Lc.nz - 1 ? inplane(2 * K + 2) : vzero<V>();
    const R w0 = K > 0 ? R(0.25) : R(0);
    const R w1 = K == 0 ? R(0.5) : R(0.75);
    const R w2 = K == Lc.nz - 1 ? R(0.5) : R(0.75);
    const R w3 = K < Lc.nz - 1 ? R(0.25) : R(0);
    fb[K * cplane + m.ip] = vadd(vadd(vscale(sa, w0), vscale(sb, w1)), vadd(vscale(sc, w2), vscale(sd, w3)));
    sa = sc;
    sb = sd;
  }
}

// x += P e_c (cell-centred multilinear prolongation), z-marching over the fine grid
template <class R>
__global__ void __launch_bounds__(kT) prolong_zm_kernel(LevelViewT<R> Lf, LevelViewT<R> Lc, int ax, int ay, int az,
                                                        Batch bt, const typename CT<R>::V* __restrict__ ec,
                                                        typename CT<R>::V* __restrict__ xf) {
  using V = typename CT<R>::V;
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZmMap m = zm_map(Lf, cb);
  if (!m.in) return;
  const int64_t plane = (int64_t)Lf.nx * Lf.ny;
  const V* eb = ec + (int64_t)b * Lc.n;
  V* xb = xf + (int64_t)b * Lf.n;
  for (int k = m.k0; k < m.k1; ++k) {
    const int64_t a = k * plane + m.ip;
    xb[a] = vadd(xb[a], prolong_at(Lc, ax, ay, az, eb, m.i, m.j, k, Lf.dim));
  }
}

// q = A p, partial p^T q (FP64), z-marching
__global__ void __launch_bounds__(kT) apply_dot_zm_kernel(LevelView L, Batch bt, const double2* __restrict__ taus,
                                                          const double2* __restrict__ p, double2* __restrict__ q,
                                                          double2* __restrict__ part, int nblk) {
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZmMap m = zm_map(L, cb);
  const int64_t plane = (int64_t)L.nx * L.ny;
  const double2* pb = p + (int64_t)b * L.n;
  double2* qb = q + (int64_t)b * L.n;
  const double2 tau = taus[b];
  const int nxp1 = L.nx + 1;
  double2 acc = make_double2(0.0, 0.0);
  if (m.in) {
    double2 xm = m.k0 > 0 ? pb[(m.k0 - 1) * plane + m.ip] : make_double2(0.0, 0.0);
    double2 xc = pb[m.k0 * plane + m.ip];
    double2 xp = m.k0 + 1 < L.nz ? pb[(m.k0 + 1) * plane + m.ip] : make_double2(0.0, 0.0);
    for (int k = m.k0; k < m.k1; ++k) {
      const double2 xn = (k + 1 < m.k1 && k + 2 < L.nz) ? pb[(k + 2) * plane + m.ip] : make_double2(0.0, 0.0);
      const int64_t a = k * plane + m.ip;
      const double* Txk = L.Tx + (int64_t)k * L.ny * nxp1;
      const double* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx;
      const int ex = m.j * nxp1 + m.i;
      const double tw = __ldg(Txk + ex), te = __ldg(Txk + ex + 1);
      const double ts = __ldg(Tyk + m.ip), tn = __ldg(Tyk + m.ip + L.nx);
      const double tb = __ldg(L.Tz + a), tt = __ldg(L.Tz + a + plane);
      const double dk = tw + te + ts + tn + tb + tt;
      double2 o = make_double2(0.0, 0.0);
      if (m.i > 0) o = cfma(make_double2(tw, 0.0), pb[a - 1], o);
      if (m.i < L.nx - 1) o = cfma(make_double2(te, 0.0), pb[a + 1], o);
      if (m.j > 0) o = cfma(make_double2(ts, 0.0), pb[a - L.nx], o);
      if (m.j < L.ny - 1) o = cfma(make_double2(tn, 0.0), pb[a + L.nx], o);
      if (k > 0) o = cfma(make_double2(tb, 0.0), xm, o);
      if (k < L.nz - 1) o = cfma(make_double2(tt, 0.0), xp, o);
      const double mm = __ldg(L.M + a);
      const double2 d = make_double2(dk + tau.x * mm, tau.y * mm);
      const double2 qa = csub(cmul(d, xc), o);
      qb[a] = qa;
      acc = cadd(acc, cmul(xc, qa));
      xm = xc;
      xc = xp;
      xp = xn;
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = acc;
}

// q = A p, partial p^T q
template <int DIM>
__global__ void __launch_bounds__(kT) apply_dot_kernel(LevelView L, Batch bt, const double2* __restrict__ taus,
                                                       const double2* __restrict__ p, double2* __restrict__ q,
                                                       double2* __restrict__ part, int nblk) {
  TILE_PROLOGUE(L);
  double2 s = make_double2(0.0, 0.0);
  if (in) {
    const double2* pb = p + b * L.n;
    const double2 qa = stencil_apply<DIM>(L, pb, a, i, j, k, taus[b]);
    q[b * L.n + a] = qa;
    s = cmul(pb[a], qa);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// x += alpha p (x = alpha p on the first iteration), r -= alpha q, rmg = (VM) r, partial ||r||^2
__global__ void __launch_bounds__(kT) axpy_norm_kernel(int64_t n, Batch bt, const double2* __restrict__ alpha,
                                                       const double2* __restrict__ p, const double2* __restrict__ q,
                                                       double2* __restrict__ x, int64_t xs, double2* __restrict__ r,
                                                       VM* __restrict__ rmg, int first, double* __restrict__ part,
                                                       int nblk) {
  ITEM_PROLOGUE(n);
  double s = 0.0;
  if (in) {
    const double2 al = alpha[b];
    const double2 pa = p[b * n + a];
    double2* xa = x + b * xs + a;
    *xa = first ? cmul(al, pa) : cfma(al, pa, *xa);
    double2 ra = csub(r[b * n + a], cmul(al, q[b * n + a]));
    r[b * n + a] = ra;
    rmg[b * n + a] = vfrom<VM>(ra);
    s = cabs2(ra);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// p = z + beta p (p = z when first)
__global__ void __launch_bounds__(kT) pupdate_kernel(int64_t n, Batch bt, const double2* __restrict__ beta,
                                                     const VM* __restrict__ z, double2* __restrict__ p, int first) {
  ITEM_PROLOGUE(n);
  if (!in) return;
  const double2 za = vto(z[b * n + a]);
  p[b * n + a] = first ? za : cfma(beta[b], p[b * n + a], za);
}

// x = 0 for items whose right-hand side is zero
__global__ void zero_kernel(int64_t n, const int* __restrict__ zero_item, double2* __restrict__ x, int64_t xs, int B) {
  const int b = blockIdx.y;
  if (!zero_item[b]) return;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    x[b * xs + a] = make_double2(0.0, 0.0);
}

// ---- per-item scalar updates (one block per item, deterministic order) -----------------
enum ScalarOp { OP_BB = 0, OP_RHO = 1, OP_ALPHA = 2, OP_RR = 3, OP_BETA = 4 };

struct Scalars {
  double* bb;
  double* rr;
  double2* rho;
  double2* alpha;
  double2* beta;
};

__global__ void __launch_bounds__(kT) scalar_kernel(int op, Batch bt, const void* part, int nblk, Scalars sc) {
  const int b = blockIdx.x;
  if (bt.done[b]) return;
  if (op == OP_BB || op == OP_RR) {
    const double* pp = static_cast<const double*>(part) + (int64_t)b * nblk;
    double s = 0.0;
    for (int k = threadIdx.x; k < nblk; k += blockDim.x) s += pp[k];
    s = block_sum(s);
    if (threadIdx.x == 0) {
      if (op == OP_BB) sc.bb[b] = s;
      else sc.rr[b] = s;
    }
  } else {
    const double2* pp = static_cast<const double2*>(part) + (int64_t)b * nblk;
    double2 s = make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < nblk; k += blockDim.x) s = cadd(s, pp[k]);
    s = block_sum(s);
    if (threadIdx.x == 0) {
      if (op == OP_RHO) sc.rho[b] = s;
      else if (op == OP_ALPHA) sc.alpha[b] = cdiv(sc.rho[b], s);
      else { sc.beta[b] = cdiv(s, sc.rho[b]); sc.rho[b] = s; }
    }
  }
}

// ---- P1 node-grid multigrid (2-D, vertex-centred) ---------------------------------------
// 7-point operator A = K + tau M (K: 5-point edges, M: E/W/N/S/NE/SW couplings); (i + j) % 3
// is a valid colouring (no two same-colour nodes are coupled), so each colour is updated in
// place without races.  Prolongation = linear interpolation on the nested coarse triangles,
// restriction = its transpose, coarse operators = P1 assembly of the averaged element fields.
template <class R>
__device__ __forceinline__ typename CT<R>::V p1_offsum(const LevelViewT<R>& L, const typename CT<R>::V* u, int64_t a,
                                                       int i, int j, R tr, R ti, R& dk) {
  // returns sum_b T_ab u_b - tau sum_b M_ab u_b (the negated off-diagonal action of A)
  using V = typename CT<R>::V;
  const int64_t ex = (int64_t)j * (L.nx + 1) + i, ey = (int64_t)j * L.nx + i;
  const R tw = L.Tx[ex], te = L.Tx[ex + 1], ts = L.Ty[ey], tn = L.Ty[ey + L.nx];
  dk = tw + te + ts + tn;
  V k{0, 0};
  if (i > 0) k = vadd(k, vscale(u[a - 1], tw));
  if (i < L.nx - 1) k = vadd(k, vscale(u[a + 1], te));
  if (j > 0) k = vadd(k, vscale(u[a - L.nx], ts));
  if (j < L.ny - 1) k = vadd(k, vscale(u[a + L.nx], tn));
  const V mo = mass_off(L, u, a, i, j);
  return V{k.x - (tr * mo.x - ti * mo.y), k.y - (tr * mo.y + ti * mo.x)};
}

template <class R>
__global__ void __launch_bounds__(kT) p1_gs_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                   const typename CT<R>::V* __restrict__ f, typename CT<R>::V* x,
                                                   int color, int zero_init) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(L);
  if (!in) return;
  V* xb = x + (int64_t)b * L.n;
  const bool mine = (i + j) % 3 == color;
  if (zero_init && !mine) {
    xb[a] = vzero<V>();
    return;
  }
  if (!mine) return;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  R dk;
  V o = f[(int64_t)b * L.n + a];
  if (zero_init) {
    const int64_t ex = (int64_t)j * (L.nx + 1) + i, ey = (int64_t)j * L.nx + i;
    dk = L.Tx[ex] + L.Tx[ex + 1] + L.Ty[ey] + L.Ty[ey + L.nx];
  } else {
    o = vadd(o, p1_offsum<R>(L, xb, a, i, j, tr, ti, dk));
  }
  xb[a] = diag_solve_r<R, V>(dk, L.M[a], tr, ti, o);
}

template <class R>
__global__ void __launch_bounds__(kT) p1_residual_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                         const typename CT<R>::V* __restrict__ f,
                                                         const typename CT<R>::V* __restrict__ x,
                                                         typename CT<R>::V* __restrict__ r) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(L);
  if (!in) return;
  const V* xb = x + (int64_t)b * L.n;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  R dk;
  const V o = p1_offsum<R>(L, xb, a, i, j, tr, ti, dk);
  const R mm = L.M[a];
  const R dr = dk + tr * mm, di = ti * mm;
  const V xa = xb[a];
  const V ax = V{dr * xa.x - di * xa.y - o.x, dr * xa.y + di * xa.x - o.y};
  r[(int64_t)b * L.n + a] = vsub(f[(int64_t)b * L.n + a], ax);
}

// f_c = P^T r: coarse node C = fine free (2ic+1, 2jc+1) collects itself and 1/2 of its
// E/W/N/S and NE/SW fine neighbours (the fine nodes interpolating from C).
template <class R>
__global__ void __launch_bounds__(kT) p1_restrict_kernel(LevelViewT<R> Lf, LevelViewT<R> Lc, Batch bt,
                                                         const typename CT<R>::V* __restrict__ rf,
                                                         typename CT<R>::V* __restrict__ fc) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(Lc);
  if (!in) return;
  const V* rb = rf + (int64_t)b * Lf.n;
  const int fi = 2 * i + 1, fj = 2 * j + 1;
  const int64_t c = (int64_t)fj * Lf.nx + fi;
  V s = vadd(vadd(vadd(rb[c - 1], rb[c + 1]), vadd(rb[c - Lf.nx], rb[c + Lf.nx])),
             vadd(rb[c + Lf.nx + 1], rb[c - Lf.nx - 1]));
  fc[(int64_t)b * Lc.n + a] = vadd(rb[c], vscale(s, R(0.5)));
}

template <class R>
__global__ void __launch_bounds__(kT) p1_prolong_kernel(LevelViewT<R> Lf, LevelViewT<R> Lc, Batch bt,
                                                        const typename CT<R>::V* __restrict__ ec,
                                                        typename CT<R>::V* __restrict__ xf) {
  using V = typename CT<R>::V;
  TILE_PROLOGUE(Lf);
  if (!in) return;
  const V* eb = ec + (int64_t)b * Lc.n;
  auto cval = [&](int Ic, int Jc) {  // coarse node coordinates; Dirichlet nodes are zero
    return (Ic >= 1 && Ic <= Lc.nx && Jc >= 1 && Jc <= Lc.ny) ? eb[(int64_t)(Jc - 1) * Lc.nx + (Ic - 1)] : vzero<V>();
  };
  const int I = i + 1, J = j + 1;
  V v;
  if ((I & 1) == 0 && (J & 1) == 0) v = cval(I >> 1, J >> 1);
  else if ((J & 1) == 0) v = vscale(vadd(cval(I >> 1, J >> 1), cval((I + 1) >> 1, J >> 1)), R(0.5));
  else if ((I & 1) == 0) v = vscale(vadd(cval(I >> 1, J >> 1), cval(I >> 1, (J + 1) >> 1)), R(0.5));
  else v = vscale(vadd(cval(I >> 1, J >> 1), cval((I + 1) >> 1, (J + 1) >> 1)), R(0.5));
  xf[(int64_t)b * Lf.n + a] = vadd(xf[(int64_t)b * Lf.n + a], v);
}

// ---- V-cycle driver --------------------------------------------------------------------
template <class R>
LevelViewT<R> mg_view(lt_pencil p, int l);
template <>
LevelViewT<double> mg_view<double>(lt_pencil p, int l) { return p->view(l); }
template <>
LevelViewT<float> mg_view<float>(lt_pencil p, int l) { return p->view32(l); }

// Returns the buffer holding the level-l V-cycle output (Bc x n_l).
template <class R, int DIM>
const typename CT<R>::V* vcycle(lt_pencil p, int l, int Bc, const Batch& bt, const double2* taus,
                                const typename CT<R>::V* const* inv, int64_t inv_ld, int64_t inv_off,
                                std::vector<typename CT<R>::V*>& X, std::vector<typename CT<R>::V*>& F,
                                std::vector<typename CT<R>::V*>& Rr) {
  using V = typename CT<R>::V;
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int last = (int)p->levels.size() - 1;
  LevelViewT<R> L = mg_view<R>(p, l);
  const double vb = sizeof(V), rb = sizeof(R);
  const double cell_bytes = (double)L.n * Bc;
  const double coef = (double)L.n * rb * (DIM + 1);
  if (p->kind == LT_GRID_P1_TRI && l < last) {
    // P1: symmetric 3-colour Gauss-Seidel V-cycle on the node grid
    LevelViewT<R> Lc = mg_view<R>(p, l + 1);
    const unsigned grid = (unsigned)L.ntiles * (unsigned)Bc;
    const double cb6 = coef + (double)L.n * rb * 3;  // + the three mass-coupling arrays
    for (int c = 0; c < 3; ++c)
      launch(ctx, "mg_smooth", cell_bytes * 3 * vb + cb6, [&] {
        p1_gs_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], c, c == 0);
      });
    launch(ctx, "mg_residual", cell_bytes * 3 * vb + cb6, [&] {
      p1_residual_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
    });
    launch(ctx, "mg_restrict", cell_bytes * vb + (double)Lc.n * Bc * vb, [&] {
      p1_restrict_kernel<R><<<(unsigned)Lc.ntiles * Bc, kT, 0, st>>>(L, Lc, bt, Rr[l], F[l + 1]);
    });
    const V* ec = vcycle<R, DIM>(p, l + 1, Bc, bt, taus, inv, inv_ld, inv_off, X, F, Rr);
    launch(ctx, "mg_prolong", cell_bytes * 2 * vb + (double)Lc.n * Bc * vb, [&] {
      p1_prolong_kernel<R><<<grid, kT, 0, st>>>(L, Lc, bt, ec, X[l]);
    });
    for (int c = 2; c >= 0; --c)
      launch(ctx, "mg_smooth", cell_bytes * 3 * vb + cb6, [&] {
        p1_gs_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], c, 0);
      });
    return X[l];
  }
  if (l == last) {
    dim3 g(blocks_for(L.n, kT / 32), Bc);
    launch(ctx, "mg_coarse_solve", cell_bytes * 2 * vb, [&] {
      coarse_solve_kernel<V><<<g, kT, 0, st>>>((int)L.n, bt, inv, inv_ld, inv_off, F[l], X[l]);
    });
    return X[l];
  }
  LevelViewT<R> Lc = mg_view<R>(p, l + 1);
  const Level& lev = *p->levels[l];
  const unsigned grid = (unsigned)L.ntiles * (unsigned)Bc;
  const unsigned sgrid = (unsigned)(((L.nx + SW_TX - 1) / SW_TX) * ((L.ny + SW_TY - 1) / SW_TY)) * (unsigned)Bc;
  const size_t ssmem = sweep_smem<R>(DIM);
  static bool attr_set = false;
  if (!attr_set) {
    LT_CUDA(cudaFuncSetAttribute(rb_sweep_kernel<R, DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
    attr_set = true;
  }
  static const bool zm_smoother = [] {
    const char* e = std::getenv("LT_SMOOTHER");
    return !(e && std::string(e) == "smem");
  }();
  const unsigned zgrid = (unsigned)zm_blocks(L) * (unsigned)Bc;
  if (zm_smoother) {
    // pre-smoothing: red half sweep from zero (f read, x written), black half sweep
    launch(ctx, "mg_smooth", cell_bytes * 2 * vb + coef, [&] {
      rbhalf_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], 0, 1);
    });
    launch(ctx, "mg_smooth", cell_bytes * 3 * vb + coef, [&] {
      rbhalf_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], 1, 0);
    });
  } else {
    // pre-smoothing: one fused red-black sweep (red first) from a zero iterate
    launch(ctx, "mg_smooth", cell_bytes * 2 * vb + coef, [&] {
      rb_sweep_kernel<R, DIM><<<sgrid, kT, ssmem, st>>>(L, bt, taus, F[l], nullptr, X[l], 0, 1, Lc, 1, 1, 1, nullptr);
    });
  }
  launch(ctx, "mg_residual", cell_bytes * 3 * vb + coef, [&] {
    if (DIM == 3)
      residual_zm_kernel<R><<<(unsigned)zm_blocks(L) * Bc, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
    else
      residual_kernel<R, DIM><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
  });
  const unsigned gridc = (unsigned)Lc.ntiles * (unsigned)Bc;
  launch(ctx, "mg_restrict", cell_bytes * vb + (double)Lc.n * Bc * vb, [&] {
    if (zm_smoother)
      restrict_zm_kernel<R><<<(unsigned)zm_blocks(Lc) * Bc, kT, 0, st>>>(L, Lc, lev.agg[0], lev.agg[1], lev.agg[2], bt,
                                                                        Rr[l], F[l + 1]);
    else
      restrict_kernel<R, DIM><<<gridc, kT, 0, st>>>(L, Lc, lev.agg[0], lev.agg[1], lev.agg[2], bt, Rr[l], F[l + 1]);
  });
  const V* ec = vcycle<R, DIM>(p, l + 1, Bc, bt, taus, inv, inv_ld, inv_off, X, F, Rr);
  if (zm_smoother) {
    // coarse correction, then the transpose of the pre-smoother (black, red), in place
    launch(ctx, "mg_prolong", cell_bytes * 2 * vb + (double)Lc.n * Bc * vb, [&] {
      prolong_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, Lc, lev.agg[0], lev.agg[1], lev.agg[2], bt, ec, X[l]);
    });
    launch(ctx, "mg_smooth", cell_bytes * 3 * vb + coef, [&] {
      rbhalf_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], 1, 0);
    });
    launch(ctx, "mg_smooth", cell_bytes * 3 * vb + coef, [&] {
      rbhalf_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], 0, 0);
    });
    return X[l];
  }
  // post-smoothing: coarse correction x + P e_c fused into one black-first sweep (the
  // transpose of the pre-smoother), written out of place into Rr[l]
  launch(ctx, "mg_smooth", cell_bytes * 3 * vb + (double)Lc.n * Bc * vb + coef, [&] {
    rb_sweep_kernel<R, DIM><<<sgrid, kT, ssmem, st>>>(L, bt, taus, F[l], X[l], Rr[l], 1, 0, Lc, lev.agg[0],
                                                      lev.agg[1], lev.agg[2], ec);
  });
  return Rr[l];
}

template <int DIM>
void inner_chunk(lt_pencil p, int Bc, const double2* taus_host, const double2* v, int64_t vs, double2* u,
                 int64_t us) {
  using R = MgReal;
  using V = VM;
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int nl = (int)p->levels.size();
  const int64_t n = p->n;
  const int nblk = (int)blocks_for(n, kT);
  LevelView L0 = p->view(0);

  // coarse factors for each distinct tau (cached on the pencil)
  std::vector<const V*> inv_host(Bc);
  const int64_t nc = p->levels.back()->n;
  const bool fp64 = sizeof(R) == 8;
  for (int b = 0; b < Bc; ++b) {
    const CoarseFactor& fc = p->factor(taus_host[b]);
    inv_host[b] = fp64 ? reinterpret_cast<const V*>(fc.inverse.get()) : reinterpret_cast<const V*>(fc.inverse32.get());
  }
  const int64_t inv_ld = fp64 ? 2 * nc : nc, inv_off = fp64 ? nc : 0;

  // small per-item state: taus, inverse pointers, done flags, scalars
  const size_t small_bytes = sizeof(double2) * Bc * 4 + sizeof(double) * Bc * 2 + sizeof(void*) * Bc +
                             sizeof(int) * Bc + 64;
  DeviceBuffer small(small_bytes, st);
  char* sp = small.as<char>();
  double2* d_taus = reinterpret_cast<double2*>(sp);
  double2* d_rho = d_taus + Bc;
  double2* d_alpha = d_rho + Bc;
  double2* d_beta = d_alpha + Bc;
  double* d_bb = reinterpret_cast<double*>(d_beta + Bc);
  double* d_rr = d_bb + Bc;
  const V** d_inv = reinterpret_cast<const V**>(d_rr + Bc);
  int* d_done = reinterpret_cast<int*>(d_inv + Bc);
  LT_CUDA(cudaMemcpyAsync(d_taus, taus_host, sizeof(double2) * Bc, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(d_inv, inv_host.data(), sizeof(void*) * Bc, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemsetAsync(d_done, 0, sizeof(int) * Bc, st));
  Scalars sc{d_bb, d_rr, d_rho, d_alpha, d_beta};
  Batch bt{Bc, d_done};

  // workspace: FP64 Krylov vectors r, p, q; multigrid vectors (precision R) per level
  DeviceBuffer partials(sizeof(double2) * (size_t)Bc *
                            std::max<int64_t>(std::max<int64_t>(nblk, L0.ntiles), zm_blocks(L0)), st);
  DeviceBuffer vec(sizeof(double2) * (size_t)Bc * n * 3, st);
  double2* r = vec.as<double2>();
  double2* pp = r + Bc * n;
  double2* q = pp + Bc * n;
  std::vector<DeviceBuffer> lvl(nl);
  std::vector<V*> X(nl), F(nl), Rr(nl);
  for (int l = 0; l < nl; ++l) {
    const int64_t nlv = p->levels[l]->n;
    lvl[l].allocate(sizeof(V) * (size_t)Bc * nlv * 3, st);
    X[l] = lvl[l].as<V>();
    F[l] = X[l] + Bc * nlv;
    Rr[l] = X[l] + 2 * Bc * nlv;
  }
  V* rmg = F[0];  // the multigrid copy of the COCG residual
  const unsigned grid = (unsigned)nblk * (unsigned)Bc;
  const double nb = (double)n * Bc;
  const double coef = (double)n * 8.0 * (DIM + 1);
  const double vb = sizeof(V);

  launch(ctx, "cocg_vec", nb * (32.0 + vb), [&] {
    copy_norm_kernel<<<grid, kT, 0, st>>>(n, bt, v, vs, r, rmg, (double*)partials.get(), nblk);
  });
  launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_BB, bt, partials.get(), nblk, sc); });
  std::vector<double> bb(Bc), rr(Bc), best(Bc);
  LT_CUDA(cudaMemcpyAsync(bb.data(), d_bb, sizeof(double) * Bc, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  std::vector<int> done(Bc, 0), zero(Bc, 0), stall(Bc, 0);
  bool any_zero = false;
  for (int b = 0; b < Bc; ++b)
    if (!(bb[b] > 0.0)) { done[b] = 1; zero[b] = 1; any_zero = true; }
  if (any_zero) {
    DeviceBuffer dz(sizeof(int) * Bc, st);
    LT_CUDA(cudaMemcpyAsync(dz.get(), zero.data(), sizeof(int) * Bc, cudaMemcpyHostToDevice, st));
    launch(ctx, "cocg_vec", nb * 16.0, [&] {
      zero_kernel<<<dim3(blocks_for(n, kT), Bc), kT, 0, st>>>(n, dz.as<int>(), u, us, Bc);
    });
    LT_CUDA(cudaMemcpyAsync(d_done, done.data(), sizeof(int) * Bc, cudaMemcpyHostToDevice, st));
  }
  int active = 0;
  for (int b = 0; b < Bc; ++b) active += !done[b];
  if (active == 0) return;

  const double tol2 = p->inner_tol * p->inner_tol;
  int iters_seen = 0;
  double sync_ms = 0.0;
  const auto wall0 = std::chrono::steady_clock::now();
  for (int b = 0; b < Bc; ++b) best[b] = bb[b];
  // z = B r ; rho = r^T z ; p = z
  const V* z = vcycle<R, DIM>(p, 0, Bc, bt, d_taus, d_inv, inv_ld, inv_off, X, F, Rr);
  launch(ctx, "cocg_vec", nb * (16.0 + vb), [&] {
    bdot_kernel<<<grid, kT, 0, st>>>(n, bt, r, z, partials.as<double2>(), nblk);
  });
  launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_RHO, bt, partials.get(), nblk, sc); });
  launch(ctx, "cocg_vec", nb * (16.0 + vb), [&] { pupdate_kernel<<<grid, kT, 0, st>>>(n, bt, d_beta, z, pp, 1); });
  for (int it = 0; it < p->inner_maxit; ++it) {
    const int nblk_apply = DIM == 3 ? zm_blocks(L0) : L0.ntiles;
    launch(ctx, "cocg_apply", nb * 32.0 + coef, [&] {
      if (DIM == 3)
        apply_dot_zm_kernel<<<(unsigned)nblk_apply * Bc, kT, 0, st>>>(L0, bt, d_taus, pp, q, partials.as<double2>(),
                                                                      nblk_apply);
      else
        apply_dot_kernel<DIM><<<(unsigned)nblk_apply * Bc, kT, 0, st>>>(L0, bt, d_taus, pp, q,
                                                                        partials.as<double2>(), nblk_apply);
    });
    launch(ctx, "cocg_scalar", 0.0, [&] {
      scalar_kernel<<<Bc, kT, 0, st>>>(OP_ALPHA, bt, partials.get(), nblk_apply, sc);
    });
    launch(ctx, "cocg_vec", nb * ((it == 0 ? 64.0 : 80.0) + vb), [&] {
      axpy_norm_kernel<<<grid, kT, 0, st>>>(n, bt, d_alpha, pp, q, u, us, r, rmg, it == 0, (double*)partials.get(),
                                            nblk);
    });
    launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_RR, bt, partials.get(), nblk, sc); });
    LT_CUDA(cudaMemcpyAsync(rr.data(), d_rr, sizeof(double) * Bc, cudaMemcpyDeviceToHost, st));
    {
      const auto s0 = std::chrono::steady_clock::now();
      LT_CUDA(cudaStreamSynchronize(st));
      if (inner_trace())
        sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count();
    }
    bool changed = false;
    for (int b = 0; b < Bc; ++b) {
      if (done[b]) continue;
      if (rr[b] <= tol2 * bb[b]) { done[b] = 1; changed = true; continue; }
      // stagnation at the rounding floor: within 1e4 of the tolerance and no halving of the
      // residual in 6 iterations.  (Far from the floor COCG's residual is non-monotone on the
      // indefinite pencils Re tau < 0 gives -- plateaus there are not stagnation.)
      if (rr[b] < 0.25 * best[b]) { best[b] = rr[b]; stall[b] = 0; }
      else if (rr[b] <= 1e8 * tol2 * bb[b] && ++stall[b] >= 6) { done[b] = 1; changed = true; }
    }
    if (changed) {
      active = 0;
      for (int b = 0; b < Bc; ++b) active += !done[b];
      if (active == 0) break;
      LT_CUDA(cudaMemcpyAsync(d_done, done.data(), sizeof(int) * Bc, cudaMemcpyHostToDevice, st));
    }
    z = vcycle<R, DIM>(p, 0, Bc, bt, d_taus, d_inv, inv_ld, inv_off, X, F, Rr);
    launch(ctx, "cocg_vec", nb * (16.0 + vb), [&] {
      bdot_kernel<<<grid, kT, 0, st>>>(n, bt, r, z, partials.as<double2>(), nblk);
    });
    launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_BETA, bt, partials.get(), nblk, sc); });
    launch(ctx, "cocg_vec", nb * (32.0 + vb), [&] { pupdate_kernel<<<grid, kT, 0, st>>>(n, bt, d_beta, z, pp, 0); });
    if (inner_trace()) iters_seen = it + 1;
  }
  LT_CUDA(cudaStreamSynchronize(st));
  if (inner_trace())
    std::fprintf(stderr, "[inner] chunk B=%d iters=%d wall=%.3f ms sync-wait=%.3f ms\n", Bc, iters_seen + 1,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count(), sync_ms);
  if (inner_trace() >= 2)
    for (int b = 0; b < Bc; ++b)
      std::fprintf(stderr, "[inner] tau=(%.4g,%.4g) it<=%d rel=%.3e %s\n", taus_host[b].x, taus_host[b].y,
                   iters_seen + 1, std::sqrt(rr[b] / bb[b]), rr[b] <= tol2 * bb[b] ? "ok" : "STAGNATED");
}

}  // namespace

void inner_solve(lt_pencil p, int B, const double2* taus_host, const double2* v, int64_t vs, double2* u, int64_t us) {
  // Chunk so that the Krylov + multigrid workspace stays bounded.
  const int64_t n = p->n;
  const double avail = available_device_bytes(p->ctx);
  const double per_item = (double)n * (sizeof(double2) * 3.0 + sizeof(VM) * 3.0 * 1.2);
  int chunk = (int)std::max(1.0, std::min(128.0, 0.5 * avail / per_item));
  if (inner_trace())
    std::fprintf(stderr, "[inner] B=%d chunk=%d available=%.1fGB\n", B, chunk, avail / 1e9);
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int bc = std::min(chunk, B - b0);
    if (p->dim == 3) inner_chunk<3>(p, bc, taus_host + b0, v + b0 * vs, vs, u + b0 * us, us);
    else inner_chunk<2>(p, bc, taus_host + b0, v + b0 * vs, vs, u + b0 * us, us);
  }
}

}  // namespace lt
