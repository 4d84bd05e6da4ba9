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
#include <cooperative_groups.h>

#include "stencil.cuh"

namespace lt {
namespace cg = cooperative_groups;

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
__device__ __forceinline__ int warp_sum(int v) {
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

// Grid-stride COCG vector kernels: G = gridDim.x / B blocks per item (a few per SM in total,
// chunk_vec_blocks), so a launch over finished items costs G blocks per item, not n / 256.
#define ITEM_GRID_PROLOGUE                                        \
  LT_ITEM_BLOCK(bt.B, b, cb)                                      \
  if (bt.done[b]) return;                                         \
  const int64_t stride_ = (int64_t)(gridDim.x / bt.B) * blockDim.x;

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

// Storage index of cell (i, j, k) of a level: natural, or colour-split (see the colour-split
// TMA kernels below)
template <class VW>
__device__ __forceinline__ int64_t rb_index(const VW& L, int i, int j, int k) {
  const int64_t row = ((int64_t)k * L.ny + j) * L.nx;
  return L.split ? row + (int64_t)(((i + j + k) & 1) * (L.nx >> 1)) + (i >> 1) : row + i;
}
// natural flat index a -> storage index (nx == 0: natural layout)
__device__ __forceinline__ int64_t rb_flat(int64_t a, int nx, int ny) {
  if (nx == 0) return a;
  const int64_t t = a / nx;
  const int i = (int)(a - t * nx);
  const int64_t k = t / ny;
  const int j = (int)(t - k * ny);
  return t * nx + (int64_t)(((i + j + (int)(k & 1)) & 1) * (nx >> 1)) + (i >> 1);
}


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

// r = v, rmg = (VM) v, u = 0, partial ||v||^2
__global__ void __launch_bounds__(kT) copy_norm_kernel(int64_t n, Batch bt, const double2* __restrict__ v, int64_t vs,
                                                       double2* __restrict__ r, VM* __restrict__ rmg,
                                                       double2* __restrict__ u, int64_t us, double* __restrict__ part,
                                                       int nblk, int snx, int sny) {
  ITEM_GRID_PROLOGUE
  double s = 0.0;
  for (int64_t a = cb * (int64_t)blockDim.x + threadIdx.x; a < n; a += stride_) {
    const double2 x = v[b * vs + a];
    r[b * n + a] = x;
    rmg[b * n + rb_flat(a, snx, sny)] = vfrom<VM>(x);
    u[b * us + a] = make_double2(0.0, 0.0);
    s += cabs2(x);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// partial sum_a r_a z_a (bilinear, no conjugation), z from the V-cycle
__global__ void __launch_bounds__(kT) bdot_kernel(int64_t n, Batch bt, const double2* __restrict__ x,
                                                  const VM* __restrict__ y, double2* __restrict__ part, int nblk,
                                                  int snx, int sny) {
  ITEM_GRID_PROLOGUE
  double2 s = make_double2(0.0, 0.0);
  for (int64_t a = cb * (int64_t)blockDim.x + threadIdx.x; a < n; a += stride_)
    s = cfma(x[b * n + a], vto(y[b * n + rb_flat(a, snx, sny)]), s);
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

// ---- transfers for aggregation 2 in x, y and z (3-D), natural or colour-split levels ------
// Both kernels work on fine cell PAIRS (2I, 2I + 1): they share the coarse x index I, and in
// the colour-split layout they sit at position I of the two colour halves; in the natural
// layout they are one 16-byte word.  Lanes are consecutive I, so every load is coalesced and
// the x-neighbours 2I - 1 / 2I + 2 (restriction) or coarse I -+ 1 (prolongation) come from
// the adjacent lanes by shuffle.  The z direction is a register ring as in the zm kernels.
// (The per-cell zm kernels read 16 strided fine values per coarse cell and fine plane and
// were latency-bound at 0.7-1.7 TB/s.)
constexpr int TP_TY = 4, TP_ZC = 16;  // restriction: 32 x 4 coarse columns x 16 coarse planes

// fine cells (2I, 2I + 1) of row (j, k) of a level
__device__ __forceinline__ void pair_load(const LevelViewT<float>& L, const float2* __restrict__ v, int I, int j,
                                          int k, float2& e, float2& o) {
  const int64_t row = ((int64_t)k * L.ny + j) * L.nx;
  if (L.split) {
    const int s = (j + k) & 1, h = L.nx >> 1;  // even cells in colour half s
    e = v[row + s * h + I];
    o = v[row + (s ^ 1) * h + I];
  } else {
    const float4 p = *reinterpret_cast<const float4*>(v + row + 2 * I);
    e = make_float2(p.x, p.y);
    o = make_float2(p.z, p.w);
  }
}
__device__ __forceinline__ void pair_store(const LevelViewT<float>& L, float2* __restrict__ v, int I, int j, int k,
                                           float2 e, float2 o) {
  const int64_t row = ((int64_t)k * L.ny + j) * L.nx;
  if (L.split) {
    const int s = (j + k) & 1, h = L.nx >> 1;
    v[row + s * h + I] = e;
    v[row + (s ^ 1) * h + I] = o;
  } else {
    *reinterpret_cast<float4*>(v + row + 2 * I) = make_float4(e.x, e.y, o.x, o.y);
  }
}
__device__ __forceinline__ float2 shfl_f2(float2 v, int src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ float2 f2fma(float w, float2 a, float2 acc) {
  return make_float2(fmaf(w, a.x, acc.x), fmaf(w, a.y, acc.y));
}

// f_c = P^T r_f.  Thread = coarse column (I, J), CTA = 32 x TP_TY columns x TP_ZC coarse
// planes, z-marching over the fine planes with the loads of fine plane kf + 1 in flight while
// plane kf is reduced (software pipeline; one coarse cell per thread with all loads
// independent was bound by CTA turnover at 1 CTA per SM, the unpipelined march by its serial
// plane chain).
struct RowsRaw {
  float2 e[4], o[4], m[4], p[4];  // fine rows 2J-1 .. 2J+2: cells 2I, 2I+1, 2I-1 (lane 0), 2I+2 (lane 31)
};
__global__ void __launch_bounds__(32 * TP_TY) restrict_pair_kernel(LevelViewT<float> Lf, LevelViewT<float> Lc,
                                                                   Batch bt, const float2* __restrict__ rf,
                                                                   float2* __restrict__ fc) {
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int tx = (Lc.nx + 31) / 32, ty = (Lc.ny + TP_TY - 1) / TP_TY;
  const int tile = cb % (tx * ty), chunk = cb / (tx * ty);
  const int lane = threadIdx.x & 31;
  const int I = (tile % tx) * 32 + lane, J = (tile / tx) * TP_TY + (threadIdx.x >> 5);
  if (J >= Lc.ny) return;  // whole warp
  const bool in = I < Lc.nx;
  const int K0 = chunk * TP_ZC, K1 = min(Lc.nz, K0 + TP_ZC);
  const float2* rb = rf + (int64_t)b * Lf.n;
  const float wxm = I > 0 ? 0.25f : 0.f, wx0 = I == 0 ? 0.5f : 0.75f;
  const float wx1 = I == Lc.nx - 1 ? 0.5f : 0.75f, wxp = I < Lc.nx - 1 ? 0.25f : 0.f;
  const float wyv[4] = {J > 0 ? 0.25f : 0.f, J == 0 ? 0.5f : 0.75f, J == Lc.ny - 1 ? 0.5f : 0.75f,
                        J < Lc.ny - 1 ? 0.25f : 0.f};
  auto load = [&](int kf, RowsRaw& R) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      R.e[r] = R.o[r] = R.m[r] = R.p[r] = make_float2(0.f, 0.f);
      if (wyv[r] == 0.f) continue;  // warp-uniform
      const int jf = 2 * J - 1 + r;
      if (in) pair_load(Lf, rb, I, jf, kf, R.e[r], R.o[r]);
      float2 t;
      if (lane == 0 && in && I > 0) pair_load(Lf, rb, I - 1, jf, kf, t, R.m[r]);
      if (lane == 31 && I + 1 < Lc.nx) pair_load(Lf, rb, I + 1, jf, kf, R.p[r], t);
    }
  };
  auto reduce = [&](const RowsRaw& R) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (wyv[r] == 0.f) continue;
      float2 om = shfl_f2(R.o[r], (lane + 31) & 31), ep = shfl_f2(R.e[r], (lane + 1) & 31);
      if (lane == 0) om = R.m[r];
      if (lane == 31) ep = R.p[r];
      float2 xr = make_float2(0.f, 0.f);
      xr = f2fma(wxm, om, xr);
      xr = f2fma(wx0, R.e[r], xr);
      xr = f2fma(wx1, R.o[r], xr);
      xr = f2fma(wxp, ep, xr);
      acc = f2fma(wyv[r], xr, acc);
    }
    return acc;
  };
  float2* fb = fc + (int64_t)b * Lc.n;
  // coarse K collects fine planes 2K-1 (1/4), 2K (3/4 | 1/2 at K = 0), 2K+1 (3/4 | 1/2 at the
  // top), 2K+2 (1/4)
  const int kbeg = max(2 * K0 - 1, 0), kend = min(2 * K1, Lf.nz - 1);
  float2 sa = make_float2(0.f, 0.f), sb = sa, sc = sa;
  RowsRaw cur, nxt;
  load(kbeg, cur);
  for (int kf = kbeg; kf <= kend; ++kf) {
    if (kf < kend) load(kf + 1, nxt);
    const float2 S = reduce(cur);
    if (kf < 2 * K0) {
      sa = S;
    } else if (kf == 2 * K0) {
      sb = S;
    } else {
      const bool odd = kf & 1;
      const int K = odd ? (kf - 1) >> 1 : (kf >> 1) - 1;
      if (odd) sc = S;
      if (!odd || K == Lc.nz - 1) {
        const float2 sd = odd ? make_float2(0.f, 0.f) : S;
        float2 v = make_float2(0.f, 0.f);
        v = f2fma(K > 0 ? 0.25f : 0.f, sa, v);
        v = f2fma(K == 0 ? 0.5f : 0.75f, sb, v);
        v = f2fma(K == Lc.nz - 1 ? 0.5f : 0.75f, sc, v);
        v = f2fma(K < Lc.nz - 1 ? 0.25f : 0.f, sd, v);
        if (in) fb[rb_index(Lc, I, J, K)] = v;
        sa = sc;
        sb = sd;
      }
    }
    cur = nxt;
  }
}

// x_f += P e_c.  Thread = fine pair (2I, 2I + 1) of one fine row, CTA 32 x 8 fine rows x a chunk
// of ZM_ZC fine planes, z-marching with the next fine pair and the next-but-one coarse plane's
// rows in flight (register ring over the coarse planes).
struct CoarseRaw {
  float2 c[2], m[2], p[2];  // coarse rows of the fine row: I, I - 1 (lane 0), I + 1 (lane 31)
};
__global__ void __launch_bounds__(kT) prolong_pair_kernel(LevelViewT<float> Lf, LevelViewT<float> Lc, Batch bt,
                                                          const float2* __restrict__ ec, float2* __restrict__ xf) {
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int nh = Lf.nx >> 1;  // pairs per fine row (= coarse nx)
  const int tx = (nh + 31) / 32, ty = (Lf.ny + 7) / 8;
  const int tile = cb % (tx * ty), chunk = cb / (tx * ty);
  const int lane = threadIdx.x & 31;
  const int I = (tile % tx) * 32 + lane, j = (tile / tx) * 8 + (threadIdx.x >> 5);
  if (j >= Lf.ny) return;  // whole warp
  const bool in = I < nh;
  const int k0 = chunk * ZM_ZC, k1 = min(Lf.nz, k0 + ZM_ZC);
  const float2* eb = ec + (int64_t)b * Lc.n;
  float2* xb = xf + (int64_t)b * Lf.n;
  // coarse rows of fine row j and their weights (Dirichlet ghost at the ends: 1/2 of J)
  const int J = j >> 1;
  int Jr[2];
  float wr[2];
  if ((j & 1) == 0) {
    Jr[0] = J; wr[0] = J == 0 ? 0.5f : 0.75f; Jr[1] = J - 1; wr[1] = J > 0 ? 0.25f : 0.f;
  } else {
    Jr[0] = J; wr[0] = J == Lc.ny - 1 ? 0.5f : 0.75f; Jr[1] = J + 1; wr[1] = J < Lc.ny - 1 ? 0.25f : 0.f;
  }
  const float wxe0 = I == 0 ? 0.5f : 0.75f, wxe1 = I > 0 ? 0.25f : 0.f;            // fine 2I: I, I - 1
  const float wxo0 = I == nh - 1 ? 0.5f : 0.75f, wxo1 = I < nh - 1 ? 0.25f : 0.f;  // fine 2I+1: I, I + 1
  auto at = [&](int Ic, int Jc, int Kc) { return eb[rb_index(Lc, Ic, Jc, Kc)]; };
  auto load = [&](int K, CoarseRaw& R) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      R.c[r] = R.m[r] = R.p[r] = make_float2(0.f, 0.f);
      if (K < 0 || K >= Lc.nz || wr[r] == 0.f) continue;  // warp-uniform
      if (in) R.c[r] = at(I, Jr[r], K);
      if (lane == 0 && in && I > 0) R.m[r] = at(I - 1, Jr[r], K);
      if (lane == 31 && I + 1 < nh) R.p[r] = at(I + 1, Jr[r], K);
    }
  };
  // bilinear in-plane values (fine 2I, fine 2I + 1) of one coarse plane
  auto interp = [&](const CoarseRaw& R, float2& pe, float2& po) {
    pe = make_float2(0.f, 0.f);
    po = pe;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float2 m1 = shfl_f2(R.c[r], (lane + 31) & 31), p1 = shfl_f2(R.c[r], (lane + 1) & 31);
      if (lane == 0) m1 = R.m[r];
      if (lane == 31) p1 = R.p[r];
      pe = f2fma(wr[r] * wxe0, R.c[r], f2fma(wr[r] * wxe1, m1, pe));
      po = f2fma(wr[r] * wxo0, R.c[r], f2fma(wr[r] * wxo1, p1, po));
    }
  };
  int K = k0 >> 1;
  float2 sme, smo, sce, sco, spe, spo;
  CoarseRaw raw;
  load(K - 1, raw);
  interp(raw, sme, smo);
  load(K, raw);
  interp(raw, sce, sco);
  load(K + 1, raw);
  interp(raw, spe, spo);
  load(K + 2, raw);  // in flight: the next coarse plane to enter the ring
  float2 e = make_float2(0.f, 0.f), o = e, en = e, on = e;
  if (in) pair_load(Lf, xb, I, j, k0, e, o);
  for (int k = k0; k < k1; ++k) {
    if (in && k + 1 < k1) pair_load(Lf, xb, I, j, k + 1, en, on);
    if ((k >> 1) != K) {
      K = k >> 1;
      sme = sce; smo = sco;
      sce = spe; sco = spo;
      interp(raw, spe, spo);
      load(K + 2, raw);
    }
    float2 ve = make_float2(0.f, 0.f), vo = ve;
    if ((k & 1) == 0) {
      const float w0 = K == 0 ? 0.5f : 0.75f, w1 = K > 0 ? 0.25f : 0.f;
      ve = f2fma(w1, sme, f2fma(w0, sce, ve));
      vo = f2fma(w1, smo, f2fma(w0, sco, vo));
    } else {
      const float w0 = K == Lc.nz - 1 ? 0.5f : 0.75f, w1 = K < Lc.nz - 1 ? 0.25f : 0.f;
      ve = f2fma(w1, spe, f2fma(w0, sce, ve));
      vo = f2fma(w1, spo, f2fma(w0, sco, vo));
    }
    if (in) pair_store(Lf, xb, I, j, k, make_float2(e.x + ve.x, e.y + ve.y), make_float2(o.x + vo.x, o.y + vo.y));
    e = en;
    o = on;
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
    if (Lf.split) {
      for (int p = 0; p < nyy; ++p)
        for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(rb[rb_index(Lf, Fx[o], Fy[p], kf)], (R)(wy[p] * wx[o])));
      return s;
    }
    const V* pl = rb + kf * fplane;
    for (int p = 0; p < nyy; ++p) {
      const V* row = pl + (int64_t)Fy[p] * Lf.nx;
      for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(row[Fx[o]], (R)(wy[p] * wx[o])));
    }
    return s;
  };
  if (az == 1 || Lf.dim == 2) {
    for (int K = m.k0; K < m.k1; ++K) {
      const V v = inplane(K);
      if (m.in) fb[rb_index(Lc, m.i, m.j, K)] = v;
    }
    return;
  }
  // coarse K collects fine planes 2K-1 (1/4), 2K (3/4 | 1/2 at K = 0), 2K+1 (3/4 | 1/2 at the
  // top), 2K+2 (1/4)
  V sa = m.k0 > 0 ? inplane(2 * m.k0 - 1) : vzero<V>();  // S(2K-1)
  V sb = inplane(2 * m.k0);                              // S(2K)
  for (int K = m.k0; K < m.k1; ++K) {
    const V sc = inplane(2 * K + 1);
    const V sd = K < Lc.nz - 1 ? inplane(2 * K + 2) : vzero<V>();
    const R z0 = K > 0 ? R(0.25) : R(0);
    const R z1 = K == 0 ? R(0.5) : R(0.75);
    const R z2 = K == Lc.nz - 1 ? R(0.5) : R(0.75);
    const R z3 = K < Lc.nz - 1 ? R(0.25) : R(0);
    const V v = vadd(vadd(vscale(sa, z0), vscale(sb, z1)), vadd(vscale(sc, z2), vscale(sd, z3)));
    if (m.in) fb[rb_index(Lc, m.i, m.j, K)] = v;
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
  // the column's bilinear in-plane weights, applied once per coarse plane (register ring
  // over the coarse planes instead of 8 coarse loads per fine cell)
  int Ix[2], Iy[2];
  float wx[2], wy[2];
  const int nxx = p1d_terms(m.i, ax, Lc.nx, Ix, wx);
  const int nyy = p1d_terms(m.j, ay, Lc.ny, Iy, wy);
  const int64_t cplane = (int64_t)Lc.nx * Lc.ny;
  auto inplane = [&](int K) {
    V s = vzero<V>();
    if (K < 0 || K >= Lc.nz) return s;
    if (Lc.split) {
      for (int p = 0; p < nyy; ++p)
        for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(eb[rb_index(Lc, Ix[o], Iy[p], K)], (R)(wy[p] * wx[o])));
      return s;
    }
    const V* pl = eb + K * cplane;
    for (int p = 0; p < nyy; ++p)
      for (int o = 0; o < nxx; ++o) s = vadd(s, vscale(pl[(int64_t)Iy[p] * Lc.nx + Ix[o]], (R)(wy[p] * wx[o])));
    return s;
  };
  if (Lf.dim == 2 || az == 1) {
    for (int k = m.k0; k < m.k1; ++k) {
      const int64_t a = rb_index(Lf, m.i, m.j, k);
      xb[a] = vadd(xb[a], inplane(Lf.dim == 2 ? 0 : k));
    }
    return;
  }
  // aggregation 2 in z: fine k takes 3/4 of coarse K = k / 2 and 1/4 of K - 1 (k even) or
  // K + 1 (k odd); at the ends the Dirichlet ghost makes it 1/2 of K (p1d_terms)
  int K = m.k0 >> 1;
  V sm = inplane(K - 1), sc = inplane(K), sp = inplane(K + 1);
  V xn = xb[rb_index(Lf, m.i, m.j, m.k0)];
  for (int k = m.k0; k < m.k1; ++k) {
    const int64_t a = rb_index(Lf, m.i, m.j, k);
    const V xc = xn;
    if (k + 1 < m.k1) xn = xb[rb_index(Lf, m.i, m.j, k + 1)];
    if ((k >> 1) != K) {
      K = k >> 1;
      sm = sc;
      sc = sp;
      sp = inplane(K + 1);
    }
    V v;
    if ((k & 1) == 0) v = K == 0 ? vscale(sc, R(0.5)) : vadd(vscale(sc, R(0.75)), vscale(sm, R(0.25)));
    else v = K == Lc.nz - 1 ? vscale(sc, R(0.5)) : vadd(vscale(sc, R(0.75)), vscale(sp, R(0.25)));
    xb[a] = vadd(xc, v);
  }
}

// q = A p, partial p^T q (FP64), z-marching; the operands of plane k + 1 (coefficients and the
// in-plane neighbours) are loaded while plane k is computed (software pipeline), the in-row
// neighbours come from the adjacent lanes
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
  const int lane = threadIdx.x & 31;
  const bool d3 = L.dim == 3;
  const double2 zero = make_double2(0.0, 0.0);
  double2 pm = zero, pc = zero, pp = zero;
  if (m.in) {
    if (m.k0 > 0) pm = pb[(m.k0 - 1) * plane + m.ip];
    pc = pb[m.k0 * plane + m.ip];
    if (m.k0 + 1 < L.nz) pp = pb[(m.k0 + 1) * plane + m.ip];
  }
  struct Ops {
    double tw, te, ts, tn, tb, tt, mm;
    double2 ps, pn, pw, pe;  // y neighbours, x neighbours across the tile edge
  };
  auto load_ops = [&](int k, Ops& o) {
    const int64_t a = k * plane + m.ip;
    const double* Txk = L.Tx + (int64_t)k * L.ny * nxp1 + (int64_t)m.j * nxp1 + m.i;
    const double* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx + m.ip;
    o.tw = __ldg(Txk);
    o.te = __ldg(Txk + 1);
    o.ts = __ldg(Tyk);
    o.tn = __ldg(Tyk + L.nx);
    o.tb = d3 ? __ldg(L.Tz + a) : 0.0;
    o.tt = d3 ? __ldg(L.Tz + a + plane) : 0.0;
    o.mm = __ldg(L.M + a);
    o.ps = m.j > 0 ? pb[a - L.nx] : zero;
    o.pn = m.j < L.ny - 1 ? pb[a + L.nx] : zero;
    o.pw = (lane == 0 && m.i > 0) ? pb[a - 1] : zero;
    o.pe = (lane == 31 && m.i + 1 < L.nx) ? pb[a + 1] : zero;
  };
  Ops cur, nxt;
  if (m.in) load_ops(m.k0, cur);
  double2 acc = zero;
  for (int k = m.k0; k < m.k1; ++k) {
    double2 pq = zero;
    if (m.in && k + 2 < L.nz && k + 1 < m.k1) pq = pb[(k + 2) * plane + m.ip];
    if (m.in && k + 1 < m.k1) load_ops(k + 1, nxt);
    const double2 up = make_double2(__shfl_up_sync(0xffffffffu, pc.x, 1), __shfl_up_sync(0xffffffffu, pc.y, 1));
    const double2 dn = make_double2(__shfl_down_sync(0xffffffffu, pc.x, 1), __shfl_down_sync(0xffffffffu, pc.y, 1));
    if (m.in) {
      const int64_t a = k * plane + m.ip;
      const double2 west = lane > 0 ? up : cur.pw;
      const double2 east = lane < 31 ? dn : cur.pe;
      const double dk = cur.tw + cur.te + cur.ts + cur.tn + cur.tb + cur.tt;
      double2 o = cscale(west, cur.tw);
      o = cfma(make_double2(cur.te, 0.0), east, o);
      o = cfma(make_double2(cur.ts, 0.0), cur.ps, o);
      o = cfma(make_double2(cur.tn, 0.0), cur.pn, o);
      o = cfma(make_double2(cur.tb, 0.0), pm, o);
      o = cfma(make_double2(cur.tt, 0.0), pp, o);
      const double2 d = make_double2(dk + tau.x * cur.mm, tau.y * cur.mm);
      const double2 qa = csub(cmul(d, pc), o);
      qb[a] = qa;
      acc = cfma(pc, qa, acc);
    }
    pm = pc;
    pc = pp;
    pp = pq;
    cur = nxt;
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = acc;
}

// ---- pair z-marching kernels (nx even) ----------------------------------------------------
// A thread owns two x-adjacent cells (i0, i0 + 1), i0 even.  In a red-black half sweep exactly
// one of the two has the sweep's colour on every plane, so every lane does useful work (the
// one-cell kernel idles half its lanes and was issue-bound), the pair moves as one 16-byte
// access, and the in-row neighbours come from the adjacent lanes by shuffle (a warp is one
// row of 64 cells).  CTA = 32 pairs x 8 rows x a chunk of ZM_ZC planes.
// The chunk of planes per CTA shrinks on the small levels (ZM_ZC on nz >= 64, else nz / 8, at
// least 2): they are latency-bound, and with 32-plane chunks a 32^3 level had 4 CTAs per item.
constexpr int ZP_TX = 32;
__host__ __device__ __forceinline__ int zp_chunk(int nz) { return nz >= 64 ? ZM_ZC : (nz >= 16 ? nz / 8 : 2); }

// Rows of <= 32 cells: a warp covers two rows (16 pairs each), so no lane idles; the tile is
// then 32 x 16 cells.
__host__ __device__ __forceinline__ int zp_rows(int nx) { return nx <= ZP_TX ? 2 : 1; }

template <class VW>
inline int zp_blocks(const VW& L) {
  const int zc = zp_chunk(L.nz), ty = ZM_TY * zp_rows(L.nx);
  return ((L.nx + 2 * ZP_TX - 1) / (2 * ZP_TX)) * ((L.ny + ty - 1) / ty) * ((L.nz + zc - 1) / zc);
}

template <class V>
struct Pair {
  V a, c;  // cells i0, i0 + 1
};

template <class V>
__device__ __forceinline__ Pair<V> ld_pair(const V* p) {
  if constexpr (sizeof(V) == 8) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    return {V{t.x, t.y}, V{t.z, t.w}};
  } else {
    return {p[0], p[1]};
  }
}

template <class V>
__device__ __forceinline__ void st_pair(V* p, const Pair<V>& v) {
  if constexpr (sizeof(V) == 8) {
    *reinterpret_cast<float4*>(p) = make_float4(v.a.x, v.a.y, v.c.x, v.c.y);
  } else {
    p[0] = v.a;
    p[1] = v.c;
  }
}

template <class V>
__device__ __forceinline__ V shfl_up1(V v) {
  return V{__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1)};
}
template <class V>
__device__ __forceinline__ V shfl_down1(V v) {
  return V{__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1)};
}

template <class V>
__device__ __forceinline__ V pick(const Pair<V>& p, int o) {
  return o ? p.c : p.a;
}

struct ZpMap {
  int i0, j, k0, k1, lane;
  bool first, last;  // first / last pair of the warp's row segment (x-neighbours from memory)
  bool in;
  int64_t ip;
};

template <class VW>
__device__ __forceinline__ ZpMap zp_map(const VW& L, int cb) {
  const int rows = zp_rows(L.nx), seg = 32 / rows;  // row segments per warp, pairs per segment
  const int tiles_x = (L.nx + 2 * ZP_TX - 1) / (2 * ZP_TX), tiles_y = (L.ny + ZM_TY * rows - 1) / (ZM_TY * rows);
  const int ntile = tiles_x * tiles_y;
  const int tile = cb % ntile, chunk = cb / ntile;
  ZpMap m;
  m.lane = threadIdx.x & 31;
  const int rl = m.lane % seg;
  m.first = rl == 0;
  m.last = rl == seg - 1;
  m.i0 = (tile % tiles_x) * 2 * ZP_TX + 2 * rl;
  m.j = (tile / tiles_x) * ZM_TY * rows + (threadIdx.x >> 5) * rows + m.lane / seg;
  m.in = m.i0 < L.nx && m.j < L.ny;
  const int zc = zp_chunk(L.nz);
  m.k0 = chunk * zc;
  m.k1 = min(L.nz, m.k0 + zc);
  m.ip = (int64_t)m.j * L.nx + m.i0;
  return m;
}

// Red-black half sweep of colour `color` on cell pairs, in place (see rbhalf_zm_kernel for why
// in place is race free).  zero_init: x = 0 on entry.  dot != null: also the partial
// sum_a f_a x_a over all cells after the sweep (the COCG rho = r^T z fused into the last
// sweep of the V-cycle: f is the multigrid copy of r on the finest level).
template <class R>
__global__ void __launch_bounds__(kT, 3) rbpair_zm_kernel(LevelViewT<R> L, Batch bt, const double2* __restrict__ taus,
                                                       const typename CT<R>::V* __restrict__ f,
                                                       typename CT<R>::V* x, int color, int zero_init,
                                                       double2* __restrict__ dot, int nblk) {
  using V = typename CT<R>::V;
  using PV = Pair<V>;
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZpMap m = zp_map(L, cb);
  const int64_t plane = (int64_t)L.nx * L.ny;
  V* xb = x + (int64_t)b * L.n;
  const V* fb = f + (int64_t)b * L.n;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  const int nxp1 = L.nx + 1;
  const bool d3 = L.dim == 3;
  const PV pz{vzero<V>(), vzero<V>()};
  PV xm = pz, xc = pz, xp = pz;
  if (m.in && !zero_init) {
    if (m.k0 > 0) xm = ld_pair(xb + (m.k0 - 1) * plane + m.ip);
    xc = ld_pair(xb + m.k0 * plane + m.ip);
    if (m.k0 + 1 < L.nz) xp = ld_pair(xb + (m.k0 + 1) * plane + m.ip);
  }
  struct Ops {
    R tw, te, ts, tn, tb, tt, mm;
    PV fv, ns, nn;
    V xw, xe;  // x-neighbours across the tile edge (lanes 0 / 31 only)
  };
  auto load_ops = [&](int k, Ops& o) {
    const int off = (m.j + k + color) & 1;
    const int64_t a = k * plane + m.ip;
    const int ic = m.i0 + off;
    const R* Txk = L.Tx + (int64_t)k * L.ny * nxp1 + (int64_t)m.j * nxp1 + ic;
    const R* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx + (int64_t)m.j * L.nx + ic;
    o.tw = __ldg(Txk);
    o.te = __ldg(Txk + 1);
    o.ts = __ldg(Tyk);
    o.tn = __ldg(Tyk + L.nx);
    o.tb = d3 ? __ldg(L.Tz + a + off) : R(0);
    o.tt = d3 ? __ldg(L.Tz + a + off + plane) : R(0);
    o.mm = __ldg(L.M + a + off);
    o.fv = ld_pair(fb + a);
    o.ns = pz;
    o.nn = pz;
    o.xw = vzero<V>();
    o.xe = vzero<V>();
    if (!zero_init) {
      if (m.j > 0) o.ns = ld_pair(xb + a - L.nx);
      if (m.j < L.ny - 1) o.nn = ld_pair(xb + a + L.nx);
      if (off == 0 && m.first && m.i0 > 0) o.xw = xb[a - 1];
      if (off == 1 && m.last && m.i0 + 2 < L.nx) o.xe = xb[a + 2];
    }
  };
  Ops cur, nxt;
  if (m.in) load_ops(m.k0, cur);
  double2 acc = make_double2(0.0, 0.0);
  for (int k = m.k0; k < m.k1; ++k) {
    PV xn = pz;
    if (m.in && !zero_init && k + 2 < L.nz && k + 1 < m.k1) xn = ld_pair(xb + (k + 2) * plane + m.ip);
    if (m.in && k + 1 < m.k1) load_ops(k + 1, nxt);
    const int off = (m.j + k + color) & 1;
    // in-row neighbours of the colour cell from the adjacent lanes (every lane shuffles)
    const V up = shfl_up1(xc.c), dn = shfl_down1(xc.a);
    if (m.in) {
      const V west = off ? xc.a : (!m.first ? up : cur.xw);
      const V east = off ? (!m.last ? dn : cur.xe) : xc.c;
      const R dk = cur.tw + cur.te + cur.ts + cur.tn + cur.tb + cur.tt;
      V o = pick(cur.fv, off);
      o = vadd(o, vadd(vadd(vscale(west, cur.tw), vscale(east, cur.te)),
                       vadd(vscale(pick(cur.ns, off), cur.ts), vscale(pick(cur.nn, off), cur.tn))));
      o = vadd(o, vadd(vscale(pick(xm, off), cur.tb), vscale(pick(xp, off), cur.tt)));
      const V nv = diag_solve_r<R, V>(dk, cur.mm, tr, ti, o);
      PV out = xc;
      if (off) out.c = nv;
      else out.a = nv;
      st_pair(xb + k * plane + m.ip, out);
      if (dot) {
        const double2 fa = vto(cur.fv.a), fc = vto(cur.fv.c);
        acc = cfma(fa, vto(out.a), acc);
        acc = cfma(fc, vto(out.c), acc);
      }
    }
    xm = xc;
    xc = xp;
    xp = xn;
    cur = nxt;
  }
  if (dot) {
    acc = block_sum(acc);
    if (threadIdx.x == 0) dot[(int64_t)b * nblk + cb] = acc;
  }
}

// r = f - A(tau) x on cell pairs (precision R)
template <class R>
__global__ void __launch_bounds__(kT, 3) residual_pair_zm_kernel(LevelViewT<R> L, Batch bt,
                                                              const double2* __restrict__ taus,
                                                              const typename CT<R>::V* __restrict__ f,
                                                              const typename CT<R>::V* __restrict__ x,
                                                              typename CT<R>::V* __restrict__ r) {
  using V = typename CT<R>::V;
  using PV = Pair<V>;
  using R2 = typename CT<R>::V;  // two coefficients of a pair
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const ZpMap m = zp_map(L, cb);
  const int64_t plane = (int64_t)L.nx * L.ny;
  const V* xb = x + (int64_t)b * L.n;
  const V* fb = f + (int64_t)b * L.n;
  V* rb = r + (int64_t)b * L.n;
  const R tr = (R)taus[b].x, ti = (R)taus[b].y;
  const int nxp1 = L.nx + 1;
  const bool d3 = L.dim == 3;
  const PV pz{vzero<V>(), vzero<V>()};
  PV xm = pz, xc = pz, xp = pz;
  if (m.in) {
    if (m.k0 > 0) xm = ld_pair(xb + (m.k0 - 1) * plane + m.ip);
    xc = ld_pair(xb + m.k0 * plane + m.ip);
    if (m.k0 + 1 < L.nz) xp = ld_pair(xb + (m.k0 + 1) * plane + m.ip);
  }
  struct Ops {
    R tx0, tx1, tx2;
    R2 ts, tn, tb, tt, mm;
    PV fv, ns, nn;
    V xw, xe;
  };
  auto ld_r2 = [](const R* p) { return R2{__ldg(p), __ldg(p + 1)}; };
  auto load_ops = [&](int k, Ops& o) {
    const int64_t a = k * plane + m.ip;
    const R* Txk = L.Tx + (int64_t)k * L.ny * nxp1 + (int64_t)m.j * nxp1 + m.i0;
    const R* Tyk = L.Ty + (int64_t)k * (L.ny + 1) * L.nx + m.ip;
    o.tx0 = __ldg(Txk);
    o.tx1 = __ldg(Txk + 1);
    o.tx2 = __ldg(Txk + 2);
    o.ts = ld_r2(Tyk);
    o.tn = ld_r2(Tyk + L.nx);
    o.tb = d3 ? ld_r2(L.Tz + a) : R2{0, 0};
    o.tt = d3 ? ld_r2(L.Tz + a + plane) : R2{0, 0};
    o.mm = ld_r2(L.M + a);
    o.fv = ld_pair(fb + a);
    o.ns = m.j > 0 ? ld_pair(xb + a - L.nx) : pz;
    o.nn = m.j < L.ny - 1 ? ld_pair(xb + a + L.nx) : pz;
    o.xw = (m.first && m.i0 > 0) ? xb[a - 1] : vzero<V>();
    o.xe = (m.last && m.i0 + 2 < L.nx) ? xb[a + 2] : vzero<V>();
  };
  Ops cur, nxt;
  if (m.in) load_ops(m.k0, cur);
  for (int k = m.k0; k < m.k1; ++k) {
    PV xn = pz;
    if (m.in && k + 2 < L.nz && k + 1 < m.k1) xn = ld_pair(xb + (k + 2) * plane + m.ip);
    if (m.in && k + 1 < m.k1) load_ops(k + 1, nxt);
    const V up = shfl_up1(xc.c), dn = shfl_down1(xc.a);
    if (m.in) {
      const V west = !m.first ? up : cur.xw;
      const V east = !m.last ? dn : cur.xe;
      PV out;
      {  // cell i0: neighbours west, xc.c
        const R dk = cur.tx0 + cur.tx1 + cur.ts.x + cur.tn.x + cur.tb.x + cur.tt.x;
        V o = vadd(vadd(vscale(west, cur.tx0), vscale(xc.c, cur.tx1)),
                   vadd(vscale(cur.ns.a, cur.ts.x), vscale(cur.nn.a, cur.tn.x)));
        o = vadd(o, vadd(vscale(xm.a, cur.tb.x), vscale(xp.a, cur.tt.x)));
        const R dr = dk + tr * cur.mm.x, di = ti * cur.mm.x;
        out.a = V{cur.fv.a.x - (dr * xc.a.x - di * xc.a.y - o.x), cur.fv.a.y - (dr * xc.a.y + di * xc.a.x - o.y)};
      }
      {  // cell i0 + 1: neighbours xc.a, east
        const R dk = cur.tx1 + cur.tx2 + cur.ts.y + cur.tn.y + cur.tb.y + cur.tt.y;
        V o = vadd(vadd(vscale(xc.a, cur.tx1), vscale(east, cur.tx2)),
                   vadd(vscale(cur.ns.c, cur.ts.y), vscale(cur.nn.c, cur.tn.y)));
        o = vadd(o, vadd(vscale(xm.c, cur.tb.y), vscale(xp.c, cur.tt.y)));
        const R dr = dk + tr * cur.mm.y, di = ti * cur.mm.y;
        out.c = V{cur.fv.c.x - (dr * xc.c.x - di * xc.c.y - o.x), cur.fv.c.y - (dr * xc.c.y + di * xc.c.x - o.y)};
      }
      st_pair(rb + k * plane + m.ip, out);
    }
    xm = xc;
    xc = xp;
    xp = xn;
    cur = nxt;
  }
}

// ---- TMA-fed z-marching kernels (large levels, nx even) -----------------------------------
// A CTA owns an (x, y) tile and marches a chunk of planes.  One thread issues the tensor-memory
// copies of each plane's operand tiles -- the iterate with a halo, the right-hand side and the
// packed coefficients -- into a ring of TZ_D plane slots in shared memory, TZ_D - 2 planes
// ahead of the plane being computed, each slot signalled by an mbarrier.  The bytes in flight
// no longer depend on registers and occupancy (the register-pipelined kernels reached only
// ~50% of HBM bandwidth), neighbours come from shared memory (no shuffles or edge loads), and
// the domain boundary is the TMA out-of-bounds zero fill.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Ring bookkeeping shared by the kernels: plane p (k0 - 1 <= p <= k1) lives in slot
// (p - k0 + 1) % D, and its barrier phase parity is ((p - k0 + 1) / D) & 1.
template <int D>
struct ZRing {
  int k0;
  __device__ __forceinline__ int slot(int p) const { return (p - k0 + 1) % D; }
  __device__ __forceinline__ uint32_t parity(int p) const { return (uint32_t)(((p - k0 + 1) / D) & 1); }
};

struct TzDims {
  int nx, ny, nz;
  int64_t n;
};

// FP32 multigrid tiles: 64 x 8 cells (32 pairs x 8 rows)
constexpr int TZ_W = 64, TZ_H = 8;
constexpr int TZ_XW = TZ_W + 4, TZ_XH = TZ_H + 2;  // iterate x0-2 .. x0+65, y0-1 .. y0+8
constexpr int TZ_CW = TZ_W + 1, TZ_CH = TZ_H + 1;  // packed coefficients x0 .. x0+64, y0 .. y0+8
constexpr int TZ_D = 5;
constexpr uint32_t TZ_XB = sizeof(float2) * TZ_XW * TZ_XH;  // 5440
constexpr uint32_t TZ_FB = sizeof(float2) * TZ_W * TZ_H;    // 4096
constexpr uint32_t TZ_CB = sizeof(float4) * TZ_CW * TZ_CH;  // 9360
constexpr uint32_t TZ_OFF_F = 5504, TZ_OFF_C = TZ_OFF_F + 4096, TZ_SLOT = TZ_OFF_C + 9472;  // 128-byte aligned
constexpr size_t TZ_SMEM = (size_t)TZ_SLOT * TZ_D;

template <class VW>
inline int tz_blocks(const VW& L) {
  return ((L.nx + TZ_W - 1) / TZ_W) * ((L.ny + TZ_H - 1) / TZ_H) * ((L.nz + ZM_ZC - 1) / ZM_ZC);
}

// Producer / consumer layout of the TMA kernels: warps 0..7 compute (one (x, y) cell or pair
// each), warp 8 is the producer -- one lane issues each plane's copies into the ring once the
// eight consumer warps have released that slot (per-slot "empty" barrier, one arrival per
// consumer warp), so consumer warps never wait on each other and the loads run TZ_D - 2
// planes ahead of the slowest warp.
constexpr int kTP = kT + 32;

// mode 0: red-black half sweep of `color` in place on x (zero_init: x = 0 on entry; dot: also
// the partials of f^T x after the sweep); mode 1: r = f - A x.
template <int MODE>
__global__ void __launch_bounds__(kTP, 2) mg_tma_kernel(const __grid_constant__ CUtensorMap mx,
                                                        const __grid_constant__ CUtensorMap mf,
                                                        const __grid_constant__ CUtensorMap mc, TzDims L, Batch bt,
                                                        const double2* __restrict__ taus, float2* __restrict__ out,
                                                        int color, int zero_init, double2* __restrict__ dot, int nblk) {
  extern __shared__ __align__(128) unsigned char tz_smem[];
  __shared__ __align__(8) uint64_t full[TZ_D], empty[TZ_D];
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int tiles_x = (L.nx + TZ_W - 1) / TZ_W, tiles_y = (L.ny + TZ_H - 1) / TZ_H;
  const int ntile = tiles_x * tiles_y;
  const int tile = cb % ntile, chunk = cb / ntile;
  const int x0 = (tile % tiles_x) * TZ_W, y0 = (tile / tiles_x) * TZ_H;
  const int k0 = chunk * ZM_ZC, k1 = min(L.nz, k0 + ZM_ZC);
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  const ZRing<TZ_D> ring{k0};
  if (tid == 0) {
    for (int s = 0; s < TZ_D; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kT / 32);
    }
    mbar_init_fence();
  }
  __syncthreads();
  double2 acc = make_double2(0.0, 0.0);
  if (wy == kT / 32) {  // producer warp
    if (lane == 0) {
      const bool ldx = MODE == 1 || !zero_init;
      for (int p = k0 - 1; p <= k1; ++p) {
        const int use = (p - k0 + 1) / TZ_D, s = ring.slot(p);
        if (use > 0) mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
        unsigned char* sp = tz_smem + (size_t)s * TZ_SLOT;
        const bool lf = p >= k0 && p < k1, lc = p >= k0;
        mbar_arrive_tx(&full[s], (ldx ? TZ_XB : 0u) + (lf ? TZ_FB : 0u) + (lc ? TZ_CB : 0u));
        if (ldx) tma_load4(sp, &mx, x0 - 2, y0 - 1, p, b, &full[s]);
        if (lf) tma_load4(sp + TZ_OFF_F, &mf, x0, y0, p, b, &full[s]);
        if (lc) tma_load3(sp + TZ_OFF_C, &mc, 2 * x0, y0, p, &full[s]);
      }
    }
  } else {
    const int i0 = x0 + 2 * lane, j = y0 + wy;
    const bool in = i0 < L.nx && j < L.ny;
    const float tr = (float)taus[b].x, ti = (float)taus[b].y;
    const int64_t plane = (int64_t)L.nx * L.ny;
    float2* ob = out + (int64_t)b * L.n;
    for (int k = k0; k < k1; ++k) {
      mbar_wait(&full[ring.slot(k - 1)], ring.parity(k - 1));
      mbar_wait(&full[ring.slot(k)], ring.parity(k));
      mbar_wait(&full[ring.slot(k + 1)], ring.parity(k + 1));
      const unsigned char* sm = tz_smem + (size_t)ring.slot(k - 1) * TZ_SLOT;
      const unsigned char* s0 = tz_smem + (size_t)ring.slot(k) * TZ_SLOT;
      const unsigned char* sp = tz_smem + (size_t)ring.slot(k + 1) * TZ_SLOT;
      auto X = [](const unsigned char* s, int yy, int xx) { return reinterpret_cast<const float2*>(s)[yy * TZ_XW + xx]; };
      auto F = [](const unsigned char* s, int yy, int xx) {
        return reinterpret_cast<const float2*>(s + TZ_OFF_F)[yy * TZ_W + xx];
      };
      auto Cf = [](const unsigned char* s, int yy, int xx) {
        return reinterpret_cast<const float4*>(s + TZ_OFF_C)[yy * TZ_CW + xx];
      };
      if (in) {
        const int c0 = 2 * lane;  // pair's first cell in F / C tile coordinates (X: + 2, + 1 row)
        float2* dst = ob + k * plane + (int64_t)j * L.nx + i0;
        if (MODE == 0) {
          const int off = (j + k + color) & 1;
          const int cx = c0 + off, xx = cx + 2;
          const float4 cc = Cf(s0, wy, cx);
          const float te = Cf(s0, wy, cx + 1).x, tn = Cf(s0, wy + 1, cx).y, tt = Cf(sp, wy, cx).z;
          const float dk = cc.x + te + cc.y + tn + cc.z + tt;
          float2 o = F(s0, wy, cx);
          float4 pr = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!zero_init) {
            pr = *reinterpret_cast<const float4*>(&reinterpret_cast<const float2*>(s0)[(wy + 1) * TZ_XW + c0 + 2]);
            const float2 w = X(s0, wy + 1, xx - 1), e = X(s0, wy + 1, xx + 1);
            const float2 so = X(s0, wy, xx), no = X(s0, wy + 2, xx);
            const float2 dn = X(sm, wy + 1, xx), up = X(sp, wy + 1, xx);
            o.x += cc.x * w.x + te * e.x + cc.y * so.x + tn * no.x + cc.z * dn.x + tt * up.x;
            o.y += cc.x * w.y + te * e.y + cc.y * so.y + tn * no.y + cc.z * dn.y + tt * up.y;
          }
          const float2 nv = diag_solve_r<float, float2>(dk, cc.w, tr, ti, o);
          if (off) {
            pr.z = nv.x;
            pr.w = nv.y;
          } else {
            pr.x = nv.x;
            pr.y = nv.y;
          }
          *reinterpret_cast<float4*>(dst) = pr;
          if (dot) {
            const float2 fa = F(s0, wy, c0), fc = F(s0, wy, c0 + 1);
            acc = cfma(make_double2(fa.x, fa.y), make_double2(pr.x, pr.y), acc);
            acc = cfma(make_double2(fc.x, fc.y), make_double2(pr.z, pr.w), acc);
          }
        } else {
          const float4 pr =
              *reinterpret_cast<const float4*>(&reinterpret_cast<const float2*>(s0)[(wy + 1) * TZ_XW + c0 + 2]);
          const float2 xa = make_float2(pr.x, pr.y), xc = make_float2(pr.z, pr.w);
          float4 res;
          {
            const float4 ca = Cf(s0, wy, c0);
            const float te = Cf(s0, wy, c0 + 1).x, tn = Cf(s0, wy + 1, c0).y, tt = Cf(sp, wy, c0).z;
            const float2 w = X(s0, wy + 1, c0 + 1), so = X(s0, wy, c0 + 2), no = X(s0, wy + 2, c0 + 2);
            const float2 dn = X(sm, wy + 1, c0 + 2), up = X(sp, wy + 1, c0 + 2);
            const float dk = ca.x + te + ca.y + tn + ca.z + tt;
            const float dr = dk + tr * ca.w, di = ti * ca.w;
            const float ox = ca.x * w.x + te * xc.x + ca.y * so.x + tn * no.x + ca.z * dn.x + tt * up.x;
            const float oy = ca.x * w.y + te * xc.y + ca.y * so.y + tn * no.y + ca.z * dn.y + tt * up.y;
            const float2 f = F(s0, wy, c0);
            res.x = f.x - (dr * xa.x - di * xa.y - ox);
            res.y = f.y - (dr * xa.y + di * xa.x - oy);
          }
          {
            const float4 ca = Cf(s0, wy, c0 + 1);
            const float te = Cf(s0, wy, c0 + 2).x, tn = Cf(s0, wy + 1, c0 + 1).y, tt = Cf(sp, wy, c0 + 1).z;
            const float2 e = X(s0, wy + 1, c0 + 4), so = X(s0, wy, c0 + 3), no = X(s0, wy + 2, c0 + 3);
            const float2 dn = X(sm, wy + 1, c0 + 3), up = X(sp, wy + 1, c0 + 3);
            const float dk = ca.x + te + ca.y + tn + ca.z + tt;
            const float dr = dk + tr * ca.w, di = ti * ca.w;
            const float ox = ca.x * xa.x + te * e.x + ca.y * so.x + tn * no.x + ca.z * dn.x + tt * up.x;
            const float oy = ca.x * xa.y + te * e.y + ca.y * so.y + tn * no.y + ca.z * dn.y + tt * up.y;
            const float2 f = F(s0, wy, c0 + 1);
            res.z = f.x - (dr * xc.x - di * xc.y - ox);
            res.w = f.y - (dr * xc.y + di * xc.x - oy);
          }
          *reinterpret_cast<float4*>(dst) = res;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ring.slot(k - 1)]);  // this warp is done with plane k - 1
    }
  }
  if (MODE == 0 && dot) {
    acc = block_sum(acc);
    if (threadIdx.x == 0) dot[(int64_t)b * nblk + cb] = acc;
  }
}

// ---- colour-split (red-black ordered) TMA kernels -----------------------------------------
// On levels with nx % 4 == 0 and nx >= 64 the multigrid vectors are stored colour-split: in
// every row (j, k) the cells of colour 0 ((i + j + k) even) come first, ordered by i, then
// those of colour 1; cell i sits at position i / 2 of its colour's half (rb_index).  Then
//  * every cell of one colour in a row is one contiguous run, and so are its six neighbours
//    (W / E at positions m - 1 + s / m + s of the other half, s = the row's parity offset;
//    S / N / down / up at position m of the other half of the adjacent rows / planes), so a
//    warp on 32 same-colour cells reads every operand as one 256-byte run: the natural-layout
//    half sweep read stride-2 cells and stride-32-byte coefficient records, and was bound by
//    shared-memory wavefronts (~64 per 64 cells), not by HBM;
//  * a half sweep moves only half of each vector: it reads the other colour of x and its own
//    colour of f and writes its own colour -- 1.5 complex64 per cell instead of 3 -- and the
//    first sweep from zero reads no x at all.
// The coefficients are stored the same way, planar (Level::packrb), so E = W(i + 1), N and T
// are contiguous runs of the other half as well.
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

// Tile: 32 positions (one warp, 64 cells of a row) x RB_H rows, z-march over ZM_ZC planes,
// for NI items at once (the items share the coefficient tiles and every coefficient-derived
// register: a half sweep runs 2 items per CTA, the residual 1).  Per plane slot and item: x
// (the other colour for a half sweep, both for the residual) over rows y0-1 .. y0+RB_H and
// positions m0-2 .. m0+33, f over the tile (own colour; both with dot or for the residual);
// once per slot the coefficients of both colours over rows y0 .. y0+RB_H, positions
// m0 .. m0+35.
#ifndef RB_DEPTH
#define RB_DEPTH (RB_BF16 ? 7 : 5)
#endif
#ifndef RB_MINB
#define RB_MINB 2
#endif
#ifndef RB_NI
#define RB_NI 2  // items per CTA of the colour-split half sweeps
#endif
// coefficient rows of the slot: RB_P + 1 positions, padded to a 16-byte multiple
constexpr int RB_P = 32, RB_H = 8, RB_XP = RB_P + 4, RB_CP = RB_P + (RB_BF16 ? 8 : 4), RB_D = RB_DEPTH;
__device__ __forceinline__ float rb_coef(float v) { return v; }
__device__ __forceinline__ float rb_coef(unsigned short v) { return __uint_as_float((uint32_t)v << 16); }  // bf16 bits
// persistent launches of the colour-split half sweeps (RB_PERSIST=0: one CTA per work item).
// Measured at configs[4], 80 items: half sweeps 128^3 38.8 -> 38.3 ms, 64^3 13.3 -> 12.4 ms per
// inner solve; the residual (one item per CTA) is faster with one CTA per work item (8.2 vs
// 9.6 ms) and stays that way.
#ifndef RB_PERSIST
#define RB_PERSIST 1
#endif
template <int MODE, int NI>
struct RbSlot {
  static constexpr int NX = MODE == 0 ? 1 : 2;  // colours of x in the slot
  static constexpr uint32_t XB = sizeof(float2) * RB_XP * NX * (RB_H + 2);     // per item
  static constexpr uint32_t XBA = (XB + 127) / 128 * 128;
  // f per item: both colours when NI == 1 (residual, or a sweep forming f^T x), else its own
  static constexpr uint32_t FB = sizeof(float2) * RB_P * (NI == 1 ? 2 : 1) * RB_H;
  static constexpr uint32_t CB = sizeof(rb_coef_t) * RB_CP * 2 * 4 * (RB_H + 1);
  static constexpr uint32_t OFF_F = XBA * NI;
  static constexpr uint32_t OFF_C = OFF_F + FB * NI;
  // the slot's own full / empty mbarriers sit behind its data, so one slot address reaches
  // the data and both barriers with immediate offsets
  static constexpr uint32_t OFF_FULL = (OFF_C + CB + 15) / 16 * 16, OFF_EMPTY = OFF_FULL + 8;
  static constexpr uint32_t SLOT = (OFF_EMPTY + 8 + 127) / 128 * 128;
  static constexpr int D = NI >= 4 ? 4 : RB_D;  // ring depth (4 items: 4 deep, 2 CTAs per SM)
  static constexpr size_t SMEM = (size_t)SLOT * D;
};

// planes per CTA: ZM_ZC on the finest levels; shorter chunks below (64^3 x 80 items with 32-plane
// chunks is 640 CTAs = 2.2 waves of 296 resident CTAs, a 16%-full last wave)
#ifndef RB_ZC_SMALL
#define RB_ZC_SMALL 16
#endif
__host__ __device__ __forceinline__ int rb_zc(int nz) { return nz >= 128 ? ZM_ZC : RB_ZC_SMALL; }

// CTAs of a persistent launch: RB_MINB per SM
inline unsigned rb_persist_grid(lt_ctx ctx) {
  return RB_PERSIST ? (unsigned)(ctx->num_sms * RB_MINB) : 0xffffffffu;
}

template <class VW>
inline int rb_blocks(const VW& L) {
  const int zc = rb_zc(L.nz);
  return ((L.nx / 2 + RB_P - 1) / RB_P) * ((L.ny + RB_H - 1) / RB_H) * ((L.nz + zc - 1) / zc);
}

__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
// 1 / x by MUFU alone (1 ulp-class; __frcp_rn adds a range check and a slow path per call).  The
// half sweep's diagonal inverse only has to be the same in the pre- and the post-smoother.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// MODE 0: red-black half sweep of `color`, in place on the colour's half of x (ZI: x = 0 on
// entry, so no x is read; DOT: also the partials of f^T x over the colour's cells, written to
// dot[((item * 2 + color) * nblk + block] -- the last black and the last red sweep of the
// post-smoother together form f^T x).  MODE 1: r = f - A x on both
// colours.  mx / mf: 5-D maps {pos, colour, y, z, item} of x and f with the slot's boxes, mc:
// {pos, colour, comp, y, z} of Level::packrb.  Work items: rb_blocks(L) per group of NI
// consecutive items (item group fastest), zc planes each.
//
// The consumer loop is written for instruction count (ncu: the previous version issued 231
// warp instructions per plane, 2.9x its loads and arithmetic, at 64-68% issue utilisation):
// every shared-memory operand is one of six per-plane base registers plus an immediate, the
// store pointers advance by a plane, and ZI / DOT are compile time.
template <int MODE, int NI, bool ZI, bool DOT>
__global__ void __launch_bounds__(kTP, RB_MINB) mg_rb_kernel(const __grid_constant__ CUtensorMap mx,
                                                       const __grid_constant__ CUtensorMap mf,
                                                       const __grid_constant__ CUtensorMap mc, TzDims L, Batch bt,
                                                       const double2* __restrict__ taus, float2* __restrict__ out,
                                                       int color, double2* __restrict__ dot, int nblk, int zc) {
  using S = RbSlot<MODE, NI>;
  extern __shared__ __align__(128) unsigned char rb_smem[];
  // Work items w = block * ngroups + item group, taken grid-strided: a persistent launch (fewer
  // CTAs than work items) keeps its plane ring running across work items, so
  // the next item's first planes are in flight while the last planes of this one are computed.
  const int ngroups = (bt.B + NI - 1) / NI;
  const int nwork = nblk * ngroups;
  const int nh = L.nx >> 1;
  const int tiles_x = (nh + RB_P - 1) / RB_P, tiles_y = (L.ny + RB_H - 1) / RB_H;
  const int ntile = tiles_x * tiles_y;
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  constexpr bool fboth = NI == 1 && MODE == 1;  // f of both colours in the slot (residual)
  constexpr int nf = fboth ? 2 : 1;
  const uint32_t ring0 = smem_u32(rb_smem);
  constexpr uint32_t RING = (uint32_t)(S::D * S::SLOT);
  if (tid == 0) {
    for (int q = 0; q < S::D; ++q) {
      mbar_init(reinterpret_cast<uint64_t*>(rb_smem + (size_t)q * S::SLOT + S::OFF_FULL), 1);
      mbar_init(reinterpret_cast<uint64_t*>(rb_smem + (size_t)q * S::SLOT + S::OFF_EMPTY), kT / 32);
    }
    mbar_init_fence();
  }
  __syncthreads();
  double2 acc[NI];
#pragma unroll
  for (int t = 0; t < NI; ++t) acc[t] = make_double2(0.0, 0.0);
  __shared__ double2 dsh[2][NI][kT / 32];  // DOT: per-warp partials of a work item
  int par = 0;
  uint32_t an = 0;      // slot (byte offset in the ring) of the next plane: the same sequence in producer and consumers
  uint32_t un = 0;      // its use count (producer) / phase parity (consumers)
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int grp = w % ngroups, cb = w / ngroups;
    bool live[NI];
    int nlive = 0;
#pragma unroll
    for (int t = 0; t < NI; ++t) {
      const int b = grp * NI + t;
      live[t] = b < bt.B && !bt.done[b];
      nlive += live[t];
    }
    if (nlive == 0) continue;
    const int tile = cb % ntile, chunk = cb / ntile;
    const int m0 = (tile % tiles_x) * RB_P, y0 = (tile / tiles_x) * RB_H;
    const int k0 = chunk * zc, k1 = min(L.nz, k0 + zc);
    if (wy == kT / 32) {  // producer warp
      if (lane == 0) {
        constexpr bool ldx = MODE == 1 || !ZI;
        constexpr uint32_t fb = fboth || NI > 1 ? S::FB : S::FB / 2;
        const uint32_t bytes_xf = ldx ? (uint32_t)nlive * S::XB : 0u;
        for (int p = k0 - 1; p <= k1; ++p) {
          unsigned char* sp = rb_smem + an;
          uint64_t* fullb = reinterpret_cast<uint64_t*>(sp + S::OFF_FULL);
          if (un > 0) mbar_wait(reinterpret_cast<uint64_t*>(sp + S::OFF_EMPTY), (un - 1) & 1u);
          const bool lf = p >= k0 && p < k1, lc = p >= k0;
          const uint32_t bytes = bytes_xf + (lc ? S::CB : 0u) + (lf ? (uint32_t)nlive * fb : 0u);
          mbar_arrive_tx(fullb, bytes);  // 0 bytes (plane k0 - 1 of a sweep from zero) completes the phase
#pragma unroll
          for (int t = 0; t < NI; ++t) {
            if (!live[t]) continue;
            const int b = grp * NI + t;
            if (ldx) tma_load5(sp + t * S::XBA, &mx, m0 - 2, MODE == 0 ? color ^ 1 : 0, y0 - 1, p, b, fullb);
            if (lf) tma_load5(sp + S::OFF_F + t * S::FB, &mf, m0, fboth ? 0 : color, y0, p, b, fullb);
          }
          if (lc) tma_load5(sp + S::OFF_C, &mc, m0, 0, 0, y0, p, fullb);
          an += S::SLOT;
          if (an == RING) { an = 0; ++un; }
        }
      }
    } else {
      const int m = m0 + lane, j = y0 + wy;
      const bool in = m < nh && j < L.ny;
      float tr[NI], ti[NI];
      float2* op[NI];  // this thread's output cell of plane k, colour 0's half of the row
#pragma unroll
      for (int t = 0; t < NI; ++t) {
        const int b = min(grp * NI + t, bt.B - 1);
        tr[t] = (float)taus[b].x;
        ti[t] = (float)taus[b].y;
        op[t] = out + (int64_t)b * L.n + ((int64_t)k0 * L.ny + j) * L.nx + m + (MODE == 0 ? (int64_t)color * nh : 0);
      }
      const int64_t plane = (int64_t)L.nx * L.ny;
      // ring: planes k - 1, k, k + 1 in slots am, a0, au; au's phase parity pu
      uint32_t am = an;
      mbar_wait_u32(ring0 + an + S::OFF_FULL, un);
      an += S::SLOT;
      if (an == RING) { an = 0; un ^= 1u; }
      uint32_t a0 = an;
      mbar_wait_u32(ring0 + an + S::OFF_FULL, un);
      an += S::SLOT;
      if (an == RING) { an = 0; un ^= 1u; }
      uint32_t au = an, pu = un;
      // byte offsets of this thread's operands inside a slot
      constexpr uint32_t XROW = sizeof(float2) * RB_XP * S::NX, XCOL = sizeof(float2) * RB_XP;
      constexpr uint32_t CW = sizeof(rb_coef_t), CROW = CW * RB_CP * 8, CCOMP = CW * RB_CP * 2, CCOL = CW * RB_CP;
      const uint32_t xoff = (uint32_t)(wy + 1) * XROW + (uint32_t)(lane + 2) * 8u;
      const uint32_t foff = S::OFF_F + ((uint32_t)(wy * nf) * RB_P + lane) * 8u;
      const uint32_t coff = S::OFF_C + (uint32_t)wy * CROW + (uint32_t)lane * CW;
      const unsigned char* base = rb_smem;  // + slot offset + operand offset: plain shared-memory addressing
      auto LX = [](const unsigned char* p, uint32_t off) { return *reinterpret_cast<const float2*>(p + off); };
      auto LC = [](const unsigned char* p, uint32_t off) {
        return rb_coef(*reinterpret_cast<const rb_coef_t*>(p + off));
      };
      int sft0 = (j + k0) & 1;  // (j + k) & 1, toggled per plane
      // the plane loop, compiled twice: every item of the group live (no per-item branches), or not
      auto planes = [&](auto allc) {
      constexpr bool all = decltype(allc)::value;
      for (int k = k0; k < k1; ++k) {
        mbar_wait_u32(ring0 + au + S::OFF_FULL, pu);
        if (in) {
          const unsigned char* xm = base + (am + xoff);
          const unsigned char* x0 = base + (a0 + xoff);
          const unsigned char* xu = base + (au + xoff);
          const unsigned char* f0 = base + (a0 + foff);
          const unsigned char* c0 = base + (a0 + coff);
          const unsigned char* cu = base + (au + coff);
          // colour c: the cell at (row j, position m) is i = 2m + sft; coefficients W, S, B, M of
          // its own colour, E = the other colour's W at position m + sft, N = its S of row j + 1,
          // T = its B of plane k + 1; the six neighbours are of the other colour (xh: that
          // colour's index in the slot)
          auto sweep = [&](const int c, const int xh, auto&& emit) {
            const int sft = sft0 ^ c;
            const uint32_t own = (uint32_t)c * CCOL, oth = (uint32_t)(c ^ 1) * CCOL;
            const float tw = LC(c0, own), ts = LC(c0, own + CCOMP), tb = LC(c0, own + 2 * CCOMP);
            const float mm = LC(c0, own + 3 * CCOMP);
            const float te = LC(c0, oth + (uint32_t)sft * CW), tn = LC(c0, oth + CROW + CCOMP);
            const float tt = LC(cu, oth + 2 * CCOMP);
            const float dk = tw + te + ts + tn + tb + tt;
            const uint32_t xc = (uint32_t)xh * XCOL, xs = xc + (uint32_t)sft * 8u;
#pragma unroll
            for (int t = 0; t < NI; ++t) {
              if (!all && !live[t]) continue;
              float2 os = make_float2(0.f, 0.f);
              if (MODE == 1 || !ZI) {
                const uint32_t it = (uint32_t)t * S::XBA;
                const float2 w = LX(x0, it + xs - 8u), e = LX(x0, it + xs);
                const float2 so = LX(x0, it + xc - XROW), no = LX(x0, it + xc + XROW);
                const float2 dn = LX(xm, it + xc), up = LX(xu, it + xc);
                os = make_float2(tw * w.x + te * e.x + ts * so.x + tn * no.x + tb * dn.x + tt * up.x,
                                 tw * w.y + te * e.y + ts * so.y + tn * no.y + tb * dn.y + tt * up.y);
              }
              const float dr = dk + tr[t] * mm, di = ti[t] * mm;
              emit(t, c, os, dr, di);
            }
          };
          if (MODE == 0) {
            sweep(color, 0, [&](int t, int c, float2 os, float dr, float di) {
              const float2 fcol = LX(f0, (uint32_t)t * S::FB + (fboth ? (uint32_t)c * RB_P * 8u : 0u));
              const float2 o = make_float2(fcol.x + os.x, fcol.y + os.y);
              const float inv = rcp_approx(dr * dr + di * di);
              const float2 xn = make_float2((o.x * dr + o.y * di) * inv, (o.y * dr - o.x * di) * inv);
              op[t][0] = xn;
              if (DOT) acc[t] = cfma(make_double2(fcol.x, fcol.y), make_double2(xn.x, xn.y), acc[t]);
            });
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c)
              sweep(c, c ^ 1, [&](int t, int cc, float2 os, float dr, float di) {
                const float2 xa = LX(x0, (uint32_t)t * S::XBA + (uint32_t)cc * XCOL);
                const float2 f = LX(f0, (uint32_t)t * S::FB + (uint32_t)cc * RB_P * 8u);
                op[t][cc ? nh : 0] =
                    make_float2(f.x - (dr * xa.x - di * xa.y - os.x), f.y - (dr * xa.y + di * xa.x - os.y));
              });
          }
        }
#pragma unroll
        for (int t = 0; t < NI; ++t) op[t] += plane;
        sft0 ^= 1;
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(ring0 + am + S::OFF_EMPTY);  // this warp is done with plane k - 1
        am = a0;
        a0 = au;
        au += S::SLOT;
        if (au == RING) { au = 0; pu ^= 1u; }
      }
      };
      if (nlive == NI) planes(std::true_type{});
      else planes(std::false_type{});
      // planes k1 - 1 and k1 go back to the producer as well; the next work item starts at au
      if (lane == 0) {
        mbar_arrive_u32(ring0 + am + S::OFF_EMPTY);
        mbar_arrive_u32(ring0 + a0 + S::OFF_EMPTY);
      }
      an = au;
      un = pu;
      if (MODE == 0 && DOT) {
        // this work item's partial of f^T x: the consumer warps alone reduce through shared
        // memory (named barrier 1; the producer warp never joins), in a fixed order.  The
        // scratch is double-buffered by work item, so one barrier per item is enough: a warp
        // writes buffer `par` again only after passing the barrier of the item in between,
        // which warp 0 reaches after reading it.
#pragma unroll
        for (int t = 0; t < NI; ++t) {
          const double2 v = warp_sum(acc[t]);
          if (lane == 0) dsh[par][t][wy] = v;
          acc[t] = make_double2(0.0, 0.0);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kT) : "memory");
        if (wy == 0) {
#pragma unroll
          for (int t = 0; t < NI; ++t) {
            double2 v = lane < kT / 32 ? dsh[par][t][lane] : make_double2(0.0, 0.0);
            v = warp_sum(v);
            const int b = grp * NI + t;
            if (lane == 0 && b < bt.B) dot[((int64_t)b * 2 + color) * nblk + cb] = v;
          }
        }
        par ^= 1;
      }
    }
  }
}

// ---- TMA-fed restriction from a colour-split fine level (aggregation 2 x 2 x 2) ----------
// f_c = P^T r_f.  CTA = 32 x 4 coarse columns (warp = coarse row J, lane = coarse I) x RT_ZC
// coarse planes; a producer warp streams each fine plane's tile (rows 2J0-1 .. 2J0+8, the
// positions I0-2 .. I0+33 of both colours) into a ring; the x / y reduction reads shared
// memory directly (cell 2I of a row sits at position I of colour (j + k) & 1, cell 2I + 1 at
// position I of the other colour, 2I - 1 / 2I + 2 at positions I - 1 / I + 1), and the z
// direction is the register ring of the pair restriction.  Every fine value is read from HBM
// once; the register-pipelined pair kernel was latency-bound at ~1.8 TB/s.
constexpr int RT_ZC = 16, RT_D = 6, RT_P = 36, RT_R = 10;
constexpr uint32_t RT_SLOT = sizeof(float2) * RT_P * 2 * RT_R;  // 5760
constexpr size_t RT_SMEM = (size_t)RT_SLOT * RT_D;
constexpr int kRT = 32 * 4 + 32;

__global__ void __launch_bounds__(kRT) restrict_tma_kernel(const __grid_constant__ CUtensorMap mr, TzDims L,
                                                          LevelViewT<float> Lc, Batch bt, float2* __restrict__ fc) {
  extern __shared__ __align__(128) unsigned char rt_smem[];
  __shared__ __align__(8) uint64_t full[RT_D], empty[RT_D];
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int tx = (Lc.nx + 31) / 32, ty = (Lc.ny + 3) / 4;
  const int tile = cb % (tx * ty), chunk = cb / (tx * ty);
  const int I0 = (tile % tx) * 32, J0 = (tile / tx) * 4;
  const int K0 = chunk * RT_ZC, K1 = min(Lc.nz, K0 + RT_ZC);
  const int kbeg = max(2 * K0 - 1, 0), kend = min(2 * K1, L.nz - 1);  // fine planes
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < RT_D; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 4);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  if (wy == 4) {  // producer warp
    if (lane == 0) {
      int sl = 0, use = 0;
      for (int p = kbeg; p <= kend; ++p) {
        if (use > 0) mbar_wait(&empty[sl], (uint32_t)((use - 1) & 1));
        mbar_arrive_tx(&full[sl], RT_SLOT);
        tma_load5(rt_smem + (size_t)sl * RT_SLOT, &mr, I0 - 2, 0, 2 * J0 - 1, p, b, &full[sl]);
        if (++sl == RT_D) { sl = 0; ++use; }
      }
    }
    return;
  }
  const int I = I0 + lane, J = J0 + wy;
  const bool own = I < Lc.nx && J < Lc.ny;
  const float wxm = I > 0 ? 0.25f : 0.f, wx0 = I == 0 ? 0.5f : 0.75f;
  const float wx1 = I == Lc.nx - 1 ? 0.5f : 0.75f, wxp = I < Lc.nx - 1 ? 0.25f : 0.f;
  const float wyv[4] = {J > 0 ? 0.25f : 0.f, J == 0 ? 0.5f : 0.75f, J == Lc.ny - 1 ? 0.5f : 0.75f,
                        J < Lc.ny - 1 ? 0.25f : 0.f};
  float2* fcb = fc + (int64_t)b * Lc.n;
  float2 sa = make_float2(0.f, 0.f), sb = sa, sc = sa;
  int sl = 0;
  uint32_t par = 0;
  for (int p = kbeg; p <= kend; ++p) {
    mbar_wait_u32(full0 + 8 * sl, par);
    const float2* T = reinterpret_cast<const float2*>(rt_smem + (size_t)sl * RT_SLOT);  // [row][colour][pos]
    float2 S = make_float2(0.f, 0.f);
    const int q = lane + 2;  // position I in the tile
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int rr = 2 * wy + r, jf = 2 * J - 1 + r;
      const int s = (jf + p) & 1;  // colour of the row's even cells
      const float2* E = T + (rr * 2 + s) * RT_P;
      const float2* O = T + (rr * 2 + (s ^ 1)) * RT_P;
      float2 xr = make_float2(0.f, 0.f);
      xr = f2fma(wxm, O[q - 1], xr);
      xr = f2fma(wx0, E[q], xr);
      xr = f2fma(wx1, O[q], xr);
      xr = f2fma(wxp, E[q + 1], xr);
      S = f2fma(wyv[r], xr, S);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty0 + 8 * sl);
    if (++sl == RT_D) { sl = 0; par ^= 1u; }
    if (p < 2 * K0) {
      sa = S;
    } else if (p == 2 * K0) {
      sb = S;
    } else {
      const bool odd = p & 1;
      const int K = odd ? (p - 1) >> 1 : (p >> 1) - 1;
      if (odd) sc = S;
      if (!odd || K == Lc.nz - 1) {
        const float2 sd = odd ? make_float2(0.f, 0.f) : S;
        float2 v = make_float2(0.f, 0.f);
        v = f2fma(K > 0 ? 0.25f : 0.f, sa, v);
        v = f2fma(K == 0 ? 0.5f : 0.75f, sb, v);
        v = f2fma(K == Lc.nz - 1 ? 0.5f : 0.75f, sc, v);
        v = f2fma(K < Lc.nz - 1 ? 0.25f : 0.f, sd, v);
        if (own) fcb[rb_index(Lc, I, J, K)] = v;
        sa = sc;
        sb = sd;
      }
    }
  }
}

// ---- TMA-fed prolongation onto a colour-split fine level (aggregation 2 x 2 x 2) ---------
// x_f += P e_c.  CTA = 32 fine pairs (positions I0 .. I0+31 = coarse I) x 8 fine rows x ZM_ZC
// fine planes; producer lane 0 streams the fine x tiles (both colours), lane 1 the coarse e
// tiles (coarse rows j0/2-1 .. j0/2+4, coarse x I0-2 .. I0+33: natural, or positions
// I0/2-2 .. I0/2+17 of both colours when the coarse level is colour-split too) into two
// rings; the bilinear in-plane values of each coarse plane are formed once (register ring over
// the coarse planes, as in prolong_pair_kernel) from shared memory.
constexpr int PT_D = 6, PT_CD = 5;                         // fine / coarse ring depths
constexpr int PT_CR = 6, PT_CXN = 36, PT_CXS = 20;         // coarse rows; x extent natural / split positions
constexpr uint32_t PT_FSLOT = sizeof(float2) * 32 * 2 * 8;  // 4096
template <bool CSPLIT>
struct PtGeom {
  static constexpr uint32_t CSLOT = CSPLIT ? sizeof(float2) * PT_CXS * 2 * PT_CR : sizeof(float2) * PT_CXN * PT_CR;
  static constexpr uint32_t CSLOT_A = (CSLOT + 127) / 128 * 128;
  static constexpr size_t SMEM = (size_t)PT_FSLOT * PT_D + (size_t)CSLOT_A * PT_CD;
};

template <bool CSPLIT>
__global__ void __launch_bounds__(kTP) prolong_tma_kernel(const __grid_constant__ CUtensorMap mxf,
                                                         const __grid_constant__ CUtensorMap mec, TzDims L,
                                                         LevelViewT<float> Lc, Batch bt, float2* __restrict__ xf) {
  using G = PtGeom<CSPLIT>;
  extern __shared__ __align__(128) unsigned char pt_smem[];
  __shared__ __align__(8) uint64_t ffull[PT_D], fempty[PT_D], cfull[PT_CD], cempty[PT_CD];
  LT_ITEM_BLOCK(bt.B, b, cb);
  if (bt.done[b]) return;
  const int nh = L.nx >> 1;  // fine pairs per row (= coarse nx)
  const int tx = (nh + 31) / 32, ty = (L.ny + 7) / 8;
  const int tile = cb % (tx * ty), chunk = cb / (tx * ty);
  const int I0 = (tile % tx) * 32, j0 = (tile / tx) * 8;
  const int k0 = chunk * ZM_ZC, k1 = min(L.nz, k0 + ZM_ZC);
  const int Kb = (k0 >> 1) - 1, Ke = ((k1 - 1) >> 1) + 1;  // coarse planes used (out of range: zero tiles)
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  unsigned char* fring = pt_smem;
  unsigned char* cring = pt_smem + (size_t)PT_FSLOT * PT_D;
  if (tid == 0) {
    for (int q = 0; q < PT_D; ++q) { mbar_init(&ffull[q], 1); mbar_init(&fempty[q], 8); }
    for (int q = 0; q < PT_CD; ++q) { mbar_init(&cfull[q], 1); mbar_init(&cempty[q], 8); }
    mbar_init_fence();
  }
  __syncthreads();
  if (wy == 8) {  // producer warp: lane 0 fine planes, lane 1 coarse planes
    if (lane == 0) {
      int sl = 0, use = 0;
      for (int k = k0; k < k1; ++k) {
        if (use > 0) mbar_wait(&fempty[sl], (uint32_t)((use - 1) & 1));
        mbar_arrive_tx(&ffull[sl], PT_FSLOT);
        tma_load5(fring + (size_t)sl * PT_FSLOT, &mxf, I0, 0, j0, k, b, &ffull[sl]);
        if (++sl == PT_D) { sl = 0; ++use; }
      }
    } else if (lane == 1) {
      int sl = 0, use = 0;
      for (int K = Kb; K <= Ke; ++K) {
        if (use > 0) mbar_wait(&cempty[sl], (uint32_t)((use - 1) & 1));
        mbar_arrive_tx(&cfull[sl], G::CSLOT);
        unsigned char* dst = cring + (size_t)sl * G::CSLOT_A;
        if (CSPLIT) tma_load5(dst, &mec, (I0 >> 1) - 2, 0, (j0 >> 1) - 1, K, b, &cfull[sl]);
        else tma_load4(dst, &mec, I0 - 2, (j0 >> 1) - 1, K, b, &cfull[sl]);
        if (++sl == PT_CD) { sl = 0; ++use; }
      }
    }
    return;
  }
  const int I = I0 + lane, j = j0 + wy;
  const bool in = I < nh && j < L.ny;
  const uint32_t ff0 = smem_u32(ffull), fe0 = smem_u32(fempty), cf0 = smem_u32(cfull), ce0 = smem_u32(cempty);
  // coarse rows of fine row j and their weights (Dirichlet ghost at the ends: 1/2 of J)
  const int J = j >> 1;
  int Jr[2];
  float wr[2];
  if ((j & 1) == 0) {
    Jr[0] = J; wr[0] = J == 0 ? 0.5f : 0.75f; Jr[1] = J - 1; wr[1] = J > 0 ? 0.25f : 0.f;
  } else {
    Jr[0] = J; wr[0] = J == Lc.ny - 1 ? 0.5f : 0.75f; Jr[1] = J + 1; wr[1] = J < Lc.ny - 1 ? 0.25f : 0.f;
  }
  const float wxe0 = I == 0 ? 0.5f : 0.75f, wxe1 = I > 0 ? 0.25f : 0.f;            // fine 2I: I, I - 1
  const float wxo0 = I == nh - 1 ? 0.5f : 0.75f, wxo1 = I < nh - 1 ? 0.25f : 0.f;  // fine 2I+1: I, I + 1
  // coarse ring: plane K in slot (K - Kb) % PT_CD
  int cnext = Kb;  // next coarse plane to wait for
  auto interp = [&](int K, float2& pe, float2& po) {
    pe = make_float2(0.f, 0.f);
    po = pe;
    const int q = (K - Kb) % PT_CD;
    const float2* C = reinterpret_cast<const float2*>(cring + (size_t)q * G::CSLOT_A);
    auto E = [&](int Jc, int Ic) {
      const int rr = Jc - ((j0 >> 1) - 1);
      if (CSPLIT) return C[(rr * 2 + ((Ic + Jc + K) & 1)) * PT_CXS + (Ic >> 1) - ((I0 >> 1) - 2)];
      return C[rr * PT_CXN + Ic - (I0 - 2)];
    };
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float2 c = E(Jr[r], I), m1 = E(Jr[r], I - 1), p1 = E(Jr[r], I + 1);
      pe = f2fma(wr[r] * wxe0, c, f2fma(wr[r] * wxe1, m1, pe));
      po = f2fma(wr[r] * wxo0, c, f2fma(wr[r] * wxo1, p1, po));
    }
  };
  auto wait_coarse = [&](int K) {  // planes up to K are resident
    while (cnext <= K) {
      const int u = cnext - Kb;
      mbar_wait_u32(cf0 + 8 * (u % PT_CD), (uint32_t)((u / PT_CD) & 1));
      ++cnext;
    }
  };
  auto release_coarse = [&](int K) {
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(ce0 + 8 * ((K - Kb) % PT_CD));
  };
  int K = k0 >> 1;
  float2 sme, smo, sce, sco, spe, spo;
  wait_coarse(K + 1);
  interp(K - 1, sme, smo);
  interp(K, sce, sco);
  interp(K + 1, spe, spo);
  release_coarse(K - 1);
  int fs = 0;
  uint32_t fp = 0;
  float2* xb = xf + (int64_t)b * L.n;
  for (int k = k0; k < k1; ++k) {
    if ((k >> 1) != K) {
      K = k >> 1;
      sme = sce; smo = sco;
      sce = spe; sco = spo;
      wait_coarse(K + 1);
      interp(K + 1, spe, spo);
      release_coarse(K - 1);
    }
    float2 ve = make_float2(0.f, 0.f), vo = ve;
    if ((k & 1) == 0) {
      const float w0 = K == 0 ? 0.5f : 0.75f, w1 = K > 0 ? 0.25f : 0.f;
      ve = f2fma(w1, sme, f2fma(w0, sce, ve));
      vo = f2fma(w1, smo, f2fma(w0, sco, vo));
    } else {
      const float w0 = K == Lc.nz - 1 ? 0.5f : 0.75f, w1 = K < Lc.nz - 1 ? 0.25f : 0.f;
      ve = f2fma(w1, spe, f2fma(w0, sce, ve));
      vo = f2fma(w1, spo, f2fma(w0, sco, vo));
    }
    mbar_wait_u32(ff0 + 8 * fs, fp);
    const float2* T = reinterpret_cast<const float2*>(fring + (size_t)fs * PT_FSLOT);  // [row][colour][pos]
    const int s = (j + k) & 1;  // colour of the row's even cells
    if (in) {
      const float2 e = T[(wy * 2 + s) * 32 + lane], o = T[(wy * 2 + (s ^ 1)) * 32 + lane];
      const int64_t row = ((int64_t)k * L.ny + j) * L.nx;
      xb[row + (int64_t)s * nh + I] = make_float2(e.x + ve.x, e.y + ve.y);
      xb[row + (int64_t)(s ^ 1) * nh + I] = make_float2(o.x + vo.x, o.y + vo.y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(fe0 + 8 * fs);
    if (++fs == PT_D) { fs = 0; fp ^= 1u; }
  }
  // the coarse planes still held: release so the producer is never left waiting (it is done)
}

// FP64 operator tiles: 32 x 8 cells, one per thread (warp = one row of 32 cells).  The
// coefficients come planar (Level::pack64: [k][j][W, S, B, M][i]), so every coefficient read
// of a warp is one contiguous 256-byte run, and the in-row neighbours of p come from the
// adjacent lanes: the interleaved {W, S, B, M} records made each coefficient read 8 shared
// wavefronts and bound the kernel by shared memory at ~3.4 TB/s.
constexpr int TA_W = 32, TA_H = 8;  // one consumer warp per row
constexpr int kTA = 32 * TA_H + 32;        // + the producer warp
constexpr int TA_XW = TA_W + 2, TA_XH = TA_H + 2;  // p: x0-1 .. x0+32, y0-1 .. y0+8
constexpr int TA_CW = TA_W + 2, TA_CH = TA_H + 1;  // coefficients x0 .. x0+33 (x0+32 used), y0 .. y0+8
constexpr uint32_t TA_XB = sizeof(double2) * TA_XW * TA_XH;     // 5440 (TA_H = 8)
constexpr uint32_t TA_CB = sizeof(double) * 4 * TA_CW * TA_CH;  // 9792
constexpr uint32_t TA_OFF_C = (TA_XB + 127) / 128 * 128, TA_SLOT = (TA_OFF_C + TA_CB + 127) / 128 * 128;

// The same operator on two items per CTA: the coefficient tiles (9.8 KB per plane, 64% of a
// one-item slot) are brought in once for both items and every coefficient-derived register is
// shared, as in the colour-split sweeps.  5-deep ring (2 CTAs per SM).
constexpr int TA2_D = 5;
constexpr uint32_t TA2_XBA = (TA_XB + 127) / 128 * 128;
constexpr uint32_t TA2_OFF_C = 2 * TA2_XBA, TA2_SLOT = (TA2_OFF_C + TA_CB + 127) / 128 * 128;
constexpr size_t TA2_SMEM = (size_t)TA2_SLOT * TA2_D;

__global__ void __launch_bounds__(kTA, 2) apply_tma2_kernel(const __grid_constant__ CUtensorMap mp,
                                                           const __grid_constant__ CUtensorMap mc, TzDims L, Batch bt,
                                                           const double2* __restrict__ taus, double2* __restrict__ q,
                                                           double2* __restrict__ part, int nblk) {
  extern __shared__ __align__(128) unsigned char ta_smem[];
  __shared__ __align__(8) uint64_t full[TA2_D], empty[TA2_D];
  const int Bp = (bt.B + 1) / 2;
  LT_ITEM_BLOCK(Bp, bp, cb);
  const int b0 = 2 * bp;
  const bool has1 = b0 + 1 < bt.B;
  const bool live0 = !bt.done[b0], live1 = has1 && !bt.done[b0 + 1];
  if (!live0 && !live1) return;
  const int tiles_x = (L.nx + TA_W - 1) / TA_W, tiles_y = (L.ny + TA_H - 1) / TA_H;
  const int ntile = tiles_x * tiles_y;
  const int tile = cb % ntile, chunk = cb / ntile;
  const int x0 = (tile % tiles_x) * TA_W, y0 = (tile / tiles_x) * TA_H;
  const int k0 = chunk * ZM_ZC, k1 = min(L.nz, k0 + ZM_ZC);
  const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < TA2_D; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TA_H);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
  if (wy == TA_H) {  // producer warp
    if (lane == 0) {
      int sl = 0, use = 0;
      for (int p = k0 - 1; p <= k1; ++p) {
        if (use > 0) mbar_wait(&empty[sl], (uint32_t)((use - 1) & 1));
        unsigned char* sp = ta_smem + (size_t)sl * TA2_SLOT;
        const bool lc = p >= k0;
        mbar_arrive_tx(&full[sl], TA_XB * (has1 ? 2u : 1u) + (lc ? TA_CB : 0u));
        tma_load4(sp, &mp, 2 * (x0 - 1), y0 - 1, p, b0, &full[sl]);
        if (has1) tma_load4(sp + TA2_XBA, &mp, 2 * (x0 - 1), y0 - 1, p, b0 + 1, &full[sl]);
        if (lc) tma_load4(sp + TA2_OFF_C, &mc, x0, 0, y0, p, &full[sl]);
        if (++sl == TA2_D) { sl = 0; ++use; }
      }
    }
  } else {
    const int i = x0 + lane, j = y0 + wy;
    const bool in = i < L.nx && j < L.ny;
    const double2 tau0 = taus[b0], tau1 = has1 ? taus[b0 + 1] : tau0;
    const int64_t plane = (int64_t)L.nx * L.ny;
    double2* qb0 = q + (int64_t)b0 * L.n;
    double2* qb1 = q + (int64_t)(b0 + 1) * L.n;
    // The consumers hold two slots (planes k, k + 1): the value below comes from a register (the
    // centre of the previous step), so a plane's slot goes back to the producer as soon as its
    // own step is done and D - 2 = 3 planes are in flight instead of 2.
    auto X = [](const unsigned char* sl, int it, int yy, int xx) {
      return reinterpret_cast<const double2*>(sl + it * TA2_XBA)[yy * TA_XW + xx];
    };
    int q0 = 1, qu = 2;
    uint32_t pu = 0;
    mbar_wait_u32(full0, 0);
    double2 below[2];
#pragma unroll
    for (int it = 0; it < 2; ++it)
      below[it] = (it == 0 || has1) ? X(ta_smem, it, wy + 1, lane + 1) : make_double2(0.0, 0.0);
    __syncwarp();
    if (lane == 0) mbar_arrive_u32(empty0);  // plane k0 - 1 is in registers
    mbar_wait_u32(full0 + 8 * q0, 0);
    for (int k = k0; k < k1; ++k) {
      mbar_wait_u32(full0 + 8 * qu, pu);
      const unsigned char* s0 = ta_smem + (size_t)q0 * TA2_SLOT;
      const unsigned char* sp = ta_smem + (size_t)qu * TA2_SLOT;
      auto C = [](const unsigned char* sl, int comp, int yy, int xx) {
        return reinterpret_cast<const double*>(sl + TA2_OFF_C)[(yy * 4 + comp) * TA_CW + xx];
      };
      const double tw = C(s0, 0, wy, lane), ts = C(s0, 1, wy, lane), tb = C(s0, 2, wy, lane);
      const double mm = C(s0, 3, wy, lane);
      const double te = C(s0, 0, wy, lane + 1), tn = C(s0, 1, wy + 1, lane), tt = C(sp, 2, wy, lane);
      const double dk = tw + te + ts + tn + tb + tt;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        if (it == 1 && !has1) break;  // uniform
        const double2 pc = X(s0, it, wy + 1, lane + 1);
        double2 w, e;
        w.x = __shfl_up_sync(0xffffffffu, pc.x, 1);
        w.y = __shfl_up_sync(0xffffffffu, pc.y, 1);
        e.x = __shfl_down_sync(0xffffffffu, pc.x, 1);
        e.y = __shfl_down_sync(0xffffffffu, pc.y, 1);
        if (lane == 0) w = X(s0, it, wy + 1, 0);
        if (lane == 31) e = X(s0, it, wy + 1, TA_XW - 1);
        if (in) {
          const double2 so = X(s0, it, wy, lane + 1), no = X(s0, it, wy + 2, lane + 1);
          const double2 dn = below[it], up = X(sp, it, wy + 1, lane + 1);
          const double ox = tw * w.x + te * e.x + ts * so.x + tn * no.x + tb * dn.x + tt * up.x;
          const double oy = tw * w.y + te * e.y + ts * so.y + tn * no.y + tb * dn.y + tt * up.y;
          const double2 tau = it == 0 ? tau0 : tau1;
          const double dr = dk + tau.x * mm, di = tau.y * mm;
          const double2 qa = make_double2(dr * pc.x - di * pc.y - ox, dr * pc.y + di * pc.x - oy);
          const int64_t o = k * plane + (int64_t)j * L.nx + i;
          if (it == 0) {
            if (live0) qb0[o] = qa;
            acc0 = cfma(pc, qa, acc0);
          } else {
            if (live1) qb1[o] = qa;
            acc1 = cfma(pc, qa, acc1);
          }
        }
        below[it] = pc;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(empty0 + 8 * q0);  // plane k is done: its centre stays in `below`
      q0 = qu;
      if (++qu == TA2_D) { qu = 0; pu ^= 1u; }
    }
  }
  acc0 = block_sum(acc0);
  if (threadIdx.x == 0 && live0) part[(int64_t)b0 * nblk + cb] = acc0;
  if (has1) {
    __syncthreads();
    acc1 = block_sum(acc1);
    if (threadIdx.x == 0 && live1) part[(int64_t)(b0 + 1) * nblk + cb] = acc1;
  }
}

// per-level tensor maps of one inner solve (ok = the level runs the TMA kernels)
struct TzMaps {
  bool ok = false;
  CUtensorMap x, f, c;
  bool rb = false;                // colour-split level: the mg_rb kernels and maps below
  CUtensorMap rx0, rx1, rf1, rf2, rc;  // x (one / both colours), f (one / both), coefficients
  CUtensorMap rt;                 // the residual's tiles for restrict_tma_kernel
  bool pt = false, pt_csplit = false;  // prolong_tma_kernel onto this level (coarse level split?)
  CUtensorMap ptf, ptc;           // fine x tiles, coarse e tiles
};

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

// r -= alpha q, rmg = (VM) r, partial ||r||^2.  (The solution update u += alpha p is deferred
// into the next direction update, which reads p anyway.)
__global__ void __launch_bounds__(kT) axpy_norm_kernel(int64_t n, Batch bt, const double2* __restrict__ alpha,
                                                       const double2* __restrict__ q, double2* __restrict__ r,
                                                       VM* __restrict__ rmg, double* __restrict__ part, int nblk,
                                                       int snx, int sny) {
  ITEM_GRID_PROLOGUE
  const double2 al = alpha[b];
  double s = 0.0;
  for (int64_t a = cb * (int64_t)blockDim.x + threadIdx.x; a < n; a += stride_) {
    const double2 ra = csub(r[b * n + a], cmul(al, q[b * n + a]));
    r[b * n + a] = ra;
    rmg[b * n + rb_flat(a, snx, sny)] = vfrom<VM>(ra);
    s += cabs2(ra);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

// u += alpha p (the deferred solution update of this iteration), then p = z + beta p;
// first: p = z only
__global__ void __launch_bounds__(kT) pupdate_kernel(int64_t n, Batch bt, const double2* __restrict__ alpha,
                                                     const double2* __restrict__ beta, const VM* __restrict__ z,
                                                     double2* __restrict__ p, double2* __restrict__ u, int64_t us,
                                                     int first, int snx, int sny) {
  ITEM_GRID_PROLOGUE
  const double2 al = alpha[b], be = beta[b];
  for (int64_t a = cb * (int64_t)blockDim.x + threadIdx.x; a < n; a += stride_) {
    const double2 za = vto(z[b * n + rb_flat(a, snx, sny)]);
    if (first) {
      p[b * n + a] = za;
      continue;
    }
    const double2 pa = p[b * n + a];
    double2* ua = u + b * us + a;
    *ua = cfma(al, pa, *ua);
    p[b * n + a] = cfma(be, pa, za);
  }
}

// u += alpha p for the items whose last update is still pending (mask)
__global__ void uupdate_kernel(int64_t n, const int* __restrict__ mask, const double2* __restrict__ alpha,
                               const double2* __restrict__ p, double2* __restrict__ u, int64_t us) {
  const int b = blockIdx.y;
  if (!mask[b]) return;
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    u[b * us + a] = cfma(alpha[b], p[b * n + a], u[b * us + a]);
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


// 2-D: 1 / 2 / 4 (the coarse levels are 1/4 of their parent, not 1/8, and the launches of the
// small levels are latency-bound: configs[1] / [2] at 8.3k -> 9.0k / 13.2k -> 16.4k solves/s)
// red-black sweeps per pre- / post-smoothing on the finest, the next and the coarser 3-D levels
#ifndef LT_NU3D_0
#define LT_NU3D_0 2
#endif
#ifndef LT_NU3D_1
#define LT_NU3D_1 4
#endif
#ifndef LT_NU3D_2
#define LT_NU3D_2 8
#endif
#ifndef LT_NU2D_0
#define LT_NU2D_0 1
#define LT_NU2D_1 2
#define LT_NU2D_2 4
#endif

// ---- the bottom of the V-cycle in one launch ----------------------------------------------
// The small levels (<= kBottomCells cells down to the coarsest) are latency-bound: each of
// their ~70 kernels per V-cycle moves a few hundred KB.  Here one CTA per item runs that whole
// sub-cycle -- the same red-black smoothing, residual, R = P^T, dense coarsest solve and P as
// the level-by-level kernels, on the same FP32 coefficients -- with every vector of those
// levels in shared memory and a block barrier between steps.
constexpr int kBottomCells = 4096, kBottomLevels = 8, kBT = 1024;
#ifdef LT_NO_BOTTOM
constexpr bool kBottom = false;  // A/B build: the level-by-level kernels all the way down
#else
constexpr bool kBottom = true;
#endif

struct BottomLevels {
  int L, dim;
  int nx[kBottomLevels], ny[kBottomLevels], nz[kBottomLevels], nu[kBottomLevels];
  int ax[kBottomLevels], ay[kBottomLevels], az[kBottomLevels];
  int off[kBottomLevels];  // float2 offset of the level's x (f = x + n, r = f + n)
  const float* Tx[kBottomLevels];
  const float* Ty[kBottomLevels];
  const float* Tz[kBottomLevels];
  const float* M[kBottomLevels];
};

__global__ void __launch_bounds__(kBT) bottom_vcycle_kernel(BottomLevels P, Batch bt, const double2* __restrict__ taus,
                                                         const float2* const* __restrict__ inv, int64_t inv_ld,
                                                         int64_t inv_off, const float2* __restrict__ f0,
                                                         float2* __restrict__ x0) {
  extern __shared__ __align__(16) float2 bsm[];
  const int b = blockIdx.x;
  if (bt.done[b]) return;
  const int tid = threadIdx.x;
  const float tr = (float)taus[b].x, ti = (float)taus[b].y;
  auto nof = [&](int l) { return P.nx[l] * P.ny[l] * P.nz[l]; };
  auto X = [&](int l) { return bsm + P.off[l]; };
  auto F = [&](int l) { return bsm + P.off[l] + nof(l); };
  auto R = [&](int l) { return bsm + P.off[l] + 2 * nof(l); };
  // the level's operator at cell a = (i, j, k): returns sum_nb T x_nb, with dk and m
  auto offsum = [&](int l, const float2* x, int i, int j, int k, float& dk, float& m) {
    const int nx = P.nx[l], ny = P.ny[l], nz = P.nz[l];
    const int a = (k * ny + j) * nx + i;
    const float tw = __ldg(P.Tx[l] + (k * ny + j) * (nx + 1) + i), te = __ldg(P.Tx[l] + (k * ny + j) * (nx + 1) + i + 1);
    const float ts = __ldg(P.Ty[l] + (k * (ny + 1) + j) * nx + i), tn = __ldg(P.Ty[l] + (k * (ny + 1) + j + 1) * nx + i);
    float2 o = make_float2(0.f, 0.f);
    auto add = [&](float t, float2 v) { o.x += t * v.x; o.y += t * v.y; };
    if (i > 0) add(tw, x[a - 1]);
    if (i < nx - 1) add(te, x[a + 1]);
    if (j > 0) add(ts, x[a - nx]);
    if (j < ny - 1) add(tn, x[a + nx]);
    dk = tw + te + ts + tn;
    if (P.dim == 3) {
      const int plane = nx * ny;
      const float tb = __ldg(P.Tz[l] + a), tt = __ldg(P.Tz[l] + a + plane);
      if (k > 0) add(tb, x[a - plane]);
      if (k < nz - 1) add(tt, x[a + plane]);
      dk += tb + tt;
    }
    m = __ldg(P.M[l] + a);
    return o;
  };
  auto half = [&](int l, int color) {
    const int n = nof(l), nx = P.nx[l], ny = P.ny[l];
    float2* x = X(l);
    const float2* f = F(l);
    for (int a = tid; a < n; a += kBT) {
      const int i = a % nx, j = (a / nx) % ny, k = a / (nx * ny);
      if (((i + j + k) & 1) != color) continue;
      float dk, m;
      const float2 o = offsum(l, x, i, j, k, dk, m);
      const float2 rhs = make_float2(f[a].x + o.x, f[a].y + o.y);
      const float dr = dk + tr * m, di = ti * m;
      const float inv_d = 1.0f / (dr * dr + di * di);
      x[a] = make_float2((rhs.x * dr + rhs.y * di) * inv_d, (rhs.y * dr - rhs.x * di) * inv_d);
    }
    __syncthreads();
  };
  // f of the top level from global memory, x = 0
  {
    const int n = nof(0);
    for (int a = tid; a < n; a += kBT) {
      F(0)[a] = f0[(int64_t)b * n + a];
      X(0)[a] = make_float2(0.f, 0.f);
    }
    __syncthreads();
  }
  // down: pre-smoothing, residual, restriction
  for (int l = 0; l < P.L - 1; ++l) {
    if (l > 0) {
      for (int a = tid; a < nof(l); a += kBT) X(l)[a] = make_float2(0.f, 0.f);
      __syncthreads();
    }
    for (int s = 0; s < P.nu[l]; ++s) {
      half(l, 0);
      half(l, 1);
    }
    {
      const int n = nof(l), nx = P.nx[l], ny = P.ny[l];
      for (int a = tid; a < n; a += kBT) {
        const int i = a % nx, j = (a / nx) % ny, k = a / (nx * ny);
        float dk, m;
        const float2 o = offsum(l, X(l), i, j, k, dk, m);
        const float2 xa = X(l)[a], fa = F(l)[a];
        const float dr = dk + tr * m, di = ti * m;
        R(l)[a] = make_float2(fa.x - (dr * xa.x - di * xa.y - o.x), fa.y - (dr * xa.y + di * xa.x - o.y));
      }
      __syncthreads();
    }
    {
      const int nc = nof(l + 1), cx = P.nx[l + 1], cy = P.ny[l + 1], fx = P.nx[l], fy = P.ny[l];
      for (int c = tid; c < nc; c += kBT) {
        const int I = c % cx, J = (c / cx) % cy, K = c / (cx * cy);
        int Fx[4], Fy[4], Fz[4];
        float wx[4], wy[4], wz[4];
        const int nxx = r1d_terms(I, P.ax[l], cx, Fx, wx), nyy = r1d_terms(J, P.ay[l], cy, Fy, wy);
        const int nzz = P.dim == 3 ? r1d_terms(K, P.az[l], P.nz[l + 1], Fz, wz) : 1;
        if (P.dim != 3) { Fz[0] = 0; wz[0] = 1.0f; }
        float2 s2 = make_float2(0.f, 0.f);
        for (int r = 0; r < nzz; ++r)
          for (int q = 0; q < nyy; ++q)
            for (int o = 0; o < nxx; ++o) {
              const float w = wz[r] * wy[q] * wx[o];
              const float2 v = R(l)[(Fz[r] * fy + Fy[q]) * fx + Fx[o]];
              s2.x += w * v.x;
              s2.y += w * v.y;
            }
        F(l + 1)[c] = s2;
      }
      __syncthreads();
    }
  }
  // the coarsest level: dense inverse
  {
    const int l = P.L - 1, nc = nof(l);
    const float2* A = inv[b] + inv_off;
    for (int r = tid; r < nc; r += kBT) {
      float2 s2 = make_float2(0.f, 0.f);
      for (int c = 0; c < nc; ++c) {
        const float2 m = A[(int64_t)r * inv_ld + c], v = F(l)[c];
        s2.x += m.x * v.x - m.y * v.y;
        s2.y += m.x * v.y + m.y * v.x;
      }
      X(l)[r] = s2;
    }
    __syncthreads();
  }
  // up: prolongation, post-smoothing (the pre-smoother's transpose order)
  for (int l = P.L - 2; l >= 0; --l) {
    {
      const int n = nof(l), fx = P.nx[l], fy = P.ny[l], cx = P.nx[l + 1], cy = P.ny[l + 1];
      const float2* e = X(l + 1);
      for (int a = tid; a < n; a += kBT) {
        const int i = a % fx, j = (a / fx) % fy, k = a / (fx * fy);
        int Ix[2], Iy[2], Iz[2];
        float wx[2], wy[2], wz[2];
        const int nxx = p1d_terms(i, P.ax[l], cx, Ix, wx), nyy = p1d_terms(j, P.ay[l], cy, Iy, wy);
        int nzz = 1;
        if (P.dim == 3) nzz = p1d_terms(k, P.az[l], P.nz[l + 1], Iz, wz);
        else { Iz[0] = 0; wz[0] = 1.0f; }
        float2 s2 = X(l)[a];
        for (int r = 0; r < nzz; ++r)
          for (int q = 0; q < nyy; ++q)
            for (int o = 0; o < nxx; ++o) {
              const float w = wz[r] * wy[q] * wx[o];
              const float2 v = e[(Iz[r] * cy + Iy[q]) * cx + Ix[o]];
              s2.x += w * v.x;
              s2.y += w * v.y;
            }
        X(l)[a] = s2;
      }
      __syncthreads();
    }
    for (int s = 0; s < P.nu[l]; ++s) {
      half(l, 1);
      half(l, 0);
    }
  }
  {
    const int n = nof(0);
    for (int a = tid; a < n; a += kBT) x0[(int64_t)b * n + a] = X(0)[a];
  }
}

// ---- all sweeps of a mid level in one launch: one thread-block cluster per item -----------
// The levels between the colour-split ones and the fused bottom (32^3 at configs[4], 32 x 32 x 16
// at configs[3]) are L2-resident and their half sweeps issue-bound: a 32^3 half sweep of 80 items
// took 24 us as its own launch, 8 + 8 sweeps = 32 launches per V-cycle.  Here a cluster of CL CTAs
// owns one item: CTA r keeps planes [r slab, (r + 1) slab) of x in its shared memory for the
// whole pre- or post-smoothing, reads the two planes next to its slab from its neighbours'
// shared memory (DSMEM) and separates half sweeps by a cluster barrier -- a half sweep of one
// colour reads only the other colour, which no CTA writes between two barriers, so one barrier
// per half sweep is enough and no halo copies are kept.  f and the FP32 coefficients come
// from global memory (L2) as before; x is read once (or starts at zero) and written once.
// Thread = one cell pair (2 ip, 2 ip + 1) of a row, marching the slab's planes: exactly one cell
// of the pair has the sweep's colour on every plane.  Same arithmetic as the pair kernel
// (diag_solve_r on f + sum T x_nb).
#ifndef LT_MID_CLUSTER
#define LT_MID_CLUSTER 1
#endif
constexpr bool kMidCluster = LT_MID_CLUSTER != 0;
constexpr int kMT = 256;  // three CTAs per SM (<= 85 registers): 111 four-CTA clusters resident
#ifndef LT_MID_SMEM_KB
#define LT_MID_SMEM_KB 32
#endif
constexpr size_t kMidSmem = LT_MID_SMEM_KB * 1024;  // x slab per CTA (32^3: clusters of 8; 64 KB / clusters of 4 measured 5.9 vs 5.1 ms per inner solve)
struct MidLevel {
  int nx, ny, nz, slab;
  const float* Tx;
  const float* Ty;
  const float* Tz;
  const float* M;
};

__global__ void __launch_bounds__(kMT, 3) mid_sweeps_kernel(MidLevel P, Batch bt, const double2* __restrict__ taus,
                                                        const float2* __restrict__ f, float2* __restrict__ x,
                                                        int first_color, int n_half, int zero_init) {
  extern __shared__ __align__(16) float2 msm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  const int b = (int)blockIdx.x / CL;
  if (bt.done[b]) return;  // the same for every CTA of the cluster
  const int tid = threadIdx.x;
  const int nx = P.nx, ny = P.ny, plane = nx * ny, hx = nx >> 1, pairs = hx * ny;
  const int kb = rank * P.slab, nloc = P.slab * plane;
  const int64_t n = (int64_t)plane * P.nz;
  const float2* fb = f + (int64_t)b * n + (int64_t)kb * plane;
  float2* xb = x + (int64_t)b * n + (int64_t)kb * plane;
  for (int a = tid; a < nloc; a += kMT) msm[a] = zero_init ? make_float2(0.f, 0.f) : xb[a];
  // the neighbours' slabs: the plane below is the last plane of rank - 1, the plane above the
  // first plane of rank + 1 (the domain boundary is the Dirichlet ghost: no neighbour term)
  const float2* below = rank > 0 ? cl.map_shared_rank(msm, rank - 1) + (P.slab - 1) * plane : nullptr;
  const float2* above = rank < CL - 1 ? cl.map_shared_rank(msm, rank + 1) : nullptr;
  const float tr = (float)taus[b].x, ti = (float)taus[b].y;
  cl.sync();
  for (int h = 0; h < n_half; ++h) {
    const int color = first_color ^ (h & 1);
    for (int p = tid; p < pairs; p += kMT) {
      const int j = p / hx, ip = p - j * hx;
      const float* Txr = P.Tx + ((int64_t)kb * ny + j) * (nx + 1) + 2 * ip;
      const float* Tyr = P.Ty + ((int64_t)kb * (ny + 1) + j) * nx + 2 * ip;
      const int c0 = j * nx + 2 * ip;  // the pair's first cell within a plane
      const float* Tzr = P.Tz + (int64_t)kb * plane + c0;
      const float* Mr = P.M + (int64_t)kb * plane + c0;
      const int sx = ny * (nx + 1), sy = (ny + 1) * nx;  // plane strides of Tx, Ty
#pragma unroll 8
      for (int kl = 0; kl < P.slab; ++kl) {
        const int o = (j + kb + kl + color) & 1;  // which cell of the pair has the colour
        const int i = 2 * ip + o, a = kl * plane + c0 + o;
        const float tw = __ldg(Txr + kl * sx + o), te = __ldg(Txr + kl * sx + o + 1);
        const float ts = __ldg(Tyr + kl * sy + o), tn = __ldg(Tyr + kl * sy + nx + o);
        const float tb = __ldg(Tzr + kl * plane + o), tt = __ldg(Tzr + (kl + 1) * plane + o);
        const float mm = __ldg(Mr + kl * plane + o);
        const float2 fv = fb[a];
        float2 acc = fv;
        auto add = [&](float t, float2 v) { acc.x += t * v.x; acc.y += t * v.y; };
        if (i > 0) add(tw, msm[a - 1]);
        if (i < nx - 1) add(te, msm[a + 1]);
        if (j > 0) add(ts, msm[a - nx]);
        if (j < ny - 1) add(tn, msm[a + nx]);
        if (kl > 0) add(tb, msm[a - plane]);
        else if (below) add(tb, below[c0 + o]);
        if (kl < P.slab - 1) add(tt, msm[a + plane]);
        else if (above) add(tt, above[c0 + o]);
        msm[a] = diag_solve_r<float, float2>(tw + te + ts + tn + tb + tt, mm, tr, ti, acc);
      }
    }
    cl.sync();
  }
  for (int a = tid; a < nloc; a += kMT) xb[a] = msm[a];
}

// cluster size for a level, 0 when the cluster kernel does not apply
template <class VW>
inline int mid_cluster(const VW& L) {
  if (L.dim != 3 || (L.nx & 1) || !L.Tz) return 0;
  for (int cl = 1; cl <= 8; cl *= 2)
    if (L.nz % cl == 0 && (size_t)(L.n / cl) * sizeof(float2) <= kMidSmem) return cl;
  return 0;
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
// dot_part != null (finest level only): the last sweep also writes per-block partials of
// f^T x, and *dot_nblk their count per item (0 when this level could not fuse them).
const typename CT<R>::V* vcycle(lt_pencil p, int l, int Bc, const Batch& bt, const double2* taus,
                                const typename CT<R>::V* const* inv, int64_t inv_ld, int64_t inv_off,
                                std::vector<typename CT<R>::V*>& X, std::vector<typename CT<R>::V*>& F,
                                std::vector<typename CT<R>::V*>& Rr, double2* dot_part, int* dot_nblk,
                                const TzMaps* tz) {
  if (dot_nblk) *dot_nblk = 0;
  using V = typename CT<R>::V;
  // per-level kernel names (class:level) for the profile
  static const char* const kSmooth[] = {"mg_smooth:l0", "mg_smooth_coarse:l1", "mg_smooth_coarse:l2",
                                        "mg_smooth_coarse:l3", "mg_smooth_coarse:l4", "mg_smooth_coarse:l5",
                                        "mg_smooth_coarse:l6", "mg_smooth_coarse:l7", "mg_smooth_coarse:l8"};
  static const char* const kResid[] = {"mg_residual:l0", "mg_residual:l1", "mg_residual:l2", "mg_residual:l3",
                                       "mg_residual:l4", "mg_residual:l5", "mg_residual:l6", "mg_residual:l7",
                                       "mg_residual:l8"};
  static const char* const kRestr[] = {"mg_restrict:l0", "mg_restrict:l1", "mg_restrict:l2", "mg_restrict:l3",
                                       "mg_restrict:l4", "mg_restrict:l5", "mg_restrict:l6", "mg_restrict:l7",
                                       "mg_restrict:l8"};
  static const char* const kProl[] = {"mg_prolong:l0", "mg_prolong:l1", "mg_prolong:l2", "mg_prolong:l3",
                                      "mg_prolong:l4", "mg_prolong:l5", "mg_prolong:l6", "mg_prolong:l7",
                                      "mg_prolong:l8"};
  const int ln = l < 8 ? l : 8;
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int last = (int)p->levels.size() - 1;
  LevelViewT<R> L = mg_view<R>(p, l);
  L.split = tz && tz[l].rb;
  const double vb = sizeof(V), rb = sizeof(R);
  const double cell_bytes = (double)L.n * Bc;
  const double coef = (double)L.n * rb * (DIM + 1);
  if (p->kind == LT_GRID_P1_TRI && l < last) {
    // P1: symmetric 3-colour Gauss-Seidel V-cycle on the node grid
    LevelViewT<R> Lc = mg_view<R>(p, l + 1);
    const unsigned grid = (unsigned)L.ntiles * (unsigned)Bc;
    const double cb6 = coef + (double)L.n * rb * 3;  // + the three mass-coupling arrays
    for (int c = 0; c < 3; ++c)
      launch(ctx, kSmooth[ln], cell_bytes * 3 * vb + cb6, [&] {
        p1_gs_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], c, c == 0);
      });
    launch(ctx, kResid[ln], cell_bytes * 3 * vb + cb6, [&] {
      p1_residual_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
    });
    launch(ctx, kRestr[ln], cell_bytes * vb + (double)Lc.n * Bc * vb, [&] {
      p1_restrict_kernel<R><<<(unsigned)Lc.ntiles * Bc, kT, 0, st>>>(L, Lc, bt, Rr[l], F[l + 1]);
    });
    const V* ec = vcycle<R, DIM>(p, l + 1, Bc, bt, taus, inv, inv_ld, inv_off, X, F, Rr, nullptr, nullptr, tz);
    launch(ctx, kProl[ln], cell_bytes * 2 * vb + (double)Lc.n * Bc * vb, [&] {
      p1_prolong_kernel<R><<<grid, kT, 0, st>>>(L, Lc, bt, ec, X[l]);
    });
    for (int c = 2; c >= 0; --c)
      launch(ctx, kSmooth[ln], cell_bytes * 3 * vb + cb6, [&] {
        p1_gs_kernel<R><<<grid, kT, 0, st>>>(L, bt, taus, F[l], X[l], c, 0);
      });
    return X[l];
  }
  if constexpr (std::is_same<R, float>::value) {
    if (kBottom && p->kind != LT_GRID_P1_TRI && l < last && L.n <= kBottomCells && !(tz && tz[l].rb)) {
      BottomLevels P{};
      P.L = last - l + 1;
      P.dim = DIM;
      int off = 0;
      bool fits = P.L <= kBottomLevels;
      for (int q = 0; fits && q < P.L; ++q) {
        const Level& Lq = *p->levels[l + q];
        P.nx[q] = Lq.nx;
        P.ny[q] = Lq.ny;
        P.nz[q] = Lq.nz;
        P.ax[q] = Lq.agg[0];
        P.ay[q] = Lq.agg[1];
        P.az[q] = Lq.agg[2];
        const int lv = l + q;
        P.nu[q] = lv == 0 ? (DIM == 3 ? LT_NU3D_0 : LT_NU2D_0) : lv == 1 ? (DIM == 3 ? LT_NU3D_1 : LT_NU2D_1) : (DIM == 3 ? LT_NU3D_2 : LT_NU2D_2);
        P.Tx[q] = Lq.Tx32;
        P.Ty[q] = Lq.Ty32;
        P.Tz[q] = Lq.Tz32;
        P.M[q] = Lq.M32;
        P.off[q] = off;
        off += (int)Lq.n * (q == P.L - 1 ? 2 : 3);
      }
      const size_t smem = sizeof(float2) * (size_t)off;
      if (fits && smem <= 200 * 1024) {
        static bool attr = false;
        if (!attr) {
          LT_CUDA(cudaFuncSetAttribute(bottom_vcycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
          attr = true;
        }
        double bytes = 0.0;
        for (int q = 0; q < P.L; ++q) bytes += (double)p->levels[l + q]->n * (double)Bc * 16.0;
        launch(ctx, "mg_bottom:fused", bytes, [&] {
          bottom_vcycle_kernel<<<Bc, kBT, smem, st>>>(P, bt, taus, reinterpret_cast<const float2* const*>(inv), inv_ld,
                                                      inv_off, reinterpret_cast<const float2*>(F[l]),
                                                      reinterpret_cast<float2*>(X[l]));
        });
        return X[l];
      }
    }
  }
  if (l == last) {
    dim3 g(blocks_for(L.n, kT / 32), Bc);
    launch(ctx, "mg_coarse_solve:dense", cell_bytes * 2 * vb, [&] {
      coarse_solve_kernel<V><<<g, kT, 0, st>>>((int)L.n, bt, inv, inv_ld, inv_off, F[l], X[l]);
    });
    return X[l];
  }
  LevelViewT<R> Lc = mg_view<R>(p, l + 1);
  Lc.split = tz && tz[l + 1].rb;
  const Level& lev = *p->levels[l];
  // red-black sweeps per pre/post smoothing, by level: 2 on the finest, 4 on the next, 8 on
  // the coarser ones.  Convergence is set by the coarse levels' smoothing, while their sweeps
  // are cheap: at configs[4] (80 items) this takes the inner solve from 17 to 12 COCG
  // iterations, 194 -> 163 ms; more finest-level sweeps do not reduce the count, fewer raise it
  const int nu0 = DIM == 3 ? LT_NU3D_0 : LT_NU2D_0, nu1 = DIM == 3 ? LT_NU3D_1 : LT_NU2D_1, nu_c = DIM == 3 ? LT_NU3D_2 : LT_NU2D_2;
  const int nu = l == 0 ? nu0 : l == 1 ? nu1 : nu_c;
  // half sweeps on cell pairs when the rows have even length, else one cell per thread
  const bool pairs = (L.nx & 1) == 0;
  const unsigned zgrid = (unsigned)zm_blocks(L) * (unsigned)Bc;
  const unsigned pgrid = (unsigned)zp_blocks(L) * (unsigned)Bc;
  const bool tma = tz && tz[l].ok;
  const unsigned tgrid = (unsigned)tz_blocks(L) * (unsigned)Bc;
  const TzDims tdims{L.nx, L.ny, L.nz, L.n};
  const bool rbk = tz && tz[l].rb;
  const unsigned rgrid = (unsigned)rb_blocks(L) * (unsigned)Bc;
  const unsigned rgrid2 = (unsigned)rb_blocks(L) * (unsigned)((Bc + RB_NI - 1) / RB_NI);
  auto half = [&](int color, int zero_init, double2* dot) {
    // finest-level sweeps are their own class (the roofline kernel); coarser levels pooled.
    // Colour-split: a half sweep moves half of f and of x twice (1.5 c per cell, 1 from zero)
    const double hb = rbk ? cell_bytes * (zero_init ? 1.0 : 1.5) * vb : cell_bytes * (zero_init ? 2 : 3) * vb;
    launch(ctx, kSmooth[ln], hb + coef, [&] {
      if (rbk) {
        const unsigned pg = std::min(rgrid2, rb_persist_grid(ctx));
        const int nb = rb_blocks(L), zc = rb_zc(L.nz);
        float2* xo = (float2*)X[l];
        if (dot)
          mg_rb_kernel<0, RB_NI, false, true><<<pg, kTP, RbSlot<0, RB_NI>::SMEM, st>>>(
              tz[l].rx0, tz[l].rf1, tz[l].rc, tdims, bt, taus, xo, color, dot, nb, zc);
        else if (zero_init)
          mg_rb_kernel<0, RB_NI, true, false><<<pg, kTP, RbSlot<0, RB_NI>::SMEM, st>>>(
              tz[l].rx0, tz[l].rf1, tz[l].rc, tdims, bt, taus, xo, color, nullptr, nb, zc);
        else
          mg_rb_kernel<0, RB_NI, false, false><<<pg, kTP, RbSlot<0, RB_NI>::SMEM, st>>>(
              tz[l].rx0, tz[l].rf1, tz[l].rc, tdims, bt, taus, xo, color, nullptr, nb, zc);
      }
      else if (tma)
        mg_tma_kernel<0><<<tgrid, kTP, TZ_SMEM, st>>>(tz[l].x, tz[l].f, tz[l].c, tdims, bt, taus, (float2*)X[l], color,
                                                   zero_init, dot, tz_blocks(L));
      else if (pairs)
        rbpair_zm_kernel<R><<<pgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], color, zero_init, dot, zp_blocks(L));
      else
        rbhalf_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], color, zero_init);
    });
  };
  // mid levels (not colour-split, small enough for a cluster's shared memory): all half sweeps
  // of the pre- / post-smoothing in one cluster launch
  int mid_cl = 0;
  if constexpr (std::is_same<R, float>::value && DIM == 3) {
    if (kMidCluster && l > 0 && !rbk && !tma && pairs && p->kind != LT_GRID_P1_TRI) mid_cl = mid_cluster(L);
  }
  auto mid = [&](int first_color, int zero_init) {
    if constexpr (std::is_same<R, float>::value) {
      // x read (unless from zero) and written once, f once per sweep of its colour
      const double mb = cell_bytes * vb * ((zero_init ? 1.0 : 2.0) + nu) + coef;
      launch(ctx, kSmooth[ln], mb, [&] {
        const MidLevel M{L.nx, L.ny, L.nz, L.nz / mid_cl, L.Tx, L.Ty, L.Tz, L.M};
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(Bc * mid_cl));
        cfg.blockDim = dim3(kMT);
        cfg.dynamicSmemBytes = sizeof(float2) * (size_t)(L.n / mid_cl);
        cfg.stream = st;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = (unsigned)mid_cl;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        LT_CUDA(cudaLaunchKernelEx(&cfg, mid_sweeps_kernel, M, bt, taus, (const float2*)F[l], (float2*)X[l],
                                   first_color, 2 * nu, zero_init));
      });
    }
  };
  // pre-smoothing: red half sweep from zero (f read, x written), then black, red, ...
  if (mid_cl) {
    mid(0, 1);
  } else {
    half(0, 1, nullptr);
    half(1, 0, nullptr);
    for (int s = 1; s < nu; ++s) {
      half(0, 0, nullptr);
      half(1, 0, nullptr);
    }
  }
  launch(ctx, kResid[ln], cell_bytes * 3 * vb + coef, [&] {
    if (rbk)
      mg_rb_kernel<1, 1, false, false><<<rgrid, kTP, RbSlot<1, 1>::SMEM, st>>>(
          tz[l].rx1, tz[l].rf2, tz[l].rc, tdims, bt, taus, (float2*)Rr[l], 0, nullptr, rb_blocks(L), rb_zc(L.nz));
    else if (tma)
      mg_tma_kernel<1><<<tgrid, kTP, TZ_SMEM, st>>>(tz[l].x, tz[l].f, tz[l].c, tdims, bt, taus, (float2*)Rr[l], 0, 0,
                                                 nullptr, 0);
    else if (pairs)
      residual_pair_zm_kernel<R><<<pgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
    else if (DIM == 3)
      residual_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
    else
      residual_kernel<R, DIM><<<(unsigned)L.ntiles * (unsigned)Bc, kT, 0, st>>>(L, bt, taus, F[l], X[l], Rr[l]);
  });
  // pair transfers for aggregation 2 in every direction (3-D, FP32 V-cycle)
  const bool ptr = std::is_same<R, float>::value && DIM == 3 && lev.agg[0] == 2 && lev.agg[1] == 2 &&
                   lev.agg[2] == 2 && (L.nx & 1) == 0;
  launch(ctx, kRestr[ln], cell_bytes * vb + (double)Lc.n * Bc * vb, [&] {
    if constexpr (std::is_same<R, float>::value) {
      if (ptr && rbk) {
        const unsigned g = (unsigned)(((Lc.nx + 31) / 32) * ((Lc.ny + 3) / 4) * ((Lc.nz + RT_ZC - 1) / RT_ZC));
        restrict_tma_kernel<<<g * Bc, kRT, RT_SMEM, st>>>(tz[l].rt, tdims, Lc, bt, (float2*)F[l + 1]);
        return;
      }
      if (ptr) {
        const unsigned g = (unsigned)(((Lc.nx + 31) / 32) * ((Lc.ny + TP_TY - 1) / TP_TY) * ((Lc.nz + TP_ZC - 1) / TP_ZC));
        restrict_pair_kernel<<<g * Bc, 32 * TP_TY, 0, st>>>(L, Lc, bt, Rr[l], F[l + 1]);
        return;
      }
    }
    restrict_zm_kernel<R><<<(unsigned)zm_blocks(Lc) * Bc, kT, 0, st>>>(L, Lc, lev.agg[0], lev.agg[1], lev.agg[2], bt,
                                                                      Rr[l], F[l + 1]);
  });
  const V* ec = vcycle<R, DIM>(p, l + 1, Bc, bt, taus, inv, inv_ld, inv_off, X, F, Rr, nullptr, nullptr, tz);
  // coarse correction, then the transpose of the pre-smoother (black, red, ...), in place
  launch(ctx, kProl[ln], cell_bytes * 2 * vb + (double)Lc.n * Bc * vb, [&] {
    if constexpr (std::is_same<R, float>::value) {
      if (ptr && rbk && tz[l].pt) {
        const unsigned g = (unsigned)(((L.nx / 2 + 31) / 32) * ((L.ny + 7) / 8) * ((L.nz + ZM_ZC - 1) / ZM_ZC));
        if (tz[l].pt_csplit)
          prolong_tma_kernel<true><<<g * Bc, kTP, PtGeom<true>::SMEM, st>>>(tz[l].ptf, tz[l].ptc, tdims, Lc, bt,
                                                                           (float2*)X[l]);
        else
          prolong_tma_kernel<false><<<g * Bc, kTP, PtGeom<false>::SMEM, st>>>(tz[l].ptf, tz[l].ptc, tdims, Lc, bt,
                                                                             (float2*)X[l]);
        return;
      }
      if (ptr) {
        const unsigned g = (unsigned)(((L.nx / 2 + 31) / 32) * ((L.ny + 7) / 8) * ((L.nz + ZM_ZC - 1) / ZM_ZC));
        prolong_pair_kernel<<<g * Bc, kT, 0, st>>>(L, Lc, bt, ec, X[l]);
        return;
      }
    }
    prolong_zm_kernel<R><<<zgrid, kT, 0, st>>>(L, Lc, lev.agg[0], lev.agg[1], lev.agg[2], bt, ec, X[l]);
  });
  if (mid_cl) mid(1, 0);
  for (int s = 0; s < (mid_cl ? 0 : nu); ++s) {
    // the last half sweeps also form the partial sums of f^T x when asked (and possible):
    // colour-split, each of the last black and red sweeps over its own colour; else the last
    // (red) sweep over both
    const bool last_sweep = s == nu - 1;
    half(1, 0, last_sweep && rbk ? dot_part : nullptr);
    half(0, 0, last_sweep && pairs ? dot_part : nullptr);
  }
  if (dot_nblk) *dot_nblk = !dot_part ? 0 : rbk ? 2 * rb_blocks(L) : (tma || pairs) ? zp_blocks(L) : 0;
  return X[l];
}

// Device-resident COCG control (one block): items masked out by the caller start done.
__global__ void cocg_mask_kernel(int B, const int* __restrict__ active, int* __restrict__ done) {
  for (int b = threadIdx.x; b < B; b += blockDim.x) done[b] = active ? !active[b] : 0;
}

// After ||v||^2: items with a zero right-hand side are done with u = 0; stagnation state.
__global__ void cocg_init_kernel(int B, int* __restrict__ done, int* __restrict__ zero, const double* __restrict__ bb,
                                 double* __restrict__ rr, double* __restrict__ best, int* __restrict__ stall,
                                 int* __restrict__ pending, int* __restrict__ counts) {
  int cnt = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int z = !done[b] && !(bb[b] > 0.0);
    zero[b] = z;
    if (z) { done[b] = 1; rr[b] = 0.0; }
    best[b] = bb[b];
    stall[b] = 0;
    pending[b] = 0;
    cnt += !done[b];
  }
  cnt = block_sum(cnt);
  if (counts && threadIdx.x == 0) counts[0] = cnt;
}

// block-wide max, valid in thread 0
__device__ __forceinline__ double block_max(double v) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffff, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)((blockDim.x + 31) >> 5) ? sh[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffff, v, o));
  }
  return v;
}

// Per iteration, after ||r||^2: converged at ||r|| <= tol ||v||; stagnated at the rounding
// floor (within kInnerFloor of the tolerance and no halving of the residual in 6 iterations; far from
// the floor COCG's residual is non-monotone on the indefinite pencils Re tau < 0 gives, so
// plateaus there are not stagnation).  An item stopping here still owes its deferred u += alpha p
// (pending).  The count of items still iterating and the worst remaining ratio to the tolerance
// go to the host through mapped pinned memory, slot (*counter)++ % ring, which the host reads an
// iteration later (no pipeline drain); counts (profiling only) keeps the whole count sequence
// for the byte accounting.
__global__ void cocg_control_kernel(int B, int* __restrict__ done, const double* __restrict__ rr,
                                    const double* __restrict__ bb, double* __restrict__ best, int* __restrict__ stall,
                                    int* __restrict__ pending, double tol2, int* __restrict__ counter,
                                    volatile FlagSlot* __restrict__ host_ring, int ring, int* __restrict__ counts) {
  int cnt = 0;
  double worst = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    if (done[b]) continue;
    const double r = rr[b], lim = tol2 * bb[b];
    bool stop = r <= lim;
    if (!stop) {
      if (r < 0.25 * best[b]) { best[b] = r; stall[b] = 0; }
      else if (r <= kInnerFloor * kInnerFloor * lim && ++stall[b] >= 6) stop = true;
    }
    if (stop) { done[b] = 1; pending[b] = 1; }
    else { ++cnt; worst = fmax(worst, r / lim); }
  }
  cnt = block_sum(cnt);
  worst = block_max(worst);
  if (threadIdx.x == 0) {
    const int s = *counter;
    *counter = s + 1;
    host_ring[s % ring].worst = worst;
    host_ring[s % ring].active = cnt;
    if (counts) counts[s + 1] = cnt;
  }
}

#ifdef LT_TMA_2D
constexpr bool kTma2d = true;  // A/B build: the TMA z-march kernels on 2-D levels too
#else
constexpr bool kTma2d = false;
#endif

template <int DIM>
void inner_chunk(lt_pencil p, int Bc, const double2* taus_host, const double2* v, int64_t vs, double2* u,
                 int64_t us, const int* active, double* rel_out) {
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

  // small per-item state: taus, scalars, inverse pointers, control flags
  const size_t small_bytes = sizeof(double2) * Bc * 4 + sizeof(double) * Bc * 3 + sizeof(void*) * Bc +
                             sizeof(int) * (Bc * 5 + 1) + 64;
  DeviceBuffer small(small_bytes, st);
  char* sp = small.as<char>();
  double2* d_taus = reinterpret_cast<double2*>(sp);
  double2* d_rho = d_taus + Bc;
  double2* d_alpha = d_rho + Bc;
  double2* d_beta = d_alpha + Bc;
  double* d_bb = reinterpret_cast<double*>(d_beta + Bc);
  double* d_rr = d_bb + Bc;
  double* d_best = d_rr + Bc;
  const V** d_inv = reinterpret_cast<const V**>(d_best + Bc);
  int* d_done = reinterpret_cast<int*>(d_inv + Bc);
  int* d_zero = d_done + Bc;
  int* d_stall = d_zero + Bc;
  int* d_pending = d_stall + Bc;
  int* d_counter = d_pending + Bc;
  LT_CUDA(cudaMemcpyAsync(d_taus, taus_host, sizeof(double2) * Bc, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(d_inv, inv_host.data(), sizeof(void*) * Bc, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemsetAsync(d_counter, 0, sizeof(int), st));
  Scalars sc{d_bb, d_rr, d_rho, d_alpha, d_beta};
  Batch bt{Bc, d_done};

  // workspace: FP64 Krylov vectors r, p, q; multigrid vectors (precision R) per level
  DeviceBuffer partials(sizeof(double2) * (size_t)Bc *
                            std::max<int64_t>(std::max<int64_t>(nblk, L0.ntiles),
                                              std::max(zm_blocks(L0), zp_blocks(L0))),
                        st);
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

  // TMA tensor maps (FD levels with even rows of >= 64 cells; FP32 V-cycle only) and the
  // FP64 operator's maps on the finest level; the other levels run the register-pipelined
  // z-march kernels
  std::vector<TzMaps> tzm(nl);
  {
    static bool attr = false;
    if (!attr) {
      LT_CUDA(cudaFuncSetAttribute(mg_tma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TZ_SMEM));
      LT_CUDA(cudaFuncSetAttribute(mg_tma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TZ_SMEM));
      LT_CUDA(cudaFuncSetAttribute(apply_tma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TA2_SMEM));
      LT_CUDA(cudaFuncSetAttribute(mg_rb_kernel<0, RB_NI, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)RbSlot<0, RB_NI>::SMEM));
      LT_CUDA(cudaFuncSetAttribute(mg_rb_kernel<0, RB_NI, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)RbSlot<0, RB_NI>::SMEM));
      LT_CUDA(cudaFuncSetAttribute(mg_rb_kernel<0, RB_NI, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)RbSlot<0, RB_NI>::SMEM));
      LT_CUDA(cudaFuncSetAttribute(mg_rb_kernel<1, 1, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)RbSlot<1, 1>::SMEM));
      LT_CUDA(cudaFuncSetAttribute(restrict_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RT_SMEM));
      LT_CUDA(cudaFuncSetAttribute(mid_sweeps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMidSmem));
      LT_CUDA(cudaFuncSetAttribute(prolong_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)PtGeom<true>::SMEM));
      LT_CUDA(cudaFuncSetAttribute(prolong_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)PtGeom<false>::SMEM));
      attr = true;
    }
  }
  if (p->kind != LT_GRID_P1_TRI && sizeof(R) == 4) {
    for (int l = 0; l < nl - 1; ++l) {
      const Level& Lv = *p->levels[l];
      // the TMA z-march kernels pay on 3-D levels; a 2-D level is one plane, where the ring set-up
      // and the producer warp are pure overhead (the register kernels run it)
      if (Lv.nx % 2 != 0 || Lv.nx < 64 || (DIM != 3 && !kTma2d)) continue;
      const uint64_t nx = Lv.nx, ny = Lv.ny, nz = Lv.nz;
      const uint64_t dims[4] = {nx, ny, nz, (uint64_t)Bc};
      const uint64_t str[3] = {nx * 8, nx * ny * 8, nx * ny * nz * 8};
      const uint32_t bx[4] = {TZ_XW, TZ_XH, 1, 1}, bf[4] = {TZ_W, TZ_H, 1, 1};
      const uint64_t cd[3] = {2 * (nx + 1), ny + 1, nz + 1};
      const uint64_t cs[2] = {(nx + 1) * 16, (nx + 1) * (ny + 1) * 16};
      const uint32_t bc[3] = {2 * TZ_CW, TZ_CH, 1};
      tzm[l].x = tma_map_8b(X[l], 4, dims, str, bx);
      tzm[l].f = tma_map_8b(F[l], 4, dims, str, bf);
      tzm[l].c = tma_map_8b(Lv.pack32.get(), 3, cd, cs, bc);
      tzm[l].ok = true;
      if (Lv.packrb.get() && nx % 4 == 0) {
        // colour-split maps: vectors {pos, colour, y, z, item}, coefficients {pos, colour,
        // comp, y, z} (Level::packrb)
        const uint64_t vd[5] = {nx / 2, 2, ny, nz, (uint64_t)Bc};
        const uint64_t vs[4] = {nx / 2 * 8, nx * 8, nx * ny * 8, nx * ny * nz * 8};
        const uint32_t bx0[5] = {RB_XP, 1, RB_H + 2, 1, 1}, bx1[5] = {RB_XP, 2, RB_H + 2, 1, 1};
        const uint32_t bf1[5] = {RB_P, 1, RB_H, 1, 1}, bf2[5] = {RB_P, 2, RB_H, 1, 1};
        const uint64_t P = (uint64_t)Lv.rb_P;
        const uint64_t kd[5] = {P, 2, 4, ny + 1, nz + 1};
        const uint64_t cw = sizeof(rb_coef_t);
        const uint64_t ks[4] = {P * cw, 2 * P * cw, 8 * P * cw, 8 * P * cw * (ny + 1)};
        const uint32_t kb[5] = {RB_CP, 2, 4, RB_H + 1, 1};
        tzm[l].rx0 = tma_map_8b(X[l], 5, vd, vs, bx0);
        tzm[l].rx1 = tma_map_8b(X[l], 5, vd, vs, bx1);
        tzm[l].rf1 = tma_map_8b(F[l], 5, vd, vs, bf1);
        tzm[l].rf2 = tma_map_8b(F[l], 5, vd, vs, bf2);
        tzm[l].rc = RB_BF16 ? tma_map_2b(Lv.packrb.get(), 5, kd, ks, kb) : tma_map_4b(Lv.packrb.get(), 5, kd, ks, kb);
        tzm[l].rb = true;
        const uint32_t brt[5] = {RT_P, 2, RT_R, 1, 1};
        tzm[l].rt = tma_map_8b(Rr[l], 5, vd, vs, brt);
      }
    }
  }
  // prolongation onto colour-split levels with aggregation 2 x 2 x 2: fine x and coarse e maps
  for (int l = 0; l + 1 < nl; ++l) {
    const Level& Lv = *p->levels[l];
    if (!tzm[l].rb || !(Lv.agg[0] == 2 && Lv.agg[1] == 2 && Lv.agg[2] == 2))
      continue;
    const Level& Lc = *p->levels[l + 1];
    const uint64_t nx = Lv.nx, ny = Lv.ny, nz = Lv.nz;
    const uint64_t vd[5] = {nx / 2, 2, ny, nz, (uint64_t)Bc};
    const uint64_t vs[4] = {nx / 2 * 8, nx * 8, nx * ny * 8, nx * ny * nz * 8};
    const uint32_t bf[5] = {32, 2, 8, 1, 1};
    tzm[l].ptf = tma_map_8b(X[l], 5, vd, vs, bf);
    const uint64_t cx = Lc.nx, cy = Lc.ny, cz = Lc.nz;
    tzm[l].pt_csplit = tzm[l + 1].rb;
    if (tzm[l + 1].rb) {
      const uint64_t cd[5] = {cx / 2, 2, cy, cz, (uint64_t)Bc};
      const uint64_t cs[4] = {cx / 2 * 8, cx * 8, cx * cy * 8, cx * cy * cz * 8};
      const uint32_t bc[5] = {PT_CXS, 2, PT_CR, 1, 1};
      tzm[l].ptc = tma_map_8b(X[l + 1], 5, cd, cs, bc);
    } else {
      const uint64_t cd[4] = {cx, cy, cz, (uint64_t)Bc};
      const uint64_t cs[3] = {cx * 8, cx * cy * 8, cx * cy * cz * 8};
      const uint32_t bc[4] = {PT_CXN, PT_CR, 1, 1};
      tzm[l].ptc = tma_map_8b(X[l + 1], 4, cd, cs, bc);
    }
    tzm[l].pt = true;
  }
  // the residual kernel reads x through the level's x map and writes Rr[l]; the smoother
  // reads and writes X[l]
  const bool ta_ok = (DIM == 3 || kTma2d) && p->kind != LT_GRID_P1_TRI && p->levels[0]->pack64.get() != nullptr && L0.nx >= 32 &&
                     L0.nx % 2 == 0;
  CUtensorMap map_p{}, map_c64{};
  if (ta_ok) {
    const uint64_t nx = L0.nx, ny = L0.ny, nz = L0.nz;
    const uint64_t dims[4] = {2 * nx, ny, nz, (uint64_t)Bc};
    const uint64_t str[3] = {nx * 16, nx * ny * 16, nx * ny * nz * 16};
    const uint32_t bx[4] = {2 * TA_XW, TA_XH, 1, 1};
    // planar coefficients [k][j][comp][i], rows of nx + 2 (Level::pack64)
    const uint64_t P = nx + 2;
    const uint64_t cd[4] = {P, 4, ny + 1, nz + 1};
    const uint64_t cs[3] = {P * 8, 4 * P * 8, 4 * P * 8 * (ny + 1)};
    const uint32_t bc[4] = {TA_CW, 4, TA_CH, 1};
    map_p = tma_map_8b(pp, 4, dims, str, bx);
    map_c64 = tma_map_8b(p->levels[0]->pack64.get(), 4, cd, cs, bc);
  }
  // COCG vector kernels: vblk grid-stride blocks per item (about LT_VBLK_SM per SM over the batch)
#ifndef LT_VBLK_SM
#define LT_VBLK_SM 64
#endif
  const int vblk = (int)std::min<int64_t>(nblk, std::max<int64_t>(4, ((int64_t)LT_VBLK_SM * ctx->num_sms + Bc - 1) / Bc));
  const unsigned grid = (unsigned)vblk * (unsigned)Bc;
  // the finest level's multigrid vectors (rmg, z) are colour-split when its kernels are
  const int snx = tzm[0].rb ? L0.nx : 0, sny = tzm[0].rb ? L0.ny : 0;
  const double nb = (double)n * Bc;
  const double coef = (double)n * 8.0 * (DIM + 1);
  const double vb = sizeof(V);
  const unsigned cblk = (unsigned)std::min(1024, (Bc + 31) / 32 * 32);

  // r = v, u = 0, ||v||^2; items masked out by the caller and zero right-hand sides are done
  launch(ctx, "cocg_scalar", 0.0, [&] { cocg_mask_kernel<<<1, cblk, 0, st>>>(Bc, active, d_done); });
  launch(ctx, "cocg_vec:copy_norm", nb * (48.0 + vb), [&] {
    copy_norm_kernel<<<grid, kT, 0, st>>>(n, bt, v, vs, r, rmg, u, us, (double*)partials.get(), vblk, snx, sny);
  });
  launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_BB, bt, partials.get(), vblk, sc); });
  // profiling: the number of items still active at every step (bytes of the launches of a
  // step are charged for those items only)
  DeviceBuffer counts;
  const bool prof = ctx->profiling;
  if (prof) counts.allocate(sizeof(int) * (size_t)(p->inner_maxit + 2), st);
  int* d_counts = prof ? counts.as<int>() : nullptr;
  launch(ctx, "cocg_scalar", 0.0, [&] {
    cocg_init_kernel<<<1, cblk, 0, st>>>(Bc, d_done, d_zero, d_bb, d_rr, d_best, d_stall, d_pending, d_counts);
  });
  const size_t pend0 = ctx->pending.size();
  if (prof) ctx->profile_tag = 0;
  launch(ctx, "cocg_vec:zero", nb * 16.0, [&] {
    zero_kernel<<<dim3(std::min<unsigned>(blocks_for(n, kT), 2 * ctx->num_sms), Bc), kT, 0, st>>>(n, d_zero, u, us, Bc);
  });

  // FD: rho = r^T z is fused into the V-cycle's last sweep (partials of f^T x on the finest
  // level, f the multigrid copy of r); P1 keeps the separate dot kernel
  const bool fused = p->kind != LT_GRID_P1_TRI;
  const V* z = nullptr;
  auto precondition = [&](int op) {
    int dnb = 0;
    z = vcycle<R, DIM>(p, 0, Bc, bt, d_taus, d_inv, inv_ld, inv_off, X, F, Rr, fused ? partials.as<double2>() : nullptr,
                       &dnb, tzm.data());
    if (dnb == 0) {
      dnb = vblk;
      launch(ctx, "cocg_vec:bdot", nb * (16.0 + vb), [&] {
        bdot_kernel<<<grid, kT, 0, st>>>(n, bt, r, z, partials.as<double2>(), vblk, snx, sny);
      });
    }
    launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(op, bt, partials.get(), dnb, sc); });
  };
  // z = B r ; rho = r^T z ; p = z
  precondition(OP_RHO);
  launch(ctx, "cocg_vec:pupdate", nb * (16.0 + vb), [&] {
    pupdate_kernel<<<grid, kT, 0, st>>>(n, bt, d_alpha, d_beta, z, pp, u, us, 1, snx, sny);
  });

  const bool zm = DIM == 3 || p->kind != LT_GRID_P1_TRI;
  const int nblk_apply = ta_ok ? ((L0.nx + TA_W - 1) / TA_W) * ((L0.ny + TA_H - 1) / TA_H) * ((L0.nz + ZM_ZC - 1) / ZM_ZC)
                               : zm ? zm_blocks(L0) : L0.ntiles;
  const double tol2 = p->inner_tol * p->inner_tol;
  FlagSlot* host_ring = ctx->flag_ring_dev();
  // one COCG iteration; u += alpha p is deferred into the direction update (pupdate)
  auto body = [&] {
    launch(ctx, "cocg_apply:operator", nb * 32.0 + coef, [&] {
      if (ta_ok)
        apply_tma2_kernel<<<(unsigned)nblk_apply * ((Bc + 1) / 2), kTA, TA2_SMEM, st>>>(
            map_p, map_c64, TzDims{L0.nx, L0.ny, L0.nz, L0.n}, bt, d_taus, q, partials.as<double2>(), nblk_apply);
      else if (zm)
        apply_dot_zm_kernel<<<(unsigned)nblk_apply * Bc, kT, 0, st>>>(L0, bt, d_taus, pp, q, partials.as<double2>(),
                                                                      nblk_apply);
      else
        apply_dot_kernel<DIM><<<(unsigned)nblk_apply * Bc, kT, 0, st>>>(L0, bt, d_taus, pp, q,
                                                                        partials.as<double2>(), nblk_apply);
    });
    launch(ctx, "cocg_scalar", 0.0, [&] {
      scalar_kernel<<<Bc, kT, 0, st>>>(OP_ALPHA, bt, partials.get(), nblk_apply, sc);
    });
    launch(ctx, "cocg_vec:axpy_norm", nb * (48.0 + vb), [&] {
      axpy_norm_kernel<<<grid, kT, 0, st>>>(n, bt, d_alpha, q, r, rmg, (double*)partials.get(), vblk, snx, sny);
    });
    launch(ctx, "cocg_scalar", 0.0, [&] { scalar_kernel<<<Bc, kT, 0, st>>>(OP_RR, bt, partials.get(), vblk, sc); });
    launch(ctx, "cocg_scalar", 0.0, [&] {
      cocg_control_kernel<<<1, cblk, 0, st>>>(Bc, d_done, d_rr, d_bb, d_best, d_stall, d_pending, tol2, d_counter,
                                              host_ring, kFlagRing, d_counts);
    });
    if (prof) ++ctx->profile_tag;
    precondition(OP_BETA);
    launch(ctx, "cocg_vec:pupdate", nb * (64.0 + vb), [&] {
      pupdate_kernel<<<grid, kT, 0, st>>>(n, bt, d_alpha, d_beta, z, pp, u, us, 0, snx, sny);
    });
  };

  // The host never drains the stream inside the loop: it issues iteration `it`, then waits
  // for iteration it - kFlagLag (already followed by queued work) and stops once that one
  // reported no active item.  The iteration issued after it is a no-op (every kernel skips
  // done items).  Without profiling the iteration body is one CUDA graph launch.
  const bool graph = !ctx->profiling && !debug_sync();
  cudaGraphExec_t exec = nullptr;
  int64_t body_launches = 0;
  if (graph) {
    const int64_t l0 = ctx->launches;
    cudaGraph_t g = nullptr;
    LT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    body();
    LT_CUDA(cudaStreamEndCapture(st, &g));
    body_launches = ctx->launches - l0;
    ctx->launches = l0;
    exec = p->graph_exec(g);
    LT_CUDA(cudaGraphDestroy(g));
  }
  // Near the end the host predicts the last iteration from the worst item's contraction and
  // waits for that iteration itself instead of issuing a speculative no-op one.
  volatile FlagSlot* ring = ctx->flag_ring_host();
  double w_prev = -1.0, w_last = -1.0;  // worst ratios of the last two iterations read
  auto read = [&](int k) -> bool {     // false: no item left after iteration k
    const int s = k % kFlagRing;
    LT_CUDA(cudaEventSynchronize(ctx->flag_ev[s]));
    if (ring[s].active == 0) return false;
    w_prev = w_last;
    w_last = ring[s].worst;
    return true;
  };
  int issued = 0;
  for (int it = 0; it < p->inner_maxit; ++it) {
    if (prof) ctx->profile_tag = it;
    if (graph) {
      LT_CUDA(cudaGraphLaunch(exec, st));
      ctx->launches += body_launches;
    } else {
      body();
    }
    LT_CUDA(cudaEventRecord(ctx->flag_ev[it % kFlagRing], st));
    issued = it + 1;
    if (it < kFlagLag) continue;
    if (!read(it - kFlagLag)) break;
    // predicted ratio after iteration it: the last one times the last contraction
    const bool last = w_prev > 0.0 && w_last < w_prev && w_last * (w_last / w_prev) <= 1.0;
    if (last && !read(it)) break;
  }
  if (prof) {
    // charge every tagged launch of this chunk for the items active at its step
    std::vector<int> cnt(issued + 1, Bc);
    LT_CUDA(cudaMemcpyAsync(cnt.data(), d_counts, sizeof(int) * (size_t)(issued + 1), cudaMemcpyDeviceToHost, st));
    stream_sync(ctx);
    for (size_t e = pend0; e < ctx->pending.size(); ++e) {
      auto& pe = ctx->pending[e];
      if (pe.tag >= 0 && pe.tag < (int)cnt.size()) pe.bytes *= (double)cnt[pe.tag] / Bc;
      pe.tag = -1;
    }
    ctx->profile_tag = -1;
  }
  // the last deferred solution update of the items that stopped after an r update
  launch(ctx, "cocg_vec:uupdate", nb * 48.0, [&] {
    uupdate_kernel<<<dim3(std::min<unsigned>(blocks_for(n, kT), 2 * ctx->num_sms), Bc), kT, 0, st>>>(
        n, d_pending, d_alpha, pp, u, us);
  });
  if (rel_out || inner_trace()) {
    std::vector<double> rr(Bc), bb(Bc);
    std::vector<int> done(Bc);
    LT_CUDA(cudaMemcpyAsync(rr.data(), d_rr, sizeof(double) * Bc, cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaMemcpyAsync(bb.data(), d_bb, sizeof(double) * Bc, cudaMemcpyDeviceToHost, st));
    stream_sync(ctx);
    for (int b = 0; b < Bc; ++b) {
      const double rel = bb[b] > 0.0 ? std::sqrt(rr[b] / bb[b]) : 0.0;
      if (rel_out) rel_out[b] = rel;
      if (inner_trace() >= 2)
        std::fprintf(stderr, "[inner] tau=(%.4g,%.4g) rel=%.3e\n", taus_host[b].x, taus_host[b].y, rel);
    }
    if (inner_trace()) std::fprintf(stderr, "[inner] chunk B=%d iterations issued=%d\n", Bc, issued);
  }
}

void inner_solve_mg(lt_pencil p, int B, const double2* taus_host, const double2* v, int64_t vs, double2* u,
                    int64_t us, const int* active, double* rel_out) {
  // Chunk so that the Krylov + multigrid workspace stays bounded.
  const int64_t n = p->n;
  const double avail = available_device_bytes(p->ctx);
  const double per_item = (double)n * (sizeof(double2) * 3.0 + sizeof(VM) * 3.0 * 1.2);
  int chunk = (int)std::max(1.0, std::min(128.0, 0.5 * avail / per_item));
  if (inner_trace())
    std::fprintf(stderr, "[inner] B=%d chunk=%d available=%.1fGB\n", B, chunk, avail / 1e9);
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int bc = std::min(chunk, B - b0);
    const int* act = active ? active + b0 : nullptr;
    double* rel = rel_out ? rel_out + b0 : nullptr;
    if (p->dim == 3) inner_chunk<3>(p, bc, taus_host + b0, v + b0 * vs, vs, u + b0 * us, us, act, rel);
    else inner_chunk<2>(p, bc, taus_host + b0, v + b0 * vs, vs, u + b0 * us, us, act, rel);
  }
}

}  // namespace

void inner_solve(lt_pencil p, int B, const double2* taus_host, const double2* v, int64_t vs, double2* u, int64_t us,
                 const int* active, double* rel_out) {
  // Items whose shift is known to need the exact banded solve (2-D pencils, strongly indefinite
  // shifts) take it directly; the others run MG-COCG, and an item that does not reach the
  // stagnation floor (kInnerFloor x the inner tolerance) is redone by the banded solve when the pencil
  // allows it (band.cu) -- else the preconditioner has failed (FactorizationError).
  std::vector<int> act(B, 1);
  if (active) {
    LT_CUDA(cudaMemcpyAsync(act.data(), active, sizeof(int) * B, cudaMemcpyDeviceToHost, p->ctx->stream));
    LT_CUDA(cudaStreamSynchronize(p->ctx->stream));
  }
  auto is_band = [&](double2 t) {
    for (const double2& b : p->band_taus)
      if (b.x == t.x && b.y == t.y) return true;
    return false;
  };
  std::vector<int> band(B, 0), mg(B, 0);
  int n_band = 0, n_mg = 0;
  for (int b = 0; b < B; ++b) {
    if (!act[b]) continue;
    if (is_band(taus_host[b])) { band[b] = 1; ++n_band; }
    else { mg[b] = 1; ++n_mg; }
  }
  std::vector<double> rel(B, 0.0);
  if (n_mg) {
    DeviceBuffer dmask;
    const int* mask = active;
    if (n_band) {
      dmask.allocate(sizeof(int) * B, p->ctx->stream);
      LT_CUDA(cudaMemcpyAsync(dmask.get(), mg.data(), sizeof(int) * B, cudaMemcpyHostToDevice, p->ctx->stream));
      mask = dmask.as<int>();
    }
    inner_solve_mg(p, B, taus_host, v, vs, u, us, mask, rel.data());
    for (int b = 0; b < B; ++b) {
      if (!mg[b] || rel[b] <= kInnerFloor * p->inner_tol) continue;
      if (!band_feasible(p)) {
        if (rel_out) continue;  // the caller reports it
        throw Error(LT_ERR_PRECONDITIONER, "shift-and-invert solve: the multigrid-preconditioned inner solve did not "
                                           "converge (relative residual " + std::to_string(rel[b]) + ")");
      }
      if (!is_band(taus_host[b])) p->band_taus.push_back(taus_host[b]);
      band[b] = 1;
      ++n_band;
    }
  }
  if (n_band) {
    for (int b = 0; b < B; ++b) {
      if (!band[b]) continue;
      const BandFactor& f = pencil_band_factor(p, taus_host[b]);
      // every item of this shift in one launch (one warp each)
      int b1 = b;
      while (b1 + 1 < B && band[b1 + 1] && taus_host[b1 + 1].x == taus_host[b].x && taus_host[b1 + 1].y == taus_host[b].y)
        ++b1;
      band_solve(p, f, b1 - b + 1, v + b * vs, vs, u + b * us, us);
      for (int q = b; q <= b1; ++q) {
        rel[q] = 0.0;  // exact LU, like the reference's factorisation
        band[q] = 0;
      }
      b = b1;
    }
  }
  if (rel_out)
    for (int b = 0; b < B; ++b) rel_out[b] = rel[b];
}

}  // namespace lt
