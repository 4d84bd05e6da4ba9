// Device helpers of the heterogeneous 5-point (2-D) / 7-point (3-D) cell-centred operator
//   (A(tau) u)_a = sum_f T_f (u_a - u_b) + tau M_a u_a,   u_b = 0 across Dirichlet faces.
#pragma once

#include "lt_internal.hpp"

namespace lt {

template <class VW>
__device__ __forceinline__ int64_t fx(const VW& L, int i, int j, int k) {
  return ((int64_t)k * L.ny + j) * (L.nx + 1) + i;
}
template <class VW>
__device__ __forceinline__ int64_t fy(const VW& L, int i, int j, int k) {
  return ((int64_t)k * (L.ny + 1) + j) * L.nx + i;
}

// Cell of thread threadIdx.x in tile `cb` of a level (256-thread x-y tiles, one plane);
// false for threads past the grid edge.
template <class VW>
__device__ __forceinline__ bool tile_cell(const VW& L, int cb, int& i, int& j, int& k, int64_t& a) {
  const int bx = cb % L.tiles_x;
  const int t = cb / L.tiles_x;
  const int by = t % L.tiles_y;
  k = t / L.tiles_y;
  i = (bx << L.tws) + (threadIdx.x & (L.tw - 1));
  j = by * L.th + (threadIdx.x >> L.tws);
  a = ((int64_t)k * L.ny + j) * L.nx + i;
  return i < L.nx && j < L.ny;
}

// (dk + tau m)^{-1} (f + off) with one real division
__device__ __forceinline__ double2 diag_solve(double dk, double m, double2 tau, double2 rhs) {
  const double dr = dk + tau.x * m, di = tau.y * m;
  const double inv = 1.0 / (dr * dr + di * di);
  return make_double2((rhs.x * dr + rhs.y * di) * inv, (rhs.y * dr - rhs.x * di) * inv);
}

template <int DIM>
__device__ __forceinline__ void decode(const LevelView& L, int64_t a, int& i, int& j, int& k) {
  i = (int)(a % L.nx);
  int64_t t = a / L.nx;
  if (DIM == 3) {
    j = (int)(t % L.ny);
    k = (int)(t / L.ny);
  } else {
    j = (int)t;
    k = 0;
  }
}

template <class VW>
__device__ __forceinline__ double diag_k(const VW& L, int i, int j, int k) {
  double d = L.Tx[fx(L, i, j, k)] + L.Tx[fx(L, i + 1, j, k)] + L.Ty[fy(L, i, j, k)] + L.Ty[fy(L, i, j + 1, k)];
  if (L.dim == 3) {
    int64_t a = ((int64_t)k * L.ny + j) * L.nx + i;
    d += L.Tz[a] + L.Tz[a + (int64_t)L.nx * L.ny];
  }
  return d;
}

// Gathers sum_f T_f u_b (neighbour coupling) and sum_f T_f (diagonal of K) at cell a.
template <int DIM>
__device__ __forceinline__ void gather(const LevelView& L, const double2* __restrict__ u, int64_t a, int i,
                                       int j, int k, double2& off, double& dk) {
  const int64_t ex = fx(L, i, j, k);
  const double tw = __ldg(L.Tx + ex), te = __ldg(L.Tx + ex + 1);
  const int64_t ey = fy(L, i, j, k);
  const double ts = __ldg(L.Ty + ey), tn = __ldg(L.Ty + ey + L.nx);
  dk = tw + te + ts + tn;
  double2 o = make_double2(0.0, 0.0);
  if (i > 0) { double2 v = u[a - 1]; o.x += tw * v.x; o.y += tw * v.y; }
  if (i < L.nx - 1) { double2 v = u[a + 1]; o.x += te * v.x; o.y += te * v.y; }
  if (j > 0) { double2 v = u[a - L.nx]; o.x += ts * v.x; o.y += ts * v.y; }
  if (j < L.ny - 1) { double2 v = u[a + L.nx]; o.x += tn * v.x; o.y += tn * v.y; }
  if (DIM == 3) {
    const int64_t plane = (int64_t)L.nx * L.ny;
    const double tb = __ldg(L.Tz + a), tt = __ldg(L.Tz + a + plane);
    dk += tb + tt;
    if (k > 0) { double2 v = u[a - plane]; o.x += tb * v.x; o.y += tb * v.y; }
    if (k < L.nz - 1) { double2 v = u[a + plane]; o.x += tt * v.x; o.y += tt * v.y; }
  }
  off = o;
}

// P1 only (2-D node grid): off-diagonal mass coupling sum_nb M_{a,nb} u_nb over the
// E/W/N/S edges and the NE/SW diagonal; Dirichlet neighbours contribute nothing.
template <class R, class V>
__device__ __forceinline__ V mass_off(const LevelViewT<R>& L, const V* __restrict__ u, int64_t a, int i, int j) {
  V o{0, 0};
  const int64_t ex = (int64_t)j * (L.nx + 1) + i;
  const int64_t ey = (int64_t)j * L.nx + i;
  if (i > 0) { const R w = L.Mx[ex]; const V v = u[a - 1]; o.x += w * v.x; o.y += w * v.y; }
  if (i < L.nx - 1) { const R w = L.Mx[ex + 1]; const V v = u[a + 1]; o.x += w * v.x; o.y += w * v.y; }
  if (j > 0) { const R w = L.My[ey]; const V v = u[a - L.nx]; o.x += w * v.x; o.y += w * v.y; }
  if (j < L.ny - 1) { const R w = L.My[ey + L.nx]; const V v = u[a + L.nx]; o.x += w * v.x; o.y += w * v.y; }
  if (i < L.nx - 1 && j < L.ny - 1) { const R w = L.Md[a]; const V v = u[a + L.nx + 1]; o.x += w * v.x; o.y += w * v.y; }
  if (i > 0 && j > 0) { const R w = L.Md[a - L.nx - 1]; const V v = u[a - L.nx - 1]; o.x += w * v.x; o.y += w * v.y; }
  return o;
}

// (M u)_a, including the P1 off-diagonal couplings when present
__device__ __forceinline__ double2 mass_apply(const LevelView& L, const double2* __restrict__ u, int64_t a, int i,
                                              int j) {
  double2 r = cscale(u[a], __ldg(L.M + a));
  if (L.Mx) r = cadd(r, mass_off(L, u, a, i, j));
  return r;
}

template <int DIM>
__device__ __forceinline__ double2 stencil_apply(const LevelView& L, const double2* __restrict__ u, int64_t a,
                                                 int i, int j, int k, double2 tau) {
  double2 off;
  double dk;
  gather<DIM>(L, u, a, i, j, k, off, dk);
  const double m = __ldg(L.M + a);
  const double2 ua = u[a];
  // (dk + tau m) ua - off  (+ tau * P1 mass couplings)
  const double2 d = make_double2(dk + tau.x * m, tau.y * m);
  double2 r = csub(cmul(d, ua), off);
  if (L.Mx) r = cadd(r, cmul(tau, mass_off(L, u, a, i, j)));
  return r;
}

}  // namespace lt
