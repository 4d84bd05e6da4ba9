// Flexible shifted FOM/GMRES (FGMRES-Sh, Algorithm 1) on the device, batched over B
// right-hand sides in lockstep.  Restates run_flexible (shifted_solver.cpp:132-287):
//   v0 = b/beta;  per iteration j:  u_j = (K + tau_j M)^{-1} v_j  (inner.cu);  s = M u_j;
//   Gram-Schmidt of s against V_{j+1} with one conditional re-orthogonalisation when the
//   norm drops below 1/sqrt(2) of its value (cpp:196-210; classical GS passes, which equal
//   the reference's MGS in exact arithmetic and read each basis vector once);
//   h_{j+1,j} = ||s||, breakdown at <= 1e-14 ||s0||;  per unconverged shift the small
//   problem on Hbar(z; T) = [I; 0] + Hbar (z I - T) (cpp:26-65: GMRES least squares via
//   Givens QR, FOM via Hessenberg partial-pivot LU), estimate/beta <= verify_at triggers
//   the true-residual check ||b - (K + zM) U y|| / beta (fused stencil kernel) and a
//   freeze, otherwise verify_at = estimate/2 (cpp:235-249).
// Solutions stay in basis form (U, y); expand_solutions materialises x = U y on demand.
#include <algorithm>
#include <cmath>
#include <vector>

#include "lt_internal.hpp"
#include "stencil.cuh"

namespace lt {

namespace {

constexpr int kT = 256;
constexpr double kBreakdownTol = 1e-14;

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffff, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum_c(double2 v) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffff, v.x, o);
    v.y += __shfl_down_sync(0xffffffff, v.y, o);
  }
  return v;
}
// block reduction into thread 0 using caller-provided shared scratch of 32 entries
__device__ __forceinline__ double2 block_sum_c(double2 v, double2* sh) {
  v = warp_sum_c(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : make_double2(0.0, 0.0);
    v = warp_sum_c(v);
  }
  return v;
}
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    v = warp_sum_d(v);
  }
  return v;
}

struct State {
  int B, ns, maxit, cap;
  int64_t n;
  int nblk;
  int nblk_tile;  // tiles per item of the fine level (verify_residual partials)
  double tol;
  int variant;
  int record_history;
  int* active;           // B: item still iterating
  const double* beta;    // B
  const double2* shifts; // B*ns
  const double2* taus;   // B*maxit (tau applied at iteration j)
  double2* H;            // B*maxit*(maxit+1): H[(b*maxit + j)*(maxit+1) + i] = h_{i,j}
  int* conv;             // B*ns
  int* iter;
  double* est;
  double* true_res;
  double* verify_at;
  int* flag;             // B*ns: verify requested this iteration
  int* m_used;           // B*ns
  double2* Y;            // B*ns*maxit
  double* history;       // B*ns*maxit or null
  double2* scratch;      // B*ns*(cap+1)*cap
  double* norm0;         // B: ||s|| before orthogonalisation
  double* norm1;         // B: ||s|| after the first pass
  int* reorth;           // B
  int* breakdown;        // B
  double* hnext;         // B
  int* n_unconv;         // B
};

// s = M u (written into V_{j+1}), partial conj(V_i) . s for i <= j and ||s||^2
template <int DIM>
__global__ void __launch_bounds__(kT) mass_multidot(LevelView L, State S, int j, const double2* __restrict__ u,
                                                    double2* __restrict__ s_out, const double2* const* __restrict__ Vcols,
                                                    double2* __restrict__ part) {
  __shared__ double2 sh[32];
  LT_ITEM_BLOCK(S.B, b, cb);
  if (!S.active[b]) return;
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  const bool in = a < L.n;
  double2 s = make_double2(0.0, 0.0);
  if (in) {
    s = cscale(u[b * L.n + a], __ldg(L.M + a));
    if (L.Mx) s = cadd(s, mass_off(L, u + b * L.n, a, (int)(a % L.nx), (int)(a / L.nx)));  // P1 (2-D)
    s_out[b * L.n + a] = s;
  }
  double2* pb = part + (int64_t)b * (j + 2) * S.nblk;
  for (int i = 0; i <= j; ++i) {
    double2 v = in ? Vcols[i][b * L.n + a] : make_double2(0.0, 0.0);
    double2 d = block_sum_c(cmulc(v, s), sh);
    if (threadIdx.x == 0) pb[(int64_t)i * S.nblk + cb] = d;
  }
  double2 nn = block_sum_c(make_double2(cabs2(s), 0.0), sh);
  if (threadIdx.x == 0) pb[(int64_t)(j + 1) * S.nblk + cb] = nn;
}

// partial conj(V_i) . s for i <= j (re-orthogonalisation pass, items with reorth set)
__global__ void __launch_bounds__(kT) multidot(State S, int j, const double2* __restrict__ s_in,
                                               const double2* const* __restrict__ Vcols, double2* __restrict__ part) {
  __shared__ double2 sh[32];
  LT_ITEM_BLOCK(S.B, b, cb);
  if (!S.active[b] || !S.reorth[b]) return;
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  const bool in = a < S.n;
  const double2 s = in ? s_in[b * S.n + a] : make_double2(0.0, 0.0);
  double2* pb = part + (int64_t)b * (j + 2) * S.nblk;
  for (int i = 0; i <= j; ++i) {
    double2 v = in ? Vcols[i][b * S.n + a] : make_double2(0.0, 0.0);
    double2 d = block_sum_c(cmulc(v, s), sh);
    if (threadIdx.x == 0) pb[(int64_t)i * S.nblk + cb] = d;
  }
}

// sum the partials: coefficients into hcoef[b*(j+1) + i] (pass 0: set; pass 1: add into H),
// norm into norm0 (pass 0)
__global__ void __launch_bounds__(kT) reduce_dots(State S, int j, const double2* __restrict__ part, int pass,
                                                  double2* __restrict__ hcoef) {
  __shared__ double2 sh[32];
  const int b = blockIdx.x / (j + 2);
  const int i = blockIdx.x % (j + 2);
  if (!S.active[b]) return;
  if (pass == 1 && (!S.reorth[b] || i == j + 1)) return;
  const double2* pb = part + ((int64_t)b * (j + 2) + i) * S.nblk;
  double2 s = make_double2(0.0, 0.0);
  for (int k = threadIdx.x; k < S.nblk; k += blockDim.x) s = cadd(s, pb[k]);
  s = block_sum_c(s, sh);
  if (threadIdx.x != 0) return;
  if (i == j + 1) {
    S.norm0[b] = sqrt(s.x);
    return;
  }
  hcoef[b * (j + 1) + i] = s;
  double2* Hc = S.H + ((int64_t)b * S.maxit + j) * (S.maxit + 1);
  if (pass == 0) Hc[i] = s;
  else Hc[i] = cadd(Hc[i], s);
}

// s -= sum_i c_i V_i ; partial ||s||^2 (pass 1 only for reorth items)
__global__ void __launch_bounds__(kT) gs_update(State S, int j, int pass, double2* __restrict__ s_io,
                                                const double2* const* __restrict__ Vcols,
                                                const double2* __restrict__ hcoef, double* __restrict__ part) {
  __shared__ double sh[32];
  LT_ITEM_BLOCK(S.B, b, cb);
  if (!S.active[b]) return;
  if (pass == 1 && !S.reorth[b]) return;
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  double nn = 0.0;
  if (a < S.n) {
    double2 s = s_io[b * S.n + a];
    for (int i = 0; i <= j; ++i) s = csub(s, cmul(hcoef[b * (j + 1) + i], Vcols[i][b * S.n + a]));
    s_io[b * S.n + a] = s;
    nn = cabs2(s);
  }
  nn = block_sum_d(nn, sh);
  if (threadIdx.x == 0) part[(int64_t)b * S.nblk + cb] = nn;
}

// after pass `pass`: norm of s; pass 0 decides re-orthogonalisation; the final pass
// sets h_{j+1,j}, breakdown and 1/h.
__global__ void __launch_bounds__(kT) reduce_norm(State S, int j, int pass, const double* __restrict__ part) {
  __shared__ double sh[32];
  const int b = blockIdx.x;
  if (!S.active[b]) return;
  if (pass == 1 && !S.reorth[b]) return;
  const double* pb = part + (int64_t)b * S.nblk;
  double s = 0.0;
  for (int k = threadIdx.x; k < S.nblk; k += blockDim.x) s += pb[k];
  s = block_sum_d(s, sh);
  if (threadIdx.x != 0) return;
  const double nrm = sqrt(s);
  if (pass == 0) {
    S.norm1[b] = nrm;
    S.reorth[b] = nrm < S.norm0[b] / sqrt(2.0);
  }
  if (pass == 1 || !S.reorth[b]) {
    double2* Hc = S.H + ((int64_t)b * S.maxit + j) * (S.maxit + 1);
    Hc[j + 1] = make_double2(nrm, 0.0);
    S.hnext[b] = nrm;
    S.breakdown[b] = nrm <= kBreakdownTol * S.norm0[b];
  }
}

__global__ void __launch_bounds__(kT) normalize(State S, double2* __restrict__ v) {
  LT_ITEM_BLOCK(S.B, b, cb);
  if (!S.active[b] || S.breakdown[b]) return;
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  if (a < S.n) {
    const double inv = 1.0 / S.hnext[b];
    v[b * S.n + a] = cscale(v[b * S.n + a], inv);
  }
}

// hz(i, l) = h_{i,l} (z - tau_l) + delta_il, i <= l + 1
__device__ __forceinline__ double2 hz_entry(const State& S, int b, int i, int l, double2 z) {
  if (i > l + 1) return make_double2(0.0, 0.0);
  const double2 h = S.H[((int64_t)b * S.maxit + l) * (S.maxit + 1) + i];
  double2 v = cmul(h, csub(z, S.taus[(int64_t)b * S.maxit + l]));
  if (i == l) v.x += 1.0;
  return v;
}

// Per (item, shift): small least-squares (GMRES) / square (FOM) solve on Hbar_m(z; T_m),
// history, verify decision.  force: best-effort pass for unconverged shifts at the end.
__global__ void small_solve(State S, int m, int force) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S.B * S.ns) return;
  const int b = t / S.ns;
  S.flag[t] = 0;
  if (!S.active[b]) return;
  if (S.conv[t]) return;
  const double2 z = S.shifts[t];
  const double beta = S.beta[b];
  const int ld = m + 1;
  double2* W = S.scratch + (int64_t)t * (S.cap + 1) * S.cap;  // column-major (m+1) x m
  for (int l = 0; l < m; ++l)
    for (int i = 0; i <= m; ++i) W[(int64_t)l * ld + i] = hz_entry(S, b, i, l, z);
  double2* y = S.Y + (int64_t)t * S.maxit;
  bool valid = true;
  double estimate = INFINITY;
  if (S.variant == LT_VARIANT_GMRES) {
    // Givens QR of the Hessenberg hz; rhs g = beta e1 (stored in y[0..m], y has maxit >= m+1? no)
    // rotated rhs g = beta e1: g_0..g_{m-1} live in y, g_m in gm
    double2 g[2];
    y[0] = make_double2(beta, 0.0);
    for (int l = 1; l < m; ++l) y[l] = make_double2(0.0, 0.0);
    double2 gm = make_double2(0.0, 0.0);
    for (int l = 0; l < m; ++l) {
      const double2 x1 = W[(int64_t)l * ld + l];
      const double2 x2 = W[(int64_t)l * ld + l + 1];
      const double ax = sqrt(cabs2(x1)), r = sqrt(cabs2(x1) + cabs2(x2));
      if (!(r > 0.0)) { valid = false; break; }
      double cs;
      double2 sn, ph;
      if (ax == 0.0) {
        cs = 0.0; sn = make_double2(1.0, 0.0); ph = make_double2(1.0, 0.0);
      } else {
        cs = ax / r;
        ph = cscale(x1, 1.0 / ax);
        sn = cmul(ph, cscale(cconj(x2), 1.0 / r));  // (a/|a|) conj(b) / r
      }
      // rows l, l+1:  [cs  sn; -conj(sn)  cs]
      for (int c = l; c < m; ++c) {
        const double2 a1 = W[(int64_t)c * ld + l], a2 = W[(int64_t)c * ld + l + 1];
        W[(int64_t)c * ld + l] = cadd(cscale(a1, cs), cmul(sn, a2));
        W[(int64_t)c * ld + l + 1] = csub(cscale(a2, cs), cmul(cconj(sn), a1));
      }
      const double2 g1 = y[l];
      const double2 g2 = (l + 1 < m) ? y[l + 1] : gm;
      g[0] = cadd(cscale(g1, cs), cmul(sn, g2));
      g[1] = csub(cscale(g2, cs), cmul(cconj(sn), g1));
      y[l] = g[0];
      if (l + 1 < m) y[l + 1] = g[1]; else gm = g[1];
    }
    if (valid) {
      for (int l = m - 1; l >= 0; --l) {
        double2 acc = y[l];
        for (int c = l + 1; c < m; ++c) acc = csub(acc, cmul(W[(int64_t)c * ld + l], y[c]));
        y[l] = cdiv(acc, W[(int64_t)l * ld + l]);
        if (!isfinite(y[l].x) || !isfinite(y[l].y)) valid = false;
      }
    }
    if (valid) {
      // explicit ||beta e1 - hz y|| (cpp:61)
      double ss = 0.0;
      for (int i = 0; i <= m; ++i) {
        double2 r = make_double2(i == 0 ? beta : 0.0, 0.0);
        const int l0 = i > 0 ? i - 1 : 0;
        for (int l = l0; l < m; ++l) r = csub(r, cmul(hz_entry(S, b, i, l, z), y[l]));
        ss += cabs2(r);
      }
      estimate = sqrt(ss);
    }
  } else {
    // FOM: Hessenberg LU with partial pivoting on the m x m top (cpp:36-51)
    y[0] = make_double2(beta, 0.0);
    for (int l = 1; l < m; ++l) y[l] = make_double2(0.0, 0.0);
    for (int l = 0; l < m && valid; ++l) {
      if (l + 1 < m) {
        const double2 p1 = W[(int64_t)l * ld + l], p2 = W[(int64_t)l * ld + l + 1];
        if (cabs2(p2) > cabs2(p1)) {
          for (int c = l; c < m; ++c) {
            double2 tmp = W[(int64_t)c * ld + l];
            W[(int64_t)c * ld + l] = W[(int64_t)c * ld + l + 1];
            W[(int64_t)c * ld + l + 1] = tmp;
          }
          double2 tmp = y[l]; y[l] = y[l + 1]; y[l + 1] = tmp;
        }
        const double2 piv = W[(int64_t)l * ld + l];
        if (!(cabs2(piv) > 0.0)) { valid = false; break; }
        const double2 f = cdiv(W[(int64_t)l * ld + l + 1], piv);
        for (int c = l; c < m; ++c)
          W[(int64_t)c * ld + l + 1] = csub(W[(int64_t)c * ld + l + 1], cmul(f, W[(int64_t)c * ld + l]));
        y[l + 1] = csub(y[l + 1], cmul(f, y[l]));
      }
    }
    if (valid) {
      for (int l = m - 1; l >= 0; --l) {
        double2 acc = y[l];
        for (int c = l + 1; c < m; ++c) acc = csub(acc, cmul(W[(int64_t)c * ld + l], y[c]));
        y[l] = cdiv(acc, W[(int64_t)l * ld + l]);
        if (!isfinite(y[l].x) || !isfinite(y[l].y)) valid = false;
      }
    }
    if (valid) {
      const double2 hmm = hz_entry(S, b, m, m - 1, z);
      estimate = sqrt(cabs2(cmul(hmm, y[m - 1])));
    }
  }
  if (!valid) {
    if (!force && S.record_history) S.history[(int64_t)t * S.maxit + (m - 1)] = S.est[t];
    return;
  }
  if (force) {
    S.flag[t] = 1;
    return;
  }
  S.est[t] = estimate / beta;
  if (S.record_history) S.history[(int64_t)t * S.maxit + (m - 1)] = S.est[t];
  if (S.est[t] <= S.verify_at[t] || S.breakdown[b]) S.flag[t] = 1;
}

// True residual r = b - (K + z M) U y for every flagged shift of an item:
// partial ||r||^2 per (item, shift).  K u_j and M u_j are formed once per column and
// accumulated as sum_j y_jq K u_j + (y_jq z_q) M u_j (y z staged in shared memory); the KC
// per-shift partial norms are reduced together (one barrier per chunk, not one per shift).
// Blocks: (x-y tile of the fine level, chunk of VR_Z planes) per item; each thread marches its
// column through the chunk and accumulates its cells' |r|^2 per shift in registers, so the
// per-shift block reductions run once per chunk instead of once per cell.
constexpr int VR_Z = 16;
inline int verify_blocks(const LevelView& L) { return L.tiles_x * L.tiles_y * ((L.nz + VR_Z - 1) / VR_Z); }

template <int DIM>
__global__ void __launch_bounds__(kT, 2) verify_residual(LevelView L, State S, int m, const double2* __restrict__ rhs,
                                                         const double2* const* __restrict__ Ucols,
                                                         double* __restrict__ part) {
  constexpr int KC = 16;  // shifts per register chunk
  constexpr int MJ = 16;  // Krylov columns whose coefficients are staged in shared memory
  constexpr int NW = kT / 32;
  __shared__ int flagged[256];
  __shared__ int nflag;
  __shared__ double2 ysm[MJ][KC], yzsm[MJ][KC];
  __shared__ double nsm[KC][kT];  // per-thread running |r|^2 per shift
  LT_ITEM_BLOCK(S.B, b, cb);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tpp = L.tiles_x * L.tiles_y;
  const int tile = (int)(cb % tpp), zc = (int)(cb / tpp);
  const int kz0 = DIM == 3 ? zc * VR_Z : 0, kz1 = DIM == 3 ? min(L.nz, kz0 + VR_Z) : 1;
  int i, jj, kk;
  int64_t a0;
  const bool in = tile_cell(L, tile, i, jj, kk, a0);  // (i, jj) of the column; plane 0
  const int64_t plane = (int64_t)L.nx * L.ny;
  // the flagged shifts of this item, in windows of 256 shift indices
  for (int base = 0; base < S.ns; base += 256) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int k = base; k < S.ns && k < base + 256; ++k)
      if (S.flag[b * S.ns + k]) flagged[c++] = k;
    nflag = c;
  }
  __syncthreads();
  if (nflag == 0) continue;  // uniform
  for (int c0 = 0; c0 < nflag; c0 += KC) {
    const int nc = min(KC, nflag - c0);
    const bool staged = m <= MJ;
    __syncthreads();
    if (staged) {
      for (int e = threadIdx.x; e < KC * MJ; e += blockDim.x) {
        const int j = e / KC, q = e % KC;
        double2 y = make_double2(0.0, 0.0), yz = y;
        if (q < nc && j < m) {
          const int t = b * S.ns + flagged[c0 + q];
          y = S.Y[(int64_t)t * S.maxit + j];
          yz = cmul(y, S.shifts[t]);
        }
        ysm[j][q] = y;
        yzsm[j][q] = yz;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < KC; ++q) nsm[q][threadIdx.x] = 0.0;
    if (in) {
      for (int k = kz0; k < kz1; ++k) {
        const int64_t a = a0 + k * plane;
        const double2 bv = rhs[b * L.n + a];
        const double mval = __ldg(L.M + a);
        double2 acc[KC];
#pragma unroll
        for (int q = 0; q < KC; ++q) acc[q] = make_double2(0.0, 0.0);
        for (int j = 0; j < m; ++j) {
          const double2* ub = Ucols[j] + b * L.n;
          double2 off;
          double dk;
          gather<DIM>(L, ub, a, i, jj, k, off, dk);
          const double2 ua = ub[a];
          const double2 Ku = csub(cscale(ua, dk), off);
          double2 Mu = cscale(ua, mval);
          if (L.Mx) Mu = cadd(Mu, mass_off(L, ub, a, i, jj));
#pragma unroll
          for (int q = 0; q < KC; ++q) {
            if (q < nc) {
              double2 y, yz;
              if (staged) {
                y = ysm[j][q];
                yz = yzsm[j][q];
              } else {
                const int t = b * S.ns + flagged[c0 + q];
                y = S.Y[(int64_t)t * S.maxit + j];
                yz = cmul(y, S.shifts[t]);
              }
              acc[q] = cfma(y, Ku, cfma(yz, Mu, acc[q]));
            }
          }
        }
#pragma unroll
        for (int q = 0; q < KC; ++q)
          if (q < nc) nsm[q][threadIdx.x] += cabs2(csub(bv, acc[q]));
      }
    }
    // per-shift partial norms: warp w reduces shifts w, w + NW over the block
    __syncthreads();
    for (int q = w; q < nc; q += NW) {
      double t = 0.0;
      for (int v = lane; v < kT; v += 32) t += nsm[q][v];
      t = warp_sum_d(t);
      if (lane == 0) part[((int64_t)b * S.ns + flagged[c0 + q]) * S.nblk_tile + cb] = t;
    }
  }
  }  // window
}

// The same true residuals for the first outer iterations (m <= 4 Krylov columns: every
// BASELINE config converges in 2-4), FD pencils.  K u_j and M u_j of all columns stay in
// registers and the shifts are walked one after the other with a single accumulator, so a
// thread holds 4 m + 16 doubles instead of the 32 + 16 of the general kernel (which ncu shows
// latency-bound at 25% occupancy, FP64 pipe 20% busy: 128 registers, one shared-memory
// read-modify-write per shift and plane) and the per-shift norms live in registers.
// A formulation on the FP64 tensor cores (one m8n8k4 per 8 cells, column and 4 shifts; lane =
// one real of K u / M u) was built and measured 1.5x SLOWER at these small m: with 8 cells per
// warp instruction the per-cell set-up (coefficients, offsets, right-hand side) costs 4x more
// instructions than the products it feeds.
template <int DIM, int MC>
__global__ void __launch_bounds__(kT, MC <= 1 ? 3 : 2) verify_residual_small(LevelView L, State S, const double2* __restrict__ rhs,
                                                               const double2* const* __restrict__ Ucols,
                                                               double* __restrict__ part) {
  constexpr int KC = 16, NW = kT / 32;
  __shared__ int flagged[256];
  __shared__ int nflag;
  __shared__ double2 ysm[MC][KC], yzsm[MC][KC];
  __shared__ double nsm[NW][KC];
  LT_ITEM_BLOCK(S.B, b, cb);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tpp = L.tiles_x * L.tiles_y;
  const int tile = (int)(cb % tpp), zc = (int)(cb / tpp);
  const int kz0 = DIM == 3 ? zc * VR_Z : 0, kz1 = DIM == 3 ? min(L.nz, kz0 + VR_Z) : 1;
  int i, jj, kk;
  int64_t a0;
  const bool in = tile_cell(L, tile, i, jj, kk, a0);
  const int64_t plane = (int64_t)L.nx * L.ny;
  const double2* ub[MC];
#pragma unroll
  for (int j = 0; j < MC; ++j) ub[j] = Ucols[j] + b * L.n;
  for (int base = 0; base < S.ns; base += 256) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int cnt = 0;
      for (int k = base; k < S.ns && k < base + 256; ++k)
        if (S.flag[b * S.ns + k]) flagged[cnt++] = k;
      nflag = cnt;
    }
    __syncthreads();
    if (nflag == 0) continue;  // uniform
    for (int c0 = 0; c0 < nflag; c0 += KC) {
      const int nc = min(KC, nflag - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < KC * MC; e += blockDim.x) {
        const int j = e / KC, q = e % KC;
        double2 y = make_double2(0.0, 0.0), yz = y;
        if (q < nc) {
          const int t = b * S.ns + flagged[c0 + q];
          y = S.Y[(int64_t)t * S.maxit + j];
          yz = cmul(y, S.shifts[t]);
        }
        ysm[j][q] = y;
        yzsm[j][q] = yz;
      }
      __syncthreads();
      double nrm[KC];
#pragma unroll
      for (int q = 0; q < KC; ++q) nrm[q] = 0.0;
      if (in) {
        for (int k = kz0; k < kz1; ++k) {
          const int64_t a = a0 + k * plane;
          const double2 bv = rhs[b * L.n + a];
          const double mval = __ldg(L.M + a);
          double2 Ku[MC], Mu[MC];
#pragma unroll
          for (int j = 0; j < MC; ++j) {
            double2 off;
            double dk;
            gather<DIM>(L, ub[j], a, i, jj, k, off, dk);
            const double2 ua = ub[j][a];
            Ku[j] = csub(cscale(ua, dk), off);
            Mu[j] = cscale(ua, mval);
          }
#pragma unroll
          for (int q = 0; q < KC; ++q) {
            if (q < nc) {
              double2 r = bv;
#pragma unroll
              for (int j = 0; j < MC; ++j) {
                const double2 y = ysm[j][q], yz = yzsm[j][q];
                r.x -= y.x * Ku[j].x - y.y * Ku[j].y + yz.x * Mu[j].x - yz.y * Mu[j].y;
                r.y -= y.x * Ku[j].y + y.y * Ku[j].x + yz.x * Mu[j].y + yz.y * Mu[j].x;
              }
              nrm[q] += r.x * r.x + r.y * r.y;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        const double v = warp_sum_d(nrm[q]);
        if (lane == 0) nsm[w][q] = v;
      }
      __syncthreads();
      if (threadIdx.x < nc) {
        double t = 0.0;
        for (int v = 0; v < NW; ++v) t += nsm[v][threadIdx.x];
        part[((int64_t)b * S.ns + flagged[c0 + threadIdx.x]) * S.nblk_tile + cb] = t;
      }
    }
  }  // window
}

// verify_residual: the small-m kernel when it applies (FD, m <= 4)
#ifndef LT_VERIFY_SMALL
#define LT_VERIFY_SMALL 1
#endif
template <int DIM>
static void launch_verify_dim(const LevelView& L0, const State& S, int m, const double2* rhs,
                              const double2* const* Ucols, double* part, unsigned grid, cudaStream_t st) {
  if (LT_VERIFY_SMALL && !L0.Mx && m <= 4) {
    switch (m) {
      case 1: verify_residual_small<DIM, 1><<<grid, kT, 0, st>>>(L0, S, rhs, Ucols, part); return;
      case 2: verify_residual_small<DIM, 2><<<grid, kT, 0, st>>>(L0, S, rhs, Ucols, part); return;
      case 3: verify_residual_small<DIM, 3><<<grid, kT, 0, st>>>(L0, S, rhs, Ucols, part); return;
      default: verify_residual_small<DIM, 4><<<grid, kT, 0, st>>>(L0, S, rhs, Ucols, part); return;
    }
  }
  verify_residual<DIM><<<grid, kT, 0, st>>>(L0, S, m, rhs, Ucols, part);
}
static void launch_verify(lt_pencil p, const LevelView& L0, const State& S, int m, const double2* rhs,
                          const double2* const* Ucols, double* part, int B, cudaStream_t st) {
  const unsigned grid = (unsigned)S.nblk_tile * (unsigned)B;
  if (p->dim == 3) launch_verify_dim<3>(L0, S, m, rhs, Ucols, part, grid, st);
  else launch_verify_dim<2>(L0, S, m, rhs, Ucols, part, grid, st);
}

// per (item, shift) flagged: true_rel; freeze or back off.  best_effort: record only.
__global__ void __launch_bounds__(kT) verify_finalize(State S, int m, const double* __restrict__ part, int best_effort) {
  __shared__ double sh[32];
  const int t = blockIdx.x;
  if (!S.flag[t]) return;
  const int b = t / S.ns;
  const double* pb = part + (int64_t)t * S.nblk_tile;
  double s = 0.0;
  for (int k = threadIdx.x; k < S.nblk_tile; k += blockDim.x) s += pb[k];
  s = block_sum_d(s, sh);
  if (threadIdx.x != 0) return;
  const double true_rel = sqrt(s) / S.beta[b];
  S.flag[t] = 0;
  if (best_effort) {
    S.true_res[t] = true_rel;
    S.m_used[t] = m;
    return;
  }
  if (true_rel <= S.tol || S.breakdown[b]) {
    S.conv[t] = 1;
    S.iter[t] = m;
    S.true_res[t] = true_rel;
    S.m_used[t] = m;
  } else {
    S.verify_at[t] = S.est[t] / 2.0;
  }
}

// After the freeze checks of iteration m: unconverged shifts per item; an item whose shifts
// all froze, or that broke down, stops iterating (cpp:250-262).
__global__ void outer_control(State S, int m, int* __restrict__ iterations) {
  for (int b = threadIdx.x; b < S.B; b += blockDim.x) {
    if (!S.active[b]) continue;
    int c = 0;
    for (int k = 0; k < S.ns; ++k) c += !S.conv[b * S.ns + k];
    S.n_unconv[b] = c;
    iterations[b] = m;
    if (c == 0 || S.breakdown[b]) S.active[b] = 0;
  }
}

// dense batch <-> item positions: to = 0: out[q] = in[idx[q]]; to = 1: out[idx[q]] = in[q]
__global__ void __launch_bounds__(kT) pack_items(int64_t n, const int* __restrict__ idx, const double2* __restrict__ in,
                                                 double2* __restrict__ out, int to) {
  const int q = blockIdx.y;
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int64_t src = (to ? q : idx[q]) * n + a, dst = (to ? idx[q] : q) * n + a;
  out[dst] = in[src];
}

// beta = ||b|| known: beta == 0 items are done, every shift converged with zero estimate and
// residual (cpp:147-156); the others iterate.
__global__ void outer_init(State S) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= S.B * S.ns) return;
  const int b = t / S.ns;
  const bool zero = !(S.beta[b] > 0.0);
  if (t % S.ns == 0) S.active[b] = !zero;
  if (zero) {
    S.conv[t] = 1;
    S.est[t] = 0.0;
    S.true_res[t] = 0.0;
  }
}

__global__ void __launch_bounds__(kT) norm_kernel(int64_t n, int B, const double2* __restrict__ x, double* __restrict__ part,
                                                  int nblk) {
  __shared__ double sh[32];
  LT_ITEM_BLOCK(B, b, cb);
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  double s = a < n ? cabs2(x[b * n + a]) : 0.0;
  s = block_sum_d(s, sh);
  if (threadIdx.x == 0) part[(int64_t)b * nblk + cb] = s;
}

__global__ void __launch_bounds__(kT) reduce_beta(int B, int nblk, const double* __restrict__ part, double* __restrict__ beta) {
  __shared__ double sh[32];
  const int b = blockIdx.x;
  double s = 0.0;
  for (int k = threadIdx.x; k < nblk; k += blockDim.x) s += part[(int64_t)b * nblk + k];
  s = block_sum_d(s, sh);
  if (threadIdx.x == 0) beta[b] = sqrt(s);
}

__global__ void __launch_bounds__(kT) scale_to(int64_t n, int B, const double2* __restrict__ x, const double* __restrict__ beta,
                                               double2* __restrict__ v) {
  LT_ITEM_BLOCK(B, b, cb);
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const double bt = beta[b];
  v[b * n + a] = bt > 0.0 ? cscale(x[b * n + a], 1.0 / bt) : make_double2(0.0, 0.0);
}

// x_out[(b*ns + k)*n + a] = scale_{b,k} sum_{j < m_used} Y[b,k,j] U_j[b][a]
__global__ void __launch_bounds__(kT) expand_kernel(int64_t n, int B, int ns, int maxit, const double2* const* __restrict__ Ucols,
                                                    const double2* __restrict__ Y, const int* __restrict__ m_used,
                                                    const double2* __restrict__ scale, double2* __restrict__ out) {
  LT_ITEM_BLOCK(B, b, cb);
  const int64_t a = cb * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  int mmax = 0;
  for (int k = 0; k < ns; ++k) mmax = max(mmax, m_used[b * ns + k]);
  constexpr int KC = 16;
  for (int k0 = 0; k0 < ns; k0 += KC) {
    double2 acc[KC];
#pragma unroll
    for (int q = 0; q < KC; ++q) acc[q] = make_double2(0.0, 0.0);
    for (int j = 0; j < mmax; ++j) {
      const double2 u = Ucols[j][b * n + a];
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        const int k = k0 + q;
        if (k < ns && j < m_used[b * ns + k]) acc[q] = cfma(Y[((int64_t)b * ns + k) * maxit + j], u, acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      const int k = k0 + q;
      if (k < ns) out[((int64_t)b * ns + k) * n + a] = scale ? cmul(scale[b * ns + k], acc[q]) : acc[q];
    }
  }
}

// Cell-major variant for the Jacobian: out[(k n + a) B + b] (all items of a (shift, cell)
// contiguous).  A block takes 32 cells x 8 items: basis reads are coalesced along the cells of
// one item, each shift's 32 x 8 values are transposed through shared memory and written as
// 8-item (128-byte) runs.
__global__ void __launch_bounds__(256) expand_cm_kernel(int64_t n, int B, int ns, int maxit,
                                                        const double2* const* __restrict__ Ucols,
                                                        const double2* __restrict__ Y, const int* __restrict__ m_used,
                                                        const double2* __restrict__ scale, double2* __restrict__ out) {
  constexpr int CX = 32, IY = 8, KC = 16;
  __shared__ double2 tile[CX][IY + 1];
  const int cl = threadIdx.x % CX, il = threadIdx.x / CX;
  const int64_t a0 = (int64_t)blockIdx.x * CX;
  const int b0 = blockIdx.y * IY;
  const int64_t a = a0 + cl;
  const int b = b0 + il;
  const bool in = a < n && b < B;
  int mmax = 0;
  if (b < B)
    for (int k = 0; k < ns; ++k) mmax = max(mmax, m_used[b * ns + k]);
  for (int k0 = 0; k0 < ns; k0 += KC) {
    double2 acc[KC];
#pragma unroll
    for (int q = 0; q < KC; ++q) acc[q] = make_double2(0.0, 0.0);
    if (in)
      for (int j = 0; j < mmax; ++j) {
        const double2 u = Ucols[j][b * n + a];
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          const int k = k0 + q;
          if (k < ns && j < m_used[b * ns + k]) acc[q] = cfma(Y[((int64_t)b * ns + k) * maxit + j], u, acc[q]);
        }
      }
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      const int k = k0 + q;
      if (k >= ns) break;  // uniform
      __syncthreads();
      tile[cl][il] = (in && scale) ? cmul(scale[b * ns + k], acc[q]) : acc[q];
      __syncthreads();
      // write: thread -> (cell c = t / IY, item i = t % IY): 8 consecutive items per cell
      const int c = threadIdx.x / IY, i = threadIdx.x % IY;
      if (a0 + c < n && b0 + i < B) out[((int64_t)k * n + a0 + c) * B + b0 + i] = tile[c][i];
    }
  }
}

// Cell-major expansion, v2: the (scaled, column-masked) coefficients of all items and shifts,
// ys[(k mmax + j) B + b] = scale_bk y_bk[j] (0 for j >= m_bk), are staged once per block in
// shared memory; thread <-> (cell, item) pairs in item-fastest order, so for every shift a
// warp writes one contiguous 512-byte run of out[(k n + a) B + b] (the block's CT x B pairs
// are one contiguous run per shift) and reads its coefficients conflict-free.  No per-shift
// barriers (the v1 kernel transposed every shift through shared memory, 2 barriers each).
__global__ void expand_coeffs(int B, int ns, int maxit, int mmax, const double2* __restrict__ Y,
                              const int* __restrict__ m_used, const double2* __restrict__ scale,
                              double2* __restrict__ ys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns * mmax * B) return;
  const int b = i % B, j = (i / B) % mmax, k = i / (B * mmax);
  const int bk = b * ns + k;
  double2 v = make_double2(0.0, 0.0);
  if (j < m_used[bk]) v = Y[(int64_t)bk * maxit + j];
  if (scale) v = cmul(scale[bk], v);
  ys[i] = v;
}

template <int MAXM>
__global__ void __launch_bounds__(256) expand_cm2_kernel(int64_t n, int B, int ns, int mmax, int CT,
                                                         const double2* const* __restrict__ Ucols,
                                                         const double2* __restrict__ ysg, double2* __restrict__ out) {
  extern __shared__ double2 ys[];  // [k][j][b]
  for (int i = threadIdx.x; i < ns * mmax * B; i += blockDim.x) ys[i] = ysg[i];
  __syncthreads();
  const int64_t a0 = (int64_t)blockIdx.x * CT;
  const int npairs = (int)(n - a0 < (int64_t)CT ? n - a0 : (int64_t)CT) * B;
  for (int idx = threadIdx.x; idx < npairs; idx += blockDim.x) {
    const int c = idx / B, b = idx - c * B;
    const int64_t a = a0 + c;
    double2 u[MAXM];
#pragma unroll
    for (int j = 0; j < MAXM; ++j) u[j] = j < mmax ? Ucols[j][(int64_t)b * n + a] : make_double2(0.0, 0.0);
    double2* o = out + a0 * B + idx;
    for (int k = 0; k < ns; ++k) {
      const double2* yk = ys + (k * mmax) * B + b;
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < MAXM; ++j)
        if (j < mmax) acc = cfma(yk[j * B], u[j], acc);
      o[(int64_t)k * n * B] = acc;
    }
  }
}

}  // namespace

void outer_solve(lt_pencil p, const OuterProblem& prob, OuterResult& res) {
  p->ctx->mem_probe_valid = false;  // re-read the device's free memory once per outer solve
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int B = prob.B, ns = prob.n_shifts;
  const int64_t n = p->n;
  const int nblk = (int)blocks_for(n, kT);
  const int maxit = prob.maxit > 0 ? (int)std::min<int64_t>(n, prob.maxit) : (int)std::min<int64_t>(n, 10 * (int64_t)ns);
  res.B = B;
  res.n_shifts = ns;
  res.maxit = maxit;
  res.iterations.assign(B, 0);
  res.status.assign((size_t)B * ns, lt_shift_status{0, 0, INFINITY, NAN});
  res.m_used.assign((size_t)B * ns, 0);
  res.U.clear();
  if (prob.record_history) res.history.assign((size_t)B * ns * maxit, NAN);
  if (B == 0 || ns == 0) return;

  // ---- device state ----
  int cap = std::min(maxit, 8);
  const size_t n_bs = (size_t)B * ns;
  DeviceBuffer dH(sizeof(double2) * (size_t)B * maxit * (maxit + 1), st);
  LT_CUDA(cudaMemsetAsync(dH.get(), 0, dH.bytes(), st));
  DeviceBuffer dTaus(sizeof(double2) * (size_t)B * maxit, st);
  DeviceBuffer dShifts(sizeof(double2) * n_bs, st);
  DeviceBuffer dY(sizeof(double2) * n_bs * maxit, st);
  LT_CUDA(cudaMemsetAsync(dY.get(), 0, dY.bytes(), st));
  DeviceBuffer dHist(prob.record_history ? sizeof(double) * n_bs * maxit : 8, st);
  DeviceBuffer ints(sizeof(int) * (n_bs * 4 + (size_t)B * 5), st);
  DeviceBuffer dbls(sizeof(double) * (n_bs * 3 + (size_t)B * 4), st);
  int* conv = ints.as<int>();
  int* iter = conv + n_bs;
  int* flag = iter + n_bs;
  int* m_used = flag + n_bs;
  int* active = m_used + n_bs;
  int* reorth = active + B;
  int* brk = reorth + B;
  int* n_unconv = brk + B;
  double* est = dbls.as<double>();
  double* true_res = est + n_bs;
  double* verify_at = true_res + n_bs;
  double* beta = verify_at + n_bs;
  double* norm0 = beta + B;
  double* norm1 = norm0 + B;
  double* hnext = norm1 + B;
  LT_CUDA(cudaMemsetAsync(ints.get(), 0, ints.bytes(), st));
  {
    std::vector<double> init(n_bs * 3);
    for (size_t t = 0; t < n_bs; ++t) {
      init[t] = INFINITY;
      init[n_bs + t] = NAN;
      init[2 * n_bs + t] = prob.tol;
    }
    LT_CUDA(cudaMemcpyAsync(est, init.data(), sizeof(double) * n_bs * 3, cudaMemcpyHostToDevice, st));
    std::vector<double2> taus((size_t)B * maxit);
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < maxit; ++j) taus[(size_t)b * maxit + j] = prob.tau_table[b][j];
    LT_CUDA(cudaMemcpyAsync(dTaus.get(), taus.data(), sizeof(double2) * taus.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dShifts.get(), prob.shifts.data(), sizeof(double2) * n_bs, cudaMemcpyHostToDevice, st));
    if (prob.record_history) {
      std::vector<double> h(n_bs * maxit, NAN);
      LT_CUDA(cudaMemcpyAsync(dHist.get(), h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, st));
    }
  }
  DeviceBuffer dScratch(sizeof(double2) * n_bs * (cap + 1) * cap, st);
  DeviceBuffer dColPtr(sizeof(void*) * (maxit + 1) * 2, st);
  const double2** dVcols = dColPtr.as<const double2*>();
  const double2** dUcols = dVcols + (maxit + 1);
  std::vector<DeviceBuffer> Vc;
  std::vector<const double2*> vptr, uptr;
  auto add_v = [&]() {
    Vc.emplace_back(sizeof(double2) * (size_t)B * n, st);
    vptr.push_back(Vc.back().as<double2>());
  };
  auto add_u = [&]() {
    res.U.emplace_back(sizeof(double2) * (size_t)B * n, st);
    uptr.push_back(res.U.back().as<double2>());
  };
  DeviceBuffer partials;
  DeviceBuffer hcoef(sizeof(double2) * (size_t)B * (maxit + 1), st);

  State S{};
  S.B = B; S.ns = ns; S.maxit = maxit; S.cap = cap; S.n = n; S.nblk = nblk;
  S.nblk_tile = verify_blocks(p->view(0));
  S.tol = prob.tol; S.variant = prob.variant; S.record_history = prob.record_history;
  S.active = active; S.beta = beta; S.shifts = dShifts.as<double2>(); S.taus = dTaus.as<double2>();
  S.H = dH.as<double2>(); S.conv = conv; S.iter = iter; S.est = est; S.true_res = true_res;
  S.verify_at = verify_at; S.flag = flag; S.m_used = m_used; S.Y = dY.as<double2>();
  S.history = prob.record_history ? dHist.as<double>() : nullptr; S.scratch = dScratch.as<double2>();
  S.norm0 = norm0; S.norm1 = norm1; S.reorth = reorth; S.breakdown = brk; S.hnext = hnext; S.n_unconv = n_unconv;

  const unsigned grid = (unsigned)nblk * (unsigned)B;
  const double nb = (double)n * B;
  LevelView L0 = p->view(0);

  // beta = ||b||, v0 = b / beta
  partials.ensure(sizeof(double2) * (size_t)B * nblk * 2, st);
  launch(ctx, "fgmres_vec", nb * 16.0, [&] { norm_kernel<<<grid, kT, 0, st>>>(n, B, prob.b, partials.as<double>(), nblk); });
  launch(ctx, "fgmres_small", 0.0, [&] { reduce_beta<<<B, kT, 0, st>>>(B, nblk, partials.as<double>(), beta); });
  add_v();
  launch(ctx, "fgmres_vec", nb * 32.0, [&] { scale_to<<<grid, kT, 0, st>>>(n, B, prob.b, beta, Vc[0].as<double2>()); });
  launch(ctx, "fgmres_small", 0.0, [&] { outer_init<<<blocks_for(n_bs, 128), 128, 0, st>>>(S); });

  // Per outer iteration the host reads the active flags once (one small copy, after the
  // iteration's last kernel): the next inner solve runs on the active items only, packed into a
  // dense batch, so the two-items-per-CTA kernels never pair a live item with a finished one.
  // The inner COCG loop itself is device-resident (inner.cu).
  DeviceBuffer dIter(sizeof(int) * B, st);
  LT_CUDA(cudaMemsetAsync(dIter.get(), 0, sizeof(int) * B, st));
  int* d_iterations = dIter.as<int>();
  std::vector<int> h_active(B, 0);
  LT_CUDA(cudaMemcpyAsync(h_active.data(), active, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  stream_sync(ctx);
  std::vector<double2> taus_j(B);
  DeviceBuffer gather_v, gather_u, gather_idx;
  for (int j = 0; j < maxit; ++j) {
    int n_active = 0;
    for (int b = 0; b < B; ++b) n_active += h_active[b];
    if (n_active == 0) break;
    if (j >= cap) {
      const int new_cap = std::min(maxit, 2 * cap);
      dScratch.allocate(sizeof(double2) * n_bs * (new_cap + 1) * new_cap, st);
      cap = new_cap;
      S.cap = cap;
      S.scratch = dScratch.as<double2>();
    }
    // 1. u_j = (K + tau_j M)^{-1} v_j  for the active items
    add_u();
    LT_CUDA(cudaMemcpyAsync(dUcols + j, &uptr[j], sizeof(void*), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dVcols + j, &vptr[j], sizeof(void*), cudaMemcpyHostToDevice, st));
    double2* Uj = const_cast<double2*>(uptr[j]);
    const double2* Vj = vptr[j];
    if (n_active == B) {
      for (int b = 0; b < B; ++b) taus_j[b] = prob.tau_table[b][j];
      inner_solve(p, B, taus_j.data(), Vj, n, Uj, n);
    } else {
      // pack the active items' v_j, solve, scatter u_j back (one launch each way)
      std::vector<int> idx;
      for (int b = 0; b < B; ++b)
        if (h_active[b]) {
          taus_j[idx.size()] = prob.tau_table[b][j];
          idx.push_back(b);
        }
      gather_v.ensure(sizeof(double2) * (size_t)n_active * n, st);
      gather_u.ensure(sizeof(double2) * (size_t)n_active * n, st);
      gather_idx.ensure(sizeof(int) * B, st);
      LT_CUDA(cudaMemcpyAsync(gather_idx.get(), idx.data(), sizeof(int) * n_active, cudaMemcpyHostToDevice, st));
      const dim3 g2((unsigned)nblk, (unsigned)n_active);
      launch(ctx, "fgmres_vec", (double)n * n_active * 32.0, [&] {
        pack_items<<<g2, kT, 0, st>>>(n, gather_idx.as<int>(), Vj, gather_v.as<double2>(), 0);
      });
      inner_solve(p, n_active, taus_j.data(), gather_v.as<double2>(), n, gather_u.as<double2>(), n);
      launch(ctx, "fgmres_vec", (double)n * n_active * 32.0, [&] {
        pack_items<<<g2, kT, 0, st>>>(n, gather_idx.as<int>(), gather_u.as<double2>(), Uj, 1);
      });
    }
    // 2. s = M u_j into V_{j+1}; Gram-Schmidt with conditional re-orthogonalisation
    add_v();
    LT_CUDA(cudaMemcpyAsync(dVcols + j + 1, &vptr[j + 1], sizeof(void*), cudaMemcpyHostToDevice, st));
    double2* s = const_cast<double2*>(vptr[j + 1]);
    partials.ensure(sizeof(double2) * (size_t)B * (j + 2) * nblk, st);
    // bytes are charged for the items still iterating (the others' blocks exit at once)
    const double nba = (double)n * n_active;
    launch(ctx, "fgmres_orth:mass_multidot", nba * (16.0 * (j + 3)) + n * 8.0, [&] {
      if (p->dim == 3)
        mass_multidot<3><<<grid, kT, 0, st>>>(L0, S, j, Uj, s, dVcols, partials.as<double2>());
      else
        mass_multidot<2><<<grid, kT, 0, st>>>(L0, S, j, Uj, s, dVcols, partials.as<double2>());
    });
    launch(ctx, "fgmres_small", 0.0, [&] {
      reduce_dots<<<B * (j + 2), kT, 0, st>>>(S, j, partials.as<double2>(), 0, hcoef.as<double2>());
    });
    launch(ctx, "fgmres_orth:gs_update", nba * (16.0 * (j + 3)), [&] {
      gs_update<<<grid, kT, 0, st>>>(S, j, 0, s, dVcols, hcoef.as<double2>(), partials.as<double>());
    });
    launch(ctx, "fgmres_small", 0.0, [&] { reduce_norm<<<B, kT, 0, st>>>(S, j, 0, partials.as<double>()); });
    // re-orthogonalisation pass (items whose norm dropped by more than 1/sqrt(2))
    launch(ctx, "fgmres_orth:multidot", 0.0, [&] { multidot<<<grid, kT, 0, st>>>(S, j, s, dVcols, partials.as<double2>()); });
    launch(ctx, "fgmres_small", 0.0, [&] {
      reduce_dots<<<B * (j + 2), kT, 0, st>>>(S, j, partials.as<double2>(), 1, hcoef.as<double2>());
    });
    launch(ctx, "fgmres_orth:gs_update", 0.0, [&] {
      gs_update<<<grid, kT, 0, st>>>(S, j, 1, s, dVcols, hcoef.as<double2>(), partials.as<double>());
    });
    launch(ctx, "fgmres_small", 0.0, [&] { reduce_norm<<<B, kT, 0, st>>>(S, j, 1, partials.as<double>()); });
    launch(ctx, "fgmres_vec", nba * 32.0, [&] { normalize<<<grid, kT, 0, st>>>(S, s); });
    const int m = j + 1;
    // 3. per-shift small solves, verification, freeze
    launch(ctx, "fgmres_small", 0.0, [&] { small_solve<<<blocks_for(n_bs, 128), 128, 0, st>>>(S, m, 0); });
    partials.ensure(sizeof(double) * n_bs * std::max(nblk, S.nblk_tile), st);
    launch(ctx, "fgmres_verify:verify_residual", nba * (16.0 * (m + 1)) + n * 8.0 * (p->dim + 1), [&] {
      launch_verify(p, L0, S, m, prob.b, dUcols, partials.as<double>(), B, st);
    });
    launch(ctx, "fgmres_small", 0.0, [&] { verify_finalize<<<(unsigned)n_bs, kT, 0, st>>>(S, m, partials.as<double>(), 0); });
    launch(ctx, "fgmres_small", 0.0, [&] {
      outer_control<<<1, 256, 0, st>>>(S, m, d_iterations);
    });
    LT_CUDA(cudaMemcpyAsync(h_active.data(), active, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
    stream_sync(ctx);
  }
  std::vector<double> h_beta(B);
  std::vector<int> h_brk(B, 0), h_unconv(B, 0);
  LT_CUDA(cudaMemcpyAsync(h_beta.data(), beta, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(res.iterations.data(), d_iterations, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_unconv.data(), n_unconv, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_brk.data(), brk, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  stream_sync(ctx);
  int m_global = 0;
  for (int b = 0; b < B; ++b) m_global = std::max(m_global, res.iterations[b]);
  res.cap = maxit;

  // best-effort iterates for unconverged shifts (cpp:270-285), at each item's own m
  bool any_unconv = false;
  for (int b = 0; b < B; ++b) any_unconv |= (h_unconv[b] > 0 && res.iterations[b] > 0);
  if (any_unconv && m_global > 0) {
    // items may have stopped at different m; run per distinct m
    std::vector<int> ms;
    for (int b = 0; b < B; ++b)
      if (h_unconv[b] > 0 && res.iterations[b] > 0) ms.push_back(res.iterations[b]);
    std::sort(ms.begin(), ms.end());
    ms.erase(std::unique(ms.begin(), ms.end()), ms.end());
    for (int m : ms) {
      std::vector<int> act(B, 0);
      for (int b = 0; b < B; ++b) act[b] = (h_unconv[b] > 0 && res.iterations[b] == m);
      LT_CUDA(cudaMemcpyAsync(active, act.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
      launch(ctx, "fgmres_small", 0.0, [&] { small_solve<<<blocks_for(n_bs, 128), 128, 0, st>>>(S, m, 1); });
      // restrict flags to the items of this m
      launch(ctx, "fgmres_verify:verify_residual", 0.0, [&] {
        launch_verify(p, L0, S, m, prob.b, dUcols, partials.as<double>(), B, st);
      });
      launch(ctx, "fgmres_small", 0.0, [&] { verify_finalize<<<(unsigned)n_bs, kT, 0, st>>>(S, m, partials.as<double>(), 1); });
    }
  }

  // ---- read back status ----
  std::vector<int> h_conv(n_bs), h_iter(n_bs), h_mu(n_bs);
  std::vector<double> h_est(n_bs), h_true(n_bs);
  LT_CUDA(cudaMemcpyAsync(h_conv.data(), conv, sizeof(int) * n_bs, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_iter.data(), iter, sizeof(int) * n_bs, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_mu.data(), m_used, sizeof(int) * n_bs, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_est.data(), est, sizeof(double) * n_bs, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaMemcpyAsync(h_true.data(), true_res, sizeof(double) * n_bs, cudaMemcpyDeviceToHost, st));
  if (prob.record_history)
    LT_CUDA(cudaMemcpyAsync(res.history.data(), dHist.get(), sizeof(double) * n_bs * maxit, cudaMemcpyDeviceToHost, st));
  stream_sync(ctx);
  for (size_t t = 0; t < n_bs; ++t) {
    res.status[t] = lt_shift_status{h_conv[t], h_iter[t], h_est[t], h_true[t]};
    res.m_used[t] = h_mu[t];
  }
  res.Y = std::move(dY);
  // column pointers for expand_solutions
  res.cap = maxit;

  if (prob.keep_basis) {
    KeptBasis& kb = p->kept;
    kb.n_rhs = B;
    kb.steps = res.iterations;
    kb.beta = h_beta;
    kb.V.assign(B, {});
    kb.U.assign(B, {});
    kb.H.assign(B, {});
    kb.taus.assign(B, {});
    std::vector<double2> hH((size_t)B * maxit * (maxit + 1));
    LT_CUDA(cudaMemcpyAsync(hH.data(), dH.get(), sizeof(double2) * hH.size(), cudaMemcpyDeviceToHost, st));
    stream_sync(ctx);
    for (int b = 0; b < B; ++b) {
      const int m = res.iterations[b];
      kb.V[b].assign((size_t)n * (m + 1), make_double2(0, 0));
      kb.U[b].assign((size_t)n * m, make_double2(0, 0));
      for (int jj = 0; jj <= m; ++jj) {
        if (jj == m && h_brk[b]) break;  // V(:, m) zeroed on breakdown (cpp:259)
        LT_CUDA(cudaMemcpyAsync(kb.V[b].data() + (size_t)jj * n, vptr[jj] + (size_t)b * n, sizeof(double2) * n,
                                cudaMemcpyDeviceToHost, st));
      }
      for (int jj = 0; jj < m; ++jj)
        LT_CUDA(cudaMemcpyAsync(kb.U[b].data() + (size_t)jj * n, uptr[jj] + (size_t)b * n, sizeof(double2) * n,
                                cudaMemcpyDeviceToHost, st));
      kb.H[b].assign((size_t)(m + 1) * m, make_double2(0, 0));
      for (int jj = 0; jj < m; ++jj)
        for (int i = 0; i <= m; ++i) kb.H[b][(size_t)jj * (m + 1) + i] = hH[((size_t)b * maxit + jj) * (maxit + 1) + i];
      kb.taus[b].assign(prob.tau_table[b].begin(), prob.tau_table[b].begin() + m);
    }
    stream_sync(ctx);
  }
}

void expand_solutions(lt_pencil p, const OuterResult& res, const double2* scale_dev, double2* x_out, bool cell_major) {
  const int ncols = (int)res.U.size();
  std::vector<const double2*> cols(std::max(ncols, 1), nullptr);
  for (int j = 0; j < ncols; ++j) cols[j] = res.U[j].as<double2>();
  expand_raw(p->ctx, p->n, res.B, res.n_shifts, cols, res.Y.as<double2>(), res.maxit, res.m_used, scale_dev, x_out,
             cell_major);
}

void expand_raw(lt_ctx ctx, int64_t n, int B, int ns, const std::vector<const double2*>& cols, const double2* Y,
                int ystride, const std::vector<int>& m_used, const double2* scale_dev, double2* x_out, bool cell_major) {
  cudaStream_t st = ctx->stream;
  if (B == 0 || ns == 0) return;
  const int ncols = (int)cols.size();
  DeviceBuffer dcols(sizeof(void*) * cols.size(), st);
  DeviceBuffer dmu(sizeof(int) * m_used.size(), st);
  LT_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(void*) * cols.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dmu.get(), m_used.data(), sizeof(int) * m_used.size(), cudaMemcpyHostToDevice, st));
  const int nblk = (int)blocks_for(n, kT);
  int mmax = 0;
  for (int v : m_used) mmax = std::max(mmax, v);
  constexpr int kCT = 32;
  const size_t ys_bytes = sizeof(double2) * (size_t)ns * std::max(mmax, 1) * B;
  // cell-major v2 (coefficients staged in shared memory) up to 8 basis columns; the v1 kernel
  // (per-shift shared-memory transpose) for longer bases
  if (cell_major && mmax >= 1 && mmax <= 8 && mmax <= ncols && ys_bytes <= 110 * 1024) {
    DeviceBuffer ys(ys_bytes, st);
    const int ny = ns * mmax * B;
    expand_coeffs<<<(unsigned)((ny + 255) / 256), 256, 0, st>>>(B, ns, ystride, mmax, Y,
                                                                 dmu.as<int>(), scale_dev, ys.as<double2>());
    auto fn = mmax <= 4 ? expand_cm2_kernel<4> : expand_cm2_kernel<8>;
    LT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ys_bytes));
    launch(ctx, "expand", (double)n * B * 16.0 * (mmax + ns), [&] {
      fn<<<(unsigned)((n + kCT - 1) / kCT), 256, ys_bytes, st>>>(n, B, ns, mmax, kCT, dcols.as<const double2*>(),
                                                                  ys.as<double2>(), x_out);
    });
    stream_sync(ctx);
    return;
  }
  launch(ctx, "expand", (double)n * B * 16.0 * (ncols + ns), [&] {
    if (cell_major)
      expand_cm_kernel<<<dim3((unsigned)((n + 31) / 32), (unsigned)((B + 7) / 8)), 256, 0, st>>>(
          n, B, ns, ystride, dcols.as<const double2*>(), Y, dmu.as<int>(), scale_dev, x_out);
    else
      expand_kernel<<<(unsigned)nblk * B, kT, 0, st>>>(n, B, ns, ystride, dcols.as<const double2*>(),
                                                        Y, dmu.as<int>(), scale_dev, x_out);
  });
  stream_sync(ctx);
}

}  // namespace lt
