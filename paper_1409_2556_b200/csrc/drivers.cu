// Physics drivers on the device: per-time contour forward solves (solve_forward /
// solve_forward_batch, forward.cpp:75-198), quadrature recombination in basis form
// (phi(t) = 2 Re U c, c_j = sum_k w_k qhat_k y_kj; talbot.cpp:82-94 + forward.cpp:104-115),
// adjoint solves (jacobian.cpp:47-55) and the adjoint-state Jacobian assembly
// (sensitivity_row_conductivity / _storativity, jacobian.cpp:57-125, FD form of SURVEY
// App. A) for all source/receiver pairs of a time slice.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "drivers.hpp"
#include "lt_internal.hpp"
#include "stencil.cuh"
#include "talbot_host.hpp"

namespace lt {

thread_local std::vector<int> g_last_unconverged;

namespace {

constexpr int kT = 256;
using cd = std::complex<double>;

inline double2 d2(cd c) { return make_double2(c.real(), c.imag()); }

// heads[dst[b] + a] += 2 Re sum_j c[b][j] U_j[b][a]   (dst[b] < 0: item skipped)
__global__ void __launch_bounds__(kT) recombine_kernel(int64_t n, int B, int mc, const double2* const* __restrict__ Ucols,
                                                       const double2* __restrict__ c, const int64_t* __restrict__ dst,
                                                       double* __restrict__ heads) {
  LT_ITEM_BLOCK(B, b, cb);
  const int64_t a = (int64_t)cb * blockDim.x + threadIdx.x;
  if (a >= n || dst[b] < 0) return;
  double s = 0.0;
  for (int j = 0; j < mc; ++j) {
    const double2 cj = c[b * mc + j];
    const double2 u = Ucols[j][b * n + a];
    s += cj.x * u.x - cj.y * u.y;
  }
  heads[dst[b] + a] += 2.0 * s;
}

// drawdown[b][r] = sum_q w_q heads[b][idx_q]
__global__ void gather_points(int64_t n, int B, int n_pts, const double* __restrict__ heads, const int64_t* __restrict__ idx,
                              const double* __restrict__ w, const int* __restrict__ cnt, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B * n_pts) return;
  const int b = t / n_pts, r = t % n_pts;
  double s = 0.0;
  for (int q = 0; q < cnt[r]; ++q) s += w[r * 8 + q] * heads[b * n + idx[r * 8 + q]];
  out[t] = s;
}

// predictions[s][r] = 2 Re sum_k w_k sum_q wq phi_{s,k}[idx_q]
__global__ void predict_kernel(int64_t n, int n_src, int n_rec, int ns, const double2* __restrict__ fields,
                               const double2* __restrict__ w, const int64_t* __restrict__ idx, const double* __restrict__ wt,
                               const int* __restrict__ cnt, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_src * n_rec) return;
  const int s = t / n_rec, r = t % n_rec;
  double2 acc = make_double2(0.0, 0.0);
  for (int k = 0; k < ns; ++k) {
    const double2* f = fields + ((int64_t)s * ns + k) * n;
    double2 v = make_double2(0.0, 0.0);
    for (int q = 0; q < cnt[r]; ++q) v = cadd(v, cscale(f[idx[r * 8 + q]], wt[r * 8 + q]));
    acc = cadd(acc, cmul(w[k], v));
  }
  out[t] = 2.0 * acc.x;
}

// rhs[item*n + idx] += w for the sparse point weights of each item (zeroed beforehand)
__global__ void scatter_points(int64_t n, int n_items, const int64_t* __restrict__ idx, const double* __restrict__ w,
                               const int* __restrict__ cnt, double2* __restrict__ rhs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_items * 8) return;
  const int it = t / 8, q = t % 8;
  if (q >= cnt[it]) return;
  rhs[(int64_t)it * n + idx[it * 8 + q]].x += w[it * 8 + q];
}

__global__ void real_to_complex(int64_t n, const double* __restrict__ x, double2* __restrict__ y) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) y[a] = make_double2(x[a], 0.0);
}

// ---- Jacobian assembly -----------------------------------------------------------------
// J_k[(s,r), a] = 2 Re sum_k w_k sum_{f in faces(a)} dT_f/dln k_a (phi_a - phi_b)(psi_a - psi_b)
// J_S[(s,r), a] = 2 Re sum_k w_k z_k^p S_a h^d phi_a psi_a
// A CTA owns TC consecutive cells of one row and all (source-block x receiver-block)
// register tiles.  Per shift k, every field value at the tile (centre) and its 2d face
// neighbours is loaded once, the 2d weighted face differences and the storativity term of
// all sources (P) and receivers (Q) are staged in shared memory, and every thread
// accumulates its SB x RB tile of Re(P Q) for one cell over the 2d+1 stages.
constexpr int SB = 4;
constexpr int RB = 8;

template <int DIM>
__global__ void __launch_bounds__(kT, 2) jacobian_kernel(LevelView L, const double* __restrict__ kappa,
                                                      const double* __restrict__ stor, double hd, double face_scale,
                                                      const double2* __restrict__ fields, int n_src, int n_rec, int ns,
                                                      const double2* __restrict__ w, const double2* __restrict__ wz,
                                                      int TC, int tiles_x, int nsub_r, int nsub_total,
                                                      double* __restrict__ Jk, double* __restrict__ Js, int64_t ldj) {
  constexpr int NF = 2 * DIM + 1;  // faces + storativity stage
  extern __shared__ double2 smem[];
  const int n_items = n_src + n_rec;
  double2* P = smem;                                    // [2 DIM][n_src][TC]
  double2* Q = smem + (size_t)2 * DIM * n_src * TC;     // [2 DIM][n_rec][TC]
  double* wt = reinterpret_cast<double*>(Q + (size_t)2 * DIM * n_rec * TC);  // [NF][TC]
  int64_t* nb = reinterpret_cast<int64_t*>(wt + NF * TC);             // [2 DIM][TC] neighbour index or -1
  const int64_t n = L.n;
  // tile -> (row, x offset); cells of one tile are consecutive in x
  const int tile = blockIdx.x;
  const int tx = tile % tiles_x;
  const int64_t row = tile / tiles_x;  // k * ny + j
  const int i0 = tx * TC;
  const int ncell = min(TC, L.nx - i0);
  const int64_t a0 = row * L.nx + i0;
  const int j = (int)(row % L.ny);
  const int kz = (int)(row / L.ny);
  const int tid = threadIdx.x;
  const int c = tid % TC;
  const int sub = tid / TC;
  const bool owner = sub < nsub_total && c < ncell;
  const int s0 = owner ? (sub / nsub_r) * SB : 0;
  const int r0 = owner ? (sub % nsub_r) * RB : 0;

  if (tid < NF * TC) {
    const int f = tid / TC, cc = tid % TC;
    double wv = 0.0;
    int64_t nbi = -1;
    if (cc < ncell) {
      const int64_t a = a0 + cc;
      if (f == 2 * DIM) {
        wv = stor[a] * hd;
      } else {
        const int d = f >> 1, hi = f & 1;
        const int coord = d == 0 ? i0 + cc : (d == 1 ? j : kz);
        const int ext = d == 0 ? L.nx : (d == 1 ? L.ny : L.nz);
        const int64_t stride = d == 0 ? 1 : (d == 1 ? (int64_t)L.nx : (int64_t)L.nx * L.ny);
        const double ka = kappa[a];
        const bool boundary = hi ? coord == ext - 1 : coord == 0;
        if (boundary) {
          wv = 2.0 * ka * face_scale;  // dT/dln k_a = T = 2 k_a h^(d-2); ghost value 0
        } else {
          nbi = hi ? a + stride : a - stride;
          const double kb = kappa[nbi];
          const double T = 2.0 * ka * kb / (ka + kb) * face_scale;
          wv = T * kb / (ka + kb);
        }
      }
    }
    wt[f * TC + cc] = wv;
    if (f < 2 * DIM) nb[f * TC + cc] = nbi;
  }

  __syncthreads();
  // phase 0: kappa block over the 2d face stages; phase 1: storativity block (centre stage).
  // Two phases keep one SB x RB accumulator tile per thread (2 CTAs per SM).
  for (int phase = 0; phase < (Js ? 2 : 1); ++phase) {
    double acc[SB][RB];
#pragma unroll
    for (int i = 0; i < SB; ++i)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[i][q] = 0.0;
    const int nstage = phase == 0 ? 2 * DIM : 1;
    for (int k = 0; k < ns; ++k) {
      const double2 wk = w[k], wzk = wz[k];
      // stage: one centre (+ 2d neighbour) loads per (item, cell)
      for (int e = tid; e < n_items * TC; e += blockDim.x) {
        const int it = e / TC, cc = e % TC;
        const double2* fld = fields + ((int64_t)it * ns + k) * n;
        const double2 fa = cc < ncell ? fld[a0 + cc] : make_double2(0.0, 0.0);
        if (phase == 0) {
          double2 fn[2 * DIM];
#pragma unroll
          for (int f = 0; f < 2 * DIM; ++f) {
            const int64_t q = cc < ncell ? nb[f * TC + cc] : -1;
            fn[f] = q >= 0 ? fld[q] : make_double2(0.0, 0.0);
          }
          if (it < n_src) {
#pragma unroll
            for (int f = 0; f < 2 * DIM; ++f)
              P[((size_t)f * n_src + it) * TC + cc] = cscale(cmul(wk, csub(fa, fn[f])), wt[f * TC + cc]);
          } else {
            const int r = it - n_src;
#pragma unroll
            for (int f = 0; f < 2 * DIM; ++f) Q[((size_t)f * n_rec + r) * TC + cc] = csub(fa, fn[f]);
          }
        } else {
          if (it < n_src) P[(size_t)it * TC + cc] = cscale(cmul(wzk, fa), wt[2 * DIM * TC + cc]);
          else Q[(size_t)(it - n_src) * TC + cc] = fa;
        }
      }
      __syncthreads();
      if (owner) {
#pragma unroll 1
        for (int f = 0; f < nstage; ++f) {
          double2 pv[SB];
#pragma unroll
          for (int i = 0; i < SB; ++i)
            pv[i] = (s0 + i < n_src) ? P[((size_t)f * n_src + s0 + i) * TC + c] : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const double2 qv = (r0 + q < n_rec) ? Q[((size_t)f * n_rec + r0 + q) * TC + c] : make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < SB; ++i) acc[i][q] = fma(pv[i].x, qv.x, fma(-pv[i].y, qv.y, acc[i][q]));
          }
        }
      }
      __syncthreads();
    }
    if (owner) {
      double* Jout = phase == 0 ? Jk : Js;
      const int64_t a = a0 + c;
#pragma unroll
      for (int i = 0; i < SB; ++i) {
        if (s0 + i >= n_src) continue;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          if (r0 + q >= n_rec) continue;
          const int64_t rowj = (int64_t)(s0 + i) * n_rec + (r0 + q);
          Jout[rowj * ldj + a] = 2.0 * acc[i][q];
        }
      }
    }
  }
}

// P1 rows (sensitivity_row_conductivity / _storativity, jacobian.cpp:57-125) on the node
// grid of build_mesh: per element e (2c lower (a,b,c), 2c+1 upper (a,c,d) of cell c)
//   J_k[e] = 2 Re sum_k w_k (kappa_e / 2) (D0 phi D0 psi + D1 phi D1 psi)
//     (exact P1 gradients: area h^2/2, grad = edge differences / h)
//   J_S[e] = 2 Re sum_k w_k z_k (S_e h^2 / 24) ((sum phi)(sum psi) + sum_i phi_i psi_i)
//     (exact P1 product integral area/12 sum (1 + d_ij) phi_i psi_j)
// Dirichlet nodes carry zero.  A CTA owns TC cells (2 TC elements) of one row.
__global__ void __launch_bounds__(kT, 2) jacobian_p1_kernel(int nx, double h2, const double* __restrict__ kappa,
                                                            const double* __restrict__ stor,
                                                            const double2* __restrict__ fields, int n_src, int n_rec,
                                                            int ns, const double2* __restrict__ w,
                                                            const double2* __restrict__ wz, int TC, int tiles_x,
                                                            int nsub_r, int nsub_total, double* __restrict__ Jk,
                                                            double* __restrict__ Js, int64_t ldj) {
  extern __shared__ double2 smem[];
  const int n_items = n_src + n_rec;
  const int U = 2 * TC;                                  // elements per tile
  double2* P = smem;                                     // [4][n_src][U]
  double2* Q = smem + (size_t)4 * n_src * U;             // [4][n_rec][U]
  double* wt = reinterpret_cast<double*>(Q + (size_t)4 * n_rec * U);  // [2][U]: kappa_e/2, S_e h^2/24
  const int nc = nx + 1;
  const int64_t n = (int64_t)nx * nx;
  const int cj = blockIdx.x / tiles_x;
  const int ci0 = (blockIdx.x % tiles_x) * TC;
  const int ncell = min(TC, nc - ci0);
  const int tid = threadIdx.x;
  const int c = tid % U;
  const int sub = tid / U;
  const bool owner = sub < nsub_total && (c >> 1) < ncell;
  const int s0 = owner ? (sub / nsub_r) * SB : 0;
  const int r0 = owner ? (sub % nsub_r) * RB : 0;
  if (tid < U) {
    const int ci = ci0 + (tid >> 1);
    const int64_t e = 2 * ((int64_t)cj * nc + ci) + (tid & 1);
    wt[tid] = (tid >> 1) < ncell ? 0.5 * kappa[e] : 0.0;
    wt[U + tid] = (tid >> 1) < ncell ? stor[e] * h2 / 24.0 : 0.0;
  }
  __syncthreads();
  auto nodev = [&](const double2* fld, int I, int J) {
    return (I >= 1 && I <= nx && J >= 1 && J <= nx) ? fld[(int64_t)(J - 1) * nx + (I - 1)] : make_double2(0.0, 0.0);
  };
  for (int phase = 0; phase < (Js ? 2 : 1); ++phase) {
    const int nstage = phase == 0 ? 2 : 4;
    double acc[SB][RB];
#pragma unroll
    for (int i = 0; i < SB; ++i)
#pragma unroll
      for (int q = 0; q < RB; ++q) acc[i][q] = 0.0;
    for (int k = 0; k < ns; ++k) {
      const double2 wk = phase == 0 ? w[k] : wz[k];
      for (int e = tid; e < n_items * TC; e += blockDim.x) {
        const int it = e / TC, cc = e % TC;
        double2 v[2][4];
        if (cc < ncell) {
          const double2* fld = fields + ((int64_t)it * ns + k) * n;
          const int ci = ci0 + cc;
          const double2 fa = nodev(fld, ci, cj), fb = nodev(fld, ci + 1, cj);
          const double2 fc = nodev(fld, ci + 1, cj + 1), fd = nodev(fld, ci, cj + 1);
          if (phase == 0) {
            v[0][0] = csub(fb, fa); v[0][1] = csub(fc, fb);  // lower (a, b, c)
            v[1][0] = csub(fc, fd); v[1][1] = csub(fd, fa);  // upper (a, c, d)
          } else {
            v[0][0] = cadd(cadd(fa, fb), fc); v[0][1] = fa; v[0][2] = fb; v[0][3] = fc;
            v[1][0] = cadd(cadd(fa, fc), fd); v[1][1] = fa; v[1][2] = fc; v[1][3] = fd;
          }
        } else {
          for (int q = 0; q < 4; ++q) v[0][q] = v[1][q] = make_double2(0.0, 0.0);
        }
        for (int el = 0; el < 2; ++el) {
          const int u = 2 * cc + el;
          for (int f = 0; f < nstage; ++f) {
            if (it < n_src) P[((size_t)f * n_src + it) * U + u] = cscale(cmul(wk, v[el][f]), wt[phase * U + u]);
            else Q[((size_t)f * n_rec + (it - n_src)) * U + u] = v[el][f];
          }
        }
      }
      __syncthreads();
      if (owner) {
#pragma unroll 1
        for (int f = 0; f < nstage; ++f) {
          double2 pv[SB];
#pragma unroll
          for (int i = 0; i < SB; ++i)
            pv[i] = (s0 + i < n_src) ? P[((size_t)f * n_src + s0 + i) * U + c] : make_double2(0.0, 0.0);
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const double2 qv = (r0 + q < n_rec) ? Q[((size_t)f * n_rec + r0 + q) * U + c] : make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < SB; ++i) acc[i][q] = fma(pv[i].x, qv.x, fma(-pv[i].y, qv.y, acc[i][q]));
          }
        }
      }
      __syncthreads();
    }
    if (owner) {
      double* Jout = phase == 0 ? Jk : Js;
      const int64_t e = 2 * ((int64_t)cj * nc + ci0 + (c >> 1)) + (c & 1);
#pragma unroll
      for (int i = 0; i < SB; ++i) {
        if (s0 + i >= n_src) continue;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          if (r0 + q >= n_rec) continue;
          Jout[((int64_t)(s0 + i) * n_rec + (r0 + q)) * ldj + e] = 2.0 * acc[i][q];
        }
      }
    }
  }
}

struct PointSet {
  std::vector<int64_t> idx;  // n_pts * 8
  std::vector<double> w;
  std::vector<int> cnt;
};

PointSet make_points(lt_pencil p, const double* pts, int n_pts) {
  PointSet ps;
  ps.idx.assign((size_t)n_pts * 8, 0);
  ps.w.assign((size_t)n_pts * 8, 0.0);
  ps.cnt.assign(n_pts, 0);
  for (int r = 0; r < n_pts; ++r)
    point_weights(p, pts + (size_t)r * p->dim, ps.idx.data() + r * 8, ps.w.data() + r * 8, &ps.cnt[r]);
  return ps;
}

void throw_unconverged(const OuterResult& res, const char* what) {
  for (int b = 0; b < res.B; ++b) {
    std::vector<int> bad;
    for (int k = 0; k < res.n_shifts; ++k)
      if (!res.status[(size_t)b * res.n_shifts + k].converged) bad.push_back(k);
    if (!bad.empty()) {
      g_last_unconverged = bad;
      throw Error(LT_ERR_NOT_CONVERGED, std::string(what) + ": " + std::to_string(bad.size()) + " of " +
                                            std::to_string(res.n_shifts) + " shifts unconverged after " +
                                            std::to_string(res.iterations[b]) + " iterations");
    }
  }
}

// Shifts and schedule of one family (solve_family, forward.cpp:40-71).
void fill_schedule(OuterProblem& prob, int b, const std::vector<cd>& shifts, int kind, int maxit_eff) {
  Schedule sch = select_schedule(shifts);
  if (kind == LT_SOLVER_SINGLE) {
    sch.taus = {sch.taus[0]};
    sch.pattern = {0};
  }
  prob.tau_table[b].resize(maxit_eff);
  for (int j = 0; j < maxit_eff; ++j) prob.tau_table[b][j] = d2(sch.tau_at(j));
  for (size_t k = 0; k < shifts.size(); ++k) prob.shifts[(size_t)b * shifts.size() + k] = d2(shifts[k]);
}

int effective_maxit(int64_t n, int maxit, int ns) {
  return maxit > 0 ? (int)std::min<int64_t>(n, maxit) : (int)std::min<int64_t>(n, 10 * (int64_t)ns);
}

// Direct mode (solve_shifted_direct): one exact shift-and-invert solve per shift, stored as a
// basis whose coefficient vectors select column k.
void direct_solve(lt_pencil p, int B, const double2* b_dev, const std::vector<cd>& shifts_all, int ns,
                  OuterResult& res) {
  cudaStream_t st = p->ctx->stream;
  const int64_t n = p->n;
  res.B = B;
  res.n_shifts = ns;
  res.maxit = ns;
  res.cap = ns;
  res.iterations.assign(B, 0);
  res.status.assign((size_t)B * ns, lt_shift_status{1, 0, 0.0, 0.0});
  res.m_used.assign((size_t)B * ns, 0);
  res.U.clear();
  std::vector<double2> Y((size_t)B * ns * ns, make_double2(0, 0));
  for (int k = 0; k < ns; ++k) {
    res.U.emplace_back(sizeof(double2) * (size_t)B * n, st);
    std::vector<double2> taus(B);
    for (int b = 0; b < B; ++b) taus[b] = d2(shifts_all[(size_t)b * ns + k]);
    inner_solve(p, B, taus.data(), b_dev, n, res.U.back().as<double2>(), n);
    for (int b = 0; b < B; ++b) {
      Y[((size_t)b * ns + k) * ns + k] = make_double2(1.0, 0.0);
      res.m_used[(size_t)b * ns + k] = k + 1;
    }
  }
  res.Y.allocate(sizeof(double2) * Y.size(), st);
  LT_CUDA(cudaMemcpyAsync(res.Y.get(), Y.data(), sizeof(double2) * Y.size(), cudaMemcpyHostToDevice, st));
}

// Run one batch of families (same n_shifts) with the configured solver.
void solve_families(lt_pencil p, const lt_solver_config& cfg, int B, const double2* b_dev,
                    const std::vector<std::vector<cd>>& shifts, OuterResult& res) {
  const int ns = (int)shifts[0].size();
  if (cfg.kind == LT_SOLVER_DIRECT) {
    std::vector<cd> all;
    for (auto& s : shifts) all.insert(all.end(), s.begin(), s.end());
    direct_solve(p, B, b_dev, all, ns, res);
    return;
  }
  OuterProblem prob;
  prob.B = B;
  prob.n_shifts = ns;
  prob.b = b_dev;
  prob.variant = cfg.variant;
  prob.tol = cfg.tol;
  prob.maxit = cfg.maxit;
  prob.record_history = false;
  const int me = effective_maxit(p->n, cfg.maxit, ns);
  prob.shifts.resize((size_t)B * ns);
  prob.tau_table.resize(B);
  for (int b = 0; b < B; ++b) fill_schedule(prob, b, shifts[b], cfg.kind, me);
  outer_solve(p, prob, res);
}

// c[b][j] = sum_k coef[b][k] y[b][k][j]  (j < m_used[b][k])
std::vector<double2> basis_coefficients(const OuterResult& res, const std::vector<cd>& coef, int& mc,
                                        int k_begin, int k_end, cudaStream_t st) {
  const int B = res.B, ns = res.n_shifts;
  std::vector<double2> Y((size_t)B * ns * res.maxit);
  LT_CUDA(cudaMemcpyAsync(Y.data(), res.Y.get(), sizeof(double2) * Y.size(), cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
  mc = (int)res.U.size();
  std::vector<double2> c((size_t)B * std::max(mc, 1), make_double2(0, 0));
  for (int b = 0; b < B; ++b)
    for (int k = k_begin; k < k_end; ++k) {
      const cd ck = coef[(size_t)b * ns + k];
      const int mu = res.m_used[(size_t)b * ns + k];
      for (int j = 0; j < mu; ++j) {
        const double2 y = Y[((size_t)b * ns + k) * res.maxit + j];
        const cd v = ck * cd(y.x, y.y);
        c[(size_t)b * mc + j].x += v.real();
        c[(size_t)b * mc + j].y += v.imag();
      }
    }
  return c;
}

void recombine(lt_pencil p, const OuterResult& res, const std::vector<double2>& c, int mc,
               const std::vector<int64_t>& dst, double* heads_dev) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  const int B = res.B;
  std::vector<const double2*> cols(std::max(mc, 1), nullptr);
  for (int j = 0; j < mc; ++j) cols[j] = res.U[j].as<double2>();
  DeviceBuffer dcols(sizeof(void*) * cols.size(), st), dc(sizeof(double2) * c.size(), st),
      ddst(sizeof(int64_t) * dst.size(), st);
  LT_CUDA(cudaMemcpyAsync(dcols.get(), cols.data(), sizeof(void*) * cols.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dc.get(), c.data(), sizeof(double2) * c.size(), cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(ddst.get(), dst.data(), sizeof(int64_t) * dst.size(), cudaMemcpyHostToDevice, st));
  launch(ctx, "recombine", (double)n * B * (16.0 * mc + 16.0), [&] {
    recombine_kernel<<<blocks_for(n, kT) * B, kT, 0, st>>>(n, B, mc, dcols.as<const double2*>(), dc.as<double2>(),
                                                            ddst.as<int64_t>(), heads_dev);
  });
  LT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

void forward(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
             const double* times, int n_times, int n_quad, const lt_talbot_params& contour, const lt_solver_config& cfg,
             bool pooled, int mem, double* heads_out, const double* receivers, int n_rec, double* drawdown_out,
             lt_time_diag* diag_out, double* shift_residuals) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  LT_REQUIRE(n_src >= 1, "solve_forward: no source");
  LT_REQUIRE(n_times >= 1, "solve_forward: no target times");
  double previous = 0.0;
  for (int t = 0; t < n_times; ++t) {
    LT_REQUIRE(times[t] > 0.0, "solve_forward: times must be positive");
    LT_REQUIRE(times[t] >= previous, "solve_forward: times must be ascending");
    previous = times[t];
  }
  LT_REQUIRE(n_quad >= 4 && n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
  const int nh = n_quad / 2;
  std::vector<std::vector<cd>> nodes(n_times), weights(n_times);
  for (int t = 0; t < n_times; ++t) talbot_build(n_quad, times[t], contour, nullptr, &nodes[t], nullptr, &weights[t]);

  // host copies of the source vectors (and initial heads) for the families
  auto kind = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DeviceBuffer src_dev(sizeof(double) * (size_t)n * n_src, st);
  LT_CUDA(cudaMemcpyAsync(src_dev.get(), sources, sizeof(double) * n * n_src, kind, st));
  std::vector<double> ih_h;
  std::vector<int> with_initial(n_src, 0);
  DeviceBuffer ih_dev;
  if (initial_head) {
    ih_dev.allocate(sizeof(double) * (size_t)n * n_src, st);
    LT_CUDA(cudaMemcpyAsync(ih_dev.get(), initial_head, sizeof(double) * n * n_src, kind, st));
    ih_h.resize((size_t)n * n_src);
    LT_CUDA(cudaMemcpyAsync(ih_h.data(), ih_dev.get(), sizeof(double) * n * n_src, cudaMemcpyDeviceToHost, st));
  }
  LT_CUDA(cudaStreamSynchronize(st));
  for (int s = 0; s < n_src && initial_head; ++s) {
    double mx = 0.0;
    for (int64_t a = 0; a < n; ++a) mx = std::max(mx, std::fabs(ih_h[(size_t)s * n + a]));
    with_initial[s] = mx > 0.0;
  }

  // Families: (source, time) items with the rate transform, and (source, time) items with
  // rhs M phi0 when the initial head is nonzero.  Pooled mode: one item per source with the
  // pooled shifts of every time.
  struct Fam { int s; int t; bool initial; };
  std::vector<Fam> fams;
  for (int s = 0; s < n_src; ++s) {
    if (pooled) {
      if (rates[s] != 0.0) fams.push_back({s, -1, false});
      if (with_initial[s]) fams.push_back({s, -1, true});
    } else {
      for (int t = 0; t < n_times; ++t) {
        if (rates[s] != 0.0) fams.push_back({s, t, false});
        if (with_initial[s]) fams.push_back({s, t, true});
      }
    }
  }
  const int F = (int)fams.size();
  const int ns = pooled ? nh * n_times : nh;
  DeviceBuffer heads_dev(sizeof(double) * (size_t)n * n_times * n_src, st);
  LT_CUDA(cudaMemsetAsync(heads_dev.get(), 0, heads_dev.bytes(), st));
  std::vector<lt_time_diag> diags(n_times, lt_time_diag{0, 1});
  if (shift_residuals)
    for (size_t q = 0; q < (size_t)n_src * n_times * nh; ++q) shift_residuals[q] = NAN;

  // item chunks bounded by memory: ~ (2 maxit-columns) vectors per item
  const double per_item = (double)n * sizeof(double2) * 14.0;
  const int chunk = std::max(1, (int)std::min<double>(F, 0.6 * available_device_bytes(p->ctx) / per_item));

  for (int f0 = 0; f0 < F; f0 += chunk) {
    const int B = std::min(chunk, F - f0);
    // right-hand sides
    DeviceBuffer rhs(sizeof(double2) * (size_t)B * n, st);
    std::vector<std::vector<cd>> shifts(B);
    for (int q = 0; q < B; ++q) {
      const Fam& fm = fams[f0 + q];
      if (pooled) {
        for (int t = 0; t < n_times; ++t) shifts[q].insert(shifts[q].end(), nodes[t].begin(), nodes[t].end());
      } else {
        shifts[q] = nodes[fm.t];
      }
      double2* dst = rhs.as<double2>() + (size_t)q * n;
      if (!fm.initial) {
        const double* srcp = src_dev.as<double>() + (size_t)fm.s * n;
        launch(ctx, "rhs", 24.0 * n, [&] { real_to_complex<<<blocks_for(n, kT), kT, 0, st>>>(n, srcp, dst); });
      } else {
        // rhs = M phi0 (apply_mass, forward.cpp:91-93)
        DeviceBuffer tmp(sizeof(double2) * n, st);
        const double* ihp = ih_dev.as<double>() + (size_t)fm.s * n;
        launch(ctx, "rhs", 24.0 * n, [&] { real_to_complex<<<blocks_for(n, kT), kT, 0, st>>>(n, ihp, tmp.as<double2>()); });
        apply_batch(p, 0, nullptr, tmp.as<double2>(), n, dst, n, 1, true, "apply_mass");
      }
    }
    OuterResult res;
    solve_families(p, cfg, B, rhs.as<double2>(), shifts, res);
    // diagnostics and convergence (forward.cpp:57-69)
    for (int q = 0; q < B; ++q) {
      const Fam& fm = fams[f0 + q];
      for (int t = 0; t < n_times; ++t) {
        if (!pooled && fm.t != t) continue;
        diags[t].iterations = std::max(diags[t].iterations, res.iterations[q]);
        for (int k = 0; k < ns; ++k) {
          const auto& stt = res.status[(size_t)q * ns + k];
          if (!stt.converged) diags[t].all_converged = 0;
        }
      }
      if (shift_residuals && !fm.initial) {
        for (int k = 0; k < ns; ++k) {
          const int t = pooled ? k / nh : fm.t;
          const int kk = pooled ? k % nh : k;
          shift_residuals[((size_t)fm.s * n_times + t) * nh + kk] = res.status[(size_t)q * ns + k].true_residual;
        }
      }
    }
    throw_unconverged(res, pooled ? "batch solve" : "shifted solve");
    // recombination per time into heads[s][t]
    for (int t = 0; t < n_times; ++t) {
      std::vector<cd> coef((size_t)B * ns, cd(0.0, 0.0));
      bool any = false;
      for (int q = 0; q < B; ++q) {
        const Fam& fm = fams[f0 + q];
        if (!pooled && fm.t != t) continue;
        any = true;
        for (int k = 0; k < nh; ++k) {
          const int kk = pooled ? t * nh + k : k;
          const cd z = nodes[t][k];
          const cd qh = fm.initial ? cd(1.0, 0.0) : rates[fm.s] / z;  // qhat_step
          coef[(size_t)q * ns + kk] = weights[t][k] * qh;
        }
      }
      if (!any) continue;
      int mc = 0;
      std::vector<double2> c = basis_coefficients(res, coef, mc, 0, ns, st);
      // two passes so the rate and initial-head families of one (s, t) never race
      for (int pass = 0; pass < 2; ++pass) {
        std::vector<int64_t> dst(B, -1);
        bool anyp = false;
        for (int q = 0; q < B; ++q) {
          const Fam& fm = fams[f0 + q];
          if ((!pooled && fm.t != t) || (int)fm.initial != pass) continue;
          dst[q] = ((int64_t)fm.s * n_times + t) * n;
          anyp = true;
        }
        if (anyp) recombine(p, res, c, mc, dst, heads_dev.as<double>());
      }
      LT_CUDA(cudaStreamSynchronize(st));
    }
  }
  if (heads_out) {
    auto k2 = mem == LT_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    LT_CUDA(cudaMemcpyAsync(heads_out, heads_dev.get(), sizeof(double) * (size_t)n * n_times * n_src, k2, st));
  }
  if (receivers && n_rec > 0 && drawdown_out) {
    PointSet ps = make_points(p, receivers, n_rec);
    DeviceBuffer didx(sizeof(int64_t) * ps.idx.size(), st), dw(sizeof(double) * ps.w.size(), st),
        dcnt(sizeof(int) * ps.cnt.size(), st), dout(sizeof(double) * (size_t)n_src * n_times * n_rec, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), ps.idx.data(), sizeof(int64_t) * ps.idx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dw.get(), ps.w.data(), sizeof(double) * ps.w.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), ps.cnt.data(), sizeof(int) * ps.cnt.size(), cudaMemcpyHostToDevice, st));
    const int Bh = n_src * n_times;
    launch(ctx, "gather_points", 0.0, [&] {
      gather_points<<<blocks_for((int64_t)Bh * n_rec, 128), 128, 0, st>>>(n, Bh, n_rec, heads_dev.as<double>(),
                                                                          didx.as<int64_t>(), dw.as<double>(), dcnt.as<int>(),
                                                                          dout.as<double>());
    });
    std::vector<double> g((size_t)Bh * n_rec);
    LT_CUDA(cudaMemcpyAsync(g.data(), dout.get(), sizeof(double) * g.size(), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    // reorder (s, t, r) -> (s, r, t)  (ThtExperiment::measurement_index, jacobian.hpp:37-41)
    for (int s = 0; s < n_src; ++s)
      for (int t = 0; t < n_times; ++t)
        for (int r = 0; r < n_rec; ++r)
          drawdown_out[((size_t)s * n_rec + r) * n_times + t] = g[((size_t)s * n_times + t) * n_rec + r];
  }
  LT_CUDA(cudaStreamSynchronize(st));
  if (diag_out)
    for (int t = 0; t < n_times; ++t) diag_out[t] = diags[t];
}

void jacobian_slice(lt_pencil p, const lt_experiment& ex, int t, int mem, double* jac_out, double* pred_out) {
  lt_ctx ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = p->n;
  const int n_src = ex.n_src, n_rec = ex.n_rec;
  LT_REQUIRE(n_src >= 1 && n_rec >= 1 && ex.n_times >= 1, "ThtForwardModel: experiment must be nonempty");
  LT_REQUIRE(t >= 0 && t < ex.n_times, "jacobian_slice: time index out of range");
  LT_REQUIRE(ex.n_quad >= 4 && ex.n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
  LT_REQUIRE(ex.times[t] > 0.0, "build_contour: time must be positive");
  TraceScope trace_all(ctx, "jacobian_slice", t);
  const int ns = ex.n_quad / 2;
  std::vector<cd> nodes, weights;
  talbot_build(ex.n_quad, ex.times[t], ex.contour, nullptr, &nodes, nullptr, &weights);

  PointSet src = make_points(p, ex.sources, n_src);
  PointSet rec = make_points(p, ex.receivers, n_rec);
  const int B = n_src + n_rec;
  // rhs: sources b_s, receivers -e_r  (jacobian.cpp:216, 227, solve_adjoint_fields cpp:49)
  // sparse point weights of all items (sources +w, receivers -w), scattered on the device
  std::vector<int64_t> pidx((size_t)B * 8, 0);
  std::vector<double> pw((size_t)B * 8, 0.0);
  std::vector<int> pcnt(B, 0);
  for (int s = 0; s < n_src; ++s) {
    pcnt[s] = src.cnt[s];
    for (int q = 0; q < src.cnt[s]; ++q) { pidx[s * 8 + q] = src.idx[s * 8 + q]; pw[s * 8 + q] = src.w[s * 8 + q]; }
  }
  for (int r = 0; r < n_rec; ++r) {
    pcnt[n_src + r] = rec.cnt[r];
    for (int q = 0; q < rec.cnt[r]; ++q) {
      pidx[(n_src + r) * 8 + q] = rec.idx[r * 8 + q];
      pw[(n_src + r) * 8 + q] = -rec.w[r * 8 + q];
    }
  }
  DeviceBuffer rhs(sizeof(double2) * (size_t)B * n, st);
  {
    DeviceBuffer didx(sizeof(int64_t) * pidx.size(), st), dwt(sizeof(double) * pw.size(), st), dcnt(sizeof(int) * B, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), pidx.data(), sizeof(int64_t) * pidx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dwt.get(), pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), pcnt.data(), sizeof(int) * B, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemsetAsync(rhs.get(), 0, rhs.bytes(), st));
    launch(ctx, "rhs", 0.0, [&] {
      scatter_points<<<blocks_for((int64_t)B * 8, 128), 128, 0, st>>>(n, B, didx.as<int64_t>(), dwt.as<double>(),
                                                                      dcnt.as<int>(), rhs.as<double2>());
    });
  }
  std::vector<std::vector<cd>> shifts(B, nodes);
  OuterResult res;
  {
    TraceScope tr(ctx, "  solve_families", B);
    solve_families(p, ex.solver, B, rhs.as<double2>(), shifts, res);
  }
  // forward failures first (jacobian.cpp:214-218), then adjoint
  {
    OuterResult* r = &res;
    for (int b = 0; b < B; ++b) {
      std::vector<int> bad;
      for (int k = 0; k < ns; ++k)
        if (!r->status[(size_t)b * ns + k].converged) bad.push_back(k);
      if (!bad.empty()) {
        g_last_unconverged = bad;
        throw Error(LT_ERR_NOT_CONVERGED, std::string(b < n_src ? "forward solve" : "adjoint solve") + ": " +
                                              std::to_string(bad.size()) + " of " + std::to_string(ns) +
                                              " shifts unconverged after " + std::to_string(r->iterations[b]) + " iterations");
      }
    }
  }
  // fields: phi_{s,k} = qhat_k U_s y_{s,k}; psi_{r,k} = U_r y_{r,k}
  std::vector<double2> scale((size_t)B * ns, make_double2(1.0, 0.0));
  for (int s = 0; s < n_src; ++s)
    for (int k = 0; k < ns; ++k) scale[(size_t)s * ns + k] = d2(ex.rates[s] / nodes[k]);
  DeviceBuffer dscale(sizeof(double2) * scale.size(), st);
  LT_CUDA(cudaMemcpyAsync(dscale.get(), scale.data(), sizeof(double2) * scale.size(), cudaMemcpyHostToDevice, st));
  DeviceBuffer fields(sizeof(double2) * (size_t)B * ns * n, st);
  {
    TraceScope tr(ctx, "  expand", B);
    expand_solutions(p, res, dscale.as<double2>(), fields.as<double2>());
  }
  res.U.clear();  // free the bases before the slice

  std::vector<double2> w(ns), wz(ns);
  for (int k = 0; k < ns; ++k) {
    w[k] = d2(weights[k]);
    wz[k] = d2(ex.storativity_z_factor ? weights[k] * nodes[k] : weights[k]);
  }
  DeviceBuffer dw(sizeof(double2) * 2 * ns, st);
  LT_CUDA(cudaMemcpyAsync(dw.get(), w.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));
  LT_CUDA(cudaMemcpyAsync(dw.as<double2>() + ns, wz.data(), sizeof(double2) * ns, cudaMemcpyHostToDevice, st));

  if (jac_out && p->kind == LT_GRID_P1_TRI) {
    TraceScope tr(ctx, "  jacobian_p1", B);
    const int nx = p->levels[0]->nx, nc = nx + 1;
    const int64_t nelem = 2 * (int64_t)nc * nc;
    const int64_t n_param = ex.include_storativity ? 2 * nelem : nelem;
    double* J = jac_out;
    DeviceBuffer jtmp;
    if (mem != LT_MEM_DEVICE) {
      jtmp.allocate(sizeof(double) * (size_t)n_src * n_rec * n_param, st);
      J = jtmp.as<double>();
    }
    const int nsub_r = (n_rec + RB - 1) / RB;
    const int nsub_total = ((n_src + SB - 1) / SB) * nsub_r;
    LT_REQUIRE(nsub_total <= kT / 2, "jacobian: too many source/receiver blocks for one CTA (n_src*n_rec too large)");
    int TC = std::max(1, kT / (2 * nsub_total));
    TC = std::min(TC, nc);
    auto smem_for = [&](int tc) { return sizeof(double2) * (size_t)4 * B * 2 * tc + sizeof(double) * 4 * tc; };
    while (TC > 1 && smem_for(TC) > 110 * 1024) TC /= 2;
    const size_t smem = smem_for(TC);
    const int tiles_x = (nc + TC - 1) / TC;
    LT_CUDA(cudaFuncSetAttribute(jacobian_p1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const double h = p->grid.h;
    const double bytes = (double)n * 16.0 * ns * B + (double)nelem * 8.0 * n_src * n_rec * (ex.include_storativity ? 2 : 1);
    launch(ctx, "jacobian", bytes, [&] {
      jacobian_p1_kernel<<<(unsigned)(tiles_x * (int64_t)nc), kT, smem, st>>>(
          nx, h * h, p->kappa.as<double>(), p->storativity.as<double>(), fields.as<double2>(), n_src, n_rec, ns,
          dw.as<double2>(), dw.as<double2>() + ns, TC, tiles_x, nsub_r, nsub_total, J,
          ex.include_storativity ? J + nelem : nullptr, n_param);
    });
    if (mem != LT_MEM_DEVICE)
      LT_CUDA(cudaMemcpyAsync(jac_out, J, sizeof(double) * (size_t)n_src * n_rec * n_param, cudaMemcpyDeviceToHost, st));
  } else if (jac_out) {
    TraceScope tr(ctx, "  jacobian", B);
    const int64_t n_param = ex.include_storativity ? 2 * n : n;
    double* J = jac_out;
    DeviceBuffer jtmp;
    if (mem != LT_MEM_DEVICE) {
      jtmp.allocate(sizeof(double) * (size_t)n_src * n_rec * n_param, st);
      J = jtmp.as<double>();
    }
    const int nsub_s = (n_src + SB - 1) / SB, nsub_r = (n_rec + RB - 1) / RB;
    const int nsub_total = nsub_s * nsub_r;
    LT_REQUIRE(nsub_total <= kT, "jacobian: too many source/receiver blocks for one CTA (n_src*n_rec too large)");
    const int nf = 2 * p->dim + 1;
    int TC = std::max(1, kT / nsub_total);
    LevelView L = p->view(0);
    TC = std::min(TC, L.nx);
    auto smem_for = [&](int tc) {
      return sizeof(double2) * (size_t)(nf - 1) * B * tc + sizeof(double) * nf * tc + sizeof(int64_t) * 2 * p->dim * tc;
    };
    while (TC > 1 && smem_for(TC) > 110 * 1024) TC /= 2;  // two CTAs per SM
    LT_REQUIRE(nf * TC <= kT, "jacobian: tile too wide");
    const size_t smem = smem_for(TC);
    const int tiles_x = (L.nx + TC - 1) / TC;
    const unsigned grid = (unsigned)(tiles_x * (int64_t)L.ny * L.nz);
    const double h = p->grid.h;
    const double face_scale = p->dim == 3 ? h : 1.0;
    const double hd = p->dim == 3 ? h * h * h : h * h;
    const double bytes = (double)n * (16.0 * ns * B + 8.0 * n_src * n_rec * (ex.include_storativity ? 2 : 1));
    auto fn = p->dim == 3 ? jacobian_kernel<3> : jacobian_kernel<2>;
    LT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch(ctx, "jacobian", bytes, [&] {
      fn<<<grid, kT, smem, st>>>(L, p->kappa.as<double>(), p->storativity.as<double>(), hd, face_scale,
                                 fields.as<double2>(), n_src, n_rec, ns, dw.as<double2>(), dw.as<double2>() + ns, TC,
                                 tiles_x, nsub_r, nsub_total, J, ex.include_storativity ? J + n : nullptr, n_param);
    });
    if (mem != LT_MEM_DEVICE)
      LT_CUDA(cudaMemcpyAsync(jac_out, J, sizeof(double) * (size_t)n_src * n_rec * n_param, cudaMemcpyDeviceToHost, st));
  }
  if (pred_out) {
    DeviceBuffer didx(sizeof(int64_t) * rec.idx.size(), st), dwt(sizeof(double) * rec.w.size(), st),
        dcnt(sizeof(int) * rec.cnt.size(), st), dout(sizeof(double) * (size_t)n_src * n_rec, st);
    LT_CUDA(cudaMemcpyAsync(didx.get(), rec.idx.data(), sizeof(int64_t) * rec.idx.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dwt.get(), rec.w.data(), sizeof(double) * rec.w.size(), cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaMemcpyAsync(dcnt.get(), rec.cnt.data(), sizeof(int) * rec.cnt.size(), cudaMemcpyHostToDevice, st));
    launch(ctx, "predict", 0.0, [&] {
      predict_kernel<<<blocks_for((int64_t)n_src * n_rec, 128), 128, 0, st>>>(n, n_src, n_rec, ns, fields.as<double2>(),
                                                                             dw.as<double2>(), didx.as<int64_t>(),
                                                                             dwt.as<double>(), dcnt.as<int>(), dout.as<double>());
    });
    LT_CUDA(cudaMemcpyAsync(pred_out, dout.get(), sizeof(double) * (size_t)n_src * n_rec, cudaMemcpyDeviceToHost, st));
  }
  LT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace lt
