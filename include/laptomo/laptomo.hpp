// laptomo/laptomo.hpp — C++ mirror of the reference's public solver API
// (/root/reference/proj/include/laptomo/{talbot,shifted_solver,forward,jacobian,errors}.hpp)
// over the C ABI of include/laptomo_gpu.h.  Header-only; link liblaptomo_gpu.so.
//
// Same names, argument meaning and exceptions as the reference:
//   std::invalid_argument, laptomo::FactorizationError, laptomo::ConvergenceError
//   (unconverged_shifts).  Vectors are std::vector<double> / std::vector<Complex>;
//   matrices are column-major (n rows), like the Eigen objects they replace.  With Eigen
//   available, the Eigen overloads at the end accept/return Eigen types.
//
// Difference at the boundary: the device operator is matrix-free on a structured grid, so a
// pencil is built either from a grid and per-cell (per-element) log fields, assembled on the
// device, or from an assembled sparse pair (K, M) declared on its grid (ShiftedPencil(ctx,
// grid, K, M): the FD cell-centred operator or the reference's own P1 pair from assemble()).
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "laptomo_gpu.h"

namespace laptomo {

using Complex = std::complex<double>;

// ---- errors (errors.hpp:14-31) ------------------------------------------------------------
class FactorizationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class ConvergenceError : public std::runtime_error {
 public:
  ConvergenceError(const std::string& what, std::vector<int> unconverged)
      : std::runtime_error(what), unconverged_shifts(std::move(unconverged)) {}
  std::vector<int> unconverged_shifts;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(lt_status s) {
  if (s == LT_OK) return;
  const std::string msg = lt_last_error();
  switch (s) {
    case LT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LT_ERR_PRECONDITIONER: throw FactorizationError(msg);
    case LT_ERR_NOT_CONVERGED: {
      std::vector<int> idx(4096);
      const int n = lt_last_unconverged(idx.data(), (int)idx.size());
      idx.resize(n < 4096 ? n : 4096);
      throw ConvergenceError(msg, idx);
    }
    default: throw DeviceError(msg);
  }
}
inline const lt_complex* c(const Complex* p) { return reinterpret_cast<const lt_complex*>(p); }
inline lt_complex* c(Complex* p) { return reinterpret_cast<lt_complex*>(p); }
inline lt_complex c(Complex z) { return lt_complex{z.real(), z.imag()}; }
}  // namespace detail

// ---- context --------------------------------------------------------------------------
class Context {
 public:
  explicit Context(int device = 0) { detail::check(lt_ctx_create(device, &h_)); }
  ~Context() { if (h_) lt_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lt_ctx handle() const { return h_; }

 private:
  lt_ctx h_ = nullptr;
};

// ---- talbot (talbot.hpp:23-63) --------------------------------------------------------
struct TalbotParams {
  double sigma0 = -0.6122;
  double mu0 = 0.5017;
  double nu = 0.2645 / 0.5017;
  double alpha = 0.6407;
  lt_talbot_params c() const { return lt_talbot_params{sigma0, mu0, nu, alpha}; }
};

struct TalbotContour {
  int n_quad = 0;
  double time = 0.0;
  double sigma = 0.0, mu = 0.0, nu = 0.0, alpha = 0.0;
  std::vector<double> thetas;
  std::vector<Complex> nodes, dnodes, weights;
  int n_half() const { return static_cast<int>(nodes.size()); }
};

inline TalbotContour build_contour(int n_quad, double time, const TalbotParams& params = {}) {
  TalbotContour out;
  const int nh = n_quad > 0 ? n_quad / 2 : 0;
  out.thetas.resize(nh);
  out.nodes.resize(nh);
  out.dnodes.resize(nh);
  out.weights.resize(nh);
  const lt_talbot_params p = params.c();
  detail::check(lt_talbot_build(n_quad, time, &p, out.thetas.data(), detail::c(out.nodes.data()),
                                detail::c(out.dnodes.data()), detail::c(out.weights.data())));
  out.n_quad = n_quad;
  out.time = time;
  out.sigma = params.sigma0 * n_quad / time;
  out.mu = params.mu0 * n_quad / time;
  out.nu = params.nu;
  out.alpha = params.alpha;
  return out;
}

inline double inverse_laplace_sum(const TalbotContour& contour, const std::vector<Complex>& values) {
  if ((int)values.size() != contour.n_half())
    throw std::invalid_argument("inverse_laplace_sum: one value per retained node required");
  Complex s = 0.0;
  for (int k = 0; k < contour.n_half(); ++k) s += contour.weights[k] * values[k];
  return 2.0 * s.real();
}

inline Complex qhat_step(double q0, Complex z) {
  lt_complex out;
  detail::check(lt_qhat_step(q0, detail::c(z), &out));
  return {out.re, out.im};
}

// ---- fields (sample_field_on_mesh, fields.hpp:41-44): structured-grid GRF on the device ----
// log-field realisation, x fastest, covariance variance * exp(-|r / l|) (one l per axis)
inline std::vector<double> sample_field_grid(const Context& ctx, const std::vector<int>& shape, double h,
                                             double variance, const std::vector<double>& corr_lengths,
                                             double mean_log, std::uint64_t seed) {
  if (shape.size() != corr_lengths.size()) throw std::invalid_argument("sample_field_grid: one length per axis");
  std::size_t n = 1;
  for (int v : shape) n *= static_cast<std::size_t>(v > 0 ? v : 0);
  std::vector<double> out(n);
  detail::check(lt_sample_field_grid(ctx.handle(), static_cast<int>(shape.size()), shape.data(), h, variance,
                                     corr_lengths.data(), mean_log, seed, nullptr, LT_MEM_HOST, out.data()));
  return out;
}

// ---- shifted solver (shifted_solver.hpp:21-132) ---------------------------------------
enum class KrylovVariant { Fom, Gmres };

struct PreconditionerSchedule {
  std::vector<Complex> taus;
  std::vector<int> pattern;
  Complex tau_at(int iteration) const { return taus[pattern[iteration % pattern.size()]]; }
};

inline PreconditionerSchedule single_tau_schedule(Complex tau) { return {{tau}, {0}}; }

inline PreconditionerSchedule select_preconditioner_shifts(const std::vector<Complex>& shifts) {
  lt_complex taus[2];
  int nt = 0, pat[5], pl = 0;
  detail::check(lt_select_preconditioner_shifts(detail::c(shifts.data()), (int)shifts.size(), taus, &nt, pat, &pl));
  PreconditionerSchedule s;
  for (int i = 0; i < nt; ++i) s.taus.emplace_back(taus[i].re, taus[i].im);
  s.pattern.assign(pat, pat + pl);
  return s;
}

struct ShiftedSolveOptions {
  KrylovVariant variant = KrylovVariant::Gmres;
  double tol = 1e-10;
  int maxit = 0;
  bool keep_basis = false;
  bool record_history = true;
};

struct ShiftStatus {
  bool converged = false;
  int iteration = 0;
  double estimate = 0.0;
  double true_residual = 0.0;
  std::vector<double> history;
};

/// Arnoldi data of the flexible iteration after m steps (shifted_solver.hpp:63-74):
///   (K + z M) U_m = V_{m+1} Hbar_m(z; T_m),  Hbar_m(z; T_m) = [I; 0] + Hbar_m (z I - T_m).
struct FlexibleBasisState {
  std::vector<Complex> V;     // n x (m+1), column-major, orthonormal
  std::vector<Complex> U;     // n x m, preconditioned basis
  std::vector<Complex> Hbar;  // (m+1) x m, column-major
  std::vector<Complex> taus;  // applied tau_j, j = 1..m
  double beta = 0.0;          // ||b||
  int m = 0;
  int steps() const { return m; }
  /// Hbar_m(z; T_m) for a probe shift, (m+1) x m column-major.
  std::vector<Complex> shifted_hessenberg(Complex z) const {
    std::vector<Complex> hz(Hbar);
    for (int l = 0; l < m; ++l) {
      for (int i = 0; i <= m; ++i) hz[(size_t)l * (m + 1) + i] *= (z - taus[l]);
      hz[(size_t)l * (m + 1) + l] += 1.0;
    }
    return hz;
  }
};

/// residual_estimate (shifted_solver.cpp:334-343): the FOM residual norm |eta_k|.
inline double residual_estimate(const FlexibleBasisState& state, Complex z, const std::vector<Complex>& y_fom) {
  double out = 0.0;
  detail::check(lt_residual_estimate(detail::c(state.Hbar.data()), detail::c(state.taus.data()), state.m, detail::c(z),
                                     detail::c(y_fom.data()), (int)y_fom.size(), &out));
  return out;
}

struct ShiftedSolveResult {
  std::vector<Complex> solutions;  // n x n_shifts, column-major
  int iterations = 0;
  bool all_converged = false;
  std::vector<ShiftStatus> shifts;
  bool has_basis = false;          // std::optional<FlexibleBasisState> basis (keep_basis)
  FlexibleBasisState basis;
  std::vector<int> unconverged() const {
    std::vector<int> out;
    for (int k = 0; k < (int)shifts.size(); ++k)
      if (!shifts[k].converged) out.push_back(k);
    return out;
  }
};

/// Cell-centred grid (x fastest): dims 2 or 3.  p1_mesh(n, L) declares the reference's P1
/// mesh build_mesh(n, L) instead (mesh.cpp:14-52).
struct Grid {
  int dim = 2;
  int shape[3] = {1, 1, 1};
  double h = 1.0;
  int kind = LT_GRID_FD_CELL;
  lt_grid c() const { return lt_grid{kind, dim, {shape[0], shape[1], shape[2]}, h}; }
  static Grid p1_mesh(int n_per_side, double side_length) {
    Grid g;
    g.kind = LT_GRID_P1_TRI;
    g.shape[0] = g.shape[1] = n_per_side;
    g.h = side_length / (n_per_side - 1);
    return g;
  }
};

/// An assembled sparse matrix in compressed rows (SparseReal of the reference; K and M being
/// symmetric, the compressed columns of Eigen's default SparseMatrix<double> work as well).
struct SparseMatrix {
  long n = 0;
  std::vector<std::int64_t> outer;  // n + 1
  std::vector<std::int64_t> inner;  // nnz
  std::vector<double> values;       // nnz
  lt_sparse c() const { return lt_sparse{outer.data(), inner.data(), values.data(), 8}; }
};

class ShiftedPencil;

/// SparseComplexFactorization view of a prepared tau (factorization.hpp:19-27).
class Factorization {
 public:
  Factorization(const ShiftedPencil* p, Complex tau) : p_(p), tau_(tau) {}
  long rows() const;
  std::vector<Complex> solve(const std::vector<Complex>& rhs) const;
  std::vector<Complex> solve_adjoint(const std::vector<Complex>& rhs) const;

 private:
  const ShiftedPencil* p_;
  Complex tau_;
};

class ShiftedPencil {
 public:
  ShiftedPencil(const Context& ctx, const Grid& grid, const std::vector<double>& log_kappa,
                const std::vector<double>& log_storativity) {
    const lt_grid g = grid.c();
    detail::check(lt_pencil_create_grid(ctx.handle(), &g, log_kappa.data(), log_storativity.data(), LT_MEM_HOST, &h_));
  }
  /// ShiftedPencil(const SparseReal& K, const SparseReal& M) (shifted_solver.hpp:90) on `grid`.
  ShiftedPencil(const Context& ctx, const Grid& grid, const SparseMatrix& K, const SparseMatrix& M) {
    if (K.n != M.n) throw std::invalid_argument("ShiftedPencil: K and M dimensions disagree");
    const lt_grid g = grid.c();
    const lt_sparse k = K.c(), m = M.c();
    detail::check(lt_pencil_create_csr(ctx.handle(), &g, K.n, &k, &m, &h_));
  }
  ~ShiftedPencil() { if (h_) lt_pencil_destroy(h_); }
  ShiftedPencil(const ShiftedPencil&) = delete;
  ShiftedPencil& operator=(const ShiftedPencil&) = delete;

  long rows() const { return (long)lt_pencil_rows(h_); }
  std::vector<Complex> apply(Complex z, const std::vector<Complex>& x) const {
    std::vector<Complex> y(x.size());
    detail::check(lt_pencil_apply(h_, detail::c(z), detail::c(x.data()), detail::c(y.data()), 1, LT_MEM_HOST));
    return y;
  }
  std::vector<Complex> apply_adjoint(Complex z, const std::vector<Complex>& x) const {
    std::vector<Complex> y(x.size());
    detail::check(lt_pencil_apply_adjoint(h_, detail::c(z), detail::c(x.data()), detail::c(y.data()), 1, LT_MEM_HOST));
    return y;
  }
  std::vector<Complex> apply_mass(const std::vector<Complex>& x) const {
    std::vector<Complex> y(x.size());
    detail::check(lt_pencil_apply_mass(h_, detail::c(x.data()), detail::c(y.data()), 1, LT_MEM_HOST));
    return y;
  }
  Factorization factorization(Complex tau) const {
    const lt_complex t = detail::c(tau);
    detail::check(lt_pencil_prepare(h_, &t, 1));
    return Factorization(this, tau);
  }
  int factorization_count() const { return lt_pencil_factorization_count(h_); }
  lt_pencil handle() const { return h_; }

 private:
  lt_pencil h_ = nullptr;
};

inline long Factorization::rows() const { return p_->rows(); }
inline std::vector<Complex> Factorization::solve(const std::vector<Complex>& rhs) const {
  std::vector<Complex> u(rhs.size());
  detail::check(lt_pencil_solve(p_->handle(), detail::c(tau_), detail::c(rhs.data()), detail::c(u.data()), 1, LT_MEM_HOST));
  return u;
}
inline std::vector<Complex> Factorization::solve_adjoint(const std::vector<Complex>& rhs) const {
  std::vector<Complex> u(rhs.size());
  detail::check(lt_pencil_solve_adjoint(p_->handle(), detail::c(tau_), detail::c(rhs.data()), detail::c(u.data()), 1,
                                        LT_MEM_HOST));
  return u;
}

inline ShiftedSolveResult solve_shifted_flexible(const ShiftedPencil& pencil, const std::vector<Complex>& b,
                                                 const std::vector<Complex>& shifts,
                                                 const PreconditionerSchedule& schedule,
                                                 const ShiftedSolveOptions& options = {}) {
  if (schedule.taus.empty() || schedule.pattern.empty())
    throw std::invalid_argument("solve_shifted_flexible: empty preconditioner schedule");
  const long n = pencil.rows();
  const int ns = (int)shifts.size();
  lt_solve_options o{options.variant == KrylovVariant::Fom ? LT_VARIANT_FOM : LT_VARIANT_GMRES, options.tol,
                     options.maxit, options.keep_basis ? 1 : 0, options.record_history ? 1 : 0};
  ShiftedSolveResult r;
  r.solutions.assign((size_t)n * ns, Complex(0.0));
  std::vector<lt_shift_status> st(ns > 0 ? ns : 1);
  int iters = 0;
  // the C API writes min(n, maxit) entries per shift (capi.cu), maxit defaulting to 10 n_shifts
  const long maxit_req = options.maxit > 0 ? options.maxit : 10L * ns;
  const int maxit = (int)std::min<long>(n, maxit_req);
  std::vector<double> hist((size_t)(ns > 0 ? ns : 1) * (maxit > 0 ? maxit : 1));
  detail::check(lt_solve_shifted(pencil.handle(), detail::c(b.data()), 1, detail::c(shifts.data()), ns,
                                 detail::c(schedule.taus.data()), (int)schedule.taus.size(), schedule.pattern.data(),
                                 (int)schedule.pattern.size(), &o, LT_MEM_HOST, detail::c(r.solutions.data()), st.data(),
                                 &iters, options.record_history ? hist.data() : nullptr));
  r.iterations = iters;
  r.all_converged = true;
  for (int k = 0; k < ns; ++k) {
    ShiftStatus s{st[k].converged != 0, st[k].iteration, st[k].estimate, st[k].true_residual, {}};
    if (options.record_history)
      for (int j = 0; j < iters && j < maxit; ++j) {
        const double v = hist[(size_t)k * maxit + j];
        if (v == v) s.history.push_back(v);
      }
    r.all_converged = r.all_converged && s.converged;
    r.shifts.push_back(std::move(s));
  }
  if (options.keep_basis) {
    FlexibleBasisState& bs = r.basis;
    detail::check(lt_last_basis(pencil.handle(), 0, &bs.m, &bs.beta, nullptr, nullptr, nullptr, nullptr));
    const int m = bs.m;
    bs.V.assign((size_t)n * (m + 1), Complex(0.0));
    bs.U.assign((size_t)n * (m > 0 ? m : 1), Complex(0.0));
    bs.Hbar.assign((size_t)(m + 1) * (m > 0 ? m : 1), Complex(0.0));
    bs.taus.assign(m > 0 ? m : 1, Complex(0.0));
    detail::check(lt_last_basis(pencil.handle(), 0, nullptr, nullptr, detail::c(bs.V.data()), detail::c(bs.U.data()),
                                detail::c(bs.Hbar.data()), detail::c(bs.taus.data())));
    bs.U.resize((size_t)n * m);
    bs.Hbar.resize((size_t)(m + 1) * m);
    bs.taus.resize(m);
    r.has_basis = true;
  }
  return r;
}

/// The (K, M) overloads (shifted_solver.hpp:114-128): a temporary pencil on `grid`.
inline ShiftedSolveResult solve_shifted_flexible(const Context& ctx, const Grid& grid, const SparseMatrix& K,
                                                 const SparseMatrix& M, const std::vector<Complex>& b,
                                                 const std::vector<Complex>& shifts,
                                                 const PreconditionerSchedule& schedule,
                                                 const ShiftedSolveOptions& options = {}) {
  ShiftedPencil p(ctx, grid, K, M);
  return solve_shifted_flexible(p, b, shifts, schedule, options);
}

inline ShiftedSolveResult solve_shifted_single(const ShiftedPencil& pencil, const std::vector<Complex>& b,
                                               const std::vector<Complex>& shifts, Complex tau,
                                               const ShiftedSolveOptions& options = {}) {
  return solve_shifted_flexible(pencil, b, shifts, single_tau_schedule(tau), options);
}

inline ShiftedSolveResult solve_shifted_single(const Context& ctx, const Grid& grid, const SparseMatrix& K,
                                               const SparseMatrix& M, const std::vector<Complex>& b,
                                               const std::vector<Complex>& shifts, Complex tau,
                                               const ShiftedSolveOptions& options = {}) {
  ShiftedPencil p(ctx, grid, K, M);
  return solve_shifted_flexible(p, b, shifts, single_tau_schedule(tau), options);
}

inline std::vector<Complex> solve_shifted_direct(const ShiftedPencil& pencil, const std::vector<Complex>& b,
                                                 const std::vector<Complex>& shifts) {
  std::vector<Complex> x((size_t)pencil.rows() * shifts.size());
  detail::check(lt_solve_shifted_direct(pencil.handle(), detail::c(b.data()), 1, detail::c(shifts.data()),
                                        (int)shifts.size(), LT_MEM_HOST, detail::c(x.data())));
  return x;
}

// ---- forward (forward.hpp:16-61) ------------------------------------------------------
enum class SolverKind { Single, Flexible, Direct };

struct SolverConfig {
  SolverKind kind = SolverKind::Flexible;
  KrylovVariant variant = KrylovVariant::Gmres;
  double tol = 1e-10;
  int maxit = 0;
  lt_solver_config c() const {
    return lt_solver_config{kind == SolverKind::Single ? LT_SOLVER_SINGLE
                                                       : (kind == SolverKind::Direct ? LT_SOLVER_DIRECT : LT_SOLVER_FLEXIBLE),
                            variant == KrylovVariant::Fom ? LT_VARIANT_FOM : LT_VARIANT_GMRES, tol, maxit};
  }
};

struct ForwardProblem {
  std::vector<double> source;        // free-dof interpolation weights of the source
  double rate = 0.0;
  std::vector<double> initial_head;  // empty: zero
  std::vector<double> times;
  int n_quad = 40;
  TalbotParams contour;
};

struct TimeDiagnostics {
  int iterations = 0;
  bool all_converged = true;
  std::vector<double> shift_residuals;
};

struct HeadSolution {
  std::vector<double> heads;  // n x n_times, column-major
  std::vector<TimeDiagnostics> diagnostics;
};

namespace detail {
inline HeadSolution forward(const ShiftedPencil& pencil, const ForwardProblem& pb, const SolverConfig& s, int pooled) {
  const long n = pencil.rows();
  const int nt = (int)pb.times.size();
  HeadSolution out;
  out.heads.assign((size_t)n * nt, 0.0);
  std::vector<lt_time_diag> diag(nt > 0 ? nt : 1);
  std::vector<double> res((size_t)(nt > 0 ? nt : 1) * (pb.n_quad > 1 ? pb.n_quad / 2 : 1));
  const lt_talbot_params tp = pb.contour.c();
  const lt_solver_config sc = s.c();
  const double rate = pb.rate;
  detail::check(lt_forward(pencil.handle(), pb.source.data(), &rate, 1,
                           pb.initial_head.empty() ? nullptr : pb.initial_head.data(), pb.times.data(), nt, pb.n_quad, &tp,
                           &sc, pooled, LT_MEM_HOST, out.heads.data(), nullptr, 0, nullptr, diag.data(), res.data()));
  for (int t = 0; t < nt; ++t) {
    TimeDiagnostics d{diag[t].iterations, diag[t].all_converged != 0, {}};
    d.shift_residuals.assign(res.begin() + (size_t)t * (pb.n_quad / 2), res.begin() + (size_t)(t + 1) * (pb.n_quad / 2));
    out.diagnostics.push_back(std::move(d));
  }
  return out;
}
}  // namespace detail

inline HeadSolution solve_forward(const ShiftedPencil& pencil, const ForwardProblem& problem,
                                  const SolverConfig& solver = {}) {
  return detail::forward(pencil, problem, solver, 0);
}

inline HeadSolution solve_forward_batch(const ShiftedPencil& pencil, const ForwardProblem& problem,
                                        const SolverConfig& solver = {}) {
  return detail::forward(pencil, problem, solver, 1);
}

/// crank_nicolson (forward.cpp:200-258): the head at each sample time, n x n_samples column-major.
inline std::vector<double> crank_nicolson(const ShiftedPencil& pencil, const std::vector<double>& source, double rate,
                                          const std::vector<double>& initial_head, double dt,
                                          const std::vector<double>& sample_times, int* steps_out = nullptr) {
  std::vector<double> out((size_t)pencil.rows() * sample_times.size());
  detail::check(lt_crank_nicolson(pencil.handle(), source.data(), &rate, 1,
                                  initial_head.empty() ? nullptr : initial_head.data(), dt,
                                  sample_times.empty() ? nullptr : sample_times.data(), (int)sample_times.size(),
                                  LT_MEM_HOST, out.data(), steps_out));
  return out;
}

/// estimate_condition_1norm (condest.cpp:43-49) with the actions of K + z M (apply, adjoint,
/// shift-and-invert solve and its adjoint).
inline double estimate_condition_1norm(const ShiftedPencil& pencil, Complex z) {
  double cond = 0.0;
  detail::check(lt_pencil_condest(pencil.handle(), detail::c(z), nullptr, nullptr, &cond));
  return cond;
}

// ---- Jacobian (jacobian.hpp:22-101) ---------------------------------------------------
struct ThtExperiment {
  Grid grid;
  std::vector<std::vector<double>> sources;    // points (dim coordinates each)
  std::vector<double> rates;
  std::vector<std::vector<double>> receivers;
  std::vector<double> times;
  int n_quad = 20;
  TalbotParams contour;
  SolverConfig solver;
  bool include_storativity = false;
  bool storativity_z_factor = true;

  int n_measurements() const { return (int)(sources.size() * receivers.size() * times.size()); }
  int measurement_index(int source, int receiver, int time) const {
    return (source * (int)receivers.size() + receiver) * (int)times.size() + time;
  }
};

struct JacobianResult {
  std::vector<double> jacobian;  // n_measurements x n_parameters, row-major
  std::vector<double> predictions;
};

class ThtForwardModel {
 public:
  ThtForwardModel(const Context& ctx, ThtExperiment experiment, std::vector<double> log_storativity)
      : ctx_(ctx), ex_(std::move(experiment)), log_s_(std::move(log_storativity)) {
    if (ex_.sources.empty() || ex_.receivers.empty() || ex_.times.empty())
      throw std::invalid_argument("ThtForwardModel: experiment must be nonempty");
    if (ex_.rates.size() != ex_.sources.size())
      throw std::invalid_argument("ThtForwardModel: one rate per source required");
  }
  int n_measurements() const { return ex_.n_measurements(); }
  long n_parameters(long n_cells) const { return ex_.include_storativity ? 2 * n_cells : n_cells; }

  std::vector<double> predict(const std::vector<double>& log_kappa) const { return predict_with(log_kappa, log_s_); }
  std::vector<double> predict_with(const std::vector<double>& log_kappa, const std::vector<double>& log_s) const {
    ShiftedPencil p(ctx_, ex_.grid, log_kappa, log_s);
    std::vector<double> src, rec;
    lt_experiment e = c(src, rec);
    std::vector<double> out(n_measurements());
    detail::check(lt_predict(p.handle(), &e, out.data()));
    return out;
  }
  JacobianResult jacobian(const std::vector<double>& log_kappa) const {
    ShiftedPencil p(ctx_, ex_.grid, log_kappa, log_s_);
    std::vector<double> src, rec;
    lt_experiment e = c(src, rec);
    JacobianResult r;
    r.jacobian.assign((size_t)n_measurements() * n_parameters(p.rows()), 0.0);
    r.predictions.assign(n_measurements(), 0.0);
    detail::check(lt_jacobian(p.handle(), &e, r.jacobian.data(), r.predictions.data()));
    return r;
  }

 private:
  lt_experiment c(std::vector<double>& src, std::vector<double>& rec) const {
    lt_experiment e;
    lt_experiment_defaults(&e);
    for (const auto& q : ex_.sources) src.insert(src.end(), q.begin(), q.end());
    for (const auto& q : ex_.receivers) rec.insert(rec.end(), q.begin(), q.end());
    e.sources = src.data();
    e.rates = ex_.rates.data();
    e.n_src = (int)ex_.sources.size();
    e.receivers = rec.data();
    e.n_rec = (int)ex_.receivers.size();
    e.times = ex_.times.data();
    e.n_times = (int)ex_.times.size();
    e.n_quad = ex_.n_quad;
    e.contour = ex_.contour.c();
    e.solver = ex_.solver.c();
    e.include_storativity = ex_.include_storativity ? 1 : 0;
    e.storativity_z_factor = ex_.storativity_z_factor ? 1 : 0;
    return e;
  }
  const Context& ctx_;
  ThtExperiment ex_;
  std::vector<double> log_s_;
};

inline JacobianResult assemble_jacobian(const Context& ctx, const ThtExperiment& experiment,
                                        const std::vector<double>& log_kappa,
                                        const std::vector<double>& log_storativity) {
  return ThtForwardModel(ctx, experiment, log_storativity).jacobian(log_kappa);
}

}  // namespace laptomo

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
namespace laptomo {
// Eigen adapters (the reference's vector types): contiguous Eigen vectors map directly.
inline Eigen::VectorXcd to_eigen(const std::vector<Complex>& v) {
  return Eigen::Map<const Eigen::VectorXcd>(v.data(), (Eigen::Index)v.size());
}
inline std::vector<Complex> from_eigen(const Eigen::VectorXcd& v) { return {v.data(), v.data() + v.size()}; }
}  // namespace laptomo
#endif
#endif
