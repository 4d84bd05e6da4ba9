// extern "C" boundary (include/laptomo_gpu.h): argument checks, exception -> status mapping,
// host/device staging of caller buffers.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "drivers.hpp"
#include "lt_internal.hpp"
#include "talbot_host.hpp"

namespace lt {
lt_ctx ctx_create(int device);
void ctx_destroy(lt_ctx ctx);
}  // namespace lt

namespace {

thread_local std::string g_err;

template <class F>
lt_status guard(F&& f) {
  try {
    f();
    return LT_OK;
  } catch (const lt::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return LT_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LT_ERR_INTERNAL;
  }
}

using cd = std::complex<double>;

void set_device(lt_ctx ctx) { LT_CUDA(cudaSetDevice(ctx->device)); }

// Stage an n_vals complex buffer onto the device (no copy when already device memory).
struct Staged {
  lt::DeviceBuffer buf;
  double2* ptr = nullptr;
};

Staged stage_in(const lt_complex* x, size_t count, int mem, cudaStream_t st) {
  Staged s;
  if (mem == LT_MEM_DEVICE) {
    s.ptr = reinterpret_cast<double2*>(const_cast<lt_complex*>(x));
  } else {
    s.buf.allocate(sizeof(double2) * count, st);
    s.ptr = s.buf.as<double2>();
    LT_CUDA(cudaMemcpyAsync(s.ptr, x, sizeof(double2) * count, cudaMemcpyHostToDevice, st));
  }
  return s;
}

Staged stage_out(lt_complex* y, size_t count, int mem, cudaStream_t st) {
  Staged s;
  if (mem == LT_MEM_DEVICE) {
    s.ptr = reinterpret_cast<double2*>(y);
  } else {
    s.buf.allocate(sizeof(double2) * count, st);
    s.ptr = s.buf.as<double2>();
  }
  return s;
}

void finish_out(lt_complex* y, const Staged& s, size_t count, int mem, cudaStream_t st) {
  if (mem != LT_MEM_DEVICE)
    LT_CUDA(cudaMemcpyAsync(y, s.ptr, sizeof(double2) * count, cudaMemcpyDeviceToHost, st));
  LT_CUDA(cudaStreamSynchronize(st));
}

void check_pencil(lt_pencil p) { LT_REQUIRE(p != nullptr, "null pencil"); }

void apply_common(lt_pencil p, double2 z, const lt_complex* x, lt_complex* y, int n_rhs, int mem, bool mass) {
  check_pencil(p);
  LT_REQUIRE(n_rhs >= 0, "n_rhs must be nonnegative");
  if (n_rhs == 0) return;
  set_device(p->ctx);
  cudaStream_t st = p->ctx->stream;
  const size_t count = (size_t)p->n * n_rhs;
  Staged xin = stage_in(x, count, mem, st);
  Staged yout = stage_out(y, count, mem, st);
  std::vector<double2> taus(n_rhs, z);
  lt::DeviceBuffer dt(sizeof(double2) * n_rhs, st);
  LT_CUDA(cudaMemcpyAsync(dt.get(), taus.data(), sizeof(double2) * n_rhs, cudaMemcpyHostToDevice, st));
  lt::apply_batch(p, 0, dt.as<double2>(), xin.ptr, p->n, yout.ptr, p->n, n_rhs, mass, mass ? "apply_mass" : "apply");
  finish_out(y, yout, count, mem, st);
}

__global__ void conj_kernel(const double2* in, double2* out, int64_t n) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) out[a] = lt::cconj(in[a]);
}

// A shift-and-invert solve (the reference's exact LU) that ended above the inner solve's
// stagnation floor (kInnerFloor x its tolerance) fails with LT_ERR_NOT_CONVERGED; lt_last_unconverged
// lists the offending right-hand sides (or shifts).
void check_inner(lt_pencil p, const std::vector<double>& rel, int shift = -1) {
  std::vector<int> bad;
  double worst = 0.0;
  for (size_t b = 0; b < rel.size(); ++b)
    if (!(rel[b] <= kInnerFloor * p->inner_tol)) {
      bad.push_back(shift >= 0 ? shift : (int)b);
      worst = std::max(worst, rel[b]);
    }
  if (bad.empty()) return;
  lt::g_last_unconverged = bad;
  throw lt::Error(LT_ERR_NOT_CONVERGED, "shift-and-invert solve: relative residual " + std::to_string(worst) +
                                            " above " + std::to_string(kInnerFloor * p->inner_tol) + " after " +
                                            std::to_string(p->inner_maxit) + " iterations");
}

// adjoint: (K + tau M)^{-H} v = conj((K + tau M)^{-1} conj(v)) since K, M are real symmetric,
// so the adjoint solve reuses the factorisation of tau (factorization.hpp:25).
void solve_common(lt_pencil p, double2 tau, const lt_complex* v, lt_complex* u, int n_rhs, int mem, bool adjoint) {
  check_pencil(p);
  LT_REQUIRE(n_rhs >= 0, "n_rhs must be nonnegative");
  if (n_rhs == 0) return;
  set_device(p->ctx);
  cudaStream_t st = p->ctx->stream;
  const size_t count = (size_t)p->n * n_rhs;
  Staged vin = stage_in(v, count, mem, st);
  Staged uout = stage_out(u, count, mem, st);
  std::vector<double2> taus(n_rhs, tau);
  lt::DeviceBuffer vc;
  const double2* vsrc = vin.ptr;
  if (adjoint) {
    vc.allocate(sizeof(double2) * count, st);
    lt::launch(p->ctx, "conj", 32.0 * count, [&] {
      conj_kernel<<<lt::blocks_for((int64_t)count, 256), 256, 0, st>>>(vin.ptr, vc.as<double2>(), (int64_t)count);
    });
    vsrc = vc.as<double2>();
  }
  std::vector<double> rel(n_rhs, 0.0);
  lt::inner_solve(p, n_rhs, taus.data(), vsrc, p->n, uout.ptr, p->n, nullptr, rel.data());
  check_inner(p, rel);
  if (adjoint)
    lt::launch(p->ctx, "conj", 32.0 * count, [&] {
      conj_kernel<<<lt::blocks_for((int64_t)count, 256), 256, 0, st>>>(uout.ptr, uout.ptr, (int64_t)count);
    });
  finish_out(u, uout, count, mem, st);
}

}  // namespace

extern "C" {

const char* lt_version(void) { return "laptomo-b200 0.1 (sm_100a, FP64)"; }
const char* lt_last_error(void) { return g_err.c_str(); }

int lt_last_unconverged(int* indices, int capacity) {
  const auto& v = lt::g_last_unconverged;
  for (int i = 0; i < (int)v.size() && i < capacity; ++i) indices[i] = v[i];
  return (int)v.size();
}

lt_status lt_ctx_create(int device, lt_ctx* out) {
  return guard([&] {
    LT_REQUIRE(out != nullptr, "lt_ctx_create: null output");
    *out = lt::ctx_create(device);
  });
}

lt_status lt_ctx_destroy(lt_ctx ctx) {
  return guard([&] { lt::ctx_destroy(ctx); });
}

lt_status lt_ctx_synchronize(lt_ctx ctx) {
  return guard([&] {
    LT_REQUIRE(ctx, "null context");
    LT_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

void* lt_ctx_stream(lt_ctx ctx) { return ctx ? (void*)ctx->stream : nullptr; }

lt_status lt_ctx_set_profiling(lt_ctx ctx, int enabled) {
  return guard([&] {
    LT_REQUIRE(ctx, "null context");
    ctx->resolve_profile();
    ctx->profiling = enabled != 0;
  });
}

lt_status lt_ctx_reset_profile(lt_ctx ctx) {
  return guard([&] {
    LT_REQUIRE(ctx, "null context");
    ctx->resolve_profile();
    ctx->profile.clear();
    ctx->class_counter.clear();
    ctx->launches = 0;
    ctx->gap_ms = 0.0;
    ctx->gap_count = 0;
  });
}

lt_status lt_ctx_set_profile_sampling(lt_ctx ctx, int every) {
  return guard([&] {
    LT_REQUIRE(ctx && every >= 1, "lt_ctx_set_profile_sampling: every must be >= 1");
    ctx->sample_every = every;
  });
}

int lt_ctx_profile(lt_ctx ctx, int capacity, char* name_buf, double* total_ms, int64_t* launches,
                   double* algorithmic_bytes) {
  if (!ctx) return -1;
  try {
    ctx->resolve_profile();
  } catch (const lt::Error& e) {
    g_err = e.what();
    return -1;
  }
  // the host gaps after stream synchronisations, as a pseudo entry
  if (ctx->gap_count > 0) {
    auto& e = ctx->profile["host_gap"];
    e.ms = ctx->gap_ms;
    e.launches = ctx->gap_count;
    e.bytes = 0.0;
  }
  // with 1-in-N sampling, scale the timed launches of a class to all its launches
  std::map<std::string, int64_t> total;
  for (const auto& kv : ctx->class_counter) total[kv.first] += kv.second;
  int i = 0;
  for (const auto& kv : ctx->profile) {
    if (i < capacity) {
      if (name_buf) {
        std::strncpy(name_buf + 64 * i, kv.first.c_str(), 63);
        name_buf[64 * i + 63] = 0;
      }
      const int64_t timed = kv.second.launches;
      const int64_t all = std::max<int64_t>(timed, total.count(kv.first) ? total[kv.first] : timed);
      const double f = timed > 0 ? (double)all / (double)timed : 1.0;
      if (total_ms) total_ms[i] = kv.second.ms * f;
      if (launches) launches[i] = all;
      if (algorithmic_bytes) algorithmic_bytes[i] = kv.second.bytes * f;
    }
    ++i;
  }
  return i;
}

int64_t lt_ctx_launch_count(lt_ctx ctx) { return ctx ? ctx->launches : -1; }

void lt_talbot_default_params(lt_talbot_params* out) {
  if (out) *out = lt_talbot_params{-0.6122, 0.5017, 0.2645 / 0.5017, 0.6407};
}

lt_status lt_talbot_build(int n_quad, double time, const lt_talbot_params* params, double* thetas,
                          lt_complex* nodes, lt_complex* dnodes, lt_complex* weights) {
  return guard([&] {
    LT_REQUIRE(n_quad >= 4 && n_quad % 2 == 0, "build_contour: n_quad must be even and at least 4");
    LT_REQUIRE(time > 0.0, "build_contour: time must be positive");
    lt_talbot_params p;
    if (params) p = *params; else lt_talbot_default_params(&p);
    std::vector<double> th;
    std::vector<cd> z, dz, w;
    lt::talbot_build(n_quad, time, p, &th, &z, &dz, &w);
    for (size_t k = 0; k < z.size(); ++k) {
      if (thetas) thetas[k] = th[k];
      if (nodes) nodes[k] = lt_complex{z[k].real(), z[k].imag()};
      if (dnodes) dnodes[k] = lt_complex{dz[k].real(), dz[k].imag()};
      if (weights) weights[k] = lt_complex{w[k].real(), w[k].imag()};
    }
  });
}

lt_status lt_sample_field_grid(lt_ctx ctx, int dim, const int* shape, double h, double variance,
                               const double* corr_lengths, double mean, uint64_t seed, const lt_complex* noise,
                               int mem, double* out) {
  return guard([&] {
    lt::sample_field_grid(ctx, dim, shape, h, variance, corr_lengths, mean, seed,
                          reinterpret_cast<const double2*>(noise), mem, out);
  });
}

lt_status lt_qhat_step(double q0, lt_complex z, lt_complex* out) {
  return guard([&] {
    LT_REQUIRE(!(z.re == 0.0 && z.im == 0.0), "qhat_step: z must be nonzero");
    const cd v = q0 / cd(z.re, z.im);
    *out = lt_complex{v.real(), v.imag()};
  });
}

lt_status lt_select_preconditioner_shifts(const lt_complex* shifts, int n_shifts, lt_complex* taus, int* n_taus,
                                          int* pattern, int* pattern_len) {
  return guard([&] {
    LT_REQUIRE(n_shifts > 0, "select_preconditioner_shifts: empty shift list");
    std::vector<cd> s(n_shifts);
    for (int k = 0; k < n_shifts; ++k) s[k] = cd(shifts[k].re, shifts[k].im);
    lt::Schedule sch = lt::select_schedule(s);
    *n_taus = (int)sch.taus.size();
    for (size_t i = 0; i < sch.taus.size(); ++i) taus[i] = lt_complex{sch.taus[i].real(), sch.taus[i].imag()};
    *pattern_len = (int)sch.pattern.size();
    for (size_t i = 0; i < sch.pattern.size(); ++i) pattern[i] = sch.pattern[i];
  });
}

lt_status lt_pencil_create_grid(lt_ctx ctx, const lt_grid* grid, const double* log_kappa, const double* log_storativity,
                                int mem, lt_pencil* out) {
  return guard([&] {
    LT_REQUIRE(ctx && grid && out, "lt_pencil_create_grid: null argument");
    LT_REQUIRE(grid->kind == LT_GRID_FD_CELL || grid->kind == LT_GRID_P1_TRI,
               "lt_pencil_create_grid: unsupported grid kind");
    if (grid->kind == LT_GRID_P1_TRI) {
      // build_mesh(n, L) (mesh.cpp:14-20): at least one interior node for a nonempty pencil
      LT_REQUIRE(grid->dim == 2, "lt_pencil_create_grid: the P1 mesh is 2-D");
      LT_REQUIRE(grid->shape[0] >= 3, "build_mesh: n_per_side must be at least 3 for interior unknowns");
    } else {
      LT_REQUIRE(grid->dim == 2 || grid->dim == 3, "lt_pencil_create_grid: dim must be 2 or 3");
      for (int d = 0; d < grid->dim; ++d) LT_REQUIRE(grid->shape[d] >= 1, "lt_pencil_create_grid: empty grid");
    }
    LT_REQUIRE(grid->h > 0.0, "lt_pencil_create_grid: spacing must be positive");
    LT_REQUIRE(log_kappa && log_storativity, "assemble: one kappa and one storativity value per element");
    set_device(ctx);
    auto* p = new lt_pencil_s();
    p->ctx = ctx;
    p->grid = *grid;
    p->kind = grid->kind;
    if (grid->dim == 2) p->grid.shape[2] = 1;
    if (grid->kind == LT_GRID_P1_TRI) p->grid.shape[1] = grid->shape[0];
    p->dim = grid->dim;
    try {
      lt::pencil_build(p, log_kappa, log_storativity, mem);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

lt_status lt_pencil_create_csr(lt_ctx ctx, const lt_grid* grid, int64_t n, const lt_sparse* K, const lt_sparse* M,
                               lt_pencil* out) {
  return guard([&] {
    LT_REQUIRE(ctx && grid && K && M && out, "ShiftedPencil(K, M): null argument");
    LT_REQUIRE(K->outer && K->inner && K->values && M->outer && M->inner && M->values,
               "ShiftedPencil(K, M): null matrix array");
    LT_REQUIRE((K->index_bytes == 4 || K->index_bytes == 8) && (M->index_bytes == 4 || M->index_bytes == 8),
               "ShiftedPencil(K, M): index_bytes must be 4 or 8");
    LT_REQUIRE(n >= 1, "ShiftedPencil(K, M): empty matrices");
    LT_REQUIRE(grid->h > 0.0, "ShiftedPencil(K, M): grid spacing must be positive");
    if (grid->kind == LT_GRID_P1_TRI) {
      LT_REQUIRE(grid->dim == 2 && grid->shape[0] >= 3, "ShiftedPencil(K, M): the P1 mesh is 2-D with n_per_side >= 3");
    } else {
      LT_REQUIRE(grid->kind == LT_GRID_FD_CELL && (grid->dim == 2 || grid->dim == 3),
                 "ShiftedPencil(K, M): unsupported grid");
      for (int d = 0; d < grid->dim; ++d) LT_REQUIRE(grid->shape[d] >= 1, "ShiftedPencil(K, M): empty grid");
    }
    set_device(ctx);
    auto* p = new lt_pencil_s();
    p->ctx = ctx;
    p->grid = *grid;
    p->kind = grid->kind;
    if (grid->dim == 2) p->grid.shape[2] = 1;
    if (grid->kind == LT_GRID_P1_TRI) p->grid.shape[1] = grid->shape[0];
    p->dim = grid->dim;
    p->n = n;
    p->from_csr = true;
    try {
      lt::pencil_build_csr(p, K, M);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

lt_status lt_pencil_destroy(lt_pencil p) {
  return guard([&] {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    cudaStreamSynchronize(p->ctx->stream);
    delete p;
    cudaStreamSynchronize(nullptr);
  });
}

int64_t lt_pencil_rows(lt_pencil p) { return p ? p->n : -1; }

int64_t lt_pencil_parameters(lt_pencil p) {
  if (!p) return -1;
  if (p->from_csr) return 0;
  if (p->kind == LT_GRID_P1_TRI) {
    const int64_t nc = p->grid.shape[0] - 1;
    return 2 * nc * nc;
  }
  return p->n;
}
int lt_pencil_levels(lt_pencil p) { return p ? (int)p->levels.size() : -1; }

lt_status lt_pencil_apply(lt_pencil p, lt_complex z, const lt_complex* x, lt_complex* y, int n_rhs, int mem) {
  return guard([&] { apply_common(p, make_double2(z.re, z.im), x, y, n_rhs, mem, false); });
}

lt_status lt_pencil_apply_adjoint(lt_pencil p, lt_complex z, const lt_complex* x, lt_complex* y, int n_rhs, int mem) {
  // K and M are real symmetric: (K + z M)^H = K + conj(z) M (shifted_solver.cpp:112-116)
  return guard([&] { apply_common(p, make_double2(z.re, -z.im), x, y, n_rhs, mem, false); });
}

lt_status lt_pencil_apply_mass(lt_pencil p, const lt_complex* x, lt_complex* y, int n_rhs, int mem) {
  return guard([&] { apply_common(p, make_double2(0, 0), x, y, n_rhs, mem, true); });
}

lt_status lt_pencil_prepare(lt_pencil p, const lt_complex* taus, int n_taus) {
  return guard([&] {
    check_pencil(p);
    set_device(p->ctx);
    for (int i = 0; i < n_taus; ++i) p->factor(make_double2(taus[i].re, taus[i].im));
  });
}

int lt_pencil_factorization_count(lt_pencil p) { return p ? (int)p->factors.size() : -1; }

lt_status lt_pencil_set_inner_tolerance(lt_pencil p, double rel_tol, int max_iterations) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(rel_tol > 0.0 && max_iterations > 0, "inner tolerance and iteration cap must be positive");
    p->inner_tol = rel_tol;
    p->inner_maxit = max_iterations;
  });
}

lt_status lt_pencil_solve(lt_pencil p, lt_complex tau, const lt_complex* v, lt_complex* u, int n_rhs, int mem) {
  return guard([&] { solve_common(p, make_double2(tau.re, tau.im), v, u, n_rhs, mem, false); });
}

lt_status lt_pencil_solve_adjoint(lt_pencil p, lt_complex tau, const lt_complex* v, lt_complex* u, int n_rhs, int mem) {
  return guard([&] { solve_common(p, make_double2(tau.re, tau.im), v, u, n_rhs, mem, true); });
}

lt_status lt_pencil_point_weights(lt_pencil p, const double* point, int64_t* indices, double* weights, int* count) {
  return guard([&] {
    check_pencil(p);
    lt::point_weights(p, point, indices, weights, count);
  });
}

void lt_solve_default_options(lt_solve_options* out) {
  if (out) *out = lt_solve_options{LT_VARIANT_GMRES, 1e-10, 0, 0, 1};
}

lt_status lt_solve_shifted(lt_pencil p, const lt_complex* b, int n_rhs, const lt_complex* shifts, int n_shifts,
                           const lt_complex* taus, int n_taus, const int* pattern, int pattern_len,
                           const lt_solve_options* options, int mem, lt_complex* x_out, lt_shift_status* status,
                           int* iterations, double* history) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(n_taus > 0 && pattern_len > 0 && taus && pattern,
               "solve_shifted_flexible: empty preconditioner schedule");
    for (int i = 0; i < pattern_len; ++i)
      LT_REQUIRE(pattern[i] >= 0 && pattern[i] < n_taus, "solve_shifted_flexible: pattern index out of range");
    LT_REQUIRE(n_rhs >= 1 && n_shifts >= 0, "lt_solve_shifted: bad sizes");
    set_device(p->ctx);
    cudaStream_t st = p->ctx->stream;
    lt_solve_options opt;
    if (options) opt = *options; else lt_solve_default_options(&opt);
    const int64_t n = p->n;
    Staged bin = stage_in(b, (size_t)n * n_rhs, mem, st);
    lt::OuterProblem prob;
    prob.B = n_rhs;
    prob.n_shifts = n_shifts;
    prob.b = bin.ptr;
    prob.variant = opt.variant;
    prob.tol = opt.tol;
    prob.maxit = opt.maxit;
    prob.record_history = history != nullptr && opt.record_history;
    prob.keep_basis = opt.keep_basis != 0;
    const int me = opt.maxit > 0 ? (int)std::min<int64_t>(n, opt.maxit) : (int)std::min<int64_t>(n, 10 * (int64_t)n_shifts);
    prob.shifts.resize((size_t)n_rhs * n_shifts);
    prob.tau_table.assign(n_rhs, std::vector<double2>(std::max(me, 1)));
    for (int r = 0; r < n_rhs; ++r) {
      for (int k = 0; k < n_shifts; ++k) prob.shifts[(size_t)r * n_shifts + k] = make_double2(shifts[k].re, shifts[k].im);
      for (int j = 0; j < me; ++j) {
        const lt_complex t = taus[pattern[j % pattern_len]];
        prob.tau_table[r][j] = make_double2(t.re, t.im);
      }
    }
    lt::OuterResult res;
    lt::outer_solve(p, prob, res);
    if (x_out && n_shifts > 0) {
      const size_t count = (size_t)n * n_shifts * n_rhs;
      Staged xo = stage_out(x_out, count, mem, st);
      lt::expand_solutions(p, res, nullptr, xo.ptr);
      finish_out(x_out, xo, count, mem, st);
    }
    if (status)
      for (size_t t = 0; t < res.status.size(); ++t) status[t] = res.status[t];
    if (iterations)
      for (int r = 0; r < n_rhs; ++r) iterations[r] = res.iterations[r];
    if (history && prob.record_history) {
      for (int r = 0; r < n_rhs; ++r)
        for (int k = 0; k < n_shifts; ++k)
          for (int j = 0; j < me; ++j)
            history[((size_t)r * n_shifts + k) * me + j] = res.history[((size_t)r * n_shifts + k) * res.maxit + j];
    }
  });
}

lt_status lt_last_basis(lt_pencil p, int rhs, int* steps_out, double* beta_out, lt_complex* V, lt_complex* U,
                        lt_complex* Hbar, lt_complex* taus) {
  return guard([&] {
    check_pencil(p);
    const auto& kb = p->kept;
    LT_REQUIRE(rhs >= 0 && rhs < kb.n_rhs, "lt_last_basis: no kept basis for this rhs (keep_basis = 1?)");
    const int m = kb.steps[rhs];
    if (steps_out) *steps_out = m;
    if (beta_out) *beta_out = kb.beta[rhs];
    if (V) std::memcpy(V, kb.V[rhs].data(), sizeof(double2) * kb.V[rhs].size());
    if (U) std::memcpy(U, kb.U[rhs].data(), sizeof(double2) * kb.U[rhs].size());
    if (Hbar) std::memcpy(Hbar, kb.H[rhs].data(), sizeof(double2) * kb.H[rhs].size());
    if (taus) std::memcpy(taus, kb.taus[rhs].data(), sizeof(double2) * kb.taus[rhs].size());
  });
}

lt_status lt_residual_estimate(const lt_complex* Hbar, const lt_complex* taus, int m, lt_complex z, const lt_complex* y_fom,
                               int y_len, double* out) {
  return guard([&] {
    LT_REQUIRE(out != nullptr, "residual_estimate: null output");
    if (m < 1 || y_len != m || !Hbar || !taus || !y_fom)
      throw lt::Error(LT_ERR_INVALID_ARGUMENT, "residual_estimate: FOM coefficients of length m required");
    const std::complex<double> h_next(Hbar[(size_t)(m - 1) * (m + 1) + m].re, Hbar[(size_t)(m - 1) * (m + 1) + m].im);
    const std::complex<double> tau_m(taus[m - 1].re, taus[m - 1].im), zz(z.re, z.im), y(y_fom[m - 1].re, y_fom[m - 1].im);
    *out = std::abs(h_next * (zz - tau_m) * y);
  });
}

lt_status lt_solve_shifted_direct(lt_pencil p, const lt_complex* b, int n_rhs, const lt_complex* shifts, int n_shifts,
                                  int mem, lt_complex* x_out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(n_rhs >= 1 && n_shifts >= 0 && x_out, "lt_solve_shifted_direct: bad arguments");
    set_device(p->ctx);
    cudaStream_t st = p->ctx->stream;
    const int64_t n = p->n;
    Staged bin = stage_in(b, (size_t)n * n_rhs, mem, st);
    const size_t count = (size_t)n * n_shifts * n_rhs;
    Staged xo = stage_out(x_out, count, mem, st);
    std::vector<int> bad;
    double worst = 0.0;
    for (int k = 0; k < n_shifts; ++k) {
      std::vector<double2> t(n_rhs, make_double2(shifts[k].re, shifts[k].im));
      std::vector<double> rel(n_rhs, 0.0);
      lt::inner_solve(p, n_rhs, t.data(), bin.ptr, n, xo.ptr + (size_t)k * n, (int64_t)n * n_shifts, nullptr,
                      rel.data());
      for (double r : rel)
        if (!(r <= kInnerFloor * p->inner_tol)) {
          if (bad.empty() || bad.back() != k) bad.push_back(k);
          worst = std::max(worst, r);
        }
    }
    finish_out(x_out, xo, count, mem, st);
    if (!bad.empty()) {
      lt::g_last_unconverged = bad;
      throw lt::Error(LT_ERR_NOT_CONVERGED, "solve_shifted_direct: " + std::to_string(bad.size()) +
                                                " shifts above the shift-and-invert floor (worst relative residual " +
                                                std::to_string(worst) + ")");
    }
    return;
    finish_out(x_out, xo, count, mem, st);
  });
}

void lt_solver_default_config(lt_solver_config* out) {
  if (out) *out = lt_solver_config{LT_SOLVER_FLEXIBLE, LT_VARIANT_GMRES, 1e-10, 0};
}

lt_status lt_forward(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
                     const double* times, int n_times, int n_quad, const lt_talbot_params* contour,
                     const lt_solver_config* solver, int pooled, int mem, double* heads_out, const double* receivers,
                     int n_rec, double* drawdown_out, lt_time_diag* diag_out, double* shift_residuals) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(sources && rates && times, "solve_forward: missing operators");
    set_device(p->ctx);
    lt_talbot_params tp;
    if (contour) tp = *contour; else lt_talbot_default_params(&tp);
    lt_solver_config cfg;
    if (solver) cfg = *solver; else lt_solver_default_config(&cfg);
    lt::forward(p, sources, rates, n_src, initial_head, times, n_times, n_quad, tp, cfg, pooled != 0, mem, heads_out,
                receivers, n_rec, drawdown_out, diag_out, shift_residuals);
  });
}

void lt_experiment_defaults(lt_experiment* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  out->n_quad = 20;
  lt_talbot_default_params(&out->contour);
  lt_solver_default_config(&out->solver);
  out->include_storativity = 0;
  out->storativity_z_factor = 1;
}

lt_status lt_jacobian_slice(lt_pencil p, const lt_experiment* exp, int time_index, int mem, double* jac_out,
                            double* predictions_out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(exp, "null experiment");
    set_device(p->ctx);
    lt::jacobian_slice(p, *exp, time_index, mem, jac_out, predictions_out);
  });
}

lt_status lt_jacobian(lt_pencil p, const lt_experiment* exp, double* jac_out, double* predictions_out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(exp, "null experiment");
    LT_REQUIRE(!(jac_out && p->from_csr),
               "ThtForwardModel::jacobian: the pencil was created from (K, M) and carries no parameter fields");
    set_device(p->ctx);
    const int64_t n_param = exp->include_storativity ? 2 * lt_pencil_parameters(p) : lt_pencil_parameters(p);
    const int pairs = exp->n_src * exp->n_rec;
    std::vector<double> slice(jac_out ? (size_t)pairs * n_param : 0), pred(pairs);
    for (int t = 0; t < exp->n_times; ++t) {
      lt::jacobian_slice(p, *exp, t, LT_MEM_HOST, jac_out ? slice.data() : nullptr, pred.data());
      for (int q = 0; q < pairs; ++q) {
        const size_t row = (size_t)q * exp->n_times + t;  // (s*n_rec + r)*n_times + t
        if (jac_out) std::memcpy(jac_out + row * n_param, slice.data() + (size_t)q * n_param, sizeof(double) * n_param);
        if (predictions_out) predictions_out[row] = pred[q];
      }
    }
  });
}

lt_status lt_predict(lt_pencil p, const lt_experiment* exp, double* predictions_out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(exp && predictions_out, "null argument");
    LT_REQUIRE(exp->n_src >= 1 && exp->n_rec >= 1 && exp->n_times >= 1, "ThtForwardModel: experiment must be nonempty");
    set_device(p->ctx);
    const int64_t n = p->n;
    std::vector<double> src((size_t)n * exp->n_src, 0.0);
    for (int s = 0; s < exp->n_src; ++s) {
      int64_t idx[8];
      double w[8];
      int cnt = 0;
      lt::point_weights(p, exp->sources + (size_t)s * p->dim, idx, w, &cnt);
      for (int q = 0; q < cnt; ++q) src[(size_t)s * n + idx[q]] += w[q];
    }
    lt::forward(p, src.data(), exp->rates, exp->n_src, nullptr, exp->times, exp->n_times, exp->n_quad, exp->contour,
                exp->solver, false, LT_MEM_HOST, nullptr, exp->receivers, exp->n_rec, predictions_out, nullptr, nullptr);
  });
}

lt_status lt_crank_nicolson(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
                            double dt, const double* sample_times, int n_samples, int mem, double* samples_out,
                            int* steps_out) {
  return guard([&] {
    check_pencil(p);
    set_device(p->ctx);
    lt::crank_nicolson(p, sources, rates, n_src, initial_head, dt, sample_times, n_samples, mem, samples_out, steps_out);
  });
}

lt_status lt_pencil_condest(lt_pencil p, lt_complex z, double* norm_a, double* norm_inv, double* cond) {
  return guard([&] {
    check_pencil(p);
    set_device(p->ctx);
    lt::condition_estimate(p, lt::to_d2(z), norm_a, norm_inv, cond);
  });
}

void lt_gn_default_options(lt_gn_options* out) {
  if (out) *out = lt_gn_options{15, 1e-3, 1, 5};
}

lt_status lt_gn_step(lt_ctx ctx, const lt_gn_problem* problem, const double* s, const double* beta,
                     const lt_gn_options* options, double* s_out, double* beta_out, double* xi_out, lt_gn_stats* stats) {
  return guard([&] {
    LT_REQUIRE(ctx && problem && s && s_out && (problem->p == 0 || (beta && beta_out)), "gauss_newton_step: null argument");
    set_device(ctx);
    lt_gn_options o;
    if (options) o = *options; else lt_gn_default_options(&o);
    lt::gn_step(ctx, *problem, s, beta, o, s_out, beta_out, xi_out, stats);
  });
}

lt_status lt_gn_invert(lt_ctx ctx, const lt_gn_problem* problem, const double* s0, const double* beta0,
                       const lt_gn_options* options, double* s_hat, double* beta_hat, lt_gn_stats* history, int* steps_out,
                       int* converged, char* reason, int reason_capacity) {
  return guard([&] {
    LT_REQUIRE(ctx && problem && s0 && s_hat && (problem->p == 0 || (beta0 && beta_hat)), "invert: null argument");
    set_device(ctx);
    lt_gn_options o;
    if (options) o = *options; else lt_gn_default_options(&o);
    const int k = lt::gn_invert(ctx, *problem, s0, beta0, o, s_hat, beta_hat, history, o.max_gn, converged, reason,
                                reason_capacity);
    if (steps_out) *steps_out = k;
  });
}

lt_status lt_gn_objective(lt_ctx ctx, const lt_gn_problem* problem, const double* s, const double* beta,
                          double* objective, double* misfit, double* prior) {
  return guard([&] {
    LT_REQUIRE(ctx && problem && s && (problem->p == 0 || beta), "objective: null argument");
    set_device(ctx);
    const double o = lt::gn_objective(ctx, *problem, s, beta, misfit, prior);
    if (objective) *objective = o;
  });
}

lt_status lt_split_solve(lt_pencil p, const lt_experiment* exp, int time_index, int item0, int item1, lt_split* out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(exp && out, "lt_split_solve: null argument");
    LT_REQUIRE(exp->n_src >= 1 && exp->n_rec >= 1 && exp->n_times >= 1, "ThtForwardModel: experiment must be nonempty");
    set_device(p->ctx);
    auto* s = new lt_split_s();
    s->p = p;
    s->t = time_index;
    s->item0 = item0;
    s->item1 = item1;
    const int d = p->dim;
    s->sources.assign(exp->sources, exp->sources + (size_t)exp->n_src * d);
    s->receivers.assign(exp->receivers, exp->receivers + (size_t)exp->n_rec * d);
    s->rates.assign(exp->rates, exp->rates + exp->n_src);
    s->times.assign(exp->times, exp->times + exp->n_times);
    s->ex = *exp;
    s->ex.sources = s->sources.data();
    s->ex.receivers = s->receivers.data();
    s->ex.rates = s->rates.data();
    s->ex.times = s->times.data();
    try {
      lt::split_solve(s);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int lt_split_columns(lt_split s) { return s ? (int)s->res.U.size() : -1; }

lt_status lt_split_coefficients(lt_split s, int m_pad, lt_complex* Y, int* m_used) {
  return guard([&] {
    LT_REQUIRE(s && Y && m_used, "lt_split_coefficients: null argument");
    set_device(s->p->ctx);
    lt::split_coefficients(s, reinterpret_cast<double2*>(Y), m_used, m_pad);
  });
}

lt_status lt_split_export(lt_split s, int plane0, int plane1, int m_pad, lt_complex* dst, int mem) {
  return guard([&] {
    LT_REQUIRE(s && dst, "lt_split_export: null argument");
    set_device(s->p->ctx);
    lt::split_export(s, plane0, plane1, m_pad, reinterpret_cast<double2*>(dst), mem);
  });
}

lt_status lt_split_predictions(lt_split s, double* predictions_out) {
  return guard([&] {
    LT_REQUIRE(s && predictions_out, "lt_split_predictions: null argument");
    set_device(s->p->ctx);
    lt::split_predictions(s, predictions_out);
  });
}

lt_status lt_split_destroy(lt_split s) {
  return guard([&] {
    if (!s) return;
    set_device(s->p->ctx);
    cudaStreamSynchronize(s->p->ctx->stream);
    delete s;
  });
}

lt_status lt_jacobian_assemble_slab(lt_pencil p, const lt_experiment* exp, int time_index, int plane0, int plane1,
                                    const lt_complex* U_slab, int m, const lt_complex* Y, const int* m_used, int mem,
                                    double* jac_out) {
  return guard([&] {
    check_pencil(p);
    LT_REQUIRE(exp && U_slab && Y && m_used && jac_out, "lt_jacobian_assemble_slab: null argument");
    LT_REQUIRE(exp->n_src >= 1 && exp->n_rec >= 1 && exp->n_times >= 1, "ThtForwardModel: experiment must be nonempty");
    set_device(p->ctx);
    const int nplanes = p->dim == 3 ? p->grid.shape[2] : p->grid.shape[1];
    const int lo = plane0 > 0 ? 1 : 0, hi = plane1 < nplanes ? 1 : 0;
    lt::jacobian_assemble_slab(p, *exp, time_index, plane0, plane1, lo, hi, reinterpret_cast<const double2*>(U_slab), m,
                               reinterpret_cast<const double2*>(Y), m_used, mem, jac_out);
  });
}

}  // extern "C"
