// Device check of the C++ mirror (include/laptomo/laptomo.hpp) of the reference API, driven by
// tests/test_gpu_boundary.py::test_cpp_mirror_on_device: reads a case written by the test,
// runs it through the mirror (which calls the C ABI of liblaptomo_gpu.so) and writes the
// results for the test to compare with the CPU oracle.
//
//   cpp_mirror_device_check <in.bin> <out.bin>
// in:  int32 nx, ny; f64 h; f64 log_kappa[n], log_s[n]; K and M as (int64 nnz, int64 outer[n+1],
//      int64 inner[nnz], f64 values[nnz]); f64 source[n]; f64 time
// out: f64 pairs (re, im) of: flexible solutions from the field pencil [n x 16], from the
//      (K, M) pencil [n x 16], direct solutions of the (K, M) pencil for shifts 0..2 [n x 3];
//      then f64: FOM |eta| and the explicit residual for shifts 0..15 (32 values), the heads
//      of solve_forward on the (K, M) pencil at `time` [n], the number of unconverged shifts of
//      the ConvergenceError thrown at maxit = 1, and the kept basis' m.
#include <cmath>
#include <complex>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <vector>

#include "laptomo/laptomo.hpp"

using namespace laptomo;

template <class T>
static void rd(std::ifstream& f, T* p, size_t n) {
  f.read(reinterpret_cast<char*>(p), sizeof(T) * n);
  if (!f) throw std::runtime_error("short input");
}

static SparseMatrix read_sparse(std::ifstream& f, long n) {
  SparseMatrix s;
  s.n = n;
  std::int64_t nnz = 0;
  rd(f, &nnz, 1);
  s.outer.resize(n + 1);
  s.inner.resize(nnz);
  s.values.resize(nnz);
  rd(f, s.outer.data(), n + 1);
  rd(f, s.inner.data(), nnz);
  rd(f, s.values.data(), nnz);
  return s;
}

// y = H_m(z)^{-1} beta e1 (the square top of shifted_hessenberg), partial-pivot Gaussian elimination
static std::vector<Complex> fom_coefficients(const FlexibleBasisState& st, Complex z) {
  const int m = st.m;
  const std::vector<Complex> hz = st.shifted_hessenberg(z);
  std::vector<Complex> A((size_t)m * m), y(m, 0.0);
  for (int c = 0; c < m; ++c)
    for (int r = 0; r < m; ++r) A[(size_t)r * m + c] = hz[(size_t)c * (m + 1) + r];
  y[0] = st.beta;
  for (int k = 0; k < m; ++k) {
    int piv = k;
    for (int r = k + 1; r < m; ++r)
      if (std::abs(A[(size_t)r * m + k]) > std::abs(A[(size_t)piv * m + k])) piv = r;
    for (int c = 0; c < m; ++c) std::swap(A[(size_t)k * m + c], A[(size_t)piv * m + c]);
    std::swap(y[k], y[piv]);
    for (int r = k + 1; r < m; ++r) {
      const Complex f = A[(size_t)r * m + k] / A[(size_t)k * m + k];
      for (int c = k; c < m; ++c) A[(size_t)r * m + c] -= f * A[(size_t)k * m + c];
      y[r] -= f * y[k];
    }
  }
  for (int k = m - 1; k >= 0; --k) {
    Complex s = y[k];
    for (int c = k + 1; c < m; ++c) s -= A[(size_t)k * m + c] * y[c];
    y[k] = s / A[(size_t)k * m + k];
  }
  return y;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1], std::ios::binary);
  int nx = 0, ny = 0;
  double h = 0.0;
  rd(f, &nx, 1);
  rd(f, &ny, 1);
  rd(f, &h, 1);
  const long n = (long)nx * ny;
  std::vector<double> lk(n), ls(n), src(n);
  rd(f, lk.data(), n);
  rd(f, ls.data(), n);
  const SparseMatrix K = read_sparse(f, n), M = read_sparse(f, n);
  rd(f, src.data(), n);
  double time = 0.0;
  rd(f, &time, 1);

  Context ctx(0);
  Grid g;
  g.dim = 2;
  g.shape[0] = nx;
  g.shape[1] = ny;
  g.h = h;
  ShiftedPencil pf(ctx, g, lk, ls);
  ShiftedPencil pc(ctx, g, K, M);
  const TalbotContour c = build_contour(32, time);
  const PreconditionerSchedule sched = select_preconditioner_shifts(c.nodes);
  std::vector<Complex> b(src.begin(), src.end());
  ShiftedSolveOptions opt;
  const ShiftedSolveResult r1 = solve_shifted_flexible(pf, b, c.nodes, sched, opt);
  const ShiftedSolveResult r2 = solve_shifted_flexible(ctx, g, K, M, b, c.nodes, sched, opt);
  const std::vector<Complex> three(c.nodes.begin(), c.nodes.begin() + 3);
  const std::vector<Complex> xd = solve_shifted_direct(pc, b, three);

  // FOM with the kept basis: residual_estimate against the explicit residual
  ShiftedSolveOptions fom;
  fom.variant = KrylovVariant::Fom;
  fom.keep_basis = true;
  const ShiftedSolveResult rf = solve_shifted_flexible(pc, b, c.nodes, sched, fom);
  std::vector<double> eta;
  for (int k = 0; k < c.n_half(); ++k) {
    const std::vector<Complex> y = fom_coefficients(rf.basis, c.nodes[k]);
    std::vector<Complex> x(n, 0.0);
    for (int j = 0; j < rf.basis.m; ++j)
      for (long a = 0; a < n; ++a) x[a] += rf.basis.U[(size_t)j * n + a] * y[j];
    const std::vector<Complex> ax = pc.apply(c.nodes[k], x);
    double r2n = 0.0;
    for (long a = 0; a < n; ++a) r2n += std::norm(b[a] - ax[a]);
    eta.push_back(residual_estimate(rf.basis, c.nodes[k], y));
    eta.push_back(std::sqrt(r2n));
  }

  ForwardProblem pb;
  pb.source = src;
  pb.rate = 1e-4;
  pb.times = {time};
  pb.n_quad = 32;
  const HeadSolution hs = solve_forward(pc, pb);
  double n_unconv = -1.0;
  try {
    SolverConfig sc;
    sc.maxit = 1;
    solve_forward(pc, pb, sc);
  } catch (const ConvergenceError& e) {
    n_unconv = (double)e.unconverged_shifts.size();
  }

  std::ofstream o(argv[2], std::ios::binary);
  auto wc = [&](const std::vector<Complex>& v) { o.write(reinterpret_cast<const char*>(v.data()), sizeof(Complex) * v.size()); };
  auto wd = [&](const std::vector<double>& v) { o.write(reinterpret_cast<const char*>(v.data()), sizeof(double) * v.size()); };
  wc(r1.solutions);
  wc(r2.solutions);
  wc(xd);
  wd(eta);
  wd(hs.heads);
  wd({n_unconv, (double)rf.basis.m});
  std::printf("ok: m=%d iterations=%d/%d unconverged-at-maxit-1=%g\n", rf.basis.m, r1.iterations, r2.iterations, n_unconv);
  return 0;
}
