// Compiles against the C++ mirror (include/laptomo/laptomo.hpp) and links liblaptomo_gpu.so.
// Host-only calls run anywhere; device calls need an sm_100 GPU (otherwise DeviceError).
#include <cmath>
#include <cstdio>
#include <vector>

#include "laptomo/laptomo.hpp"

int main() {
  using namespace laptomo;
  const TalbotContour c = build_contour(24, 1.0);
  std::vector<Complex> f(c.n_half());
  for (int k = 0; k < c.n_half(); ++k) f[k] = 1.0 / (c.nodes[k] + 1.0);
  std::printf("inverse_laplace(1/(z+1), t=1) - exp(-1) = %.3e\n", inverse_laplace_sum(c, f) - std::exp(-1.0));
  const PreconditionerSchedule s = select_preconditioner_shifts(c.nodes);
  std::printf("taus %zu pattern %zu\n", s.taus.size(), s.pattern.size());
  try {
    build_contour(7, 1.0);
  } catch (const std::invalid_argument&) {
    std::printf("invalid_argument ok\n");
  }
  try {
    Context ctx(0);
    Grid g;
    g.dim = 2;
    g.shape[0] = 32;
    g.shape[1] = 32;
    g.h = 1.0 / 32;
    std::vector<double> lk(32 * 32, -9.0), ls(32 * 32, std::log(1e-5));
    ShiftedPencil p(ctx, g, lk, ls);
    ForwardProblem pb;
    pb.source.assign(32 * 32, 0.0);
    pb.source[16 * 32 + 16] = 1.0;
    pb.rate = 1e-4;
    pb.times = {100.0, 1000.0};
    pb.n_quad = 32;
    const HeadSolution h = solve_forward(p, pb);
    std::printf("device: head at source t=100: %.6e, iterations %d\n", h.heads[16 * 32 + 16],
                h.diagnostics[0].iterations);
  } catch (const DeviceError& e) {
    std::printf("no device: %s\n", e.what());
  }
  return 0;
}
