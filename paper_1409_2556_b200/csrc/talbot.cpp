// Host arithmetic of the contour and the preconditioner schedule (tiny, O(n_quad)):
// talbot.cpp:25-101 and shifted_solver.cpp:81-104 of the reference.
#include <cmath>
#include <complex>
#include <vector>

#include "laptomo_gpu.h"
#include "talbot_host.hpp"

namespace lt {

void talbot_build(int n_quad, double time, const lt_talbot_params& p, std::vector<double>* thetas,
                  std::vector<std::complex<double>>* nodes, std::vector<std::complex<double>>* dnodes,
                  std::vector<std::complex<double>>* weights) {
  const double scale = n_quad / time;
  const double sigma = p.sigma0 * scale;
  const double mu = p.mu0 * scale;
  const double a = p.alpha;
  const int n_half = n_quad / 2;
  const double spacing = 2.0 * M_PI / n_quad;
  for (int k = 0; k < n_half; ++k) {
    const double theta = (k + 0.5) * spacing;
    // contour_point: theta cot(alpha theta) -> 1/alpha at theta = 0 (never sampled).
    const double cot_term = theta == 0.0 ? 1.0 / a : theta * std::cos(a * theta) / std::sin(a * theta);
    const std::complex<double> z(sigma + mu * cot_term, mu * p.nu * theta);
    double dcot = 0.0;
    if (theta != 0.0) {
      const double s = std::sin(a * theta);
      dcot = std::cos(a * theta) / s - a * theta / (s * s);
    }
    const std::complex<double> dz(mu * dcot, mu * p.nu);
    if (thetas) thetas->push_back(theta);
    if (nodes) nodes->push_back(z);
    if (dnodes) dnodes->push_back(dz);
    if (weights)
      weights->push_back(-std::complex<double>(0.0, 1.0) / double(n_quad) * std::exp(z * time) * dz);
  }
}

Schedule select_schedule(const std::vector<std::complex<double>>& shifts) {
  auto less = [](const std::complex<double>& x, const std::complex<double>& y) {
    if (x.real() != y.real()) return x.real() < y.real();
    return x.imag() < y.imag();
  };
  size_t i_min = 0, i_max = 0;
  for (size_t i = 1; i < shifts.size(); ++i) {
    if (less(shifts[i], shifts[i_min])) i_min = i;
    if (less(shifts[i_max], shifts[i])) i_max = i;
  }
  Schedule s;
  if (shifts[i_min] == shifts[i_max]) {
    s.taus = {shifts[i_min]};
    s.pattern = {0};
  } else {
    s.taus = {shifts[i_min], shifts[i_max]};
    s.pattern = {0, 0, 0, 1, 1};
  }
  return s;
}

}  // namespace lt
