#pragma once
#include <complex>
#include <vector>

#include "laptomo_gpu.h"

namespace lt {

struct Schedule {
  std::vector<std::complex<double>> taus;
  std::vector<int> pattern;
  std::complex<double> tau_at(int j) const { return taus[pattern[j % pattern.size()]]; }
};

void talbot_build(int n_quad, double time, const lt_talbot_params& p, std::vector<double>* thetas,
                  std::vector<std::complex<double>>* nodes, std::vector<std::complex<double>>* dnodes,
                  std::vector<std::complex<double>>* weights);

Schedule select_schedule(const std::vector<std::complex<double>>& shifts);

}  // namespace lt
