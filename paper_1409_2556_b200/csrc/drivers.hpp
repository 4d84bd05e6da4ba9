#pragma once
#include <vector>

#include <cstdint>

#include <cuda_runtime.h>

#include "laptomo_gpu.h"

namespace lt {

extern thread_local std::vector<int> g_last_unconverged;

void forward(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
             const double* times, int n_times, int n_quad, const lt_talbot_params& contour, const lt_solver_config& cfg,
             bool pooled, int mem, double* heads_out, const double* receivers, int n_rec, double* drawdown_out,
             lt_time_diag* diag_out, double* shift_residuals);

void jacobian_slice(lt_pencil p, const lt_experiment& ex, int t, int mem, double* jac_out, double* pred_out);

void sample_field_grid(lt_ctx ctx, int dim, const int* shape, double h, double variance, const double* corr,
                       double mean, uint64_t seed, const double2* noise, int mem, double* out);

}  // namespace lt
