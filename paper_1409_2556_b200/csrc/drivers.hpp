#pragma once
#include <vector>

#include <cstdint>

#include <cuda_runtime.h>

#include "laptomo_gpu.h"

struct lt_split_s;

namespace lt {

extern thread_local std::vector<int> g_last_unconverged;

void forward(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
             const double* times, int n_times, int n_quad, const lt_talbot_params& contour, const lt_solver_config& cfg,
             bool pooled, int mem, double* heads_out, const double* receivers, int n_rec, double* drawdown_out,
             lt_time_diag* diag_out, double* shift_residuals);

void jacobian_slice(lt_pencil p, const lt_experiment& ex, int t, int mem, double* jac_out, double* pred_out);

// timestep.cu
void crank_nicolson(lt_pencil p, const double* sources, const double* rates, int n_src, const double* initial_head,
                    double dt, const double* sample_times, int n_samples, int mem, double* out, int* steps_out);
void condition_estimate(lt_pencil p, double2 z, double* norm_a, double* norm_inv, double* cond);

// gn.cu
void gn_step(lt_ctx ctx, const lt_gn_problem& pb, const double* s, const double* beta, const lt_gn_options& opt,
             double* s_out, double* beta_out, double* xi_out, lt_gn_stats* stats);
int gn_invert(lt_ctx ctx, const lt_gn_problem& pb, const double* s0, const double* beta0, const lt_gn_options& opt,
              double* s_hat, double* beta_hat, lt_gn_stats* history, int history_cap, int* converged, char* reason,
              int reason_cap);
double gn_objective(lt_ctx ctx, const lt_gn_problem& pb, const double* s, const double* beta, double* misfit,
                    double* prior);

// split build of one time slice
void split_solve(lt_split_s* sp);
void split_export(lt_split_s* sp, int plane0, int plane1, int m_pad, double2* dst, int mem);
void split_coefficients(lt_split_s* sp, double2* Y, int* m_used, int m_pad);
void split_predictions(lt_split_s* sp, double* out);
void jacobian_assemble_slab(lt_pencil p, const lt_experiment& ex, int t, int plane0, int plane1, int halo_lo,
                            int halo_hi, const double2* U, int m, const double2* Y, const int* m_used, int mem,
                            double* jac_out);

void sample_field_grid(lt_ctx ctx, int dim, const int* shape, double h, double variance, const double* corr,
                       double mean, uint64_t seed, const double2* noise, int mem, double* out);

}  // namespace lt
