/*
 * laptomo_gpu.h — C ABI of the B200-native shifted-FGMRES / Laplace-THT hot path.
 *
 * Drop-in boundary for the reference's solver API (/root/reference/proj/include/laptomo).
 * Every entry point below names the reference interface it replaces (file:line).
 * Plain pointers and sizes only: complex numbers are interleaved (re, im) doubles,
 * layout-compatible with std::complex<double>, Eigen::VectorXcd data and CUDA double2.
 *
 * Conventions
 *  - Every call returns an lt_status; on failure lt_last_error() (thread-local) holds a
 *    message.  The reference's exceptions map to codes:
 *      std::invalid_argument  -> LT_ERR_INVALID_ARGUMENT
 *      FactorizationError     -> LT_ERR_PRECONDITIONER
 *      ConvergenceError       -> LT_ERR_NOT_CONVERGED  (indices via lt_last_unconverged)
 *  - One lt_ctx = one device + one CUDA stream.  Calls are synchronous at return.
 *    A handle is not thread-safe; distinct handles may be used concurrently.
 *  - `mem` arguments say where caller buffers live: LT_MEM_HOST or LT_MEM_DEVICE.
 *  - Multi-RHS buffers are RHS-major: rhs b occupies [b*n, (b+1)*n).
 *  - There is no CPU fallback: without a usable sm_100 device every compute call fails
 *    with LT_ERR_CUDA.
 */
#ifndef LAPTOMO_GPU_H
#define LAPTOMO_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} lt_complex;

typedef enum {
  LT_OK = 0,
  LT_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                      */
  LT_ERR_PRECONDITIONER = 2,   /* FactorizationError (errors.hpp:14-17)       */
  LT_ERR_NOT_CONVERGED = 3,    /* ConvergenceError (errors.hpp:20-25)         */
  LT_ERR_CUDA = 4,
  LT_ERR_OOM = 5,
  LT_ERR_INTERNAL = 6
} lt_status;

enum { LT_MEM_HOST = 0, LT_MEM_DEVICE = 1 };

/* KrylovVariant (shifted_solver.hpp:21) */
enum { LT_VARIANT_FOM = 0, LT_VARIANT_GMRES = 1 };
/* SolverKind (forward.hpp:16) */
enum { LT_SOLVER_SINGLE = 0, LT_SOLVER_FLEXIBLE = 1, LT_SOLVER_DIRECT = 2 };
/* Discretisations:
 *   FD_CELL = cell-centred finite volume (BASELINE configs), per-cell fields;
 *   P1_TRI  = the reference's own P1 FEM on build_mesh(n, L) (mesh.cpp:14-52,
 *             assembly.cpp:24-113): shape[0] = n_per_side nodes, h = L/(n-1), per-element
 *             fields (element 2c lower / 2c+1 upper triangle of cell c), unknowns = interior
 *             nodes in ascending node order (the reference's free dofs). */
enum { LT_GRID_FD_CELL = 0, LT_GRID_P1_TRI = 1 };

typedef struct lt_ctx_s* lt_ctx;
typedef struct lt_pencil_s* lt_pencil;

/* ---- library / context ------------------------------------------------------------- */
const char* lt_version(void);
const char* lt_last_error(void);
/* Unconverged shift indices of the last LT_ERR_NOT_CONVERGED (ConvergenceError::unconverged_shifts). */
int lt_last_unconverged(int* indices, int capacity);

lt_status lt_ctx_create(int device, lt_ctx* out);
lt_status lt_ctx_destroy(lt_ctx ctx);
lt_status lt_ctx_synchronize(lt_ctx ctx);
/* The cudaStream_t all work of this context is issued on. */
void* lt_ctx_stream(lt_ctx ctx);

/* Per-kernel-class device timing (CUDA events on the context stream) for roofline reporting. */
lt_status lt_ctx_set_profiling(lt_ctx ctx, int enabled);
lt_status lt_ctx_reset_profile(lt_ctx ctx);
/* Time only 1 in `every` launches of each kernel class (default 1) to keep the event
 * overhead out of long timed regions; lt_ctx_profile then scales each class's timed
 * launches to all of its launches (estimated totals; `launches` = all launches). */
lt_status lt_ctx_set_profile_sampling(lt_ctx ctx, int every);
/* Returns the number of kernel classes; fills up to `capacity` entries. name_buf holds
 * capacity*64 chars (NUL-terminated names). */
int lt_ctx_profile(lt_ctx ctx, int capacity, char* name_buf, double* total_ms, int64_t* launches,
                   double* algorithmic_bytes);
/* Total kernel launches issued by this context since creation / last reset. */
int64_t lt_ctx_launch_count(lt_ctx ctx);

/* ---- talbot (talbot.hpp:23-63; host arithmetic, no device work) ---------------------- */
typedef struct {
  double sigma0, mu0, nu, alpha; /* TalbotParams (talbot.hpp:23-28) */
} lt_talbot_params;

void lt_talbot_default_params(lt_talbot_params* out);
/* build_contour (talbot.cpp:49-80): n_quad/2 entries per output (any output may be NULL). */
lt_status lt_talbot_build(int n_quad, double time, const lt_talbot_params* params, double* thetas,
                          lt_complex* nodes, lt_complex* dnodes, lt_complex* weights);
/* qhat_step (talbot.cpp:96-101). */
lt_status lt_qhat_step(double q0, lt_complex z, lt_complex* out);
/* select_preconditioner_shifts (shifted_solver.cpp:85-104): taus[2], pattern[5]. */
lt_status lt_select_preconditioner_shifts(const lt_complex* shifts, int n_shifts, lt_complex* taus,
                                          int* n_taus, int* pattern, int* pattern_len);

/* ---- pencil (ShiftedPencil, shifted_solver.hpp:88-104; assemble, assembly.hpp:37-39) -- */
typedef struct {
  int kind;     /* LT_GRID_FD_CELL */
  int dim;      /* 2 or 3 */
  int shape[3]; /* cells along x, y, z (z ignored for dim 2); cell a = (k*ny + j)*nx + i */
  double h;     /* uniform spacing */
} lt_grid;

/* Assembles (K, M) on the device from per-cell log fields (host or device arrays of n
 * doubles) and builds the preconditioner hierarchy.  Replaces assemble() +
 * ShiftedPencil(K, M) (assembly.cpp:69-113, shifted_solver.cpp:106-107). */
lt_status lt_pencil_create_grid(lt_ctx ctx, const lt_grid* grid, const double* log_kappa,
                                const double* log_storativity, int mem, lt_pencil* out);
/* A compressed sparse matrix, 0-based: outer[n + 1] offsets, inner[nnz] indices, values[nnz].
 * Compressed rows (CSR) or, K and M being symmetric, compressed columns (the layout of Eigen's
 * default column-major SparseMatrix<double>); index_bytes = 4 (Eigen's int StorageIndex) or 8. */
typedef struct {
  const void* outer;
  const void* inner;
  const double* values;
  int index_bytes;
} lt_sparse;

/* ShiftedPencil(const SparseReal& K, const SparseReal& M) (shifted_solver.hpp:90,
 * shifted_solver.cpp:106-107) for an assembled pair on a declared structured grid: K, M host
 * matrices of n rows.  The device operator is matrix-free, so the pair is checked against the
 * grid's stencil and converted to its coefficients:
 *   LT_GRID_FD_CELL  K the 5-/7-point cell-centred operator, M diagonal (n = cells);
 *   LT_GRID_P1_TRI   the reference's assemble() pair on build_mesh(shape[0], L) interior nodes
 *                    (assembly.cpp:69-113; K's NE/SW hypotenuse entries zero), n = (shape[0]-2)^2.
 * Entries off the stencil, an asymmetric pair or a negative boundary coupling give
 * LT_ERR_INVALID_ARGUMENT.  The pencil then solves and applies exactly like a grid pencil (same
 * multigrid shift-and-invert, coarsened from the given operator); it carries no parameter
 * fields, so lt_jacobian / lt_predict need lt_pencil_create_grid. */
lt_status lt_pencil_create_csr(lt_ctx ctx, const lt_grid* grid, int64_t n, const lt_sparse* K,
                               const lt_sparse* M, lt_pencil* out);
lt_status lt_pencil_destroy(lt_pencil p);
int64_t lt_pencil_rows(lt_pencil p);
/* Number of per-parameter cells of the log fields: cells (FD) or elements (P1); 0 for a
 * pencil created from (K, M). */
int64_t lt_pencil_parameters(lt_pencil p);
int lt_pencil_levels(lt_pencil p);

/* (K + z M) x, (K + conj(z) M) x, M x for n_rhs RHS (shifted_solver.cpp:109-118). */
lt_status lt_pencil_apply(lt_pencil p, lt_complex z, const lt_complex* x, lt_complex* y,
                          int n_rhs, int mem);
lt_status lt_pencil_apply_adjoint(lt_pencil p, lt_complex z, const lt_complex* x, lt_complex* y,
                                  int n_rhs, int mem);
lt_status lt_pencil_apply_mass(lt_pencil p, const lt_complex* x, lt_complex* y, int n_rhs,
                               int mem);

/* The factorisation-cache analogue (ShiftedPencil::factorization, cpp:120-128): prepares
 * the exact shift-and-invert preconditioner for each tau (cached by exact value). */
lt_status lt_pencil_prepare(lt_pencil p, const lt_complex* taus, int n_taus);
int lt_pencil_factorization_count(lt_pencil p);
/* Inner-solve accuracy of the shift-and-invert preconditioner (relative residual). */
lt_status lt_pencil_set_inner_tolerance(lt_pencil p, double rel_tol, int max_iterations);
/* u = (K + tau M)^{-1} v  (SparseComplexFactorization::solve, factorization.hpp:23) and
 * u = (K + tau M)^{-H} v (solve_adjoint, factorization.hpp:25). */
lt_status lt_pencil_solve(lt_pencil p, lt_complex tau, const lt_complex* v, lt_complex* u,
                          int n_rhs, int mem);
lt_status lt_pencil_solve_adjoint(lt_pencil p, lt_complex tau, const lt_complex* v,
                                  lt_complex* u, int n_rhs, int mem);

/* Multilinear cell-centre weights of a point (FD analogue of point_source, mesh.cpp:91-125). */
lt_status lt_pencil_point_weights(lt_pencil p, const double* point, int64_t* indices,
                                  double* weights, int* count);

/* ---- shifted solver (shifted_solver.hpp:44-132) ------------------------------------- */
typedef struct {
  int variant;        /* LT_VARIANT_GMRES (default) | LT_VARIANT_FOM */
  double tol;         /* 1e-10 */
  int maxit;          /* 0 -> min(n, 10 n_shifts) */
  int keep_basis;     /* 0 */
  int record_history; /* 1 */
} lt_solve_options;

void lt_solve_default_options(lt_solve_options* out);

typedef struct {
  int converged;
  int iteration;        /* Arnoldi step at which the shift froze (1-based) */
  double estimate;      /* relative */
  double true_residual; /* relative, checked at freeze */
} lt_shift_status;

/* solve_shifted_flexible / solve_shifted_single (shifted_solver.cpp:291-322) for n_rhs
 * right-hand sides in lockstep, all with the same shifts and schedule.
 *   b         n * n_rhs
 *   x_out     n * n_shifts * n_rhs (RHS-major, then shift), may be NULL
 *   status    n_rhs * n_shifts, iterations n_rhs (both host, may be NULL)
 *   history   n_rhs * n_shifts * maxit estimates (host, NaN-padded), may be NULL
 * Never fails on non-convergence (like run_flexible): check status. */
lt_status lt_solve_shifted(lt_pencil p, const lt_complex* b, int n_rhs, const lt_complex* shifts,
                           int n_shifts, const lt_complex* taus, int n_taus, const int* pattern,
                           int pattern_len, const lt_solve_options* options, int mem,
                           lt_complex* x_out, lt_shift_status* status, int* iterations,
                           double* history);

/* FlexibleBasisState (shifted_solver.hpp:63-74) of the last lt_solve_shifted with
 * keep_basis = 1, for rhs index `rhs`.  Sizes: V n*(m+1), U n*m, Hbar (m+1)*m column-major,
 * taus m.  Pass NULL buffers to query m (steps_out) first. */
lt_status lt_last_basis(lt_pencil p, int rhs, int* steps_out, double* beta_out, lt_complex* V,
                        lt_complex* U, lt_complex* Hbar, lt_complex* taus);

/* residual_estimate (shifted_solver.cpp:334-343): |h_{m+1,m} (z - tau_m) y_m|, the FOM residual
 * norm, on a FlexibleBasisState as lt_last_basis returns it (Hbar (m+1) x m column-major, taus m)
 * for FOM coefficients y_fom of length y_len (must equal m >= 1).  Host arithmetic. */
lt_status lt_residual_estimate(const lt_complex* Hbar, const lt_complex* taus, int m, lt_complex z,
                               const lt_complex* y_fom, int y_len, double* out);

/* solve_shifted_direct (shifted_solver.cpp:324-332): one shift-and-invert solve per shift.
 * LT_ERR_NOT_CONVERGED (shift indices via lt_last_unconverged) if a solve ended above the
 * inner solve's floor (1e4 x its tolerance); x_out is written either way. */
lt_status lt_solve_shifted_direct(lt_pencil p, const lt_complex* b, int n_rhs,
                                  const lt_complex* shifts, int n_shifts, int mem,
                                  lt_complex* x_out);

/* ---- drivers (forward.hpp:52-61, jacobian.hpp:79-101) -------------------------------- */
typedef struct {
  int kind;    /* LT_SOLVER_* (SolverConfig, forward.hpp:18-23) */
  int variant; /* LT_VARIANT_* */
  double tol;
  int maxit;
} lt_solver_config;

void lt_solver_default_config(lt_solver_config* out);

typedef struct {
  int iterations;
  int all_converged;
} lt_time_diag;

/* solve_forward (forward.cpp:75-118) for n_src independent problems that share times,
 * n_quad, contour and solver (each its own source vector and rate), batched in lockstep.
 *   sources        n * n_src weight vectors (free dofs)
 *   initial_head   n * n_src or NULL (phi0 = 0)
 *   heads_out      n * n_times * n_src (per source: column t of HeadSolution.heads), or NULL
 *   receivers      n_rec receiver points (dim doubles each) -> drawdown_out
 *                  n_src * n_rec * n_times ((s*n_rec + r)*n_times + t), either may be NULL
 *   shift_residuals n_src * n_times * n_half (verified relative residual per shift), or NULL
 * pooled != 0 selects solve_forward_batch (forward.cpp:126-198).
 * Throws-equivalent: LT_ERR_NOT_CONVERGED when shifts fail to converge. */
lt_status lt_forward(lt_pencil p, const double* sources, const double* rates, int n_src,
                     const double* initial_head, const double* times, int n_times, int n_quad,
                     const lt_talbot_params* contour, const lt_solver_config* solver, int pooled,
                     int mem, double* heads_out, const double* receivers, int n_rec,
                     double* drawdown_out, lt_time_diag* diag_out, double* shift_residuals);

/* ThtExperiment (jacobian.hpp:22-42) with point coordinates (dim doubles per point). */
typedef struct {
  const double* sources;   /* n_src * dim */
  const double* rates;     /* n_src */
  int n_src;
  const double* receivers; /* n_rec * dim */
  int n_rec;
  const double* times;     /* n_times */
  int n_times;
  int n_quad;
  lt_talbot_params contour;
  lt_solver_config solver;
  int include_storativity;
  int storativity_z_factor;
} lt_experiment;

void lt_experiment_defaults(lt_experiment* out);

/* One time slice of ThtForwardModel::jacobian (jacobian.cpp:189-247) on the pencil's
 * fields: rows (s*n_rec + r) of the slice, row-major, n_param = n (kappa block) or 2n
 * (storativity block appended).  jac_out is n_src*n_rec*n_param doubles (host or device
 * per `mem`), predictions_out n_src*n_rec (host).  Either may be NULL. */
lt_status lt_jacobian_slice(lt_pencil p, const lt_experiment* exp, int time_index, int mem,
                            double* jac_out, double* predictions_out);

/* Full ThtForwardModel::jacobian: J n_meas x n_param row-major in the reference's row
 * order (s*n_rec + r)*n_times + t (jacobian.hpp:37-41), predictions n_meas.  Host only. */
lt_status lt_jacobian(lt_pencil p, const lt_experiment* exp, double* jac_out,
                      double* predictions_out);

/* ThtForwardModel::predict (jacobian.cpp:158-187): n_meas predictions. */
lt_status lt_predict(lt_pencil p, const lt_experiment* exp, double* predictions_out);

/* ---- time stepping and conditioning (forward.hpp:63-68, shifted_solver.hpp:141-149) ---- */
/* crank_nicolson (forward.cpp:200-258): (M + dt/2 K) h_{n+1} = (M - dt/2 K) h_n + dt q b from
 * h_0 = initial_head (NULL: zero) until the last sample time, for n_src problems in lockstep
 * (sources n x n_src weights, rates n_src); samples_out[(s n_samples + i) n + a] = the head at
 * sample_times[i] (linear interpolation between the two steps around it, as the reference).
 * The step solve is the pencil's shift-and-invert at tau = 2/dt (the reference's LDLT of
 * M + dt/2 K); steps_out may be NULL.  dt <= 0 or no sample times: LT_ERR_INVALID_ARGUMENT. */
lt_status lt_crank_nicolson(lt_pencil p, const double* sources, const double* rates, int n_src,
                            const double* initial_head, double dt, const double* sample_times,
                            int n_samples, int mem, double* samples_out, int* steps_out);
/* estimate_condition_1norm (condest.cpp:11-49) of A = K + z M: Hager 1-norm lower bounds of A
 * (apply / apply_adjoint) and of A^{-1} (shift-and-invert solve / its adjoint) and their
 * product (never above kappa_1(A)); any output may be NULL. */
lt_status lt_pencil_condest(lt_pencil p, lt_complex z, double* norm_a, double* norm_inv, double* cond);

/* ---- Gauss-Newton step of the geostatistical inversion (inversion.hpp:17-91) ----------
 * InversionProblem: y (n_y), r_diag (n_y, > 0), drift X (n_s x p, column-major like Eigen) and
 * the prior Q, either dense (prior != NULL: n_s x n_s, the reference's matrix; jittered
 * Cholesky for the prior term) or, prior == NULL, a stationary exponential covariance
 * variance[b] exp(-|(dx/l0, dy/l1, dz/l2)|) between the cells of `grid` for each of n_blocks
 * parameter blocks (s = [block 0 cells, block 1 cells]: log kappa then log S), applied exactly by
 * FFT (Q J^T) and inverted by CG for the prior term.  The forward handles are
 * callbacks (InversionProblem::predict / jacobian_and_predict, inversion.hpp:25-26): s and h
 * are host arrays, J_out a DEVICE buffer of n_y x n_s doubles (row-major, rows in y's order),
 * e.g. filled by lt_jacobian_slice with LT_MEM_DEVICE; a nonzero return is raised as that
 * lt_status.                                                                             */
typedef int (*lt_predict_fn)(void* user, const double* s, double* h_out);
typedef int (*lt_jacobian_fn)(void* user, const double* s, double* J_out_device, double* h_out);
typedef struct {
  int n_y, n_s, p;
  const double* y;
  const double* r_diag;
  const double* drift;
  const double* prior;
  lt_grid grid;
  int n_blocks;
  double variance[2];
  double corr[2][3];
  lt_predict_fn predict;
  lt_jacobian_fn jacobian_and_predict;
  void* user;
} lt_gn_problem;

typedef struct { /* GnOptions (inversion.hpp:29-34) */
  int max_gn;       /* 15 */
  double rtol;      /* 1e-3 */
  int damping;      /* 1 */
  int max_halvings; /* 5 */
} lt_gn_options;

typedef struct { /* GnIterate scalars (inversion.hpp:36-47) */
  double objective, misfit, prior, step_norm, alpha, saddle_residual, drift_violation;
} lt_gn_stats;

void lt_gn_default_options(lt_gn_options* out);
/* GaussNewtonSolver::step (inversion.cpp:78-148): s_out (n_s), beta_out (p), xi_out (n_y or NULL). */
lt_status lt_gn_step(lt_ctx ctx, const lt_gn_problem* problem, const double* s, const double* beta,
                     const lt_gn_options* options, double* s_out, double* beta_out, double* xi_out,
                     lt_gn_stats* stats);
/* GaussNewtonSolver::invert (inversion.cpp:150-186): returns the number of steps taken in
 * *steps_out; history (max_gn entries) may be NULL; reason is the stop_reason (NUL-terminated). */
lt_status lt_gn_invert(lt_ctx ctx, const lt_gn_problem* problem, const double* s0, const double* beta0,
                       const lt_gn_options* options, double* s_hat, double* beta_hat, lt_gn_stats* history,
                       int* steps_out, int* converged, char* reason, int reason_capacity);
/* GaussNewtonSolver::objective = misfit(predict(s)) + prior_term(s, beta) (inversion.cpp:58-76). */
lt_status lt_gn_objective(lt_ctx ctx, const lt_gn_problem* problem, const double* s, const double* beta,
                          double* objective, double* misfit, double* prior);

/* ---- split build of one Jacobian time slice across ranks -------------
 * The rows of jacobian.cpp:205-246 are independent, and each needs phi_s and psi_r on the same
 * cells: one rank per GPU solves a contiguous range of the slice's items (sources, then
 * receivers: the lockstep batch of lt_jacobian_slice) and keeps their bases; the caller moves
 * every z-slab's basis rows (the slab's planes plus one halo plane on each interior side) to
 * the slab's owner in one all-to-all (NCCL over NVLink; paper_1409_2556_b200/split_build.py);
 * each rank then assembles the J columns of its slab.  J rows need no reduction.
 * Planes are z-planes (3-D) or rows (2-D) of the FD grid pencil.                           */
typedef struct lt_split_s* lt_split;
/* Solves items [item0, item1) of time slice `time_index` (ConvergenceError like
 * lt_jacobian_slice). */
lt_status lt_split_solve(lt_pencil p, const lt_experiment* exp, int time_index, int item0, int item1,
                         lt_split* out);
/* m: basis columns of this part (the all-to-all pads every part to the max over ranks). */
int lt_split_columns(lt_split s);
/* Y[(b ns + k) m_pad + j] (zero for j >= m_used), m_used[b ns + k] for this part's items
 * (host arrays; ns = n_quad / 2). */
lt_status lt_split_coefficients(lt_split s, int m_pad, lt_complex* Y, int* m_used);
/* Basis rows of planes [plane0, plane1): dst[(j (item1-item0) + b) cells + a'], j < m_pad
 * (zero columns past this part's m), cells = (plane1-plane0) x plane size; host or device. */
lt_status lt_split_export(lt_split s, int plane0, int plane1, int m_pad, lt_complex* dst, int mem);
/* Predictions (jacobian.cpp:241-244) of this part's sources at every receiver: (s, r) row-major
 * over the part's sources (none if the part holds only receivers). */
lt_status lt_split_predictions(lt_split s, double* predictions_out);
lt_status lt_split_destroy(lt_split s);
/* The J columns of slab [plane0, plane1) from every item's basis rows over the slab and its
 * halo planes (planes plane0 - (plane0 > 0) .. plane1 + (plane1 < planes)):
 *   U_slab[(j B + b) view_cells + a'], B = n_src + n_rec, j < m;  Y, m_used as
 *   lt_split_coefficients over all B items (host);
 *   jac_out rows (s n_rec + r), kappa block then storativity block, n_slab columns each. */
lt_status lt_jacobian_assemble_slab(lt_pencil p, const lt_experiment* exp, int time_index, int plane0,
                                    int plane1, const lt_complex* U_slab, int m, const lt_complex* Y,
                                    const int* m_used, int mem, double* jac_out);

/* ---- fields (sample_field / sample_field_on_mesh, fields.hpp:27-44, fields.cpp:84-123) --
 * The reference draws mean + C zeta with C C^T = Q, Q the dense exponential covariance over
 * the element centres (Cholesky).  On a structured grid this draws the same Gaussian law by
 * circulant embedding on a torus twice the grid (cuFFT): covariance variance *
 * exp(-|(dx/l0, dy/l1, dz/l2)|) between cell centres (isotropic: equal lengths), grid spacing
 * h, shape[dim] cells, out = n cells (x fastest; host or device per `mem`).  noise == NULL:
 * complex standard normals from Philox(seed); else prod(2 shape) complex standard normals
 * (x fastest over the doubled grid, same `mem`), the deterministic path. */
lt_status lt_sample_field_grid(lt_ctx ctx, int dim, const int* shape, double h, double variance,
                               const double* corr_lengths, double mean, uint64_t seed,
                               const lt_complex* noise, int mem, double* out);

#ifdef __cplusplus
}
#endif

#endif /* LAPTOMO_GPU_H */
