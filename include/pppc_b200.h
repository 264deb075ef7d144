/*
 * pppc_b200.h — C ABI of the B200-native PP-PC hot path.
 *
 * The reference (`parasteady`, /root/reference/proj) is an in-process C++ library
 * with no FFI; its hot path sits behind these C++ entry points, each of which is
 * replaced by one or more functions below (reference file:line in brackets):
 *
 *   PeriodicProblem(M, K_fn, J_fn, excitation)      [proj/include/parasteady/problem.hpp:74-104]
 *        -> ps_problem_desc + ps_create
 *   newton_step(problem, u_prev, t_next, dt, s)     [proj/include/parasteady/propagators.hpp:39-40,
 *                                                    proj/src/propagators.cpp:27-58]
 *        -> ps_newton_step
 *   Propagator::fine_propagate(n, u)                [proj/include/parasteady/propagators.hpp:59,
 *                                                    proj/src/propagators.cpp:102-115]
 *        -> ps_fine_propagate_batch (all subintervals in one call; replaces the
 *           parallel_for at proj/src/engine.cpp:226-227)
 *   Propagator::coarse_propagate(n, u)              [proj/include/parasteady/propagators.hpp:58,
 *                                                    proj/src/propagators.cpp:96-100]
 *        -> ps_coarse_propagate_batch (replaces proj/src/engine.cpp:231-232 and :216)
 *   frozen_coarse_linearization(problem, ref)       [proj/src/engine.cpp:66-74]
 *        -> ps_create_frozen
 *   make_cyclic_system / MultiharmonicCyclicSolver  [proj/src/spectral.cpp:118-132, 233-255]
 *        -> ps_mh_setup
 *   assemble_rhs(F, G, sys, problem, mesh)          [proj/src/spectral.cpp:134-150]
 *        -> ps_assemble_rhs
 *   MultiharmonicCyclicSolver::solve(rhs)           [proj/src/spectral.cpp:257-279]
 *        -> ps_mh_solve
 *   forward_dft / inverse_dft                       [proj/src/spectral.cpp:105-116]
 *        -> ps_forward_dft / ps_inverse_dft
 *   jump_norm(current, previous)                    [proj/src/engine.cpp:54-64]
 *        -> ps_jump_norm (and fused into ps_pppc_correct)
 *   solve_pp_pc(problem, settings, Multiharmonic)   [proj/src/engine.cpp:187-270]
 *        -> ps_pppc_solve (host C++ driver over the calls above)
 *   fine_periodicity_defect(problem, traj, mesh)    [proj/src/engine.cpp:272-290]
 *        -> ps_fine_periodicity_defect
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *   - Host-array functions take states in the reference's order: [count][dim]
 *     (one StateVector per subinterval, time-major).  `_dev` variants take device
 *     pointers in the same order.  Internally the library keeps every batch
 *     interleaved [dim][count] (system index fastest) in HBM.
 *   - Every function returns PS_OK (0) or a PS_ERR_* code; no exception crosses
 *     the ABI.  ps_last_error(ctx) returns the reference-style message
 *     (e.g. "propagator: Newton did not converge at t = 0.005 (residual 1e-3)").
 *   - All arithmetic is IEEE fp64.  Results do not depend on `count` or on how a
 *     batch is split (bitwise), mirroring the worker-count independence contract
 *     of proj/tests/test_engine.cpp:253-271.
 *   - There is no CPU fallback: on a machine without a usable sm_100 device every
 *     compute entry point fails with PS_ERR_CUDA.
 */
#ifndef PPPC_B200_H
#define PPPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ codes */
enum {
  PS_OK = 0,
  PS_ERR_BAD_ARG = 1,           /* invalid argument (message says which) */
  PS_ERR_NEWTON_MAXITER = 2,    /* "propagator: Newton did not converge"  propagators.cpp:57 */
  PS_ERR_NEWTON_DIVERGED = 3,   /* "propagator: Newton iteration diverged" propagators.cpp:54 */
  PS_ERR_SINGULAR = 4,          /* "propagator: step system singular"      propagators.cpp:46,92 */
  PS_ERR_PCG_MAXITER = 5,       /* "propagator: PCG did not converge" (new: iterative solver) */
  PS_ERR_NONFINITE = 6,         /* "spectral: harmonic solve produced non-finite values" spectral.cpp:266 */
  PS_ERR_ODD_BLOCKS = 7,        /* "spectral: ... requires an even number of blocks" spectral.cpp:86-90 */
  PS_ERR_SINGULAR_BLOCK = 8,    /* "spectral: harmonic block p = k is singular"    spectral.cpp:248-251 */
  PS_ERR_CONJ_SYMMETRY = 9,     /* "spectral: conjugate symmetry violated"        spectral.cpp:78-80 */
  PS_ERR_CUDA = 10,             /* CUDA runtime error / no device */
  PS_ERR_NOT_LINEAR = 11,       /* "spectral: cyclic system requires a linear problem (freeze ...)" spectral.cpp:119-121 */
  PS_ERR_NOT_SETUP = 12,        /* multiharmonic solve before ps_mh_setup */
  PS_ERR_COCG_MAXITER = 13,     /* "spectral: COCG did not converge" (new: iterative solver) */
  PS_ERR_WATCHDOG = 14          /* device-side barrier watchdog fired (should never happen) */
};

/* ---------------------------------------------------------- problem data */
/* Reluctivity curve [proj/include/parasteady/problem.hpp:43-60, proj/src/problem.cpp:65-98]:
 * kind 0: constant nu; kind 1: Brauer nu(B^2) = min(k1*exp(min(k2*B^2,700)) + k3, 1/mu0). */
typedef struct {
  int32_t kind;
  int32_t pad_;
  double nu;
  double k1, k2, k3;
} ps_curve;

/* Structured description of  M u' + K(u) u = f(t),  u(0) = u(T)
 * [proj/include/parasteady/problem.hpp:74-104].  The opaque std::function
 * assembly callbacks of the reference cannot be offloaded, so the operator is
 * given by its elements instead:
 *     K(u) = sum_e nu(b2_e) S_e,   b2_e = u_e^T S_e u_e * inv_area_e,
 *     J(u) = sum_e nu S_e + 2 nu'(b2_e) inv_area_e (S_e u_e)(S_e u_e)^T.
 * With 2-node elements S_e = w[[1,-1],[-1,1]], inv_area = 1/(w h^2) this is the
 * reference's radial cable (proj/src/problem.cpp:204-237, 344-359) exactly; with
 * 3-node P1 triangles it is the 2-D cable of BASELINE.json.
 * A problem is linear iff `stiffness` != NULL (then the element fields are ignored). */
typedef struct {
  int32_t dim;                 /* d: free DOFs */
  int32_t nnz;                 /* CSR nonzeros of the (symmetric) step-matrix pattern */
  const int32_t* row_ptr;      /* [dim+1] */
  const int32_t* col_idx;      /* [nnz], sorted per row, includes the diagonal */
  const double* mass;          /* [nnz] M on the pattern */
  const double* stiffness;     /* [nnz] constant K (linear problems) or NULL */
  int32_t n_elem;              /* nonlinear problems: elements */
  int32_t nodes_per_elem;      /* 2 or 3 */
  const int32_t* elem_nodes;   /* [n_elem*npe], -1 = Dirichlet (eliminated) node */
  const double* elem_stiff;    /* [n_elem*npe*npe] unit stiffness S_e, row-major, symmetric */
  const double* elem_inv_area; /* [n_elem] */
  const int32_t* elem_curve;   /* [n_elem] index into curves */
  int32_t n_curves;
  int32_t pad_;
  const ps_curve* curves;      /* [n_curves] */
  /* excitation f(t) = sum_k amplitude_k sin(2 pi freq_k tau + phase_k) pattern_k,
   * tau = fmod(t, T) [proj/src/problem.cpp:36-63] */
  double period;
  int32_t n_terms;
  int32_t pad2_;
  const double* patterns;      /* [n_terms*dim] */
  const double* amplitude;     /* [n_terms] */
  const double* frequency_hz;  /* [n_terms] */
  const double* phase_rad;     /* [n_terms] */
} ps_problem_desc;

/* TimeMesh [proj/include/parasteady/types.hpp:21-40] */
typedef struct {
  int32_t subintervals; /* N */
  int32_t fine_steps;   /* s */
  double period;        /* T */
} ps_time_mesh;

/* NewtonSettings [proj/include/parasteady/propagators.hpp:19-24] (same defaults) */
typedef struct {
  double tol_abs;   /* 1e-9 */
  double tol_rel;   /* 1e-8 */
  int32_t max_iter; /* 30 */
  /* Extension (default 0 = the reference's update u += damping*delta): up to
   * `line_search` step halvings until ||R(u)|| <= (1 - 1e-4 lambda) ||R_pre||.
   * Needed for the deep-saturation BASELINE configs, where the undamped Newton of
   * proj/src/propagators.cpp:27-58 enters a 2-cycle across the nu = 1/mu0 cap. */
  int32_t line_search;
  double damping;   /* 1.0 */
} ps_newton_settings;

typedef struct {
  double tol_rel;     /* stop at ||r||_2 <= tol_rel * ||b||_2 (1e-12) */
  int32_t max_iter;   /* 20000 */
  int32_t warm_start; /* COCG only: start each multiharmonic solve of a context from the
                         solution of its previous successful solve (0 = from zero; the
                         reference's direct solve has no start value) */
} ps_krylov_settings;

typedef struct {
  ps_newton_settings newton;
  ps_krylov_settings pcg;   /* Jacobi-PCG for every step system (replaces SimplicialLDLT) */
  ps_krylov_settings cocg;  /* Jacobi-COCG per harmonic block (replaces complex SparseLU) */
  int32_t max_batch;        /* systems resident per batch (0 = subintervals) */
  int32_t engine;           /* fine batches of nonlinear element problems: 0 = by size (one
                               thread-block cluster per system when its vectors fit in a cluster's
                               shared memory, else one block per system when they fit in one
                               block's, else one warp lane per system), 1 = lane engine,
                               2 = block engine, 3 = cluster engine */
} ps_solver_settings;

/* Outcome of one batched call.  On error `code` != PS_OK and `failed_index`
 * is the lowest failing batch member (deterministic), like the reference's
 * first-exception rethrow (proj/include/parasteady/parallel.hpp:23-40). */
typedef struct {
  int32_t code;
  int32_t failed_index;
  double t_next;                 /* time of the failing step */
  double residual;               /* last residual norm of the failing system */
  int64_t newton_iterations;     /* summed over systems and steps */
  int64_t pcg_iterations;        /* summed over systems, steps and Newton iterations */
  int32_t max_newton_iterations; /* max over single steps */
  int32_t max_pcg_iterations;    /* max over single solves */
  int64_t lockstep_pcg_iterations; /* batched iterations executed (lock-step, summed over groups) */
  double algorithmic_bytes;      /* canonical bytes of the call's kernels */
  double kernel_ms;              /* device time of the call's compute kernels (CUDA events) */
} ps_batch_status;

typedef struct ps_ctx ps_ctx;

/* ---------------------------------------------------------------- context */
/* stream: a cudaStream_t to launch on (NULL = the library creates one). */
int ps_create(const ps_problem_desc* problem, const ps_time_mesh* mesh,
              const ps_solver_settings* settings, void* stream, ps_ctx** out);
void ps_destroy(ps_ctx* ctx);
const char* ps_last_error(const ps_ctx* ctx);
/* Which engine ran the context's last propagation (1 lane, 2 block, 3 cluster; 0 =
 * none yet) and, for the cluster engine, the CTAs per cluster and the clusters
 * the device holds at once.  Diagnostics for the bench line; any pointer may be NULL. */
int ps_last_engine(const ps_ctx* ctx, int32_t* engine, int32_t* cluster_ctas, int32_t* coresident_clusters);
/* Error string for failures that happen before a context exists. */
const char* ps_global_error(void);
int ps_dim(const ps_ctx* ctx);
int ps_is_linear(const ps_ctx* ctx);
/* Linear surrogate K = K(u_ref) (u_ref NULL => zero state) sharing mesh and settings
 * [proj/src/engine.cpp:66-74]; linear problems are copied through unchanged. */
int ps_create_frozen(ps_ctx* ctx, const double* u_ref, ps_ctx** out);
int ps_default_settings(ps_solver_settings* out);
int ps_device_info(char* name, int name_len, int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------ propagation */
/* newton_step for `count` independent systems, each with its own t_next
 * [proj/src/propagators.cpp:27-58].  iterations/residual_norms may be NULL;
 * residual_norms is [count][newton.max_iter] (post-update norms, zero-padded). */
int ps_newton_step(ps_ctx* ctx, int32_t count, const double* U_prev, const double* t_next,
                   double dt, double* U_out, int32_t* iterations, double* residual_norms,
                   ps_batch_status* status);
/* F_n for n = n_first .. n_first+count-1 (1-based, like the reference),
 * U_start[i] = state at T_{n-1}; U_end[i] = F_n(U_start[i]). */
int ps_fine_propagate_batch(ps_ctx* ctx, int32_t n_first, int32_t count, const double* U_start,
                            double* U_end, ps_batch_status* status);
int ps_fine_propagate_batch_dev(ps_ctx* ctx, int32_t n_first, int32_t count,
                                const double* dU_start, double* dU_end, ps_batch_status* status);
/* G_n: one implicit-Euler step of dT = T/N to boundary(n). */
int ps_coarse_propagate_batch(ps_ctx* ctx, int32_t n_first, int32_t count, const double* U_start,
                              double* U_end, ps_batch_status* status);
int ps_coarse_propagate_batch_dev(ps_ctx* ctx, int32_t n_first, int32_t count,
                                  const double* dU_start, double* dU_end, ps_batch_status* status);
/* Initial PP-PC iterate: U[0] = 0, U[n] = G_n(U[n-1]) for n = 1..N-1
 * [proj/src/engine.cpp:213-218].  U is [N][dim]. */
int ps_coarse_sweep(ps_ctx* ctx, double* U, ps_batch_status* status);

/* K(u) and J(u) values on the CSR pattern for `count` states (diagnostics / KATs)
 * [proj/src/problem.cpp:136-144, 344-359].  Either output may be NULL. [count][nnz]. */
int ps_assemble_operators(ps_ctx* ctx, int32_t count, const double* U, double* K_values,
                          double* J_values);
/* f(t) for `count` times [proj/src/problem.cpp:52-63]; out is [count][dim]. */
int ps_eval_excitation(ps_ctx* ctx, int32_t count, const double* t, double* out);

/* --------------------------------------------------------------- spectral */
/* Bin set for the multiharmonic solve: bins 0..N/2 (conjugate symmetry, reference
 * default) or 0..N-1; `bin_mask` (length N, NULL = all) zeroes unsolved bins
 * (the opt-in odd-harmonic truncation of BASELINE.json).
 * shift_kind 0 = reference block Q - exp(-2 pi i p/N) C [spectral.cpp:224-231];
 * shift_kind 1 = continuous K + j w_p M (BASELINE wording, variant only). */
int ps_mh_setup(ps_ctx* linear_ctx, int32_t use_conjugate_symmetry, const int32_t* bin_mask,
                int32_t shift_kind);
/* rhs_row = Q (F_sub - G_sub) + f(T_sub), sub = row == 0 ? N : row. [N][dim] arrays. */
int ps_assemble_rhs(ps_ctx* linear_ctx, const double* F, const double* G, double* rhs);
int ps_mh_solve(ps_ctx* linear_ctx, const double* rhs, double* U, ps_batch_status* status);
/* The PP-PC correction: assemble_rhs -> multiharmonic solve -> jump_norm, in place on U. */
int ps_pppc_correct(ps_ctx* linear_ctx, const double* F, const double* G, double* U_inout,
                    double* jump, ps_batch_status* status);
/* Unitary DFT across n blocks of d components; spectrum is [n][d][2] (re, im), bins in
 * FFT order [proj/src/spectral.cpp:32-63].  ps_inverse_dft fails with
 * PS_ERR_CONJ_SYMMETRY when the imaginary residue exceeds 1e-8*max(1, max|re|). */
int ps_forward_dft(int32_t n, int32_t d, const double* U, double* spectrum);
int ps_inverse_dft(int32_t n, int32_t d, const double* spectrum, double* U);
/* max_n ||cur_n - prev_n|| / max(1, max_n ||cur_n||) on the device. */
int ps_jump_norm(int32_t count, int32_t d, const double* cur, const double* prev, double* out);
/* Brauer / constant curve evaluation (device code path), for KATs. */
int ps_eval_reluctivity(const ps_curve* curve, int32_t n, const double* b2, double* nu,
                        double* nu_prime);

/* ----------------------------------------------------------------- driver */
typedef struct {
  double tol;                      /* 1e-6  [proj/include/parasteady/engine.hpp:60] */
  int32_t max_iterations;          /* 50 */
  int32_t use_conjugate_symmetry;  /* 1 */
  const int32_t* bin_mask;         /* NULL = every bin */
  int32_t shift_kind;              /* 0 = reference */
  int32_t pad_;
} ps_engine_settings;

#define PS_MAX_HISTORY 256
typedef struct {
  int32_t iterations;              /* PP-PC iterations performed */
  int32_t converged;
  double jumps[PS_MAX_HISTORY];
  double fine_ms, coarse_ms, spectral_ms, total_ms;
  int64_t fine_pcg_iterations, coarse_pcg_iterations, cocg_iterations, newton_iterations;
  double fine_bytes;               /* canonical algorithmic bytes of the fine kernels */
  double final_defect;             /* PP-IC: relative_defect(u_N, u_0) of the last iterate */
  int64_t cocg_per_iteration[PS_MAX_HISTORY];  /* PP-PC: COCG iterations (all bins) per iteration */
  double fine_ms_per_iteration[PS_MAX_HISTORY];
  double spectral_ms_per_iteration[PS_MAX_HISTORY];
} ps_history;

/* solve_pp_pc with the multiharmonic coarse solver [proj/src/engine.cpp:187-270].
 * frozen_ref NULL = zero state.  U_out is [N][dim] (states at T_0..T_{N-1}).
 * iterates (optional, [max_iterations][N][dim]) receives every iterate U^k. */
int ps_pppc_solve(ps_ctx* fine_ctx, const ps_engine_settings* settings, const double* frozen_ref,
                  double* U_out, double* iterates, ps_history* history);
int ps_fine_periodicity_defect(ps_ctx* ctx, const double* U, double* defect);

/* classic_parareal [proj/src/engine.cpp:76-129]: initial-value Parareal from u0
 * (dim) with the context's own problem as fine and coarse propagator.  U_out
 * is [N+1][dim] (states at T_0..T_N); iterates (or NULL) [max_iterations][N+1][dim]. */
int ps_classic_parareal(ps_ctx* ctx, const ps_engine_settings* settings, const double* u0,
                        double* U_out, double* iterates, ps_history* history);
/* solve_pp_ic [proj/src/engine.cpp:131-185]: periodic Parareal with initial-value
 * relaxation u_0 <- u_N; converged when jump and relative_defect(u_N, u_0) are
 * both <= tol.  U_out is [N][dim] (T_0..T_{N-1}); iterates [k][N+1][dim]. */
int ps_pp_ic_solve(ps_ctx* ctx, const ps_engine_settings* settings, double* U_out,
                   double* iterates, ps_history* history);
/* sequential_steady_state [proj/src/propagators.cpp:117-149]: U_out [N][dim] holds
 * the last period's states T_0..T_{N-1}; defects (or NULL) [max_periods]. */
int ps_sequential_steady_state(ps_ctx* ctx, double tol, int32_t max_periods, double* U_out,
                               int32_t* periods, int32_t* converged, double* defects);

/* Diagnostics: time one PCG phase of the last nonlinear propagation's batch as a
 * standalone (ncu-replayable) kernel: mode 1 = SpMV phase, 2 = update phase,
 * 3 = the update phase's streams as a flat copy.  bytes_out = the phase's bytes
 * by the SURVEY.md §8d stream count. */
int ps_phase_probe(ps_ctx* ctx, int32_t mode, int32_t reps, double* ms_out, double* bytes_out);

/* Test probes of the hot-path kernels themselves (not of a whole solve).
 * ps_refill_probe: one fused refill (refill_row_ell / refill_long_rows /
 *   refill_finish inside the persistent propagation kernel) of `count` systems
 *   at (U, U_prev, t_next, dt): A = M/dt + J(U) [count][nnz], R = M (U - U_prev)/dt
 *   + K(U) U - f(t_next) [count][dim], Dinv = 1/diag(A) [count][dim]; any output
 *   may be NULL [proj/src/propagators.cpp:13-17, proj/src/problem.cpp:344-359].
 * ps_mh_bins: the solved bins of the context's spectral setup (returns their
 *   count, or minus an error code).
 * ps_mh_forward: dft_forward_kernel, rhs [N][dim] -> spectrum [H][dim] complex
 *   (re, im pairs) on the solved bins [proj/src/spectral.cpp:32-63].
 * ps_mh_inverse: idft_jump_kernel + jump_finalize_kernel, spectrum [H][dim] ->
 *   mirrored, realified U [N][dim] and jump_norm against U_old (or NULL)
 *   [proj/src/spectral.cpp:72-84,270-278, proj/src/engine.cpp:54-64]. */
int ps_refill_probe(ps_ctx* ctx, int32_t count, const double* U, const double* U_prev,
                    const double* t_next, double dt, double* A_out, double* R_out, double* Dinv_out);
int ps_mh_bins(ps_ctx* ctx, int32_t* bins, int32_t cap);
int ps_mh_forward(ps_ctx* ctx, const double* rhs, double* spectrum);
int ps_mh_inverse(ps_ctx* ctx, const double* spectrum, const double* U_old, double* U, double* jump);

/* --------------------------------------------------------------- builders */
typedef struct ps_problem ps_problem;
/* 2-D structured polar P1 cable (BASELINE.json configs). */
typedef struct {
  int32_t nr, ntheta;
  double radius;                  /* outer (Dirichlet) radius, 5e-3 */
  double r_conductor;             /* 2e-3 */
  double r_insulator;             /* 4e-3 */
  double sigma_conductor;         /* 5.8e7 */
  double sigma_insulator;         /* 0 */
  double sigma_sheath;            /* 1e6 */
  double brauer_k1, brauer_k2, brauer_k3; /* 3.8, 2.17, 396.2 */
  int32_t linear_sheath;          /* freeze the sheath at nu(0) = k1 + k3 */
  int32_t return_in_sheath;       /* 1: -unit current in the sheath */
  double current;                 /* I0 = 2000 A */
  double frequency_hz;            /* 50 */
  int32_t ripple_terms;           /* odd-harmonic square-ripple terms (config 4: 5) */
  int32_t pad_;
  double ripple_fraction;         /* 0.1 */
  double ripple_frequency_hz;     /* 1000 */
} ps_polar_cable_params;
int ps_polar_cable_defaults(ps_polar_cable_params* p);
int ps_build_polar_cable(const ps_polar_cable_params* params, ps_problem** out);

/* The reference's own 1-D radial coax cable, CoaxCableParams
 * [proj/include/parasteady/problem.hpp:122-144, proj/src/problem.cpp:242-361]. */
typedef struct {
  int32_t n_r;
  int32_t source_region;
  double r1, r2, r3;
  double sigma_wire, sigma_sleeve, sigma_shield;
  double brauer_k1, brauer_k2, brauer_k3;
  int32_t linear_sleeve;
  int32_t pad_;
  double current;
  double frequency_hz;
} ps_radial_cable_params;
int ps_radial_cable_defaults(ps_radial_cable_params* p);
int ps_build_radial_cable(const ps_radial_cable_params* params, ps_problem** out);
const ps_problem_desc* ps_problem_get_desc(const ps_problem* p);
/* node coordinates (x, y) of the free DOFs, [dim][2] (polar builder only; NULL otherwise) */
const double* ps_problem_coordinates(const ps_problem* p);
void ps_problem_free(ps_problem* p);
/* Error message of the last failed builder call on this thread. */
const char* ps_builder_error(void);
/* Seeded N(0, sigma^2) samples: std::mt19937_64(seed) + explicit Box-Muller. */
/* Files (host C++, no device work).
 * Matrix Market [proj/src/matrix_market.cpp:30-93]: coordinate real general or
 * symmetric storage, duplicates summed; written in column-major entry order with
 * shortest round-trip values.  Errors: ps_builder_error(). */
typedef struct ps_csr ps_csr;
int ps_mm_read(const char* path, ps_csr** out);
int ps_csr_shape(const ps_csr* m, int32_t* rows, int32_t* cols, int64_t* nnz);
const int32_t* ps_csr_row_ptr(const ps_csr* m);
const int32_t* ps_csr_col_idx(const ps_csr* m);
const double* ps_csr_values(const ps_csr* m);
void ps_csr_free(ps_csr* m);
int ps_mm_write(const char* path, int32_t rows, int32_t cols, const int32_t* row_ptr, const int32_t* col_idx,
                const double* values);
/* load_problem [proj/src/problem.cpp:363-421]: linear problem from M, K Matrix
 * Market files and the excitation JSON (parse_excitation_text's schema). */
int ps_load_problem(const char* mass_path, const char* stiffness_path, const char* excitation_path,
                    ps_problem** out);
/* format_double, write_trajectory_csv, write_history_csv [proj/src/io.cpp:151-178] */
int ps_format_double(double value, char* buf, int32_t len);
int ps_write_trajectory_csv(const char* path, int32_t count, int32_t dim, const double* states,
                            const ps_time_mesh* mesh);
int ps_write_history_csv(const char* path, int32_t count, const double* jumps, const double* seconds);

void ps_seeded_normal(uint64_t seed, int64_t count, double sigma, double* out);
/* Seeded U(lo, hi) samples: mt19937_64 53-bit mantissa mapping. */
void ps_seeded_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif /* PPPC_B200_H */
