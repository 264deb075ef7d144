/*
 * oracle.h — CPU ORACLE for the PP-PC hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain C++ restatement of the reference algorithm (parasteady,
 * /root/reference/proj), used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg as the CHECKER — never as the product
 * path.  The reference itself cannot be built here (Eigen >= 3.4 and FFTW3 are
 * absent, proj/CMakeLists.txt:12-16), so the oracle restates its call graph
 * function by function (each function cites the reference file:line it follows)
 * and substitutes the third-party arithmetic:
 *   Eigen::SimplicialLDLT / SparseLU  -> an up-looking sparse LDL^T (real or
 *                                        complex-symmetric) with a nested-dissection
 *                                        or natural ordering      (mode OR_DIRECT)
 *   FFTW plan_many_dft                -> a direct unitary DFT with an exact twiddle table
 * and, for parity with the device path, implements the device algorithm's
 * iterative solvers (Jacobi-PCG, Jacobi-COCG) step for step (mode OR_ITERATIVE).
 *
 * Parity pins: the restatement is checked against every known-answer test the
 * reference holds for this path in tests/test_oracle_kat.py, and
 * against SciPy as an independent third implementation on small cases.
 */
#ifndef PPPC_ORACLE_H
#define PPPC_ORACLE_H

#include <stdint.h>

#include "../include/pppc_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_DIRECT = 0, OR_ITERATIVE = 1 };

typedef struct or_problem or_problem;

typedef struct {
  int64_t newton_iterations;
  int64_t pcg_iterations;
  int32_t max_newton_iterations;
  int32_t max_pcg_iterations;
  int32_t failed_index;
  int32_t code;
} or_stats;

const char* or_last_error(void);
int or_create(const ps_problem_desc* desc, const double* coords, or_problem** out);
void or_free(or_problem* p);
int or_dim(const or_problem* p);
int or_nnz(const or_problem* p);
int or_is_linear(const or_problem* p);
int or_frozen(const or_problem* p, const double* u_ref, or_problem** out);

void or_nu(const ps_curve* curve, int32_t n, const double* b2, double* nu, double* nu_prime);
int or_excitation(const or_problem* p, double t, double* f);
int or_stiffness_at(const or_problem* p, const double* u, double* K);
int or_newton_matrix_at(const or_problem* p, const double* u, double* J);

int or_newton_step(const or_problem* p, const ps_solver_settings* s, int32_t mode,
                   const double* u_prev, double t_next, double dt, double* u_out,
                   int32_t* iterations, double* trace, int64_t* pcg_iterations);
int or_fine_propagate_batch(const or_problem* p, const ps_time_mesh* mesh,
                            const ps_solver_settings* s, int32_t mode, int32_t n_first,
                            int32_t count, const double* U_start, double* U_end, int32_t workers,
                            or_stats* stats);
int or_coarse_propagate_batch(const or_problem* p, const ps_time_mesh* mesh,
                              const ps_solver_settings* s, int32_t mode, int32_t n_first,
                              int32_t count, const double* U_start, double* U_end,
                              int32_t workers, or_stats* stats);
int or_coarse_sweep(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                    int32_t mode, double* U);

int or_forward_dft(int32_t n, int32_t d, const double* U, double* spectrum);
int or_inverse_dft(int32_t n, int32_t d, const double* spectrum, double* U);
int or_assemble_rhs(const or_problem* lin, const ps_time_mesh* mesh, const double* F,
                    const double* G, double* rhs);
/* seconds of the last DIRECT or_mh_solve: per-bin factorizations and
 * back-substitutions summed over bins, and the wall time of its bin loop */
int or_last_direct_timing(double* factor_s, double* solve_s, double* wall_s);
int or_mh_solve(const or_problem* lin, const ps_time_mesh* mesh, const ps_solver_settings* s,
                int32_t mode, int32_t use_conjugate_symmetry, const int32_t* bin_mask,
                int32_t shift_kind, const double* rhs, double* U, int32_t workers,
                int64_t* cocg_iterations);
int or_solve_cyclic_direct(const or_problem* lin, const ps_time_mesh* mesh, const double* rhs,
                           double* U);
double or_jump_norm(int32_t count, int32_t d, const double* cur, const double* prev);

int or_pppc_solve(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                  const ps_engine_settings* e, int32_t mode, const double* frozen_ref,
                  double* U_out, double* iterates, ps_history* history, int32_t workers);
int or_classic_parareal(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                        const ps_engine_settings* e, int32_t mode, const double* u0, double* U_out,
                        double* iterates, ps_history* history, int32_t workers);
int or_pp_ic_solve(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                   const ps_engine_settings* e, int32_t mode, double* U_out, double* iterates,
                   ps_history* history, int32_t workers);
int or_fine_periodicity_defect(const or_problem* p, const ps_time_mesh* mesh,
                               const ps_solver_settings* s, int32_t mode, const double* U,
                               double* defect, int32_t workers);
int or_sequential_steady_state(const or_problem* p, const ps_time_mesh* mesh,
                               const ps_solver_settings* s, int32_t mode, double tol,
                               int32_t max_periods, double* U_out, int32_t* periods,
                               int32_t* converged, double* defects);

/* The oracle's own builders and seeded generators (polar_mesh.cpp): the canonical
 * polar P1 cable of SURVEY.md App. A.1 and the SURVEY.md §8(d) generators,
 * independent of the product library's builders. */
typedef struct or_mesh or_mesh;
int or_polar_cable_defaults(ps_polar_cable_params* p);
int or_build_polar_cable(const ps_polar_cable_params* params, or_mesh** out);
const char* or_mesh_error(void);
const ps_problem_desc* or_mesh_desc(const or_mesh* m);
const double* or_mesh_coordinates(const or_mesh* m);
void or_mesh_free(or_mesh* m);
void or_seeded_normal(uint64_t seed, int64_t count, double sigma, double* out);
void or_seeded_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif
