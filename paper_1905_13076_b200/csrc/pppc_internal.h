// Internal declarations shared by the device kernels (kernels.cu), the C ABI
// (capi.cu) and the host PP-PC driver (driver.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/pppc_b200.h"

namespace pppc {

constexpr int kWarps = 16;             // warps per block of the persistent kernels
constexpr int kThreads = kWarps * 32;  // 512
constexpr int kMaxCurves = 8;
constexpr int kMaxTerms = 16;
constexpr int kNDots = 4;
constexpr int kDbgSlots = 21;          // debug timing: 9 timing words + 9 action counts + 3 release times
constexpr int kRegularRow = 7;         // rows with <= 7 slots (the P1 polar mesh) use register accumulators
constexpr int kLongRow = 32;           // rows with > 32 slots are split across a block's warps
// Row records: rowrec[3i] = {first slot, length, kind (1 = per-system values),
// 0}; rowrec[3i+1..3i+2] = the row's column indices padded to kEll with the
// row's own index (rows longer than kEll keep using row_ptr / col_idx).  The
// persistent kernels copy their block's records into shared memory once.
constexpr int kEll = 8;
constexpr int kRecInts4 = 3;                          // int4 per row record
constexpr size_t kScrSmem = static_cast<size_t>(kWarps) * kEll * 32 * sizeof(double);  // refill slot scratch
constexpr size_t kRecSmemMax = 144 * 1024;            // dynamic shared memory for records (after the scratch)

// Per-system outcome written by block 0 of every group.
struct SysOut {
  int32_t code;
  int32_t newton_last;     // Newton iterations of the last step
  double t_fail;
  double residual;
  int64_t newton_total;
  int64_t pcg_total;
  int32_t max_newton;
  int32_t max_pcg;
};

// Everything the persistent propagation kernel needs (passed by value).
struct PropParams {
  // geometry of the launch
  int d, nnz;
  int stride;      // interleaved stride = batch count N
  int count;       // systems in the batch
  int G, C, L, Lp, R;
  const int* warp_row_begin;  // [C*kWarps + 1] contiguous row ranges per (block, warp)
  int n_long;                 // rows longer than kLongRow and the block that owns each
  const int* long_rows;
  const int* long_owner;
  // pattern
  const int* rp;
  const int* ci;
  const int* diag;
  const int4* rowrec;   // [d][kRecInts4]
  int rec_rows;          // >0: largest block row range; records are staged in shared memory
  const double* ME;      // [d][kEll] padded mass rows
  const double* KE;      // [d][kEll] padded shared stiffness rows (K linear, K_const element problems)
  int chunk_rot;         // chunk k of kWarps rows belongs to block (k + chunk_rot) mod C
  int g_base;            // storage group of launch-local group 0 (sequential group launches)
  int r_smem;            // 1: the PCG residual r of the block's rows (<= kLongRow slots) lives in shared memory
  int pf_dist;           // phase-A L2 prefetch distance in rows; 0 = off
  int hub_split;         // 1: the single long row's phase-A product goes through the reduction
  int probe_refill;      // 1: every lane runs one refill (ACT_R, u vs uprev) and stops (ps_refill_probe)
  const double* M;
  const double* Klin;     // linear K (Newton on a linear problem)
  // shared step matrix M/dt + K (linear problems) or M/dt + K_const (element
  // problems, rows of rowkind 0) and its Jacobi diagonal
  const double* Ash;
  const double* Dsh;
  const double* AshE;  // [d][kEll] padded rows of Ash (rows of <= kEll slots)
  const unsigned char* rowkind;  // element problems: 1 = row touches a nonlinear element
  const double* Kc;              // constant-nu stiffness (rows of rowkind 0)
  // element data (nonlinear)
  const int* adj_ptr;
  const int2* adj;        // (element, local index)
  const int* adj_rel;     // [n_adj*npe] slot offset within the row, -1 Dirichlet
  const int* en;
  const double* eS;
  const double* einvA;
  const int* ecurve;
  ps_curve curves[kMaxCurves];
  int ncurves;
  // excitation
  int nterms;
  const double* pat;       // [nterms][d]
  const double* coef;      // [steps][count][nterms]
  const double* t_next;    // [steps][count]
  int steps;
  double dt;
  // state (interleaved [d][stride]); nonlinear: u (state), uprev; linear: ubuf[2]
  double* u;
  double* uprev;
  double* ubuf0;
  double* ubuf1;
  double* x;
  double* r;
  double* p;
  double* q;
  double* Dinv;   // per-system Jacobi (nonlinear)
  double* A;      // per-system step-matrix values [nnz][stride] (nonlinear)
  // settings
  double newton_tol_abs, newton_tol_rel, damping;
  int newton_max;
  int line_search;
  double pcg_tol;
  int pcg_max;
  // sync + outputs
  unsigned long long* sync;   // [G] monotone arrival counters
  double* partials;           // [2][G][C][kNDots][32]
  int* abort_flag;
  SysOut* out;                // [count]
  double* trace;              // [count][newton_max] or null
  int64_t* lockstep;          // [G] lock-step PCG iterations executed
  unsigned long long* dbg;    // optional [G*C][kDbgSlots] timing (PPPC_DEBUG_TIMING)
};

struct DftPlan;

// System-per-block engine (kernels.cu sysblock_kernel): one thread block runs
// one system's whole propagation (every step, Newton iteration and PCG
// iteration) with block barriers only; per-system vectors are contiguous
// ([count][d], thread = row), so the SpMV gathers are coalesced across rows.
struct SysParams {
  double* su;           // state u [count][d] (the start state is gathered from P.u, group-blocked)
  double* sA;           // per-system step-matrix values of rows <= kEll slots, ELL [count][kEll][d]
  double* hubA;         // per-system values of the hub row [count][hub_len] (rows > kEll slots: at most one)
  const int* ciT;       // [kEll][d] padded ELL columns (pad = the row itself)
  const double* MT;     // [kEll][d] padded mass values
  const double* KT;     // [kEll][d] padded shared stiffness values (K_const)
  const double* AshT;   // [kEll][d] padded shared step-matrix values M/dt + K_const (per dt)
  int hub;              // the row longer than kEll, or -1
  int hub_len;
  int smem_vectors;     // 1: u, u_prev, x, r, p, q, Dinv in shared memory (7 d doubles)
  // sparsity-pattern dictionary (cluster engine): row i's pattern id; pattern p's
  // kEll column entries (relative to the row; 0 where the bit of pat_meta's
  // absolute mask is set: that column is the hub) and pat_meta = length | absolute mask << 8
  const unsigned char* pat_id;   // [d], kPatIrregular = not in the dictionary
  const int* pat_cols;           // [kPatMax][kEll]
  const int* pat_meta;           // [kPatMax]
  int ell_width;                 // longest row among the rows of <= kEll slots
};
constexpr int kPatMax = 256;
constexpr int kPatIrregular = kPatMax - 1;
size_t sysblock_smem(int d);
constexpr size_t kSbSmemMax = 200 * 1024;

// System-per-cluster engine (cluster_engine.cuh): a thread-block cluster of C
// CTAs runs one system; CTA c owns the contiguous rows [row_begin[c],
// row_begin[c+1]) and keeps p over the column window [win_lo[c], win_hi[c])
// (its rows plus the halo they gather), r and x of its rows in shared memory.
constexpr int kClusterMaxC = 16;
struct ClusterGeom {
  int C;
  int rows_max;   // largest row range
  int win_max;    // largest window
  int hub_len;    // slots of the hub row (0 = none): its values and window indices sit in shared memory
  int row_begin[kClusterMaxC + 1];
  int win_lo[kClusterMaxC];
  int win_hi[kClusterMaxC];
};

// Device-resident problem + work buffers owned by a context.
struct DevProblem {
  int d = 0, nnz = 0;
  bool linear = true;
  int npe = 0;
  int ne = 0;
  int* rp = nullptr;
  int* ci = nullptr;
  int* diag = nullptr;
  int4* rowrec = nullptr;
  double* ME = nullptr;  // [d][kEll] padded mass rows
  double* KE = nullptr;  // [d][kEll] padded shared stiffness rows (K or K_const)
  double* M = nullptr;
  double* K = nullptr;        // linear K (or frozen K-bar)
  int* adj_ptr = nullptr;
  int2* adj = nullptr;
  int* adj_rel = nullptr;
  int* en = nullptr;
  double* eS = nullptr;
  double* einvA = nullptr;
  int* ecurve = nullptr;
  std::vector<ps_curve> curves;
  int nterms = 0;
  double* pat = nullptr;
  double period = 0.0;
  std::vector<double> amp, freq, phase;
  // host copies needed for setup
  std::vector<int> h_rp, h_ci, h_diag;
  std::vector<double> h_M, h_K;
  int max_row_len = 0;
  // element problems: rows touching only constant-nu elements share their values
  unsigned char* rowkind = nullptr;
  double* Kc = nullptr;
  // system-per-block engine: transposed padded rows; sb_ok = the pattern qualifies
  // (every row <= kEll slots but at most one longer row)
  bool sb_ok = false;
  int sb_hub = -1;
  int ell_width = 1;   // longest row among the rows of <= kEll slots
  int* ciT = nullptr;
  unsigned char* pat_id = nullptr;
  int* pat_cols = nullptr;
  int* pat_meta = nullptr;
  double* MT = nullptr;
  double* KT = nullptr;
  std::vector<unsigned char> h_rowkind;
  std::vector<double> h_Kc;
};

// launches (kernels.cu)
int launch_propagate(const PropParams& prm, bool linear, int npe, cudaStream_t st, std::string* err);
int max_coresident_blocks(bool linear, int npe, int* out);
// host-order [count][d] <-> group-blocked [G][d][32] (L systems per group)
void launch_to_blocked(const double* src, double* dst, int count, int d, int L, cudaStream_t st);
void launch_from_blocked(const double* src, double* dst, int count, int d, int L, cudaStream_t st);
// interleaved [d][stride] <-> group-blocked
void launch_il_blocked(const double* src, double* dst, int d, int count, int stride, int L, bool to_blocked,
                       cudaStream_t st);
void launch_to_interleaved(const double* src, double* dst, int count, int d, int stride,
                           cudaStream_t st);
void launch_from_interleaved(const double* src, double* dst, int count, int d, int stride,
                             cudaStream_t st);
void launch_assemble_ops(const DevProblem& p, int count, const double* u_il, double* K_out,
                         double* J_out, cudaStream_t st);
void launch_excitation(const DevProblem& p, int count, const double* coef, double* out_il,
                       cudaStream_t st);
void launch_fill(double* dst, double v, size_t n, cudaStream_t st);
void launch_axpby_shared(const double* a, double sa, const double* b, double sb, double* out,
                         size_t n, cudaStream_t st);
void launch_eval_curve(const ps_curve& c, int n, const double* b2, double* nu, double* nup,
                       cudaStream_t st);
void launch_frozen_K(const DevProblem& p, const double* u_ref, double* K_out, cudaStream_t st);
int launch_phase_probe(const PropParams& prm, int mode, double* sink, cudaStream_t st);
int launch_sysblock(const PropParams& prm, const SysParams& sp, int npe, cudaStream_t st, std::string* err);
// system-per-cluster engine: shared memory of one CTA, rows a CTA can own at most,
// co-resident clusters (0 = this geometry cannot launch), launch
size_t syscluster_smem(const ClusterGeom& gm);
int syscluster_max_rows();
int syscluster_max_clusters(int npe, int ell_width, const ClusterGeom& gm);
int launch_syscluster(const PropParams& prm, const SysParams& sp, const ClusterGeom& gm, int npe, cudaStream_t st,
                      std::string* err);

// spectral (spectral.cu)
struct SpectralState;
int spectral_setup(SpectralState** out, const DevProblem& p, int N, double period,
                   int use_conj, const int32_t* mask, int shift_kind, std::string* err);
void spectral_free(SpectralState* s);
int spectral_assemble_rhs(SpectralState* s, const DevProblem& p, const double* F_il,
                          const double* G_il, double* rhs_il, cudaStream_t st);
int spectral_solve(SpectralState* s, const DevProblem& p, const ps_krylov_settings& cocg,
                   const double* rhs_il, double* U_il, double* U_prev_il, double* jump,
                   ps_batch_status* status, cudaStream_t st, std::string* err);
int dft_forward_standalone(int n, int d, const double* U, double* spec, std::string* err);
int spectral_forward_probe(SpectralState* s, const double* rhs, double* spec, std::string* err);
int spectral_inverse_probe(SpectralState* s, const double* spec, const double* U_old, double* U, double* jump,
                           std::string* err);
int spectral_bins(const SpectralState* s, int32_t* bins, int32_t cap);
int dft_inverse_standalone(int n, int d, const double* spec, double* U, std::string* err);
int jump_norm_device(int count, int d, const double* cur_il, const double* prev_il, int stride,
                     double* out, cudaStream_t st);

}  // namespace pppc
