// Batched fine / coarse propagation on B200 (sm_100a), fp64.
//
// One persistent cooperative kernel runs a whole batch of implicit-Euler
// propagations  (proj/src/propagators.cpp:96-115):  every time step, every
// Newton iteration (proj/src/propagators.cpp:27-58) and every Jacobi-PCG
// iteration of the step solve stays on the device.  The host only sees the
// final states and a per-system status word.
//
// Layout: every per-system vector is interleaved [row][system]
// so that, for one CSR slot, the column index is read once and the values /
// gathered operands of all systems are contiguous.  Systems are split into
// groups of L <= 32; a warp lane holds one (row, system) pair, a group is
// served by C blocks of 512 threads that synchronise only among themselves
// through a monotone arrival counter (no grid-wide barrier).  Every block
// reduces the group's dot-product partials redundantly in a fixed order, so
// all blocks hold bit-identical per-system scalars (alpha, beta, convergence
// flags) and take identical branches; results are deterministic and do not
// depend on which other systems share the batch.
#include "group_sync.cuh"
#include "pppc_internal.h"

#include <cstdio>

namespace pppc {
namespace {

constexpr double kVacuumReluctivity = 1.0 / (4.0e-7 * 3.14159265358979323846);

__device__ __forceinline__ double std_min(double a, double b) { return (b < a) ? b : a; }

// ReluctivityCurve::nu / nu_prime (proj/src/problem.cpp:84-98); one exp shared.
__device__ __forceinline__ void curve_eval(const ps_curve& c, double b2, double& nu, double& nup) {
  if (c.kind == 0) {
    nu = c.nu;
    nup = 0.0;
    return;
  }
  const double expo = std_min(c.k2 * b2, 700.0);
  const double ex = exp(expo);
  const double unc = c.k1 * ex + c.k3;
  nu = std_min(unc, kVacuumReluctivity);
  nup = (unc >= kVacuumReluctivity) ? 0.0 : c.k1 * c.k2 * ex;
}

// Per-lane (= per-system) scalar state.  Every thread whose lane maps to the
// same system holds an identical copy, in every block of the group.
struct Lane {
  bool alive;
  int code;
  double t_fail, res_fail;
  double tol;
  int nit;
  bool nact;
  bool pact;
  int pit;
  double rho, stop, alpha, beta;
  double res_pre;
  double lambda;   // current Newton step length (damping, halved on backtracks)
  int ls_k;        // backtracks taken in this Newton iteration
  bool upd;        // needs an update + residual round
  bool bt;         // the pending round is a backtrack
  bool zero_dx;    // the step solve took 0 iterations (delta = 0)
  long long newton_total, pcg_total;
  int max_nit, max_pit, last_nit;
};

__device__ __forceinline__ void lane_fail(Lane& s, int code, double res, double t) {
  if (!s.alive) return;
  s.alive = false;
  s.nact = false;
  s.pact = false;
  s.upd = false;
  s.code = code;
  s.res_fail = res;
  s.t_fail = t;
}

__device__ __forceinline__ void pcg_start(Lane& s, double rho, double bb, double tol) {
  s.rho = rho;
  s.stop = (tol * tol) * bb;
  s.pit = 0;
  s.pact = s.alive && (bb != 0.0);
}

template <int NPE>
struct Elem {
  double ue[NPE], g[NPE], S[NPE * NPE];
  double nu, cc;
};

template <int NPE>
__device__ __forceinline__ void eval_elem(const PropParams& P, const ps_curve* curves, int e,
                                          const double* u, size_t stride, int sys,
                                          Elem<NPE>& E) {
#pragma unroll
  for (int b = 0; b < NPE; ++b) {
    const int n = __ldg(P.en + e * NPE + b);
    E.ue[b] = n >= 0 ? u[static_cast<size_t>(n) * stride + sys] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < NPE * NPE; ++k) E.S[k] = __ldg(P.eS + static_cast<size_t>(e) * NPE * NPE + k);
  double b2 = 0.0;
#pragma unroll
  for (int a = 0; a < NPE; ++a) {
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < NPE; ++b) s += E.S[a * NPE + b] * E.ue[b];
    E.g[a] = s;
    b2 += E.ue[a] * s;
  }
  const double inva = __ldg(P.einvA + e);
  b2 *= inva;
  double nup;
  curve_eval(curves[__ldg(P.ecurve + e)], b2, E.nu, nup);
  E.cc = 2.0 * nup * inva;
}

// Fused residual + Jacobian refill + Jacobi diagonal + PCG init for one row
// and one system: writes A = M/dt + J(u) into the
// fixed CSR pattern, Dinv, r = -R, p = Dinv r, x = 0.
template <int NPE>
__device__ __forceinline__ void refill_row(const PropParams& P, const ps_curve* curves, int i,
                                           int sys, int step, bool first, double (&acc)[kNDots]) {
  const size_t st = static_cast<size_t>(P.stride);
  const size_t iv = static_cast<size_t>(i) * st + sys;
  const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
  const int len = end - base;
  const bool regular = len <= kRegularRow;
  double jv[kRegularRow];
#pragma unroll
  for (int s = 0; s < kRegularRow; ++s) jv[s] = 0.0;
  if (!regular)
    for (int k = base; k < end; ++k) P.A[static_cast<size_t>(k) * st + sys] = 0.0;
  double ku = 0.0;
  if constexpr (NPE == 0) {
    // linear problem under newton_step semantics: J = K (proj/src/problem.cpp:141-144)
    for (int k = base; k < end; ++k) {
      const double kk = __ldg(P.Klin + k);
      ku += kk * P.u[static_cast<size_t>(__ldg(P.ci + k)) * st + sys];
      if (regular) {
#pragma unroll
        for (int s = 0; s < kRegularRow; ++s) jv[s] += (k - base == s) ? kk : 0.0;
      } else {
        P.A[static_cast<size_t>(k) * st + sys] = kk;
      }
    }
  } else {
    const int q0 = __ldg(P.adj_ptr + i), q1 = __ldg(P.adj_ptr + i + 1);
    for (int q = q0; q < q1; ++q) {
      const int2 ea = __ldg(P.adj + q);
      Elem<NPE> E;
      eval_elem<NPE>(P, curves, ea.x, P.u, st, sys, E);
      const int a = ea.y;
      ku += E.nu * E.g[a];
  #pragma unroll
      for (int b = 0; b < NPE; ++b) {
        const int rel = __ldg(P.adj_rel + static_cast<size_t>(q) * NPE + b);
        if (rel < 0) continue;
        const double v = E.nu * E.S[a * NPE + b] + E.cc * (E.g[a] * E.g[b]);
        if (regular) {
  #pragma unroll
          for (int s = 0; s < kRegularRow; ++s) jv[s] += (rel == s) ? v : 0.0;
        } else {
          P.A[static_cast<size_t>(base + rel) * st + sys] += v;
        }
      }
    }
  }
  // excitation f_i = sum_t c_t(t_next) pattern_t[i]  (proj/src/problem.cpp:52-63)
  double f = 0.0;
  const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
  for (int t = 0; t < P.nterms; ++t) f += cf[t] * __ldg(P.pat + static_cast<size_t>(t) * P.d + i);
  // mass term M (u - u_prev)/dt, zero at the first Newton iterate of a step
  double mr = 0.0, dval = 0.0;
  const int dslot = __ldg(P.diag + i);
  for (int k = base; k < end; ++k) {
    const double mk = __ldg(P.M + k);
    if (!first) {
      const size_t jv2 = static_cast<size_t>(__ldg(P.ci + k)) * st + sys;
      mr += mk * ((P.u[jv2] - P.uprev[jv2]) / P.dt);
    }
    double jk;
    if (regular) {
      jk = 0.0;
#pragma unroll
      for (int s = 0; s < kRegularRow; ++s) jk = (k - base == s) ? jv[s] : jk;
    } else {
      jk = P.A[static_cast<size_t>(k) * st + sys];
    }
    const double av = mk / P.dt + jk;
    P.A[static_cast<size_t>(k) * st + sys] = av;
    if (k == dslot) dval = av;
  }
  const double dinv = 1.0 / dval;
  const double R = mr + ku - f;
  const double r = -R;
  const double z = dinv * r;
  P.Dinv[iv] = dinv;
  P.r[iv] = r;
  P.p[iv] = z;
  if (first) P.uprev[iv] = P.u[iv];
  acc[0] += R * R;
  acc[1] += f * f;
  acc[2] += r * z;
  acc[3] += r * r;
}

// q_i = (A p)_i for one row and one system, plus the phase-A dot partials
// p.q, q.z, q.Dq (z = D r).  Regular rows (<= 8 slots) issue all column-index,
// value and gathered-operand loads before the first FMA (memory-level
// parallelism); long rows (the polar hub) take a plain loop.
template <bool LINEAR>
__device__ __forceinline__ void spmv_row(const PropParams& P, int i, int sys, double (&acc)[kNDots]) {
  const size_t st = static_cast<size_t>(P.stride);
  const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
  const int len = end - base;
  double qv = 0.0;
  if (len <= kRegularRow) {
    int cj[kRegularRow];
    double av[kRegularRow], pv[kRegularRow];
#pragma unroll
    for (int k = 0; k < kRegularRow; ++k) cj[k] = k < len ? __ldg(P.ci + base + k) : i;
#pragma unroll
    for (int k = 0; k < kRegularRow; ++k) {
      if (LINEAR)
        av[k] = k < len ? __ldg(P.Ash + base + k) : 0.0;
      else
        av[k] = k < len ? P.A[static_cast<size_t>(base + k) * st + sys] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kRegularRow; ++k) pv[k] = k < len ? P.p[static_cast<size_t>(cj[k]) * st + sys] : 0.0;
#pragma unroll
    for (int k = 0; k < kRegularRow; ++k)
      if (k < len) qv += av[k] * pv[k];
  } else {
    for (int k = base; k < end; ++k) {
      const int j0 = __ldg(P.ci + k);
      const double a0 = LINEAR ? __ldg(P.Ash + k) : P.A[static_cast<size_t>(k) * st + sys];
      qv += a0 * P.p[static_cast<size_t>(j0) * st + sys];
    }
  }
  const size_t iv = static_cast<size_t>(i) * st + sys;
  P.q[iv] = qv;
  const double di = LINEAR ? __ldg(P.Dsh + i) : P.Dinv[iv];
  const double pi = P.p[iv], ri = P.r[iv];
  const double zi = di * ri;
  acc[0] += pi * qv;
  acc[1] += qv * zi;
  acc[2] += qv * (di * qv);
}

// Phase B for two consecutive rows (loads of both rows issued together):
// x += alpha p (x = alpha p on the first iteration), r -= alpha q, z = D r,
// p = z + beta p; partials r.r and r.z.
template <bool LINEAR>
__device__ __forceinline__ void update_rows(const PropParams& P, double* x, int i, bool two, int sys, double alpha,
                                            double beta, bool first, double (&acc)[kNDots]) {
  const size_t st = static_cast<size_t>(P.stride);
  const size_t iv0 = static_cast<size_t>(i) * st + sys;
  const size_t iv1 = iv0 + st;
  double d0, d1 = 0.0, p0, p1 = 0.0, q0, q1 = 0.0, r0, r1 = 0.0, x0 = 0.0, x1 = 0.0;
  d0 = LINEAR ? __ldg(P.Dsh + i) : P.Dinv[iv0];
  p0 = P.p[iv0];
  q0 = P.q[iv0];
  r0 = P.r[iv0];
  if (!first) x0 = x[iv0];
  if (two) {
    d1 = LINEAR ? __ldg(P.Dsh + i + 1) : P.Dinv[iv1];
    p1 = P.p[iv1];
    q1 = P.q[iv1];
    r1 = P.r[iv1];
    if (!first) x1 = x[iv1];
  }
  // x0 = 0: the first update writes alpha p (the refill leaves the previous
  // Newton update in x so a line-search backtrack can still use it)
  x[iv0] = first ? alpha * p0 : x0 + alpha * p0;
  r0 -= alpha * q0;
  const double z0 = d0 * r0;
  P.r[iv0] = r0;
  P.p[iv0] = z0 + beta * p0;
  acc[0] += r0 * r0;
  acc[1] += r0 * z0;
  if (two) {
    x[iv1] = first ? alpha * p1 : x1 + alpha * p1;
    r1 -= alpha * q1;
    const double z1 = d1 * r1;
    P.r[iv1] = r1;
    P.p[iv1] = z1 + beta * p1;
    acc[0] += r1 * r1;
    acc[1] += r1 * z1;
  }
}

// Per-lane actions: one action per group-barrier interval, so every system
// advances through its own steps, Newton iterations, backtracks and PCG
// iterations without waiting for the other systems of its group.
enum : int { ACT_IDLE = 0, ACT_R0, ACT_A, ACT_B, ACT_U, ACT_R, ACT_L0, ACT_LU };

template <bool LINEAR, int NPE>
__global__ void __launch_bounds__(kThreads, 1) propagate_kernel(const PropParams P) {
  __shared__ SyncShared<kNDots> sh;
  __shared__ ps_curve sh_curves[kMaxCurves];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x / P.C, c = blockIdx.x % P.C;
  const int sub = lane / P.Lp, sl = lane % P.Lp;
  const int sys = g * P.L + sl;
  const bool valid = (sl < P.L) && (sys < P.count);
  if (threadIdx.x < P.ncurves) sh_curves[threadIdx.x] = P.curves[threadIdx.x];
  if (threadIdx.x == 0) sh.abort = 0;
  __syncthreads();
  SyncCtx X;
  X.sync = P.sync;
  X.partials = P.partials;
  X.abort_flag = P.abort_flag;
  X.G = P.G;
  X.C = P.C;
  X.Lp = P.Lp;
  const int row_begin = P.warp_row_begin[c * kWarps + warp];
  const int row_end = P.warp_row_begin[c * kWarps + warp + 1];
  unsigned long long target = 0;
  int bar_idx = 0;
  const bool writer = (c == 0) && (warp == 0) && (sub == 0) && valid;

  Lane s;
  s.alive = valid;
  s.code = PS_OK;
  s.t_fail = 0.0;
  s.res_fail = 0.0;
  s.tol = 0.0;
  s.nit = 0;
  s.nact = false;
  s.pact = false;
  s.pit = 0;
  s.rho = s.stop = s.alpha = s.beta = 0.0;
  s.res_pre = 0.0;
  s.lambda = 1.0;
  s.ls_k = 0;
  s.upd = s.bt = s.zero_dx = false;
  s.newton_total = s.pcg_total = 0;
  s.max_nit = s.max_pit = s.last_nit = 0;
  int act = valid ? (LINEAR ? ACT_L0 : ACT_R0) : ACT_IDLE;
  int step = 0;

  double acc[kNDots] = {0.0, 0.0, 0.0, 0.0};
  long long lockstep = 0;

  while (__syncthreads_or(act != ACT_IDLE)) {
    const double t_now = (act != ACT_IDLE) ? P.t_next[static_cast<size_t>(step) * P.count + sys] : 0.0;
    double* xs = LINEAR ? ((step & 1) ? P.ubuf0 : P.ubuf1) : P.x;
    // ------------------------------------------------ this lane's action
    if (act == ACT_A) {
      for (int i = row_begin + sub; i < row_end; i += P.R) spmv_row<LINEAR>(P, i, sys, acc);
    } else if (act == ACT_B) {
      const bool first = s.pit == 0;
      if (P.R == 1) {
        for (int i = row_begin; i < row_end; i += 2)
          update_rows<LINEAR>(P, xs, i, i + 1 < row_end, sys, s.alpha, s.beta, first, acc);
      } else {
        for (int i = row_begin + sub; i < row_end; i += P.R)
          update_rows<LINEAR>(P, xs, i, false, sys, s.alpha, s.beta, first, acc);
      }
    } else if (act == ACT_R0 || act == ACT_R) {
      if constexpr (!LINEAR)
        for (int i = row_begin + sub; i < row_end; i += P.R)
          refill_row<NPE>(P, sh_curves, i, sys, step, act == ACT_R0, acc);
    } else if (act == ACT_U) {
      if (!s.zero_dx)
        for (int i = row_begin + sub; i < row_end; i += P.R) {
          // trial u += lambda delta (propagators.cpp:46-48), or a backtrack
          // u -= lambda delta with lambda already halved; delta must be finite
          const size_t iv = static_cast<size_t>(i) * P.stride + sys;
          const double dx = P.x[iv];
          if (s.bt) {
            P.u[iv] -= s.lambda * dx;
          } else {
            acc[0] += isfinite(dx) ? 0.0 : 1.0;
            P.u[iv] += s.lambda * dx;
          }
        }
    } else if (act == ACT_L0) {
      // b = M (u/dt) + f, x = 0, r = b, p = D b (proj/src/propagators.cpp:85-94)
      const double* uin = (step & 1) ? P.ubuf1 : P.ubuf0;
      const size_t st = static_cast<size_t>(P.stride);
      const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
      for (int i = row_begin + sub; i < row_end; i += P.R) {
        const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
        double mv = 0.0;
        for (int k = base; k < end; ++k)
          mv += __ldg(P.M + k) * (uin[static_cast<size_t>(__ldg(P.ci + k)) * st + sys] / P.dt);
        double f = 0.0;
        for (int t = 0; t < P.nterms; ++t) f += cf[t] * __ldg(P.pat + static_cast<size_t>(t) * P.d + i);
        const double b = mv + f;
        const size_t iv = static_cast<size_t>(i) * st + sys;
        const double z = __ldg(P.Dsh + i) * b;
        xs[iv] = 0.0;
        P.r[iv] = b;
        P.p[iv] = z;
        acc[0] += b * z;
        acc[1] += b * b;
      }
    } else if (act == ACT_LU) {
      // the step solution must be finite (propagators.cpp:92); x0 = 0 when b = 0
      for (int i = row_begin + sub; i < row_end; i += P.R) {
        const size_t iv = static_cast<size_t>(i) * P.stride + sys;
        if (s.pit == 0) xs[iv] = 0.0;
        acc[0] += isfinite(xs[iv]) ? 0.0 : 1.0;
      }
    }
    if (!group_sync_reduce<kNDots, 4>(X, sh, acc, g, c, target, bar_idx)) return;
    ++lockstep;
    const double t0v = sh.tot[0][sl], t1v = sh.tot[1][sl], t2v = sh.tot[2][sl], t3v = sh.tot[3][sl];
    // ------------------------------------------------ this lane's transition
    switch (act) {
      case ACT_R0: {
        s.nact = true;
        s.tol = P.newton_tol_abs + P.newton_tol_rel * sqrt(t1v);
        s.nit = 1;
        s.res_pre = sqrt(t0v);
        pcg_start(s, t2v, t3v, P.pcg_tol);
        s.upd = true;
        s.bt = false;
        s.zero_dx = !s.pact;
        s.lambda = P.damping;
        s.ls_k = 0;
        act = s.pact ? ACT_A : ACT_U;
        break;
      }
      case ACT_A: {
        if (!isfinite(t0v) || t0v == 0.0) {
          lane_fail(s, PS_ERR_SINGULAR, LINEAR ? 0.0 : s.res_pre, t_now);
        } else {
          s.alpha = s.rho / t0v;
          const double rho_est = s.rho - 2.0 * s.alpha * t1v + s.alpha * s.alpha * t2v;
          s.beta = rho_est / s.rho;
          act = ACT_B;
        }
        break;
      }
      case ACT_B: {
        const double rr = t0v;
        s.rho = t1v;
        s.pit += 1;
        if (rr <= s.stop) {
          s.pact = false;
          s.pcg_total += s.pit;
          s.max_pit = max(s.max_pit, s.pit);
          act = LINEAR ? ACT_LU : ACT_U;
        } else if (!isfinite(rr)) {
          lane_fail(s, PS_ERR_SINGULAR, LINEAR ? 0.0 : s.res_pre, t_now);
        } else if (s.pit >= P.pcg_max) {
          lane_fail(s, PS_ERR_PCG_MAXITER, LINEAR ? 0.0 : s.res_pre, t_now);
        } else {
          act = ACT_A;
        }
        break;
      }
      case ACT_U: {
        if (!s.bt && t0v > 0.0)
          lane_fail(s, PS_ERR_SINGULAR, s.res_pre, t_now);
        else
          act = ACT_R;
        break;
      }
      case ACT_R: {
        const double post = sqrt(t0v);
        if (P.line_search > 0 && s.ls_k < P.line_search && !(post <= s.tol) &&
            !(post <= (1.0 - 1e-4 * s.lambda) * s.res_pre)) {
          s.lambda *= 0.5;
          s.ls_k += 1;
          s.bt = true;
          act = ACT_U;
          break;
        }
        s.bt = false;
        if (writer && P.trace) P.trace[static_cast<size_t>(sys) * P.newton_max + (s.nit - 1)] = post;
        if (!isfinite(post)) {
          lane_fail(s, PS_ERR_NEWTON_DIVERGED, post, t_now);
        } else if (post <= s.tol) {
          s.nact = false;
          s.newton_total += s.nit;
          s.last_nit = s.nit;
          s.max_nit = max(s.max_nit, s.nit);
          ++step;
          act = step < P.steps ? ACT_R0 : ACT_IDLE;
        } else if (s.nit >= P.newton_max) {
          lane_fail(s, PS_ERR_NEWTON_MAXITER, post, t_now);
        } else {
          s.nit += 1;
          s.res_pre = post;
          pcg_start(s, t2v, t3v, P.pcg_tol);
          s.zero_dx = !s.pact;
          s.lambda = P.damping;
          s.ls_k = 0;
          act = s.pact ? ACT_A : ACT_U;
        }
        break;
      }
      case ACT_L0: {
        pcg_start(s, t0v, t1v, P.pcg_tol);
        act = s.pact ? ACT_A : ACT_LU;
        break;
      }
      case ACT_LU: {
        if (t0v > 0.0) {
          lane_fail(s, PS_ERR_SINGULAR, 0.0, t_now);
        } else {
          s.newton_total += 1;
          s.last_nit = 1;
          s.max_nit = max(s.max_nit, 1);
          ++step;
          act = step < P.steps ? ACT_L0 : ACT_IDLE;
        }
        break;
      }
      default:
        break;
    }
    if (!s.alive) act = ACT_IDLE;
  }

  if (writer) {
    SysOut o;
    o.code = s.code;
    o.newton_last = s.last_nit;
    o.t_fail = s.t_fail;
    o.residual = s.res_fail;
    o.newton_total = s.newton_total;
    o.pcg_total = s.pcg_total;
    o.max_newton = s.max_nit;
    o.max_pcg = s.max_pit;
    P.out[sys] = o;
  }
  if (c == 0 && threadIdx.x == 0) P.lockstep[g] = lockstep;
}

// ------------------------------------------------------------ small kernels
__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst, int rows,
                                 int cols, int ld_src, int ld_dst) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + y, cc = c0 + threadIdx.x;
    if (r < rows && cc < cols) tile[y][threadIdx.x] = src[static_cast<size_t>(r) * ld_src + cc];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int cc = c0 + y, r = r0 + threadIdx.x;
    if (r < rows && cc < cols) dst[static_cast<size_t>(cc) * ld_dst + r] = tile[threadIdx.x][y];
  }
}

template <int NPE>
__global__ void assemble_ops_kernel(const PropParams P, int count, const double* __restrict__ u_il,
                                    double* K_out, double* J_out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(count) * P.d) return;
  const int sys = static_cast<int>(t % count), i = static_cast<int>(t / count);
  const int base = P.rp[i], end = P.rp[i + 1];
  double* Kr = K_out ? K_out + static_cast<size_t>(sys) * P.nnz : nullptr;
  double* Jr = J_out ? J_out + static_cast<size_t>(sys) * P.nnz : nullptr;
  for (int k = base; k < end; ++k) {
    if (Kr) Kr[k] = 0.0;
    if (Jr) Jr[k] = 0.0;
  }
  for (int q = P.adj_ptr[i]; q < P.adj_ptr[i + 1]; ++q) {
    const int2 ea = P.adj[q];
    Elem<NPE> E;
    eval_elem<NPE>(P, P.curves, ea.x, u_il, static_cast<size_t>(count), sys, E);
    const int a = ea.y;
    for (int b = 0; b < NPE; ++b) {
      const int rel = P.adj_rel[static_cast<size_t>(q) * NPE + b];
      if (rel < 0) continue;
      if (Kr) Kr[base + rel] += E.nu * E.S[a * NPE + b];
      if (Jr) Jr[base + rel] += E.nu * E.S[a * NPE + b] + E.cc * (E.g[a] * E.g[b]);
    }
  }
}

__global__ void excitation_kernel(const double* __restrict__ pat, const double* __restrict__ coef, int nterms,
                                  int d, int count, double* out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(count) * d) return;
  const int sys = static_cast<int>(t % count), i = static_cast<int>(t / count);
  double f = 0.0;
  for (int k = 0; k < nterms; ++k) f += coef[static_cast<size_t>(sys) * nterms + k] * pat[static_cast<size_t>(k) * d + i];
  out[t] = f;
}

__global__ void fill_kernel(double* dst, double v, size_t n) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) dst[t] = v;
}

__global__ void axpby_kernel(const double* a, double sa, const double* b, double sb, double* out, size_t n) {
  const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = a[t] / sa + b[t] * sb;
}

__global__ void curve_kernel(ps_curve c, int n, const double* b2, double* nu, double* nup) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v, vp;
  curve_eval(c, b2[t], v, vp);
  if (nu) nu[t] = v;
  if (nup) nup[t] = vp;
}

template <bool LINEAR, int NPE>
void* kernel_ptr() {
  return reinterpret_cast<void*>(&propagate_kernel<LINEAR, NPE>);
}

void* select_kernel(bool linear, int npe) {
  if (linear) return kernel_ptr<true, 0>();
  if (npe == 0) return kernel_ptr<false, 0>();
  return npe == 2 ? kernel_ptr<false, 2>() : kernel_ptr<false, 3>();
}

}  // namespace

int max_coresident_blocks(bool linear, int npe, int* out) {
  (void)linear;
  (void)npe;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PS_ERR_CUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return PS_ERR_CUDA;
  // every variant must fit: the capacity is the minimum over all instantiations
  int best = 1 << 30;
  void* fns[] = {kernel_ptr<true, 0>(), kernel_ptr<false, 0>(), kernel_ptr<false, 2>(), kernel_ptr<false, 3>()};
  for (void* fn : fns) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess) return PS_ERR_CUDA;
    best = per_sm < best ? per_sm : best;
  }
  *out = sms * best;
  return PS_OK;
}

int launch_propagate(const PropParams& prm, bool linear, int npe, cudaStream_t st, std::string* err) {
  void* fn = select_kernel(linear, npe);
  PropParams local = prm;
  void* args[] = {&local};
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(prm.G * prm.C), dim3(kThreads), args, 0, st);
  if (e != cudaSuccess) {
    if (err) *err = std::string("cuda: propagate launch failed: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

void launch_to_interleaved(const double* src, double* dst, int count, int d, int stride, cudaStream_t st) {
  // src [count][d] -> dst [d][stride]
  dim3 grid((d + 31) / 32, (count + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, dst, count, d, d, stride);
}

void launch_from_interleaved(const double* src, double* dst, int count, int d, int stride, cudaStream_t st) {
  // src [d][stride] (first count columns) -> dst [count][d]
  dim3 grid((count + 31) / 32, (d + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, dst, d, count, stride, d);
}

void launch_assemble_ops(const DevProblem& p, int count, const double* u_il, double* K_out, double* J_out,
                         cudaStream_t st) {
  PropParams P{};
  P.d = p.d;
  P.nnz = p.nnz;
  P.rp = p.rp;
  P.adj_ptr = p.adj_ptr;
  P.adj = p.adj;
  P.adj_rel = p.adj_rel;
  P.en = p.en;
  P.eS = p.eS;
  P.einvA = p.einvA;
  P.ecurve = p.ecurve;
  P.ncurves = static_cast<int>(p.curves.size());
  for (int k = 0; k < P.ncurves && k < kMaxCurves; ++k) P.curves[k] = p.curves[k];
  const int64_t total = static_cast<int64_t>(count) * p.d;
  const int blocks = static_cast<int>((total + 255) / 256);
  if (p.npe == 2)
    assemble_ops_kernel<2><<<blocks, 256, 0, st>>>(P, count, u_il, K_out, J_out);
  else
    assemble_ops_kernel<3><<<blocks, 256, 0, st>>>(P, count, u_il, K_out, J_out);
}

void launch_excitation(const DevProblem& p, int count, const double* coef, double* out_il, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(count) * p.d;
  excitation_kernel<<<static_cast<int>((total + 255) / 256), 256, 0, st>>>(p.pat, coef, p.nterms, p.d, count,
                                                                           out_il);
}

void launch_fill(double* dst, double v, size_t n, cudaStream_t st) {
  if (n == 0) return;
  fill_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(dst, v, n);
}

// out = a / sa + b * sb  (used for M/dt + K)
void launch_axpby_shared(const double* a, double sa, const double* b, double sb, double* out, size_t n,
                         cudaStream_t st) {
  if (n == 0) return;
  axpby_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(a, sa, b, sb, out, n);
}

void launch_eval_curve(const ps_curve& c, int n, const double* b2, double* nu, double* nup, cudaStream_t st) {
  if (n <= 0) return;
  curve_kernel<<<(n + 255) / 256, 256, 0, st>>>(c, n, b2, nu, nup);
}

void launch_frozen_K(const DevProblem& p, const double* u_ref, double* K_out, cudaStream_t st) {
  launch_assemble_ops(p, 1, u_ref, K_out, nullptr, st);
}

}  // namespace pppc
