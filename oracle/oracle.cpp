// CPU ORACLE — test infrastructure only (see oracle.h).  Restates the
// reference's hot path (parasteady, /root/reference/proj) in plain C++.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <chrono>
#include <complex>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;
// proj/include/parasteady/problem.hpp:62
constexpr double kVacuumReluctivity = 1.0 / (4.0e-7 * 3.14159265358979323846);
// proj/src/spectral.cpp:21
constexpr double kImagResidualTol = 1e-8;

thread_local std::string g_error;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// proj/src/propagators.cpp:19-23
Error step_failure_error(int code, const char* what, double t_next, double residual) {
  std::ostringstream msg;
  msg << "propagator: " << what << " at t = " << t_next << " (residual " << residual << ")";
  return Error(code, msg.str());
}
#define step_failure(...) throw step_failure_error(__VA_ARGS__)

// proj/include/parasteady/parallel.hpp:15-41 — fork/join strided map; the lowest
// failing index wins (deterministic variant of "first exception observed").
void parallel_for(int count, int workers, const std::function<void(int)>& fn) {
  if (count <= 0) return;
  const int n_threads = std::max(1, std::min(workers, count));
  std::vector<std::exception_ptr> errors(static_cast<size_t>(count));
  auto body = [&](int t) {
    for (int i = t; i < count; i += n_threads) {
      try {
        fn(i);
      } catch (...) {
        errors[i] = std::current_exception();
      }
    }
  };
  if (n_threads == 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < n_threads; ++t) pool.emplace_back(body, t);
    for (auto& th : pool) th.join();
  }
  for (int i = 0; i < count; ++i)
    if (errors[i]) std::rethrow_exception(errors[i]);
}

// ---------------------------------------------------------------- curves
// proj/src/problem.cpp:84-98
double curve_nu(const ps_curve& c, double b2) {
  if (c.kind == 0) return c.nu;
  const double expo = std::min(c.k2 * b2, 700.0);
  return std::min(c.k1 * std::exp(expo) + c.k3, kVacuumReluctivity);
}
double curve_nu_prime(const ps_curve& c, double b2) {
  if (c.kind == 0) return 0.0;
  const double expo = std::min(c.k2 * b2, 700.0);
  const double uncapped = c.k1 * std::exp(expo) + c.k3;
  if (uncapped >= kVacuumReluctivity) return 0.0;
  return c.k1 * c.k2 * std::exp(expo);
}

// --------------------------------------------------------------- problem
struct Problem {
  int d = 0;
  int64_t nnz = 0;
  std::vector<int32_t> rp, ci;
  std::vector<double> M, K;
  bool linear = true;
  int ne = 0, npe = 0;
  std::vector<int32_t> en, ecurve;
  std::vector<double> eS, einvA;
  std::vector<ps_curve> curves;
  double T = 0.0;
  int nterms = 0;
  std::vector<double> pat, amp, freq, phase;
  std::vector<double> coords;
  std::vector<int64_t> eslot;  // [ne][npe][npe] pattern slot, -1 for Dirichlet pairs
  std::vector<int32_t> order;  // fill-reducing ordering for the direct solver

  int64_t slot(int32_t r, int32_t c) const {
    const auto b = ci.begin() + rp[r], e = ci.begin() + rp[r + 1];
    const auto it = std::lower_bound(b, e, c);
    if (it == e || *it != c) return -1;
    return it - ci.begin();
  }
};

void nested_dissection(const Problem& p, std::vector<int32_t>& nodes, std::vector<int32_t>& out,
                       std::vector<int32_t>& mark, int tag_base, int& tag) {
  if (nodes.size() <= 96 || p.coords.empty()) {
    out.insert(out.end(), nodes.begin(), nodes.end());
    return;
  }
  double xmin = 1e300, xmax = -1e300, ymin = 1e300, ymax = -1e300;
  for (int32_t v : nodes) {
    xmin = std::min(xmin, p.coords[2 * v]);
    xmax = std::max(xmax, p.coords[2 * v]);
    ymin = std::min(ymin, p.coords[2 * v + 1]);
    ymax = std::max(ymax, p.coords[2 * v + 1]);
  }
  const int axis = (xmax - xmin) >= (ymax - ymin) ? 0 : 1;
  std::vector<double> key(nodes.size());
  for (size_t i = 0; i < nodes.size(); ++i) key[i] = p.coords[2 * nodes[i] + axis];
  std::vector<double> sorted = key;
  std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
  const double median = sorted[sorted.size() / 2];
  const int left_tag = ++tag;
  std::vector<int32_t> left, right, sep;
  for (size_t i = 0; i < nodes.size(); ++i) {
    if (key[i] < median) {
      left.push_back(nodes[i]);
      mark[nodes[i]] = left_tag;
    }
  }
  for (size_t i = 0; i < nodes.size(); ++i) {
    if (key[i] < median) continue;
    const int32_t v = nodes[i];
    bool touches = false;
    for (int32_t k = p.rp[v]; k < p.rp[v + 1]; ++k)
      if (mark[p.ci[k]] == left_tag) {
        touches = true;
        break;
      }
    (touches ? sep : right).push_back(v);
  }
  if (left.empty() || right.empty()) {
    out.insert(out.end(), nodes.begin(), nodes.end());
    return;
  }
  (void)tag_base;
  nested_dissection(p, left, out, mark, tag_base, tag);
  nested_dissection(p, right, out, mark, tag_base, tag);
  out.insert(out.end(), sep.begin(), sep.end());
}

std::shared_ptr<Problem> make_problem(const ps_problem_desc* desc, const double* coords) {
  auto p = std::make_shared<Problem>();
  p->d = desc->dim;
  p->nnz = desc->nnz;
  p->rp.assign(desc->row_ptr, desc->row_ptr + p->d + 1);
  p->ci.assign(desc->col_idx, desc->col_idx + p->nnz);
  p->M.assign(desc->mass, desc->mass + p->nnz);
  p->linear = desc->stiffness != nullptr;
  if (p->linear) p->K.assign(desc->stiffness, desc->stiffness + p->nnz);
  if (!p->linear) {
    p->ne = desc->n_elem;
    p->npe = desc->nodes_per_elem;
    const int64_t ne = p->ne, npe = p->npe;
    p->en.assign(desc->elem_nodes, desc->elem_nodes + ne * npe);
    p->eS.assign(desc->elem_stiff, desc->elem_stiff + ne * npe * npe);
    p->einvA.assign(desc->elem_inv_area, desc->elem_inv_area + ne);
    p->ecurve.assign(desc->elem_curve, desc->elem_curve + ne);
    p->curves.assign(desc->curves, desc->curves + desc->n_curves);
    p->eslot.assign(ne * npe * npe, -1);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < npe; ++a)
        for (int b = 0; b < npe; ++b) {
          const int32_t na = p->en[e * npe + a], nb = p->en[e * npe + b];
          if (na < 0 || nb < 0) continue;
          const int64_t s = p->slot(na, nb);
          if (s < 0) throw Error(PS_ERR_BAD_ARG, "problem: element coupling missing from pattern");
          p->eslot[(e * npe + a) * npe + b] = s;
        }
  }
  p->T = desc->period;
  p->nterms = desc->n_terms;
  // Excitation ctor (proj/src/problem.cpp:36-50)
  if (!(p->T > 0.0)) throw Error(PS_ERR_BAD_ARG, "problem: excitation period must be positive");
  for (int k = 0; k < p->nterms; ++k) {
    const double fk = desc->frequency_hz[k];
    if (!(fk > 0.0)) throw Error(PS_ERR_BAD_ARG, "problem: excitation frequency must be positive");
    const double cycles = fk * p->T;
    if (std::abs(cycles - std::round(cycles)) > 1e-9 * std::max(1.0, cycles))
      throw Error(PS_ERR_BAD_ARG, "problem: excitation frequency is not an integer multiple of 1/period");
  }
  p->pat.assign(desc->patterns, desc->patterns + static_cast<int64_t>(p->nterms) * p->d);
  p->amp.assign(desc->amplitude, desc->amplitude + p->nterms);
  p->freq.assign(desc->frequency_hz, desc->frequency_hz + p->nterms);
  p->phase.assign(desc->phase_rad, desc->phase_rad + p->nterms);
  if (coords) p->coords.assign(coords, coords + 2 * static_cast<int64_t>(p->d));
  std::vector<int32_t> all(p->d);
  std::iota(all.begin(), all.end(), 0);
  if (!p->coords.empty()) {
    std::vector<int32_t> mark(p->d, 0);
    int tag = 0;
    p->order.reserve(p->d);
    nested_dissection(*p, all, p->order, mark, 0, tag);
  } else {
    p->order = all;
  }
  return p;
}

// proj/src/problem.cpp:52-63
void excitation(const Problem& p, double t, double* f) {
  double tau = std::fmod(t, p.T);
  if (tau < 0.0) tau += p.T;
  std::fill(f, f + p.d, 0.0);
  for (int k = 0; k < p.nterms; ++k) {
    const double arg = 2.0 * kPi * p.freq[k] * tau + p.phase[k];
    const double c = p.amp[k] * std::sin(arg);
    const double* pk = &p.pat[static_cast<int64_t>(k) * p.d];
    for (int i = 0; i < p.d; ++i) f[i] += c * pk[i];
  }
}

// K(u) = sum_e nu(b2_e) S_e  and  J(u) = sum_e nu S_e + 2 nu' invA (S u)(S u)^T,
// accumulated element by element like the triplet assembly of
// proj/src/problem.cpp:204-223,344-359.
void assemble(const Problem& p, const double* u, double* K, double* J) {
  if (p.linear) {
    if (K) std::copy(p.K.begin(), p.K.end(), K);
    if (J) std::copy(p.K.begin(), p.K.end(), J);
    return;
  }
  if (K) std::fill(K, K + p.nnz, 0.0);
  if (J) std::fill(J, J + p.nnz, 0.0);
  const int npe = p.npe;
  double ue[4], g[4];
  for (int64_t e = 0; e < p.ne; ++e) {
    const double* S = &p.eS[e * npe * npe];
    for (int a = 0; a < npe; ++a) {
      const int32_t n = p.en[e * npe + a];
      ue[a] = n >= 0 ? u[n] : 0.0;
    }
    double b2 = 0.0;
    for (int a = 0; a < npe; ++a) {
      double s = 0.0;
      for (int b = 0; b < npe; ++b) s += S[a * npe + b] * ue[b];
      g[a] = s;
      b2 += ue[a] * s;
    }
    b2 *= p.einvA[e];
    const ps_curve& cv = p.curves[p.ecurve[e]];
    const double nu = curve_nu(cv, b2);
    const double c = 2.0 * curve_nu_prime(cv, b2) * p.einvA[e];
    for (int a = 0; a < npe; ++a)
      for (int b = 0; b < npe; ++b) {
        const int64_t s = p.eslot[(e * npe + a) * npe + b];
        if (s < 0) continue;
        if (K) K[s] += nu * S[a * npe + b];
        if (J) J[s] += nu * S[a * npe + b] + c * (g[a] * g[b]);
      }
  }
}

void spmv(const Problem& p, const double* vals, const double* x, double* y) {
  for (int i = 0; i < p.d; ++i) {
    double s = 0.0;
    for (int32_t k = p.rp[i]; k < p.rp[i + 1]; ++k) s += vals[k] * x[p.ci[k]];
    y[i] = s;
  }
}

double norm2(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

// ------------------------------------------------------------ sparse LDL^T
// Up-looking LDL^T of P A P^T (Eigen SimplicialLDLT / SparseLU substitute).
// Works for real symmetric and complex symmetric (no conjugation) matrices.
template <class S>
struct Ldlt {
  int n = 0;
  std::vector<int32_t> perm, iperm, parent, Lp, Lnz, Li;
  std::vector<S> Lx, D;
  bool ok = false;

  // values(k) gives the value of pattern slot k of the original matrix.
  template <class ValueFn>
  void factor(const Problem& p, ValueFn values) {
    n = p.d;
    perm = p.order;
    iperm.assign(n, 0);
    for (int i = 0; i < n; ++i) iperm[perm[i]] = i;
    parent.assign(n, -1);
    Lnz.assign(n, 0);
    std::vector<int32_t> flag(n, -1);
    for (int k = 0; k < n; ++k) {
      flag[k] = k;
      const int32_t row = perm[k];
      for (int32_t q = p.rp[row]; q < p.rp[row + 1]; ++q) {
        int32_t i = iperm[p.ci[q]];
        if (i >= k) continue;
        for (; flag[i] != k; i = parent[i]) {
          if (parent[i] == -1) parent[i] = k;
          Lnz[i]++;
          flag[i] = k;
        }
      }
    }
    Lp.assign(n + 1, 0);
    for (int k = 0; k < n; ++k) Lp[k + 1] = Lp[k] + Lnz[k];
    Li.assign(Lp[n], 0);
    Lx.assign(Lp[n], S(0));
    D.assign(n, S(0));
    std::vector<S> Y(n, S(0));
    std::vector<int32_t> pattern(n);
    std::fill(Lnz.begin(), Lnz.end(), 0);
    std::fill(flag.begin(), flag.end(), -1);
    ok = true;
    for (int k = 0; k < n; ++k) {
      int top = n;
      flag[k] = k;
      const int32_t row = perm[k];
      for (int32_t q = p.rp[row]; q < p.rp[row + 1]; ++q) {
        int32_t i = iperm[p.ci[q]];
        if (i > k) continue;
        Y[i] += values(q);
        int len = 0;
        for (; flag[i] != k; i = parent[i]) {
          pattern[len++] = i;
          flag[i] = k;
        }
        while (len > 0) pattern[--top] = pattern[--len];
      }
      D[k] = Y[k];
      Y[k] = S(0);
      for (; top < n; ++top) {
        const int32_t i = pattern[top];
        const S yi = Y[i];
        Y[i] = S(0);
        const int32_t p2 = Lp[i] + Lnz[i];
        for (int32_t q = Lp[i]; q < p2; ++q) Y[Li[q]] -= Lx[q] * yi;
        const S l_ki = yi / D[i];
        D[k] -= l_ki * yi;
        Li[p2] = k;
        Lx[p2] = l_ki;
        Lnz[i]++;
      }
      if (D[k] == S(0)) ok = false;
    }
  }

  void solve(const S* b, S* x) const {
    std::vector<S> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int j = 0; j < n; ++j)
      for (int32_t q = Lp[j]; q < Lp[j + 1]; ++q) y[Li[q]] -= Lx[q] * y[j];
    for (int j = 0; j < n; ++j) y[j] /= D[j];
    for (int j = n - 1; j >= 0; --j)
      for (int32_t q = Lp[j]; q < Lp[j + 1]; ++q) y[j] -= Lx[q] * y[Li[q]];
    for (int i = 0; i < n; ++i) x[perm[i]] = y[i];
  }
};

// ------------------------------------------------- Jacobi-PCG (device algorithm)
// The exact algorithm the device kernels run: x0 = 0,
// two-phase iteration, beta from the expanded recurrence
//   rho_est = rho - 2 alpha (q.z) + alpha^2 (q.Dq),
// rho recomputed exactly after the update, stop at ||r||^2 <= tol^2 ||b||^2.
// Returns the iteration count; throws on breakdown / budget exhaustion.
template <class S>
S dotu(const S* a, const S* b, int n) {
  S s(0);
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
inline double abs2(double v) { return v * v; }
inline double abs2(const cd& v) { return std::norm(v); }

struct KrylovFailure {
  int kind;  // 0 breakdown, 1 max iterations
};

template <class S, class MatVec>
int jacobi_cg(const Problem& p, MatVec matvec, const S* dinv, const S* b, S* x, double tol,
              int max_iter, bool warm = false) {
  // warm: x holds the start value (r = b - A x; the stop stays relative to b, and
  // a start that already meets it takes no iteration); cold: x = 0, r = b
  const int n = p.d;
  std::vector<S> r(b, b + n), z(n), pv(n), q(n);
  double bb = 0.0;
  for (int i = 0; i < n; ++i) bb += abs2(b[i]);
  if (warm && bb != 0.0) {
    matvec(x, q.data());
    for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];
  } else {
    std::fill(x, x + n, S(0));
  }
  for (int i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
  pv = z;
  S rho = dotu(r.data(), z.data(), n);
  if (bb == 0.0) return 0;
  const double stop = (tol * tol) * bb;
  if (warm) {
    double rr0 = 0.0;
    for (int i = 0; i < n; ++i) rr0 += abs2(r[i]);
    if (rr0 <= stop) return 0;
  }
  int it = 0;
  for (;;) {
    matvec(pv.data(), q.data());
    S pq(0), qz(0), qdq(0);
    for (int i = 0; i < n; ++i) {
      pq += pv[i] * q[i];
      qz += q[i] * z[i];
      qdq += q[i] * (dinv[i] * q[i]);
    }
    if (!(std::isfinite(std::abs(pq))) || pq == S(0)) throw KrylovFailure{0};
    const S alpha = rho / pq;
    const S rho_est = rho - S(2.0) * alpha * qz + alpha * alpha * qdq;
    const S beta = rho_est / rho;
    double rr = 0.0;
    S rz(0);
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * pv[i];
      r[i] -= alpha * q[i];
      z[i] = dinv[i] * r[i];
      pv[i] = z[i] + beta * pv[i];
      rr += abs2(r[i]);
      rz += r[i] * z[i];
    }
    rho = rz;
    ++it;
    if (rr <= stop) return it;
    if (!std::isfinite(rr)) throw KrylovFailure{0};
    if (it >= max_iter) throw KrylovFailure{1};
  }
}

// Solves A x = b for a real step matrix A given by CSR values.
struct RealSolver {
  int mode;
  double tol;
  int max_iter;
  int64_t iterations = 0;
  int last_iterations = 0;

  // returns false if the factorization has a zero pivot
  bool solve(const Problem& p, const std::vector<double>& A, const double* b, double* x) {
    if (mode == OR_DIRECT) {
      Ldlt<double> f;
      f.factor(p, [&](int64_t q) { return A[q]; });
      if (!f.ok) return false;
      f.solve(b, x);
      last_iterations = 0;
      return true;
    }
    std::vector<double> dinv(p.d);
    for (int i = 0; i < p.d; ++i) {
      const int64_t s = p.slot(i, i);
      dinv[i] = 1.0 / (s >= 0 ? A[s] : 0.0);
    }
    auto mv = [&](const double* in, double* out) { spmv(p, A.data(), in, out); };
    last_iterations = jacobi_cg<double>(p, mv, dinv.data(), b, x, tol, max_iter);
    iterations += last_iterations;
    return true;
  }
};

// ------------------------------------------------------------- newton_step
// proj/src/propagators.cpp:13-17 (residual) and :27-58 (Newton)
struct StepOut {
  int iterations = 0;
  std::vector<double> trace;
  int64_t pcg = 0;
  int max_pcg = 0;
};

void step_residual(const Problem& p, const std::vector<double>& K, const double* u,
                   const double* u_prev, double dt, const double* f, double* R) {
  std::vector<double> v(p.d), mv(p.d), ku(p.d);
  for (int i = 0; i < p.d; ++i) v[i] = (u[i] - u_prev[i]) / dt;
  spmv(p, p.M.data(), v.data(), mv.data());
  spmv(p, K.data(), u, ku.data());
  for (int i = 0; i < p.d; ++i) R[i] = mv[i] + ku[i] - f[i];
}

void newton_step(const Problem& p, const ps_solver_settings& s, int mode, const double* u_prev,
                 double t_next, double dt, double* u_out, StepOut* out) {
  const ps_newton_settings& ns = s.newton;
  if (!(dt > 0.0)) throw Error(PS_ERR_BAD_ARG, "propagator: step size must be positive");
  if (ns.max_iter < 1) throw Error(PS_ERR_BAD_ARG, "propagator: Newton needs at least one iteration");
  std::vector<double> f(p.d);
  excitation(p, t_next, f.data());
  const double tol = ns.tol_abs + ns.tol_rel * norm2(f.data(), p.d);
  std::vector<double> u(u_prev, u_prev + p.d), K(p.nnz), J(p.nnz), A(p.nnz), R(p.d), rhs(p.d),
      upd(p.d);
  assemble(p, u.data(), K.data(), nullptr);
  RealSolver solver{mode, s.pcg.tol_rel, s.pcg.max_iter};
  for (int it = 1; it <= ns.max_iter; ++it) {
    step_residual(p, K, u.data(), u_prev, dt, f.data(), R.data());
    assemble(p, u.data(), nullptr, J.data());
    for (int64_t q = 0; q < p.nnz; ++q) A[q] = p.M[q] / dt + J[q];
    for (int i = 0; i < p.d; ++i) rhs[i] = -R[i];
    bool ok;
    try {
      ok = solver.solve(p, A, rhs.data(), upd.data());
    } catch (const KrylovFailure& kf) {
      if (kf.kind == 0) step_failure(PS_ERR_SINGULAR, "step system singular", t_next, norm2(R.data(), p.d));
      step_failure(PS_ERR_PCG_MAXITER, "PCG did not converge", t_next, norm2(R.data(), p.d));
    }
    if (!ok) step_failure(PS_ERR_SINGULAR, "step system not factorizable", t_next, 0.0);
    out->max_pcg = std::max(out->max_pcg, solver.last_iterations);
    for (int i = 0; i < p.d; ++i)
      if (!std::isfinite(upd[i])) step_failure(PS_ERR_SINGULAR, "step system singular", t_next, norm2(R.data(), p.d));
    const double res_pre = norm2(R.data(), p.d);
    double lambda = ns.damping;
    for (int i = 0; i < p.d; ++i) u[i] += lambda * upd[i];
    assemble(p, u.data(), K.data(), nullptr);
    step_residual(p, K, u.data(), u_prev, dt, f.data(), R.data());
    double post = norm2(R.data(), p.d);
    // opt-in residual backtracking (ps_newton_settings.line_search halvings, 0 = the
    // reference's plain damped update): accept when ||R|| <= (1 - 1e-4 lambda) ||R_pre||
    for (int k = 0; k < ns.line_search && !(post <= tol) && !(post <= (1.0 - 1e-4 * lambda) * res_pre); ++k) {
      lambda *= 0.5;
      for (int i = 0; i < p.d; ++i) u[i] -= lambda * upd[i];
      assemble(p, u.data(), K.data(), nullptr);
      step_residual(p, K, u.data(), u_prev, dt, f.data(), R.data());
      post = norm2(R.data(), p.d);
    }
    out->trace.push_back(post);
    out->iterations = it;
    out->pcg = solver.iterations;
    if (!std::isfinite(post)) step_failure(PS_ERR_NEWTON_DIVERGED, "Newton iteration diverged", t_next, post);
    if (post <= tol) {
      std::copy(u.begin(), u.end(), u_out);
      return;
    }
  }
  step_failure(PS_ERR_NEWTON_MAXITER, "Newton did not converge", t_next, out->trace.back());
}

// ------------------------------------------------------------- propagator
// proj/src/propagators.cpp:65-115, TimeMesh proj/include/parasteady/types.hpp:21-40
struct Mesh {
  int N, s;
  double T;
  double coarse_dt() const { return T / N; }
  double fine_dt() const { return coarse_dt() / s; }
  double boundary(int n) const {
    if (n == N) return T;
    return static_cast<double>(n) * T / N;
  }
};

Mesh make_mesh(const ps_time_mesh* m) {
  if (m->subintervals < 2) throw Error(PS_ERR_BAD_ARG, "mesh: need at least 2 subintervals");
  if (m->fine_steps < 1) throw Error(PS_ERR_BAD_ARG, "mesh: need at least 1 fine step per subinterval");
  if (!(m->period > 0.0)) throw Error(PS_ERR_BAD_ARG, "mesh: period must be positive");
  return Mesh{m->subintervals, m->fine_steps, m->period};
}

struct Propagator {
  const Problem& p;
  Mesh mesh;
  ps_solver_settings s;
  int mode;
  mutable std::mutex mu;
  mutable std::map<double, std::shared_ptr<Ldlt<double>>> cache;  // linear_factor, propagators.cpp:71-83
  mutable std::map<double, std::shared_ptr<std::vector<double>>> acache;

  Propagator(const Problem& pr, Mesh m, const ps_solver_settings& st, int md)
      : p(pr), mesh(m), s(st), mode(md) {
    if (p.T != mesh.T) throw Error(PS_ERR_BAD_ARG, "propagator: mesh period does not match the problem");
  }

  std::shared_ptr<std::vector<double>> step_matrix(double dt) const {
    std::lock_guard<std::mutex> lock(mu);
    auto it = acache.find(dt);
    if (it != acache.end()) return it->second;
    auto A = std::make_shared<std::vector<double>>(p.nnz);
    for (int64_t q = 0; q < p.nnz; ++q) (*A)[q] = p.M[q] / dt + p.K[q];
    acache.emplace(dt, A);
    return A;
  }

  std::shared_ptr<Ldlt<double>> linear_factor(double dt) const {
    auto A = step_matrix(dt);
    {
      std::lock_guard<std::mutex> lock(mu);
      auto it = cache.find(dt);
      if (it != cache.end()) return it->second;
    }
    auto f = std::make_shared<Ldlt<double>>();
    f->factor(p, [&](int64_t q) { return (*A)[q]; });
    if (!f->ok) throw Error(PS_ERR_SINGULAR, "propagator: linear step system not factorizable");
    std::lock_guard<std::mutex> lock(mu);
    return cache.emplace(dt, f).first->second;
  }

  // proj/src/propagators.cpp:85-94
  void step(const double* u_prev, double t_next, double dt, double* u, StepOut* st) const {
    if (!p.linear) {
      StepOut o;
      newton_step(p, s, mode, u_prev, t_next, dt, u, &o);
      st->iterations += o.iterations;
      st->pcg += o.pcg;
      st->max_pcg = std::max(st->max_pcg, o.max_pcg);
      st->trace = o.trace;
      return;
    }
    std::vector<double> v(p.d), mv(p.d), f(p.d), rhs(p.d);
    for (int i = 0; i < p.d; ++i) v[i] = u_prev[i] / dt;
    spmv(p, p.M.data(), v.data(), mv.data());
    excitation(p, t_next, f.data());
    for (int i = 0; i < p.d; ++i) rhs[i] = mv[i] + f[i];
    if (mode == OR_DIRECT) {
      linear_factor(dt)->solve(rhs.data(), u);
    } else {
      auto A = step_matrix(dt);
      std::vector<double> dinv(p.d);
      for (int i = 0; i < p.d; ++i) dinv[i] = 1.0 / (*A)[p.slot(i, i)];
      auto mvf = [&](const double* in, double* out) { spmv(p, A->data(), in, out); };
      int its;
      try {
        its = jacobi_cg<double>(p, mvf, dinv.data(), rhs.data(), u, s.pcg.tol_rel, s.pcg.max_iter);
      } catch (const KrylovFailure& kf) {
        if (kf.kind == 0) step_failure(PS_ERR_SINGULAR, "step system singular", t_next, 0.0);
        step_failure(PS_ERR_PCG_MAXITER, "PCG did not converge", t_next, 0.0);
      }
      st->pcg += its;
      st->max_pcg = std::max(st->max_pcg, its);
    }
    st->iterations += 1;
    for (int i = 0; i < p.d; ++i)
      if (!std::isfinite(u[i])) step_failure(PS_ERR_SINGULAR, "step system singular", t_next, 0.0);
  }

  void coarse_propagate(int n, const double* u0, double* u1, StepOut* st) const {
    if (n < 1 || n > mesh.N) throw Error(PS_ERR_BAD_ARG, "propagator: subinterval index out of range");
    step(u0, mesh.boundary(n), mesh.coarse_dt(), u1, st);
  }

  void fine_propagate(int n, const double* u0, double* u1, StepOut* st) const {
    if (n < 1 || n > mesh.N) throw Error(PS_ERR_BAD_ARG, "propagator: subinterval index out of range");
    const double t_left = mesh.boundary(n - 1);
    const double dt = mesh.fine_dt();
    std::vector<double> u(u0, u0 + p.d), nxt(p.d);
    for (int j = 1; j <= mesh.s; ++j) {
      const double t_next = j == mesh.s ? mesh.boundary(n) : t_left + j * dt;
      step(u.data(), t_next, dt, nxt.data(), st);
      u.swap(nxt);
    }
    std::copy(u.begin(), u.end(), u1);
  }
};

// ---------------------------------------------------------------- spectral
// dft_bins (proj/src/spectral.cpp:32-63): unitary DFT across the list index,
// FFT bin order, both directions scaled by N^{-1/2}.  Direct summation with an
// exact twiddle table replaces FFTW.
void dft_bins(int n, int d, const cd* in, cd* out, int sign) {
  std::vector<cd> tw(n);
  for (int k = 0; k < n; ++k) {
    const double ang = 2.0 * kPi * k / n;
    tw[k] = cd(std::cos(ang), sign < 0 ? -std::sin(ang) : std::sin(ang));
  }
  const double scale = 1.0 / std::sqrt(static_cast<double>(n));
  if (n >= 64 && (n & (n - 1)) == 0) {
    // large power-of-two block counts: iterative radix-2 FFT per DOF (the
    // reference runs FFTW, proj/src/spectral.cpp:42-50), same unitary scale
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    std::vector<cd> a(n);
    for (int j = 0; j < d; ++j) {
      for (int m = 0; m < n; ++m) {
        int r = 0;
        for (int bit = 0; bit < lg; ++bit) r |= ((m >> bit) & 1) << (lg - 1 - bit);
        a[r] = in[static_cast<int64_t>(m) * d + j];
      }
      for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1, step = n / len;
        for (int i0 = 0; i0 < n; i0 += len)
          for (int k = 0; k < half; ++k) {
            const cd t = tw[static_cast<int64_t>(k) * step] * a[i0 + k + half];
            a[i0 + k + half] = a[i0 + k] - t;
            a[i0 + k] += t;
          }
      }
      for (int b = 0; b < n; ++b) out[static_cast<int64_t>(b) * d + j] = scale * a[b];
    }
    return;
  }
  for (int b = 0; b < n; ++b) {
    for (int j = 0; j < d; ++j) {
      cd acc(0.0, 0.0);
      for (int m = 0; m < n; ++m) acc += in[static_cast<int64_t>(m) * d + j] * tw[(static_cast<int64_t>(b) * m) % n];
      out[static_cast<int64_t>(b) * d + j] = scale * acc;
    }
  }
}

void require_even_blocks(int n, const char* where) {
  if (n < 2 || n % 2 != 0)
    throw Error(PS_ERR_ODD_BLOCKS, std::string("spectral: ") + where +
                                       " requires an even number of blocks >= 2, got " + std::to_string(n));
}

// realify (proj/src/spectral.cpp:72-84)
void realify(int n, int d, const cd* bins, double* out) {
  double real_max = 0.0, imag_max = 0.0;
  const int64_t total = static_cast<int64_t>(n) * d;
  for (int64_t i = 0; i < total; ++i) {
    real_max = std::max(real_max, std::fabs(bins[i].real()));
    imag_max = std::max(imag_max, std::fabs(bins[i].imag()));
  }
  if (imag_max > kImagResidualTol * std::max(1.0, real_max))
    throw Error(PS_ERR_CONJ_SYMMETRY,
                "spectral: conjugate symmetry violated (imaginary residue " + std::to_string(imag_max) + ")");
  for (int64_t i = 0; i < total; ++i) out[i] = bins[i].real();
}

int harmonic_index(int bin, int n) { return bin <= n / 2 ? bin : bin - n; }  // spectral.cpp:94-103

// proj/src/spectral.cpp:134-150
void assemble_rhs(const Problem& lin, const Mesh& mesh, const double* F, const double* G, double* rhs) {
  const int n = mesh.N, d = lin.d;
  const double dT = mesh.coarse_dt();
  std::vector<double> q(lin.nnz), jump(d), qj(d), f(d);
  for (int64_t k = 0; k < lin.nnz; ++k) {
    const double c = lin.M[k] / dT;
    q[k] = c + lin.K[k];
  }
  for (int row = 0; row < n; ++row) {
    const int sub = row == 0 ? n : row;
    for (int i = 0; i < d; ++i)
      jump[i] = F[static_cast<int64_t>(sub - 1) * d + i] - G[static_cast<int64_t>(sub - 1) * d + i];
    spmv(lin, q.data(), jump.data(), qj.data());
    excitation(lin, mesh.boundary(sub), f.data());
    for (int i = 0; i < d; ++i) rhs[static_cast<int64_t>(row) * d + i] = qj[i] + f[i];
  }
}

// per-bin factor / back-substitution seconds of the last DIRECT mh_solve (summed
// over bins) and the wall seconds of its bin loop (or_last_direct_timing)
std::mutex g_direct_timing_mu;
double g_direct_timing[3] = {0.0, 0.0, 0.0};

// MultiharmonicCyclicSolver (proj/src/spectral.cpp:224-279) with the bin mask
// and shift-kind extensions of SURVEY.md App. A.3/A.4.
// warm (ITERATIVE, s.cocg.warm_start): the previous solve's spectrum, used as
// the COCG start value of every solved bin and replaced by this solve's
// (empty on the first solve: cold start).
void mh_solve(const Problem& lin, const Mesh& mesh, const ps_solver_settings& s, int mode,
              bool conj, const int32_t* mask, int shift_kind, const double* rhs, double* U,
              int workers, int64_t* cocg_iters, std::vector<cd>* warm = nullptr) {
  const int n = mesh.N, d = lin.d;
  require_even_blocks(n, "multiharmonic solve");
  const double dT = mesh.coarse_dt();
  std::vector<double> C(lin.nnz), Q(lin.nnz);
  for (int64_t k = 0; k < lin.nnz; ++k) {
    C[k] = lin.M[k] / dT;
    Q[k] = C[k] + lin.K[k];
  }
  std::vector<cd> in(static_cast<int64_t>(n) * d), hat(in.size()), sol(in.size(), cd(0, 0)), back(in.size());
  const bool warm_start = warm && s.cocg.warm_start && mode != OR_DIRECT && warm->size() == sol.size();
  if (warm_start) sol = *warm;
  for (int64_t i = 0; i < static_cast<int64_t>(in.size()); ++i) in[i] = cd(rhs[i], 0.0);
  dft_bins(n, d, in.data(), hat.data(), -1);
  const int last = conj ? n / 2 : n - 1;
  std::vector<int64_t> its(last + 1, 0);
  if (mode == OR_DIRECT) g_direct_timing[0] = g_direct_timing[1] = 0.0;
  const auto t_loop = std::chrono::steady_clock::now();
  parallel_for(last + 1, workers, [&](int bin) {
    if (mask && mask[bin] == 0) return;
    const int p = harmonic_index(bin, n);
    std::vector<cd> lam(lin.nnz);
    if (shift_kind == 0) {
      const cd phase = std::exp(cd(0.0, -2.0 * kPi * p / n));  // harmonic_block, spectral.cpp:224-231
      for (int64_t k = 0; k < lin.nnz; ++k) lam[k] = cd(Q[k], 0.0) - phase * cd(C[k], 0.0);
    } else {
      const double omega = 2.0 * kPi * p / mesh.T;
      for (int64_t k = 0; k < lin.nnz; ++k) lam[k] = cd(lin.K[k], 0.0) + cd(0.0, omega) * cd(lin.M[k], 0.0);
    }
    cd* x = &sol[static_cast<int64_t>(bin) * d];
    const cd* b = &hat[static_cast<int64_t>(bin) * d];
    if (mode == OR_DIRECT) {
      // factor once per bin (the solver's constructor, proj/src/spectral.cpp:233-255),
      // then the per-iteration back-substitution (:257-279); both timed per bin
      const auto t0 = std::chrono::steady_clock::now();
      Ldlt<cd> f;
      f.factor(lin, [&](int64_t q) { return lam[q]; });
      const auto t1 = std::chrono::steady_clock::now();
      if (!f.ok) {
        std::ostringstream msg;
        msg << "spectral: harmonic block p = " << p << " is singular";
        throw Error(PS_ERR_SINGULAR_BLOCK, msg.str());
      }
      f.solve(b, x);
      const auto t2 = std::chrono::steady_clock::now();
      std::lock_guard<std::mutex> lk(g_direct_timing_mu);
      g_direct_timing[0] += std::chrono::duration<double>(t1 - t0).count();
      g_direct_timing[1] += std::chrono::duration<double>(t2 - t1).count();
    } else {
      std::vector<cd> dinv(d);
      for (int i = 0; i < d; ++i) dinv[i] = cd(1.0, 0.0) / lam[lin.slot(i, i)];
      auto mv = [&](const cd* xin, cd* yout) {
        for (int i = 0; i < d; ++i) {
          cd acc(0, 0);
          for (int32_t k = lin.rp[i]; k < lin.rp[i + 1]; ++k) acc += lam[k] * xin[lin.ci[k]];
          yout[i] = acc;
        }
      };
      try {
        its[bin] = jacobi_cg<cd>(lin, mv, dinv.data(), b, x, s.cocg.tol_rel, s.cocg.max_iter, warm_start);
      } catch (const KrylovFailure& kf) {
        std::ostringstream msg;
        if (kf.kind == 0) {
          msg << "spectral: harmonic block p = " << p << " is singular";
          throw Error(PS_ERR_SINGULAR_BLOCK, msg.str());
        }
        msg << "spectral: COCG did not converge for harmonic block p = " << p;
        throw Error(PS_ERR_COCG_MAXITER, msg.str());
      }
    }
    for (int i = 0; i < d; ++i)
      if (!std::isfinite(x[i].real()) || !std::isfinite(x[i].imag()))
        throw Error(PS_ERR_NONFINITE, "spectral: harmonic solve produced non-finite values");
  });
  if (mode == OR_DIRECT)
    g_direct_timing[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_loop).count();
  if (cocg_iters) *cocg_iters += std::accumulate(its.begin(), its.end(), int64_t{0});
  if (warm && s.cocg.warm_start && mode != OR_DIRECT) *warm = sol;
  if (conj)
    for (int bin = n / 2 + 1; bin < n; ++bin)
      for (int i = 0; i < d; ++i)
        sol[static_cast<int64_t>(bin) * d + i] = std::conj(sol[static_cast<int64_t>(n - bin) * d + i]);
  dft_bins(n, d, sol.data(), back.data(), +1);
  realify(n, d, back.data(), U);
}

// proj/src/engine.cpp:54-64
double jump_norm(int count, int d, const double* cur, const double* prev) {
  if (count < 1) throw Error(PS_ERR_BAD_ARG, "engine: jump_norm needs two state lists of equal length");
  double change = 0.0, scale = 1.0;
  for (int n = 0; n < count; ++n) {
    double c = 0.0, s = 0.0;
    for (int i = 0; i < d; ++i) {
      const double a = cur[static_cast<int64_t>(n) * d + i];
      const double df = a - prev[static_cast<int64_t>(n) * d + i];
      c += df * df;
      s += a * a;
    }
    change = std::max(change, std::sqrt(c));
    scale = std::max(scale, std::sqrt(s));
  }
  return change / scale;
}

// proj/src/engine.cpp:66-74
std::shared_ptr<Problem> frozen(const Problem& p, const double* ref) {
  auto lin = std::make_shared<Problem>(p);
  if (p.linear) return lin;
  std::vector<double> zero(p.d, 0.0);
  lin->K.assign(p.nnz, 0.0);
  assemble(p, ref ? ref : zero.data(), lin->K.data(), nullptr);
  lin->linear = true;
  return lin;
}

}  // namespace orc

using namespace orc;

struct or_problem {
  std::shared_ptr<Problem> p;
};

namespace {
template <class Fn>
int guard(Fn fn) {
  try {
    fn();
    return PS_OK;
  } catch (const Error& e) {
    g_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}
}  // namespace

extern "C" {

const char* or_last_error(void) { return g_error.c_str(); }

int or_create(const ps_problem_desc* desc, const double* coords, or_problem** out) {
  return guard([&] { *out = new or_problem{make_problem(desc, coords)}; });
}
void or_free(or_problem* p) { delete p; }
int or_dim(const or_problem* p) { return p->p->d; }
int or_nnz(const or_problem* p) { return static_cast<int>(p->p->nnz); }
int or_is_linear(const or_problem* p) { return p->p->linear ? 1 : 0; }
int or_frozen(const or_problem* p, const double* u_ref, or_problem** out) {
  return guard([&] { *out = new or_problem{frozen(*p->p, u_ref)}; });
}

void or_nu(const ps_curve* curve, int32_t n, const double* b2, double* nu, double* nu_prime) {
  for (int i = 0; i < n; ++i) {
    if (nu) nu[i] = curve_nu(*curve, b2[i]);
    if (nu_prime) nu_prime[i] = curve_nu_prime(*curve, b2[i]);
  }
}

int or_excitation(const or_problem* p, double t, double* f) {
  return guard([&] { excitation(*p->p, t, f); });
}
int or_stiffness_at(const or_problem* p, const double* u, double* K) {
  return guard([&] { assemble(*p->p, u, K, nullptr); });
}
int or_newton_matrix_at(const or_problem* p, const double* u, double* J) {
  return guard([&] { assemble(*p->p, u, nullptr, J); });
}

int or_newton_step(const or_problem* p, const ps_solver_settings* s, int32_t mode,
                   const double* u_prev, double t_next, double dt, double* u_out,
                   int32_t* iterations, double* trace, int64_t* pcg_iterations) {
  StepOut o;
  const int rc = guard([&] { newton_step(*p->p, *s, mode, u_prev, t_next, dt, u_out, &o); });
  if (iterations) *iterations = o.iterations;
  if (trace)
    for (size_t i = 0; i < o.trace.size(); ++i) trace[i] = o.trace[i];
  if (pcg_iterations) *pcg_iterations = o.pcg;
  return rc;
}

static int propagate_batch(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                           int32_t mode, int32_t n_first, int32_t count, const double* U_start,
                           double* U_end, int32_t workers, or_stats* stats, bool fine) {
  std::vector<StepOut> outs(count > 0 ? count : 0);
  const int rc = guard([&] {
    const Mesh m = make_mesh(mesh);
    Propagator prop(*p->p, m, *s, mode);
    const int d = p->p->d;
    parallel_for(count, workers, [&](int i) {
      const double* u0 = U_start + static_cast<int64_t>(i) * d;
      double* u1 = U_end + static_cast<int64_t>(i) * d;
      if (fine)
        prop.fine_propagate(n_first + i, u0, u1, &outs[i]);
      else
        prop.coarse_propagate(n_first + i, u0, u1, &outs[i]);
    });
  });
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    for (const auto& o : outs) {
      stats->newton_iterations += o.iterations;
      stats->pcg_iterations += o.pcg;
      stats->max_pcg_iterations = std::max(stats->max_pcg_iterations, o.max_pcg);
    }
    stats->code = rc;
    stats->failed_index = -1;
  }
  return rc;
}

int or_fine_propagate_batch(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                            int32_t mode, int32_t n_first, int32_t count, const double* U_start,
                            double* U_end, int32_t workers, or_stats* stats) {
  return propagate_batch(p, mesh, s, mode, n_first, count, U_start, U_end, workers, stats, true);
}
int or_coarse_propagate_batch(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                              int32_t mode, int32_t n_first, int32_t count, const double* U_start,
                              double* U_end, int32_t workers, or_stats* stats) {
  return propagate_batch(p, mesh, s, mode, n_first, count, U_start, U_end, workers, stats, false);
}

// proj/src/engine.cpp:213-218
int or_coarse_sweep(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                    int32_t mode, double* U) {
  return guard([&] {
    const Mesh m = make_mesh(mesh);
    Propagator prop(*p->p, m, *s, mode);
    const int d = p->p->d;
    std::fill(U, U + d, 0.0);
    StepOut st;
    for (int n = 1; n < m.N; ++n)
      prop.coarse_propagate(n, U + static_cast<int64_t>(n - 1) * d, U + static_cast<int64_t>(n) * d, &st);
  });
}

int or_forward_dft(int32_t n, int32_t d, const double* U, double* spectrum) {
  return guard([&] {
    require_even_blocks(n, "forward_dft");
    std::vector<cd> in(static_cast<int64_t>(n) * d);
    for (size_t i = 0; i < in.size(); ++i) in[i] = cd(U[i], 0.0);
    dft_bins(n, d, in.data(), reinterpret_cast<cd*>(spectrum), -1);
  });
}

int or_inverse_dft(int32_t n, int32_t d, const double* spectrum, double* U) {
  return guard([&] {
    require_even_blocks(n, "inverse_dft");
    std::vector<cd> back(static_cast<int64_t>(n) * d);
    dft_bins(n, d, reinterpret_cast<const cd*>(spectrum), back.data(), +1);
    realify(n, d, back.data(), U);
  });
}

int or_assemble_rhs(const or_problem* lin, const ps_time_mesh* mesh, const double* F, const double* G,
                    double* rhs) {
  return guard([&] {
    if (!lin->p->linear)
      throw Error(PS_ERR_NOT_LINEAR,
                  "spectral: cyclic system requires a linear problem (freeze the coarse operator first)");
    assemble_rhs(*lin->p, make_mesh(mesh), F, G, rhs);
  });
}

int or_mh_solve(const or_problem* lin, const ps_time_mesh* mesh, const ps_solver_settings* s,
                int32_t mode, int32_t use_conjugate_symmetry, const int32_t* bin_mask,
                int32_t shift_kind, const double* rhs, double* U, int32_t workers,
                int64_t* cocg_iterations) {
  return guard([&] {
    if (!lin->p->linear)
      throw Error(PS_ERR_NOT_LINEAR,
                  "spectral: cyclic system requires a linear problem (freeze the coarse operator first)");
    if (cocg_iterations) *cocg_iterations = 0;
    mh_solve(*lin->p, make_mesh(mesh), *s, mode, use_conjugate_symmetry != 0, bin_mask, shift_kind,
             rhs, U, workers, cocg_iterations);
  });
}

int or_last_direct_timing(double* factor_s, double* solve_s, double* wall_s) {
  std::lock_guard<std::mutex> lk(g_direct_timing_mu);
  if (factor_s) *factor_s = g_direct_timing[0];
  if (solve_s) *solve_s = g_direct_timing[1];
  if (wall_s) *wall_s = g_direct_timing[2];
  return PS_OK;
}

// solve_cyclic_direct (proj/src/spectral.cpp:152-188): dense (N d)^2 Gaussian
// elimination with partial pivoting; test-size systems only.
int or_solve_cyclic_direct(const or_problem* lin, const ps_time_mesh* mesh, const double* rhs, double* U) {
  return guard([&] {
    const Problem& p = *lin->p;
    const Mesh m{mesh->subintervals, mesh->fine_steps, mesh->period};
    const int n = m.N, d = p.d;
    const int64_t sz = static_cast<int64_t>(n) * d;
    if (sz > 4096) throw Error(PS_ERR_BAD_ARG, "oracle: direct cyclic solve limited to N*d <= 4096");
    const double dT = m.coarse_dt();
    std::vector<double> big(sz * sz, 0.0), x(rhs, rhs + sz);
    for (int row = 0; row < n; ++row) {
      const int prev = (row + n - 1) % n;
      for (int i = 0; i < d; ++i)
        for (int32_t k = p.rp[i]; k < p.rp[i + 1]; ++k) {
          const double c = p.M[k] / dT;
          big[(row * d + i) * sz + row * d + p.ci[k]] += c + p.K[k];
          big[(row * d + i) * sz + prev * d + p.ci[k]] += -c;
        }
    }
    for (int64_t c = 0; c < sz; ++c) {
      int64_t piv = c;
      for (int64_t r = c + 1; r < sz; ++r)
        if (std::fabs(big[r * sz + c]) > std::fabs(big[piv * sz + c])) piv = r;
      if (big[piv * sz + c] == 0.0) throw Error(PS_ERR_SINGULAR, "spectral: cyclic system is singular");
      if (piv != c) {
        for (int64_t k = 0; k < sz; ++k) std::swap(big[c * sz + k], big[piv * sz + k]);
        std::swap(x[c], x[piv]);
      }
      for (int64_t r = c + 1; r < sz; ++r) {
        const double f = big[r * sz + c] / big[c * sz + c];
        if (f == 0.0) continue;
        for (int64_t k = c; k < sz; ++k) big[r * sz + k] -= f * big[c * sz + k];
        x[r] -= f * x[c];
      }
    }
    for (int64_t c = sz - 1; c >= 0; --c) {
      double s = x[c];
      for (int64_t k = c + 1; k < sz; ++k) s -= big[c * sz + k] * x[k];
      x[c] = s / big[c * sz + c];
    }
    std::copy(x.begin(), x.end(), U);
  });
}

double or_jump_norm(int32_t count, int32_t d, const double* cur, const double* prev) {
  double out = -1.0;
  guard([&] { out = jump_norm(count, d, cur, prev); });
  return out;
}

// solve_pp_pc with the multiharmonic coarse solver (proj/src/engine.cpp:187-270)
int or_pppc_solve(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                  const ps_engine_settings* e, int32_t mode, const double* frozen_ref, double* U_out,
                  double* iterates, ps_history* history, int32_t workers) {
  return guard([&] {
    if (!(e->tol > 0.0)) throw Error(PS_ERR_BAD_ARG, "engine: tolerance must be positive");
    if (e->max_iterations < 1) throw Error(PS_ERR_BAD_ARG, "engine: need at least one iteration");
    const Mesh m = make_mesh(mesh);
    const Problem& prob = *p->p;
    const int n_sub = m.N, d = prob.d;
    const int64_t nd = static_cast<int64_t>(n_sub) * d;
    auto coarse_problem = frozen(prob, frozen_ref);
    Propagator fine(prob, m, *s, mode);
    Propagator coarse(*coarse_problem, m, *s, mode);
    require_even_blocks(n_sub, "multiharmonic solve");
    ps_history h;
    std::memset(&h, 0, sizeof(h));
    std::vector<double> u(nd, 0.0), fine_end(nd), coarse_end(nd), rhs(nd), next(nd);
    StepOut sweep;
    for (int n = 1; n < n_sub; ++n)
      coarse.coarse_propagate(n, &u[static_cast<int64_t>(n - 1) * d], &u[static_cast<int64_t>(n) * d], &sweep);
    h.coarse_pcg_iterations += sweep.pcg;
    std::vector<cd> warm;  // the previous iteration's spectrum (COCG warm start)
    for (int k = 0; k < e->max_iterations; ++k) {
      std::vector<StepOut> fo(n_sub), co(n_sub);
      parallel_for(n_sub, workers, [&](int i) {
        fine.fine_propagate(i + 1, &u[static_cast<int64_t>(i) * d], &fine_end[static_cast<int64_t>(i) * d], &fo[i]);
      });
      parallel_for(n_sub, workers, [&](int i) {
        coarse.coarse_propagate(i + 1, &u[static_cast<int64_t>(i) * d], &coarse_end[static_cast<int64_t>(i) * d], &co[i]);
      });
      for (int i = 0; i < n_sub; ++i) {
        h.fine_pcg_iterations += fo[i].pcg;
        h.newton_iterations += fo[i].iterations;
        h.coarse_pcg_iterations += co[i].pcg;
      }
      assemble_rhs(*coarse_problem, m, fine_end.data(), coarse_end.data(), rhs.data());
      int64_t cocg = 0;
      mh_solve(*coarse_problem, m, *s, mode, e->use_conjugate_symmetry != 0, e->bin_mask, e->shift_kind,
               rhs.data(), next.data(), workers, &cocg, &warm);
      h.cocg_iterations += cocg;
      if (k < PS_MAX_HISTORY) h.cocg_per_iteration[k] = cocg;
      const double jump = jump_norm(n_sub, d, next.data(), u.data());
      if (k < PS_MAX_HISTORY) h.jumps[k] = jump;
      h.iterations = k + 1;
      u.swap(next);
      if (iterates) std::copy(u.begin(), u.end(), iterates + static_cast<int64_t>(k) * nd);
      if (jump <= e->tol) {
        h.converged = 1;
        break;
      }
    }
    std::copy(u.begin(), u.end(), U_out);
    if (history) *history = h;
  });
}

// proj/src/engine.cpp:76-129 (classic_parareal) and :131-185 (solve_pp_ic):
// fine batch over all subintervals, then the sequential coarse sweep with the
// correction u_n = F_n + (G_new - G_old); the coarse propagator is the same
// (nonlinear) problem over one coarse step.  U_out holds N + 1 states
// (classic) or the N states T_0..T_{N-1} (PP-IC); iterates [k][N+1][d].
namespace {
int parareal_family(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                    const ps_engine_settings* e, int32_t mode, const double* u0, bool periodic, double* U_out,
                    double* iterates, ps_history* history, int32_t workers) {
  return guard([&] {
    if (!(e->tol > 0.0)) throw Error(PS_ERR_BAD_ARG, "engine: tolerance must be positive");
    if (e->max_iterations < 1) throw Error(PS_ERR_BAD_ARG, "engine: need at least one iteration");
    if (workers < 1) throw Error(PS_ERR_BAD_ARG, "engine: worker count must be >= 1");
    const Mesh m = make_mesh(mesh);
    const Problem& prob = *p->p;
    const int n_sub = m.N, d = prob.d;
    const int64_t nd1 = static_cast<int64_t>(n_sub + 1) * d;
    Propagator prop(prob, m, *s, mode);
    ps_history h;
    std::memset(&h, 0, sizeof(h));
    std::vector<double> u(nd1, 0.0), g_old(static_cast<int64_t>(n_sub) * d), fine_end(static_cast<int64_t>(n_sub) * d),
        g_new(d);
    if (!periodic) std::copy(u0, u0 + d, u.begin());
    {
      StepOut st;
      for (int n = 1; n <= n_sub; ++n) {
        prop.coarse_propagate(n, &u[static_cast<int64_t>(n - 1) * d], &u[static_cast<int64_t>(n) * d], &st);
        std::copy(&u[static_cast<int64_t>(n) * d], &u[static_cast<int64_t>(n) * d] + d,
                  &g_old[static_cast<int64_t>(n - 1) * d]);
      }
      h.coarse_pcg_iterations += st.pcg;
    }
    for (int k = 0; k < e->max_iterations; ++k) {
      const std::vector<double> u_old = u;
      std::vector<StepOut> fo(n_sub);
      parallel_for(n_sub, workers, [&](int i) {
        prop.fine_propagate(i + 1, &u_old[static_cast<int64_t>(i) * d], &fine_end[static_cast<int64_t>(i) * d],
                            &fo[i]);
      });
      for (int i = 0; i < n_sub; ++i) {
        h.fine_pcg_iterations += fo[i].pcg;
        h.newton_iterations += fo[i].iterations;
      }
      // periodicity by relaxation (PP-IC): the new period start is the old end
      if (periodic)
        std::copy(&u_old[static_cast<int64_t>(n_sub) * d], &u_old[static_cast<int64_t>(n_sub) * d] + d, u.begin());
      StepOut st;
      for (int n = 1; n <= n_sub; ++n) {
        prop.coarse_propagate(n, &u[static_cast<int64_t>(n - 1) * d], g_new.data(), &st);
        double* un = &u[static_cast<int64_t>(n) * d];
        const double* fe = &fine_end[static_cast<int64_t>(n - 1) * d];
        double* go = &g_old[static_cast<int64_t>(n - 1) * d];
        for (int i = 0; i < d; ++i) {
          un[i] = fe[i] + (g_new[i] - go[i]);
          go[i] = g_new[i];
        }
      }
      h.coarse_pcg_iterations += st.pcg;
      const double jump = jump_norm(n_sub + 1, d, u.data(), u_old.data());
      if (k < PS_MAX_HISTORY) h.jumps[k] = jump;
      h.iterations = k + 1;
      if (iterates) std::copy(u.begin(), u.end(), iterates + static_cast<int64_t>(k) * nd1);
      bool done = jump <= e->tol;
      if (periodic) {
        // relative_defect(u[N], u[0]), proj/src/engine.cpp:26-28
        const double* w = &u[static_cast<int64_t>(n_sub) * d];
        double df = 0.0, nw = 0.0;
        for (int i = 0; i < d; ++i) {
          df += (w[i] - u[i]) * (w[i] - u[i]);
          nw += w[i] * w[i];
        }
        h.final_defect = std::sqrt(df) / std::max(1.0, std::sqrt(nw));
        done = done && h.final_defect <= e->tol;
      }
      if (done) {
        h.converged = 1;
        break;
      }
    }
    std::copy(u.begin(), u.begin() + (periodic ? nd1 - d : nd1), U_out);
    if (history) *history = h;
  });
}
}  // namespace

int or_classic_parareal(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                        const ps_engine_settings* e, int32_t mode, const double* u0, double* U_out, double* iterates,
                        ps_history* history, int32_t workers) {
  if (!u0) return PS_ERR_BAD_ARG;
  return parareal_family(p, mesh, s, e, mode, u0, false, U_out, iterates, history, workers);
}

int or_pp_ic_solve(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                   const ps_engine_settings* e, int32_t mode, double* U_out, double* iterates, ps_history* history,
                   int32_t workers) {
  return parareal_family(p, mesh, s, e, mode, nullptr, true, U_out, iterates, history, workers);
}

// proj/src/engine.cpp:272-290
int or_fine_periodicity_defect(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                               int32_t mode, const double* U, double* defect, int32_t workers) {
  return guard([&] {
    const Mesh m = make_mesh(mesh);
    const int n_sub = m.N, d = p->p->d;
    Propagator prop(*p->p, m, *s, mode);
    std::vector<double> out(static_cast<int64_t>(n_sub) * d);
    std::vector<StepOut> st(n_sub);
    parallel_for(n_sub, workers, [&](int i) {
      prop.fine_propagate(i + 1, U + static_cast<int64_t>(i) * d, &out[static_cast<int64_t>(i) * d], &st[i]);
    });
    double scale = 0.0;
    for (int n = 0; n < n_sub; ++n) scale = std::max(scale, norm2(U + static_cast<int64_t>(n) * d, d));
    scale = std::max(1.0, scale);
    double worst = 0.0;
    for (int n = 0; n < n_sub; ++n) {
      const double* target = U + static_cast<int64_t>((n + 1) % n_sub) * d;
      double acc = 0.0;
      for (int i = 0; i < d; ++i) {
        const double df = out[static_cast<int64_t>(n) * d + i] - target[i];
        acc += df * df;
      }
      worst = std::max(worst, std::sqrt(acc));
    }
    *defect = worst / scale;
  });
}

// proj/src/propagators.cpp:117-149
int or_sequential_steady_state(const or_problem* p, const ps_time_mesh* mesh, const ps_solver_settings* s,
                               int32_t mode, double tol, int32_t max_periods, double* U_out,
                               int32_t* periods, int32_t* converged, double* defects) {
  return guard([&] {
    if (!(tol > 0.0)) throw Error(PS_ERR_BAD_ARG, "propagator: tolerance must be positive");
    if (max_periods < 1) throw Error(PS_ERR_BAD_ARG, "propagator: need at least one period");
    const Mesh m = make_mesh(mesh);
    const int d = p->p->d;
    Propagator prop(*p->p, m, *s, mode);
    std::vector<double> u(d, 0.0), traj(static_cast<int64_t>(m.N) * d), u_end(d);
    *converged = 0;
    StepOut st;
    for (int per = 1; per <= max_periods; ++per) {
      std::copy(u.begin(), u.end(), traj.begin());
      for (int n = 1; n < m.N; ++n)
        prop.fine_propagate(n, &traj[static_cast<int64_t>(n - 1) * d], &traj[static_cast<int64_t>(n) * d], &st);
      prop.fine_propagate(m.N, &traj[static_cast<int64_t>(m.N - 1) * d], u_end.data(), &st);
      double diff = 0.0;
      for (int i = 0; i < d; ++i) diff += (u_end[i] - u[i]) * (u_end[i] - u[i]);
      const double defect = std::sqrt(diff) / std::max(1.0, norm2(u_end.data(), d));
      if (defects) defects[per - 1] = defect;
      *periods = per;
      std::copy(traj.begin(), traj.end(), U_out);
      u = u_end;
      if (defect <= tol) {
        *converged = 1;
        break;
      }
    }
  });
}

}  // extern "C"
