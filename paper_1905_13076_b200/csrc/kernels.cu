// Batched fine / coarse propagation on B200 (sm_100a), fp64.
//
// One persistent cooperative kernel runs a whole batch of implicit-Euler
// propagations (proj/src/propagators.cpp:96-115): every time step, every
// Newton iteration (proj/src/propagators.cpp:27-58) and every Jacobi-PCG
// iteration of the step solve stays on the device.  The host only sees the
// final states and a per-system status word.
//
// Layout: systems are split into groups of L <= 32; group g's
// vectors are stored row-major with 32 padded lanes, element (row i, lane l)
// at  g*d*32 + i*32 + l  (per-system matrix values: g*nnz*32 + k*32 + l).  A
// warp lane owns one system; one CSR slot's column index is a broadcast and
// the group's 32 lanes read one aligned 256-byte segment, and every block
// streams a contiguous region of each array.  A group is served by C blocks of
// 512 threads that synchronise only among themselves through a monotone
// arrival counter (group_sync.cuh).  Every block reduces the group's
// dot-product partials redundantly in a fixed order, so all blocks hold
// bit-identical per-system scalars and take identical branches.  Each lane runs
// its own state machine (one action per barrier interval), so systems never
// wait for one another's Newton or PCG iteration counts.
#include "group_sync.cuh"
#include "pppc_internal.h"

#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>

namespace pppc {
namespace {

constexpr double kVacuumReluctivity = 1.0 / (4.0e-7 * 3.14159265358979323846);
constexpr int kLanes = 32;  // padded lanes per group row

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
  bool pact;
  int pit;
  double rho, stop, alpha, beta;
  double res_pre;
  double lambda;   // current Newton step length (damping, halved on backtracks)
  int ls_k;        // backtracks taken in this Newton iteration
  bool bt;         // the pending update round is a backtrack
  bool zero_dx;    // the step solve took 0 iterations (delta = 0)
  long long newton_total, pcg_total;
  int max_nit, max_pit, last_nit;
};

__device__ __forceinline__ void lane_fail(Lane& s, int code, double res, double t) {
  if (!s.alive) return;
  s.alive = false;
  s.pact = false;
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

// Element quantities from the state u (element (n) at u[off + n*rs]).
template <int NPE>
__device__ __forceinline__ void eval_elem(const PropParams& P, const ps_curve* curves, int e, const double* u,
                                          size_t off, size_t rs, Elem<NPE>& E) {
#pragma unroll
  for (int b = 0; b < NPE; ++b) {
    const int n = __ldg(P.en + e * NPE + b);
    E.ue[b] = n >= 0 ? u[off + static_cast<size_t>(n) * rs] : 0.0;
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

// row a of S_e and g_a by selects (no dynamically indexed local arrays)
template <int NPE>
__device__ __forceinline__ void elem_row(const Elem<NPE>& E, int a, double& ga, double (&Sa)[NPE]) {
  ga = E.g[0];
#pragma unroll
  for (int b = 0; b < NPE; ++b) Sa[b] = E.S[b];
#pragma unroll
  for (int aa = 1; aa < NPE; ++aa)
    if (a == aa) {
      ga = E.g[aa];
#pragma unroll
      for (int b = 0; b < NPE; ++b) Sa[b] = E.S[aa * NPE + b];
    }
}

// Fused residual + Jacobian refill + Jacobi diagonal + PCG init for one row
// and one system: writes A = M/dt + J(u) into the
// fixed CSR pattern, Dinv, r = -R, p = Dinv r.  x keeps the previous Newton
// update (a line-search backtrack still needs it); the first PCG update
// overwrites it.  vo / ao: this lane's vector / matrix-value base offsets.
// A row whose step-matrix values are the same for every system (linear
// problems, and rows touching only constant-nu elements).
__device__ __forceinline__ bool row_shared(const PropParams& P, int i) {
  return P.rowkind == nullptr || __ldg(P.rowkind + i) == 0;
}

__device__ __forceinline__ void refill_finish(const PropParams& P, int i, int sys, size_t vo, int step, bool first,
                                              bool shared_row, double ku, double mr, double dval, double* rdst,
                                              double (&acc)[kNDots]);

template <int NPE>
__device__ __forceinline__ void refill_row(const PropParams& P, const ps_curve* curves, int i, int sys, size_t vo,
                                           size_t ao, int step, bool first, double* rdst, double (&acc)[kNDots]) {
  const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
  const int len = end - base;
  const bool regular = len <= kRegularRow;
  const bool shared_row = row_shared(P, i);
  double jv[kRegularRow];
#pragma unroll
  for (int s = 0; s < kRegularRow; ++s) jv[s] = 0.0;
  if (!regular && !shared_row)
    for (int k = base; k < end; ++k) P.A[ao + static_cast<size_t>(k) * kLanes] = 0.0;
  double ku = 0.0;
  if (shared_row) {
    // J = K on this row (linear problems under newton_step semantics,
    // proj/src/problem.cpp:141-144, or constant-nu elements): K u by CSR; the
    // step-matrix values and Jacobi diagonal come from the shared copy
    const double* Kr = NPE == 0 ? P.Klin : P.Kc;
    for (int k = base; k < end; ++k)
      ku += __ldg(Kr + k) * P.u[vo + static_cast<size_t>(__ldg(P.ci + k)) * kLanes];
  } else if constexpr (NPE > 0) {
    const int q0 = __ldg(P.adj_ptr + i), q1 = __ldg(P.adj_ptr + i + 1);
    for (int q = q0; q < q1; ++q) {
      const int2 ea = __ldg(P.adj + q);
      Elem<NPE> E;
      eval_elem<NPE>(P, curves, ea.x, P.u, vo, kLanes, E);
      double ga, Sa[NPE];
      elem_row<NPE>(E, ea.y, ga, Sa);
      ku += E.nu * ga;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        const int rel = __ldg(P.adj_rel + static_cast<size_t>(q) * NPE + b);
        if (rel < 0) continue;
        const double v = E.nu * Sa[b] + E.cc * (ga * E.g[b]);
        if (regular) {
#pragma unroll
          for (int s = 0; s < kRegularRow; ++s) jv[s] += (rel == s) ? v : 0.0;
        } else {
          P.A[ao + static_cast<size_t>(base + rel) * kLanes] += v;
        }
      }
    }
  }
  // mass term M (u - u_prev)/dt, zero at the first Newton iterate of a step
  double mr = 0.0, dval = 0.0;
  const int dslot = __ldg(P.diag + i);
  for (int k = base; k < end; ++k) {
    const double mk = __ldg(P.M + k);
    if (!first) {
      const size_t jv2 = vo + static_cast<size_t>(__ldg(P.ci + k)) * kLanes;
      mr += mk * ((P.u[jv2] - P.uprev[jv2]) / P.dt);
    }
    if (shared_row) continue;
    double jk;
    if (regular) {
      jk = 0.0;
#pragma unroll
      for (int s = 0; s < kRegularRow; ++s) jk = (k - base == s) ? jv[s] : jk;
    } else {
      jk = P.A[ao + static_cast<size_t>(k) * kLanes];
    }
    const double av = mk / P.dt + jk;
    P.A[ao + static_cast<size_t>(k) * kLanes] = av;
    if (k == dslot) dval = av;
  }
  refill_finish(P, i, sys, vo, step, first, shared_row, ku, mr, dval, rdst, acc);
}

// refill_row for a row of <= kEll slots, driven by its record (pppc_internal.h):
// the row's u and u_prev entries are gathered in one go (the element nodes of
// every element adjacent to row i are columns of row i, so the element loop
// reads them from the warp's shared-memory slot scratch `us` through adj_rel
// instead of chasing element -> node -> u), the padded mass / shared stiffness
// rows come as uniform loads.  Same arithmetic, same order as refill_row.
template <int NPE>
__device__ __forceinline__ void refill_row_ell(const PropParams& P, const ps_curve* curves, const int4* rec, int ri,
                                               int i, int sys, size_t vo, size_t ao, int step, bool first,
                                               double (*us)[32], double* rdst, double (&acc)[kNDots]) {
  const int lane = threadIdx.x & 31;
  const int4 h = rec[kRecInts4 * ri];
  const int4 c03 = rec[kRecInts4 * ri + 1], c47 = rec[kRecInts4 * ri + 2];
  const int base = h.x, len = h.y;
  const bool shared_row = P.rowkind == nullptr || h.z == 0;
  const int c[kEll] = {c03.x, c03.y, c03.z, c03.w, c47.x, c47.y, c47.z, c47.w};
  // the operands of the row's later rounds (shared stiffness row, excitation
  // coefficients and patterns, Jacobi entry, element adjacency) are requested
  // into L1 now, so those rounds hit L1 instead of waiting on L2
  {
    const char* ke = reinterpret_cast<const char*>(P.KE + static_cast<size_t>(i) * kEll);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(ke));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(ke + 32));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms));
    for (int t = 0; t < P.nterms; ++t)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P.pat + static_cast<size_t>(t) * P.d + i));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.Dsh + i));
    if (!shared_row) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P.adj_ptr + i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(P.adj + __ldg(P.adj_ptr + i)));
    }
  }
  // the row's u and u_prev entries and padded mass row are all issued in one
  // round (one memory latency per row instead of three); u then goes to the
  // lane's scratch column
  const double* me = P.ME + static_cast<size_t>(i) * kEll;
  double mr = 0.0;
  {
    double uc[kEll], upc[kEll], mv[kEll];
#pragma unroll
    for (int k = 0; k < kEll; ++k) uc[k] = P.u[vo + static_cast<size_t>(c[k]) * kLanes];
#pragma unroll
    for (int k = 0; k < kEll; ++k) upc[k] = first ? 0.0 : P.uprev[vo + static_cast<size_t>(c[k]) * kLanes];
#pragma unroll
    for (int k = 0; k < kEll; ++k) mv[k] = __ldg(me + k);
#pragma unroll
    for (int k = 0; k < kEll; ++k) us[k][lane] = uc[k];
    // mass term M (u - u_prev)/dt, zero at the first Newton iterate of a step
    if (!first) {
#pragma unroll
      for (int k = 0; k < kEll; ++k)
        if (k < len) mr += mv[k] * ((uc[k] - upc[k]) / P.dt);
    }
  }
  double ku = 0.0;
  if (shared_row) {
    const double* ke = P.KE + static_cast<size_t>(i) * kEll;
#pragma unroll
    for (int k = 0; k < kEll; ++k)
      if (k < len) ku += __ldg(ke + k) * us[k][lane];
    refill_finish(P, i, sys, vo, step, first, true, ku, mr, 0.0, rdst, acc);
    return;
  }
  double jv[kEll];
#pragma unroll
  for (int k = 0; k < kEll; ++k) jv[k] = 0.0;
  if constexpr (NPE > 0) {
    // each lane reads back only its own scratch column: no warp sync (lanes of
    // a warp may be in different actions)
    const int q0 = __ldg(P.adj_ptr + i), q1 = __ldg(P.adj_ptr + i + 1);
    for (int q = q0; q < q1; ++q) {
      const int2 ea = __ldg(P.adj + q);
      const int e = ea.x;
      int rel[NPE];
      Elem<NPE> E;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        rel[b] = __ldg(P.adj_rel + static_cast<size_t>(q) * NPE + b);
        E.ue[b] = rel[b] >= 0 ? us[rel[b]][lane] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < NPE * NPE; ++k) E.S[k] = __ldg(P.eS + static_cast<size_t>(e) * NPE * NPE + k);
      double b2 = 0.0;
#pragma unroll
      for (int a = 0; a < NPE; ++a) {
        double sg = 0.0;
#pragma unroll
        for (int b = 0; b < NPE; ++b) sg += E.S[a * NPE + b] * E.ue[b];
        E.g[a] = sg;
        b2 += E.ue[a] * sg;
      }
      const double inva = __ldg(P.einvA + e);
      b2 *= inva;
      double nup;
      curve_eval(curves[__ldg(P.ecurve + e)], b2, E.nu, nup);
      E.cc = 2.0 * nup * inva;
      double ga, Sa[NPE];
      elem_row<NPE>(E, ea.y, ga, Sa);
      ku += E.nu * ga;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        if (rel[b] < 0) continue;
        const double v = E.nu * Sa[b] + E.cc * (ga * E.g[b]);
#pragma unroll
        for (int sl = 0; sl < kEll; ++sl) jv[sl] += (rel[b] == sl) ? v : 0.0;
      }
    }
  }
  double dval = 0.0;
  const int dslot = __ldg(P.diag + i) - base;
  double* Arow = P.A + ao + static_cast<size_t>(base) * kLanes;
#pragma unroll
  for (int k = 0; k < kEll; ++k) {
    if (k >= len) break;
    const double av = __ldg(me + k) / P.dt + jv[k];
    Arow[k * kLanes] = av;
    if (k == dslot) dval = av;
  }
  refill_finish(P, i, sys, vo, step, first, false, ku, mr, dval, rdst, acc);
}

// Row epilogue of the refill: excitation, residual R = M(u - u_prev)/dt + K(u)u
// - f, Jacobi diagonal, r = -R, p = Dinv r, and the row's dot partials.
__device__ __forceinline__ void refill_finish(const PropParams& P, int i, int sys, size_t vo, int step, bool first,
                                              bool shared_row, double ku, double mr, double dval, double* rdst,
                                              double (&acc)[kNDots]) {
  const size_t iv = vo + static_cast<size_t>(i) * kLanes;
  // excitation f_i = sum_t c_t(t_next) pattern_t[i]  (proj/src/problem.cpp:52-63)
  double f = 0.0;
  const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
  for (int t = 0; t < P.nterms; ++t) f += cf[t] * __ldg(P.pat + static_cast<size_t>(t) * P.d + i);
  const double dinv = shared_row ? __ldg(P.Dsh + i) : 1.0 / dval;
  const double R = mr + ku - f;
  const double r = -R;
  const double z = dinv * r;
  if (!shared_row) P.Dinv[iv] = dinv;
  *rdst = r;
  P.p[iv] = z;
  if (first) P.uprev[iv] = P.u[iv];
  acc[0] += R * R;
  acc[1] += f * f;
  acc[2] += r * z;
  acc[3] += r * r;
}

// Phase-A epilogue for one row: store q, accumulate p.q, q.z, q.Dq (z = D r).
__device__ __forceinline__ void spmv_epilogue(const PropParams& P, int i, size_t vo, double qv, bool sh,
                                              double (&acc)[kNDots]) {
  const size_t iv = vo + static_cast<size_t>(i) * kLanes;
  P.q[iv] = qv;
  const double di = sh ? __ldg(P.Dsh + i) : P.Dinv[iv];
  const double pi = P.p[iv], ri = P.r[iv];
  const double zi = di * ri;
  acc[0] += pi * qv;
  acc[1] += qv * zi;
  acc[2] += qv * (di * qv);
}

// Per-phase base pointers.  opq() hides a kernel-parameter pointer from
// loop-invariant code motion: without it the compiler hoists every base address
// of both PCG phases out of the persistent interval loop and keeps them all in
// registers, which the phase pipelines then lack (spills).
template <class T>
__device__ __forceinline__ T* opq(T* ptr) {
  asm volatile("" : "+l"(ptr));
  return ptr;
}

struct PhasePtrs {
  const double* p;     // this lane's p (vo applied)
  const double* r;
  const double* dinv;
  const double* A;     // this lane's per-system values (ao applied)
  double* q;
  const double* dsh;   // shared Jacobi / padded shared rows / rowkind flag
  const double* ashe;
  double* rs;          // this lane's shared-memory residual column (rows <= kLongRow), or null
  bool kinds;          // rows have kinds (element problems)
};

__device__ __forceinline__ PhasePtrs phase_ptrs(const PropParams& P, size_t vo, size_t ao, double* rs = nullptr) {
  PhasePtrs Q;
  Q.rs = rs;
  Q.p = opq(P.p) + vo;
  Q.r = opq(P.r) + vo;
  Q.dinv = opq(P.Dinv) + vo;
  Q.A = opq(P.A) + ao;
  Q.q = opq(P.q) + vo;
  Q.dsh = opq(P.Dsh);
  Q.ashe = opq(P.AshE);
  Q.kinds = P.rowkind != nullptr;
  return Q;
}

// Phase A, one row: every load of row i is issued from its record (pppc_internal.h
// kEll; staged in shared memory by the persistent kernels) in one go, one row
// ahead of its use: the padded column list drives eight unpredicated gathers
// of p (pad columns point at the row itself and carry a = 0), the values come
// from the padded shared rows (AshE: four uniform 16-byte loads, zero pads) or
// the lane's per-system copy (one coalesced 256-byte segment per slot,
// immediate offsets off one row pointer; slots past the row length read
// nothing and hold 0), plus the row's own p, r and Jacobi entries.
struct RowData {
  int base, len;
  bool shared;
  double a[kEll], pv[kEll];
  double po, ro, dv;
};

__device__ __forceinline__ void issue_row(const PhasePtrs& Q, const int4* rec, int ri, int i, RowData& o) {
  const int4 h = rec[kRecInts4 * ri];
  const int4 c03 = rec[kRecInts4 * ri + 1], c47 = rec[kRecInts4 * ri + 2];
  o.base = h.x;
  o.len = h.y;
  o.shared = !Q.kinds || h.z == 0;
  const int c[kEll] = {c03.x, c03.y, c03.z, c03.w, c47.x, c47.y, c47.z, c47.w};
#pragma unroll
  for (int k = 0; k < kEll; ++k) o.pv[k] = Q.p[static_cast<ptrdiff_t>(c[k]) * kLanes];
  const size_t io = static_cast<size_t>(i) * kLanes;
  o.po = Q.p[io];
  o.ro = (Q.rs != nullptr && o.len <= kLongRow) ? Q.rs[ri * 32] : Q.r[io];
  if (o.shared) {
    o.dv = __ldg(Q.dsh + i);
    const double2* ap = reinterpret_cast<const double2*>(Q.ashe + static_cast<size_t>(i) * kEll);
#pragma unroll
    for (int k = 0; k < kEll / 2; ++k) {
      const double2 v = __ldg(ap + k);
      o.a[2 * k] = v.x;
      o.a[2 * k + 1] = v.y;
    }
  } else {
    o.dv = Q.dinv[io];
    const int n = o.len <= kEll ? o.len : 0;
    const double* ap = Q.A + static_cast<size_t>(o.base) * kLanes;
#pragma unroll
    for (int k = 0; k < kEll; ++k) o.a[k] = k < n ? ap[k * kLanes] : 0.0;
  }
}

// L2 prefetch (no register or scoreboard cost) of the streamed operands of a
// row a few rows ahead of its loads: the loads then see L2 rather than DRAM
// latency, which is what bounds a warp with one row in flight.
__device__ __forceinline__ void pf_l2(const void* ptr) { asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr)); }

__device__ __forceinline__ void prefetch_row_a(const PhasePtrs& Q, const int4* rec, int ri, int i) {
  const size_t io = static_cast<size_t>(i) * kLanes;
  pf_l2(Q.r + io);
  if (!Q.kinds) return;
  const int4 h = rec[kRecInts4 * ri];
  if (h.z == 0) return;
  pf_l2(Q.dinv + io);
  const double* ap = Q.A + static_cast<size_t>(h.x) * kLanes;
  const int n = h.y <= kEll ? h.y : 0;
#pragma unroll
  for (int k = 0; k < kEll; ++k)
    if (k < n) pf_l2(ap + k * kLanes);
}

// Row i of phase A from `cur` (issued one row earlier); issues row i1 (record
// ri1) into `nxt`.
template <bool LINEAR>
__device__ __forceinline__ void spmv_row(const PropParams& P, const PhasePtrs& Q, const int4* rec, int i, int ri1,
                                         int i1, bool more, const RowData& cur, RowData& nxt,
                                         double (&acc)[kNDots]) {
  if (more) issue_row(Q, rec, ri1, i1, nxt);
  double qv = 0.0;
  if (cur.len <= kEll) {
#pragma unroll
    for (int k = 0; k < kEll; ++k) qv += cur.a[k] * cur.pv[k];
  } else if (cur.len <= kLongRow) {
    for (int k = cur.base; k < cur.base + cur.len; ++k) {
      const double av = cur.shared ? __ldg(P.Ash + k) : Q.A[static_cast<size_t>(k) * kLanes];
      qv += av * Q.p[static_cast<ptrdiff_t>(__ldg(P.ci + k)) * kLanes];
    }
  } else {
    return;  // long rows: spmv_long_rows
  }
  Q.q[static_cast<size_t>(i) * kLanes] = qv;
  const double zi = cur.dv * cur.ro;
  acc[0] += cur.po * qv;
  acc[1] += qv * zi;
  acc[2] += qv * (cur.dv * qv);
}

// A warp's rows: row(j) = rb + j * stride (< re), record index ri0 + j * rstep.
struct RowSeq {
  int rb, re, stride, ri0, rstep;
};

// Phase A over a warp's rows: q = A p and the partials p.q, q.z, q.Dq.
// Unrolled by two so the in-flight and the consumed operand sets keep fixed
// registers.
template <bool LINEAR>
__device__ __forceinline__ void spmv_range(const PropParams& P, const int4* rec, const RowSeq& S, size_t vo,
                                           size_t ao, double* rs, double (&acc)[kNDots]) {
  if (S.rb >= S.re) return;
  const PhasePtrs Q = phase_ptrs(P, vo, ao, rs);
  RowData ra, rc;
  issue_row(Q, rec, S.ri0, S.rb, ra);
  int ri = S.ri0;
  const int pfd = P.pf_dist, pfs = pfd * S.stride, pfr = pfd * S.rstep;
  for (int i = S.rb;;) {
    if (pfd > 0 && i + pfs < S.re) prefetch_row_a(Q, rec, ri + pfr, i + pfs);
    int i1 = i + S.stride, ri1 = ri + S.rstep;
    spmv_row<LINEAR>(P, Q, rec, i, ri1, i1, i1 < S.re, ra, rc, acc);
    if (i1 >= S.re) break;
    i = i1, ri = ri1;
    if (pfd > 0 && i + pfs < S.re) prefetch_row_a(Q, rec, ri + pfr, i + pfs);
    i1 = i + S.stride, ri1 = ri + S.rstep;
    spmv_row<LINEAR>(P, Q, rec, i, ri1, i1, i1 < S.re, rc, ra, acc);
    if (i1 >= S.re) break;
    i = i1, ri = ri1;
  }
}

// Row ownership: rows go in chunks of kWarps, chunk k to block
// k mod C of the group, one row of a chunk per warp.  A group's C blocks thus
// sweep every array together through one moving window (DRAM page locality of
// a plain stream), and work per block is balanced to one chunk.  Warp w of
// block c owns rows (c + j C) kWarps + w.  The block's row records are copied
// to shared memory in that order when they fit (P.rec_rows > 0).
__device__ __forceinline__ int first_chunk(const PropParams& P, int c) {
  return (c - P.chunk_rot % P.C + P.C) % P.C;
}

__device__ __forceinline__ RowSeq warp_rows(const PropParams& P, int c, int warp) {
  RowSeq S;
  S.rb = first_chunk(P, c) * kWarps + warp;
  S.re = P.d;
  S.stride = P.C * kWarps;
  if (P.rec_rows > 0) {
    S.ri0 = warp;
    S.rstep = kWarps;
  } else {
    S.ri0 = S.rb;
    S.rstep = S.stride;
  }
  return S;
}

__device__ __forceinline__ const int4* stage_records(const PropParams& P, int c, int4* srec) {
  if (P.rec_rows <= 0) return P.rowrec;
  const int n = P.rec_rows * kRecInts4;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int lr = t / kRecInts4, part = t - lr * kRecInts4;
    const int row = (first_chunk(P, c) + (lr / kWarps) * P.C) * kWarps + (lr % kWarps);
    if (row < P.d) srec[t] = __ldg(P.rowrec + static_cast<size_t>(row) * kRecInts4 + part);
  }
  __syncthreads();
  return srec;
}

// Refill of the long rows this block owns (the polar hub: ntheta+1 slots),
// called by every thread of the block.  For a shared-value row the K u and
// mass sums are split across the 16 warps (4 slots in flight per warp) and
// combined in fixed order; warp 0 finishes the row.  A long row with
// per-system values falls back to the serial element loop on warp 0.
// `active`: this lane refills in this interval.
template <int NPE>
__device__ __forceinline__ void refill_long_rows(const PropParams& P, const ps_curve* curves, bool active,
                                                 bool first, int sys, size_t vo, size_t ao, int step, int c,
                                                 double (*lpart)[32], double (*lpart2)[32],
                                                 double (&acc)[kNDots]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < P.n_long; ++j) {
    if (__ldg(P.long_owner + j) != c) continue;
    const int i = __ldg(P.long_rows + j);
    if (!row_shared(P, i)) {
      if (warp == 0 && active)
        refill_row<NPE>(P, curves, i, sys, vo, ao, step, first, P.r + vo + static_cast<size_t>(i) * kLanes, acc);
      continue;
    }
    const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
    const double* Kr = NPE == 0 ? P.Klin : P.Kc;
    double kp = 0.0, mp = 0.0;
    if (active) {
      for (int k0 = base + warp; k0 < end; k0 += 4 * kWarps) {
        double kv[4], mv[4], uv[4], up[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * kWarps;
          const bool ok = k < end;
          const size_t jv = vo + static_cast<size_t>(ok ? __ldg(P.ci + k) : i) * kLanes;
          kv[u] = ok ? __ldg(Kr + k) : 0.0;
          mv[u] = ok ? __ldg(P.M + k) : 0.0;
          uv[u] = ok ? P.u[jv] : 0.0;
          up[u] = (ok && !first) ? P.uprev[jv] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          kp += kv[u] * uv[u];
          if (!first) mp += mv[u] * ((uv[u] - up[u]) / P.dt);
        }
      }
    }
    lpart[warp][lane] = kp;
    lpart2[warp][lane] = mp;
    __syncthreads();
    if (warp == 0 && active) {
      double ku = 0.0, mr = 0.0;
      for (int w = 0; w < kWarps; ++w) {
        ku += lpart[w][lane];
        mr += lpart2[w][lane];
      }
      refill_finish(P, i, sys, vo, step, first, true, ku, mr, 0.0, P.r + vo + static_cast<size_t>(i) * kLanes, acc);
    }
    __syncthreads();
  }
}

// The single long row (P.hub_split) in phase A: its slots are dealt to the
// group's C blocks (slot s to block s mod C, warp (s / C) mod kWarps), each
// thread adding its slots' A p products into partial slot 3 of the phase-A
// reduction.  The group barrier then sums the row's q in fixed order and the
// transitions finish it, so no block carries the 1 + ntheta slot row alone.
__device__ __forceinline__ void hub_partial(const PropParams& P, size_t vo, size_t ao, int c, int warp,
                                            double (&acc)[kNDots]) {
  const int i = __ldg(P.long_rows);
  const int base = __ldg(P.rp + i), len = __ldg(P.rp + i + 1) - base;
  const bool sh = row_shared(P, i);
  double part = 0.0;
  for (int sidx = c + P.C * warp; sidx < len; sidx += P.C * kWarps) {
    const int k = base + sidx;
    const double av = sh ? __ldg(P.Ash + k) : P.A[ao + static_cast<size_t>(k) * kLanes];
    part += av * P.p[vo + static_cast<size_t>(__ldg(P.ci + k)) * kLanes];
  }
  acc[3] += part;
}

// Long rows (the polar hub: ntheta+1 slots) walked serially by one lane would
// cost ~len dependent load rounds per SpMV and hold every block of the group at
// the next barrier.  The owning block splits the slots across its 16 warps
// (4 slots in flight per warp), combines the warp partials in fixed order and
// runs the row epilogue on warp 0.  All threads of the block execute this.
template <bool LINEAR>
__device__ __forceinline__ void spmv_long_rows(const PropParams& P, bool active, size_t vo, size_t ao, int c,
                                               double (*lpart)[32], double (&acc)[kNDots]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = 0; j < P.n_long; ++j) {
    if (__ldg(P.long_owner + j) != c) continue;
    const int i = __ldg(P.long_rows + j);
    const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
    const bool sh = row_shared(P, i);
    double part = 0.0;
    if (active) {
      for (int k0 = base + warp; k0 < end; k0 += 4 * kWarps) {
        double av[4], pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u * kWarps;
          const int cj = k < end ? __ldg(P.ci + k) : i;
          av[u] = k < end ? (sh ? __ldg(P.Ash + k) : P.A[ao + static_cast<size_t>(k) * kLanes]) : 0.0;
          pv[u] = k < end ? P.p[vo + static_cast<size_t>(cj) * kLanes] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) part += av[u] * pv[u];
      }
    }
    lpart[warp][lane] = part;
    __syncthreads();
    if (warp == 0 && active) {
      double qv = 0.0;
      for (int w = 0; w < kWarps; ++w) qv += lpart[w][lane];
      spmv_epilogue(P, i, vo, qv, sh, acc);
    }
    __syncthreads();
  }
}

// Phase B over a warp's rows: x += alpha p (x = alpha p on the first
// iteration), r -= alpha q, z = D r, p = z + beta p; partials r.r and r.z.
// Rows go in batches of four whose twenty loads are issued together.  (A
// software pipeline one batch ahead halves phase B in the standalone probe but
// spills inside the persistent kernel, where it is slower.)
struct BatchB {
  double dv[4], pv[4], qv[4], rv[4], xv[4];
  bool rsm[4];  // the row's residual lives in shared memory
};

__device__ __forceinline__ void load_batch_b(const PhasePtrs& Q, const int4* rec, const double* x, const RowSeq& S,
                                             int i0, int r0, bool first, BatchB& o) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    // rows past the end re-read row i0 (valid addresses, results unused):
    // unpredicated, branch-free loads keep all twenty in flight together
    const int i = i0 + u * S.stride;
    const bool ok = i < S.re;
    const int ii = ok ? i : i0;
    const int ri = ok ? r0 + u * S.rstep : r0;
    const size_t io = static_cast<size_t>(ii) * kLanes;
    const int4 h = rec[kRecInts4 * ri];
    const bool sh = !Q.kinds || h.z == 0;
    const double* dp = sh ? Q.dsh + ii : Q.dinv + io;
    o.dv[u] = *dp;
    o.pv[u] = Q.p[io];
    o.qv[u] = Q.q[io];
    o.rsm[u] = Q.rs != nullptr && h.y <= kLongRow;
    o.rv[u] = o.rsm[u] ? Q.rs[ri * 32] : Q.r[io];
    o.xv[u] = first ? 0.0 : x[io];
  }
}

__device__ __forceinline__ void store_batch_b(const PhasePtrs& Q, double* x, const RowSeq& S, int i0, int r0,
                                              double alpha, double beta, bool first, const BatchB& o,
                                              double (&acc)[kNDots]) {
  double* pw = const_cast<double*>(Q.p);
  double* rw = const_cast<double*>(Q.r);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + u * S.stride;
    if (i >= S.re) break;
    const size_t io = static_cast<size_t>(i) * kLanes;
    x[io] = first ? alpha * o.pv[u] : o.xv[u] + alpha * o.pv[u];
    const double r = o.rv[u] - alpha * o.qv[u];
    const double z = o.dv[u] * r;
    if (o.rsm[u])
      Q.rs[(r0 + u * S.rstep) * 32] = r;
    else
      rw[io] = r;
    pw[io] = z + beta * o.pv[u];
    acc[0] += r * r;
    acc[1] += r * z;
  }
}

template <bool LINEAR>
__device__ __forceinline__ void update_range(const PropParams& P, const int4* rec, double* x, const RowSeq& S,
                                             size_t vo, double alpha, double beta, bool first, double* rs,
                                             double (&acc)[kNDots]) {
  if (S.rb >= S.re) return;
  const PhasePtrs Q = phase_ptrs(P, vo, 0, rs);
  double* xb = opq(x) + vo;
  const int bstep = 4 * S.stride, rstep = 4 * S.rstep;
  for (int i0 = S.rb, r0 = S.ri0; i0 < S.re; i0 += bstep, r0 += rstep) {
    BatchB ba;
    load_batch_b(Q, rec, xb, S, i0, r0, first, ba);
    store_batch_b(Q, xb, S, i0, r0, alpha, beta, first, ba, acc);
  }
}

// Per-lane actions: one action per group-barrier interval.  ACT_WAIT idles one
// interval so that every lane's PCG phase A falls on an even interval: lanes of
// a warp then run the same PCG phase (no A/B divergence).
enum : int { ACT_IDLE = 0, ACT_R0, ACT_A, ACT_B, ACT_U, ACT_R, ACT_L0, ACT_LU, ACT_WAIT };

template <bool LINEAR, int NPE>
__global__ void __launch_bounds__(kThreads, 1) propagate_kernel(const PropParams P) {
  __shared__ SyncShared<kNDots> sh;
  __shared__ ps_curve sh_curves[kMaxCurves];
  __shared__ double lpart[kWarps][32];
  // Per-lane (= per-system) state lives once per block in shared memory: warp 0
  // runs the transitions after each barrier, every warp reads what its action
  // needs.  (Keeping a copy in every thread's registers would cost ~25 registers
  // the SpMV pipeline needs.)
  __shared__ Lane lanes[32];
  __shared__ int lact[32], lstep[32];
  __shared__ int any_a;  // some lane of the block runs phase A in this interval
  __shared__ int any_r;  // ... or a refill
  __shared__ double lpart2[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // g: launch-local group (barrier domain); gs: storage group (vectors, systems)
  const int g = blockIdx.x / P.C, c = blockIdx.x % P.C;
  const int gs = P.g_base + g;
  const int sl = lane;
  const int sys = gs * P.L + sl;
  const bool valid = (sl < P.L) && (sys < P.count);
  if (threadIdx.x < P.ncurves) sh_curves[threadIdx.x] = P.curves[threadIdx.x];
  sync_state_init(sh);
  if (warp == 0) {
    Lane& s = lanes[lane];
    s.alive = valid;
    s.code = PS_OK;
    s.t_fail = 0.0;
    s.res_fail = 0.0;
    s.tol = 0.0;
    s.nit = 0;
    s.pact = false;
    s.pit = 0;
    s.rho = s.stop = s.alpha = s.beta = 0.0;
    s.res_pre = 0.0;
    s.lambda = 1.0;
    s.ls_k = 0;
    s.bt = s.zero_dx = false;
    s.newton_total = s.pcg_total = 0;
    s.max_nit = s.max_pit = s.last_nit = 0;
    lact[lane] = valid ? (LINEAR ? ACT_L0 : (P.probe_refill ? ACT_R : ACT_R0)) : ACT_IDLE;
    lstep[lane] = 0;
    if (lane == 0) any_a = 0, any_r = !LINEAR;
  }
  __syncthreads();
  // dynamic shared memory: the refill slot scratch (a row's u entries per
  // warp), then the block's row records
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  double(*uscr)[kEll][32] = reinterpret_cast<double(*)[kEll][32]>(dyn_smem);
  int4* srec = reinterpret_cast<int4*>(dyn_smem + kScrSmem);
  stage_records(P, c, srec);
  // the block's residual rows [rec_rows][32] after the records (P.r_smem)
  double* rsm = P.r_smem ? reinterpret_cast<double*>(dyn_smem + kScrSmem +
                                                     static_cast<size_t>(P.rec_rows) * kRecInts4 * sizeof(int4))
                         : nullptr;
  const bool writer = (c == 0) && (warp == 0) && valid;
  double acc[kNDots] = {0.0, 0.0, 0.0, 0.0};
  // Loop-carried state is kept minimal (barrier state and counters in shared
  // memory, addresses recomputed per interval from g, c, warp, lane) so the
  // phase pipelines get the registers.
  __shared__ unsigned long long t_start, t_arr[2];  // debug timing (thread 0): arrival, release seen
  // optional per-block timing (P.dbg): work / barrier-wait ns and counts for
  // intervals where lane 0 ran phase A, phase B, or anything else
  // plus per-action lane-interval counts (dbg[9 + action])
  __shared__ unsigned long long dbg[kDbgSlots];
  if (threadIdx.x < kDbgSlots) dbg[threadIdx.x] = 0;

  // One barrier interval.  Phase A only ever runs on even intervals and B on
  // odd ones (ACT_WAIT alignment), so the loop is unrolled by two with the
  // parity static: each copy contains only one PCG phase, and the register
  // allocator never sees both phase pipelines live in one region.
  bool aborted = false;
  auto interval = [&](auto odd_tag) -> bool {
    constexpr bool ODD = decltype(odd_tag)::value;
    if (!__syncthreads_or(lact[sl] != ACT_IDLE)) return false;
    const int act = lact[sl];
    const int step = lstep[sl];
    if (P.dbg && threadIdx.x == 0) t_start = globaltimer_ns();
    const int dbg_kind = any_r ? 2 : (any_a ? 0 : 1);  // refill in the interval, else phase A, else the rest
    double* xs = LINEAR ? ((step & 1) ? P.ubuf0 : P.ubuf1) : P.x;
    // per-interval addressing from opaque copies of (g, c, warp, lane): the
    // compiler cannot hoist it and keep it live across the whole loop
    int gq = gs, cq = c, wq = warp, lq = sl;
    asm volatile("" : "+r"(gq), "+r"(cq), "+r"(wq), "+r"(lq));
    const size_t vo = static_cast<size_t>(gq) * P.d * kLanes + lq;
    const size_t ao = static_cast<size_t>(gq) * P.nnz * kLanes + lq;
    const RowSeq S = warp_rows(P, cq, wq);
    const int row_begin = S.rb, row_end = S.re, row_step = S.stride;
    const int4* rec = P.rec_rows > 0 ? static_cast<const int4*>(srec) : P.rowrec;
    double* rs = rsm != nullptr ? rsm + lq : nullptr;  // this lane's residual column
    // ------------------------------------------------ this lane's action
    if (P.n_long > 0 && any_a) {
      if (P.hub_split) {
        if (act == ACT_A) hub_partial(P, vo, ao, cq, wq, acc);
      } else {
        spmv_long_rows<LINEAR>(P, act == ACT_A, vo, ao, c, lpart, acc);
      }
    }
    if (!LINEAR)
      if (P.n_long > 0 && any_r)
        refill_long_rows<NPE>(P, sh_curves, act == ACT_R0 || act == ACT_R, act == ACT_R0, sys, vo, ao, step, c,
                              lpart, lpart2, acc);
    if (act == ACT_A) {
      if constexpr (!ODD) spmv_range<LINEAR>(P, rec, S, vo, ao, rs, acc);
    } else if (act == ACT_B) {
      if constexpr (ODD)
        update_range<LINEAR>(P, rec, xs, S, vo, lanes[sl].alpha, lanes[sl].beta, lanes[sl].pit == 0, rs, acc);
    } else if (act == ACT_R0 || act == ACT_R) {
      if (!LINEAR)
        for (int i = row_begin, ri = S.ri0; i < row_end; i += row_step, ri += S.rstep) {
          const int len = rec[kRecInts4 * ri].y;
          double* rdst = rs != nullptr ? rs + ri * 32 : P.r + vo + static_cast<size_t>(i) * kLanes;
          if (len <= kEll)
            refill_row_ell<NPE>(P, sh_curves, rec, ri, i, sys, vo, ao, step, act == ACT_R0, uscr[wq], rdst, acc);
          else if (len <= kLongRow)
            refill_row<NPE>(P, sh_curves, i, sys, vo, ao, step, act == ACT_R0, rdst, acc);
          // longer rows: refill_long_rows
        }
    } else if (act == ACT_U) {
      if (!lanes[sl].zero_dx) {
        const bool bt = lanes[sl].bt;
        const double lambda = lanes[sl].lambda;
        for (int i = row_begin; i < row_end; i += row_step) {
          // trial u += lambda delta (propagators.cpp:46-48), or a backtrack
          // u -= lambda delta with lambda already halved; delta must be finite
          const size_t iv = vo + static_cast<size_t>(i) * kLanes;
          const double dx = P.x[iv];
          if (bt) {
            P.u[iv] -= lambda * dx;
          } else {
            acc[0] += isfinite(dx) ? 0.0 : 1.0;
            P.u[iv] += lambda * dx;
          }
        }
      }
    } else if (act == ACT_L0) {
      // b = M (u/dt) + f, x = 0, r = b, p = D b (proj/src/propagators.cpp:85-94)
      const double* uin = (step & 1) ? P.ubuf1 : P.ubuf0;
      const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
      for (int i = row_begin, ri = S.ri0; i < row_end; i += row_step, ri += S.rstep) {
        const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
        double mv = 0.0;
        for (int k = base; k < end; ++k)
          mv += __ldg(P.M + k) * (uin[vo + static_cast<size_t>(__ldg(P.ci + k)) * kLanes] / P.dt);
        double f = 0.0;
        for (int t = 0; t < P.nterms; ++t) f += cf[t] * __ldg(P.pat + static_cast<size_t>(t) * P.d + i);
        const double b = mv + f;
        const size_t iv = vo + static_cast<size_t>(i) * kLanes;
        const double z = __ldg(P.Dsh + i) * b;
        xs[iv] = 0.0;
        if (rs != nullptr && end - base <= kLongRow)
          rs[ri * 32] = b;
        else
          P.r[iv] = b;
        P.p[iv] = z;
        acc[0] += b * z;
        acc[1] += b * b;
      }
    } else if (act == ACT_LU) {
      // the step solution must be finite (propagators.cpp:92); x0 = 0 when b = 0
      const bool zero = lanes[sl].pit == 0;
      for (int i = row_begin; i < row_end; i += row_step) {
        const size_t iv = vo + static_cast<size_t>(i) * kLanes;
        if (zero) xs[iv] = 0.0;
        acc[0] += isfinite(xs[iv]) ? 0.0 : 1.0;
      }
    }
    // hub row operands for the phase-A transition, loaded before the barrier so
    // their latency overlaps it
    double hub_p = 0.0, hub_r = 0.0, hub_d = 0.0;
    if (warp == 0 && act == ACT_A && P.hub_split) {
      const int hub = __ldg(P.long_rows);
      const size_t ih = static_cast<size_t>(gs) * P.d * kLanes + sl + static_cast<size_t>(hub) * kLanes;
      hub_p = P.p[ih];
      hub_r = P.r[ih];
      hub_d = row_shared(P, hub) ? __ldg(P.Dsh + hub) : P.Dinv[ih];
    }
    {
      const SyncCtx X{P.sync, P.partials, P.abort_flag, P.G, P.C, 32, P.L};
      if (!group_sync_reduce<kNDots, 4>(X, sh, acc, g, c, P.dbg ? t_arr : nullptr)) {
        aborted = true;
        return false;
      }
    }
    if (P.dbg && warp == 0 && valid) atomicAdd(&dbg[9 + act], 1ull);
    if (P.dbg && threadIdx.x == 0) {
      const unsigned long long t_end = globaltimer_ns();
      dbg[3 * dbg_kind + 0] += t_arr[0] - t_start;
      dbg[3 * dbg_kind + 1] += t_end - t_arr[0];
      dbg[3 * dbg_kind + 2] += 1;
      dbg[18 + dbg_kind] += t_arr[1] - t_arr[0];
    }
    // ------------------------------------------------ transitions (warp 0)
    if (warp == 0) {
      Lane& s = lanes[lane];
      int a = act;
      int stp = step;
      // the step's time is only needed to report a failure: read it then, not on
      // every interval's critical path
      auto t_now_of = [&]() { return P.t_next[static_cast<size_t>(stp) * P.count + sys]; };
      double t0v = sh.tot[0][sl], t1v = sh.tot[1][sl], t2v = sh.tot[2][sl];
      const double t3v = sh.tot[3][sl];
      if (a == ACT_A && P.hub_split) {
        // the single long row's q came through the reduction (slot 3): add its
        // terms to p.q, q.z, q.Dq here, identically in every block; the owner
        // stores it for phase B
        const int hub = __ldg(P.long_rows);
        const size_t ih = static_cast<size_t>(gs) * P.d * kLanes + sl + static_cast<size_t>(hub) * kLanes;
        const double qh = t3v, ph = hub_p, rh = hub_r;
        const double dh = hub_d;
        t0v += ph * qh;
        t1v += qh * (dh * rh);
        t2v += qh * (dh * qh);
        if (c == __ldg(P.long_owner)) P.q[ih] = qh;
      }
      if (P.probe_refill) a = ACT_IDLE;  // the refill probe stops after its one refill
      switch (P.probe_refill ? ACT_IDLE : a) {
        case ACT_R0: {
          s.tol = P.newton_tol_abs + P.newton_tol_rel * sqrt(t1v);
          s.nit = 1;
          s.res_pre = sqrt(t0v);
          pcg_start(s, t2v, t3v, P.pcg_tol);
          s.bt = false;
          s.zero_dx = !s.pact;
          s.lambda = P.damping;
          s.ls_k = 0;
          a = s.pact ? ACT_A : ACT_U;
          break;
        }
        case ACT_A: {
          if (!isfinite(t0v) || t0v == 0.0) {
            lane_fail(s, PS_ERR_SINGULAR, LINEAR ? 0.0 : s.res_pre, t_now_of());
          } else {
            s.alpha = s.rho / t0v;
            const double rho_est = s.rho - 2.0 * s.alpha * t1v + s.alpha * s.alpha * t2v;
            s.beta = rho_est / s.rho;
            a = ACT_B;
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
            a = LINEAR ? ACT_LU : ACT_U;
          } else if (!isfinite(rr)) {
            lane_fail(s, PS_ERR_SINGULAR, LINEAR ? 0.0 : s.res_pre, t_now_of());
          } else if (s.pit >= P.pcg_max) {
            lane_fail(s, PS_ERR_PCG_MAXITER, LINEAR ? 0.0 : s.res_pre, t_now_of());
          } else {
            a = ACT_A;
          }
          break;
        }
        case ACT_U: {
          if (!s.bt && t0v > 0.0)
            lane_fail(s, PS_ERR_SINGULAR, s.res_pre, t_now_of());
          else
            a = ACT_R;
          break;
        }
        case ACT_R: {
          const double post = sqrt(t0v);
          if (P.line_search > 0 && s.ls_k < P.line_search && !(post <= s.tol) &&
              !(post <= (1.0 - 1e-4 * s.lambda) * s.res_pre)) {
            s.lambda *= 0.5;
            s.ls_k += 1;
            s.bt = true;
            a = ACT_U;
            break;
          }
          s.bt = false;
          if (writer && P.trace) P.trace[static_cast<size_t>(sys) * P.newton_max + (s.nit - 1)] = post;
          if (!isfinite(post)) {
            lane_fail(s, PS_ERR_NEWTON_DIVERGED, post, t_now_of());
          } else if (post <= s.tol) {
            s.newton_total += s.nit;
            s.last_nit = s.nit;
            s.max_nit = max(s.max_nit, s.nit);
            ++stp;
            a = stp < P.steps ? ACT_R0 : ACT_IDLE;
          } else if (s.nit >= P.newton_max) {
            lane_fail(s, PS_ERR_NEWTON_MAXITER, post, t_now_of());
          } else {
            s.nit += 1;
            s.res_pre = post;
            pcg_start(s, t2v, t3v, P.pcg_tol);
            s.zero_dx = !s.pact;
            s.lambda = P.damping;
            s.ls_k = 0;
            a = s.pact ? ACT_A : ACT_U;
          }
          break;
        }
        case ACT_L0: {
          pcg_start(s, t0v, t1v, P.pcg_tol);
          a = s.pact ? ACT_A : ACT_LU;
          break;
        }
        case ACT_LU: {
          if (t0v > 0.0) {
            lane_fail(s, PS_ERR_SINGULAR, 0.0, t_now_of());
          } else {
            s.newton_total += 1;
            s.last_nit = 1;
            s.max_nit = max(s.max_nit, 1);
            ++stp;
            a = stp < P.steps ? ACT_L0 : ACT_IDLE;
          }
          break;
        }
        case ACT_WAIT:
          a = ACT_A;
          break;
        default:
          break;
      }
      if (!s.alive) a = ACT_IDLE;
      if (a == ACT_A && (sh.bar_idx & 1)) a = ACT_WAIT;  // phase A only on even intervals
      lact[lane] = a;
      lstep[lane] = stp;
      const unsigned am = __ballot_sync(0xffffffffu, a == ACT_A);
      const unsigned rm = __ballot_sync(0xffffffffu, a == ACT_R0 || a == ACT_R);
      if (lane == 0) any_a = am != 0u, any_r = rm != 0u;
    }
    __syncthreads();
    return true;
  };
  using EvenTag = std::integral_constant<bool, false>;
  using OddTag = std::integral_constant<bool, true>;
  for (;;) {
    if (!interval(EvenTag())) break;
    if (!interval(OddTag())) break;
  }
  if (aborted) return;

  if (writer) {
    const Lane& s = lanes[lane];
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
  if (c == 0 && threadIdx.x == 0) P.lockstep[gs] = sh.bar_idx;
  __syncthreads();
  if (P.dbg && threadIdx.x == 0)
    for (int k = 0; k < kDbgSlots; ++k) P.dbg[static_cast<size_t>(blockIdx.x) * kDbgSlots + k] = dbg[k];
}

// ------------------------------------------------- system-per-block engine
// One thread block runs one system's whole batch of implicit-Euler steps
// (proj/src/propagators.cpp:96-115): the refill, the Newton control
// (:27-58, with the same backtracking extension as propagate_kernel) and every
// Jacobi-PCG iteration, synchronising with block barriers only.  Vectors are
// contiguous per system and thread t owns rows t, t + NT, ..., so every
// operand of a row (the padded ELL column list, the shared or per-system slot
// values, the gathered p entries of neighbouring rows) is a coalesced load
// across a warp.  Same arithmetic and control flow as propagate_kernel's lane
// state machine; block reductions run in a fixed order, so a system's result
// does not depend on the batch it is in.

// Fixed-order block sum of ND values: shuffle-down tree per warp, then the
// warp partials in warp order.  Every thread returns the same totals.
template <int ND, int NT>
__device__ __forceinline__ void sb_reduce(double (&v)[ND], double (*red)[NT / 32], double* tot) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) red[k][warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < ND) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[threadIdx.x][w];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ND; ++k) v[k] = tot[k];
}

struct SbVec {
  double *u, *uprev, *x, *r, *p, *q, *D, *A, *hA;
};

__device__ __forceinline__ bool sb_shared_row(const PropParams& P, int i) {
  return P.rowkind == nullptr || __ldg(P.rowkind + i) == 0;
}

// Refill of one row of <= kEll slots (refill_row_ell's arithmetic, contiguous
// layout): excitation, residual R = M(u - u_prev)/dt + K(u)u - f, the step
// matrix values M/dt + J(u) (per-system rows), Jacobi, r = -R, p = Dinv r;
// partials {R.R, f.f, r.z, r.r}.
template <int NPE>
__device__ __forceinline__ void sb_refill_row(const PropParams& P, const SysParams& S, const ps_curve* curves,
                                              const SbVec& V, int sys, int step, bool first, int i,
                                              double (&acc)[4]) {
  const int d = P.d;
  const int base = __ldg(P.rp + i), len = __ldg(P.rp + i + 1) - base;
  const bool shared_row = sb_shared_row(P, i);
  int c[kEll];
  double uc[kEll], upc[kEll], mv[kEll];
#pragma unroll
  for (int k = 0; k < kEll; ++k) c[k] = __ldg(S.ciT + static_cast<size_t>(k) * d + i);
#pragma unroll
  for (int k = 0; k < kEll; ++k) uc[k] = V.u[c[k]];
#pragma unroll
  for (int k = 0; k < kEll; ++k) upc[k] = first ? 0.0 : V.uprev[c[k]];
#pragma unroll
  for (int k = 0; k < kEll; ++k) mv[k] = __ldg(S.MT + static_cast<size_t>(k) * d + i);
  double mr = 0.0;
  if (!first) {
#pragma unroll
    for (int k = 0; k < kEll; ++k)
      if (k < len) mr += mv[k] * ((uc[k] - upc[k]) / P.dt);
  }
  double ku = 0.0, dinv;
  if (shared_row) {
#pragma unroll
    for (int k = 0; k < kEll; ++k)
      if (k < len) ku += __ldg(S.KT + static_cast<size_t>(k) * d + i) * uc[k];
    dinv = __ldg(P.Dsh + i);
  } else {
    double jv[kEll];
#pragma unroll
    for (int k = 0; k < kEll; ++k) jv[k] = 0.0;
    const int q0 = __ldg(P.adj_ptr + i), q1 = __ldg(P.adj_ptr + i + 1);
    for (int q = q0; q < q1; ++q) {
      const int2 ea = __ldg(P.adj + q);
      const int e = ea.x;
      int rel[NPE];
      Elem<NPE> E;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        rel[b] = __ldg(P.adj_rel + static_cast<size_t>(q) * NPE + b);
        double ub = 0.0;
#pragma unroll
        for (int s = 0; s < kEll; ++s) ub = (rel[b] == s) ? uc[s] : ub;
        E.ue[b] = ub;
      }
#pragma unroll
      for (int k = 0; k < NPE * NPE; ++k) E.S[k] = __ldg(P.eS + static_cast<size_t>(e) * NPE * NPE + k);
      double b2 = 0.0;
#pragma unroll
      for (int a = 0; a < NPE; ++a) {
        double sg = 0.0;
#pragma unroll
        for (int b = 0; b < NPE; ++b) sg += E.S[a * NPE + b] * E.ue[b];
        E.g[a] = sg;
        b2 += E.ue[a] * sg;
      }
      const double inva = __ldg(P.einvA + e);
      b2 *= inva;
      double nup;
      curve_eval(curves[__ldg(P.ecurve + e)], b2, E.nu, nup);
      E.cc = 2.0 * nup * inva;
      double ga, Sa[NPE];
      elem_row<NPE>(E, ea.y, ga, Sa);
      ku += E.nu * ga;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        if (rel[b] < 0) continue;
        const double v = E.nu * Sa[b] + E.cc * (ga * E.g[b]);
#pragma unroll
        for (int sl = 0; sl < kEll; ++sl) jv[sl] += (rel[b] == sl) ? v : 0.0;
      }
    }
    double dval = 0.0;
    const int dslot = __ldg(P.diag + i) - base;
#pragma unroll
    for (int k = 0; k < kEll; ++k) {
      // pad slots hold 0 (the SpMV reads all kEll slots of a row)
      const double av = k < len ? mv[k] / P.dt + jv[k] : 0.0;
      V.A[static_cast<size_t>(k) * d + i] = av;
      if (k == dslot) dval = av;
    }
    dinv = 1.0 / dval;
    V.D[i] = dinv;
  }
  double f = 0.0;
  const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
  for (int t = 0; t < P.nterms; ++t) f += __ldg(cf + t) * __ldg(P.pat + static_cast<size_t>(t) * d + i);
  const double R = mr + ku - f;
  const double r = -R;
  const double z = dinv * r;
  V.r[i] = r;
  V.p[i] = z;
  if (first) V.uprev[i] = V.u[i];
  acc[0] += R * R;
  acc[1] += f * f;
  acc[2] += r * z;
  acc[3] += r * r;
}

// The hub row (more than kEll slots), serially by one thread: refill_row's
// arithmetic on the CSR slots.
template <int NPE>
__device__ void sb_refill_hub(const PropParams& P, const SysParams& S, const ps_curve* curves, const SbVec& V,
                              int sys, int step, bool first, double (&acc)[4]) {
  const int i = S.hub, d = P.d;
  const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
  const bool shared_row = sb_shared_row(P, i);
  double ku = 0.0;
  if (shared_row) {
    for (int k = base; k < end; ++k) ku += __ldg(P.Kc + k) * V.u[__ldg(P.ci + k)];
  } else {
    for (int k = 0; k < end - base; ++k) V.hA[k] = 0.0;
    const int q0 = __ldg(P.adj_ptr + i), q1 = __ldg(P.adj_ptr + i + 1);
    for (int q = q0; q < q1; ++q) {
      const int2 ea = __ldg(P.adj + q);
      Elem<NPE> E;
      eval_elem<NPE>(P, curves, ea.x, V.u, 0, 1, E);
      double ga, Sa[NPE];
      elem_row<NPE>(E, ea.y, ga, Sa);
      ku += E.nu * ga;
#pragma unroll
      for (int b = 0; b < NPE; ++b) {
        const int rel = __ldg(P.adj_rel + static_cast<size_t>(q) * NPE + b);
        if (rel < 0) continue;
        V.hA[rel] += E.nu * Sa[b] + E.cc * (ga * E.g[b]);
      }
    }
  }
  double mr = 0.0, dval = 0.0;
  const int dslot = __ldg(P.diag + i);
  for (int k = base; k < end; ++k) {
    const double mk = __ldg(P.M + k);
    if (!first) {
      const int j = __ldg(P.ci + k);
      mr += mk * ((V.u[j] - V.uprev[j]) / P.dt);
    }
    if (shared_row) continue;
    const double av = mk / P.dt + V.hA[k - base];
    V.hA[k - base] = av;
    if (k == dslot) dval = av;
  }
  double f = 0.0;
  const double* cf = P.coef + (static_cast<size_t>(step) * P.count + sys) * P.nterms;
  for (int t = 0; t < P.nterms; ++t) f += __ldg(cf + t) * __ldg(P.pat + static_cast<size_t>(t) * d + i);
  const double dinv = shared_row ? __ldg(P.Dsh + i) : 1.0 / dval;
  const double R = mr + ku - f;
  const double r = -R;
  const double z = dinv * r;
  if (!shared_row) V.D[i] = dinv;
  V.r[i] = r;
  V.p[i] = z;
  if (first) V.uprev[i] = V.u[i];
  acc[0] += R * R;
  acc[1] += f * f;
  acc[2] += r * z;
  acc[3] += r * r;
}

template <int NPE, int NT>
__device__ __forceinline__ void sb_refill(const PropParams& P, const SysParams& S, const ps_curve* curves,
                                          const SbVec& V, int sys, int step, bool first, double (*red)[NT / 32],
                                          double* tot, double (&t)[4]) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < P.d; i += NT)
    if (i != S.hub) sb_refill_row<NPE>(P, S, curves, V, sys, step, first, i, acc);
  // the hub row serially on the last thread (it owns the fewest rows)
  if (S.hub >= 0 && threadIdx.x == NT - 1) sb_refill_hub<NPE>(P, S, curves, V, sys, step, first, acc);
  sb_reduce<4, NT>(acc, red, tot);
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = acc[k];
}

// Phase A over this thread's rows, two rows per round with all their loads
// issued before the first FMA: q = A p and the partials p.q, q.z, q.Dq.  The
// hub row is skipped (its product goes through the reduction).
template <int NT>
__device__ __forceinline__ void sb_spmv_rows(const PropParams& P, const SysParams& S, const SbVec& V,
                                             double (&acc)[4]) {
  const int d = P.d;
  for (int i0 = threadIdx.x; i0 < d; i0 += 2 * NT) {
    int row[2] = {i0, i0 + NT};
    bool ok[2] = {i0 != S.hub, i0 + NT < d && i0 + NT != S.hub};
    double av[2][kEll], pv[2][kEll], po[2], ro[2], dv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = ok[u] ? row[u] : i0;  // a skipped row re-reads row i0 (results unused)
      // shared and per-system operands are both requested and then selected by
      // the row kind, so no load waits on the kind
      const bool sh = sb_shared_row(P, i);
      double as[kEll], ap[kEll];
#pragma unroll
      for (int k = 0; k < kEll; ++k) {
        const size_t t = static_cast<size_t>(k) * d + i;
        as[k] = __ldg(S.AshT + t);
        ap[k] = V.A[t];
        pv[u][k] = V.p[__ldg(S.ciT + t)];
      }
#pragma unroll
      for (int k = 0; k < kEll; ++k) av[u][k] = sh ? as[k] : ap[k];
      po[u] = V.p[i];
      ro[u] = V.r[i];
      const double ds = __ldg(P.Dsh + i), dp = V.D[i];
      dv[u] = sh ? ds : dp;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      double qv = 0.0;
#pragma unroll
      for (int k = 0; k < kEll; ++k) qv += av[u][k] * pv[u][k];
      V.q[row[u]] = qv;
      const double zi = dv[u] * ro[u];
      acc[0] += po[u] * qv;
      acc[1] += qv * zi;
      acc[2] += qv * (dv[u] * qv);
    }
  }
}

// Phase B over this thread's rows, two rows per round: x (+)= alpha p,
// r -= alpha q, z = D r, p = z + beta p; partials r.r, r.z.
template <int NT>
__device__ __forceinline__ void sb_update_rows(const PropParams& P, const SbVec& V, double alpha, double beta,
                                               bool first, double (&acc)[2]) {
  const int d = P.d;
  for (int i0 = threadIdx.x; i0 < d; i0 += 2 * NT) {
    const int i1 = i0 + NT < d ? i0 + NT : i0;
    const int row[2] = {i0, i1};
    double dv[2], pv[2], xv[2], rv[2], qv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = row[u];
      const double ds = __ldg(P.Dsh + i), dp = V.D[i];
      dv[u] = sb_shared_row(P, i) ? ds : dp;
      pv[u] = V.p[i];
      xv[u] = first ? 0.0 : V.x[i];
      rv[u] = V.r[i];
      qv[u] = V.q[i];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && i0 + NT >= d) break;
      const int i = row[u];
      V.x[i] = first ? alpha * pv[u] : xv[u] + alpha * pv[u];
      const double rn = rv[u] - alpha * qv[u];
      const double z = dv[u] * rn;
      V.r[i] = rn;
      V.p[i] = z + beta * pv[u];
      acc[0] += rn * rn;
      acc[1] += rn * z;
    }
  }
}

template <int NPE, int NT>
__global__ void __launch_bounds__(NT, 1) sysblock_kernel(const PropParams P, const SysParams S) {
  __shared__ double red[4][NT / 32];
  __shared__ double tot[4];
  __shared__ ps_curve curves[kMaxCurves];
  const int sys = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid < P.ncurves) curves[tid] = P.curves[tid];
  const int d = P.d;
  const size_t vb = static_cast<size_t>(sys) * d;
  SbVec V;
  if (S.smem_vectors) {
    // small systems: the seven per-row vectors live in shared memory
    extern __shared__ __align__(16) double sv[];
    V.u = sv;
    V.uprev = sv + d;
    V.x = sv + 2 * static_cast<size_t>(d);
    V.r = sv + 3 * static_cast<size_t>(d);
    V.p = sv + 4 * static_cast<size_t>(d);
    V.q = sv + 5 * static_cast<size_t>(d);
    V.D = sv + 6 * static_cast<size_t>(d);
  } else {
    V.u = S.su + vb;
    V.uprev = P.uprev + vb;
    V.x = P.x + vb;
    V.r = P.r + vb;
    V.p = P.p + vb;
    V.q = P.q + vb;
    V.D = P.Dinv + vb;
  }
  V.A = S.sA + static_cast<size_t>(sys) * kEll * d;
  V.hA = S.hub >= 0 ? S.hubA + static_cast<size_t>(sys) * S.hub_len : nullptr;
  // start state from the group-blocked layout [G][d][32] (the callers' staging)
  const int g = sys / P.L, l = sys - g * P.L;
  double* ub = P.u + static_cast<size_t>(g) * d * kLanes + l;
  for (int i = tid; i < d; i += NT) V.u[i] = ub[static_cast<size_t>(i) * kLanes];
  __syncthreads();

  const bool hub_shared = S.hub >= 0 && sb_shared_row(P, S.hub);
  const int hub_base = S.hub >= 0 ? __ldg(P.rp + S.hub) : 0;
  int code = PS_OK, last_nit = 0, max_nit = 0, max_pit = 0;
  double t_fail = 0.0, res_fail = 0.0;
  long long newton_total = 0, pcg_total = 0;
  double t[4];
  for (int step = 0; step < P.steps && code == PS_OK; ++step) {
    const double t_now = P.t_next[static_cast<size_t>(step) * P.count + sys];
    sb_refill<NPE, NT>(P, S, curves, V, sys, step, true, red, tot, t);
    const double tol = P.newton_tol_abs + P.newton_tol_rel * sqrt(t[1]);
    int nit = 1;
    double res_pre = sqrt(t[0]);
    double rho = t[2], bb = t[3];
    for (;;) {
      // ---- step solve (J delta = -R): Jacobi-PCG from delta = 0
      const bool pact = bb != 0.0;
      if (pact) {
        const double stop = (P.pcg_tol * P.pcg_tol) * bb;
        int pit = 0;
        for (;;) {
          double a4[4] = {0.0, 0.0, 0.0, 0.0};
          sb_spmv_rows<NT>(P, S, V, a4);
          if (S.hub >= 0) {
            double part = 0.0;
            for (int s = tid; s < S.hub_len; s += NT) {
              const int k = hub_base + s;
              const double av = hub_shared ? __ldg(P.Ash + k) : V.hA[s];
              part += av * V.p[__ldg(P.ci + k)];
            }
            a4[3] = part;
          }
          sb_reduce<4, NT>(a4, red, tot);
          double t0v = a4[0], t1v = a4[1], t2v = a4[2];
          if (S.hub >= 0) {
            // the hub's q came through the reduction: its terms are added to the
            // dots here (uniformly), its owner stores it for the update
            const double qh = a4[3], ph = V.p[S.hub], rh = V.r[S.hub];
            const double dh = hub_shared ? __ldg(P.Dsh + S.hub) : V.D[S.hub];
            t0v += ph * qh;
            t1v += qh * (dh * rh);
            t2v += qh * (dh * qh);
            if (tid == S.hub % NT) V.q[S.hub] = qh;
          }
          if (!isfinite(t0v) || t0v == 0.0) {
            code = PS_ERR_SINGULAR;
            res_fail = res_pre;
            t_fail = t_now;
            break;
          }
          const double alpha = rho / t0v;
          const double rho_est = rho - 2.0 * alpha * t1v + alpha * alpha * t2v;
          const double beta = rho_est / rho;
          double b2[2] = {0.0, 0.0};
          sb_update_rows<NT>(P, V, alpha, beta, pit == 0, b2);
          sb_reduce<2, NT>(b2, red, tot);
          const double rr = b2[0];
          rho = b2[1];
          pit += 1;
          if (rr <= stop) break;
          if (!isfinite(rr)) {
            code = PS_ERR_SINGULAR;
            res_fail = res_pre;
            t_fail = t_now;
            break;
          }
          if (pit >= P.pcg_max) {
            code = PS_ERR_PCG_MAXITER;
            res_fail = res_pre;
            t_fail = t_now;
            break;
          }
        }
        if (code != PS_OK) break;
        pcg_total += pit;
        max_pit = max(max_pit, pit);
      }
      // ---- trial update u += lambda delta (propagators.cpp:46-48), delta finite
      double lambda = P.damping;
      int ls_k = 0;
      if (pact) {
        double bad[1] = {0.0};
        for (int i = tid; i < d; i += NT) {
          const double dx = V.x[i];
          bad[0] += isfinite(dx) ? 0.0 : 1.0;
          V.u[i] += lambda * dx;
        }
        sb_reduce<1, NT>(bad, red, tot);
        if (bad[0] > 0.0) {
          code = PS_ERR_SINGULAR;
          res_fail = res_pre;
          t_fail = t_now;
          break;
        }
      } else {
        __syncthreads();
      }
      // ---- residual at the trial point; optional backtracking
      double post;
      for (;;) {
        sb_refill<NPE, NT>(P, S, curves, V, sys, step, false, red, tot, t);
        post = sqrt(t[0]);
        if (P.line_search > 0 && ls_k < P.line_search && !(post <= tol) &&
            !(post <= (1.0 - 1e-4 * lambda) * res_pre)) {
          lambda *= 0.5;
          ls_k += 1;
          if (pact)
            for (int i = tid; i < d; i += NT) V.u[i] -= lambda * V.x[i];
          __syncthreads();
          continue;
        }
        break;
      }
      if (tid == 0 && P.trace) P.trace[static_cast<size_t>(sys) * P.newton_max + (nit - 1)] = post;
      if (!isfinite(post)) {
        code = PS_ERR_NEWTON_DIVERGED;
        res_fail = post;
        t_fail = t_now;
        break;
      }
      if (post <= tol) {
        newton_total += nit;
        last_nit = nit;
        max_nit = max(max_nit, nit);
        break;
      }
      if (nit >= P.newton_max) {
        code = PS_ERR_NEWTON_MAXITER;
        res_fail = post;
        t_fail = t_now;
        break;
      }
      nit += 1;
      res_pre = post;
      rho = t[2];
      bb = t[3];
    }
  }
  // result back to the group-blocked layout
  for (int i = tid; i < d; i += NT) ub[static_cast<size_t>(i) * kLanes] = V.u[i];
  if (tid == 0) {
    SysOut o;
    o.code = code;
    o.newton_last = last_nit;
    o.t_fail = t_fail;
    o.residual = res_fail;
    o.newton_total = newton_total;
    o.pcg_total = pcg_total;
    o.max_newton = max_nit;
    o.max_pcg = max_pit;
    P.out[sys] = o;
    atomicMax(reinterpret_cast<unsigned long long*>(P.lockstep + g), static_cast<unsigned long long>(pcg_total));
  }
}

#include "cluster_engine.cuh"

// ------------------------------------------------------- phase probes
// One PCG phase over the whole batch with the propagation kernel's exact thread
// -> (group, row, lane) mapping and code, but no barriers or state machine:
// a normal (non-cooperative) kernel that ncu can replay and that isolates the
// memory behaviour of one phase.  mode 1: phase A (SpMV + dots), 2: phase B
// (update), 3: phase B's streams as a flat grid-stride copy (the streaming
// reference).  Dots go to `sink`.
__global__ void __launch_bounds__(kThreads, 1) phase_probe_kernel(const PropParams P, int mode, double* sink) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x / P.C, c = blockIdx.x % P.C;
  const size_t vo = static_cast<size_t>(g) * P.d * kLanes + lane;
  const size_t ao = static_cast<size_t>(g) * P.nnz * kLanes + lane;
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  const int4* rec = stage_records(P, c, reinterpret_cast<int4*>(dyn_smem + kScrSmem));
  const RowSeq S = warp_rows(P, c, warp);
  double acc[kNDots] = {0.0, 0.0, 0.0, 0.0};
  if (mode == 1)
    spmv_range<false>(P, rec, S, vo, ao, nullptr, acc);
  else if (mode == 2)
    update_range<false>(P, rec, P.x, S, vo, 1e-30, 1e-30, false, nullptr, acc);
  else {
    // mode 3: the phase-B streams (5 reads, 3 writes) as a flat grid-stride
    // loop over the whole padded batch: the streaming reference for mode 2
    const size_t n = static_cast<size_t>(P.G) * P.d * kLanes;
    const size_t nt = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t e0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; e0 < n; e0 += 4 * nt) {
      double dv[4], pv[4], qv[4], rv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t e = e0 + u * nt < n ? e0 + u * nt : e0;
        dv[u] = P.Dinv[e], pv[u] = P.p[e], qv[u] = P.q[e], rv[u] = P.r[e], xv[u] = P.x[e];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t e = e0 + u * nt;
        if (e >= n) break;
        const double r = rv[u] - 1e-30 * qv[u];
        const double z = dv[u] * r;
        P.x[e] = xv[u] + 1e-30 * pv[u];
        P.r[e] = r;
        P.p[e] = z + 1e-30 * pv[u];
        acc[0] += r * r;
        acc[1] += r * z;
      }
    }
  }
  if (acc[0] == 12345.0) sink[blockIdx.x] = acc[1] + acc[2];  // keep the dots live
}

// ------------------------------------------------------------ small kernels
__global__ void transpose_kernel(const double* __restrict__ src, double* __restrict__ dst, int rows, int cols,
                                 int ld_src, int ld_dst) {
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

// interleaved [d][stride] <-> group-blocked [G][d][32] (L lanes used per group)
__global__ void il_blocked_kernel(const double* __restrict__ src, double* __restrict__ dst, int d, int count,
                                  int stride, int L, int to_blocked) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(d) * count) return;
  const int sys = static_cast<int>(t % count), i = static_cast<int>(t / count);
  const int g = sys / L, l = sys % L;
  const size_t b = (static_cast<size_t>(g) * d + i) * kLanes + l;
  const size_t il = static_cast<size_t>(i) * stride + sys;
  if (to_blocked)
    dst[b] = src[il];
  else
    dst[il] = src[b];
}

template <int NPE>
__global__ void assemble_ops_kernel(const PropParams P, int count, const double* __restrict__ u_il, double* K_out,
                                    double* J_out) {
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
    eval_elem<NPE>(P, P.curves, ea.x, u_il, static_cast<size_t>(sys), static_cast<size_t>(count), E);
    double ga, Sa[NPE];
    elem_row<NPE>(E, ea.y, ga, Sa);
    for (int b = 0; b < NPE; ++b) {
      const int rel = P.adj_rel[static_cast<size_t>(q) * NPE + b];
      if (rel < 0) continue;
      if (Kr) Kr[base + rel] += E.nu * Sa[b];
      if (Jr) Jr[base + rel] += E.nu * Sa[b] + E.cc * (ga * E.g[b]);
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
  for (int k = 0; k < 4; ++k) {
    const size_t smem = kScrSmem + kRecSmemMax;
    if (smem &&
        cudaFuncSetAttribute(fns[k], cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
            cudaSuccess)
      return PS_ERR_CUDA;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[k], kThreads, smem) != cudaSuccess)
      return PS_ERR_CUDA;
    best = per_sm < best ? per_sm : best;
  }
  *out = sms * best;
  return PS_OK;
}

int launch_propagate(const PropParams& prm, bool linear, int npe, cudaStream_t st, std::string* err) {
  void* fn = select_kernel(linear, npe);
  PropParams local = prm;
  void* args[] = {&local};
  const size_t smem = kScrSmem + static_cast<size_t>(prm.rec_rows) * kRecInts4 * sizeof(int4) +
                      (prm.r_smem ? static_cast<size_t>(prm.rec_rows) * 32 * sizeof(double) : 0);
  const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(prm.G * prm.C), dim3(kThreads), args, smem, st);
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

void launch_to_blocked(const double* src, double* dst, int count, int d, int L, cudaStream_t st) {
  // src [count][d] -> group-blocked: group g's [d][32] block from rows g*L ..
  for (int g = 0; g * L < count; ++g) {
    const int rows = count - g * L < L ? count - g * L : L;
    dim3 grid((d + 31) / 32, (rows + 31) / 32);
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src + static_cast<size_t>(g) * L * d,
                                                   dst + static_cast<size_t>(g) * d * kLanes, rows, d, d, kLanes);
  }
}

void launch_from_blocked(const double* src, double* dst, int count, int d, int L, cudaStream_t st) {
  for (int g = 0; g * L < count; ++g) {
    const int rows = count - g * L < L ? count - g * L : L;
    dim3 grid((rows + 31) / 32, (d + 31) / 32);
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src + static_cast<size_t>(g) * d * kLanes,
                                                   dst + static_cast<size_t>(g) * L * d, d, rows, kLanes, d);
  }
}

void launch_il_blocked(const double* src, double* dst, int d, int count, int stride, int L, bool to_blocked,
                       cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(d) * count;
  il_blocked_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(src, dst, d, count, stride, L,
                                                                                to_blocked ? 1 : 0);
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

#ifndef PPPC_SB_THREADS
#define PPPC_SB_THREADS 512
#endif
constexpr int kSbThreads = PPPC_SB_THREADS;

size_t sysblock_smem(int d) { return static_cast<size_t>(7) * d * sizeof(double); }

int launch_sysblock(const PropParams& prm, const SysParams& sp, int npe, cudaStream_t st, std::string* err) {
  const size_t smem = sp.smem_vectors ? sysblock_smem(prm.d) : 0;
  void* fn = npe == 2 ? reinterpret_cast<void*>(&sysblock_kernel<2, kSbThreads>)
                      : reinterpret_cast<void*>(&sysblock_kernel<3, kSbThreads>);
  if (npe != 2 && npe != 3) return PS_ERR_BAD_ARG;
  if (smem > 0 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
                      cudaSuccess) {
    if (err) *err = "cuda: sysblock shared-memory opt-in failed";
    return PS_ERR_CUDA;
  }
  if (npe == 2)
    sysblock_kernel<2, kSbThreads><<<prm.count, kSbThreads, smem, st>>>(prm, sp);
  else
    sysblock_kernel<3, kSbThreads><<<prm.count, kSbThreads, smem, st>>>(prm, sp);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (err) *err = std::string("cuda: sysblock launch failed: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

static_assert(kClMaxC == kClusterMaxC, "cluster geometry arrays");

size_t syscluster_smem(const ClusterGeom& gm) {
  return (static_cast<size_t>(gm.win_max) + 3 * static_cast<size_t>(gm.rows_max)) * sizeof(double) +
         static_cast<size_t>((gm.rows_max + 3) & ~3) * sizeof(unsigned short) +
         static_cast<size_t>(gm.hub_len) * (sizeof(double) + sizeof(int)) + sizeof(ClShared) + 16;
}

int syscluster_max_rows() { return kClRpt * kClThreads; }

namespace {
// instantiated slot widths: 3 (2-node radial elements), 7 (P1 triangles on the
// polar mesh), kEll (anything else)
int syscluster_width(int npe, int ell_width) {
  if (npe == 2 && ell_width <= 3) return 3;
  if (npe == 3 && ell_width <= 7) return 7;
  return kEll;
}

using ClusterKernel = void (*)(const PropParams, const SysParams, const ClusterGeom);
ClusterKernel syscluster_fn(int npe, int ell_width) {
  const int w = syscluster_width(npe, ell_width);
  if (npe == 2) return w == 3 ? syscluster_kernel<2, 3> : syscluster_kernel<2, kEll>;
  return w == 7 ? syscluster_kernel<3, 7> : syscluster_kernel<3, kEll>;
}

bool syscluster_config(ClusterKernel fn, const ClusterGeom& gm, int count, cudaStream_t st, cudaLaunchConfig_t* cfg,
                       cudaLaunchAttribute* attr) {
  const size_t smem = syscluster_smem(gm);
  if (cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return false;
  if (gm.C > 8 && cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return false;
  *cfg = cudaLaunchConfig_t{};
  cfg->gridDim = dim3(static_cast<unsigned>(count) * gm.C);
  cfg->blockDim = dim3(kClThreads);
  cfg->dynamicSmemBytes = smem;
  cfg->stream = st;
  attr->id = cudaLaunchAttributeClusterDimension;
  attr->val.clusterDim.x = gm.C;
  attr->val.clusterDim.y = 1;
  attr->val.clusterDim.z = 1;
  cfg->attrs = attr;
  cfg->numAttrs = 1;
  return true;
}
}  // namespace

int syscluster_max_clusters(int npe, int ell_width, const ClusterGeom& gm) {
  if (npe != 2 && npe != 3) return 0;
  const ClusterKernel fn = syscluster_fn(npe, ell_width);
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr;
  if (!syscluster_config(fn, gm, 1, nullptr, &cfg, &attr)) {
    cudaGetLastError();
    return 0;
  }
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(fn), &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int launch_syscluster(const PropParams& prm, const SysParams& sp, const ClusterGeom& gm, int npe, cudaStream_t st,
                      std::string* err) {
  if (npe != 2 && npe != 3) return PS_ERR_BAD_ARG;
  const ClusterKernel fn = syscluster_fn(npe, sp.ell_width);
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr;
  if (!syscluster_config(fn, gm, prm.count, st, &cfg, &attr)) {
    if (err) *err = std::string("cuda: cluster engine setup failed: ") + cudaGetErrorString(cudaGetLastError());
    return PS_ERR_CUDA;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, prm, sp, gm);
  if (e != cudaSuccess) {
    if (err) *err = std::string("cuda: cluster engine launch failed: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

int launch_phase_probe(const PropParams& prm, int mode, double* sink, cudaStream_t st) {
  const size_t smem = kScrSmem + static_cast<size_t>(prm.rec_rows) * kRecInts4 * sizeof(int4);
  if (cudaFuncSetAttribute(reinterpret_cast<const void*>(phase_probe_kernel),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
    return PS_ERR_CUDA;
  phase_probe_kernel<<<prm.G * prm.C, kThreads, smem, st>>>(prm, mode, sink);
  return cudaGetLastError() == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

void launch_frozen_K(const DevProblem& p, const double* u_ref, double* K_out, cudaStream_t st) {
  launch_assemble_ops(p, 1, u_ref, K_out, nullptr, st);
}

}  // namespace pppc
