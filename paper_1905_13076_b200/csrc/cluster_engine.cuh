// System-per-cluster engine (included by kernels.cu inside its namespaces).
//
// One thread-block cluster of C CTAs runs one system's whole batch of
// implicit-Euler steps (proj/src/propagators.cpp:96-115): refill, Newton control
// (:27-58) and every Jacobi-PCG iteration, as sysblock_kernel does with one
// block, but with the rows split into C contiguous ranges, one per CTA, so that
// the Krylov vectors of a system of d ~ 50k rows stay ON CHIP for the whole
// launch:
//   * the search direction p of the CTA's rows plus the halo its rows gather
//     (the window [win_lo, win_hi) of columns) in shared memory; after every
//     update the owner pushes the entries other CTAs' windows hold into their
//     shared memory through DSMEM (st.shared::cluster via map_shared_rank);
//   * the residual r and the solution update x of the CTA's rows in shared
//     memory; q = A p of the thread's rows in registers (rows are dealt
//     thread-cyclically, at most kClRpt per thread);
//   * dot products: fixed-order block reduction, every CTA writes its partials
//     into every CTA's shared memory, one hardware cluster barrier
//     (barrier.cluster arrive.release / wait.acquire), then every CTA sums the C
//     partials in rank order -> all CTAs hold bit-identical scalars and take the
//     same branches.  The same barrier publishes the halo pushes.
// Per PCG iteration only the matrix streams from L2 (padded columns, shared or
// per-system slot values, Jacobi); nothing device-wide is synchronised and the
// hardware schedules the clusters (one per system) as CTAs drain.
// Same arithmetic per row as sysblock_kernel (sb_refill_row / sb_refill_hub are
// reused through offset pointers); a system's result depends only on (d, C).

namespace cg = cooperative_groups;

constexpr int kClThreads = 512;
constexpr int kClRpt = 18;      // rows per thread at most (q lives in registers)
constexpr int kClMaxC = 16;     // CTAs per cluster at most (8 portable)
constexpr int kClNd = 8;        // reduction slots per CTA

struct ClShared {
  double red[kClNd][kClThreads / 32];
  double cpart[2][kClMaxC][kClNd];
  ps_curve curves[kMaxCurves];
};

struct ClCtx {
  int C, rank, r0, r1, wlo, whi, par;
  double* pw;   // p window (index = column - wlo)
  double* rs;   // r of own rows (index = row - r0)
  double* xs;   // x of own rows
  ClShared* sh;
};

// Halo push: the entries of p this CTA owns that other CTAs' windows hold.
__device__ __forceinline__ void cl_push_halo(cg::cluster_group& cl, const ClusterGeom& Gm, const ClCtx& X) {
  for (int t = 0; t < X.C; ++t) {
    if (t == X.rank) continue;
    const int tlo = Gm.win_lo[t], thi = Gm.win_hi[t];
    const int lo = max(X.r0, tlo), hi = min(X.r1, thi);
    if (lo >= hi) continue;
    double* remote = cl.map_shared_rank(X.pw, t);
    for (int i = lo + threadIdx.x; i < hi; i += kClThreads) remote[i - tlo] = X.pw[i - X.wlo];
  }
}

// Fixed-order cluster sum of ND values; every thread of every CTA returns the
// same totals.  push: publish this CTA's p entries to the other windows before
// the barrier (the block barrier inside orders the owners' writes first).
template <int ND>
__device__ __forceinline__ void cl_reduce(cg::cluster_group& cl, const ClusterGeom& Gm, ClCtx& X, double (&v)[ND],
                                          bool push) {
  constexpr int NW = kClThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) X.sh->red[k][warp] = v[k];
  }
  __syncthreads();
  if (push) cl_push_halo(cl, Gm, X);
  if (threadIdx.x < ND) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += X.sh->red[threadIdx.x][w];
    for (int t = 0; t < X.C; ++t) {
      ClShared* rsh = cl.map_shared_rank(X.sh, t);
      rsh->cpart[X.par][X.rank][threadIdx.x] = s;
    }
  }
  cl.sync();
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    double s = 0.0;
    for (int t = 0; t < X.C; ++t) s += X.sh->cpart[X.par][t][k];
    v[k] = s;
  }
  X.par ^= 1;
}

// Refill over the CTA's rows (sb_refill_row / sb_refill_hub through the offset
// pointers of V), cluster totals {R.R, f.f, r.z, r.r}; publishes p.
template <int NPE>
__device__ __forceinline__ void cl_refill(cg::cluster_group& cl, const ClusterGeom& Gm, ClCtx& X,
                                          const PropParams& P, const SysParams& S, const SbVec& V, int sys, int step,
                                          bool first, double (&t)[4]) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = X.r0 + threadIdx.x; i < X.r1; i += kClThreads)
    if (i != S.hub) sb_refill_row<NPE>(P, S, X.sh->curves, V, sys, step, first, i, acc);
  if (S.hub >= X.r0 && S.hub < X.r1 && threadIdx.x == kClThreads - 1)
    sb_refill_hub<NPE>(P, S, X.sh->curves, V, sys, step, first, acc);
  cl_reduce<4>(cl, Gm, X, acc, true);
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = acc[k];
}

struct ClRow {
  int c[kEll];
  double a[kEll];
  double dv;
};

// Operands of row i that stream from L2: padded columns, slot values (shared
// M/dt + K_const or the system's own), Jacobi entry.
__device__ __forceinline__ void cl_load_row(const PropParams& P, const SysParams& S, const SbVec& V, int i, bool own,
                                            ClRow& o) {
  const int d = P.d;
  const double* As = own ? V.A : S.AshT;
  const double* Ds = own ? V.D : P.Dsh;
#pragma unroll
  for (int k = 0; k < kEll; ++k) o.c[k] = __ldg(S.ciT + static_cast<size_t>(k) * d + i);
#pragma unroll
  for (int k = 0; k < kEll; ++k) o.a[k] = As[static_cast<size_t>(k) * d + i];
  o.dv = Ds[i];
}

template <int NPE>
__global__ void __launch_bounds__(kClThreads, 1) syscluster_kernel(const PropParams P, const SysParams S,
                                                                   const ClusterGeom Gm) {
  extern __shared__ __align__(16) unsigned char cl_smem[];
  cg::cluster_group cl = cg::this_cluster();
  ClCtx X;
  X.C = Gm.C;
  X.rank = static_cast<int>(cl.block_rank());
  X.r0 = Gm.row_begin[X.rank];
  X.r1 = Gm.row_begin[X.rank + 1];
  X.wlo = Gm.win_lo[X.rank];
  X.whi = Gm.win_hi[X.rank];
  X.par = 0;
  X.pw = reinterpret_cast<double*>(cl_smem);
  X.rs = X.pw + Gm.win_max;
  X.xs = X.rs + Gm.rows_max;
  X.sh = reinterpret_cast<ClShared*>(X.xs + Gm.rows_max);
  const int sys = blockIdx.x / Gm.C;
  const int tid = threadIdx.x;
  if (tid < P.ncurves) X.sh->curves[tid] = P.curves[tid];
  const int d = P.d;
  const int r0 = X.r0, r1 = X.r1;
  const size_t vb = static_cast<size_t>(sys) * d;
  SbVec V;
  V.u = S.su + vb;
  V.uprev = P.uprev + vb;
  V.D = P.Dinv + vb;
  V.x = X.xs - r0;
  V.r = X.rs - r0;
  V.p = X.pw - X.wlo;
  V.q = nullptr;
  V.A = S.sA + static_cast<size_t>(sys) * kEll * d;
  V.hA = S.hub >= 0 ? S.hubA + static_cast<size_t>(sys) * S.hub_len : nullptr;
  // start state from the group-blocked layout [G][d][32] (the callers' staging)
  const int g = sys / P.L, l = sys - g * P.L;
  double* ub = P.u + static_cast<size_t>(g) * d * kLanes + l;
  for (int i = r0 + tid; i < r1; i += kClThreads) V.u[i] = ub[static_cast<size_t>(i) * kLanes];
  // which of this thread's rows carry per-system values
  unsigned ownmask = 0;
#pragma unroll
  for (int k = 0; k < kClRpt; ++k) {
    const int i = r0 + tid + k * kClThreads;
    if (i < r1 && !sb_shared_row(P, i)) ownmask |= 1u << k;
  }
  cl.sync();

  const bool hub_here = S.hub >= r0 && S.hub < r1;
  const bool hub_shared = S.hub >= 0 && sb_shared_row(P, S.hub);
  const int hub_base = S.hub >= 0 ? __ldg(P.rp + S.hub) : 0;
  int code = PS_OK, last_nit = 0, max_nit = 0, max_pit = 0;
  double t_fail = 0.0, res_fail = 0.0;
  long long newton_total = 0, pcg_total = 0;
  double t[4];
  double q[kClRpt];
  for (int step = 0; step < P.steps && code == PS_OK; ++step) {
    const double t_now = P.t_next[static_cast<size_t>(step) * P.count + sys];
    cl_refill<NPE>(cl, Gm, X, P, S, V, sys, step, true, t);
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
          // phase A: q = A p over this thread's rows (next row's operands in
          // flight while the current row is multiplied), partials p.q, q.z, q.Dq
          double a7[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          {
            ClRow cur, nxt;
            const int i_first = r0 + tid;
            if (i_first < r1) cl_load_row(P, S, V, i_first, ownmask & 1u, cur);
#pragma unroll
            for (int k = 0; k < kClRpt; ++k) {
              const int i = r0 + tid + k * kClThreads;
              if (i >= r1) break;
              if (k + 1 < kClRpt) {
                const int in = i + kClThreads;
                if (in < r1) cl_load_row(P, S, V, in, (ownmask >> (k + 1)) & 1u, nxt);
              }
              if (i != S.hub) {
                double qv = 0.0;
#pragma unroll
                for (int s = 0; s < kEll; ++s) qv += cur.a[s] * X.pw[cur.c[s] - X.wlo];
                q[k] = qv;
                const double zi = cur.dv * X.rs[i - r0];
                a7[0] += X.pw[i - X.wlo] * qv;
                a7[1] += qv * zi;
                a7[2] += qv * (cur.dv * qv);
              }
              cur = nxt;
            }
          }
          if (S.hub >= 0) {
            // the hub row's product: every CTA sums the slots whose column it
            // owns; the owner also sends p, D r and D of the hub through the sum
            double part = 0.0;
            for (int s = tid; s < S.hub_len; s += kClThreads) {
              const int kk = hub_base + s;
              const int col = __ldg(P.ci + kk);
              if (col >= r0 && col < r1) {
                const double av = hub_shared ? __ldg(P.Ash + kk) : V.hA[s];
                part += av * X.pw[col - X.wlo];
              }
            }
            a7[3] = part;
            if (hub_here && tid == 0) {
              const double dh = hub_shared ? __ldg(P.Dsh + S.hub) : V.D[S.hub];
              a7[4] = X.pw[S.hub - X.wlo];
              a7[5] = dh * X.rs[S.hub - r0];
              a7[6] = dh;
            }
          }
          cl_reduce<7>(cl, Gm, X, a7, false);
          double t0v = a7[0], t1v = a7[1], t2v = a7[2];
          const double qh = a7[3];
          if (S.hub >= 0) {
            t0v += a7[4] * qh;
            t1v += qh * a7[5];
            t2v += qh * (a7[6] * qh);
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
          // phase B: x (+)= alpha p, r -= alpha q, z = D r, p = z + beta p
          double b2[2] = {0.0, 0.0};
          const bool first_it = pit == 0;
#pragma unroll
          for (int k = 0; k < kClRpt; ++k) {
            const int i = r0 + tid + k * kClThreads;
            if (i >= r1) break;
            const bool own = (ownmask >> k) & 1u;
            const double dv = own ? V.D[i] : __ldg(P.Dsh + i);
            const double pv = X.pw[i - X.wlo];
            const double qv = i == S.hub ? qh : q[k];
            const double xv = first_it ? 0.0 : X.xs[i - r0];
            X.xs[i - r0] = first_it ? alpha * pv : xv + alpha * pv;
            const double rn = X.rs[i - r0] - alpha * qv;
            const double z = dv * rn;
            X.rs[i - r0] = rn;
            X.pw[i - X.wlo] = z + beta * pv;
            b2[0] += rn * rn;
            b2[1] += rn * z;
          }
          cl_reduce<2>(cl, Gm, X, b2, true);
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
        for (int i = r0 + tid; i < r1; i += kClThreads) {
          const double dx = V.x[i];
          bad[0] += isfinite(dx) ? 0.0 : 1.0;
          V.u[i] += lambda * dx;
        }
        cl_reduce<1>(cl, Gm, X, bad, false);
        if (bad[0] > 0.0) {
          code = PS_ERR_SINGULAR;
          res_fail = res_pre;
          t_fail = t_now;
          break;
        }
      } else {
        cl.sync();
      }
      // ---- residual at the trial point; optional backtracking
      double post;
      for (;;) {
        cl_refill<NPE>(cl, Gm, X, P, S, V, sys, step, false, t);
        post = sqrt(t[0]);
        if (P.line_search > 0 && ls_k < P.line_search && !(post <= tol) &&
            !(post <= (1.0 - 1e-4 * lambda) * res_pre)) {
          lambda *= 0.5;
          ls_k += 1;
          if (pact)
            for (int i = r0 + tid; i < r1; i += kClThreads) V.u[i] -= lambda * V.x[i];
          cl.sync();
          continue;
        }
        break;
      }
      if (X.rank == 0 && tid == 0 && P.trace) P.trace[static_cast<size_t>(sys) * P.newton_max + (nit - 1)] = post;
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
  for (int i = r0 + tid; i < r1; i += kClThreads) ub[static_cast<size_t>(i) * kLanes] = V.u[i];
  if (X.rank == 0 && tid == 0) {
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
  // no CTA may exit while others can still write into its shared memory
  cl.sync();
}
