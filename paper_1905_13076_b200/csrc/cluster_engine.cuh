// System-per-cluster engine (included by kernels.cu inside its namespaces).
//
// One thread-block cluster of C CTAs runs one system's whole batch of
// implicit-Euler steps (proj/src/propagators.cpp:96-115): refill, Newton control
// (:27-58) and every Jacobi-PCG iteration, as sysblock_kernel does with one
// block, but with the rows split into C contiguous ranges, one per CTA, so that
// the Krylov vectors of a system of d ~ 50k rows stay ON CHIP for the whole
// launch:
//   * the search direction p of the CTA's rows plus the halo its rows gather
//     (the window [win_lo, win_hi) of columns), the residual r, the update x and
//     q = A p of the CTA's rows live in shared memory;
//   * after every update the owning thread pushes the entries of p that other
//     CTAs' windows hold straight into their shared memory with st.async
//     (DSMEM store + complete_tx on the receiver's mbarrier): the receiver waits
//     for its known halo byte count, no fence and no cluster barrier;
//   * dot products: fixed-order block reduction, warp 0 sends the block sums to
//     every CTA (st.async into the receivers' slots, complete_tx on their
//     mbarrier), waits for the C x ND values of its own CTA and sums them in rank
//     order -> all CTAs hold bit-identical scalars and take the same branches;
//   * one reduction per PCG iteration: the exact r.z and r.r of the updated
//     residual are accumulated by the next iteration's SpMV pass (which reads r
//     and the Jacobi entry anyway), so an iteration is
//         SpMV pass -> cluster sum of {p.q, q.z, q.Dq, r.z, r.r} -> update pass
//     and convergence is seen one SpMV pass late (one wasted pass per solve).
// Per PCG iteration only the matrix streams from L2 (padded columns, shared or
// per-system slot values, Jacobi); nothing device-wide is synchronised and the
// hardware schedules the clusters (one per system) as CTAs drain.  Hardware
// cluster barriers (with their device-scope fence) are used only where global
// memory written by one CTA is read by another (the Newton state u).
// Same arithmetic per row as sysblock_kernel (sb_refill_row / sb_refill_hub are
// reused through offset pointers); a system's result depends only on (d, C).

namespace cg = cooperative_groups;

#ifndef PPPC_CL_THREADS
#define PPPC_CL_THREADS 1024
#endif
#ifndef PPPC_CL_RB
#define PPPC_CL_RB 1
#endif
constexpr int kClThreads = PPPC_CL_THREADS;
constexpr int kClRb = PPPC_CL_RB;   // rows per thread whose operands are in flight together (SpMV pass)
constexpr int kClMaxC = 16;         // CTAs per cluster at most (8 portable)
constexpr int kClNd = 8;            // reduction slots per CTA
constexpr int kClMaxRpt = 32;       // rows per thread at most (row-kind / push bit masks)

struct ClShared {
  double red[kClNd][32];
  double cpart[2][kClMaxC][kClNd];
  double tot[kClNd];
  double qh;                              // the hub row's product (owner CTA)
  unsigned long long red_mb[2], halo_mb;  // mbarriers
  int n_push;
  int push_lo[kClMaxC], push_hi[kClMaxC];
  unsigned push_base[kClMaxC];            // shared::cluster address of the target's window entry of row 0
  unsigned push_mb[kClMaxC];              // shared::cluster address of the target's halo mbarrier
  ps_curve curves[kMaxCurves];
};

struct ClCtx {
  int C, rank, r0, r1, wlo, whi;
  int par, red_phase, halo_phase;   // red_phase: bit b = phase parity of red_mb[b]
  unsigned halo_in_bytes;
  int hub;          // the hub row if this CTA owns it, else -1
  bool hub_shared;
  const double *hubD;   // Jacobi entry of the hub row (owner)
  double* pw;   // p window (index = column - wlo)
  double* rs;   // r of own rows (index = row - r0)
  double* xs;   // x of own rows
  double* qs;   // q of own rows
  ClShared* sh;
};

__device__ __forceinline__ unsigned cl_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned cl_mapa(unsigned addr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// remote (or own) shared-memory store of one double that completes 8 bytes on the
// target CTA's mbarrier
__device__ __forceinline__ void cl_st_async(unsigned addr, double v, unsigned mbar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(__double_as_longlong(v)), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void cl_mbar_init(unsigned long long* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cl_smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void cl_mbar_expect(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cl_smem_u32(mb)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cl_mbar_wait(unsigned long long* mb, unsigned parity) {
  const unsigned a = cl_smem_u32(mb);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// Sends v (row i of p, owned here) to every CTA whose window holds column i.
__device__ __forceinline__ void cl_push_row(const ClCtx& X, int i, double v) {
  const ClShared* sh = X.sh;
  for (int e = 0; e < sh->n_push; ++e)
    if (i >= sh->push_lo[e] && i < sh->push_hi[e])
      cl_st_async(sh->push_base[e] + static_cast<unsigned>(i) * 8u, v, sh->push_mb[e]);
}

// Block barrier (the CTA's own p entries are written) + arrival of the halo
// entries the other CTAs pushed since the last call.
__device__ __forceinline__ void cl_halo_sync(ClCtx& X) {
  __syncthreads();
  if (X.halo_in_bytes) {
    if (threadIdx.x == 0) cl_mbar_expect(&X.sh->halo_mb, X.halo_in_bytes);
    cl_mbar_wait(&X.sh->halo_mb, X.halo_phase);
    X.halo_phase ^= 1;
  }
}

// Fixed-order cluster sum of ND values; every thread of every CTA returns the
// same totals.  HUBFIX (PCG pass, values {p.q, q.z, q.Dq, r.z, r.r, hub part}):
// the hub row's product is the owner's block sum of slot 5; the owner adds the
// row's terms to its block sums before they are sent and keeps the product.
template <int ND, bool HUBFIX>
__device__ __forceinline__ void cl_reduce(ClCtx& X, double (&v)[ND]) {
  constexpr int NW = kClThreads / 32;
  static_assert(NW <= 32 && ND <= kClNd, "reduction geometry");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ClShared* sh = X.sh;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < ND; ++k) sh->red[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
    unsigned long long* mb = &sh->red_mb[X.par];
    constexpr int NS = HUBFIX ? ND - 1 : ND;   // values that cross the cluster
    if (lane == 0) cl_mbar_expect(mb, static_cast<unsigned>(X.C) * NS * 8u);
    double s[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      double w = lane < NW ? sh->red[k][lane] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) w += __shfl_down_sync(0xffffffffu, w, off);
      s[k] = __shfl_sync(0xffffffffu, w, 0);
    }
    if (HUBFIX && X.hub >= 0) {
      const double qh = s[ND - 1];
      const double dh = *X.hubD;
      s[0] += X.pw[X.hub - X.wlo] * qh;
      s[1] += qh * (dh * X.rs[X.hub - X.r0]);
      s[2] += qh * (dh * qh);
      if (lane == 0) sh->qh = qh;
    }
    if (lane < X.C) {
      const unsigned dst = cl_mapa(cl_smem_u32(&sh->cpart[X.par][X.rank][0]), lane);
      const unsigned rmb = cl_mapa(cl_smem_u32(mb), lane);
#pragma unroll
      for (int k = 0; k < NS; ++k) cl_st_async(dst + 8u * k, s[k], rmb);
    }
    cl_mbar_wait(mb, (X.red_phase >> X.par) & 1);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      // rank-order sum: lane t holds CTA t's value, folded by a fixed tree
      double w = lane < X.C ? sh->cpart[X.par][lane][k] : 0.0;
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) w += __shfl_down_sync(0xffffffffu, w, off);
      if (lane == 0) sh->tot[k] = w;
    }
  }
  X.red_phase ^= 1 << X.par;
  X.par ^= 1;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ND; ++k) v[k] = sh->tot[k];
}

// Refill over the CTA's rows (sb_refill_row / sb_refill_hub through the offset
// pointers of V), cluster totals {R.R, f.f, r.z, r.r}; publishes p.
template <int NPE>
__device__ __forceinline__ void cl_refill(ClCtx& X, const PropParams& P, const SysParams& S, const SbVec& V, int sys,
                                          int step, bool first, unsigned pushmask, double (&t)[4]) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = X.r0 + threadIdx.x; i < X.r1; i += kClThreads)
    if (i != S.hub) sb_refill_row<NPE>(P, S, X.sh->curves, V, sys, step, first, i, acc);
  if (X.hub >= 0 && threadIdx.x == kClThreads - 1) sb_refill_hub<NPE>(P, S, X.sh->curves, V, sys, step, first, acc);
  if (X.sh->n_push) {
    __syncthreads();  // the hub row's p entry is written by another thread than the one that pushes it
    int k = 0;
    for (int i = X.r0 + threadIdx.x; i < X.r1; i += kClThreads, ++k)
      if ((pushmask >> k) & 1u) cl_push_row(X, i, X.pw[i - X.wlo]);
  }
  cl_reduce<4, false>(X, acc);
  cl_halo_sync(X);
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
  X.red_phase = 0;
  X.halo_phase = 0;
  X.pw = reinterpret_cast<double*>(cl_smem);
  X.rs = X.pw + Gm.win_max;
  X.xs = X.rs + Gm.rows_max;
  X.qs = X.xs + Gm.rows_max;
  X.sh = reinterpret_cast<ClShared*>(X.qs + Gm.rows_max);
  ClShared* sh = X.sh;
  const int sys = blockIdx.x / Gm.C;
  const int tid = threadIdx.x;
  if (tid < P.ncurves) sh->curves[tid] = P.curves[tid];
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
  X.hub = (S.hub >= r0 && S.hub < r1) ? S.hub : -1;
  X.hub_shared = S.hub >= 0 && sb_shared_row(P, S.hub);
  X.hubD = S.hub >= 0 ? (X.hub_shared ? P.Dsh + S.hub : V.D + S.hub) : nullptr;
  // halo plan: who holds rows of mine (push list), how many bytes arrive here
  {
    unsigned in_bytes = 0;
    for (int t = 0; t < X.C; ++t) {
      if (t == X.rank) continue;
      const int lo = max(Gm.row_begin[t], X.wlo), hi = min(Gm.row_begin[t + 1], X.whi);
      if (lo < hi) in_bytes += static_cast<unsigned>(hi - lo) * 8u;
    }
    X.halo_in_bytes = in_bytes;
  }
  if (tid == 0) {
    cl_mbar_init(&sh->red_mb[0], 1);
    cl_mbar_init(&sh->red_mb[1], 1);
    cl_mbar_init(&sh->halo_mb, 1);
    int n = 0;
    for (int t = 0; t < X.C; ++t) {
      if (t == X.rank) continue;
      const int tlo = Gm.win_lo[t], thi = Gm.win_hi[t];
      const int lo = max(r0, tlo), hi = min(r1, thi);
      if (lo >= hi) continue;
      sh->push_lo[n] = lo;
      sh->push_hi[n] = hi;
      sh->push_base[n] = cl_mapa(cl_smem_u32(X.pw), t) - static_cast<unsigned>(tlo) * 8u;
      sh->push_mb[n] = cl_mapa(cl_smem_u32(&sh->halo_mb), t);
      ++n;
    }
    sh->n_push = n;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // start state from the group-blocked layout [G][d][32] (the callers' staging)
  const int g = sys / P.L, l = sys - g * P.L;
  double* ub = P.u + static_cast<size_t>(g) * d * kLanes + l;
  for (int i = r0 + tid; i < r1; i += kClThreads) V.u[i] = ub[static_cast<size_t>(i) * kLanes];
  cl.sync();
  // which of this thread's rows carry per-system values / are held by other windows
  unsigned ownmask = 0, pushmask = 0;
  {
    int k = 0;
    for (int i = r0 + tid; i < r1; i += kClThreads, ++k) {
      if (!sb_shared_row(P, i)) ownmask |= 1u << k;
      for (int e = 0; e < sh->n_push; ++e)
        if (i >= sh->push_lo[e] && i < sh->push_hi[e]) pushmask |= 1u << k;
    }
  }

  const int hub_base = S.hub >= 0 ? __ldg(P.rp + S.hub) : 0;
  int code = PS_OK, last_nit = 0, max_nit = 0, max_pit = 0;
  double t_fail = 0.0, res_fail = 0.0;
  long long newton_total = 0, pcg_total = 0;
  double t[4];
  for (int step = 0; step < P.steps && code == PS_OK; ++step) {
    const double t_now = P.t_next[static_cast<size_t>(step) * P.count + sys];
    cl_refill<NPE>(X, P, S, V, sys, step, true, pushmask, t);
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
          // SpMV pass: q = A p over this thread's rows; partials p.q, q.z, q.Dq
          // and r.z, r.r of the residual as the last update left it
          double a6[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
          {
            int k = 0;
#pragma unroll 1
            for (int i0 = r0 + tid; i0 < r1; i0 += kClThreads * kClRb, k += kClRb) {
              ClRow R[kClRb];
#pragma unroll
              for (int u = 0; u < kClRb; ++u) {
                const int i = i0 + u * kClThreads;
                if (i < r1) cl_load_row(P, S, V, i, (ownmask >> (k + u)) & 1u, R[u]);
              }
#pragma unroll
              for (int u = 0; u < kClRb; ++u) {
                const int i = i0 + u * kClThreads;
                if (i >= r1) break;
                double qv = 0.0;
#pragma unroll
                for (int s = 0; s < kEll; ++s) qv += R[u].a[s] * X.pw[R[u].c[s] - X.wlo];
                const double ri = X.rs[i - r0];
                const double zi = R[u].dv * ri;
                if (i != S.hub) {
                  X.qs[i - r0] = qv;
                  a6[0] += X.pw[i - X.wlo] * qv;
                  a6[1] += qv * zi;
                  a6[2] += qv * (R[u].dv * qv);
                }
                a6[3] += ri * zi;
                a6[4] += ri * ri;
              }
            }
          }
          if (X.hub >= 0) {
            // the hub row's product (its columns lie inside the owner's window)
            double part = 0.0;
            for (int s = tid; s < S.hub_len; s += kClThreads) {
              const int kk = hub_base + s;
              const double av = X.hub_shared ? __ldg(P.Ash + kk) : V.hA[s];
              part += av * X.pw[__ldg(P.ci + kk) - X.wlo];
            }
            a6[5] = part;
          }
          cl_reduce<6, true>(X, a6);
          const double t0v = a6[0], t1v = a6[1], t2v = a6[2];
          if (pit > 0) {
            // the state after update `pit`
            const double rr = a6[4];
            rho = a6[3];
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
          if (!isfinite(t0v) || t0v == 0.0) {
            code = PS_ERR_SINGULAR;
            res_fail = res_pre;
            t_fail = t_now;
            break;
          }
          const double alpha = rho / t0v;
          const double rho_est = rho - 2.0 * alpha * t1v + alpha * alpha * t2v;
          const double beta = rho_est / rho;
          // update pass: x (+)= alpha p, r -= alpha q, z = D r, p = z + beta p
          const bool first_it = pit == 0;
          const double qh = X.hub >= 0 ? sh->qh : 0.0;
          {
            int k = 0;
#pragma unroll 2
            for (int i = r0 + tid; i < r1; i += kClThreads, ++k) {
              const bool own = (ownmask >> k) & 1u;
              const double dv = own ? V.D[i] : __ldg(P.Dsh + i);
              const double pv = X.pw[i - X.wlo];
              const double qv = i == S.hub ? qh : X.qs[i - r0];
              const double xv = first_it ? 0.0 : X.xs[i - r0];
              X.xs[i - r0] = first_it ? alpha * pv : xv + alpha * pv;
              const double rn = X.rs[i - r0] - alpha * qv;
              const double pn = dv * rn + beta * pv;
              X.rs[i - r0] = rn;
              X.pw[i - X.wlo] = pn;
              if ((pushmask >> k) & 1u) cl_push_row(X, i, pn);
            }
          }
          pit += 1;
          cl_halo_sync(X);
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
        cl_reduce<1, false>(X, bad);
        if (bad[0] > 0.0) {
          code = PS_ERR_SINGULAR;
          res_fail = res_pre;
          t_fail = t_now;
          break;
        }
      }
      cl.sync();  // u is read across CTAs by the refill
      // ---- residual at the trial point; optional backtracking
      double post;
      for (;;) {
        cl_refill<NPE>(X, P, S, V, sys, step, false, pushmask, t);
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
    // the next step's first refill overwrites u_prev, which the last refill of
    // this step read across CTAs: its cluster sum already ordered those reads
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
