// System-per-cluster engine (included by kernels.cu inside its namespaces).
//
// One thread-block cluster of C CTAs runs one system's whole batch of
// implicit-Euler steps (proj/src/propagators.cpp:96-115): refill, Newton control
// (:27-58) and every Jacobi-PCG iteration, as sysblock_kernel does with one
// block, but with the rows split into C contiguous ranges, one per CTA, so that
// the Krylov vectors of a system of d ~ 50k rows stay ON CHIP for the whole
// launch:
//   * the search direction p of the CTA's rows plus the halo its rows gather
//     (the window [win_lo, win_hi) of columns), the residual r, q = A p and the
//     Jacobi entries of the CTA's rows live in shared memory (rows are dealt
//     thread-cyclically, at most kClRpt per thread); the solution update x, which
//     only the update pass touches, stays in L2;
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
//   * the sparsity pattern is held on chip as a dictionary: a row carries an
//     8-bit pattern id (packed in registers), the pattern's relative columns sit
//     in shared memory, so no column index is read from memory in the PCG loop
//     (rows whose pattern is not among the 255 most frequent ones fall back to
//     the padded column lists).
// Per PCG iteration only the slot values stream from L2 (shared M/dt + K_const or
// the system's own, row length many); nothing device-wide is synchronised and the
// hardware schedules the clusters (one per system) as CTAs drain.  Hardware
// cluster barriers (with their device-scope fence) are used only where global
// memory written by one CTA is read by another (the Newton state u).
// Same arithmetic per row as sysblock_kernel (sb_refill_row / sb_refill_hub are
// reused through offset pointers); a system's result depends only on (d, C).

namespace cg = cooperative_groups;

#ifndef PPPC_CL_THREADS
#define PPPC_CL_THREADS 512
#endif
#ifndef PPPC_CL_RB
#define PPPC_CL_RB 1
#endif
#ifndef PPPC_CL_RPT
#define PPPC_CL_RPT (6656 / PPPC_CL_THREADS)
#endif
constexpr int kClThreads = PPPC_CL_THREADS;
constexpr int kClRb = PPPC_CL_RB;     // rows per thread whose slot values are requested together (SpMV pass)
#ifndef PPPC_CL_PIPE
#define PPPC_CL_PIPE 1
#endif
#ifndef PPPC_CL_EXP
#define PPPC_CL_EXP 0   // timing experiments only (results are wrong): 1 no x traffic, 2 slot values not read, 4 p not gathered
#endif
constexpr int kClExp = PPPC_CL_EXP;
constexpr int kClPipe = PPPC_CL_PIPE; // groups of kClRb rows requested ahead of the one being multiplied (0, 1, 2)
constexpr int kClRpt = PPPC_CL_RPT;   // rows per thread at most (their x entries are registers)
constexpr int kClMaxC = 16;           // CTAs per cluster at most (8 portable)
constexpr int kClNd = 8;              // reduction slots per CTA
// per-row info word: pattern id | kClOwn (per-system values) | push entry + 1 in
// bits 10..13 (kClPushMany: held by more than one other window)
constexpr unsigned kClOwn = 0x100u, kClPushShift = 10u, kClPushMask = 0xfu << kClPushShift,
                   kClPushMany = 0xfu;

struct alignas(16) ClShared {
  int4 pat_cols[kPatMax][kEll / 4];       // pattern dictionary: column entries
  int pat_meta[kPatMax];                  // length | absolute mask << 8
  double red[kClNd][32];
  double cpart[2][kClMaxC][kClNd];
  double tot[kClNd];
  double qh;                              // the hub row's product (owner CTA)
  long long tm[4], tm_c[4];               // PPPC_DEBUG_TIMING: cycles of the SpMV pass, cluster sum, update
                                          // pass, halo wait; stamps (start, after sum, after update, mid-sum)
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
  double* ds;   // Jacobi entries of own rows
  double* qs;   // q of own rows
  unsigned short* info;   // per own row: pattern id | kClOwn | push entry (see kClPushShift)
  ClShared* sh;
  bool timed;          // PPPC_DEBUG_TIMING: thread 0 keeps cycle stamps in shared memory
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

// Sends v (row i of p, owned here) to the CTAs whose windows hold column i;
// code = the row's push field (entry + 1, or kClPushMany: look the targets up).
__device__ __forceinline__ void cl_push_row(const ClCtx& X, int i, double v, unsigned code) {
  const ClShared* sh = X.sh;
  if (code != kClPushMany) {
    cl_st_async(sh->push_base[code - 1] + static_cast<unsigned>(i) * 8u, v, sh->push_mb[code - 1]);
    return;
  }
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

// Sum of 8 slots over the 32 lanes in 4 + 2 + 1 + 1 + 1 exchanges (instead of
// 8 x 5): after every exchange a lane is responsible for half as many slots.  On
// return the lane holds the warp total of slot cl_slot_of(lane); the additions
// form one fixed tree.
__device__ __forceinline__ double cl_butterfly8(const double (&v)[8], int lane) {
  double w4[4], w2[2];
  const bool b4 = lane & 16;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double send = b4 ? v[j] : v[j + 4], keep = b4 ? v[j + 4] : v[j];
    w4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  const bool b3 = lane & 8;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double send = b3 ? w4[j] : w4[j + 2], keep = b3 ? w4[j + 2] : w4[j];
    w2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const bool b2 = lane & 4;
  const double send = b2 ? w2[0] : w2[1], keep = b2 ? w2[1] : w2[0];
  double w = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  w += __shfl_xor_sync(0xffffffffu, w, 2);
  w += __shfl_xor_sync(0xffffffffu, w, 1);
  return w;
}
__device__ __forceinline__ int cl_slot_of(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }
__device__ __forceinline__ int cl_lane_of(int slot) { return (slot & 4 ? 16 : 0) + (slot & 2 ? 8 : 0) + (slot & 1 ? 4 : 0); }

// Fixed-order cluster sum of ND values; every thread of every CTA returns the
// same totals.  HUBFIX (PCG pass, values {p.q, q.z, q.Dq, r.z, r.r}): the hub
// row's product (sh->qh, formed by the owner's last warp during the SpMV pass)
// enters the owner's block sums before they are sent.
template <int ND, bool HUBFIX>
__device__ __forceinline__ void cl_reduce(ClCtx& X, double (&v)[ND]) {
  constexpr int NW = kClThreads / 32;
  static_assert(NW <= 32 && ND <= kClNd, "reduction geometry");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ClShared* sh = X.sh;
  {
    double v8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v8[k] = k < ND ? v[k] : 0.0;
    const double w = cl_butterfly8(v8, lane);
    if ((lane & 3) == 0) sh->red[cl_slot_of(lane)][warp] = w;
  }
  __syncthreads();
  if (X.timed && threadIdx.x == 0) sh->tm_c[3] = clock64();
  if (warp == 0) {
    unsigned long long* mb = &sh->red_mb[X.par];
    if (lane == 0) cl_mbar_expect(mb, static_cast<unsigned>(X.C) * ND * 8u);
    double v8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v8[k] = (k < ND && lane < NW) ? sh->red[k][lane] : 0.0;
    const double w = cl_butterfly8(v8, lane);
    double s[ND];
#pragma unroll
    for (int k = 0; k < ND; ++k) s[k] = __shfl_sync(0xffffffffu, w, cl_lane_of(k));
    if (HUBFIX && X.hub >= 0) {
      const double qh = sh->qh;
      const double dh = *X.hubD;
      s[0] += X.pw[X.hub - X.wlo] * qh;
      s[1] += qh * (dh * X.rs[X.hub - X.r0]);
      s[2] += qh * (dh * qh);
    }
    if (lane < X.C) {
      const unsigned dst = cl_mapa(cl_smem_u32(&sh->cpart[X.par][X.rank][0]), lane);
      const unsigned rmb = cl_mapa(cl_smem_u32(mb), lane);
#pragma unroll
      for (int k = 0; k < ND; ++k) cl_st_async(dst + 8u * k, s[k], rmb);
    }
    cl_mbar_wait(mb, (X.red_phase >> X.par) & 1);
    // rank-order sum: lane t holds CTA t's values, folded by the same fixed tree
#pragma unroll
    for (int k = 0; k < 8; ++k) v8[k] = (k < ND && lane < X.C) ? sh->cpart[X.par][lane][k] : 0.0;
    const double tot = cl_butterfly8(v8, lane);
    if ((lane & 3) == 0) sh->tot[cl_slot_of(lane)] = tot;
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
                                       int step, bool first, double (&t)[4]) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i = X.r0 + threadIdx.x; i < X.r1; i += kClThreads)
    if (i != S.hub) sb_refill_row<NPE>(P, S, X.sh->curves, V, sys, step, first, i, acc);
  if (X.hub >= 0 && threadIdx.x == kClThreads - 1) sb_refill_hub<NPE>(P, S, X.sh->curves, V, sys, step, first, acc);
  if (X.sh->n_push) {
    __syncthreads();  // the hub row's p entry is written by another thread than the one that pushes it
    for (int i = X.r0 + threadIdx.x; i < X.r1; i += kClThreads) {
      const unsigned code = (X.info[i - X.r0] & kClPushMask) >> kClPushShift;
      if (code) cl_push_row(X, i, X.pw[i - X.wlo], code);
    }
  }
  cl_reduce<4, false>(X, acc);
  cl_halo_sync(X);
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = acc[k];
}

// W: slots read per row = the longest row among the rows of <= kEll slots
// (compile-time, so that the slot loops carry no predicates).
template <int NPE, int W>
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
  X.timed = P.dbg != nullptr;
  X.sh = reinterpret_cast<ClShared*>(cl_smem);
  X.pw = reinterpret_cast<double*>(cl_smem + sizeof(ClShared));
  X.rs = X.pw + Gm.win_max;
  X.ds = X.rs + Gm.rows_max;
  X.qs = X.ds + Gm.rows_max;
  X.info = reinterpret_cast<unsigned short*>(X.qs + Gm.rows_max);
  // the hub row's values and window indices (owner CTA), 8-byte aligned after the info words
  double* const hubv = reinterpret_cast<double*>(X.info + ((Gm.rows_max + 3) & ~3));
  int* const hubc = reinterpret_cast<int*>(hubv + Gm.hub_len);
  ClShared* sh = X.sh;
  const int sys = blockIdx.x / Gm.C;
  const int tid = threadIdx.x;
  if (tid < P.ncurves) sh->curves[tid] = P.curves[tid];
  for (int k = tid; k < kPatMax * (kEll / 4); k += kClThreads)
    (&sh->pat_cols[0][0])[k] = __ldg(reinterpret_cast<const int4*>(S.pat_cols) + k);
  for (int k = tid; k < kPatMax; k += kClThreads) sh->pat_meta[k] = __ldg(S.pat_meta + k);
  const int d = P.d;
  const int r0 = X.r0, r1 = X.r1;
  const size_t vb = static_cast<size_t>(sys) * d;
  SbVec V;
  V.u = S.su + vb;
  V.uprev = P.uprev + vb;
  V.D = P.Dinv + vb;
  V.x = P.x + vb;
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
    for (int k = 0; k < 4; ++k) sh->tm[k] = 0;
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
  // per own row: pattern id (the hub row counts as irregular), whether its values
  // are the system's own, whether other windows hold it
  for (int i = r0 + tid; i < r1; i += kClThreads) {
    unsigned v = i == S.hub ? static_cast<unsigned>(kPatIrregular) : __ldg(S.pat_id + i);
    if (!sb_shared_row(P, i)) v |= kClOwn;
    unsigned code = 0;
    for (int e = 0; e < sh->n_push; ++e)
      if (i >= sh->push_lo[e] && i < sh->push_hi[e]) code = code ? kClPushMany : static_cast<unsigned>(e + 1);
    v |= code << kClPushShift;
    X.info[i - r0] = static_cast<unsigned short>(v);
  }
  __syncthreads();
  const int hub_base = S.hub >= 0 ? __ldg(P.rp + S.hub) : 0;
  if (X.hub >= 0)
    for (int s = tid; s < S.hub_len; s += kClThreads) hubc[s] = __ldg(P.ci + hub_base + s) - X.wlo;
  // the Jacobi entries of the CTA's rows after a refill (each thread its own rows)
  // ... and the hub row's slot values (its owner; the last warp multiplies them)
  auto load_jacobi = [&]() {
    for (int i = r0 + tid; i < r1; i += kClThreads)
      X.ds[i - r0] = (X.info[i - r0] & kClOwn) ? V.D[i] : __ldg(P.Dsh + i);
    if (X.hub >= 0) {
      for (int s = tid; s < S.hub_len; s += kClThreads)
        hubv[s] = X.hub_shared ? __ldg(P.Ash + hub_base + s) : V.hA[s];
      __syncthreads();
    }
  };
  // hot-loop views: own rows by local index l = row - r0, p also by column
  const int nloc = r1 - r0;
  const int hubl = X.hub >= 0 ? X.hub - r0 : -1;
  double* __restrict__ const rs = X.rs;
  double* __restrict__ const ds = X.ds;
  double* __restrict__ const qs = X.qs;
  double* const pwo = X.pw + (r0 - X.wlo);
  const double* const pw0 = X.pw - X.wlo;
  const unsigned short* __restrict__ const info = X.info;
  double* __restrict__ const xg = V.x + r0;   // x of own rows (global)
  const double* __restrict__ const Aown = V.A + r0;
  const double* __restrict__ const Ash = S.AshT + r0;
  int code = PS_OK, last_nit = 0, max_nit = 0, max_pit = 0;
  double t_fail = 0.0, res_fail = 0.0;
  long long newton_total = 0, pcg_total = 0;
  double t[4];
  for (int step = 0; step < P.steps && code == PS_OK; ++step) {
    const double t_now = P.t_next[static_cast<size_t>(step) * P.count + sys];
    cl_refill<NPE>(X, P, S, V, sys, step, true, t);
    load_jacobi();
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
          // and r.z, r.r of the residual as the last update left it.  Software
          // pipeline: the slot values of the next kClRb rows are requested before
          // the current kClRb rows are multiplied (all W slots of a row: pads hold
          // 0 and point at the row itself; a row index past the range is clamped).
          double a5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
          if (X.timed && tid == 0) sh->tm_c[0] = clock64();
          double avA[kClRb][W], avB[kClRb][W], avC[kClRb][W];
          unsigned infA[kClRb], infB[kClRb], infC[kClRb];
          auto load_rows = [&](int l0, double (&av)[kClRb][W], unsigned (&inf)[kClRb]) {
#pragma unroll
            for (int u = 0; u < kClRb; ++u) {
              const int l = min(l0 + u * kClThreads, nloc - 1);
              inf[u] = info[l];
              const double* ap = ((inf[u] & kClOwn) ? Aown : Ash) + l;
#pragma unroll
              for (int s = 0; s < W; ++s) av[u][s] = (kClExp & 2) ? 1.0 + s : ap[static_cast<size_t>(s) * d];
            }
          };
          // Straight-line main path for all kClRb rows (so that their instructions
          // interleave): every row is treated as a dictionary row without absolute
          // entries, with a clamped index; the rare other rows are recomputed
          // afterwards, and rows past the range / the hub row are masked out.
          auto mult_rows = [&](int l0, const double (&av)[kClRb][W], const unsigned (&inf)[kClRb]) {
            double qv[kClRb], ri[kClRb], dvi[kClRb], pi[kClRb];
            bool special[kClRb];
#pragma unroll
            for (int u = 0; u < kClRb; ++u) {
              const int l = min(l0 + u * kClThreads, nloc - 1);
              const unsigned pid = inf[u] & 0xffu;
              const int4 o0 = sh->pat_cols[pid][0], o1 = sh->pat_cols[pid][1];
              const int off[kEll] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
              special[u] = pid == static_cast<unsigned>(kPatIrregular) || (sh->pat_meta[pid] >> 8) != 0;
              const double* pwi = pwo + l;   // p at this row's own column
              ri[u] = rs[l];
              dvi[u] = ds[l];
              pi[u] = pwi[0];
              // two partial sums (even / odd slots) shorten the dependent chain
              double qe = 0.0, qo = 0.0;
#pragma unroll
              for (int s = 0; s < W; s += 2) qe += av[u][s] * ((kClExp & 4) ? pi[u] + off[s] : pwi[off[s]]);
#pragma unroll
              for (int s = 1; s < W; s += 2) qo += av[u][s] * ((kClExp & 4) ? pi[u] + off[s] : pwi[off[s]]);
              qv[u] = qe + qo;
            }
#pragma unroll
            for (int u = 0; u < kClRb; ++u) {
              if (!special[u]) continue;
              const int l = min(l0 + u * kClThreads, nloc - 1);
              const unsigned pid = inf[u] & 0xffu;
              double q = 0.0;
              if (pid != static_cast<unsigned>(kPatIrregular)) {
                // dictionary row with entries kept absolute (the hub's column)
                const int4 o0 = sh->pat_cols[pid][0], o1 = sh->pat_cols[pid][1];
                const int off[kEll] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
                const int absm = sh->pat_meta[pid] >> 8;
#pragma unroll
                for (int s = 0; s < W; ++s) q += av[u][s] * (((absm >> s) & 1) ? pw0[S.hub] : pwo[l + off[s]]);
              } else {
                // outside the dictionary: padded columns from memory
                const int* cp = S.ciT + (r0 + l);
#pragma unroll
                for (int s = 0; s < W; ++s) q += av[u][s] * pw0[__ldg(cp + static_cast<size_t>(s) * d)];
              }
              qv[u] = q;
            }
#pragma unroll
            for (int u = 0; u < kClRb; ++u) {
              const int l = l0 + u * kClThreads;
              const bool in = l < nloc;
              const bool mul = in && l != hubl;   // the hub row's product comes from the last warp
              const double r = in ? ri[u] : 0.0, q = mul ? qv[u] : 0.0;
              const double zi = dvi[u] * r;
              if (mul) qs[l] = q;
              a5[0] += pi[u] * q;
              a5[1] += q * zi;
              a5[2] += q * (dvi[u] * q);
              a5[3] += r * zi;
              a5[4] += r * r;
            }
          };
          constexpr int kStride = kClThreads * kClRb;
          if (kClPipe == 0) {
            // no pipeline: the rows' values are requested, then multiplied
            (void)avB, (void)avC, (void)infB, (void)infC;
#pragma unroll 1
            for (int l0 = tid; l0 < nloc; l0 += kStride) {
              load_rows(l0, avA, infA);
              mult_rows(l0, avA, infA);
            }
          } else if (kClPipe == 1) {
            // one group of rows ahead (two register buffers)
            (void)avC, (void)infC;
            load_rows(tid, avA, infA);
#pragma unroll 1
            for (int l0 = tid; l0 < nloc; l0 += 2 * kStride) {
              load_rows(l0 + kStride, avB, infB);
              mult_rows(l0, avA, infA);
              load_rows(l0 + 2 * kStride, avA, infA);
              mult_rows(l0 + kStride, avB, infB);
            }
          } else {
            // two groups of rows ahead (three register buffers)
            load_rows(tid, avA, infA);
            load_rows(tid + kStride, avB, infB);
#pragma unroll 1
            for (int l0 = tid; l0 < nloc; l0 += 3 * kStride) {
              load_rows(l0 + 2 * kStride, avC, infC);
              mult_rows(l0, avA, infA);
              load_rows(l0 + 3 * kStride, avA, infA);
              mult_rows(l0 + kStride, avB, infB);
              load_rows(l0 + 4 * kStride, avB, infB);
              mult_rows(l0 + 2 * kStride, avC, infC);
            }
          }
          if (X.hub >= 0 && (tid >> 5) == kClThreads / 32 - 1) {
            // the hub row's product by the last warp (its columns lie inside the
            // owner's window); the cluster sum folds it in
            double part = 0.0;
            for (int s = tid & 31; s < S.hub_len; s += 32) part += hubv[s] * X.pw[hubc[s]];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if ((tid & 31) == 0) sh->qh = part;
          }
          cl_reduce<5, true>(X, a5);
          if (X.timed && tid == 0) sh->tm_c[1] = clock64();
          const double t0v = a5[0], t1v = a5[1], t2v = a5[2];
          if (pit > 0) {
            // the state after update `pit`
            const double rr = a5[4];
            rho = a5[3];
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
          // rows in batches of four; x (global, L2-resident) of the next batch is
          // requested before the current batch is updated
          {
            constexpr int kB = 4;
            double xa[kB], xn[kB];
#pragma unroll
            for (int u = 0; u < kB; ++u)
              xa[u] = (first_it || (kClExp & 1)) ? 0.0 : xg[min(tid + u * kClThreads, nloc - 1)];
#pragma unroll 1
            for (int l0 = tid; l0 < nloc; l0 += kB * kClThreads) {
#pragma unroll
              for (int u = 0; u < kB; ++u)
                xn[u] = (first_it || (kClExp & 1)) ? 0.0 : xg[min(l0 + (kB + u) * kClThreads, nloc - 1)];
              double pv[kB], qq[kB], rv[kB], dv[kB];
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                const int l = min(l0 + u * kClThreads, nloc - 1);
                pv[u] = pwo[l];
                qq[u] = l == hubl ? qh : qs[l];
                rv[u] = rs[l];
                dv[u] = ds[l];
              }
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                const int l = l0 + u * kClThreads;
                const double rn = rv[u] - alpha * qq[u];
                const double pn = dv[u] * rn + beta * pv[u];
                if (l < nloc) {
                  if (!(kClExp & 1) || l == 0) xg[l] = xa[u] + alpha * pv[u];
                  rs[l] = rn;
                  pwo[l] = pn;
                  const unsigned code = (info[l] & kClPushMask) >> kClPushShift;
                  if (code) cl_push_row(X, r0 + l, pn, code);
                }
              }
#pragma unroll
              for (int u = 0; u < kB; ++u) xa[u] = xn[u];
            }
          }
          pit += 1;
          if (X.timed && tid == 0) sh->tm_c[2] = clock64();
          cl_halo_sync(X);
          if (X.timed && tid == 0) {
            sh->tm[0] += sh->tm_c[3] - sh->tm_c[0];
            sh->tm[1] += sh->tm_c[1] - sh->tm_c[3];
            sh->tm[2] += sh->tm_c[2] - sh->tm_c[1];
            sh->tm[3] += clock64() - sh->tm_c[2];
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
        cl_refill<NPE>(X, P, S, V, sys, step, false, t);
        load_jacobi();
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
  if (X.timed && tid == 0) {
    unsigned long long* o = P.dbg + (static_cast<size_t>(sys) * X.C + X.rank) * 8;
    for (int k = 0; k < 4; ++k) o[k] = static_cast<unsigned long long>(sh->tm[k]);
    o[4] = static_cast<unsigned long long>(pcg_total);
  }
  // no CTA may exit while others can still write into its shared memory
  cl.sync();
}
