// Multiharmonic coarse solve on B200 (sm_100a), fp64.
//
//   rhs_row = Q (F_sub - G_sub) + f(T_sub)           assemble_rhs, proj/src/spectral.cpp:134-150
//   rhs_hat = unitary DFT across rows (per DOF)      dft_bins,     proj/src/spectral.cpp:32-63
//   Lambda_p x_p = rhs_hat_p  for every solved bin    MultiharmonicCyclicSolver::solve, :257-279
//   U = realify(IDFT(mirror(x)))                      :72-84, :270-278
//   jump = max_n |U_n - U_old_n| / max(1, max_n |U_n|)   jump_norm, proj/src/engine.cpp:54-64
//
// The per-bin complex sparse LU of the reference is replaced by a batched
// Jacobi-preconditioned COCG (complex-symmetric CG, unconjugated bilinear form)
// running as one persistent kernel over all bins: lane = bin, the block matrix
// Lambda_p = X + s_p Y is never materialised — X = Q and Y = C (= M/dT) are read
// once per slot for all bins of a warp and shifted on the fly.
#include "group_sync.cuh"
#include "pppc_internal.h"

#include <cmath>
#include <complex>
#include <cstring>

namespace pppc {

namespace {

constexpr int kCND = 6;  // complex dots: 3 complex values per reduction at most
constexpr double kPi = 3.14159265358979323846;
constexpr double kImagResidualTol = 1e-8;  // proj/src/spectral.cpp:21

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }

struct CocgParams {
  int d, H;   // DOFs, solved bins (interleave stride)
  int G, C, L, Lp, R;
  const int* warp_row_begin;
  int n_long;
  const int* long_rows;
  const int* long_owner;
  const int* rp;
  const int* ci;
  const int* diag;
  const double* X;  // Q (or K)
  const double* Y;  // C = M/dT (or M)
  const int4* rowrec;   // [d][3] row records (pppc_internal.h): {base, len, kind, 0}, padded columns
  const double2* XYE;   // [d][kEll] padded (X, Y) slot values of rows with <= kEll slots
  const double2* dXY;   // [d] (X, Y) at the diagonal slot
  const double2* shift;  // [H] Lambda_b = X + shift_b * Y
  const double2* b;      // rhs_hat [d][H]
  double2* x;
  double2* r;
  double2* p;
  double2* q;
  double tol;
  int max_iter;
  int warm;        // 1: x holds the start value (the previous solve's solution)
  unsigned long long* sync;
  double* partials;
  int* abort_flag;
  int* code;       // [H]
  int* iters;      // [H]
  int64_t* lockstep;
};

struct BinLane {
  bool alive, act;
  int code, it;
  double2 rho, alpha, beta;
  double stop;
};

__device__ __forceinline__ double2 lam_diag(const CocgParams& P, int i, double2 s) {
  const double2 xy = __ldg(P.dXY + i);
  return make_double2(xy.x + s.x * xy.y, s.y * xy.y);
}

__device__ __forceinline__ double2 jacobi(double2 xy, double2 s) {
  return cdiv(make_double2(1.0, 0.0), make_double2(xy.x + s.x * xy.y, s.y * xy.y));
}

// Phase A for one row of <= kEll slots: every load of the row (padded slot
// values, the eight gathered p entries, own p, r and the diagonal) is issued
// before the first FMA; the row record came one row earlier.  Pad slots carry
// (X, Y) = 0 and point at the row itself.
__device__ __forceinline__ void cocg_row_a(const CocgParams& P, int i, const int4& c03, const int4& c47, size_t H,
                                           int h, double2 s_b, double (&acc)[kCND]) {
  const int c[kEll] = {c03.x, c03.y, c03.z, c03.w, c47.x, c47.y, c47.z, c47.w};
  double2 xy[kEll], pv[kEll];
  const double2* xr = P.XYE + static_cast<size_t>(i) * kEll;
#pragma unroll
  for (int k = 0; k < kEll; ++k) xy[k] = __ldg(xr + k);
#pragma unroll
  for (int k = 0; k < kEll; ++k) pv[k] = P.p[static_cast<size_t>(c[k]) * H + h];
  const size_t iv = static_cast<size_t>(i) * H + h;
  const double2 pi = P.p[iv], ri = P.r[iv];
  const double2 dxy = __ldg(P.dXY + i);
  double2 qv = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < kEll; ++k) qv = cadd(qv, cmul(make_double2(xy[k].x + s_b.x * xy[k].y, s_b.y * xy[k].y), pv[k]));
  P.q[iv] = qv;
  const double2 dinv = jacobi(dxy, s_b);
  const double2 zi = cmul(dinv, ri);
  const double2 pq = cmul(pi, qv), qz = cmul(qv, zi), qdq = cmul(qv, cmul(dinv, qv));
  acc[0] += pq.x;
  acc[1] += pq.y;
  acc[2] += qz.x;
  acc[3] += qz.y;
  acc[4] += qdq.x;
  acc[5] += qdq.y;
}

// Phase A of one COCG iteration for this thread's rows: q = Lambda p and the
// partials p.q, q.z, q.Dq.  Called by every thread of the block (the long-row
// path uses block barriers); `act`: this lane's bin is iterating.
__device__ __forceinline__ void cocg_phase_a(const CocgParams& P, bool act, int c, int row_begin, int row_end,
                                             size_t H, int h, double2 s_b, double2 (*lpart)[32],
                                             double (&acc)[kCND]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / P.Lp;
  // long rows (the polar hub): slots split across the owning block's warps
  for (int j = 0; j < P.n_long; ++j) {
    if (__ldg(P.long_owner + j) != c) continue;
    const int i = __ldg(P.long_rows + j);
    const int base = __ldg(P.rp + i), end = __ldg(P.rp + i + 1);
    double2 part = make_double2(0.0, 0.0);
    if (act)
      for (int k = base + warp; k < end; k += kWarps) {
        const int cj = __ldg(P.ci + k);
        const double xk = __ldg(P.X + k), yk = __ldg(P.Y + k);
        part = cadd(part, cmul(make_double2(xk + s_b.x * yk, s_b.y * yk), P.p[static_cast<size_t>(cj) * H + h]));
      }
    lpart[warp][lane] = part;
    __syncthreads();
    if (warp == 0 && act) {
      double2 qv = make_double2(0.0, 0.0);
      for (int w = 0; w < kWarps; ++w) qv = cadd(qv, lpart[w][lane]);
      const size_t iv = static_cast<size_t>(i) * H + h;
      P.q[iv] = qv;
      const double2 dinv = cdiv(make_double2(1.0, 0.0), lam_diag(P, i, s_b));
      const double2 pi = P.p[iv], ri = P.r[iv];
      const double2 zi = cmul(dinv, ri);
      const double2 pq = cmul(pi, qv), qz = cmul(qv, zi), qdq = cmul(qv, cmul(dinv, qv));
      acc[0] += pq.x;
      acc[1] += pq.y;
      acc[2] += qz.x;
      acc[3] += qz.y;
      acc[4] += qdq.x;
      acc[5] += qdq.y;
    }
    __syncthreads();
  }
  if (act && row_begin + sub < row_end) {
    // row records two rows ahead of their use; the next row's gathered p
    // entries, own p / r and slot values are requested into L1 one row ahead
    // (no registers held), so the row's loads mostly hit L1
    int i = row_begin + sub;
    int4 h0 = __ldg(P.rowrec + kRecInts4 * i), c03 = __ldg(P.rowrec + kRecInts4 * i + 1),
         c47 = __ldg(P.rowrec + kRecInts4 * i + 2);
    int4 h1 = h0, d03 = c03, d47 = c47;
    if (i + P.R < row_end) {
      h1 = __ldg(P.rowrec + kRecInts4 * (i + P.R));
      d03 = __ldg(P.rowrec + kRecInts4 * (i + P.R) + 1);
      d47 = __ldg(P.rowrec + kRecInts4 * (i + P.R) + 2);
    }
    for (;;) {
      const int i1 = i + P.R, i2 = i + 2 * P.R;
      const bool more = i1 < row_end;
      int4 h2 = h1, e03 = d03, e47 = d47;
      if (i2 < row_end) {
        h2 = __ldg(P.rowrec + kRecInts4 * i2);
        e03 = __ldg(P.rowrec + kRecInts4 * i2 + 1);
        e47 = __ldg(P.rowrec + kRecInts4 * i2 + 2);
      }
      if (more && h1.y <= kEll) {
        const int cn[kEll] = {d03.x, d03.y, d03.z, d03.w, d47.x, d47.y, d47.z, d47.w};
#pragma unroll
        for (int k = 0; k < kEll; ++k)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(P.p + static_cast<size_t>(cn[k]) * H + h));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.r + static_cast<size_t>(i1) * H + h));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(P.XYE + static_cast<size_t>(i1) * kEll));
      }
      const int len = h0.y;
      if (len <= kEll) {
        cocg_row_a(P, i, c03, c47, H, h, s_b, acc);
      } else if (len <= kLongRow) {
        double2 qv = make_double2(0.0, 0.0);
        for (int k = h0.x; k < h0.x + len; ++k) {
          const int j = __ldg(P.ci + k);
          const double xk = __ldg(P.X + k), yk = __ldg(P.Y + k);
          const double2 lam = make_double2(xk + s_b.x * yk, s_b.y * yk);
          qv = cadd(qv, cmul(lam, P.p[static_cast<size_t>(j) * H + h]));
        }
        const size_t iv = static_cast<size_t>(i) * H + h;
        P.q[iv] = qv;
        const double2 dinv = cdiv(make_double2(1.0, 0.0), lam_diag(P, i, s_b));
        const double2 pi = P.p[iv], ri = P.r[iv];
        const double2 zi = cmul(dinv, ri);
        const double2 pq = cmul(pi, qv), qz = cmul(qv, zi), qdq = cmul(qv, cmul(dinv, qv));
        acc[0] += pq.x;
        acc[1] += pq.y;
        acc[2] += qz.x;
        acc[3] += qz.y;
        acc[4] += qdq.x;
        acc[5] += qdq.y;
      }
      if (!more) break;
      i = i1;
      h0 = h1;
      c03 = d03;
      c47 = d47;
      h1 = h2;
      d03 = e03;
      d47 = e47;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) cocg_kernel(const CocgParams P) {
  __shared__ SyncShared<kCND> sh;
  __shared__ double2 lpart[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = blockIdx.x / P.C, c = blockIdx.x % P.C;
  const int sub = lane / P.Lp, sl = lane % P.Lp;
  const int h = g * P.L + sl;
  const bool valid = (sl < P.L) && (h < P.H);
  sync_state_init(sh);
  __syncthreads();
  SyncCtx X;
  X.sync = P.sync;
  X.partials = P.partials;
  X.abort_flag = P.abort_flag;
  X.G = P.G;
  X.C = P.C;
  X.Lp = P.Lp;
  X.L = P.L;
  const int row_begin = P.warp_row_begin[c * kWarps + warp];
  const int row_end = P.warp_row_begin[c * kWarps + warp + 1];
  const size_t H = static_cast<size_t>(P.H);
  const double2 s_b = valid ? P.shift[h] : make_double2(0.0, 0.0);
  double acc[kCND] = {0, 0, 0, 0, 0, 0};

  BinLane s;
  s.alive = valid;
  s.act = false;
  s.code = PS_OK;
  s.it = 0;
  s.rho = s.alpha = s.beta = make_double2(0.0, 0.0);
  s.stop = 0.0;
  long long lockstep = 0;

  if (P.warm) {
    // warm start from x (the previous solve's solution): q = Lambda x with the
    // phase-A rows reading x in place of p; each row's q is read back below by
    // the thread of the same block that owns the row
    CocgParams Pw = P;
    Pw.p = P.x;
    cocg_phase_a(Pw, s.alive, c, row_begin, row_end, H, h, s_b, lpart, acc);
#pragma unroll
    for (int k = 0; k < kCND; ++k) acc[k] = 0.0;
    __syncthreads();
  }
  // init: r = b - Lambda x (x = 0 cold: r = b), z = D r, p = z, rho = r.z,
  // bb = |b|^2 (the stop stays relative to b), rr = |r|^2
  if (s.alive)
    for (int i = row_begin + sub; i < row_end; i += P.R) {
      const size_t iv = static_cast<size_t>(i) * H + h;
      const double2 bv = P.b[iv];
      const double2 rv = P.warm ? csub(bv, P.q[iv]) : bv;
      const double2 z = cdiv(make_double2(1.0, 0.0), lam_diag(P, i, s_b));
      const double2 zr = cmul(z, rv);
      if (!P.warm) P.x[iv] = make_double2(0.0, 0.0);
      P.r[iv] = rv;
      P.p[iv] = zr;
      const double2 rz = cmul(rv, zr);
      acc[0] += rz.x;
      acc[1] += rz.y;
      acc[2] += bv.x * bv.x + bv.y * bv.y;
      acc[3] += rv.x * rv.x + rv.y * rv.y;
    }
  if (!group_sync_reduce<kCND, 4>(X, sh, acc, g, c)) return;
  if (s.alive) {
    s.rho = make_double2(sh.tot[0][sl], sh.tot[1][sl]);
    const double bb = sh.tot[2][sl], rr = sh.tot[3][sl];
    s.stop = (P.tol * P.tol) * bb;
    // cold: at least one iteration unless b = 0; warm: none if x already meets the stop
    s.act = P.warm ? (bb != 0.0 && !(rr <= s.stop)) : bb != 0.0;
    if (P.warm && bb == 0.0)
      for (int i = row_begin + sub; i < row_end; i += P.R) P.x[static_cast<size_t>(i) * H + h] = make_double2(0.0, 0.0);
  }

  while (__syncthreads_or(s.act ? 1 : 0)) {
    cocg_phase_a(P, s.act, c, row_begin, row_end, H, h, s_b, lpart, acc);
    if (!group_sync_reduce<kCND, 6>(X, sh, acc, g, c)) return;
    ++lockstep;
    if (s.act) {
      const double2 mu = make_double2(sh.tot[0][sl], sh.tot[1][sl]);
      const double2 qz = make_double2(sh.tot[2][sl], sh.tot[3][sl]);
      const double2 qdq = make_double2(sh.tot[4][sl], sh.tot[5][sl]);
      if (!isfinite(mu.x) || !isfinite(mu.y) || (mu.x == 0.0 && mu.y == 0.0)) {
        s.alive = s.act = false;
        s.code = PS_ERR_SINGULAR_BLOCK;
      } else {
        s.alpha = cdiv(s.rho, mu);
        // rho_est = rho - 2 alpha qz + alpha^2 qdq
        const double2 t1 = cmul(cscale(2.0, s.alpha), qz);
        const double2 t2 = cmul(cmul(s.alpha, s.alpha), qdq);
        const double2 rho_est = cadd(csub(s.rho, t1), t2);
        s.beta = cdiv(rho_est, s.rho);
      }
    }
    if (s.act)
      // rows in pairs whose loads are issued together
      for (int i0 = row_begin + sub; i0 < row_end; i0 += 2 * P.R) {
        double2 xv[2], pv[2], qv[2], rv[2], dxy[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = i0 + u * P.R < row_end ? i0 + u * P.R : i0;
          const size_t iv = static_cast<size_t>(i) * H + h;
          dxy[u] = __ldg(P.dXY + i);
          xv[u] = P.x[iv];
          pv[u] = P.p[iv];
          qv[u] = P.q[iv];
          rv[u] = P.r[iv];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = i0 + u * P.R;
          if (i >= row_end) break;
          const size_t iv = static_cast<size_t>(i) * H + h;
          const double2 dinv = jacobi(dxy[u], s_b);
          P.x[iv] = cadd(xv[u], cmul(s.alpha, pv[u]));
          const double2 ri = csub(rv[u], cmul(s.alpha, qv[u]));
          const double2 zi = cmul(dinv, ri);
          P.r[iv] = ri;
          P.p[iv] = cadd(zi, cmul(s.beta, pv[u]));
          const double2 rz = cmul(ri, zi);
          acc[0] += ri.x * ri.x + ri.y * ri.y;
          acc[1] += rz.x;
          acc[2] += rz.y;
        }
      }
    if (!group_sync_reduce<kCND, 3>(X, sh, acc, g, c)) return;
    if (s.act) {
      const double rr = sh.tot[0][sl];
      s.rho = make_double2(sh.tot[1][sl], sh.tot[2][sl]);
      s.it += 1;
      if (rr <= s.stop) {
        s.act = false;
      } else if (!isfinite(rr)) {
        s.alive = s.act = false;
        s.code = PS_ERR_SINGULAR_BLOCK;
      } else if (s.it >= P.max_iter) {
        s.alive = s.act = false;
        s.code = PS_ERR_COCG_MAXITER;
      }
    }
  }
  if (c == 0 && warp == 0 && sub == 0 && valid) {
    P.code[h] = s.code;
    P.iters[h] = s.it;
  }
  if (c == 0 && threadIdx.x == 0) P.lockstep[g] = lockstep;
}

// rhs[i][row] = sum_k Q_k (F[c_k][sub-1] - G[c_k][sub-1]) + f_i(T_sub)
__global__ void assemble_rhs_kernel(int d, int N, const int* __restrict__ rp, const int* __restrict__ ci,
                                    const double* __restrict__ Q, const double* F, const double* Gv,
                                    const double* __restrict__ pat, const double* __restrict__ coef, int nterms,
                                    double* rhs) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(d) * N) return;
  const int row = static_cast<int>(t % N), i = static_cast<int>(t / N);
  const int sub = row == 0 ? N : row;
  double acc = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const size_t j = static_cast<size_t>(ci[k]) * N + (sub - 1);
    acc += Q[k] * (F[j] - Gv[j]);
  }
  double f = 0.0;
  for (int k = 0; k < nterms; ++k) f += coef[static_cast<size_t>(row) * nterms + k] * pat[static_cast<size_t>(k) * d + i];
  rhs[t] = acc + f;
}

// Spectral tiles: a block stages kDftRows consecutive DOFs' samples (or
// spectra) and the twiddle table in shared memory with coalesced loads, then
// every thread owns output slots of the tile.  Blocks stride over tiles.
constexpr int kDftRows = 8;

// rhs_hat[i][h] = N^{-1/2} sum_n rhs[i][n] exp(-2 pi i bin_h n / N)
// (proj/src/spectral.cpp:32-63; the same n order and incremental twiddle index
// as a per-DOF loop).  Thread slot = (row of the tile, bin): consecutive
// threads write consecutive out entries.
__global__ void dft_forward_kernel(int d, int N, int H, const int* __restrict__ bins, const double2* __restrict__ tw,
                                   const double* __restrict__ rhs, double2* __restrict__ out) {
  extern __shared__ double2 dsm[];
  double2* stw = dsm;                                              // [N]
  double* srow = reinterpret_cast<double*>(dsm + N);               // [kDftRows][N]
  int* sbin = reinterpret_cast<int*>(srow + kDftRows * N);         // [H]
  for (int k = threadIdx.x; k < N; k += blockDim.x) stw[k] = tw[k];
  for (int k = threadIdx.x; k < H; k += blockDim.x) sbin[k] = bins[k];
  const double scale = 1.0 / sqrt(static_cast<double>(N));
  const int tiles = (d + kDftRows - 1) / kDftRows;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int i0 = tile * kDftRows;
    const int rows = min(kDftRows, d - i0);
    __syncthreads();
    const double* src = rhs + static_cast<size_t>(i0) * N;
    for (int k = threadIdx.x; k < rows * N; k += blockDim.x) srow[k] = src[k];
    __syncthreads();
    for (int slot = threadIdx.x; slot < rows * H; slot += blockDim.x) {
      const int r = slot / H, hh = slot - r * H;
      const int b = sbin[hh];
      const double* row = srow + r * N;
      double ar = 0.0, ai = 0.0;
      int idx = 0;
      for (int n = 0; n < N; ++n) {
        const double v = row[n];
        const double2 w = stw[idx];
        ar += v * w.x;
        ai += v * w.y;
        idx += b;
        if (idx >= N) idx -= N;
      }
      out[static_cast<size_t>(i0) * H + slot] = make_double2(scale * ar, scale * ai);
    }
  }
}

// U_new[i][n] = N^{-1/2} sum over the (mirrored) spectrum, realified
// (proj/src/spectral.cpp:72-84,270-278); fused with the jump partials
// (proj/src/engine.cpp:54-64: per-n sums of |U_new - U_old|^2 and |U_new|^2)
// and the max |re| / max |im| of the realify check.  blockDim = k * N: thread t
// owns sample n = t mod N for rows t / N, t / N + k, ... of every tile it
// visits, so its partial sums run in a fixed order; part[block][2][N].
__global__ void idft_jump_kernel(int d, int N, int H, const int* __restrict__ bins, const double2* __restrict__ tw,
                                 int conj, const double2* __restrict__ xhat, double* U, const double* U_old,
                                 double* part, double* maxre, double* maxim) {
  // U and U_old may alias (in-place PP-PC correction): no __restrict__ on them
  extern __shared__ double2 ism[];
  double2* stw = ism;                                         // [N]
  double2* sx = ism + N;                                      // [kDftRows][H]
  double* sred = reinterpret_cast<double*>(sx + kDftRows * H);  // [blockDim] x 2
  int* sbin = reinterpret_cast<int*>(sred + 2 * blockDim.x);  // [H]
  for (int k = threadIdx.x; k < N; k += blockDim.x) stw[k] = tw[k];
  for (int k = threadIdx.x; k < H; k += blockDim.x) sbin[k] = bins[k];
  const int n = threadIdx.x % N, r0 = threadIdx.x / N, kr = blockDim.x / N;
  const double scale = 1.0 / sqrt(static_cast<double>(N));
  double dd = 0.0, nn = 0.0, mre = 0.0, mim = 0.0;
  const int tiles = (d + kDftRows - 1) / kDftRows;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int i0 = tile * kDftRows;
    const int rows = min(kDftRows, d - i0);
    __syncthreads();
    const double2* src = xhat + static_cast<size_t>(i0) * H;
    for (int k = threadIdx.x; k < rows * H; k += blockDim.x) sx[k] = src[k];
    __syncthreads();
    for (int r = r0; r < rows; r += kr) {
      const double2* xr = sx + r * H;
      double vr = 0.0, vi = 0.0;
      for (int hh = 0; hh < H; ++hh) {
        const int b = sbin[hh];
        const double2 xv = xr[hh];
        const double2 w = stw[(b * n) % N];  // exp(-2 pi i b n/N), b n < 2^20; inverse uses conj
        const double cr = xv.x * w.x + xv.y * w.y;
        const double cim = xv.y * w.x - xv.x * w.y;
        if (conj && b != 0 && 2 * b != N) {
          vr += 2.0 * cr;
        } else {
          vr += cr;
          vi += cim;
        }
      }
      vr *= scale;
      vi *= scale;
      mre = fmax(mre, fabs(vr));
      mim = fmax(mim, fabs(vi));
      const size_t iv = static_cast<size_t>(i0 + r) * N + n;
      if (U_old) {
        const double df = vr - U_old[iv];
        dd += df * df;
      }
      nn += vr * vr;
      U[iv] = vr;
    }
  }
  // per-n partials: the kr threads of sample n combine in row order
  __syncthreads();
  sred[threadIdx.x] = dd;
  sred[blockDim.x + threadIdx.x] = nn;
  __syncthreads();
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    double a = 0.0, b2 = 0.0;
    for (int k = 0; k < kr; ++k) {
      a += sred[k * N + m];
      b2 += sred[blockDim.x + k * N + m];
    }
    part[(static_cast<size_t>(blockIdx.x) * 2 + 0) * N + m] = a;
    part[(static_cast<size_t>(blockIdx.x) * 2 + 1) * N + m] = b2;
  }
  __syncthreads();
  sred[threadIdx.x] = mre;
  sred[blockDim.x + threadIdx.x] = mim;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b2 = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x); ++k) {
      a = fmax(a, sred[k]);
      b2 = fmax(b2, sred[blockDim.x + k]);
    }
    maxre[blockIdx.x] = a;
    maxim[blockIdx.x] = b2;
  }
}

// out[0] = jump, out[1] = max_n |dU_n|, out[2] = max_n |U_n|, out[3] = max|re|, out[4] = max|im|
// One block of 1024 threads: thread (n, j) sums the block partials j, j + 4,
// ... of sample n (eight loads in flight), the four sub-sums combine in order.
__global__ void jump_finalize_kernel(int N, int nblocks, int nmax, const double* part, const double* maxre,
                                     const double* maxim, double* out) {
  constexpr int kSub = 4;
  __shared__ double sa[1024], sb[1024], sd[1024], sn[1024], sr[1024], si[1024];
  const int j = threadIdx.x % kSub, t = threadIdx.x / kSub, nt = blockDim.x / kSub;
  double bd = 0.0, bn = 0.0;
  for (int n0 = 0; n0 < N; n0 += nt) {
    const int n = n0 + t;
    double a = 0.0, b = 0.0;
    if (n < N)
      for (int k0 = j; k0 < nblocks; k0 += 8 * kSub) {
        double va[8], vb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = k0 + u * kSub;
          va[u] = k < nblocks ? part[(static_cast<size_t>(k) * 2 + 0) * N + n] : 0.0;
          vb[u] = k < nblocks ? part[(static_cast<size_t>(k) * 2 + 1) * N + n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a += va[u];
          b += vb[u];
        }
      }
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    if (j == 0 && n < N) {
      double A = 0.0, B = 0.0;
      for (int q = 0; q < kSub; ++q) {
        A += sa[threadIdx.x + q];
        B += sb[threadIdx.x + q];
      }
      bd = fmax(bd, sqrt(A));
      bn = fmax(bn, sqrt(B));
    }
    __syncthreads();
  }
  double mr = 0.0, mi = 0.0;
  for (int k = threadIdx.x; k < nmax; k += blockDim.x) {
    mr = fmax(mr, maxre[k]);
    mi = fmax(mi, maxim[k]);
  }
  sd[threadIdx.x] = bd;
  sn[threadIdx.x] = bn;
  sr[threadIdx.x] = mr;
  si[threadIdx.x] = mi;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) {
      sd[threadIdx.x] = fmax(sd[threadIdx.x], sd[threadIdx.x + w]);
      sn[threadIdx.x] = fmax(sn[threadIdx.x], sn[threadIdx.x + w]);
      sr[threadIdx.x] = fmax(sr[threadIdx.x], sr[threadIdx.x + w]);
      si[threadIdx.x] = fmax(si[threadIdx.x], si[threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sd[0] / fmax(1.0, sn[0]);
    out[1] = sd[0];
    out[2] = sn[0];
    out[3] = sr[0];
    out[4] = si[0];
  }
}

// generic complex DFT for the standalone forward/inverse entry points:
// out[b][j] = N^{-1/2} sum_n in[n][j] w^{+-bn}, in/out [N][d] complex
__global__ void dft_generic_kernel(int N, int d, const double2* __restrict__ tw, int inverse, const double2* in,
                                   double2* out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(N) * d) return;
  const int j = static_cast<int>(t % d), b = static_cast<int>(t / d);
  double ar = 0.0, ai = 0.0;
  for (int n = 0; n < N; ++n) {
    double2 w = tw[(static_cast<int64_t>(b) * n) % N];
    if (inverse) w.y = -w.y;
    const double2 v = in[static_cast<size_t>(n) * d + j];
    ar += v.x * w.x - v.y * w.y;
    ai += v.x * w.y + v.y * w.x;
  }
  const double scale = 1.0 / sqrt(static_cast<double>(N));
  out[t] = make_double2(scale * ar, scale * ai);
}

__global__ void strided_jump_kernel(int count, int d, int stride, const double* cur, const double* prev,
                                    double* part) {
  // one block per system n: part[n][0] = |cur_n - prev_n|^2, part[n][1] = |cur_n|^2
  __shared__ double sa[256], sb[256];
  const int n = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const size_t iv = static_cast<size_t>(i) * stride + n;
    const double c = cur[iv], df = c - prev[iv];
    a += df * df;
    b += c * c;
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sb[threadIdx.x] += sb[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * n] = sa[0];
    part[2 * n + 1] = sb[0];
  }
}

std::vector<double2> twiddles(int N) {
  std::vector<double2> tw(N);
  for (int k = 0; k < N; ++k) {
    const double ang = 2.0 * kPi * k / N;
    tw[k] = make_double2(std::cos(ang), -std::sin(ang));
  }
  return tw;
}

template <class T>
int dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)) == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

}  // namespace

// dynamic shared memory of the two spectral tile kernels (spectral_solve)
size_t dft_forward_smem(int N, int H) {
  return static_cast<size_t>(N) * sizeof(double2) + static_cast<size_t>(kDftRows) * N * sizeof(double) +
         static_cast<size_t>(H) * sizeof(int);
}
int idft_threads(int N) { return N * std::max(1, 512 / N); }  // thread t owns sample t mod N
size_t idft_smem(int N, int H) {
  return static_cast<size_t>(N) * sizeof(double2) + static_cast<size_t>(kDftRows) * H * sizeof(double2) +
         static_cast<size_t>(2) * idft_threads(N) * sizeof(double) + static_cast<size_t>(H) * sizeof(int);
}

struct SpectralState {
  int N = 0, d = 0, nnz = 0, H = 0;
  double period = 0.0;
  int conj = 1, shift_kind = 0;
  std::vector<int> bins;
  std::vector<int> harmonic;  // signed harmonic index per solved bin
  int G = 0, C = 0, L = 0, Lp = 0, R = 0;
  int* warp_row_begin = nullptr;
  int n_long = 0;
  int* long_rows = nullptr;
  int* long_owner = nullptr;
  double* X = nullptr;
  double* Y = nullptr;
  double* Q = nullptr;  // C + K for the RHS
  double2* XYE = nullptr;  // [d][kEll] padded (X, Y) slot values
  double2* dXY = nullptr;  // [d] diagonal (X, Y)
  double2* shift = nullptr;
  double2* tw = nullptr;
  int* d_bins = nullptr;
  double* rhs = nullptr;  // [d][N]
  double2 *bhat = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;
  unsigned long long* sync = nullptr;
  double* partials = nullptr;
  int* abort_flag = nullptr;
  int* code = nullptr;
  int* iters = nullptr;
  int64_t* lockstep = nullptr;
  double* jpart = nullptr;
  double* maxre = nullptr;
  double* maxim = nullptr;
  double* jout = nullptr;
  double* coef = nullptr;  // [N][nterms] excitation at T_sub per row
  int idft_blocks = 0;
  bool warm_valid = false;  // x holds the last successful solve's solution (warm-start value)
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

// shared with capi.cu
int row_ranges(const std::vector<int>& h_rp, int C, int R, std::vector<int>* out,
               const std::vector<unsigned char>* rowkind);
int long_rows_of(const std::vector<int>& h_rp, const std::vector<int>& ranges, std::vector<int>* rows,
                 std::vector<int>* owner);

int spectral_setup(SpectralState** out, const DevProblem& p, int N, double period, int use_conj,
                   const int32_t* mask, int shift_kind, std::string* err) {
  if (N < 2 || N % 2 != 0) {
    *err = "spectral: multiharmonic solve requires an even number of blocks >= 2, got " + std::to_string(N);
    return PS_ERR_ODD_BLOCKS;
  }
  if (!p.linear) {
    *err = "spectral: cyclic system requires a linear problem (freeze the coarse operator first)";
    return PS_ERR_NOT_LINEAR;
  }
  if (N > 1024) {
    *err = "spectral: multiharmonic solve supports at most 1024 blocks, got " + std::to_string(N);
    return PS_ERR_BAD_ARG;
  }
  auto* s = new SpectralState();
  s->N = N;
  s->d = p.d;
  s->nnz = p.nnz;
  s->period = period;
  s->conj = use_conj ? 1 : 0;
  s->shift_kind = shift_kind;
  const int last = use_conj ? N / 2 : N - 1;
  for (int b = 0; b <= last; ++b) {
    if (mask && mask[b] == 0) continue;
    s->bins.push_back(b);
    s->harmonic.push_back(b <= N / 2 ? b : b - N);
  }
  s->H = static_cast<int>(s->bins.size());
  const double dT = period / N;
  // host: C = M/dT, Q = C + K  (make_cyclic_system, proj/src/spectral.cpp:118-132)
  std::vector<double> hC(p.nnz), hQ(p.nnz);
  for (int k = 0; k < p.nnz; ++k) {
    hC[k] = p.h_M[k] / dT;
    hQ[k] = hC[k] + p.h_K[k];
  }
  std::vector<double2> hs(std::max(1, s->H));
  for (int hh = 0; hh < s->H; ++hh) {
    const int pidx = s->harmonic[hh];
    if (shift_kind == 0) {
      const std::complex<double> phase = std::exp(std::complex<double>(0.0, -2.0 * kPi * pidx / N));
      hs[hh] = make_double2(-phase.real(), -phase.imag());
    } else {
      hs[hh] = make_double2(0.0, 2.0 * kPi * pidx / period);
    }
  }
  int rc = PS_OK;
  rc |= dalloc(&s->X, p.nnz);
  rc |= dalloc(&s->Y, p.nnz);
  rc |= dalloc(&s->Q, p.nnz);
  rc |= dalloc(&s->shift, std::max(1, s->H));
  rc |= dalloc(&s->tw, N);
  rc |= dalloc(&s->d_bins, std::max(1, s->H));
  rc |= dalloc(&s->rhs, static_cast<size_t>(p.d) * N);
  const size_t cvec = static_cast<size_t>(p.d) * std::max(1, s->H);
  rc |= dalloc(&s->bhat, cvec);
  rc |= dalloc(&s->x, cvec);
  rc |= dalloc(&s->r, cvec);
  rc |= dalloc(&s->p, cvec);
  rc |= dalloc(&s->q, cvec);
  if (rc != PS_OK) {
    *err = "cuda: out of memory in spectral setup";
    spectral_free(s);
    return PS_ERR_CUDA;
  }
  if (shift_kind == 0) {
    cudaMemcpy(s->X, hQ.data(), p.nnz * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(s->Y, hC.data(), p.nnz * sizeof(double), cudaMemcpyHostToDevice);
  } else {
    cudaMemcpy(s->X, p.h_K.data(), p.nnz * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(s->Y, p.h_M.data(), p.nnz * sizeof(double), cudaMemcpyHostToDevice);
  }
  cudaMemcpy(s->Q, hQ.data(), p.nnz * sizeof(double), cudaMemcpyHostToDevice);
  {
    // padded (X, Y) rows and diagonal pairs for the COCG SpMV / Jacobi
    const std::vector<double>& hX = shift_kind == 0 ? hQ : p.h_K;
    const std::vector<double>& hY = shift_kind == 0 ? hC : p.h_M;
    std::vector<double2> xye(static_cast<size_t>(p.d) * kEll, make_double2(0.0, 0.0)), dxy(p.d);
    for (int i = 0; i < p.d; ++i) {
      const int b = p.h_rp[i], len = p.h_rp[i + 1] - b;
      if (len <= kEll)
        for (int k = 0; k < len; ++k) xye[static_cast<size_t>(i) * kEll + k] = make_double2(hX[b + k], hY[b + k]);
      const int dk = p.h_diag[i];
      dxy[i] = make_double2(hX[dk], hY[dk]);
    }
    rc |= dalloc(&s->XYE, xye.size());
    rc |= dalloc(&s->dXY, dxy.size());
    if (rc == PS_OK) {
      cudaMemcpy(s->XYE, xye.data(), xye.size() * sizeof(double2), cudaMemcpyHostToDevice);
      cudaMemcpy(s->dXY, dxy.data(), dxy.size() * sizeof(double2), cudaMemcpyHostToDevice);
    }
  }
  cudaMemcpy(s->shift, hs.data(), hs.size() * sizeof(double2), cudaMemcpyHostToDevice);
  const auto tw = twiddles(N);
  cudaMemcpy(s->tw, tw.data(), N * sizeof(double2), cudaMemcpyHostToDevice);
  if (s->H > 0) cudaMemcpy(s->d_bins, s->bins.data(), s->H * sizeof(int), cudaMemcpyHostToDevice);

  // COCG launch geometry: groups of <= 32 bins, C co-resident blocks per group
  if (s->H > 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cocg_kernel, kThreads, 0);
    const int capacity = std::max(1, sms * per_sm);
    s->G = (s->H + 31) / 32;
    s->L = (s->H + s->G - 1) / s->G;
    s->Lp = 32;  // one lane per bin (the long-row split assumes R = 1)
    s->R = 1;
    const int rows_min = kWarps * s->R * 4;
    s->C = std::max(1, std::min(capacity / s->G, (p.d + rows_min - 1) / rows_min));
    if (s->G > capacity) {
      *err = "spectral: too many harmonic bins for one cooperative launch";
      spectral_free(s);
      return PS_ERR_BAD_ARG;
    }
    std::vector<int> ranges;
    row_ranges(p.h_rp, s->C, s->R, &ranges, nullptr);
    rc |= dalloc(&s->warp_row_begin, ranges.size());
    cudaMemcpy(s->warp_row_begin, ranges.data(), ranges.size() * sizeof(int), cudaMemcpyHostToDevice);
    std::vector<int> lrows, lowner;
    long_rows_of(p.h_rp, ranges, &lrows, &lowner);
    s->n_long = static_cast<int>(lrows.size());
    rc |= dalloc(&s->long_rows, std::max<size_t>(1, lrows.size()));
    rc |= dalloc(&s->long_owner, std::max<size_t>(1, lrows.size()));
    if (s->n_long) {
      cudaMemcpy(s->long_rows, lrows.data(), lrows.size() * sizeof(int), cudaMemcpyHostToDevice);
      cudaMemcpy(s->long_owner, lowner.data(), lowner.size() * sizeof(int), cudaMemcpyHostToDevice);
    }
    rc |= dalloc(&s->sync, s->G);
    rc |= dalloc(&s->partials, static_cast<size_t>(2) * s->G * s->C * kCND * 32);
    rc |= dalloc(&s->abort_flag, 1);
    rc |= dalloc(&s->code, s->H);
    rc |= dalloc(&s->iters, s->H);
    rc |= dalloc(&s->lockstep, s->G);
  }
  {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = (p.d + kDftRows - 1) / kDftRows;
    s->idft_blocks = std::max(1, std::min(tiles, sms * 8));
  }
  rc |= dalloc(&s->jpart, static_cast<size_t>(s->idft_blocks) * 2 * N);
  rc |= dalloc(&s->maxre, static_cast<size_t>(s->idft_blocks));
  rc |= dalloc(&s->maxim, static_cast<size_t>(s->idft_blocks));
  rc |= dalloc(&s->jout, 8);
  rc |= dalloc(&s->coef, static_cast<size_t>(N) * std::max(1, p.nterms));
  // excitation coefficients at T_sub for every row (assemble_rhs)
  std::vector<double> coef(static_cast<size_t>(N) * std::max(1, p.nterms), 0.0);
  for (int row = 0; row < N; ++row) {
    const int sub = row == 0 ? N : row;
    const double t = sub == N ? period : static_cast<double>(sub) * period / N;  // TimeMesh::boundary
    double tau = std::fmod(t, p.period);
    if (tau < 0.0) tau += p.period;
    for (int k = 0; k < p.nterms; ++k) {
      const double arg = 2.0 * kPi * p.freq[k] * tau + p.phase[k];
      coef[static_cast<size_t>(row) * p.nterms + k] = p.amp[k] * std::sin(arg);
    }
  }
  cudaMemcpy(s->coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice);
  // spectral tiles: opt in to the device's shared-memory maximum and reject a
  // (N, bins) combination whose tiles do not fit (e.g. N = 1024 with
  // use_conjugate_symmetry = 0 asks for ~164 KB in the inverse tile)
  {
    int dev = 0, smax = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t need = std::max(dft_forward_smem(N, s->H), idft_smem(N, s->H));
    if (need > static_cast<size_t>(smax)) {
      *err = "spectral: " + std::to_string(N) + " blocks with " + std::to_string(s->H) +
             " solved bins need " + std::to_string(need) + " bytes of shared memory per spectral tile (device max " +
             std::to_string(smax) + ")";
      spectral_free(s);
      return PS_ERR_BAD_ARG;
    }
    cudaFuncSetAttribute(reinterpret_cast<const void*>(dft_forward_kernel),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(idft_jump_kernel),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
  }
  cudaEventCreate(&s->e0);
  cudaEventCreate(&s->e1);
  if (rc != PS_OK || cudaGetLastError() != cudaSuccess) {
    *err = "cuda: spectral setup failed";
    spectral_free(s);
    return PS_ERR_CUDA;
  }
  *out = s;
  return PS_OK;
}

void spectral_free(SpectralState* s) {
  if (!s) return;
  void* ptrs[] = {s->XYE, s->dXY, s->warp_row_begin, s->long_rows, s->long_owner, s->X, s->Y, s->Q, s->shift, s->tw, s->d_bins, s->rhs, s->bhat,
                  s->x, s->r, s->p, s->q, s->sync, s->partials, s->abort_flag, s->code, s->iters,
                  s->lockstep, s->jpart, s->maxre, s->maxim, s->jout, s->coef};
  for (void* ptr : ptrs)
    if (ptr) cudaFree(ptr);
  if (s->e0) cudaEventDestroy(s->e0);
  if (s->e1) cudaEventDestroy(s->e1);
  delete s;
}

int spectral_assemble_rhs(SpectralState* s, const DevProblem& p, const double* F_il, const double* G_il,
                          double* rhs_il, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(s->d) * s->N;
  assemble_rhs_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
      s->d, s->N, p.rp, p.ci, s->Q, F_il, G_il, p.pat, s->coef, p.nterms, rhs_il ? rhs_il : s->rhs);
  return cudaGetLastError() == cudaSuccess ? PS_OK : PS_ERR_CUDA;
}

int spectral_solve(SpectralState* s, const DevProblem& p, const ps_krylov_settings& cocg, const double* rhs_il,
                   double* U_il, double* U_prev_il, double* jump, ps_batch_status* status, cudaStream_t st,
                   std::string* err) {
  const int N = s->N, d = s->d, H = s->H;
  cudaEventRecord(s->e0, st);
  const double* rhs = rhs_il ? rhs_il : s->rhs;
  // warm start (ps_krylov_settings.warm_start): from the last successful solve
  const bool warm = cocg.warm_start != 0 && s->warm_valid;
  s->warm_valid = false;
  int64_t lock_total = 0, its_total = 0;
  int max_its = 0;
  if (H > 0) {
    const int ftpb = std::min(1024, ((kDftRows * H + 31) / 32) * 32);
    dft_forward_kernel<<<s->idft_blocks, ftpb, dft_forward_smem(N, H), st>>>(d, N, H, s->d_bins, s->tw, rhs, s->bhat);
    if (const cudaError_t le = cudaGetLastError(); le != cudaSuccess) {
      *err = std::string("cuda: dft_forward launch failed: ") + cudaGetErrorString(le);
      return PS_ERR_CUDA;
    }
    cudaMemsetAsync(s->sync, 0, s->G * sizeof(unsigned long long), st);
    cudaMemsetAsync(s->abort_flag, 0, sizeof(int), st);
    CocgParams P{};
    P.d = d;
    P.H = H;
    P.G = s->G;
    P.C = s->C;
    P.L = s->L;
    P.Lp = s->Lp;
    P.R = s->R;
    P.warp_row_begin = s->warp_row_begin;
    P.n_long = s->n_long;
    P.long_rows = s->long_rows;
    P.long_owner = s->long_owner;
    P.rp = p.rp;
    P.ci = p.ci;
    P.diag = p.diag;
    P.X = s->X;
    P.Y = s->Y;
    P.rowrec = p.rowrec;
    P.XYE = s->XYE;
    P.dXY = s->dXY;
    P.shift = s->shift;
    P.b = s->bhat;
    P.x = s->x;
    P.r = s->r;
    P.p = s->p;
    P.q = s->q;
    P.tol = cocg.tol_rel;
    P.max_iter = cocg.max_iter;
    P.warm = warm ? 1 : 0;
    P.sync = s->sync;
    P.partials = s->partials;
    P.abort_flag = s->abort_flag;
    P.code = s->code;
    P.iters = s->iters;
    P.lockstep = s->lockstep;
    void* args[] = {&P};
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cocg_kernel), dim3(s->G * s->C),
                                                      dim3(kThreads), args, 0, st);
    if (e != cudaSuccess) {
      *err = std::string("cuda: cocg launch failed: ") + cudaGetErrorString(e);
      return PS_ERR_CUDA;
    }
  }
  idft_jump_kernel<<<s->idft_blocks, idft_threads(N), idft_smem(N, H), st>>>(
      d, N, H, s->d_bins, s->tw, s->conj, s->x, U_il, U_prev_il, s->jpart, s->maxre, s->maxim);
  if (const cudaError_t le = cudaGetLastError(); le != cudaSuccess) {
    *err = std::string("cuda: idft_jump launch failed: ") + cudaGetErrorString(le);
    return PS_ERR_CUDA;
  }
  jump_finalize_kernel<<<1, 1024, 0, st>>>(N, s->idft_blocks, s->idft_blocks, s->jpart, s->maxre, s->maxim, s->jout);
  if (const cudaError_t le = cudaGetLastError(); le != cudaSuccess) {
    *err = std::string("cuda: jump_finalize launch failed: ") + cudaGetErrorString(le);
    return PS_ERR_CUDA;
  }
  cudaEventRecord(s->e1, st);
  double hj[5];
  cudaMemcpyAsync(hj, s->jout, sizeof(hj), cudaMemcpyDeviceToHost, st);
  std::vector<int> codes(H), iters(H);
  std::vector<int64_t> lock(s->G);
  int abort_h = 0;
  if (H > 0) {
    cudaMemcpyAsync(codes.data(), s->code, H * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(iters.data(), s->iters, H * sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(lock.data(), s->lockstep, s->G * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&abort_h, s->abort_flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  }
  const cudaError_t ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) {
    *err = std::string("cuda: spectral solve failed: ") + cudaGetErrorString(ce);
    return PS_ERR_CUDA;
  }
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, s->e0, s->e1);
  if (abort_h) {
    *err = "cuda: device barrier watchdog fired in the COCG kernel";
    return PS_ERR_WATCHDOG;
  }
  int rc = PS_OK;
  for (int hh = 0; hh < H; ++hh) {
    its_total += iters[hh];
    max_its = std::max(max_its, iters[hh]);
    if (codes[hh] != PS_OK && rc == PS_OK) {
      rc = codes[hh];
      if (rc == PS_ERR_SINGULAR_BLOCK)
        *err = "spectral: harmonic block p = " + std::to_string(s->harmonic[hh]) + " is singular";
      else
        *err = "spectral: COCG did not converge for harmonic block p = " + std::to_string(s->harmonic[hh]);
    }
  }
  for (int g = 0; g < s->G && H > 0; ++g) lock_total += lock[g];
  if (rc == PS_OK) {
    if (!std::isfinite(hj[3]) || !std::isfinite(hj[4])) {
      rc = PS_ERR_NONFINITE;
      *err = "spectral: harmonic solve produced non-finite values";
    } else if (hj[4] > kImagResidualTol * std::max(1.0, hj[3])) {
      rc = PS_ERR_CONJ_SYMMETRY;
      *err = "spectral: conjugate symmetry violated (imaginary residue " + std::to_string(hj[4]) + ")";
    }
  }
  if (jump) *jump = hj[0];
  if (status) {
    std::memset(status, 0, sizeof(*status));
    status->code = rc;
    status->failed_index = -1;
    status->pcg_iterations = its_total;
    status->max_pcg_iterations = max_its;
    status->lockstep_pcg_iterations = lock_total;
    // canonical bytes: COCG H*160*d + 20*nnz + 4(d+1) per batched
    // iteration; DFT 8Nd + 16Hd each way; jump +8Nd
    const double dd = static_cast<double>(d), nz = static_cast<double>(s->nnz);
    double bytes = 0.0;
    for (int hh = 0; hh < H; ++hh) bytes += static_cast<double>(iters[hh]) * 160.0 * dd;
    bytes += static_cast<double>(lock_total) * (20.0 * nz + 4.0 * (dd + 1.0));
    bytes += 2.0 * (8.0 * N * dd + 16.0 * H * dd) + 8.0 * N * dd;
    if (warm) bytes += H * 32.0 * dd + 20.0 * nz + 4.0 * (dd + 1.0);  // warm start: q = Lambda x once
    status->algorithmic_bytes = bytes;
    status->kernel_ms = ms;
  }
  s->warm_valid = (rc == PS_OK && H > 0);
  return rc;
}

// Test probes of the hot-path spectral kernels with a context's solved bins
// (ps_mh_forward / ps_mh_inverse): host arrays in the reference's order.
// Forward: rhs [N][d] -> dft_forward_kernel -> spectrum [H][d] (complex pairs).
int spectral_forward_probe(SpectralState* s, const double* rhs, double* spec, std::string* err) {
  const int N = s->N, d = s->d, H = s->H;
  if (H < 1) {
    *err = "spectral: no solved bins";
    return PS_ERR_BAD_ARG;
  }
  double* tmp = nullptr;
  if (dalloc(&tmp, static_cast<size_t>(N) * d)) {
    *err = "cuda: out of memory";
    return PS_ERR_CUDA;
  }
  cudaMemcpy(tmp, rhs, static_cast<size_t>(N) * d * sizeof(double), cudaMemcpyHostToDevice);
  launch_to_interleaved(tmp, s->rhs, N, d, N, nullptr);
  const int ftpb = std::min(1024, ((kDftRows * H + 31) / 32) * 32);
  dft_forward_kernel<<<s->idft_blocks, ftpb, dft_forward_smem(N, H)>>>(d, N, H, s->d_bins, s->tw, s->rhs, s->bhat);
  cudaError_t e = cudaGetLastError();
  std::vector<double2> h(static_cast<size_t>(d) * H);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), s->bhat, h.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  if (e != cudaSuccess) {
    *err = std::string("cuda: dft_forward failed: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  for (int hh = 0; hh < H; ++hh)
    for (int i = 0; i < d; ++i) {
      spec[(static_cast<size_t>(hh) * d + i) * 2] = h[static_cast<size_t>(i) * H + hh].x;
      spec[(static_cast<size_t>(hh) * d + i) * 2 + 1] = h[static_cast<size_t>(i) * H + hh].y;
    }
  return PS_OK;
}

// Inverse: spectrum [H][d] -> idft_jump_kernel (mirror, realify check, jump
// partials against U_old [N][d] or none) + jump_finalize_kernel -> U [N][d], jump.
int spectral_inverse_probe(SpectralState* s, const double* spec, const double* U_old, double* U, double* jump,
                           std::string* err) {
  const int N = s->N, d = s->d, H = s->H;
  std::vector<double2> h(static_cast<size_t>(d) * std::max(1, H));
  for (int hh = 0; hh < H; ++hh)
    for (int i = 0; i < d; ++i)
      h[static_cast<size_t>(i) * H + hh] =
          make_double2(spec[(static_cast<size_t>(hh) * d + i) * 2], spec[(static_cast<size_t>(hh) * d + i) * 2 + 1]);
  double *tmp = nullptr, *u_il = nullptr, *old_il = nullptr;
  if (dalloc(&tmp, static_cast<size_t>(N) * d) || dalloc(&u_il, static_cast<size_t>(N) * d) ||
      dalloc(&old_il, static_cast<size_t>(N) * d)) {
    *err = "cuda: out of memory";
    return PS_ERR_CUDA;
  }
  if (H > 0) cudaMemcpy(s->x, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
  if (U_old) {
    cudaMemcpy(tmp, U_old, static_cast<size_t>(N) * d * sizeof(double), cudaMemcpyHostToDevice);
    launch_to_interleaved(tmp, old_il, N, d, N, nullptr);
  }
  idft_jump_kernel<<<s->idft_blocks, idft_threads(N), idft_smem(N, H)>>>(
      d, N, H, s->d_bins, s->tw, s->conj, s->x, u_il, U_old ? old_il : nullptr, s->jpart, s->maxre, s->maxim);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    jump_finalize_kernel<<<1, 1024>>>(N, s->idft_blocks, s->idft_blocks, s->jpart, s->maxre, s->maxim, s->jout);
    e = cudaGetLastError();
  }
  double hj[5] = {0, 0, 0, 0, 0};
  if (e == cudaSuccess) {
    launch_from_interleaved(u_il, tmp, N, d, N, nullptr);
    e = cudaMemcpy(U, tmp, static_cast<size_t>(N) * d * sizeof(double), cudaMemcpyDeviceToHost);
  }
  if (e == cudaSuccess) e = cudaMemcpy(hj, s->jout, sizeof(hj), cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  cudaFree(u_il);
  cudaFree(old_il);
  if (e != cudaSuccess) {
    *err = std::string("cuda: idft_jump failed: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  if (jump) *jump = hj[0];
  if (!std::isfinite(hj[3]) || !std::isfinite(hj[4])) {
    *err = "spectral: harmonic solve produced non-finite values";
    return PS_ERR_NONFINITE;
  }
  if (hj[4] > kImagResidualTol * std::max(1.0, hj[3])) {
    *err = "spectral: conjugate symmetry violated (imaginary residue " + std::to_string(hj[4]) + ")";
    return PS_ERR_CONJ_SYMMETRY;
  }
  return PS_OK;
}

int dft_forward_standalone(int n, int d, const double* U, double* spec, std::string* err) {
  if (n < 2 || n % 2 != 0) {
    *err = "spectral: forward_dft requires an even number of blocks >= 2, got " + std::to_string(n);
    return PS_ERR_ODD_BLOCKS;
  }
  const size_t total = static_cast<size_t>(n) * d;
  std::vector<double2> hin(total);
  for (size_t k = 0; k < total; ++k) hin[k] = make_double2(U[k], 0.0);
  double2 *din = nullptr, *dout = nullptr, *dtw = nullptr;
  if (dalloc(&din, total) || dalloc(&dout, total) || dalloc(&dtw, n)) {
    *err = "cuda: allocation failed";
    return PS_ERR_CUDA;
  }
  const auto tw = twiddles(n);
  cudaMemcpy(dtw, tw.data(), n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemcpy(din, hin.data(), total * sizeof(double2), cudaMemcpyHostToDevice);
  dft_generic_kernel<<<static_cast<unsigned>((total + 255) / 256), 256>>>(n, d, dtw, 0, din, dout);
  const cudaError_t e = cudaMemcpy(spec, dout, total * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dtw);
  if (e != cudaSuccess) {
    *err = std::string("cuda: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  return PS_OK;
}

int dft_inverse_standalone(int n, int d, const double* spec, double* U, std::string* err) {
  if (n < 2 || n % 2 != 0) {
    *err = "spectral: inverse_dft requires an even number of blocks >= 2, got " + std::to_string(n);
    return PS_ERR_ODD_BLOCKS;
  }
  const size_t total = static_cast<size_t>(n) * d;
  double2 *din = nullptr, *dout = nullptr, *dtw = nullptr;
  if (dalloc(&din, total) || dalloc(&dout, total) || dalloc(&dtw, n)) {
    *err = "cuda: allocation failed";
    return PS_ERR_CUDA;
  }
  const auto tw = twiddles(n);
  cudaMemcpy(dtw, tw.data(), n * sizeof(double2), cudaMemcpyHostToDevice);
  cudaMemcpy(din, spec, total * sizeof(double2), cudaMemcpyHostToDevice);
  dft_generic_kernel<<<static_cast<unsigned>((total + 255) / 256), 256>>>(n, d, dtw, 1, din, dout);
  std::vector<double2> hout(total);
  const cudaError_t e = cudaMemcpy(hout.data(), dout, total * sizeof(double2), cudaMemcpyDeviceToHost);
  cudaFree(din);
  cudaFree(dout);
  cudaFree(dtw);
  if (e != cudaSuccess) {
    *err = std::string("cuda: ") + cudaGetErrorString(e);
    return PS_ERR_CUDA;
  }
  double re = 0.0, im = 0.0;
  for (size_t k = 0; k < total; ++k) {
    re = std::max(re, std::fabs(hout[k].x));
    im = std::max(im, std::fabs(hout[k].y));
  }
  if (im > kImagResidualTol * std::max(1.0, re)) {
    *err = "spectral: conjugate symmetry violated (imaginary residue " + std::to_string(im) + ")";
    return PS_ERR_CONJ_SYMMETRY;
  }
  for (size_t k = 0; k < total; ++k) U[k] = hout[k].x;
  return PS_OK;
}

int spectral_bins(const SpectralState* s, int32_t* bins, int32_t cap) {
  for (int k = 0; k < s->H && k < cap; ++k) bins[k] = s->bins[k];
  return s->H;
}

int jump_norm_device(int count, int d, const double* cur_il, const double* prev_il, int stride, double* out,
                     cudaStream_t st) {
  double* part = nullptr;
  if (dalloc(&part, static_cast<size_t>(2) * count)) return PS_ERR_CUDA;
  strided_jump_kernel<<<count, 256, 0, st>>>(count, d, stride, cur_il, prev_il, part);
  std::vector<double> h(static_cast<size_t>(2) * count);
  const cudaError_t e = cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(part);
  if (e != cudaSuccess) return PS_ERR_CUDA;
  double change = 0.0, scale = 1.0;
  for (int n = 0; n < count; ++n) {
    change = std::max(change, std::sqrt(h[2 * n]));
    scale = std::max(scale, std::sqrt(h[2 * n + 1]));
  }
  *out = change / scale;
  return PS_OK;
}

}  // namespace pppc
