// Group barrier + deterministic reduction used by the persistent solver kernels.
//
// A "group" is the set of C co-resident blocks that serve one batch of <= 32
// independent systems (fine propagators or harmonic bins).  Blocks of a group
// synchronise through a monotone 64-bit arrival counter (no reset, no grid-wide
// barrier, other groups are never waited for).  Each block first reduces its
// per-lane partials in a fixed order, publishes them, arrives, waits until all C
// blocks of the group have arrived, then EVERY block reduces the C published
// partials in the same fixed order.  All blocks therefore hold bit-identical
// per-system scalars and take identical control-flow decisions without a
// second broadcast barrier.  Partials are double-buffered by barrier parity: a
// block cannot overwrite a buffer before every block has passed the barrier
// that follows its last read.
#pragma once

#include "pppc_internal.h"

namespace pppc {

constexpr unsigned long long kBarrierTimeoutNs = 60ull * 1000ull * 1000ull * 1000ull;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ int ld_volatile_i32(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int NDMAX>
struct SyncShared {
  static constexpr int S = kThreads / (NDMAX * 16);  // interleaved sub-sums per (dot, lane pair)
  double wpart[kWarps][NDMAX][32];
  double red[S][NDMAX][32];
  double tot[NDMAX][32];
  int abort;
  // barrier state (thread 0 advances it): arrival target and barrier count
  unsigned long long target;
  int bar_idx;
};

template <int NDMAX>
__device__ __forceinline__ void sync_state_init(SyncShared<NDMAX>& sh) {
  if (threadIdx.x == 0) {
    sh.abort = 0;
    sh.target = 0;
    sh.bar_idx = 0;
  }
}

struct SyncCtx {
  unsigned long long* sync;  // [G]
  double* partials;          // [2][G][C][NDMAX][32]
  int* abort_flag;
  int G, C, Lp;
  int L;                     // lanes carrying a system (the rest are padding and are not reduced)
};

// acc: this thread's partial sums (lane = system, sub-rows combined here).
// The barrier state lives in `sh` (sync_state_init before the first call), so
// nothing of it occupies registers across the caller's work loop.
template <int NDMAX, int ND>
__device__ bool group_sync_reduce(const SyncCtx& X, SyncShared<NDMAX>& sh, double (&acc)[NDMAX], int g, int c,
                                  unsigned long long* t_arrive = nullptr) {
  static_assert(ND <= NDMAX, "too many dots");
  constexpr int S = SyncShared<NDMAX>::S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int off = X.Lp; off < 32; off <<= 1) {
#pragma unroll
    for (int k = 0; k < ND; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
  }
  if (lane < X.Lp) {
#pragma unroll
    for (int k = 0; k < ND; ++k) sh.wpart[warp][k][lane] = acc[k];
  }
  const int buf = sh.bar_idx & 1;
  __syncthreads();
  double* part = X.partials + ((static_cast<size_t>(buf) * X.G + g) * X.C) * (NDMAX * 32);
  if (threadIdx.x < ND * 32) {
    const int k = threadIdx.x >> 5, l = threadIdx.x & 31;
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += sh.wpart[w][k][l];
    part[static_cast<size_t>(c) * (NDMAX * 32) + k * 32 + l] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (t_arrive) *t_arrive = globaltimer_ns();
    __threadfence();
    atomicAdd(X.sync + g, 1ull);
    const unsigned long long target = sh.target + static_cast<unsigned long long>(X.C);
    sh.target = target;
    const unsigned long long t0 = globaltimer_ns();
    int ab = 0;
    while (ld_volatile_u64(X.sync + g) < target) {
      if (ld_volatile_i32(X.abort_flag)) {
        ab = 1;
        break;
      }
      if (globaltimer_ns() - t0 > kBarrierTimeoutNs) {
        atomicExch(X.abort_flag, 1);
        ab = 1;
        break;
      }
      __nanosleep(20);
    }
    __threadfence();
    if (t_arrive) t_arrive[1] = globaltimer_ns();  // release seen (diagnostics)
    sh.abort = ab;
    sh.bar_idx += 1;
  }
  __syncthreads();
  if (sh.abort) return false;
  {
    // thread = (sub-sum s, dot k, lane pair lp): 16-byte loads of two lanes,
    // kRedIlp of them in flight, partials of block c = s, s + S, ... summed
    // in increasing c (fixed order); at C = 148 two rounds of L2 latency
    constexpr int kRedIlp = 10;
    const int t = threadIdx.x;
    const int s = t / (NDMAX * 16);
    const int k = (t / 16) % NDMAX;
    const int lp = t & 15;
    if (s < S && k < ND && 2 * lp < X.L) {
      double2 v = make_double2(0.0, 0.0);
      for (int c0 = s; c0 < X.C; c0 += kRedIlp * S) {
        double2 tmp[kRedIlp];
#pragma unroll
        for (int u = 0; u < kRedIlp; ++u) {
          const int cc = c0 + u * S;
          tmp[u] = cc < X.C ? *reinterpret_cast<const double2*>(part + static_cast<size_t>(cc) * (NDMAX * 32) +
                                                                k * 32 + 2 * lp)
                            : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kRedIlp; ++u) {
          v.x += tmp[u].x;
          v.y += tmp[u].y;
        }
      }
      sh.red[s][k][2 * lp] = v.x;
      sh.red[s][k][2 * lp + 1] = v.y;
    }
  }
  __syncthreads();
  if (threadIdx.x < ND * 32) {
    const int k = threadIdx.x >> 5, l = threadIdx.x & 31;
    double v = sh.red[0][k][l];
#pragma unroll
    for (int s = 1; s < S; ++s) v += sh.red[s][k][l];
    sh.tot[k][l] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NDMAX; ++k) acc[k] = 0.0;
  return true;
}

}  // namespace pppc
