// C ABI of the B200 PP-PC hot path (include/pppc_b200.h) and the host C++
// PP-PC driver that mirrors solve_pp_pc (proj/src/engine.cpp:187-270).
//
// The context owns every device buffer (pattern, values, work vectors,
// allocated once at ps_create); host arrays cross the ABI in the reference's
// [count][dim] order and are transposed on the device into the interleaved
// [dim][count] layout the kernels use.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pppc_internal.h"

using namespace pppc;

namespace pppc {

constexpr double kPi = 3.14159265358979323846;

thread_local std::string g_global_error;

struct Geometry {
  int G = 0, C = 0, L = 0, Lp = 0, R = 0;
  int* warp_row_begin = nullptr;
  int n_long = 0;
  int* long_rows = nullptr;
  int* long_owner = nullptr;
  int max_block_rows = 0;  // largest row range of one block (shared-memory records)
};

// Rows longer than kLongRow and the block whose warp ranges contain them.
int long_rows_of(const std::vector<int>& h_rp, const std::vector<int>& ranges, std::vector<int>* rows,
                 std::vector<int>* owner) {
  const int d = static_cast<int>(h_rp.size()) - 1;
  const int parts = static_cast<int>(ranges.size()) - 1;
  rows->clear();
  owner->clear();
  int part = 0;
  for (int i = 0; i < d; ++i) {
    while (part + 1 < parts && ranges[part + 1] <= i) ++part;
    if (h_rp[i + 1] - h_rp[i] > kLongRow) {
      rows->push_back(i);
      owner->push_back(part / kWarps);
    }
  }
  return PS_OK;
}

// Contiguous row ranges for C blocks x kWarps warps, balanced by row cost
// (slots + vector streams).  Depends only on the pattern, C and R.
int row_ranges(const std::vector<int>& h_rp, int C, int R, std::vector<int>* out,
               const std::vector<unsigned char>* rowkind) {
  const int d = static_cast<int>(h_rp.size()) - 1;
  const int parts = C * kWarps;
  std::vector<double> cum(d + 1, 0.0);
  // Near-equal row counts per warp: the PCG update phase costs the same for
  // every row and each phase ends at a group barrier, so the slowest warp sets
  // the pace (rows of the P1 mesh differ by at most 7 vs 5 slots).  Rows with
  // per-system values (rowkind 1) stream their values and Jacobi diagonal from
  // HBM instead of the shared L2-resident copy and weigh 1.3 (measured phase
  // A+B cost ratio).  Long rows are split across the owning block's warps and
  // weigh their per-warp share.
  for (int i = 0; i < d; ++i) {
    const int len = h_rp[i + 1] - h_rp[i];
    const double w = (rowkind && !rowkind->empty() && (*rowkind)[i]) ? 1.3 : 1.0;
    cum[i + 1] = cum[i] + (len > kLongRow ? 1.0 + len / double(kWarps * kRegularRow) : w);
  }
  out->assign(parts + 1, d);
  (*out)[0] = 0;
  int row = 0;
  for (int k = 1; k < parts; ++k) {
    const double goal = cum[d] * k / parts;
    while (row < d && cum[row] < goal) ++row;
    // keep ranges a multiple of R rows where possible (sub-row lanes)
    int aligned = row - (row % R);
    aligned = std::max(aligned, (*out)[k - 1]);
    (*out)[k] = std::min(aligned, d);
  }
  (*out)[parts] = d;
  return PS_OK;
}

}  // namespace pppc

struct ps_ctx {
  DevProblem P;
  ps_time_mesh mesh{};
  ps_solver_settings settings{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int max_batch = 0;
  int capacity = 0;
  // work buffers (interleaved, stride = batch count)
  double *u = nullptr, *uprev = nullptr, *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;
  double *Dinv = nullptr, *A = nullptr;
  double *io_a = nullptr, *io_b = nullptr;  // [count][d] staging
  // kernel control
  unsigned long long* sync = nullptr;
  double* partials = nullptr;
  size_t partials_len = 0;
  int* abort_flag = nullptr;
  SysOut* out = nullptr;
  double* trace = nullptr;
  int64_t* lockstep = nullptr;
  double* coef = nullptr;
  size_t coef_len = 0;
  double* tnext = nullptr;
  size_t tnext_len = 0;
  std::map<int, Geometry> geo;
  // dt -> shared step matrix M/dt + K (CSR values, Jacobi, per-row padded
  // values for the SpMV row records); the linear_factor analogue
  struct StepMatrix {
    double* A = nullptr;
    double* D = nullptr;
    double* AE = nullptr;
    double* AT = nullptr;  // AE transposed [kEll][d] (system-per-block engine)
  };
  // system-per-block engine buffers: contiguous state, per-system ELL values, hub values
  double *sb_u = nullptr, *sb_A = nullptr, *sb_hub = nullptr;
  size_t sb_u_len = 0, sb_A_len = 0, sb_hub_len = 0;
  std::map<double, StepMatrix> step_cache;
  // system-per-cluster engine geometry (cluster_geometry): C = 0 when it cannot run
  ClusterGeom cl_geo{};
  int cl_slots = 0;       // co-resident clusters
  bool cl_sized = false;
  int last_engine = 0;    // 1 lane, 2 block, 3 cluster (ps_last_engine)
  SpectralState* spec = nullptr;
  int spec_N = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::mutex mu;
  PropParams last_params{};  // parameters of the last nonlinear propagation (phase probes)
  bool has_last_params = false;
};

namespace {

template <class T>
bool dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)) == cudaSuccess;
}

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Failure(PS_ERR_CUDA, std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

template <class Fn>
int guard(ps_ctx* ctx, Fn fn) {
  try {
    fn();
    return PS_OK;
  } catch (const Failure& f) {
    if (ctx) ctx->err = f.what();
    g_global_error = f.what();
    return f.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    g_global_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

// TimeMesh (proj/include/parasteady/types.hpp:21-40)
double coarse_dt(const ps_time_mesh& m) { return m.period / m.subintervals; }
double fine_dt(const ps_time_mesh& m) { return coarse_dt(m) / m.fine_steps; }
double boundary(const ps_time_mesh& m, int n) {
  if (n == m.subintervals) return m.period;
  return static_cast<double>(n) * m.period / m.subintervals;
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    throw Failure(PS_ERR_CUDA, "cuda: no CUDA device available (the B200 path has no CPU fallback)");
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) throw Failure(PS_ERR_CUDA, "cuda: this library is built for sm_100a (B200) only");
}

void validate_desc(const ps_problem_desc* d) {
  if (!d) throw Failure(PS_ERR_BAD_ARG, "problem: null description");
  if (d->dim < 1) throw Failure(PS_ERR_BAD_ARG, "problem: excitation dimension must be positive");
  if (!d->row_ptr || !d->col_idx || !d->mass) throw Failure(PS_ERR_BAD_ARG, "problem: missing CSR arrays");
  if (d->row_ptr[0] != 0 || d->row_ptr[d->dim] != d->nnz) throw Failure(PS_ERR_BAD_ARG, "problem: bad row_ptr");
  for (int i = 0; i < d->dim; ++i) {
    if (d->row_ptr[i + 1] < d->row_ptr[i]) throw Failure(PS_ERR_BAD_ARG, "problem: bad row_ptr");
    bool diag = false;
    for (int k = d->row_ptr[i]; k < d->row_ptr[i + 1]; ++k) {
      if (d->col_idx[k] < 0 || d->col_idx[k] >= d->dim) throw Failure(PS_ERR_BAD_ARG, "problem: column out of range");
      if (k > d->row_ptr[i] && d->col_idx[k] <= d->col_idx[k - 1])
        throw Failure(PS_ERR_BAD_ARG, "problem: columns must be sorted and unique");
      diag |= d->col_idx[k] == i;
    }
    if (!diag) throw Failure(PS_ERR_BAD_ARG, "problem: pattern must contain the diagonal");
  }
  if (!(d->period > 0.0)) throw Failure(PS_ERR_BAD_ARG, "problem: excitation period must be positive");
  // Excitation ctor (proj/src/problem.cpp:36-50)
  for (int k = 0; k < d->n_terms; ++k) {
    if (!(d->frequency_hz[k] > 0.0)) throw Failure(PS_ERR_BAD_ARG, "problem: excitation frequency must be positive");
    const double cycles = d->frequency_hz[k] * d->period;
    if (std::abs(cycles - std::round(cycles)) > 1e-9 * std::max(1.0, cycles))
      throw Failure(PS_ERR_BAD_ARG, "problem: excitation frequency is not an integer multiple of 1/period");
  }
  if (!d->stiffness) {
    if (d->nodes_per_elem != 2 && d->nodes_per_elem != 3)
      throw Failure(PS_ERR_BAD_ARG, "problem: nonlinear problems need 2- or 3-node elements");
    if (d->n_curves < 1 || d->n_curves > kMaxCurves) throw Failure(PS_ERR_BAD_ARG, "problem: 1..8 curves supported");
    for (int e = 0; e < d->n_elem; ++e)
      if (d->elem_curve[e] < 0 || d->elem_curve[e] >= d->n_curves)
        throw Failure(PS_ERR_BAD_ARG, "problem: element curve index out of range");
  }
}

template <class T>
T* upload(const T* src, size_t n, const char* what) {
  T* d = nullptr;
  if (!dalloc(&d, n)) throw Failure(PS_ERR_CUDA, std::string("cuda: out of memory for ") + what);
  if (n) check(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice), what);
  return d;
}

void build_problem(ps_ctx* ctx, const ps_problem_desc* desc) {
  DevProblem& P = ctx->P;
  P.d = desc->dim;
  P.nnz = desc->nnz;
  P.linear = desc->stiffness != nullptr;
  P.h_rp.assign(desc->row_ptr, desc->row_ptr + P.d + 1);
  P.h_ci.assign(desc->col_idx, desc->col_idx + P.nnz);
  P.h_M.assign(desc->mass, desc->mass + P.nnz);
  P.h_diag.resize(P.d);
  P.max_row_len = 0;
  for (int i = 0; i < P.d; ++i) {
    P.max_row_len = std::max(P.max_row_len, P.h_rp[i + 1] - P.h_rp[i]);
    for (int k = P.h_rp[i]; k < P.h_rp[i + 1]; ++k)
      if (P.h_ci[k] == i) P.h_diag[i] = k;
  }
  P.rp = upload(P.h_rp.data(), P.h_rp.size(), "row_ptr");
  P.ci = upload(P.h_ci.data(), P.h_ci.size(), "col_idx");
  P.diag = upload(P.h_diag.data(), P.h_diag.size(), "diag");
  P.M = upload(P.h_M.data(), P.h_M.size(), "mass");
  if (P.linear) {
    P.h_K.assign(desc->stiffness, desc->stiffness + P.nnz);
    P.K = upload(P.h_K.data(), P.h_K.size(), "stiffness");
  } else {
    P.npe = desc->nodes_per_elem;
    P.ne = desc->n_elem;
    const int npe = P.npe;
    const int64_t ne = P.ne;
    P.en = upload(desc->elem_nodes, ne * npe, "elements");
    P.eS = upload(desc->elem_stiff, ne * npe * npe, "element stiffness");
    P.einvA = upload(desc->elem_inv_area, ne, "element areas");
    P.ecurve = upload(desc->elem_curve, ne, "element curves");
    P.curves.assign(desc->curves, desc->curves + desc->n_curves);
    // node -> (element, local index) adjacency in increasing element order,
    // plus the slot offset of every (a, b) coupling within row a
    std::vector<int> cnt(P.d + 1, 0);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < npe; ++a) {
        const int n = desc->elem_nodes[e * npe + a];
        if (n >= 0) cnt[n + 1]++;
      }
    for (int i = 0; i < P.d; ++i) cnt[i + 1] += cnt[i];
    std::vector<int2> adj(cnt[P.d]);
    std::vector<int> rel(static_cast<size_t>(cnt[P.d]) * npe, -1);
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < ne; ++e)
      for (int a = 0; a < npe; ++a) {
        const int n = desc->elem_nodes[e * npe + a];
        if (n < 0) continue;
        const int q = fill[n]++;
        adj[q] = make_int2(static_cast<int>(e), a);
        for (int b = 0; b < npe; ++b) {
          const int nb = desc->elem_nodes[e * npe + b];
          if (nb < 0) continue;
          const auto first = P.h_ci.begin() + P.h_rp[n], last = P.h_ci.begin() + P.h_rp[n + 1];
          const auto it = std::lower_bound(first, last, nb);
          if (it == last || *it != nb) throw Failure(PS_ERR_BAD_ARG, "problem: element coupling missing from pattern");
          rel[static_cast<size_t>(q) * npe + b] = static_cast<int>(it - first);
        }
      }
    P.adj_ptr = upload(cnt.data(), cnt.size(), "adjacency");
    P.adj = upload(adj.data(), adj.size(), "adjacency");
    P.adj_rel = upload(rel.data(), rel.size(), "adjacency slots");
    // Rows whose adjacent elements all have a constant reluctivity have the same
    // step-matrix values M/dt + sum nu S_e in every system and every Newton
    // iterate: they are read from one shared copy (h_Kc) instead of per-system
    // values.  rowkind 1 marks rows touching a nonlinear (Brauer) element.
    P.h_rowkind.assign(P.d, 0);
    P.h_Kc.assign(P.nnz, 0.0);
    for (int64_t e = 0; e < ne; ++e) {
      const ps_curve& cv = desc->curves[desc->elem_curve[e]];
      for (int a = 0; a < npe; ++a) {
        const int na = desc->elem_nodes[e * npe + a];
        if (na < 0) continue;
        if (cv.kind != 0) {
          P.h_rowkind[na] = 1;
          continue;
        }
        for (int b = 0; b < npe; ++b) {
          const int nb = desc->elem_nodes[e * npe + b];
          if (nb < 0) continue;
          const auto first = P.h_ci.begin() + P.h_rp[na], last = P.h_ci.begin() + P.h_rp[na + 1];
          const int64_t slot = std::lower_bound(first, last, nb) - P.h_ci.begin();
          P.h_Kc[slot] += cv.nu * desc->elem_stiff[(e * npe + a) * npe + b];
        }
      }
    }
    P.rowkind = upload(P.h_rowkind.data(), P.h_rowkind.size(), "row kinds");
    P.Kc = upload(P.h_Kc.data(), P.h_Kc.size(), "constant stiffness");
  }
  {
    // row records (pppc_internal.h kEll)
    std::vector<int4> rec(static_cast<size_t>(P.d) * kRecInts4);
    for (int i = 0; i < P.d; ++i) {
      const int b = P.h_rp[i], len = P.h_rp[i + 1] - b;
      int c[kEll];
      for (int k = 0; k < kEll; ++k) c[k] = (k < len && len <= kEll) ? P.h_ci[b + k] : i;
      rec[kRecInts4 * i] = make_int4(b, len, P.linear ? 0 : P.h_rowkind[i], 0);
      rec[kRecInts4 * i + 1] = make_int4(c[0], c[1], c[2], c[3]);
      rec[kRecInts4 * i + 2] = make_int4(c[4], c[5], c[6], c[7]);
    }
    P.rowrec = upload(rec.data(), rec.size(), "row records");
    // padded per-row mass and shared stiffness values (refill of rows <= kEll)
    std::vector<double> me(static_cast<size_t>(P.d) * kEll, 0.0), ke(static_cast<size_t>(P.d) * kEll, 0.0);
    const std::vector<double>& Kref = P.linear ? P.h_K : P.h_Kc;
    for (int i = 0; i < P.d; ++i) {
      const int b = P.h_rp[i], len = P.h_rp[i + 1] - b;
      if (len > kEll) continue;
      for (int k = 0; k < len; ++k) {
        me[static_cast<size_t>(i) * kEll + k] = P.h_M[b + k];
        ke[static_cast<size_t>(i) * kEll + k] = Kref[b + k];
      }
    }
    P.ME = upload(me.data(), me.size(), "padded mass rows");
    P.KE = upload(ke.data(), ke.size(), "padded stiffness rows");
    // system-per-block engine: the same padded rows transposed ([kEll][d]) and the
    // padded columns; eligible when every row has <= kEll slots but at most one
    int longer = 0, hub = -1;
    for (int i = 0; i < P.d; ++i)
      if (P.h_rp[i + 1] - P.h_rp[i] > kEll) ++longer, hub = i;
    if (!P.linear && P.npe > 0 && longer <= 1) {
      std::vector<int> cT(static_cast<size_t>(P.d) * kEll);
      std::vector<double> mT(cT.size(), 0.0), kT(cT.size(), 0.0);
      for (int i = 0; i < P.d; ++i) {
        const int b = P.h_rp[i], len = P.h_rp[i + 1] - b;
        for (int k = 0; k < kEll; ++k) {
          const size_t t = static_cast<size_t>(k) * P.d + i;
          const bool slot = len <= kEll && k < len;
          cT[t] = slot ? P.h_ci[b + k] : i;
          mT[t] = slot ? P.h_M[b + k] : 0.0;
          kT[t] = slot ? Kref[b + k] : 0.0;
        }
      }
      P.ciT = upload(cT.data(), cT.size(), "padded columns");
      P.MT = upload(mT.data(), mT.size(), "padded mass columns");
      P.KT = upload(kT.data(), kT.size(), "padded stiffness columns");
      P.sb_ok = true;
      P.sb_hub = hub;
      for (int i = 0; i < P.d; ++i) {
        const int len = P.h_rp[i + 1] - P.h_rp[i];
        if (len <= kEll) P.ell_width = std::max(P.ell_width, len);
      }
      // Sparsity-pattern dictionary for the cluster engine: a row's pattern is its
      // length and its columns relative to the row (the hub's column, which every
      // neighbour of the hub holds, is flagged absolute instead).  Structured meshes have a
      // handful of patterns; the kPatMax - 1 most frequent get an id, the other
      // rows stay "irregular" and read their padded columns from memory.
      std::map<std::vector<int>, int> freq;
      auto key_of = [&](int i) {
        const int b = P.h_rp[i], len = P.h_rp[i + 1] - b;
        std::vector<int> key(2 + kEll, 0);
        int absmask = 0;
        for (int k = 0; k < len; ++k) {
          const int c = P.h_ci[b + k];
          if (c == hub && c != i) {
            absmask |= 1 << k;   // the entry stays 0: the column is the hub
          } else {
            key[2 + k] = c - i;
          }
        }
        key[0] = len;
        key[1] = absmask;
        return key;
      };
      for (int i = 0; i < P.d; ++i)
        if (P.h_rp[i + 1] - P.h_rp[i] <= kEll) ++freq[key_of(i)];
      std::vector<std::pair<int, std::vector<int>>> order;
      for (const auto& kv : freq) order.emplace_back(kv.second, kv.first);
      std::stable_sort(order.begin(), order.end(),
                       [](const auto& a, const auto& b) { return a.first > b.first; });
      std::map<std::vector<int>, int> ids;
      std::vector<int> pcols(static_cast<size_t>(kPatMax) * kEll, 0), pmeta(kPatMax, 0);
      for (size_t n = 0; n < order.size() && n < static_cast<size_t>(kPatIrregular); ++n) {
        ids[order[n].second] = static_cast<int>(n);
        for (int k = 0; k < kEll; ++k) pcols[n * kEll + k] = order[n].second[2 + k];
        pmeta[n] = order[n].second[0] | (order[n].second[1] << 8);
      }
      std::vector<unsigned char> pid(P.d, static_cast<unsigned char>(kPatIrregular));
      for (int i = 0; i < P.d; ++i) {
        if (P.h_rp[i + 1] - P.h_rp[i] > kEll) continue;
        const auto it = ids.find(key_of(i));
        if (it != ids.end()) pid[i] = static_cast<unsigned char>(it->second);
      }
      P.pat_id = upload(pid.data(), pid.size(), "pattern ids");
      P.pat_cols = upload(pcols.data(), pcols.size(), "pattern columns");
      P.pat_meta = upload(pmeta.data(), pmeta.size(), "pattern lengths");
    }
  }
  P.nterms = desc->n_terms;
  P.period = desc->period;
  P.amp.assign(desc->amplitude, desc->amplitude + P.nterms);
  P.freq.assign(desc->frequency_hz, desc->frequency_hz + P.nterms);
  P.phase.assign(desc->phase_rad, desc->phase_rad + P.nterms);
  P.pat = upload(desc->patterns, static_cast<size_t>(P.nterms) * P.d, "excitation patterns");
}

// Work vectors use the group-blocked layout [G][d][32] (G = ceil(max_batch/32)),
// which is also large enough to serve as interleaved [d][N] scratch.
size_t lanes_padded(const ps_ctx* ctx) { return static_cast<size_t>((ctx->max_batch + 31) / 32) * 32; }

void alloc_work(ps_ctx* ctx) {
  const size_t n = static_cast<size_t>(ctx->P.d) * lanes_padded(ctx);
  const size_t nio = static_cast<size_t>(ctx->P.d) * ctx->max_batch;
  bool ok = dalloc(&ctx->u, n) && dalloc(&ctx->uprev, n) && dalloc(&ctx->x, n) && dalloc(&ctx->r, n) &&
            dalloc(&ctx->p, n) && dalloc(&ctx->q, n) && dalloc(&ctx->io_a, nio) && dalloc(&ctx->io_b, nio);
  ok = ok && dalloc(&ctx->Dinv, n);
  if (!ctx->P.linear) ok = ok && dalloc(&ctx->A, static_cast<size_t>(ctx->P.nnz) * lanes_padded(ctx));
  ok = ok && dalloc(&ctx->abort_flag, 1) && dalloc(&ctx->out, ctx->max_batch) &&
       dalloc(&ctx->lockstep, (ctx->max_batch + 31) / 32 + 1);
  if (!ok) throw Failure(PS_ERR_CUDA, "cuda: out of device memory for the work vectors");
}

void ensure(double** buf, size_t* len, size_t need) {
  if (*len >= need) return;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  if (!dalloc(buf, need)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
  *len = need;
}

// Chunk-to-block rotation (kernels.cu warp_rows); PPPC_CHUNK_ROT, diagnostics only.
int chunk_rotation() {
  static const int rot = std::getenv("PPPC_CHUNK_ROT") ? std::atoi(std::getenv("PPPC_CHUNK_ROT")) : 0;
  return rot < 0 ? 0 : rot;
}

// Sequential group launches: the groups of a batch run one after another, each
// on every co-resident block (C from one group), and the PCG residual of a
// block's rows stays in shared memory.  PPPC_SEQ=0/1 overrides the default.
bool sequential_groups() {
  static const int v = std::getenv("PPPC_SEQ") ? std::atoi(std::getenv("PPPC_SEQ")) : 0;
  return v != 0;
}

Geometry& geometry(ps_ctx* ctx, int count) {
  auto it = ctx->geo.find(count);
  if (it != ctx->geo.end()) return it->second;
  // One warp lane per system (R = 1) and a block count C fixed by (d, max_batch):
  // every call on this context uses the same per-system reduction tree, so a
  // system's result is bitwise independent of how the batch is split
  // (proj/tests/test_engine.cpp:253-271 contract).
  Geometry g;
  g.G = (count + 31) / 32;
  g.L = (count + g.G - 1) / g.G;
  g.Lp = 32;
  g.R = 1;
  const int g_max = sequential_groups() ? 1 : (ctx->max_batch + 31) / 32;
  // at least rows_min rows per block: two rows per warp.  Small problems then
  // spread over more SMs (configs[0], d = 2,497: 79 blocks, fine sweep 969 ->
  // 832 ms against four rows per warp; one row per warp is slower again, the
  // barrier then dominates).  PPPC_ROWS_MIN overrides (diagnostics).
  static const int rows_min = std::getenv("PPPC_ROWS_MIN") ? std::max(1, std::atoi(std::getenv("PPPC_ROWS_MIN")))
                                                           : kWarps * 2;
  if (g_max > ctx->capacity) throw Failure(PS_ERR_BAD_ARG, "propagator: batch too large for one cooperative launch");
  g.C = std::max(1, std::min(ctx->capacity / g_max, (ctx->P.d + rows_min - 1) / rows_min));
  std::vector<int> ranges;
  row_ranges(ctx->P.h_rp, g.C, g.R, &ranges, &ctx->P.h_rowkind);
  g.warp_row_begin = upload(ranges.data(), ranges.size(), "row ranges");
  // rows in chunks of kWarps dealt round-robin to the C blocks (kernels.cu
  // warp_rows); a block holds at most ceil(chunks / C) chunks
  const int chunks = (ctx->P.d + kWarps - 1) / kWarps;
  g.max_block_rows = ((chunks + g.C - 1) / g.C) * kWarps;
  std::vector<int> lrows, lowner;
  for (int i = 0; i < ctx->P.d; ++i)
    if (ctx->P.h_rp[i + 1] - ctx->P.h_rp[i] > kLongRow) {
      lrows.push_back(i);
      lowner.push_back((i / kWarps + chunk_rotation()) % g.C);
    }
  g.n_long = static_cast<int>(lrows.size());
  g.long_rows = upload(lrows.data(), lrows.size(), "long rows");
  g.long_owner = upload(lowner.data(), lowner.size(), "long rows");
  return ctx->geo.emplace(count, g).first->second;
}

ps_ctx::StepMatrix shared_step_matrix(ps_ctx* ctx, double dt) {
  auto it = ctx->step_cache.find(dt);
  if (it != ctx->step_cache.end()) return it->second;
  const DevProblem& P = ctx->P;
  std::vector<double> A(P.nnz), D(P.d), AE(static_cast<size_t>(P.d) * kEll, 0.0);
  // linear problems: M/dt + K; element problems: M/dt + K_const (valid on rows
  // with rowkind 0, the only rows that read it)
  const std::vector<double>& Kref = P.linear ? P.h_K : P.h_Kc;
  for (int k = 0; k < P.nnz; ++k) A[k] = P.h_M[k] / dt + Kref[k];
  for (int i = 0; i < P.d; ++i) {
    D[i] = 1.0 / A[P.h_diag[i]];
    const int b = P.h_rp[i], len = P.h_rp[i + 1] - b;
    if (len <= kEll)
      for (int k = 0; k < len; ++k) AE[static_cast<size_t>(i) * kEll + k] = A[b + k];
  }
  ps_ctx::StepMatrix m;
  m.A = upload(A.data(), A.size(), "step matrix");
  m.D = upload(D.data(), D.size(), "jacobi");
  m.AE = upload(AE.data(), AE.size(), "step matrix rows");
  if (P.sb_ok) {
    std::vector<double> AT(AE.size());
    for (int i = 0; i < P.d; ++i)
      for (int k = 0; k < kEll; ++k) AT[static_cast<size_t>(k) * P.d + i] = AE[static_cast<size_t>(i) * kEll + k];
    m.AT = upload(AT.data(), AT.size(), "step matrix columns");
  }
  return ctx->step_cache.emplace(dt, m).first->second;
}

void excitation_coef(const DevProblem& P, double t, double* out) {
  // Excitation::operator() (proj/src/problem.cpp:52-63): same double expressions
  double tau = std::fmod(t, P.period);
  if (tau < 0.0) tau += P.period;
  for (int k = 0; k < P.nterms; ++k) {
    const double arg = 2.0 * kPi * P.freq[k] * tau + P.phase[k];
    out[k] = P.amp[k] * std::sin(arg);
  }
}

const char* failure_what(int code) {
  switch (code) {
    case PS_ERR_SINGULAR: return "step system singular";
    case PS_ERR_NEWTON_MAXITER: return "Newton did not converge";
    case PS_ERR_NEWTON_DIVERGED: return "Newton iteration diverged";
    case PS_ERR_PCG_MAXITER: return "PCG did not converge";
    default: return "step failed";
  }
}

struct PropResult {
  double* state = nullptr;  // interleaved result (stride = count)
};

// Row split and column windows of the system-per-cluster engine for C CTAs:
// balanced contiguous row ranges; a CTA's window spans its rows and every
// column they gather (the hub row included: its owner forms the whole product).
ClusterGeom cluster_split(const DevProblem& P, int C) {
  ClusterGeom g{};
  g.C = C;
  g.hub_len = P.sb_hub >= 0 ? P.h_rp[P.sb_hub + 1] - P.h_rp[P.sb_hub] : 0;
  for (int c = 0; c <= C; ++c) g.row_begin[c] = static_cast<int>(static_cast<int64_t>(P.d) * c / C);
  for (int c = 0; c < C; ++c) {
    const int r0 = g.row_begin[c], r1 = g.row_begin[c + 1];
    int lo = r0, hi = r1;
    for (int i = r0; i < r1; ++i) {
      for (int k = P.h_rp[i]; k < P.h_rp[i + 1]; ++k) {
        lo = std::min(lo, P.h_ci[k]);
        hi = std::max(hi, P.h_ci[k] + 1);
      }
    }
    g.win_lo[c] = lo;
    g.win_hi[c] = hi;
    g.rows_max = std::max(g.rows_max, r1 - r0);
    g.win_max = std::max(g.win_max, hi - lo);
  }
  return g;
}

// Picks the cluster size among every C whose CTA working set (p window, r, q,
// Jacobi) fits in shared memory and whose row range fits the per-thread row
// budget.  A system runs roughly C times faster on C CTAs and the context's batch
// (max_batch systems) takes ceil(max_batch / co-resident clusters) waves, so the
// score is C * max_batch / waves: configs[1] (100 systems, d = 50,945) -> C = 9
// (15 clusters at once, the only sizes that fit are 9..16); configs[0] (20 systems,
// d = 2,497) -> C = 6 (22 clusters at once: 2.57 s per 35 PP-PC iterations against
// 4.56 s at C = 1, 3.6 s at C = 7/8 where only 15 fit, 5.35 s with the block
// engine).  The size depends on the context (d, max_batch) only, never on the
// batch of one call, so a system's result is independent of how a batch is split.
// The smaller C wins ties.  PPPC_CLUSTER=C forces a size.
void cluster_geometry(ps_ctx* ctx) {
  if (ctx->cl_sized) return;
  ctx->cl_sized = true;
  const DevProblem& P = ctx->P;
  if (!P.sb_ok) return;
  int dev = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int forced = std::getenv("PPPC_CLUSTER") ? std::atoi(std::getenv("PPPC_CLUSTER")) : 0;
  const int batch = std::max(1, ctx->max_batch);
  double best_score = 0.0;
  for (int C = 1; C <= kClusterMaxC; ++C) {
    if (forced > 0 && C != forced) continue;
    if (C > P.d) break;
    const ClusterGeom g = cluster_split(P, C);
    if (g.rows_max > syscluster_max_rows() || syscluster_smem(g) > static_cast<size_t>(smem_max)) continue;
    const int slots = syscluster_max_clusters(P.npe, P.ell_width, g);
    if (slots < 1) continue;
    const int waves = (batch + slots - 1) / slots;
    const double score = static_cast<double>(C) * batch / waves;
    if (score > best_score) {
      best_score = score;
      ctx->cl_geo = g;
      ctx->cl_slots = slots;
    }
  }
  if (std::getenv("PPPC_DEBUG_TIMING") && ctx->cl_geo.C > 0)
    std::fprintf(stderr, "[pppc cluster] C = %d, rows/CTA %d, window %d, smem %zu B, %d co-resident clusters\n",
                 ctx->cl_geo.C, ctx->cl_geo.rows_max, ctx->cl_geo.win_max, syscluster_smem(ctx->cl_geo),
                 ctx->cl_slots);
}

// Fine-propagation engine for a nonlinear element problem.
//   cluster (syscluster_kernel): one thread-block cluster of C CTAs per system,
//           Krylov vectors in the cluster's shared memory, DSMEM halo exchange and
//           sums; the default whenever the pattern qualifies (DevProblem::sb_ok) and
//           some cluster size holds a CTA's working set on chip (configs[0],
//           d = 2,497, C = 6; configs[1], d = 50,945, C = 9);
//   block   (sysblock_kernel): one block per system, block barriers only, the
//           seven vectors in one block's shared memory (small systems);
//   lane    (propagate_kernel): one warp lane per system, groups of blocks with
//           device-wide group barriers, vectors in HBM; any size (configs[3]/[4]).
// ps_solver_settings.engine (1 lane, 2 block, 3 cluster) or PPPC_ENGINE=lane|sys|cluster
// forces one; the pattern must qualify for block and cluster.
enum class Engine { Lane, Block, Cluster };
Engine select_engine(ps_ctx* ctx, bool linear_path, bool probe_refill) {
  if (linear_path || probe_refill || !ctx->P.sb_ok) return Engine::Lane;
  const int e = ctx->settings.engine;
  if (e == 1) return Engine::Lane;
  if (e == 2) return Engine::Block;
  const char* env = std::getenv("PPPC_ENGINE");
  if (e == 0 && env && std::strcmp(env, "lane") == 0) return Engine::Lane;
  if (e == 0 && env && std::strcmp(env, "sys") == 0) return Engine::Block;
  cluster_geometry(ctx);
  if (ctx->cl_geo.C > 0) return Engine::Cluster;
  if (e == 3) throw Failure(PS_ERR_BAD_ARG, "propagator: the cluster engine cannot hold this system on chip");
  if (sysblock_smem(ctx->P.d) <= kSbSmemMax) return Engine::Block;
  return Engine::Lane;
}

// Runs `steps` implicit-Euler steps of size dt for `count` systems whose
// start states are in ctx->u (interleaved, stride count).  t_next is
// [steps][count].  newton_mode: run Newton even for linear problems
// (newton_step semantics) instead of the linear fast path.
PropResult propagate(ps_ctx* ctx, int count, int steps, double dt, const std::vector<double>& t_next,
                     bool newton_mode, bool want_trace, ps_batch_status* status, bool probe_refill = false) {
  const DevProblem& P = ctx->P;
  if (count < 1 || count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "propagator: batch count out of range");
  if (!(dt > 0.0)) throw Failure(PS_ERR_BAD_ARG, "propagator: step size must be positive");
  const ps_solver_settings& S = ctx->settings;
  if (S.newton.max_iter < 1) throw Failure(PS_ERR_BAD_ARG, "propagator: Newton needs at least one iteration");
  Geometry& geo = geometry(ctx, count);
  const bool linear_path = P.linear && !newton_mode;
  if (!linear_path && !ctx->A && !dalloc(&ctx->A, static_cast<size_t>(P.nnz) * lanes_padded(ctx)))
    throw Failure(PS_ERR_CUDA, "cuda: out of device memory for the step matrices");
  const int nt = std::max(1, P.nterms);
  std::vector<double> coef(static_cast<size_t>(steps) * count * nt, 0.0);
  for (int j = 0; j < steps; ++j)
    for (int n = 0; n < count; ++n)
      excitation_coef(P, t_next[static_cast<size_t>(j) * count + n], &coef[(static_cast<size_t>(j) * count + n) * nt]);
  ensure(&ctx->coef, &ctx->coef_len, coef.size());
  ensure(&ctx->tnext, &ctx->tnext_len, t_next.size());
  check(cudaMemcpyAsync(ctx->coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
        "coef upload");
  check(cudaMemcpyAsync(ctx->tnext, t_next.data(), t_next.size() * sizeof(double), cudaMemcpyHostToDevice,
                        ctx->stream),
        "t upload");
  const size_t plen = static_cast<size_t>(2) * geo.G * geo.C * kNDots * 32;
  ensure(&ctx->partials, &ctx->partials_len, plen);
  if (!ctx->sync && !dalloc(&ctx->sync, 64)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
  if (geo.G > 64) throw Failure(PS_ERR_BAD_ARG, "propagator: batch too large");
  if (want_trace) {
    if (ctx->trace) cudaFree(ctx->trace);
    if (!dalloc(&ctx->trace, static_cast<size_t>(count) * S.newton.max_iter))
      throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    check(cudaMemsetAsync(ctx->trace, 0, static_cast<size_t>(count) * S.newton.max_iter * sizeof(double), ctx->stream),
          "trace");
  }
  check(cudaMemsetAsync(ctx->sync, 0, geo.G * sizeof(unsigned long long), ctx->stream), "sync reset");
  check(cudaMemsetAsync(ctx->abort_flag, 0, sizeof(int), ctx->stream), "abort reset");

  PropParams K{};
  K.d = P.d;
  K.nnz = P.nnz;
  K.stride = count;
  K.count = count;
  K.G = geo.G;
  K.C = geo.C;
  K.L = geo.L;
  K.Lp = geo.Lp;
  K.R = geo.R;
  K.warp_row_begin = geo.warp_row_begin;
  K.n_long = geo.n_long;
  K.long_rows = geo.long_rows;
  K.long_owner = geo.long_owner;
  K.rp = P.rp;
  K.ci = P.ci;
  K.diag = P.diag;
  K.rowrec = P.rowrec;
  K.ME = P.ME;
  K.KE = P.KE;
  K.chunk_rot = chunk_rotation();
  K.g_base = 0;
  K.hub_split = (geo.n_long == 1 && std::getenv("PPPC_NO_HUB_SPLIT") == nullptr) ? 1 : 0;
  K.probe_refill = probe_refill ? 1 : 0;
  {
    // phase-A L2 prefetch distance in rows, PPPC_PF (default 0 = off: it helps
    // the standalone phase probe but not the persistent kernel)
    static const int pf = std::getenv("PPPC_PF") ? std::atoi(std::getenv("PPPC_PF")) : 0;
    K.pf_dist = pf < 0 ? 0 : pf;
  }
  K.rec_rows = geo.max_block_rows * kRecInts4 * sizeof(int4) <= kRecSmemMax ? geo.max_block_rows : 0;
  // residual rows in shared memory when records + residual fit the opted-in size
  K.r_smem = (sequential_groups() && K.rec_rows > 0 &&
              static_cast<size_t>(K.rec_rows) * (kRecInts4 * sizeof(int4) + 32 * sizeof(double)) <= kRecSmemMax)
                 ? 1
                 : 0;
  K.M = P.M;
  K.Klin = P.K;
  K.Kc = P.Kc;
  {
    // shared step matrix M/dt + K (linear) or M/dt + K_const (constant-nu rows)
    const auto sm = shared_step_matrix(ctx, dt);
    K.Ash = sm.A;
    K.Dsh = sm.D;
    K.AshE = sm.AE;
  }
  // rows with per-system values: every row under newton_step on a linear problem
  // uses the shared matrix (J = K), element problems by rowkind
  K.rowkind = P.linear ? nullptr : P.rowkind;
  K.adj_ptr = P.adj_ptr;
  K.adj = P.adj;
  K.adj_rel = P.adj_rel;
  K.en = P.en;
  K.eS = P.eS;
  K.einvA = P.einvA;
  K.ecurve = P.ecurve;
  K.ncurves = static_cast<int>(P.curves.size());
  for (int k = 0; k < K.ncurves; ++k) K.curves[k] = P.curves[k];
  K.nterms = P.nterms;
  K.pat = P.pat;
  K.coef = ctx->coef;
  K.t_next = ctx->tnext;
  K.steps = steps;
  K.dt = dt;
  K.u = ctx->u;
  K.uprev = ctx->uprev;
  K.ubuf0 = ctx->u;
  K.ubuf1 = ctx->uprev;
  K.x = ctx->x;
  K.r = ctx->r;
  K.p = ctx->p;
  K.q = ctx->q;
  K.Dinv = ctx->Dinv;
  K.A = ctx->A;
  K.newton_tol_abs = S.newton.tol_abs;
  K.newton_tol_rel = S.newton.tol_rel;
  K.damping = S.newton.damping;
  K.newton_max = S.newton.max_iter;
  K.line_search = S.newton.line_search;
  K.pcg_tol = S.pcg.tol_rel;
  K.pcg_max = S.pcg.max_iter;
  K.sync = ctx->sync;
  K.partials = ctx->partials;
  K.abort_flag = ctx->abort_flag;
  K.out = ctx->out;
  K.trace = want_trace ? ctx->trace : nullptr;
  K.lockstep = ctx->lockstep;
  ctx->last_params = K;
  ctx->last_params.r_smem = 0;  // phase probes keep r in global memory
  ctx->has_last_params = !linear_path;

  const int npe = P.linear ? 0 : P.npe;
  // PPPC_DEBUG_TIMING=1: per-block work / barrier-wait timing summary on stderr
  static const bool debug_timing = std::getenv("PPPC_DEBUG_TIMING") != nullptr;
  unsigned long long* dbg = nullptr;
  const int nblk = geo.G * geo.C;
  const Engine engine = select_engine(ctx, linear_path, probe_refill);
  const bool sysblock = engine != Engine::Lane;
  ctx->last_engine = engine == Engine::Lane ? 1 : engine == Engine::Block ? 2 : 3;
  if (debug_timing && !sysblock && dalloc(&dbg, static_cast<size_t>(nblk) * kDbgSlots)) K.dbg = dbg;
  unsigned long long* cl_dbg = nullptr;
  if (debug_timing && engine == Engine::Cluster &&
      dalloc(&cl_dbg, static_cast<size_t>(count) * ctx->cl_geo.C * 8)) {
    cudaMemsetAsync(cl_dbg, 0, static_cast<size_t>(count) * ctx->cl_geo.C * 8 * sizeof(unsigned long long), ctx->stream);
    K.dbg = cl_dbg;
  }
  // The SpMV gathers the search direction p at +-ntheta rows; keep p resident in
  // L2 (persisting access-policy window) so the streamed matrix values and
  // vectors do not evict it between neighbour reads.  PPPC_NO_L2_PERSIST=1 off.
  static const bool l2_persist = std::getenv("PPPC_NO_L2_PERSIST") == nullptr;
  if (l2_persist) {
    int dev = 0, max_persist = 0, max_window = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    const size_t pbytes = static_cast<size_t>(geo.G) * P.d * 32 * sizeof(double);
    if (max_persist > 0 && max_window > 0) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(max_persist, pbytes));
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = ctx->p;
      attr.accessPolicyWindow.num_bytes = std::min<size_t>(pbytes, static_cast<size_t>(max_window));
      attr.accessPolicyWindow.hitRatio =
          std::min(1.0f, static_cast<float>(max_persist) / static_cast<float>(attr.accessPolicyWindow.num_bytes));
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
      cudaGetLastError();
    }
  }
  check(cudaEventRecord(ctx->e0, ctx->stream), "event");
  std::string err;
  if (sysblock) {
    ensure(&ctx->sb_u, &ctx->sb_u_len, static_cast<size_t>(count) * P.d);
    ensure(&ctx->sb_A, &ctx->sb_A_len, static_cast<size_t>(count) * kEll * P.d);
    SysParams sp{};
    sp.su = ctx->sb_u;
    sp.sA = ctx->sb_A;
    sp.hub = P.sb_hub;
    sp.hub_len = P.sb_hub >= 0 ? P.h_rp[P.sb_hub + 1] - P.h_rp[P.sb_hub] : 0;
    if (sp.hub >= 0) {
      ensure(&ctx->sb_hub, &ctx->sb_hub_len, static_cast<size_t>(count) * sp.hub_len);
      sp.hubA = ctx->sb_hub;
    }
    sp.ciT = P.ciT;
    sp.pat_id = P.pat_id;
    sp.pat_cols = P.pat_cols;
    sp.pat_meta = P.pat_meta;
    sp.ell_width = P.ell_width;
    sp.MT = P.MT;
    sp.KT = P.KT;
    sp.AshT = shared_step_matrix(ctx, dt).AT;
    static const bool no_smem = std::getenv("PPPC_SB_NO_SMEM") != nullptr;
    sp.smem_vectors = (engine == Engine::Block && !no_smem && sysblock_smem(P.d) <= kSbSmemMax) ? 1 : 0;
    check(cudaMemsetAsync(ctx->lockstep, 0, geo.G * sizeof(int64_t), ctx->stream), "lockstep reset");
    check(cudaEventRecord(ctx->e0, ctx->stream), "event");
    const int rc = engine == Engine::Cluster ? launch_syscluster(K, sp, ctx->cl_geo, npe, ctx->stream, &err)
                                             : launch_sysblock(K, sp, npe, ctx->stream, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  } else if (sequential_groups() && geo.G > 1) {
    // one launch per group, each on all C blocks, own arrival counter
    for (int gg = 0; gg < geo.G; ++gg) {
      PropParams Kg = K;
      Kg.G = 1;
      Kg.g_base = gg;
      Kg.sync = K.sync + gg;
      if (K.dbg) Kg.dbg = K.dbg + static_cast<size_t>(gg) * geo.C * kDbgSlots;
      const int rc = launch_propagate(Kg, linear_path, npe, ctx->stream, &err);
      if (rc != PS_OK) throw Failure(rc, err);
    }
  } else {
    const int rc = launch_propagate(K, linear_path, npe, ctx->stream, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  }
  check(cudaEventRecord(ctx->e1, ctx->stream), "event");
  if (cl_dbg) {
    // cluster engine: mean cycles per PCG iteration of the four parts, over all CTAs
    std::vector<unsigned long long> h(static_cast<size_t>(count) * ctx->cl_geo.C * 8);
    check(cudaMemcpyAsync(h.data(), cl_dbg, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "dbg");
    check(cudaStreamSynchronize(ctx->stream), "dbg");
    cudaFree(cl_dbg);
    K.dbg = nullptr;
    double tm[4] = {0, 0, 0, 0}, its = 0;
    for (size_t b = 0; b < h.size() / 8; ++b) {
      for (int k = 0; k < 4; ++k) tm[k] += static_cast<double>(h[b * 8 + k]);
      its += static_cast<double>(h[b * 8 + 4]);
    }
    if (its > 0)
      std::fprintf(stderr,
                   "[pppc cluster timing] cycles per PCG iteration: SpMV pass %.0f, cluster sum %.0f, update pass %.0f, "
                   "halo wait %.0f\n",
                   tm[0] / its, tm[1] / its, tm[2] / its, tm[3] / its);
  }
  std::vector<unsigned long long> h_dbg;
  if (K.dbg) {
    constexpr int W = kDbgSlots;
    std::vector<unsigned long long>& h = h_dbg;
    h.resize(static_cast<size_t>(nblk) * W);
    check(cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream), "dbg");
    check(cudaStreamSynchronize(ctx->stream), "dbg");
    cudaFree(dbg);
    const char* names[3] = {"A (no refill)", "B+other (no refill)", "with refill"};
    for (int kind = 0; kind < 3; ++kind) {
      double work = 0, wait = 0, wmin = 1e300, wmax = 0, n = 0;
      for (int b = 0; b < nblk; ++b) {
        const double cnt = static_cast<double>(h[b * W + 3 * kind + 2]);
        if (cnt == 0) continue;
        const double w = h[b * W + 3 * kind] / cnt;
        work += h[b * W + 3 * kind];
        wait += h[b * W + 3 * kind + 1];
        n += cnt;
        wmin = std::min(wmin, w);
        wmax = std::max(wmax, w);
      }
      double rel = 0;
      for (int b = 0; b < nblk; ++b) rel += static_cast<double>(h[b * W + 18 + kind]);
      if (n > 0)
        std::fprintf(stderr,
                     "[pppc timing] %s: %.0f intervals/block, work %.2f us (block min %.2f max %.2f), wait %.2f us "
                     "(arrival -> release seen %.2f us)\n",
                     names[kind], n / nblk, work / n / 1e3, wmin / 1e3, wmax / 1e3, wait / n / 1e3, rel / n / 1e3);
      if (std::getenv("PPPC_DEBUG_BLOCKS")) {
        std::fprintf(stderr, "[pppc blocks %s]", names[kind]);
        for (int b = 0; b < nblk; ++b) {
          const double cnt = static_cast<double>(h[b * W + 3 * kind + 2]);
          std::fprintf(stderr, " %.0f", cnt > 0 ? h[b * W + 3 * kind] / cnt / 1e3 : 0.0);
        }
        std::fprintf(stderr, "\n");
      }
    }
  }
  if (K.dbg) {
    // lane-interval shares per action, block 0 of every group
    const char* an[9] = {"idle", "R0", "A", "B", "U", "R", "L0", "LU", "wait"};
    for (int gg = 0; gg < geo.G; ++gg) {
      const unsigned long long* hb = h_dbg.data() + static_cast<size_t>(gg) * geo.C * kDbgSlots;
      double tot = 0;
      for (int a = 0; a < 9; ++a) tot += static_cast<double>(hb[9 + a]);
      std::fprintf(stderr, "[pppc actions g%d] lane-intervals %.0f:", gg, tot);
      for (int a = 0; a < 9; ++a)
        if (hb[9 + a]) std::fprintf(stderr, " %s %.3f", an[a], hb[9 + a] / tot);
      std::fprintf(stderr, "\n");
    }
  }
  std::vector<SysOut> outs(count);
  std::vector<int64_t> lock(geo.G);
  int abort_h = 0;
  check(cudaMemcpyAsync(outs.data(), ctx->out, count * sizeof(SysOut), cudaMemcpyDeviceToHost, ctx->stream), "status");
  check(cudaMemcpyAsync(lock.data(), ctx->lockstep, geo.G * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream),
        "status");
  check(cudaMemcpyAsync(&abort_h, ctx->abort_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "status");
  check(cudaStreamSynchronize(ctx->stream), "propagation kernel");
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, ctx->e0, ctx->e1);
  if (abort_h) throw Failure(PS_ERR_WATCHDOG, "cuda: device barrier watchdog fired in the propagation kernel");
  if (K.dbg)
    for (int gg = 0; gg < geo.G; ++gg) {
      int64_t pmax = 0, psum = 0;
      int nl = 0;
      for (int l = 0; l < geo.L && gg * geo.L + l < count; ++l, ++nl) {
        pmax = std::max<int64_t>(pmax, outs[gg * geo.L + l].pcg_total);
        psum += outs[gg * geo.L + l].pcg_total;
      }
      std::fprintf(stderr, "[pppc group g%d] intervals %lld, lanes %d, pcg per lane max %lld mean %.0f\n", gg,
                   static_cast<long long>(lock[gg]), nl, static_cast<long long>(pmax), nl ? double(psum) / nl : 0.0);
    }

  ps_batch_status st{};
  st.failed_index = -1;
  const double d = P.d, nnz = P.nnz;
  double bytes = 0.0;
  for (int n = 0; n < count; ++n) {
    const SysOut& o = outs[n];
    st.newton_iterations += o.newton_total;
    st.pcg_iterations += o.pcg_total;
    st.max_newton_iterations = std::max(st.max_newton_iterations, o.max_newton);
    st.max_pcg_iterations = std::max(st.max_pcg_iterations, o.max_pcg);
    // canonical bytes: Jacobi-PCG iteration Nb(8 nnz + 80 d) (+ shared
    // 4 nnz + 4(d+1) per batched iteration); fused refill Nb(8 nnz + 48 d) per Newton
    // iterate; the linear path reads one shared matrix (8 nnz per batched iteration).
    if (linear_path) {
      bytes += static_cast<double>(o.pcg_total) * 80.0 * d;
    } else {
      bytes += static_cast<double>(o.pcg_total) * (8.0 * nnz + 80.0 * d);
      bytes += static_cast<double>(o.newton_total + steps) * (8.0 * nnz + 48.0 * d);
    }
    if (o.code != PS_OK && st.code == PS_OK) {
      st.code = o.code;
      st.failed_index = n;
      st.t_next = o.t_fail;
      st.residual = o.residual;
    }
  }
  for (int g = 0; g < geo.G; ++g) {
    st.lockstep_pcg_iterations += lock[g];
    bytes += static_cast<double>(lock[g]) * ((linear_path ? 12.0 : 4.0) * nnz + 4.0 * (d + 1.0));
  }
  st.algorithmic_bytes = bytes;
  st.kernel_ms = ms;
  if (status) *status = st;
  if (st.code != PS_OK) {
    std::ostringstream msg;
    msg << "propagator: " << failure_what(st.code) << " at t = " << st.t_next << " (residual " << st.residual << ")";
    throw Failure(st.code, msg.str());
  }
  PropResult res;
  res.state = linear_path ? ((steps & 1) ? ctx->uprev : ctx->u) : ctx->u;
  return res;
}

__global__ void copy_column_kernel(const double* src, int src_stride, int src_col, double* dst, int dst_stride,
                                   int dst_col, int d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) dst[static_cast<size_t>(i) * dst_stride + dst_col] = src[static_cast<size_t>(i) * src_stride + src_col];
}

void copy_column(const double* src, int src_stride, int src_col, double* dst, int dst_stride, int dst_col, int d,
                 cudaStream_t st) {
  copy_column_kernel<<<(d + 255) / 256, 256, 0, st>>>(src, src_stride, src_col, dst, dst_stride, dst_col, d);
}

std::vector<double> fine_times(const ps_time_mesh& m, int n_first, int count) {
  const int s = m.fine_steps;
  std::vector<double> t(static_cast<size_t>(s) * count);
  const double dt = fine_dt(m);
  for (int i = 0; i < count; ++i) {
    const int n = n_first + i;
    const double t_left = boundary(m, n - 1);
    for (int j = 1; j <= s; ++j)
      t[static_cast<size_t>(j - 1) * count + i] = j == s ? boundary(m, n) : t_left + j * dt;
  }
  return t;
}

void check_range(const ps_time_mesh& m, int n_first, int count) {
  if (count < 1 || n_first < 1 || n_first + count - 1 > m.subintervals)
    throw Failure(PS_ERR_BAD_ARG, "propagator: subinterval index out of range");
}

int lanes_per_group(int count) {
  const int G = (count + 31) / 32;
  return (count + G - 1) / G;
}

// host [count][d] -> ctx->u group-blocked (the propagation kernels' layout)
void stage_in_host(ps_ctx* ctx, const double* U, int count) {
  const size_t n = static_cast<size_t>(count) * ctx->P.d;
  check(cudaMemcpyAsync(ctx->io_a, U, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
  launch_to_blocked(ctx->io_a, ctx->u, count, ctx->P.d, lanes_per_group(count), ctx->stream);
}
void stage_in_dev(ps_ctx* ctx, const double* dU, int count) {
  launch_to_blocked(dU, ctx->u, count, ctx->P.d, lanes_per_group(count), ctx->stream);
}
void stage_out_blocked(ps_ctx* ctx, const double* blocked, double* U, int count) {
  const size_t n = static_cast<size_t>(count) * ctx->P.d;
  launch_from_blocked(blocked, ctx->io_b, count, ctx->P.d, lanes_per_group(count), ctx->stream);
  check(cudaMemcpyAsync(U, ctx->io_b, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  check(cudaStreamSynchronize(ctx->stream), "D2H");
}
// interleaved [d][count] -> host [count][d]
void stage_out_host(ps_ctx* ctx, const double* il, double* U, int count) {
  const size_t n = static_cast<size_t>(count) * ctx->P.d;
  launch_from_interleaved(il, ctx->io_b, count, ctx->P.d, count, ctx->stream);
  check(cudaMemcpyAsync(U, ctx->io_b, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
  check(cudaStreamSynchronize(ctx->stream), "D2H");
}

int create_ctx(const ps_problem_desc* desc, const ps_time_mesh* mesh, const ps_solver_settings* settings, void* stream,
               ps_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<ps_ctx>();
  const int rc = guard(ctx.get(), [&] {
    require_device();
    validate_desc(desc);
    if (!mesh) throw Failure(PS_ERR_BAD_ARG, "mesh: null");
    if (mesh->subintervals < 2) throw Failure(PS_ERR_BAD_ARG, "mesh: need at least 2 subintervals");
    if (mesh->fine_steps < 1) throw Failure(PS_ERR_BAD_ARG, "mesh: need at least 1 fine step per subinterval");
    if (!(mesh->period > 0.0)) throw Failure(PS_ERR_BAD_ARG, "mesh: period must be positive");
    if (desc->period != mesh->period)
      throw Failure(PS_ERR_BAD_ARG, "propagator: mesh period does not match the problem");
    ctx->mesh = *mesh;
    if (settings) {
      ctx->settings = *settings;
    } else {
      ps_default_settings(&ctx->settings);
    }
    if (ctx->settings.engine < 0 || ctx->settings.engine > 3)
      throw Failure(PS_ERR_BAD_ARG, "propagator: engine must be 0 (by size), 1 (lane), 2 (block) or 3 (cluster)");
    ctx->max_batch = ctx->settings.max_batch > 0 ? ctx->settings.max_batch : mesh->subintervals;
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
      ctx->own_stream = true;
    }
    check(cudaEventCreate(&ctx->e0), "event");
    check(cudaEventCreate(&ctx->e1), "event");
    build_problem(ctx.get(), desc);
    int cap = 0;
    if (max_coresident_blocks(ctx->P.linear, ctx->P.linear ? 0 : ctx->P.npe, &cap) != PS_OK || cap < 1)
      throw Failure(PS_ERR_CUDA, "cuda: cannot size the cooperative propagation kernel");
    ctx->capacity = cap;
    alloc_work(ctx.get());
  });
  if (rc != PS_OK) {
    g_global_error = ctx->err;
    ps_destroy(ctx.release());
    return rc;
  }
  *out = ctx.release();
  return PS_OK;
}

}  // namespace

extern "C" {

int ps_default_settings(ps_solver_settings* out) {
  if (!out) return PS_ERR_BAD_ARG;
  std::memset(out, 0, sizeof(*out));
  out->newton.tol_abs = 1e-9;
  out->newton.tol_rel = 1e-8;
  out->newton.max_iter = 30;
  out->newton.damping = 1.0;
  out->newton.line_search = 0;
  out->pcg.tol_rel = 1e-12;
  out->pcg.max_iter = 20000;
  out->cocg.tol_rel = 1e-12;
  out->cocg.max_iter = 20000;
  out->max_batch = 0;
  return PS_OK;
}

const char* ps_global_error(void) { return g_global_error.c_str(); }

int ps_device_info(char* name, int name_len, int* sm_count, int* cc_major, int* cc_minor) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    g_global_error = "cuda: no CUDA device available";
    return PS_ERR_CUDA;
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, 0) != cudaSuccess) return PS_ERR_CUDA;
  if (name && name_len > 0) {
    std::strncpy(name, prop.name, name_len - 1);
    name[name_len - 1] = 0;
  }
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return PS_OK;
}

int ps_create(const ps_problem_desc* problem, const ps_time_mesh* mesh, const ps_solver_settings* settings,
              void* stream, ps_ctx** out) {
  if (!out) return PS_ERR_BAD_ARG;
  return create_ctx(problem, mesh, settings, stream, out);
}

void ps_destroy(ps_ctx* ctx) {
  if (!ctx) return;
  DevProblem& P = ctx->P;
  void* ptrs[] = {P.rowrec, P.ME, P.KE, P.rowkind, P.Kc, P.rp, P.ci, P.diag, P.M, P.K, P.adj_ptr, P.adj, P.adj_rel, P.en, P.eS, P.einvA, P.ecurve,
                  P.pat, ctx->u, ctx->uprev, ctx->x, ctx->r, ctx->p, ctx->q, ctx->Dinv, ctx->A, ctx->io_a,
                  ctx->io_b, ctx->sync, ctx->partials, ctx->abort_flag, ctx->out, ctx->trace, ctx->lockstep,
                  ctx->coef, ctx->tnext};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& kv : ctx->geo) {
    cudaFree(kv.second.warp_row_begin);
    cudaFree(kv.second.long_rows);
    cudaFree(kv.second.long_owner);
  }
  for (auto& kv : ctx->step_cache) {
    cudaFree(kv.second.A);
    cudaFree(kv.second.D);
    cudaFree(kv.second.AE);
    if (kv.second.AT) cudaFree(kv.second.AT);
  }
  void* sb[] = {P.ciT, P.MT, P.KT, ctx->sb_u, ctx->sb_A, ctx->sb_hub, P.pat_id, P.pat_cols, P.pat_meta};
  for (void* q : sb)
    if (q) cudaFree(q);
  if (ctx->spec) spectral_free(ctx->spec);
  if (ctx->e0) cudaEventDestroy(ctx->e0);
  if (ctx->e1) cudaEventDestroy(ctx->e1);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* ps_last_error(const ps_ctx* ctx) { return ctx ? ctx->err.c_str() : g_global_error.c_str(); }

int ps_last_engine(const ps_ctx* ctx, int32_t* engine, int32_t* cluster_ctas, int32_t* coresident_clusters) {
  if (!ctx) return PS_ERR_BAD_ARG;
  if (engine) *engine = ctx->last_engine;
  if (cluster_ctas) *cluster_ctas = ctx->last_engine == 3 ? ctx->cl_geo.C : 0;
  if (coresident_clusters) *coresident_clusters = ctx->last_engine == 3 ? ctx->cl_slots : 0;
  return PS_OK;
}
int ps_dim(const ps_ctx* ctx) { return ctx ? ctx->P.d : -1; }
int ps_is_linear(const ps_ctx* ctx) { return ctx && ctx->P.linear ? 1 : 0; }

// frozen_coarse_linearization (proj/src/engine.cpp:66-74)
int ps_create_frozen(ps_ctx* ctx, const double* u_ref, ps_ctx** out) {
  if (!ctx || !out) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    const DevProblem& P = ctx->P;
    std::vector<double> K(P.nnz);
    if (P.linear) {
      K = P.h_K;
    } else {
      double* dref = nullptr;
      double* dK = nullptr;
      if (!dalloc(&dref, P.d) || !dalloc(&dK, P.nnz)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
      if (u_ref)
        check(cudaMemcpy(dref, u_ref, P.d * sizeof(double), cudaMemcpyHostToDevice), "u_ref");
      else
        check(cudaMemset(dref, 0, P.d * sizeof(double)), "u_ref");
      launch_frozen_K(P, dref, dK, ctx->stream);
      check(cudaStreamSynchronize(ctx->stream), "frozen K");
      check(cudaMemcpy(K.data(), dK, P.nnz * sizeof(double), cudaMemcpyDeviceToHost), "frozen K");
      cudaFree(dref);
      cudaFree(dK);
    }
    ps_problem_desc desc{};
    desc.dim = P.d;
    desc.nnz = P.nnz;
    desc.row_ptr = P.h_rp.data();
    desc.col_idx = P.h_ci.data();
    desc.mass = P.h_M.data();
    desc.stiffness = K.data();
    desc.period = P.period;
    desc.n_terms = P.nterms;
    std::vector<double> pat(static_cast<size_t>(P.nterms) * P.d);
    if (!pat.empty())
      check(cudaMemcpy(pat.data(), P.pat, pat.size() * sizeof(double), cudaMemcpyDeviceToHost), "patterns");
    desc.patterns = pat.data();
    desc.amplitude = P.amp.data();
    desc.frequency_hz = P.freq.data();
    desc.phase_rad = P.phase.data();
    ps_solver_settings s = ctx->settings;
    const int rc = create_ctx(&desc, &ctx->mesh, &s, ctx->own_stream ? nullptr : ctx->stream, out);
    if (rc != PS_OK) throw Failure(rc, g_global_error);
  });
}

int ps_newton_step(ps_ctx* ctx, int32_t count, const double* U_prev, const double* t_next, double dt, double* U_out,
                   int32_t* iterations, double* residual_norms, ps_batch_status* status) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (count < 1 || count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "propagator: batch count out of range");
    stage_in_host(ctx, U_prev, count);
    std::vector<double> t(t_next, t_next + count);
    ps_batch_status st{};
    PropResult res;
    try {
      res = propagate(ctx, count, 1, dt, t, true, residual_norms != nullptr, &st);
    } catch (...) {
      if (status) *status = st;
      throw;
    }
    if (status) *status = st;
    stage_out_blocked(ctx, res.state, U_out, count);
    if (iterations || residual_norms) {
      std::vector<SysOut> outs(count);
      check(cudaMemcpy(outs.data(), ctx->out, count * sizeof(SysOut), cudaMemcpyDeviceToHost), "status");
      if (iterations)
        for (int n = 0; n < count; ++n) iterations[n] = outs[n].newton_last;
      if (residual_norms)
        check(cudaMemcpy(residual_norms, ctx->trace,
                         static_cast<size_t>(count) * ctx->settings.newton.max_iter * sizeof(double),
                         cudaMemcpyDeviceToHost),
              "trace");
    }
  });
}

// Test probe of the fused refill as the hot path runs
// it: every system refills once at (u, u_prev, t_next, dt) inside the persistent
// propagation kernel (refill_row_ell / refill_row / refill_long_rows /
// refill_finish) and the kernel stops.  Outputs in the reference's order:
// A = M/dt + J(u) [count][nnz] (per-system values where the kernel wrote them,
// the shared step matrix on constant-nu rows), R = M (u - u_prev)/dt + K(u) u - f
// [count][dim], Dinv = 1/diag(A) [count][dim].
int ps_refill_probe(ps_ctx* ctx, int32_t count, const double* U, const double* U_prev, const double* t_next,
                    double dt, double* A_out, double* R_out, double* Dinv_out) {
  if (!ctx || !U || !U_prev || !t_next) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    const DevProblem& P = ctx->P;
    if (count < 1 || count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "propagator: batch count out of range");
    if (P.linear) throw Failure(PS_ERR_BAD_ARG, "probe: the refill probe needs an element (nonlinear) problem");
    const int d = P.d, L = lanes_per_group(count);
    stage_in_host(ctx, U_prev, count);
    check(cudaMemcpyAsync(ctx->uprev, ctx->u, static_cast<size_t>(d) * lanes_padded(ctx) * sizeof(double),
                          cudaMemcpyDeviceToDevice, ctx->stream),
          "u_prev");
    stage_in_host(ctx, U, count);
    std::vector<double> t(t_next, t_next + count);
    ps_batch_status st{};
    propagate(ctx, count, 1, dt, t, true, false, &st, true);
    const int G = (count + L - 1) / L;
    std::vector<double> A(static_cast<size_t>(G) * P.nnz * 32), r(static_cast<size_t>(G) * d * 32),
        di(static_cast<size_t>(G) * d * 32);
    check(cudaMemcpy(A.data(), ctx->A, A.size() * sizeof(double), cudaMemcpyDeviceToHost), "A");
    check(cudaMemcpy(r.data(), ctx->r, r.size() * sizeof(double), cudaMemcpyDeviceToHost), "r");
    check(cudaMemcpy(di.data(), ctx->Dinv, di.size() * sizeof(double), cudaMemcpyDeviceToHost), "Dinv");
    for (int n = 0; n < count; ++n) {
      const int g = n / L, l = n % L;
      for (int i = 0; i < d; ++i) {
        const bool per_system = P.h_rowkind[i] != 0;
        const size_t iv = (static_cast<size_t>(g) * d + i) * 32 + l;
        double diag = 0.0;
        for (int k = P.h_rp[i]; k < P.h_rp[i + 1]; ++k) {
          const double a = per_system ? A[(static_cast<size_t>(g) * P.nnz + k) * 32 + l] : P.h_M[k] / dt + P.h_Kc[k];
          if (A_out) A_out[static_cast<size_t>(n) * P.nnz + k] = a;
          if (k == P.h_diag[i]) diag = a;
        }
        if (R_out) R_out[static_cast<size_t>(n) * d + i] = -r[iv];
        if (Dinv_out) Dinv_out[static_cast<size_t>(n) * d + i] = per_system ? di[iv] : 1.0 / diag;
      }
    }
  });
}

static int propagate_api(ps_ctx* ctx, int32_t n_first, int32_t count, const double* U_start, double* U_end,
                         ps_batch_status* status, bool fine, bool dev) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    check_range(ctx->mesh, n_first, count);
    if (count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "propagator: batch count out of range");
    if (dev)
      stage_in_dev(ctx, U_start, count);
    else
      stage_in_host(ctx, U_start, count);
    std::vector<double> t;
    int steps;
    double dt;
    if (fine) {
      t = fine_times(ctx->mesh, n_first, count);
      steps = ctx->mesh.fine_steps;
      dt = fine_dt(ctx->mesh);
    } else {
      t.resize(count);
      for (int i = 0; i < count; ++i) t[i] = boundary(ctx->mesh, n_first + i);
      steps = 1;
      dt = coarse_dt(ctx->mesh);
    }
    ps_batch_status st{};
    PropResult res;
    try {
      res = propagate(ctx, count, steps, dt, t, false, false, &st);
    } catch (...) {
      if (status) *status = st;
      throw;
    }
    if (status) *status = st;
    if (dev) {
      launch_from_blocked(res.state, U_end, count, ctx->P.d, lanes_per_group(count), ctx->stream);
      check(cudaStreamSynchronize(ctx->stream), "D2D");
    } else {
      stage_out_blocked(ctx, res.state, U_end, count);
    }
  });
}

int ps_fine_propagate_batch(ps_ctx* ctx, int32_t n_first, int32_t count, const double* U_start, double* U_end,
                            ps_batch_status* status) {
  return propagate_api(ctx, n_first, count, U_start, U_end, status, true, false);
}
int ps_fine_propagate_batch_dev(ps_ctx* ctx, int32_t n_first, int32_t count, const double* dU_start, double* dU_end,
                                ps_batch_status* status) {
  return propagate_api(ctx, n_first, count, dU_start, dU_end, status, true, true);
}
int ps_coarse_propagate_batch(ps_ctx* ctx, int32_t n_first, int32_t count, const double* U_start, double* U_end,
                              ps_batch_status* status) {
  return propagate_api(ctx, n_first, count, U_start, U_end, status, false, false);
}
int ps_coarse_propagate_batch_dev(ps_ctx* ctx, int32_t n_first, int32_t count, const double* dU_start,
                                  double* dU_end, ps_batch_status* status) {
  return propagate_api(ctx, n_first, count, dU_start, dU_end, status, false, true);
}

}  // extern "C"

namespace {

// Initial iterate U[0] = 0, U[n] = G_n(U[n-1]) on an interleaved [d][N] buffer.
void coarse_sweep_il(ps_ctx* ctx, double* U_il, ps_batch_status* total) {
  const int N = ctx->mesh.subintervals, d = ctx->P.d;
  check(cudaMemsetAsync(U_il, 0, static_cast<size_t>(d) * N * sizeof(double), ctx->stream), "zero");
  for (int n = 1; n < N; ++n) {
    // a batch of one: group 0, lane 0 of the blocked layout (row stride 32)
    copy_column(U_il, N, n - 1, ctx->u, 32, 0, d, ctx->stream);
    std::vector<double> t(1, boundary(ctx->mesh, n));
    ps_batch_status st{};
    PropResult res = propagate(ctx, 1, 1, coarse_dt(ctx->mesh), t, false, false, &st);
    copy_column(res.state, 32, 0, U_il, N, n, d, ctx->stream);
    if (total) {
      total->pcg_iterations += st.pcg_iterations;
      total->kernel_ms += st.kernel_ms;
      total->algorithmic_bytes += st.algorithmic_bytes;
    }
  }
}

void ensure_spectral(ps_ctx* lin, int use_conj, const int32_t* mask, int shift_kind) {
  if (lin->spec) {
    spectral_free(lin->spec);
    lin->spec = nullptr;
  }
  std::string err;
  const int rc = spectral_setup(&lin->spec, lin->P, lin->mesh.subintervals, lin->mesh.period, use_conj, mask,
                                shift_kind, &err);
  if (rc != PS_OK) throw Failure(rc, err);
}

}  // namespace

extern "C" {

int ps_coarse_sweep(ps_ctx* ctx, double* U, ps_batch_status* status) {
  if (!ctx || !U) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    double* U_il = nullptr;
    if (!dalloc(&U_il, static_cast<size_t>(N) * d)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    ps_batch_status st{};
    try {
      coarse_sweep_il(ctx, U_il, &st);
    } catch (...) {
      cudaFree(U_il);
      throw;
    }
    launch_from_interleaved(U_il, ctx->io_b, N, d, N, ctx->stream);
    check(cudaMemcpyAsync(U, ctx->io_b, static_cast<size_t>(N) * d * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream),
          "D2H");
    check(cudaStreamSynchronize(ctx->stream), "sweep");
    cudaFree(U_il);
    if (status) *status = st;
  });
}

int ps_assemble_operators(ps_ctx* ctx, int32_t count, const double* U, double* K_values, double* J_values) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    const DevProblem& P = ctx->P;
    if (count < 1 || count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "problem: batch count out of range");
    const size_t tot = static_cast<size_t>(count) * P.nnz;
    if (P.linear) {
      for (int n = 0; n < count; ++n) {
        if (K_values) std::copy(P.h_K.begin(), P.h_K.end(), K_values + static_cast<size_t>(n) * P.nnz);
        if (J_values) std::copy(P.h_K.begin(), P.h_K.end(), J_values + static_cast<size_t>(n) * P.nnz);
      }
      return;
    }
    check(cudaMemcpyAsync(ctx->io_a, U, static_cast<size_t>(count) * P.d * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream),
          "H2D");
    launch_to_interleaved(ctx->io_a, ctx->x, count, P.d, count, ctx->stream);
    double *dK = nullptr, *dJ = nullptr;
    if (!dalloc(&dK, tot) || !dalloc(&dJ, tot)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    launch_assemble_ops(P, count, ctx->x, dK, dJ, ctx->stream);
    check(cudaStreamSynchronize(ctx->stream), "assemble");
    if (K_values) check(cudaMemcpy(K_values, dK, tot * sizeof(double), cudaMemcpyDeviceToHost), "K");
    if (J_values) check(cudaMemcpy(J_values, dJ, tot * sizeof(double), cudaMemcpyDeviceToHost), "J");
    cudaFree(dK);
    cudaFree(dJ);
  });
}

int ps_eval_excitation(ps_ctx* ctx, int32_t count, const double* t, double* out) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    const DevProblem& P = ctx->P;
    if (count < 1 || count > ctx->max_batch) throw Failure(PS_ERR_BAD_ARG, "problem: batch count out of range");
    const int nt = std::max(1, P.nterms);
    std::vector<double> coef(static_cast<size_t>(count) * nt, 0.0);
    for (int n = 0; n < count; ++n) excitation_coef(P, t[n], &coef[static_cast<size_t>(n) * nt]);
    ensure(&ctx->coef, &ctx->coef_len, coef.size());
    check(cudaMemcpyAsync(ctx->coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream),
          "coef");
    launch_excitation(P, count, ctx->coef, ctx->u, ctx->stream);
    stage_out_host(ctx, ctx->u, out, count);
  });
}

int ps_mh_setup(ps_ctx* ctx, int32_t use_conjugate_symmetry, const int32_t* bin_mask, int32_t shift_kind) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] { ensure_spectral(ctx, use_conjugate_symmetry, bin_mask, shift_kind); });
}

// Test probes of the hot-path DFT kernels on the context's solved bins (after
// ps_mh_setup): dft_forward_kernel and idft_jump_kernel + jump_finalize_kernel.
int ps_mh_bins(ps_ctx* ctx, int32_t* bins, int32_t cap) {
  if (!ctx) return -PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (!ctx->spec) return -PS_ERR_NOT_SETUP;
  return spectral_bins(ctx->spec, bins, cap);
}

int ps_mh_forward(ps_ctx* ctx, const double* rhs, double* spectrum) {
  if (!ctx || !rhs || !spectrum) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->spec) throw Failure(PS_ERR_NOT_SETUP, "spectral: call ps_mh_setup first");
    std::string err;
    const int rc = spectral_forward_probe(ctx->spec, rhs, spectrum, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  });
}

int ps_mh_inverse(ps_ctx* ctx, const double* spectrum, const double* U_old, double* U, double* jump) {
  if (!ctx || !spectrum || !U) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->spec) throw Failure(PS_ERR_NOT_SETUP, "spectral: call ps_mh_setup first");
    std::string err;
    const int rc = spectral_inverse_probe(ctx->spec, spectrum, U_old, U, jump, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  });
}

int ps_assemble_rhs(ps_ctx* ctx, const double* F, const double* G, double* rhs) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->P.linear)
      throw Failure(PS_ERR_NOT_LINEAR,
                    "spectral: cyclic system requires a linear problem (freeze the coarse operator first)");
    if (!ctx->spec) ensure_spectral(ctx, 1, nullptr, 0);
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    const size_t n = static_cast<size_t>(N) * d;
    check(cudaMemcpyAsync(ctx->io_a, F, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "F");
    launch_to_interleaved(ctx->io_a, ctx->u, N, d, N, ctx->stream);
    check(cudaMemcpyAsync(ctx->io_b, G, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "G");
    launch_to_interleaved(ctx->io_b, ctx->uprev, N, d, N, ctx->stream);
    if (spectral_assemble_rhs(ctx->spec, ctx->P, ctx->u, ctx->uprev, ctx->x, ctx->stream) != PS_OK)
      throw Failure(PS_ERR_CUDA, "cuda: assemble_rhs failed");
    stage_out_host(ctx, ctx->x, rhs, N);
  });
}

int ps_mh_solve(ps_ctx* ctx, const double* rhs, double* U, ps_batch_status* status) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->P.linear)
      throw Failure(PS_ERR_NOT_LINEAR,
                    "spectral: cyclic system requires a linear problem (freeze the coarse operator first)");
    if (!ctx->spec) ensure_spectral(ctx, 1, nullptr, 0);
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    const size_t n = static_cast<size_t>(N) * d;
    check(cudaMemcpyAsync(ctx->io_a, rhs, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "rhs");
    launch_to_interleaved(ctx->io_a, ctx->x, N, d, N, ctx->stream);
    std::string err;
    const int rc = spectral_solve(ctx->spec, ctx->P, ctx->settings.cocg, ctx->x, ctx->u, nullptr, nullptr, status,
                                  ctx->stream, &err);
    if (rc != PS_OK) throw Failure(rc, err);
    stage_out_host(ctx, ctx->u, U, N);
  });
}

int ps_pppc_correct(ps_ctx* ctx, const double* F, const double* G, double* U_inout, double* jump,
                    ps_batch_status* status) {
  if (!ctx) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->P.linear)
      throw Failure(PS_ERR_NOT_LINEAR,
                    "spectral: cyclic system requires a linear problem (freeze the coarse operator first)");
    if (!ctx->spec) ensure_spectral(ctx, 1, nullptr, 0);
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    const size_t n = static_cast<size_t>(N) * d;
    check(cudaMemcpyAsync(ctx->io_a, F, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "F");
    launch_to_interleaved(ctx->io_a, ctx->u, N, d, N, ctx->stream);
    check(cudaMemcpyAsync(ctx->io_b, G, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "G");
    launch_to_interleaved(ctx->io_b, ctx->uprev, N, d, N, ctx->stream);
    check(cudaMemcpyAsync(ctx->io_a, U_inout, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "U");
    launch_to_interleaved(ctx->io_a, ctx->q, N, d, N, ctx->stream);
    if (spectral_assemble_rhs(ctx->spec, ctx->P, ctx->u, ctx->uprev, nullptr, ctx->stream) != PS_OK)
      throw Failure(PS_ERR_CUDA, "cuda: assemble_rhs failed");
    std::string err;
    const int rc =
        spectral_solve(ctx->spec, ctx->P, ctx->settings.cocg, nullptr, ctx->q, ctx->q, jump, status, ctx->stream, &err);
    if (rc != PS_OK) throw Failure(rc, err);
    stage_out_host(ctx, ctx->q, U_inout, N);
  });
}

int ps_forward_dft(int32_t n, int32_t d, const double* U, double* spectrum) {
  return guard(nullptr, [&] {
    require_device();
    std::string err;
    const int rc = dft_forward_standalone(n, d, U, spectrum, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  });
}

int ps_inverse_dft(int32_t n, int32_t d, const double* spectrum, double* U) {
  return guard(nullptr, [&] {
    require_device();
    std::string err;
    const int rc = dft_inverse_standalone(n, d, spectrum, U, &err);
    if (rc != PS_OK) throw Failure(rc, err);
  });
}

int ps_jump_norm(int32_t count, int32_t d, const double* cur, const double* prev, double* out) {
  return guard(nullptr, [&] {
    require_device();
    if (count < 1 || d < 1) throw Failure(PS_ERR_BAD_ARG, "engine: jump_norm needs two state lists of equal length");
    const size_t n = static_cast<size_t>(count) * d;
    double *a = nullptr, *b = nullptr, *ai = nullptr, *bi = nullptr;
    if (!dalloc(&a, n) || !dalloc(&b, n) || !dalloc(&ai, n) || !dalloc(&bi, n))
      throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    check(cudaMemcpy(a, cur, n * sizeof(double), cudaMemcpyHostToDevice), "cur");
    check(cudaMemcpy(b, prev, n * sizeof(double), cudaMemcpyHostToDevice), "prev");
    launch_to_interleaved(a, ai, count, d, count, nullptr);
    launch_to_interleaved(b, bi, count, d, count, nullptr);
    const int rc = jump_norm_device(count, d, ai, bi, count, out, nullptr);
    cudaFree(a);
    cudaFree(b);
    cudaFree(ai);
    cudaFree(bi);
    if (rc != PS_OK) throw Failure(rc, "cuda: jump_norm failed");
  });
}

int ps_eval_reluctivity(const ps_curve* curve, int32_t n, const double* b2, double* nu, double* nu_prime) {
  return guard(nullptr, [&] {
    require_device();
    double *db = nullptr, *dn = nullptr, *dp = nullptr;
    if (!dalloc(&db, n) || !dalloc(&dn, n) || !dalloc(&dp, n)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    check(cudaMemcpy(db, b2, n * sizeof(double), cudaMemcpyHostToDevice), "b2");
    launch_eval_curve(*curve, n, db, dn, dp, nullptr);
    if (nu) check(cudaMemcpy(nu, dn, n * sizeof(double), cudaMemcpyDeviceToHost), "nu");
    if (nu_prime) check(cudaMemcpy(nu_prime, dp, n * sizeof(double), cudaMemcpyDeviceToHost), "nu'");
    cudaFree(db);
    cudaFree(dn);
    cudaFree(dp);
  });
}

// solve_pp_pc with the multiharmonic coarse solver (proj/src/engine.cpp:187-270).
// All iterates stay in HBM; the host reads back one jump scalar per iteration.
int ps_pppc_solve(ps_ctx* fine, const ps_engine_settings* settings, const double* frozen_ref, double* U_out,
                  double* iterates, ps_history* history) {
  if (!fine || !settings) return PS_ERR_BAD_ARG;
  ps_ctx* coarse = nullptr;
  int rc = ps_create_frozen(fine, frozen_ref, &coarse);
  if (rc != PS_OK) return rc;
  std::lock_guard<std::mutex> lock(fine->mu);
  rc = guard(fine, [&] {
    std::unique_ptr<ps_ctx, void (*)(ps_ctx*)> hold(coarse, ps_destroy);
    if (!(settings->tol > 0.0)) throw Failure(PS_ERR_BAD_ARG, "engine: tolerance must be positive");
    if (settings->max_iterations < 1) throw Failure(PS_ERR_BAD_ARG, "engine: need at least one iteration");
    const int N = fine->mesh.subintervals, d = fine->P.d;
    if (fine->max_batch < N) throw Failure(PS_ERR_BAD_ARG, "engine: context batch smaller than N");
    cudaStream_t st = fine->stream;
    ps_history h;
    std::memset(&h, 0, sizeof(h));
    cudaEvent_t t0, t1;
    check(cudaEventCreate(&t0), "event");
    check(cudaEventCreate(&t1), "event");
    check(cudaEventRecord(t0, st), "event");
    ensure_spectral(coarse, settings->use_conjugate_symmetry, settings->bin_mask, settings->shift_kind);
    double* U = nullptr;
    if (!dalloc(&U, static_cast<size_t>(N) * d)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    std::unique_ptr<double, cudaError_t (*)(void*)> holdU(U, cudaFree);
    // the coarse context runs on its own stream; order through the host
    check(cudaStreamSynchronize(st), "sync");
    ps_batch_status cs{};
    coarse_sweep_il(coarse, U, &cs);
    h.coarse_ms += cs.kernel_ms;
    h.coarse_pcg_iterations += cs.pcg_iterations;
    check(cudaStreamSynchronize(coarse->stream), "sweep");
    const size_t nd = static_cast<size_t>(N) * d;
    for (int k = 0; k < settings->max_iterations; ++k) {
      // fine batch: F_n(U_{n-1}), all N subintervals in one launch
      const int L = lanes_per_group(N);
      launch_il_blocked(U, fine->u, d, N, N, L, true, st);
      ps_batch_status fs{};
      PropResult fr = propagate(fine, N, fine->mesh.fine_steps, fine_dt(fine->mesh), fine_times(fine->mesh, 1, N),
                                false, false, &fs);
      double* F_il = fine->io_a;
      launch_il_blocked(fr.state, F_il, d, N, N, L, false, st);
      check(cudaStreamSynchronize(st), "fine");
      h.fine_ms += fs.kernel_ms;
      h.fine_pcg_iterations += fs.pcg_iterations;
      h.newton_iterations += fs.newton_iterations;
      h.fine_bytes += fs.algorithmic_bytes;
      // coarse batch: G_n(U_{n-1}) with the frozen linear operator
      launch_il_blocked(U, coarse->u, d, N, N, L, true, coarse->stream);
      std::vector<double> tc(N);
      for (int n = 0; n < N; ++n) tc[n] = boundary(fine->mesh, n + 1);
      ps_batch_status gs{};
      PropResult gr = propagate(coarse, N, 1, coarse_dt(fine->mesh), tc, false, false, &gs);
      double* G_il = coarse->io_a;
      launch_il_blocked(gr.state, G_il, d, N, N, L, false, coarse->stream);
      h.coarse_ms += gs.kernel_ms;
      h.coarse_pcg_iterations += gs.pcg_iterations;
      // correction: rhs = Q (F - G) + f, multiharmonic solve, jump (in place on U)
      if (spectral_assemble_rhs(coarse->spec, coarse->P, F_il, G_il, nullptr, coarse->stream) != PS_OK)
        throw Failure(PS_ERR_CUDA, "cuda: assemble_rhs failed");
      double jump = 0.0;
      ps_batch_status ss{};
      std::string err;
      const int src = spectral_solve(coarse->spec, coarse->P, coarse->settings.cocg, nullptr, U, U, &jump, &ss,
                                     coarse->stream, &err);
      if (src != PS_OK) throw Failure(src, err);
      h.spectral_ms += ss.kernel_ms;
      h.cocg_iterations += ss.pcg_iterations;
      if (k < PS_MAX_HISTORY) {
        h.jumps[k] = jump;
        h.cocg_per_iteration[k] = ss.pcg_iterations;
        h.fine_ms_per_iteration[k] = fs.kernel_ms;
        h.spectral_ms_per_iteration[k] = ss.kernel_ms;
      }
      h.iterations = k + 1;
      if (iterates) {
        launch_from_interleaved(U, fine->io_b, N, d, N, coarse->stream);
        check(cudaMemcpyAsync(iterates + static_cast<size_t>(k) * nd, fine->io_b, nd * sizeof(double),
                              cudaMemcpyDeviceToHost, coarse->stream),
              "iterate");
        check(cudaStreamSynchronize(coarse->stream), "iterate");
      }
      if (jump <= settings->tol) {
        h.converged = 1;
        break;
      }
    }
    check(cudaStreamSynchronize(coarse->stream), "sync");
    check(cudaEventRecord(t1, st), "event");
    launch_from_interleaved(U, fine->io_b, N, d, N, st);
    check(cudaMemcpyAsync(U_out, fine->io_b, nd * sizeof(double), cudaMemcpyDeviceToHost, st), "U_out");
    check(cudaStreamSynchronize(st), "U_out");
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, t0, t1);
    h.total_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (history) *history = h;
  });
  return rc;
}

// ------------------------------------------------ classical Parareal and PP-IC
// proj/src/engine.cpp:76-129 (classic_parareal) and :131-185 (solve_pp_ic):
// the fine batch runs as one batched launch over all N subintervals; the coarse
// sweep is inherently sequential (u_n needs the corrected u_{n-1}) and runs one
// single-system coarse step per subinterval, each followed by the fused
// correction u_n = F_n + (G_new - G_old), G_old <- G_new.  States stay in HBM
// in the reference's [N+1][d] order; the host reads one jump (and for PP-IC one
// defect) per iteration.
}  // extern "C"

namespace {

__global__ void parareal_correct_kernel(const double* __restrict__ fine_end, const double* __restrict__ g_new,
                                        double* __restrict__ g_old, double* __restrict__ u_n, int d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d) return;
  const double gn = g_new[i];
  u_n[i] = fine_end[i] + (gn - g_old[i]);
  g_old[i] = gn;
}

// part[n] = (|cur_n - prev_n|^2, |cur_n|^2) for row-major [count][d] states
__global__ void row_jump_kernel(const double* cur, const double* prev, int d, double* part) {
  __shared__ double sa[256], sb[256];
  const int n = blockIdx.x;
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const size_t k = static_cast<size_t>(n) * d + i;
    const double c = cur[k], df = c - prev[k];
    a += df * df;
    b += c * c;
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) {
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sb[threadIdx.x] += sb[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * n] = sa[0];
    part[2 * n + 1] = sb[0];
  }
}

// jump_norm (proj/src/engine.cpp:54-64) over `count` row-major states
double row_jump(const double* cur, const double* prev, int count, int d, double* part, cudaStream_t st) {
  row_jump_kernel<<<count, 256, 0, st>>>(cur, prev, d, part);
  std::vector<double> h(static_cast<size_t>(2) * count);
  check(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "jump");
  check(cudaStreamSynchronize(st), "jump");
  double change = 0.0, scale = 1.0;
  for (int n = 0; n < count; ++n) {
    change = std::max(change, std::sqrt(h[2 * n]));
    scale = std::max(scale, std::sqrt(h[2 * n + 1]));
  }
  return change / scale;
}

int parareal_family(ps_ctx* ctx, const ps_engine_settings* settings, const double* u0, bool periodic, double* U_out,
                    double* iterates, ps_history* history) {
  if (!ctx || !settings || !U_out || (!periodic && !u0)) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!(settings->tol > 0.0)) throw Failure(PS_ERR_BAD_ARG, "engine: tolerance must be positive");
    if (settings->max_iterations < 1) throw Failure(PS_ERR_BAD_ARG, "engine: need at least one iteration");
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    if (ctx->max_batch < N) throw Failure(PS_ERR_BAD_ARG, "engine: context batch smaller than N");
    cudaStream_t st = ctx->stream;
    const size_t nd = static_cast<size_t>(N) * d, nd1 = nd + d;
    double *U = nullptr, *Uold = nullptr, *F = nullptr, *Gold = nullptr, *gnew = nullptr, *part = nullptr;
    if (!dalloc(&U, nd1) || !dalloc(&Uold, nd1) || !dalloc(&F, nd) || !dalloc(&Gold, nd) || !dalloc(&gnew, d) ||
        !dalloc(&part, 2 * static_cast<size_t>(N + 1)))
      throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    std::unique_ptr<double, cudaError_t (*)(void*)> h0(U, cudaFree), h1(Uold, cudaFree), h2(F, cudaFree),
        h3(Gold, cudaFree), h4(gnew, cudaFree), h5(part, cudaFree);
    ps_history h;
    std::memset(&h, 0, sizeof(h));
    cudaEvent_t t0, t1;
    check(cudaEventCreate(&t0), "event");
    check(cudaEventCreate(&t1), "event");
    check(cudaEventRecord(t0, st), "event");
    check(cudaMemsetAsync(U, 0, nd1 * sizeof(double), st), "init");
    if (!periodic) check(cudaMemcpyAsync(U, u0, d * sizeof(double), cudaMemcpyHostToDevice, st), "u0");
    const double dT = coarse_dt(ctx->mesh), dt = fine_dt(ctx->mesh);
    const int cblocks = (d + 255) / 256;
    // one coarse step G_n(U[n-1]) into gnew (proj/src/propagators.cpp:107-115)
    auto coarse_step = [&](int n) {
      stage_in_dev(ctx, U + static_cast<size_t>(n - 1) * d, 1);
      ps_batch_status cs{};
      PropResult r = propagate(ctx, 1, 1, dT, std::vector<double>{boundary(ctx->mesh, n)}, false, false, &cs);
      launch_from_blocked(r.state, gnew, 1, d, 1, st);
      h.coarse_ms += cs.kernel_ms;
      h.coarse_pcg_iterations += cs.pcg_iterations;
    };
    for (int n = 1; n <= N; ++n) {
      coarse_step(n);
      check(cudaMemcpyAsync(U + static_cast<size_t>(n) * d, gnew, d * sizeof(double), cudaMemcpyDeviceToDevice, st),
            "sweep");
      check(cudaMemcpyAsync(Gold + static_cast<size_t>(n - 1) * d, gnew, d * sizeof(double),
                            cudaMemcpyDeviceToDevice, st),
            "sweep");
    }
    for (int k = 0; k < settings->max_iterations; ++k) {
      check(cudaMemcpyAsync(Uold, U, nd1 * sizeof(double), cudaMemcpyDeviceToDevice, st), "u_old");
      // fine batch F_n(u_old[n-1]), n = 1..N, one launch
      stage_in_dev(ctx, Uold, N);
      ps_batch_status fs{};
      PropResult fr = propagate(ctx, N, ctx->mesh.fine_steps, dt, fine_times(ctx->mesh, 1, N), false, false, &fs);
      launch_from_blocked(fr.state, F, N, d, lanes_per_group(N), st);
      h.fine_ms += fs.kernel_ms;
      h.fine_pcg_iterations += fs.pcg_iterations;
      h.newton_iterations += fs.newton_iterations;
      h.fine_bytes += fs.algorithmic_bytes;
      // periodicity by relaxation (PP-IC): the new period start is the old end
      if (periodic)
        check(cudaMemcpyAsync(U, Uold + nd, d * sizeof(double), cudaMemcpyDeviceToDevice, st), "relax");
      for (int n = 1; n <= N; ++n) {
        coarse_step(n);
        parareal_correct_kernel<<<cblocks, 256, 0, st>>>(F + static_cast<size_t>(n - 1) * d, gnew,
                                                         Gold + static_cast<size_t>(n - 1) * d,
                                                         U + static_cast<size_t>(n) * d, d);
      }
      const double jump = row_jump(U, Uold, N + 1, d, part, st);
      if (k < PS_MAX_HISTORY) h.jumps[k] = jump;
      h.iterations = k + 1;
      if (iterates) {
        check(cudaMemcpyAsync(iterates + static_cast<size_t>(k) * nd1, U, nd1 * sizeof(double),
                              cudaMemcpyDeviceToHost, st),
              "iterate");
        check(cudaStreamSynchronize(st), "iterate");
      }
      bool done = jump <= settings->tol;
      if (periodic) {
        // relative_defect(u_N, u_0) (proj/src/engine.cpp:26-28)
        h.final_defect = row_jump(U + nd, U, 1, d, part, st);
        done = done && h.final_defect <= settings->tol;
      }
      if (done) {
        h.converged = 1;
        break;
      }
    }
    check(cudaEventRecord(t1, st), "event");
    check(cudaMemcpyAsync(U_out, U, (periodic ? nd : nd1) * sizeof(double), cudaMemcpyDeviceToHost, st), "U_out");
    check(cudaStreamSynchronize(st), "U_out");
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, t0, t1);
    h.total_ms = ms;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (history) *history = h;
  });
}

}  // namespace

extern "C" {

int ps_classic_parareal(ps_ctx* ctx, const ps_engine_settings* settings, const double* u0, double* U_out,
                        double* iterates, ps_history* history) {
  return parareal_family(ctx, settings, u0, false, U_out, iterates, history);
}

int ps_pp_ic_solve(ps_ctx* ctx, const ps_engine_settings* settings, double* U_out, double* iterates,
                   ps_history* history) {
  return parareal_family(ctx, settings, nullptr, true, U_out, iterates, history);
}

// sequential_steady_state (proj/src/propagators.cpp:117-149): period after
// period from zero, one fine propagation per subinterval (batch size 1), until
// the period map's relative defect is <= tol.  U_out [N][dim]: the last
// period's states T_0..T_{N-1}; defects [max_periods] or NULL.
int ps_sequential_steady_state(ps_ctx* ctx, double tol, int32_t max_periods, double* U_out, int32_t* periods,
                               int32_t* converged, double* defects) {
  if (!ctx || !U_out || !periods || !converged) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!(tol > 0.0)) throw Failure(PS_ERR_BAD_ARG, "propagator: tolerance must be positive");
    if (max_periods < 1) throw Failure(PS_ERR_BAD_ARG, "propagator: need at least one period");
    const int N = ctx->mesh.subintervals, d = ctx->P.d;
    cudaStream_t st = ctx->stream;
    const size_t nd = static_cast<size_t>(N) * d;
    double *traj = nullptr, *part = nullptr;
    if (!dalloc(&traj, nd + d) || !dalloc(&part, 2)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    std::unique_ptr<double, cudaError_t (*)(void*)> h0(traj, cudaFree), h1(part, cudaFree);
    check(cudaMemsetAsync(traj, 0, (nd + d) * sizeof(double), st), "init");
    const double dt = fine_dt(ctx->mesh);
    *converged = 0;
    for (int per = 1; per <= max_periods; ++per) {
      for (int n = 1; n <= N; ++n) {
        stage_in_dev(ctx, traj + static_cast<size_t>(n - 1) * d, 1);
        ps_batch_status fs{};
        PropResult r = propagate(ctx, 1, ctx->mesh.fine_steps, dt, fine_times(ctx->mesh, n, 1), false, false, &fs);
        launch_from_blocked(r.state, traj + static_cast<size_t>(n) * d, 1, d, 1, st);
      }
      // (u_end - u).norm() / max(1, u_end.norm())
      const double defect = row_jump(traj + nd, traj, 1, d, part, st);
      if (defects) defects[per - 1] = defect;
      *periods = per;
      check(cudaMemcpyAsync(U_out, traj, nd * sizeof(double), cudaMemcpyDeviceToHost, st), "U_out");
      check(cudaMemcpyAsync(traj, traj + nd, d * sizeof(double), cudaMemcpyDeviceToDevice, st), "wrap");
      check(cudaStreamSynchronize(st), "U_out");
      if (defect <= tol) {
        *converged = 1;
        break;
      }
    }
  });
}

// Diagnostic: time one PCG phase of the last nonlinear propagation's batch as a
// standalone kernel (see phase_probe_kernel).  mode 1 = phase A (SpMV + dots),
// 2 = phase B (updates), 3 = phase B's streams as a flat copy.  ms_out = mean
// over reps; bytes_out = the phase's bytes by the SURVEY.md §8d stream count.
int ps_phase_probe(ps_ctx* ctx, int32_t mode, int32_t reps, double* ms_out, double* bytes_out) {
  if (!ctx || reps < 1) return PS_ERR_BAD_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  return guard(ctx, [&] {
    if (!ctx->has_last_params) throw Failure(PS_ERR_NOT_SETUP, "probe: run a nonlinear propagation first");
    const PropParams& K = ctx->last_params;
    double* sink = nullptr;
    if (!dalloc(&sink, static_cast<size_t>(K.G) * K.C)) throw Failure(PS_ERR_CUDA, "cuda: out of memory");
    check(cudaEventRecord(ctx->e0, ctx->stream), "event");
    for (int r = 0; r < reps; ++r)
      if (launch_phase_probe(K, mode, sink, ctx->stream) != PS_OK) throw Failure(PS_ERR_CUDA, "cuda: probe launch");
    check(cudaEventRecord(ctx->e1, ctx->stream), "event");
    check(cudaStreamSynchronize(ctx->stream), "probe");
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ctx->e0, ctx->e1);
    cudaFree(sink);
    const double d = K.d, nnz = K.nnz, nb = K.count;
    if (ms_out) *ms_out = ms / reps;
    if (bytes_out) *bytes_out = mode >= 2 ? nb * 64.0 * d : nb * (8.0 * nnz + 40.0 * d);
  });
}

// fine_periodicity_defect (proj/src/engine.cpp:272-290)
int ps_fine_periodicity_defect(ps_ctx* ctx, const double* U, double* defect) {
  if (!ctx || !U || !defect) return PS_ERR_BAD_ARG;
  const int N = ctx->mesh.subintervals, d = ctx->P.d;
  std::vector<double> F(static_cast<size_t>(N) * d);
  const int rc = ps_fine_propagate_batch(ctx, 1, N, U, F.data(), nullptr);
  if (rc != PS_OK) return rc;
  double scale = 0.0;
  for (int n = 0; n < N; ++n) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += U[static_cast<size_t>(n) * d + i] * U[static_cast<size_t>(n) * d + i];
    scale = std::max(scale, std::sqrt(s));
  }
  scale = std::max(1.0, scale);
  double worst = 0.0;
  for (int n = 0; n < N; ++n) {
    const double* target = U + static_cast<size_t>((n + 1) % N) * d;
    double s = 0.0;
    for (int i = 0; i < d; ++i) {
      const double df = F[static_cast<size_t>(n) * d + i] - target[i];
      s += df * df;
    }
    worst = std::max(worst, std::sqrt(s));
  }
  *defect = worst / scale;
  return PS_OK;
}

}  // extern "C"
