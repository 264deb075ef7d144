// CPU ORACLE — test infrastructure only (see oracle.h).
//
// The oracle's own problem builders and seeded generators, so that the CPU
// checker (and bench.py's reference arm) never consumes a problem built by the
// product library.  They restate, independently of
// paper_1905_13076_b200/csrc/builders.cpp:
//  * the canonical structured polar P1 coax cable of SURVEY.md App. A.1 (the
//    2-D cross-section BASELINE.json's configs name; the reference has only the
//    1-D radial cable of proj/src/problem.cpp:242-361, so this geometry has no
//    reference line to follow — the element formulas are the P1 restatement of
//    its per-element stiffness / mass / load, proj/src/problem.cpp:204-237,
//    278-329);
//  * the seeded generators of SURVEY.md §8(d): std::mt19937_64 with an explicit
//    Box-Muller (no libstdc++ distribution objects).
// tests/test_builders.py asserts that both builders agree bit for bit.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;
// proj/include/parasteady/problem.hpp:62
constexpr double kVacuumNu = 1.0 / (4.0e-7 * 3.14159265358979323846);

thread_local std::string g_mesh_error;

// One P1 triangle of the polar mesh: node ids (-1 = Dirichlet ring), geometry
// and the radial band it lies in.
struct Tri {
  int32_t n[3];
  double S[9];
  double area;
  int band;
};

}  // namespace

struct or_mesh {
  std::vector<int32_t> rp, ci, en, ecurve;
  std::vector<double> mass, stiff, eS, einvA, pat, amp, freq, phase, xy;
  std::vector<ps_curve> curves;
  ps_problem_desc desc{};
};

extern "C" {

int or_polar_cable_defaults(ps_polar_cable_params* p) {
  if (!p) return 1;
  std::memset(p, 0, sizeof(*p));
  // BASELINE.json configs[0]: R = 5 mm, conductor r < 2 mm (sigma 5.8e7),
  // insulator 2-4 mm, Brauer steel sheath 4-5 mm (3.8, 2.17, 396.2; sigma 1e6),
  // I0 = 2000 A at 50 Hz, return in the sheath
  p->nr = 40;
  p->ntheta = 64;
  p->radius = 5.0e-3;
  p->r_conductor = 2.0e-3;
  p->r_insulator = 4.0e-3;
  p->sigma_conductor = 5.8e7;
  p->sigma_insulator = 0.0;
  p->sigma_sheath = 1.0e6;
  p->brauer_k1 = 3.8;
  p->brauer_k2 = 2.17;
  p->brauer_k3 = 396.2;
  p->linear_sheath = 0;
  p->return_in_sheath = 1;
  p->current = 2000.0;
  p->frequency_hz = 50.0;
  p->ripple_terms = 0;
  p->ripple_fraction = 0.1;
  p->ripple_frequency_hz = 1000.0;
  return 0;
}

const char* or_mesh_error(void) { return g_mesh_error.c_str(); }

int or_build_polar_cable(const ps_polar_cable_params* prm, or_mesh** out) {
  if (!prm || !out) return 1;
  *out = nullptr;
  try {
    const ps_polar_cable_params& P = *prm;
    if (P.nr < 2 || P.ntheta < 3) throw std::runtime_error("problem: polar mesh too small");
    if (!(0.0 < P.r_conductor && P.r_conductor < P.r_insulator && P.r_insulator < P.radius))
      throw std::runtime_error("problem: cable radii must satisfy 0 < r1 < r2 < R");
    const int nr = P.nr, nt = P.ntheta;
    const int dim = 1 + (nr - 1) * nt;
    auto* m = new or_mesh();
    // node (ring, j): centre 0, then ring by ring; ring nr is the Dirichlet ring
    auto id = [&](int ring, int j) -> int32_t {
      if (ring == 0) return 0;
      if (ring == nr) return -1;
      return 1 + (ring - 1) * nt + j % nt;
    };
    std::vector<double> cosj(nt), sinj(nt);
    for (int j = 0; j < nt; ++j) {
      cosj[j] = std::cos(2.0 * kPi * j / nt);
      sinj[j] = std::sin(2.0 * kPi * j / nt);
    }
    auto at = [&](int ring, int j, double* x, double* y) {
      const double r = P.radius * ring / nr;
      *x = r * cosj[j % nt];
      *y = r * sinj[j % nt];
    };
    m->xy.assign(2 * static_cast<size_t>(dim), 0.0);
    for (int ring = 1; ring < nr; ++ring)
      for (int j = 0; j < nt; ++j) at(ring, j, &m->xy[2 * id(ring, j)], &m->xy[2 * id(ring, j) + 1]);

    // elements: the centre fan, then per band two triangles per quad, split along
    // the (i, j)-(i+1, j+1) diagonal
    std::vector<Tri> tris;
    tris.reserve(static_cast<size_t>(nt) * (2 * nr - 1));
    auto tri = [&](int band, int r0, int j0, int r1, int j1, int r2, int j2) {
      Tri t{};
      const int rr[3] = {r0, r1, r2}, jj[3] = {j0, j1, j2};
      double x[3], y[3];
      for (int k = 0; k < 3; ++k) {
        at(rr[k], jj[k], &x[k], &y[k]);
        t.n[k] = id(rr[k], jj[k]);
      }
      // P1 gradients: grad phi_k = (b_k, c_k) / (2A)
      const double two_a = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
      t.area = 0.5 * std::fabs(two_a);
      double b[3], c[3];
      for (int k = 0; k < 3; ++k) {
        b[k] = y[(k + 1) % 3] - y[(k + 2) % 3];
        c[k] = x[(k + 2) % 3] - x[(k + 1) % 3];
      }
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) t.S[3 * k + l] = (b[k] * b[l] + c[k] * c[l]) / (4.0 * t.area);
      t.band = band;
      tris.push_back(t);
    };
    for (int j = 0; j < nt; ++j) tri(0, 0, 0, 1, j, 1, j + 1);
    for (int i = 1; i < nr; ++i)
      for (int j = 0; j < nt; ++j) {
        tri(i, i, j, i + 1, j, i + 1, j + 1);
        tri(i, i, j, i + 1, j + 1, i, j + 1);
      }
    const size_t ne = tris.size();

    // region of an element by its band's mid radius
    std::vector<int> region(ne);
    for (size_t e = 0; e < ne; ++e) {
      const double mid = P.radius * (tris[e].band + 0.5) / nr;
      region[e] = mid < P.r_conductor ? 0 : (mid < P.r_insulator ? 1 : 2);
    }

    // CSR pattern: every coupling of two free nodes of one element, plus the diagonal
    std::vector<std::set<int32_t>> rows(dim);
    for (int i = 0; i < dim; ++i) rows[i].insert(i);
    for (const Tri& t : tris)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          if (t.n[a] >= 0 && t.n[b] >= 0) rows[t.n[a]].insert(t.n[b]);
    m->rp.assign(dim + 1, 0);
    for (int i = 0; i < dim; ++i) {
      m->ci.insert(m->ci.end(), rows[i].begin(), rows[i].end());
      m->rp[i + 1] = static_cast<int32_t>(m->ci.size());
    }
    auto slot = [&](int32_t r, int32_t c) -> size_t {
      const auto b = m->ci.begin() + m->rp[r], e = m->ci.begin() + m->rp[r + 1];
      return static_cast<size_t>(std::lower_bound(b, e, c) - m->ci.begin());
    };

    // materials: vacuum reluctivity in the conductor and insulator, Brauer steel
    ps_curve vac{}, steel{};
    vac.kind = 0;
    vac.nu = kVacuumNu;
    if (P.linear_sheath) {
      steel.kind = 0;
      steel.nu = P.brauer_k1 + P.brauer_k3;
    } else {
      steel.kind = 1;
      steel.k1 = P.brauer_k1;
      steel.k2 = P.brauer_k2;
      steel.k3 = P.brauer_k3;
    }
    m->curves = {vac, steel};
    const double sigma[3] = {P.sigma_conductor, P.sigma_insulator, P.sigma_sheath};

    // element arrays, consistent sigma-mass sigma A / 12 [[2,1,1],[1,2,1],[1,1,2]],
    // and the unit P1 loads A / 3 of the free nodes of the source regions
    m->mass.assign(m->ci.size(), 0.0);
    std::vector<double> load_c(dim, 0.0), load_s(dim, 0.0);
    double sum_c = 0.0, sum_s = 0.0;
    for (size_t e = 0; e < ne; ++e) {
      const Tri& t = tris[e];
      for (int a = 0; a < 3; ++a) m->en.push_back(t.n[a]);
      for (int k = 0; k < 9; ++k) m->eS.push_back(t.S[k]);
      m->einvA.push_back(1.0 / t.area);
      m->ecurve.push_back(region[e] == 2 ? 1 : 0);
      const double s = sigma[region[e]];
      if (s != 0.0) {
        const double w = s * t.area / 12.0;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            if (t.n[a] >= 0 && t.n[b] >= 0) m->mass[slot(t.n[a], t.n[b])] += (a == b ? 2.0 : 1.0) * w;
      }
      if (region[e] == 1) continue;
      const double w = t.area / 3.0;
      for (int a = 0; a < 3; ++a) {
        if (t.n[a] < 0) continue;
        if (region[e] == 0) {
          load_c[t.n[a]] += w;
          sum_c += w;
        } else {
          load_s[t.n[a]] += w;
          sum_s += w;
        }
      }
    }
    // uniform current density, each source pattern normalised over the free
    // DOFs: the conductor carries +1 and the sheath returns exactly -1
    std::vector<double> pattern(dim);
    for (int i = 0; i < dim; ++i) {
      pattern[i] = sum_c > 0.0 ? load_c[i] / sum_c : 0.0;
      if (P.return_in_sheath && sum_s > 0.0) pattern[i] -= load_s[i] / sum_s;
    }
    m->pat = pattern;
    m->amp = {P.current};
    m->freq = {P.frequency_hz};
    m->phase = {0.0};
    // optional PWM-like ripple: odd-harmonic square-wave series, same pattern
    for (int k = 0; k < P.ripple_terms; ++k) {
      const int h = 2 * k + 1;
      m->pat.insert(m->pat.end(), pattern.begin(), pattern.end());
      m->amp.push_back(P.ripple_fraction * P.current * 4.0 / (kPi * h));
      m->freq.push_back(P.ripple_frequency_hz * h);
      m->phase.push_back(0.0);
    }
    if (P.linear_sheath) {
      // K = sum_e nu S_e, element by element
      m->stiff.assign(m->ci.size(), 0.0);
      for (size_t e = 0; e < ne; ++e) {
        const Tri& t = tris[e];
        const double nu = m->curves[m->ecurve[e]].nu;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b)
            if (t.n[a] >= 0 && t.n[b] >= 0) m->stiff[slot(t.n[a], t.n[b])] += nu * t.S[3 * a + b];
      }
    }
    ps_problem_desc& d = m->desc;
    std::memset(&d, 0, sizeof(d));
    d.dim = dim;
    d.nnz = static_cast<int32_t>(m->ci.size());
    d.row_ptr = m->rp.data();
    d.col_idx = m->ci.data();
    d.mass = m->mass.data();
    d.stiffness = P.linear_sheath ? m->stiff.data() : nullptr;
    d.n_elem = static_cast<int32_t>(ne);
    d.nodes_per_elem = 3;
    d.elem_nodes = m->en.data();
    d.elem_stiff = m->eS.data();
    d.elem_inv_area = m->einvA.data();
    d.elem_curve = m->ecurve.data();
    d.n_curves = 2;
    d.curves = m->curves.data();
    d.period = 1.0 / P.frequency_hz;
    d.n_terms = static_cast<int32_t>(m->amp.size());
    d.patterns = m->pat.data();
    d.amplitude = m->amp.data();
    d.frequency_hz = m->freq.data();
    d.phase_rad = m->phase.data();
    *out = m;
    return 0;
  } catch (const std::exception& e) {
    g_mesh_error = e.what();
    return 1;
  }
}

const ps_problem_desc* or_mesh_desc(const or_mesh* m) { return m ? &m->desc : nullptr; }
const double* or_mesh_coordinates(const or_mesh* m) { return m ? m->xy.data() : nullptr; }
void or_mesh_free(or_mesh* m) { delete m; }

// mt19937_64, 53-bit uniforms, explicit Box-Muller pairs
void or_seeded_normal(uint64_t seed, int64_t count, double sigma, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < count; i += 2) {
    const double u1 = (static_cast<double>(rng() >> 11) + 1.0) / 9007199254740992.0;
    const double u2 = static_cast<double>(rng() >> 11) / 9007199254740992.0;
    const double rho = std::sqrt(-2.0 * std::log(u1));
    out[i] = sigma * rho * std::cos(2.0 * kPi * u2);
    if (i + 1 < count) out[i + 1] = sigma * rho * std::sin(2.0 * kPi * u2);
  }
}

void or_seeded_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * (static_cast<double>(rng() >> 11) / 9007199254740992.0);
}

}  // extern "C"
