// Problem builders and seeded generators (host C++).
//
// These produce the structured ps_problem_desc the device path consumes:
//  * ps_build_radial_cable restates the reference's own 1-D radial coax cable
//    (proj/src/problem.cpp:242-361, CoaxCableParams at
//    proj/include/parasteady/problem.hpp:122-144) as 2-node elements, so the
//    reference's cable tests run through the GPU path;
//  * ps_build_polar_cable builds the 2-D structured polar P1 cable that
//    BASELINE.json's configs name (canonical mesh: SURVEY.md App. A.1).
#include "pppc_b200.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;
// proj/include/parasteady/problem.hpp:62
constexpr double kVacuumReluctivity = 1.0 / (4.0e-7 * 3.14159265358979323846);

thread_local std::string g_builder_error;

}  // namespace

struct ps_problem {
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<double> mass, stiffness;
  std::vector<int32_t> elem_nodes, elem_curve;
  std::vector<double> elem_stiff, elem_inv_area;
  std::vector<ps_curve> curves;
  std::vector<double> patterns, amplitude, frequency, phase;
  std::vector<double> coords;
  bool linear = false;
  int npe = 0;
  int dim = 0;
  ps_problem_desc desc{};

  void finalize() {
    std::memset(&desc, 0, sizeof(desc));
    desc.dim = dim;
    desc.nnz = static_cast<int32_t>(col_idx.size());
    desc.row_ptr = row_ptr.data();
    desc.col_idx = col_idx.data();
    desc.mass = mass.data();
    desc.stiffness = linear ? stiffness.data() : nullptr;
    desc.n_elem = static_cast<int32_t>(elem_curve.size());
    desc.nodes_per_elem = npe;
    desc.elem_nodes = elem_nodes.data();
    desc.elem_stiff = elem_stiff.data();
    desc.elem_inv_area = elem_inv_area.data();
    desc.elem_curve = elem_curve.data();
    desc.n_curves = static_cast<int32_t>(curves.size());
    desc.curves = curves.data();
    desc.n_terms = static_cast<int32_t>(amplitude.size());
    desc.patterns = patterns.data();
    desc.amplitude = amplitude.data();
    desc.frequency_hz = frequency.data();
    desc.phase_rad = phase.data();
  }

  // Symmetric CSR pattern of all element couplings between free nodes
  // (each row sorted, diagonal always present).
  void build_pattern() {
    const int64_t n_elem = static_cast<int64_t>(elem_curve.size());
    std::vector<int32_t> count(static_cast<size_t>(dim) + 1, 0);
    for (int64_t e = 0; e < n_elem; ++e)
      for (int a = 0; a < npe; ++a) {
        const int32_t na = elem_nodes[e * npe + a];
        if (na >= 0) count[na + 1] += npe;
      }
    for (int i = 0; i < dim; ++i) count[i + 1] += 1;  // diagonal
    std::vector<int64_t> start(static_cast<size_t>(dim) + 1, 0);
    for (int i = 0; i < dim; ++i) start[i + 1] = start[i] + count[i + 1];
    std::vector<int32_t> scratch(static_cast<size_t>(start[dim]));
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int i = 0; i < dim; ++i) scratch[fill[i]++] = i;
    for (int64_t e = 0; e < n_elem; ++e)
      for (int a = 0; a < npe; ++a) {
        const int32_t na = elem_nodes[e * npe + a];
        if (na < 0) continue;
        for (int b = 0; b < npe; ++b) {
          const int32_t nb = elem_nodes[e * npe + b];
          if (nb >= 0) scratch[fill[na]++] = nb;
        }
      }
    row_ptr.assign(static_cast<size_t>(dim) + 1, 0);
    col_idx.clear();
    col_idx.reserve(static_cast<size_t>(dim) * 8);
    for (int i = 0; i < dim; ++i) {
      auto b = scratch.begin() + start[i];
      auto e = scratch.begin() + fill[i];
      std::sort(b, e);
      auto last = std::unique(b, e);
      col_idx.insert(col_idx.end(), b, last);
      row_ptr[i + 1] = static_cast<int32_t>(col_idx.size());
    }
    mass.assign(col_idx.size(), 0.0);
    stiffness.assign(col_idx.size(), 0.0);
  }

  int64_t slot(int32_t row, int32_t col) const {
    const auto b = col_idx.begin() + row_ptr[row];
    const auto e = col_idx.begin() + row_ptr[row + 1];
    const auto it = std::lower_bound(b, e, col);
    if (it == e || *it != col) throw std::runtime_error("builder: pattern slot missing");
    return it - col_idx.begin();
  }

  double curve_nu0(int c) const {
    const ps_curve& cv = curves[c];
    if (cv.kind == 0) return cv.nu;
    return std::min(cv.k1 * std::exp(std::min(cv.k2 * 0.0, 700.0)) + cv.k3, kVacuumReluctivity);
  }

  // Linear problems: K = sum_e nu(0) S_e, accumulated element by element.
  void assemble_linear_stiffness() {
    const int64_t n_elem = static_cast<int64_t>(elem_curve.size());
    std::fill(stiffness.begin(), stiffness.end(), 0.0);
    for (int64_t e = 0; e < n_elem; ++e) {
      const double nu = curve_nu0(elem_curve[e]);
      for (int a = 0; a < npe; ++a) {
        const int32_t na = elem_nodes[e * npe + a];
        if (na < 0) continue;
        for (int b = 0; b < npe; ++b) {
          const int32_t nb = elem_nodes[e * npe + b];
          if (nb < 0) continue;
          stiffness[slot(na, nb)] += nu * elem_stiff[(e * npe + a) * npe + b];
        }
      }
    }
  }
};

extern "C" {

int ps_radial_cable_defaults(ps_radial_cable_params* p) {
  if (!p) return PS_ERR_BAD_ARG;
  std::memset(p, 0, sizeof(*p));
  // proj/include/parasteady/problem.hpp:122-137
  p->n_r = 200;
  p->r1 = 2.0e-3;
  p->r2 = 3.5e-3;
  p->r3 = 5.0e-3;
  p->sigma_wire = 5.96e7;
  p->sigma_sleeve = 5.0e6;
  p->sigma_shield = 0.0;
  p->brauer_k1 = 49.4;
  p->brauer_k2 = 1.46;
  p->brauer_k3 = 520.6;
  p->linear_sleeve = 0;
  p->source_region = 0;
  p->current = 100.0;
  p->frequency_hz = 50.0;
  return PS_OK;
}

int ps_polar_cable_defaults(ps_polar_cable_params* p) {
  if (!p) return PS_ERR_BAD_ARG;
  std::memset(p, 0, sizeof(*p));
  // BASELINE.json configs[0]
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
  return PS_OK;
}

// Restates build_coax_cable (proj/src/problem.cpp:242-361) in element form.
int ps_build_radial_cable(const ps_radial_cable_params* params, ps_problem** out) {
  if (!params || !out) return PS_ERR_BAD_ARG;
  try {
    const ps_radial_cable_params& P = *params;
    if (P.n_r < 3) throw std::runtime_error("problem: cable needs at least 3 radial nodes");
    if (!(0.0 < P.r1 && P.r1 < P.r2 && P.r2 < P.r3))
      throw std::runtime_error("problem: cable radii must satisfy 0 < r1 < r2 < r3");
    if (P.sigma_wire < 0.0 || P.sigma_sleeve < 0.0 || P.sigma_shield < 0.0)
      throw std::runtime_error("problem: conductivities must be non-negative");
    if (P.source_region < 0 || P.source_region > 2)
      throw std::runtime_error("problem: source region must be 0, 1 or 2");
    if (!(P.frequency_hz > 0.0)) throw std::runtime_error("problem: frequency must be positive");
    if (!P.linear_sleeve && (!(P.brauer_k1 > 0) || !(P.brauer_k2 > 0) || !(P.brauer_k3 > 0)))
      throw std::runtime_error("problem: Brauer coefficients must be positive");

    auto pb = new ps_problem();
    ps_problem& pr = *pb;
    const int n_nodes = P.n_r;
    const int n_elems = n_nodes - 1;
    pr.dim = n_nodes - 1;
    pr.npe = 2;
    const double h = P.r3 / n_elems;
    std::vector<double> radii(n_nodes);
    for (int i = 0; i < n_nodes; ++i) radii[i] = P.r3 * i / n_elems;

    ps_curve vac{};
    vac.kind = 0;
    vac.nu = kVacuumReluctivity;
    ps_curve sleeve{};
    if (P.linear_sleeve) {
      sleeve.kind = 0;
      sleeve.nu = P.brauer_k1 + P.brauer_k3;
    } else {
      sleeve.kind = 1;
      sleeve.k1 = P.brauer_k1;
      sleeve.k2 = P.brauer_k2;
      sleeve.k3 = P.brauer_k3;
    }
    pr.curves = {vac, sleeve};

    const double region_sigma[3] = {P.sigma_wire, P.sigma_sleeve, P.sigma_shield};
    const double bounds[2] = {P.r1, P.r2};
    std::vector<double> sigma(n_elems);
    for (int e = 0; e < n_elems; ++e) {
      const double mid = 0.5 * (radii[e] + radii[e + 1]);
      const int region = mid < bounds[0] ? 0 : (mid < bounds[1] ? 1 : 2);
      sigma[e] = region_sigma[region];
      pr.elem_curve.push_back(region == 1 ? 1 : 0);
      pr.elem_nodes.push_back(e < pr.dim ? e : -1);
      pr.elem_nodes.push_back(e + 1 < pr.dim ? e + 1 : -1);
      const double rbar = 0.5 * (radii[e] + radii[e + 1]);
      const double w = 2.0 * kPi * rbar / h;
      pr.elem_stiff.insert(pr.elem_stiff.end(), {w, -w, -w, w});
      pr.elem_inv_area.push_back(1.0 / (w * h * h));
    }
    pr.build_pattern();

    // conductivity mass, 2-point Gauss (proj/src/problem.cpp:278-305)
    const double gauss = 1.0 / std::sqrt(3.0);
    for (int e = 0; e < n_elems; ++e) {
      if (sigma[e] == 0.0) continue;
      const double ra = radii[e], rb = radii[e + 1];
      const double jac = 0.5 * h;
      double m[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      for (double xi : {-gauss, gauss}) {
        const double r = 0.5 * (ra + rb) + 0.5 * h * xi;
        const double phi[2] = {0.5 * (1.0 - xi), 0.5 * (1.0 + xi)};
        const double weight = sigma[e] * 2.0 * kPi * r * jac;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) m[a][b] += weight * (phi[a] * phi[b]);
      }
      const int idx[2] = {e, e + 1};
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          if (idx[a] < pr.dim && idx[b] < pr.dim) pr.mass[pr.slot(idx[a], idx[b])] += m[a][b];
    }

    // unit source current load vector (proj/src/problem.cpp:307-329)
    const double src_a = P.source_region == 0 ? 0.0 : bounds[P.source_region - 1];
    const double src_b = P.source_region == 2 ? P.r3 : bounds[P.source_region];
    const double density = 1.0 / (kPi * (src_b * src_b - src_a * src_a));
    std::vector<double> pattern(pr.dim, 0.0);
    for (int e = 0; e < n_elems; ++e) {
      const double ra = radii[e], rb = radii[e + 1];
      const double lo = std::max(ra, src_a), hi = std::min(rb, src_b);
      if (hi <= lo) continue;
      const double jac = 0.5 * (hi - lo);
      for (double xi : {-gauss, gauss}) {
        const double r = 0.5 * (lo + hi) + jac * xi;
        const double phi_a = (rb - r) / h;
        const double phi_b = (r - ra) / h;
        const double w = density * 2.0 * kPi * r * jac;
        if (e < pr.dim) pattern[e] += w * phi_a;
        if (e + 1 < pr.dim) pattern[e + 1] += w * phi_b;
      }
    }
    pr.patterns = pattern;
    pr.amplitude = {P.current};
    pr.frequency = {P.frequency_hz};
    pr.phase = {0.0};
    pr.desc.period = 1.0 / P.frequency_hz;
    pr.linear = P.linear_sleeve != 0;
    if (pr.linear) pr.assemble_linear_stiffness();
    const double period = pr.desc.period;
    pr.finalize();
    pr.desc.period = period;
    *out = pb;
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

// Canonical structured polar P1 mesh: a centre node,
// rings i = 1..nr at r_i = i R / nr with ntheta nodes each (ring nr Dirichlet),
// a centre fan of ntheta triangles and every ring quad split along the
// (i,j)-(i+1,j+1) diagonal.  d = 1 + (nr-1) ntheta, E = ntheta (2 nr - 1).
int ps_build_polar_cable(const ps_polar_cable_params* params, ps_problem** out) {
  if (!params || !out) return PS_ERR_BAD_ARG;
  try {
    const ps_polar_cable_params& P = *params;
    if (P.nr < 2 || P.ntheta < 3) throw std::runtime_error("problem: polar mesh too small");
    if (!(0.0 < P.r_conductor && P.r_conductor < P.r_insulator && P.r_insulator < P.radius))
      throw std::runtime_error("problem: cable radii must satisfy 0 < r1 < r2 < R");
    if (P.sigma_conductor < 0 || P.sigma_insulator < 0 || P.sigma_sheath < 0)
      throw std::runtime_error("problem: conductivities must be non-negative");
    if (!(P.frequency_hz > 0.0)) throw std::runtime_error("problem: frequency must be positive");
    if (!P.linear_sheath && (!(P.brauer_k1 > 0) || !(P.brauer_k2 > 0) || !(P.brauer_k3 > 0)))
      throw std::runtime_error("problem: Brauer coefficients must be positive");
    const int nr = P.nr, nt = P.ntheta;
    const int64_t dim64 = 1 + static_cast<int64_t>(nr - 1) * nt;
    const int64_t nnz64 = 1 + static_cast<int64_t>(nt) * (7 * static_cast<int64_t>(nr) - 9);
    if (dim64 > (1LL << 30) || nnz64 >= (1LL << 31))
      throw std::runtime_error("problem: polar mesh exceeds int32 indexing");

    auto pb = new ps_problem();
    ps_problem& pr = *pb;
    pr.dim = static_cast<int>(dim64);
    pr.npe = 3;
    auto node = [&](int ring, int j) -> int32_t {
      if (ring == 0) return 0;
      if (ring >= nr) return -1;
      return 1 + (ring - 1) * nt + ((j % nt) + nt) % nt;
    };
    std::vector<double> cs(nt), sn(nt);
    for (int j = 0; j < nt; ++j) {
      const double th = 2.0 * kPi * j / nt;
      cs[j] = std::cos(th);
      sn[j] = std::sin(th);
    }
    auto xy = [&](int ring, int j, double& x, double& y) {
      const double r = P.radius * ring / nr;
      const int jj = ((j % nt) + nt) % nt;
      x = r * cs[jj];
      y = r * sn[jj];
    };
    pr.coords.resize(static_cast<size_t>(pr.dim) * 2);
    pr.coords[0] = pr.coords[1] = 0.0;
    for (int ring = 1; ring < nr; ++ring)
      for (int j = 0; j < nt; ++j) {
        const int32_t id = node(ring, j);
        xy(ring, j, pr.coords[2 * id], pr.coords[2 * id + 1]);
      }

    ps_curve vac{};
    vac.kind = 0;
    vac.nu = kVacuumReluctivity;
    ps_curve steel{};
    if (P.linear_sheath) {
      steel.kind = 0;
      steel.nu = P.brauer_k1 + P.brauer_k3;
    } else {
      steel.kind = 1;
      steel.k1 = P.brauer_k1;
      steel.k2 = P.brauer_k2;
      steel.k3 = P.brauer_k3;
    }
    pr.curves = {vac, steel};

    const int64_t n_elem = static_cast<int64_t>(nt) * (2 * nr - 1);
    pr.elem_nodes.reserve(n_elem * 3);
    pr.elem_stiff.reserve(n_elem * 9);
    pr.elem_inv_area.reserve(n_elem);
    pr.elem_curve.reserve(n_elem);
    std::vector<double> area;
    std::vector<int8_t> region;
    area.reserve(n_elem);
    region.reserve(n_elem);

    auto add_tri = [&](int r0, int j0, int r1, int j1, int r2, int j2, int band) {
      double x[3], y[3];
      xy(r0, j0, x[0], y[0]);
      xy(r1, j1, x[1], y[1]);
      xy(r2, j2, x[2], y[2]);
      const double two_a = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
      const double a = 0.5 * std::fabs(two_a);
      double b[3], c[3];
      for (int k = 0; k < 3; ++k) {
        const int k1 = (k + 1) % 3, k2 = (k + 2) % 3;
        b[k] = y[k1] - y[k2];
        c[k] = x[k2] - x[k1];
      }
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) pr.elem_stiff.push_back((b[k] * b[l] + c[k] * c[l]) / (4.0 * a));
      pr.elem_nodes.push_back(node(r0, j0));
      pr.elem_nodes.push_back(node(r1, j1));
      pr.elem_nodes.push_back(node(r2, j2));
      pr.elem_inv_area.push_back(1.0 / a);
      // region by the band's mid radius, like the reference's element midpoint rule
      const double mid = P.radius * (band + 0.5) / nr;
      const int reg = mid < P.r_conductor ? 0 : (mid < P.r_insulator ? 1 : 2);
      region.push_back(static_cast<int8_t>(reg));
      pr.elem_curve.push_back(reg == 2 ? 1 : 0);
      area.push_back(a);
    };
    for (int j = 0; j < nt; ++j) add_tri(0, 0, 1, j, 1, j + 1, 0);
    for (int i = 1; i < nr; ++i)
      for (int j = 0; j < nt; ++j) {
        add_tri(i, j, i + 1, j, i + 1, j + 1, i);  // (a, d, c)
        add_tri(i, j, i + 1, j + 1, i, j + 1, i);  // (a, c, b)
      }
    pr.build_pattern();

    // consistent P1 conductivity mass sigma A/12 [[2,1,1],[1,2,1],[1,1,2]]; the
    // source patterns are uniform current densities whose P1 loads A/3 on the
    // free nodes are normalised so the conductor carries exactly +1 and the
    // sheath returns exactly -1 (the Dirichlet ring takes no share)
    const double region_sigma[3] = {P.sigma_conductor, P.sigma_insulator, P.sigma_sheath};
    std::vector<double> load_c(pr.dim, 0.0), load_s(pr.dim, 0.0);
    double sum_c = 0.0, sum_s = 0.0;
    for (int64_t e = 0; e < n_elem; ++e) {
      const double s = region_sigma[region[e]];
      const int32_t* nd = &pr.elem_nodes[e * 3];
      if (s != 0.0) {
        const double m = s * area[e] / 12.0;
        for (int a = 0; a < 3; ++a) {
          if (nd[a] < 0) continue;
          for (int b = 0; b < 3; ++b) {
            if (nd[b] < 0) continue;
            pr.mass[pr.slot(nd[a], nd[b])] += (a == b ? 2.0 : 1.0) * m;
          }
        }
      }
      if (region[e] == 1) continue;
      const double w = area[e] / 3.0;
      std::vector<double>& load = region[e] == 0 ? load_c : load_s;
      double& sum = region[e] == 0 ? sum_c : sum_s;
      for (int a = 0; a < 3; ++a)
        if (nd[a] >= 0) {
          load[nd[a]] += w;
          sum += w;
        }
    }
    std::vector<double> pattern(pr.dim, 0.0);
    for (int i = 0; i < pr.dim; ++i) {
      // (a region without elements carries no source)
      pattern[i] = sum_c > 0.0 ? load_c[i] / sum_c : 0.0;
      if (P.return_in_sheath && sum_s > 0.0) pattern[i] -= load_s[i] / sum_s;
    }

    // excitation: I0 sin(2 pi f t) plus an optional odd-harmonic square ripple
    pr.patterns = pattern;
    pr.amplitude = {P.current};
    pr.frequency = {P.frequency_hz};
    pr.phase = {0.0};
    for (int k = 0; k < P.ripple_terms; ++k) {
      const int harm = 2 * k + 1;
      pr.patterns.insert(pr.patterns.end(), pattern.begin(), pattern.end());
      pr.amplitude.push_back(P.ripple_fraction * P.current * 4.0 / (kPi * harm));
      pr.frequency.push_back(P.ripple_frequency_hz * harm);
      pr.phase.push_back(0.0);
    }
    pr.linear = P.linear_sheath != 0;
    if (pr.linear) pr.assemble_linear_stiffness();
    pr.finalize();
    pr.desc.period = 1.0 / P.frequency_hz;
    *out = pb;
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

const ps_problem_desc* ps_problem_get_desc(const ps_problem* p) { return p ? &p->desc : nullptr; }

const double* ps_problem_coordinates(const ps_problem* p) {
  return (p && !p->coords.empty()) ? p->coords.data() : nullptr;
}

void ps_problem_free(ps_problem* p) { delete p; }

const char* ps_builder_error(void) { return g_builder_error.c_str(); }

void ps_seeded_normal(uint64_t seed, int64_t count, double sigma, double* out) {
  std::mt19937_64 gen(seed);
  const double scale = 1.0 / 9007199254740992.0;  // 2^-53
  for (int64_t i = 0; i < count; i += 2) {
    const double u1 = (static_cast<double>(gen() >> 11) + 1.0) * scale;  // (0, 1]
    const double u2 = static_cast<double>(gen() >> 11) * scale;          // [0, 1)
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * kPi * u2;
    out[i] = sigma * rad * std::cos(ang);
    if (i + 1 < count) out[i + 1] = sigma * rad * std::sin(ang);
  }
}

void ps_seeded_uniform(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  std::mt19937_64 gen(seed);
  const double scale = 1.0 / 9007199254740992.0;
  for (int64_t i = 0; i < count; ++i)
    out[i] = lo + (hi - lo) * (static_cast<double>(gen() >> 11) * scale);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Files: Matrix Market, excitation JSON, shortest round-trip CSV writers
// (SURVEY.md §8f ranks 2-3).  Host C++, no third-party parser: a restatement of
// proj/src/matrix_market.cpp:30-98, proj/src/problem.cpp:363-421 (the JSON
// schema nlohmann::json parses there) and proj/src/io.cpp:151-178.
#include <cerrno>
#include <charconv>
#include <cstdlib>
#include <string_view>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>

struct ps_csr {
  int32_t rows = 0, cols = 0;
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<double> values;
};

namespace {

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

std::string shortest(double x) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof(buf), x);
  return std::string(buf, res.ptr);
}

struct Trip {
  int32_t i, j;
  double v;
};

// triplets -> CSR with duplicates summed (Eigen setFromTriplets semantics)
ps_csr to_csr(int32_t rows, int32_t cols, std::vector<Trip> t) {
  std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) { return a.i != b.i ? a.i < b.i : a.j < b.j; });
  ps_csr m;
  m.rows = rows;
  m.cols = cols;
  m.row_ptr.assign(static_cast<size_t>(rows) + 1, 0);
  for (size_t k = 0; k < t.size(); ++k) {
    if (!m.col_idx.empty() && k > 0 && t[k].i == t[k - 1].i && t[k].j == t[k - 1].j) {
      m.values.back() += t[k].v;
      continue;
    }
    m.col_idx.push_back(t[k].j);
    m.values.push_back(t[k].v);
    m.row_ptr[t[k].i + 1] = static_cast<int32_t>(m.col_idx.size());
  }
  for (int32_t r = 0; r < rows; ++r) m.row_ptr[r + 1] = std::max(m.row_ptr[r + 1], m.row_ptr[r]);
  return m;
}

// Matrix Market coordinate files (the subset read_matrix_market accepts,
// proj/src/matrix_market.cpp:30-81: real, general or symmetric, 1-based).  The
// file is read whole and walked by a cursor over its data lines; numbers are
// parsed with strtol / strtod so a stray token anywhere in a line is an error.
class MMCursor {
 public:
  MMCursor(std::string text, std::string path) : text_(std::move(text)), path_(std::move(path)) {}

  [[noreturn]] void fail(const std::string& what) const { throw std::runtime_error("matrix_market: " + what + path_); }

  // next line (without the newline); false at end of file
  bool line(std::string_view* out) {
    if (pos_ >= text_.size()) return false;
    const size_t nl = text_.find('\n', pos_);
    const size_t end = nl == std::string::npos ? text_.size() : nl;
    *out = std::string_view(text_).substr(pos_, end - pos_);
    if (!out->empty() && out->back() == '\r') out->remove_suffix(1);
    pos_ = end + 1;
    return true;
  }
  // next line that is neither blank nor a % comment
  bool data_line(std::string_view* out) {
    while (line(out)) {
      const size_t k = out->find_first_not_of(" \t");
      if (k != std::string_view::npos && (*out)[k] != '%') return true;
    }
    return false;
  }

 private:
  std::string text_, path_;
  size_t pos_ = 0;
};

// whitespace-separated fields of one line; exactly `n` of them must parse
bool mm_fields(std::string_view ln, int n, long* ints, double* real) {
  std::string buf(ln);
  const char* c = buf.c_str();
  for (int f = 0; f < n; ++f) {
    char* end = nullptr;
    errno = 0;
    if (real && f == n - 1) {
      *real = std::strtod(c, &end);
    } else {
      ints[f] = std::strtol(c, &end, 10);
    }
    if (end == c || errno != 0 || (*end != '\0' && *end != ' ' && *end != '\t')) return false;
    c = end;
  }
  while (*c == ' ' || *c == '\t') ++c;
  return *c == '\0';
}

ps_csr read_mm(const std::string& path) {
  std::ifstream file(path, std::ios::binary);
  if (!file) throw std::runtime_error("matrix_market: cannot open " + path);
  std::ostringstream whole;
  whole << file.rdbuf();
  MMCursor cur(whole.str(), " in " + path);
  std::string_view first;
  if (!cur.line(&first)) cur.fail("empty file");
  // banner: %%MatrixMarket matrix <format> <field> <symmetry>
  std::vector<std::string> word;
  {
    std::istringstream ws{std::string(first)};
    for (std::string w; ws >> w;) word.push_back(lower(w));
  }
  if (word.size() < 5 || word[0] != "%%matrixmarket" || word[1] != "matrix") cur.fail("bad header");
  if (word[2] != "coordinate") cur.fail("only coordinate format is supported");
  if (word[3] != "real") cur.fail("only real matrices are supported");
  const bool mirrored = word[4] == "symmetric";
  if (!mirrored && word[4] != "general") cur.fail("only general or symmetric storage is supported");
  std::string_view ln;
  long shape[3];
  if (!cur.data_line(&ln)) cur.fail("missing size line");
  if (!mm_fields(ln, 3, shape, nullptr) || shape[0] < 0 || shape[1] < 0 || shape[2] < 0)
    cur.fail("malformed size line");
  const long n_rows = shape[0], n_cols = shape[1], declared = shape[2];
  std::vector<Trip> entries;
  entries.reserve(static_cast<size_t>(mirrored ? 2 * declared : declared));
  long read = 0;
  for (; read < declared && cur.data_line(&ln); ++read) {
    long ij[2];
    double v = 0.0;
    if (!mm_fields(ln, 3, ij, &v)) cur.fail("malformed entry");
    if (ij[0] < 1 || ij[0] > n_rows || ij[1] < 1 || ij[1] > n_cols) cur.fail("index out of range");
    const auto r = static_cast<int32_t>(ij[0] - 1), c = static_cast<int32_t>(ij[1] - 1);
    entries.push_back({r, c, v});
    if (mirrored && r != c) entries.push_back({c, r, v});
  }
  if (read != declared)
    cur.fail("expected " + std::to_string(declared) + " entries, got " + std::to_string(read));
  return to_csr(static_cast<int32_t>(n_rows), static_cast<int32_t>(n_cols), std::move(entries));
}

// ---- a small JSON reader for the excitation schema
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JsonParser {
  const std::string& s;
  size_t p = 0;
  [[noreturn]] void fail(const std::string& what) {
    throw std::runtime_error("problem: excitation JSON parse error: " + what + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
  }
  Json value() {
    ws();
    if (p >= s.size()) fail("unexpected end of input");
    const char c = s[p];
    Json j;
    if (c == '{') {
      j.kind = Json::Obj;
      ++p;
      ws();
      if (p < s.size() && s[p] == '}') {
        ++p;
        return j;
      }
      for (;;) {
        ws();
        if (p >= s.size() || s[p] != '"') fail("expected a key");
        std::string k = string();
        ws();
        if (p >= s.size() || s[p] != ':') fail("expected ':'");
        ++p;
        j.obj.emplace_back(std::move(k), value());
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == '}') {
          ++p;
          return j;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      j.kind = Json::Arr;
      ++p;
      ws();
      if (p < s.size() && s[p] == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == ']') {
          ++p;
          return j;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      j.kind = Json::Str;
      j.str = string();
      return j;
    }
    if (s.compare(p, 4, "true") == 0) {
      p += 4;
      j.kind = Json::Bool;
      j.b = true;
      return j;
    }
    if (s.compare(p, 5, "false") == 0) {
      p += 5;
      j.kind = Json::Bool;
      return j;
    }
    if (s.compare(p, 4, "null") == 0) {
      p += 4;
      return j;
    }
    const char* b = s.c_str() + p;
    char* e = nullptr;
    j.num = std::strtod(b, &e);
    if (e == b) fail("unexpected character");
    p += static_cast<size_t>(e - b);
    j.kind = Json::Num;
    return j;
  }
  std::string string() {
    ++p;  // opening quote
    std::string out;
    while (p < s.size() && s[p] != '"') {
      if (s[p] == '\\' && p + 1 < s.size()) ++p;
      out.push_back(s[p++]);
    }
    if (p >= s.size()) fail("unterminated string");
    ++p;
    return out;
  }
};

bool is_int(const Json& j) { return j.kind == Json::Num && j.num == std::floor(j.num); }

// relative_asymmetry (proj/src/problem.cpp:21-32) of a CSR matrix
double asymmetry(const ps_csr& a) {
  std::map<std::pair<int32_t, int32_t>, double> v;
  double scale = 1.0;
  for (int32_t i = 0; i < a.rows; ++i)
    for (int32_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      v[{i, a.col_idx[k]}] += a.values[k];
      scale = std::max(scale, std::abs(a.values[k]));
    }
  double asym = 0.0;
  for (const auto& kv : v) {
    const auto it = v.find({kv.first.second, kv.first.first});
    asym = std::max(asym, std::abs(kv.second - (it == v.end() ? 0.0 : it->second)));
  }
  return asym / scale;
}

}  // namespace

extern "C" {

int ps_mm_read(const char* path, ps_csr** out) {
  if (!path || !out) return PS_ERR_BAD_ARG;
  try {
    *out = new ps_csr(read_mm(path));
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

int ps_csr_shape(const ps_csr* m, int32_t* rows, int32_t* cols, int64_t* nnz) {
  if (!m) return PS_ERR_BAD_ARG;
  if (rows) *rows = m->rows;
  if (cols) *cols = m->cols;
  if (nnz) *nnz = static_cast<int64_t>(m->col_idx.size());
  return PS_OK;
}
const int32_t* ps_csr_row_ptr(const ps_csr* m) { return m ? m->row_ptr.data() : nullptr; }
const int32_t* ps_csr_col_idx(const ps_csr* m) { return m ? m->col_idx.data() : nullptr; }
const double* ps_csr_values(const ps_csr* m) { return m ? m->values.data() : nullptr; }
void ps_csr_free(ps_csr* m) { delete m; }

// write_matrix_market (proj/src/matrix_market.cpp:83-93): general storage, the
// entries in column-major order (Eigen's compressed column order), values in
// the shortest round-trip decimal form.
int ps_mm_write(const char* path, int32_t rows, int32_t cols, const int32_t* row_ptr, const int32_t* col_idx,
                const double* values) {
  if (!path || rows < 0 || cols < 0 || !row_ptr) return PS_ERR_BAD_ARG;
  try {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("matrix_market: cannot write ") + path);
    std::vector<Trip> t;
    for (int32_t i = 0; i < rows; ++i)
      for (int32_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) t.push_back({i, col_idx[k], values[k]});
    std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) { return a.j != b.j ? a.j < b.j : a.i < b.i; });
    out << "%%MatrixMarket matrix coordinate real general\n";
    out << rows << " " << cols << " " << t.size() << "\n";
    for (const Trip& e : t) out << e.i + 1 << " " << e.j + 1 << " " << shortest(e.v) << "\n";
    if (!out) throw std::runtime_error(std::string("matrix_market: write failed for ") + path);
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

// load_problem + parse_excitation_text (proj/src/problem.cpp:363-421): linear
// problem M du/dt + K u = f(t) from two Matrix Market files and the excitation
// JSON {"period": T, "terms": [{"amplitude", "frequency", "phase"?, "dofs",
// "values"}]}.  The device pattern is the symmetric union of both patterns plus
// the diagonal; the values are the files' values (explicit zeros elsewhere).
int ps_load_problem(const char* mass_path, const char* stiffness_path, const char* excitation_path,
                    ps_problem** out) {
  if (!mass_path || !stiffness_path || !excitation_path || !out) return PS_ERR_BAD_ARG;
  *out = nullptr;
  try {
    const ps_csr M = read_mm(mass_path), K = read_mm(stiffness_path);
    if (M.rows != K.rows || M.cols != K.cols)
      throw std::runtime_error("problem: mass and stiffness dimensions do not match");
    if (M.rows != M.cols) throw std::runtime_error("problem: matrices must be square");
    std::ifstream in(excitation_path);
    if (!in) throw std::runtime_error(std::string("problem: cannot open excitation file ") + excitation_path);
    std::stringstream buf;
    buf << in.rdbuf();
    const std::string text = buf.str();
    JsonParser jp{text};
    const Json spec = jp.value();
    const int dim = M.rows;
    if (spec.kind != Json::Obj) throw std::runtime_error("problem: excitation spec must be an object");
    for (const auto& kv : spec.obj)
      if (kv.first != "period" && kv.first != "terms")
        throw std::runtime_error("problem: unknown excitation key \"" + kv.first + "\"");
    const Json* per = spec.get("period");
    const Json* terms = spec.get("terms");
    if (!per || per->kind != Json::Num) throw std::runtime_error("problem: excitation spec needs a numeric \"period\"");
    if (!terms || terms->kind != Json::Arr) throw std::runtime_error("problem: excitation spec needs a \"terms\" array");
    auto p = std::make_unique<ps_problem>();
    p->linear = true;
    p->dim = dim;
    const double period = per->num;
    for (const Json& t : terms->arr) {
      if (t.kind != Json::Obj) throw std::runtime_error("problem: excitation term must be an object");
      for (const auto& kv : t.obj)
        if (kv.first != "amplitude" && kv.first != "frequency" && kv.first != "phase" && kv.first != "dofs" &&
            kv.first != "values")
          throw std::runtime_error("problem: unknown excitation term key \"" + kv.first + "\"");
      const Json *amp = t.get("amplitude"), *fr = t.get("frequency"), *ph = t.get("phase"), *dofs = t.get("dofs"),
                 *vals = t.get("values");
      if (!amp || !fr) throw std::runtime_error("problem: excitation term needs amplitude and frequency");
      if (amp->kind != Json::Num || fr->kind != Json::Num || (ph && ph->kind != Json::Num))
        throw std::runtime_error("problem: excitation term values must be numbers");
      if (!dofs || !vals || dofs->kind != Json::Arr || vals->kind != Json::Arr || dofs->arr.size() != vals->arr.size())
        throw std::runtime_error("problem: excitation term needs matching dofs/values arrays");
      std::vector<double> pattern(static_cast<size_t>(dim), 0.0);
      for (size_t i = 0; i < dofs->arr.size(); ++i) {
        if (!is_int(dofs->arr[i]) || vals->arr[i].kind != Json::Num)
          throw std::runtime_error("problem: excitation dofs must be integers and values numbers");
        const double dof = dofs->arr[i].num;
        if (dof < 0 || dof >= dim) throw std::runtime_error("problem: excitation dof index out of range");
        pattern[static_cast<size_t>(dof)] = vals->arr[i].num;
      }
      p->patterns.insert(p->patterns.end(), pattern.begin(), pattern.end());
      p->amplitude.push_back(amp->num);
      p->frequency.push_back(fr->num);
      p->phase.push_back(ph ? ph->num : 0.0);
    }
    // Excitation::Excitation (proj/src/problem.cpp:36-50)
    if (!(period > 0.0)) throw std::runtime_error("problem: excitation period must be positive");
    for (double f : p->frequency) {
      if (!(f > 0.0)) throw std::runtime_error("problem: excitation frequency must be positive");
      const double cycles = f * period;
      if (std::abs(cycles - std::round(cycles)) > 1e-9 * std::max(1.0, cycles))
        throw std::runtime_error("problem: excitation frequency is not an integer multiple of 1/period");
    }
    // PeriodicProblem::PeriodicProblem (proj/src/problem.cpp:100-113)
    if (asymmetry(M) > 1e-12) throw std::runtime_error("problem: mass matrix is not symmetric");
    if (asymmetry(K) > 1e-12) throw std::runtime_error("problem: stiffness matrix is not symmetric");
    // symmetric union pattern with the diagonal
    std::vector<std::vector<int32_t>> cols(static_cast<size_t>(dim));
    for (const ps_csr* A : {&M, &K})
      for (int32_t i = 0; i < dim; ++i)
        for (int32_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) {
          cols[i].push_back(A->col_idx[k]);
          cols[A->col_idx[k]].push_back(i);
        }
    p->row_ptr.assign(static_cast<size_t>(dim) + 1, 0);
    for (int32_t i = 0; i < dim; ++i) {
      cols[i].push_back(i);
      std::sort(cols[i].begin(), cols[i].end());
      cols[i].erase(std::unique(cols[i].begin(), cols[i].end()), cols[i].end());
      p->col_idx.insert(p->col_idx.end(), cols[i].begin(), cols[i].end());
      p->row_ptr[i + 1] = static_cast<int32_t>(p->col_idx.size());
    }
    p->mass.assign(p->col_idx.size(), 0.0);
    p->stiffness.assign(p->col_idx.size(), 0.0);
    for (int32_t i = 0; i < dim; ++i) {
      for (int32_t k = M.row_ptr[i]; k < M.row_ptr[i + 1]; ++k) p->mass[p->slot(i, M.col_idx[k])] += M.values[k];
      for (int32_t k = K.row_ptr[i]; k < K.row_ptr[i + 1]; ++k)
        p->stiffness[p->slot(i, K.col_idx[k])] += K.values[k];
    }
    p->finalize();
    p->desc.period = period;
    *out = p.release();
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

// format_double / write_trajectory_csv / write_history_csv (proj/src/io.cpp:151-178)
int ps_format_double(double value, char* buf, int32_t len) {
  if (!buf || len < 1) return PS_ERR_BAD_ARG;
  const std::string s = shortest(value);
  if (static_cast<int32_t>(s.size()) >= len) return PS_ERR_BAD_ARG;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return PS_OK;
}

int ps_write_trajectory_csv(const char* path, int32_t count, int32_t dim, const double* states,
                            const ps_time_mesh* mesh) {
  if (!path || count < 0 || dim < 0 || (count > 0 && !states) || !mesh) return PS_ERR_BAD_ARG;
  try {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("io: cannot write ") + path);
    out << "n,t";
    for (int j = 0; j < dim; ++j) out << ",u" << j;
    out << "\n";
    for (int n = 0; n < count; ++n) {
      // TimeMesh::boundary (proj/include/parasteady/types.hpp:32-39)
      const double t = n == mesh->subintervals ? mesh->period : static_cast<double>(n) * mesh->period / mesh->subintervals;
      out << n << "," << shortest(t);
      for (int j = 0; j < dim; ++j) out << "," << shortest(states[static_cast<int64_t>(n) * dim + j]);
      out << "\n";
    }
    if (!out) throw std::runtime_error(std::string("io: write failed for ") + path);
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

int ps_write_history_csv(const char* path, int32_t count, const double* jumps, const double* seconds) {
  if (!path || count < 0 || (count > 0 && !jumps)) return PS_ERR_BAD_ARG;
  try {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(std::string("io: cannot write ") + path);
    out << "k,jump_norm,wall_time_s\n";
    for (int k = 0; k < count; ++k)
      out << k << "," << shortest(jumps[k]) << "," << shortest(seconds ? seconds[k] : 0.0) << "\n";
    if (!out) throw std::runtime_error(std::string("io: write failed for ") + path);
    return PS_OK;
  } catch (const std::exception& e) {
    g_builder_error = e.what();
    return PS_ERR_BAD_ARG;
  }
}

}  // extern "C"
