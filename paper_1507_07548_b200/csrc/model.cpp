// Host-side force-field setup for b200md.  See model.hpp.  Every constant is
// computed with the reference's operation order (no FMA contraction) so the
// device kernels consume bit-identical parameters.
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numbers>

#include "search_geometry.hpp"

namespace b2md {

namespace {

constexpr double kPi = std::numbers::pi;

struct V3 {
  double x, y, z;
};
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }

std::string fmt(const char* f, double a, double b = 0.0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b);
  return buf;
}

// Symmetric 3x3 Jacobi eigen-decomposition, eigenvalues ascending with a
// stable order for ties (the reference sorts 3 keys with std::sort, i.e. an
// insertion sort; src/model.cpp:12-60).
void jacobi3(const double m[3][3], double vals[3], double vecs[3][3]) {
  double a[3][3];
  std::memcpy(a, m, sizeof a);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vecs[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) off += a[p][q] * a[p][q];
    if (off < 1e-30) break;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (std::abs(a[p][q]) < 1e-300) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t =
            (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double kp = a[k][p], kq = a[k][q];
          a[k][p] = c * kp - s * kq;
          a[k][q] = s * kp + c * kq;
        }
        for (int k = 0; k < 3; ++k) {
          const double pk = a[p][k], qk = a[q][k];
          a[p][k] = c * pk - s * qk;
          a[q][k] = s * pk + c * qk;
        }
        for (int k = 0; k < 3; ++k) {
          const double kp = vecs[k][p], kq = vecs[k][q];
          vecs[k][p] = c * kp - s * kq;
          vecs[k][q] = s * kp + c * kq;
        }
      }
  }
  int order[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) {
    const int v = order[i];
    int j = i;
    for (; j > 0 && a[v][v] < a[order[j - 1]][order[j - 1]]; --j) order[j] = order[j - 1];
    order[j] = v;
  }
  double sorted[3][3];
  for (int j = 0; j < 3; ++j) {
    vals[j] = a[order[j]][order[j]];
    for (int i = 0; i < 3; ++i) sorted[i][j] = vecs[i][order[j]];
  }
  std::memcpy(vecs, sorted, sizeof sorted);
}

double net_charge(const ModelTables& t) {
  double q = 0.0;
  for (int s = 0; s < t.ns; ++s) q += t.counts[s] * t.species[s].net_charge;
  return q;
}

}  // namespace

int build_species(const b2md_site* in, int n, b2md_species& sp, std::string& err) {
  if (n <= 0) return err = "species: no sites", B2MD_MODEL_ERROR;
  if (n > B2MD_MAX_SITES) return err = "species: more than B2MD_MAX_SITES sites", B2MD_MODEL_ERROR;
  b2md_site s[B2MD_MAX_SITES];
  std::memcpy(s, in, sizeof(b2md_site) * n);
  double mass = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int k = 0; k < n; ++k) {
    if (s[k].kind == B2MD_SITE_DUMMY && (s[k].sigma != 0.0 || s[k].epsilon != 0.0))
      return err = "species: dummy site with nonzero sigma or epsilon", B2MD_MODEL_ERROR;
    if (s[k].kind == B2MD_SITE_LJ && s[k].sigma <= 0.0)
      return err = "species: LJ site with sigma <= 0", B2MD_MODEL_ERROR;
    if (s[k].kind == B2MD_SITE_LJ && s[k].epsilon < 0.0)
      return err = "species: LJ site with epsilon < 0", B2MD_MODEL_ERROR;
    if (s[k].mass < 0.0) return err = "species: negative site mass", B2MD_MODEL_ERROR;
    mass += s[k].mass;
    cx += s[k].body_pos[0] * s[k].mass;
    cy += s[k].body_pos[1] * s[k].mass;
    cz += s[k].body_pos[2] * s[k].mass;
  }
  if (mass <= 0.0) return err = "species: non-positive total mass", B2MD_MODEL_ERROR;
  const double inv = 1.0 / mass;
  cx *= inv;
  cy *= inv;
  cz *= inv;
  double I[3][3] = {};
  for (int k = 0; k < n; ++k) {
    s[k].body_pos[0] -= cx;
    s[k].body_pos[1] -= cy;
    s[k].body_pos[2] -= cz;
    const double x = s[k].body_pos[0], y = s[k].body_pos[1], z = s[k].body_pos[2];
    const double r2 = x * x + y * y + z * z;
    const double m = s[k].mass;
    I[0][0] += m * (r2 - x * x);
    I[1][1] += m * (r2 - y * y);
    I[2][2] += m * (r2 - z * z);
    I[0][1] -= m * x * y;
    I[0][2] -= m * x * z;
    I[1][2] -= m * y * z;
  }
  I[1][0] = I[0][1];
  I[2][0] = I[0][2];
  I[2][1] = I[1][2];
  double mom[3], ax[3][3];
  jacobi3(I, mom, ax);
  const double scale = std::max({mom[0], mom[1], mom[2], 0.0});
  for (double& m : mom)
    if (m < 1e-12 * scale || m < 1e-300) m = 0.0;
  std::memset(&sp, 0, sizeof sp);
  sp.n_sites = n;
  sp.total_mass = mass;
  for (int k = 0; k < 3; ++k) sp.inertia_principal[k] = mom[k];
  for (int k = 0; k < n; ++k) {
    const double x = s[k].body_pos[0], y = s[k].body_pos[1], z = s[k].body_pos[2];
    s[k].body_pos[0] = ax[0][0] * x + ax[1][0] * y + ax[2][0] * z;
    s[k].body_pos[1] = ax[0][1] * x + ax[1][1] * y + ax[2][1] * z;
    s[k].body_pos[2] = ax[0][2] * x + ax[1][2] * y + ax[2][2] * z;
    sp.sites[k] = s[k];
    sp.net_charge += s[k].q;
    sp.max_extent = std::max(sp.max_extent, norm({s[k].body_pos[0], s[k].body_pos[1], s[k].body_pos[2]}));
  }
  for (int k = 0; k < 3; ++k)
    if (sp.inertia_principal[k] > 0.0) ++sp.rotational_dof;
  return B2MD_OK;
}

int ewald_tune(double delta, double cutoff, double box, double& alpha, int& kmax, std::string& err) {
  if (!(delta > 0.0) || delta > 1e-2)
    return err = "ewald_tune: accuracy must lie in (0, 1e-2]", B2MD_CONFIG_ERROR;
  if (cutoff <= 0.0 || box <= 0.0) return err = "ewald_tune: bad geometry", B2MD_CONFIG_ERROR;
  double lo = 1e-6 / cutoff, hi = 40.0 / cutoff;
  if (std::erfc(lo * cutoff) < delta)
    return err = "ewald_tune: accuracy infeasible for this cutoff", B2MD_CONFIG_ERROR;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    (std::erfc(mid * cutoff) > delta ? lo : hi) = mid;
  }
  alpha = 0.5 * (lo + hi);
  const double x = std::sqrt(-std::log(delta));
  kmax = static_cast<int>(std::ceil(alpha * box * x / kPi));
  if (kmax < 1) kmax = 1;
  return B2MD_OK;
}

int count_kvectors(int kmax) {
  int c = 0;
  for (int nx = 0; nx <= kmax; ++nx)
    for (int ny = (nx == 0 ? 0 : -kmax); ny <= kmax; ++ny)
      for (int nz = (nx == 0 && ny == 0 ? 1 : -kmax); nz <= kmax; ++nz) {
        const long n2 = long(nx) * nx + long(ny) * ny + long(nz) * nz;
        if (n2 != 0 && n2 <= long(kmax) * kmax) ++c;
      }
  return c;
}

int build_tables(const b2md_composition& comp, const b2md_ff_options& opts, ModelTables& t,
                 std::string& err) {
  if (comp.n_species <= 0 || !comp.species || !comp.counts)
    return err = "composition: no molecules", B2MD_CONFIG_ERROR;
  t = ModelTables{};
  t.ns = comp.n_species;
  t.species.assign(comp.species, comp.species + t.ns);
  t.counts.assign(comp.counts, comp.counts + t.ns);
  t.box = comp.box_length;
  t.temperature = comp.temperature;
  for (const auto& sp : t.species)
    if (sp.n_sites < 1 || sp.n_sites > B2MD_MAX_SITES)
      return err = "species: site count out of range", B2MD_MODEL_ERROR;

  // ---- PairTable (src/potentials.cpp:35-83)
  const double cutoff = opts.cutoff;
  if (cutoff <= 0.0) return err = "pair table: cutoff must be positive", B2MD_CONFIG_ERROR;
  if (cutoff > 0.5 * comp.box_length + 1e-12)
    return err = fmt("pair table: cutoff %f exceeds half the box length %f", cutoff,
                     0.5 * comp.box_length),
           B2MD_CONFIG_ERROR;
  t.method = opts.method;
  t.rc = cutoff;
  t.rc2 = cutoff * cutoff;
  if (t.method == B2MD_METHOD_REACTION_FIELD) {
    const double e = opts.eps_rf;
    if (!(e > 1.0) && !std::isinf(e))
      return err = "reaction field: epsilon_rf must exceed 1", B2MD_CONFIG_ERROR;
    t.rf_factor = std::isinf(e) ? 0.5 : (e - 1.0) / (2.0 * e + 1.0);
    t.rf_r3inv = t.rf_factor / (cutoff * cutoff * cutoff);
    t.rf_shift = -(1.0 + t.rf_factor) / cutoff;
  }
  t.alpha = (t.method == B2MD_METHOD_EWALD && opts.has_ewald) ? opts.ewald_alpha : 0.0;
  if (t.method == B2MD_METHOD_EWALD && t.alpha <= 0.0)
    return err = "pair table: ewald method requires alpha > 0", B2MD_CONFIG_ERROR;
  const int ns = t.ns;
  t.lj.assign(ns * ns, {});
  t.qq.assign(ns * ns, {});
  t.rmax2.assign(ns * ns, 0.0);
  for (int sa = 0; sa < ns; ++sa)
    for (int sb = 0; sb < ns; ++sb) {
      const b2md_species& A = t.species[sa];
      const b2md_species& B = t.species[sb];
      for (int ia = 0; ia < A.n_sites; ++ia)
        for (int ib = 0; ib < B.n_sites; ++ib) {
          const b2md_site& a = A.sites[ia];
          const b2md_site& b = B.sites[ib];
          if (a.kind != B2MD_SITE_CHARGE && b.kind != B2MD_SITE_CHARGE) {
            const double eps = std::sqrt(a.epsilon * b.epsilon);
            if (eps > 0.0) {
              const double sigma = 0.5 * (a.sigma + b.sigma);
              const double s3 = sigma * sigma * sigma;
              const double s6 = s3 * s3;
              t.lj[sa * ns + sb].push_back({ia, ib, 4.0 * eps * s6 * s6, 4.0 * eps * s6});
            }
          }
          if (t.method != B2MD_METHOD_NONE && a.q != 0.0 && b.q != 0.0)
            t.qq[sa * ns + sb].push_back({ia, ib, a.q * b.q});
        }
      // COM search radius of src/potentials.cpp:212-213
      const double rmax = cutoff + A.max_extent + B.max_extent;
      t.rmax2[sa * ns + sb] = rmax * rmax;
    }
  t.single_lj_only = true;
  for (const auto& sp : t.species)
    if (sp.n_sites != 1 || sp.sites[0].kind != B2MD_SITE_LJ) t.single_lj_only = false;
  t.single_site_path = t.single_lj_only && t.method != B2MD_METHOD_EWALD;

  // ---- lj_lrc (src/potentials.cpp:7-33)
  {
    struct Ty {
      double sigma, eps;
      long count;
    };
    std::vector<Ty> ty;
    for (int s = 0; s < ns; ++s)
      for (int k = 0; k < t.species[s].n_sites; ++k) {
        const b2md_site& st = t.species[s].sites[k];
        if (st.kind != B2MD_SITE_CHARGE && st.epsilon > 0.0)
          ty.push_back({st.sigma, st.epsilon, long(t.counts[s])});
      }
    double k = 0.0;
    for (const auto& a : ty)
      for (const auto& b : ty) {
        const double sigma = 0.5 * (a.sigma + b.sigma);
        const double eps = std::sqrt(a.eps * b.eps);
        const double sr3 = sigma * sigma * sigma / (cutoff * cutoff * cutoff);
        const double sr9 = sr3 * sr3 * sr3;
        k += (8.0 * kPi / 3.0) * static_cast<double>(a.count) * static_cast<double>(b.count) * eps *
             sigma * sigma * sigma * (sr9 / 3.0 - sr3);
      }
    t.lrc_k = k;
  }

  // ---- SystemComposition::validate (src/model.cpp:244-268)
  long nmol = 0;
  for (int c : t.counts) nmol += c;
  if (nmol <= 0) return err = "composition: no molecules", B2MD_CONFIG_ERROR;
  for (int c : t.counts)
    if (c < 0) return err = "composition: negative molecule count", B2MD_CONFIG_ERROR;
  if (t.box <= 0.0) return err = "composition: box length must be positive", B2MD_CONFIG_ERROR;
  if (t.temperature <= 0.0)
    return err = "composition: temperature must be positive", B2MD_CONFIG_ERROR;
  if (t.method == B2MD_METHOD_EWALD) {
    if (std::abs(net_charge(t)) > 1e-12)
      return err = fmt("ewald requires an electro-neutral system (net charge %f)", net_charge(t)),
             B2MD_CONFIG_ERROR;
  } else if (t.method == B2MD_METHOD_REACTION_FIELD) {
    for (const auto& sp : t.species)
      if (std::abs(sp.net_charge) > 1e-12)
        return err = "reaction_field requires neutral molecules", B2MD_CONFIG_ERROR;
  } else {
    for (const auto& sp : t.species)
      for (int k = 0; k < sp.n_sites; ++k)
        if (sp.sites[k].q != 0.0)
          return err = "species has point charges; choose electrostatics = reaction_field or ewald",
                 B2MD_CONFIG_ERROR;
  }
  if (nmol > (1L << 24)) return err = "composition: too many molecules", B2MD_CONFIG_ERROR;

  // ---- scene indexing (src/potentials.cpp:94-104)
  t.n = int(nmol);
  t.species_of.resize(t.n);
  t.site_begin.resize(t.n + 1);
  int sites = 0, m = 0;
  for (int s = 0; s < ns; ++s)
    for (int c = 0; c < t.counts[s]; ++c, ++m) {
      t.species_of[m] = s;
      t.site_begin[m] = sites;
      sites += t.species[s].n_sites;
    }
  t.site_begin[t.n] = sites;
  t.total_sites = sites;
  for (const auto& sp : t.species) {
    if (sp.rotational_dof > 0) t.any_rigid = true;
    const b2md_site& s0 = sp.sites[0];
    const double n2 = s0.body_pos[0] * s0.body_pos[0] + s0.body_pos[1] * s0.body_pos[1] +
                      s0.body_pos[2] * s0.body_pos[2];
    if (sp.n_sites > 1 || n2 != 0.0) t.any_offsets = true;
  }
  t.vderiv = opts.volume_derivatives != 0;

  // ---- Ewald (src/parallel.cpp:63-69, src/ewald.cpp:30-105)
  if (t.method == B2MD_METHOD_EWALD) {
    if (!opts.has_ewald)
      return err = "force field: ewald method without ewald parameters", B2MD_CONFIG_ERROR;
    if (opts.workers != 1)
      return err = "force field: ewald summation runs single-threaded (worker count must be 1)",
             B2MD_CONFIG_ERROR;
    t.ewald = true;
    t.kmax = opts.ewald_kmax;
    const double alpha = t.alpha;
    if (alpha <= 0.0) return err = "ewald: alpha must be positive", B2MD_CONFIG_ERROR;
    if (t.kmax < 1) return err = "ewald: kmax must be at least 1", B2MD_CONFIG_ERROR;
    if (std::abs(net_charge(t)) > 1e-12)
      return err = "ewald: system is not electro-neutral", B2MD_CONFIG_ERROR;
    const double L = t.box;
    const double tail = std::exp(-std::pow(kPi * t.kmax / (alpha * L), 2));
    if (tail > 1e-2) {
      char buf[256];
      std::snprintf(buf, sizeof buf,
                    "ewald: reciprocal truncation estimate %f at kmax = %d looks too coarse", tail,
                    t.kmax);
      t.warning = buf;
    }
    double sum_q2 = 0.0, intra = 0.0;
    for (int s = 0; s < ns; ++s) {
      const b2md_species& sp = t.species[s];
      const long cnt = t.counts[s];
      std::vector<int> ch;
      for (int k = 0; k < sp.n_sites; ++k)
        if (sp.sites[k].q != 0.0) ch.push_back(k);
      for (int a : ch) sum_q2 += cnt * sp.sites[a].q * sp.sites[a].q;
      double corr = 0.0;
      for (std::size_t a = 0; a < ch.size(); ++a)
        for (std::size_t b = a + 1; b < ch.size(); ++b) {
          const b2md_site& A = sp.sites[ch[a]];
          const b2md_site& B = sp.sites[ch[b]];
          const double r = norm({A.body_pos[0] - B.body_pos[0], A.body_pos[1] - B.body_pos[1],
                                 A.body_pos[2] - B.body_pos[2]});
          const double qq = A.q * B.q;
          if (r < 1e-12)
            corr += qq * 2.0 * alpha / std::sqrt(kPi);
          else
            corr += qq * std::erf(alpha * r) / r;
        }
      intra += cnt * corr;
    }
    t.self_plus_intra = -alpha / std::sqrt(kPi) * sum_q2 - intra;
    const double two_pi_over_L = 2.0 * kPi / L;
    const double volume = L * L * L;
    const int kmax = t.kmax;
    for (int nx = 0; nx <= kmax; ++nx)
      for (int ny = (nx == 0 ? 0 : -kmax); ny <= kmax; ++ny)
        for (int nz = (nx == 0 && ny == 0 ? 1 : -kmax); nz <= kmax; ++nz) {
          const long n2 = long(nx) * nx + long(ny) * ny + long(nz) * nz;
          if (n2 == 0 || n2 > long(kmax) * kmax) continue;
          KVec k;
          k.nx = nx;
          k.ny = ny;
          k.nz = nz;
          k.kx = two_pi_over_L * nx;
          k.ky = two_pi_over_L * ny;
          k.kz = two_pi_over_L * nz;
          const double k2 = k.kx * k.kx + k.ky * k.ky + k.kz * k.kz;
          k.coeff = 2.0 * (4.0 * kPi / volume) * std::exp(-k2 / (4.0 * alpha * alpha)) / k2;
          t.kv.push_back(k);
        }
    for (int mol = 0; mol < t.n; ++mol) {
      const b2md_species& sp = t.species[t.species_of[mol]];
      for (int k = 0; k < sp.n_sites; ++k)
        if (sp.sites[k].q != 0.0) t.charged.push_back({mol, t.site_begin[mol] + k, sp.sites[k].q});
    }
    t.vderiv = false;  // src/parallel.cpp:68
  }
  return B2MD_OK;
}

void shard_plan(int n, int nk, int world, int rank, int& row_begin, int& row_end, int& k_begin,
                int& k_end, int64_t& candidates) {
  const SearchGeometry g = search_geometry(n);
  // granularity: one super-tile row = g.st tile rows of 32 molecules
  const int ngroups = g.n_super;
  auto pairs_before_row = [n](long i) -> long {  // flat index base (src/potentials.cpp:135)
    if (i > n) i = n;
    return i * n - i * (i + 1) / 2;
  };
  const long total = long(n) * (n - 1) / 2;
  auto boundary = [&](int r) -> int {
    if (r <= 0) return 0;
    if (r >= world) return ngroups;
    const double target = double(total) * r / world;
    int best = 0;
    for (int gidx = 0; gidx <= ngroups; ++gidx) {
      const long p = pairs_before_row(long(gidx) * g.st * 32);
      if (double(p) <= target) best = gidx;
    }
    // choose the closer of best and best+1
    if (best < ngroups) {
      const double lo = double(pairs_before_row(long(best) * g.st * 32));
      const double hi = double(pairs_before_row(long(best + 1) * g.st * 32));
      if (hi - target < target - lo) ++best;
    }
    return best;
  };
  const int g0 = boundary(rank), g1 = boundary(rank + 1);
  row_begin = g0 * g.st;
  row_end = std::min(g1 * g.st, g.n_tiles);
  if (g1 >= ngroups) row_end = g.n_tiles;
  row_begin = std::min(row_begin, g.n_tiles);
  candidates = pairs_before_row(long(row_end) * 32) - pairs_before_row(long(row_begin) * 32);
  k_begin = int(long(nk) * rank / world);
  k_end = int(long(nk) * (rank + 1) / world);
}

}  // namespace b2md
