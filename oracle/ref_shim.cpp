// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  A C entry layer over the
// UNMODIFIED reference library `tmd_core`, compiled from the sources where
// they lie under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libtmdref.so.  Used (1) to pin the C restatement in
// oracle/tmd_oracle.c bit for bit, (2) to generate tests/golden/, and (3) as
// the CPU baseline / `bench.py --impl reference` arm.  It contains no
// reference source, only calls through the reference's public headers:
//   tmd::build_species      include/tmd/model.hpp:42
//   tmd::ForceField         include/tmd/parallel.hpp:56-80
//   tmd::Engine             include/tmd/engine.hpp:52-112
//   tmd::ewald_tune         include/tmd/ewald.hpp:23
//   tmd::minimum_image/norm2 include/tmd/potentials.hpp:176, geom.hpp:33
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "tmd/engine.hpp"
#include "tmd/checkpoint.hpp"
#include "tmd/greenkubo.hpp"
#include "tmd/structure.hpp"
#include "tmd/parallel.hpp"
#include "../include/b200md.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const tmd::ModelError& e) {
    return fail(B2MD_MODEL_ERROR, e.what());
  } catch (const tmd::ConfigError& e) {
    return fail(B2MD_CONFIG_ERROR, e.what());
  } catch (const tmd::IoError& e) {
    return fail(B2MD_IO_ERROR, e.what());
  } catch (const tmd::NumericalError& e) {
    return fail(B2MD_NUMERICAL_ERROR, e.what());
  } catch (const std::exception& e) {
    return fail(B2MD_INVALID_ARGUMENT, e.what());
  }
}

tmd::Site to_site(const b2md_site& s) {
  tmd::Site o;
  o.kind = static_cast<tmd::SiteKind>(s.kind);
  o.body_pos = {s.body_pos[0], s.body_pos[1], s.body_pos[2]};
  o.sigma = s.sigma;
  o.epsilon = s.epsilon;
  o.q = s.q;
  o.mass = s.mass;
  return o;
}

b2md_site from_site(const tmd::Site& s) {
  b2md_site o{};
  o.kind = static_cast<int32_t>(s.kind);
  o.body_pos[0] = s.body_pos.x;
  o.body_pos[1] = s.body_pos.y;
  o.body_pos[2] = s.body_pos.z;
  o.sigma = s.sigma;
  o.epsilon = s.epsilon;
  o.q = s.q;
  o.mass = s.mass;
  return o;
}

// an already-built species is copied verbatim (no second build_species pass)
tmd::MoleculeSpecies to_species(const b2md_species& s) {
  tmd::MoleculeSpecies o;
  o.name = "s";
  for (int k = 0; k < s.n_sites; ++k) o.sites.push_back(to_site(s.sites[k]));
  o.total_mass = s.total_mass;
  o.inertia_principal = {s.inertia_principal[0], s.inertia_principal[1], s.inertia_principal[2]};
  o.net_charge = s.net_charge;
  o.rotational_dof = s.rotational_dof;
  o.max_extent = s.max_extent;
  return o;
}

tmd::SystemComposition to_comp(const b2md_composition& c) {
  tmd::SystemComposition o;
  for (int s = 0; s < c.n_species; ++s) {
    o.species.push_back(to_species(c.species[s]));
    o.counts.push_back(c.counts[s]);
  }
  o.box_length = c.box_length;
  o.temperature = c.temperature;
  return o;
}

tmd::ForceFieldOptions to_opts(const b2md_ff_options& p) {
  tmd::ForceFieldOptions o;
  o.cutoff = p.cutoff;
  o.method = static_cast<tmd::ElectrostaticsMethod>(p.method);
  o.eps_rf = p.eps_rf;
  if (p.has_ewald) o.ewald = tmd::EwaldParams{p.ewald_alpha, p.ewald_kmax};
  o.workers = p.workers;
  o.volume_derivatives = p.volume_derivatives != 0;
  return o;
}

void put_energy(const tmd::EnergyBreakdown& e, b2md_energy* out) {
  if (!out) return;
  out->lj = e.lj;
  out->elec_real = e.elec_real;
  out->elec_recip = e.elec_recip;
  out->elec_self = e.elec_self;
  out->rf = e.rf;
  out->lrc = e.lrc;
  out->du_dv_explicit = e.du_dv_explicit;
  out->du_dv_lrc = e.du_dv_lrc;
  out->d2u_dv2_explicit = e.d2u_dv2_explicit;
  out->d2u_dv2_lrc = e.d2u_dv2_lrc;
}

void put_vec3(const std::vector<tmd::Vec3>& v, double* out) {
  if (!out) return;
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[3 * i] = v[i].x;
    out[3 * i + 1] = v[i].y;
    out[3 * i + 2] = v[i].z;
  }
}

void get_state(tmd::SystemState& st, int n, const double* pos, const double* orient,
               const double* vel, const double* ang_vel) {
  st.resize(n);
  for (int i = 0; i < n; ++i) {
    if (pos) st.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    if (orient) st.orient[i] = {orient[4 * i], orient[4 * i + 1], orient[4 * i + 2], orient[4 * i + 3]};
    if (vel) st.vel[i] = {vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]};
    if (ang_vel) st.ang_vel[i] = {ang_vel[3 * i], ang_vel[3 * i + 1], ang_vel[3 * i + 2]};
  }
}

struct RefFF {
  tmd::SystemComposition comp;  // ForceField keeps a reference: must outlive it
  std::unique_ptr<tmd::ForceField> ff;
};

struct RefEngine {
  std::unique_ptr<tmd::Engine> eng;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_build_species(const b2md_site* sites, int n, b2md_species* out) {
  return guarded([&]() -> int {
    std::vector<tmd::Site> v;
    for (int k = 0; k < n; ++k) v.push_back(to_site(sites[k]));
    const tmd::MoleculeSpecies sp = tmd::build_species("s", v);
    if (sp.site_count() > B2MD_MAX_SITES) return fail(B2MD_MODEL_ERROR, "too many sites");
    std::memset(out, 0, sizeof *out);
    out->n_sites = sp.site_count();
    for (int k = 0; k < sp.site_count(); ++k) out->sites[k] = from_site(sp.sites[k]);
    out->total_mass = sp.total_mass;
    out->inertia_principal[0] = sp.inertia_principal.x;
    out->inertia_principal[1] = sp.inertia_principal.y;
    out->inertia_principal[2] = sp.inertia_principal.z;
    out->net_charge = sp.net_charge;
    out->rotational_dof = sp.rotational_dof;
    out->max_extent = sp.max_extent;
    return B2MD_OK;
  });
}

int ref_ewald_tune(double delta, double cutoff, double box, double* alpha, int* kmax) {
  return guarded([&]() -> int {
    const tmd::EwaldParams p = tmd::ewald_tune(delta, cutoff, box);
    *alpha = p.alpha;
    *kmax = p.kmax;
    return B2MD_OK;
  });
}

int ref_ff_create(const b2md_composition* comp, const b2md_ff_options* opts, void** out) {
  *out = nullptr;
  return guarded([&]() -> int {
    auto h = std::make_unique<RefFF>();
    h->comp = to_comp(*comp);
    h->ff = std::make_unique<tmd::ForceField>(h->comp, to_opts(*opts));
    *out = h.release();
    return B2MD_OK;
  });
}

void ref_ff_destroy(void* h) { delete static_cast<RefFF*>(h); }

const char* ref_ff_warning(void* h) {
  auto* f = static_cast<RefFF*>(h);
  return f->ff->ewald() ? f->ff->ewald()->warning().c_str() : "";
}

int ref_evaluate(void* h, const double* pos, const double* orient, double* force, double* torque,
                 b2md_energy* energy, double* virial) {
  return guarded([&]() -> int {
    auto* f = static_cast<RefFF*>(h);
    tmd::SystemState st;
    st.box_length = f->comp.box_length;
    get_state(st, f->comp.molecule_count(), pos, orient, nullptr, nullptr);
    f->ff->evaluate(st);
    put_vec3(st.force, force);
    put_vec3(st.torque, torque);
    put_energy(st.energy, energy);
    if (virial) *virial = st.virial;
    return B2MD_OK;
  });
}

// COM partner search using the reference's own inline minimum_image/norm2
// with the tests of src/potentials.cpp:156-158 and 209-213.
int64_t ref_pair_list(void* h, const double* pos, int32_t* pairs, int64_t capacity) {
  auto* f = static_cast<RefFF*>(h);
  const auto& comp = f->comp;
  const int n = comp.molecule_count();
  const auto& table = f->ff->table();
  const bool single = table.single_lj_only() && table.method() != tmd::ElectrostaticsMethod::ewald;
  int64_t cnt = 0;
  for (int i = 0; i < n; ++i) {
    const tmd::Vec3 ci{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    for (int j = i + 1; j < n; ++j) {
      const tmd::Vec3 cj{pos[3 * j], pos[3 * j + 1], pos[3 * j + 2]};
      const tmd::Vec3 R = tmd::minimum_image(ci - cj, comp.box_length);
      const double R2 = tmd::norm2(R);
      bool pass;
      if (single) {
        pass = R2 < table.cutoff2();
      } else {
        const double rmax = table.cutoff() + comp.species[comp.species_of_molecule(i)].max_extent +
                            comp.species[comp.species_of_molecule(j)].max_extent;
        pass = R2 < rmax * rmax;
      }
      if (pass) {
        if (pairs && cnt < capacity) {
          pairs[2 * cnt] = i;
          pairs[2 * cnt + 1] = j;
        }
        ++cnt;
      }
    }
  }
  return cnt;
}

int ref_engine_create(const b2md_composition* comp, const b2md_ff_options* opts, double dt,
                      uint64_t seed, void** out) {
  *out = nullptr;
  return guarded([&]() -> int {
    tmd::SimulationPlan plan;
    plan.dt = dt;
    plan.thermostat_interval_equil = 0;
    plan.thermostat_interval_prod = 0;
    auto h = std::make_unique<RefEngine>();
    h->eng = std::make_unique<tmd::Engine>(to_comp(*comp), to_opts(*opts), plan, seed);
    *out = h.release();
    return B2MD_OK;
  });
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_set_state(void* h, const double* pos, const double* orient, const double* vel,
                         const double* ang_vel) {
  return guarded([&]() -> int {
    auto* e = static_cast<RefEngine*>(h);
    tmd::SystemState st = e->eng->state();
    get_state(st, st.molecule_count(), pos, orient, vel, ang_vel);
    e->eng->set_state(st);
    return B2MD_OK;
  });
}

int ref_engine_step(void* h, int64_t nsteps) {
  return guarded([&]() -> int {
    auto* e = static_cast<RefEngine*>(h);
    for (int64_t s = 0; s < nsteps; ++s) e->eng->step();
    return B2MD_OK;
  });
}

int ref_engine_get_state(void* h, double* pos, double* orient, double* vel, double* ang_vel,
                         double* force, double* torque, b2md_energy* energy, double* virial) {
  auto* e = static_cast<RefEngine*>(h);
  const tmd::SystemState& st = e->eng->state();
  put_vec3(st.pos, pos);
  if (orient)
    for (int i = 0; i < st.molecule_count(); ++i) {
      orient[4 * i] = st.orient[i].w;
      orient[4 * i + 1] = st.orient[i].x;
      orient[4 * i + 2] = st.orient[i].y;
      orient[4 * i + 3] = st.orient[i].z;
    }
  put_vec3(st.vel, vel);
  put_vec3(st.ang_vel, ang_vel);
  put_vec3(st.force, force);
  put_vec3(st.torque, torque);
  put_energy(st.energy, energy);
  if (virial) *virial = st.virial;
  return B2MD_OK;
}

}  // extern "C"

// tmd::Rng (include/tmd/rng.hpp:14-76): raw draws for the RNG golden vectors.
extern "C" int ref_rng_draws(uint64_t seed, int n, uint64_t* u64, double* uniform, double* gaussian) {
  tmd::Rng a(seed), b(seed), c(seed);
  for (int k = 0; k < n; ++k) {
    u64[k] = a.next_u64();
    uniform[k] = b.uniform();
    gaussian[k] = c.gaussian();
  }
  return 0;
}

// tmd::heat_flux (include/tmd/greenkubo.hpp:93, src/greenkubo.cpp:182-266)
extern "C" int ref_heat_flux(void* h, const double* pos, const double* orient, const double* vel,
                             const double* ang_vel, const double* enthalpy, int n_enthalpy,
                             double* jq) {
  return guarded([&]() -> int {
    auto* f = static_cast<RefFF*>(h);
    tmd::SystemState st;
    st.box_length = f->comp.box_length;
    get_state(st, f->comp.molecule_count(), pos, orient, vel, ang_vel);
    std::vector<double> hh(enthalpy, enthalpy + n_enthalpy);
    const tmd::Vec3 j = tmd::heat_flux(f->comp, st, f->ff->table(), hh);
    jq[0] = j.x;
    jq[1] = j.y;
    jq[2] = j.z;
    return B2MD_OK;
  });
}

// ---------------------------------------------- tmd::RdfHistogram (structure.cpp)
extern "C" int ref_rdf_create(void* ffh, double bin_width, double r_max, void** out) {
  return guarded([&]() -> int {
    auto* f = static_cast<RefFF*>(ffh);
    *out = new tmd::RdfHistogram(f->comp, bin_width, r_max);
    return B2MD_OK;
  });
}

extern "C" void ref_rdf_destroy(void* h) { delete static_cast<tmd::RdfHistogram*>(h); }

extern "C" int ref_rdf_accumulate(void* h, void* ffh, const double* pos, const double* orient) {
  return guarded([&]() -> int {
    auto* f = static_cast<RefFF*>(ffh);
    tmd::SystemState st;
    st.box_length = f->comp.box_length;
    get_state(st, f->comp.molecule_count(), pos, orient, nullptr, nullptr);
    static_cast<tmd::RdfHistogram*>(h)->accumulate(st);
    return B2MD_OK;
  });
}

// RdfHistogram::serialize bytes (structure.cpp:130-140); returns the length
extern "C" int64_t ref_rdf_serialize(void* h, char* buf, int64_t cap) {
  tmd::ByteWriter w;
  static_cast<tmd::RdfHistogram*>(h)->serialize(w);
  const std::string& d = w.data();
  if (buf && cap >= static_cast<int64_t>(d.size())) std::memcpy(buf, d.data(), d.size());
  return static_cast<int64_t>(d.size());
}

// RdfHistogram::finalize (structure.cpp:78-128), flattened per table:
// species_a, species_b, partner_density, bin_width, snapshots, bins, then
// bins x (r_mid, g, n_cum).  Returns the number of doubles.
extern "C" int64_t ref_rdf_finalize(void* h, double* out, int64_t cap) {
  std::vector<double> v;
  try {
    for (const auto& t : static_cast<tmd::RdfHistogram*>(h)->finalize()) {
      v.insert(v.end(), {double(t.species_a), double(t.species_b), t.partner_density, t.bin_width,
                         double(t.snapshots), double(t.g.size())});
      for (std::size_t b = 0; b < t.g.size(); ++b) v.insert(v.end(), {t.r_mid[b], t.g[b], t.n_cum[b]});
    }
  } catch (const std::exception& e) {
    fail(B2MD_CONFIG_ERROR, e.what());
    return -1;
  }
  if (out && cap >= static_cast<int64_t>(v.size())) std::memcpy(out, v.data(), v.size() * 8);
  return static_cast<int64_t>(v.size());
}

extern "C" double ref_first_minimum(const double* r_mid, const double* g, int n) {
  return tmd::first_minimum(std::vector<double>(r_mid, r_mid + n), std::vector<double>(g, g + n));
}

extern "C" double ref_solvation_number(double bin_width, const double* g, int n,
                                       double partner_density, double r_min) {
  tmd::RdfTable t;
  t.bin_width = bin_width;
  t.g.assign(g, g + n);
  return tmd::solvation_number(t, partner_density, r_min);
}

// ------------------------------------------- Engine checkpoints (engine.cpp:420-541)
extern "C" int64_t ref_engine_checkpoint(void* h, char* buf, int64_t cap) {
  const std::string d = static_cast<RefEngine*>(h)->eng->checkpoint_bytes();
  if (buf && cap >= static_cast<int64_t>(d.size())) std::memcpy(buf, d.data(), d.size());
  return static_cast<int64_t>(d.size());
}

// What a restart does with a checkpoint file: the container header (magic,
// version, embedded config text — written by checkpoint_bytes, engine.cpp:
// 421-423), then Engine::restore_dynamic for the rest.
extern "C" int ref_engine_restore(void* h, const char* buf, int64_t len) {
  return guarded([&]() -> int {
    tmd::ByteReader r(std::string(buf, static_cast<std::size_t>(len)));
    char magic[8];
    r.bytes(magic, 8);
    if (std::string(magic, 8) != "TMDCKPT1") throw tmd::IoError("checkpoint: bad magic");
    if (r.u32() != 1) throw tmd::IoError("checkpoint: unsupported version");
    (void)r.str();
    static_cast<RefEngine*>(h)->eng->restore_dynamic(r);
    return B2MD_OK;
  });
}

// Engine::run with samplers (engine.cpp:197-300), then checkpoint_bytes: a
// checkpoint with every sampler section.  flags: 1 massieu, 2 rdf, 4 self
// diffusion, 8 electric conductivity, 16 thermal conductivity, 32 residence.
extern "C" int64_t ref_run_sampled_checkpoint(const b2md_composition* comp,
                                              const b2md_ff_options* opts, double dt,
                                              uint64_t seed, int64_t n_equil, int64_t n_prod,
                                              int n_ext, int corr_length, int n_blocks, int flags,
                                              const double* enthalpy, int n_enthalpy,
                                              int res_solute, int res_solvent, double res_radius,
                                              const char* config_text, char* buf, int64_t cap) {
  std::string d;
  const int rc = guarded([&]() -> int {
    tmd::SimulationPlan plan;
    plan.dt = dt;
    plan.n_equilibration = n_equil;
    plan.n_production = n_prod;
    plan.n_ext = n_ext;
    plan.corr_length = corr_length;
    plan.n_blocks = n_blocks;
    plan.sample_massieu = flags & 1;
    plan.sample_rdf = flags & 2;
    plan.sample_self_diffusion = flags & 4;
    plan.sample_electric_conductivity = flags & 8;
    plan.sample_thermal_conductivity = flags & 16;
    plan.sample_residence = flags & 32;
    plan.enthalpy.assign(enthalpy, enthalpy + n_enthalpy);
    plan.residence_solute = res_solute;
    plan.residence_solvent = res_solvent;
    plan.residence_radius = res_radius;
    plan.config_text = config_text ? config_text : "";
    tmd::Engine eng(to_comp(*comp), to_opts(*opts), plan, seed);
    (void)eng.run();
    d = eng.checkpoint_bytes();
    return B2MD_OK;
  });
  if (rc) return -1;
  if (buf && cap >= static_cast<int64_t>(d.size())) std::memcpy(buf, d.data(), d.size());
  return static_cast<int64_t>(d.size());
}

// ------------------------------------------------ thermostat (engine.cpp:145-160)
extern "C" int ref_engine_apply_thermostat(void* h) {
  return guarded([&]() -> int {
    static_cast<RefEngine*>(h)->eng->apply_thermostat();
    return B2MD_OK;
  });
}

extern "C" int ref_kinetic_energy(void* ffh, const double* vel, const double* ang_vel, double* out) {
  return guarded([&]() -> int {
    auto* f = static_cast<RefFF*>(ffh);
    tmd::SystemState st;
    get_state(st, f->comp.molecule_count(), nullptr, nullptr, vel, ang_vel);
    out[0] = tmd::kinetic_energy_trans(f->comp, st);
    out[1] = tmd::kinetic_energy_rot(f->comp, st);
    return B2MD_OK;
  });
}

// ---------------------- scalar accumulators (massieu.cpp:9-70, results.hpp:21-51)
#include "tmd/massieu.hpp"
#include "tmd/results.hpp"

extern "C" int64_t ref_derivative_accumulator(double temperature, double volume, int64_t n_mol,
                                              int n_blocks, int64_t expected,
                                              const double* samples, int k, char* buf,
                                              int64_t cap) {
  std::string d;
  const int rc = guarded([&]() -> int {
    tmd::DerivativeAccumulator a(temperature, volume, n_mol, n_blocks, expected);
    for (int i = 0; i < k; ++i) a.add(samples[3 * i], samples[3 * i + 1], samples[3 * i + 2]);
    tmd::ByteWriter w;
    a.serialize(w);
    d = w.data();
    return B2MD_OK;
  });
  if (rc) return -1;
  if (buf && cap >= static_cast<int64_t>(d.size())) std::memcpy(buf, d.data(), d.size());
  return static_cast<int64_t>(d.size());
}

extern "C" int64_t ref_block_stat(int n_blocks, int64_t expected, const double* x, int k, char* buf,
                                  int64_t cap) {
  tmd::BlockStat b(n_blocks, expected);
  for (int i = 0; i < k; ++i) b.add(x[i]);
  tmd::ByteWriter w;
  b.serialize(w);
  const std::string& d = w.data();
  if (buf && cap >= static_cast<int64_t>(d.size())) std::memcpy(buf, d.data(), d.size());
  return static_cast<int64_t>(d.size());
}
