// tmd_gpu.hpp — the binding a tmd maintainer adds to the reference to use the
// B200 path: tmd::GpuForceField / tmd::GpuEngine over the C ABI of
// include/b200md.h, with the reference's own types (include/tmd/*.hpp) and
// exceptions (include/tmd/error.hpp).  Header-only; link libb200md.so.
//
//   tmd::ForceField::evaluate(SystemState&)  (src/parallel.cpp:79-122)
//     -> tmd::GpuForceField::evaluate(SystemState&)     same contract
//   tmd::Engine::set_state / step / state      (src/engine.cpp:91-143)
//     -> tmd::GpuEngine::set_state / step / state        device-resident
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200md.h"
#include "tmd/engine.hpp"
#include "tmd/checkpoint.hpp"
#include "tmd/massieu.hpp"
#include "tmd/parallel.hpp"
#include "tmd/structure.hpp"

namespace tmd {

namespace b2md_detail {

inline void check(int rc) {
  if (rc == B2MD_OK) return;
  const std::string msg = b2md_last_error();
  switch (rc) {
    case B2MD_MODEL_ERROR: throw ModelError(msg);
    case B2MD_CONFIG_ERROR: throw ConfigError(msg);
    case B2MD_IO_ERROR: throw IoError(msg);
    case B2MD_NUMERICAL_ERROR: throw NumericalError(msg);
    default: throw Error(msg);
  }
}

// an already-built tmd::MoleculeSpecies -> b2md_species (no second build pass)
inline b2md_species to_c(const MoleculeSpecies& sp) {
  if (sp.site_count() > B2MD_MAX_SITES) throw ModelError("b200md: too many sites in species");
  b2md_species o;
  std::memset(&o, 0, sizeof o);
  o.n_sites = sp.site_count();
  o.rotational_dof = sp.rotational_dof;
  for (int k = 0; k < sp.site_count(); ++k) {
    const Site& s = sp.sites[k];
    o.sites[k].kind = static_cast<int32_t>(s.kind);
    o.sites[k].body_pos[0] = s.body_pos.x;
    o.sites[k].body_pos[1] = s.body_pos.y;
    o.sites[k].body_pos[2] = s.body_pos.z;
    o.sites[k].sigma = s.sigma;
    o.sites[k].epsilon = s.epsilon;
    o.sites[k].q = s.q;
    o.sites[k].mass = s.mass;
  }
  o.total_mass = sp.total_mass;
  o.inertia_principal[0] = sp.inertia_principal.x;
  o.inertia_principal[1] = sp.inertia_principal.y;
  o.inertia_principal[2] = sp.inertia_principal.z;
  o.net_charge = sp.net_charge;
  o.max_extent = sp.max_extent;
  return o;
}

inline b2md_ff_options to_c(const ForceFieldOptions& f) {
  b2md_ff_options o;
  std::memset(&o, 0, sizeof o);
  o.cutoff = f.cutoff;
  o.method = static_cast<int32_t>(f.method);
  o.eps_rf = f.eps_rf;
  o.has_ewald = f.ewald ? 1 : 0;
  if (f.ewald) {
    o.ewald_alpha = f.ewald->alpha;
    o.ewald_kmax = f.ewald->kmax;
  }
  o.workers = f.workers;
  o.volume_derivatives = f.volume_derivatives ? 1 : 0;
  return o;
}

inline void from_c(const b2md_energy& e, EnergyBreakdown& o) {
  o.lj = e.lj;
  o.elec_real = e.elec_real;
  o.elec_recip = e.elec_recip;
  o.elec_self = e.elec_self;
  o.rf = e.rf;
  o.lrc = e.lrc;
  o.du_dv_explicit = e.du_dv_explicit;
  o.du_dv_lrc = e.du_dv_lrc;
  o.d2u_dv2_explicit = e.d2u_dv2_explicit;
  o.d2u_dv2_lrc = e.d2u_dv2_lrc;
}

// Vec3 / Quat are plain structs of doubles (geom.hpp:9-38): AoS as the ABI expects
static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 layout");
static_assert(sizeof(Quat) == 4 * sizeof(double), "Quat layout");

class Context {
 public:
  Context(const SystemComposition& comp, const ForceFieldOptions& opts, double dt, int device) {
    std::vector<b2md_species> sp;
    for (const auto& s : comp.species) sp.push_back(to_c(s));
    std::vector<int32_t> counts(comp.counts.begin(), comp.counts.end());
    b2md_composition c;
    std::memset(&c, 0, sizeof c);
    c.n_species = comp.species_count();
    c.species = sp.data();
    c.counts = counts.data();
    c.box_length = comp.box_length;
    c.temperature = comp.temperature;
    const b2md_ff_options o = to_c(opts);
    check(b2md_create(device, &c, &o, dt, 1, &ctx_));
  }
  ~Context() { b2md_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  b2md_ctx* get() const { return ctx_; }

 private:
  b2md_ctx* ctx_ = nullptr;
};

}  // namespace b2md_detail

// Drop-in for tmd::ForceField (parallel.hpp:56-80).
class GpuForceField {
 public:
  GpuForceField(const SystemComposition& comp, const ForceFieldOptions& opts, int device = 0)
      : comp_(comp), ctx_(comp, opts, 0.0, device) {}

  void evaluate(SystemState& state) {
    const int n = state.molecule_count();
    state.force.resize(n);
    state.torque.resize(n);
    b2md_energy e;
    b2md_eval_stats st;
    b2md_detail::check(b2md_evaluate(ctx_.get(), &state.pos[0].x, &state.orient[0].w,
                                     &state.force[0].x, &state.torque[0].x, &e, &st));
    b2md_detail::from_c(e, state.energy);
    state.virial = st.virial;
  }

  const char* warning() const { return b2md_warning(ctx_.get()); }
  b2md_ctx* context() const { return ctx_.get(); }

  // tmd::heat_flux(comp, state, table, h) (greenkubo.hpp:93, greenkubo.cpp:182-266)
  // with this force field's pair table; state taken as given.
  Vec3 heat_flux(const SystemState& state, const std::vector<double>& h_per_species) {
    Vec3 jq;
    b2md_detail::check(b2md_heat_flux_state(ctx_.get(), &state.pos[0].x, &state.orient[0].w,
                                            &state.vel[0].x, &state.ang_vel[0].x,
                                            h_per_species.data(),
                                            static_cast<int>(h_per_species.size()), &jq.x));
    return jq;
  }

 private:
  const SystemComposition& comp_;
  b2md_detail::Context ctx_;
};

// Free-function form next to tmd::heat_flux.
inline Vec3 heat_flux(GpuForceField& ff, const SystemState& state,
                      const std::vector<double>& h_per_species) {
  return ff.heat_flux(state, h_per_species);
}

// The step path of tmd::Engine (engine.hpp:52-112), device resident.
class GpuEngine {
 public:
  GpuEngine(const SystemComposition& comp, const ForceFieldOptions& opts, double dt, int device = 0)
      : comp_(comp), ctx_(comp, opts, dt, device) {
    if (dt <= 0.0) throw ConfigError("engine: time step must be positive");
  }

  void set_state(const SystemState& s) {  // engine.cpp:91-98
    if (s.molecule_count() != comp_.molecule_count())
      throw ConfigError("engine: state does not match composition");
    b2md_detail::check(b2md_set_state(ctx_.get(), &s.pos[0].x, &s.orient[0].w, &s.vel[0].x,
                                      &s.ang_vel[0].x));
  }

  void step(long n = 1) { b2md_detail::check(b2md_step(ctx_.get(), n)); }  // engine.cpp:102-143

  SystemState state() const {
    SystemState s;
    s.resize(comp_.molecule_count());
    s.box_length = comp_.box_length;
    b2md_energy e;
    b2md_eval_stats st;
    b2md_detail::check(b2md_get_state(ctx_.get(), &s.pos[0].x, &s.orient[0].w, &s.vel[0].x,
                                      &s.ang_vel[0].x, &s.force[0].x, &s.torque[0].x, &e, &st));
    b2md_detail::from_c(e, s.energy);
    s.virial = st.virial;
    return s;
  }

  b2md_ctx* context() const { return ctx_.get(); }

  // EnergyBreakdown of the resident state (no array download)
  EnergyBreakdown energy() const {
    b2md_energy e;
    b2md_detail::check(b2md_get_state(ctx_.get(), nullptr, nullptr, nullptr, nullptr, nullptr,
                                      nullptr, &e, nullptr));
    EnergyBreakdown out;
    b2md_detail::from_c(e, out);
    return out;
  }

  // Engine::sample_extended_step's Massieu sample (engine.cpp:228-229): the
  // device-side U, dU/dV and d2U/dV2 fed to the reference's OWN
  // DerivativeAccumulator (massieu.cpp:53-70) -- the estimator stays host code
  void sample_massieu(DerivativeAccumulator& acc) const {
    const EnergyBreakdown e = energy();
    acc.add(e.total(), e.du_dv(), e.d2u_dv2());
  }

  // checkpoint state block (engine.cpp:432-441) of the device state, for
  // Engine::checkpoint_bytes; restore = restore_dynamic's state part + forces
  std::string checkpoint_state_block() const {
    std::string buf(b2md_state_block_size(ctx_.get()), '\0');
    b2md_detail::check(b2md_save_state_block(ctx_.get(), 0, reinterpret_cast<std::uint8_t*>(&buf[0]),
                                             buf.size()));
    return buf;
  }
  void restore_state_block(const std::string& block) {
    b2md_detail::check(b2md_restore_state_block(
        ctx_.get(), 0, reinterpret_cast<const std::uint8_t*>(block.data()), block.size()));
  }

  // J_q of the resident state, as Engine::run samples it every n_ext steps
  // (engine.cpp:235-238)
  Vec3 heat_flux(const std::vector<double>& h_per_species) const {
    Vec3 jq;
    b2md_detail::check(b2md_heat_flux(ctx_.get(), h_per_species.data(),
                                      static_cast<int>(h_per_species.size()), &jq.x));
    return jq;
  }

 private:
  SystemComposition comp_;
  b2md_detail::Context ctx_;
};

// RdfHistogram (structure.hpp:29-67) accumulated on the GPU.  The counts
// are the reference's (bit-exact); finalize() hands them to the reference's
// own class through its deserialize (structure.cpp:142-153), so tables,
// first_minimum and solvation_number are the reference's arithmetic.
class GpuRdfHistogram {
 public:
  template <typename Owner>  // GpuForceField or GpuEngine
  GpuRdfHistogram(const SystemComposition& comp, Owner& owner, double bin_width, double r_max)
      : comp_(comp), bin_width_(bin_width), r_max_(r_max) {
    b2md_detail::check(b2md_rdf_create(owner.context(), bin_width, r_max, &h_));
    b2md_detail::check(b2md_rdf_shape(h_, nullptr, &bins_, &pairs_));
  }
  ~GpuRdfHistogram() { b2md_rdf_destroy(h_); }
  GpuRdfHistogram(const GpuRdfHistogram&) = delete;
  GpuRdfHistogram& operator=(const GpuRdfHistogram&) = delete;

  void accumulate(const SystemState& s) {  // structure.cpp:38-76
    b2md_detail::check(b2md_rdf_accumulate_state(h_, &s.pos[0].x, &s.orient[0].w));
  }
  void accumulate() { b2md_detail::check(b2md_rdf_accumulate(h_)); }  // resident state

  // the reference histogram holding the GPU counts (RdfHistogram::serialize layout)
  RdfHistogram to_reference() const {
    std::vector<std::uint64_t> counts(std::size_t(pairs_) * bins_);
    std::int64_t snaps = 0;
    b2md_detail::check(b2md_rdf_counts(h_, 0, counts.data(), &snaps));
    ByteWriter w;
    w.f64(bin_width_);
    w.f64(r_max_);
    w.u32(static_cast<std::uint32_t>(bins_));
    w.i64(snaps);
    w.u64(static_cast<std::uint64_t>(pairs_));
    for (int p = 0; p < pairs_; ++p) {
      w.u64(static_cast<std::uint64_t>(bins_));
      for (int b = 0; b < bins_; ++b) w.u64(counts[std::size_t(p) * bins_ + b]);
    }
    RdfHistogram h(comp_, bin_width_, r_max_);
    ByteReader r(w.data());
    h.deserialize(r);
    return h;
  }
  std::vector<RdfTable> finalize() const { return to_reference().finalize(); }

 private:
  const SystemComposition& comp_;
  double bin_width_, r_max_;
  int bins_ = 0, pairs_ = 0;
  b2md_rdf* h_ = nullptr;
};

}  // namespace tmd
