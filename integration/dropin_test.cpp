// dropin_test.cpp — the reference's own types, generators and CPU ForceField /
// Engine next to the GPU drop-ins of tmd_gpu.hpp.  Built where the reference
// headers exist (integration/Makefile); the binary runs on the GPU box.
// Exit status 0 iff forces/torques agree to 1e-10 x max|F|, energies and
// 50-step trajectories to 1e-9.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "tmd/greenkubo.hpp"
#include "tmd_gpu.hpp"

using namespace tmd;

namespace {

Site lj(double x, double y, double z, double s, double e, double m) {
  Site t;
  t.kind = SiteKind::lj;
  t.body_pos = {x, y, z};
  t.sigma = s;
  t.epsilon = e;
  t.mass = m;
  return t;
}

Site charge(double x, double y, double z, double q, double m) {
  Site t;
  t.kind = SiteKind::charge;
  t.body_pos = {x, y, z};
  t.q = q;
  t.mass = m;
  return t;
}

double max_abs(const std::vector<Vec3>& a) {
  double m = 0.0;
  for (const auto& v : a) m = std::max({m, std::abs(v.x), std::abs(v.y), std::abs(v.z)});
  return m;
}

double max_diff(const std::vector<Vec3>& a, const std::vector<Vec3>& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i)
    m = std::max({m, std::abs(a[i].x - b[i].x), std::abs(a[i].y - b[i].y), std::abs(a[i].z - b[i].z)});
  return m;
}

int failures = 0;

void expect(bool ok, const char* what, double v) {
  std::printf("  %-44s %.3e %s\n", what, v, ok ? "ok" : "FAIL");
  if (!ok) ++failures;
}

void compare_eval(const char* name, const SystemComposition& comp, const ForceFieldOptions& opts,
                  const SystemState& st) {
  std::printf("%s (N=%d)\n", name, comp.molecule_count());
  ForceField cpu(comp, opts);
  GpuForceField gpu(comp, opts);
  SystemState a = st, b = st;
  cpu.evaluate(a);
  gpu.evaluate(b);
  const double fs = std::max(1.0, max_abs(a.force)), ts = std::max(1.0, max_abs(a.torque));
  expect(max_diff(a.force, b.force) <= 1e-10 * fs, "max |dF| / max |F|", max_diff(a.force, b.force) / fs);
  expect(max_diff(a.torque, b.torque) <= 1e-10 * ts, "max |dtau| / max |tau|", max_diff(a.torque, b.torque) / ts);
  const double de = std::abs(a.energy.total() - b.energy.total()) / std::abs(a.energy.total());
  expect(de <= 1e-9, "|dU| / |U|", de);
  const double dv = std::abs(a.virial - b.virial) / std::max(1.0, std::abs(a.virial));
  expect(dv <= 1e-9, "|dW| / |W|", dv);
  // heat flux (greenkubo.cpp:182-266) of the same state, one enthalpy per species
  std::vector<double> h;
  for (int k = 0; k < comp.species_count(); ++k) h.push_back(0.3 - 0.7 * k);
  const Vec3 jr = heat_flux(comp, st, cpu.table(), h);
  const Vec3 jg = heat_flux(gpu, st, h);
  const double js = std::max({1.0, std::abs(jr.x), std::abs(jr.y), std::abs(jr.z)});
  const double dj = std::max({std::abs(jr.x - jg.x), std::abs(jr.y - jg.y), std::abs(jr.z - jg.z)}) / js;
  expect(dj <= 1e-10, "heat flux |dJq| / max |Jq|", dj);
}

}  // namespace

int main() {
  // 2CLJ (BASELINE config 1 shape, smaller N), reference init_lattice
  {
    SystemComposition comp;
    comp.species = {build_species("2clj", {lj(0.25, 0, 0, 1, 1, 0.5), lj(-0.25, 0, 0, 1, 1, 0.5)})};
    comp.counts = {500};
    comp.box_length = std::cbrt(500 / 0.3);
    comp.temperature = 2.0;
    ForceFieldOptions opts;
    opts.cutoff = 0.45 * comp.box_length;
    const SystemState st = init_lattice(comp, 7);
    compare_eval("2CLJ", comp, opts, st);

    SimulationPlan plan;
    plan.dt = 0.002;
    plan.thermostat_interval_equil = 0;
    plan.thermostat_interval_prod = 0;
    Engine ref(comp, opts, plan, 7);
    GpuEngine gpu(comp, opts, 0.002);
    ref.set_state(st);
    gpu.set_state(st);
    // Massieu sampling every 5 steps into the reference's own accumulator:
    // the CPU engine's energies vs the GPU engine's device-side scalars
    DerivativeAccumulator mref(comp.temperature, comp.volume(), comp.molecule_count(), 2, 10);
    DerivativeAccumulator mgpu(comp.temperature, comp.volume(), comp.molecule_count(), 2, 10);
    for (int k = 0; k < 10; ++k) {
      for (int q = 0; q < 5; ++q) ref.step();
      gpu.step(5);
      const EnergyBreakdown& e = ref.state().energy;
      mref.add(e.total(), e.du_dv(), e.d2u_dv2());
      gpu.sample_massieu(mgpu);
    }
    const SystemState a = ref.state(), b = gpu.state();
    double dp = 0.0;
    for (int i = 0; i < comp.molecule_count(); ++i)
      for (int k = 0; k < 3; ++k) {
        double d = a.pos[i][k] - b.pos[i][k];
        d -= comp.box_length * std::nearbyint(d / comp.box_length);
        dp = std::max(dp, std::abs(d));
      }
    std::printf("2CLJ engine, 50 steps\n");
    expect(dp / comp.box_length <= 1e-9, "max |dpos| / L", dp / comp.box_length);
    const double de = std::abs(a.energy.total() - b.energy.total()) / std::abs(a.energy.total());
    expect(de <= 1e-9, "|dU| / |U|", de);
    // J_q of the stepped states: the reference on its state, the GPU on its resident one
    ForceField table_owner(comp, opts);
    const Vec3 jr = heat_flux(comp, a, table_owner.table(), {0.4});
    const Vec3 jg = gpu.heat_flux({0.4});
    const double js = std::max({1.0, std::abs(jr.x), std::abs(jr.y), std::abs(jr.z)});
    const double dj = std::max({std::abs(jr.x - jg.x), std::abs(jr.y - jg.y), std::abs(jr.z - jg.z)}) / js;
    expect(dj <= 1e-9, "heat flux after 50 steps |dJq| / max |Jq|", dj);
    // the reference's Massieu estimators from the two sample streams
    const DerivativeReport ra = mref.finalize(), rg = mgpu.finalize();
    double dm = 0.0;
    for (std::size_t k = 0; k < ra.entries.size(); ++k)
      dm = std::max(dm, std::abs(ra.entries[k].value - rg.entries[k].value) /
                            std::max(1.0, std::abs(ra.entries[k].value)));
    expect(mref.samples() == mgpu.samples() && dm <= 1e-8, "Massieu derivatives (GPU scalars)", dm);

    // RDF: GPU counts finalized by the reference's own RdfHistogram, on a
    // host state and on the GPU engine's resident state (b = its download)
    RdfHistogram cpu2(comp, 0.05, 0.5 * comp.box_length);
    GpuRdfHistogram gpu2(comp, gpu, 0.05, 0.5 * comp.box_length);
    cpu2.accumulate(a);
    gpu2.accumulate(a);
    cpu2.accumulate(b);
    gpu2.accumulate();
    const auto tc = cpu2.finalize(), tg = gpu2.finalize();
    double dg = tc.size() == tg.size() ? 0.0 : 1.0;
    for (std::size_t t = 0; t < tc.size() && t < tg.size(); ++t)
      for (std::size_t k = 0; k < tc[t].g.size(); ++k)
        dg = std::max({dg, std::abs(tc[t].g[k] - tg[t].g[k]), std::abs(tc[t].n_cum[k] - tg[t].n_cum[k])});
    expect(dg == 0.0, "RDF tables (GPU counts) vs reference, max |d|", dg);

    // checkpoint state block: a fresh pair of engines on the same state
    Engine ref2(comp, opts, plan, 7);
    GpuEngine gpu3(comp, opts, 0.002);
    ref2.set_state(st);
    gpu3.set_state(st);
    const std::string full = ref2.checkpoint_bytes();
    const std::string block = gpu3.checkpoint_state_block();
    const std::size_t off = 8 + 4 + 8 + plan.config_text.size() + 3 * 8 + 4 * 8;  // engine.cpp:421-429
    const bool same = full.compare(off, block.size(), block) == 0;
    expect(same, "checkpoint state block == reference bytes", same ? 0.0 : 1.0);
    gpu3.restore_state_block(block);
    const SystemState r3 = gpu3.state();
    const double dfr = max_diff(r3.force, ref2.state().force) / std::max(1.0, max_abs(ref2.state().force));
    expect(dfr <= 1e-10, "forces after state-block restore", dfr);
  }
  // charged rigid dimers + LJ with reaction field (test_potentials.cpp:214-258 shape)
  {
    SystemComposition comp;
    comp.species = {build_species("pair", {charge(0.2, 0, 0, 0.5, 1), charge(-0.2, 0, 0, -0.5, 1),
                                           lj(0, 0, 0, 1, 1, 1)})};
    comp.counts = {256};
    comp.box_length = std::cbrt(256 / 0.5);
    comp.temperature = 1.0;
    ForceFieldOptions opts;
    opts.cutoff = 0.45 * comp.box_length;
    opts.method = ElectrostaticsMethod::reaction_field;
    opts.eps_rf = 65.0;
    compare_eval("RF dimers", comp, opts, init_lattice(comp, 3));
  }
  // ions with Ewald (reference ewald_tune)
  {
    SystemComposition comp;
    comp.species = {build_species("cat", {lj(0, 0, 0, 1.0, 0.5, 1.0)}),
                    build_species("ani", {lj(0, 0, 0, 1.2, 0.5, 1.0)})};
    comp.species[0].sites[0].q = 1.0;
    comp.species[0].net_charge = 1.0;
    comp.species[1].sites[0].q = -1.0;
    comp.species[1].net_charge = -1.0;
    comp.counts = {108, 108};
    comp.box_length = std::cbrt(216 / 0.4);
    comp.temperature = 1.0;
    ForceFieldOptions opts;
    opts.cutoff = 0.45 * comp.box_length;
    opts.method = ElectrostaticsMethod::ewald;
    opts.ewald = ewald_tune(1e-6, opts.cutoff, comp.box_length);
    compare_eval("Ewald ions", comp, opts, init_lattice(comp, 5));
  }
  std::printf("%s\n", failures ? "FAILED" : "PASSED");
  return failures ? 1 : 0;
}
