"""CPU: pins the oracle (oracle/tmd_oracle.c) to the reference.

(1) bit-exact against the committed golden vectors generated from the
unmodified reference (tests/golden/make_golden.py); (2) bit-exact against the
reference library itself (oracle/_ref) at BASELINE sizes when it is built;
(3) the known-answer values of the reference's own tests
(tests/test_potentials.cpp, test_ewald.cpp, test_parallel.cpp)."""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle
from paper_1507_07548_b200 import configs
from paper_1507_07548_b200.configs import Rng

import golden_cases
import systems

GOLDEN = Path(__file__).resolve().parent / "golden"
EVAL_CASES = golden_cases.eval_cases()
TRAJ_CASES = golden_cases.traj_cases()


def energy_vec(e):
    return np.array([getattr(e, f) for f in golden_cases.ENERGY_FIELDS])


def test_rng_matches_reference_draws():
    g = np.load(GOLDEN / "rng.npz")
    for k, seed in enumerate(g["seeds"]):
        a, b, c = Rng(int(seed)), Rng(int(seed)), Rng(int(seed))
        assert [a.next_u64() for _ in range(32)] == [int(x) for x in g["u64"][k]]
        assert np.array_equal([b.uniform() for _ in range(32)], g["uniform"][k])
        assert np.array_equal([c.gaussian() for _ in range(32)], g["gaussian"][k])


@pytest.mark.parametrize("name", list(golden_cases.species_cases()))
def test_oracle_build_species_bitexact(name):
    g = np.load(GOLDEN / "species.npz")
    sp = pyoracle.build_species_c(golden_cases.species_cases()[name], "oracle")
    body = np.array([sp.sites[k].body_pos[:] for k in range(sp.n_sites)])
    assert np.array_equal(body, g[name + "_body"])
    assert np.array_equal(np.array(sp.inertia_principal[:]), g[name + "_inertia"])
    assert np.array_equal([sp.total_mass, sp.net_charge, sp.max_extent, sp.rotational_dof],
                          g[name + "_scalars"])


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_oracle_evaluate_bitexact_vs_golden(name):
    comp, opts, _ = EVAL_CASES[name]
    g = np.load(GOLDEN / f"eval_{name}.npz")
    o = pyoracle.OracleFF(comp, opts)
    r = o.evaluate(g["pos"], g["orient"])
    assert np.array_equal(r["force"], g["force"])
    assert np.array_equal(r["torque"], g["torque"])
    assert np.array_equal(energy_vec(r["energy"]), g["energy"])
    assert r["virial"] == float(g["virial"])
    assert np.array_equal(o.pair_list(g["pos"]), g["pairs"])
    assert o.warning == str(g["warning"])


@pytest.mark.parametrize("name", list(TRAJ_CASES))
def test_oracle_trajectory_bitexact_vs_golden(name):
    comp, opts, _, dt, steps = TRAJ_CASES[name]
    g = np.load(GOLDEN / f"traj_{name}.npz")
    o = pyoracle.OracleFF(comp, opts)
    r = o.run(float(g["dt"]), int(g["steps"]), g["pos0"], g["orient0"], g["vel0"], g["ang_vel0"])
    for k in ("pos", "orient", "vel", "ang_vel", "force", "torque"):
        assert np.array_equal(r[k], g[k]), k
    assert np.array_equal(energy_vec(r["energy"]), g["energy"])


needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg4"])
def test_oracle_bitexact_vs_reference_at_baseline_sizes(cfg):
    wl = configs.make(cfg) if cfg != "cfg4" else configs.make("cfg4", replicas=1)
    st = wl.states[0]
    a = pyoracle.OracleFF(wl.comp, wl.opts).evaluate(st.pos, st.orient)
    ref = pyoracle.RefFF(wl.comp, wl.opts)
    b = ref.evaluate(st.pos, st.orient)
    assert np.array_equal(a["force"], b["force"])
    assert np.array_equal(a["torque"], b["torque"])
    assert np.array_equal(energy_vec(a["energy"]), energy_vec(b["energy"]))
    assert a["virial"] == b["virial"]
    assert np.array_equal(pyoracle.OracleFF(wl.comp, wl.opts).pair_list(st.pos), ref.pair_list(st.pos))


@needs_ref
def test_oracle_steps_bitexact_vs_reference_engine():
    wl = configs.make("cfg0")
    st = wl.states[0]
    eng = pyoracle.RefEngine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st.pos, st.orient, st.vel, st.ang_vel)
    eng.step(10)
    b = eng.state()
    a = pyoracle.OracleFF(wl.comp, wl.opts).run(wl.dt, 10, st.pos, st.orient, st.vel, st.ang_vel)
    for k in ("pos", "vel", "force"):
        assert np.array_equal(a[k], b[k]), k


@needs_ref
def test_ewald_tune_matches_reference():
    for args in [(1e-6, 2.0, 4.0), (1e-6, 3.0, 6.0), (1e-4, 5.0, 10.0), (1e-14, 4.0, 8.0)]:
        assert pyoracle.ewald_tune(*args, which="oracle") == pyoracle.ewald_tune(*args, which="ref")


# ---- known answers of the reference's own tests, on the oracle


def two_body(r, rc=4.0, box=10.0):
    comp = systems.lj_fluid(2, box)
    pos = np.array([[4.0, 5.0, 5.0], [4.0 + r, 5.0, 5.0]])
    orient = np.tile([1.0, 0, 0, 0], (2, 1))
    return pyoracle.OracleFF(comp, systems.lj_opts(rc)).evaluate(pos, orient)


def test_lj_closed_forms():  # test_potentials.cpp:10-39
    assert abs(two_body(1.0)["energy"].lj) < 1e-14
    rmin = 2.0 ** (1.0 / 6.0)
    r = two_body(rmin)
    assert r["energy"].lj == pytest.approx(-1.0, rel=1e-14)
    assert np.abs(r["force"]).max() < 1e-13
    assert two_body(2.0)["energy"].lj == pytest.approx(-0.0615234375, rel=1e-14)


def test_lrc_against_quadrature():  # test_potentials.cpp:56-85
    comp = systems.lj_fluid(100, 5.0)
    o = pyoracle.OracleFF(comp, systems.lj_opts(2.5))
    st = systems.random_state(comp, 1, 0.8)
    e = o.evaluate(st.pos, st.orient)["energy"]
    a = 1.0 / 2.5  # integral_0^{1/rc} 4 (s^8 - s^2) ds, closed form of the quadrature oracle
    tail = 4.0 * (a ** 9 / 9.0 - a ** 3 / 3.0)
    expected = 2.0 * math.pi * (100.0 * 100.0 / 125.0) * tail
    assert e.lrc == pytest.approx(expected, rel=1e-10)


def test_virial_matches_minus_3v_dudv():  # test_potentials.cpp:293-301
    comp = systems.lj_fluid(25, 6.0, 1.2)
    st = systems.random_state(comp, 21, 0.9)
    r = pyoracle.OracleFF(comp, systems.lj_opts(2.8)).evaluate(st.pos, st.orient)
    assert r["virial"] == pytest.approx(-3.0 * comp.volume() * r["energy"].du_dv_explicit, rel=1e-12)


def test_third_law():  # test_parallel.cpp:98-120
    comp, opts = systems.dimer_mono_mixture()
    st = systems.random_state(comp, 31, 0.85)
    f = pyoracle.OracleFF(comp, opts).evaluate(st.pos, st.orient)["force"]
    assert np.all(np.abs(f.sum(axis=0)) < 1e-10 * max(1.0, np.abs(f).max()))


def test_madelung_constant():  # test_ewald.cpp:52-76
    comp, opts, st = systems.rock_salt()
    e = pyoracle.OracleFF(comp, opts).evaluate(st.pos, st.orient)["energy"]
    assert e.total() / 32.0 == pytest.approx(-1.747565, rel=1e-3 / 1.747565)


def test_coincident_neutral_charges_zero_energy():  # test_ewald.cpp:33-50
    from paper_1507_07548_b200 import SystemComposition, build_species, make_charge_site
    comp = SystemComposition([build_species("z", [make_charge_site(0, 0, 0, 0.7, 1.0),
                                                  make_charge_site(0, 0, 0, -0.7, 1.0)])], [3], 10.0, 1.0)
    from paper_1507_07548_b200 import EwaldParams
    opts = systems.ewald_opts(4.0, EwaldParams(0.8, 6))
    pos = np.array([[1.0, 1.0, 1.0], [5.0, 5.5, 4.0], [8.0, 2.0, 7.0]])
    e = pyoracle.OracleFF(comp, opts).evaluate(pos, np.tile([1.0, 0, 0, 0], (3, 1)))["energy"]
    assert abs(e.total()) < 1e-12


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_random_ions_vs_direct_image_sum(seed):  # test_ewald.cpp:78-93
    from paper_1507_07548_b200 import ewald_tune
    comp = systems.ion_pair_comp(4, 6.0)
    st = systems.random_state(comp, seed, 1.0)
    q = [1, 1, 1, 1, -1, -1, -1, -1]
    oracle_u = systems.direct_image_sum_converged(st.pos, q, 6.0)
    opts = systems.ewald_opts(3.0, ewald_tune(1e-6, 3.0, 6.0))
    u = pyoracle.OracleFF(comp, opts).evaluate(st.pos, st.orient)["energy"].total()
    assert u == pytest.approx(oracle_u, rel=1e-4)
