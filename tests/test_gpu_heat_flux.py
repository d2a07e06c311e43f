"""GPU parity of the heat flux J_q (k_heat_flux through b2md_heat_flux /
b2md_heat_flux_state) against the reference's golden vectors, the oracle
(tmd_oracle.c: oracle_heat_flux, pinned bit-exact to tmd::heat_flux) and the
reference's own known answers (tests/test_greenkubo.cpp:172-287).

Tolerance: |dJ_q| <= 1e-10 * scale per component, scale = max(|J_q|, sum_i
|(e_kin_i - h_i) v_i|, 1) (flux_checks.flux_scale) — the force tolerance of
BASELINE.json's north_star applied to a sum whose terms can cancel.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

import flux_checks
import golden_cases

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
J_TOL = 1e-10


def check_flux(comp, st, h, jq, ref, what=""):
    scale = flux_checks.flux_scale(comp, st, h, ref)
    err = float(np.abs(np.asarray(jq) - ref).max()) / scale
    assert err <= J_TOL, f"{what}: {err:.3e} > {J_TOL} (jq={jq}, ref={ref})"


def state_of(comp, pos, orient, vel, ang_vel):
    st = b2.SystemState(comp.molecule_count(), comp.box_length)
    st.pos, st.orient, st.vel, st.ang_vel = (np.array(a, dtype=np.float64)
                                             for a in (pos, orient, vel, ang_vel))
    return st


@pytest.mark.parametrize("name", list(golden_cases.eval_cases()))
def test_golden_heat_flux(name):
    comp, opts, _ = golden_cases.eval_cases()[name]
    g = np.load(GOLDEN / f"flux_{name}.npz")
    st = state_of(comp, g["pos"], g["orient"], g["vel"], g["ang_vel"])
    jq = b2.ForceField(comp, opts).heat_flux(st, g["h"])
    check_flux(comp, st, g["h"], jq, g["jq"], name)


def test_heat_flux_rest_and_ideal_gas():  # test_greenkubo.cpp:172-216
    comp, opts, st, h, expected = flux_checks.ideal_gas_case()
    ff = b2.ForceField(comp, opts)
    np.testing.assert_allclose(ff.heat_flux(st, h), expected, rtol=1e-12)
    rest = st.copy()
    rest.vel[:] = 0.0
    rest.ang_vel[:] = 0.0
    assert np.linalg.norm(ff.heat_flux(rest, [0.0])) < 1e-15


def test_heat_flux_independent_double_loop():  # test_greenkubo.cpp:218-287
    comp, opts, st, h = flux_checks.dimer_case()
    jq = b2.heat_flux(b2.ForceField(comp, opts), st, h)
    ind = flux_checks.independent_flux(comp, opts.cutoff, st, h)
    np.testing.assert_allclose(jq, ind, rtol=1e-12, atol=1e-12 * np.abs(ind).max())


def test_heat_flux_enthalpy_count_is_config_error():  # greenkubo.cpp:184-185
    comp, opts, st, _, _ = flux_checks.ideal_gas_case()
    ff = b2.ForceField(comp, opts)
    for h in ([], [1.0, 2.0]):
        with pytest.raises(b2.ConfigError, match="enthalpy"):
            ff.heat_flux(st, h)
    eng = b2.Engine(comp, opts, 0.002)
    with pytest.raises(b2.ConfigError):
        eng.heat_flux([0.0])  # no state yet
    eng.set_state(st)
    with pytest.raises(b2.ConfigError, match="enthalpy"):
        eng.heat_flux([])


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_heat_flux_baseline_configs(cfg):
    wl = configs.make(cfg)
    st0 = wl.states[0]
    vel, ang_vel, h = golden_cases.flux_inputs(cfg, wl.comp)
    st = state_of(wl.comp, st0.pos, st0.orient, vel, ang_vel)
    jq = b2.ForceField(wl.comp, wl.opts).heat_flux(st, h)
    ref = pyoracle.OracleFF(wl.comp, wl.opts).heat_flux(st.pos, st.orient, vel, ang_vel, h)
    check_flux(wl.comp, st, h, jq, ref, cfg)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_heat_flux_of_engine_state_after_steps(cfg):
    """b2md_heat_flux on the device-resident state (Engine::run's sampling,
    engine.cpp:235-238) equals the oracle on the downloaded state."""
    wl = configs.make(cfg)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(wl.states[0])
    eng.step(10)
    h = golden_cases.flux_inputs(cfg, wl.comp)[2]
    jq = eng.heat_flux(h)
    s = eng.state()
    ref = pyoracle.OracleFF(wl.comp, wl.opts).heat_flux(s.pos, s.orient, s.vel, s.ang_vel, h)
    check_flux(wl.comp, s, h, jq, ref, cfg)


def test_heat_flux_replicas_cfg4():
    wl = configs.make("cfg4", replicas=4, steps=5)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=4)
    eng.set_state(wl.states)
    eng.step(5)
    h = np.array([-1.5])
    jq = eng.heat_fluxes(h)
    assert jq.shape == (4, 3)
    ora = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, s in enumerate(eng.states()):
        ref = ora.heat_flux(s.pos, s.orient, s.vel, s.ang_vel, h)
        check_flux(wl.comp, s, h, jq[r], ref, f"replica {r}")


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
@pytest.mark.parametrize("world", [2, 3])
def test_heat_flux_shards_sum_to_full(cfg, world):
    """Row shards (no communicator): the partial fluxes sum to the whole.
    cfg2 takes the bit-matrix walk (pair parts split by tiles, the kinetic
    part on rank 0 only), cfg3 the cluster walk (each rank owns disjoint rows
    and adds their kinetic terms)."""
    wl = configs.make(cfg)
    st0 = wl.states[0]
    vel, ang_vel, h = golden_cases.flux_inputs(cfg, wl.comp)
    st = state_of(wl.comp, st0.pos, st0.orient, vel, ang_vel)
    full = b2.ForceField(wl.comp, wl.opts).heat_flux(st, h)
    total = np.zeros(3)
    for rank in range(world):
        ff = b2.ForceField(wl.comp, wl.opts)
        ff.set_shard(rank, world)
        total += ff.heat_flux(st, h)
    check_flux(wl.comp, st, h, total, full, f"world {world}")


def test_heat_flux_deterministic():
    wl = configs.make("cfg1")
    st0 = wl.states[0]
    vel, ang_vel, h = golden_cases.flux_inputs("cfg1", wl.comp)
    st = state_of(wl.comp, st0.pos, st0.orient, vel, ang_vel)
    ff = b2.ForceField(wl.comp, wl.opts)
    a = ff.heat_flux(st, h)
    b = ff.heat_flux(st, h)
    assert np.array_equal(a, b)
