"""GPU: kinetic energies, Engine::apply_thermostat and Engine::run's
thermostatted loop (b2md_kinetic_energy / b2md_apply_thermostat /
b2md_step_thermostat) against the oracle (pinned bit-exact to the reference's
thermostat in tests/test_sampling.py).  The device reduces the kinetic
energies in a fixed tree order (the reference sums serially), so the bar is
1e-13 relative on energies and scales and 1e-9 on thermostatted trajectories."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_kinetic_energy_and_thermostat(cfg):
    wl = configs.make(cfg)
    st = wl.states[0].copy()
    st.vel *= 1.3
    st.ang_vel *= 0.7
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    kt, kr = eng.kinetic_energies()
    ref = o.kinetic_energy(st.vel, st.ang_vel)
    assert abs(kt[0] - ref[0]) <= 1e-13 * ref[0]
    assert abs(kr[0] - ref[1]) <= 1e-13 * max(ref[1], 1.0)
    eng.apply_thermostat()
    s = eng.state()
    v, w = o.apply_thermostat(st.vel, st.ang_vel)
    assert np.abs(s.vel - v).max() <= 1e-13 * np.abs(v).max()
    assert np.abs(s.ang_vel - w).max() <= 1e-13 * max(np.abs(w).max(), 1.0)
    dof_t = 3 * wl.comp.molecule_count() - 3
    kt2, _ = eng.kinetic_energies()
    assert kt2[0] == pytest.approx(0.5 * dof_t * wl.comp.temperature, rel=1e-12)


def test_thermostat_zero_energy_is_numerical_error():
    wl = configs.make("cfg1")
    st = wl.states[0].copy()
    st.ang_vel[:] = 0.0
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    with pytest.raises(b2.NumericalError, match="zero rotational kinetic energy"):
        eng.apply_thermostat()
    st.vel[:] = 0.0
    eng.set_state(st)
    with pytest.raises(b2.NumericalError, match="zero translational kinetic energy"):
        eng.apply_thermostat()


@pytest.mark.parametrize("cfg,interval,done", [("cfg1", 3, 1), ("cfg0", 4, 0), ("cfg3", 5, 2)])
def test_thermostatted_run_tracks_oracle(cfg, interval, done):
    """engine.cpp:273-296: the rescale after every step whose number (counted
    from the phase start, `done` steps already taken) divides `interval`."""
    wl = configs.make(cfg)
    st = wl.states[0]
    nsteps = 11 if cfg == "cfg3" else 17
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    eng.step_thermostat(nsteps, interval, done)
    s = eng.state()
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    pos, q, v, w = st.pos.copy(), st.orient.copy(), st.vel.copy(), st.ang_vel.copy()
    k = 0
    while k < nsteps:
        step_no = done + k
        chunk = min(interval - step_no % interval, nsteps - k)
        r = o.run(wl.dt, chunk, pos, q, v, w)
        pos, q, v, w = r["pos"], r["orient"], r["vel"], r["ang_vel"]
        k += chunk
        if (done + k) % interval == 0:
            v, w = o.apply_thermostat(v, w)
    L = wl.comp.box_length
    d = s.pos - pos
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= 1e-9
    assert np.abs(s.vel - v).max() <= 1e-9 * np.abs(v).max()


def test_thermostat_replicas():
    wl = configs.make("cfg4", replicas=3, steps=2)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=3)
    eng.set_state(wl.states)
    eng.apply_thermostat()
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, s in enumerate(eng.states()):
        v, w = o.apply_thermostat(wl.states[r].vel, wl.states[r].ang_vel)
        assert np.abs(s.vel - v).max() <= 1e-13 * np.abs(v).max()
