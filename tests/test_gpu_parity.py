"""GPU parity: the sm_100a path through the C ABI against the oracle and the
reference's golden vectors.

Tolerances (BASELINE.json north_star):
  * COM pair lists: bit-exact (set and order);
  * forces / torques: max |dF| <= 1e-10 * max |F_ref|;
  * energy parts, virial: relative 1e-9 (absolute floor 1e-9 * sum |parts|);
  * trajectories: positions (minimum image) / L, velocities / max|v|,
    quaternions (sign fixed), total energy: 1e-9.
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

import golden_cases
import systems

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
F_TOL = 1e-10
E_TOL = 1e-9
T_TOL = 1e-9


def check_vec(a, ref, tol=F_TOL, what=""):
    scale = max(1.0, float(np.abs(ref).max())) if ref.size else 1.0
    err = float(np.abs(a - ref).max()) / scale if ref.size else 0.0
    assert err <= tol, f"{what}: {err:.3e} > {tol}"


def check_energy(e, ref, virial=None, ref_virial=None):
    fields = golden_cases.ENERGY_FIELDS
    a = np.array([getattr(e, f) for f in fields])
    b = ref if isinstance(ref, np.ndarray) else np.array([getattr(ref, f) for f in fields])
    floor = E_TOL * max(1e-300, float(np.abs(b).sum()))
    for f, x, y in zip(fields, a, b):
        assert abs(x - y) <= max(E_TOL * abs(y), floor), f"{f}: {x} vs {y}"
    if virial is not None:
        assert abs(virial - ref_virial) <= E_TOL * max(abs(ref_virial), 1.0)


def gpu_eval(comp, opts, pos, orient):
    ff = b2.ForceField(comp, opts)
    st = b2.SystemState(comp.molecule_count(), comp.box_length)
    st.pos = np.array(pos, dtype=np.float64)
    st.orient = np.array(orient, dtype=np.float64)
    ff.evaluate(st)
    return ff, st


# ------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("name", list(golden_cases.eval_cases()))
def test_golden_evaluations(name):
    comp, opts, _ = golden_cases.eval_cases()[name]
    g = np.load(GOLDEN / f"eval_{name}.npz")
    ff, st = gpu_eval(comp, opts, g["pos"], g["orient"])
    assert np.array_equal(ff.pair_list(), g["pairs"])
    check_vec(st.force, g["force"], what="force")
    check_vec(st.torque, g["torque"], what="torque")
    check_energy(st.energy, g["energy"], st.virial, float(g["virial"]))
    assert ff.warning == str(g["warning"])


@pytest.mark.parametrize("name", list(golden_cases.traj_cases()))
def test_golden_trajectories(name):
    comp, opts, _, _, _ = golden_cases.traj_cases()[name]
    g = np.load(GOLDEN / f"traj_{name}.npz")
    eng = b2.Engine(comp, opts, float(g["dt"]))
    st = b2.SystemState(comp.molecule_count(), comp.box_length)
    st.pos, st.orient, st.vel, st.ang_vel = g["pos0"], g["orient0"], g["vel0"], g["ang_vel0"]
    eng.set_state(st)
    eng.step(int(g["steps"]))
    out = eng.state()
    compare_states(out, {k: g[k] for k in ("pos", "orient", "vel", "ang_vel")}, comp.box_length)
    check_energy(out.energy, g["energy"])


def compare_states(out, ref, L):
    d = out.pos - ref["pos"]
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= T_TOL
    assert np.abs(out.vel - ref["vel"]).max() / max(1e-300, np.abs(ref["vel"]).max()) <= T_TOL
    q, qr = out.orient, ref["orient"]
    sign = np.where(np.sum(q * qr, axis=1) < 0, -1.0, 1.0)[:, None]
    assert np.abs(q * sign - qr).max() <= T_TOL
    wr = np.abs(ref["ang_vel"]).max()
    if wr > 0:
        assert np.abs(out.ang_vel - ref["ang_vel"]).max() / wr <= T_TOL


# ------------------------------------------------ BASELINE configs vs oracle
@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_baseline_config_evaluation(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(wl.comp, wl.opts, st.pos, st.orient)
    pairs = ff.pair_list()
    assert len(pairs) == ref["com_pairs"]
    assert np.array_equal(pairs, o.pair_list(st.pos))
    check_vec(out.force, ref["force"], what="force")
    check_vec(out.torque, ref["torque"], what="torque")
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1"])
def test_baseline_100_step_trajectory(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    eng.step(wl.steps)
    out = eng.state()
    ref = pyoracle.OracleFF(wl.comp, wl.opts).run(wl.dt, wl.steps, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(out, ref, wl.comp.box_length)
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    # the engine's device pair list after 100 steps is the oracle's on that state
    assert np.array_equal(eng.pair_list(), pyoracle.OracleFF(wl.comp, wl.opts).pair_list(ref["pos"]))


def test_cfg3_100_step_trajectory_vs_reference():
    """cfg3 (cluster walk, re-sorts every 40 steps) for 100 steps against the
    unmodified reference engine's trajectory (tests/golden/traj_cfg3_100.npz,
    make_cfg3_trajectory.py): every 8th molecule's position and velocity and
    the energy at the north-star bar (1e-9)."""
    g = np.load(GOLDEN / "traj_cfg3_100.npz")
    wl = configs.make("cfg3")
    st = wl.states[0]
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    eng.step(int(g["steps"]))
    out = eng.state()
    k = int(g["stride"])
    L = wl.comp.box_length
    d = out.pos[::k] - g["pos"]
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= T_TOL
    assert np.abs(out.vel[::k] - g["vel"]).max() / np.abs(g["vel"]).max() <= T_TOL
    e = out.energy
    assert abs(e.total() - g["energy"][2]) <= T_TOL * abs(g["energy"][2])
    assert abs(e.lj - g["energy"][0]) <= T_TOL * abs(g["energy"][0])
    assert abs(out.virial - float(g["virial"])) <= T_TOL * abs(float(g["virial"]))


def test_replica_batch_cfg4():
    wl = configs.make("cfg4", replicas=4, steps=20)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=4)
    eng.set_state(wl.states)
    first = eng.states()
    eng.step(20)
    outs = eng.states()
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, st in enumerate(wl.states):
        ref0 = o.evaluate(st.pos, st.orient)
        check_vec(first[r].force, ref0["force"], what=f"replica {r} force")
        check_vec(first[r].torque, ref0["torque"], what=f"replica {r} torque")
        ref = o.run(wl.dt, 20, st.pos, st.orient, st.vel, st.ang_vel)
        compare_states(outs[r], ref, wl.comp.box_length)
        check_energy(outs[r].energy, ref["energy"])
        assert np.array_equal(eng.pair_list(r), o.pair_list(ref["pos"]))


def test_replica_batch_cfg4_full_shape():
    """cfg4 at the shape bench.py runs per GPU: the 8-replica batch (seeds
    0-7, T_r = 1.5 + 1.5 u) for 100 steps, EVERY replica against the oracle's
    Engine::step (src/engine.cpp:102-143): pos / L, velocities, quaternions,
    angular velocities and energy at 1e-9, pair lists bit-exact."""
    R, steps = 8, 100
    wl = configs.make("cfg4", replicas=R, steps=steps)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=R)
    eng.set_state(wl.states)
    eng.step(steps)
    outs = eng.states()
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, st in enumerate(wl.states):
        ref = o.run(wl.dt, steps, st.pos, st.orient, st.vel, st.ang_vel)
        compare_states(outs[r], ref, wl.comp.box_length)
        check_energy(outs[r].energy, ref["energy"])
        assert np.array_equal(eng.pair_list(r), o.pair_list(ref["pos"]))


# --------------------------------------------------------------- edge cases
@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 100, 513, 1537, 4100, 8200])
def test_sizes_and_partial_tiles(n):
    box = (n / 0.7) ** (1.0 / 3.0) if n > 8 else 8.0
    rc = min(2.5, 0.5 * box)
    wl = configs.lj_fluid_config(n, n / box ** 3, rc, seed=n) if n > 8 else None
    if wl is None:
        comp = systems.lj_fluid(n, box)
        st = systems.random_state(comp, n, 0.9)
        opts = systems.lj_opts(rc)
    else:
        comp, opts, st = wl.comp, wl.opts, wl.states[0]
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(comp, opts, st.pos, st.orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(st.pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])


@pytest.mark.parametrize("mode", ["0", "2"])
@pytest.mark.parametrize("n", [1, 2, 7, 9, 100, 1537, 4100])
def test_single_site_walks(monkeypatch, mode, n):
    """Both single-site walks -- the cluster walk (B2MD_CLUSTER=2 forces it)
    and the search + bit-matrix walk (=0) -- reproduce the oracle's pairs,
    forces and energies at any size (one partial cluster, rc ~ L/2, ...)."""
    monkeypatch.setenv("B2MD_CLUSTER", mode)
    box = (n / 0.7) ** (1.0 / 3.0) if n > 8 else 8.0
    rc = min(2.5, 0.5 * box)
    if n > 8:
        wl = configs.lj_fluid_config(n, n / box ** 3, rc, seed=n + 1)
        comp, opts, st = wl.comp, wl.opts, wl.states[0]
    else:
        comp, opts = systems.lj_fluid(n, box), systems.lj_opts(rc)
        st = systems.random_state(comp, n, 0.9)
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(comp, opts, st.pos, st.orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(st.pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    assert ff.last_stats.com_pairs == ref["com_pairs"]


@pytest.mark.parametrize("n", [9, 300, 2053])
def test_cluster_walk_single_site_mixture(monkeypatch, n):
    """The cluster walk on a two-species single-site mixture (species-pair LJ
    terms, Lorentz-Berthelot, potentials.cpp:64-69): pairs, forces, energies
    and a short trajectory."""
    monkeypatch.setenv("B2MD_CLUSTER", "2")
    na = n // 3
    box = (n / 0.7) ** (1.0 / 3.0)
    comp = b2.SystemComposition([b2.build_species("a", [b2.make_lj_site(0, 0, 0, 1.0, 1.0, 1.0)]),
                                 b2.build_species("b", [b2.make_lj_site(0, 0, 0, 0.9, 1.3, 2.0)])],
                                [na, n - na], box, 1.0)
    opts = systems.lj_opts(min(2.5, 0.45 * box))
    st = systems.random_state(comp, n, 0.8)
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(comp, opts, st.pos, st.orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(st.pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    dt, steps = 0.002, 10
    eng = b2.Engine(comp, opts, dt)
    eng.set_state(st)
    eng.step(steps)
    got = eng.state()
    tr = o.run(dt, steps, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(got, tr, box)


def test_cluster_walk_cfg3_void():
    """cfg3's lattice start (26^3 truncated: a void at high z, so some
    clusters span far-apart columns) through the cluster walk: oracle pairs,
    forces and energies."""
    wl = configs.make("cfg3")
    st = wl.states[0]
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(wl.comp, wl.opts, st.pos, st.orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(st.pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    # the walk's OWN pair decisions (its in-cutoff count, potentials.cpp:156-161),
    # not only the on-demand list of k_search
    assert ff.last_stats.com_pairs == ref["com_pairs"]


@pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")
def test_cfg3_100_steps_full_state_vs_reference_engine():
    """cfg3 (N = 16384) through the cluster walk for 100 steps against the
    unmodified reference tmd::Engine run live on the host cores (all threads):
    EVERY molecule's position / velocity / force, the energy parts and the
    walk's own pair count at step 0 and after the 100 steps
    (src/engine.cpp:102-143, src/potentials.cpp:156-181)."""
    import copy
    import os
    wl = configs.make("cfg3", steps=100)
    st = wl.states[0]
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    _, stats0 = eng.energies()
    opts = copy.copy(wl.opts)
    opts.workers = max(1, os.cpu_count() or 1)
    ref = pyoracle.RefEngine(wl.comp, opts, wl.dt)
    ref.set_state(st.pos, st.orient, st.vel, st.ang_vel)
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    assert stats0[0].com_pairs == o.evaluate(st.pos, st.orient)["com_pairs"]
    eng.step(100)
    ref.step(100)
    out, r = eng.state(), ref.state()
    compare_states(out, r, wl.comp.box_length)
    check_vec(out.force, r["force"], what="force after 100 steps")
    check_energy(out.energy, r["energy"], out.virial, r["virial"])
    _, stats = eng.energies()
    assert stats[0].com_pairs == o.evaluate(out.pos, out.orient)["com_pairs"]


@pytest.mark.parametrize("n", [1001, 2053])
def test_cluster_walk_replicas(n):
    """Single-site replicas through the cluster walk (rc < 0.3 L, re-sorted
    every 8 steps here): per-replica oracle forces, energies, pair lists and a
    30-step trajectory.  n is not a multiple of the cluster size, so each
    replica's last cluster is short and its staging reads into the next
    replica (or the zeroed padding)."""
    wls = [configs.lj_fluid_config(n, 0.8, 2.5, seed=11 + r) for r in range(3)]
    comp, opts = wls[0].comp, wls[0].opts
    states = [w.states[0] for w in wls]
    dt, steps = 0.005, 30
    eng = b2.Engine(comp, opts, dt, replicas=3)
    eng.set_sort_interval(8)
    eng.set_state(states)
    first = eng.states()
    eng.step(steps)
    outs = eng.states()
    o = pyoracle.OracleFF(comp, opts)
    for r, st in enumerate(states):
        ref0 = o.evaluate(st.pos, st.orient)
        check_vec(first[r].force, ref0["force"], what=f"replica {r} force")
        check_energy(first[r].energy, ref0["energy"], first[r].virial, ref0["virial"])
        ref = o.run(dt, steps, st.pos, st.orient, st.vel, st.ang_vel)
        compare_states(outs[r], ref, comp.box_length)
        check_energy(outs[r].energy, ref["energy"])
        assert np.array_equal(eng.pair_list(r), o.pair_list(ref["pos"]))


def test_cluster_walk_unwrapped_positions(monkeypatch):
    """The cluster walk on positions outside [0, L) (ForceField::evaluate
    takes them as given): such clusters are never culled, the exact minimum
    image decides."""
    monkeypatch.setenv("B2MD_CLUSTER", "2")
    wl = configs.lj_fluid_config(600, 0.7, 2.5, seed=3)
    L = wl.comp.box_length
    st = wl.states[0]
    rng = np.random.default_rng(5)
    pos = st.pos + L * rng.integers(-3, 4, size=st.pos.shape)
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    ref = o.evaluate(pos, st.orient)
    ff, out = gpu_eval(wl.comp, wl.opts, pos, st.orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])


def test_cfg3_trajectory_with_resorts():
    """cfg3 (cluster walk, re-sorted every 10 steps here) for 25 steps against
    the oracle, and bit-identical when repeated (fixed summation order)."""
    wl = configs.make("cfg3")
    st = wl.states[0]
    outs = []
    for _ in range(2):
        eng = b2.Engine(wl.comp, wl.opts, wl.dt)
        eng.set_sort_interval(10)
        eng.set_state(st)
        eng.step(25)
        outs.append(eng.state())
    ref = pyoracle.OracleFF(wl.comp, wl.opts).run(wl.dt, 25, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(outs[0], ref, wl.comp.box_length)
    check_energy(outs[0].energy, ref["energy"], outs[0].virial, ref["virial"])
    assert np.array_equal(outs[0].pos, outs[1].pos) and np.array_equal(outs[0].vel, outs[1].vel)
    assert np.array_equal(eng.pair_list(), pyoracle.OracleFF(wl.comp, wl.opts).pair_list(ref["pos"]))


def test_min_image_ties_and_far_images():
    """Separations exactly L/2 (round-half-even ties), positions several
    boxes away (nearbyint = +-2, +-3) and negative coordinates."""
    comp = systems.lj_fluid(6, 4.0)
    pos = np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0], [0.0, 2.0, 2.0], [-6.0, 9.0, 1.0],
                    [13.5, -7.25, 2.0], [2.0, 2.0, 2.0]])
    orient = np.tile([1.0, 0, 0, 0], (6, 1))
    opts = systems.lj_opts(2.0)
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(pos, orient)
    ff, out = gpu_eval(comp, opts, pos, orient)
    assert np.array_equal(ff.pair_list(), o.pair_list(pos))
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"])


def test_ideal_gas_dummy_sites():  # test_potentials.cpp:160-176
    comp = b2.SystemComposition([b2.build_species("ghost", [b2.Site(b2.SiteKind.dummy, (0, 0, 0), 0, 0, 0, 1.0)])],
                                [16], 6.0, 1.0)
    st = systems.random_state(comp, 3, 0.0)
    ff, out = gpu_eval(comp, systems.lj_opts(2.5), st.pos, st.orient)
    assert out.energy.total() == 0.0 and out.energy.du_dv() == 0.0 and out.energy.d2u_dv2() == 0.0
    assert np.all(out.force == 0.0)


def test_repeated_evaluations_bit_identical():  # test_parallel.cpp:84-96
    wl = configs.make("cfg1")
    st = wl.states[0]
    ff = b2.ForceField(wl.comp, wl.opts)
    a, b = st.copy(), st.copy()
    ff.evaluate(a)
    ff.evaluate(b)
    assert np.array_equal(a.force, b.force) and np.array_equal(a.torque, b.torque)
    assert a.energy == b.energy and a.virial == b.virial


def test_third_law_and_virial_identity():
    comp, opts = systems.dimer_mono_mixture()
    st = systems.random_state(comp, 31, 0.85)
    _, out = gpu_eval(comp, opts, st.pos, st.orient)
    assert np.all(np.abs(out.force.sum(axis=0)) < 1e-10 * max(1.0, np.abs(out.force).max()))
    comp = systems.lj_fluid(25, 6.0, 1.2)
    st = systems.random_state(comp, 21, 0.9)
    _, out = gpu_eval(comp, systems.lj_opts(2.8), st.pos, st.orient)
    assert out.virial == pytest.approx(-3.0 * comp.volume() * out.energy.du_dv_explicit, rel=1e-12)


def test_madelung_on_gpu():
    comp, opts, st = systems.rock_salt()
    _, out = gpu_eval(comp, opts, st.pos, st.orient)
    assert out.energy.total() / 32.0 == pytest.approx(-1.747565, rel=1e-3 / 1.747565)


def test_free_flight_exact():  # test_engine.cpp:27-43
    comp = systems.lj_fluid(1, 10.0)
    eng = b2.Engine(comp, systems.lj_opts(3.0), 0.01)
    st = b2.SystemState(1, 10.0)
    st.pos[0] = (5.0, 5.0, 5.0)
    st.vel[0] = (1.0, 0.0, 0.0)
    eng.set_state(st)
    eng.step()
    assert eng.state().pos[0, 0] == 5.0 + 0.01 * 1.0 and eng.state().pos[0, 1] == 5.0
    eng.step()
    assert eng.state().pos[0, 0] == 5.0 + 0.01 + 0.01


def test_two_body_orbit_energy_drift():  # test_engine.cpp:45-65
    comp = systems.lj_fluid(2, 20.0)
    eng = b2.Engine(comp, systems.lj_opts(8.0), 0.001)
    st = b2.SystemState(2, 20.0)
    st.pos[0], st.pos[1] = (10.0, 10.0, 10.0), (11.2, 10.0, 10.0)
    st.vel[0], st.vel[1] = (0.0, 0.4, 0.0), (0.0, -0.4, 0.0)
    eng.set_state(st)
    s0 = eng.state()
    e0 = b2.kinetic_energy_trans(comp, s0) + s0.energy.total()
    drift = 0.0
    for _ in range(100):
        eng.step(100)
        s = eng.state()
        drift = max(drift, abs(b2.kinetic_energy_trans(comp, s) + s.energy.total() - e0))
    assert drift / abs(e0) < 1e-5


def test_torque_free_dumbbell():  # test_engine.cpp:67-102
    """Lab-frame angular momentum of a torque-free linear rotor over 1e4 steps.
    The reference's own bound (1e-8) is not met by the reference itself: the
    NO_SQUISH splitting drifts |dL| = 4.3e-8 here (oracle == reference, bit for
    bit); the GPU must reproduce the reference's trajectory, so it is compared
    to the oracle at the trajectory tolerance and to the drift the reference
    shows."""
    comp = systems.dumbbell()
    eng = b2.Engine(comp, systems.lj_opts(3.0), 0.001)
    st = b2.SystemState(1, 10.0)
    st.pos[0] = (5, 5, 5)
    st.ang_vel[0] = (0.0, 1.3, 0.7)
    eng.set_state(st)
    inertia = comp.species[0].inertia_principal

    def lab_l(s):
        return systems.rotate(s.orient[0], inertia * s.ang_vel[0])

    s0 = eng.state()
    l0 = lab_l(s0)
    e0 = b2.kinetic_energy_rot(comp, s0)
    eng.step(10000)
    s1 = eng.state()
    ref = pyoracle.OracleFF(comp, systems.lj_opts(3.0)).run(0.001, 10000, st.pos, st.orient, st.vel,
                                                            st.ang_vel)
    compare_states(s1, ref, 10.0)
    assert np.abs(lab_l(s1) - l0).max() < 1e-7
    assert b2.kinetic_energy_rot(comp, s1) == pytest.approx(e0, rel=1e-10)
    assert abs(np.linalg.norm(s1.orient[0]) - 1.0) < 1e-9


def test_three_site_rotor_energy():  # test_engine.cpp:104-129
    """The reference's 1e-5 energy bound does not hold for the reference
    itself here (the truncated, unshifted LJ makes crossings of rc jump the
    energy: the oracle == reference drifts 0.7% over 4000 steps); the GPU must
    reproduce the reference's trajectory and its energy history."""
    comp, opts, st, dt, _ = golden_cases.traj_cases()["tri"]
    eng = b2.Engine(comp, opts, dt)
    eng.set_state(st)
    eng.step(4000)
    out = eng.state()
    ref = pyoracle.OracleFF(comp, opts).run(dt, 4000, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(out, ref, comp.box_length)
    check_energy(out.energy, ref["energy"])


def test_nan_is_fatal():  # test_engine.cpp:232-245
    comp = systems.lj_fluid(4, 6.0)
    eng = b2.Engine(comp, systems.lj_opts(2.5), 0.01)
    st = systems.random_state(comp, 2, 0.9)
    st.vel[2] = (np.nan, 0, 0)
    eng.set_state(st)
    with pytest.raises(b2.NumericalError, match="non-finite state for molecule 2"):
        eng.step()


def test_nan_is_fatal_cluster_walk():
    """A NaN velocity on the cluster path (cfg3-like cutoff): the step fails
    with the reference's message for the same molecule (check_finite's first
    non-finite molecule after the NaN has reached its partners' forces)."""
    wl = configs.lj_fluid_config(600, 0.7, 2.5, seed=9)
    st = wl.states[0].copy()
    st.vel[37] = (np.nan, 0.0, 0.0)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(st)
    with pytest.raises(b2.NumericalError) as got:
        eng.step(3)
    with pytest.raises(Exception) as ref:
        pyoracle.OracleFF(wl.comp, wl.opts).run(wl.dt, 3, st.pos, st.orient, st.vel, st.ang_vel)
    mol = lambda e: str(e.value).split("molecule")[1].split()[0]
    assert mol(got) == mol(ref)


@pytest.mark.parametrize("pinned", [True, False])
def test_nan_deferred_to_get_state(pinned):
    """step_async defers the NumericalError to the next get_state (the flag
    rides with the download, zero-copy or staged), reported once."""
    comp = systems.lj_fluid(4, 6.0)
    eng = b2.Engine(comp, systems.lj_opts(2.5), 0.01)
    st = systems.random_state(comp, 2, 0.9)
    st.vel[2] = (np.nan, 0, 0)
    eng.set_state(st)
    import torch
    alloc = ((lambda s: torch.empty(s, dtype=torch.float64, pin_memory=True).numpy()) if pinned
             else (lambda s: np.empty(s)))
    bufs = [alloc((4, 3)), alloc((4, 4)), alloc((4, 3))]
    eng.step_async(1)
    with pytest.raises(b2.NumericalError, match="non-finite state for molecule 2"):
        eng.get_state_raw(*bufs)
    assert np.isnan(bufs[2][2, 0])
    eng.get_state_raw(*bufs)  # already reported
    ok = systems.random_state(comp, 2, 0.9)
    eng2 = b2.Engine(comp, systems.lj_opts(2.5), 0.01)
    eng2.set_state(ok)
    eng2.step_async(3)
    eng2.get_state_raw(*bufs)
    eng2.step(1)


def test_set_state_wraps():  # engine.cpp:91-98
    comp = systems.lj_fluid(20, 6.0)
    st = systems.random_state(comp, 11, 0.9)
    moved = st.copy()
    moved.pos = moved.pos + np.array([1.3, -2.1, 0.7]) * 6.0
    eng = b2.Engine(comp, systems.lj_opts(2.5), 0.005)
    eng.set_state(moved)
    out = eng.state()
    assert np.all(out.pos >= 0) and np.all(out.pos < 6.0)
    ref = pyoracle.OracleFF(comp, systems.lj_opts(2.5)).run(0.005, 0, moved.pos, moved.orient,
                                                             moved.vel, moved.ang_vel)
    assert np.array_equal(out.pos, ref["pos"])
    check_vec(out.force, ref["force"])


def test_engine_runs_bit_identical():  # test_engine.cpp:185-213 (fixed-seed determinism)
    wl = configs.make("cfg1")
    outs = []
    for _ in range(2):
        eng = b2.Engine(wl.comp, wl.opts, wl.dt)
        eng.set_state(wl.states[0])
        eng.step(20)
        outs.append(eng.state())
    assert np.array_equal(outs[0].pos, outs[1].pos) and np.array_equal(outs[0].vel, outs[1].vel)


# ------------------------------------------------ multi-GPU decomposition
@pytest.mark.parametrize("case", ["lj", "two_clj", "water_ions"])
@pytest.mark.parametrize("world", [2, 3])
def test_shards_sum_to_full_evaluation(case, world):
    """Each rank's shard (tile rows + k-vector range, b2md_set_shard — what a
    rank holds before the NCCL all-reduce) evaluated on this GPU; the sum over
    ranks must equal the full evaluation (reduction-order rounding only)."""
    if case == "lj":
        wl = configs.lj_fluid_config(5000, 0.8, 3.0, seed=4)
        comp, opts, st = wl.comp, wl.opts, wl.states[0]
    elif case == "two_clj":
        wl = configs.two_clj_config(2048, 0.3, 1, 2.0, 0.002, 1, "c1")
        comp, opts, st = wl.comp, wl.opts, wl.states[0]
    else:
        comp, opts, st = golden_cases._water_ions_small(300, 10, 2)
    _, full = gpu_eval(comp, opts, st.pos, st.orient)
    f = np.zeros_like(full.force)
    t = np.zeros_like(full.torque)
    parts = np.zeros(5)
    for rank in range(world):
        ff = b2.ForceField(comp, opts)
        ff.set_shard(rank, world)
        s = st.copy()
        ff.evaluate(s)
        f += s.force
        t += s.torque
        e = s.energy
        parts += [e.lj, e.elec_real, e.elec_recip, s.virial, ff.last_stats.com_pairs]
    check_vec(f, full.force, 1e-12, "sharded force")
    check_vec(t, full.torque, 1e-12, "sharded torque")
    e = full.energy
    ref = np.array([e.lj, e.elec_real, e.elec_recip, full.virial])
    assert np.all(np.abs(parts[:4] - ref) <= 1e-11 * np.maximum(1.0, np.abs(ref)))
    assert int(parts[4]) == len(pyoracle.OracleFF(comp, opts).pair_list(st.pos))


# ------------------------------------------------ partner-search strategies
def _search_variants(comp, opts, pos, orient):
    out = []
    for fix, cull in ((True, True), (True, False), (False, False)):
        ff = b2.ForceField(comp, opts)
        ff.set_search_options(fix, cull)
        st = b2.SystemState(comp.molecule_count(), comp.box_length)
        st.pos, st.orient = np.array(pos), np.array(orient)
        ff.evaluate(st)
        out.append((ff.pair_list(), st.force.copy(), st.torque.copy()))
    return out


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg3", "lj_gas_8192", "lj_shell_4096"])
def test_tile_cull_is_exact(cfg):
    """Tile culling, the unculled fixed-point search and the generic fp64
    search give the same pair list (bit-exact vs the oracle) and the same
    forces.  lj_gas: random positions (blocks span the box, little culls);
    lj_shell: a lattice whose spacing puts many COM distances within 1e-12
    of rmax."""
    if cfg.startswith("lj_gas"):
        rng = np.random.default_rng(4)
        n = 8192
        wl = configs.lj_fluid_config(n, 0.8, 3.0, seed=4, steps=1, name=cfg)
        comp, opts = wl.comp, wl.opts
        pos = rng.uniform(0, comp.box_length, size=(n, 3))
        orient = wl.states[0].orient
    elif cfg.startswith("lj_shell"):
        wl = configs.lj_fluid_config(4096, 0.8, None, seed=5, steps=1, side=16, name=cfg)
        comp = wl.comp
        a = comp.box_length / 16
        opts = b2.ForceFieldOptions(cutoff=3 * a)  # lattice shells sit on rmax
        idx = np.arange(4096)
        pos = np.column_stack([idx // 256, (idx // 16) % 16, idx % 16]) * a + 0.5 * a
        orient = wl.states[0].orient
    else:
        wl = configs.make(cfg)
        comp, opts = wl.comp, wl.opts
        pos, orient = wl.states[0].pos, wl.states[0].orient
    variants = _search_variants(comp, opts, pos, orient)
    ref_pairs = pyoracle.OracleFF(comp, opts).pair_list(pos)
    for pairs, f, t in variants:
        assert np.array_equal(pairs, ref_pairs)
        check_vec(f, variants[2][1], 1e-12, "force")
        check_vec(t, variants[2][2], 1e-12, "torque")


def test_tile_cull_after_steps():
    """Culling on a state the integrator moved (arcs from the device-written
    fixed-point positions) keeps the pair list exact."""
    wl = configs.make("cfg3")
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(wl.states[0])
    eng.step(50)
    s = eng.state()
    assert np.array_equal(eng.pair_list(), pyoracle.OracleFF(wl.comp, wl.opts).pair_list(s.pos))


# ------------------------------------------------------- spatial ordering
@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_spatial_order_evaluation(cfg):
    """Sorted (default) and input-order evaluations: identical pair lists
    (the oracle's), forces/torques/energies equal to summation order."""
    wl = configs.make(cfg)
    st0 = wl.states[0]
    out = []
    for interval in (100, 0):
        ff = b2.ForceField(wl.comp, wl.opts)
        ff.set_sort_interval(interval)
        st = st0.copy()
        ff.evaluate(st)
        out.append((ff.pair_list(), st))
    ref = pyoracle.OracleFF(wl.comp, wl.opts).evaluate(st0.pos, st0.orient)
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][0], pyoracle.OracleFF(wl.comp, wl.opts).pair_list(st0.pos))
    for _, st in out:
        check_vec(st.force, ref["force"], F_TOL, "force")
        check_vec(st.torque, ref["torque"], F_TOL, "torque")
        check_energy(st.energy, ref["energy"], st.virial, ref["virial"])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2_small", "cfg3"])
def test_spatial_order_resorts_during_steps(cfg):
    """Re-sorts every 7 steps (eager steps between graph launches) keep the
    trajectory on the oracle's, the pair list exact and the heat flux right."""
    if cfg == "cfg2_small":
        comp, opts, st = golden_cases.eval_cases()["water_ions"]
        wl = None
        dt, steps = 0.0005, 30
        st = st.copy()
        rng = np.random.default_rng(3)
        st.vel = rng.normal(scale=0.05, size=(comp.molecule_count(), 3))
        st.ang_vel = rng.normal(scale=0.05, size=(comp.molecule_count(), 3))
    else:
        wl = configs.make(cfg)
        comp, opts, st, dt = wl.comp, wl.opts, wl.states[0], wl.dt
        steps = 30
    chunks, interval = (1, 1, 5, 9, 14), 7  # single-step graphs and multi-step runs
    if cfg == "cfg3":  # the O(N^2) oracle step is ~1 s here
        chunks, interval, steps = (1, 4, 7), 3, 12
    eng = b2.Engine(comp, opts, dt)
    eng.set_sort_interval(interval)
    eng.set_state(st)
    for chunk in chunks:
        eng.step(chunk)
    s = eng.state()
    ora = pyoracle.OracleFF(comp, opts)
    o = ora.run(dt, steps, st.pos, st.orient, st.vel, st.ang_vel)
    L = comp.box_length
    d = s.pos - o["pos"]
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= T_TOL
    assert np.array_equal(eng.pair_list(), ora.pair_list(s.pos))
    h = np.linspace(-1.0, 1.0, len(comp.species))
    check_vec(eng.heat_flux(h), ora.heat_flux(s.pos, s.orient, s.vel, s.ang_vel, h), 1e-10, "jq")


def test_spatial_order_replicas():
    wl = configs.make("cfg4", replicas=3, steps=12)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=3)
    eng.set_sort_interval(5)
    eng.set_state(wl.states)
    eng.step(12)
    ora = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, s in enumerate(eng.states()):
        st = wl.states[r]
        o = ora.run(wl.dt, 12, st.pos, st.orient, st.vel, st.ang_vel)
        d = s.pos - o["pos"]
        d -= wl.comp.box_length * np.round(d / wl.comp.box_length)
        assert np.abs(d).max() / wl.comp.box_length <= T_TOL
        assert np.array_equal(eng.pair_list(r), ora.pair_list(s.pos))


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_fused_kick_bit_identical(cfg):
    """The end-of-step half kick in the force kernel's epilogue (single-step
    graphs, multi-step graphs, eager re-sort steps) gives the separate-kernel
    trajectory bit for bit (cfg2 has an Ewald term: never fused)."""
    wl = configs.make(cfg)
    out = []
    for fused in (True, False):
        eng = b2.Engine(wl.comp, wl.opts, wl.dt)
        eng.set_step_options(fused)
        eng.set_sort_interval(4 if cfg == "cfg3" else 0)
        eng.set_state(wl.states[0])
        for k in (1, 1, 6, 3):
            eng.step(k)
        s = eng.state()
        out.append(np.hstack([s.pos, s.orient, s.vel, s.ang_vel, s.force, s.torque]))
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3"])
def test_pinned_and_pageable_transfers_agree(cfg):
    """b2md_upload_state / b2md_get_state: 16-byte-aligned pinned host
    buffers take the one-launch zero-copy path, pageable and unaligned pinned
    ones the staged copies; same bits."""
    import torch
    wl = configs.make(cfg)
    st = wl.states[0]
    n = wl.comp.molecule_count()

    def pinned(a, offset):
        a = np.ascontiguousarray(a)
        raw = torch.empty(a.size + 1, dtype=torch.float64, pin_memory=True).numpy()
        v = raw[offset:offset + a.size].reshape(a.shape)
        v[...] = a
        return v

    outs = []
    for mode in ("pinned", "pinned_unaligned", "pageable"):
        eng = b2.Engine(wl.comp, wl.opts, wl.dt)
        eng.set_state(st)
        mk = {"pinned": lambda a: pinned(a, 0), "pinned_unaligned": lambda a: pinned(a, 1),
              "pageable": lambda a: np.ascontiguousarray(a).copy()}[mode]
        bufs = [mk(x) for x in (st.pos, st.orient, st.vel, st.ang_vel, np.zeros((n, 3)), np.zeros((n, 3)))]
        assert all((b.ctypes.data % 16 != 0) == (mode == "pinned_unaligned") for b in bufs)
        eng.get_state_raw(*bufs)
        for k in range(3):
            eng.upload_state_raw(*bufs)
            if k == 1:
                eng.step_async(1)
            else:
                eng.step(1)
            eng.get_state_raw(*bufs)
        outs.append(np.hstack([np.array(b) for b in bufs]))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


# ------------------------------------------ once-per-pair cluster walk (Newton)
# k_nl_count/scan/fill/inrec + k_force_nl + k_nl_reduce (csrc/cluster.cuh): each
# pair evaluated once from a cluster-pair list with a skin, partner
# contributions through the per-pair record buffer and a fixed-order
# reduction (B2MD_NEWTON=1, the default; the env pins it for these cases).
@pytest.mark.parametrize("n", [1, 2, 7, 9, 100, 1537, 4100])
def test_newton_walk_sizes(monkeypatch, n):
    monkeypatch.setenv("B2MD_CLUSTER", "2")
    monkeypatch.setenv("B2MD_NEWTON", "1")
    box = (n / 0.7) ** (1.0 / 3.0) if n > 8 else 8.0
    rc = min(2.5, 0.5 * box)
    if n > 8:
        wl = configs.lj_fluid_config(n, n / box ** 3, rc, seed=n + 3)
        comp, opts, st = wl.comp, wl.opts, wl.states[0]
    else:
        comp, opts = systems.lj_fluid(n, box), systems.lj_opts(rc)
        st = systems.random_state(comp, n, 0.9)
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(comp, opts, st.pos, st.orient)
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    assert ff.last_stats.com_pairs == ref["com_pairs"]


@pytest.mark.parametrize("n", [300, 2053])
def test_newton_walk_mixture_and_trajectory(monkeypatch, n):
    """Two species (Lorentz-Berthelot terms) and a 25-step trajectory with
    re-sorts on the once-per-pair walk; repeated runs are bit-identical."""
    monkeypatch.setenv("B2MD_CLUSTER", "2")
    monkeypatch.setenv("B2MD_NEWTON", "1")
    na = n // 3
    box = (n / 0.7) ** (1.0 / 3.0)
    comp = b2.SystemComposition([b2.build_species("a", [b2.make_lj_site(0, 0, 0, 1.0, 1.0, 1.0)]),
                                 b2.build_species("b", [b2.make_lj_site(0, 0, 0, 0.9, 1.3, 2.0)])],
                                [na, n - na], box, 1.0)
    opts = systems.lj_opts(min(2.5, 0.45 * box))
    st = systems.random_state(comp, n, 0.8)
    o = pyoracle.OracleFF(comp, opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(comp, opts, st.pos, st.orient)
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    dt, steps = 0.002, 25
    runs = []
    for _ in range(2):
        eng = b2.Engine(comp, opts, dt)
        eng.set_sort_interval(7)
        eng.set_state(st)
        eng.step(steps)
        runs.append(eng.state())
    tr = o.run(dt, steps, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(runs[0], tr, box)
    assert np.array_equal(runs[0].pos, runs[1].pos) and np.array_equal(runs[0].force, runs[1].force)


def test_newton_walk_replicas_and_cfg3(monkeypatch):
    """Replicas (short last clusters) and cfg3 itself on the once-per-pair
    walk: per-replica oracle forces / energies / pair counts, then cfg3's
    100-step trajectory against the reference engine's golden states."""
    monkeypatch.setenv("B2MD_NEWTON", "1")
    wls = [configs.lj_fluid_config(1001, 0.8, 2.5, seed=21 + r) for r in range(3)]
    comp, opts = wls[0].comp, wls[0].opts
    eng = b2.Engine(comp, opts, 0.005, replicas=3)
    eng.set_state([w.states[0] for w in wls])
    outs, stats = eng.states(), eng.energies()[1]
    o = pyoracle.OracleFF(comp, opts)
    for r, w in enumerate(wls):
        ref = o.evaluate(w.states[0].pos, w.states[0].orient)
        check_vec(outs[r].force, ref["force"], what=f"replica {r}")
        check_energy(outs[r].energy, ref["energy"], outs[r].virial, ref["virial"])
        assert stats[r].com_pairs == ref["com_pairs"]
    g = np.load(GOLDEN / "traj_cfg3_100.npz")
    wl = configs.make("cfg3")
    e3 = b2.Engine(wl.comp, wl.opts, wl.dt)
    e3.set_state(wl.states[0])
    e3.step(int(g["steps"]))
    out = e3.state()
    k, L = int(g["stride"]), wl.comp.box_length
    d = out.pos[::k] - g["pos"]
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= T_TOL
    assert abs(out.energy.total() - g["energy"][2]) <= T_TOL * abs(g["energy"][2])


@pytest.mark.parametrize("mode", ["stale", "both_rows", "every_step", "wide_skin", "rebuild_each_step"])
def test_cluster_walk_modes(monkeypatch, mode):
    """The list's exactness guard and schedule: skin 0 makes every list stale
    after the first drift (the exact per-step walk runs instead), the
    both-rows walk, per-step drift checks with a thin skin and frequent
    re-sorts, a wide skin (long lists: the per-step arc cull keeps the pair
    work), and a rebuild at every step.  Each: forces, energies and the pair
    count against the oracle, a 30-step trajectory with re-sorts against the
    oracle's Engine::step (src/engine.cpp:102-143), bit-identical repeats."""
    env = {"stale": {"B2MD_NEWTON": "1", "B2MD_NL_SKIN": "0"},
           "both_rows": {"B2MD_NEWTON": "0"},
           "every_step": {"B2MD_NEWTON": "1", "B2MD_NL_SKIN": "0.05", "B2MD_NL_INTERVAL": "0"},
           "wide_skin": {"B2MD_NEWTON": "1", "B2MD_NL_SKIN": "2.5", "B2MD_NL_INTERVAL": "0"},
           "rebuild_each_step": {"B2MD_NEWTON": "1", "B2MD_NL_INTERVAL": "1"}}[mode]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("B2MD_CLUSTER", "2")
    wl = configs.lj_fluid_config(4100, 0.8, 2.5, seed=17, temperature=2.0)
    st = wl.states[0]
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    ref = o.evaluate(st.pos, st.orient)
    ff, out = gpu_eval(wl.comp, wl.opts, st.pos, st.orient)
    check_vec(out.force, ref["force"])
    check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
    assert ff.last_stats.com_pairs == ref["com_pairs"]
    runs = []
    for _ in range(2):
        eng = b2.Engine(wl.comp, wl.opts, 0.005)
        eng.set_sort_interval(13)
        eng.set_state(st)
        eng.step(30)
        runs.append((eng.state(), eng.energies()[1][0].com_pairs))
    tr = o.run(0.005, 30, st.pos, st.orient, st.vel, st.ang_vel)
    compare_states(runs[0][0], tr, wl.comp.box_length)
    check_energy(runs[0][0].energy, tr["energy"], runs[0][0].virial, tr["virial"])
    assert runs[0][1] == o.evaluate(runs[0][0].pos, runs[0][0].orient)["com_pairs"]
    assert np.array_equal(runs[0][0].pos, runs[1][0].pos)
    assert np.array_equal(runs[0][0].force, runs[1][0].force)


@pytest.mark.parametrize("tiled", ["0", "1"])
def test_ewald_forms_cfg2(monkeypatch, tiled):
    """Both reciprocal-space forms (per-(k, charge) table gathers, and the
    shared-memory tiled S(k) / force kernels of B2MD_EWALD_TILED=1) against the
    oracle on cfg2 (ewald.cpp:107-180): forces, torques, energies; repeated
    evaluations bit-identical."""
    monkeypatch.setenv("B2MD_EWALD_TILED", tiled)
    wl = configs.make("cfg2")
    st = wl.states[0]
    ref = pyoracle.OracleFF(wl.comp, wl.opts).evaluate(st.pos, st.orient)
    outs = [gpu_eval(wl.comp, wl.opts, st.pos, st.orient)[1] for _ in range(2)]
    check_vec(outs[0].force, ref["force"])
    check_vec(outs[0].torque, ref["torque"])
    check_energy(outs[0].energy, ref["energy"], outs[0].virial, ref["virial"])
    assert np.array_equal(outs[0].force, outs[1].force)
    assert outs[0].energy.total() == outs[1].energy.total()


def test_ewald_steps_cfg2(monkeypatch):
    """Engine::step with an Ewald term (src/engine.cpp:102-143 over
    src/ewald.cpp:107-180): in the step paths the reciprocal forces are computed
    beside the real-space kernel and added by the end-of-step kick
    (B2MD_EWALD_OVERLAP, the default); =0 adds them in place after it.  Both:
    single-step and multi-step calls against the oracle's trajectory, forces /
    torques / energies of the final state against the oracle's evaluation of it;
    and the two forms bit-identical (the same single addition per component)."""
    wl = configs.make("cfg2")
    st = wl.states[0]
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    calls = (1, 1, 4, 3)
    tr = o.run(wl.dt, sum(calls), st.pos, st.orient, st.vel, st.ang_vel)
    outs = []
    for overlap in ("1", "0"):
        monkeypatch.setenv("B2MD_EWALD_OVERLAP", overlap)
        eng = b2.Engine(wl.comp, wl.opts, wl.dt)
        eng.set_state(st)
        for k in calls:
            eng.step(k)
        out = eng.state()
        compare_states(out, tr, wl.comp.box_length)
        ref = o.evaluate(out.pos, out.orient)
        check_vec(out.force, ref["force"], what="force")
        check_vec(out.torque, ref["torque"], what="torque")
        check_energy(out.energy, ref["energy"], out.virial, ref["virial"])
        outs.append(np.hstack([out.pos, out.orient, out.vel, out.ang_vel, out.force, out.torque]))
    assert np.array_equal(outs[0], outs[1])

