"""GPU parity of the RDF histograms (b2md_rdf_*, csrc/rdf.cuh) against the
reference's golden vectors, the oracle (oracle_rdf_*, pinned bit-exact to
tmd::RdfHistogram) and the known answers of tests/test_structure.cpp.

Counts are integers: the bar is bit-exact (and so are finalize and the
serialized bytes, which are host arithmetic on the counts)."""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

import host_rdf

import golden_cases
from test_rdf_oracle import flatten, lj_fluid

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def finalize(h, replica=0):
    """The device counts through the reference's finalize arithmetic
    (structure.cpp:78-128; tests/host_rdf.py, pinned to the reference)."""
    counts, snaps = h.counts(replica)
    return host_rdf.finalize_tables(h.comp, h.types, h.bin_width, h.r_max, counts, snaps)


def state_of(comp, pos, orient):
    st = b2.SystemState(comp.molecule_count(), comp.box_length)
    st.pos, st.orient = np.array(pos, dtype=np.float64), np.array(orient, dtype=np.float64)
    return st


@pytest.mark.parametrize("name", list(golden_cases.eval_cases()))
def test_golden_rdf(name):
    comp, opts, _ = golden_cases.eval_cases()[name]
    g = np.load(GOLDEN / f"rdf_{name}.npz")
    ff = b2.ForceField(comp, opts)
    h = b2.RdfHistogram(ff, float(g["bin_width"]), float(g["r_max"]))
    for pos, orient in zip(g["pos"], g["orient"]):
        h.accumulate(state_of(comp, pos, orient))
    counts, snaps = h.counts()
    assert snaps == int(g["snapshots"])
    assert np.array_equal(counts, g["counts"])
    if int(g["counts"].size):
        assert np.array_equal(flatten(finalize(h)), g["finalize"])
    assert h.serialize() == g["serialized"].tobytes()


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_rdf_baseline_configs(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    L = wl.comp.box_length
    h = b2.RdfHistogram(b2.ForceField(wl.comp, wl.opts), L / 300, 0.5 * L)
    h.accumulate(st)
    o = pyoracle.OracleRdf(pyoracle.OracleFF(wl.comp, wl.opts), L / 300, 0.5 * L)
    o.accumulate(st.pos, st.orient)
    assert np.array_equal(h.counts()[0], o.counts()[0])


def test_rdf_global_atomic_path():
    """A histogram too large for shared memory (pairs x bins > 12288) takes
    the global-atomic kernel: same counts."""
    comp, opts, st = golden_cases.eval_cases()["mixture"]
    L = comp.box_length
    bw = L / 6000
    h = b2.RdfHistogram(b2.ForceField(comp, opts), bw, 0.5 * L)
    assert h._pairs * h.bins() > 12 * 1024
    h.accumulate(st)
    o = pyoracle.OracleRdf(pyoracle.OracleFF(comp, opts), bw, 0.5 * L)
    o.accumulate(st.pos, st.orient)
    assert np.array_equal(h.counts()[0], o.counts()[0])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg3"])
def test_rdf_of_engine_state(cfg):
    """b2md_rdf_accumulate on the resident state after steps (the engine's
    sampler, engine.cpp:259 / 294) equals the oracle on the downloaded state."""
    wl = configs.make(cfg)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt)
    eng.set_state(wl.states[0])
    L = wl.comp.box_length
    h = b2.RdfHistogram(eng, L / 250, 0.5 * L)
    o = pyoracle.OracleRdf(pyoracle.OracleFF(wl.comp, wl.opts), L / 250, 0.5 * L)
    for _ in range(2):
        eng.step(5)
        h.accumulate()
        s = eng.state()
        o.accumulate(s.pos, s.orient)
    assert np.array_equal(h.counts()[0], o.counts()[0])
    assert h.snapshots() == 2


def test_rdf_replicas():
    wl = configs.make("cfg4", replicas=3, steps=4)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=3)
    eng.set_state(wl.states)
    eng.step(4)
    L = wl.comp.box_length
    h = b2.RdfHistogram(eng, 0.05, 0.5 * L)
    h.accumulate()
    ora = pyoracle.OracleFF(wl.comp, wl.opts)
    for r, s in enumerate(eng.states()):
        o = pyoracle.OracleRdf(ora, 0.05, 0.5 * L)
        o.accumulate(s.pos, s.orient)
        assert np.array_equal(h.counts(r)[0], o.counts()[0])


def test_rdf_serialize_round_trip():  # structure.cpp:130-153
    comp, opts, st = golden_cases.eval_cases()["two_clj"]
    ff = b2.ForceField(comp, opts)
    L = comp.box_length
    a = b2.RdfHistogram(ff, 0.05, 0.5 * L)
    a.accumulate(st)
    a.accumulate(st)
    data = a.serialize()
    b = b2.RdfHistogram(ff, 0.05, 0.5 * L)
    assert b.deserialize(data) == len(data)
    assert np.array_equal(a.counts()[0], b.counts()[0]) and b.snapshots() == 2
    b.accumulate(st)
    assert np.array_equal(b.counts()[0], 3 * (a.counts()[0] // 2))
    with pytest.raises(b2.IoError):
        b.deserialize(data[:-3])


# ---- known answers of tests/test_structure.cpp on the GPU path
def test_single_pair_bin():  # :10-32
    comp = lj_fluid(2, 10.0)
    h = b2.RdfHistogram(b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.5)), 0.05, 5.0)
    h.accumulate(state_of(comp, [[2.0, 2, 2], [2.0, 2, 3.234]], [[1.0, 0, 0, 0]] * 2))
    t = finalize(h)[0]
    nz = [b for b, g in enumerate(t.g) if g > 0.0]
    assert nz == [int(1.234 / 0.05)]
    assert t.n_cum[-1] == pytest.approx(1.0)


def test_fcc_first_shell_twelve_neighbours():  # :51-76
    a, cells = 1.5, 4
    base = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]])
    pos = np.array([(np.array([i, j, k]) + b) * a for i in range(cells) for j in range(cells)
                    for k in range(cells) for b in base]) + 0.01
    comp = lj_fluid(len(pos), a * cells)
    h = b2.RdfHistogram(b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.0)), 0.02,
                        0.5 * comp.box_length)
    h.accumulate(state_of(comp, pos, [[1.0, 0, 0, 0]] * len(pos)))
    t = finalize(h)[0]
    first = next(b for b, g in enumerate(t.g) if g > 0.0)
    assert abs(first - int(a / math.sqrt(2.0) / 0.02)) <= 1
    assert t.n_cum[first] == pytest.approx(12.0, rel=1e-12)


def test_ideal_gas_and_counting_identities():  # :79-101, :147-217
    n, L = 500, 7.937
    comp = lj_fluid(n, L)
    ff = b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.5))
    h = b2.RdfHistogram(ff, 0.05, 0.5 * L)
    rng = np.random.default_rng(41)
    direct = 0.0
    for _ in range(400):
        pos = rng.uniform(0, L, size=(n, 3))
        h.accumulate(state_of(comp, pos, np.tile([1.0, 0, 0, 0], (n, 1))))
    t = finalize(h)[0]
    for r, g in zip(t.r_mid, t.g):
        if 0.2 * 0.5 * L <= r <= 0.5 * L:
            assert g == pytest.approx(1.0, rel=0.02)
    # n_cum / solvation_number == direct neighbour counting (small system)
    n, L = 120, 6.0
    comp = lj_fluid(n, L)
    h = b2.RdfHistogram(b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.5)), 0.05, 3.0)
    rng = np.random.default_rng(9)
    for _ in range(25):
        pos = rng.uniform(0, L, size=(n, 3))
        h.accumulate(state_of(comp, pos, np.tile([1.0, 0, 0, 0], (n, 1))))
        d = pos[:, None, :] - pos[None, :, :]
        d -= L * np.round(d / L)
        r = np.sqrt((d * d).sum(-1))
        direct += float(((r < 1.5) & (r > 0)).sum())
    direct /= 25 * n
    t = finalize(h)[0]
    assert host_rdf.solvation_number(t, t.partner_density, 1.5) == pytest.approx(direct, rel=1e-10)
    assert t.n_cum[int(1.5 / 0.05) - 1] == pytest.approx(direct, rel=1e-10)


def test_dummy_and_charge_sites():  # :219-261
    sp = b2.build_species("mol", [b2.make_lj_site(0, 0, 0, 1, 1, 1),
                                  b2.Site(b2.SiteKind.dummy, (0.3, 0, 0), 0.0, 0.0, 0.0, 0.0)])
    comp = b2.SystemComposition([sp], [20], 6.0, 1.0)
    h = b2.RdfHistogram(b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.5)), 0.05, 3.0)
    assert h.site_type_count() == 2
    rng = np.random.default_rng(6)
    q = rng.normal(size=(20, 4))
    h.accumulate(state_of(comp, rng.uniform(0, 6, size=(20, 3)), q / np.linalg.norm(q, axis=1)[:, None]))
    assert len(finalize(h)) == 3
    ion = b2.build_species("ion_pair", [b2.make_charge_site(0.2, 0, 0, 0.5, 1.0),
                                        b2.make_charge_site(-0.2, 0, 0, -0.5, 1.0),
                                        b2.make_lj_site(0, 0, 0, 1, 1, 1)])
    comp = b2.SystemComposition([ion], [4], 8.0, 1.0)
    opts = b2.ForceFieldOptions(cutoff=2.5, method=b2.ElectrostaticsMethod.reaction_field, eps_rf=10.0)
    assert b2.RdfHistogram(b2.ForceField(comp, opts), 0.05, 4.0).site_type_count() == 1


def test_rdf_validation():  # :263-269
    comp = lj_fluid(10, 6.0)
    ff = b2.ForceField(comp, b2.ForceFieldOptions(cutoff=2.5))
    for bw, rmax in ((0.0, 3.0), (0.02, 3.5)):
        with pytest.raises(b2.ConfigError):
            b2.RdfHistogram(ff, bw, rmax)
    with pytest.raises(b2.Error, match="no snapshots"):
        finalize(b2.RdfHistogram(ff, 0.02, 3.0))
