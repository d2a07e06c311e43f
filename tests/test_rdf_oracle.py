"""CPU: pins the RDF checker and the host-side RDF arithmetic to the
reference's tmd::RdfHistogram (src/structure.cpp).

(1) the oracle's counts (oracle_rdf_*, tmd_oracle.c) bit-exact against the
golden vectors written by the unmodified reference and, when oracle/_ref is
built, against the reference at BASELINE sizes; (2) the package's finalize /
serialize / first_minimum / solvation_number restatements
(paper_1507_07548_b200/structure.py) bit-exact against the reference's
outputs on the same counts; (3) known answers of tests/test_structure.cpp."""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle
from paper_1507_07548_b200 import (
    SystemComposition,
    build_species,
    configs,
    make_charge_site,
    make_lj_site,
    rdf_site_types,
    serialize_counts,
)
from host_rdf import finalize_tables, first_minimum, solvation_number

import golden_cases

GOLDEN = Path(__file__).resolve().parent / "golden"
EVAL_CASES = golden_cases.eval_cases()
needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")


def flatten(tables):
    if not tables:
        return np.zeros(0)
    return np.concatenate([np.concatenate([[t.species_a, t.species_b, t.partner_density, t.bin_width,
                                            t.snapshots, len(t.g)],
                                           np.column_stack([t.r_mid, t.g, t.n_cum]).ravel()])
                           for t in tables])


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_oracle_rdf_counts_bitexact_vs_golden(name):
    comp, opts, _ = EVAL_CASES[name]
    g = np.load(GOLDEN / f"rdf_{name}.npz")
    o = pyoracle.OracleRdf(pyoracle.OracleFF(comp, opts), float(g["bin_width"]), float(g["r_max"]))
    for pos, orient in zip(g["pos"], g["orient"]):
        o.accumulate(pos, orient)
    counts, snaps = o.counts()
    assert snaps == int(g["snapshots"])
    assert np.array_equal(counts, g["counts"])


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_host_rdf_arithmetic_bitexact_vs_golden(name):
    comp, _, _ = EVAL_CASES[name]
    g = np.load(GOLDEN / f"rdf_{name}.npz")
    bw, rmax, counts, snaps = float(g["bin_width"]), float(g["r_max"]), g["counts"], int(g["snapshots"])
    tables = finalize_tables(comp, rdf_site_types(comp), bw, rmax, counts, snaps)
    assert np.array_equal(flatten(tables), g["finalize"])
    bins = int(math.ceil(rmax / bw))
    assert serialize_counts(bw, rmax, bins, snaps, counts) == g["serialized"].tobytes()
    fm = np.array([first_minimum(t.r_mid, t.g) for t in tables])
    assert np.array_equal(fm, g["first_minimum"], equal_nan=True)
    sv = np.array([solvation_number(t, t.partner_density, 0.6 * rmax) for t in tables])
    assert np.array_equal(sv, g["solvation_number"])


@needs_ref
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_oracle_rdf_bitexact_vs_reference_at_baseline_sizes(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    L = wl.comp.box_length
    o = pyoracle.OracleRdf(pyoracle.OracleFF(wl.comp, wl.opts), L / 200, 0.5 * L)
    r = pyoracle.RefRdf(pyoracle.RefFF(wl.comp, wl.opts), L / 200, 0.5 * L)
    o.accumulate(st.pos, st.orient)
    r.accumulate(st.pos, st.orient)
    assert np.array_equal(o.counts()[0], r.counts()[0])


def lj_fluid(n, box):
    return SystemComposition([build_species("lj", [make_lj_site(0, 0, 0, 1, 1, 1)])], [n], box, 1.0)


def test_two_molecules_single_count():  # test_structure.cpp:10-32
    comp = lj_fluid(2, 10.0)
    ff = pyoracle.OracleFF(comp, _opts(2.5))
    h = pyoracle.OracleRdf(ff, 0.05, 5.0)
    h.accumulate(np.array([[2.0, 2, 2], [2.0, 2, 3.234]]), np.tile([1.0, 0, 0, 0], (2, 1)))
    counts, snaps = h.counts()
    assert counts.sum() == 1 and counts[0, int(1.234 / 0.05)] == 1
    t = finalize_tables(comp, rdf_site_types(comp), 0.05, 5.0, counts, snaps)[0]
    assert t.n_cum[-1] == pytest.approx(1.0)


def test_intramolecular_pairs_excluded():  # test_structure.cpp:34-49
    sp = build_species("dimer", [make_lj_site(0.4, 0, 0, 1, 1, 1), make_lj_site(-0.4, 0, 0, 1, 1, 1)])
    comp = SystemComposition([sp], [1], 8.0, 1.0)
    h = pyoracle.OracleRdf(pyoracle.OracleFF(comp, _opts(2.5)), 0.02, 4.0)
    h.accumulate(np.array([[4.0, 4, 4]]), np.array([[1.0, 0, 0, 0]]))
    assert h.counts()[0].sum() == 0


def test_charge_sites_are_not_sampling_centres():  # test_structure.cpp:251-261
    sp = build_species("ion_pair", [make_charge_site(0.2, 0, 0, 0.5, 1.0),
                                    make_charge_site(-0.2, 0, 0, -0.5, 1.0),
                                    make_lj_site(0, 0, 0, 1, 1, 1)])
    comp = SystemComposition([sp], [4], 8.0, 1.0)
    assert len(rdf_site_types(comp)) == 1
    from paper_1507_07548_b200 import ElectrostaticsMethod, ForceFieldOptions
    opts = ForceFieldOptions(cutoff=2.5, method=ElectrostaticsMethod.reaction_field, eps_rf=10.0)
    h = pyoracle.OracleRdf(pyoracle.OracleFF(comp, opts), 0.05, 4.0)
    assert h.n_types == 1


def test_rdf_validation():  # test_structure.cpp:263-269
    comp = lj_fluid(10, 6.0)
    ff = pyoracle.OracleFF(comp, _opts(2.5))
    for bw, rmax in ((0.0, 3.0), (0.02, 3.5)):
        with pytest.raises(pyoracle.OracleError) as ei:
            pyoracle.OracleRdf(ff, bw, rmax)
        assert ei.value.code == 2
    with pytest.raises(Exception, match="no snapshots"):
        finalize_tables(comp, rdf_site_types(comp), 0.02, 3.0, np.zeros((1, 150), np.uint64), 0)


def test_first_minimum_and_solvation_closed_forms():  # test_structure.cpp:131-165
    r = [0.02 * (i + 0.5) for i in range(150)]
    g = [1.0 + 1.8 * math.exp(-30.0 * (x - 1.1) ** 2) - 0.6 * math.exp(-25.0 * (x - 1.6) ** 2) for x in r]
    assert first_minimum(r, g) == pytest.approx(1.6, rel=0.02 / 1.6 + 0.02)
    assert math.isnan(first_minimum(r, [1.0] * 150))
    from host_rdf import RdfTable
    t = RdfTable(bin_width=0.05, g=[1.0] * 100)
    assert solvation_number(t, 0.7, 1.5) == pytest.approx(4.0 / 3.0 * math.pi * 0.7 * 1.5 ** 3, rel=1e-12)
    t.g = [0.0] * 100
    assert solvation_number(t, 0.7, 1.5) == 0.0


def _opts(rc):
    from paper_1507_07548_b200 import ForceFieldOptions
    return ForceFieldOptions(cutoff=rc)
