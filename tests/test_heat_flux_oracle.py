"""CPU: pins the heat-flux oracle (oracle_heat_flux, tmd_oracle.c) to the
reference tmd::heat_flux (src/greenkubo.cpp:182-266).

(1) bit-exact against the golden vectors written by the unmodified reference
(tests/golden/flux_*.npz); (2) bit-exact against oracle/_ref at BASELINE
sizes when it is built; (3) the reference's own known answers: rest, ideal
gas and the independent double loop (tests/test_greenkubo.cpp:172-287), and
the ConfigError on a missing enthalpy (test_greenkubo.cpp:215)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle
from paper_1507_07548_b200 import configs

import flux_checks
import golden_cases

GOLDEN = Path(__file__).resolve().parent / "golden"
EVAL_CASES = golden_cases.eval_cases()
needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("name", list(EVAL_CASES))
def test_oracle_heat_flux_bitexact_vs_golden(name):
    comp, opts, _ = EVAL_CASES[name]
    g = np.load(GOLDEN / f"flux_{name}.npz")
    jq = pyoracle.OracleFF(comp, opts).heat_flux(g["pos"], g["orient"], g["vel"], g["ang_vel"], g["h"])
    assert np.array_equal(jq, g["jq"])


@needs_ref
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_oracle_heat_flux_bitexact_vs_reference_at_baseline_sizes(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    vel, ang_vel, h = golden_cases.flux_inputs(cfg, wl.comp)
    a = pyoracle.OracleFF(wl.comp, wl.opts).heat_flux(st.pos, st.orient, vel, ang_vel, h)
    b = pyoracle.RefFF(wl.comp, wl.opts).heat_flux(st.pos, st.orient, vel, ang_vel, h)
    assert np.array_equal(a, b)


def test_heat_flux_at_rest_is_zero():  # test_greenkubo.cpp:188-190
    comp, opts, st, _, _ = flux_checks.ideal_gas_case()
    st.vel[:] = 0.0
    st.ang_vel[:] = 0.0
    jq = pyoracle.OracleFF(comp, opts).heat_flux(st.pos, st.orient, st.vel, st.ang_vel, [0.0])
    assert np.linalg.norm(jq) < 1e-15


def test_heat_flux_ideal_gas_closed_form():  # test_greenkubo.cpp:192-213
    comp, opts, st, h, expected = flux_checks.ideal_gas_case()
    jq = pyoracle.OracleFF(comp, opts).heat_flux(st.pos, st.orient, st.vel, st.ang_vel, h)
    np.testing.assert_allclose(jq, expected, rtol=1e-12)


def test_heat_flux_matches_independent_double_loop():  # test_greenkubo.cpp:218-287
    comp, opts, st, h = flux_checks.dimer_case()
    jq = pyoracle.OracleFF(comp, opts).heat_flux(st.pos, st.orient, st.vel, st.ang_vel, h)
    ind = flux_checks.independent_flux(comp, opts.cutoff, st, h)
    # some pair must interact, or the check is vacuous
    ideal = flux_checks.independent_flux(comp, 1e-9, st, h)
    assert np.abs(ind - ideal).max() > 1e-3
    np.testing.assert_allclose(jq, ind, rtol=1e-12, atol=1e-12 * np.abs(ind).max())


def test_heat_flux_requires_one_enthalpy_per_species():  # greenkubo.cpp:184-185
    comp, opts, st, _, _ = flux_checks.ideal_gas_case()
    impls = [pyoracle.OracleFF] + ([pyoracle.RefFF] if pyoracle.ref_available() else [])
    for cls in impls:
        ff = cls(comp, opts)
        for h in (np.zeros(0), np.zeros(2)):
            with pytest.raises(pyoracle.OracleError) as ei:
                ff.heat_flux(st.pos, st.orient, st.vel, st.ang_vel, h)
            assert ei.value.code == 2  # B2MD_CONFIG_ERROR
            assert "enthalpy" in str(ei.value)
