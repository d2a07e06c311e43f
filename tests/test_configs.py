"""CPU: the seeded BASELINE workloads are deterministic and have the stated
shapes (BASELINE.json configs)."""
import math

import numpy as np
import pytest

from paper_1507_07548_b200 import configs, kinetic_energy_trans, translational_dof


def test_cfg0_shape_and_determinism():
    a = configs.make("cfg0")
    b = configs.make("cfg0")
    st = a.states[0]
    assert st.pos.shape == (1000, 3)
    assert a.comp.box_length == pytest.approx((1000 / 0.8) ** (1 / 3))
    assert a.opts.cutoff == pytest.approx(0.45 * a.comp.box_length)
    assert np.array_equal(st.pos, b.states[0].pos) and np.array_equal(st.vel, b.states[0].vel)
    assert np.all(st.pos >= 0) and np.all(st.pos < a.comp.box_length)
    assert np.allclose(st.vel.sum(axis=0), 0.0, atol=1e-12)
    assert kinetic_energy_trans(a.comp, st) == pytest.approx(0.5 * translational_dof(a.comp) * 1.0,
                                                            rel=1e-12)


def test_cfg1_and_cfg3_and_cfg4():
    c1 = configs.make("cfg1")
    assert c1.comp.molecule_count() == 2048 and c1.comp.species[0].rotational_dof == 2
    assert c1.comp.species[0].inertia_principal[1] == pytest.approx(0.0625)
    c3 = configs.make("cfg3")
    assert c3.comp.molecule_count() == 16384 and c3.opts.cutoff == 5.0
    assert c3.comp.box_length == pytest.approx(27.359615, rel=1e-6)
    c4 = configs.make("cfg4", replicas=3)
    assert c4.replicas == 3
    for st in c4.states:
        assert st.pos.shape == (1000, 3)
    assert not np.array_equal(c4.states[0].pos, c4.states[1].pos)


def test_cfg2_water_ions():
    c2 = configs.make("cfg2")
    assert c2.comp.counts == [1000, 50, 50]
    assert c2.comp.box_length * configs.SIGMA_REF_A == pytest.approx(32.67, abs=0.01)
    assert configs.Q_REDUCED == pytest.approx(25.9795, rel=1e-4)
    assert abs(sum(c * s.net_charge for s, c in zip(c2.comp.species, c2.comp.counts))) < 1e-9
    assert c2.opts.ewald.kmax == 7
