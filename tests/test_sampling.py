"""CPU: scalar sampling (engine.cpp:218-229) and the thermostat oracle.

The host restatements of tmd::DerivativeAccumulator (massieu.cpp:9-70,
148-190) and BlockStat::add (results.hpp:30-37) serialize to the bytes the
reference writes for the same samples (tests/golden/sampling.npz); the
oracle's kinetic energies and apply_thermostat (engine.cpp:145-160) are
bit-exact against the reference when oracle/_ref is built."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle
from host_checkpoint import BlockStat, ByteReader, ByteWriter
from host_sampling import DerivativeAccumulator
from paper_1507_07548_b200 import configs

G = np.load(Path(__file__).resolve().parent / "golden" / "sampling.npz")
needs_ref = pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("k", range(5))
def test_derivative_accumulator_bytes(k):
    nb, expected, _ = (int(v) for v in G["cases"][k])
    a = DerivativeAccumulator.create(1.5, 812.0, 256, nb, expected)
    for u, uv, uvv in G[f"da_{k}_samples"]:
        a.add(float(u), float(uv), float(uvv))
    w = ByteWriter()
    a.serialize(w)
    assert w.data() == G[f"da_{k}_bytes"].tobytes()
    back = DerivativeAccumulator.deserialize(ByteReader(w.data()))
    assert back == a


@pytest.mark.parametrize("k", range(5))
def test_block_stat_add_bytes(k):
    nb, expected, _ = (int(v) for v in G["cases"][k])
    b = BlockStat.fresh(nb, expected)
    for x in G[f"bs_{k}_x"]:
        b.add(float(x))
    w = ByteWriter()
    b.serialize(w)
    assert w.data() == G[f"bs_{k}_bytes"].tobytes()


def test_derivative_accumulator_errors():
    from paper_1507_07548_b200 import ConfigError, NumericalError
    with pytest.raises(ConfigError, match="bad state constants"):
        DerivativeAccumulator.create(0.0, 1.0, 10)
    a = DerivativeAccumulator.create(1.0, 1.0, 10)
    with pytest.raises(NumericalError, match="non-finite snapshot"):
        a.add(float("nan"), 0.0, 0.0)


@needs_ref
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_oracle_thermostat_bitexact_vs_reference(cfg):
    wl = configs.make(cfg)
    st = wl.states[0]
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    r = pyoracle.RefFF(wl.comp, wl.opts)
    assert np.array_equal(o.kinetic_energy(st.vel, st.ang_vel), r.kinetic_energy(st.vel, st.ang_vel))
    e = pyoracle.RefEngine(wl.comp, wl.opts, wl.dt)
    e.set_state(st.pos, st.orient, st.vel * 1.3, st.ang_vel * 0.7)
    e.apply_thermostat()
    s = e.state()
    v, w = o.apply_thermostat(st.vel * 1.3, st.ang_vel * 0.7)
    assert np.array_equal(v, s["vel"]) and np.array_equal(w, s["ang_vel"])


def test_oracle_thermostat_zero_energy_messages():
    wl = configs.make("cfg1")
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    n = wl.comp.molecule_count()
    with pytest.raises(pyoracle.OracleError, match="zero translational kinetic energy"):
        o.apply_thermostat(np.zeros((n, 3)), np.ones((n, 3)))
    with pytest.raises(pyoracle.OracleError, match="zero rotational kinetic energy"):
        o.apply_thermostat(np.ones((n, 3)), np.zeros((n, 3)))
