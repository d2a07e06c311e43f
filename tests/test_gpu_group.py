"""b2md_create_group: one process driving several GPUs (SURVEY.md 8(b) item 8,
8(e)) -- the single-process caller shape of tmd::Engine (src/engine.cpp:
100-143) over the row-sharded step (src/parallel.cpp:84-95's split, one packed
NCCL all-reduce per evaluation).

On one device the group is a plain context (rank 0 of 1): bit-identical to an
Engine.  With two or more visible devices the sharded group is checked against
the oracle (forces, energies, trajectories at the BASELINE tolerances); those
tests skip on a one-GPU box."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

pytestmark = pytest.mark.gpu
T_TOL = 1e-9


def n_devices():
    import torch
    return torch.cuda.device_count()


def _cases():
    return {
        "lj-cluster": configs.lj_fluid_config(2048, 0.8, 2.5, seed=5, steps=20, name="g-lj"),
        "lj-bitmatrix": configs.lj_fluid_config(500, 0.8, None, seed=4, steps=20, name="g-lj45"),
        "2clj": configs.two_clj_config(300, 0.3, 5, 2.0, 0.002, 20, "g-2clj"),
    }


@pytest.mark.parametrize("case", ["lj-cluster", "lj-bitmatrix", "2clj"])
def test_group_of_one_equals_engine(case):
    wl = _cases()[case]
    st = wl.states[0]
    g = b2.EngineGroup(wl.comp, wl.opts, wl.dt, devices=[0])
    assert g.size() == 1
    g.set_state(st)
    g.step(wl.steps)
    a = g.state()
    e = b2.Engine(wl.comp, wl.opts, wl.dt, device=0)
    e.set_state(st)
    e.step(wl.steps)
    b = e.state()
    for f in ("pos", "vel", "orient", "ang_vel", "force"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.energy.total() == b.energy.total()
    g.close()


@pytest.mark.parametrize("case", ["lj-cluster", "lj-bitmatrix", "2clj"])
def test_group_sharded_against_oracle(case):
    nd = n_devices()
    if nd < 2:
        pytest.skip("one CUDA device visible: the sharded group needs >= 2")
    wl = _cases()[case]
    st = wl.states[0]
    g = b2.EngineGroup(wl.comp, wl.opts, wl.dt, devices=list(range(min(nd, 4))))
    g.set_state(st)
    g.step(wl.steps)
    out = g.state()
    ref = pyoracle.OracleFF(wl.comp, wl.opts).run(wl.dt, wl.steps, st.pos, st.orient, st.vel,
                                                  st.ang_vel)
    L = wl.comp.box_length
    d = out.pos - ref["pos"]
    d -= L * np.round(d / L)
    assert np.abs(d).max() / L <= T_TOL
    assert np.abs(out.vel - ref["vel"]).max() / np.abs(ref["vel"]).max() <= T_TOL
    assert abs(out.energy.total() - ref["energy"].total()) <= T_TOL * abs(ref["energy"].total())
    # every rank holds the same replicated state after the all-reduce
    for e in g.engines[1:]:
        assert np.array_equal(e.state().pos, out.pos)
    g.close()


def test_group_bad_arguments():
    wl = _cases()["lj-bitmatrix"]
    with pytest.raises(b2.Error):
        b2.EngineGroup(wl.comp, wl.opts, wl.dt, devices=[n_devices() + 7])
