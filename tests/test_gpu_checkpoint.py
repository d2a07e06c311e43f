"""GPU: checkpoint / restart through the device state block
(b2md_save_state_block / b2md_restore_state_block) against checkpoints
written by the unmodified reference (tests/golden/ckpt.npz) and the oracle.

* a GPU engine after set_state writes the reference's bytes exactly;
* a restored reference checkpoint gives the file's state bit for bit, forces
  equal to the oracle's on it, and re-emits the same bytes;
* restart is bit-exact where the summation order is a function of the state
  alone (fixed spatial order, row / both-rows walks); with periodic re-sorting
  or the once-per-pair list (rebuilt from the restored positions) it agrees to
  rounding."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import configs

from host_checkpoint import EngineCheckpoint, checkpoint_bytes, restore_checkpoint

import golden_cases

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).resolve().parent / "golden" / "ckpt.npz")


def records(s: b2.SystemState) -> np.ndarray:
    return np.hstack([s.pos, s.orient, s.vel, s.ang_vel])


def test_fresh_engine_checkpoint_equals_reference():
    comp, opts, st = golden_cases.eval_cases()["two_clj"]
    eng = b2.Engine(comp, opts, 0.002)
    eng.set_state(st)
    meta = EngineCheckpoint.fresh(int(G["fresh_seed"]), n_blocks=10, n_production=0)
    assert checkpoint_bytes(eng, meta) == G["fresh_two_clj"].tobytes()


def test_restore_reference_checkpoint():
    comp, opts, _ = golden_cases.eval_cases()["water_ions"]
    data = G["sampled_water"].tobytes()
    eng = b2.Engine(comp, opts, 0.0005)
    meta = restore_checkpoint(eng, data)
    s = eng.state()
    assert np.array_equal(records(s), meta.state)  # restore does not wrap (engine.cpp:483-491)
    ref = pyoracle.OracleFF(comp, opts).evaluate(meta.state[:, 0:3], meta.state[:, 3:7])
    scale = max(1.0, np.abs(ref["force"]).max())
    assert np.abs(s.force - ref["force"]).max() <= 1e-10 * scale
    assert np.abs(s.torque - ref["torque"]).max() <= 1e-10 * max(1.0, np.abs(ref["torque"]).max())
    assert checkpoint_bytes(eng, meta) == data


@pytest.mark.parametrize("cfg,sort,walk", [("cfg1", 0, None), ("cfg3", 0, "both_rows"),
                                           ("cfg3", 0, "list"), ("cfg3", 100, "list")])
def test_restart_continues_the_trajectory(monkeypatch, cfg, sort, walk):
    """A restart is bit-exact when the summation order is a function of the
    state alone: a fixed slot order and the row / both-rows walks.  The
    once-per-pair list (cfg3's default) is rebuilt from the restored positions,
    so its batches group the i-side sums differently from the uninterrupted
    run's list: the restart then agrees to rounding, as across a re-sort."""
    if walk is not None:
        monkeypatch.setenv("B2MD_NEWTON", "1" if walk == "list" else "0")
    wl = configs.make(cfg)
    a = b2.Engine(wl.comp, wl.opts, wl.dt)
    a.set_sort_interval(sort)
    a.set_state(wl.states[0])
    a.step(7)
    data = checkpoint_bytes(a)
    a.step(9)
    b = b2.Engine(wl.comp, wl.opts, wl.dt)
    b.set_sort_interval(sort)
    restore_checkpoint(b, data)
    b.step(9)
    ra, rb = records(a.state()), records(b.state())
    if sort == 0 and walk != "list":
        assert np.array_equal(ra, rb)  # bit-exact restart
    else:
        assert np.abs(ra - rb).max() <= 1e-12 * max(1.0, np.abs(ra).max())


def test_restore_into_one_replica():
    wl = configs.make("cfg4", replicas=2, steps=3)
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=2)
    eng.set_state(wl.states)
    before = [records(s) for s in eng.states()]
    src = b2.Engine(wl.comp, wl.opts, wl.dt)
    src.set_state(wl.states[0])
    src.step(3)
    block = src.state_block()
    eng.restore_state_block(block, replica=1)
    after = [records(s) for s in eng.states()]
    assert np.array_equal(after[0], before[0])
    assert np.array_equal(after[1], records(src.state()))


def test_restore_errors():
    comp, opts, st = golden_cases.eval_cases()["two_clj"]
    eng = b2.Engine(comp, opts, 0.002)
    eng.set_state(st)
    with pytest.raises(b2.IoError, match="molecule count mismatch"):
        restore_checkpoint(eng, G["sampled_water"].tobytes())
    block = eng.state_block()
    with pytest.raises(b2.IoError, match=r"truncated or corrupted data \(need 8 bytes at offset 116\)"):
        eng.restore_state_block(block[:120])
    bad = bytearray(block)
    bad[4:12] = np.float64(comp.box_length * 1.5).tobytes()
    with pytest.raises(b2.IoError, match="box length"):
        eng.restore_state_block(bytes(bad))
