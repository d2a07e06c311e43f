"""Generates tests/golden/traj_cfg3_100.npz: the UNMODIFIED reference engine
(oracle/_ref/libtmdref.so, tmd::Engine with ForceFieldOptions.workers = all
host cores) run for cfg3's 100 velocity-Verlet steps (BASELINE.json configs[3]:
N = 16384, rc = 5, dt = 0.005) from the seeded cfg3 state.  Stored: every 8th
molecule's final position and velocity (2048 molecules), the energy parts and
the virial -- the GPU test compares the cluster walk's 100-step trajectory
against them at the north-star bar (1e-9).

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_cfg3_trajectory.py
"""
from __future__ import annotations

import copy
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle  # noqa: E402
from paper_1507_07548_b200 import configs  # noqa: E402

STRIDE = 8
STEPS = 100  # the north-star trajectory bar (cfg3 itself runs 1000)


def main() -> None:
    wl = configs.make("cfg3")
    st = wl.states[0]
    opts = copy.copy(wl.opts)
    opts.workers = os.cpu_count() or 1
    eng = pyoracle.RefEngine(wl.comp, opts, wl.dt)
    eng.set_state(st.pos, st.orient, st.vel, st.ang_vel)
    t0 = time.perf_counter()
    eng.step(STEPS)
    out = eng.state()
    e = out["energy"]
    np.savez_compressed(
        Path(__file__).resolve().parent / "traj_cfg3_100.npz",
        stride=STRIDE, steps=STEPS, workers=opts.workers,
        pos=out["pos"][::STRIDE], vel=out["vel"][::STRIDE],
        energy=np.array([e.lj, e.lrc, e.total()]), virial=out["virial"])
    print(f"{STEPS} reference steps in {time.perf_counter() - t0:.1f} s "
          f"(W={opts.workers}); E_total={e.total():.12g}")


if __name__ == "__main__":
    main()
