"""Smoke-size runs of every hot kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): the cluster walk (k_force_cpair,
k_step_drift_arcs, k_heat_flux_cpair), the search + bit-matrix walk
(k_search, k_force_single), the rigid and multi-site kernels (k_force_rigid,
k_force_multi), the Ewald kernels (k_ewald_tables / _sk / _force) and the RDF
kernels (k_rdf_stage / k_rdf_pairs).  Each case is checked against the oracle
so a sanitizer run also proves the instrumented path computed the right
answer.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_1507_07548_b200 as b2  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_1507_07548_b200 import configs  # noqa: E402


def check(name, wl, steps=3):
    st = wl.states[0]
    ff = b2.ForceField(wl.comp, wl.opts)
    s = st.copy()
    ff.evaluate(s)
    o = pyoracle.OracleFF(wl.comp, wl.opts)
    ref = o.evaluate(st.pos, st.orient)
    df = np.abs(s.force - ref["force"]).max() / max(1.0, np.abs(ref["force"]).max())
    assert df <= 1e-10, (name, df)
    assert np.array_equal(ff.pair_list(), o.pair_list(st.pos)), name
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, replicas=len(wl.states))
    eng.set_state(wl.states)
    eng.step(steps)
    h = np.full(len(wl.comp.species), -0.3)
    eng.heat_fluxes(h)
    rdf = b2.RdfHistogram(eng, 0.05, 0.5 * wl.comp.box_length)
    rdf.accumulate()
    rdf.counts()
    print(f"{name}: dF={df:.2e} ok", flush=True)


def main():
    only = sys.argv[1:] or ["cluster", "newton", "bitmatrix", "rigid", "tile", "ewald", "replicas"]
    if "cluster" in only:
        os.environ["B2MD_CLUSTER"] = "2"
        os.environ["B2MD_NEWTON"] = "0"  # the both-rows walk (the list is the default)
        check("cluster walk (single-site, rc < 0.3 L)", configs.lj_fluid_config(1200, 0.8, 2.5, seed=5,
                                                                               name="san-cluster"))
        os.environ.pop("B2MD_CLUSTER")
        os.environ.pop("B2MD_NEWTON")
    if "newton" in only:
        os.environ["B2MD_CLUSTER"] = "2"
        os.environ["B2MD_NEWTON"] = "1"
        check("once-per-pair cluster walk", configs.lj_fluid_config(1200, 0.8, 2.5, seed=5,
                                                                   name="san-newton"))
        os.environ.pop("B2MD_CLUSTER")
        os.environ.pop("B2MD_NEWTON")
    if "bitmatrix" in only:
        check("search + bit-matrix walk", configs.lj_fluid_config(300, 0.8, None, seed=3, name="san-lj"))
    if "rigid" in only:
        check("rigid 2CLJ", configs.two_clj_config(200, 0.3, 5, 2.0, 0.002, 3, "san-2clj"))
    if "tile" in only:
        os.environ["B2MD_TILE"] = "1"
        check("rigid 2CLJ block-pair tiles", configs.two_clj_config(200, 0.3, 5, 2.0, 0.002, 3,
                                                                    "san-2clj-tile"))
        os.environ.pop("B2MD_TILE")
    if "ewald" in only:
        wl = configs.make("cfg2")
        check("water + ions, Ewald (cfg2)", wl, steps=1)
    if "replicas" in only:
        check("2CLJ replicas", configs.replica_batch_config(3, 0, 3))


if __name__ == "__main__":
    main()
