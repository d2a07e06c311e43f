"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libtmdref.so, built by `make -C oracle` from /root/reference).

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_golden.py
Each case stores the inputs (composition is rebuilt from tests/systems.py by
name), the reference outputs of tmd::ForceField::evaluate / Engine::step and
the COM partner list computed with the reference's own minimum_image/norm2.
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import pyoracle  # noqa: E402
from paper_1507_07548_b200 import configs  # noqa: E402
import golden_cases  # noqa: E402

OUT = Path(__file__).resolve().parent


def rng_vectors():
    lib = pyoracle.ref_lib()
    lib.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
    seeds = [0, 1, 77, (1 << 63) + 5]
    n = 32
    u64 = np.zeros((len(seeds), n), dtype=np.uint64)
    uni = np.zeros((len(seeds), n))
    gau = np.zeros((len(seeds), n))
    for k, s in enumerate(seeds):
        lib.ref_rng_draws(s, n, u64[k].ctypes.data_as(C.POINTER(C.c_uint64)),
                          uni[k].ctypes.data_as(C.POINTER(C.c_double)),
                          gau[k].ctypes.data_as(C.POINTER(C.c_double)))
    np.savez_compressed(OUT / "rng.npz", seeds=np.array(seeds, dtype=np.uint64), u64=u64,
                        uniform=uni, gaussian=gau)


def species_vectors():
    out = {}
    for name, sites in golden_cases.species_cases().items():
        sp = pyoracle.build_species_c(sites, "ref")
        out[name + "_body"] = np.array([sp.sites[k].body_pos[:] for k in range(sp.n_sites)])
        out[name + "_inertia"] = np.array(sp.inertia_principal[:])
        out[name + "_scalars"] = np.array([sp.total_mass, sp.net_charge, sp.max_extent,
                                           sp.rotational_dof])
    np.savez_compressed(OUT / "species.npz", **out)


def eval_vectors():
    for name, (comp, opts, st) in golden_cases.eval_cases().items():
        ref = pyoracle.RefFF(comp, opts)
        r = ref.evaluate(st.pos, st.orient)
        e = r["energy"]
        np.savez_compressed(
            OUT / f"eval_{name}.npz", pos=st.pos, orient=st.orient, force=r["force"],
            torque=r["torque"], virial=r["virial"],
            energy=np.array([getattr(e, f) for f in golden_cases.ENERGY_FIELDS]),
            pairs=ref.pair_list(st.pos), warning=np.array(ref.warning))


def flux_vectors():
    """tmd::heat_flux (src/greenkubo.cpp:182-266) on every eval case with
    seeded velocities, angular velocities and enthalpies."""
    for name, (comp, opts, st) in golden_cases.eval_cases().items():
        vel, ang_vel, h = golden_cases.flux_inputs(name, comp)
        ref = pyoracle.RefFF(comp, opts)
        jq = ref.heat_flux(st.pos, st.orient, vel, ang_vel, h)
        np.savez_compressed(OUT / f"flux_{name}.npz", pos=st.pos, orient=st.orient, vel=vel,
                            ang_vel=ang_vel, h=h, jq=jq)


def rdf_vectors():
    """tmd::RdfHistogram (structure.cpp:10-153) on every eval case: counts,
    serialize bytes and finalize tables of two snapshots, and first_minimum /
    solvation_number of each table."""
    for name, (comp, opts, st) in golden_cases.eval_cases().items():
        bw, rmax, snaps = golden_cases.rdf_inputs(name, comp, st)
        ref = pyoracle.RefRdf(pyoracle.RefFF(comp, opts), bw, rmax)
        for pos, orient in snaps:
            ref.accumulate(pos, orient)
        counts, n_snap = ref.counts()
        tables = ref.finalize()
        flat = np.concatenate([np.concatenate([[t["species_a"], t["species_b"], t["partner_density"],
                                                t["bin_width"], t["snapshots"], len(t["g"])],
                                               np.column_stack([t["r_mid"], t["g"], t["n_cum"]]).ravel()])
                               for t in tables]) if tables else np.zeros(0)
        fmin = np.array([pyoracle.ref_first_minimum(t["r_mid"], t["g"]) for t in tables])
        solv = np.array([pyoracle.ref_solvation_number(t["bin_width"], t["g"], t["partner_density"],
                                                       0.6 * rmax) for t in tables])
        np.savez_compressed(
            OUT / f"rdf_{name}.npz", bin_width=bw, r_max=rmax,
            pos=np.stack([p for p, _ in snaps]), orient=np.stack([o for _, o in snaps]),
            counts=counts, snapshots=n_snap, serialized=np.frombuffer(ref.serialize(), np.uint8),
            finalize=flat, first_minimum=fmin, solvation_number=solv)


def checkpoint_vectors():
    """tmd::Engine::checkpoint_bytes (engine.cpp:420-462): two sampled runs
    (Engine::run with every sampler section the reference has) and a fresh
    engine after set_state; plus the reference's restore error on truncated
    copies of one of them."""
    cases = golden_cases.eval_cases()
    comp, opts, st = cases["water_ions"]
    a = pyoracle.ref_run_sampled_checkpoint(comp, opts, 0.0005, 7, 20, 40, n_ext=2, corr_length=6,
                                            n_blocks=4, flags=62, enthalpy=[-1.0, 0.5, 0.7],
                                            residence=(1, 0, 0.0),
                                            config_text="[system]\nexample = true\n")
    comp, opts, st = cases["rf"]
    b = pyoracle.ref_run_sampled_checkpoint(comp, opts, 0.001, 3, 10, 30, n_ext=1, corr_length=5,
                                            n_blocks=3, flags=1 | 2 | 4 | 16, enthalpy=[0.3],
                                            config_text="rf")
    comp, opts, st = cases["two_clj"]
    eng = pyoracle.RefEngine(comp, opts, 0.002, seed=5)
    eng.set_state(st.pos, st.orient, st.vel, st.ang_vel)
    fresh = eng.checkpoint_bytes()
    # the reference's restore of truncated water-ions copies
    comp_w, opts_w, _ = cases["water_ions"]
    cuts = [9, 40, 200, 1000, len(a) // 2, len(a) - 3]
    msgs = []
    for cut in cuts:
        e = pyoracle.RefEngine(comp_w, opts_w, 0.0005, seed=7)
        try:
            e.restore(a[:cut])
            msgs.append("")
        except pyoracle.OracleError as exc:
            msgs.append(str(exc))
    np.savez_compressed(OUT / "ckpt.npz", sampled_water=np.frombuffer(a, np.uint8),
                        sampled_rf=np.frombuffer(b, np.uint8), fresh_two_clj=np.frombuffer(fresh, np.uint8),
                        fresh_seed=5, cuts=np.array(cuts), cut_messages=np.array(msgs))


def sampling_vectors():
    """tmd::DerivativeAccumulator (massieu.cpp:9-70) and tmd::BlockStat
    (results.hpp:21-51) fed seeded samples, serialized by the reference."""
    rng = np.random.default_rng(2718)
    out = {}
    cases = [(1, 0, 5), (4, 20, 20), (4, 10, 23), (7, 30, 13), (3, 1, 4)]
    for k, (nb, expected, count) in enumerate(cases):
        smp = rng.normal(size=(count, 3)) * [50.0, 3.0, 0.2] + [-900.0, 4.0, 0.5]
        x = rng.normal(size=count)
        out[f"da_{k}_samples"] = smp
        out[f"da_{k}_bytes"] = np.frombuffer(
            pyoracle.ref_derivative_accumulator(1.5, 812.0, 256, nb, expected, smp), np.uint8)
        out[f"bs_{k}_x"] = x
        out[f"bs_{k}_bytes"] = np.frombuffer(pyoracle.ref_block_stat(nb, expected, x), np.uint8)
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT / "sampling.npz", **out)


def traj_vectors():
    for name, (comp, opts, st, dt, steps) in golden_cases.traj_cases().items():
        eng = pyoracle.RefEngine(comp, opts, dt, seed=1)
        eng.set_state(st.pos, st.orient, st.vel, st.ang_vel)
        eng.step(steps)
        s = eng.state()
        e = s["energy"]
        np.savez_compressed(
            OUT / f"traj_{name}.npz", pos0=st.pos, orient0=st.orient, vel0=st.vel,
            ang_vel0=st.ang_vel, dt=dt, steps=steps, pos=s["pos"], orient=s["orient"],
            vel=s["vel"], ang_vel=s["ang_vel"], force=s["force"], torque=s["torque"],
            virial=s["virial"], energy=np.array([getattr(e, f) for f in golden_cases.ENERGY_FIELDS]))


if __name__ == "__main__":
    if not pyoracle.ref_available():
        sys.exit("oracle/_ref/libtmdref.so missing: run `make -C oracle` with /root/reference present")
    rng_vectors()
    species_vectors()
    eval_vectors()
    flux_vectors()
    rdf_vectors()
    checkpoint_vectors()
    sampling_vectors()
    traj_vectors()
    print("golden vectors written to", OUT)
