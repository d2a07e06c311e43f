"""Definitions of the golden-vector cases (inputs only).  Outputs come from
the reference (tests/golden/make_golden.py) and are committed as .npz."""
from __future__ import annotations

import math

import numpy as np

from paper_1507_07548_b200 import (
    ElectrostaticsMethod,
    ForceFieldOptions,
    Site,
    SiteKind,
    SystemComposition,
    build_species,
    configs,
    ewald_tune,
    make_charge_site,
    make_lj_site,
)
from paper_1507_07548_b200.model import _ENERGY_FIELDS

import systems

ENERGY_FIELDS = _ENERGY_FIELDS


def species_cases():
    d = 1.0 / 3.166
    half = math.radians(109.47) / 2.0
    return {
        "lj": [make_lj_site(0, 0, 0, 1.0, 1.0, 1.0)],
        "two_clj": [make_lj_site(0.25, 0, 0, 1.0, 1.0, 0.5), make_lj_site(-0.25, 0, 0, 1.0, 1.0, 0.5)],
        "tri": [make_lj_site(0.3, 0, 0, 1.0, 0.8, 1), make_lj_site(-0.2, 0.25, 0, 0.9, 1.2, 1),
                make_lj_site(-0.1, -0.2, 0.15, 1.1, 0.6, 2)],
        "rotor3": [make_lj_site(0.3, 0, 0, 0.9, 0.7, 1.0), make_lj_site(-0.2, 0.25, 0, 1.0, 1.0, 1.5),
                   make_lj_site(0, -0.2, 0.2, 1.1, 0.5, 0.8)],
        "water": [Site(SiteKind.lj, (0, 0, 0), 1.0, 1.0, -0.8476, 15.9994),
                  Site(SiteKind.charge, (d * math.sin(half), d * math.cos(half), 0), 0, 0, 0.4238, 1.008),
                  Site(SiteKind.charge, (-d * math.sin(half), d * math.cos(half), 0), 0, 0, 0.4238, 1.008)],
        "dummy": [Site(SiteKind.dummy, (0.1, 0.2, 0.3), 0.0, 0.0, 0.0, 1.0),
                  make_lj_site(0.5, -0.1, 0.0, 1.0, 1.0, 2.0)],
    }


def _water_ions_small(n_water=40, n_ion=2, seed=3):
    wl = configs.water_ions_config(seed)
    water, na, cl = wl.comp.species
    n = n_water + 2 * n_ion
    L = wl.comp.box_length * (n / 1100.0) ** (1.0 / 3.0)
    comp = SystemComposition([water, na, cl], [n_water, n_ion, n_ion], L, wl.comp.temperature)
    st = systems.random_state(comp, seed, 0.55)
    opts = ForceFieldOptions(cutoff=0.45 * L, method=ElectrostaticsMethod.ewald,
                             ewald=configs.EwaldParams(5.6 / L, 5), workers=1)
    return comp, opts, st


def eval_cases():
    cases = {}
    comp = systems.lj_fluid(64, 6.0, 1.0)
    st = systems.random_state(comp, 5, 0.9)
    cases["lj64"] = (comp, systems.lj_opts(2.5), st)
    moved = st.copy()
    moved.pos = moved.pos + np.array([1.3, -2.1, 0.7]) * np.array([1.0, 3.0, 11.0])
    cases["lj64_unwrapped"] = (comp, systems.lj_opts(2.5), moved)
    comp, opts = systems.dimer_mono_mixture()
    cases["mixture"] = (comp, opts, systems.random_state(comp, 31, 0.85))
    comp, opts = systems.tri_rotor()
    cases["tri"] = (comp, opts, systems.random_state(comp, 10, 0.9))
    comp, opts = systems.rf_dimers()
    cases["rf"] = (comp, opts, systems.random_state(comp, 2, 0.9))
    comp = systems.ion_pair_comp(4, 6.0)
    cases["ewald_ions"] = (comp, systems.ewald_opts(3.0, ewald_tune(1e-6, 3.0, 6.0)),
                           systems.random_state(comp, 11, 1.0))
    comp, opts = systems.rigid_dipoles()
    cases["ewald_dipoles"] = (comp, opts, systems.random_state(comp, 9, 0.8))
    comp, opts, st = systems.rock_salt()
    cases["madelung"] = (comp, opts, st)
    cases["water_ions"] = _water_ions_small()
    wl = configs.two_clj_config(120, 0.3, 4, 2.0, 0.002, 10, "2clj120")
    cases["two_clj"] = (wl.comp, wl.opts, wl.states[0])
    return cases


def traj_cases():
    cases = {}
    wl = configs.lj_fluid_config(108, 0.8, 2.5, seed=9, dt=0.005, steps=20)
    cases["lj108"] = (wl.comp, wl.opts, wl.states[0], 0.005, 20)
    wl = configs.two_clj_config(120, 0.3, 4, 2.0, 0.002, 20, "2clj120")
    cases["two_clj"] = (wl.comp, wl.opts, wl.states[0], 0.002, 20)
    comp, opts = systems.tri_rotor(8, 8.0, 3.5)
    st = systems.random_state(comp, 12, 1.05)
    rng = configs.Rng(4)
    for i in range(8):
        st.vel[i] = (0.2 * rng.gaussian(), 0.2 * rng.gaussian(), 0.2 * rng.gaussian())
        st.ang_vel[i] = (0.3 * rng.gaussian(), 0.3 * rng.gaussian(), 0.3 * rng.gaussian())
    cases["tri"] = (comp, opts, st, 0.0005, 40)
    return cases


def flux_inputs(name, comp):
    """Seeded velocities, angular velocities (body frame) and one enthalpy per
    species for the heat-flux golden vectors (stored with them, so the seed
    only fixes what make_golden.py writes)."""
    seed = sum(name.encode()) * 7919
    rng = np.random.default_rng(seed)
    n = comp.molecule_count()
    vel = rng.normal(size=(n, 3))
    ang_vel = rng.normal(size=(n, 3))
    h = rng.normal(size=comp.species_count()) * 2.0
    return vel, ang_vel, h


def rdf_inputs(name, comp, st):
    """Two seeded snapshots (the case's state and a displaced / re-oriented
    copy), bin width and r_max = L/2 (the engine's choice, engine.cpp:204)."""
    seed = sum(name.encode()) * 104729
    rng = np.random.default_rng(seed)
    n = comp.molecule_count()
    pos2 = st.pos + rng.normal(scale=0.3, size=(n, 3))
    q = rng.normal(size=(n, 4))
    orient2 = q / np.linalg.norm(q, axis=1, keepdims=True)
    L = comp.box_length
    return L / 150.0, 0.5 * L, [(st.pos, st.orient), (pos2, orient2)]
