"""Heat-flux test systems and independent checks (test infrastructure).

Restates the known-answer set-ups of the reference's own heat-flux tests
(tests/test_greenkubo.cpp:172-216 rest / ideal gas, 218-287 independent
double loop) with this repo's seeded numpy inputs.
"""
from __future__ import annotations

import numpy as np

from paper_1507_07548_b200 import (
    ElectrostaticsMethod,
    ForceFieldOptions,
    SystemComposition,
    SystemState,
    build_species,
    make_lj_site,
)


def rotate(q, v):
    """geom.hpp:62-66 in numpy: v + 2w (u x v) + 2 u x (u x v)."""
    u = np.asarray(q[1:])
    t = np.cross(u, v)
    return v + 2.0 * q[0] * t + 2.0 * np.cross(u, t)


def random_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def ideal_gas_case(seed=8):
    """test_greenkubo.cpp:172-216: three rotors 15 apart in a box of 40 with
    rc 2.5 — no pair inside the cutoff, so J_q = sum (e_kin - h) v."""
    sp = build_species("rotor", [make_lj_site(0.4, 0, 0, 1, 1, 1.0), make_lj_site(-0.4, 0, 0, 1, 1, 1.0)])
    comp = SystemComposition([sp], [3], 40.0, 1.0)
    opts = ForceFieldOptions(cutoff=2.5, method=ElectrostaticsMethod.none)
    st = SystemState(3, 40.0)
    st.pos = np.array([[5.0, 5, 5], [20, 20, 20], [35, 35, 35]])
    rng = np.random.default_rng(seed)
    st.vel = rng.normal(size=(3, 3))
    st.ang_vel = np.column_stack([np.zeros(3), rng.normal(size=(3, 2))])
    st.orient = random_quats(rng, 3)
    h = np.array([2.5])
    inertia = sp.inertia_principal
    expected = np.zeros(3)
    for i in range(3):
        w = st.ang_vel[i]
        e = 0.5 * sp.total_mass * st.vel[i] @ st.vel[i] + 0.5 * float(inertia @ (w * w))
        expected += (e - h[0]) * st.vel[i]
    return comp, opts, st, h, expected


def dimer_case(seed=17, n=6):
    """test_greenkubo.cpp:218-287: six LJ dimers with unequal sites, box 7,
    rc 3 (many site pairs straddle the cutoff)."""
    sp = build_species("dimer", [make_lj_site(0.3, 0, 0, 1.0, 0.9, 1.0),
                                 make_lj_site(-0.3, 0, 0, 0.9, 1.1, 1.2)])
    comp = SystemComposition([sp], [n], 7.0, 1.0)
    opts = ForceFieldOptions(cutoff=3.0, method=ElectrostaticsMethod.none)
    rng = np.random.default_rng(seed)
    st = SystemState(n, 7.0)
    # rejection-sampled so no two centres are closer than 0.9
    pos = []
    while len(pos) < n:
        p = rng.uniform(0, 7.0, size=3)
        if all(np.linalg.norm((p - q) - 7.0 * np.round((p - q) / 7.0)) > 0.9 for q in pos):
            pos.append(p)
    st.pos = np.array(pos)
    st.orient = random_quats(rng, n)
    st.vel = rng.normal(size=(n, 3))
    st.ang_vel = rng.normal(size=(n, 3))
    return comp, opts, st, np.array([0.37])


def independent_flux(comp, rc, st, h):
    """From-scratch double loop over ordered pairs (i != j), the molecule-pair
    decomposition of test_greenkubo.cpp:236-283: LJ with Lorentz-Berthelot
    site parameters, each row collecting 0.5 u_ij and
    0.5 (f_ij.v_i + g_ij.w_i) r_ij."""
    n = comp.molecule_count()
    L = comp.box_length
    sp = comp.species[0]
    sites = sp.sites
    off = [[rotate(st.orient[i], np.array(s.body_pos)) for s in sites] for i in range(n)]
    pot = np.zeros(n)
    transport = np.zeros(3)
    for i in range(n):
        w_lab = rotate(st.orient[i], st.ang_vel[i])
        for j in range(n):
            if i == j:
                continue
            d = st.pos[i] - st.pos[j]
            rij = d - L * np.round(d / L)
            f_ij = np.zeros(3)
            g_ij = np.zeros(3)
            u_ij = 0.0
            for a in range(len(sites)):
                for b in range(len(sites)):
                    rv = rij + off[i][a] - off[j][b]
                    r = np.linalg.norm(rv)
                    if r >= rc:
                        continue
                    sig = 0.5 * (sites[a].sigma + sites[b].sigma)
                    eps = np.sqrt(sites[a].epsilon * sites[b].epsilon)
                    sr6 = (sig / r) ** 6
                    u_ij += 4 * eps * (sr6 * sr6 - sr6)
                    dudr = -4 * eps * (12 * sr6 * sr6 - 6 * sr6) / r
                    f = (-dudr / r) * rv
                    f_ij += f
                    g_ij += np.cross(off[i][a], f)
            pot[i] += 0.5 * u_ij
            transport += 0.5 * (f_ij @ st.vel[i] + g_ij @ w_lab) * rij
    out = transport.copy()
    inertia = sp.inertia_principal
    for i in range(n):
        w = st.ang_vel[i]
        e = 0.5 * sp.total_mass * st.vel[i] @ st.vel[i] + 0.5 * float(inertia @ (w * w)) + pot[i]
        out += (e - h[0]) * st.vel[i]
    return out


def flux_scale(comp, st, h, jq):
    """Magnitude the heat-flux tolerance is relative to: the larger of |J_q|
    and the convective sum of |(e_kin_i - h_i) v_i| (J_q itself can cancel)."""
    idx = comp.species_index()
    total = np.zeros(3)
    for k, sp in enumerate(comp.species):
        sel = idx == k
        v = st.vel[sel]
        w = st.ang_vel[sel]
        ek = 0.5 * sp.total_mass * (v * v).sum(1) + 0.5 * (w * w * sp.inertia_principal).sum(1)
        total += np.abs((ek - h[k])[:, None] * v).sum(0)
    return max(float(np.abs(jq).max()), float(total.max()), 1.0)
