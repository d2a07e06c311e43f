"""Small test systems, restating the reference's test fixtures
(tests/test_helpers.hpp:14-87) with this repo's seeded generator: LJ fluids,
multi-site molecules, charged dimers, ion pairs, rigid dipoles, rock salt.
Shared by the parity tests and tests/golden/make_golden.py."""
from __future__ import annotations

import math

import numpy as np

from paper_1507_07548_b200 import (
    ElectrostaticsMethod,
    EwaldParams,
    ForceFieldOptions,
    Site,
    SiteKind,
    SystemComposition,
    SystemState,
    build_species,
    ewald_tune,
    make_charge_site,
    make_lj_site,
)
from paper_1507_07548_b200.configs import Rng


def lj_fluid(n, box, temperature=1.0, sigma=1.0, eps=1.0):  # test_helpers.hpp:34-40
    return SystemComposition([build_species("lj", [make_lj_site(0, 0, 0, sigma, eps, 1.0)])],
                             [n], box, temperature)


def quat_from_axis_angle(axis, angle):  # geom.hpp:47-52
    n = math.sqrt(sum(a * a for a in axis))
    if n == 0.0:
        return (1.0, 0.0, 0.0, 0.0)
    s = math.sin(0.5 * angle) / n
    return (math.cos(0.5 * angle), axis[0] * s, axis[1] * s, axis[2] * s)


def rotate(q, v):  # geom.hpp:62-66 (numpy, for fixtures only)
    w, u = q[0], np.array(q[1:])
    t = np.cross(u, v)
    return v + 2.0 * w * t + 2.0 * np.cross(u, t)


def random_state(comp: SystemComposition, seed: int, min_sep: float = 0.85) -> SystemState:
    """Rejection-sampled non-overlapping configuration (test_helpers.hpp:43-87)."""
    rng = Rng(seed)
    n = comp.molecule_count()
    L = comp.box_length
    st = SystemState(n, L)
    spec = comp.species_index()
    body = [np.array([s.body_pos for s in sp.sites]) for sp in comp.species]
    placed = []
    for i in range(n):
        sp = comp.species[spec[i]]
        for attempt in range(200000):
            r = np.array([rng.uniform(0, L), rng.uniform(0, L), rng.uniform(0, L)])
            q = (1.0, 0.0, 0.0, 0.0)
            if sp.rotational_dof > 0:
                axis = (rng.gaussian(), rng.gaussian(), rng.gaussian())
                q = quat_from_axis_angle(axis, rng.uniform(0, 2 * math.pi))
                nq = math.sqrt(sum(c * c for c in q))
                q = tuple(c / nq for c in q)
            mine = np.array([r + rotate(q, b) for b in body[spec[i]]])
            ok = True
            for other in placed:
                d = mine[:, None, :] - other[None, :, :]
                d -= L * np.round(d / L)
                if np.min(np.sum(d * d, axis=2)) < min_sep * min_sep:
                    ok = False
                    break
            if ok:
                st.pos[i] = r
                st.orient[i] = q
                placed.append(mine)
                break
        else:
            raise RuntimeError("random_state: cannot place molecules")
        sv = math.sqrt(comp.temperature / sp.total_mass)
        st.vel[i] = (sv * rng.gaussian(), sv * rng.gaussian(), sv * rng.gaussian())
    return st


def lj_opts(cutoff, **kw):
    return ForceFieldOptions(cutoff=cutoff, **kw)


def dimer_mono_mixture():  # test_parallel.cpp:98-120
    comp = SystemComposition(
        [build_species("dimer", [make_lj_site(0.4, 0, 0, 1, 1, 1), make_lj_site(-0.4, 0, 0, 1, 1, 1)]),
         build_species("mono", [make_lj_site(0, 0, 0, 0.9, 1.3, 1)])], [40, 40], 7.0, 1.0)
    return comp, lj_opts(2.5)


def tri_rotor(n=8, box=7.0, cutoff=3.0):  # test_potentials.cpp:193-212
    comp = SystemComposition([build_species("tri", [
        make_lj_site(0.3, 0, 0, 1.0, 0.8, 1), make_lj_site(-0.2, 0.25, 0, 0.9, 1.2, 1),
        make_lj_site(-0.1, -0.2, 0.15, 1.1, 0.6, 2)])], [n], box, 1.0)
    return comp, lj_opts(cutoff)


def rf_dimers(n=10):  # test_potentials.cpp:214-258
    comp = SystemComposition([build_species("pair", [
        make_charge_site(0.2, 0, 0, 0.5, 1.0), make_charge_site(-0.2, 0, 0, -0.5, 1.0),
        make_lj_site(0, 0, 0, 1.0, 1.0, 1.0)])], [n], 8.0, 1.0)
    opts = ForceFieldOptions(cutoff=3.5, method=ElectrostaticsMethod.reaction_field, eps_rf=65.0)
    return comp, opts


def ion_pair_comp(n_each, box):  # test_ewald.cpp:10-19
    return SystemComposition([build_species("cat", [make_charge_site(0, 0, 0, 1.0, 1.0)]),
                              build_species("ani", [make_charge_site(0, 0, 0, -1.0, 1.0)])],
                             [n_each, n_each], box, 1.0)


def ewald_opts(cutoff, params: EwaldParams):
    return ForceFieldOptions(cutoff=cutoff, method=ElectrostaticsMethod.ewald, ewald=params, workers=1)


def rock_salt():  # test_ewald.cpp:52-76
    cells = 4
    comp = ion_pair_comp(32, float(cells))
    st = SystemState(64, float(cells))
    plus, minus = 0, 32
    for x in range(cells):
        for y in range(cells):
            for z in range(cells):
                if (x + y + z) % 2 == 0:
                    st.pos[plus] = (x, y, z)
                    plus += 1
                else:
                    st.pos[minus] = (x, y, z)
                    minus += 1
    return comp, ewald_opts(2.0, ewald_tune(1e-6, 2.0, cells)), st


def rigid_dipoles():  # test_ewald.cpp:112-148
    comp = SystemComposition([build_species("dipole", [make_charge_site(0.25, 0, 0, 0.6, 1.0),
                                                       make_charge_site(-0.25, 0, 0, -0.6, 1.0)])],
                             [6], 7.0, 1.0)
    return comp, ewald_opts(3.5, ewald_tune(1e-6, 3.5, 7.0))


def dumbbell():  # test_engine.cpp:67-102
    return SystemComposition([build_species("dumbbell", [make_lj_site(0.5, 0, 0, 1, 1, 1),
                                                         make_lj_site(-0.5, 0, 0, 1, 1, 1)])],
                             [1], 10.0, 1.0)


def image_cube_sum(pos, q, box, n_img):  # test_helpers.hpp:220-247
    pos = np.asarray(pos)
    q = np.asarray(q)
    rng_ = np.arange(-n_img, n_img + 1)
    shifts = np.stack(np.meshgrid(rng_, rng_, rng_, indexing="ij"), -1).reshape(-1, 3) * box
    u = 0.0
    n = len(q)
    for i in range(n):
        d = pos[i] - pos  # (n,3)
        im = d[:, None, :] + shifts[None, :, :]
        r = np.sqrt(np.sum(im * im, axis=2))
        qq = q[i] * q
        if True:
            r[i, (shifts == 0).all(axis=1)] = np.inf
        u += 0.5 * np.sum(qq[:, None] / r)
    dip = np.sum(q[:, None] * pos, axis=0)
    u -= 2.0 * math.pi * np.dot(dip, dip) / (3.0 * box ** 3)
    return u


def direct_image_sum_converged(pos, q, box):  # test_helpers.hpp:249-268
    j = [image_cube_sum(pos, q, box, n) for n in (3, 4, 5)]
    m = np.array([[1, 1 / 9, 1 / 27], [1, 1 / 16, 1 / 64], [1, 1 / 25, 1 / 125]])
    return float(np.linalg.solve(m, np.array(j))[0])
