"""Seeded synthetic systems for the five BASELINE.json configs.

There is no public dataset on this path: the configs are synthetic.  All
randomness flows through the reference's generator algorithm — xoshiro256++
seeded by splitmix64, 53-bit uniforms, Box-Muller cosine branch,
Fisher-Yates shuffle (include/tmd/rng.hpp:14-76) — restated here.  The
Maxwell-Boltzmann draw, drift removal and exact kinetic rescale follow
init_lattice (src/model.cpp:391-423); Shoemake orientations follow
random_orientation (src/model.cpp:341-347).  Gaps in BASELINE.json are filled
as SURVEY.md Appendix A recommends and DESIGN.md records.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .forcefield import EwaldParams, ForceFieldOptions
from .model import (
    ElectrostaticsMethod,
    SiteKind,
    Site,
    SystemComposition,
    SystemState,
    build_species as _build_species_native,
    kinetic_energy_rot,
    kinetic_energy_trans,
    make_lj_site,
    rotational_dof,
    translational_dof,
)

_M64 = (1 << 64) - 1

# Species builder of the generators: tmd::build_species (src/model.cpp:68-129).
# Default: b2md_build_species (the native library's bit-exact restatement).
# bench.py's reference arm swaps in the reference's OWN build_species
# (oracle/_ref) through `species_builder`, so that arm loads no product code.
_species_builder = None


def build_species(name, sites):
    return (_species_builder or _build_species_native)(name, sites)


class Rng:
    """xoshiro256++ 1.0 seeded via splitmix64 (rng.hpp:14-76)."""

    def __init__(self, seed: int):
        x = seed & _M64
        self.s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & _M64
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            self.s.append(z ^ (z >> 31))

    @staticmethod
    def _rotl(v, k):
        return ((v << k) | (v >> (64 - k))) & _M64

    def next_u64(self) -> int:
        s = self.s
        result = (self._rotl((s[0] + s[3]) & _M64, 23) + s[0]) & _M64
        t = (s[1] << 17) & _M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return result

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = float(self.next_u64() >> 11) * (2.0 ** -53)
        if lo is None:
            return u
        return lo + (hi - lo) * u

    def uniform_below(self, n: int) -> int:
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= threshold:
                return r % n

    def gaussian(self) -> float:
        u1 = 1.0 - self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.uniform_below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


def random_orientation(rng: Rng):
    """Shoemake uniform unit quaternion (model.cpp:341-347)."""
    u1, u2, u3 = rng.uniform(), rng.uniform(), rng.uniform()
    a, b = math.sqrt(1.0 - u1), math.sqrt(u1)
    t2, t3 = 2.0 * math.pi * u2, 2.0 * math.pi * u3
    return (b * math.cos(t3), a * math.sin(t2), a * math.cos(t2), b * math.sin(t3))


@dataclass
class Workload:
    name: str
    comp: SystemComposition
    opts: ForceFieldOptions
    dt: float
    steps: int
    states: list = field(default_factory=list)  # one SystemState per replica
    description: str = ""

    @property
    def replicas(self) -> int:
        return len(self.states)


def _lattice_state(comp: SystemComposition, rng: Rng, side: int, jitter: float,
                   shuffle_slots: bool) -> SystemState:
    """Simple-cubic lattice ((c + 1/2) a), seeded jitter, random orientation,
    Maxwell-Boltzmann velocities with drift removal and exact rescale."""
    n = comp.molecule_count()
    L = comp.box_length
    a = L / side
    slots = list(range(side ** 3))
    if shuffle_slots:
        rng.shuffle(slots)
    st = SystemState(n, L)
    for i in range(n):
        s = slots[i]
        cx, cy, cz = s % side, (s // side) % side, s // (side * side)
        st.pos[i] = ((cx + 0.5) * a + rng.uniform(-jitter, jitter),
                     (cy + 0.5) * a + rng.uniform(-jitter, jitter),
                     (cz + 0.5) * a + rng.uniform(-jitter, jitter))
    spec = comp.species_index()
    for i in range(n):
        sp = comp.species[spec[i]]
        st.orient[i] = random_orientation(rng) if sp.rotational_dof > 0 else (1.0, 0.0, 0.0, 0.0)
    T = comp.temperature
    for i in range(n):
        sp = comp.species[spec[i]]
        sv = math.sqrt(T / sp.total_mass)
        st.vel[i] = (sv * rng.gaussian(), sv * rng.gaussian(), sv * rng.gaussian())
        inertia = sp.inertia_principal
        w = [0.0, 0.0, 0.0]
        for k in range(3):
            if inertia[k] > 0.0:
                w[k] = math.sqrt(T / inertia[k]) * rng.gaussian()
        st.ang_vel[i] = w
    m = np.array([comp.species[s].total_mass for s in spec])
    p = (m[:, None] * st.vel).sum(axis=0)
    st.vel -= p / m.sum()
    ket = kinetic_energy_trans(comp, st)
    if ket > 0.0:
        st.vel *= math.sqrt(0.5 * translational_dof(comp) * T / ket)
    ker = kinetic_energy_rot(comp, st)
    dof_r = rotational_dof(comp)
    if dof_r > 0 and ker > 0.0:
        st.ang_vel *= math.sqrt(0.5 * dof_r * T / ker)
    st.wrap()
    return st


def lj_fluid_config(n: int, density: float, cutoff: float | None, seed: int = 0,
                    temperature: float = 1.0, dt: float = 0.005, steps: int = 100,
                    side: int | None = None, name: str = "cfg0") -> Workload:
    """cfg0 / cfg3: single-site LJ on a jittered SC lattice (lattice order)."""
    L = (n / density) ** (1.0 / 3.0)
    comp = SystemComposition([build_species("lj", [make_lj_site(0, 0, 0, 1.0, 1.0, 1.0)])],
                             [n], L, temperature)
    if side is None:
        side = int(round(n ** (1.0 / 3.0)))
        while side ** 3 < n:
            side += 1
    rc = 0.45 * L if cutoff is None else cutoff
    st = _lattice_state(comp, Rng(seed), side, 0.1, shuffle_slots=False)
    return Workload(name, comp, ForceFieldOptions(cutoff=rc), dt, steps, [st])


def two_clj_species():
    """Rigid 2CLJ: sites +-0.25 sigma, eps = sigma = 1, mass 0.5 per site."""
    return build_species("2clj", [make_lj_site(0.25, 0, 0, 1.0, 1.0, 0.5),
                                  make_lj_site(-0.25, 0, 0, 1.0, 1.0, 0.5)])


def two_clj_config(n: int, density: float, seed: int, temperature: float, dt: float,
                   steps: int, name: str) -> Workload:
    L = (n / density) ** (1.0 / 3.0)
    comp = SystemComposition([two_clj_species()], [n], L, temperature)
    side = 1
    while side ** 3 < n:
        side += 1
    rng = Rng(seed)
    st = _lattice_state(comp, rng, side, 0.1, shuffle_slots=False)
    return Workload(name, comp, ForceFieldOptions(cutoff=0.45 * L), dt, steps, [st])


# ---- SPC/E water + ions (cfg2), reduced units sigma_ref = 3.166 A, eps_ref/k = 78.2 K
SIGMA_REF_A = 3.166
EPS_REF_K = 78.2
_E = 1.602176634e-19
_EPS0 = 8.8541878128e-12
_KB = 1.380649e-23
_NA = 6.02214076e23
Q_REDUCED = _E / math.sqrt(4.0 * math.pi * _EPS0 * SIGMA_REF_A * 1e-10 * _KB * EPS_REF_K)
KCAL_PER_MOL_K = 4184.0 / (_NA * _KB)  # 1 kcal/mol in K


def water_ions_config(seed: int = 0) -> Workload:
    d = 1.0 / SIGMA_REF_A
    half = math.radians(109.47) / 2.0
    qO, qH = -0.8476 * Q_REDUCED, 0.4238 * Q_REDUCED
    water = build_species("spce", [
        Site(SiteKind.lj, (0.0, 0.0, 0.0), 1.0, 1.0, qO, 15.9994),
        Site(SiteKind.charge, (d * math.sin(half), d * math.cos(half), 0.0), 0.0, 0.0, qH, 1.008),
        Site(SiteKind.charge, (-d * math.sin(half), d * math.cos(half), 0.0), 0.0, 0.0, qH, 1.008),
    ])
    # Smith-Dang ion LJ (sigma per BASELINE.json; eps 0.13 / 0.10 kcal/mol, recorded in DESIGN.md)
    na = build_species("na", [Site(SiteKind.lj, (0.0, 0.0, 0.0), 2.35 / SIGMA_REF_A,
                                   0.13 * KCAL_PER_MOL_K / EPS_REF_K, Q_REDUCED, 22.98977)])
    cl = build_species("cl", [Site(SiteKind.lj, (0.0, 0.0, 0.0), 4.40 / SIGMA_REF_A,
                                   0.10 * KCAL_PER_MOL_K / EPS_REF_K, -Q_REDUCED, 35.453)])
    counts = [1000, 50, 50]
    mass_g_mol = 1000 * water.total_mass + 50 * na.total_mass + 50 * cl.total_mass
    volume_a3 = mass_g_mol / _NA / 0.997 * 1e24  # 997 kg/m^3 = 0.997 g/cm^3
    L = volume_a3 ** (1.0 / 3.0) / SIGMA_REF_A
    T = 298.15 / EPS_REF_K
    comp = SystemComposition([water, na, cl], counts, L, T)
    st = _lattice_state(comp, Rng(seed), 11, 0.1 / SIGMA_REF_A, shuffle_slots=True)
    opts = ForceFieldOptions(cutoff=0.45 * L, method=ElectrostaticsMethod.ewald,
                             ewald=EwaldParams(5.6 / L, 7), workers=1)
    return Workload("cfg2", comp, opts, 0.002, 1, [st])


def replica_batch_config(replicas: int = 8, first_seed: int = 0, steps: int = 500) -> Workload:
    """cfg4: independent 2CLJ N=1000 systems, seeds first_seed.., T_r = 1.5 + 1.5 u."""
    n, density = 1000, 0.3
    L = (n / density) ** (1.0 / 3.0)
    comp = SystemComposition([two_clj_species()], [n], L, 2.25)
    states = []
    temps = []
    for r in range(replicas):
        rng = Rng(first_seed + r)
        T = 1.5 + 1.5 * rng.uniform()
        temps.append(T)
        c = SystemComposition(comp.species, comp.counts, L, T)
        states.append(_lattice_state(c, rng, 10, 0.1, shuffle_slots=False))
    wl = Workload("cfg4", comp, ForceFieldOptions(cutoff=0.45 * L), 0.002, steps, states)
    wl.description = "temperatures " + ",".join(f"{t:.4f}" for t in temps)
    return wl


def make(name: str, species_builder=None, **kw) -> Workload:
    """One of the five BASELINE.json configs.  species_builder(name, sites) ->
    MoleculeSpecies replaces the native build_species (same bits)."""
    global _species_builder
    if species_builder is not None:
        prev, _species_builder = _species_builder, species_builder
        try:
            return make(name, **kw)
        finally:
            _species_builder = prev
    if name == "cfg0":
        return lj_fluid_config(1000, 0.8, None, seed=kw.get("seed", 0), dt=0.005, steps=100,
                               side=10, name="cfg0")
    if name == "cfg1":
        return two_clj_config(2048, 0.3, kw.get("seed", 0), 2.0, 0.002, 100, "cfg1")
    if name == "cfg2":
        return water_ions_config(kw.get("seed", 0))
    if name == "cfg3":
        return lj_fluid_config(16384, 0.8, 5.0, seed=kw.get("seed", 0), dt=0.005,
                               steps=kw.get("steps", 1000), side=26, name="cfg3")
    if name == "cfg4":
        return replica_batch_config(kw.get("replicas", 8), kw.get("first_seed", 0),
                                    kw.get("steps", 500))
    raise ValueError(f"unknown config {name}")
