"""Model types mirroring include/tmd/model.hpp and include/tmd/energy.hpp.

Species are built by the native library (b2md_build_species restates
tmd::build_species, src/model.cpp:68-129, bit for bit).  States are numpy
arrays in the reference's AoS layouts: pos/vel/ang_vel/force/torque are
(n, 3) float64, orient is (n, 4) (w, x, y, z) — include/tmd/geom.hpp:9-38.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import check


class SiteKind(enum.IntEnum):  # model.hpp:16
    lj = _abi.SITE_LJ
    charge = _abi.SITE_CHARGE
    dummy = _abi.SITE_DUMMY


class ElectrostaticsMethod(enum.IntEnum):  # model.hpp:52
    none = _abi.METHOD_NONE
    reaction_field = _abi.METHOD_REACTION_FIELD
    ewald = _abi.METHOD_EWALD


@dataclass
class Site:  # model.hpp:18-25
    kind: SiteKind = SiteKind.lj
    body_pos: tuple = (0.0, 0.0, 0.0)
    sigma: float = 0.0
    epsilon: float = 0.0
    q: float = 0.0
    mass: float = 0.0

    def to_c(self) -> _abi.b2md_site:
        s = _abi.b2md_site()
        s.kind = int(self.kind)
        s.body_pos[:] = [float(v) for v in self.body_pos]
        s.sigma, s.epsilon, s.q, s.mass = self.sigma, self.epsilon, self.q, self.mass
        return s


def make_lj_site(x, y, z, sigma, eps, mass) -> Site:
    return Site(SiteKind.lj, (x, y, z), sigma, eps, 0.0, mass)


def make_charge_site(x, y, z, q, mass) -> Site:
    return Site(SiteKind.charge, (x, y, z), 0.0, 0.0, q, mass)


class MoleculeSpecies:
    """A built species (model.hpp:29-40), backed by the C struct."""

    def __init__(self, name: str, c: _abi.b2md_species):
        self.name = name
        self.c = c

    @property
    def n_sites(self) -> int:
        return self.c.n_sites

    def site_count(self) -> int:
        return self.c.n_sites

    @property
    def sites(self) -> list[Site]:
        out = []
        for k in range(self.c.n_sites):
            s = self.c.sites[k]
            out.append(Site(SiteKind(s.kind), tuple(s.body_pos), s.sigma, s.epsilon, s.q, s.mass))
        return out

    @property
    def total_mass(self) -> float:
        return self.c.total_mass

    @property
    def inertia_principal(self) -> np.ndarray:
        return np.array(self.c.inertia_principal[:], dtype=np.float64)

    @property
    def rotational_dof(self) -> int:
        return self.c.rotational_dof

    @property
    def max_extent(self) -> float:
        return self.c.max_extent

    @property
    def net_charge(self) -> float:
        return self.c.net_charge

    def has_charges(self) -> bool:
        return any(s.q != 0.0 for s in self.sites)


def build_species(name: str, sites: list[Site]) -> MoleculeSpecies:
    """tmd::build_species (src/model.cpp:68-129) via b2md_build_species."""
    arr = (_abi.b2md_site * max(len(sites), 1))(*[s.to_c() for s in sites])
    out = _abi.b2md_species()
    check(_abi.lib().b2md_build_species(arr, len(sites), C.byref(out)))
    return MoleculeSpecies(name, out)


@dataclass
class SystemComposition:  # model.hpp:54-72
    species: list = field(default_factory=list)
    counts: list = field(default_factory=list)
    box_length: float = 0.0
    temperature: float = 0.0

    def species_count(self) -> int:
        return len(self.species)

    def molecule_count(self) -> int:
        return int(sum(self.counts))

    def volume(self) -> float:
        return self.box_length * self.box_length * self.box_length

    def species_of_molecule(self, mol: int) -> int:
        off = 0
        for s, c in enumerate(self.counts):
            off += c
            if mol < off:
                return s
        raise IndexError("molecule index out of range")

    def species_index(self) -> np.ndarray:
        return np.repeat(np.arange(len(self.counts)), self.counts)

    def to_c(self):
        """Returns (struct, keepalive) — the struct points into keepalive."""
        sp = (_abi.b2md_species * max(len(self.species), 1))(*[s.c for s in self.species])
        counts = (C.c_int32 * max(len(self.counts), 1))(*[int(c) for c in self.counts])
        c = _abi.b2md_composition()
        c.n_species = len(self.species)
        c.species = C.cast(sp, C.POINTER(_abi.b2md_species))
        c.counts = C.cast(counts, C.POINTER(C.c_int32))
        c.box_length = float(self.box_length)
        c.temperature = float(self.temperature)
        return c, (sp, counts)


_ENERGY_FIELDS = [f for f, _ in _abi.b2md_energy._fields_]


@dataclass
class EnergyBreakdown:  # energy.hpp:9-25
    lj: float = 0.0
    elec_real: float = 0.0
    elec_recip: float = 0.0
    elec_self: float = 0.0
    rf: float = 0.0
    lrc: float = 0.0
    du_dv_explicit: float = 0.0
    du_dv_lrc: float = 0.0
    d2u_dv2_explicit: float = 0.0
    d2u_dv2_lrc: float = 0.0

    def total(self) -> float:
        return self.lj + self.elec_real + self.elec_recip + self.elec_self + self.rf + self.lrc

    def du_dv(self) -> float:
        return self.du_dv_explicit + self.du_dv_lrc

    def d2u_dv2(self) -> float:
        return self.d2u_dv2_explicit + self.d2u_dv2_lrc

    @classmethod
    def from_c(cls, e: _abi.b2md_energy) -> "EnergyBreakdown":
        return cls(**{f: getattr(e, f) for f in _ENERGY_FIELDS})

    @classmethod
    def list_from_c(cls, e_arr, count: int) -> list["EnergyBreakdown"]:
        """`count` b2md_energy structs (all doubles, in field order) in one pass."""
        nf = len(_ENERGY_FIELDS)
        vals = np.frombuffer(e_arr, dtype=np.float64, count=count * nf).tolist()
        return [cls(*vals[r * nf:(r + 1) * nf]) for r in range(count)]


class SystemState:
    """model.hpp:75-92 with numpy arrays."""

    def __init__(self, n: int = 0, box_length: float = 0.0):
        self.pos = np.zeros((n, 3))
        self.orient = np.zeros((n, 4))
        self.orient[:, 0] = 1.0
        self.vel = np.zeros((n, 3))
        self.ang_vel = np.zeros((n, 3))
        self.box_length = float(box_length)
        self.force = np.zeros((n, 3))
        self.torque = np.zeros((n, 3))
        self.energy = EnergyBreakdown()
        self.virial = 0.0

    def molecule_count(self) -> int:
        return self.pos.shape[0]

    def copy(self) -> "SystemState":
        s = SystemState(0, self.box_length)
        for k in ("pos", "orient", "vel", "ang_vel", "force", "torque"):
            setattr(s, k, getattr(self, k).copy())
        s.energy = EnergyBreakdown(**vars(self.energy))
        s.virial = self.virial
        return s

    def wrap(self) -> None:  # model.cpp:279-286
        L = self.box_length
        self.pos -= L * np.floor(self.pos / L)


# kinetic bookkeeping (model.cpp:304-337), host-side scalars for checks
def kinetic_energy_trans(comp: SystemComposition, state: SystemState) -> float:
    m = np.array([comp.species[s].total_mass for s in comp.species_index()])
    return float(np.sum(0.5 * m * np.sum(state.vel * state.vel, axis=1)))


def kinetic_energy_rot(comp: SystemComposition, state: SystemState) -> float:
    inertia = np.array([comp.species[s].inertia_principal for s in comp.species_index()])
    return float(np.sum(0.5 * np.sum(inertia * state.ang_vel * state.ang_vel, axis=1)))


def translational_dof(comp: SystemComposition) -> int:
    return 3 * comp.molecule_count() - 3


def rotational_dof(comp: SystemComposition) -> int:
    return int(sum(c * s.rotational_dof for s, c in zip(comp.species, comp.counts)))
