"""TEST INFRASTRUCTURE (not the product): the reference's host samplers
restated to check the device scalars against the reference's bytes.
Scalar sampling of tmd::Engine::run (src/engine.cpp:218-229) and the
Massieu derivative accumulator it feeds (src/massieu.cpp:9-70, 148-190):
host arithmetic on the few scalars a step produces on the device (kinetic
energies, U, dU/dV, d2U/dV2, virial).  The reference's operation order is
kept, so the accumulators serialize to the reference's bytes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from host_checkpoint import BlockStat, ByteReader, ByteWriter
from paper_1507_07548_b200.errors import ConfigError, IoError, NumericalError


def block_stat_add(b: BlockStat, x: float) -> None:
    """BlockStat::add (results.hpp:30-37)."""
    k = 0
    if b.expected > 0:
        k = (b.total * b.n_blocks) // b.expected
    if k >= b.n_blocks:
        k = b.n_blocks - 1
    b.sum[k] += x
    b.cnt[k] += 1
    b.total += 1


BlockStat.add = block_stat_add


@dataclass
class _Moments:  # massieu.hpp:59-69
    n: int = 0
    x: float = 0.0
    x2: float = 0.0
    x3: float = 0.0
    y: float = 0.0
    yx: float = 0.0
    yx2: float = 0.0
    y2: float = 0.0
    y2x: float = 0.0
    z: float = 0.0
    zx: float = 0.0

    def add(self, xs, ys, zs):  # massieu.cpp:22-35
        self.n += 1
        w = 1.0 / float(self.n)
        self.x += (xs - self.x) * w
        self.x2 += (xs * xs - self.x2) * w
        self.x3 += (xs * xs * xs - self.x3) * w
        self.y += (ys - self.y) * w
        self.yx += (ys * xs - self.yx) * w
        self.yx2 += (ys * xs * xs - self.yx2) * w
        self.y2 += (ys * ys - self.y2) * w
        self.y2x += (ys * ys * xs - self.y2x) * w
        self.z += (zs - self.z) * w
        self.zx += (zs * xs - self.zx) * w


@dataclass
class DerivativeAccumulator:
    """tmd::DerivativeAccumulator (massieu.hpp:41-80): block moments of
    (U, dU/dV, d2U/dV2) for the Massieu derivatives."""
    beta: float = 0.0
    volume: float = 0.0
    n_molecules: int = 0
    n_blocks: int = 1
    expected: int = 0
    total: int = 0
    shift_set: bool = False
    shift_u: float = 0.0
    shift_uv: float = 0.0
    shift_uvv: float = 0.0
    blocks: list = field(default_factory=list)

    @classmethod
    def create(cls, temperature: float, volume: float, n_molecules: int, n_blocks: int = 10,
               expected_samples: int = 0) -> "DerivativeAccumulator":
        """massieu.cpp:9-20."""
        if temperature <= 0.0 or volume <= 0.0 or n_molecules <= 0:
            raise ConfigError("derivative accumulator: bad state constants")
        nb = n_blocks if expected_samples > 0 else 1
        nb = max(1, nb)
        return cls(1.0 / temperature, volume, n_molecules, nb, expected_samples,
                   blocks=[_Moments() for _ in range(nb)])

    def add(self, u: float, du_dv: float, d2u_dv2: float) -> None:
        """massieu.cpp:53-70."""
        if not (math.isfinite(u) and math.isfinite(du_dv) and math.isfinite(d2u_dv2)):
            raise NumericalError("derivative accumulator: non-finite snapshot")
        if not self.shift_set:
            self.shift_u, self.shift_uv, self.shift_uvv = u, du_dv, d2u_dv2
            self.shift_set = True
        block = 0
        if self.expected > 0 and self.expected > 1:
            block = (self.total * self.n_blocks) // self.expected
        if block >= self.n_blocks:
            block = self.n_blocks - 1
        self.blocks[block].add(u - self.shift_u, du_dv - self.shift_uv, d2u_dv2 - self.shift_uvv)
        self.total += 1

    def samples(self) -> int:
        return self.total

    def serialize(self, w: ByteWriter) -> None:  # massieu.cpp:148-163
        w.f64(self.beta)
        w.f64(self.volume)
        w.i64(self.n_molecules)
        w.u32(self.n_blocks)
        w.i64(self.expected)
        w.i64(self.total)
        w.u8(1 if self.shift_set else 0)
        w.f64(self.shift_u)
        w.f64(self.shift_uv)
        w.f64(self.shift_uvv)
        for b in self.blocks:
            w.i64(b.n)
            for v in (b.x, b.x2, b.x3, b.y, b.yx, b.yx2, b.y2, b.y2x, b.z, b.zx):
                w.f64(v)

    @classmethod
    def deserialize(cls, r: ByteReader) -> "DerivativeAccumulator":  # massieu.cpp:165-190
        a = cls()
        a.beta, a.volume, a.n_molecules = r.f64(), r.f64(), r.i64()
        a.n_blocks, a.expected, a.total = r.u32(), r.i64(), r.i64()
        a.shift_set = r.u8() != 0
        a.shift_u, a.shift_uv, a.shift_uvv = r.f64(), r.f64(), r.f64()
        a.blocks = []
        for _ in range(a.n_blocks):
            m = _Moments(r.i64())
            (m.x, m.x2, m.x3, m.y, m.yx, m.yx2, m.y2, m.y2x, m.z, m.zx) = (r.f64() for _ in range(10))
            a.blocks.append(m)
        return a


def accumulate_scalars(comp, ke_trans: float, ke_rot: float, energy, virial: float, stats) -> None:
    """Engine::accumulate_scalars (engine.cpp:218-225) into the four
    BlockStats (tkin, tkin_rot, u, virial)."""
    dof_t = 3 * comp.molecule_count() - 3  # model.cpp:321-323
    stats[0].add(2.0 * ke_trans / dof_t)
    dof_r = sum(c * sp.rotational_dof for c, sp in zip(comp.counts, comp.species))
    if dof_r > 0:
        stats[1].add(2.0 * ke_rot / dof_r)
    stats[2].add(energy.total())
    stats[3].add(virial)
