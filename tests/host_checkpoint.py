"""TEST INFRASTRUCTURE (not the product): the checkpoint container of
tmd::Engine restated to check the device state block inside the reference's
full checkpoint bytes.  Checkpoint / restart byte format of tmd::Engine (src/engine.cpp:420-541,
include/tmd/checkpoint.hpp:15-100, src/results.cpp:39-57).

The container is host data except its state block (u32 n, f64 box, 13 x f64
per molecule), which is packed and restored on the device through the C ABI
(b2md_save_state_block / b2md_restore_state_block).  Sampler sections this
path does not run (Massieu, correlation sets, residence) are carried as the
exact byte spans of their serialized form, parsed only to find their extent,
so a reference checkpoint round-trips byte for byte; the RDF sections are
the RdfHistogram format (paper_1507_07548_b200.structure).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from paper_1507_07548_b200.configs import Rng
from paper_1507_07548_b200.errors import IoError

MAGIC = b"TMDCKPT1"
VERSION = 1


class ByteWriter:  # checkpoint.hpp:15-38 (little-endian raw host bytes)
    def __init__(self):
        self._b = bytearray()

    def u8(self, v):
        self._b += struct.pack("<B", v)

    def u32(self, v):
        self._b += struct.pack("<I", v)

    def u64(self, v):
        self._b += struct.pack("<Q", v)

    def i64(self, v):
        self._b += struct.pack("<q", v)

    def f64(self, v):
        self._b += struct.pack("<d", v)

    def str(self, s: str):
        b = s.encode()
        self.u64(len(b))
        self._b += b

    def f64_vec(self, v):
        self.u64(len(v))
        self._b += np.ascontiguousarray(v, dtype="<f8").tobytes()

    def bytes(self, b: bytes):
        self._b += b

    def data(self) -> bytes:
        return bytes(self._b)


class ByteReader:  # checkpoint.hpp:40-100
    def __init__(self, data: bytes, pos: int = 0):
        self.data = data
        self.pos = pos

    def need(self, n: int):
        if n < 0 or self.pos + n > len(self.data):
            raise IoError(f"checkpoint: truncated or corrupted data (need {n} bytes at offset {self.pos})")

    def _take(self, n: int) -> bytes:
        self.need(n)
        b = self.data[self.pos:self.pos + n]
        self.pos += n
        return b

    def u8(self):
        return self._take(1)[0]

    def u32(self):
        return struct.unpack("<I", self._take(4))[0]

    def u64(self):
        return struct.unpack("<Q", self._take(8))[0]

    def i64(self):
        return struct.unpack("<q", self._take(8))[0]

    def f64(self):
        return struct.unpack("<d", self._take(8))[0]

    def str(self) -> str:
        n = self.u64()
        return self._take(n).decode()

    def f64_vec(self):
        n = self.u64()
        if n > (len(self.data) - self.pos) // 8:
            self.need(8 * n)
        return list(np.frombuffer(self._take(8 * n), dtype="<f8"))

    def bytes(self, n: int) -> bytes:
        return self._take(n)

    def elements(self, count: int, size: int) -> bytes:
        """`count` reads of `size` bytes each, as the reference's element
        loops do: a truncation fails at the first element that does not fit."""
        avail = (len(self.data) - self.pos) // size
        if count > avail:
            self.pos += avail * size
            self.need(size)
        return self._take(count * size)

    def at_end(self) -> bool:
        return self.pos == len(self.data)


@dataclass
class BlockStat:  # results.hpp:21-51, serialize results.cpp:39-57
    n_blocks: int = 1
    expected: int = 0
    total: int = 0
    sum: list = field(default_factory=lambda: [0.0])
    cnt: list = field(default_factory=lambda: [0])

    @classmethod
    def fresh(cls, n_blocks: int = 10, expected: int = 0) -> "BlockStat":
        nb = n_blocks if expected > 0 else 1
        nb = max(1, nb)
        return cls(nb, expected, 0, [0.0] * nb, [0] * nb)

    def serialize(self, w: ByteWriter):
        w.u32(self.n_blocks)
        w.i64(self.expected)
        w.i64(self.total)
        w.f64_vec(self.sum)
        w.u64(len(self.cnt))
        for v in self.cnt:
            w.i64(v)

    @classmethod
    def deserialize(cls, r: ByteReader) -> "BlockStat":
        nb = r.u32()
        expected = r.i64()
        total = r.i64()
        s = r.f64_vec()
        n = r.u64()
        cnt = list(np.frombuffer(r.elements(n, 8), dtype="<i8").astype(int))
        if nb < 1 or len(s) != nb or len(cnt) != len(s):
            raise IoError("block stat: corrupted payload")
        return cls(nb, expected, total, s, cnt)


# ---- extents of sampler sections, read with the reference's deserializers'
# granularity and checks (so truncations fail with the same message)
def _span(r: ByteReader, parse) -> bytes:
    start = r.pos
    parse(r)
    return r.data[start:r.pos]


def _derivative_accumulator(r: ByteReader):  # massieu.cpp:165-190
    r.f64(), r.f64(), r.i64()
    nb = r.u32()
    r.i64(), r.i64(), r.u8(), r.f64(), r.f64(), r.f64()
    r.elements(nb * 11, 8)


def _correlation_set(r: ByteReader):  # greenkubo.cpp:115-138
    dim, length, nb = r.u32(), r.u32(), r.u32()
    r.i64()
    pushes = r.i64()
    if dim < 1 or length < 2 or nb < 1 or pushes < 0:
        raise IoError("correlation set: corrupted header")
    ring, weight = r.f64_vec(), r.f64_vec()
    nv = r.u64()
    r.elements(nv, 1)
    acf = r.f64_vec()
    nc = r.u64()
    r.elements(nc, 8)
    if (len(ring) != length * dim or len(weight) != length or nv != length or
            len(acf) != nb * length or nc != len(acf)):
        raise IoError("correlation set: corrupted payload length")


def _residence(r: ByteReader):  # greenkubo.cpp:435-456
    ns, nv = r.u32(), r.u32()
    r.u32(), r.u32(), r.i64(), r.i64()
    if ns < 1 or nv < 1:
        raise IoError("residence tracker: corrupted header")
    r.elements(r.u64() * ns * nv, 1)
    r.elements(r.u64(), 8)
    for _ in range(ns):
        _correlation_set(r)


def _rdf(r: ByteReader):  # structure.cpp:142-153 (pair / bin counts checked by the owner)
    r.f64(), r.f64(), r.u32(), r.i64()
    for _ in range(r.u64()):
        r.elements(r.u64(), 8)


@dataclass
class EngineCheckpoint:
    """Everything Engine::checkpoint_bytes writes (engine.cpp:420-462)."""
    config_text: str = ""
    seed: int = 0
    equil_done: int = 0
    prod_done: int = 0
    rng_state: tuple = (0, 0, 0, 0)
    box_length: float = 0.0
    state: np.ndarray = field(default_factory=lambda: np.zeros((0, 13)))  # pos, q.wxyz, vel, w
    stats: list = field(default_factory=lambda: [BlockStat() for _ in range(4)])  # tkin, tkin_rot, u, virial
    samplers_ready: bool = False
    residence_radius_used: float = 0.0
    massieu: bytes | None = None
    je_corr: bytes | None = None
    jq_corr: bytes | None = None
    vacf: list = field(default_factory=list)
    residence: bytes | None = None
    rdf: bytes | None = None
    rdf_prepass: bytes | None = None

    @classmethod
    def fresh(cls, seed: int, n_blocks: int = 10, n_production: int = 0,
              config_text: str = "") -> "EngineCheckpoint":
        """The metadata of an Engine right after construction (engine.cpp:
        63-89): seeded RNG (rng.hpp), empty block statistics, no samplers."""
        return cls(config_text=config_text, seed=seed, rng_state=tuple(Rng(seed).s),
                   stats=[BlockStat.fresh(n_blocks, n_production) for _ in range(4)])

    # --- the state block (engine.cpp:432-441)
    def state_block(self) -> bytes:
        return (struct.pack("<Id", self.state.shape[0], self.box_length) +
                np.ascontiguousarray(self.state, dtype="<f8").tobytes())

    def set_state_block(self, block: bytes):
        r = ByteReader(block)
        n = r.u32()
        self.box_length = r.f64()
        raw = r.bytes(104 * n)
        self.state = np.frombuffer(raw, dtype="<f8").reshape(n, 13).copy()

    def to_bytes(self) -> bytes:
        w = ByteWriter()
        w.bytes(MAGIC)
        w.u32(VERSION)
        w.str(self.config_text)
        w.u64(self.seed)
        w.i64(self.equil_done)
        w.i64(self.prod_done)
        for word in self.rng_state:
            w.u64(word)
        w.bytes(self.state_block())
        for s in self.stats:
            s.serialize(w)
        w.u8(1 if self.samplers_ready else 0)
        w.f64(self.residence_radius_used)
        for sec in (self.massieu, self.je_corr, self.jq_corr):
            w.u8(1 if sec is not None else 0)
            if sec is not None:
                w.bytes(sec)
        w.u32(len(self.vacf))
        for v in self.vacf:
            w.bytes(v)
        for sec in (self.residence, self.rdf, self.rdf_prepass):
            w.u8(1 if sec is not None else 0)
            if sec is not None:
                w.bytes(sec)
        w.bytes(b"END!")
        return w.data()

    @classmethod
    def from_bytes(cls, data: bytes, n_molecules: int | None = None) -> "EngineCheckpoint":
        """The container header, then restore_dynamic's reads (engine.cpp:
        472-537) with the reference's IoError messages."""
        r = ByteReader(data)
        if r.bytes(8) != MAGIC:
            raise IoError("checkpoint: bad magic")
        if r.u32() != VERSION:
            raise IoError("checkpoint: unsupported version")
        c = cls(config_text=r.str())
        c.seed, c.equil_done, c.prod_done = r.u64(), r.i64(), r.i64()
        c.rng_state = tuple(r.u64() for _ in range(4))
        n = r.u32()
        if n_molecules is not None and n != n_molecules:
            raise IoError("checkpoint: molecule count mismatch")
        c.box_length = r.f64()
        c.state = np.frombuffer(r.elements(13 * n, 8), dtype="<f8").reshape(n, 13).copy()
        c.stats = [BlockStat.deserialize(r) for _ in range(4)]
        c.samplers_ready = r.u8() != 0
        c.residence_radius_used = r.f64()
        c.massieu = _span(r, _derivative_accumulator) if r.u8() else None
        c.je_corr = _span(r, _correlation_set) if r.u8() else None
        c.jq_corr = _span(r, _correlation_set) if r.u8() else None
        c.vacf = [_span(r, _correlation_set) for _ in range(r.u32())]
        c.residence = _span(r, _residence) if r.u8() else None
        c.rdf = _span(r, _rdf) if r.u8() else None
        c.rdf_prepass = _span(r, _rdf) if r.u8() else None
        if r.bytes(4) != b"END!":
            raise IoError("checkpoint: missing end marker")
        return c


def checkpoint_bytes(engine, meta=None, replica: int = 0) -> bytes:
    """Engine::checkpoint_bytes: `meta` (header, counters, RNG, statistics,
    sampler sections) around the engine's device-packed state block."""
    meta = meta if meta is not None else EngineCheckpoint.fresh(0)
    meta.set_state_block(engine.state_block(replica))
    return meta.to_bytes()


def restore_checkpoint(engine, data: bytes, replica: int = 0):
    """Parses a checkpoint container and restores its state block into the
    engine's `replica` on the device; returns the host-side metadata."""
    meta = EngineCheckpoint.from_bytes(data, engine._c.n)
    engine.restore_state_block(meta.state_block(), replica)
    return meta
