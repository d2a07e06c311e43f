"""Radial distribution functions: the host mirror of tmd's structure module
(include/tmd/structure.hpp, src/structure.cpp).

The O(N^2 s^2) histogram accumulation runs on the GPU (b2md_rdf_*, csrc/rdf.cuh);
the integer counts are bit-exact with the reference.  serialize() writes them
in RdfHistogram::serialize's byte layout (structure.cpp:130-140), which the
reference's own RdfHistogram::deserialize reads: finalize, first_minimum and
solvation_number (structure.cpp:78-194) stay the reference's host code
(integration/tmd_gpu.hpp hands the counts to it).
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _abi
from .errors import ConfigError, Error, IoError, check
from .model import SystemComposition, SystemState


def rdf_site_types(comp: SystemComposition) -> list[tuple[int, int, str]]:
    """structure.cpp:17-32: (species, site, label) of every LJ / dummy site in
    (species, site) order; charge-only sites are not sampling centres."""
    out = []
    for s, sp in enumerate(comp.species):
        for k, site in enumerate(sp.sites):
            if int(site.kind) != 1:  # SiteKind::charge
                out.append((s, k, sp.name + str(k + 1)))
    return out


def serialize_counts(bin_width: float, r_max: float, bins: int, snapshots: int,
                     counts: np.ndarray) -> bytes:
    """RdfHistogram::serialize (structure.cpp:130-140), little-endian
    ByteWriter layout (checkpoint.hpp:15-38)."""
    npairs = counts.shape[0]
    out = [struct.pack("<ddIqQ", bin_width, r_max, bins, snapshots, npairs)]
    for p in range(npairs):
        out.append(struct.pack("<Q", bins))
        out.append(np.ascontiguousarray(counts[p], dtype="<u8").tobytes())
    return b"".join(out)


class RdfHistogram:
    """tmd::RdfHistogram (structure.hpp:29-67) on a ForceField's or Engine's
    device context: one histogram per replica."""

    def __init__(self, owner, bin_width: float, r_max: float):
        self._owner = owner  # keeps the context alive
        self._c = owner._c
        self.comp: SystemComposition = self._c.comp
        h = C.c_void_p()
        check(_abi.lib().b2md_rdf_create(self._c.ctx, float(bin_width), float(r_max), C.byref(h)))
        self._h = h
        self.bin_width = float(bin_width)
        self.r_max = float(r_max)
        t, b, p = C.c_int(), C.c_int(), C.c_int()
        check(_abi.lib().b2md_rdf_shape(self._h, C.byref(t), C.byref(b), C.byref(p)))
        self._types, self._bins, self._pairs = t.value, b.value, p.value
        sp = (C.c_int * max(1, self._types))()
        st = (C.c_int * max(1, self._types))()
        check(_abi.lib().b2md_rdf_types(self._h, sp, st))
        # labels "<species><siteOrdinal>" (structure.cpp:27)
        self.types = [(sp[k], st[k], self.comp.species[sp[k]].name + str(st[k] + 1))
                      for k in range(self._types)]

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _abi.lib().b2md_rdf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bins(self) -> int:
        return self._bins

    def site_type_count(self) -> int:
        return self._types

    def pair_index(self, ta: int, tb: int) -> int:  # structure.hpp:51-54, ta <= tb
        return ta * self._types - ta * (ta + 1) // 2 + tb

    def accumulate(self, state: SystemState | None = None) -> None:
        """structure.cpp:38-76.  With `state` None the context's device state
        (an Engine's current one, every replica) is sampled."""
        if state is None:
            check(_abi.lib().b2md_rdf_accumulate(self._h))
            return
        n = self.comp.molecule_count()
        pos = np.ascontiguousarray(state.pos, dtype=np.float64).reshape(n, 3)
        orient = np.ascontiguousarray(state.orient, dtype=np.float64).reshape(n, 4)
        check(_abi.lib().b2md_rdf_accumulate_state(self._h, _abi.dptr(pos), _abi.dptr(orient)))

    def counts(self, replica: int = 0) -> tuple[np.ndarray, int]:
        out = np.zeros((self._pairs, self._bins), dtype=np.uint64)
        snaps = C.c_int64()
        check(_abi.lib().b2md_rdf_counts(self._h, replica,
                                         out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(snaps)))
        return out, snaps.value

    def snapshots(self, replica: int = 0) -> int:
        return self.counts(replica)[1]

    def serialize(self, replica: int = 0) -> bytes:
        """structure.cpp:130-140 byte layout."""
        counts, snaps = self.counts(replica)
        return serialize_counts(self.bin_width, self.r_max, self._bins, snaps, counts)

    def deserialize(self, data: bytes, replica: int = 0) -> int:
        """Restores the counts; returns the number of bytes consumed."""
        need = 36
        if len(data) < need:
            raise IoError("checkpoint: truncated or corrupted data")
        bw, rm, bins, snaps, npairs = struct.unpack_from("<ddIqQ", data, 0)
        if npairs != self._pairs:
            raise IoError("rdf: checkpoint does not match the composition")
        o = 36
        counts = np.zeros((self._pairs, bins), dtype=np.uint64)
        for p in range(self._pairs):
            if len(data) < o + 8:
                raise IoError("checkpoint: truncated or corrupted data")
            (nb,) = struct.unpack_from("<Q", data, o)
            if nb != self._bins or nb != bins:
                raise IoError("rdf: corrupted bin count")
            if len(data) < o + 8 + 8 * nb:
                raise IoError("checkpoint: truncated or corrupted data")
            counts[p] = np.frombuffer(data, "<u8", nb, o + 8)
            o += 8 + 8 * nb
        self.bin_width, self.r_max = bw, rm
        check(_abi.lib().b2md_rdf_set_counts(
            self._h, replica, np.ascontiguousarray(counts).ctypes.data_as(C.POINTER(C.c_uint64)),
            int(snaps)))
        return o
