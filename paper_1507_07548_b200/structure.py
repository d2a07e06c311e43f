"""Radial distribution functions: the host mirror of tmd's structure module
(include/tmd/structure.hpp, src/structure.cpp).

The O(N^2 s^2) histogram accumulation runs on the GPU (b2md_rdf_*, csrc/rdf.cuh);
the integer counts are bit-exact with the reference.  finalize, first_minimum,
solvation_number and the serialize byte format are the reference's host
arithmetic, restated here with the same operation order.
"""
from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigError, Error, IoError, check
from .model import SystemComposition, SystemState


@dataclass
class RdfTable:  # structure.hpp:18-27
    label_a: str = ""
    label_b: str = ""
    species_a: int = 0
    species_b: int = 0
    r_mid: list = field(default_factory=list)
    g: list = field(default_factory=list)
    n_cum: list = field(default_factory=list)
    bin_width: float = 0.0
    partner_density: float = 0.0
    snapshots: int = 0


def rdf_site_types(comp: SystemComposition) -> list[tuple[int, int, str]]:
    """structure.cpp:17-32: (species, site, label) of every LJ / dummy site in
    (species, site) order; charge-only sites are not sampling centres."""
    out = []
    for s, sp in enumerate(comp.species):
        for k, site in enumerate(sp.sites):
            if int(site.kind) != 1:  # SiteKind::charge
                out.append((s, k, sp.name + str(k + 1)))
    return out


def finalize_tables(comp: SystemComposition, types, bin_width: float, r_max: float,
                    counts: np.ndarray, snapshots: int) -> list[RdfTable]:
    """RdfHistogram::finalize (structure.cpp:78-128) on [pair][bin] counts."""
    if snapshots < 1:
        raise Error("rdf: no snapshots accumulated")
    volume = comp.box_length * comp.box_length * comp.box_length  # model.hpp:63
    bins = counts.shape[1] if counts.ndim == 2 else 0
    T = len(types)
    tables = []
    for ta in range(T):
        for tb in range(ta, T):
            sa, _, la = types[ta]
            sb, _, lb = types[tb]
            n_a = float(comp.counts[sa])
            n_b = float(comp.counts[sb])
            if sa != sb:
                norm_pairs = n_a * n_b
            elif ta != tb:
                norm_pairs = n_a * (n_a - 1.0)
            else:
                norm_pairs = n_a * (n_a - 1.0) / 2.0
            if norm_pairs <= 0.0:
                continue
            tab = RdfTable(la, lb, sa, sb, bin_width=bin_width, snapshots=snapshots)
            tab.partner_density = ((n_b - 1.0) if sa == sb else n_b) / volume
            cnt = counts[ta * T - ta * (ta + 1) // 2 + tb]
            cum_pairs = 0.0
            center_count = n_a
            multiplicity = 2.0 if ta == tb else 1.0
            for b in range(bins):
                r_lo = b * bin_width
                r_hi = min((b + 1) * bin_width, r_max)
                shell = 4.0 * math.pi / 3.0 * (r_hi * r_hi * r_hi - r_lo * r_lo * r_lo)
                mean_count = float(cnt[b]) / float(snapshots)
                tab.r_mid.append(0.5 * (r_lo + r_hi))
                tab.g.append(mean_count * volume / (norm_pairs * shell))
                cum_pairs += mean_count
                tab.n_cum.append(cum_pairs * multiplicity / center_count)
            tables.append(tab)
    return tables


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

    def finalize(self, replica: int = 0) -> list[RdfTable]:
        """structure.cpp:78-128."""
        counts, snaps = self.counts(replica)
        return finalize_tables(self.comp, self.types, self.bin_width, self.r_max, counts, snaps)

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


def first_minimum(r_mid, g) -> float:
    """structure.cpp:157-182: first local minimum after the first peak above 1
    of the 3-point smoothed g; NaN when there is none."""
    n = len(g)
    if n < 5:
        return math.nan
    smooth = [0.0] * n
    for i in range(n):
        lo, hi = max(0, i - 1), min(n - 1, i + 1)
        s = 0.0
        for k in range(lo, hi + 1):
            s += g[k]
        smooth[i] = s / (hi - lo + 1)
    peak = -1
    for i in range(1, n - 1):
        if smooth[i] > 1.0 and smooth[i] >= smooth[i - 1] and smooth[i] > smooth[i + 1]:
            peak = i
            break
    if peak < 0:
        return math.nan
    for i in range(peak + 1, n - 1):
        if smooth[i] <= smooth[i - 1] and smooth[i] < smooth[i + 1]:
            return r_mid[i]
    return math.nan


def solvation_number(table: RdfTable, partner_density: float, r_min: float) -> float:
    """structure.cpp:184-194."""
    n = 0.0
    for b in range(len(table.g)):
        r_lo = b * table.bin_width
        r_hi = min((b + 1) * table.bin_width, r_min)
        if r_hi <= r_lo:
            break
        shell = 4.0 * math.pi / 3.0 * (r_hi * r_hi * r_hi - r_lo * r_lo * r_lo)
        n += partner_density * table.g[b] * shell
    return n
