"""RdfHistogram host arithmetic of the reference (structure.cpp:78-194),
restated for the TESTS only: finalize / first_minimum / solvation_number are
host code of the reference (out of the GPU path's scope); the tests use this
restatement, pinned bit-exact to the reference's outputs in
tests/test_rdf_oracle.py, to check the device counts end to end.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from paper_1507_07548_b200.errors import Error


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
