"""CPU: the C-ABI library loads, exports every symbol include/b200md.h
declares, its host-only entry points (species building, Ewald tuning, shard
plans, configuration validation) match the reference, and device entry
points fail loudly without a GPU (there is no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1507_07548_b200 as b2
from oracle import pyoracle
from paper_1507_07548_b200 import _abi

import golden_cases
import systems

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def declared_symbols():
    text = (ROOT / "include" / "b200md.h").read_text()
    return sorted(set(re.findall(r"\b(b2md_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _abi.SIGNATURES, f"{name} missing from the ctypes mirror"
    assert lib.b2md_abi_version() == 1


def test_struct_layouts():
    assert C.sizeof(_abi.b2md_site) == 64
    assert C.sizeof(_abi.b2md_energy) == 80
    assert C.sizeof(_abi.b2md_ff_options) == 48


@pytest.mark.parametrize("name", list(golden_cases.species_cases()))
def test_build_species_bitexact(name):
    g = np.load(GOLDEN / "species.npz")
    sp = b2.build_species(name, golden_cases.species_cases()[name])
    body = np.array([s.body_pos for s in sp.sites])
    assert np.array_equal(body, g[name + "_body"])
    assert np.array_equal(sp.inertia_principal, g[name + "_inertia"])
    assert np.array_equal([sp.total_mass, sp.net_charge, sp.max_extent, sp.rotational_dof],
                          g[name + "_scalars"])


def test_build_species_errors():  # model.cpp:69-84
    with pytest.raises(b2.ModelError):
        b2.build_species("empty", [])
    with pytest.raises(b2.ModelError):
        b2.build_species("d", [b2.Site(b2.SiteKind.dummy, (0, 0, 0), 1.0, 0.0, 0.0, 1.0)])
    with pytest.raises(b2.ModelError):
        b2.build_species("s", [b2.make_lj_site(0, 0, 0, -1.0, 1.0, 1.0)])
    with pytest.raises(b2.ModelError):
        b2.build_species("m", [b2.make_lj_site(0, 0, 0, 1.0, 1.0, 0.0)])


def test_ewald_tune_and_kvectors():
    for args in [(1e-6, 2.0, 4.0), (1e-6, 3.0, 6.0), (1e-4, 5.0, 10.0)]:
        p = b2.ewald_tune(*args)
        assert (p.alpha, p.kmax) == pyoracle.ewald_tune(*args, which="oracle")
    with pytest.raises(b2.ConfigError):
        b2.ewald_tune(0.5, 5.0, 10.0)
    with pytest.raises(b2.ConfigError):
        b2.ewald_tune(0.0, 5.0, 10.0)
    # spherical half-space rule of ewald.cpp:77-104: 709 vectors at kmax = 7
    assert b2.kvector_count(7) == 709
    assert b2.kvector_count(1) == 3


def _gpu_present() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_config_errors_match_reference():
    """ConfigError cases of PairTable / validate / ForceField ctor are raised
    before any device work, exactly where the reference throws."""
    comp = systems.lj_fluid(10, 5.0)
    cases = [
        (comp, systems.lj_opts(2.6)),                                      # rc > L/2
        (comp, systems.lj_opts(-1.0)),                                     # rc <= 0
        (systems.ion_pair_comp(2, 8.0), systems.lj_opts(3.0)),             # charges w/o method
    ]
    comp_rf, opts_rf = systems.rf_dimers()
    opts_rf.eps_rf = 0.5
    cases.append((comp_rf, opts_rf))                                        # eps_rf <= 1
    comp_i = systems.ion_pair_comp(2, 8.0)
    opts_w = systems.ewald_opts(3.0, b2.EwaldParams(1.0, 5))
    opts_w.workers = 4
    cases.append((comp_i, opts_w))                                          # ewald + workers
    bad = b2.SystemComposition([comp_i.species[0]], [4], 8.0, 1.0)
    cases.append((bad, systems.ewald_opts(3.0, b2.EwaldParams(1.0, 5))))    # non-neutral
    for c, o in cases:
        with pytest.raises(b2.ConfigError):
            b2.ForceField(c, o)
        if pyoracle.ref_available():
            with pytest.raises(pyoracle.OracleError) as ei:
                pyoracle.RefFF(c, o)
            assert ei.value.code == _abi.CONFIG_ERROR


@pytest.mark.skipif(_gpu_present(), reason="checks the no-GPU failure mode")
def test_device_path_fails_loudly_without_gpu():
    comp = systems.lj_fluid(10, 6.0)
    with pytest.raises(b2.CudaError):
        b2.ForceField(comp, systems.lj_opts(2.5))


@pytest.mark.parametrize("n", [1, 2, 31, 33, 1000, 2048, 5000, 16384])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_partitions_the_pair_triangle(n, world):
    total = n * (n - 1) // 2
    n_tiles = (n + 31) // 32
    nk = 709
    plans = [b2.shard_plan(n, nk, world, r) for r in range(world)]
    assert plans[0]["row_begin"] == 0 and plans[-1]["row_end"] == n_tiles
    for a, b in zip(plans, plans[1:]):
        assert a["row_end"] == b["row_begin"] and a["k_end"] == b["k_begin"]
    assert plans[0]["k_begin"] == 0 and plans[-1]["k_end"] == nk
    assert sum(p["candidate_pairs"] for p in plans) == total
    if world > 1 and n >= 16384:  # balanced like the reference's static split
        c = [p["candidate_pairs"] for p in plans]
        assert max(c) <= 1.15 * total / world
