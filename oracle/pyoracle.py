"""Python bindings of the CPU checkers.  TEST INFRASTRUCTURE ONLY — imported
by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg, never by the product package.

  OracleFF      oracle/liboracle.so      C restatement (tmd_oracle.c)
  RefFF/RefEngine oracle/_ref/libtmdref.so the unmodified reference tmd_core
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_1507_07548_b200 import _abi
from paper_1507_07548_b200.model import EnergyBreakdown, SystemComposition

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libtmdref.so"

_D = C.POINTER(C.c_double)
_oracle = None
_ref = None


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not ORACLE_LIB.exists():
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_LIB))
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_build_species.argtypes = [C.POINTER(_abi.b2md_site), C.c_int, C.POINTER(_abi.b2md_species)]
        L.oracle_ewald_tune.argtypes = [C.c_double, C.c_double, C.c_double, _D, C.POINTER(C.c_int)]
        L.oracle_ff_create.argtypes = [C.POINTER(_abi.b2md_composition), C.POINTER(_abi.b2md_ff_options), C.POINTER(C.c_void_p)]
        L.oracle_ff_destroy.argtypes = [C.c_void_p]
        L.oracle_ff_warning.argtypes = [C.c_void_p]
        L.oracle_ff_warning.restype = C.c_char_p
        L.oracle_ff_kvector_count.argtypes = [C.c_void_p]
        L.oracle_evaluate.argtypes = [C.c_void_p, _D, _D, _D, _D, C.POINTER(_abi.b2md_energy), C.POINTER(_abi.b2md_eval_stats)]
        L.oracle_evaluate_shard.argtypes = [C.c_void_p, _D, _D, C.c_int, C.c_int, C.c_int, C.c_int, _D, _D, _D]
        L.oracle_pair_list.argtypes = [C.c_void_p, _D, C.POINTER(C.c_int32), C.c_int64]
        L.oracle_pair_list.restype = C.c_int64
        L.oracle_wrap.argtypes = [C.c_int, C.c_double, _D]
        L.oracle_kinetic_energy.argtypes = [C.c_void_p, _D, _D, _D]
        L.oracle_apply_thermostat.argtypes = [C.c_void_p, _D, _D]
        L.oracle_heat_flux.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, C.c_int, _D]
        L.oracle_rdf_create.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.oracle_rdf_destroy.argtypes = [C.c_void_p]
        L.oracle_rdf_accumulate.argtypes = [C.c_void_p, _D, _D]
        L.oracle_rdf_shape.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.oracle_rdf_counts.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
        L.oracle_step.argtypes = [C.c_void_p, C.c_double, C.c_int64, _D, _D, _D, _D, _D, _D,
                                  C.POINTER(_abi.b2md_energy), C.POINTER(_abi.b2md_eval_stats)]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return REF_LIB.exists()


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(str(REF_LIB))
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_species.argtypes = [C.POINTER(_abi.b2md_site), C.c_int, C.POINTER(_abi.b2md_species)]
        L.ref_ewald_tune.argtypes = [C.c_double, C.c_double, C.c_double, _D, C.POINTER(C.c_int)]
        L.ref_ff_create.argtypes = [C.POINTER(_abi.b2md_composition), C.POINTER(_abi.b2md_ff_options), C.POINTER(C.c_void_p)]
        L.ref_ff_destroy.argtypes = [C.c_void_p]
        L.ref_ff_warning.argtypes = [C.c_void_p]
        L.ref_ff_warning.restype = C.c_char_p
        L.ref_evaluate.argtypes = [C.c_void_p, _D, _D, _D, _D, C.POINTER(_abi.b2md_energy), _D]
        L.ref_pair_list.argtypes = [C.c_void_p, _D, C.POINTER(C.c_int32), C.c_int64]
        L.ref_pair_list.restype = C.c_int64
        L.ref_engine_apply_thermostat.argtypes = [C.c_void_p]
        L.ref_kinetic_energy.argtypes = [C.c_void_p, _D, _D, _D]
        L.ref_heat_flux.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, C.c_int, _D]
        L.ref_rdf_create.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(C.c_void_p)]
        L.ref_rdf_destroy.argtypes = [C.c_void_p]
        L.ref_rdf_accumulate.argtypes = [C.c_void_p, C.c_void_p, _D, _D]
        L.ref_rdf_serialize.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_rdf_serialize.restype = C.c_int64
        L.ref_rdf_finalize.argtypes = [C.c_void_p, _D, C.c_int64]
        L.ref_rdf_finalize.restype = C.c_int64
        L.ref_first_minimum.argtypes = [_D, _D, C.c_int]
        L.ref_first_minimum.restype = C.c_double
        L.ref_solvation_number.argtypes = [C.c_double, _D, C.c_int, C.c_double, C.c_double]
        L.ref_solvation_number.restype = C.c_double
        L.ref_engine_checkpoint.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_engine_checkpoint.restype = C.c_int64
        L.ref_engine_restore.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_run_sampled_checkpoint.argtypes = [
            C.POINTER(_abi.b2md_composition), C.POINTER(_abi.b2md_ff_options), C.c_double, C.c_uint64,
            C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, _D, C.c_int, C.c_int, C.c_int,
            C.c_double, C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_run_sampled_checkpoint.restype = C.c_int64
        L.ref_engine_create.argtypes = [C.POINTER(_abi.b2md_composition), C.POINTER(_abi.b2md_ff_options), C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_set_state.argtypes = [C.c_void_p, _D, _D, _D, _D]
        L.ref_engine_step.argtypes = [C.c_void_p, C.c_int64]
        L.ref_engine_get_state.argtypes = [C.c_void_p, _D, _D, _D, _D, _D, _D, C.POINTER(_abi.b2md_energy), _D]
        _ref = L
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(lib, prefix, rc):
    if rc:
        raise OracleError(rc, getattr(lib, prefix + "_last_error")().decode())


def build_species_c(sites, which="oracle") -> _abi.b2md_species:
    lib = oracle_lib() if which == "oracle" else ref_lib()
    arr = (_abi.b2md_site * max(len(sites), 1))(*[s.to_c() for s in sites])
    out = _abi.b2md_species()
    fn = lib.oracle_build_species if which == "oracle" else lib.ref_build_species
    _check(lib, which if which == "oracle" else "ref", fn(arr, len(sites), C.byref(out)))
    return out


def ref_species_builder(name, sites):
    """configs.make(species_builder=...) hook: the reference's own
    tmd::build_species (oracle/_ref), wrapped as a MoleculeSpecies."""
    from paper_1507_07548_b200.model import MoleculeSpecies
    return MoleculeSpecies(name, build_species_c(sites, "ref"))


def ewald_tune(delta, cutoff, box, which="oracle"):
    lib = oracle_lib() if which == "oracle" else ref_lib()
    a, k = C.c_double(), C.c_int()
    fn = lib.oracle_ewald_tune if which == "oracle" else lib.ref_ewald_tune
    _check(lib, "oracle" if which == "oracle" else "ref", fn(delta, cutoff, box, C.byref(a), C.byref(k)))
    return a.value, k.value


class _FF:
    prefix = "oracle"

    def __init__(self, comp: SystemComposition, opts):
        self.lib = oracle_lib() if self.prefix == "oracle" else ref_lib()
        self.comp = comp
        self.n = comp.molecule_count()
        cc, self._keep = comp.to_c()
        oc = opts.to_c()
        h = C.c_void_p()
        _check(self.lib, self.prefix, getattr(self.lib, self.prefix + "_ff_create")(C.byref(cc), C.byref(oc), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            getattr(self.lib, self.prefix + "_ff_destroy")(self.h)
            self.h = None

    @property
    def warning(self) -> str:
        return getattr(self.lib, self.prefix + "_ff_warning")(self.h).decode()

    def kinetic_energy(self, vel, ang_vel):
        """kinetic_energy_trans / _rot (model.cpp:304-319)."""
        return _kinetic(self, vel, ang_vel)

    def pair_list(self, pos) -> np.ndarray:
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        fn = getattr(self.lib, self.prefix + "_pair_list")
        n = fn(self.h, _d(pos), None, 0)
        out = np.zeros((n, 2), dtype=np.int32)
        if n:
            fn(self.h, _d(pos), out.ctypes.data_as(C.POINTER(C.c_int32)), n)
        return out


def _heat_flux(ff, pos, orient, vel, ang_vel, enthalpy):
    n = ff.n
    arr = [np.ascontiguousarray(a, dtype=np.float64).reshape(n, w)
           for a, w in ((pos, 3), (orient, 4), (vel, 3), (ang_vel, 3))]
    h = np.ascontiguousarray(enthalpy, dtype=np.float64).reshape(-1)
    out = np.zeros(3)
    _check(ff.lib, ff.prefix, getattr(ff.lib, ff.prefix + "_heat_flux")(
        ff.h, *[_d(a) for a in arr], _d(h) if h.size else None, int(h.size), _d(out)))
    return out


def _kinetic(ff, vel, ang_vel):
    v = np.ascontiguousarray(vel, dtype=np.float64).reshape(ff.n, 3)
    w = np.ascontiguousarray(ang_vel, dtype=np.float64).reshape(ff.n, 3)
    out = np.zeros(2)
    _check(ff.lib, ff.prefix, getattr(ff.lib, ff.prefix + "_kinetic_energy")(ff.h, _d(v), _d(w), _d(out)))
    return out


class OracleFF(_FF):
    """C restatement (serial ForceField::evaluate + Engine::step)."""

    prefix = "oracle"

    def apply_thermostat(self, vel, ang_vel):
        """Engine::apply_thermostat on copies; returns (vel, ang_vel)."""
        v = np.array(vel, dtype=np.float64).reshape(self.n, 3)
        w = np.array(ang_vel, dtype=np.float64).reshape(self.n, 3)
        _check(self.lib, "oracle", self.lib.oracle_apply_thermostat(self.h, _d(v), _d(w)))
        return v, w

    def heat_flux(self, pos, orient, vel, ang_vel, enthalpy):
        return _heat_flux(self, pos, orient, vel, ang_vel, enthalpy)

    def evaluate(self, pos, orient):
        n = self.n
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(n, 3)
        orient = np.ascontiguousarray(orient, dtype=np.float64).reshape(n, 4)
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        e = _abi.b2md_energy()
        s = _abi.b2md_eval_stats()
        _check(self.lib, "oracle", self.lib.oracle_evaluate(self.h, _d(pos), _d(orient), _d(f), _d(t), C.byref(e), C.byref(s)))
        return {"force": f, "torque": t, "energy": EnergyBreakdown.from_c(e), "virial": s.virial,
                "s1": s.s1, "s2": s.s2, "com_pairs": s.com_pairs}

    def evaluate_shard(self, pos, orient, row_begin, row_end, k_begin, k_end):
        n = self.n
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        orient = np.ascontiguousarray(orient, dtype=np.float64)
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        sums = np.zeros(8)
        _check(self.lib, "oracle", self.lib.oracle_evaluate_shard(self.h, _d(pos), _d(orient), row_begin, row_end, k_begin, k_end, _d(f), _d(t), _d(sums)))
        return f, t, sums

    def run(self, dt, nsteps, pos, orient, vel, ang_vel):
        """set_state (wrap + forces) then Engine::step x nsteps; returns the state."""
        n = self.n
        pos = np.array(pos, dtype=np.float64).reshape(n, 3)
        orient = np.array(orient, dtype=np.float64).reshape(n, 4)
        vel = np.array(vel, dtype=np.float64).reshape(n, 3)
        ang = np.array(ang_vel, dtype=np.float64).reshape(n, 3)
        self.lib.oracle_wrap(n, self.comp.box_length, _d(pos))
        r = self.evaluate(pos, orient)
        f, t = r["force"], r["torque"]
        e = _abi.b2md_energy()
        s = _abi.b2md_eval_stats()
        if nsteps > 0:
            _check(self.lib, "oracle", self.lib.oracle_step(self.h, dt, nsteps, _d(pos), _d(orient), _d(vel), _d(ang), _d(f), _d(t), C.byref(e), C.byref(s)))
            energy, virial = EnergyBreakdown.from_c(e), s.virial
        else:
            energy, virial = r["energy"], r["virial"]
        return {"pos": pos, "orient": orient, "vel": vel, "ang_vel": ang, "force": f, "torque": t,
                "energy": energy, "virial": virial}


class RefFF(_FF):
    """The unmodified reference tmd::ForceField (workers from opts)."""

    prefix = "ref"

    def heat_flux(self, pos, orient, vel, ang_vel, enthalpy):
        return _heat_flux(self, pos, orient, vel, ang_vel, enthalpy)

    def evaluate(self, pos, orient):
        n = self.n
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(n, 3)
        orient = np.ascontiguousarray(orient, dtype=np.float64).reshape(n, 4)
        f = np.zeros((n, 3))
        t = np.zeros((n, 3))
        e = _abi.b2md_energy()
        v = np.zeros(1)
        _check(self.lib, "ref", self.lib.ref_evaluate(self.h, _d(pos), _d(orient), _d(f), _d(t), C.byref(e), _d(v)))
        return {"force": f, "torque": t, "energy": EnergyBreakdown.from_c(e), "virial": float(v[0])}


class RefEngine:
    """The unmodified reference tmd::Engine (thermostat off, NVE steps)."""

    def __init__(self, comp: SystemComposition, opts, dt: float, seed: int = 1):
        self.lib = ref_lib()
        self.comp = comp
        self.n = comp.molecule_count()
        cc, self._keep = comp.to_c()
        oc = opts.to_c()
        h = C.c_void_p()
        _check(self.lib, "ref", self.lib.ref_engine_create(C.byref(cc), C.byref(oc), dt, seed, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.ref_engine_destroy(self.h)
            self.h = None

    def set_state(self, pos, orient, vel, ang_vel):
        arr = [np.ascontiguousarray(a, dtype=np.float64) for a in (pos, orient, vel, ang_vel)]
        _check(self.lib, "ref", self.lib.ref_engine_set_state(self.h, *[_d(a) for a in arr]))

    def checkpoint_bytes(self) -> bytes:
        n = self.lib.ref_engine_checkpoint(self.h, None, 0)
        buf = C.create_string_buffer(int(n))
        self.lib.ref_engine_checkpoint(self.h, buf, n)
        return buf.raw

    def apply_thermostat(self) -> None:
        _check(self.lib, "ref", self.lib.ref_engine_apply_thermostat(self.h))

    def restore(self, data: bytes) -> None:
        _check(self.lib, "ref", self.lib.ref_engine_restore(self.h, data, len(data)))

    def step(self, n=1):
        _check(self.lib, "ref", self.lib.ref_engine_step(self.h, n))

    def state(self):
        n = self.n
        out = {k: np.zeros((n, w)) for k, w in (("pos", 3), ("orient", 4), ("vel", 3), ("ang_vel", 3), ("force", 3), ("torque", 3))}
        e = _abi.b2md_energy()
        v = np.zeros(1)
        self.lib.ref_engine_get_state(self.h, *[_d(out[k]) for k in ("pos", "orient", "vel", "ang_vel", "force", "torque")], C.byref(e), _d(v))
        out["energy"] = EnergyBreakdown.from_c(e)
        out["virial"] = float(v[0])
        return out


class OracleRdf:
    """oracle_rdf_*: the C restatement of tmd::RdfHistogram accumulate."""

    def __init__(self, ff: "OracleFF", bin_width: float, r_max: float):
        self.ff = ff
        self.lib = ff.lib
        h = C.c_void_p()
        _check(self.lib, "oracle", self.lib.oracle_rdf_create(ff.h, bin_width, r_max, C.byref(h)))
        self.h = h
        t, b, p = C.c_int(), C.c_int(), C.c_int()
        self.lib.oracle_rdf_shape(self.h, C.byref(t), C.byref(b), C.byref(p))
        self.n_types, self.bins, self.n_pairs = t.value, b.value, p.value

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.oracle_rdf_destroy(self.h)
            self.h = None

    def accumulate(self, pos, orient):
        n = self.ff.n
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(n, 3)
        orient = np.ascontiguousarray(orient, dtype=np.float64).reshape(n, 4)
        _check(self.lib, "oracle", self.lib.oracle_rdf_accumulate(self.h, _d(pos), _d(orient)))

    def counts(self):
        out = np.zeros((self.n_pairs, self.bins), dtype=np.uint64)
        snaps = C.c_int64()
        self.lib.oracle_rdf_counts(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(snaps))
        return out, snaps.value


class RefRdf:
    """The unmodified tmd::RdfHistogram (oracle/_ref)."""

    def __init__(self, ff: "RefFF", bin_width: float, r_max: float):
        self.ff = ff
        self.lib = ff.lib
        h = C.c_void_p()
        _check(self.lib, "ref", self.lib.ref_rdf_create(ff.h, bin_width, r_max, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.ref_rdf_destroy(self.h)
            self.h = None

    def accumulate(self, pos, orient):
        n = self.ff.n
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(n, 3)
        orient = np.ascontiguousarray(orient, dtype=np.float64).reshape(n, 4)
        _check(self.lib, "ref", self.lib.ref_rdf_accumulate(self.h, self.ff.h, _d(pos), _d(orient)))

    def serialize(self) -> bytes:
        n = self.lib.ref_rdf_serialize(self.h, None, 0)
        buf = C.create_string_buffer(int(n))
        self.lib.ref_rdf_serialize(self.h, buf, n)
        return buf.raw

    def counts(self):
        """Counts parsed from RdfHistogram::serialize (structure.cpp:130-140)."""
        b = self.serialize()
        bins = int(np.frombuffer(b, np.uint32, 1, 16)[0])
        snaps = int(np.frombuffer(b, np.int64, 1, 20)[0])
        npairs = int(np.frombuffer(b, np.uint64, 1, 28)[0])
        out = np.zeros((npairs, bins), dtype=np.uint64)
        o = 36
        for p in range(npairs):
            nb = int(np.frombuffer(b, np.uint64, 1, o)[0])
            out[p] = np.frombuffer(b, np.uint64, nb, o + 8)
            o += 8 + 8 * nb
        return out, snaps

    def finalize(self):
        n = self.lib.ref_rdf_finalize(self.h, None, 0)
        if n < 0:
            raise OracleError(2, self.lib.ref_last_error().decode())
        v = np.zeros(int(n))
        self.lib.ref_rdf_finalize(self.h, _d(v), n)
        tables, o = [], 0
        while o < len(v):
            sa, sb, dens, bw, snaps, nb = v[o:o + 6]
            nb = int(nb)
            body = v[o + 6:o + 6 + 3 * nb].reshape(nb, 3)
            tables.append({"species_a": int(sa), "species_b": int(sb), "partner_density": dens,
                           "bin_width": bw, "snapshots": int(snaps), "r_mid": body[:, 0].copy(),
                           "g": body[:, 1].copy(), "n_cum": body[:, 2].copy()})
            o += 6 + 3 * nb
        return tables


def ref_first_minimum(r_mid, g):
    L = ref_lib()
    r_mid = np.ascontiguousarray(r_mid, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    return L.ref_first_minimum(_d(r_mid), _d(g), len(g))


def ref_solvation_number(bin_width, g, partner_density, r_min):
    L = ref_lib()
    g = np.ascontiguousarray(g, dtype=np.float64)
    return L.ref_solvation_number(bin_width, _d(g), len(g), partner_density, r_min)


def ref_run_sampled_checkpoint(comp, opts, dt, seed, n_equil, n_prod, *, n_ext=1, corr_length=20,
                               n_blocks=4, flags=0, enthalpy=(), residence=(0, 0, 0.0),
                               config_text=""):
    """tmd::Engine::run with samplers, then Engine::checkpoint_bytes (bytes)."""
    L = ref_lib()
    cc, keep = comp.to_c()
    oc = opts.to_c()
    h = np.ascontiguousarray(enthalpy, dtype=np.float64).reshape(-1)
    args = (C.byref(cc), C.byref(oc), dt, seed, n_equil, n_prod, n_ext, corr_length, n_blocks, flags,
            _d(h) if h.size else None, int(h.size), residence[0], residence[1], float(residence[2]),
            config_text.encode())
    n = L.ref_run_sampled_checkpoint(*args, None, 0)
    if n < 0:
        raise OracleError(2, L.ref_last_error().decode())
    buf = C.create_string_buffer(int(n))
    L.ref_run_sampled_checkpoint(*args, buf, n)
    return buf.raw


def ref_derivative_accumulator(temperature, volume, n_mol, n_blocks, expected, samples) -> bytes:
    """tmd::DerivativeAccumulator fed `samples` (k x 3), serialized."""
    L = ref_lib()
    L.ref_derivative_accumulator.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_int, C.c_int64, _D,
                                             C.c_int, C.c_char_p, C.c_int64]
    L.ref_derivative_accumulator.restype = C.c_int64
    smp = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 3)
    args = (temperature, volume, n_mol, n_blocks, expected, _d(smp), len(smp))
    n = L.ref_derivative_accumulator(*args, None, 0)
    if n < 0:
        raise OracleError(2, L.ref_last_error().decode())
    buf = C.create_string_buffer(int(n))
    L.ref_derivative_accumulator(*args, buf, n)
    return buf.raw


def ref_block_stat(n_blocks, expected, x) -> bytes:
    """tmd::BlockStat fed `x`, serialized."""
    L = ref_lib()
    L.ref_block_stat.argtypes = [C.c_int, C.c_int64, _D, C.c_int, C.c_char_p, C.c_int64]
    L.ref_block_stat.restype = C.c_int64
    xs = np.ascontiguousarray(x, dtype=np.float64)
    n = L.ref_block_stat(n_blocks, expected, _d(xs), len(xs), None, 0)
    buf = C.create_string_buffer(int(n))
    L.ref_block_stat(n_blocks, expected, _d(xs), len(xs), buf, n)
    return buf.raw
