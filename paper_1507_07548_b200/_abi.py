"""ctypes mirror of include/b200md.h and the loader of the native library.

The native library (paper_1507_07548_b200/lib/libb200md.so) is the product:
there is no Python or CPU fallback.  If it is missing, importing the device
entry points raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

B2MD_MAX_SITES = 16

# status codes (include/tmd/error.hpp:8-30)
OK, MODEL_ERROR, CONFIG_ERROR, IO_ERROR, NUMERICAL_ERROR, CUDA_ERROR, INVALID_ARGUMENT = range(7)

SITE_LJ, SITE_CHARGE, SITE_DUMMY = 0, 1, 2
METHOD_NONE, METHOD_REACTION_FIELD, METHOD_EWALD = 0, 1, 2


class b2md_site(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("pad_", C.c_int32),
        ("body_pos", C.c_double * 3),
        ("sigma", C.c_double),
        ("epsilon", C.c_double),
        ("q", C.c_double),
        ("mass", C.c_double),
    ]


class b2md_species(C.Structure):
    _fields_ = [
        ("n_sites", C.c_int32),
        ("rotational_dof", C.c_int32),
        ("sites", b2md_site * B2MD_MAX_SITES),
        ("total_mass", C.c_double),
        ("inertia_principal", C.c_double * 3),
        ("net_charge", C.c_double),
        ("max_extent", C.c_double),
    ]


class b2md_composition(C.Structure):
    _fields_ = [
        ("n_species", C.c_int32),
        ("pad_", C.c_int32),
        ("species", C.POINTER(b2md_species)),
        ("counts", C.POINTER(C.c_int32)),
        ("box_length", C.c_double),
        ("temperature", C.c_double),
    ]


class b2md_ff_options(C.Structure):
    _fields_ = [
        ("cutoff", C.c_double),
        ("method", C.c_int32),
        ("has_ewald", C.c_int32),
        ("eps_rf", C.c_double),
        ("ewald_alpha", C.c_double),
        ("ewald_kmax", C.c_int32),
        ("workers", C.c_int32),
        ("volume_derivatives", C.c_int32),
        ("pad_", C.c_int32),
    ]


class b2md_energy(C.Structure):
    _fields_ = [
        (name, C.c_double)
        for name in (
            "lj",
            "elec_real",
            "elec_recip",
            "elec_self",
            "rf",
            "lrc",
            "du_dv_explicit",
            "du_dv_lrc",
            "d2u_dv2_explicit",
            "d2u_dv2_lrc",
        )
    ]


class b2md_eval_stats(C.Structure):
    _fields_ = [
        ("virial", C.c_double),
        ("s1", C.c_double),
        ("s2", C.c_double),
        ("com_pairs", C.c_int64),
    ]


_D = C.POINTER(C.c_double)
_CTX = C.c_void_p

# name -> (restype, argtypes): every symbol include/b200md.h declares
SIGNATURES = {
    "b2md_last_error": (C.c_char_p, []),
    "b2md_abi_version": (C.c_int, []),
    "b2md_build_species": (C.c_int, [C.POINTER(b2md_site), C.c_int, C.POINTER(b2md_species)]),
    "b2md_ewald_tune": (C.c_int, [C.c_double, C.c_double, C.c_double, _D, C.POINTER(C.c_int)]),
    "b2md_ewald_kvector_count": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "b2md_shard_plan": (
        C.c_int,
        [C.c_int, C.c_int, C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 4 + [C.POINTER(C.c_int64)],
    ),
    "b2md_create": (
        C.c_int,
        [C.c_int, C.POINTER(b2md_composition), C.POINTER(b2md_ff_options), C.c_double, C.c_int,
         C.POINTER(_CTX)],
    ),
    "b2md_destroy": (None, [_CTX]),
    "b2md_warning": (C.c_char_p, [_CTX]),
    "b2md_evaluate": (
        C.c_int,
        [_CTX, _D, _D, _D, _D, C.POINTER(b2md_energy), C.POINTER(b2md_eval_stats)],
    ),
    "b2md_set_state": (C.c_int, [_CTX, _D, _D, _D, _D]),
    "b2md_step": (C.c_int, [_CTX, C.c_int64]),
    "b2md_step_async": (C.c_int, [_CTX, C.c_int64]),
    "b2md_sync": (C.c_int, [_CTX]),
    "b2md_upload_state": (C.c_int, [_CTX, _D, _D, _D, _D, _D, _D]),
    "b2md_get_state": (
        C.c_int,
        [_CTX, _D, _D, _D, _D, _D, _D, C.POINTER(b2md_energy), C.POINTER(b2md_eval_stats)],
    ),
    "b2md_pair_list": (
        C.c_int,
        [_CTX, C.c_int, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_int64)],
    ),
    "b2md_set_search_options": (C.c_int, [_CTX, C.c_int, C.c_int]),
    "b2md_set_sort_interval": (C.c_int, [_CTX, C.c_int]),
    "b2md_get_sort_interval": (C.c_int, [_CTX, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "b2md_nlist_info": (C.c_int, [_CTX, C.c_int, C.POINTER(C.c_int64)]),
    "b2md_set_step_options": (C.c_int, [_CTX, C.c_int]),
    "b2md_heat_flux": (C.c_int, [_CTX, _D, C.c_int, _D]),
    "b2md_heat_flux_state": (C.c_int, [_CTX, _D, _D, _D, _D, _D, C.c_int, _D]),
    "b2md_kinetic_energy": (C.c_int, [_CTX, _D, _D]),
    "b2md_apply_thermostat": (C.c_int, [_CTX]),
    "b2md_step_thermostat": (C.c_int, [_CTX, C.c_int64, C.c_int, C.c_int64]),
    "b2md_state_block_size": (C.c_size_t, [_CTX]),
    "b2md_save_state_block": (C.c_int, [_CTX, C.c_int, C.c_char_p, C.c_size_t]),
    "b2md_restore_state_block": (C.c_int, [_CTX, C.c_int, C.c_char_p, C.c_size_t]),
    "b2md_rdf_create": (C.c_int, [_CTX, C.c_double, C.c_double, C.POINTER(C.c_void_p)]),
    "b2md_rdf_destroy": (None, [C.c_void_p]),
    "b2md_rdf_shape": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "b2md_rdf_types": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "b2md_rdf_accumulate": (C.c_int, [C.c_void_p]),
    "b2md_rdf_accumulate_state": (C.c_int, [C.c_void_p, _D, _D]),
    "b2md_rdf_counts": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]),
    "b2md_rdf_set_counts": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64), C.c_int64]),
    "b2md_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "b2md_attach_nccl": (C.c_int, [_CTX, C.c_char_p, C.c_int, C.c_int]),
    "b2md_create_group": (
        C.c_int,
        [C.c_int, C.POINTER(C.c_int), C.POINTER(b2md_composition), C.POINTER(b2md_ff_options),
         C.c_double, C.c_int, C.POINTER(_CTX)],
    ),
    "b2md_destroy_group": (None, [_CTX]),
    "b2md_group_size": (C.c_int, [_CTX]),
    "b2md_group_context": (_CTX, [_CTX, C.c_int]),
    "b2md_group_set_state": (C.c_int, [_CTX, _D, _D, _D, _D]),
    "b2md_group_step": (C.c_int, [_CTX, C.c_int64]),
    "b2md_group_step_async": (C.c_int, [_CTX, C.c_int64]),
    "b2md_group_sync": (C.c_int, [_CTX]),
    "b2md_group_get_state": (
        C.c_int,
        [_CTX, _D, _D, _D, _D, _D, _D, C.POINTER(b2md_energy), C.POINTER(b2md_eval_stats)],
    ),
    "b2md_set_shard": (C.c_int, [_CTX, C.c_int, C.c_int]),
    "b2md_stream": (C.c_void_p, [_CTX]),
    "b2md_profile_enable": (C.c_int, [_CTX, C.c_int]),
    "b2md_kernel_times": (
        C.c_int,
        [_CTX, C.c_int, C.c_void_p, _D, C.POINTER(C.c_int64), C.POINTER(C.c_int)],
    ),
    "b2md_set_graphs": (C.c_int, [_CTX, C.c_int]),
    "b2md_measure_fp64_peak": (C.c_int, [C.c_int, _D]),
}

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libb200md.so"
_lib = None


def library_path() -> Path:
    return Path(os.environ.get("B2MD_LIBRARY", str(LIB_PATH)))


def _prefer_python_nccl() -> None:
    """NCCL is loaded by the library at first multi-GPU use; point it at the
    NCCL of this Python environment's PyTorch (nvidia-nccl wheel) so a later
    `import torch` finds the same, compatible library in the process."""
    if os.environ.get("B2MD_NCCL_LIBRARY"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = Path(base) / "lib" / "libnccl.so.2"
        if cand.exists():
            os.environ["B2MD_NCCL_LIBRARY"] = str(cand)
            return


def lib():
    """Load libb200md.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        path = library_path()
        if not path.exists():
            raise RuntimeError(
                f"b200md native library missing at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
            )
        _prefer_python_nccl()
        handle = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


# ndarray -> double* conversions cost ~3 us each in ctypes; a caller that steps
# through the same (pinned) buffers pays it once per buffer.  The cache keeps
# the array alive, so its id and data pointer cannot be reused while cached.
_PTR_CACHE: dict[int, tuple[np.ndarray, object]] = {}
_PTR_CACHE_MAX = 64


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    hit = _PTR_CACHE.get(id(a))
    if hit is not None and hit[0] is a:
        return hit[1]
    assert a.dtype == np.float64 and a.flags.c_contiguous
    p = a.ctypes.data_as(_D)
    if len(_PTR_CACHE) >= _PTR_CACHE_MAX:
        _PTR_CACHE.clear()
    _PTR_CACHE[id(a)] = (a, p)
    return p
