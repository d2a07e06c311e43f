"""paper_1507_07548_b200 — B200-native (sm_100a) force/energy/partner-search
and rigid-body step path of the ms2 2.0 / tmd reference, behind the
reference's ForceField / Engine interface (include/tmd/parallel.hpp,
include/tmd/engine.hpp) and the C ABI in include/b200md.h."""
from .errors import ConfigError, CudaError, Error, IoError, ModelError, NumericalError
from .forcefield import (
    Engine,
    EngineGroup,
    EvalStats,
    EwaldParams,
    ForceField,
    ForceFieldOptions,
    ewald_tune,
    heat_flux,
    kvector_count,
    measure_fp64_peak,
    nccl_unique_id,
    shard_plan,
)
from .structure import RdfHistogram, rdf_site_types, serialize_counts
from .model import (
    ElectrostaticsMethod,
    EnergyBreakdown,
    MoleculeSpecies,
    Site,
    SiteKind,
    SystemComposition,
    SystemState,
    build_species,
    kinetic_energy_rot,
    kinetic_energy_trans,
    make_charge_site,
    make_lj_site,
    rotational_dof,
    translational_dof,
)

__all__ = [n for n in dir() if not n.startswith("_")]
