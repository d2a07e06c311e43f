"""ForceField / Engine mirrors of include/tmd/parallel.hpp:45-80 and
include/tmd/engine.hpp:52-112 over the b200md C ABI (include/b200md.h).

Same names, argument meaning and error behaviour as the reference: a
ForceField is built from a SystemComposition and ForceFieldOptions and its
evaluate(state) overwrites state.force / torque / virial / energy
(src/parallel.cpp:79-122).  Everything runs on the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import check
from .model import (
    ElectrostaticsMethod,
    EnergyBreakdown,
    SystemComposition,
    SystemState,
)


@dataclass
class EwaldParams:  # ewald.hpp:15-18
    alpha: float = 0.0
    kmax: int = 0


def ewald_tune(delta: float, cutoff: float, box_length: float) -> EwaldParams:
    """tmd::ewald_tune (src/ewald.cpp:8-28)."""
    a = C.c_double()
    k = C.c_int()
    check(_abi.lib().b2md_ewald_tune(delta, cutoff, box_length, C.byref(a), C.byref(k)))
    return EwaldParams(a.value, k.value)


def kvector_count(kmax: int) -> int:
    c = C.c_int()
    check(_abi.lib().b2md_ewald_kvector_count(kmax, C.byref(c)))
    return c.value


@dataclass
class ForceFieldOptions:  # parallel.hpp:45-52
    cutoff: float = 0.0
    method: ElectrostaticsMethod = ElectrostaticsMethod.none
    eps_rf: float = math.inf
    ewald: EwaldParams | None = None
    workers: int = 1
    volume_derivatives: bool = True

    def to_c(self) -> _abi.b2md_ff_options:
        o = _abi.b2md_ff_options()
        o.cutoff = float(self.cutoff)
        o.method = int(self.method)
        o.eps_rf = float(self.eps_rf)
        o.has_ewald = 1 if self.ewald is not None else 0
        if self.ewald is not None:
            o.ewald_alpha = float(self.ewald.alpha)
            o.ewald_kmax = int(self.ewald.kmax)
        o.workers = int(self.workers)
        o.volume_derivatives = 1 if self.volume_derivatives else 0
        return o


@dataclass
class EvalStats:
    virial: float = 0.0
    s1: float = 0.0
    s2: float = 0.0
    com_pairs: int = 0


def _f64(a, shape) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if out.shape != shape:
        out = out.reshape(shape)
    return out


class _Context:
    """Owns one b2md_ctx (device memory + stream)."""

    def __init__(self, comp: SystemComposition, opts: ForceFieldOptions, dt: float, replicas: int,
                 device: int):
        self.comp = comp
        self.opts = opts
        self.n = comp.molecule_count()
        self.replicas = int(replicas)
        self.device = int(device)
        cc, self._keep = comp.to_c()
        oc = opts.to_c()
        ctx = C.c_void_p()
        check(_abi.lib().b2md_create(self.device, C.byref(cc), C.byref(oc), float(dt),
                                     self.replicas, C.byref(ctx)))
        self.ctx = ctx

    def close(self) -> None:
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            _abi.lib().b2md_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def warning(self) -> str:
        return _abi.lib().b2md_warning(self.ctx).decode()

    def energies(self, e_arr, s_arr):
        es = EnergyBreakdown.list_from_c(e_arr, self.replicas)
        ss = [EvalStats(s_arr[r].virial, s_arr[r].s1, s_arr[r].s2, s_arr[r].com_pairs)
              for r in range(self.replicas)]
        return es, ss

    def pair_list(self, replica: int = 0) -> np.ndarray:
        """(n_pairs, 2) int32 i<j molecule pairs passing the COM partner
        search of the last evaluation, sorted by i then j."""
        n = C.c_int64()
        check(_abi.lib().b2md_pair_list(self.ctx, replica, None, 0, C.byref(n)))
        out = np.zeros((n.value, 2), dtype=np.int32)
        if n.value:
            check(_abi.lib().b2md_pair_list(
                self.ctx, replica, out.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n)))
        return out


class ForceField:
    """tmd::ForceField (parallel.hpp:56-80) on a B200."""

    def __init__(self, comp: SystemComposition, opts: ForceFieldOptions, device: int = 0):
        self._c = _Context(comp, opts, 0.0, 1, device)
        self.last_stats = EvalStats()

    def composition(self) -> SystemComposition:
        return self._c.comp

    @property
    def warning(self) -> str:
        return self._c.warning

    def evaluate(self, state: SystemState) -> None:
        """ForceField::evaluate (src/parallel.cpp:79-122): fills state.force,
        torque, virial and energy.  Positions are used as given (not wrapped)."""
        n = self._c.n
        pos = _f64(state.pos, (n, 3))
        orient = _f64(state.orient, (n, 4))
        force = np.empty((n, 3))
        torque = np.empty((n, 3))
        e = (_abi.b2md_energy * 1)()
        s = (_abi.b2md_eval_stats * 1)()
        check(_abi.lib().b2md_evaluate(self._c.ctx, _abi.dptr(pos), _abi.dptr(orient),
                                       _abi.dptr(force), _abi.dptr(torque), e, s))
        es, ss = self._c.energies(e, s)
        state.force = force
        state.torque = torque
        state.energy = es[0]
        state.virial = ss[0].virial
        self.last_stats = ss[0]

    def pair_list(self) -> np.ndarray:
        return self._c.pair_list(0)

    def set_sort_interval(self, steps: int) -> None:
        """b2md_set_sort_interval: re-sort period of the internal spatial order
        (0 keeps the input order; results differ only in summation order)."""
        check(_abi.lib().b2md_set_sort_interval(self._c.ctx, int(steps)))

    def nlist_info(self, replica: int = 0) -> dict:
        """b2md_nlist_info: the once-per-pair cluster-pair list (diagnostics)."""
        buf = (C.c_int64 * 8)()
        check(_abi.lib().b2md_nlist_info(self._c.ctx, int(replica), buf))
        keys = ("active", "entries", "incoming", "stale", "evaluations", "steps_since_build",
                "interval", "skin_e6")
        return dict(zip(keys, [int(x) for x in buf]))

    def set_search_options(self, fix_prefilter: bool = True, tile_cull: bool = True) -> None:
        """b2md_set_search_options: partner-search strategy (same results)."""
        check(_abi.lib().b2md_set_search_options(self._c.ctx, int(fix_prefilter), int(tile_cull)))

    def heat_flux(self, state: SystemState, h_per_species) -> np.ndarray:
        """tmd::heat_flux(comp, state, table, h_per_species) (src/greenkubo.cpp:182-266)
        of `state` (positions as given) with this force field's pair table."""
        n = self._c.n
        return _heat_flux_state(self._c, _f64(state.pos, (n, 3)), _f64(state.orient, (n, 4)),
                                _f64(state.vel, (n, 3)), _f64(state.ang_vel, (n, 3)),
                                h_per_species)[0]

    def set_shard(self, rank: int, world: int) -> None:
        """Evaluate only `rank`'s shard of a `world`-way decomposition (partial
        results, no communicator) — b2md_set_shard."""
        check(_abi.lib().b2md_set_shard(self._c.ctx, rank, world))

    def close(self) -> None:
        self._c.close()


class Engine:
    """The NVE hot path of tmd::Engine (engine.hpp:52-112): set_state,
    compute_forces, step — device resident.  `replicas` independent systems
    of the same composition are stepped together (one launch each kernel)."""

    def __init__(self, comp: SystemComposition, ff_opts: ForceFieldOptions, dt: float,
                 device: int = 0, replicas: int = 1):
        if dt <= 0.0:
            from .errors import ConfigError
            raise ConfigError("engine: time step must be positive")
        self._c = _Context(comp, ff_opts, dt, replicas, device)
        self.dt = float(dt)
        self.replicas = int(replicas)

    @property
    def ctx(self):
        return self._c.ctx

    @property
    def n(self) -> int:
        return self._c.n

    def composition(self) -> SystemComposition:
        return self._c.comp

    def set_state(self, states) -> None:
        """Engine::set_state (src/engine.cpp:91-98): upload, wrap, forces."""
        if isinstance(states, SystemState):
            states = [states]
        if len(states) != self.replicas:
            raise ValueError("one state per replica required")
        n = self._c.n
        for s in states:
            if s.molecule_count() != n:
                from .errors import ConfigError
                raise ConfigError("engine: state does not match composition")
        cat = lambda k, w: np.ascontiguousarray(
            np.concatenate([_f64(getattr(s, k), (n, w)) for s in states]), dtype=np.float64)
        check(_abi.lib().b2md_set_state(self._c.ctx, _abi.dptr(cat("pos", 3)),
                                        _abi.dptr(cat("orient", 4)), _abi.dptr(cat("vel", 3)),
                                        _abi.dptr(cat("ang_vel", 3))))

    def set_state_raw(self, pos, orient, vel, ang_vel) -> None:
        """set_state from replica-major contiguous float64 host buffers."""
        check(_abi.lib().b2md_set_state(self._c.ctx, _abi.dptr(pos), _abi.dptr(orient),
                                        _abi.dptr(vel), _abi.dptr(ang_vel)))

    def step(self, nsteps: int = 1) -> None:
        """Engine::step (src/engine.cpp:102-143) x nsteps."""
        check(_abi.lib().b2md_step(self._c.ctx, int(nsteps)))

    def step_async(self, nsteps: int = 1) -> None:
        """Enqueue steps without waiting; sync() waits and raises like step()."""
        check(_abi.lib().b2md_step_async(self._c.ctx, int(nsteps)))

    def sync(self) -> None:
        check(_abi.lib().b2md_sync(self._c.ctx))

    def upload_state_raw(self, pos, orient, vel, ang_vel, force=None, torque=None) -> None:
        """b2md_upload_state from contiguous float64 host buffers (no evaluation)."""
        check(_abi.lib().b2md_upload_state(self._c.ctx, *map(_abi.dptr, (pos, orient, vel, ang_vel, force, torque))))

    def get_state_raw(self, pos=None, orient=None, vel=None, ang_vel=None, force=None, torque=None):
        """Download into caller-provided float64 host buffers; returns energies."""
        R = self.replicas
        e = (_abi.b2md_energy * R)()
        s = (_abi.b2md_eval_stats * R)()
        check(_abi.lib().b2md_get_state(self._c.ctx, *map(_abi.dptr, (pos, orient, vel, ang_vel, force, torque)), e, s))
        return self._c.energies(e, s)

    def states(self) -> list[SystemState]:
        n, R = self._c.n, self.replicas
        pos = np.empty((R * n, 3))
        orient = np.empty((R * n, 4))
        vel = np.empty((R * n, 3))
        ang = np.empty((R * n, 3))
        force = np.empty((R * n, 3))
        torque = np.empty((R * n, 3))
        e = (_abi.b2md_energy * R)()
        s = (_abi.b2md_eval_stats * R)()
        check(_abi.lib().b2md_get_state(self._c.ctx, *(map(_abi.dptr, (pos, orient, vel, ang, force, torque))), e, s))
        es, ss = self._c.energies(e, s)
        out = []
        for r in range(R):
            st = SystemState(0, self._c.comp.box_length)
            sl = slice(r * n, (r + 1) * n)
            st.pos, st.orient, st.vel, st.ang_vel = pos[sl], orient[sl], vel[sl], ang[sl]
            st.force, st.torque = force[sl], torque[sl]
            st.energy, st.virial = es[r], ss[r].virial
            out.append(st)
        self.last_stats = ss
        return out

    def state(self) -> SystemState:
        return self.states()[0]

    def energies(self):
        """Per-replica (EnergyBreakdown, EvalStats) without downloading arrays."""
        R = self.replicas
        e = (_abi.b2md_energy * R)()
        s = (_abi.b2md_eval_stats * R)()
        check(_abi.lib().b2md_get_state(self._c.ctx, None, None, None, None, None, None, e, s))
        return self._c.energies(e, s)

    def pair_list(self, replica: int = 0) -> np.ndarray:
        return self._c.pair_list(replica)

    def set_sort_interval(self, steps: int) -> None:
        """b2md_set_sort_interval: re-sort period of the internal spatial order
        (0 keeps the input order; results differ only in summation order)."""
        check(_abi.lib().b2md_set_sort_interval(self._c.ctx, int(steps)))

    nlist_info = ForceField.nlist_info

    def sort_interval(self) -> tuple[int, int]:
        """(re-sort period, steps taken since the last re-sort)."""
        a, b = C.c_int(), C.c_int()
        check(_abi.lib().b2md_get_sort_interval(self._c.ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_search_options(self, fix_prefilter: bool = True, tile_cull: bool = True) -> None:
        """b2md_set_search_options: partner-search strategy (same results)."""
        check(_abi.lib().b2md_set_search_options(self._c.ctx, int(fix_prefilter), int(tile_cull)))

    def set_step_options(self, fused_kick: bool = True) -> None:
        """b2md_set_step_options: end-of-step kick fused into the force kernel
        (same results bit for bit)."""
        check(_abi.lib().b2md_set_step_options(self._c.ctx, int(fused_kick)))

    # --- thermostat (engine.cpp:145-160, 273-296) and kinetic energies
    def kinetic_energies(self) -> tuple[np.ndarray, np.ndarray]:
        """(kinetic_energy_trans, kinetic_energy_rot) of every replica
        (model.cpp:304-319), reduced on the device."""
        kt = np.zeros(self.replicas)
        kr = np.zeros(self.replicas)
        check(_abi.lib().b2md_kinetic_energy(self._c.ctx, _abi.dptr(kt), _abi.dptr(kr)))
        return kt, kr

    def apply_thermostat(self) -> None:
        """Engine::apply_thermostat: isokinetic rescale to the composition's
        temperature (every replica)."""
        check(_abi.lib().b2md_apply_thermostat(self._c.ctx))

    def step_thermostat(self, nsteps: int, interval: int, done: int = 0) -> None:
        """Engine::run's loop: steps done+1 .. done+nsteps of a phase with the
        rescale after each step whose number is a multiple of `interval`."""
        check(_abi.lib().b2md_step_thermostat(self._c.ctx, int(nsteps), int(interval), int(done)))

    # --- checkpoint / restart (engine.cpp:420-541)
    def state_block(self, replica: int = 0) -> bytes:
        """The state block of Engine::checkpoint_bytes (engine.cpp:432-441),
        packed on the device: u32 n, f64 box, 13 f64 per molecule."""
        size = _abi.lib().b2md_state_block_size(self._c.ctx)
        buf = C.create_string_buffer(size)
        check(_abi.lib().b2md_save_state_block(self._c.ctx, replica, buf, size))
        return buf.raw

    def restore_state_block(self, block: bytes, replica: int = 0) -> None:
        """restore_dynamic's state part + compute_forces (engine.cpp:479-491, 540)."""
        check(_abi.lib().b2md_restore_state_block(self._c.ctx, replica, block, len(block)))

    def heat_fluxes(self, h_per_species) -> np.ndarray:
        """(replicas, 3) J_q of the device-resident state (what Engine::run
        samples every n_ext steps, src/engine.cpp:235-238)."""
        h = np.ascontiguousarray(h_per_species, dtype=np.float64).reshape(-1)
        out = np.empty((self.replicas, 3))
        check(_abi.lib().b2md_heat_flux(self._c.ctx, _abi.dptr(h), int(h.size), _abi.dptr(out)))
        return out

    def heat_flux(self, h_per_species) -> np.ndarray:
        return self.heat_fluxes(h_per_species)[0]

    def attach_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        check(_abi.lib().b2md_attach_nccl(self._c.ctx, unique_id, rank, world))

    def set_graphs(self, enable: bool) -> None:
        check(_abi.lib().b2md_set_graphs(self._c.ctx, 1 if enable else 0))

    def profile(self, enable, level: int = 1) -> None:
        """Per-kernel CUDA-event timing: level 1 all kernels, 2 search only."""
        check(_abi.lib().b2md_profile_enable(self._c.ctx, int(level) if enable else 0))

    def kernel_times(self) -> dict:
        rows = 16
        names = (C.c_char * 32 * rows)()
        ms = (C.c_double * rows)()
        cnt = (C.c_int64 * rows)()
        nr = C.c_int()
        check(_abi.lib().b2md_kernel_times(self._c.ctx, rows, names, ms, cnt, C.byref(nr)))
        return {names[k].value.decode(): (ms[k], cnt[k]) for k in range(nr.value)}

    def stream(self) -> int:
        return _abi.lib().b2md_stream(self._c.ctx)

    def close(self) -> None:
        self._c.close()


def _heat_flux_state(c: _Context, pos, orient, vel, ang_vel, h_per_species) -> np.ndarray:
    h = np.ascontiguousarray(h_per_species, dtype=np.float64).reshape(-1)
    out = np.empty((c.replicas, 3))
    check(_abi.lib().b2md_heat_flux_state(c.ctx, _abi.dptr(pos), _abi.dptr(orient), _abi.dptr(vel),
                                          _abi.dptr(ang_vel), _abi.dptr(h), int(h.size),
                                          _abi.dptr(out)))
    return out


def heat_flux(ff: ForceField, state: SystemState, h_per_species) -> np.ndarray:
    """Free-function form of tmd::heat_flux (include/tmd/greenkubo.hpp:93)."""
    return ff.heat_flux(state, h_per_species)


class _ContextView(_Context):
    """A context owned by a b2md_group (not destroyed here)."""

    def __init__(self, comp, opts, replicas, device, ctx):
        self.comp = comp
        self.opts = opts
        self.n = comp.molecule_count()
        self.replicas = int(replicas)
        self.device = int(device)
        self.ctx = C.c_void_p(ctx)

    def close(self) -> None:
        self.ctx = None


class EngineGroup:
    """b2md_create_group: one process driving several GPUs -- the single-process
    caller shape of tmd::Engine (src/engine.cpp:100-143) over a row-sharded
    system (src/parallel.cpp:84-95's split, one packed NCCL all-reduce per
    evaluation).  `engines[k]` is rank k's context (streams, profiling,
    energies); stepping goes through the group (all devices together)."""

    def __init__(self, comp: SystemComposition, ff_opts: ForceFieldOptions, dt: float,
                 devices=None, replicas: int = 1):
        devs = list(range(_device_count())) if devices is None else [int(d) for d in devices]
        if not devs:
            from .errors import CudaError
            raise CudaError("create_group: no CUDA device")
        self.comp, self.dt, self.replicas = comp, float(dt), int(replicas)
        cc, self._keep = comp.to_c()
        oc = ff_opts.to_c()
        arr = (C.c_int * len(devs))(*devs)
        g = C.c_void_p()
        check(_abi.lib().b2md_create_group(len(devs), arr, C.byref(cc), C.byref(oc), float(dt),
                                           self.replicas, C.byref(g)))
        self._g = g
        self.devices = devs
        self.engines = []
        for k, d in enumerate(devs):
            e = Engine.__new__(Engine)
            e._c = _ContextView(comp, ff_opts, self.replicas, d,
                                _abi.lib().b2md_group_context(g, k))
            e.dt, e.replicas = self.dt, self.replicas
            self.engines.append(e)

    def size(self) -> int:
        return int(_abi.lib().b2md_group_size(self._g))

    def set_state(self, states) -> None:
        if isinstance(states, SystemState):
            states = [states]
        n = self.comp.molecule_count()
        cat = lambda k, w: np.ascontiguousarray(
            np.concatenate([_f64(getattr(s, k), (n, w)) for s in states]), dtype=np.float64)
        check(_abi.lib().b2md_group_set_state(self._g, _abi.dptr(cat("pos", 3)),
                                              _abi.dptr(cat("orient", 4)), _abi.dptr(cat("vel", 3)),
                                              _abi.dptr(cat("ang_vel", 3))))

    def step(self, nsteps: int = 1) -> None:
        check(_abi.lib().b2md_group_step(self._g, int(nsteps)))

    def step_async(self, nsteps: int = 1) -> None:
        check(_abi.lib().b2md_group_step_async(self._g, int(nsteps)))

    def sync(self) -> None:
        check(_abi.lib().b2md_group_sync(self._g))

    def states(self) -> list[SystemState]:
        """rank 0's copy (every rank holds the whole replicated state)."""
        self.sync()
        return self.engines[0].states()

    def state(self) -> SystemState:
        return self.states()[0]

    def close(self) -> None:
        if getattr(self, "_g", None) is not None and self._g.value:
            for e in self.engines:
                e._c.close()
            _abi.lib().b2md_destroy_group(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_count() -> int:
    n = C.c_int(0)
    try:
        cudart = C.CDLL("libcudart.so")
    except OSError:
        import torch
        return torch.cuda.device_count()
    cudart.cudaGetDeviceCount(C.byref(n))
    return int(n.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_abi.lib().b2md_nccl_unique_id(buf))
    return buf.raw


def shard_plan(n_molecules: int, n_kvectors: int, world: int, rank: int) -> dict:
    """b2md_shard_plan: tile-row and k-vector ranges of `rank`."""
    vals = [C.c_int() for _ in range(4)]
    cand = C.c_int64()
    check(_abi.lib().b2md_shard_plan(n_molecules, n_kvectors, world, rank,
                                     *[C.byref(v) for v in vals], C.byref(cand)))
    rb, re, kb, ke = (v.value for v in vals)
    return {"row_begin": rb, "row_end": re, "k_begin": kb, "k_end": ke,
            "candidate_pairs": cand.value}


def measure_fp64_peak(device: int = 0) -> float:
    g = C.c_double()
    check(_abi.lib().b2md_measure_fp64_peak(device, C.byref(g)))
    return g.value
