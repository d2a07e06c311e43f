#!/usr/bin/env python
"""Benchmark of the B200 MD hot path (one JSON line on rank 0).

Workload (default): BASELINE config 3 — LJ fluid N=16384, rho*=0.8, rc=5 sigma,
fp64, the 16384-molecule system the north_star's FP64-roofline target and the
multi-GPU row-sharding spec are quoted on.  A "step" is one Engine::step
(src/engine.cpp:102-143): half kick + drift + wrap, partner search, forces,
energies, half kick.  `--config cfg0..cfg4` selects the other configs.

  python bench.py [--gpus N --steps K --warmup W]          # this implementation
  python bench.py --impl reference [...]                    # reference CPU arm
N > 1 is launched by torchrun (one rank per GPU): the pair triangle is
row-sharded and one packed NCCL all-reduce per step combines forces and
energy sums (strong scaling; cfg4 runs independent replicas per rank).

Timing: W untimed steps, then K steps, each bracketed on the library's stream
by CUDA events; the L2 is flushed (256 MiB memset, outside the events)
between timed steps; barrier + synchronize around the region; max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "site-site pair interactions/s and MD steps/s; fraction of B200 FP64 peak"
# algorithmic fp64 work per unit
FLOP_CANDIDATE = 17
FLOP_LJ_SINGLE = 32


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg3")
    p.add_argument("--e2e-steps", type=int, default=50)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-flush", action="store_true")
    p.add_argument("--group", action="store_true",
                   help="one process for all --gpus devices (b2md_create_group); the default "
                        "when --gpus N > 1 is given without torchrun")
    p.add_argument("--equil", type=int, default=-1,
                   help="untimed equilibration steps before the timed region (-1: 1000 for cfg3, "
                        "else 0); with a re-sort interval the count is padded so the first timed "
                        "step re-sorts")
    p.add_argument("--op", default="step", choices=["step", "heat_flux", "rdf"],
                   help="step: Engine::step (the north_star path); heat_flux: tmd::heat_flux, "
                        "rdf: RdfHistogram::accumulate (SURVEY 8(f) rows 1-2) of the set state")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(name, rank, world, species_builder=None):
    from paper_1507_07548_b200 import configs
    if name == "cfg4":  # replicas only: 8 independent replicas per rank
        return configs.make("cfg4", replicas=8, first_seed=8 * rank, species_builder=species_builder)
    return configs.make(name, species_builder=species_builder)


def physical_cores():
    """Physical cores of the host (W = all physical cores)."""
    try:
        import psutil
        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:
        pass
    cores = set()
    try:
        phys = core = None
        for line in open("/proc/cpuinfo"):
            if line.startswith("physical id"):
                phys = line.split(":")[1].strip()
            elif line.startswith("core id"):
                core = line.split(":")[1].strip()
            elif not line.strip() and core is not None:
                cores.add((phys, core))
                phys = core = None
    except OSError:
        pass
    return len(cores) or (os.cpu_count() or 1)


def product_libs_loaded():
    """The repo's own native libraries mapped into this process (the reference
    arm must map none of them)."""
    try:
        maps = open("/proc/self/maps").read()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps.splitlines()
                   if "libb200md" in ln or "paper_1507_07548_b200" in ln})


def algorithmic(wl, pairs_in_cutoff):
    n = wl.comp.molecule_count()
    cand = n * (n - 1) // 2
    return cand, cand * FLOP_CANDIDATE


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def cpu_reference_run(wl, steps_wanted, budget_s, threads, min_steps=1):
    """The reference tmd::Engine (oracle/_ref, built from /root/reference) on the
    host cores: set_state then step() x k, bounded to ~budget_s seconds."""
    from oracle import pyoracle
    opts = wl.opts
    if opts.method != 2:  # ewald forces workers = 1 (parallel.cpp:65-66)
        import copy
        opts = copy.copy(opts)
        opts.workers = threads
    st = wl.states[0]
    eng = pyoracle.RefEngine(wl.comp, opts, wl.dt)
    eng.set_state(st.pos, st.orient, st.vel, st.ang_vel)
    t0 = time.perf_counter()
    eng.step(1)  # warm-up + per-step estimate
    est = time.perf_counter() - t0
    k = max(min_steps, min(steps_wanted, int(budget_s / max(est, 1e-6))))
    t0 = time.perf_counter()
    eng.step(k)
    dt = time.perf_counter() - t0
    return k / dt, k, opts.workers


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle
    if not pyoracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtmdref.so not built"}))
        return
    # the same seeded workload, its species built by the reference's own
    # tmd::build_species: nothing of the product is loaded on this arm
    wl = workload(args.config, 0, 1, species_builder=pyoracle.ref_species_builder)
    threads = os.cpu_count() or 1
    # each of the K steps is one reference step; bound the whole run to ~3 min
    value, k, workers = cpu_reference_run(wl, args.steps, 150.0, threads)
    loaded = product_libs_loaded()
    if loaded:
        raise SystemExit(f"reference arm loaded product code: {loaded}")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "steps/s",
        "n_gpus": args.gpus,
        "steps": k,
        "warmup": 1,
        "ms_per_step": 1e3 / value,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator, paper_1507_07548_b200/configs.py)",
        "config": {"workload": f"{args.config}: {describe(wl)}"},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": workers, "kind": "reference",
                         "physical_cores": physical_cores(),
                         "sample": f"{k} tmd::Engine::step calls after set_state, W={workers} threads "
                                   f"(all logical CPUs)"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_libs_loaded": loaded,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------- sampler ops
# SURVEY.md 8(f) rows measured like the step: device value on the resident
# state, e2e through the host-buffer C-ABI call, roofline on the op's kernel,
# the reference's own CPU implementation as the baseline.
#
# heat_flux (greenkubo.cpp:182-266): fp64 work per visit of an in-cutoff
# single-site pair from one row (each pair is visited from both rows):
# min image 12, r^2 5, 1/r^2 5, LJ 9, force 5, 0.5 f.v 6, s R accumulate 6,
# u 1, cutoff test 1  ("heat flux")
FLUX_FLOP_PER_VISIT = 50
# RdfHistogram::accumulate (structure.cpp:60-73): per intermolecular site pair
# min image 12 (3 x sub, div, round, mul-sub), norm2 5, sqrt 1, div 1
RDF_FLOP_PER_PAIR = 19
OPS = {
    "heat_flux": {"metric": "heat-flux J_q evaluations/s (tmd::heat_flux)", "unit": "evals/s",
                  "family": "heat_flux"},
    "rdf": {"metric": "RDF histogram accumulations/s (tmd::RdfHistogram::accumulate)",
            "unit": "snapshots/s", "family": "rdf"},
}
RDF_BIN_WIDTH = 0.02  # SimulationPlan::rdf_bin_width default (engine.hpp:34)


def flux_inputs(wl):
    rng = np.random.default_rng(12345)
    n = wl.comp.molecule_count() * wl.replicas
    return rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=len(wl.comp.species))


def rdf_site_pairs(wl):
    """Intermolecular pairs of RDF sampling sites (LJ and dummy) per replica."""
    per_species = [sum(1 for s in sp.sites if int(s.kind) != 1) for sp in wl.comp.species]
    sites = [per_species[k] for k in wl.comp.species_index()]
    tot = sum(sites)
    return (tot * tot - sum(x * x for x in sites)) // 2


def cpu_reference_op(op, wl, calls_wanted, budget_s):
    """The reference's own serial implementation of the op (oracle/_ref)."""
    from oracle import pyoracle
    st = wl.states[0]
    n = wl.comp.molecule_count()
    vel, ang, h = flux_inputs(wl)
    ff = pyoracle.RefFF(wl.comp, wl.opts)
    if op == "heat_flux":
        call = lambda: ff.heat_flux(st.pos, st.orient, vel[:n], ang[:n], h)
    else:
        rdf = pyoracle.RefRdf(ff, RDF_BIN_WIDTH, 0.5 * wl.comp.box_length)
        call = lambda: rdf.accumulate(st.pos, st.orient)
    t0 = time.perf_counter()
    call()
    est = time.perf_counter() - t0
    k = max(1, min(calls_wanted, int(budget_s / max(est, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(k):
        call()
    return k / (time.perf_counter() - t0), k


def run_op_reference(args):
    rank, _, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle
    if not pyoracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtmdref.so not built"}))
        return
    wl = workload(args.config, 0, 1, species_builder=pyoracle.ref_species_builder)
    spec = OPS[args.op]
    value, k = cpu_reference_op(args.op, wl, args.steps, 150.0)
    loaded = product_libs_loaded()
    if loaded:
        raise SystemExit(f"reference arm loaded product code: {loaded}")
    line = {
        "impl": "reference", "op": args.op, "metric": spec["metric"], "value": value,
        "unit": spec["unit"], "n_gpus": args.gpus, "steps": k, "warmup": 1, "ms_per_step": 1e3 / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_1507_07548_b200/configs.py)",
        "config": {"workload": f"{args.config}: {describe(wl)}"},
        "cpu_baseline": {"value": value, "unit": spec["unit"], "cores": 1, "kind": "reference",
                         "sample": f"{k} calls of the reference's {args.op} (serial in the reference)"},
        "e2e": {"value": value, "unit": spec["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_op(args):
    """A sampler op on the device-resident state (what Engine::run calls every
    n_ext / rdf_stride steps), K calls each bracketed by CUDA events with an L2
    flush between; e2e through the host-state C-ABI entry with pinned buffers."""
    rank, world, local = dist_env()
    import torch
    import paper_1507_07548_b200 as b2
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workload(args.config, rank, world)
    spec = OPS[args.op]
    R, n = wl.replicas, wl.comp.molecule_count()
    L = wl.comp.box_length
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, device=local, replicas=R)
    if world > 1 and args.config != "cfg4" and args.op == "heat_flux":
        uid = [b2.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.attach_nccl(uid[0], rank, world)
    vel, ang, h = flux_inputs(wl)
    states = wl.states
    for r, s in enumerate(states):
        s.vel, s.ang_vel = vel[r * n:(r + 1) * n], ang[r * n:(r + 1) * n]
    eng.set_state(states)
    _, stats = eng.energies()
    pairs_total = int(sum(s.com_pairs for s in stats))
    peak_gflops = b2.measure_fp64_peak(local)
    stream = torch.cuda.ExternalStream(eng.stream(), device=local)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    rdf = b2.RdfHistogram(eng, RDF_BIN_WIDTH, 0.5 * L) if args.op == "rdf" else None
    op_call = (lambda: eng.heat_fluxes(h)) if args.op == "heat_flux" else (lambda: rdf.accumulate())
    for _ in range(max(3, args.warmup)):
        op_call()

    def timed(k):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        with torch.cuda.stream(stream):
            for i in range(k):
                starts[i].record(stream)
                op_call()
                ends[i].record(stream)
                if flush is not None:
                    flush.zero_()
        torch.cuda.synchronize()
        return float(sum(a.elapsed_time(b) for a, b in zip(starts, ends)))

    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    total_ms = timed(args.steps)
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    eng.profile(True, 1)
    timed(args.steps)
    kt = eng.kernel_times()
    eng.profile(False)
    # e2e: the reference's host-state form (upload + device work + result back)
    ff = b2.ForceField(wl.comp, wl.opts, device=local)
    if world > 1 and args.config != "cfg4" and args.op == "heat_flux":
        ff.set_shard(rank, world)  # partial per rank; the e2e time is what counts
    hs = wl.states[0]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hs.pos, hs.orient, hs.vel, hs.ang_vel = map(pin, (hs.pos, hs.orient, hs.vel, hs.ang_vel))
    if args.op == "heat_flux":
        e2e_call = lambda: ff.heat_flux(hs, h)
        h2d, d2h = 8 * n * 13, 8 * 3
    else:
        rdf_h = b2.RdfHistogram(ff, RDF_BIN_WIDTH, 0.5 * L)
        e2e_call = lambda: (rdf_h.accumulate(hs), rdf_h.counts())
        h2d, d2h = 8 * n * 7, 8 * rdf_h._pairs * rdf_h.bins()
    e2e_call()
    k_e2e = max(1, args.e2e_steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        e2e_call()
    e2e_s = time.perf_counter() - t0
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    evals = args.steps * (R * world if args.config == "cfg4" else 1)
    value = evals / (total_ms * 1e-3)
    k_ms, k_n = kt.get(spec["family"], (0.0, 0))
    avg_s = k_ms * 1e-3 / max(1, k_n)
    if args.op == "heat_flux":
        work = 2 * pairs_total * FLUX_FLOP_PER_VISIT
        kernel = f"k_heat_flux ({FLUX_FLOP_PER_VISIT} flop per pair visit, 2 visits per in-cutoff pair)"
    else:
        work = rdf_site_pairs(wl) * R * RDF_FLOP_PER_PAIR
        kernel = (f"k_rdf_pairs ({RDF_FLOP_PER_PAIR} flop per intermolecular site pair, "
                  f"bin width {RDF_BIN_WIDTH}, r_max L/2)")
    achieved = work / avg_s / 1e12 if avg_s > 0 else 0.0
    peak = peak_gflops / 1e3
    line = {
        "op": args.op, "metric": spec["metric"], "value": value, "unit": spec["unit"],
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config == "cfg4" else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator; velocities N(0,1))",
        "config": {"workload": f"{args.config}: {describe(wl)}",
                   "l2": "flushed between timed calls (256 MiB memset outside the events)"
                   if flush is not None else "not flushed",
                   "timing": "per-call CUDA events on the library stream (kernels + small readback)"},
        "e2e": {"value": k_e2e * (R if args.config == "cfg4" else 1) / e2e_s, "unit": spec["unit"],
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": ("b2md_heat_flux_state" if args.op == "heat_flux" else
                         "b2md_rdf_accumulate_state + b2md_rdf_counts") + ", pinned host buffers"},
        "roofline": {"bound": "fp64", "kernel": kernel, "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": None,
                     "launch_ms": avg_s * 1e3},
        "kernel_ms_per_launch": {k: v[0] / max(1, v[1]) for k, v in kt.items()},
        "gpu_launches": int(sum(c for _, c in kt.values())),
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import pyoracle
            if pyoracle.ref_available():
                v, k = cpu_reference_op(args.op, wl, 10 ** 6, args.cpu_seconds)
                line["cpu_baseline"] = {"value": v, "unit": spec["unit"], "cores": 1, "kind": "reference",
                                        "sample": f"{k} calls of the reference's {args.op} on {args.config} (serial)"}
        except Exception as exc:
            line["cpu_baseline"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def tile_cull_kept_fraction(eng, wl):
    """Fraction of the upper-triangle 32x32 tiles the search's bounding-arc
    cull keeps on the final state, re-sorted as the device orders it (the
    arithmetic of k_search's arcs)."""
    L = wl.comp.box_length
    pos = eng.state().pos % L
    n = len(pos)
    # the device's slot order (k_sort_keys): columns of c^2 = 32 / (rho L), x inside
    G = max(1, min(1024, int(L / np.sqrt(32.0 / (n / L ** 3 * L)))))
    col = np.clip((pos[:, 2] / L * G).astype(np.int64), 0, G - 1) * G + \
        np.clip((pos[:, 1] / L * G).astype(np.int64), 0, G - 1)
    xq = np.clip((pos[:, 0] / L * 2 ** 20).astype(np.int64), 0, 2 ** 20 - 1)
    pos = pos[np.argsort((col << 20) | xq, kind="stable")]
    u = np.floor(pos * (2.0 ** 32 / L) + 0.5).astype(np.int64) % (1 << 32)
    nb = (n + 31) // 32
    pad = np.zeros((nb * 32, 3), dtype=np.int64)
    pad[:n] = u
    blk = pad.reshape(nb, 32, 3)
    off = ((blk - blk[:, :1, :] + (1 << 31)) % (1 << 32)) - (1 << 31)
    mn, mx = off.min(1), off.max(1)
    c = (blk[:, 0, :] + (mn + mx) // 2) % (1 << 32)
    h = (mx - mn + 1) // 2 + 1
    rmax = wl.opts.cutoff + 2 * max(sp.max_extent for sp in wl.comp.species)
    ru = rmax * 2.0 ** 32 / L
    kept, total = 0, 0
    for b in range(nb):
        d = np.abs(((c[b] - c[b:] + (1 << 31)) % (1 << 32)) - (1 << 31))
        g = np.maximum(d - h[b] - h[b:] - 2, 0).astype(float)
        kept += int(((g * g).sum(-1) <= ru * ru * (1 + 1e-6)).sum())
        total += nb - b
    return kept / total


def describe(wl):
    n = wl.comp.molecule_count()
    return (f"N={n} x {wl.replicas} replica(s), {len(wl.comp.species)} species, L={wl.comp.box_length:.6f}, "
            f"rc={wl.opts.cutoff:.6f}, dt={wl.dt}, method={int(wl.opts.method)}")


def run_group(args):
    """--gpus N > 1 in ONE process (no torchrun): b2md_create_group -- one
    context per device, ncclCommInitAll, the row-sharded step with its packed
    all-reduce, every device's calls on its own worker thread -- or, for the
    cfg4 replica batch, N independent engines (8 replicas each, no traffic).
    Per-step CUDA events on every device's stream, L2 flushed on every device
    between steps, the step time is the max over devices."""
    import torch
    import paper_1507_07548_b200 as b2
    N = args.gpus
    if torch.cuda.device_count() < N:
        raise SystemExit(f"--gpus {N}: only {torch.cuda.device_count()} CUDA device(s) visible")
    devs = list(range(N))
    if args.config == "cfg4":
        wls = [workload("cfg4", k, N) for k in devs]
        engines = [b2.Engine(w.comp, w.opts, w.dt, device=k, replicas=w.replicas) for k, w in zip(devs, wls)]
        for e, w in zip(engines, wls):
            e.set_state(w.states)
        wl = wls[0]
        group = None

        def step_all(k):
            for e in engines:
                e.step_async(k)

        def sync_all():
            for e in engines:
                e.sync()
    else:
        wl = workload(args.config, 0, 1)
        group = b2.EngineGroup(wl.comp, wl.opts, wl.dt, devices=devs, replicas=wl.replicas)
        group.set_state(wl.states)
        engines = group.engines
        step_all, sync_all = group.step_async, group.sync
    R, n = wl.replicas, wl.comp.molecule_count()
    streams = [torch.cuda.ExternalStream(e.stream(), device=k) for k, e in zip(devs, engines)]
    flushes = [None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{k}")
               for k in devs]
    for _ in range(max(3, args.warmup)):
        step_all(1)
    sync_all()
    interval, since = engines[0].sort_interval()
    equil = args.equil if args.equil >= 0 else (1000 if args.config == "cfg3" else 0)
    extra = (interval - since + interval * max(0, -(-(equil - (interval - since)) // interval))
             if interval > 0 else equil)
    if extra > 0:
        step_all(extra)
        sync_all()

    def timed_pass(steps):
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)] for _ in devs]
        for k in range(steps):
            for d in devs:
                ev[d][k][0].record(streams[d])
            step_all(1)
            for d in devs:
                ev[d][k][1].record(streams[d])
                if flushes[d] is not None:
                    with torch.cuda.stream(streams[d]):
                        flushes[d].zero_()
        sync_all()
        for d in devs:
            torch.cuda.synchronize(d)
        return max(float(sum(a.elapsed_time(b) for a, b in ev[d])) for d in devs)

    clocks = ClockSampler(0)
    clocks.start()
    total_ms = timed_pass(args.steps)
    clk = clocks.stop()
    for e in engines:
        e.profile(True, 1)
    n_all = min(args.steps, 50)
    timed_pass(n_all)
    kts = [e.kernel_times() for e in engines]
    for e in engines:
        e.profile(False)
    kt = kts[0]
    launches = sum(c for kt_ in kts for name, (ms, c) in kt_.items()) / max(1, n_all)
    _, stats = engines[0].energies()
    pairs_total = int(sum(s.com_pairs for s in stats))
    # end to end: host state to every device, the step, rank 0's state back
    nt = n * R
    pinned = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    bufs = [[pinned((nt, 3)), pinned((nt, 4)), pinned((nt, 3)), pinned((nt, 3)), pinned((nt, 3)),
             pinned((nt, 3))] for _ in (devs if group is None else devs[:1])]
    for e, b in zip(engines, bufs):
        e.get_state_raw(*b)
    point = all(sp.rotational_dof == 0 for sp in wl.comp.species)
    sel = (lambda b: (b[0], None, b[2], None, b[4], None)) if point else (lambda b: tuple(b))
    per_dev = 8 * nt * ((3 + 3 + 3) if point else (3 + 4 + 3 + 3 + 3 + 3))
    e2e_steps = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if group is None:
            for e, b in zip(engines, bufs):
                e.upload_state_raw(*sel(b))
                e.step_async(1)
            for e, b in zip(engines, bufs):
                e.get_state_raw(*sel(b))
        else:
            for e in engines:
                e.upload_state_raw(*sel(bufs[0]))
            group.step_async(1)
            group.sync()
            engines[0].get_state_raw(*sel(bufs[0]))
    e2e_s = time.perf_counter() - t0
    mult = R * N if args.config == "cfg4" else 1
    line = {
        "metric": METRIC, "value": args.steps * mult / (total_ms * 1e-3), "unit": "steps/s",
        "n_gpus": N, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.config == "cfg4" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded xoshiro256++ generator, paper_1507_07548_b200/configs.py)",
        "config": {
            "workload": f"{args.config}: {describe(wl)}",
            "parallelism": (f"replicas x{N} (one process, N engines)" if group is None else
                            f"row-sharded x{N} + NCCL all-reduce (one process: b2md_create_group)"),
            "l2": "flushed between timed steps on every device" if flushes[0] is not None else "not flushed",
            "timing": "per-step CUDA events on every device's library stream; max over devices",
        },
        "pair_interactions_per_s": pairs_total * args.steps * (N if args.config == "cfg4" else 1)
        / (total_ms * 1e-3),
        "e2e": {"value": e2e_steps * mult / e2e_s, "unit": "steps/s",
                "h2d_bytes_per_step": per_dev * N, "d2h_bytes_per_step": per_dev * (N if group is None else 1),
                "path": "b2md_upload_state on every device + step + b2md_get_state (pinned host buffers)"},
        "kernel_ms_per_launch": {k: v[0] / max(1, v[1]) for k, v in kt.items()},
        "gpu_launches": int(round(launches * args.steps)),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if group is not None:
        group.close()


def main():
    args = parse()
    if args.op != "step":
        (run_op_reference if args.impl == "reference" else run_op)(args)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.group or (args.gpus > 1 and "WORLD_SIZE" not in os.environ):
        run_group(args)
        return
    rank, world, local = dist_env()
    import torch
    import paper_1507_07548_b200 as b2

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workload(args.config, rank, world)
    R = wl.replicas
    n = wl.comp.molecule_count()
    eng = b2.Engine(wl.comp, wl.opts, wl.dt, device=local, replicas=R)
    if world > 1 and args.config != "cfg4":
        uid = [b2.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.attach_nccl(uid[0], rank, world)
    eng.set_state(wl.states)
    peak_gflops = b2.measure_fp64_peak(local)

    stream = torch.cuda.ExternalStream(eng.stream(), device=local)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    # ---- warm-up: W steps (single-step graphs instantiated) and one step at
    # every profiling level the later passes use (their graphs instantiated)
    done = 0
    for _ in range(max(3, args.warmup)):
        eng.step_async(1)
        done += 1
    eng.sync()
    for level in (3, 2, 1):
        eng.profile(True, level)
        eng.step_async(1)
        eng.sync()
        eng.profile(False)
        done += 1
    # ---- equilibration away from the lattice start (the cull is tightest on
    # the ordered start), padded so that the FIRST timed step re-sorts: a
    # K-step window then holds ceil(K / interval) re-sorts, never fewer than
    # its share
    interval, since = eng.sort_interval()
    equil = args.equil if args.equil >= 0 else (1000 if args.config == "cfg3" else 0)
    if interval > 0:
        to_due = interval - since
        extra = to_due + interval * max(0, -(-(equil - to_due) // interval))
    else:
        extra = equil
    if extra > 0:
        eng.step_async(extra)
        eng.sync()
        done += extra

    def timed_pass(steps, flush_between):
        """K single steps, each bracketed by CUDA events on the library's stream."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        with torch.cuda.stream(stream):
            for k in range(steps):
                starts[k].record(stream)
                eng.step_async(1)
                ends[k].record(stream)
                if flush_between is not None:
                    flush_between.zero_()
        eng.sync()
        torch.cuda.synchronize()
        return float(sum(s.elapsed_time(e) for s, e in zip(starts, ends)))

    # ---- timed region: device-resident steps as CUDA graphs, no per-kernel events
    clocks = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    total_ms = timed_pass(args.steps, flush)
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    if dist is not None:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    energies, stats = eng.energies()

    # ---- live kernel timing (CUDA events on the library stream, same step
    # structure, L2 flushed between steps): (1) events around the partner
    # search only; (2) events around the force kernel only, harvested after
    # every step -- the roofline's launch time is the MEDIAN per launch; (3)
    # events around every kernel, a short pass -- the per-kernel breakdown and
    # launch counts.  Event-record nodes stall the graph pipeline, so they are
    # kept out of the headline region.
    eng.profile(True, 2)
    timed_pass(args.steps, flush)
    kt_search = eng.kernel_times()
    eng.profile(False)

    def per_launch(level, family, steps):
        eng.profile(True, level)
        out, prev = [], (0.0, 0)
        with torch.cuda.stream(stream):
            for _ in range(steps):
                eng.step_async(1)
                ms, n_l = eng.kernel_times().get(family, (0.0, 0))  # harvest (syncs)
                if n_l > prev[1]:
                    out.append((ms - prev[0]) / (n_l - prev[1]))
                prev = (ms, n_l)
                if flush is not None:
                    flush.zero_()
        eng.sync()
        eng.profile(False)
        return out

    force_samples = per_launch(3, "force", args.steps)
    n_all = min(args.steps, 50)
    eng.profile(True, 1)
    timed_pass(n_all, flush)
    kt = eng.kernel_times()
    eng.profile(False)
    launches_per_step = sum(c for name, (ms, c) in kt.items()) / max(1, n_all)
    pairs_total = int(sum(s.com_pairs for s in stats))

    # ---- end to end through the C ABI with host buffers (pinned):
    # per step upload the full dynamic state (b2md_upload_state), step, download it
    def pinned(shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    nt = n * R
    hp, hq, hv, hw, hf, ht = (pinned((nt, 3)), pinned((nt, 4)), pinned((nt, 3)), pinned((nt, 3)),
                              pinned((nt, 3)), pinned((nt, 3)))
    eng.get_state_raw(hp, hq, hv, hw, hf, ht)
    # point molecules (rotational_dof 0 everywhere): the step neither reads nor
    # writes orientations, angular velocities or torques (engine.cpp:107-141
    # skips the rotor), so the per-step transfer is pos, vel and the cached
    # forces; rigid molecules move the full dynamic state
    point = all(sp.rotational_dof == 0 for sp in wl.comp.species)
    if point:
        hq = hw = ht = None
        h2d = d2h = 8 * nt * (3 + 3 + 3)
    else:
        h2d = d2h = 8 * nt * (3 + 4 + 3 + 3 + 3 + 3)
    e2e_steps = max(1, args.e2e_steps)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.upload_state_raw(hp, hq, hv, hw, hf, ht)
        eng.step_async(1)  # its NumericalError is reported by get_state
        eng.get_state_raw(hp, hq, hv, hw, hf, ht)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    replica_steps = args.steps * (R * world if args.config == "cfg4" else 1)
    value = replica_steps / (total_ms * 1e-3)
    e2e_value = e2e_steps * (R * world if args.config == "cfg4" else 1) / e2e_s

    # ---- roofline of the dominant kernel: the force walk (fp64 CUDA cores).
    # Algorithmic work: 32 flop per single-site LJ pair in
    # cutoff; multi-site: 86 per LJ term, counted as if every term of a passing
    # molecule pair were inside rc (an upper bound).
    peak = peak_gflops / 1e3
    avg_force_s = statistics.median(force_samples) * 1e-3 if force_samples else 0.0
    single_site = all(sp.n_sites == 1 for sp in wl.comp.species)
    cand = n * (n - 1) // 2 * R
    # cluster walk: no search launches -- the force kernel decides every
    # candidate pair itself (partner search fused into the LJ kernel), so its
    # algorithmic work is the search's plus the forces'
    fused_search = single_site and kt_search.get("search", (0.0, 0))[1] == 0
    nlist = eng.nlist_info() if fused_search else {"active": 0}
    if fused_search:
        force_flop = cand * FLOP_CANDIDATE + pairs_total * FLOP_LJ_SINGLE
        walk = ("k_force_nl: once-per-pair cluster-pair list (each pair evaluated once, partner-side "
                "sums written to per-entry records; the fixed-order record reduction k_nl_reduce is "
                "timed apart as force_jsum)" if nlist["active"] else
                "k_force_cpair: both-rows cluster walk")
        force_note = (f"{walk}; partner search fused with LJ; {FLOP_CANDIDATE} flop per "
                      f"candidate pair i<j decided + {FLOP_LJ_SINGLE} per pair in cutoff")
    elif single_site:
        force_flop = pairs_total * FLOP_LJ_SINGLE
        force_note = f"{FLOP_LJ_SINGLE} flop per single-site LJ pair in cutoff"
    else:
        terms = max(sp.n_sites for sp in wl.comp.species) ** 2
        force_flop = pairs_total * (2 + 86 * terms)
        force_note = f"(2 + 86 x {terms} terms) flop per passing molecule pair (upper bound)"
    achieved = force_flop / avg_force_s / 1e12 if avg_force_s > 0 else 0.0
    traffic = None
    executed = None
    prof = ROOT / "profiles" / f"ncu_{args.config}_force.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get("dram_bytes_per_launch")
            executed = pj.get("fp64_pipe_pct")
        except Exception:
            traffic = None
    # partner search: share of the step and the tiles the bounding-arc cull kept
    search_ms, search_launches = kt_search.get("search", (0.0, 0))
    avg_search_s = search_ms * 1e-3 / max(1, search_launches)
    kept = tile_cull_kept_fraction(eng, wl) if single_site and R == 1 and not fused_search else None
    step_s = total_ms * 1e-3 / args.steps
    fp64_step = ((cand * FLOP_CANDIDATE + pairs_total * FLOP_LJ_SINGLE) / step_s / 1e12 / peak
                 if single_site and world == 1 else None)
    step_kernels = sum(c for name, (ms, c) in kt.items() if name != "allreduce")

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "steps/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if args.config == "cfg4" else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded xoshiro256++ generator, paper_1507_07548_b200/configs.py)",
        "config": {
            "workload": f"{args.config}: {describe(wl)}",
            "parallelism": (f"replicas x{world}" if args.config == "cfg4" else
                            (f"row-sharded x{world} + NCCL all-reduce" if world > 1 else "single GPU")),
            "l2": "flushed between timed steps (256 MiB memset outside the per-step events)"
            if flush is not None else "not flushed",
            "timing": "per-step CUDA events on the library stream; max over ranks",
            "pre_steps": done,
            "sort": (f"re-sort every {interval} steps; the first timed step re-sorts "
                     f"({-(-args.steps // interval)} re-sorts in the window)" if interval > 0
                     else "fixed slot order"),
        },
        "pair_interactions_per_s": pairs_total * args.steps * (world if args.config == "cfg4" else 1)
        / (total_ms * 1e-3),
        "pairs_in_cutoff_per_step": pairs_total,
        "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "b2md_upload_state + b2md_step_async + b2md_get_state (one host sync), pinned host buffers"
                        + ("; point molecules: pos, vel, forces (orientations / angular velocities / "
                           "torques are not read or written by their step and stay resident)" if point else
                           "; full dynamic state (pos, quaternion, vel, angular vel, forces, torques)")},
        "roofline": {
            "bound": "fp64",
            "kernel": f"k_force_* partner walk ({force_note})",
            "achieved": achieved,
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None,
            "traffic": traffic,
            "peak_source": "DFMA microbenchmark measured in this run (MEASURED_PEAKS.json has no fp64 entry)",
            "launch_ms": avg_force_s * 1e3,
            "launch_ms_stats": ({"median": statistics.median(force_samples), "min": min(force_samples),
                                 "max": max(force_samples), "launches": len(force_samples)}
                                if force_samples else None),
            "share_of_step": avg_force_s / max(1e-12, step_s),
            "fp64_pipe_pct_executed": executed,
            "executed_note": "ncu sm__pipe_fp64_cycles_active of the same kernel (profiles/): the fp64 "
                             "work actually issued, vs the algorithmic count above",
            "launch_timing": "median of per-launch CUDA-event times around the force kernel only "
                             "(a second K-step pass, same graph step structure, L2 flushed between "
                             "steps, profiling graph warmed before); ncu launch list in profiles/",
        },
        "search": ({
            "launch_ms": None,
            "candidates": cand,
            "note": "fused into the force kernel: cluster pairs (8 x 8 slots) that are provably > rc "
                    "apart are skipped (bounding arcs / member distances at the list build less the "
                    "displacement since, exact); the rest are decided on the reference's fp64 r2 "
                    "per pair",
            "pair_list": ({"entries": nlist["entries"], "rebuild_interval": nlist["interval"],
                           "skin": nlist["skin_e6"] * 1e-6, "stale": bool(nlist["stale"])}
                          if nlist["active"] else None),
        } if fused_search else {
            "launch_ms": avg_search_s * 1e3,
            "share_of_step": avg_search_s / max(1e-12, step_s),
            "candidates": cand,
            "tile_cull_kept_fraction": kept,
            "note": "32x32 tiles whose blocks' bounding arcs are > rmax apart are skipped (exact)",
        }),
        "fp64_fraction_step": fp64_step,
        "fp64_fraction_step_def": "(all n(n-1)/2 candidates x 17 + pairs in cutoff x 32) flop per "
                                  "step / device step time / fp64 peak (SURVEY.md 8(d) convention; "
                                  "culled candidates count as work the reference does)",
        "kernel_ms_per_launch": {k: v[0] / max(1, v[1]) for k, v in kt.items()},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            from oracle import pyoracle
            if pyoracle.ref_available():
                # the reference engine at W = all physical cores (the value) and
                # at W = 1, on the same workload and starting state
                phys = physical_cores()
                v, k, w = cpu_reference_run(wl, 10 ** 6, 0.65 * args.cpu_seconds, phys, min_steps=2)
                v1, k1, _ = cpu_reference_run(wl, 10 ** 6, 0.35 * args.cpu_seconds, 1, min_steps=1)
                line["cpu_baseline"] = {
                    "value": v, "unit": "steps/s", "cores": w, "kind": "reference",
                    "sample": f"{k} tmd::Engine::step of {args.config} at W={w} (all physical cores) "
                              f"after set_state of the same start state",
                    "w1": {"value": v1, "unit": "steps/s", "cores": 1,
                           "sample": f"{k1} tmd::Engine::step at W=1"},
                    "logical_cpus": os.cpu_count()}
        except Exception as exc:  # the GPU number stands without it
            line["cpu_baseline"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
