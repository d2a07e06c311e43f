"""CPU, world_size 2 over gloo: the multi-GPU decomposition (tile-row shards
of the i<j triangle + k-vector ranges, b2md_shard_plan) followed by one
all-reduce of (forces, torques, energy sums) reproduces the full evaluation.
This is the host logic of the NCCL path (b2md_attach_nccl), exercised with
the oracle as each rank's compute."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import systems
    from paper_1507_07548_b200 import configs
    if name == "lj":
        wl = configs.lj_fluid_config(700, 0.8, 3.0, seed=2)
        return wl.comp, wl.opts, wl.states[0]
    if name == "water":
        import golden_cases
        return golden_cases._water_ions_small(60, 3, 5)
    comp, opts = systems.tri_rotor(90, 9.0, 3.5)
    return comp, opts, systems.random_state(comp, 3, 0.9)


def _worker(rank, world, port, name, q):
    sys.path.insert(0, ROOT)
    from oracle import pyoracle
    import paper_1507_07548_b200 as b2
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    comp, opts, st = _case(name)
    o = pyoracle.OracleFF(comp, opts)
    nk = pyoracle.oracle_lib().oracle_ff_kvector_count(o.h)
    plan = b2.shard_plan(comp.molecule_count(), nk, world, rank)
    f, t, sums = o.evaluate_shard(st.pos, st.orient, plan["row_begin"], plan["row_end"],
                                  plan["k_begin"], plan["k_end"])
    packed = torch.from_numpy(np.concatenate([f.ravel(), t.ravel(), sums]))
    dist.all_reduce(packed)
    if rank == 0:
        q.put(packed.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lj", "tri", "water"])
def test_two_rank_shards_reproduce_full_evaluation(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle import pyoracle
    comp, opts, st = _case(name)
    full = pyoracle.OracleFF(comp, opts).evaluate(st.pos, st.orient)
    n = comp.molecule_count()
    f, t, sums = got[:3 * n].reshape(n, 3), got[3 * n:6 * n].reshape(n, 3), got[6 * n:]
    fs = max(1.0, np.abs(full["force"]).max())
    assert np.abs(f - full["force"]).max() <= 1e-12 * fs
    assert np.abs(t - full["torque"]).max() <= 1e-12 * max(1.0, np.abs(full["torque"]).max())
    e = full["energy"]
    assert sums[0] == pytest.approx(e.lj, rel=1e-12, abs=1e-12)
    assert sums[1] == pytest.approx(e.elec_real, rel=1e-12, abs=1e-12)
    assert sums[5] == pytest.approx(full["virial"], rel=1e-12, abs=1e-12)
    assert sums[6] == pytest.approx(e.elec_recip, rel=1e-12, abs=1e-12)
    assert int(sums[7]) == full["com_pairs"]
