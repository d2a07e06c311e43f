"""Host-side breakdown of one end-to-end step (b2md_upload_state + b2md_step_async +
b2md_get_state with pinned host buffers): wall time of each call, and the same three
stages timed on the device with CUDA events.  Usage: python tools/e2e_breakdown.py [cfg]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1507_07548_b200 import Engine, configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wl = configs.make(cfg)
R = len(wl.states)
eng = Engine(wl.comp, wl.opts, wl.dt, replicas=R) if R > 1 else Engine(wl.comp, wl.opts, wl.dt)
eng.set_state(wl.states if R > 1 else wl.states[0])
eng.step(100)
nt = wl.comp.molecule_count() * R


def pinned(shape):
    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


hp, hq, hv, hw, hf, ht = (pinned((nt, 3)), pinned((nt, 4)), pinned((nt, 3)), pinned((nt, 3)),
                          pinned((nt, 3)), pinned((nt, 3)))
eng.get_state_raw(hp, hq, hv, hw, hf, ht)
if all(sp.rotational_dof == 0 for sp in wl.comp.species):
    hq = hw = ht = None
K = 300
t = np.zeros((K, 4))
for k in range(K):
    t0 = time.perf_counter()
    eng.upload_state_raw(hp, hq, hv, hw, hf, ht)
    t1 = time.perf_counter()
    eng.step_async(1)
    t2 = time.perf_counter()
    eng.get_state_raw(hp, hq, hv, hw, hf, ht)
    t3 = time.perf_counter()
    t[k] = (t1 - t0, t2 - t1, t3 - t2, t3 - t0)
m = np.median(t[50:], axis=0) * 1e6
print(f"{cfg}: upload call {m[0]:.1f} us, step_async call {m[1]:.1f} us, get_state call (with the sync) "
      f"{m[2]:.1f} us, total {m[3]:.1f} us")
# device-only timing of the three stages (stream-ordered events around the same calls)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(K):
    eng.step_async(1)
eng.sync()
print(f"{cfg}: device-resident steps {(time.perf_counter() - t0) / K * 1e6:.1f} us each (no transfers, no L2 flush)")
