"""Diagnostics: per-launch device times of one sweep for the small configs, and the phase
split of the e2e solve on C5 (create from pinned host / sweeps / read back)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_X, Solver  # noqa: E402
from synth import make_config  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for name in sys.argv[1:] or ["C2", "C4"]:
    p = make_config(name)
    s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho)
    s.sweep(3)
    s.sync()
    prof = s.profile_sweep()
    print(name, "launches", len(prof), "sum us", round(1e3 * sum(prof), 1))
    print("  ", " ".join(f"{1e3 * t:.1f}" for t in prof))

p = make_config("C5")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
obs, mask, g0 = pin(p.observed), pin(p.mask), pin(p.G0)
out = torch.empty(p.n, dtype=torch.float32).pin_memory()
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.sweep(50, trace=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s.reconstruct(IFCTN_X, out=out)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    s.close()
    print(f"e2e C5 create {t1 - t0:.3f}s  50 sweeps(trace) {t2 - t1:.3f}s  readback {t3 - t2:.3f}s")
