"""A/B timing of one library build (IFCTN_LIB) on one config: graph-replayed fused sweeps
(ms/sweep, CUDA events) and the per-launch split of one profiled sweep."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tag = sys.argv[3] if len(sys.argv) > 3 else os.environ.get("IFCTN_LIB", "default")
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho)
s.sweep(n)
s.sync()
ts = []
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    s.sweep(n)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / n)
prof = s.profile_sweep()
passes = [prof[3 * b] for b in range(len(prof) // 3)]
print(f"{tag:28s} {name} fused {min(ts):.3f} ms/sweep (reps {' '.join(f'{t:.3f}' for t in ts)})  "
      f"a2 mean {1e3 * np.mean(passes):.1f} us  refill {1e3 * prof[-2]:.1f} us")
