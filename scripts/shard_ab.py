"""A/B of one library build (IFCTN_LIB) on the rank-0 shard of a W-way sharded config (one
process, no-op host all-reduce): per-block a2 pass times of one profiled sweep and GB/s."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from paper_2511_16358_b200 import dist as D  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tag = sys.argv[3] if len(sys.argv) > 3 else os.environ.get("IFCTN_LIB", "default")
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
sm, sb, se = D.shard_range(p.dims, world, 0)
obs = D.shard_tensor(p.observed, p.dims, sm, sb, se)
d = D.make_dist(0, world, -1, host_allreduce=lambda a: None)
s = Solver(p.dims, p.ranks, dev(obs), dev(D.shard_tensor(p.mask, p.dims, sm, sb, se)),
           dev(D.shard_factors(p.G0, p.dims, p.ranks, sm, sb, se)), rho=p.rho, dist=d)
best = None
for rep in range(3):
    prof = s.profile_sweep()
    t, k2 = 0, []
    for k in range(p.N):
        for i in range(p.N):
            if i == k:
                continue
            k2.append(prof[t])
            t += 2 + (2 if k != sm else 1)
    if best is None or sum(k2) < sum(best):
        best = k2
gbs = obs.size * p.dtype.itemsize / (statistics.mean(best) / 1e3) / 1e9
print(f"{tag:24s} {name}/{world} rank0 a2 mean {1e3 * statistics.mean(best):.1f} us = {gbs:.0f} GB/s; "
      f"by block " + " ".join(f"{1e3 * v:.0f}" for v in best))
