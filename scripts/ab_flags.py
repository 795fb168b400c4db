"""Graph-replayed ms/sweep of several configs under several ifctn_create flags, interleaved
(A/B in one process).  usage: ab_flags.py CONFIG[,CONFIG..] FLAG[,FLAG..] [ROUNDS]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

cfgs = sys.argv[1].split(",")
flags = [int(f) for f in sys.argv[2].split(",")]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for name in cfgs:
    p = make_config(name)
    n = 20 if name == "C5" else 100
    obs, mask, g0 = dev(p.observed), dev(p.mask), dev(p.G0)
    for r in range(rounds):
        for fl in flags:
            s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho, flags=fl)
            s.sweep(n)
            s.sync()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.sweep(n)
            b.record()
            torch.cuda.synchronize()
            print(f"{name} flags={fl:3d} {1e3 * a.elapsed_time(b) / n:9.1f} us/sweep", flush=True)
            s.close()
