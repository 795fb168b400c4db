"""Per-block launch times of one profiled sweep (ifctn_profile_sweep: [a2, reduce, solve] per
block, then refill/finaliser) under several create flags.  usage: block_flags.py CFG FLAG[,FLAG..]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2r"
flags = [int(f) for f in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
blocks = [(k, i) for k in range(p.N) for i in range(p.N) if i != k]
for fl in flags:
    s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=fl)
    s.sweep(2)
    best = None
    for _ in range(5):
        prof = s.profile_sweep()
        if best is None or sum(prof) < sum(best):
            best = prof
    s.close()
    print(f"{name} flags={fl}: per block us [a2 | reduce | solve]")
    for b, (k, i) in enumerate(blocks):
        print(f"  ({k},{i}) {1e3 * best[3 * b]:7.1f} | {1e3 * best[3 * b + 1]:6.1f} | {1e3 * best[3 * b + 2]:6.1f}")
    print("  rest:", " ".join(f"{1e3 * x:.1f}" for x in best[3 * len(blocks):]), f" total {1e3 * sum(best):.1f} us")
