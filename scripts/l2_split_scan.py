"""Per-block a2 times (ifctn_profile_sweep) of one config under pinned L2-pass splits
(IFCTN_L2_KEPT="CG,wpi,Z", IFCTN_L2_RED="TL,Z"; 0 = free).  usage: l2_split_scan.py CFG kept|red SPEC[;SPEC..]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

name, kind, specs = sys.argv[1], sys.argv[2], sys.argv[3].split(";")
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
obs, mask, g0 = dev(p.observed), dev(p.mask), dev(p.G0)
blocks = [(k, i) for k in range(p.N) for i in range(p.N) if i != k]
sel = [b for b, (k, i) in enumerate(blocks) if ((k == 0 or i == 0) == (kind == "kept"))]
print(name, kind, "blocks", [blocks[b] for b in sel])
for spec in specs:
    os.environ["IFCTN_L2_KEPT" if kind == "kept" else "IFCTN_L2_RED"] = spec
    try:
        s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho)
    except Exception as e:  # split not feasible for some block
        print(f"{spec:>10s}  infeasible ({e})")
        continue
    s.sweep(2)
    best = None
    for _ in range(5):
        prof = s.profile_sweep()
        if best is None or sum(prof) < sum(best):
            best = prof
    s.close()
    print(f"{spec:>10s} ", " ".join(f"{1e3 * best[3 * b]:6.1f}" for b in sel), f"  sum {1e3 * sum(best[3 * b] for b in sel):7.1f}")
