"""Per-block launch times of one profiled sweep (ifctn_profile_sweep: [a2, reduce, solve] per
block, then refill/finaliser) for the default build with and without given create flags."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_FLAG_NO_L2PASS, Solver  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
blocks = [(k, i) for k in range(p.N) for i in range(p.N) if i != k]
res = {}
for tag, fl in (("l2", 0), ("walk", IFCTN_FLAG_NO_L2PASS)):
    s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=fl)
    s.sweep(2)
    best = None
    for _ in range(3):
        prof = s.profile_sweep()
        if best is None or sum(prof) < sum(best):
            best = prof
    res[tag] = best
    s.close()
print(f"{name}: per block us  [a2+reduce | solve]  l2 vs walk")
for b, (k, i) in enumerate(blocks):
    a = res["l2"][3 * b] + res["l2"][3 * b + 1]
    w = res["walk"][3 * b] + res["walk"][3 * b + 1]
    print(f"  ({k},{i}) dims {p.dims[k]}x{p.dims[i]}: l2 {1e3 * a:7.1f} | {1e3 * res['l2'][3 * b + 2]:6.1f}   "
          f"walk {1e3 * w:7.1f} | {1e3 * res['walk'][3 * b + 2]:6.1f}")
print(f"  total l2 {1e3 * sum(res['l2']):.1f} us, walk {1e3 * sum(res['walk']):.1f} us")
