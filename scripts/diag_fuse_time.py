"""Graph-replayed sweep time on one config with the default (fused) path vs NO_FUSE vs
NO_VBLOCK, device-timed with CUDA events on the solver's stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_FLAG_NO_FUSE, IFCTN_FLAG_NO_VBLOCK, Solver  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
obs, mask, g0 = dev(p.observed), dev(p.mask), dev(p.G0)
for fl, lab in ((0, "fused"), (IFCTN_FLAG_NO_FUSE, "no_fuse"), (IFCTN_FLAG_NO_FUSE | IFCTN_FLAG_NO_VBLOCK, "plain")):
    s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho, flags=fl)
    s.sweep(n)
    s.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    s.sweep(n)
    b.record()
    torch.cuda.synchronize()
    print(f"{name} {lab:8s} {a.elapsed_time(b) / n:.3f} ms/sweep  launches {s.launch_count()}")
    s.close()
