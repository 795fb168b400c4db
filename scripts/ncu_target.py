"""Small driver for ncu captures: create one config's solver and run a few plain-launch
sweeps (no CUDA graph) so every kernel shows up as its own launch."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_FLAG_NO_GRAPH, Solver  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--sweeps", type=int, default=2)
ap.add_argument("--flags", type=int, default=IFCTN_FLAG_NO_GRAPH)
a = ap.parse_args()
p = make_config(a.config)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=a.flags)
s.sweep(a.sweeps)
s.sync()
print("ok", a.config, a.sweeps, s.rse(dev(p.truth)))
