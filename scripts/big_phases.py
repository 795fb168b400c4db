"""Per-phase clocks of one block_solve_big CTA (IFCTN_EXP_PHASE_CLOCKS build via IFCTN_LIB):
usage: IFCTN_LIB=exp/phase.so python scripts/big_phases.py CONFIG FLAGS"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

p = make_config(sys.argv[1])
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=int(sys.argv[2]))
s.sweep(3)
s.sync()
