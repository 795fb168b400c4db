"""Small workload for compute-sanitizer: C1 (fp64) and C2s/C2rs-sized runs through
the graph/fused path, plain launches, a traced run, the large-rank solve, metrics, RSE and
the rank-grid driver."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_FLAG_NO_GRAPH, Solver  # noqa: E402
from paper_2511_16358_b200.grid import rank_grid  # noqa: E402
from synth import MSI_GRID, grid_rank_matrix, init_factors, make_config  # noqa: E402

dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
for name in ("C1", "C2s", "C2rs", "C4s"):
    p = make_config(name)
    for fl in (0, IFCTN_FLAG_NO_GRAPH):
        s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=fl)
        s.sweep(3)
        s.sweep(2, trace=True)
        s.rse(dev(p.truth))
        s.metrics(dev(p.truth))
        s.close()
    print(name, "ok", flush=True)
p = make_config("C2s")
inst = []
for (r12, r3) in MSI_GRID[:3]:
    R = grid_rank_matrix(r12, r3)
    g, _ = init_factors(p.dims, R, p.observed, p.mask, p.dtype, "uniform", 0)
    inst.append(dict(ranks=R, rho=p.rho, init=g))
rank_grid(p.dims, dev(p.observed), dev(p.mask), inst, 2, truth=dev(p.truth), concurrency=2)
print("grid ok")
