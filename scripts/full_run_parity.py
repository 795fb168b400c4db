"""Full-run RSE parity on the configured sweep counts (north star: final RSE within 1e-3
relative after the full run) for configs C1–C4 and C2r: GPU (fused graph path, fp32/fp64 as
configured) vs the float64 oracle from the same seeded inputs.  One JSON document."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

O.build()
O.set_threads(os.cpu_count() or 1)
out = {}
for name in (sys.argv[1:] or ["C1", "C2", "C3", "C4", "C2r"]):
    p = make_config(name)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho)
    s.sweep(p.sweeps)
    s.sync()
    rse_gpu = s.rse(dev(p.truth))
    met = s.metrics(dev(p.truth))
    s.close()
    sh = O.Shape(p.dims, p.ranks)
    G = p.G0.astype(np.float64)
    X = O.init_x(p.observed, p.mask)
    t0 = time.time()
    r, _ = O.solve(sh, G, X, p.mask, p.rho, p.sweeps, 0.0, True)
    el = time.time() - t0
    rse_orc = O.rse(p.truth.astype(np.float64), X)
    tol = 1e-3 * rse_orc + (1e-10 if p.dtype == np.float64 else 1e-5)
    out[name] = {"sweeps": p.sweeps, "rse_gpu": rse_gpu, "rse_oracle": rse_orc,
                 "gap": abs(rse_gpu - rse_orc), "bound_R22": tol, "within": abs(rse_gpu - rse_orc) <= tol,
                 "oracle_status": int(r), "oracle_s": el,
                 "gpu_metrics": {k: (v if v == v and abs(v) != float("inf") else str(v)) for k, v in met.items()}}
    print(name, out[name], file=sys.stderr, flush=True)
print(json.dumps(out))
