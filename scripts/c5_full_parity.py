"""Full-size C5 parity (the final-RSE parity of the headline config needs the
oracle to run in full).  50 sweeps of C5 on the GPU (fp32, traced) and in the float64 oracle
(all host cores); reports per-sweep objective traces, final RSE of both, their gap against
reading R22, and the relative difference of the final X.  Output: one JSON document."""
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

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
t0 = time.time()
p = make_config("C5")
gen_s = time.time() - t0
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho)
t1 = time.time()
done, rows = s.sweep(sweeps, trace=True)
gpu_s = time.time() - t1
rse_gpu = s.rse(dev(p.truth))
Xg = s.reconstruct().cpu().numpy()
s.close()
del s
torch.cuda.empty_cache()

O.build()
threads = os.cpu_count() or 1
O.set_threads(threads)
sh = O.Shape(p.dims, p.ranks)
G = p.G0.astype(np.float64)
X = O.init_x(p.observed, p.mask)
t2 = time.time()
r, trace = O.solve(sh, G, X, p.mask, p.rho, sweeps, 0.0, True)
orc_s = time.time() - t2
rse_orc = O.rse(p.truth.astype(np.float64), X)
nX = np.linalg.norm(X)
xdiff = float(np.linalg.norm(Xg.astype(np.float64) - X) / nX)
obj_gpu = [row["objective"] for row in rows]
obj_orc = [float(t[1]) for t in trace]
out = {"config": "C5", "sweeps": sweeps, "gpu_sweeps_done": done, "oracle_status": int(r),
       "oracle_threads": threads, "generation_s": gen_s, "gpu_s_traced": gpu_s, "oracle_s": orc_s,
       "rse_gpu": rse_gpu, "rse_oracle": rse_orc,
       "rse_gap": abs(rse_gpu - rse_orc), "rse_bound_R22": 1e-3 * rse_orc + 1e-5,
       "rse_within_R22": abs(rse_gpu - rse_orc) <= 1e-3 * rse_orc + 1e-5,
       "x_rel_diff_final": xdiff,
       "objective_rel_gap_per_sweep": [abs(a - b) / abs(b) for a, b in zip(obj_gpu, obj_orc)],
       "objective_gpu": obj_gpu, "objective_oracle": obj_orc}
print(json.dumps(out))
