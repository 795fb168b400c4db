"""Graph-replayed us/sweep of several configs under several IFCTN_TUNE_* environment settings
(read by ifctn_create), interleaved in one process.
usage: ab_env.py CONFIG[,CONFIG..] 'VAR=V[;VAR=V]' ['VAR=V' ..]   ('-' = no override)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

cfgs = sys.argv[1].split(",")
settings = sys.argv[2:] or ["-"]
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
keys = {kv.split("=")[0] for st in settings if st != "-" for kv in st.split(";")}
for name in cfgs:
    p = make_config(name)
    n = 20 if name == "C5" else 100
    obs, mask, g0 = dev(p.observed), dev(p.mask), dev(p.G0)
    for r in range(2):
        for st in settings:
            for k in keys:
                os.environ.pop(k, None)
            if st != "-":
                for kv in st.split(";"):
                    k, v = kv.split("=")
                    os.environ[k] = v
            s = Solver(p.dims, p.ranks, obs, mask, g0, rho=p.rho)
            s.sweep(n)
            s.sync()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.sweep(n)
            b.record()
            torch.cuda.synchronize()
            print(f"{name} {st:40s} {1e3 * a.elapsed_time(b) / n:9.1f} us/sweep", flush=True)
            s.close()
