"""Per-CTA timeline of the a2 passes (diagnosis build IFCTN_EXP_TIMELINE, IFCTN_LIB=exp/tl.so):
for every block, one ifctn_block_coefficients call (pass + reduce, plain launches) and the
%globaltimer stamps [start, prologue end, end] of each CTA: launch ramp, prologue, work, tail."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16358_b200 import IFCTN_FLAG_NO_GRAPH, Solver, _abi  # noqa: E402
from synth import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = make_config(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
lib = _abi.lib()
tl = lib.ifctn_exp_timeline
tl.argtypes = [ctypes.c_void_p, ctypes.c_int]
if world > 1:
    from paper_2511_16358_b200 import dist as D
    sm, sb, se = D.shard_range(p.dims, world, 0)
    d = D.make_dist(0, world, -1, host_allreduce=lambda a: None)
    s = Solver(p.dims, p.ranks, dev(D.shard_tensor(p.observed, p.dims, sm, sb, se)),
               dev(D.shard_tensor(p.mask, p.dims, sm, sb, se)),
               dev(D.shard_factors(p.G0, p.dims, p.ranks, sm, sb, se)), rho=p.rho, dist=d,
               flags=IFCTN_FLAG_NO_GRAPH)
else:
    s = Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, flags=IFCTN_FLAG_NO_GRAPH)
buf = np.zeros(3 * 4096, dtype=np.uint64)
for rep in range(2):
    for k in range(p.N):
        for i in range(p.N):
            if i == k:
                continue
            tl(None, -1)
            s.block_coefficients(k, i)
            tl(buf.ctypes.data, 4096)
            t = buf.reshape(-1, 3).astype(np.int64)
            t = t[t[:, 0] > 0]
            if rep == 0 or len(t) == 0:
                continue
            t0 = t[:, 0].min()
            st, pe, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
            print(f"{name} block ({k},{i}) CTAs {len(t):4d}: start last {st.max():6.2f} us | prologue med "
                  f"{np.median(pe - st):5.2f} | CTA time med {np.median(en - st):6.2f} min {np.min(en - st):6.2f} "
                  f"max {np.max(en - st):6.2f} | first end {en.min():6.2f} last end {en.max():6.2f}")
