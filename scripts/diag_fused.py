import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from gpu_util import make_solver, oracle_state, rel
from oracle import oracle as O
from synth import make_config
from paper_2511_16358_b200 import IFCTN_FLAG_NO_FUSE, IFCTN_FLAG_NO_VBLOCK
for name in ['C5s', 'C2s']:
    p = make_config(name)
    for ns in (1, 2, 3):
        sh, G, X = oracle_state(p)
        F = O.objective(sh, G, X)
        for _ in range(ns): O.sweep(sh, G, X, p.mask, p.rho, F, False)
        out = []
        for fl in (0, IFCTN_FLAG_NO_FUSE, IFCTN_FLAG_NO_FUSE | IFCTN_FLAG_NO_VBLOCK):
            s = make_solver(p, flags=fl); s.sweep(ns)
            out.append((rel(s.factors().cpu().numpy(), G), rel(s.reconstruct().cpu().numpy(), X)))
        print(name, ns, ['G %.2e X %.2e' % o for o in out])
