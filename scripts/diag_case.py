"""Per-block parity of one sweep for one random case (tests/test_gpu_random.py), in fp32 and
fp64 and under the diagnostic flags that switch kernel paths."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from gpu_util import make_solver, oracle_state, rel  # noqa: E402
from oracle import oracle as O  # noqa: E402
from synth import make_problem  # noqa: E402
from test_gpu_random import _case  # noqa: E402
from paper_2511_16358_b200 import (IFCTN_FLAG_NO_FUSE, IFCTN_FLAG_NO_SOLVE_REDUCE,  # noqa: E402
                                   IFCTN_FLAG_NO_VBLOCK)

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 18
dims, R, dtype = _case(seed)
for dt in (dtype, "float64"):
    p = make_problem(f"rand{seed}", dims, R, dt, "normal", sr=0.3, init_kind="normal", seed=seed)
    sh, G, X = oracle_state(p)
    st, _, _ = O.sweep(sh, G, X, p.mask, p.rho, O.objective(sh, G, X), False)
    for fl, lab in ((0, "default"), (IFCTN_FLAG_NO_VBLOCK, "no_vblock"), (IFCTN_FLAG_NO_SOLVE_REDUCE, "no_solve_reduce"),
                    (IFCTN_FLAG_NO_VBLOCK | IFCTN_FLAG_NO_SOLVE_REDUCE | IFCTN_FLAG_NO_FUSE, "all_off")):
        s = make_solver(p, flags=fl)
        s.sweep(1)
        Gg = s.factors().cpu().numpy()
        errs = []
        for k in range(p.N):
            for i in range(p.N):
                if i != k:
                    errs.append(f"({k},{i}) {rel(O.factor(sh, Gg, k, i), O.factor(sh, G, k, i)):.1e}")
        print(dt, lab, "X", f"{rel(s.reconstruct().cpu().numpy(), X):.2e}", " ".join(errs))
