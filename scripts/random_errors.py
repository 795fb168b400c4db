"""Per-seed one-sweep errors of tests/test_gpu_random.py's cases (GPU vs float64 oracle) in
the case's own dtype and in float64 — to size the tolerance from data, not guesswork."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from oracle import oracle as O  # noqa: E402
from synth import make_problem  # noqa: E402
from gpu_util import make_solver, oracle_state, rel  # noqa: E402
from test_gpu_random import _case  # noqa: E402

O.set_threads(8)
for seed in range(24):
    dims, R, dtype = _case(seed)
    row = [seed, dims, int(R.max())]
    for dt in (dtype, "float64"):
        p = make_problem(f"rand{seed}", dims, R, dt, "normal", sr=0.3, init_kind="normal", seed=seed)
        s = make_solver(p)
        sh, G, X = oracle_state(p)
        O.sweep(sh, G, X, p.mask, p.rho, O.objective(sh, G, X), False)
        s.sweep(1)
        row += [dt, f"{rel(s.factors().cpu().numpy(), G):.2e}", f"{rel(s.reconstruct().cpu().numpy(), X):.2e}"]
    print(*row, flush=True)
