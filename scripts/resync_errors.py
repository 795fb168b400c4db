import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import oracle as O
from synth import make_config
from gpu_util import make_solver, rel
from paper_2511_16358_b200 import IFCTN_FLAG_NO_L2PASS
for name in ["C5s", "C3s", "C4s"]:
    for fl in (0, IFCTN_FLAG_NO_L2PASS):
        p = make_config(name)
        s = make_solver(p, flags=fl)
        sh = O.Shape(p.dims, p.ranks)
        out = []
        for sweep in range(4):
            G = s.factors().cpu().numpy().astype(np.float64)
            X = s.reconstruct().cpu().numpy().astype(np.float64)
            st, _, _ = O.sweep(sh, G, X, p.mask, p.rho, O.objective(sh, G, X), False)
            s.sweep(1)
            out.append((rel(s.factors().cpu().numpy(), G), rel(s.reconstruct().cpu().numpy(), X)))
        print(name, "flags", fl, " ".join(f"G {a:.2e} X {b:.2e} |" for a, b in out))
