"""The library's real multi-process path on one GPU (-m gpu): W separate processes, each with
its own CUDA context and its own ifctn context over its shard, the per-block
Gram/RHS partials summed across processes by a gloo all_reduce through the ifctn_dist
host_allreduce hook (tests/mp_rank_worker.py).  The gathered result must reproduce the
single-GPU run (1e-5) and the float64 oracle (north-star bar, 1e-4)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from synth import make_config

from gpu_util import make_solver, oracle_state, rel, requires_cuda, tol_for

pytestmark = [pytest.mark.gpu, requires_cuda]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,world,sweeps", [("C2s", 2, 1), ("C4s", 2, 2), ("C3s", 3, 1)])
def test_multiprocess_sharded_sweep(tmp_path, name, world, sweeps):
    from paper_2511_16358_b200.dist import gather_factors, gather_tensor
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(world))
    procs = []
    for r in range(world):
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_rank_worker.py"),
                                       name, str(sweeps), str(tmp_path)],
                                      env=dict(env, RANK=str(r)), stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [pr.communicate(timeout=540)[0] for pr in procs]
    for pr, o in zip(procs, outs):
        assert pr.returncode == 0, o[-3000:]
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert len({int(x["pid"]) for x in res}) == world          # really separate processes
    p = make_config(name)
    sm = int(res[0]["sm"])
    bounds = [(int(x["b"]), int(x["e"])) for x in res]
    X = gather_tensor([x["X"] for x in res], p.dims, sm)
    G = gather_factors([x["G"] for x in res], p.dims, p.ranks, sm, bounds)
    # every rank reports the same global objective trace (all-reduced norms)
    for x in res[1:]:
        assert np.array_equal(x["objective"], res[0]["objective"])
    ref = make_solver(p)
    ref.sweep(sweeps)
    assert rel(X, ref.reconstruct().cpu().numpy()) <= tol_for(p, 1e-5, 1e-12)
    assert rel(G, ref.factors().cpu().numpy()) <= tol_for(p, 1e-5, 1e-12)
    sh, Go, Xo = oracle_state(p)
    F = O.objective(sh, Go, Xo)
    for _ in range(sweeps):
        st, F, _ = O.sweep(sh, Go, Xo, p.mask, p.rho, F, True)
        assert st == 0
    assert rel(X, Xo) <= tol_for(p)
    assert rel(G, Go) <= tol_for(p)
    obs = p.mask.astype(bool)
    assert np.array_equal(X[obs].view(np.uint8), p.observed[obs].view(np.uint8))
