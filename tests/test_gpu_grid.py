"""Multi-instance driver (ifctn_grid_run) on the GPU (-m gpu).

Every instance of a concurrent grid run is bit-identical to a lone run of the same instance
(same kernels, deterministic reductions), for any concurrency; one instance matches the
float64 oracle's final RSE (reading R22); per-instance failures are reported per instance.
"""
import numpy as np
import pytest

from oracle import oracle as O
from synth import MSI_GRID, TRAFFIC_GRID, grid_rank_matrix, init_factors, make_config

from gpu_util import dev, rel, requires_cuda, torch

pytestmark = [pytest.mark.gpu, requires_cuda]


def _grid(p, pairs):
    out = []
    for (r12, r3) in pairs:
        R = grid_rank_matrix(r12, r3)
        g, _ = init_factors(p.dims, R, p.observed, p.mask, p.dtype, "uniform", 0)
        out.append(dict(ranks=R, rho=p.rho, init=g))
    return out


def _lone(p, d, sweeps):
    from paper_2511_16358_b200 import Solver
    s = Solver(p.dims, d["ranks"], dev(p.observed), dev(p.mask), dev(d["init"]), rho=d["rho"])
    s.sweep(sweeps)
    s.sync()
    return s.objective(), s.rse(dev(p.truth))


@pytest.mark.parametrize("concurrency", [1, 3, 8])
def test_grid_equals_lone_runs(concurrency):
    from paper_2511_16358_b200.grid import rank_grid
    p = make_config("C2s")
    inst = _grid(p, MSI_GRID[::3])            # 6 instances, R_{1,2} from 3 to 36
    res = rank_grid(p.dims, dev(p.observed), dev(p.mask), inst, 4, truth=dev(p.truth),
                    concurrency=concurrency)
    assert [r["status"] for r in res] == [0] * len(inst)
    for d, r in zip(inst, res):
        f, e = _lone(p, d, 4)
        assert r["objective"] == f and r["rse"] == e
        assert r["seconds"] > 0


def test_grid_host_inputs_and_oracle_rse():
    from paper_2511_16358_b200.grid import rank_grid
    p = make_config("C2s")
    inst = _grid(p, [(36, 9), (6, 3)])
    res = rank_grid(p.dims, p.observed, p.mask, inst, 10, truth=p.truth, concurrency=2)
    for d, r in zip(inst, res):
        sh = O.Shape(p.dims, d["ranks"])
        G = d["init"].astype(np.float64)
        X = O.init_x(p.observed, p.mask)
        for _ in range(10):
            O.sweep(sh, G, X, p.mask, d["rho"], 0.0, False)
        e = O.rse(p.truth.astype(np.float64), X)
        assert abs(r["rse"] - e) <= 1e-3 * e + 1e-5   # reading R22


def test_grid_reports_bad_instance():
    from paper_2511_16358_b200._abi import IfctnError
    from paper_2511_16358_b200.grid import rank_grid
    p = make_config("C2s")
    inst = _grid(p, [(6, 3)])
    bad = dict(inst[0])
    bad["ranks"] = np.array([[0, 65, 3], [65, 0, 3], [3, 3, 0]], np.int32)   # above IFCTN_MAX_RANK
    with pytest.raises(IfctnError):
        rank_grid(p.dims, dev(p.observed), dev(p.mask), [inst[0], bad], 2, concurrency=2)


@pytest.mark.parametrize("pair", [(2, 3), (9, 6), (36, 12)])
def test_traffic_grid_instances_vs_oracle_rse(pair):
    """The paper's traffic rank grid on the Guangzhou-shaped C4 recipe (C4g,
    214×61×144, fibre mask 70%): spot-check instances — smallest, middle, largest R_{1,2} —
    of a grid run against the float64 oracle's RSE after 10 sweeps (reading R22)."""
    import os
    from paper_2511_16358_b200.grid import rank_grid
    O.set_threads(max(1, min(16, os.cpu_count() or 1)))
    p = make_config("C4g")
    assert len(TRAFFIC_GRID) == 28 and pair in TRAFFIC_GRID
    inst = _grid(p, [pair, (4, 9)])
    res = rank_grid(p.dims, dev(p.observed), dev(p.mask), inst, 10, truth=dev(p.truth), concurrency=2)
    assert all(r["status"] == 0 for r in res)
    d = inst[0]
    sh = O.Shape(p.dims, d["ranks"])
    G = np.asarray(d["init"], np.float64).copy()
    X = O.init_x(p.observed, p.mask)
    r, _ = O.solve(sh, G, X, p.mask, p.rho, 10, 0.0, False)
    assert r == 10
    ro = O.rse(p.truth.astype(np.float64), X)
    assert abs(res[0]["rse"] - ro) <= 1e-3 * ro + 1e-5, (res[0]["rse"], ro)
