"""Evaluation metrics on the GPU (ifctn_metrics) against the float64 numpy
definitions of oracle/metrics.py, on the same X (-m gpu)."""
import numpy as np
import pytest

from oracle import metrics as M
from synth import make_config, make_problem

from gpu_util import dev, make_solver, requires_cuda, torch

pytestmark = [pytest.mark.gpu, requires_cuda]


def _check(p, s, tol=1e-10):
    X = s.reconstruct().cpu().numpy()
    g = s.metrics(dev(p.truth))
    assert g["rse"] == pytest.approx(M.rse(p.truth, X), rel=tol)
    r = M.rmse_missing(p.truth, X, p.mask)
    if np.isnan(r):
        assert np.isnan(g["rmse"])
    else:
        assert g["rmse"] == pytest.approx(r, rel=tol)
    ps = M.psnr_bands(p.truth, X, p.dims)
    assert g["psnr"] == (pytest.approx(ps, rel=tol) if np.isfinite(ps) else ps)
    if p.N == 3:
        assert g["ssim"] == pytest.approx(M.ssim_bands(p.truth, X, p.dims), rel=tol, abs=1e-12)
    else:
        assert np.isnan(g["ssim"])
    assert g["missing"] == int(p.n - p.mask.sum())
    return g


@pytest.mark.parametrize("name,sweeps", [("C2s", 5), ("C2rs", 3), ("C3s", 3), ("C4s", 3)])
def test_metrics_match_definitions(name, sweeps):
    p = make_config(name)
    s = make_solver(p)
    s.sweep(sweeps)
    _check(p, s)


def test_metrics_small_images_whole_window():
    p = make_problem("small_img", (8, 9, 3), 2, "float32", "normal", sr=0.4, init_kind="normal", seed=5)
    s = make_solver(p)
    s.sweep(2)
    _check(p, s)


def test_metrics_exact_and_host_truth():
    p = make_problem("full", (12, 14, 3), 2, "float32", "normal", sr=1.0, init_kind="normal")
    s = make_solver(p)
    s.sweep(1)
    g = _check(p, s)
    assert g["rse"] == 0.0 and g["psnr"] == float("inf") and np.isnan(g["rmse"]) and g["ssim"] == 1.0
    q = make_config("C2s")
    s = make_solver(q)
    s.sweep(2)
    a = s.metrics(dev(q.truth))
    b = s.metrics(np.ascontiguousarray(q.truth))                       # pageable host
    c = s.metrics(torch.from_numpy(np.ascontiguousarray(q.truth)).pin_memory())   # pinned host
    assert a == b == c
