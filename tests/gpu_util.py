"""Helpers shared by the GPU parity tests (marshalling only; no method arithmetic)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

requires_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def make_solver(p, **kw):
    from paper_2511_16358_b200 import Solver
    return Solver(p.dims, p.ranks, dev(p.observed), dev(p.mask), dev(p.G0), rho=p.rho, **kw)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def oracle_state(p):
    sh = O.Shape(p.dims, p.ranks)
    return sh, p.G0.astype(np.float64), O.init_x(p.observed, p.mask)


def tol_for(p, f32=1e-4, f64=1e-10):
    return f64 if p.dtype == np.float64 else f32
