"""The L2-resident contraction (csrc/l2pass.cuh, default when X ≤ 48 MB) against the
HBM-streaming fibre walk (IFCTN_FLAG_NO_L2PASS) and the float64 oracle: β/ω of every block,
one full sweep, and the split-across-CTAs (Z > 1) partial sums."""
import numpy as np
import pytest

from oracle import oracle as O
from synth import make_config

from gpu_util import make_solver, oracle_state, rel, requires_cuda, tol_for

pytestmark = [pytest.mark.gpu, requires_cuda]

# the L2 pass serves third-order tensors (csrc/ifctn.cu make_l2); the others check the switch
SMALL = ["C1", "C2s", "C3s", "C4s", "C5s", "C2rs"]


@pytest.mark.parametrize("name", SMALL + ["C2", "C2r"])
def test_l2pass_block_coefficients_match_fibre_walk_and_oracle(name):
    from paper_2511_16358_b200 import IFCTN_FLAG_NO_L2PASS
    p = make_config(name)
    a = make_solver(p)
    b = make_solver(p, flags=IFCTN_FLAG_NO_L2PASS)
    sh, G, X = oracle_state(p)
    small = p.n <= 200_000
    t = tol_for(p, 1e-5, 1e-11)
    for k in range(p.N):
        for i in range(p.N):
            if i == k:
                continue
            ba, wa = a.block_coefficients(k, i)
            bb, wb = b.block_coefficients(k, i)
            assert rel(ba, bb) <= t and rel(wa, wb) <= t, (k, i, rel(ba, bb), rel(wa, wb))
            if small:
                bo, wo = O.block_contract(sh, G, X, k, i)
                assert rel(ba, bo) <= t and rel(wa, wo) <= t, (k, i)
                # per element: |Δ| within the fp32 accumulation bound of the largest entries
                sc = np.abs(wo).max()
                assert np.max(np.abs(wa - wo)) <= 1e-5 * sc + 1e-300, (k, i)


@pytest.mark.parametrize("name", ["C2s", "C2rs", "C1"])
def test_l2pass_one_sweep_matches_oracle(name):
    p = make_config(name)
    s = make_solver(p)
    sh, G, X = oracle_state(p)
    st, _, _ = O.sweep(sh, G, X, p.mask, p.rho, O.objective(sh, G, X), True)
    assert st == 0
    s.sweep(1, trace=True)
    assert rel(s.factors().cpu().numpy(), G) <= tol_for(p)
    assert rel(s.reconstruct().cpu().numpy(), X) <= tol_for(p)


def test_l2pass_split_partials_are_deterministic():
    """Blocks with few kept values split each v over Z CTAs (last-arriving CTA sums in z
    order): repeated calls are bit-identical."""
    p = make_config("C2")
    s = make_solver(p)
    for (k, i) in ((0, 2), (2, 0), (2, 1)):
        b1, w1 = s.block_coefficients(k, i)
        b2, w2 = s.block_coefficients(k, i)
        assert np.array_equal(b1, b2) and np.array_equal(w1, w2)
