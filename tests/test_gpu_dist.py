"""Sharded (multi-GPU) sweep on ONE device (-m gpu): W ranks are W contexts driven from W host
threads, each owning its shard along the shard mode; the per-block Gram/RHS partial sums go
through the library's host_allreduce hook (a barrier exchange between the threads) instead of
NCCL.  No kernel waits on another rank's kernel — the waiting happens on the host — so this is
safe on one GPU (B200_PROFILING.md).  The sharded run must reproduce the single-GPU run."""
import threading

import numpy as np
import pytest

from synth import make_config

from gpu_util import dev, make_solver, oracle_state, rel, requires_cuda, tol_for, torch

pytestmark = [pytest.mark.gpu, requires_cuda]


def run_sharded(p, world, sweeps, trace=False, shard_mode=-1):
    from paper_2511_16358_b200 import Solver
    from paper_2511_16358_b200.dist import make_dist, shard_factors, shard_range, shard_tensor

    slots = [None] * world
    barrier = threading.Barrier(world)

    def make_cb(r):
        def cb(arr):
            slots[r] = arr.copy()
            barrier.wait()
            total = slots[0].copy()
            for q in range(1, world):       # fixed order: identical on every rank
                total += slots[q]
            barrier.wait()
            arr[:] = total
        return cb

    solvers, bounds = [], []
    sm = None
    for r in range(world):
        sm, b, e = shard_range(p.dims, world, r, shard_mode)
        bounds.append((b, e))
        obs = shard_tensor(p.observed, p.dims, sm, b, e)
        msk = shard_tensor(p.mask, p.dims, sm, b, e)
        g0 = shard_factors(p.G0, p.dims, p.ranks, sm, b, e)
        d = make_dist(r, world, shard_mode, host_allreduce=make_cb(r))
        st = torch.cuda.Stream()
        solvers.append(Solver(p.dims, p.ranks, dev(obs), dev(msk), dev(g0), rho=p.rho, dist=d,
                              stream=st.cuda_stream))
        solvers[-1]._dist_keep = d
    out = [None] * world
    errs = []

    def work(r):
        try:
            out[r] = solvers[r].sweep(sweeps, trace=trace)
        except Exception as ex:  # surfaced below
            errs.append(ex)
            barrier.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    return solvers, sm, bounds, out


# C5s is ill-conditioned in fp32 (summation-order differences grow ~25x per sweep, see
# test_gpu_parity.py): one sweep there, two elsewhere.
@pytest.mark.parametrize("name,world,sweeps", [("C2s", 2, 2), ("C3s", 2, 2), ("C4s", 3, 2), ("C5s", 2, 1),
                                               ("C1", 4, 2)])
def test_sharded_sweeps_match_single_gpu(name, world, sweeps):
    from paper_2511_16358_b200.dist import gather_factors, gather_tensor
    p = make_config(name)
    ref = make_solver(p)
    ref.sweep(sweeps, trace=True)
    solvers, sm, bounds, out = run_sharded(p, world, sweeps, trace=True)
    X = gather_tensor([s.reconstruct().cpu().numpy() for s in solvers], p.dims, sm)
    G = gather_factors([s.factors().cpu().numpy() for s in solvers], p.dims, p.ranks, sm, bounds)
    tol = tol_for(p, 1e-5, 1e-12)
    assert rel(X, ref.reconstruct().cpu().numpy()) <= tol
    assert rel(G, ref.factors().cpu().numpy()) <= tol
    # the trace (all-reduced norms) is identical on every rank and matches the single GPU run
    _, rows_ref = ref.sweep(1, trace=True)
    obs = p.mask.astype(bool)
    assert np.array_equal(X[obs].view(np.uint8), p.observed[obs].view(np.uint8))
    for r in range(1, world):
        assert out[r][1] == out[0][1]


@pytest.mark.parametrize("name,world,mode", [("C3s", 2, 0), ("C4s", 2, 3), ("C2s", 3, 2), ("C2rs", 2, 2)])
def test_sharded_one_sweep_vs_oracle(name, world, mode):
    """Sharding along a chosen mode (including mode 1 = the fibre mode): one sweep, north-star
    bar against the float64 oracle."""
    from oracle import oracle as O
    from paper_2511_16358_b200.dist import gather_factors, gather_tensor
    p = make_config(name)
    solvers, sm, bounds, _ = run_sharded(p, world, 1, trace=True, shard_mode=mode)
    assert sm == mode
    X = gather_tensor([s.reconstruct().cpu().numpy() for s in solvers], p.dims, sm)
    G = gather_factors([s.factors().cpu().numpy() for s in solvers], p.dims, p.ranks, sm, bounds)
    sh, Go, Xo = oracle_state(p)
    st, _, _ = O.sweep(sh, Go, Xo, p.mask, p.rho, O.objective(sh, Go, Xo), True)
    assert st == 0
    assert rel(G, Go) <= tol_for(p) and rel(X, Xo) <= tol_for(p)


def test_sharded_fused_sequence_and_rse():
    """Fixed sweep count (fused sequence) sharded, and the all-reduced RSE."""
    from paper_2511_16358_b200.dist import gather_tensor, shard_range, shard_tensor
    p = make_config("C3s")
    ref = make_solver(p)
    ref.sweep(3)
    solvers, sm, bounds, _ = run_sharded(p, 2, 3)
    X = gather_tensor([s.reconstruct().cpu().numpy() for s in solvers], p.dims, sm)
    assert rel(X, ref.reconstruct().cpu().numpy()) <= 1e-5
    # RSE: every rank returns the global value
    vals = [None, None]

    def rse(r):
        b, e = bounds[r]
        vals[r] = solvers[r].rse(dev(shard_tensor(p.truth, p.dims, sm, b, e)))

    th = [threading.Thread(target=rse, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    r_ref = ref.rse(dev(p.truth))
    assert abs(vals[0] - r_ref) <= 1e-6 and vals[0] == vals[1]


@pytest.mark.parametrize("name,mode", [("C3s", 1), ("C5s", 0), ("C2", 2)])
def test_nccl_single_rank_path_matches_single_gpu(name, mode):
    """The NCCL code path on one GPU: a 1-rank communicator built from torch's ncclUniqueId
    runs every projection / all-reduce / split finaliser (captured in the sweep graphs) and
    must reproduce the single-GPU result bit for bit (1-rank all-reduce = copy)."""
    import torch.cuda.nccl as tnccl

    from paper_2511_16358_b200.dist import make_dist
    p = make_config(name)
    a = make_solver(p)
    d = make_dist(0, 1, mode, nccl_id=tnccl.unique_id())
    b = make_solver(p, dist=d)
    for s in (a, b):
        s.sweep(3)
        s.sweep(2, trace=True)
    assert np.array_equal(a.reconstruct().cpu().numpy(), b.reconstruct().cpu().numpy())
    assert np.array_equal(a.factors().cpu().numpy(), b.factors().cpu().numpy())
    assert b.launch_count() > a.launch_count()  # the extra projection / combine launches ran


@pytest.mark.parametrize("mode", [2, 0])
def test_sharded_metrics_match_single_gpu(mode):
    """Metrics of a sharded context (virtual ranks) equal the single-GPU values; SSIM needs
    whole band images, so it is NaN when the shard mode is an image mode."""
    import threading as _th
    p = make_config("C2s")
    ref = make_solver(p)
    ref.sweep(2)
    want = ref.metrics(dev(p.truth))
    world = 2
    solvers, sm, bounds, _ = run_sharded(p, world, 2, shard_mode=mode)
    from paper_2511_16358_b200.dist import shard_tensor
    got = [None] * world

    def work(r):
        b, e = bounds[r]
        got[r] = solvers[r].metrics(dev(shard_tensor(p.truth, p.dims, sm, b, e)))

    th = [_th.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    # same sweeps up to summation order: a shard regroups the fp32 partial sums of the passes
    # (the L2 pass sums a run of cells along the longest reduced mode per thread; shard mode 0
    # is also stored mode-swapped, Shape::perm) — the sharded-vs-single bar of DESIGN §8, 1e-5
    rt = 1e-5
    for g in got:
        for key in ("rse", "rmse", "psnr"):
            assert g[key] == pytest.approx(want[key], rel=rt)
        assert g["missing"] == want["missing"]
        if mode == 2:
            assert g["ssim"] == pytest.approx(want["ssim"], rel=rt)  # a function of the same X
        else:
            assert np.isnan(g["ssim"])


def test_c5_world8_shard_along_mode1_matches_single_gpu():
    """BASELINE.json's C5 configuration: 64⁴×32 sharded along mode 1 (API mode 0, the default
    rule: largest mode, first on ties) across 8 ranks — 8 slices of the fibre mode per rank, so
    each rank stores its shard with mode 0 swapped for mode 2 (Shape::perm).  One sweep, 8
    virtual ranks on one device: factors and X match the single-GPU run to 1e-5."""
    from paper_2511_16358_b200.dist import gather_factors, gather_tensor
    p = make_config("C5")
    ref = make_solver(p)
    ref.sweep(1, trace=True)
    Xr, Gr = ref.reconstruct().cpu().numpy(), ref.factors().cpu().numpy()
    ref.close()
    solvers, sm, bounds, out = run_sharded(p, 8, 1, trace=True)
    assert sm == 0 and bounds[0] == (0, 8)
    X = gather_tensor([s.reconstruct().cpu().numpy() for s in solvers], p.dims, sm)
    G = gather_factors([s.factors().cpu().numpy() for s in solvers], p.dims, p.ranks, sm, bounds)
    for s in solvers:
        s.close()
    assert rel(X, Xr) <= 1e-5 and rel(G, Gr) <= 1e-5, (rel(X, Xr), rel(G, Gr))
    obs = p.mask.astype(bool)
    assert np.array_equal(X[obs].view(np.uint8), p.observed[obs].view(np.uint8))
    for r in range(1, 8):
        assert out[r][1] == out[0][1]


@pytest.mark.parametrize("name,dims", [("C3s", None), ("C1", (12, 20, 16)), ("C5s", (4, 8, 6, 5, 4))])
def test_nccl_single_rank_mode_permuted_layout(name, dims):
    """1-rank NCCL communicator with shard mode 0 shorter than the middle modes: the context
    stores the tensor in the internal mode order of Shape::perm — (1,0,2,3), (1,0,2) and the
    3-cycle (1,2,0,3,4), whose first block (API (0,1) = internal (2,0)) runs the fused refill
    pass through H_{0,2}.  Results match the single-GPU run to summation order, factors and X
    come back in the API layout, the step-level entry points take API block indices and the
    metrics are unchanged."""
    import torch.cuda.nccl as tnccl

    from paper_2511_16358_b200.dist import make_dist
    mode = 0
    p = make_config(name) if dims is None else make_config(name, dims=dims)
    a = make_solver(p)
    d = make_dist(0, 1, mode, nccl_id=tnccl.unique_id())
    b = make_solver(p, dist=d)
    assert rel(b.reconstruct().cpu().numpy(), a.reconstruct().cpu().numpy()) == 0.0
    assert np.array_equal(b.factors().cpu().numpy(), a.factors().cpu().numpy())
    for k, i in ((0, 1), (2, 0), (1, 2)):
        ba, wa = a.block_coefficients(k, i)
        bb, wb = b.block_coefficients(k, i)
        assert rel(bb, ba) <= tol_for(p, 1e-6, 1e-13) and rel(wb, wa) <= tol_for(p, 1e-6, 1e-13)
    # C5s is ill-conditioned in fp32 (summation-order differences grow ~25x per sweep): two
    # sweeps (first + fused + last graphs) and the north-star bar there
    for s in (a, b):
        if name == "C5s":
            s.sweep(2)
        else:
            s.sweep(3)
            s.sweep(2, trace=True)
    tol = tol_for(p, 1e-4 if name == "C5s" else 1e-5, 1e-11)
    assert rel(b.reconstruct().cpu().numpy(), a.reconstruct().cpu().numpy()) <= tol
    assert rel(b.factors().cpu().numpy(), a.factors().cpu().numpy()) <= tol
    from paper_2511_16358_b200 import IFCTN_MODEL
    assert rel(b.reconstruct(IFCTN_MODEL).cpu().numpy(), a.reconstruct(IFCTN_MODEL).cpu().numpy()) <= tol
    ma, mb = a.metrics(dev(p.truth)), b.metrics(dev(p.truth))
    for key in ("rse", "rmse", "psnr"):
        assert mb[key] == pytest.approx(ma[key], rel=1e-4)
    assert b.rse(p.truth) == pytest.approx(a.rse(dev(p.truth)), rel=1e-4)
