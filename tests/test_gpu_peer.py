"""Device-side exchange over peer memory (IFCTN_XCHG_PEER, csrc/peer.cuh).

* The protocol (publish epoch, wait for every rank, rank-ordered sum, two slots, epoch
  counter) under real concurrency: W = 2..16 virtual ranks in ONE cooperative launch
  (ranks whose kernels wait on one another must not be separate launches on one GPU,
  B200_PROFILING.md), with the same device functions the solve kernels use.
* The library's peer path at world 1: the FROM_PROJ solves publish / wait / sum themselves,
  the norms and RSE go through peer_allreduce, all inside the sweep graphs — bit-identical to
  the single-GPU path and to the 1-rank NCCL path.
"""
import numpy as np
import pytest

from synth import make_config

from gpu_util import dev, make_solver, rel, requires_cuda, tol_for, torch

pytestmark = [pytest.mark.gpu, requires_cuda]


@pytest.mark.parametrize("world", [2, 3, 4, 8, 16])
def test_peer_protocol_selftest(world):
    from paper_2511_16358_b200 import _abi
    assert _abi.ifctn_peer_selftest(world, 64, 1000) == 0


def test_peer_selftest_rejects_bad_sizes():
    from paper_2511_16358_b200 import IfctnError, _abi
    for w in (1, 17):
        with pytest.raises(IfctnError):
            _abi.ifctn_peer_selftest(w, 1, 10)


@pytest.mark.parametrize("name,mode", [("C3s", 1), ("C2", 2), ("C2rs", 2), ("C5s", 3)])
def test_peer_single_rank_matches_single_gpu(name, mode):
    """World-1 peer exchange: every dist block runs PROJECT then the fused exchange+solve;
    results are bit-identical to the single-GPU path (1-rank sums are copies)."""
    from paper_2511_16358_b200.dist import make_dist
    p = make_config(name)
    a = make_solver(p)
    d = make_dist(0, 1, mode, peer=True)
    b = make_solver(p, dist=d)
    for s in (a, b):
        s.sweep(3)
        _, rows = s.sweep(2, trace=True)
        s.sweep(1, eps=1e-30, trace=True)  # plain per-sweep graph with the stop test
    assert np.array_equal(a.reconstruct().cpu().numpy(), b.reconstruct().cpu().numpy())
    assert np.array_equal(a.factors().cpu().numpy(), b.factors().cpu().numpy())
    assert b.launch_count() > a.launch_count()
    assert b.rse(dev(p.truth)) == a.rse(dev(p.truth))
    ma, mb = a.metrics(dev(p.truth)), b.metrics(dev(p.truth))
    for key in ("rse", "rmse", "psnr"):
        assert mb[key] == pytest.approx(ma[key], rel=1e-12)


def test_peer_and_nccl_single_rank_agree():
    import torch.cuda.nccl as tnccl

    from paper_2511_16358_b200.dist import make_dist
    p = make_config("C4s")
    a = make_solver(p, dist=make_dist(0, 1, 0, nccl_id=tnccl.unique_id()))
    b = make_solver(p, dist=make_dist(0, 1, 0, peer=True))
    for s in (a, b):
        s.sweep(4)
    assert np.array_equal(a.reconstruct().cpu().numpy(), b.reconstruct().cpu().numpy())
    assert np.array_equal(a.factors().cpu().numpy(), b.factors().cpu().numpy())


def test_peer_permuted_layout_single_rank():
    """Peer exchange with a mode-0 shard (internal mode order, Shape::perm) vs single GPU."""
    from paper_2511_16358_b200.dist import make_dist
    p = make_config("C3s")
    a = make_solver(p)
    b = make_solver(p, dist=make_dist(0, 1, 0, peer=True))
    for s in (a, b):
        s.sweep(3)
    assert rel(b.reconstruct().cpu().numpy(), a.reconstruct().cpu().numpy()) <= tol_for(p, 1e-5, 1e-11)
