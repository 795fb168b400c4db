"""Host logic of the sharded (multi-GPU) sweep on CPU (-m "not gpu").

* shard/gather round trips of tensors and factor chains (paper_2511_16358_b200.dist);
* a world_size-2 torch.distributed **gloo** run of the sharded PAM sweep decomposition the
  library implements: each rank contracts its shard (float64 oracle), projects
  its partial (β, ω) onto the Gram/RHS of Eq. 8, blocks with k ≠ s all-reduce the projections,
  every rank solves redundantly, the X update is local and the norms are all-reduced — and the
  gathered result equals the unsharded oracle sweep.
"""
import os

import numpy as np
import pytest

from synth import make_config


@pytest.fixture(scope="module")
def dist_mod():
    from paper_2511_16358_b200 import build
    build.build()
    from paper_2511_16358_b200 import dist
    return dist


@pytest.mark.parametrize("dims,mode,world", [((5, 4, 3), 0, 2), ((5, 4, 3), 2, 3), ((3, 7, 2, 4), 1, 4),
                                             ((6, 2, 3, 2, 5), 4, 2)])
def test_shard_gather_roundtrip(dist_mod, dims, mode, world):
    rng = np.random.default_rng(0)
    N = len(dims)
    ranks = np.full((N, N), 2)
    np.fill_diagonal(ranks, 0)
    n = int(np.prod(dims))
    x = rng.standard_normal(n)
    G = rng.standard_normal(sum(2 * dims[k] for k in range(N) for i in range(N) if i != k))
    shards, fs, bounds = [], [], []
    for r in range(world):
        sm, b, e = dist_mod.shard_range(dims, world, r, mode)
        assert sm == mode
        bounds.append((b, e))
        shards.append(dist_mod.shard_tensor(x, dims, mode, b, e))
        fs.append(dist_mod.shard_factors(G, dims, ranks, mode, b, e))
    assert bounds[0][0] == 0 and bounds[-1][1] == dims[mode]
    assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
    assert np.array_equal(dist_mod.gather_tensor(shards, dims, mode), x)
    assert np.array_equal(dist_mod.gather_factors(fs, dims, ranks, mode, bounds), G)


def _layout(dims, ranks):
    N = len(dims)
    out, off = {}, 0
    for k in range(N):
        for i in range(N):
            if i != k:
                R = int(ranks[k][i])
                out[(k, i)] = (off, R, int(dims[k]))
                off += R * int(dims[k])
    return out


def _sharded_sweep(rank, world, name, mode, q):
    """One process of the gloo run (spawned)."""
    import torch
    import torch.distributed as tdist

    from oracle import oracle as O
    from paper_2511_16358_b200 import dist as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    tdist.init_process_group("gloo", rank=rank, world_size=world,
                             init_method=f"tcp://127.0.0.1:{q['port']}")
    try:
        p = make_config(name)
        sm, b, e = D.shard_range(p.dims, world, rank, mode)
        ld = list(p.dims)
        ld[sm] = e - b
        sh = O.Shape(ld, p.ranks)
        G = D.shard_factors(p.G0, p.dims, p.ranks, sm, b, e).astype(np.float64)
        X = O.init_x(D.shard_tensor(p.observed, p.dims, sm, b, e), D.shard_tensor(p.mask, p.dims, sm, b, e))
        mask = D.shard_tensor(p.mask, p.dims, sm, b, e)
        lay = _layout(ld, p.ranks)

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            tdist.all_reduce(t)
            return t.numpy()

        dg2_shard = dg2_rep = 0.0
        N = p.N
        for k in range(N):
            for i in range(N):
                if i == k:
                    continue
                beta, omega = O.block_contract(sh, G, X, k, i)      # this rank's partial sums
                off_i, R, Ii = lay[(i, k)]
                gik = G[off_i:off_i + R * Ii].reshape(Ii, R)         # rows = local a
                gram = np.einsum("aj,ar,as->jrs", omega, gik, gik)   # Σ_a ω g gᵀ (local a)
                rhs = np.einsum("aj,ar->jr", beta, gik)
                if k != sm:                                          # exchange (§8(e))
                    gram = allreduce(gram)
                    rhs = allreduce(rhs)
                off_k, _, Ik = lay[(k, i)]
                cold = G[off_k:off_k + R * Ik].reshape(Ik, R).copy()
                cnew = np.stack([np.linalg.solve(gram[j] + p.rho * np.eye(R), rhs[j] + p.rho * cold[j])
                                 for j in range(Ik)])
                d = float(np.sum((cnew - cold) ** 2))
                if k == sm:
                    dg2_shard += d
                else:
                    dg2_rep += d
                G[off_k:off_k + R * Ik] = cnew.reshape(-1)
        dx2, x2, f = O.refill(sh, G, X, mask, p.rho)
        s4 = allreduce(np.array([dx2, x2, f, dg2_shard]))
        q["res"][rank] = (X.copy(), G.copy(), (b, e), sm, s4, dg2_rep)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("name,mode", [("C3s", -1), ("C4s", 0), ("C2s", 2)])
def test_gloo_world2_sharded_sweep_equals_oracle(dist_mod, name, mode):
    import socket

    import torch.multiprocessing as mp

    from oracle import oracle as O

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    q = mgr.dict()
    q["port"] = port
    q["res"] = mgr.dict()
    mp.spawn(_sharded_sweep, args=(2, name, mode, q), nprocs=2, join=True)
    res = [q["res"][r] for r in range(2)]
    p = make_config(name)
    sm = res[0][3]
    X = dist_mod.gather_tensor([r[0] for r in res], p.dims, sm)
    G = dist_mod.gather_factors([r[1] for r in res], p.dims, p.ranks, sm, [r[2] for r in res])
    sh = O.Shape(p.dims, p.ranks)
    Go = p.G0.astype(np.float64)
    Xo = O.init_x(p.observed, p.mask)
    F0 = O.objective(sh, Go, Xo)
    st, F1, row = O.sweep(sh, Go, Xo, p.mask, p.rho, F0, False)
    np.testing.assert_allclose(G, Go, rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(X, Xo, rtol=1e-9, atol=1e-10)
    s4, dg2_rep = res[0][4], res[0][5]
    assert np.allclose(s4, res[1][4]) and dg2_rep == res[1][5]   # replicated state identical
    assert abs(s4[2] - F1) <= 1e-9 * max(1, F1)                   # all-reduced objective (½ applied per rank)
    assert abs((s4[3] + dg2_rep) - row[3]) <= 1e-9 * max(1, row[3])  # ΔG² accounting


def _peer_allgather(rank, world, q):
    """One process: the IPC-handle all-gather of the peer exchange (make_dist(peer=True)),
    called through the C function pointer the library calls inside ifctn_create."""
    import ctypes

    import torch.distributed as tdist

    from paper_2511_16358_b200 import dist as D

    tdist.init_process_group("gloo", rank=rank, world_size=world,
                             init_method=f"tcp://127.0.0.1:{q['port']}")
    try:
        d = D.make_dist(rank, world, -1, peer=True, allgather=D.torch_allgather())
        assert d.exchange == 1 and bool(d.host_allgather)
        mine = bytes([rank * 16 + b % 16 for b in range(64)])
        src = ctypes.create_string_buffer(mine, 64)
        out = ctypes.create_string_buffer(64 * world)
        d.host_allgather(ctypes.cast(src, ctypes.c_void_p), ctypes.cast(out, ctypes.c_void_p), 64, None)
        q["res"][rank] = out.raw
    finally:
        tdist.destroy_process_group()


def test_gloo_world2_peer_handle_allgather(dist_mod):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    q = mgr.dict()
    q["port"] = port
    q["res"] = mgr.dict()
    mp.spawn(_peer_allgather, args=(2, q), nprocs=2, join=True)
    want = b"".join(bytes([r * 16 + b % 16 for b in range(64)]) for r in range(2))
    assert q["res"][0] == want and q["res"][1] == want
