"""Host logic of the multi-instance driver on CPU (-m "not gpu").

The instance list is dealt round-robin to the ranks and the results gathered with
torch.distributed: a world_size-2 gloo run in which every rank solves its share of a small
rank grid with the float64 oracle reproduces the serial oracle run of the whole grid.
"""
import os

import numpy as np
import pytest

from synth import MSI_GRID, grid_rank_matrix, init_factors, make_config


def _grid(n_inst=5):
    p = make_config("C2s")
    out = []
    for (r12, r3) in MSI_GRID[:n_inst]:
        R = grid_rank_matrix(r12, r3)
        g, _ = init_factors(p.dims, R, p.observed, p.mask, p.dtype, "uniform", 0)
        out.append(dict(ranks=R, rho=p.rho, init=g))
    return p, out


def _oracle_instance(p, d, sweeps):
    from oracle import oracle as O
    sh = O.Shape(p.dims, d["ranks"])
    G = d["init"].astype(np.float64)
    X = O.init_x(p.observed, p.mask)
    for _ in range(sweeps):
        O.sweep(sh, G, X, p.mask, d["rho"], 0.0, False)
    return dict(rse=O.rse(p.truth.astype(np.float64), X), objective=O.objective(sh, G, X))


def test_round_robin_partition_covers_once():
    from paper_2511_16358_b200.grid import shard_instances
    for count in (0, 1, 5, 18):
        for world in (1, 2, 3, 8):
            parts = [shard_instances(count, r, world) for r in range(world)]
            flat = sorted(q for part in parts for q in part)
            assert flat == list(range(count))
            assert max(len(x) for x in parts) - min(len(x) for x in parts) <= 1


def _worker(rank, world, q):
    import torch.distributed as tdist

    from paper_2511_16358_b200.grid import gather_results, shard_instances

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    tdist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{q['port']}")
    try:
        p, inst = _grid()
        mine = shard_instances(len(inst), rank, world)
        local = [_oracle_instance(p, inst[i], 2) for i in mine]
        full = gather_results(local, mine, len(inst))
        q["res"][rank] = full
    finally:
        tdist.destroy_process_group()


def test_gloo_world2_grid_equals_serial():
    import socket

    import torch.multiprocessing as mp

    from paper_2511_16358_b200 import build
    build.build()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    q = mgr.dict()
    q["port"] = port
    q["res"] = mgr.dict()
    mp.spawn(_worker, args=(2, q), nprocs=2, join=True)
    p, inst = _grid()
    serial = [_oracle_instance(p, d, 2) for d in inst]
    for r in range(2):
        got = q["res"][r]
        assert len(got) == len(inst)
        for a, b in zip(got, serial):
            assert a == b   # same float64 oracle, same inputs: identical
