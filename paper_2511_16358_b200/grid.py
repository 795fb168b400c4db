"""Multi-instance (rank-grid) driver — SURVEY §8(f2); marshalling over `ifctn_grid_run`.

The paper tunes the iFCTN ranks over a grid and reports the total time including tuning
(P:L485-489).  `rank_grid` solves a list of instances that share (O, Ω) on one GPU, several
at a time on independent streams (csrc/grid.cu).  Across GPUs the instance list is dealt
round-robin to the ranks (`shard_instances`) — independent problems, no data-path collective —
and the per-instance results are gathered to every rank (`gather_results`, torch.distributed).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._abi import IFCTN_F32, IFCTN_F64


def _ptr(x):
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(x.ctypes.data)


def rank_grid(dims, observed, mask, instances, t_max, truth=None, concurrency=8, dtype=None):
    """Solve every instance (dict with `ranks` (N×N), `rho`, `init` (flat G⁰)) for t_max
    sweeps; returns one dict per instance: rse, objective, seconds (device), status."""
    import torch
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    if dtype is None:
        dt = observed.dtype
        is64 = (dt == np.float64) if isinstance(dt, np.dtype) else (dt == torch.float64)
        dtype = IFCTN_F64 if is64 else IFCTN_F32
    from . import check_buffer, factor_layout
    if isinstance(mask, np.ndarray) and mask.dtype == np.bool_:
        mask = mask.view(np.uint8)
    kind = "f64" if dtype == IFCTN_F64 else "f32"
    n = int(np.prod(dims))
    check_buffer(observed, "observed", kind, n)
    check_buffer(mask, "mask", "u8", n)
    if truth is not None:
        check_buffer(truth, "truth", kind, n)
    keep = []
    inst = []
    for q, d in enumerate(instances):
        R = np.asarray(d["ranks"], dtype=np.int32).reshape(N, N)
        g = d["init"]
        lay = factor_layout(dims, R)
        check_buffer(g, f"instances[{q}].init", kind, lay[-1][2] + lay[-1][3] * lay[-1][4])
        keep.append(g)
        inst.append(([int(v) for v in R.reshape(-1)], float(d.get("rho", 0.1)), _ptr(g)))
    return _abi.ifctn_grid_run(N, dims, dtype, _ptr(observed), _ptr(mask), _ptr(truth), inst,
                               int(t_max), int(concurrency))


def shard_instances(count: int, rank: int, world: int) -> list:
    """Instance indices of one rank: round-robin, so a cost-sorted list stays balanced."""
    return list(range(rank, count, world))


def gather_results(local: list, indices: list, count: int) -> list:
    """All ranks' (index, result) pairs → the full result list (torch.distributed)."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(zip(indices, local)))
    out = [None] * count
    for part in parts:
        for q, r in part:
            out[q] = r
    return out
