"""Multi-GPU host logic: sharding of the inputs along the shard mode, the
factor-chain column split, gathering, and the torch.distributed plumbing that hands NCCL's
unique id to the library.  No arithmetic of the method lives here: every sweep step — the
per-rank contraction, the projection onto Gram/RHS partials and the solves — runs in
libifctn.so, which sums the partials with NCCL (or a host callback in tests).

Layouts are the C-ABI's (include/ifctn.h): tensors flat mode-1-fastest; factors concatenated
(k asc, i asc, i≠k), each R_{k,i}×I_k column-major.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi


def shard_range(dims, world: int, rank: int, shard_mode: int = -1):
    """(shard mode, begin, end) of this rank's slice — the library's own rule (reading R21:
    ⌈I_s/W⌉ slices first, then ⌊I_s/W⌋; shard mode = largest, the first on ties)."""
    d = _abi.ifctn_dist(None, rank, world, shard_mode)
    return _abi.ifctn_shard_range(len(dims), dims, d if world > 1 else None)


def _as_nd(x, dims):
    a = np.asarray(x)
    return a.reshape(tuple(int(v) for v in dims), order="F")


def shard_tensor(x, dims, mode: int, begin: int, end: int):
    """Slice [begin, end) of `mode` of a flat mode-1-fastest tensor (numpy), flat again."""
    a = _as_nd(x, dims)
    sl = [slice(None)] * len(dims)
    sl[mode] = slice(begin, end)
    return np.ascontiguousarray(a[tuple(sl)].reshape(-1, order="F"))


def gather_tensor(shards, dims, mode: int):
    """Inverse of shard_tensor over all ranks (shards in rank order)."""
    parts = []
    for sh in shards:
        ld = list(dims)
        ld[mode] = -1
        n_other = int(np.prod([d for m, d in enumerate(dims) if m != mode]))
        ld[mode] = len(sh) // n_other
        parts.append(np.asarray(sh).reshape(ld, order="F"))
    return np.concatenate(parts, axis=mode).reshape(-1, order="F")


def _layout(dims, ranks):
    N = len(dims)
    r = np.asarray(ranks).reshape(N, N)
    out, off = [], 0
    for k in range(N):
        for i in range(N):
            if i != k:
                out.append((k, i, off, int(r[k, i]), int(dims[k])))
                off += int(r[k, i]) * int(dims[k])
    return out


def shard_factors(G, dims, ranks, mode: int, begin: int, end: int):
    """The factor array of one rank: chains G_{mode,·} keep columns [begin, end)."""
    G = np.asarray(G)
    parts = []
    for (k, i, off, R, Ik) in _layout(dims, ranks):
        blk = G[off:off + R * Ik].reshape(Ik, R)   # row = column of G_{k,i}
        if k == mode:
            blk = blk[begin:end]
        parts.append(blk.reshape(-1))
    return np.ascontiguousarray(np.concatenate(parts))


def gather_factors(shards, dims, ranks, mode: int, bounds):
    """Inverse of shard_factors: replicated chains from rank 0, shard chains concatenated."""
    out = []
    ld = [list(dims) for _ in shards]
    for r, (b, e) in enumerate(bounds):
        ld[r][mode] = e - b
    lays = [_layout(ld[r], ranks) for r in range(len(shards))]
    for t, (k, i, off, R, Ik) in enumerate(_layout(dims, ranks)):
        if k == mode:
            cols = []
            for r, sh in enumerate(shards):
                _, _, o, Rr, Ikr = lays[r][t]
                cols.append(np.asarray(sh)[o:o + Rr * Ikr].reshape(Ikr, Rr))
            out.append(np.concatenate(cols, axis=0).reshape(-1))
        else:
            _, _, o, Rr, Ikr = lays[0][t]
            out.append(np.asarray(shards[0])[o:o + Rr * Ikr])
    return np.concatenate(out)


def make_dist(rank: int, world: int, shard_mode: int = -1, nccl_id: bytes | None = None,
              host_allreduce=None, user=None, peer: bool = False, allgather=None):
    """ifctn_dist for rank/world.  Either nccl_id (128 bytes, identical on all ranks), a
    Python host_allreduce(np_view) callback summing a float64 buffer across ranks in place, or
    peer=True: the device-side exchange over peer memory (IFCTN_XCHG_PEER), whose CUDA IPC
    handles are all-gathered once at create by allgather(bytes) -> [bytes per rank] (host
    plumbing, e.g. torch_allgather below; not needed at world 1)."""
    d = _abi.ifctn_dist()
    d.rank, d.world, d.shard_mode = rank, world, shard_mode
    keep = []
    if peer:
        d.exchange = _abi.IFCTN_XCHG_PEER
        if allgather is not None:
            def _ag(mine, out, nbytes, _user):
                got = allgather(ctypes.string_at(mine, nbytes))
                if len(got) != world or any(len(g) != nbytes for g in got):
                    raise RuntimeError("host_allgather: wrong result shape")
                ctypes.memmove(out, b"".join(got), nbytes * world)
            cbg = _abi.HOST_ALLGATHER(_ag)
            keep.append(cbg)
            d.host_allgather = cbg
    if nccl_id is not None:
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        keep.append(buf)
        d.nccl_unique_id = ctypes.cast(buf, ctypes.c_void_p)
    if host_allreduce is not None:
        def _cb(ptr, count, _user):
            arr = np.ctypeslib.as_array(ptr, shape=(count,))
            host_allreduce(arr)
        cb = _abi.HOST_ALLREDUCE(_cb)
        keep.append(cb)
        d.host_allreduce = cb
    d._keep = keep  # keep the buffer / callback alive with the struct
    return d


def nccl_unique_id_from_torch(group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId (through torch's NCCL binding) and broadcasts it."""
    import torch
    import torch.distributed as dist
    if dist.get_rank(group) == 0:
        uid = torch.cuda.nccl.unique_id()
    else:
        uid = bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def torch_allgather(group=None):
    """allgather(bytes) -> [bytes per rank] over torch.distributed (host objects; gloo or
    NCCL process groups): the IPC-handle exchange of make_dist(peer=True)."""
    import torch.distributed as dist

    def ag(b: bytes):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, b, group=group)
        return out
    return ag
