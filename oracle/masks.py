"""The paper's missingness protocols (RM and FM) as exact-count draws, written out plainly.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): the reference the on-device generators
`ifctn_mask_uniform` / `ifctn_mask_fibres` are checked against; never
imported by the product package.

Protocols ("random-missing (RM) and fiber-missing (FM)"; "fiber-wise
missingness"), with DESIGN.md reading R12 (exact count, uniform without replacement) and
R30 (the counter-based key stream both sides implement):

  key(u)  = the u-th output (u = 0, 1, …) of splitmix64 started at state `seed`:
            s_u = seed + (u+1)·0x9E3779B97F4A7C15 (mod 2^64), key = fmix64(s_u),
            fmix64: z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27; z *= 0x94D049BB133111EB;
            z ^= z>>31.
  RM      mask[u] = 1 iff u is one of the `observed` indices with the smallest keys.
  FM      fibre id of entry u: its linear index with mode m removed (remaining modes ascending,
          lowest fastest); the `missing` fibres with the smallest keys (over fibre ids) are
          0 along their whole length, every other entry 1.
Tensors are flat, mode-1-fastest (the repository's linearisation).
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix64_keys(seed: int, count: int, start: int = 0) -> np.ndarray:
    """key(start..start+count-1) as uint64 (numpy uint64 arithmetic wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        u = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + u * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def smallest(keys: np.ndarray, k: int) -> np.ndarray:
    """Boolean selector of the k smallest keys (keys distinct)."""
    sel = np.zeros(keys.size, dtype=bool)
    if k > 0:
        sel[np.argsort(keys, kind="stable")[:k]] = True
    return sel


def mask_uniform(n: int, observed: int, seed: int) -> np.ndarray:
    """RM: exactly `observed` of n entries observed (uint8, 1 = observed)."""
    return smallest(splitmix64_keys(seed, n), observed).astype(np.uint8)


def mask_fibres(dims, mode: int, missing: int, seed: int) -> np.ndarray:
    """FM: exactly `missing` whole mode-`mode` fibres unobserved (uint8, 1 = observed)."""
    dims = [int(d) for d in dims]
    n = int(np.prod(dims))
    inner = int(np.prod(dims[:mode]))
    span = inner * dims[mode]
    nf = n // dims[mode]
    miss_f = smallest(splitmix64_keys(seed, nf), missing)
    u = np.arange(n, dtype=np.int64)
    fib = u % inner + inner * (u // span)
    return (~miss_f[fib]).astype(np.uint8)
