"""Seeded generators for the synthetic stand-ins of the paper's workloads.

Recipes follow SURVEY §8(d) and the readings listed in DESIGN.md §Inputs:

* C1 — 20×20×20 float64, all ranks 2, G_true i.i.d. N(0,1), T = t(G_true), 30% uniform mask.
* C2 — 256×256×31 float32 ("MSI-shaped", paper P:L481), ranks 4, smooth G_true (rows are
  sums of 3 low-frequency cosines with N(0,1) weights), T = minmax(minmax(t) + 0.01 ε),
  10% uniform mask (RM 90%, Table 5 protocol P:L872).
* C3 — 144×176×3×50 float32 (video-shaped; BASELINE.json only), ranks 3, G_true N(0,1),
  T = minmax(minmax(t) + 0.01 ε), 5% uniform mask.
* C4 — 214×61×144×4 float32 (Guangzhou-shaped 214×61×144, plus a 4-week mode),
  ranks 5, mode-3 rows 1 + cos(2π h τ/144 + φ), others U[0,1), T = minmax(minmax(t)+0.05 ε),
  fibre mask: exactly 36,551 of the 52,216 mode-3 fibres missing (FM 70%).
* C5 — 64×64×64×64×32 float32, ranks 4, G_true N(0,1), T = t(G_true) raw, 5% uniform mask.

"t(G)" for a *truth* is built here as the planted product Π_{p<q} A_{p,q}(i_p,i_q) of
random rank-R pair matrices A_{p,q} = G_{p,q}ᵀ G_{q,p} — a data recipe, not the solver: the
truth only enters the method as observed values on Ω and in the RSE.

Random streams (numpy Generator(Philox(seed + offset))):
  +0 truth factors, +1 G⁰, +2 mask keys, +3 noise ε.
Every array is produced in float64 and rounded once to the config dtype; the same rounded
arrays go to both sides.  Layout: flat, mode-1-fastest; factors concatenated (k asc, i asc,
i≠k), each R_{k,i}×I_k column-major (the C-ABI layout, include/ifctn.h).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


def _rng(seed: int, offset: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed + offset))


def mask_count(sr: float, n: int) -> int:
    """Exact observed count round-half-up(SR·n) (reading R12)."""
    return int(math.floor(sr * n + 0.5))


def _k_smallest_mask(keys: np.ndarray, k: int) -> np.ndarray:
    """Boolean mask of the k smallest keys (a uniform random k-subset for i.i.d. keys)."""
    if k >= keys.size:
        return np.ones(keys.size, dtype=bool)
    if k <= 0:
        return np.zeros(keys.size, dtype=bool)
    thr = np.partition(keys, k - 1)[k - 1]
    m = keys <= thr
    if int(m.sum()) != k:  # ties at the threshold: astronomically unlikely with 63-bit keys
        raise RuntimeError("mask key tie at threshold; change seed")
    return m


def uniform_mask(n: int, count: int, seed: int) -> np.ndarray:
    """Exactly `count` observed entries drawn uniformly without replacement (uint8, 1=observed)."""
    keys = _rng(seed, 2).integers(0, 2**63 - 1, size=n, dtype=np.int64)
    return _k_smallest_mask(keys, count).astype(np.uint8)


def fibre_mask(dims, fibre_mode: int, missing_fibres: int, seed: int) -> np.ndarray:
    """Exactly `missing_fibres` whole mode-`fibre_mode` fibres missing (reading R12)."""
    other = [d for m, d in enumerate(dims) if m != fibre_mode]
    nf = int(np.prod(other))
    keys = _rng(seed, 2).integers(0, 2**63 - 1, size=nf, dtype=np.int64)
    miss = _k_smallest_mask(keys, missing_fibres)
    # fibre id: remaining modes ascending, lowest fastest → array shape (rev other) in C order
    obs_f = (~miss).astype(np.uint8).reshape(list(reversed(other)))
    full = np.expand_dims(obs_f, axis=len(dims) - 1 - fibre_mode)
    rev = list(reversed(dims))
    full = np.broadcast_to(full, rev)
    return np.ascontiguousarray(full).reshape(-1)


def factor_sizes(dims, ranks):
    N = len(dims)
    return [(k, i, int(ranks[k][i]), int(dims[k])) for k in range(N) for i in range(N) if i != k]


def planted_tensor(G: dict, dims) -> np.ndarray:
    """Π_{p<q} A_{p,q}(i_p,i_q) with A_{p,q} = G_{p,q}ᵀG_{q,p}; flat mode-1-fastest float64.
    (Truth recipe only; see module docstring.)"""
    N = len(dims)
    rev = tuple(reversed(dims))
    T = None
    for p in range(N):
        for q in range(p + 1, N):
            A = G[(p, q)].T @ G[(q, p)]                 # (I_p, I_q)
            shape = [1] * N
            shape[N - 1 - p] = dims[p]
            shape[N - 1 - q] = dims[q]
            # axis order in `rev` is descending mode; A must be laid out (…q…p…)
            Ab = A.T.reshape(shape) if q > p else A.reshape(shape)
            if T is None:
                T = np.broadcast_to(Ab, rev).copy()
            else:
                T *= Ab
    if T is None:
        T = np.ones(rev)
    return T.reshape(-1)


def minmax(x: np.ndarray) -> np.ndarray:
    lo, hi = x.min(), x.max()
    return (x - lo) / (hi - lo)


@dataclasses.dataclass
class Problem:
    name: str
    dims: tuple
    ranks: np.ndarray          # (N, N) int32, symmetric, zero diagonal
    dtype: np.dtype            # float32 or float64
    rho: float
    sweeps: int
    truth: np.ndarray          # flat, dtype
    mask: np.ndarray           # flat uint8, 1 = observed
    observed: np.ndarray       # flat, dtype; P_Ω(truth), zeros off Ω
    G0: np.ndarray             # flat factors, dtype
    recipe: dict

    @property
    def N(self):
        return len(self.dims)

    @property
    def n(self):
        return int(np.prod(self.dims))


def _truth_factors(kind: str, dims, ranks, rng) -> dict:
    G = {}
    for (k, i, R, Ik) in factor_sizes(dims, ranks):
        if kind == "normal":
            G[(k, i)] = rng.standard_normal(R * Ik).reshape(Ik, R).T
        elif kind == "smooth":   # C2: rows = Σ_{h=0..2} a_{r,h} cos(π h (x+½)/I_k)
            a = rng.standard_normal((R, 3))
            x = (np.arange(Ik) + 0.5) / Ik
            basis = np.stack([np.cos(np.pi * h * x) for h in range(3)])   # (3, I_k)
            G[(k, i)] = a @ basis
        elif kind == "traffic":  # C4: mode 3 (index 2) periodic daily profile, others U[0,1)
            if k == 2:
                phi = rng.uniform(0.0, 2.0 * np.pi, R)
                tau = np.arange(Ik)
                G[(k, i)] = np.stack([1.0 + np.cos(2.0 * np.pi * (r + 1) * tau / Ik + phi[r])
                                      for r in range(R)])
            else:
                G[(k, i)] = rng.random(R * Ik).reshape(Ik, R).T
        else:
            raise ValueError(kind)
    return G


def init_factors(dims, ranks, observed, mask, dtype, init_kind="uniform", seed=0):
    """G⁰ (stream seed+1) for the given rank matrix: N(0,1), or U[0,s) with
    s = (m·4^P / Π_{p<q} R_{p,q})^{1/(2P)}, m = mean |O| on Ω (reading R8)."""
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    ranks = np.asarray(ranks)
    rng1 = _rng(seed, 1)
    P = N * (N - 1) // 2
    sizes = factor_sizes(dims, ranks)
    total = sum(R_ * Ik for (_, _, R_, Ik) in sizes)
    if init_kind == "normal":
        G0 = rng1.standard_normal(total)
        irec = {"kind": "normal"}
    else:
        m = float(np.mean(np.abs(observed[mask.astype(bool)].astype(np.float64))))
        pr = float(np.prod([ranks[p][q] for p in range(N) for q in range(p + 1, N)]))
        s = (m * 4.0 ** P / pr) ** (1.0 / (2 * P))
        G0 = rng1.uniform(0.0, s, total)
        irec = {"kind": "uniform", "s": s}
    return G0.astype(dtype), irec


# The paper's MSI rank grid: R_{1,2} ∈ {3,6,9,15,30,36}, R_{1,3} = R_{2,3} ∈ {3,6,9}
MSI_GRID = [(r12, r3) for r12 in (3, 6, 9, 15, 30, 36) for r3 in (3, 6, 9)]


# The paper's traffic rank grid: R_{1,2} ∈ {2,3,4,6,9,12,36}, R_{1,3} = R_{2,3} ∈ {3,6,9,12}
TRAFFIC_GRID = [(r12, r3) for r12 in (2, 3, 4, 6, 9, 12, 36) for r3 in (3, 6, 9, 12)]


def grid_rank_matrix(r12: int, r3: int) -> np.ndarray:
    return np.array([[0, r12, r3], [r12, 0, r3], [r3, r3, 0]], np.int32)


def make_problem(name, dims, R, dtype, truth_kind, *, scale_noise=None, mask_kind="uniform",
                 sr=None, fibre_missing_ratio=None, fibre_mode=2, init_kind="normal",
                 rho=0.1, sweeps=10, seed=0) -> Problem:
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    ranks = np.full((N, N), int(R), dtype=np.int32) if np.isscalar(R) else np.asarray(R, np.int32)
    np.fill_diagonal(ranks, 0)
    dtype = np.dtype(dtype)
    n = int(np.prod(dims))

    Gt = _truth_factors(truth_kind, dims, ranks, _rng(seed, 0))
    t = planted_tensor(Gt, dims)
    if scale_noise is not None:
        eps = _rng(seed, 3).standard_normal(n)
        t = minmax(minmax(t) + scale_noise * eps)
    truth = t.astype(dtype)

    if mask_kind == "uniform":
        cnt = mask_count(sr, n)
        mask = uniform_mask(n, cnt, seed)
        mrec = {"kind": "uniform", "sr": sr, "observed": cnt}
    elif mask_kind == "fibre":
        other = int(np.prod([d for m, d in enumerate(dims) if m != fibre_mode]))
        miss = int(math.floor(fibre_missing_ratio * other + 0.5))
        mask = fibre_mask(dims, fibre_mode, miss, seed)
        mrec = {"kind": "fibre", "fibre_mode": fibre_mode, "fibres": other,
                "missing_fibres": miss, "observed": (other - miss) * dims[fibre_mode]}
    else:
        raise ValueError(mask_kind)
    observed = np.where(mask.astype(bool), truth, np.zeros((), dtype)).astype(dtype)

    G0, irec = init_factors(dims, ranks, observed, mask, dtype, init_kind, seed)

    recipe = {"truth": truth_kind, "noise_sigma": scale_noise, "mask": mrec, "init": irec,
              "seed": seed}
    return Problem(name, dims, ranks, dtype, rho, sweeps, truth, mask, observed, G0, recipe)


# name -> (dims, R, dtype, truth kind, kwargs)
CONFIGS = {
    "C1": dict(dims=(20, 20, 20), R=2, dtype="float64", truth_kind="normal", sr=0.30,
               init_kind="normal", sweeps=10),
    "C2": dict(dims=(256, 256, 31), R=4, dtype="float32", truth_kind="smooth", scale_noise=0.01,
               sr=0.10, init_kind="uniform", sweeps=100),
    "C3": dict(dims=(144, 176, 3, 50), R=3, dtype="float32", truth_kind="normal",
               scale_noise=0.01, sr=0.05, init_kind="uniform", sweeps=100),
    "C4": dict(dims=(214, 61, 144, 4), R=5, dtype="float32", truth_kind="traffic",
               scale_noise=0.05, mask_kind="fibre", fibre_missing_ratio=0.70, fibre_mode=2,
               init_kind="uniform", sweeps=200),
    # The 3rd-order Guangzhou shape itself (214×61×144) on the C4 recipe: the tensor
    # the paper's traffic rank grid (TRAFFIC_GRID) is tuned on (f2 bench).
    "C4g": dict(dims=(214, 61, 144), R=5, dtype="float32", truth_kind="traffic", scale_noise=0.05,
                mask_kind="fibre", fibre_missing_ratio=0.70, fibre_mode=2, init_kind="uniform",
                sweeps=100),
    "C5": dict(dims=(64, 64, 64, 64, 32), R=4, dtype="float32", truth_kind="normal", sr=0.05,
               init_kind="normal", sweeps=50),
    # Reduced-size twins with the same recipes, for oracle-speed parity tests (ragged mode-1
    # sizes on purpose: 27, 18 and 9 are not multiples of 4).
    "C2s": dict(dims=(40, 36, 7), R=4, dtype="float32", truth_kind="smooth", scale_noise=0.01,
                sr=0.10, init_kind="uniform", sweeps=20),
    "C3s": dict(dims=(18, 22, 3, 6), R=3, dtype="float32", truth_kind="normal",
                scale_noise=0.01, sr=0.20, init_kind="uniform", sweeps=20),
    "C4s": dict(dims=(27, 9, 18, 4), R=5, dtype="float32", truth_kind="traffic",
                scale_noise=0.05, mask_kind="fibre", fibre_missing_ratio=0.70, fibre_mode=2,
                init_kind="uniform", sweeps=20),
    "C5s": dict(dims=(9, 8, 6, 5, 4), R=4, dtype="float32", truth_kind="normal", sr=0.20,
                init_kind="normal", sweeps=10),
    # Large-rank operating point of the paper's MSI grid: R_{1,2} = 36,
    # R_{1,3} = R_{2,3} = 9, the largest values of P:L485, on the C2 recipe; and its
    # oracle-speed twin.
    "C2r": dict(dims=(256, 256, 31), R=[[0, 36, 9], [36, 0, 9], [9, 9, 0]], dtype="float32",
                truth_kind="smooth", scale_noise=0.01, sr=0.10, init_kind="uniform", sweeps=100),
    "C2rs": dict(dims=(40, 36, 7), R=[[0, 36, 9], [36, 0, 9], [9, 9, 0]], dtype="float32",
                 truth_kind="smooth", scale_noise=0.01, sr=0.10, init_kind="uniform", sweeps=20),
}


def make_config(name: str, seed: int = 0, **overrides) -> Problem:
    kw = dict(CONFIGS[name])
    kw.update(overrides)
    dims = kw.pop("dims")
    R = kw.pop("R")
    dtype = kw.pop("dtype")
    truth_kind = kw.pop("truth_kind")
    return make_problem(name, dims, R, dtype, truth_kind, seed=seed, **kw)
