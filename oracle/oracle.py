"""ctypes front-end of the float64 C oracle (oracle/ifctn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg — never by the product package
(paper_2511_16358_b200/), which shares no code with it.

Every function here is argument marshalling; the arithmetic, and the paper passage each
step follows, is in ifctn_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ifctn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        i64p, i32p, dp = P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_double)
        vp, u8p = ctypes.c_void_p, P(ctypes.c_uint8)
        c_int, c_i64, c_d = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        sig = {
            "orc_set_threads": (None, [c_int]),
            "orc_get_threads": (c_int, []),
            "orc_num_params": (c_i64, [c_int, i64p, i32p]),
            "orc_factor_offset": (c_i64, [c_int, i64p, i32p, c_int, c_int]),
            "orc_pair_gram": (None, [c_int, i64p, i32p, dp, c_int, c_int, dp]),
            "orc_model": (None, [c_int, i64p, i32p, dp, dp]),
            "orc_model_at": (c_d, [c_int, i64p, i32p, dp, i64p]),
            "orc_block_contract": (None, [c_int, i64p, i32p, dp, vp, c_int, c_int, c_int, dp, dp]),
            "orc_block_contract_at": (None, [c_int, i64p, i32p, dp, vp, c_int, c_int, c_int,
                                             c_i64, c_i64, dp, dp]),
            "orc_column_solve": (c_int, [c_int, c_i64, dp, dp, dp, dp, c_d, dp]),
            "orc_block_update": (c_int, [c_int, i64p, i32p, dp, vp, c_int, c_int, c_int, c_d, dp]),
            "orc_refill": (None, [c_int, i64p, i32p, dp, dp, u8p, c_d, dp]),
            "orc_objective": (c_d, [c_int, i64p, i32p, dp, dp]),
            "orc_init_x": (None, [c_i64, vp, c_int, u8p, dp]),
            "orc_rse": (c_d, [c_i64, dp, dp]),
            "orc_sweep": (c_int, [c_int, i64p, i32p, dp, dp, u8p, c_d, dp, dp, c_int]),
            "orc_solve": (c_int, [c_int, i64p, i32p, dp, dp, u8p, c_d, c_int, c_d, dp, c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


class Shape:
    """dims (N,), ranks (N,N) symmetric with zero diagonal."""

    def __init__(self, dims, ranks):
        self.dims = _i64(dims)
        self.ranks = _i32(np.asarray(ranks).reshape(len(dims), len(dims)))
        self.N = len(dims)
        self.n = int(np.prod(self.dims))

    @property
    def args(self):
        return (self.N, _p(self.dims, ctypes.c_int64), _p(self.ranks, ctypes.c_int32))


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def get_threads() -> int:
    return lib().orc_get_threads()


def num_params(sh: Shape) -> int:
    return int(lib().orc_num_params(*sh.args))


def factor_offset(sh: Shape, k: int, i: int) -> int:
    return int(lib().orc_factor_offset(*sh.args, k, i))


def factor(sh: Shape, G, k: int, i: int):
    """View of G_{k,i} as an (R, I_k) array (column-major storage, r fastest)."""
    off = factor_offset(sh, k, i)
    R, Ik = int(sh.ranks[k, i]), int(sh.dims[k])
    return np.asarray(G)[off:off + R * Ik].reshape(Ik, R).T


def pair_gram(sh: Shape, G, p: int, q: int):
    G = _f64(G)
    H = np.empty(int(sh.dims[p] * sh.dims[q]), dtype=np.float64)
    lib().orc_pair_gram(*sh.args, _p(G, ctypes.c_double), p, q, _p(H, ctypes.c_double))
    return H.reshape(int(sh.dims[q]), int(sh.dims[p])).T  # (I_p, I_q)


def model(sh: Shape, G):
    """t = iFCTN(G), flat mode-1-fastest (length n)."""
    G = _f64(G)
    t = np.empty(sh.n, dtype=np.float64)
    lib().orc_model(*sh.args, _p(G, ctypes.c_double), _p(t, ctypes.c_double))
    return t


def model_at(sh: Shape, G, idx) -> float:
    G = _f64(G)
    idx = _i64(idx)
    return float(lib().orc_model_at(*sh.args, _p(G, ctypes.c_double), _p(idx, ctypes.c_int64)))


def _xarg(X):
    X = np.ascontiguousarray(X)
    if X.dtype == np.float32:
        return X, 1
    X = _f64(X)
    return X, 0


def block_contract(sh: Shape, G, X, k: int, i: int):
    """(β, ω) of block (k,i) as (I_i, I_k) arrays."""
    G = _f64(G)
    X, isf = _xarg(X)
    Ii, Ik = int(sh.dims[i]), int(sh.dims[k])
    b = np.empty(Ii * Ik, dtype=np.float64)
    w = np.empty(Ii * Ik, dtype=np.float64)
    lib().orc_block_contract(*sh.args, _p(G, ctypes.c_double), X.ctypes.data, isf, k, i,
                             _p(b, ctypes.c_double), _p(w, ctypes.c_double))
    return b.reshape(Ik, Ii).T, w.reshape(Ik, Ii).T


def block_contract_at(sh: Shape, G, X, k: int, i: int, a: int, j: int):
    G = _f64(G)
    X, isf = _xarg(X)
    b = ctypes.c_double()
    w = ctypes.c_double()
    lib().orc_block_contract_at(*sh.args, _p(G, ctypes.c_double), X.ctypes.data, isf, k, i,
                                int(a), int(j), ctypes.byref(b), ctypes.byref(w))
    return b.value, w.value


def column_solve(Gik, beta_col, omega_col, c_old, rho):
    """Gik: (R, I_i). Returns (status, c_new)."""
    Gik = _f64(np.asarray(Gik).T)  # column-major R×I_i == row-major I_i×R
    R = Gik.shape[1]
    beta_col, omega_col, c_old = _f64(beta_col), _f64(omega_col), _f64(c_old)
    c = np.empty(R, dtype=np.float64)
    st = lib().orc_column_solve(R, Gik.shape[0], _p(Gik, ctypes.c_double),
                                _p(beta_col, ctypes.c_double), _p(omega_col, ctypes.c_double),
                                _p(c_old, ctypes.c_double), float(rho), _p(c, ctypes.c_double))
    return st, c


def block_update(sh: Shape, G, X, k: int, i: int, rho: float):
    """In-place update of G (float64 array) for block (k,i). Returns (status, dG2)."""
    assert G.dtype == np.float64 and G.flags.c_contiguous
    X, isf = _xarg(X)
    d = ctypes.c_double(0.0)
    st = lib().orc_block_update(*sh.args, _p(G, ctypes.c_double), X.ctypes.data, isf, k, i,
                                float(rho), ctypes.byref(d))
    return st, d.value


def refill(sh: Shape, G, X, mask, rho):
    """In-place X update. Returns (dX2, X2_old, f_new)."""
    assert X.dtype == np.float64 and X.flags.c_contiguous
    G = _f64(G)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.zeros(3, dtype=np.float64)
    lib().orc_refill(*sh.args, _p(G, ctypes.c_double), _p(X, ctypes.c_double),
                     _p(mask, ctypes.c_uint8), float(rho), _p(out, ctypes.c_double))
    return tuple(out)


def objective(sh: Shape, G, X) -> float:
    G, X = _f64(G), _f64(X)
    return float(lib().orc_objective(*sh.args, _p(G, ctypes.c_double), _p(X, ctypes.c_double)))


def init_x(O, mask):
    O = np.ascontiguousarray(O)
    isf = 1 if O.dtype == np.float32 else 0
    if not isf:
        O = _f64(O)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    X = np.empty(O.size, dtype=np.float64)
    lib().orc_init_x(O.size, O.ctypes.data, isf, _p(mask, ctypes.c_uint8), _p(X, ctypes.c_double))
    return X


def rse(truth, X) -> float:
    truth, X = _f64(truth), _f64(X)
    return float(lib().orc_rse(truth.size, _p(truth, ctypes.c_double), _p(X, ctypes.c_double)))


def sweep(sh: Shape, G, X, mask, rho, F_prev: float, check_lemma2: bool = True):
    """One PAM sweep in place. Returns (status, F_new, row[rel, F, dX2, dG2])."""
    assert G.dtype == np.float64 and X.dtype == np.float64
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    F = ctypes.c_double(F_prev)
    row = np.zeros(4, dtype=np.float64)
    st = lib().orc_sweep(*sh.args, _p(G, ctypes.c_double), _p(X, ctypes.c_double),
                         _p(mask, ctypes.c_uint8), float(rho), ctypes.byref(F),
                         _p(row, ctypes.c_double), int(check_lemma2))
    return st, F.value, row


def solve(sh: Shape, G, X, mask, rho, t_max, eps=0.0, check_lemma2=True):
    """Algorithm 1 in place on (G, X). Returns (sweeps_done_or_-status, trace (s,4))."""
    assert G.dtype == np.float64 and X.dtype == np.float64
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    trace = np.zeros((t_max, 4), dtype=np.float64)
    r = lib().orc_solve(*sh.args, _p(G, ctypes.c_double), _p(X, ctypes.c_double),
                        _p(mask, ctypes.c_uint8), float(rho), int(t_max), float(eps),
                        _p(trace, ctypes.c_double), int(check_lemma2))
    return r, trace[:max(r, 0)]
