"""paper_2511_16358_b200 — B200-native iFCTN tensor-completion PAM sweep (arxiv 2511.16358).

The product is the C-ABI shared library ``libifctn.so`` (include/ifctn.h, sources in
csrc/).  This package is its thin Python binding: ``_abi`` exposes every C entry point
under its own name; :class:`Solver` marshals torch/numpy buffers into those calls.  PyTorch
is used for device memory (the workspace), streams and process groups only.

There is no CPU fallback: importing :mod:`paper_2511_16358_b200._abi` without the built
library raises.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._abi import (IFCTN_F32, IFCTN_F64, IFCTN_FLAG_NO_FUSE, IFCTN_FLAG_NO_GRAPH,  # noqa: F401
                   IFCTN_FLAG_GRAM_GEMM, IFCTN_FLAG_NO_DMMA, IFCTN_FLAG_NO_L2PASS, IFCTN_FLAG_NO_PDL, IFCTN_FLAG_NO_SOLVE_REDUCE, IFCTN_FLAG_NO_VBLOCK,
                   IFCTN_FLAG_NONE, IFCTN_FLAG_X_FULL, IFCTN_MODEL, IFCTN_X, IfctnError,
                   ifctn_dist, ifctn_trace_row)

__all__ = ["Solver", "IfctnError", "IFCTN_F32", "IFCTN_F64", "IFCTN_MODEL", "IFCTN_X", "mask_uniform", "mask_fibres",
           "factor_layout", "num_params"]


def _ranks_matrix(ranks, N):
    r = np.asarray(ranks, dtype=np.int64)
    if r.ndim == 0:
        r = np.full((N, N), int(r), dtype=np.int64)
        np.fill_diagonal(r, 0)
    return r.reshape(N, N)


def factor_layout(dims, ranks):
    """[(k, i, offset, R, I_k)] of the concatenated factor array (k asc, i asc, i≠k)."""
    N = len(dims)
    r = _ranks_matrix(ranks, N)
    out, off = [], 0
    for k in range(N):
        for i in range(N):
            if i != k:
                out.append((k, i, off, int(r[k, i]), int(dims[k])))
                off += int(r[k, i]) * int(dims[k])
    return out


def num_params(dims, ranks) -> int:
    lay = factor_layout(dims, ranks)
    return lay[-1][2] + lay[-1][3] * lay[-1][4] if lay else 0


def _ptr(x):
    """Device or host address of a torch tensor / numpy array (kept alive by the caller)."""
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr())
    return ctypes.c_void_p(x.ctypes.data)


def check_buffer(x, name, kind, count):
    """Validate a buffer before its raw address crosses the C-ABI (the library cannot see
    dtype, extent or strides): `kind` is "f32", "f64" or "u8" (mask: uint8 or bool bytes),
    `count` the element count the call reads or writes.  Raises IfctnError(E_ARG)."""
    if x is None:
        raise IfctnError(1, f"{name} must not be None")
    if hasattr(x, "data_ptr"):  # torch tensor
        import torch
        ok = {"f32": (torch.float32,), "f64": (torch.float64,), "u8": (torch.uint8, torch.bool)}[kind]
        dt, n, contig = x.dtype, x.numel(), x.is_contiguous()
    elif isinstance(x, np.ndarray):
        ok = {"f32": (np.dtype(np.float32),), "f64": (np.dtype(np.float64),),
              "u8": (np.dtype(np.uint8), np.dtype(np.bool_))}[kind]
        dt, n, contig = x.dtype, x.size, x.flags["C_CONTIGUOUS"]
    else:
        raise IfctnError(1, f"{name} must be a torch tensor or a numpy array")
    if dt not in ok:
        raise IfctnError(1, f"{name} has dtype {dt}, expected {kind}")
    if n != count:
        raise IfctnError(1, f"{name} has {n} elements, expected {count}")
    if not contig:
        raise IfctnError(1, f"{name} must be contiguous")


class Solver:
    """One iFCTN-TC problem on one GPU (or one rank's shard).

    Arguments follow Algorithm 1's input: observed tensor O, mask Ω, ranks R,
    ρ; plus the initial factors G⁰.  Tensors are flat mode-1-fastest (torch CUDA/CPU tensors
    or numpy arrays); the library copies them in ``ifctn_create``.
    """

    def __init__(self, dims, ranks, observed, mask, init_factors, rho=0.1, dtype=None,
                 dist=None, flags=0, stream=None, workspace=True):
        import torch

        self.dims = tuple(int(d) for d in dims)
        self.N = len(self.dims)
        self.ranks = _ranks_matrix(ranks, self.N)
        if dtype is None:
            dt = observed.dtype
            is64 = (dt == np.float64) if isinstance(dt, np.dtype) else (dt == torch.float64)
            dtype = IFCTN_F64 if is64 else IFCTN_F32
        self.dtype = dtype
        self.rho = float(rho)
        self.dist = dist
        self._torch_dtype = torch.float64 if dtype == IFCTN_F64 else torch.float32
        flat = [int(v) for v in self.ranks.reshape(-1)]
        self.ws_bytes = _abi.ifctn_workspace_bytes(self.N, self.dims, flat, dtype, dist)
        if isinstance(mask, np.ndarray) and mask.dtype == np.bool_:
            mask = mask.view(np.uint8)
        # local extents (this rank's shard under dist) — every buffer is checked against them
        if dist is not None and dist.world > 1:
            sm, b, e = _abi.ifctn_shard_range(self.N, self.dims, dist)
            self.shard_mode, self.shard_begin, self.shard_end = sm, b, e
            ld = list(self.dims)
            ld[sm] = e - b
            self.local_dims = tuple(ld)
        else:
            self.shard_mode, self.shard_begin, self.shard_end = 0, 0, self.dims[0]
            self.local_dims = self.dims
        self.n_local = int(np.prod(self.local_dims))
        lay = factor_layout(self.local_dims, self.ranks)
        self.n_params_local = lay[-1][2] + lay[-1][3] * lay[-1][4]
        self._kind = "f64" if dtype == IFCTN_F64 else "f32"
        check_buffer(observed, "observed", self._kind, self.n_local)
        check_buffer(mask, "mask", "u8", self.n_local)
        check_buffer(init_factors, "init_factors", self._kind, self.n_params_local)
        # Ω must be non-empty (Algorithm 1 needs an observation); the library checks host masks
        # itself, device masks are checked here (single GPU: a shard may be empty)
        if hasattr(mask, "data_ptr") and mask.is_cuda and (dist is None or dist.world <= 1):
            if not bool(mask.any()):
                raise IfctnError(11, "the mask has no observed entry")
        self.workspace = None
        ws_ptr = None
        if workspace:
            self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device="cuda")
            base = self.workspace.data_ptr()
            ws_ptr = ctypes.c_void_p((base + 255) // 256 * 256)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        self.stream = stream
        self.ctx = _abi.ifctn_create(self.N, self.dims, flat, dtype, self.rho, _ptr(observed),
                                     _ptr(mask), _ptr(init_factors), ws_ptr, self.ws_bytes, dist,
                                     ctypes.c_void_p(stream), flags)

    # -- Algorithm 1 -------------------------------------------------------------------
    def sweep(self, t_max, eps=0.0, trace=False):
        """Run up to t_max sweeps. Returns sweeps done, or (done, rows) with trace=True."""
        if trace:
            rows = (ifctn_trace_row * max(int(t_max), 1))()
            done = _abi.ifctn_sweep(self.ctx, t_max, eps, rows)
            out = [dict(sweep=rows[s].sweep, rel_change=rows[s].rel_change,
                        objective=rows[s].objective, dx2=rows[s].dx2, dg2=rows[s].dg2)
                   for s in range(done)]
            return done, out
        return _abi.ifctn_sweep(self.ctx, t_max, eps, None)

    def sync(self):
        _abi.ifctn_sync(self.ctx)

    def profile_sweep(self):
        """One sweep with per-launch CUDA-event timings (ms), see ifctn_profile_sweep."""
        return _abi.ifctn_profile_sweep(self.ctx)

    def reconstruct(self, what=IFCTN_X, out=None):
        import torch
        if out is None:
            out = torch.empty(self.n_local, dtype=self._torch_dtype, device="cuda")
        check_buffer(out, "out", self._kind, self.n_local)
        _abi.ifctn_reconstruct(self.ctx, what, _ptr(out))
        return out

    def factors(self, out=None):
        import torch
        if out is None:
            out = torch.empty(self.n_params_local, dtype=self._torch_dtype, device="cuda")
        check_buffer(out, "out", self._kind, self.n_params_local)
        _abi.ifctn_get_factors(self.ctx, _ptr(out))
        return out

    def rse(self, truth) -> float:
        check_buffer(truth, "truth", self._kind, self.n_local)
        return _abi.ifctn_rse(self.ctx, _ptr(truth))

    def metrics(self, truth) -> dict:
        """RSE, RMSE on Ω^c, band-mean PSNR, SSIM (ifctn_metrics)."""
        check_buffer(truth, "truth", self._kind, self.n_local)
        return _abi.ifctn_metrics(self.ctx, _ptr(truth))

    def objective(self) -> float:
        return _abi.ifctn_objective(self.ctx)

    # -- step-level entry points --------------------------------------------------------
    def block_coefficients(self, k, i):
        """(β, ω) of block (k,i) as float64 numpy arrays of shape (I_i, I_k)."""
        Ii, Ik = self.local_dims[i], self.local_dims[k]
        b = np.empty(Ii * Ik, dtype=np.float64)
        w = np.empty(Ii * Ik, dtype=np.float64)
        _abi.ifctn_block_coefficients(self.ctx, k, i, _ptr(b), _ptr(w))
        return b.reshape(Ik, Ii).T, w.reshape(Ik, Ii).T

    def block_update(self, k, i):
        _abi.ifctn_block_update(self.ctx, k, i)

    def x_update(self):
        n = np.zeros(4, dtype=np.float64)
        _abi.ifctn_x_update(self.ctx, _ptr(n))
        return n

    def launch_count(self) -> int:
        return _abi.ifctn_launch_count(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            _abi.ifctn_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def mask_uniform(n, observed, seed=0, device=None):
    """RM sampling set on the device (ifctn_mask_uniform): uint8[n], exactly `observed` ones."""
    import torch
    m = torch.empty(int(n), dtype=torch.uint8, device=device or "cuda")
    stream = torch.cuda.current_stream(m.device).cuda_stream
    _abi.ifctn_mask_uniform(m.data_ptr() if n else None, n, observed, seed, stream)
    return m


def mask_fibres(dims, mode, missing, seed=0, device=None):
    """FM sampling set on the device (ifctn_mask_fibres): uint8[Π dims], mode-1-fastest, with
    exactly `missing` whole mode-`mode` fibres unobserved."""
    import torch
    m = torch.empty(int(np.prod(dims)), dtype=torch.uint8, device=device or "cuda")
    stream = torch.cuda.current_stream(m.device).cuda_stream
    _abi.ifctn_mask_fibres(m.data_ptr(), dims, mode, missing, seed, stream)
    return m
