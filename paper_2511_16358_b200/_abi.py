"""ctypes binding of libifctn.so (include/ifctn.h) — argument marshalling only.

Every function here has the name of the C entry point it calls.  No arithmetic of the
method happens in Python: each step of the sweep runs in the sm_100a kernels of
csrc/.  If the shared library is missing this module raises at import time — there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# IFCTN_LIB: an experiment build of the same library (scripts/variants.sh), never a fallback
LIB_PATH = os.environ.get("IFCTN_LIB") or os.path.join(_HERE, "libifctn.so")

IFCTN_F32, IFCTN_F64 = 0, 1
IFCTN_MODEL, IFCTN_X = 0, 1
IFCTN_FLAG_NONE, IFCTN_FLAG_NO_GRAPH, IFCTN_FLAG_X_FULL, IFCTN_FLAG_NO_VBLOCK = 0, 1, 2, 8
IFCTN_FLAG_NO_FUSE = 16
IFCTN_FLAG_NO_SOLVE_REDUCE = 64
IFCTN_FLAG_NO_L2PASS = 128
IFCTN_FLAG_GRAM_GEMM = 256
IFCTN_FLAG_NO_PDL = 512
IFCTN_FLAG_NO_DMMA = 1024
IFCTN_MAX_ORDER, IFCTN_MAX_RANK = 6, 64

STATUS = ["IFCTN_OK", "IFCTN_E_ARG", "IFCTN_E_SHAPE", "IFCTN_E_RANKS", "IFCTN_E_WORKSPACE",
          "IFCTN_E_CUDA", "IFCTN_E_NCCL", "IFCTN_E_NOT_SPD", "IFCTN_E_NONFINITE", "IFCTN_E_STATE",
          "IFCTN_E_UNSUPPORTED", "IFCTN_E_NO_OBSERVED"]


class IfctnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{name}: {msg}")


HOST_ALLREDUCE = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t, ctypes.c_void_p)
HOST_ALLGATHER = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
IFCTN_XCHG_NCCL, IFCTN_XCHG_PEER = 0, 1


class ifctn_dist(ctypes.Structure):
    _fields_ = [("nccl_unique_id", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("shard_mode", ctypes.c_int),
                ("host_allreduce", HOST_ALLREDUCE), ("user", ctypes.c_void_p),
                ("exchange", ctypes.c_int), ("host_allgather", HOST_ALLGATHER)]


class ifctn_trace_row(ctypes.Structure):
    _fields_ = [("sweep", ctypes.c_int), ("rel_change", ctypes.c_double),
                ("objective", ctypes.c_double), ("dx2", ctypes.c_double), ("dg2", ctypes.c_double)]


class ifctn_instance(ctypes.Structure):
    _fields_ = [("ranks", ctypes.POINTER(ctypes.c_int32)), ("rho", ctypes.c_double),
                ("init_factors", ctypes.c_void_p)]


class ifctn_instance_result(ctypes.Structure):
    _fields_ = [("rse", ctypes.c_double), ("objective", ctypes.c_double),
                ("seconds", ctypes.c_double), ("status", ctypes.c_int)]


_lib = None

# name -> (restype, argtypes); the exported C-ABI (checked against include/ifctn.h by tests)
_VP, _I, _D, _U = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_uint
_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)
SIGNATURES = {
    "ifctn_workspace_bytes": (_I, [_I, _I64P, _I32P, _I, ctypes.POINTER(ifctn_dist), ctypes.POINTER(ctypes.c_size_t)]),
    "ifctn_shard_range": (_I, [_I, _I64P, ctypes.POINTER(ifctn_dist), ctypes.POINTER(ctypes.c_int), _I64P, _I64P]),
    "ifctn_create": (_I, [ctypes.POINTER(_VP), _I, _I64P, _I32P, _I, _D, _VP, _VP, _VP, _VP,
                          ctypes.c_size_t, ctypes.POINTER(ifctn_dist), _VP, _U]),
    "ifctn_sweep": (_I, [_VP, _I, _D, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ifctn_trace_row)]),
    "ifctn_sync": (_I, [_VP]),
    "ifctn_profile_sweep": (_I, [_VP, ctypes.POINTER(ctypes.c_float), _I, ctypes.POINTER(ctypes.c_int)]),
    "ifctn_reconstruct": (_I, [_VP, _I, _VP]),
    "ifctn_get_factors": (_I, [_VP, _VP]),
    "ifctn_rse": (_I, [_VP, _VP, ctypes.POINTER(ctypes.c_double)]),
    "ifctn_objective": (_I, [_VP, ctypes.POINTER(ctypes.c_double)]),
    "ifctn_metrics": (_I, [_VP, _VP, ctypes.POINTER(ctypes.c_double)]),
    "ifctn_block_coefficients": (_I, [_VP, _I, _I, _VP, _VP]),
    "ifctn_block_update": (_I, [_VP, _I, _I]),
    "ifctn_x_update": (_I, [_VP, _VP]),
    "ifctn_destroy": (_I, [_VP]),
    "ifctn_status_string": (ctypes.c_char_p, [_I]),
    "ifctn_last_error": (ctypes.c_char_p, [_VP]),
    "ifctn_launch_count": (ctypes.c_int64, [_VP]),
    "ifctn_mask_uniform": (_I, [_VP, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, _VP]),
    "ifctn_mask_fibres": (_I, [_VP, _I, _I64P, _I, ctypes.c_int64, ctypes.c_uint64, _VP]),
    "ifctn_grid_run": (_I, [_I, _I64P, _I, _VP, _VP, _VP, ctypes.POINTER(ifctn_instance), _I, _I, _I,
                            ctypes.POINTER(ifctn_instance_result)]),
    "ifctn_peer_selftest": (_I, [_I, _I, ctypes.c_int64, _I64P]),
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(the CUDA extension is required; there is no fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, ctx=None):
    if status != 0:
        msg = lib().ifctn_last_error(ctx)
        raise IfctnError(status, msg.decode() if msg else "")


def _i64arr(vals):
    a = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return a


def _i32arr(vals):
    a = (ctypes.c_int32 * len(vals))(*[int(v) for v in vals])
    return a


def ifctn_workspace_bytes(order, dims, ranks_flat, dtype, dist=None) -> int:
    out = ctypes.c_size_t(0)
    check(lib().ifctn_workspace_bytes(order, _i64arr(dims), _i32arr(ranks_flat), dtype,
                                      ctypes.byref(dist) if dist is not None else None, ctypes.byref(out)))
    return out.value


def ifctn_shard_range(order, dims, dist=None):
    sm = ctypes.c_int(0)
    b = ctypes.c_int64(0)
    e = ctypes.c_int64(0)
    check(lib().ifctn_shard_range(order, _i64arr(dims), ctypes.byref(dist) if dist is not None else None,
                                  ctypes.byref(sm), ctypes.byref(b), ctypes.byref(e)))
    return sm.value, b.value, e.value


def ifctn_create(order, dims, ranks_flat, dtype, rho, observed_ptr, mask_ptr, init_ptr,
                 workspace_ptr, workspace_bytes, dist, stream_ptr, flags):
    ctx = ctypes.c_void_p(0)
    st = lib().ifctn_create(ctypes.byref(ctx), order, _i64arr(dims), _i32arr(ranks_flat), dtype,
                            float(rho), observed_ptr, mask_ptr, init_ptr, workspace_ptr,
                            int(workspace_bytes), ctypes.byref(dist) if dist is not None else None,
                            stream_ptr, int(flags))
    if st != 0:
        msg = lib().ifctn_last_error(None)
        raise IfctnError(st, msg.decode() if msg else "")
    return ctx


def ifctn_sweep(ctx, t_max, eps=0.0, trace=None):
    done = ctypes.c_int(0)
    check(lib().ifctn_sweep(ctx, int(t_max), float(eps), ctypes.byref(done), trace), ctx)
    return done.value


def ifctn_sync(ctx):
    check(lib().ifctn_sync(ctx), ctx)


def ifctn_profile_sweep(ctx, capacity=4096):
    ms = (ctypes.c_float * capacity)()
    cnt = ctypes.c_int(0)
    check(lib().ifctn_profile_sweep(ctx, ms, capacity, ctypes.byref(cnt)), ctx)
    return [ms[t] for t in range(min(cnt.value, capacity))]


def ifctn_reconstruct(ctx, what, out_ptr):
    check(lib().ifctn_reconstruct(ctx, int(what), out_ptr), ctx)


def ifctn_get_factors(ctx, out_ptr):
    check(lib().ifctn_get_factors(ctx, out_ptr), ctx)


def ifctn_rse(ctx, truth_ptr) -> float:
    r = ctypes.c_double(0)
    check(lib().ifctn_rse(ctx, truth_ptr, ctypes.byref(r)), ctx)
    return r.value


def ifctn_objective(ctx) -> float:
    r = ctypes.c_double(0)
    check(lib().ifctn_objective(ctx, ctypes.byref(r)), ctx)
    return r.value


def ifctn_metrics(ctx, truth_ptr) -> dict:
    out = (ctypes.c_double * 5)()
    check(lib().ifctn_metrics(ctx, truth_ptr, out), ctx)
    return dict(rse=out[0], rmse=out[1], psnr=out[2], ssim=out[3], missing=int(out[4]))


def ifctn_block_coefficients(ctx, k, i, beta_ptr, omega_ptr):
    check(lib().ifctn_block_coefficients(ctx, int(k), int(i), beta_ptr, omega_ptr), ctx)


def ifctn_block_update(ctx, k, i):
    check(lib().ifctn_block_update(ctx, int(k), int(i)), ctx)


def ifctn_x_update(ctx, norms_ptr=None):
    check(lib().ifctn_x_update(ctx, norms_ptr), ctx)


def ifctn_destroy(ctx):
    check(lib().ifctn_destroy(ctx))


def ifctn_status_string(s: int) -> str:
    return lib().ifctn_status_string(int(s)).decode()


def ifctn_last_error(ctx=None) -> str:
    r = lib().ifctn_last_error(ctx)
    return r.decode() if r else ""


def ifctn_launch_count(ctx) -> int:
    return int(lib().ifctn_launch_count(ctx))


def ifctn_grid_run(order, dims, dtype, observed_ptr, mask_ptr, truth_ptr, instances, t_max,
                   concurrency):
    """instances: list of (ranks_flat, rho, init_ptr); returns a list of result dicts."""
    n = len(instances)
    arr = (ifctn_instance * max(n, 1))()
    keep = []
    for q, (ranks_flat, rho, init_ptr) in enumerate(instances):
        r = _i32arr(ranks_flat)
        keep.append(r)
        arr[q].ranks = ctypes.cast(r, ctypes.POINTER(ctypes.c_int32))
        arr[q].rho = float(rho)
        arr[q].init_factors = init_ptr
    res = (ifctn_instance_result * max(n, 1))()
    st = lib().ifctn_grid_run(order, _i64arr(dims), dtype, observed_ptr, mask_ptr, truth_ptr, arr, n,
                              int(t_max), int(concurrency), res)
    out = [dict(rse=res[q].rse, objective=res[q].objective, seconds=res[q].seconds,
                status=res[q].status) for q in range(n)]
    if st != 0:
        msg = lib().ifctn_last_error(None)
        raise IfctnError(st, (msg.decode() if msg else "") + f" (per-instance: {[o['status'] for o in out]})")
    return out


def ifctn_mask_uniform(mask_ptr, n, observed, seed, stream=None):
    check(lib().ifctn_mask_uniform(mask_ptr, int(n), int(observed), int(seed), stream))


def ifctn_mask_fibres(mask_ptr, dims, mode, missing_fibres, seed, stream=None):
    check(lib().ifctn_mask_fibres(mask_ptr, len(dims), _i64arr(dims), int(mode), int(missing_fibres),
                                  int(seed), stream))


def ifctn_peer_selftest(world: int, rounds: int, n: int) -> int:
    """Peer-exchange protocol self-test on the current device; returns the mismatch count."""
    err = ctypes.c_int64(-1)
    check(lib().ifctn_peer_selftest(world, rounds, n, ctypes.byref(err)))
    return err.value
