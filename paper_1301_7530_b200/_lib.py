"""ctypes binding of ``librcg.so`` (the C ABI declared in ``include/rcg.h``).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every device operation raises.  ``EXPORTS`` lists every symbol the
header declares (the CPU test suite checks the built library exports them).
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

from .core_errors import ContractViolation, NumericalFailure, RankDeficient

import os as _os
# RCG_LIB overrides the library path (A/B comparisons of builds on one box)
_LIB_PATH = Path(_os.environ.get("RCG_LIB") or (Path(__file__).resolve().parent / "librcg.so"))

RCG_OK, RCG_ERR_CONTRACT, RCG_ERR_RANK_DEFICIENT, RCG_ERR_NUMERICAL, RCG_ERR_CUDA, RCG_ERR_OOM = range(6)
FAIL_NONE, FAIL_RZ, FAIL_WAW = 0, 1, 2

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


class RcgCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_offsets", C.c_void_p),
                ("row_offsets_64", C.c_int32), ("block", C.c_int32),
                ("col_indices", C.c_void_p), ("values", C.c_void_p),
                ("bsr_row_offsets", C.c_void_p), ("bsr_col_indices", C.c_void_p), ("bsr_values", C.c_void_p),
                ("bsr_slice", C.c_int32), ("dia_count", C.c_int32), ("dia_block", C.c_int32), ("rem_rows", C.c_int32),
                ("dia_offsets", C.c_void_p), ("dia_values", C.c_void_p),
                ("rem_row_ids", C.c_void_p), ("rem_col_indices", C.c_void_p), ("rem_values", C.c_void_p),
                ("rem_width", C.c_int32), ("pad2", C.c_int32)]


class RcgDeflation(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_c", C.c_int64), ("C", C.c_void_p), ("ldc", C.c_int64),
                ("AC", C.c_void_p), ("ldac", C.c_int64), ("L", C.c_void_p), ("Ginv", C.c_void_p)]


class RcgSolveCfg(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64), ("reorthogonalize", C.c_int32),
                ("trace_capture", C.c_int32), ("store_directions", C.c_int32), ("batch", C.c_int32),
                ("krylov_cap", C.c_int64)]


class RcgTraceView(C.Structure):
    _fields_ = [("n", C.c_int64), ("iterations", C.c_int64), ("n_betas", C.c_int64),
                ("converged", C.c_int32), ("failure", C.c_int32), ("early_exit", C.c_int32),
                ("pad_", C.c_int32), ("r0_norm", C.c_double), ("b_norm", C.c_double),
                ("alphas", C.c_void_p), ("betas", C.c_void_p), ("rz_inner", C.c_void_p),
                ("residual_norms", C.c_void_p), ("Z", C.c_void_p), ("W", C.c_void_p),
                ("AW", C.c_void_p), ("R", C.c_void_p), ("waw", C.c_void_p), ("ld", C.c_int64),
                ("device_seconds", C.c_double)]


class RcgHalo(C.Structure):
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("n_local", C.c_int64), ("n_ghost", C.c_int64),
                ("send_idx", C.c_void_p), ("send_off", C.c_void_p), ("recv_off", C.c_void_p),
                ("send_buf", C.c_void_p)]


class RcgKernelStat(C.Structure):
    _fields_ = [("launches", C.c_int64), ("seconds", C.c_double), ("bytes", C.c_double)]


KCLASSES = ("spmv", "update", "coarse", "precond", "colreduce", "wupdate", "actr", "halo", "allreduce")

_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_d = C.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "rcg_ctx_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "rcg_ctx_destroy": (None, [_vp]),
    "rcg_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "rcg_last_error": (C.c_char_p, [_vp]),
    "rcg_version": (C.c_int, []),
    "rcg_num_kernel_launches": (C.c_int, [_vp, c_int64_p]),
    "rcg_debug_guard_violations": (C.c_int64, []),
    "rcg_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "rcg_ctx_kernel_stats": (C.c_int, [_vp, C.POINTER(RcgKernelStat), C.c_int]),
    "rcg_ctx_reset_stats": (C.c_int, [_vp]),
    "rcg_comm_unique_id": (C.c_int, [C.c_char_p, _vp]),
    "rcg_comm_init": (C.c_int, [_vp, C.c_char_p, _vp, C.c_int, C.c_int]),
    "rcg_comm_destroy": (C.c_int, [_vp]),
    "rcg_allreduce_sum": (C.c_int, [_vp, _vp, _i64]),
    "rcg_halo_exchange": (C.c_int, [_vp, C.POINTER(RcgHalo), _vp]),
    "rcg_loop_group_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "rcg_loop_group_destroy": (None, [_vp]),
    "rcg_comm_init_loopback": (C.c_int, [_vp, _vp, C.c_int]),
    "rcg_spmv": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _vp]),
    "rcg_spmm": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _i64, _i64, _vp, _i64]),
    "rcg_csr_diagonal": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _vp]),
    "rcg_csr_block3_analyze": (C.c_int, [_vp, C.POINTER(RcgCsr), C.POINTER(_i32)]),
    "rcg_csr_block3_build": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _vp, _vp]),
    "rcg_gen_diffusion_rows": (C.c_int, [_vp, _vp, C.c_int32, _vp, C.POINTER(C.c_int64)]),
    "rcg_gen_diffusion_fill": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "rcg_gen_elasticity_rows": (C.c_int, [_vp, C.c_int64, _vp, C.POINTER(C.c_int64)]),
    "rcg_gen_elasticity_fill": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "rcg_csr_dia_analyze": (C.c_int, [_vp, C.POINTER(RcgCsr), C.c_int32, _vp, C.POINTER(C.c_int32)]),
    "rcg_csr_dia_build": (C.c_int, [_vp, C.POINTER(RcgCsr), C.c_int32, _vp, C.c_int32, _vp, C.POINTER(C.c_int32)]),
    "rcg_csr_block3_slice_plan": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, C.POINTER(C.c_int64)]),
    "rcg_csr_block3_slice_build": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _vp, _vp]),
    "rcg_diag_apply": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "rcg_gemm_tn": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i32]),
    "rcg_gemm_nn": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    "rcg_dense_cholesky": (C.c_int, [_vp, _vp, _i64, _d, _vp, _vp, c_int64_p]),
    "rcg_deflation_build": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _i64, _i64, _vp, _i64, _vp, _vp, c_int64_p]),
    "rcg_project": (C.c_int, [_vp, C.POINTER(RcgDeflation), _vp, _vp]),
    "rcg_initial_guess": (C.c_int, [_vp, C.POINTER(RcgDeflation), _vp, _vp]),
    "rcg_apcg_solve": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, C.POINTER(RcgDeflation), _vp, _vp,
                                 C.POINTER(RcgSolveCfg), C.POINTER(_vp)]),
    "rcg_apcg_solve_sharded": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, C.POINTER(RcgDeflation), _vp, _vp,
                                         C.POINTER(RcgSolveCfg), C.POINTER(RcgHalo), C.POINTER(_vp)]),
    "rcg_deflation_build_sharded": (C.c_int, [_vp, C.POINTER(RcgCsr), _vp, _i64, _i64, _vp, _i64, _vp, _vp,
                                              C.POINTER(RcgHalo), c_int64_p]),
    "rcg_trace_get_view": (C.c_int, [_vp, C.POINTER(RcgTraceView)]),
    "rcg_trace_free": (None, [_vp]),
    "rcg_lanczos_tridiag": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "rcg_tridiag_eigvals": (C.c_int, [_vp, _vp, _vp, _i64, _vp]),
    "rcg_tridiag_eigvecs": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "rcg_select_converged": (C.c_int, [_vp, _vp, _vp, _i64, _d, _vp]),
    "rcg_cluster_filter": (C.c_int, [_vp, _vp, _i64, _i64, c_int64_p]),
    "rcg_ritz_select": (C.c_int, [_vp, _vp, _vp, _i64, _d, _vp, _vp, _vp, _vp, _vp]),
    "rcg_ritz_vectors": (C.c_int, [_vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _i64, _i32, _vp, _i64]),
    "rcg_column_norms": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _vp]),
    "rcg_column_norms_sharded": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _vp]),
    "rcg_scale_columns": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _i64]),
}
EXPORTS = tuple(SIGNATURES)

_lib = None
_lib_lock = threading.Lock()


def lib_path():
    return _LIB_PATH


def load(path=None):
    """Load (once) and type the library; raises if it is not built."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else _LIB_PATH
        if not p.exists():
            raise RuntimeError(f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(the B200 path has no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


# ---------------------------------------------------------------------------
# per-thread contexts on the current torch stream


_tls = threading.local()


def _torch():
    import torch
    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch


class Context:
    """Owns one ``rcg_ctx`` (device scratch, counters) bound to a stream."""

    def __init__(self, device):
        self.lib = load()
        self.device = device
        torch = require_cuda()
        stream = torch.cuda.current_stream(device).cuda_stream
        h = _vp()
        rc = self.lib.rcg_ctx_create(device, _vp(stream), C.byref(h))
        if rc != RCG_OK or not h.value:
            raise RuntimeError(f"rcg_ctx_create failed with status {rc}")
        self.h = h
        self.stream = stream

    def bind_stream(self):
        torch = _torch()
        s = torch.cuda.current_stream(self.device).cuda_stream
        if s != self.stream:
            self.lib.rcg_ctx_set_stream(self.h, _vp(s))
            self.stream = s
        return self

    def check(self, rc, what=""):
        if rc == RCG_OK:
            return
        msg = (self.lib.rcg_last_error(self.h) or b"").decode(errors="replace")
        if rc == RCG_ERR_CONTRACT:
            raise ContractViolation(msg or what)
        if rc == RCG_ERR_NUMERICAL:
            raise NumericalFailure(msg or what)
        if rc == RCG_ERR_OOM:
            raise MemoryError(msg or what)
        raise RuntimeError(f"{what}: {msg} (status {rc})")

    def set_profiling(self, on):
        self.lib.rcg_ctx_set_profiling(self.h, 1 if on else 0)

    def reset_stats(self):
        self.lib.rcg_ctx_reset_stats(self.h)

    def kernel_stats(self):
        arr = (RcgKernelStat * len(KCLASSES))()
        self.lib.rcg_ctx_kernel_stats(self.h, arr, len(KCLASSES))
        return {k: dict(launches=arr[i].launches, seconds=arr[i].seconds, bytes=arr[i].bytes)
                for i, k in enumerate(KCLASSES)}

    def launches(self):
        v = C.c_int64(0)
        self.lib.rcg_num_kernel_launches(self.h, C.byref(v))
        return v.value

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                self.lib.rcg_ctx_destroy(self.h)
                self.h = _vp()
        except Exception:
            pass


def context(device=None):
    torch = require_cuda()
    if device is None:
        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    ctx = ctxs.get(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device)
    return ctx.bind_stream()


def total_launches():
    """Kernel launches issued by this thread's contexts (bench `gpu_launches`)."""
    ctxs = getattr(_tls, "ctxs", None) or {}
    return sum(c.launches() for c in ctxs.values())


def ptr(t):
    """Raw device pointer of a torch tensor (or None)."""
    return None if t is None else _vp(t.data_ptr())


class CudaArray:
    """``__cuda_array_interface__`` over library-owned memory; keeps the owner
    alive for as long as any tensor made from it is alive."""

    def __init__(self, owner, data_ptr, shape, strides_elems):
        self.owner = owner
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape),
            "typestr": "<f8",
            "data": (int(data_ptr), False),
            "version": 3,
            "strides": tuple(8 * int(s) for s in strides_elems),
            "stream": None,
        }


def as_numpy_bool(t):
    return np.asarray(t.cpu().numpy(), dtype=bool)
