"""Device-resident consumer of the assembled CSR: sparse products and the
conjugate-gradient SPD solve of ``surriga/solvers.py`` on the GPU.

Mirrors the reference interface (``SolveOptions`` with the same validation messages,
``solve_spd(A, b, opts)`` with the same ``RuntimeError`` messages, ``solvers.py:40-155``).  The
matrix may be a ``SparseMatrix`` / scipy matrix / dense array (uploaded once), or a device-resident
``_lib.Result`` from ``assemble_device`` / ``surrogate_device`` (no D2H of the CSR at all).

Only the conjugate-gradient method runs here: the reference's ``method="direct"`` is a scipy
SuperLU factorisation (``solvers.py:104-105``), which is not part of the B200 path; asking for it
raises ``NotImplementedError`` (never a silent CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .assembly import _exec

__all__ = ["SolveOptions", "solve_spd", "spmv", "DeviceCSR", "to_device"]

_METHODS = ("direct", "conjugate-gradient")
_PRECONDITIONERS = ("none", "diagonal")


@dataclass(frozen=True)
class SolveOptions:
    """solvers.py:40-71 (same fields, defaults and validation messages)."""

    method: str = "direct"
    tolerance: float = 1e-10
    max_iterations: int | None = None
    preconditioner: str = "none"

    def __post_init__(self):
        method = "conjugate-gradient" if self.method == "cg" else self.method
        object.__setattr__(self, "method", method)
        if self.method not in _METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if not 0.0 < self.tolerance < 1.0:
            raise ValueError("tolerance must lie in (0, 1)")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.preconditioner not in _PRECONDITIONERS:
            raise ValueError(f"unknown preconditioner {self.preconditioner!r}")


class DeviceCSR:
    """A square CSR matrix resident on the GPU (owning handle)."""

    def __init__(self, result: _lib.Result, shape):
        self.result = result
        self.shape = tuple(shape)

    def free(self):
        self.result.free()


def to_device(A, device=None) -> DeviceCSR:
    """Upload ``A`` (SparseMatrix, scipy sparse or dense) once; solvers.py:31-35 accepts the same."""
    mat = getattr(A, "mat", A)
    mat = mat.tocsr() if sp.issparse(mat) else sp.csr_matrix(np.asarray(mat, dtype=float))
    mat.sort_indices()
    n = mat.shape[0]
    ip = np.ascontiguousarray(mat.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(mat.indices, dtype=np.int32)
    d = np.ascontiguousarray(mat.data, dtype=np.float64)
    h = C.c_void_p()
    dev = _exec(device).device
    _lib.check(_lib.lib().sg_result_from_host(dev, n, d.size, ip.ctypes.data_as(_lib._i64), ix.ctypes.data_as(_lib._i32),
                                              _lib.dptr(d), C.byref(h)))
    return DeviceCSR(_lib.Result(h.value), mat.shape)


def _device_matrix(A, device=None):
    """-> (DeviceCSR, owned) ; a Result from assemble_device is used in place."""
    if isinstance(A, DeviceCSR):
        return A, False
    if isinstance(A, _lib.Result):
        nr, _ = A.sizes()
        return DeviceCSR(A, (nr, nr)), False
    return to_device(A, device), True


def spmv(A, x, device=None) -> np.ndarray:
    """``A @ x`` on the GPU (the reference's ``mat @ x``)."""
    dA, owned = _device_matrix(A, device)
    try:
        n = dA.shape[0]
        xv = np.ascontiguousarray(np.asarray(x, dtype=float).ravel())
        if xv.size != dA.shape[1]:
            raise ValueError("matrix and vector sizes do not match")
        y = np.empty(n)
        _lib.check(_lib.lib().sg_spmv(dA.result.h, _lib.dptr(xv), _lib.dptr(y), C.byref(_exec(device))))
        return y
    finally:
        if owned:
            dA.free()


def solve_spd(A, b, opts: SolveOptions | None = None, device=None) -> np.ndarray:
    """solvers.py:74-115: solve ``A x = b`` for SPD ``A`` by conjugate gradient on the GPU."""
    opts = opts or SolveOptions()
    if opts.method == "direct":
        raise NotImplementedError("the direct (SuperLU) solve is not part of the B200 path; "
                                  "use SolveOptions(method='conjugate-gradient')")
    dA, owned = _device_matrix(A, device)
    try:
        n = dA.shape[0]
        rhs = np.ascontiguousarray(np.asarray(b, dtype=float).ravel())
        if dA.shape[0] != dA.shape[1] or dA.shape[0] != rhs.size:
            raise ValueError("matrix and right-hand side sizes do not match")
        normb = np.linalg.norm(rhs)
        if normb == 0.0:
            return np.zeros_like(rhs)
        maxit = opts.max_iterations if opts.max_iterations is not None else 10 * n
        x = np.empty(n)
        st = _lib.SgCgStats()
        prec = 1 if opts.preconditioner == "diagonal" else 0
        _lib.check(_lib.lib().sg_cg_solve(dA.result.h, _lib.dptr(rhs), _lib.dptr(x), float(opts.tolerance), int(maxit),
                                          prec, C.byref(_exec(device)), C.byref(st)))
        if st.status == 2:
            raise RuntimeError("non-positive diagonal entry; system is not positive definite")
        if st.status == 1:
            raise RuntimeError(f"negative curvature at iteration {st.iterations}; system is not positive definite")
        if st.status == 3:
            raise RuntimeError(f"conjugate gradient did not converge in {maxit} iterations "
                               f"(relative residual {st.rel_residual:.3e})")
        if st.rel_residual > opts.tolerance:
            raise RuntimeError(f"solve residual {st.rel_residual:.3e} exceeds tolerance {opts.tolerance:.1e}")
        return x
    finally:
        if owned:
            dA.free()

