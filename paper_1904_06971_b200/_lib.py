"""ctypes binding of ``libsurriga_b200.so`` (C ABI in ``include/surriga_b200.h``).

There is no CPU fallback: if the library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsurriga_b200.so")

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_i32 = C.POINTER(C.c_int32)


class SgProblem(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("p", C.c_int32), ("form", C.c_int32), ("m", C.c_int32 * 3), ("g", C.c_int32),
        ("knots", _d * 3), ("qpts", _d * 3), ("qwts", _d * 3), ("sol_w", _d),
        ("geo_p", C.c_int32), ("geo_m", C.c_int32 * 3), ("geo_knots", _d * 3), ("geo_hom", _d),
        ("coefficient", C.c_double),
    ]


class SgExec(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("slab_lo", C.c_int64), ("slab_hi", C.c_int64)]


class SgSurrogateParams(C.Structure):
    _fields_ = [
        ("M", C.c_int32), ("q", C.c_int32), ("mode", C.c_int32), ("nlat", C.c_int32 * 3), ("lat_idx", _i64 * 3),
        ("qd", C.c_int32 * 3), ("interp_knots", _d * 3), ("colloc_inv", _d * 3), ("box_pts", _d * 3),
    ]


class SgSurrogateStats(C.Structure):
    _fields_ = [("n_interp_rows", C.c_int64), ("n_quad_rows", C.c_int64), ("n_interp_entries", C.c_int64),
                ("n_zero_dropped", C.c_int64), ("n_reset_rows", C.c_int64)]


class SgCgStats(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int64), ("norm_b", C.c_double), ("rel_residual", C.c_double)]


class NativeError(RuntimeError):
    pass


class UnsupportedError(NativeError, NotImplementedError):
    """Status -2: valid for the reference but outside what this build supports (e.g. p > 4)."""


_lock = threading.Lock()
_lib = None


def lib():
    """Load the sm_100a library (once).  Raises if it is missing -- no fallback path exists."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} not built; run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        L.sg_last_error.restype = C.c_char_p
        L.sg_version.restype = C.c_char_p
        L.sg_assemble.argtypes = [C.POINTER(SgProblem), _i64, C.c_int64, C.POINTER(SgExec), C.POINTER(C.c_void_p)]
        L.sg_surrogate.argtypes = [C.POINTER(SgProblem), C.POINTER(SgSurrogateParams), C.POINTER(SgExec),
                                   C.POINTER(C.c_void_p), C.POINTER(SgSurrogateStats)]
        L.sg_surrogate_begin.argtypes = [C.POINTER(SgProblem), C.POINTER(SgSurrogateParams), C.POINTER(SgExec),
                                         C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _i64]
        L.sg_surrogate_finish.argtypes = [C.c_void_p, C.POINTER(SgSurrogateParams), C.POINTER(C.c_void_p),
                                          C.POINTER(SgSurrogateStats)]
        L.sg_surrogate_state_free.argtypes = [C.c_void_p]
        L.sg_result_sizes.argtypes = [C.c_void_p, _i64, _i64]
        L.sg_result_copy.argtypes = [C.c_void_p, _i32, _i32, _d]
        L.sg_result_copy_i64.argtypes = [C.c_void_p, _i64, _i32, _d]
        L.sg_host_staging_init.argtypes = [C.c_int]
        L.sg_host_register.argtypes = [C.c_void_p, C.c_size_t]
        L.sg_map_points.argtypes = [C.POINTER(SgProblem), C.POINTER(SgExec), _d]
        L.sg_assemble_load.argtypes = [C.POINTER(SgProblem), _d, C.POINTER(SgExec), _d]
        L.sg_host_unregister.argtypes = [C.c_void_p]
        L.sg_assemble_divergence.argtypes = [C.POINTER(SgProblem), C.POINTER(SgProblem), _i64, C.c_int64,
                                             C.POINTER(SgExec), C.POINTER(C.c_void_p)]
        L.sg_surrogate_divergence.argtypes = [C.POINTER(SgProblem), C.POINTER(SgProblem), C.POINTER(SgSurrogateParams),
                                              C.POINTER(C.c_int32), _i64, C.c_int64, C.POINTER(SgExec),
                                              C.POINTER(C.c_void_p), C.POINTER(SgSurrogateStats)]
        L.sg_result_device_ptrs.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.sg_result_checksum.argtypes = [C.c_void_p, _d]
        L.sg_result_free.argtypes = [C.c_void_p]
        L.sg_last_timing.argtypes = [_d, _i32]
        L.sg_last_kernel_times.argtypes = [C.c_char_p, C.c_int32, _d, C.c_int32, _i32]
        L.sg_result_from_host.argtypes = [C.c_int32, C.c_int64, C.c_int64, _i64, _i32, _d, C.POINTER(C.c_void_p)]
        L.sg_spmv.argtypes = [C.c_void_p, _d, _d, C.POINTER(SgExec)]
        L.sg_last_dmma_count.argtypes = [_i64]
        L.sg_quadrature_fields.argtypes = [C.POINTER(SgProblem), _d, C.c_int32, C.POINTER(SgExec), _d, _d, _d, _d, _d]
        L.sg_write_matrix_market_host.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _i64, _i32, _d, C.c_int32, C.c_int32]
        L.sg_write_matrix_market.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int32, C.c_int32]
        L.sg_cg_solve.argtypes = [C.c_void_p, _d, _d, C.c_double, C.c_int64, C.c_int32, C.POINTER(SgExec),
                                  C.POINTER(SgCgStats)]
        _lib = L
    return _lib


SYMBOLS = ("sg_assemble", "sg_surrogate", "sg_surrogate_begin", "sg_surrogate_finish", "sg_surrogate_state_free", "sg_result_sizes", "sg_result_copy", "sg_result_copy_i64",
           "sg_result_device_ptrs", "sg_result_checksum", "sg_result_free", "sg_last_timing",
           "sg_last_kernel_times", "sg_last_error", "sg_version", "sg_max_degree", "sg_host_staging_init",
           "sg_assemble_divergence", "sg_surrogate_divergence", "sg_host_register", "sg_host_unregister",
           "sg_map_points", "sg_assemble_load", "sg_result_from_host", "sg_spmv", "sg_cg_solve",
           "sg_quadrature_fields", "sg_write_matrix_market_host", "sg_write_matrix_market", "sg_last_dmma_count")


def check(rc):
    if rc != 0:
        msg = lib().sg_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        if rc == -6:
            raise IndexError(msg)
        if rc == -2:
            raise UnsupportedError(f"surriga_b200 error {rc}: {msg}")
        raise NativeError(f"surriga_b200 error {rc}: {msg}")


def dptr(a):
    return a.ctypes.data_as(_d) if a is not None else None


class _HostPool:
    """Reusable host buffers for CSR results (large arrays only).

    A result array is a view of a pooled base buffer; the base is reused once no view of it is alive
    (its reference count drops back to the pool's own), so repeated assemblies copy into memory whose
    pages are already mapped instead of paying first-touch page faults on every D2H.  Bases that get
    reused are registered with the driver (cudaHostRegister, ~13 GB/s, done by a background thread
    after the base's first copy), after which the D2H runs straight into them at the PCIe rate
    (57 GB/s) instead of through the staging ring (~36 GB/s, host-memory bound).  At most ``keep``
    idle bases per dtype are retained.  SG_HOST_POOL=0 disables the pool (plain np.empty)."""

    MIN_BYTES = 64 << 20

    def __init__(self, keep=2):
        self.keep = keep
        self.bases = {}
        self.lock = threading.Lock()
        self.enabled = os.environ.get("SG_HOST_POOL", "1") != "0"
        self.registered = {}     # id(base) -> True once pinned
        self.fresh = []          # bases created by the last take(): registered at the next take()
        self.jobs = []
        self.worker = None

    @staticmethod
    def _idle(b):
        return sys.getrefcount(b) <= 4  # pool list + caller loop variable + parameter + getrefcount argument

    def _register_async(self, bases):
        def run(items):
            for b in items:
                if check_quiet(lib().sg_host_register(C.c_void_p(b.ctypes.data), C.c_size_t(b.nbytes))):
                    # no pool lock here: take() may hold it while it joins this thread (sync());
                    # a single dict store is atomic under the GIL
                    self.registered[id(b)] = True

        t = threading.Thread(target=run, args=(list(bases),), daemon=True)
        t.start()
        self.jobs.append(t)

    def sync(self):
        """Wait for pending registrations (call outside timed regions)."""
        for t in self.jobs:
            t.join()
        self.jobs = []

    def release(self):
        self.sync()
        self.fresh = []
        with self.lock:
            for lst in self.bases.values():
                x = None
                for x in [b for b in lst if self._idle(b)]:
                    self._drop(lst, x)
                x = None

    def _drop(self, lst, x):
        if self.registered.pop(id(x), False):
            lib().sg_host_unregister(C.c_void_p(x.ctypes.data))
        for i, b in enumerate(lst):  # by identity (list.remove would compare arrays elementwise)
            if b is x:
                del lst[i]
                break

    def begin(self):
        """Start of a result copy: bases created by earlier copies are filled -> pin them now."""
        with self.lock:
            fresh, self.fresh = self.fresh, []
        if fresh:
            self._register_async(fresh)

    def take(self, n, dtype):
        dtype = np.dtype(dtype)
        if not self.enabled or n * dtype.itemsize < self.MIN_BYTES:
            return np.empty(n, dtype=dtype)
        with self.lock:
            lst = self.bases.setdefault(dtype.str, [])
            best = None
            for b in lst:
                if b.size >= n and self._idle(b) and (best is None or b.size < best.size):
                    best = b
            b = None
            if best is None:
                best = np.empty(n, dtype=dtype)
                lst.append(best)
                self.fresh.append(best)
            idle = [x for x in lst if x is not best and self._idle(x)]
            x = None
            if len(idle) > self.keep:
                self.sync()
                for x in sorted(idle, key=lambda a: a.size)[:len(idle) - self.keep]:
                    self._drop(lst, x)
                x = None
            return best[:n]


def check_quiet(rc):
    return rc == 0


_pool = _HostPool(keep=int(os.environ.get("SG_HOST_POOL_KEEP", "2")))


class Result:
    """Owning handle of a device-resident CSR produced by the library."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def sizes(self):
        nr, nz = C.c_int64(), C.c_int64()
        check(lib().sg_result_sizes(self.h, C.byref(nr), C.byref(nz)))
        return nr.value, nz.value

    def to_host(self):
        """D2H copy -> (indptr, indices, data) with scipy's index dtype (int32 when it fits)."""
        nrows, nnz = self.sizes()
        _pool.begin()
        indices = _pool.take(nnz, np.int32)
        data = _pool.take(nnz, np.float64)
        if nnz < 2**31 - 1:
            indptr = np.empty(nrows + 1, dtype=np.int32)
            check(lib().sg_result_copy(self.h, indptr.ctypes.data_as(_i32), indices.ctypes.data_as(_i32), dptr(data)))
        else:
            indptr = np.empty(nrows + 1, dtype=np.int64)
            check(lib().sg_result_copy_i64(self.h, indptr.ctypes.data_as(_i64), indices.ctypes.data_as(_i32), dptr(data)))
        return indptr, indices, data

    def device_ptrs(self):
        a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().sg_result_device_ptrs(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def checksum(self):
        out = np.zeros(5)
        check(lib().sg_result_checksum(self.h, dptr(out)))
        return out

    def free(self):
        if self.h is not None and self.h.value:
            lib().sg_result_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def host_staging_init(device=0):
    """Allocate the pinned D2H staging ring + host copy pool now (else on the first large copy)."""
    check(lib().sg_host_staging_init(int(device)))


def host_pool_sync():
    """Finish pending registrations of reused host result buffers (call outside timed regions)."""
    _pool.sync()


def host_pool_release():
    """Unpin and drop every idle pooled host buffer (e.g. before forking worker processes)."""
    _pool.release()


def last_timing():
    ms = C.c_double()
    n = C.c_int32()
    lib().sg_last_timing(C.byref(ms), C.byref(n))
    return ms.value, n.value


def last_dmma_count():
    """DMMA (m8n8k4 f64, 512 flops) instructions executed by the assembly kernel in the last call."""
    c = C.c_int64()
    lib().sg_last_dmma_count(C.byref(c))
    return c.value


def last_kernel_times(copies: bool = False):
    """(name, device ms) of each kernel of the last call; ``copies`` adds the timed host->device
    staging copies ("h2d_*")."""
    names = C.create_string_buffer(4096)
    ms = (C.c_double * 64)()
    cnt = C.c_int32()
    lib().sg_last_kernel_times(names, 4096, ms, 64, C.byref(cnt))
    nm = names.value.decode().split(",") if cnt.value else []
    out = list(zip(nm, [ms[i] for i in range(min(cnt.value, 64))]))
    return out if copies else [(n, t) for n, t in out if not n.startswith("h2d_")]
