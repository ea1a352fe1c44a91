"""Thin ctypes binding of libsdpc (include/sdpc.h).  Argument marshalling only.

Every step of the hot path runs in the CUDA library; nothing here computes.  If
libsdpc.so is missing or cannot find an sm_100 device, calls fail loudly (there is
no CPU fallback).  PyTorch supplies device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDPC_LIB") or os.path.join(_HERE, "libsdpc.so")  # SDPC_LIB: experiments only

SDPC_OK, SDPC_ERR_INVALID_ARG, SDPC_ERR_NOT_PD, SDPC_ERR_OOM, SDPC_ERR_CUDA, SDPC_ERR_NCCL, SDPC_ERR_STATE = range(7)

# (name, restype, argtypes) for every symbol declared in include/sdpc.h
_P = C.c_void_p
_SIGS = [
    ("sdpc_create", C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, C.c_int32, C.c_int32,
                              C.c_int32, _P]),
    ("sdpc_get_unique_id", C.c_int, [_P]),
    ("sdpc_get_structure", C.c_int, [_P, _P]),
    ("sdpc_get_scm_layout", C.c_int, [_P, _P]),
    ("sdpc_factor_xinv", C.c_int, [_P, _P, _P]),
    ("sdpc_get_xinv_factor", C.c_int, [_P, _P, _P, _P]),
    ("sdpc_scm_build", C.c_int, [_P, _P, _P, C.c_int64, _P]),
    ("sdpc_get_y_factor", C.c_int, [_P, _P, _P, _P]),
    ("sdpc_get_inverse_columns", C.c_int, [_P, _P, C.c_int32, _P, _P, _P]),
    ("sdpc_scm_cholesky", C.c_int, [_P, _P, C.c_int64, _P, _P]),
    ("sdpc_scm_solve", C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int32, _P]),
    ("sdpc_scm_cholesky_virtual", C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P]),
    ("sdpc_potrf_tile", C.c_int, [_P, _P, C.c_int32, C.c_int64, _P, _P, _P]),
    ("sdpc_trsm_panel", C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, C.c_int64, _P, C.c_int32, _P]),
    ("sdpc_update_tiles", C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                    _P]),
    ("sdpc_iteration", C.c_int, [_P, _P, _P, _P, C.c_int64, _P, _P]),
    ("sdpc_iteration_host", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("sdpc_get_phase_times", C.c_int, [_P, _P]),
    ("sdpc_get_kernel_times", C.c_int, [_P, _P]),
    ("sdpc_search_direction", C.c_int, [_P, _P, _P, C.c_double, _P, C.c_int64, _P, _P, _P, _P, _P]),
    ("sdpc_step_lengths", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    ("sdpc_set_timing", C.c_int, [_P, C.c_int32]),
    ("sdpc_set_truncation", C.c_int, [_P, C.c_int32]),
    ("sdpc_set_cholesky_schedule", C.c_int, [_P, C.c_int32]),
    ("sdpc_set_cholesky_trace", C.c_int, [_P, C.c_int64]),
    ("sdpc_get_cholesky_trace", C.c_int, [_P, _P, C.c_int64, _P]),
    ("sdpc_launch_count", C.c_int64, [_P]),
    ("sdpc_fp64_peak", C.c_int, [C.c_int32, C.c_double, _P, _P]),
    ("sdpc_destroy", C.c_int, [_P]),
    ("sdpc_status_string", C.c_char_p, [C.c_int]),
    ("sdpc_last_info", C.c_int64, [_P]),
    ("sdpc_last_error_message", C.c_char_p, [_P]),
]
SYMBOLS = [s[0] for s in _SIGS]


class _Structure(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("nnzE", C.c_int64), ("perm", _P), ("parent", _P),
                ("colptr", _P), ("rowind", _P), ("nsuper", C.c_int32), ("super_ptr", _P)]


class _Layout(C.Structure):
    _fields_ = [("nb", C.c_int32), ("Pr", C.c_int32), ("Pc", C.c_int32), ("myrow", C.c_int32),
                ("mycol", C.c_int32), ("mloc", C.c_int64), ("nloc", C.c_int64), ("lld", C.c_int64)]


_lib = None


def lib():
    """Load libsdpc.so (raises if it was not built; there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libsdpc.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SdpcError(RuntimeError):
    def __init__(self, status, info=0, where=""):
        self.status = status
        self.info = info
        msg = lib().sdpc_status_string(status).decode()
        super().__init__(f"{where}: {msg} (status {status}, info {info})")


def _ptr(a):
    """Raw pointer of a numpy array (host) or torch tensor (device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class Handle:
    """One libsdpc handle (one problem, one GPU).  Mirrors the C ABI names."""

    def __init__(self, n, m, a_ptr, a_row, a_col, a_val, b, perm=None, device=0, nranks=1, rank=0, nccl_id=None):
        L = lib()
        self._keep = [np.ascontiguousarray(a_ptr, dtype=np.int64), np.ascontiguousarray(a_row, dtype=np.int32),
                      np.ascontiguousarray(a_col, dtype=np.int32), np.ascontiguousarray(a_val, dtype=np.float64),
                      np.ascontiguousarray(b, dtype=np.float64)]
        pp = None if perm is None else np.ascontiguousarray(perm, dtype=np.int32)
        h = _P()
        nid = None
        if nccl_id is not None:
            self._nid = (C.c_char * 128).from_buffer_copy(bytes(nccl_id))
            nid = C.addressof(self._nid)
        st = L.sdpc_create(C.byref(h), int(n), int(m), *[_ptr(x) for x in self._keep], _ptr(pp), int(device),
                           int(nranks), int(rank), nid)
        if st != SDPC_OK:
            raise SdpcError(st, 0, "sdpc_create")
        self.h = h
        self.n, self.m = int(n), int(m)
        self.device = device

    @classmethod
    def from_instance(cls, inst, device=0, with_perm=True, nranks=1, rank=0, nccl_id=None):
        return cls(inst.n, inst.m, inst.a_ptr, inst.a_row, inst.a_col, inst.a_val, inst.b,
                   inst.perm if with_perm else None, device, nranks, rank, nccl_id)

    def _check(self, st, where):
        if st != SDPC_OK:
            msg = lib().sdpc_last_error_message(self.h).decode()
            raise SdpcError(st, lib().sdpc_last_info(self.h), where + (f" [{msg}]" if msg else ""))

    def get_structure(self):
        s = _Structure()
        self._check(lib().sdpc_get_structure(self.h, C.byref(s)), "sdpc_get_structure")

        def arr(p, cnt, dt):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(dt)), shape=(cnt,)).copy()
        return dict(n=s.n, m=s.m, nnzE=s.nnzE, nsuper=s.nsuper, perm=arr(s.perm, s.n, C.c_int32),
                    parent=arr(s.parent, s.n, C.c_int32), colptr=arr(s.colptr, s.n + 1, C.c_int64),
                    rowind=arr(s.rowind, s.nnzE, C.c_int32), super_ptr=arr(s.super_ptr, s.nsuper + 1, C.c_int32))

    def get_scm_layout(self):
        s = _Layout()
        self._check(lib().sdpc_get_scm_layout(self.h, C.byref(s)), "sdpc_get_scm_layout")
        return {f: getattr(s, f) for f, _ in _Layout._fields_}

    def factor_xinv(self, xbar_E, stream=None):
        self._check(lib().sdpc_factor_xinv(self.h, _ptr(xbar_E), _stream(stream)), "sdpc_factor_xinv")

    def get_xinv_factor(self, L_E, D, stream=None):
        self._check(lib().sdpc_get_xinv_factor(self.h, _ptr(L_E), _ptr(D), _stream(stream)), "sdpc_get_xinv_factor")

    def scm_build(self, y_E, B, ldb=None, stream=None):
        ldb = self.m if ldb is None else ldb
        self._check(lib().sdpc_scm_build(self.h, _ptr(y_E), _ptr(B), int(ldb), _stream(stream)), "sdpc_scm_build")

    def get_y_factor(self, LY_E, DY, stream=None):
        self._check(lib().sdpc_get_y_factor(self.h, _ptr(LY_E), _ptr(DY), _stream(stream)), "sdpc_get_y_factor")

    def get_inverse_columns(self, cols, X_out, Y_out, stream=None):
        c = np.ascontiguousarray(cols, dtype=np.int32)
        self._check(lib().sdpc_get_inverse_columns(self.h, _ptr(c), int(c.size), _ptr(X_out), _ptr(Y_out),
                                                   _stream(stream)), "sdpc_get_inverse_columns")

    def scm_cholesky(self, B, ldb=None, stream=None, raise_not_pd=True):
        ldb = self.m if ldb is None else ldb
        info = C.c_int32(0)
        st = lib().sdpc_scm_cholesky(self.h, _ptr(B), int(ldb), C.byref(info), _stream(stream))
        if st == SDPC_ERR_NOT_PD and not raise_not_pd:
            return int(info.value)
        self._check(st, "sdpc_scm_cholesky")
        return int(info.value)

    def scm_solve(self, R, G, ldr=None, ldg=None, nrhs=1, stream=None):
        """(R R^T) X = G in place (the SCE B dz = g with the SCM factor)."""
        ldr = self.m if ldr is None else ldr
        ldg = self.m if ldg is None else ldg
        self._check(lib().sdpc_scm_solve(self.h, _ptr(R), int(ldr), _ptr(G), int(ldg), int(nrhs), _stream(stream)),
                    "sdpc_scm_solve")

    # -- distributed SCM Cholesky tile entries (asynchronous; see sdpc.h) --
    def potrf_tile(self, A, n, lda, inv, info_dev, stream=None):
        self._check(lib().sdpc_potrf_tile(self.h, _ptr(A), int(n), int(lda), _ptr(inv), _ptr(info_dev),
                                          _stream(stream)), "sdpc_potrf_tile")

    def trsm_panel(self, A, rows, lda, L, ldl, inv, kb, stream=None):
        self._check(lib().sdpc_trsm_panel(self.h, _ptr(A), int(rows), int(lda), _ptr(L), int(ldl), _ptr(inv),
                                          int(kb), _stream(stream)), "sdpc_trsm_panel")

    def update_tiles(self, C_loc, ldc, P, ldp, k1, K, stream=None, jlo=0, jhi=0):
        self._check(lib().sdpc_update_tiles(self.h, _ptr(C_loc), int(ldc), _ptr(P), int(ldp), int(k1), int(K),
                                            int(jlo), int(jhi), _stream(stream)), "sdpc_update_tiles")

    def iteration(self, xbar_E, y_E, B, ldb=None, stream=None, raise_not_pd=True):
        """(a1) || (a2) -> (b) -> (c) -> (d) on device buffers; returns the Cholesky info."""
        ldb = self.m if ldb is None else ldb
        info = C.c_int32(0)
        st = lib().sdpc_iteration(self.h, _ptr(xbar_E), _ptr(y_E), _ptr(B), int(ldb), C.byref(info), _stream(stream))
        if st == SDPC_ERR_NOT_PD and not raise_not_pd and info.value > 0:
            return int(info.value)
        self._check(st, "sdpc_iteration")
        return int(info.value)

    def iteration_host(self, xbar_E, y_E, rdiag=None, stream=None):
        x = np.ascontiguousarray(xbar_E, dtype=np.float64)
        y = np.ascontiguousarray(y_E, dtype=np.float64)
        info = C.c_int32(0)
        st = lib().sdpc_iteration_host(self.h, _ptr(x), _ptr(y), _ptr(rdiag), C.byref(info), _stream(stream))
        if st == SDPC_ERR_NOT_PD:
            return int(info.value)
        self._check(st, "sdpc_iteration_host")
        return int(info.value)

    def phase_times(self):
        t = (C.c_double * 8)()
        self._check(lib().sdpc_get_phase_times(self.h, t), "sdpc_get_phase_times")
        return list(t)

    def search_direction(self, xbar_E, G_E, beta_mu, R, ldr, g, dz, dY_E, dX_E, stream=None):
        """sdpc_search_direction: g, dz, dY, dX (device tensors) of the HKM direction."""
        self._check(lib().sdpc_search_direction(self.h, _ptr(xbar_E), _ptr(G_E), float(beta_mu), _ptr(R), int(ldr),
                                                _ptr(g), _ptr(dz), _ptr(dY_E), _ptr(dX_E), _stream(stream)),
                    "sdpc_search_direction")

    def step_lengths(self, xbar_E, dX_E, y_E, dY_E, stream=None):
        """sdpc_step_lengths -> (alpha_p, alpha_d)."""
        ap, ad = C.c_double(0), C.c_double(0)
        self._check(lib().sdpc_step_lengths(self.h, _ptr(xbar_E), _ptr(dX_E), _ptr(y_E), _ptr(dY_E), C.byref(ap),
                                            C.byref(ad), _stream(stream)), "sdpc_step_lengths")
        return ap.value, ad.value

    def kernel_times(self):
        t = (C.c_double * 8)()
        self._check(lib().sdpc_get_kernel_times(self.h, t), "sdpc_get_kernel_times")
        return list(t)

    def set_truncation(self, on):
        self._check(lib().sdpc_set_truncation(self.h, int(bool(on))), "sdpc_set_truncation")

    def set_cholesky_schedule(self, task_graph):
        self._check(lib().sdpc_set_cholesky_schedule(self.h, int(bool(task_graph))), "sdpc_set_cholesky_schedule")

    def set_cholesky_trace(self, cap):
        self._check(lib().sdpc_set_cholesky_trace(self.h, int(cap)), "sdpc_set_cholesky_trace")

    def get_cholesky_trace(self, cap):
        out = np.zeros((int(cap), 4), dtype=np.uint64)
        n = C.c_int64(0)
        self._check(lib().sdpc_get_cholesky_trace(self.h, _ptr(out), int(cap), C.byref(n)), "sdpc_get_cholesky_trace")
        return out[: n.value], out.reshape(-1)

    def set_timing(self, on):
        self._check(lib().sdpc_set_timing(self.h, int(bool(on))), "sdpc_set_timing")

    def launch_count(self):
        return int(lib().sdpc_launch_count(self.h))

    def last_info(self):
        return int(lib().sdpc_last_info(self.h))

    def destroy(self):
        if getattr(self, "h", None):
            lib().sdpc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def get_unique_id():
    """sdpc_get_unique_id: the 128-byte NCCL id (bytes) for Handle(..., nccl_id=...)."""
    buf = (C.c_char * 128)()
    st = lib().sdpc_get_unique_id(buf)
    if st != SDPC_OK:
        raise SdpcError(st, 0, "sdpc_get_unique_id")
    return bytes(buf)


def scm_cholesky_virtual(handles, Bs, ldb, stream=None):
    """sdpc_scm_cholesky_virtual: the distributed Cholesky with every rank's handle in this process
    (one device).  Returns info."""
    P = len(handles)
    hs = (_P * P)(*[h.h for h in handles])
    bp = (_P * P)(*[_ptr(b) for b in Bs])
    info = C.c_int32(0)
    st = lib().sdpc_scm_cholesky_virtual(hs, P, bp, int(ldb), C.byref(info), _stream(stream))
    if st == SDPC_ERR_NOT_PD:
        return int(info.value)
    if st != SDPC_OK:
        raise SdpcError(st, 0, "sdpc_scm_cholesky_virtual [" + lib().sdpc_last_error_message(handles[0].h).decode() + "]")
    return int(info.value)


def fp64_peak(device=0, ms=2000.0):
    a, b = C.c_double(0), C.c_double(0)
    st = lib().sdpc_fp64_peak(int(device), float(ms), C.byref(a), C.byref(b))
    if st != SDPC_OK:
        raise SdpcError(st, 0, "sdpc_fp64_peak")
    return a.value, b.value
