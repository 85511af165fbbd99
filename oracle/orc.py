"""TEST INFRASTRUCTURE — ctypes binding of the C restatement (oracle/_lib/
libkrylov_oracle.so, built from oracle/krylov_oracle.c by oracle/Makefile).

Same call shapes as oracle/ref.py, so a test can run one scenario through the
reference, the restatement and the product and compare."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import ref as _ref

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_LIB = os.path.join(HERE, "_lib", "libkrylov_oracle.so")

i64, i32, dbl, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
P_dbl, P_i64 = C.POINTER(C.c_double), C.POINTER(C.c_int64)
kry_solver_config, kry_report = _ref.kry_solver_config, _ref.kry_report
kry_append_outcome, kry_store_info = _ref.kry_append_outcome, _ref.kry_store_info

SIGS = {
    "orc_last_error": (C.c_char_p, []),
    "orc_laplace2d": (C.c_int, [i64, i64, P_i64, P_i64, P_i64, P_i64, P_dbl]),
    "orc_laplace3d": (C.c_int, [i64, i64, i64, P_i64, P_i64, P_i64, P_i64, P_dbl]),
    "orc_spmv": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl]),
    "orc_mpk": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, i64, P_dbl]),
    "orc_gram": (C.c_int, [i64, i64, P_dbl, P_dbl]),
    "orc_try_cholesky": (C.c_int, [i64, P_dbl, P_dbl, P_i64]),
    "orc_bcgs_pip_partial": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "orc_bcgs_pip": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "orc_bcgs_pip2": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "orc_store_create": (C.c_int, [i64, i64, i64, i64, C.POINTER(vp)]),
    "orc_store_destroy": (None, [vp]),
    "orc_store_append_block": (C.c_int, [vp, P_dbl, i64, C.c_int, i32, C.POINTER(kry_append_outcome), P_i64]),
    "orc_store_preprocess_block": (C.c_int, [vp, P_dbl, i64, C.c_int, C.POINTER(kry_append_outcome), P_i64]),
    "orc_store_finalize_big_panel": (C.c_int, [vp, C.POINTER(kry_append_outcome), P_i64]),
    "orc_store_get_info": (C.c_int, [vp, C.POINTER(kry_store_info)]),
    "orc_store_coefficients": (C.c_int, [vp, P_dbl]),
    "orc_store_columns": (C.c_int, [vp, i64, i64, P_dbl]),
    "orc_store_hessenberg": (C.c_int, [vp, i64, P_dbl, P_i64]),
    "orc_hessenberg_lsq": (C.c_int, [i64, P_dbl, dbl, P_dbl, P_dbl, P_i64]),
    "orc_sstep_gmres": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl, C.POINTER(kry_solver_config),
                                  C.POINTER(kry_report), P_dbl]),
    "orc_standard_gmres": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl, C.POINTER(kry_solver_config),
                                     C.POINTER(kry_report), P_dbl]),
}

_lib = None


def available() -> bool:
    return os.path.exists(ORC_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{ORC_LIB} not built (make -C oracle oracle)")
        L = C.CDLL(ORC_LIB)
        for k, (r, a) in SIGS.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg, pivot=0):
        super().__init__(f"[{code}] {msg}")
        self.code, self.pivot = code, pivot


def _chk(rc, pivot=0):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode(), pivot)


_f, _p = _ref._f, _ref._p


def _csr(fn, *dims):
    n, nnz = C.c_int64(), C.c_int64()
    _chk(fn(*dims, C.byref(n), C.byref(nnz), None, None, None))
    rp = np.zeros(n.value + 1, np.int64)
    ci = np.zeros(nnz.value, np.int64)
    v = np.zeros(nnz.value)
    _chk(fn(*dims, C.byref(n), C.byref(nnz), rp.ctypes.data_as(P_i64), ci.ctypes.data_as(P_i64), _p(v)))
    return _ref.Csr(n.value, rp, ci, v)


def laplace2d(nx, ny):
    return _csr(lib().orc_laplace2d, nx, ny)


def laplace3d(nx, ny, nz):
    return _csr(lib().orc_laplace3d, nx, ny, nz)


def spmv(a, x):
    x = _f(x)
    y = np.zeros(a.n)
    _chk(lib().orc_spmv(a.n, *a.ptrs(), _p(x), _p(y)))
    return y


def mpk(a, start, s):
    out = np.zeros((a.n, s + 1), order="F")
    _chk(lib().orc_mpk(a.n, *a.ptrs(), _p(_f(start)), s, _p(out)))
    return out


def gram(v):
    v = _f(v, 2)
    g = np.zeros((v.shape[1], v.shape[1]), order="F")
    _chk(lib().orc_gram(v.shape[0], v.shape[1], _p(v), _p(g)))
    return g


def try_cholesky(s):
    s = _f(s, 2)
    r = np.zeros(s.shape, order="F")
    piv = C.c_int64()
    _chk(lib().orc_try_cholesky(s.shape[0], _p(s), _p(r), C.byref(piv)))
    return r, piv.value


def _pip(fn, q_prev, v):
    v = _f(v, 2)
    n, w = v.shape
    q, c0 = (None, 0) if q_prev is None or np.asarray(q_prev).size == 0 else (_f(q_prev, 2), np.asarray(q_prev).shape[1])
    out = np.zeros((n, w), order="F")
    rc = np.zeros((c0, w), order="F")
    rj = np.zeros((w, w), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    code = fn(n, _p(q), c0, _p(v), w, _p(out), _p(rc), _p(rj), C.byref(piv), C.byref(red))
    return code, out, rc, rj, piv.value, red.value


def bcgs_pip(q_prev, v):
    code, q, rc, rj, piv, red = _pip(lib().orc_bcgs_pip, q_prev, v)
    _chk(code, piv)
    return q, rc, rj, red


def bcgs_pip2(q_prev, v):
    code, q, rc, rj, piv, red = _pip(lib().orc_bcgs_pip2, q_prev, v)
    _chk(code, piv)
    return q, rc, rj, red


class Store:
    def __init__(self, n, m, s, shat):
        h = C.c_void_p()
        _chk(lib().orc_store_create(n, m, s, shat, C.byref(h)))
        self._h, self.n, self.m = h, n, m

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_store_destroy(self._h)
            self._h = None

    def info(self):
        inf = kry_store_info()
        _chk(lib().orc_store_get_info(self._h, C.byref(inf)))
        return inf

    def append_block(self, v, overlap, kind):
        v = _f(v, 2)
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().orc_store_append_block(self._h, _p(v), v.shape[1], int(overlap), int(kind), C.byref(o),
                                          C.byref(d)))
        return o, d.value

    def preprocess_block(self, v, overlap):
        v = _f(v, 2)
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().orc_store_preprocess_block(self._h, _p(v), v.shape[1], int(overlap), C.byref(o), C.byref(d)))
        return o, d.value

    def finalize_big_panel(self):
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().orc_store_finalize_big_panel(self._h, C.byref(o), C.byref(d)))
        return o, d.value

    def coefficients(self):
        r = np.zeros((self.m + 1, self.m + 1), order="F")
        _chk(lib().orc_store_coefficients(self._h, _p(r)))
        return r

    def columns(self, first, count):
        out = np.zeros((self.n, count), order="F")
        if count:
            _chk(lib().orc_store_columns(self._h, first, count, _p(out)))
        return out

    def all(self):
        return self.columns(0, self.info().filled)

    def column(self, j):
        return self.columns(j, 1)[:, 0]

    def hessenberg(self, k):
        h = np.zeros((k + 1, k), order="F")
        col = C.c_int64()
        _chk(lib().orc_store_hessenberg(self._h, k, _p(h), C.byref(col)))
        return h


def solve(a, b, x0, cfg, standard=False, cap=200000):
    b = _f(b)
    x0a = None if x0 is None else _f(x0)
    x = np.zeros(a.n)
    rep = kry_report()
    cyc = np.zeros(cap)
    pb = np.zeros(cap, np.int64)
    pbp = np.zeros(cap, np.int64)
    rep.cycle_residuals, rep.cycle_residuals_cap = cyc.ctypes.data_as(P_dbl), cap
    rep.per_block, rep.per_block_cap = pb.ctypes.data_as(P_i64), cap
    rep.per_big_panel, rep.per_big_panel_cap = pbp.ctypes.data_as(P_i64), cap
    fn = lib().orc_standard_gmres if standard else lib().orc_sstep_gmres
    _chk(fn(a.n, *a.ptrs(), _p(b), _p(x0a), C.byref(cfg), C.byref(rep), _p(x)))
    return _ref.RefReport(rep.status, rep.iterations, rep.restarts, rep.initial_residual,
                          rep.final_relative_residual, list(cyc[: rep.n_cycle_residuals]), bool(rep.breakdown),
                          rep.breakdown_kappa, rep.reduces, list(pb[: rep.n_per_block]),
                          list(pbp[: rep.n_per_big_panel]), rep.reduces_per_iteration, rep.wall_seconds, x)
