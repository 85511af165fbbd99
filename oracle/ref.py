"""TEST INFRASTRUCTURE — ctypes binding of oracle/_ref/libkrylov_ref.so.

libkrylov_ref.so is the unmodified CPU reference (/root/reference/proj/include,
compiled in place by oracle/Makefile with the reference's Release flags)
behind oracle/ref_shim.cpp.  Only tests/, tests/golden/make_golden.py,
__graft_entry__.smoke() and bench.py's CPU legs import this module; the
product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libkrylov_ref.so")

i64, i32, dbl, vp = C.c_int64, C.c_int32, C.c_double, C.c_void_p
P_dbl, P_i64, P_i32 = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)


def _capi():
    # Share the struct layouts with the product header (include/krylov_b200.h)
    # without importing the product package (which needs the CUDA library).
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_kry_capi_structs", os.path.join(HERE, "..", "paper_2402_15033_b200", "_capi.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


_S = _capi()
kry_solver_config, kry_report = _S.kry_solver_config, _S.kry_report
kry_append_outcome, kry_store_info = _S.kry_append_outcome, _S.kry_store_info

SIGS = {
    "kref_last_error": (C.c_char_p, []),
    "kref_last_pivot": (i64, []),
    "kref_laplace2d_size": (C.c_int, [i64, i64, C.c_int, P_i64, P_i64]),
    "kref_laplace2d": (C.c_int, [i64, i64, C.c_int, P_i64, P_i64, P_dbl]),
    "kref_laplace3d_size": (C.c_int, [i64, i64, i64, P_i64, P_i64]),
    "kref_laplace3d": (C.c_int, [i64, i64, i64, P_i64, P_i64, P_dbl]),
    "kref_gen_glued": (C.c_int, [i64, i64, i64, dbl, dbl, dbl, C.c_uint64, P_dbl]),
    "kref_gen_logscaled": (C.c_int, [i64, i64, dbl, C.c_uint64, P_dbl]),
    "kref_spmv": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl]),
    "kref_mpk": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, i64, P_dbl]),
    "kref_gram": (C.c_int, [i64, i64, P_dbl, P_dbl]),
    "kref_mat_mul_tn": (C.c_int, [i64, i64, P_dbl, i64, P_dbl, P_dbl]),
    "kref_try_cholesky": (C.c_int, [i64, P_dbl, P_dbl, P_i64]),
    "kref_tri_solve_right": (C.c_int, [i64, i64, P_dbl, P_dbl, P_dbl]),
    "kref_ortho_error": (C.c_int, [i64, i64, P_dbl, P_dbl]),
    "kref_bcgs_pip_partial": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_bcgs_pip": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_bcgs_pip2": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_cholqr": (C.c_int, [i64, P_dbl, i64, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_cholqr2": (C.c_int, [i64, P_dbl, i64, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_bcgs_project": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_i64]),
    "kref_bcgs2": (C.c_int, [i64, P_dbl, i64, P_dbl, i64, i32, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kref_householder_q": (C.c_int, [i64, i64, P_dbl, P_dbl]),
    "kref_store_create": (C.c_int, [i64, i64, i64, i64, C.POINTER(vp)]),
    "kref_store_destroy": (None, [vp]),
    "kref_store_reset": (C.c_int, [vp]),
    "kref_store_seed_unit_column": (C.c_int, [vp, P_dbl]),
    "kref_store_append_block": (C.c_int, [vp, P_dbl, i64, C.c_int, i32, i64, C.POINTER(kry_append_outcome), P_i64]),
    "kref_store_preprocess_block": (C.c_int, [vp, P_dbl, i64, C.c_int, C.POINTER(kry_append_outcome), P_i64]),
    "kref_store_finalize_big_panel": (C.c_int, [vp, C.POINTER(kry_append_outcome), P_i64]),
    "kref_store_get_info": (C.c_int, [vp, C.POINTER(kry_store_info)]),
    "kref_store_coefficients": (C.c_int, [vp, P_dbl]),
    "kref_store_columns": (C.c_int, [vp, i64, i64, P_dbl]),
    "kref_store_panel_states": (C.c_int, [vp, P_i32]),
    "kref_store_block_record": (C.c_int, [vp, i64, P_i64, P_i64, P_i32, P_dbl, P_dbl]),
    "kref_store_hessenberg": (C.c_int, [vp, i64, P_dbl]),
    "kref_hessenberg_lsq": (C.c_int, [i64, P_dbl, dbl, P_dbl, P_dbl, P_i64]),
    "kref_sstep_gmres": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl, C.POINTER(kry_solver_config),
                                   C.POINTER(kry_report), P_dbl]),
    "kref_standard_gmres": (C.c_int, [i64, P_i64, P_i64, P_dbl, P_dbl, P_dbl, C.POINTER(kry_solver_config),
                                      C.POINTER(kry_report), P_dbl]),
}

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def _load(path):
    L = C.CDLL(path)
    for k, (r, a) in SIGS.items():
        f = getattr(L, k)
        f.restype, f.argtypes = r, a
    return L


def lib():
    global _lib
    if _lib is None:
        if os.environ.get("KRY_REF_VARIANT") == "fma":  # rounding-envelope measurement only
            _lib = _load(os.path.join(HERE, "_ref", "libkrylov_ref_fma.so"))
            return _lib
        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref)")
        _lib = _load(REF_LIB)
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg, pivot=0):
        super().__init__(f"[{code}] {msg}")
        self.code, self.pivot = code, pivot


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().kref_last_error().decode(), lib().kref_last_pivot())


def _f(a, ndim=None):
    a = np.asfortranarray(a, dtype=np.float64)
    if ndim == 2 and a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(P_dbl)


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    def ptrs(self):
        return (self.row_ptr.ctypes.data_as(P_i64), self.col_idx.ctypes.data_as(P_i64),
                self.vals.ctypes.data_as(P_dbl))


def laplace2d(nx, ny, stencil=5) -> Csr:
    n, nnz = C.c_int64(), C.c_int64()
    _chk(lib().kref_laplace2d_size(nx, ny, stencil, C.byref(n), C.byref(nnz)))
    rp = np.zeros(n.value + 1, np.int64)
    ci = np.zeros(nnz.value, np.int64)
    v = np.zeros(nnz.value)
    _chk(lib().kref_laplace2d(nx, ny, stencil, rp.ctypes.data_as(P_i64), ci.ctypes.data_as(P_i64), _p(v)))
    return Csr(n.value, rp, ci, v)


def laplace3d(nx, ny, nz) -> Csr:
    n, nnz = C.c_int64(), C.c_int64()
    _chk(lib().kref_laplace3d_size(nx, ny, nz, C.byref(n), C.byref(nnz)))
    rp = np.zeros(n.value + 1, np.int64)
    ci = np.zeros(nnz.value, np.int64)
    v = np.zeros(nnz.value)
    _chk(lib().kref_laplace3d(nx, ny, nz, rp.ctypes.data_as(P_i64), ci.ctypes.data_as(P_i64), _p(v)))
    return Csr(n.value, rp, ci, v)


def gen_glued(n, p, s, kappa_panel, growth, coupling, seed) -> np.ndarray:
    out = np.zeros((n, p * s), order="F")
    _chk(lib().kref_gen_glued(n, p, s, kappa_panel, growth, coupling, seed, _p(out)))
    return out


def gen_logscaled(n, k, kappa, seed) -> np.ndarray:
    out = np.zeros((n, k), order="F")
    _chk(lib().kref_gen_logscaled(n, k, kappa, seed, _p(out)))
    return out


def spmv(a: Csr, x) -> np.ndarray:
    x = _f(x)
    y = np.zeros(a.n)
    _chk(lib().kref_spmv(a.n, *a.ptrs(), _p(x), _p(y)))
    return y


def mpk(a: Csr, start, s) -> np.ndarray:
    start = _f(start)
    out = np.zeros((a.n, s + 1), order="F")
    _chk(lib().kref_mpk(a.n, *a.ptrs(), _p(start), s, _p(out)))
    return out


def gram(v) -> np.ndarray:
    v = _f(v, 2)
    g = np.zeros((v.shape[1], v.shape[1]), order="F")
    _chk(lib().kref_gram(v.shape[0], v.shape[1], _p(v), _p(g)))
    return g


def mat_mul_tn(a, b) -> np.ndarray:
    a, b = _f(a, 2), _f(b, 2)
    c = np.zeros((a.shape[1], b.shape[1]), order="F")
    _chk(lib().kref_mat_mul_tn(a.shape[0], a.shape[1], _p(a), b.shape[1], _p(b), _p(c)))
    return c


def try_cholesky(s):
    s = _f(s, 2)
    k = s.shape[0]
    r = np.zeros((k, k), order="F")
    piv = C.c_int64()
    _chk(lib().kref_try_cholesky(k, _p(s), _p(r), C.byref(piv)))
    return r, piv.value


def ortho_error(q) -> float:
    q = _f(q, 2)
    e = C.c_double()
    _chk(lib().kref_ortho_error(q.shape[0], q.shape[1], _p(q), C.byref(e)))
    return e.value


def _pip(fn, q_prev, v):
    v = _f(v, 2)
    n, w = v.shape
    if q_prev is None or np.asarray(q_prev).size == 0:
        q, c0 = None, 0
    else:
        q = _f(q_prev, 2)
        c0 = q.shape[1]
    out = np.zeros((n, w), order="F")
    rc = np.zeros((c0, w), order="F")
    rj = np.zeros((w, w), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    code = fn(n, _p(q), c0, _p(v), w, _p(out), _p(rc), _p(rj), C.byref(piv), C.byref(red))
    return code, out, rc, rj, piv.value, red.value


def bcgs_pip(q_prev, v):
    code, q, rc, rj, piv, red = _pip(lib().kref_bcgs_pip, q_prev, v)
    if code:
        raise RefError(code, lib().kref_last_error().decode(), piv)
    return q, rc, rj, red


def bcgs_pip2(q_prev, v):
    code, q, rc, rj, piv, red = _pip(lib().kref_bcgs_pip2, q_prev, v)
    if code:
        raise RefError(code, lib().kref_last_error().decode(), piv)
    return q, rc, rj, red


def cholqr2(v):
    """cholqr2 (block_ortho.hpp:57): (q, r, reduces)."""
    v = _f(v, 2)
    n, w = v.shape
    q = np.zeros((n, w), order="F")
    r = np.zeros((w, w), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    code = lib().kref_cholqr2(n, _p(v), w, _p(q), _p(r), C.byref(piv), C.byref(red))
    if code:
        raise RefError(code, lib().kref_last_error().decode(), piv.value)
    return q, r, red.value


def bcgs_project(q_prev, v):
    """bcgs_project (block_ortho.hpp:70): (vhat, r_block, reduces)."""
    v = _f(v, 2)
    n, w = v.shape
    if q_prev is None or np.asarray(q_prev).size == 0:
        q, c0 = None, 0
    else:
        q = _f(q_prev, 2)
        c0 = q.shape[1]
    vhat = np.zeros((n, w), order="F")
    rb = np.zeros((c0, w), order="F")
    red = C.c_int64(0)
    _chk(lib().kref_bcgs_project(n, _p(q), c0, _p(v), w, _p(vhat), _p(rb), C.byref(red)))
    return vhat, rb, red.value


def bcgs2(q_prev, v, intra="cholqr2"):
    """bcgs2 (block_ortho.hpp:102): (q, r_col, r_jj, reduces)."""
    kind = {"hhqr": 0, "cholqr2": 1}[intra]
    code, q, rc, rj, piv, red = _pip(lambda n, qq, c0, vv, w, out, rcp, rjp, pv, rd:
                                     lib().kref_bcgs2(n, qq, c0, vv, w, kind, out, rcp, rjp, pv, rd), q_prev, v)
    if code:
        raise RefError(code, lib().kref_last_error().decode(), piv)
    return q, rc, rj, red


def bcgs_pip_partial(q_prev, v):
    code, q, rc, rj, piv, red = _pip(lib().kref_bcgs_pip_partial, q_prev, v)
    _chk(code)
    return q if piv == 0 else None, rc, rj, piv, red


class Store:
    """krylov::BasisStore through the shim (host, reference arithmetic)."""

    def __init__(self, n, m, s, shat):
        h = C.c_void_p()
        _chk(lib().kref_store_create(n, m, s, shat, C.byref(h)))
        self._h, self.n, self.m = h, n, m

    def __del__(self):
        if getattr(self, "_h", None):
            lib().kref_store_destroy(self._h)
            self._h = None

    def info(self):
        inf = kry_store_info()
        _chk(lib().kref_store_get_info(self._h, C.byref(inf)))
        return inf

    def append_block(self, v, overlap, kind, shat=0):
        v = _f(v, 2)
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().kref_store_append_block(self._h, _p(v), v.shape[1], int(overlap), int(kind), shat,
                                           C.byref(o), C.byref(d)))
        return o, d.value

    def preprocess_block(self, v, overlap):
        v = _f(v, 2)
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().kref_store_preprocess_block(self._h, _p(v), v.shape[1], int(overlap), C.byref(o), C.byref(d)))
        return o, d.value

    def finalize_big_panel(self):
        o, d = kry_append_outcome(), C.c_int64()
        _chk(lib().kref_store_finalize_big_panel(self._h, C.byref(o), C.byref(d)))
        return o, d.value

    def seed_unit_column(self, v):
        _chk(lib().kref_store_seed_unit_column(self._h, _p(_f(v))))

    def reset(self):
        _chk(lib().kref_store_reset(self._h))

    def coefficients(self):
        k = self.m + 1
        r = np.zeros((k, k), order="F")
        _chk(lib().kref_store_coefficients(self._h, _p(r)))
        return r

    def columns(self, first, count):
        out = np.zeros((self.n, count), order="F")
        if count:
            _chk(lib().kref_store_columns(self._h, first, count, _p(out)))
        return out

    def all(self):
        return self.columns(0, self.info().filled)

    def column(self, j):
        return self.columns(j, 1)[:, 0]

    def panel_states(self):
        k = self.info().n_panel_states
        st = np.zeros(max(k, 1), np.int32)
        _chk(lib().kref_store_panel_states(self._h, st.ctypes.data_as(P_i32)))
        return [int(s) for s in st[:k]]

    def block_records(self):
        out = []
        for i in range(self.info().n_records):
            c0, w, ov, diag = C.c_int64(), C.c_int64(), C.c_int32(), C.c_double()
            car = np.zeros(self.m + 2)
            _chk(lib().kref_store_block_record(self._h, i, C.byref(c0), C.byref(w), C.byref(ov), _p(car),
                                               C.byref(diag)))
            out.append((c0.value, w.value, bool(ov.value), car[: c0.value].copy() if ov.value else np.zeros(0),
                        diag.value))
        return out

    def hessenberg(self, k):
        h = np.zeros((k + 1, k), order="F")
        _chk(lib().kref_store_hessenberg(self._h, k, _p(h)))
        return h


@dataclass
class RefReport:
    status: int
    iterations: int
    restarts: int
    initial_residual: float
    final_relative_residual: float
    cycle_residuals: List[float]
    breakdown: bool
    breakdown_kappa: float
    reduces: int
    per_block: List[int]
    per_big_panel: List[int]
    reduces_per_iteration: float
    wall_seconds: float
    solution: Optional[np.ndarray] = field(default=None, repr=False)


def make_config(m=60, s=5, big_step=0, kind=2, shat=0, rel_tol=1e-6, max_iters=500000):
    c = kry_solver_config()
    c.restart_len, c.step, c.big_step = m, s, big_step
    c.scheme_kind, c.scheme_big_panel_size = kind, shat
    c.rel_tol, c.max_iters = rel_tol, max_iters
    return c


def solve(a: Csr, b, x0, cfg, standard=False, cap=200000) -> RefReport:
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
    fn = lib().kref_standard_gmres if standard else lib().kref_sstep_gmres
    _chk(fn(a.n, *a.ptrs(), _p(b), _p(x0a), C.byref(cfg), C.byref(rep), _p(x)))
    return RefReport(rep.status, rep.iterations, rep.restarts, rep.initial_residual,
                     rep.final_relative_residual, list(cyc[: rep.n_cycle_residuals]), bool(rep.breakdown),
                     rep.breakdown_kappa, rep.reduces, list(pb[: rep.n_per_block]),
                     list(pbp[: rep.n_per_big_panel]), rep.reduces_per_iteration, rep.wall_seconds, x)
