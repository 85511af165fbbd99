"""B200-native hot path of s-step GMRES with two-stage block orthogonalization.

Python mirror of the reference's C++ API (/root/reference/proj/include/krylov)
over the C ABI of include/krylov_b200.h — the same names, argument meaning
and error behaviour, so the parity tests read like the reference's own
(tests/test_block_ortho.cpp, test_sparse_core.cpp).  Everything computes on
the GPU through libkrylov_b200.so; there is no CPU fallback.

    reference (krylov::)                 here
    ---------------------------------    ---------------------------------
    sstep_gmres  gmres.hpp:396           sstep_gmres(op, b, x0, cfg)
    standard_gmres gmres.hpp:404         standard_gmres(op, b, x0, cfg)
    bcgs_pip / _partial / 2, cholqr      bcgs_pip(...), ... (block_ortho.hpp)
    BasisStore  basis_store.hpp:42       BasisStore(n, m, s, ŝ)
    spmv / mpk_monomial                  Operator.spmv / Operator.mpk
    CsrMatrix / gen_laplace2d/3d         CsrOperator / Laplace2D / Laplace3D
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import (P_dbl, P_i32, P_i64, kry_append_outcome, kry_report, kry_solver_config,
                    kry_store_info)

__all__ = [
    "KrylovError", "DimensionMismatch", "NotPositiveDefinite", "SingularFactor", "SingularR",
    "Unsupported", "DeviceError", "OrthoKind", "SolveStatus", "PanelState", "OrthoScheme",
    "SolverConfig", "SyncCounter", "AppendOutcome", "BlockRecord", "SolveReport", "Context",
    "cholqr2", "bcgs_project", "bcgs2",
    "get_context", "CsrOperator", "Laplace2D", "Laplace3D", "BasisStore", "bcgs_pip",
    "bcgs_pip_partial", "bcgs_pip2", "cholqr", "gram", "gram_full", "try_cholesky",
    "solve_hessenberg_lsq", "sstep_gmres", "standard_gmres", "sstep_gmres_device", "lib",
]

lib = _capi.lib


# ---- errors (types.hpp) ------------------------------------------------------
class KrylovError(RuntimeError):
    pass


class DimensionMismatch(KrylovError, ValueError):
    pass


class NotPositiveDefinite(KrylovError):
    def __init__(self, msg, pivot):
        super().__init__(msg)
        self.pivot = int(pivot)


class SingularFactor(KrylovError):
    pass


class SingularR(KrylovError):
    def __init__(self, msg, column):
        super().__init__(msg)
        self.column = int(column)


class Unsupported(KrylovError):
    pass


class DeviceError(KrylovError):
    pass


def _check(rc: int, aux: int = 0) -> None:
    if rc == _capi.KRY_OK:
        return
    msg = lib().kry_last_error().decode(errors="replace")
    if rc == _capi.KRY_DIMENSION_MISMATCH:
        raise DimensionMismatch(msg)
    if rc == _capi.KRY_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefinite(msg, aux)
    if rc == _capi.KRY_SINGULAR_FACTOR:
        raise SingularFactor(msg)
    if rc == _capi.KRY_SINGULAR_R:
        raise SingularR(msg, aux)
    if rc == _capi.KRY_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == _capi.KRY_UNSUPPORTED:
        raise Unsupported(msg)
    raise DeviceError(f"{lib().kry_status_name(rc).decode()}: {msg}")


# ---- enums and value types (block_ortho.hpp, basis_store.hpp, gmres.hpp) -------
class OrthoKind(enum.IntEnum):
    BCGS2_HHQR = 0
    BCGS2_CHOLQR2 = 1
    BCGS_PIP2 = 2
    TWO_STAGE = 3


class SolveStatus(enum.IntEnum):
    CONVERGED = 0
    MAX_ITERS = 1
    ORTHO_BREAKDOWN = 2
    STAGNATION = 3


class PanelState(enum.IntEnum):
    RAW = 0
    PREPROCESSED = 1
    FINAL = 2


@dataclass
class OrthoScheme:
    kind: OrthoKind = OrthoKind.BCGS_PIP2
    big_panel_size: int = 0


@dataclass
class SolverConfig:
    restart_len: int = 60
    step: int = 5
    big_step: int = 0
    scheme: OrthoScheme = field(default_factory=OrthoScheme)
    rel_tol: float = 1e-6
    max_iters: int = 500000

    def effective_big_step(self) -> int:
        return self.restart_len if self.big_step == 0 else self.big_step

    def to_c(self) -> kry_solver_config:
        c = kry_solver_config()
        c.restart_len, c.step, c.big_step = self.restart_len, self.step, self.big_step
        c.scheme_kind = int(self.scheme.kind)
        c.scheme_big_panel_size = self.scheme.big_panel_size
        c.rel_tol, c.max_iters = self.rel_tol, self.max_iters
        return c


@dataclass
class SyncCounter:
    reduces: int = 0
    per_block: List[int] = field(default_factory=list)
    per_big_panel: List[int] = field(default_factory=list)

    def add(self, k: int = 1) -> None:
        self.reduces += k


@dataclass
class AppendOutcome:
    committed: int = 0
    truncated: bool = False
    breakdown: bool = False
    pivot: int = 0
    kappa_estimate: float = 0.0


@dataclass
class BlockRecord:
    c0: int
    width: int
    overlap: bool
    carried: np.ndarray
    carried_diag: float


@dataclass
class BlockOrthoResult:
    q: np.ndarray
    r_col: np.ndarray
    r_jj: np.ndarray


@dataclass
class PipOutcome:
    r_col: np.ndarray
    r_chol: np.ndarray
    q: Optional[np.ndarray]
    bad_pivot: int


@dataclass
class BlockQr:
    q: np.ndarray
    r: np.ndarray


@dataclass
class SolveReport:
    status: SolveStatus
    iterations: int
    restarts: int
    initial_residual: float
    final_relative_residual: float
    cycle_residuals: List[float]
    breakdown: bool
    breakdown_kappa: float
    sync: SyncCounter
    reduces_per_iteration: float
    wall_seconds: float
    solution: Optional[np.ndarray]
    telemetry: dict


# ---- helpers -------------------------------------------------------------------
def _f64(a, ndim=None) -> np.ndarray:
    a = np.asfortranarray(a, dtype=np.float64)
    if ndim == 2 and a.ndim == 1:
        a = a.reshape(-1, 1, order="F")
    return a


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(P_dbl)


def _report_cap(cfg: "SolverConfig", standard: bool = False) -> int:
    """History entries a solve can produce: one per-block entry per s
    iterations (plus truncation retries), at most one cycle per s iterations."""
    step = 1 if standard else max(1, cfg.step)
    return 2 * (min(cfg.max_iters, 1 << 40) // step) + 64


def _report_from_c(rep: kry_report, cyc, pb, pbp, solution) -> SolveReport:
    n1, n2, n3 = rep.n_cycle_residuals, rep.n_per_block, rep.n_per_big_panel
    if n1 > len(cyc) or n2 > len(pb) or n3 > len(pbp):  # never truncate the history silently
        raise KrylovError(f"report history overflow ({n1}/{n2}/{n3} entries, capacity {len(cyc)})")
    tel = {k: getattr(rep, k) for k in (
        "mpk_seconds", "ortho_seconds", "gram_kernel_seconds", "update_kernel_seconds",
        "restart_seconds", "mpk_bytes", "ortho_bytes", "gram_bytes", "update_bytes",
        "gram_launches", "update_launches", "gpu_launches", "allreduces",
        "fused_kernel_seconds", "fused_bytes", "fused_launches")}
    return SolveReport(
        status=SolveStatus(rep.status), iterations=rep.iterations, restarts=rep.restarts,
        initial_residual=rep.initial_residual, final_relative_residual=rep.final_relative_residual,
        cycle_residuals=list(cyc[:n1]), breakdown=bool(rep.breakdown),
        breakdown_kappa=rep.breakdown_kappa,
        sync=SyncCounter(rep.reduces, [int(v) for v in pb[:n2]], [int(v) for v in pbp[:n3]]),
        reduces_per_iteration=rep.reduces_per_iteration, wall_seconds=rep.wall_seconds,
        solution=solution, telemetry=tel)


def _new_report(cap=200000):
    rep = kry_report()
    cyc = np.zeros(cap, dtype=np.float64)
    pb = np.zeros(cap, dtype=np.int64)
    pbp = np.zeros(cap, dtype=np.int64)
    rep.cycle_residuals, rep.cycle_residuals_cap = cyc.ctypes.data_as(P_dbl), cap
    rep.per_block, rep.per_block_cap = pb.ctypes.data_as(P_i64), cap
    rep.per_big_panel, rep.per_big_panel_cap = pbp.ctypes.data_as(P_i64), cap
    return rep, cyc, pb, pbp


# ---- context ---------------------------------------------------------------------
class Context:
    """One GPU + stream (+ NCCL communicator when nranks > 1)."""

    def __init__(self, device: int = 0, nranks: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None):
        h = C.c_void_p()
        idbuf = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        _check(lib().kry_ctx_create(device, nranks, rank, idbuf, C.byref(h)))
        self._h = h
        self.device, self.nranks, self.rank = device, nranks, rank

    @property
    def handle(self):
        return self._h

    def set_timing(self, on: bool) -> None:
        _check(lib().kry_ctx_set_timing(self._h, int(bool(on))))

    def synchronize(self) -> None:
        _check(lib().kry_ctx_synchronize(self._h))

    def stream_handle(self) -> int:
        """cudaStream_t (as an integer) all kernels of this context run on."""
        v = C.c_void_p()
        _check(lib().kry_ctx_stream(self._h, C.byref(v)))
        return v.value or 0

    def launch_count(self) -> int:
        v = C.c_int64()
        _check(lib().kry_ctx_launch_count(self._h, C.byref(v)))
        return v.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().kry_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        n = lib().kry_nccl_unique_id_size()
        buf = C.create_string_buffer(n)
        _check(lib().kry_nccl_get_unique_id(buf))
        return buf.raw


_default_ctx: Optional[Context] = None


def get_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def device_count() -> int:
    n = C.c_int()
    lib().kry_device_count(C.byref(n))
    return n.value


# ---- operators (csr_matrix.hpp, matgen.hpp) ------------------------------------------
class Operator:
    _h = None

    def __init__(self, ctx: Optional[Context]):
        self.ctx = ctx or get_context()

    def _rows(self):
        ng, rb, nl = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().kry_operator_rows(self._h, C.byref(ng), C.byref(rb), C.byref(nl)))
        self.n_global, self.row_begin, self.n = ng.value, rb.value, nl.value

    @property
    def handle(self):
        return self._h

    def spmv(self, x) -> np.ndarray:
        """y = A·x for this rank's rows (spmv, csr_matrix.hpp:69)."""
        x = _f64(x)
        if x.shape != (self.n,):
            raise DimensionMismatch("dimension mismatch: spmv vector length")
        y = np.empty(self.n, dtype=np.float64)
        _check(lib().kry_spmv(self.ctx.handle, self._h, _p(x), _p(y)))
        return y

    def mpk(self, start, s: int) -> np.ndarray:
        """mpk_monomial (gmres.hpp:80-90): n×(s+1), column 0 = start."""
        start = _f64(start)
        if start.shape != (self.n,):
            raise DimensionMismatch("dimension mismatch: mpk start vector length")
        v = np.empty((self.n, s + 1), dtype=np.float64, order="F")
        _check(lib().kry_mpk(self.ctx.handle, self._h, _p(start), s, _p(v)))
        return v

    def jacobi(self) -> "Operator":
        """Left Jacobi preconditioning on the device: from now on this operator
        is D⁻¹A and solves take the original b (kry_operator_jacobi)."""
        _check(lib().kry_operator_jacobi(self._h))
        return self

    @property
    def is_jacobi(self) -> bool:
        e = C.c_int()
        _check(lib().kry_operator_is_jacobi(self._h, C.byref(e)))
        return bool(e.value)

    def close(self):
        if self._h:
            lib().kry_operator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CsrOperator(Operator):
    """CSR rows [row_begin, row_begin+n_local) of an n_global×n_global matrix."""

    def __init__(self, row_ptr, col_idx, vals, n_global: Optional[int] = None, row_begin: int = 0,
                 ctx: Optional[Context] = None):
        super().__init__(ctx)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        vv = np.ascontiguousarray(vals, dtype=np.float64)
        n_local = rp.shape[0] - 1
        if n_global is None:
            n_global = n_local
        h = C.c_void_p()
        _check(lib().kry_operator_create_csr(self.ctx.handle, n_global, row_begin, n_local,
                                             rp.ctypes.data_as(P_i64), ci.ctypes.data_as(P_i64),
                                             vv.ctypes.data_as(P_dbl), C.byref(h)))
        self._h = h
        self._rows()
        self.nnz = int(rp[-1])


def gen_random_sparse(n_global: int, row_begin: int = 0, n_local: Optional[int] = None, per_row: int = 30,
                      seed: int = 1, diag_factor: float = 0.15, jacobi: bool = False):
    """BASELINE configs[4] rows on the host (kry_gen_random_sparse): int64
    row_ptr (from 0), int64 global columns, fp64 values."""
    n_local = n_global - row_begin if n_local is None else n_local
    rp = np.empty(n_local + 1, dtype=np.int64)
    ci = np.empty(n_local * per_row, dtype=np.int64)
    vv = np.empty(n_local * per_row, dtype=np.float64)
    _check(lib().kry_gen_random_sparse(n_global, row_begin, n_local, per_row, seed, diag_factor, int(jacobi),
                                       rp.ctypes.data_as(P_i64), ci.ctypes.data_as(P_i64),
                                       vv.ctypes.data_as(P_dbl)))
    return rp, ci, vv


class Laplace2D(Operator):
    """Matrix-free gen_laplace2d(nx, ny, 5) (matgen.hpp:134-164)."""

    def __init__(self, nx: int, ny: int, ctx: Optional[Context] = None):
        super().__init__(ctx)
        h = C.c_void_p()
        _check(lib().kry_operator_create_laplace2d(self.ctx.handle, nx, ny, C.byref(h)))
        self._h = h
        self.nx, self.ny = nx, ny
        self._rows()


class Laplace3D(Operator):
    """Matrix-free gen_laplace3d(nx, ny, nz) (matgen.hpp:167-187)."""

    def __init__(self, nx: int, ny: int, nz: int, ctx: Optional[Context] = None):
        super().__init__(ctx)
        h = C.c_void_p()
        _check(lib().kry_operator_create_laplace3d(self.ctx.handle, nx, ny, nz, C.byref(h)))
        self._h = h
        self.nx, self.ny, self.nz = nx, ny, nz
        self._rows()


# ---- block orthogonalization (block_ortho.hpp) -------------------------------------------
def _prefix(q_prev, n):
    if q_prev is None:
        return None, 0
    q = _f64(q_prev, 2)
    if q.shape[1] == 0:
        return None, 0
    if q.shape[0] != n:
        raise DimensionMismatch("dimension mismatch: prefix rows")
    return q, q.shape[1]


def gram(q_prev, v, ctx: Optional[Context] = None):
    """[Q_prev V]ᵀV on the device: (Q_prevᵀV, VᵀV)."""
    ctx = ctx or get_context()
    v = _f64(v, 2)
    n, w = v.shape
    q, c0 = _prefix(q_prev, n)
    rc = np.zeros((c0, w), order="F")
    g = np.zeros((w, w), order="F")
    _check(lib().kry_gram(ctx.handle, n, _p(q), c0, _p(v), w, _p(rc), _p(g)))
    return rc, g


def gram_full(q, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or get_context()
    q = _f64(q, 2)
    g = np.zeros((q.shape[1], q.shape[1]), order="F")
    _check(lib().kry_gram_full(ctx.handle, q.shape[0], _p(q), q.shape[1], _p(g)))
    return g


def bcgs_pip_partial(q_prev, v, sync: SyncCounter, ctx: Optional[Context] = None) -> PipOutcome:
    ctx = ctx or get_context()
    v = _f64(v, 2)
    n, w = v.shape
    q, c0 = _prefix(q_prev, n)
    out = np.zeros((n, w), order="F")
    rc = np.zeros((c0, w), order="F")
    rj = np.zeros((w, w), order="F")
    bad, red = C.c_int64(0), C.c_int64(0)
    _check(lib().kry_bcgs_pip_partial(ctx.handle, n, _p(q), c0, _p(v), w, _p(out), _p(rc), _p(rj),
                                      C.byref(bad), C.byref(red)))
    sync.add(red.value)
    return PipOutcome(rc, rj, out if bad.value == 0 else None, bad.value)


def _pip_call(fn, q_prev, v, sync, ctx):
    ctx = ctx or get_context()
    v = _f64(v, 2)
    n, w = v.shape
    q, c0 = _prefix(q_prev, n)
    out = np.zeros((n, w), order="F")
    rc = np.zeros((c0, w), order="F")
    rj = np.zeros((w, w), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    rc_code = fn(ctx.handle, n, _p(q), c0, _p(v), w, _p(out), _p(rc), _p(rj), C.byref(piv), C.byref(red))
    sync.add(red.value)
    _check(rc_code, piv.value)
    return BlockOrthoResult(out, rc, rj)


def bcgs_pip(q_prev, v, sync: SyncCounter, ctx: Optional[Context] = None) -> BlockOrthoResult:
    """bcgs_pip (block_ortho.hpp:180): raises NotPositiveDefinite(pivot)."""
    return _pip_call(lib().kry_bcgs_pip, q_prev, v, sync, ctx)


def bcgs_pip2(q_prev, v, sync: SyncCounter, ctx: Optional[Context] = None) -> BlockOrthoResult:
    """bcgs_pip2 (block_ortho.hpp:192): two reduces."""
    return _pip_call(lib().kry_bcgs_pip2, q_prev, v, sync, ctx)


def cholqr(v, sync: SyncCounter, ctx: Optional[Context] = None) -> BlockQr:
    """cholqr (block_ortho.hpp:49): one reduce."""
    r = bcgs_pip(None, v, sync, ctx)
    return BlockQr(r.q, r.r_jj)


def cholqr2(v, sync: SyncCounter, ctx: Optional[Context] = None) -> BlockQr:
    """cholqr2 (block_ortho.hpp:57): CholQR twice, R = R2·R1; two reduces."""
    ctx = ctx or get_context()
    v = _f64(v, 2)
    n, w = v.shape
    q = np.zeros((n, w), order="F")
    r = np.zeros((w, w), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    rc = lib().kry_cholqr2(ctx.handle, n, _p(v), w, _p(q), _p(r), C.byref(piv), C.byref(red))
    sync.add(red.value)
    _check(rc, piv.value)
    return BlockQr(q, r)


def bcgs_project(q_prev, v, sync: SyncCounter, ctx: Optional[Context] = None):
    """bcgs_project (block_ortho.hpp:70): (vhat, r_block); one reduce (none for an empty prefix)."""
    ctx = ctx or get_context()
    v = _f64(v, 2)
    n, w = v.shape
    q, c0 = _prefix(q_prev, n)
    vhat = np.zeros((n, w), order="F")
    rb = np.zeros((c0, w), order="F")
    red = C.c_int64(0)
    _check(lib().kry_bcgs_project(ctx.handle, n, _p(q), c0, _p(v), w, _p(vhat), _p(rb), C.byref(red)))
    sync.add(red.value)
    return vhat, rb


def bcgs2(q_prev, v, sync: SyncCounter, intra: str = "cholqr2", ctx: Optional[Context] = None) -> BlockOrthoResult:
    """bcgs2 (block_ortho.hpp:102): project, intra (CholQR2; 'hhqr' is not on
    the device path for blocks wider than one column), re-project, CholQR."""
    kind = {"hhqr": 0, "cholqr2": 1}[intra]
    return _pip_call(lambda h, n, q, c0, vv, w, out, rc, rj, piv, red:
                     lib().kry_bcgs2(h, n, q, c0, vv, w, kind, out, rc, rj, piv, red), q_prev, v, sync, ctx)


def try_cholesky(s):
    """try_cholesky (dense_kernels.hpp:111): (R, pivot) — host arithmetic of the library."""
    s = _f64(s, 2)
    k = s.shape[0]
    r = np.zeros((k, k), order="F")
    piv = C.c_int64()
    _check(lib().kry_try_cholesky(k, _p(s), _p(r), C.byref(piv)))
    return r, piv.value


def solve_hessenberg_lsq(h, gamma: float):
    """solve_hessenberg_lsq (gmres.hpp:146): (y, implicit_residual, valid_cols)."""
    h = _f64(h, 2)
    k = h.shape[1]
    y = np.zeros(max(k, 1))
    imp, valid = C.c_double(), C.c_int64()
    _check(lib().kry_hessenberg_lsq(k, _p(h), gamma, _p(y), C.byref(imp), C.byref(valid)))
    return y[: valid.value], imp.value, valid.value


# ---- basis store (basis_store.hpp) ----------------------------------------------------------
class BasisStore:
    """Device-resident krylov::BasisStore(n, m, panel_size, big_panel_size)."""

    def __init__(self, n: int, m: int, panel_size: int, big_panel_size: int, ctx: Optional[Context] = None):
        self.ctx = ctx or get_context()
        h = C.c_void_p()
        _check(lib().kry_store_create(self.ctx.handle, n, m, panel_size, big_panel_size, C.byref(h)))
        self._h = h
        self.n, self.m = n, m

    def close(self):
        if getattr(self, "_h", None):
            lib().kry_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _info(self) -> kry_store_info:
        info = kry_store_info()
        _check(lib().kry_store_get_info(self._h, C.byref(info)))
        return info

    def rows(self): return self._info().rows
    def capacity(self): return self._info().capacity
    def filled(self): return self._info().filled
    def finalized_count(self): return self._info().finalized
    def big_panel_start(self): return self._info().big_panel_start
    def panel_size(self): return self._info().panel_size
    def big_panel_size(self): return self._info().big_panel_size
    def has_seam_column(self): return bool(self._info().seam_valid)
    def big_panel_open(self): return bool(self._info().big_panel_open)
    def big_panel_full(self): return bool(self._info().big_panel_full)

    @staticmethod
    def _outcome(o: kry_append_outcome) -> AppendOutcome:
        return AppendOutcome(o.committed, bool(o.truncated), bool(o.breakdown), o.pivot, o.kappa_estimate)

    def append_block(self, v, overlap: bool, scheme: OrthoScheme, sync: SyncCounter) -> AppendOutcome:
        v = _f64(v, 2)
        if v.shape[0] != self.n:
            raise DimensionMismatch("dimension mismatch: block row count")
        o, d = kry_append_outcome(), C.c_int64()
        _check(lib().kry_store_append_block(self._h, _p(v), v.shape[1], int(overlap), int(scheme.kind),
                                            scheme.big_panel_size, C.byref(o), C.byref(d)))
        sync.add(d.value)
        sync.per_block.append(d.value)
        return self._outcome(o)

    def preprocess_block(self, v, overlap: bool, sync: SyncCounter) -> AppendOutcome:
        return self.append_block(v, overlap, OrthoScheme(OrthoKind.TWO_STAGE, self.big_panel_size()), sync)

    def finalize_big_panel(self, sync: SyncCounter) -> AppendOutcome:
        info = self._info()
        o, d = kry_append_outcome(), C.c_int64()
        _check(lib().kry_store_finalize_big_panel(self._h, C.byref(o), C.byref(d)))
        if info.filled > info.big_panel_start:  # the reference records a delta only for an open panel
            sync.add(d.value)
            sync.per_big_panel.append(d.value)
        return self._outcome(o)

    def mpk(self, op: Operator, start, c0: int, s: int) -> None:
        sp = None if start is None else _f64(start)
        _check(lib().kry_store_mpk(self._h, op.handle, _p(sp), c0, s))

    def append_inplace(self, w: int, overlap: bool, scheme: OrthoScheme, sync: SyncCounter) -> AppendOutcome:
        o, d = kry_append_outcome(), C.c_int64()
        _check(lib().kry_store_append_inplace(self._h, w, int(overlap), int(scheme.kind),
                                              scheme.big_panel_size, C.byref(o), C.byref(d)))
        sync.add(d.value)
        sync.per_block.append(d.value)
        return self._outcome(o)

    def reset(self):
        _check(lib().kry_store_reset(self._h))

    def seed_unit_column(self, v):
        _check(lib().kry_store_seed_unit_column(self._h, _p(_f64(v))))

    def coefficients(self) -> np.ndarray:
        k = self.m + 1
        r = np.zeros((k, k), order="F")
        _check(lib().kry_store_coefficients(self._h, _p(r)))
        return r

    def columns(self, first: int, count: int) -> np.ndarray:
        out = np.zeros((self.n, count), order="F")
        if count:
            _check(lib().kry_store_columns(self._h, first, count, _p(out)))
        return out

    def column(self, j: int) -> np.ndarray:
        return self.columns(j, 1)[:, 0]

    def all(self) -> np.ndarray:
        return self.columns(0, self.filled())

    def finalized(self) -> np.ndarray:
        return self.columns(0, self.finalized_count())

    def panel_states(self) -> List[PanelState]:
        n = self._info().n_panel_states
        st = np.zeros(max(n, 1), dtype=np.int32)
        _check(lib().kry_store_panel_states(self._h, st.ctypes.data_as(P_i32)))
        return [PanelState(int(s)) for s in st[:n]]

    def block_records(self) -> List[BlockRecord]:
        out = []
        for i in range(self._info().n_records):
            c0, w, ov, diag = C.c_int64(), C.c_int64(), C.c_int32(), C.c_double()
            carried = np.zeros(self.m + 2)
            _check(lib().kry_store_block_record(self._h, i, C.byref(c0), C.byref(w), C.byref(ov), _p(carried),
                                                C.byref(diag)))
            out.append(BlockRecord(c0.value, w.value, bool(ov.value),
                                   carried[: c0.value].copy() if ov.value else np.zeros(0), diag.value))
        return out

    def hessenberg(self, k: int) -> np.ndarray:
        h = np.zeros((k + 1, k), order="F")
        col = C.c_int64()
        _check(lib().kry_store_hessenberg(self._h, k, _p(h), C.byref(col)), col.value)
        return h


# ---- solvers (gmres.hpp) ---------------------------------------------------------------
def _solve(fn, op: Operator, b, x0, cfg: SolverConfig, want_solution=True) -> SolveReport:
    b = _f64(b)
    if b.shape != (op.n,):
        raise DimensionMismatch("dimension mismatch: rhs length")
    x0a = None
    if x0 is not None and len(x0) > 0:
        x0a = _f64(x0)
        if x0a.shape != (op.n,):
            raise DimensionMismatch("dimension mismatch: x0 length")
    x = np.zeros(op.n) if want_solution else None
    rep, cyc, pb, pbp = _new_report(_report_cap(cfg, fn == lib().kry_standard_gmres))
    c = cfg.to_c()
    _check(fn(op.ctx.handle, op.handle, _p(b), _p(x0a), C.byref(c), C.byref(rep), _p(x)))
    return _report_from_c(rep, cyc, pb, pbp, x)


def sstep_gmres(op: Operator, b, x0, cfg: SolverConfig) -> SolveReport:
    """sstep_gmres (gmres.hpp:396): host vectors in, host solution out."""
    return _solve(lib().kry_sstep_gmres, op, b, x0, cfg)


def standard_gmres(op: Operator, b, x0, cfg: SolverConfig) -> SolveReport:
    """standard_gmres (gmres.hpp:404): s = 1, BCGS2-CholQR2 (CGS2)."""
    return _solve(lib().kry_standard_gmres, op, b, x0, cfg)


def _solve_device(fn, op: Operator, d_b: int, d_x0: Optional[int], cfg: SolverConfig,
                  d_x_out: Optional[int]) -> SolveReport:
    rep, cyc, pb, pbp = _new_report(_report_cap(cfg, fn == lib().kry_standard_gmres_device))
    c = cfg.to_c()
    _check(fn(op.ctx.handle, op.handle, C.c_void_p(d_b), C.c_void_p(d_x0) if d_x0 else None, C.byref(c),
              C.byref(rep), C.c_void_p(d_x_out) if d_x_out else None))
    return _report_from_c(rep, cyc, pb, pbp, None)


def sstep_gmres_device(op: Operator, d_b: int, d_x0: Optional[int], cfg: SolverConfig,
                       d_x_out: Optional[int] = None) -> SolveReport:
    """Inputs already resident in HBM (raw device pointers, e.g. tensor.data_ptr())."""
    return _solve_device(lib().kry_sstep_gmres_device, op, d_b, d_x0, cfg, d_x_out)


def standard_gmres_device(op: Operator, d_b: int, d_x0: Optional[int], cfg: SolverConfig,
                          d_x_out: Optional[int] = None) -> SolveReport:
    """standard_gmres (gmres.hpp:404) with inputs resident in HBM."""
    return _solve_device(lib().kry_standard_gmres_device, op, d_b, d_x0, cfg, d_x_out)
