"""Preconditioners on the device (mirror of src/precond.py).

Jacobi (src/precond.py:77-95): z = r * inv_diag.  For the cavity operator
the diagonal is the constant 6/h^2, so the fused CG forms z in registers
from r (no extra HBM pass) -- ``JacobiPreconditioner.constant`` carries the
scalar when every entry is equal.

DIC (src/precond.py:98-151): the simplified diagonal-based incomplete
Cholesky.  Its recurrence and sweeps are sequential by row; on the device
they run as level-scheduled sweeps (rows grouped by dependency depth; for
the 7-point operator a level is a hyperplane i+j+k = const), each row
evaluated with the reference's operand order, so the preconditioner and
its iteration counts are the reference's.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .grid import as_device, to_host
from .sparse import CsrMatrix, SymCsrMatrix, StencilOperator, _as_f64, _as_i64


class JacobiPreconditioner:
    """Reciprocal-diagonal scaling (src/precond.py:77-95)."""

    kind = "jacobi"

    def __init__(self, inv_diag):
        self.inv_diag, _ = as_device(inv_diag)
        self.inv_diag = self.inv_diag.contiguous()
        # constant diagonal (the cavity operator) -> the fused CG forms z in registers
        n = self.inv_diag.shape[0]
        first = self.inv_diag[:1]
        self.constant = (float(first.item()) if n and bool(torch.all(self.inv_diag == first).item()) else None)

    @property
    def n(self) -> int:
        return self.inv_diag.shape[0]

    def apply(self, r, out=None):
        rd, host = as_device(r)
        if rd.shape[0] != self.n:
            raise ValueError(f"preconditioner has dimension {self.n}, vector {rd.shape[0]}")
        y = torch.empty_like(rd) if out is None or not isinstance(out, torch.Tensor) else out
        lib = _lib.load_library()
        _lib.check(lib.cf_mul(rd.contiguous().data_ptr(), self.inv_diag.data_ptr(), y.data_ptr(), self.n,
                              _lib.stream()), "jacobi apply")
        if out is not None and not isinstance(out, torch.Tensor):
            out[...] = to_host(y)
            return out
        return to_host(y) if host and out is None else y


def _diag_of(a) -> np.ndarray:
    if isinstance(a, SymCsrMatrix):
        return a.diag
    if isinstance(a, (CsrMatrix, StencilOperator)):
        return a.diagonal()
    raise TypeError(f"unsupported matrix type {type(a).__name__}")


def jacobi_from(a) -> JacobiPreconditioner:
    """src/precond.py:127-138."""
    diag = _diag_of(a)
    zero = np.flatnonzero(diag == 0.0)
    if len(zero):
        raise ValueError(f"zero diagonal entry at row {zero[0]}")
    return JacobiPreconditioner(1.0 / diag)


def _triangles(a):
    """Strict lower / upper triangles (int64 CSR), diagonal, n (src/precond.py:57-74)."""
    if isinstance(a, SymCsrMatrix):
        lower = (a.t_row_ptr, a.t_col_idx, a.lower_values())
        return lower, a.diag.copy(), (a.row_ptr, a.col_idx, a.values), a.n
    if isinstance(a, CsrMatrix):
        if a.n_rows != a.n_cols:
            raise ValueError(f"matrix must be square, got {a.shape}")
        rows = a.row_indices()
        parts = []
        for m in (a.col_idx < rows, a.col_idx > rows):
            ptr = np.concatenate(([0], np.cumsum(np.bincount(rows[m], minlength=a.n_rows)))).astype(np.int64)
            parts.append((ptr, _as_i64(a.col_idx[m]), _as_f64(a.values[m])))
        return parts[0], a.diagonal(), parts[1], a.n_rows
    if isinstance(a, StencilOperator):
        # the 7-point pattern generated directly (lower: k-1, j-1, i-1; upper:
        # i+1, j+1, k+1 -- ascending columns, as the CSR triangles would be)
        nx, ny, nz, num = a.nx, a.ny, a.nz, a.num
        idx = np.arange(num, dtype=np.int64)
        i, j, k = idx % nx, (idx // nx) % ny, idx // (nx * ny)
        off = -1.0 / (a.h * a.h)
        pl = nx * ny
        out = []
        for cols, mask in (((idx - pl, idx - nx, idx - 1), (k > 0, j > 0, i > 0)),
                           ((idx + 1, idx + nx, idx + pl), (i < nx - 1, j < ny - 1, k < nz - 1))):
            c = np.stack(cols, axis=1)
            m = np.stack(mask, axis=1)
            ptr = np.concatenate(([0], np.cumsum(m.sum(axis=1)))).astype(np.int64)
            cc = c.ravel()[m.ravel()]
            out.append((ptr, cc, np.full(len(cc), off)))
        return out[0], a.diagonal(), out[1], num
    raise TypeError(f"unsupported matrix type {type(a).__name__}")


def _levels(a, lower, n):
    """Level of every row: 1 + max level of its lower columns."""
    if isinstance(a, StencilOperator):
        idx = np.arange(n, dtype=np.int64)
        return (idx % a.nx + (idx // a.nx) % a.ny + idx // (a.nx * a.ny)).astype(np.int32)
    lib = _lib.host_library()
    lv = np.empty(n, dtype=np.int32)
    nl = np.zeros(1, dtype=np.int32)
    _lib.check(lib.cf_level_schedule(n, lower[0].ctypes.data, lower[1].ctypes.data, lv.ctypes.data,
                                     nl.ctypes.data), "level schedule")
    return lv


class DicPreconditioner:
    """Simplified DIC over the fixed pattern (src/precond.py:98-124), on the
    device by level-scheduled sweeps with the reference's per-row order."""

    kind = "dic"

    def __init__(self, lower, diag, upper, n, levels):
        from .sparse import _i32_dev

        self.n = int(n)
        self._lower = tuple(_i32_dev(t) if t.dtype == np.int64 else as_device(t)[0] for t in lower)
        self._upper = tuple(_i32_dev(t) if t.dtype == np.int64 else as_device(t)[0] for t in upper)
        order = np.argsort(levels, kind="stable")
        counts = np.bincount(levels) if len(levels) else np.zeros(0, dtype=np.int64)
        self._level_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        self._rows = _i32_dev(order.astype(np.int64))
        self.nlevels = len(counts)
        self.modified_diag = torch.empty(self.n, dtype=torch.float64, device=self._rows.device)
        diag_d, _ = as_device(diag)
        lib = _lib.load_library()
        bad = np.zeros(1, dtype=np.int64)
        rc = lib.cf_dic_factor(self.n, *(t.data_ptr() for t in self._lower), diag_d.data_ptr(),
                               self._rows.data_ptr(), self._level_ptr.ctypes.data, self.nlevels,
                               self.modified_diag.data_ptr(), bad.ctypes.data, _lib.stream())
        if rc == _lib.CF_EINVAL and bad[0] >= 0:
            d = float(to_host(self.modified_diag[int(bad[0]):int(bad[0]) + 1])[0])
            raise ValueError(f"DIC breakdown at row {int(bad[0])}: modified diagonal {d!r} <= 0 "
                             "(matrix not SPD or pattern pathological)")
        _lib.check(rc, "dic factor")

    def _args(self):
        return (*(t.data_ptr() for t in self._lower), *(t.data_ptr() for t in self._upper),
                self.modified_diag.data_ptr(), self._rows.data_ptr(), self._level_ptr.ctypes.data,
                self.nlevels)

    def apply(self, r, out=None):
        rd, host = as_device(r)
        if rd.shape[0] != self.n:
            raise ValueError(f"preconditioner has dimension {self.n}, vector {rd.shape[0]}")
        rd = rd.contiguous()
        z = out if isinstance(out, torch.Tensor) and out.is_cuda else torch.empty_like(rd)
        w = torch.empty_like(rd)
        lib = _lib.load_library()
        lp, lc, lv = (t.data_ptr() for t in self._lower)
        up, uc, uv = (t.data_ptr() for t in self._upper)
        _lib.check(lib.cf_dic_apply(self.n, lp, lc, lv, up, uc, uv, self.modified_diag.data_ptr(),
                                    self._rows.data_ptr(), self._level_ptr.ctypes.data, self.nlevels,
                                    rd.data_ptr(), w.data_ptr(), z.data_ptr(), _lib.stream()), "dic apply")
        if out is not None and not isinstance(out, torch.Tensor):
            out[...] = to_host(z)
            return out
        return to_host(z) if host and out is None else z

    def _fused_solve(self, ws, b, x, x0, tol, max_iter, its, res):
        import ctypes

        lib = _lib.load_library()
        # the workspace holds raw pointers to the bound factor: rebind whenever
        # another preconditioner was bound last, and keep this one alive while
        # the workspace points at it
        if getattr(ws, "_dic_owner", None) is not self:
            _lib.check(lib.cf_cg_set_dic(ws._h, *self._args()), "cf_cg_set_dic")
            ws._dic_owner = self
        return lib.cf_cg_solve(ws._h, b.data_ptr(), x.data_ptr(), _lib.ptr(x0), float(tol), int(max_iter),
                               _lib.PRECOND_DIC, None, ctypes.byref(its), ctypes.byref(res), _lib.stream())


def dic_from(a) -> DicPreconditioner:
    """Simplified DIC preconditioner (src/precond.py:141-151)."""
    lower, diag, upper, n = _triangles(a)
    return DicPreconditioner(lower, diag, upper, n, _levels(a, lower, n))


def apply(p, r, out):
    """out = M^-1 r (src/precond.py:154-156)."""
    return p.apply(r, out=out)
