"""Sparse operators and vector kernels on the device (mirror of src/sparse.py).

Storage types keep the reference's constructor signatures and validation
(host-side, numpy: structure checks are setup, not hot path) and mirror
themselves into HBM with int32 indices (half the index traffic of the
reference's int64).  Kernels take CUDA tensors; numpy inputs are accepted
for drop-in use and are uploaded, computed on the GPU and copied back, so a
caller that passes host arrays gets host arrays.

``StencilOperator`` is the matrix-free form of the pressure operator: the
fast path of the CG solve (no matrix stream at all).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .grid import as_device, to_host


def _as_i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x), dtype=np.int64)


def _as_f64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x), dtype=np.float64)


def _validate_csr(n_rows, n_cols, row_ptr, col_idx, values):
    """Same acceptance rules and messages as src/sparse.py:72-96."""
    if row_ptr.shape != (n_rows + 1,):
        raise ValueError(f"row_ptr must have length {n_rows + 1}, got {row_ptr.shape}")
    if row_ptr[0] != 0:
        raise ValueError(f"row_ptr[0] must be 0, got {row_ptr[0]}")
    if len(col_idx) != len(values):
        raise ValueError(f"col_idx and values lengths differ: {len(col_idx)} vs {len(values)}")
    if row_ptr[-1] != len(values):
        raise ValueError(f"row_ptr[-1]={row_ptr[-1]} must equal nnz={len(values)}")
    steps = np.diff(row_ptr)
    if np.any(steps < 0):
        raise ValueError(f"row_ptr decreases at row {int(np.argmax(steps < 0))}")
    if len(col_idx) and (col_idx.min() < 0 or col_idx.max() >= n_cols):
        raise ValueError(f"column index out of range [0, {n_cols})")
    if len(col_idx) > 1:
        rows = np.repeat(np.arange(n_rows, dtype=np.int64), steps)
        same_row = rows[1:] == rows[:-1]
        bad = same_row & (np.diff(col_idx) <= 0)
        if np.any(bad):
            raise ValueError(
                f"column indices not strictly increasing in row {int(rows[1:][bad][0])}")


def _i32_dev(a: np.ndarray) -> torch.Tensor:
    if len(a) and (a.max() >= 2 ** 31 or a.min() < -(2 ** 31)):
        raise ValueError("index exceeds the int32 device range")
    return torch.as_tensor(a.astype(np.int32), device=as_device(np.zeros(0))[0].device)


class CsrMatrix:
    """Compressed-row sparse matrix (src/sparse.py:29-69)."""

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col_idx, values):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.row_ptr = _as_i64(row_ptr)
        self.col_idx = _as_i64(col_idx)
        self.values = _as_f64(values)
        _validate_csr(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, self.values)
        self._dev = None

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @classmethod
    def from_dense(cls, a) -> "CsrMatrix":
        a = _as_f64(a)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
        rows, cols = np.nonzero(a)
        ptr = np.concatenate(([0], np.cumsum(np.bincount(rows, minlength=a.shape[0]))))
        return cls(a.shape[0], a.shape[1], ptr, cols, a[rows, cols])

    def row_indices(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))

    def diagonal(self) -> np.ndarray:
        d = np.zeros(min(self.n_rows, self.n_cols))
        rows = self.row_indices()
        on = rows == self.col_idx
        d[rows[on]] = self.values[on]
        return d

    def device(self):
        """(row_ptr, col_idx) int32 and values fp64 in HBM, uploaded once."""
        if self._dev is None:
            self._dev = (_i32_dev(self.row_ptr), _i32_dev(self.col_idx), as_device(self.values)[0])
        return self._dev


class SymCsrMatrix:
    """Diagonal plus strict upper triangle, with the cached transpose pattern
    (src/sparse.py:99-137)."""

    def __init__(self, n: int, diag, row_ptr, col_idx, values):
        self.n = int(n)
        self.diag = _as_f64(diag)
        self.row_ptr = _as_i64(row_ptr)
        self.col_idx = _as_i64(col_idx)
        self.values = _as_f64(values)
        if self.diag.shape != (self.n,):
            raise ValueError(f"diag must have length {self.n}, got {self.diag.shape}")
        _validate_csr(self.n, self.n, self.row_ptr, self.col_idx, self.values)
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        below = self.col_idx <= rows
        if np.any(below):
            b = int(np.flatnonzero(below)[0])
            raise ValueError(f"upper triangle holds entry ({rows[b]}, {self.col_idx[b]}) with col <= row")
        order = np.lexsort((rows, self.col_idx))
        counts = np.bincount(self.col_idx, minlength=self.n)
        self.t_row_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        self.t_col_idx = rows[order]
        self.t_perm = order.astype(np.int64)
        self._dev = None

    @property
    def nnz_stored(self) -> int:
        return self.n + len(self.values)

    def lower_values(self) -> np.ndarray:
        return self.values[self.t_perm]

    def device(self):
        if self._dev is None:
            self._dev = (as_device(self.diag)[0], _i32_dev(self.row_ptr), _i32_dev(self.col_idx),
                         as_device(self.values)[0], _i32_dev(self.t_row_ptr), _i32_dev(self.t_col_idx),
                         _i32_dev(self.t_perm))
        return self._dev


def to_symmetric(a: CsrMatrix) -> SymCsrMatrix:
    """Diagonal + upper storage of an exactly symmetric CSR matrix (src/sparse.py:140-177)."""
    if a.n_rows != a.n_cols:
        raise ValueError(f"matrix must be square, got {a.shape}")
    rows = a.row_indices()
    up = a.col_idx > rows
    lo = a.col_idx < rows
    diag = np.zeros(a.n_rows)
    on = a.col_idx == rows
    diag[rows[on]] = a.values[on]
    ur, uc, uv = rows[up], a.col_idx[up], a.values[up]
    lr, lc, lv = rows[lo], a.col_idx[lo], a.values[lo]
    upper = set(zip(ur.tolist(), uc.tolist()))
    mirrored = {(j, i) for i, j in zip(lr.tolist(), lc.tolist())}
    if upper != mirrored:
        i, j = sorted(upper.symmetric_difference(mirrored))[0]
        raise ValueError(f"matrix is not symmetric: entry ({i},{j}) has no stored mirror ({j},{i})")
    order = np.lexsort((ur, uc))  # transpose of U in lower-triangle order
    tuv = uv[order]
    mism = tuv != lv
    if np.any(mism):
        p = int(np.flatnonzero(mism)[0])
        raise ValueError(f"matrix is not symmetric: A[{uc[order][p]},{ur[order][p]}]={tuv[p]!r} "
                         f"but A[{lr[p]},{lc[p]}]={lv[p]!r}")
    ptr = np.concatenate(([0], np.cumsum(np.bincount(ur, minlength=a.n_rows))))
    return SymCsrMatrix(a.n_rows, diag, ptr, uc, uv)


# ---------------------------------------------------------------------------
# kernels


def _out_like(out, n, host):
    if out is None:
        return torch.empty(n, dtype=torch.float64, device=as_device(np.zeros(0))[0].device), None
    if isinstance(out, torch.Tensor) and out.is_cuda:
        return out, None
    # host out= buffer: compute on the device, copy back into it
    return torch.empty(n, dtype=torch.float64, device=as_device(np.zeros(0))[0].device), out


def _finish(y, host_out, host):
    if host_out is not None:
        host_out[...] = to_host(y)
        return host_out
    return to_host(y) if host else y


def spmv(a: CsrMatrix, x, out=None, pool=None):
    """y = A x, full CSR (src/sparse.py:236-247)."""
    xd, host = as_device(x)
    if xd.shape[0] != a.n_cols:
        raise ValueError(f"matrix has {a.n_cols} columns but x has length {xd.shape[0]}")
    y, host_out = _out_like(out, a.n_rows, host)
    rp, ci, val = a.device()
    lib = _lib.load_library()
    _lib.check(lib.cf_csr_spmv(a.n_rows, rp.data_ptr(), ci.data_ptr(), val.data_ptr(),
                               xd.contiguous().data_ptr(), y.data_ptr(), _lib.stream()), "spmv")
    return _finish(y, host_out, host)


def spmv_sym(s: SymCsrMatrix, x, out=None, pool=None):
    """y = (D + U + U^T) x (src/sparse.py:250-267)."""
    xd, host = as_device(x)
    if xd.shape[0] != s.n:
        raise ValueError(f"matrix has dimension {s.n} but x has length {xd.shape[0]}")
    y, host_out = _out_like(out, s.n, host)
    d = s.device()
    lib = _lib.load_library()
    _lib.check(lib.cf_sym_spmv(s.n, *(t.data_ptr() for t in d), xd.contiguous().data_ptr(), y.data_ptr(),
                               _lib.stream()), "spmv_sym")
    return _finish(y, host_out, host)


def _check_same_length(x, y):
    if len(x) != len(y):
        raise ValueError(f"vector lengths differ: {len(x)} vs {len(y)}")


def dot(x, y, pool=None) -> float:
    """x . y with a fixed two-level device reduction (src/sparse.py:270-281)."""
    _check_same_length(x, y)
    xd, _ = as_device(x)
    yd, _ = as_device(y)
    r = _lib.dbl_out()
    lib = _lib.load_library()
    _lib.check(lib.cf_dot(xd.contiguous().data_ptr(), yd.contiguous().data_ptr(), xd.shape[0],
                          _lib.byref(r), _lib.stream()), "dot")
    return float(r.value)


def multiply_add_inplace(y, alpha: float, x, pool=None) -> None:
    """y += alpha * x in place, unfused (src/sparse.py:284-290)."""
    _check_same_length(x, y)
    yd, host = as_device(y)
    xd, _ = as_device(x)
    if not yd.is_contiguous():
        raise ValueError("y must be contiguous")
    lib = _lib.load_library()
    _lib.check(lib.cf_axpy(yd.data_ptr(), float(alpha), xd.contiguous().data_ptr(), yd.shape[0],
                           _lib.stream()), "multiply_add_inplace")
    if host:
        y[...] = to_host(yd)


def add(x, y):
    """x + y in a fresh vector (src/sparse.py:293-296)."""
    _check_same_length(x, y)
    xd, host = as_device(x)
    yd, _ = as_device(y)
    out = torch.empty_like(xd)
    lib = _lib.load_library()
    _lib.check(lib.cf_add(xd.contiguous().data_ptr(), yd.contiguous().data_ptr(), out.data_ptr(),
                          xd.shape[0], _lib.stream()), "add")
    return to_host(out) if host else out


def scale(alpha: float, x):
    """alpha * x in a fresh vector (src/sparse.py:299-301)."""
    xd, host = as_device(x)
    out = torch.empty_like(xd)
    lib = _lib.load_library()
    _lib.check(lib.cf_scale(float(alpha), xd.contiguous().data_ptr(), out.data_ptr(), xd.shape[0],
                            _lib.stream()), "scale")
    return to_host(out) if host else out


class StencilOperator:
    """Matrix-free 7-point pressure operator of src/sim.py:296-333.

    ``op(x, out=None)`` has the ``apply_a`` signature pcg expects
    (src/solver.py:44-48).  ``order`` selects the summation order of
    ``spmv`` (CSR, the baseline variant) or ``spmv_sym`` (the optimized
    variant) so results are bit-identical to the matching reference SpMV.
    """

    def __init__(self, n: int, h: float, order: str = "sym", shape=None):
        if order not in ("csr", "sym"):
            raise ValueError("order must be 'csr' or 'sym'")
        self.n, self.h = int(n), float(h)
        # shape (extension): an nx*ny*nz box; the reference operator is the n-cube
        self.nx, self.ny, self.nz = (self.n,) * 3 if shape is None else tuple(int(s) for s in shape)
        self.order = _lib.ORDER_CSR if order == "csr" else _lib.ORDER_SYM
        self.num = self.nx * self.ny * self.nz
        self.inv_diag_value = 1.0 / (6.0 / (self.h * self.h))  # jacobi_from's 1.0 / diag

    def __call__(self, x, out=None):
        xd, host = as_device(x)
        if xd.shape[0] != self.num:
            raise ValueError(f"operator has dimension {self.num} but x has length {xd.shape[0]}")
        y, host_out = _out_like(out, self.num, host)
        lib = _lib.load_library()
        _lib.check(lib.cf_stencil7_apply(self.nx, self.ny, self.nz, self.h, self.order,
                                         xd.contiguous().data_ptr(), y.data_ptr(), _lib.stream()),
                   "stencil7_apply")
        return _finish(y, host_out, host)

    def diagonal(self) -> np.ndarray:
        return np.full(self.num, 6.0 / (self.h * self.h))
