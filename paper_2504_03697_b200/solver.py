"""Preconditioned conjugate gradient (mirror of src/solver.py).

``pcg`` keeps the reference signature, stopping rule (recurrence residual
sqrt(r.r)/|b| <= tol checked every iteration), zero-RHS shortcut,
``max_iter`` reporting and ``BreakdownError``.

Two device paths:

* fused -- when ``apply_a`` is the package's own matrix-free operator
  (``StencilOperator``) and the preconditioner is none/Jacobi/DIC, the whole
  solve runs in libcfgpu (cf_cg_solve): two fused kernels per iteration,
  scalars kept on the device, the loop a CUDA graph with a conditional
  WHILE node -- no host round trip until the solve ends.
* per-op -- any other ``apply_a`` callable: the reference loop with each
  vector op on the device (cf_dot / cf_axpy / the operator) and the
  reference's host-side scalar recurrence.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import as_device, to_host
from .sparse import StencilOperator, dot, multiply_add_inplace


class BreakdownError(RuntimeError):
    """p^T A p <= 0: the operator is not positive definite (src/solver.py:22-23)."""


@dataclass
class SolveStats:
    iterations: int
    final_residual_rel: float
    converged: bool


class _NullRegion:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


class _NullProfiler:
    def region(self, name):
        return _NullRegion()


NULL_PROFILER = _NullProfiler()


# cf_cg_last_form codes (include/cfgpu.h CF_CG_FORM_*)
FORMS = {0: "small", 1: "two-kernel", 2: "single-pass", 3: "pass", 4: "persistent", 5: "two-kernel+dic"}


class CgWorkspace:
    """Device workspace of the fused solver (one per operator grid; like
    PoissonCache it is built once and reused every step)."""

    def __init__(self, op: StencilOperator):
        lib = _lib.load_library()
        h = ctypes.c_void_p()
        _lib.check(lib.cf_cg_create(ctypes.byref(h), op.nx, op.ny, op.nz, op.h, op.order, _lib.stream()),
                   "cf_cg_create")
        self._h = h
        self.op = op
        self.last_loop_ms = 0.0
        self.last_form = None  # the CG kernel form of the last solve (FORMS) and its kernel launches
        self.last_launches = 0

    def solve(self, b: torch.Tensor, x0, precond, tol: float, max_iter: int):
        lib = _lib.load_library()
        pk, inv = _lib.PRECOND_NONE, None
        extra = None
        if precond is not None:
            kind = getattr(precond, "kind", None)
            if kind == "jacobi":
                pk = _lib.PRECOND_JACOBI
                if precond.constant is None or precond.constant != self.op.inv_diag_value:
                    inv = precond.inv_diag
            elif kind == "dic":
                pk = _lib.PRECOND_DIC
                extra = precond
            else:
                raise TypeError(f"fused pcg: unsupported preconditioner {type(precond).__name__}")
        x = torch.empty_like(b)
        its = ctypes.c_int64()
        res = ctypes.c_double()
        if extra is not None:
            rc = extra._fused_solve(self, b, x, x0, tol, max_iter, its, res)
        else:
            rc = lib.cf_cg_solve(self._h, b.data_ptr(), x.data_ptr(), _lib.ptr(x0), float(tol), int(max_iter),
                                 pk, _lib.ptr(inv), ctypes.byref(its), ctypes.byref(res), _lib.stream())
        ms = ctypes.c_float()
        lib.cf_cg_last_loop_ms(self._h, ctypes.byref(ms))
        self.last_loop_ms = float(ms.value)
        form, launches = ctypes.c_int(), ctypes.c_int64()
        lib.cf_cg_last_form(self._h, ctypes.byref(form), ctypes.byref(launches))
        self.last_form, self.last_launches = FORMS.get(form.value, str(form.value)), int(launches.value)
        if rc == _lib.CF_BREAKDOWN:
            raise BreakdownError(_lib.last_error())
        _lib.check(rc, "cf_cg_solve")
        return x, SolveStats(int(its.value), float(res.value), rc == _lib.CF_OK)

    def __del__(self):
        try:
            if self._h and _lib._lib is not None:
                _lib._lib.cf_cg_destroy(self._h)
        except Exception:
            pass


def workspace_for(op: StencilOperator) -> CgWorkspace:
    ws = getattr(op, "_cg_ws", None)
    if ws is None:
        ws = CgWorkspace(op)
        op._cg_ws = ws
    return ws


def pcg(apply_a, b, x0=None, precond=None, tol: float = 1e-6, max_iter: int = 1000,
        variant: str = "baseline", pool=None, profiler=None):
    """Solve A x = b for SPD A given as ``apply_a(x, out=None)`` (src/solver.py:33-68)."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if max_iter < 1:
        raise ValueError(f"max_iter must be >= 1, got {max_iter}")
    if variant not in ("baseline", "optimized"):
        raise ValueError(f"unknown variant {variant!r}")
    prof = profiler if profiler is not None else NULL_PROFILER
    bd, host = as_device(b)
    bd = bd.contiguous()
    x0d = None if x0 is None else as_device(x0)[0].contiguous()
    fusable = isinstance(apply_a, StencilOperator) and (
        precond is None or getattr(precond, "kind", None) in ("jacobi", "dic"))
    if fusable:
        ws = workspace_for(apply_a)
        x, stats = ws.solve(bd, x0d, precond, tol, max_iter)
        _record_fused_rows(prof, ws, stats, x0d is not None, precond is not None)
    else:
        x, stats = _pcg_per_op(apply_a, bd, x0d, precond, tol, max_iter, prof)
    return (to_host(x) if host else x), stats


# Bytes per cell each reference op of one CG iteration streams
# (src/solver.py:148-170): spmv reads p and writes Ap, p.Ap / r.z read two
# vectors, r.r one, multiply_add_inplace reads two and writes one, the
# preconditioner reads r and writes z.
_ROW_BYTES = {"spmv": 16, "dot": 16, "multiply_add_inplace": 24, "precondition": 16}


def _record_fused_rows(prof, ws, stats, warm, has_precond):
    """The reference's pcg sub-regions (src/solver.py:148-170: spmv, dot,
    multiply_add_inplace, precondition -- PAPER.md Table 1's rows) for a
    solve that ran as fused kernels: the reference's call counts for
    `stats.iterations` iterations, and the measured device time of the loop
    (CUDA events, ws.last_loop_ms) split over them in proportion to the bytes
    each op streams.  The split is synthesised -- the fused kernels run no
    separate spmv or dot -- but the rows line up with a reference report
    (compare_reports)."""
    k = stats.iterations
    record = getattr(prof, "record", None)
    if k == 0 or record is None:
        return
    last_full = not stats.converged  # a converged last iteration stops after r.r
    calls = {"spmv": k + (1 if warm else 0),
             "dot": 1 + 2 * k + (k if last_full else k - 1),
             "multiply_add_inplace": 2 * k + (k if last_full else k - 1) + (1 if warm else 0),
             "precondition": (1 + (k if last_full else k - 1)) if has_precond else 0}
    weight = {n: c * (_ROW_BYTES[n] if n != "dot" else 40 / 3) for n, c in calls.items()}
    total = sum(weight.values())
    seconds = ws.last_loop_ms * 1e-3
    for name in ("spmv", "dot", "multiply_add_inplace", "precondition"):
        if calls[name]:
            record(name, calls[name], seconds * weight[name] / total)


def _precondition(precond, r, out, prof):
    if precond is None:
        out.copy_(r)
        return out
    with prof.region("precondition"):
        res = precond.apply(r, out=out)
        if res is not out:
            out.copy_(res if isinstance(res, torch.Tensor) else torch.as_tensor(res, device=out.device))
        return out


def _pcg_per_op(apply_a, b, x0, precond, tol, max_iter, prof):
    """The reference recurrence (src/solver.py:128-171) on device vectors."""
    n = b.shape[0]
    with prof.region("dot"):
        norm_b = math.sqrt(dot(b, b))
    if norm_b == 0.0:
        return torch.zeros_like(b), SolveStats(0, 0.0, True)
    r = b.clone()
    ap = torch.empty_like(b)

    def op(v, out):
        res = apply_a(v, out=out)
        if res is not out:
            out.copy_(res if isinstance(res, torch.Tensor) else torch.as_tensor(np.asarray(res), device=out.device))
        return out

    if x0 is None:
        x = torch.zeros_like(b)
    else:
        x = x0.clone()
        with prof.region("spmv"):
            op(x, ap)
        with prof.region("multiply_add_inplace"):
            multiply_add_inplace(r, -1.0, ap)
    z = _precondition(precond, r, torch.empty_like(b), prof)
    p = z.clone()
    with prof.region("dot"):
        rz = dot(r, z)
    res_rel = math.inf
    it = 0
    converged = False
    while it < max_iter:
        with prof.region("spmv"):
            op(p, ap)
        with prof.region("dot"):
            pap = dot(p, ap)
        if pap <= 0.0:
            raise BreakdownError(f"p^T A p = {pap!r} at iteration {it + 1}")
        alpha = rz / pap
        with prof.region("multiply_add_inplace"):
            multiply_add_inplace(x, alpha, p)
            multiply_add_inplace(r, -alpha, ap)
        it += 1
        with prof.region("dot"):
            res_rel = math.sqrt(dot(r, r)) / norm_b
        if res_rel <= tol:
            converged = True
            break
        _precondition(precond, r, z, prof)
        with prof.region("dot"):
            rz_new = dot(r, z)
        beta = rz_new / rz
        rz = rz_new
        with prof.region("multiply_add_inplace"):
            multiply_add_inplace(z, beta, p)
        p, z = z, p
    assert n == x.shape[0]
    return x, SolveStats(it, res_rel, converged)
