"""CPU oracle for the cavityflow time-step hot path.

TEST INFRASTRUCTURE ONLY -- this package is the parity checker, never the
product.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product
package ``paper_2504_03697_b200`` never imports it and has no CPU fallback.

It restates the reference algorithm (``/root/reference/pkg/src/cavityflow``,
abbreviated ``src/`` below) as numpy glue over the plain-C kernels in
``cf_oracle.c``.  Each function cites the reference lines it follows.  The
restatement is *pinned*: ``tests/test_oracle.py`` checks it bit-for-bit (or
at the reference's own tolerances) against ``tests/golden/*.npz``, which
``tests/golden/make_golden.py`` produced by importing and running the
reference itself in the build container.

Layouts follow the reference: velocity components are C-order numpy arrays
``u (n+1,n,n)``, ``v (n,n+1,n)``, ``w (n,n,n+1)`` (k fastest); scalars are
flat with i fastest (``src/grid.py:44-48``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    """Compile cf_oracle.c into liboracle.so (idempotent)."""
    src = os.path.join(_HERE, "cf_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_spmv_csr.argtypes = [_ip, _ip, _dp, _dp, _dp, _ip, ctypes.c_int]
        L.orc_spmv_sym.argtypes = [_dp, _ip, _ip, _dp, _ip, _ip, _ip, _dp, _dp, _ip, ctypes.c_int]
        L.orc_dot.argtypes = [_dp, _dp, _ip, ctypes.c_int, _dp]
        L.orc_maxpy.argtypes = [_dp, ctypes.c_double, _dp, _ip, ctypes.c_int]
        L.orc_dic_diag.argtypes = [_ip, _ip, _dp, _dp, _dp, ctypes.c_int64]
        L.orc_dic_diag.restype = ctypes.c_int64
        L.orc_dic_apply.argtypes = [_ip, _ip, _dp, _ip, _ip, _dp, _dp, _dp, _dp, _dp, ctypes.c_int64]
        L.orc_advect.argtypes = [_dp, _dp, _dp, _dp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_double, ctypes.c_double, _ip, ctypes.c_int]
        L.orc_divergence.argtypes = [_dp, _dp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_double, _dp, ctypes.c_int]
        _lib = L
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def chunk_bounds(n_items: int, threads: int) -> np.ndarray:
    """src/parallel.py:24-26 -- one contiguous chunk per worker."""
    chunks = max(1, min(threads, n_items)) if n_items > 0 else 1
    return np.linspace(0, n_items, chunks + 1).astype(np.int64)


# ---------------------------------------------------------------------------
# sparse storage and kernels (src/sparse.py)


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.n_rows, dtype=np.int64), np.diff(self.row_ptr))

    def diagonal(self) -> np.ndarray:
        d = np.zeros(min(self.n_rows, self.n_cols))
        r = self.rows()
        on = r == self.col_idx
        d[r[on]] = self.values[on]
        return d


@dataclass
class SymCsr:
    n: int
    diag: np.ndarray
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    t_row_ptr: np.ndarray = field(init=False)
    t_col_idx: np.ndarray = field(init=False)
    t_perm: np.ndarray = field(init=False)

    def __post_init__(self):
        # src/sparse.py:123-129: transpose pattern, sorted by (col, row)
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))
        order = np.lexsort((rows, self.col_idx))
        counts = np.bincount(self.col_idx, minlength=self.n)
        self.t_row_ptr = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        self.t_col_idx = np.ascontiguousarray(rows[order])
        self.t_perm = order.astype(np.int64)


def _cell_ijk(nx: int, ny: int, nz: int):
    idx = np.arange(nx * ny * nz, dtype=np.int64)
    return idx, idx % nx, (idx // nx) % ny, idx // (nx * ny)


def _box(n, shape):
    return tuple(shape) if shape is not None else (n, n, n)


def poisson_csr(n: int, h: float, shape=None) -> Csr:
    """src/sim.py:296-317 -- full CSR, columns ascending (k-1,j-1,i-1,d,i+1,j+1,k+1).
    ``shape`` (extension): an nx*ny*nz box instead of the cube."""
    nx, ny, nz = _box(n, shape)
    idx, i, j, k = _cell_ijk(nx, ny, nz)
    pl = nx * ny
    cand = np.stack([idx - pl, idx - nx, idx - 1, idx, idx + 1, idx + nx, idx + pl], axis=1)
    keep = np.stack([k > 0, j > 0, i > 0, np.ones_like(i, dtype=bool), i < nx - 1, j < ny - 1,
                     k < nz - 1], axis=1)
    vals = np.full(cand.shape, -1.0 / (h * h))
    vals[:, 3] = 6.0 / (h * h)
    row_ptr = np.concatenate(([0], np.cumsum(keep.sum(axis=1)))).astype(np.int64)
    m = keep.ravel()
    num = nx * ny * nz
    return Csr(num, num, row_ptr, np.ascontiguousarray(cand.ravel()[m]),
               np.ascontiguousarray(vals.ravel()[m]))


def poisson_sym(n: int, h: float, shape=None) -> SymCsr:
    """src/sim.py:320-333 -- diagonal plus strict upper (i+1, j+1, k+1)."""
    nx, ny, nz = _box(n, shape)
    idx, i, j, k = _cell_ijk(nx, ny, nz)
    cand = np.stack([idx + 1, idx + nx, idx + nx * ny], axis=1)
    keep = np.stack([i < nx - 1, j < ny - 1, k < nz - 1], axis=1)
    vals = np.full(cand.shape, -1.0 / (h * h))
    row_ptr = np.concatenate(([0], np.cumsum(keep.sum(axis=1)))).astype(np.int64)
    m = keep.ravel()
    num = nx * ny * nz
    return SymCsr(num, np.full(num, 6.0 / (h * h)), row_ptr,
                  np.ascontiguousarray(cand.ravel()[m]), np.ascontiguousarray(vals.ravel()[m]))


def spmv(a: Csr, x: np.ndarray, threads: int = 1, out=None) -> np.ndarray:
    """src/sparse.py:236-247."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(a.n_rows) if out is None else out
    b = chunk_bounds(a.n_rows, threads)
    lib().orc_spmv_csr(_i(a.row_ptr), _i(a.col_idx), _d(a.values), _d(x), _d(out), _i(b), len(b) - 1)
    return out


def spmv_sym(s: SymCsr, x: np.ndarray, threads: int = 1, out=None) -> np.ndarray:
    """src/sparse.py:250-267."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(s.n) if out is None else out
    b = chunk_bounds(s.n, threads)
    lib().orc_spmv_sym(_d(s.diag), _i(s.row_ptr), _i(s.col_idx), _d(s.values), _i(s.t_row_ptr),
                       _i(s.t_col_idx), _i(s.t_perm), _d(x), _d(out), _i(b), len(b) - 1)
    return out


def dot(x: np.ndarray, y: np.ndarray, threads: int = 1) -> float:
    """src/sparse.py:270-281 -- chunk partials summed in chunk order."""
    b = chunk_bounds(len(x), threads) if threads > 1 else np.array([0, len(x)], dtype=np.int64)
    part = np.empty(len(b) - 1)
    lib().orc_dot(_d(x), _d(y), _i(b), len(b) - 1, _d(part))
    if threads == 1:
        return float(part[0])
    return float(sum(part.tolist()))


def maxpy(y: np.ndarray, alpha: float, x: np.ndarray, threads: int = 1) -> None:
    """src/sparse.py:284-290 -- y += alpha * x in place."""
    b = chunk_bounds(len(y), threads)
    lib().orc_maxpy(_d(y), float(alpha), _d(x), _i(b), len(b) - 1)


# ---------------------------------------------------------------------------
# preconditioners (src/precond.py)


class Jacobi:
    """src/precond.py:77-95, :127-138."""

    def __init__(self, diag: np.ndarray):
        zero = np.flatnonzero(diag == 0.0)
        if len(zero):
            raise ValueError(f"zero diagonal entry at row {zero[0]}")
        self.inv_diag = 1.0 / diag

    def apply(self, r, out=None):
        out = np.empty(len(r)) if out is None else out
        np.multiply(r, self.inv_diag, out=out)
        return out


def _triangles(a):
    """src/precond.py:57-74 -- strict lower / upper triangles in CSR form."""
    if isinstance(a, SymCsr):
        lower = (a.t_row_ptr, a.t_col_idx, np.ascontiguousarray(a.values[a.t_perm]))
        return lower, a.diag.copy(), (a.row_ptr, a.col_idx, a.values), a.n
    rows = a.rows()
    parts = []
    for m in (a.col_idx < rows, a.col_idx > rows):
        ptr = np.concatenate(([0], np.cumsum(np.bincount(rows[m], minlength=a.n_rows)))).astype(np.int64)
        parts.append((ptr, np.ascontiguousarray(a.col_idx[m]), np.ascontiguousarray(a.values[m])))
    return parts[0], a.diagonal(), parts[1], a.n_rows


class Dic:
    """src/precond.py:98-124, :141-151 -- simplified DIC, sequential sweeps."""

    def __init__(self, a):
        self.lower, diag, self.upper, self.n = _triangles(a)
        self.modified_diag = np.empty(self.n)
        bad = lib().orc_dic_diag(_i(self.lower[0]), _i(self.lower[1]), _d(self.lower[2]), _d(diag),
                                 _d(self.modified_diag), self.n)
        if bad >= 0:
            raise ValueError(f"DIC breakdown at row {bad}")

    def apply(self, r, out=None):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.empty(self.n) if out is None else out
        w = np.empty(self.n)
        lo, up = self.lower, self.upper
        lib().orc_dic_apply(_i(lo[0]), _i(lo[1]), _d(lo[2]), _i(up[0]), _i(up[1]), _d(up[2]),
                            _d(self.modified_diag), _d(r), _d(w), _d(out), self.n)
        return out


def jacobi_from(a) -> Jacobi:
    return Jacobi(a.diag if isinstance(a, SymCsr) else a.diagonal())


# ---------------------------------------------------------------------------
# PCG (src/solver.py)


class Breakdown(RuntimeError):
    pass


@dataclass
class Stats:
    iterations: int
    final_residual_rel: float
    converged: bool


def pcg(apply_a, b, x0=None, precond=None, tol=1e-6, max_iter=1000, variant="optimized",
        threads=1, max_count=None):
    """src/solver.py:33-68 with the loop of :128-171.

    The baseline variant (:81-125) performs the same per-element operations
    (``add(x, scale(a, p))`` == ``x + a*p``), and its dots are serial, so it
    is the optimized loop with ``threads`` forced to 1 for the dots.
    ``max_count`` (oracle-only) stops after that many iterations, for
    bounded CPU-baseline samples.
    """
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    dthreads = threads if variant == "optimized" else 1
    norm_b = math.sqrt(dot(b, b, dthreads))
    if norm_b == 0.0:
        return np.zeros(n), Stats(0, 0.0, True)
    r = b.copy()
    ap = np.empty(n)
    if x0 is None:
        x = np.zeros(n)
    else:
        x = np.array(x0, dtype=np.float64)
        apply_a(x, ap)
        maxpy(r, -1.0, ap, threads)
    z = r.copy() if precond is None else precond.apply(r, np.empty(n))
    p = z.copy()
    rz = dot(r, z, dthreads)
    res = math.inf
    it = 0
    converged = False
    limit = max_iter if max_count is None else min(max_iter, max_count)
    while it < limit:
        apply_a(p, ap)
        pap = dot(p, ap, dthreads)
        if pap <= 0.0:
            raise Breakdown(f"p^T A p = {pap!r} at iteration {it + 1}")
        alpha = rz / pap
        maxpy(x, alpha, p, threads)
        maxpy(r, -alpha, ap, threads)
        it += 1
        res = math.sqrt(dot(r, r, dthreads)) / norm_b
        if res <= tol:
            converged = True
            break
        if precond is None:
            z[:] = r
        else:
            precond.apply(r, z)
        rz_new = dot(r, z, dthreads)
        beta = rz_new / rz
        rz = rz_new
        maxpy(z, beta, p, threads)
        p, z = z, p
    return x, Stats(it, res, converged)


# ---------------------------------------------------------------------------
# time step (src/sim.py, src/grid.py)


@dataclass
class Cfg:
    """Mirror of src/sim.py:53-70 (validation lives in the product)."""

    n: int = 100
    h: float = 1.0
    dt: float = 0.4
    t_end: float = 6.0
    lid_accel: float = 1.0
    density: float = 1.0
    tol: float = 1e-6
    max_iter: int = 1000
    preconditioner: str = "dic"
    variant: str = "baseline"
    threads: int = 1
    warm_start: bool = False
    shape: tuple | None = None  # extension: an nx*ny*nz box (the reference is the n-cube)

    @property
    def num_steps(self) -> int:
        return round(self.t_end / self.dt)

    @property
    def box(self):
        return _box(self.n, self.shape)


@dataclass
class State:
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    p: np.ndarray
    t: float = 0.0
    step: int = 0


@dataclass
class StepResult:
    solve: Stats
    div_pre: float
    div_post: float


def initial_state(n: int, shape=None) -> State:
    """src/sim.py:126-131 -- rest under unit pressure."""
    nx, ny, nz = _box(n, shape)
    return State(np.zeros((nx + 1, ny, nz)), np.zeros((nx, ny + 1, nz)), np.zeros((nx, ny, nz + 1)),
                 np.ones(nx * ny * nz))


def apply_forces(s: State, cfg: Cfg) -> None:
    """src/sim.py:134-137 -- lid offset on the top-layer u faces."""
    nx, ny, _ = cfg.box
    s.u[1:nx, ny - 1, :] += cfg.lid_accel * cfg.dt


def enforce_boundaries(s: State) -> None:
    """src/sim.py:140-149 -- zero the wall-normal faces."""
    s.u[0], s.u[-1] = 0.0, 0.0
    s.v[:, 0], s.v[:, -1] = 0.0, 0.0
    s.w[:, :, 0], s.w[:, :, -1] = 0.0, 0.0


def advect(u, v, w, n: int, h: float, dt: float, threads: int = 1):
    """src/sim.py:259-289 -- new (u, v, w) with wall-normal planes zeroed.
    (The box extents come from the arrays; n is kept for the reference call shape.)"""
    u, v, w = (np.ascontiguousarray(a, dtype=np.float64) for a in (u, v, w))
    nx, ny, nz = u.shape[0] - 1, u.shape[1], u.shape[2]
    outs = []
    for comp, shape in enumerate(((nx + 1, ny, nz), (nx, ny + 1, nz), (nx, ny, nz + 1))):
        out = np.empty(shape)
        b = chunk_bounds(out.size, threads)
        lib().orc_advect(_d(u), _d(v), _d(w), _d(out), comp, nx, ny, nz, h, dt, _i(b), len(b) - 1)
        outs.append(out)
    nu, nv, nw = outs
    nu[0], nu[nx] = 0.0, 0.0
    nv[:, 0], nv[:, ny] = 0.0, 0.0
    nw[:, :, 0], nw[:, :, nz] = 0.0, 0.0
    return nu, nv, nw


_LATTICE = ((0.0, 0.5, 0.5), (0.5, 0.0, 0.5), (0.5, 0.5, 0.0))


def _trilinear(arr, a, b, c):
    """src/grid.py:102-121 -- clamp to the lattice hull, then lerp x, y, z."""
    na, nb, nc = arr.shape
    a = min(max(a, 0.0), na - 1.0)
    b = min(max(b, 0.0), nb - 1.0)
    c = min(max(c, 0.0), nc - 1.0)
    i0, j0, k0 = min(int(a), max(na - 2, 0)), min(int(b), max(nb - 2, 0)), min(int(c), max(nc - 2, 0))
    i1, j1, k1 = min(i0 + 1, na - 1), min(j0 + 1, nb - 1), min(k0 + 1, nc - 1)
    fa, fb, fc = a - i0, b - j0, c - k0

    def lx(j, k):
        return arr[i0, j, k] * (1.0 - fa) + arr[i1, j, k] * fa

    return (lx(j0, k0) * (1.0 - fb) + lx(j1, k0) * fb) * (1.0 - fc) + (lx(j0, k1) * (1.0 - fb) + lx(j1, k1) * fb) * fc


def sample_velocity(u, v, w, h: float, point) -> np.ndarray:
    """src/grid.py:124-142 -- each component on its own face lattice."""
    p = np.asarray(point, dtype=np.float64)
    if p.shape != (3,) or not np.all(np.isfinite(p)):
        raise ValueError(f"bad sample point {p!r}")
    return np.array([_trilinear(arr, p[0] / h - o[0], p[1] / h - o[1], p[2] / h - o[2])
                     for arr, o in zip((u, v, w), _LATTICE)])


def divergence(u, v, w, h: float, threads: int = 1) -> np.ndarray:
    """src/grid.py:145-154 -- flat, i fastest."""
    nx, ny, nz = u.shape[0] - 1, u.shape[1], u.shape[2]
    out = np.empty(nx * ny * nz)
    lib().orc_divergence(_d(np.ascontiguousarray(u)), _d(np.ascontiguousarray(v)),
                         _d(np.ascontiguousarray(w)), nx, ny, nz, h, _d(out), threads)
    return out


class Cache:
    """src/sim.py:336-349 -- the optimized variant keeps its symmetric matrix."""

    def __init__(self):
        self.matrix = None


def assemble(s: State, cfg: Cfg, cache: Cache | None = None):
    """src/sim.py:352-372."""
    b = (-cfg.density / cfg.dt) * divergence(s.u, s.v, s.w, cfg.h, cfg.threads)
    if cfg.variant == "optimized":
        if cache is None:
            return poisson_sym(cfg.n, cfg.h, cfg.shape), b
        if cache.matrix is None:
            cache.matrix = poisson_sym(cfg.n, cfg.h, cfg.shape)
        return cache.matrix, b
    return poisson_csr(cfg.n, cfg.h, cfg.shape), b


def solve_pressure(s: State, cfg: Cfg, cache: Cache | None = None, max_count=None):
    """src/sim.py:379-423 -- returns (stats, div_pre); writes s.p in place."""
    a, b = assemble(s, cfg, cache)
    div_pre = float(np.abs(b).max()) * cfg.dt / cfg.density if len(b) else 0.0
    pre = Dic(a) if cfg.preconditioner == "dic" else jacobi_from(a)
    th = cfg.threads
    if isinstance(a, SymCsr):
        def op(x, out):
            return spmv_sym(a, x, th, out)
    else:
        def op(x, out):
            return spmv(a, x, th, out)
    x0 = s.p.copy() if (cfg.warm_start and s.step > 0) else None
    x, st = pcg(op, b, x0, pre, cfg.tol, cfg.max_iter, cfg.variant, th, max_count)
    s.p[:] = x
    return st, div_pre


def correct(s: State, cfg: Cfg) -> float:
    """src/sim.py:426-449 -- gradient subtract with ghost p = 0, div_post, walls."""
    nx, ny, nz = cfg.box
    coef = cfg.dt / (cfg.density * cfg.h)
    p3 = s.p.reshape((nx, ny, nz), order="F")
    s.u[1:nx] -= coef * (p3[1:] - p3[:-1])
    s.v[:, 1:ny] -= coef * (p3[:, 1:] - p3[:, :-1])
    s.w[:, :, 1:nz] -= coef * (p3[:, :, 1:] - p3[:, :, :-1])
    s.u[0] -= coef * p3[0]
    s.u[nx] -= coef * (0.0 - p3[nx - 1])
    s.v[:, 0] -= coef * p3[:, 0]
    s.v[:, ny] -= coef * (0.0 - p3[:, ny - 1])
    s.w[:, :, 0] -= coef * p3[:, :, 0]
    s.w[:, :, nz] -= coef * (0.0 - p3[:, :, nz - 1])
    div_post = float(np.abs(divergence(s.u, s.v, s.w, cfg.h, cfg.threads)).max())
    enforce_boundaries(s)
    return div_post


def step(s: State, cfg: Cfg, cache: Cache | None = None) -> StepResult:
    """src/sim.py:452-474 -- one time step."""
    apply_forces(s, cfg)
    enforce_boundaries(s)
    s.u, s.v, s.w = advect(s.u, s.v, s.w, cfg.n, cfg.h, cfg.dt, cfg.threads)
    enforce_boundaries(s)
    st, div_pre = solve_pressure(s, cfg, cache)
    div_post = correct(s, cfg)
    enforce_boundaries(s)
    s.step += 1
    s.t = s.step * cfg.dt
    return StepResult(st, div_pre, div_post)


def run(cfg: Cfg):
    """src/sim.py:477-505 without snapshot output."""
    s = initial_state(cfg.n, cfg.shape)
    cache = Cache()
    results = [step(s, cfg, cache) for _ in range(cfg.num_steps)]
    return s, results


def snapshot_columns(s: State, h: float):
    """src/snapshots.py:46-62 -- cell-centred x,y,z,u,v,w,p columns."""
    n = s.u.shape[1]
    c = (np.arange(n) + 0.5) * h
    x, y, z = np.meshgrid(c, c, c, indexing="ij")
    uc = 0.5 * (s.u[:-1] + s.u[1:])
    vc = 0.5 * (s.v[:, :-1] + s.v[:, 1:])
    wc = 0.5 * (s.w[:, :, :-1] + s.w[:, :, 1:])
    f = lambda a: a.flatten(order="F")  # noqa: E731
    return {"x": f(x), "y": f(y), "z": f(z), "u": f(uc), "v": f(vc), "w": f(wc), "p": s.p.copy()}


def format_value(v: float) -> str:
    """src/snapshots.py:65-70 -- shortest round-trip repr, integral '.0' dropped."""
    s = repr(float(v))
    return s[:-2] if s.endswith(".0") else s


def snapshot_csv(cols: dict) -> bytes:
    """src/snapshots.py:73-108 -- the CSV bytes of a column dict (either mode)."""
    names = ("x", "y", "z", "u", "v", "w", "p")
    rows = zip(*(cols[c].tolist() for c in names))
    body = "".join(",".join(format_value(a) for a in r) + "\n" for r in rows)
    return ("x,y,z,u,v,w,p\n" + body).encode()
