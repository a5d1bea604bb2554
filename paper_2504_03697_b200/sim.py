"""The cavity time step on the device (mirror of src/sim.py).

Substep sequence and semantics are the reference's (src/sim.py:452-474):
forces -> walls -> semi-Lagrangian advection -> walls -> pressure solve ->
gradient correction (+ walls) -> walls.  Each substep is one sm_100a kernel
(cf_forces_bc, cf_advect, cf_divergence, the fused CG, cf_pressure_correct)
on device-resident fields; the only host synchronisations per step are the
three scalars StepStats reports (div_pre, the solve stats, div_post).

Fusions relative to the reference: forcing and the wall clamp are one
kernel; advection zeroes the wall planes itself (the reference's following
enforce_boundaries is then the identity and is skipped); the divergence
kernel emits the scaled right-hand side and max|b| in one pass; the
correction kernel computes the corrected faces, div_post and the wall clamp
in one pass, out of place into the spare velocity buffer (swapped in, as
solve_advection swaps in a new field in the reference).
"""

from __future__ import annotations

import logging
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grid import GridSpec, ScalarField, VelocityField, _divergence_into, divergence
from .precond import jacobi_from
from .solver import NULL_PROFILER, SolveStats, pcg
from .sparse import CsrMatrix, StencilOperator, SymCsrMatrix

log = logging.getLogger("cavityflow")

ROOT_REGION = "cavityflow"
PRECONDITIONERS = ("dic", "jacobi")
VARIANTS = ("baseline", "optimized")


@dataclass
class SimConfig:
    """All run parameters; defaults reproduce the reference configuration (src/sim.py:53-100)."""

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
    output_dir: str | None = None
    threads: int = 1
    advect_block: int = 8
    warm_start: bool = False
    # --- physics extension beyond the (inviscid) reference, SURVEY.md §8 f2;
    # the defaults reproduce the reference physics exactly
    viscosity: float = 0.0               # kinematic nu: explicit diffusion after advection
    lid_velocity: float | None = None    # Dirichlet lid u = U at y = L (via the diffusion ghosts)
    no_slip: bool = False                # tangential ghosts negated on the walls
    initial_pressure: float = 1.0        # the reference starts from p = 1 (dynamically inert)
    diffusion: str = "explicit"          # "explicit" | "implicit" (backward Euler, CG per component)
    diffusion_tol: float = 1e-10
    shape: tuple | None = None           # an nx*ny*nz box instead of the n-cube

    def __post_init__(self):
        if self.viscosity < 0:
            raise ValueError(f"viscosity must be >= 0, got {self.viscosity}")
        if self.diffusion not in ("explicit", "implicit"):
            raise ValueError("diffusion must be 'explicit' or 'implicit'")
        if (self.diffusion == "explicit" and self.viscosity > 0
                and self.viscosity * self.dt / (self.h * self.h) > 1.0 / 6.0):
            raise ValueError(
                f"explicit diffusion is unstable: nu*dt/h^2 = {self.viscosity * self.dt / self.h ** 2:.3f} > 1/6 "
                "(use diffusion='implicit')")
        if self.n < 2:
            raise ValueError(f"n must be >= 2, got {self.n}")
        if not self.dt > 0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if self.t_end < 0:
            raise ValueError(f"t_end must be >= 0, got {self.t_end}")
        if not self.density > 0:
            raise ValueError(f"density must be positive, got {self.density}")
        if not self.tol > 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.preconditioner not in PRECONDITIONERS:
            raise ValueError(f"preconditioner must be one of {PRECONDITIONERS}")
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}")
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        if self.advect_block < 1:
            raise ValueError(f"advect_block must be >= 1, got {self.advect_block}")

    @property
    def spec(self) -> GridSpec:
        return GridSpec(self.n, self.h, tuple(self.shape) if self.shape is not None else None)

    @property
    def num_steps(self) -> int:
        return round(self.t_end / self.dt)


@dataclass
class SimState:
    vel: VelocityField
    p: ScalarField
    t: float = 0.0
    step: int = 0


@dataclass
class StepStats:
    solve: SolveStats
    div_pre: float
    div_post: float


@dataclass
class RunReport:
    steps: list = field(default_factory=list)
    snapshot_paths: list = field(default_factory=list)
    regions: list = field(default_factory=list)
    wall_seconds: float = 0.0


def initial_state(cfg: SimConfig) -> SimState:
    """Fluid at rest under uniform unit pressure (src/sim.py:126-131)."""
    spec = cfg.spec
    p = ScalarField(spec)
    p.data.fill_(cfg.initial_pressure)
    return SimState(vel=VelocityField(spec), p=p)


def _box(vel: VelocityField):
    """(nx, ny, nz, z0, z1, halo, ldu, ldv, ldw) of the whole box for the cf_*_slab entry points."""
    nx, ny, nz = vel.spec.dims
    return (nx, ny, nz, 0, nz, 0, vel.ld[0], vel.ld[1], vel.ld[2])


def apply_forces(state: SimState, cfg: SimConfig):
    """Lid offset g*dt on the top-layer u faces (src/sim.py:134-137)."""
    nx, ny, _ = state.vel.spec.dims
    state.vel.u[1:nx, ny - 1, :] += cfg.lid_accel * cfg.dt


def enforce_boundaries(state: SimState):
    """Zero every wall-normal face (src/sim.py:140-149)."""
    lib = _lib.load_library()
    _lib.check(lib.cf_forces_bc_slab(*state.vel.ptrs(), *_box(state.vel), 0.0, 0, _lib.stream()),
               "enforce_boundaries")


def _forces_and_walls(state: SimState, cfg: SimConfig):
    lib = _lib.load_library()
    _lib.check(lib.cf_forces_bc_slab(*state.vel.ptrs(), *_box(state.vel), cfg.lid_accel * cfg.dt, 1,
                                     _lib.stream()), "forces_bc")


def _advect_into(src: VelocityField, dst: VelocityField, cfg: SimConfig):
    lib = _lib.load_library()
    _lib.check(lib.cf_advect_slab(*src.ptrs(), *dst.ptrs(), *_box(src), src.spec.h, cfg.dt, _lib.stream()),
               "advect")


def _diffuse_into(src: VelocityField, dst: VelocityField, cfg: SimConfig):
    lib = _lib.load_library()
    kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
    lid = cfg.lid_velocity
    _lib.check(lib.cf_diffuse_slab(*src.ptrs(), *dst.ptrs(), *_box(src), kdt, 0.0 if lid is None else float(lid),
                                   0 if lid is None else 1, 1 if cfg.no_slip else 0, _lib.stream()), "diffuse")


class HelmholtzOperator:
    """(I - kdt L) for one velocity component on its physical padded array
    (cf_helmholtz); an ``apply_a`` for pcg's per-op path."""

    def __init__(self, comp: int, dims: tuple, ld: int, kdt: float, lid_velocity, no_slip: bool):
        self.comp, self.dims, self.ld, self.kdt = comp, tuple(dims), ld, float(kdt)
        self.lid = 0.0 if lid_velocity is None else float(lid_velocity)
        self.dirichlet = 0 if lid_velocity is None else 1
        self.no_slip = 1 if no_slip else 0

    def _run(self, mode, x, y):
        lib = _lib.load_library()
        _lib.check(lib.cf_helmholtz(mode, self.comp, x.data_ptr() if x is not None else None, y.data_ptr(),
                                    *self.dims, self.ld, self.kdt, self.lid, self.dirichlet, self.no_slip,
                                    _lib.stream()),
                   "helmholtz")
        return y

    def __call__(self, x, out=None):
        return self._run(0, x, torch.empty_like(x) if out is None else out)

    def diagonal_tensor(self, like):
        return self._run(1, like, torch.empty_like(like))

    def rhs(self, ustar):
        return self._run(2, ustar, torch.empty_like(ustar))


def _diffuse_implicit(vel: VelocityField, cfg: SimConfig):
    """Backward-Euler diffusion in place: per component (I - kdt L) u = u*,
    Jacobi-PCG on the device (per-op path), warm-started from u*."""
    from .precond import JacobiPreconditioner

    kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
    stats = []
    for comp, phys in enumerate(vel._phys):
        flat = phys.view(-1)
        op = HelmholtzOperator(comp, vel.spec.dims, vel.ld[comp], kdt, cfg.lid_velocity, cfg.no_slip)
        b = op.rhs(flat)
        pre = JacobiPreconditioner(1.0 / op.diagonal_tensor(flat))
        x, st = pcg(op, b, x0=flat, precond=pre, tol=cfg.diffusion_tol, max_iter=10000, variant="optimized")
        flat.copy_(x)
        stats.append(st)
    return stats


def solve_diffusion(state: SimState, cfg: SimConfig) -> VelocityField:
    """Extension: one viscous diffusion step into a new field
    (explicit, or backward Euler when cfg.diffusion == 'implicit')."""
    if cfg.diffusion == "implicit":
        new = state.vel.copy()
        _diffuse_implicit(new, cfg)
        return new
    new = VelocityField(state.vel.spec)
    _diffuse_into(state.vel, new, cfg)
    return new


def solve_advection(state: SimState, cfg: SimConfig, pool=None) -> VelocityField:
    """Semi-Lagrangian backtrace + resample into a new field (src/sim.py:259-289)."""
    new = VelocityField(state.vel.spec)
    _advect_into(state.vel, new, cfg)
    return new


def poisson_full_csr(n: int, h: float) -> CsrMatrix:
    """7-point negative Laplacian, Dirichlet ghost pressure, full CSR (src/sim.py:296-317)."""
    num = n ** 3
    idx = np.arange(num, dtype=np.int64)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    nn = n * n
    cols = np.stack([idx - nn, idx - n, idx - 1, idx, idx + 1, idx + n, idx + nn], axis=1)
    exists = np.stack([k > 0, j > 0, i > 0, np.ones(num, dtype=bool), i < n - 1, j < n - 1, k < n - 1], axis=1)
    vals = np.full((num, 7), -1.0 / (h * h))
    vals[:, 3] = 6.0 / (h * h)
    ptr = np.concatenate(([0], np.cumsum(exists.sum(axis=1))))
    keep = exists.ravel()
    return CsrMatrix(num, num, ptr, cols.ravel()[keep], vals.ravel()[keep])


def poisson_symmetric(n: int, h: float) -> SymCsrMatrix:
    """Same operator as diagonal + strict upper triangle (src/sim.py:320-333)."""
    num = n ** 3
    idx = np.arange(num, dtype=np.int64)
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    cols = np.stack([idx + 1, idx + n, idx + n * n], axis=1)
    exists = np.stack([i < n - 1, j < n - 1, k < n - 1], axis=1)
    vals = np.full((num, 3), -1.0 / (h * h))
    ptr = np.concatenate(([0], np.cumsum(exists.sum(axis=1))))
    keep = exists.ravel()
    return SymCsrMatrix(num, np.full(num, 6.0 / (h * h)), ptr, cols.ravel()[keep], vals.ravel()[keep])


def _build_preconditioner(a, kind: str):
    """src/sim.py:375-376 (built once per cached operator here: the matrix is constant)."""
    from .precond import dic_from

    return dic_from(a) if kind == "dic" else jacobi_from(a)


class PoissonCache:
    """Per-grid device state reused across steps (src/sim.py:336-349).

    ``matrix`` keeps the reference meaning (the symmetric pattern for the
    optimized variant).  On the device the solve never streams a matrix: it
    uses the matrix-free operator and the fused-CG workspace held here, plus
    the right-hand-side buffer and the spare velocity field.
    """

    def __init__(self):
        self.matrix: SymCsrMatrix | None = None
        self._ops = {}
        self._precond = {}
        self.rhs: torch.Tensor | None = None
        self.spare: VelocityField | None = None

    def refresh_values(self, n: int, h: float):
        self.matrix.diag[:] = 6.0 / (h * h)
        self.matrix.values[:] = -1.0 / (h * h)

    def operator(self, cfg: SimConfig) -> StencilOperator:
        # optimized variant <-> spmv_sym order, baseline <-> spmv (CSR) order
        key = (cfg.n, cfg.h, cfg.variant, cfg.spec.dims)
        if key not in self._ops:
            self._ops[key] = StencilOperator(cfg.n, cfg.h, "sym" if cfg.variant == "optimized" else "csr",
                                             shape=cfg.spec.dims)
        return self._ops[key]

    def preconditioner(self, cfg: SimConfig, op: StencilOperator):
        key = (cfg.n, cfg.h, cfg.preconditioner, cfg.spec.dims)
        if key not in self._precond:
            self._precond[key] = _build_preconditioner(op, cfg.preconditioner)
        return self._precond[key]

    def rhs_buffer(self, spec: GridSpec) -> torch.Tensor:
        if self.rhs is None or self.rhs.shape[0] != spec.num_cells:
            self.rhs = torch.empty(spec.num_cells, dtype=torch.float64, device=torch.device("cuda"))
        return self.rhs

    def spare_field(self, spec: GridSpec) -> VelocityField:
        if self.spare is None or self.spare.spec != spec:
            self.spare = VelocityField(spec)
        return self.spare


def assemble_pressure_system(state: SimState, cfg: SimConfig, cache: PoissonCache | None = None):
    """(A, b) with b = -(rho/dt) * divergence (src/sim.py:352-372)."""
    div = divergence(state.vel)
    b = (-cfg.density / cfg.dt) * div.data
    if cfg.variant == "optimized":
        if cache is None:
            a = poisson_symmetric(cfg.n, cfg.h)
        elif cache.matrix is None:
            cache.matrix = poisson_symmetric(cfg.n, cfg.h)
            a = cache.matrix
        else:
            cache.refresh_values(cfg.n, cfg.h)
            a = cache.matrix
    else:
        a = poisson_full_csr(cfg.n, cfg.h)
    return a, b


def solve_pressure_correction(state: SimState, cfg: SimConfig, cache: PoissonCache | None = None,
                              pool=None, profiler=None):
    """Pressure Poisson solve into state.p (src/sim.py:379-423).

    Returns ``(pressure, stats, div_pre)``.  The operator is the matrix-free
    stencil in the variant's SpMV summation order; b is produced straight
    into the device RHS buffer by the divergence kernel.
    """
    prof = profiler if profiler is not None else NULL_PROFILER
    cache = cache if cache is not None else PoissonCache()
    b = cache.rhs_buffer(state.vel.spec)
    max_b = _divergence_into(state.vel, -cfg.density / cfg.dt, b, want_max=True)
    div_pre = float(max_b) * cfg.dt / cfg.density
    op = cache.operator(cfg)
    precond = cache.preconditioner(cfg, op)
    x0 = state.p.data if (cfg.warm_start and state.step > 0) else None
    with prof.region("pcg"):
        x, stats = pcg(op, b, x0=x0, precond=precond, tol=cfg.tol, max_iter=cfg.max_iter,
                       variant=cfg.variant, pool=pool, profiler=prof)
    if not stats.converged:
        log.warning(
            "pressure solve did not converge in %d iterations (rel residual %.3e); "
            "continuing with best iterate", stats.iterations, stats.final_residual_rel)
    state.p.data.copy_(x)
    return state.p, stats, div_pre


def _correct_into(src: VelocityField, dst: VelocityField, p: ScalarField, cfg: SimConfig) -> float:
    lib = _lib.load_library()
    coef = cfg.dt / (cfg.density * cfg.h)
    out = _lib.dbl_out()
    _lib.check(lib.cf_pressure_correct_slab(*src.ptrs(), *dst.ptrs(), p.data.data_ptr(), *_box(src), cfg.h, coef,
                                            _lib.byref(out), _lib.stream()), "pressure_correct")
    return float(out.value)


def apply_pressure_correction(state: SimState, p: ScalarField, cfg: SimConfig) -> float:
    """Subtract (dt/rho) grad p, report div_post, clamp walls (src/sim.py:426-449)."""
    tmp = VelocityField(state.vel.spec)
    div_post = _correct_into(state.vel, tmp, p, cfg)
    state.vel.copy_from(tmp)  # in place, as the reference mutates state.vel
    return div_post


def step(state: SimState, cfg: SimConfig, cache: PoissonCache | None = None, pool=None,
         profiler=None) -> StepStats:
    """Advance one time step (src/sim.py:452-474)."""
    prof = profiler if profiler is not None else NULL_PROFILER
    cache = cache if cache is not None else PoissonCache()
    spec = state.vel.spec
    with prof.region("applyForces"):
        _forces_and_walls(state, cfg)  # + enforce_boundaries
    with prof.region("solveAdvection"):
        new = cache.spare_field(spec)
        _advect_into(state.vel, new, cfg)  # wall planes zeroed in-kernel
        cache.spare, state.vel = state.vel, new
    if cfg.viscosity > 0.0:  # extension: viscous diffusion
        with prof.region("solveDiffusion"):
            if cfg.diffusion == "implicit":
                _diffuse_implicit(state.vel, cfg)
            else:
                new = cache.spare_field(spec)
                _diffuse_into(state.vel, new, cfg)
                cache.spare, state.vel = state.vel, new
    with prof.region("solvePressureCorrection"):
        p, stats, div_pre = solve_pressure_correction(state, cfg, cache, pool, prof)
    with prof.region("applyPressureCorrection"):
        dst = cache.spare_field(spec)
        div_post = _correct_into(state.vel, dst, p, cfg)  # + walls
        cache.spare, state.vel = state.vel, dst
    state.step += 1
    state.t = state.step * cfg.dt
    return StepStats(solve=stats, div_pre=div_pre, div_post=div_post)


def run(cfg: SimConfig, profiler=None):
    """Run the configured simulation (src/sim.py:477-505).  ``profiler``
    (extension) is a fresh ``Profiler`` to time with, e.g.
    ``Profiler(timer="events")``; the default is the reference's wall clock."""
    from .profiling import Profiler
    from . import snapshots

    state = initial_state(cfg)
    report = RunReport()
    profiler = Profiler() if profiler is None else profiler
    cache = PoissonCache()
    if cfg.output_dir is not None:
        os.makedirs(cfg.output_dir, exist_ok=True)

    def write(step_index: int):
        if cfg.output_dir is None:
            return
        path = os.path.join(cfg.output_dir, snapshots.snapshot_filename(step_index))
        with profiler.region("write_to_file"):
            snapshots.write_snapshot(state, path)
        report.snapshot_paths.append(path)

    with profiler.region(ROOT_REGION):
        write(0)
        for _ in range(cfg.num_steps):
            report.steps.append(step(state, cfg, cache, None, profiler))
            write(state.step)
    report.regions = profiler.stats()
    for rec in report.regions:
        if rec.name == ROOT_REGION:
            report.wall_seconds = rec.inclusive_seconds
    return state, report
