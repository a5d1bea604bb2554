"""Oracle for the physics EXTENSION -- TEST INFRASTRUCTURE.

The reference is inviscid; BASELINE configs 1,
4, 5 add viscosity, a moving lid and no-slip walls.  Parity for these is NOT
pinned by the reference (there is nothing to pin against): this module is the
repo's own numpy restatement of the extension, written in the conventions of
src/sim.py, and the CUDA kernels are checked against it bit-for-bit.

Explicit diffusion on each component's lattice (same operation order as
cf_diffuse in include/cfgpu.h):

    new = c + kdt * (((((( xm + xp) + ym) + yp) + zm) + zp) - 6*c),   kdt = nu*dt/h^2

with tangential ghosts across walls mirrored (free slip) or negated (no
slip); the lid y = L, when it has a velocity U, is a Dirichlet wall:
ghost u = 2U - c, ghost w = -c.  Wall-normal faces stay zero.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import Cfg, advect, apply_forces, correct, enforce_boundaries, solve_pressure, StepResult


def _neighbours(a, axis, lo_ghost, hi_ghost):
    """(minus, plus) neighbour arrays of `a` along `axis`, ghosts at the ends."""
    m = np.empty_like(a)
    p = np.empty_like(a)
    sl = [slice(None)] * 3

    def idx(s):
        t = list(sl)
        t[axis] = s
        return tuple(t)

    m[idx(slice(1, None))] = a[idx(slice(None, -1))]
    m[idx(slice(0, 1))] = lo_ghost(a[idx(slice(0, 1))])
    p[idx(slice(None, -1))] = a[idx(slice(1, None))]
    p[idx(slice(-1, None))] = hi_ghost(a[idx(slice(-1, None))])
    return m, p


def diffuse(u, v, w, n, kdt, lid_u=None, no_slip=False):
    """One explicit diffusion step of (u, v, w) (C order [i, j, k])."""
    wallg = (lambda c: -c) if no_slip else (lambda c: c)
    out = []
    for comp, a in enumerate((u, v, w)):
        ghosts = []
        for axis in range(3):
            if axis == comp:  # own axis: the wall-normal faces exist (zero)
                ghosts.append((lambda c: np.zeros_like(c), lambda c: np.zeros_like(c)))
                continue
            hi = wallg
            if axis == 1 and lid_u is not None:  # the lid, a Dirichlet wall
                hi = (lambda c: 2.0 * lid_u - c) if comp == 0 else (lambda c: -c)
            ghosts.append((wallg, hi))
        xm, xp = _neighbours(a, 0, *ghosts[0])
        ym, yp = _neighbours(a, 1, *ghosts[1])
        zm, zp = _neighbours(a, 2, *ghosts[2])
        s = xm + xp
        s = s + ym
        s = s + yp
        s = s + zm
        s = s + zp
        s = s - 6.0 * a
        new = a + kdt * s
        if comp == 0:
            new[0], new[-1] = 0.0, 0.0
        elif comp == 1:
            new[:, 0], new[:, -1] = 0.0, 0.0
        else:
            new[:, :, 0], new[:, :, -1] = 0.0, 0.0
        out.append(new)
    return tuple(out)


def helmholtz_apply(comp, x, n, kdt, lid_u=None, no_slip=False):
    """(I - kdt L) x for one component array (reference C-order layout).
    Ghosts fold into the diagonal (+1 mirror / -1 negate; the moving lid is a
    -1); along the component's own axis the wall faces are fixed zeros (no
    term).  Wall-normal faces are identity rows."""
    g = -1.0 if no_slip else 1.0
    shape = x.shape
    idx = np.indices(shape)
    s = np.zeros_like(x)
    gsum = np.zeros_like(x)
    for axis in range(3):
        pos = idx[axis]
        hi_lim = shape[axis] - 1
        if axis == comp:  # own axis: real neighbours only between the walls
            has_m, has_p = pos > 1, pos < hi_lim - 1
        else:
            has_m, has_p = pos > 0, pos < hi_lim
        xm = np.zeros_like(x)
        xp = np.zeros_like(x)
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[axis], sl_hi[axis] = slice(1, None), slice(None, -1)
        xm[tuple(sl_lo)] = x[tuple(sl_hi)]
        xp[tuple(sl_hi)] = x[tuple(sl_lo)]
        s = s + np.where(has_m, xm, 0.0) + np.where(has_p, xp, 0.0)
        if axis != comp:
            gsum = gsum + np.where(has_m, 0.0, g)
            if axis == 1 and lid_u is not None:
                gsum = gsum + np.where(has_p, 0.0, -1.0)
            else:
                gsum = gsum + np.where(has_p, 0.0, g)
    y = (1.0 + kdt * (6.0 - gsum)) * x - kdt * s
    wall = idx[comp]
    fixed = (wall == 0) | (wall == shape[comp] - 1)
    return np.where(fixed, x, y), np.where(fixed, 1.0, 1.0 + kdt * (6.0 - gsum))


def diffuse_implicit(u, v, w, n, kdt, lid_u=None, no_slip=False, tol=1e-10):
    """Backward Euler per component with the oracle's Jacobi-PCG (src/solver.py)."""
    from . import Jacobi, pcg

    out = []
    for comp, a in enumerate((u, v, w)):
        shape = a.shape

        def op(vec, o, comp=comp, shape=shape):
            o[:] = helmholtz_apply(comp, vec.reshape(shape), n, kdt, lid_u, no_slip)[0].ravel()
            return o

        _, dia = helmholtz_apply(comp, a, n, kdt, lid_u, no_slip)
        b = a.copy()
        if lid_u is not None and comp == 0:
            b[1:shape[0] - 1, shape[1] - 1, :] += kdt * (2.0 * lid_u)
        x, _ = pcg(op, b.ravel(), x0=a.ravel(), precond=Jacobi(dia.ravel()), tol=tol, max_iter=10000)
        out.append(x.reshape(shape))
    return tuple(out)


@dataclass
class ExtCfg(Cfg):
    viscosity: float = 0.0
    lid_velocity: float | None = None
    no_slip: bool = False
    diffusion: str = "explicit"
    diffusion_tol: float = 1e-10


def step(s, cfg: ExtCfg, cache=None) -> StepResult:
    """forces -> walls -> advect -> walls -> diffuse -> project -> walls."""
    apply_forces(s, cfg)
    enforce_boundaries(s)
    s.u, s.v, s.w = advect(s.u, s.v, s.w, cfg.n, cfg.h, cfg.dt, cfg.threads)
    enforce_boundaries(s)
    if cfg.viscosity > 0.0:
        kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
        if cfg.diffusion == "implicit":
            s.u, s.v, s.w = diffuse_implicit(s.u, s.v, s.w, cfg.n, kdt, cfg.lid_velocity, cfg.no_slip,
                                             cfg.diffusion_tol)
        else:
            s.u, s.v, s.w = diffuse(s.u, s.v, s.w, cfg.n, kdt, cfg.lid_velocity, cfg.no_slip)
    st, div_pre = solve_pressure(s, cfg, cache)
    div_post = correct(s, cfg)
    enforce_boundaries(s)
    s.step += 1
    s.t = s.step * cfg.dt
    return StepResult(st, div_pre, div_post)
