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
            new[0], new[n] = 0.0, 0.0
        elif comp == 1:
            new[:, 0], new[:, n] = 0.0, 0.0
        else:
            new[:, :, 0], new[:, :, n] = 0.0, 0.0
        out.append(new)
    return tuple(out)


@dataclass
class ExtCfg(Cfg):
    viscosity: float = 0.0
    lid_velocity: float | None = None
    no_slip: bool = False


def step(s, cfg: ExtCfg, cache=None) -> StepResult:
    """forces -> walls -> advect -> walls -> diffuse -> project -> walls."""
    apply_forces(s, cfg)
    enforce_boundaries(s)
    s.u, s.v, s.w = advect(s.u, s.v, s.w, cfg.n, cfg.h, cfg.dt, cfg.threads)
    enforce_boundaries(s)
    if cfg.viscosity > 0.0:
        kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
        s.u, s.v, s.w = diffuse(s.u, s.v, s.w, cfg.n, kdt, cfg.lid_velocity, cfg.no_slip)
    st, div_pre = solve_pressure(s, cfg, cache)
    div_post = correct(s, cfg)
    enforce_boundaries(s)
    s.step += 1
    s.t = s.step * cfg.dt
    return StepResult(st, div_pre, div_post)
