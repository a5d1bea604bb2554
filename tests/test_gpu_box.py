"""GPU: non-cubic nx*ny*nz boxes (extension) against the
oracle's box restatement (oracle/__init__.py, ``shape=``).

The reference only builds the n-cube; the box generalises every index
formula (cell id i + nx*(j + ny*k), face extents) without touching the
arithmetic, so the same bars apply as for the cube:
  * bit-exact: stencil (both summation orders), advection, divergence,
    pressure correction + div_post, explicit diffusion;
  * CG: iterations within +-2 of the oracle; solution rel-L2 <= 1e-8 at
    tol 1e-10;
  * whole runs at CG tol 1e-6: velocity rel-L2 <= 1e-7, pressure <= 1e-6;
  * emulated z-slabs vs the single-domain box at tol 1e-12: rel-L2 1e-10.
Shapes are chosen to hit every device path: the single-block small CG
(n^3 <= 5120), the LDG stencil (odd nx), and the TMA pipeline (nx >= 32,
even, ny not a multiple of the 16-row tile).
"""

import numpy as np
import pytest
import torch

import oracle as orc
from oracle import physics_ext as ext

pytestmark = pytest.mark.gpu

BOXES = [(7, 5, 9), (16, 12, 20), (33, 10, 14), (48, 20, 24)]


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def random_field(shape, seed, scale=0.3):
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    u = scale * rng.standard_normal((nx + 1, ny, nz))
    v = scale * rng.standard_normal((nx, ny + 1, nz))
    w = scale * rng.standard_normal((nx, ny, nz + 1))
    u[0] = u[nx] = 0.0
    v[:, 0] = v[:, ny] = 0.0
    w[:, :, 0] = w[:, :, nz] = 0.0
    return u, v, w


def flat(*arrs):
    return np.concatenate([np.asarray(a).ravel() for a in arrs])


@pytest.mark.parametrize("shape", BOXES)
@pytest.mark.parametrize("order", ["csr", "sym"])
def test_box_stencil_bitwise(cuda, shape, order):
    h = 1.0 / max(shape)
    op = cuda.StencilOperator(max(shape), h, order, shape=shape)
    x = np.random.default_rng(1).standard_normal(int(np.prod(shape)))
    got = op(torch.as_tensor(x, device="cuda")).cpu().numpy()
    if order == "csr":
        want = orc.spmv(orc.poisson_csr(0, h, shape), x)
    else:
        want = orc.spmv_sym(orc.poisson_sym(0, h, shape), x)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("shape", BOXES)
def test_box_step_kernels_bitwise(cuda, shape):
    from paper_2504_03697_b200 import sim

    nx, ny, nz = shape
    h, dt = 1.0 / max(shape), 0.05
    u, v, w = random_field(shape, 7)
    cfg = cuda.SimConfig(n=max(shape), h=h, dt=dt, t_end=0.0, shape=shape)
    p = np.random.default_rng(8).standard_normal(nx * ny * nz)
    st = cuda.SimState(vel=cuda.VelocityField(cfg.spec, u, v, w), p=cuda.ScalarField(cfg.spec, p))
    new = sim.solve_advection(st, cfg)
    want = orc.advect(u, v, w, max(shape), h, dt)
    for c, a, b in zip("uvw", new.numpy(), want):
        assert np.array_equal(a, b), c
    assert np.array_equal(cuda.divergence(st.vel).numpy(), orc.divergence(u, v, w, h))
    st2 = cuda.SimState(vel=new, p=st.p)
    div_post = sim.apply_pressure_correction(st2, st.p, cfg)
    ost = orc.State(*(a.copy() for a in want), p.copy())
    assert div_post == orc.correct(ost, orc.Cfg(n=max(shape), h=h, dt=dt, shape=shape))
    for c, a, b in zip("uvw", st2.vel.numpy(), (ost.u, ost.v, ost.w)):
        assert np.array_equal(a, b), c


@pytest.mark.parametrize("shape", [(33, 10, 14), (32, 16, 8)])
def test_box_step_kernels_flat_forms(cuda, monkeypatch, shape):
    """The one-thread-per-cell forms of the divergence / correction / diffusion
    kernels (CF_DIVERGENCE / CF_CORRECT / CF_DIFFUSE = flat) against the
    z-marches that replaced them as the default: bit-identical outputs (both
    are also pinned to the oracle by the tests around this one), with h a
    power of two (32: the exact-multiplication branch) and not."""
    from paper_2504_03697_b200 import sim
    from paper_2504_03697_b200.sim import solve_diffusion

    nx, ny, nz = shape
    n = max(shape)
    u, v, w = random_field(shape, 11)
    p = np.random.default_rng(12).standard_normal(nx * ny * nz)
    cfg = cuda.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.0, viscosity=0.05 * (24.0 / n) ** 2 / 4,
                         lid_velocity=1.0, no_slip=True, shape=shape)
    out = []
    for form in ("flat", None):
        for k in ("CF_DIVERGENCE", "CF_CORRECT", "CF_DIFFUSE"):
            if form:
                monkeypatch.setenv(k, form)
            else:
                monkeypatch.delenv(k, raising=False)
        st = cuda.SimState(vel=cuda.VelocityField(cfg.spec, u, v, w), p=cuda.ScalarField(cfg.spec, p))
        div = cuda.divergence(st.vel).numpy()
        dif = solve_diffusion(st, cfg).numpy()
        div_post = sim.apply_pressure_correction(st, st.p, cfg)
        out.append((div, flat(*dif), div_post, flat(*st.vel.numpy())))
    for a, b in zip(*out):
        assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("shape", [(16, 12, 20), (48, 20, 24)])
def test_box_diffusion_bitwise(cuda, shape):
    from paper_2504_03697_b200.sim import solve_diffusion

    n = max(shape)
    u, v, w = random_field(shape, 3)
    cfg = cuda.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.0, viscosity=0.05 * (24.0 / n) ** 2 / 4,
                         lid_velocity=1.0, no_slip=True, shape=shape)
    st = cuda.SimState(vel=cuda.VelocityField(cfg.spec, u, v, w), p=cuda.ScalarField(cfg.spec))
    got = solve_diffusion(st, cfg).numpy()
    kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
    for g, wv in zip(got, ext.diffuse(u, v, w, n, kdt, 1.0, True)):
        assert np.array_equal(g, wv)


@pytest.mark.parametrize("shape", BOXES)
@pytest.mark.parametrize("precond", ["jacobi", "dic"])
def test_box_pcg_vs_oracle(cuda, shape, precond):
    h = 1.0 / max(shape)
    op = cuda.StencilOperator(max(shape), h, "sym", shape=shape)
    b = np.random.default_rng(2).standard_normal(int(np.prod(shape)))
    pc = cuda.jacobi_from(op) if precond == "jacobi" else cuda.dic_from(op)
    x, st = cuda.pcg(op, torch.as_tensor(b, device="cuda"), precond=pc, tol=1e-10, max_iter=5000)
    a = orc.poisson_sym(0, h, shape)
    opc = orc.jacobi_from(a) if precond == "jacobi" else orc.Dic(a)
    xo, so = orc.pcg(lambda v, o: orc.spmv_sym(a, v, 1, o), b, precond=opc, tol=1e-10, max_iter=5000)
    assert st.converged and so.converged
    assert abs(st.iterations - so.iterations) <= 2, (st.iterations, so.iterations)
    assert rel(x.cpu().numpy(), xo) <= 1e-8


@pytest.mark.parametrize("shape", [(16, 12, 20), (48, 20, 24)])
def test_box_cavity_run_vs_oracle(cuda, shape):
    n = max(shape)
    kw = dict(n=n, h=1.0 / n, dt=0.01, t_end=0.05, tol=1e-6, max_iter=10000, variant="optimized",
              preconditioner="jacobi", shape=shape)
    cfg = cuda.SimConfig(**kw)
    st = cuda.initial_state(cfg)
    cache = cuda.PoissonCache()
    ocfg = orc.Cfg(**kw)
    ost = orc.initial_state(n, shape)
    ocache = orc.Cache()
    for _ in range(cfg.num_steps):
        a = cuda.step(st, cfg, cache)
        b = orc.step(ost, ocfg, ocache)
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
        assert a.div_pre == pytest.approx(b.div_pre, rel=1e-6)
        assert a.div_post <= 1e-3 * a.div_pre
    u, v, w = st.vel.numpy()
    assert rel(flat(u, v, w), flat(ost.u, ost.v, ost.w)) <= 1e-7
    assert rel(st.p.numpy(), ost.p) <= 1e-6


def test_box_extension_physics_run(cuda):
    """Lid velocity + no-slip + explicit diffusion on a 24x16x32 box vs the restatement."""
    shape = (24, 16, 32)
    n = max(shape)
    kw = dict(n=n, h=1.0 / n, dt=0.01, t_end=0.04, tol=1e-6, max_iter=10000, variant="optimized",
              preconditioner="jacobi", lid_accel=0.0, shape=shape)
    ekw = dict(viscosity=0.01, lid_velocity=1.0, no_slip=True)
    cfg = cuda.SimConfig(initial_pressure=0.0, **kw, **ekw)
    st = cuda.initial_state(cfg)
    cache = cuda.PoissonCache()
    ocfg = ext.ExtCfg(**kw, **ekw)
    ost = orc.initial_state(n, shape)
    ost.p[:] = 0.0
    for _ in range(cfg.num_steps):
        a = cuda.step(st, cfg, cache)
        b = ext.step(ost, ocfg, orc.Cache())
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
    u, v, w = st.vel.numpy()
    assert rel(flat(u, v, w), flat(ost.u, ost.v, ost.w)) <= 1e-7
    assert rel(st.p.numpy(), ost.p) <= 1e-6


@pytest.mark.parametrize("shape,bounds", [((40, 24, 30), [0, 9, 20, 30]), ((34, 17, 12), [0, 6, 12])])
def test_box_slabs_match_single_domain(cuda, shape, bounds):
    from paper_2504_03697_b200.distributed import SlabSim

    n = max(shape)
    cfg = cuda.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.03, tol=1e-12, max_iter=20000, variant="optimized",
                         preconditioner="jacobi", shape=shape)
    u0, v0, w0 = random_field(shape, 11, scale=0.5)
    ref = cuda.initial_state(cfg)
    ref.vel.load_host(u0, v0, w0)
    cache = cuda.PoissonCache()
    sim = SlabSim(cfg, bounds)
    sim.load_global(u0, v0, w0)
    for _ in range(cfg.num_steps):
        a = cuda.step(ref, cfg, cache)
        b = sim.step()
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
        assert b.div_pre == pytest.approx(a.div_pre, rel=1e-12)
    su, sv, sw, sp = sim.gather()
    ru, rv, rw = ref.vel.numpy()
    assert rel(flat(su, sv, sw), flat(ru, rv, rw)) <= 1e-10
    assert rel(sp, ref.p.numpy()) <= 1e-9


def test_box_slabs_need_tma_rows(cuda):
    """The NCCL z-slab solver is TMA-only (even nx >= 32); the peer-memory one needs an even nx."""
    from paper_2504_03697_b200.distributed import SlabSim

    cfg = cuda.SimConfig(n=33, h=1.0 / 33, dt=0.01, t_end=0.01, shape=(17, 33, 12),
                         preconditioner="jacobi", variant="optimized")
    with pytest.raises(ValueError, match="even nx >= 32"):
        SlabSim(cfg, [0, 6, 12], collective="nccl")
    with pytest.raises(ValueError, match="nx even"):
        SlabSim(cfg, [0, 6, 12])
