"""GPU: physics extension beyond the reference --
viscous diffusion, moving-lid Dirichlet wall, no-slip walls -- against the
repo's numpy restatement (oracle/physics_ext.py).  The reference is inviscid
so nothing upstream pins this physics; parity here is kernel == restatement,
bit-exact for the diffusion kernel, rel-L2 1e-7 (velocity) / 1e-6 (pressure)
for whole steps at CG tol 1e-6 (reduction order only).
"""

import numpy as np
import pytest

import oracle as orc
from oracle import physics_ext as ext

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def random_field(n, seed, scale=0.3):
    rng = np.random.default_rng(seed)
    u = scale * rng.standard_normal((n + 1, n, n))
    v = scale * rng.standard_normal((n, n + 1, n))
    w = scale * rng.standard_normal((n, n, n + 1))
    u[0] = u[n] = 0.0
    v[:, 0] = v[:, n] = 0.0
    w[:, :, 0] = w[:, :, n] = 0.0
    return u, v, w


@pytest.mark.parametrize("lid,no_slip", [(None, False), (None, True), (1.0, True), (0.5, False)])
def test_diffusion_kernel_bitwise(cuda, lid, no_slip):
    from paper_2504_03697_b200.sim import solve_diffusion

    n = 12
    u, v, w = random_field(n, 3)
    cfg = cuda.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.0, viscosity=0.05, lid_velocity=lid, no_slip=no_slip)
    st = cuda.SimState(vel=cuda.VelocityField(cfg.spec, u, v, w), p=cuda.ScalarField(cfg.spec))
    got = solve_diffusion(st, cfg).numpy()
    kdt = 0.05 * 0.01 / (1.0 / n) ** 2
    want = ext.diffuse(u, v, w, n, kdt, lid, no_slip)
    for g, wv in zip(got, want):
        assert np.array_equal(g, wv)


def test_config1_physics_run_vs_restatement(cuda):
    """BASELINE config 1 in full: 16^3, nu=0.01, lid velocity 1 (no lid
    acceleration), no-slip, p0 = 0, dt=0.01, 10 steps, CG tol 1e-6."""
    kw = dict(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000, variant="optimized",
              preconditioner="jacobi", lid_accel=0.0)
    ekw = dict(viscosity=0.01, lid_velocity=1.0, no_slip=True)
    cfg = cuda.SimConfig(initial_pressure=0.0, **kw, **ekw)
    st = cuda.initial_state(cfg)
    cache = cuda.PoissonCache()
    ocfg = ext.ExtCfg(**kw, **ekw)
    ost = orc.initial_state(16)
    ost.p[:] = 0.0
    ocache = orc.Cache()
    for _ in range(cfg.num_steps):
        a = cuda.step(st, cfg, cache)
        b = ext.step(ost, ocfg, ocache)
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
    u, v, w = st.vel.numpy()
    assert rel(np.concatenate([u.ravel(), v.ravel(), w.ravel()]),
               np.concatenate([ost.u.ravel(), ost.v.ravel(), ost.w.ravel()])) <= 1e-7
    assert rel(st.p.numpy(), ost.p) <= 1e-6
    # the lid drives the flow: positive u under the lid
    assert u[1:16, 15, :].mean() > 0.0


def test_explicit_diffusion_stability_guard(cuda):
    with pytest.raises(ValueError, match="unstable"):
        cuda.SimConfig(n=512, h=1.0 / 512, dt=0.001, viscosity=0.001)  # BASELINE config 5: 0.262 > 1/6


def test_slab_run_with_extension_physics(cuda):
    """Config-4 physics on emulated z-slabs equals the single-domain run."""
    from paper_2504_03697_b200.distributed import SlabSim

    n = 32
    kw = dict(n=n, h=1.0 / n, dt=0.01, t_end=0.03, tol=1e-12, max_iter=20000, variant="optimized",
              preconditioner="jacobi", lid_accel=0.0, viscosity=0.01, lid_velocity=1.0, no_slip=True)
    cfg = cuda.SimConfig(**kw)
    ref = cuda.initial_state(cfg)
    cache = cuda.PoissonCache()
    sim = SlabSim(cfg, [0, 11, 20, 32])
    for _ in range(cfg.num_steps):
        a = cuda.step(ref, cfg, cache)
        b = sim.step()
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
    su, sv, sw, _ = sim.gather()
    ru, rv, rw = ref.vel.numpy()
    assert rel(np.concatenate([su.ravel(), sv.ravel(), sw.ravel()]),
               np.concatenate([ru.ravel(), rv.ravel(), rw.ravel()])) <= 1e-10


@pytest.mark.parametrize("lid,no_slip", [(None, False), (1.0, True)])
def test_implicit_diffusion_vs_restatement(cuda, lid, no_slip):
    """Backward-Euler diffusion (CG per component, device per-op path) against
    the oracle's restatement, both solved to tol 1e-12: rel-L2 <= 1e-9."""
    from paper_2504_03697_b200.sim import solve_diffusion

    n = 12
    u, v, w = random_field(n, 5)
    nu = 0.3 * (1.0 / n) ** 2 / 0.01  # nu*dt/h^2 = 0.3 > 1/6: explicit would be unstable
    cfg = cuda.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.0, viscosity=nu, lid_velocity=lid, no_slip=no_slip,
                         diffusion="implicit", diffusion_tol=1e-12)
    st = cuda.SimState(vel=cuda.VelocityField(cfg.spec, u, v, w), p=cuda.ScalarField(cfg.spec))
    got = solve_diffusion(st, cfg).numpy()
    want = ext.diffuse_implicit(u, v, w, n, 0.3, lid, no_slip, tol=1e-12)
    for g, wv in zip(got, want):
        assert rel(g, wv) <= 1e-9


def test_config5_ratio_implicit_run(cuda):
    """Config-5 diffusion number (nu*dt/h^2 = 0.262) on a 32^3 run: implicit
    diffusion, lid velocity, no-slip; matches the restatement step by step."""
    n = 32
    h, dt = 1.0 / n, 0.01
    nu = 0.262 * h * h / dt
    kw = dict(n=n, h=h, dt=dt, t_end=0.02, tol=1e-8, max_iter=20000, variant="optimized",
              preconditioner="jacobi", lid_accel=0.0)
    ekw = dict(viscosity=nu, lid_velocity=1.0, no_slip=True, diffusion="implicit", diffusion_tol=1e-12)
    cfg = cuda.SimConfig(**kw, **ekw)
    st = cuda.initial_state(cfg)
    cache = cuda.PoissonCache()
    ost = orc.initial_state(n)
    ocfg = ext.ExtCfg(**kw, **ekw)
    for _ in range(cfg.num_steps):
        a = cuda.step(st, cfg, cache)
        b = ext.step(ost, ocfg, orc.Cache())
        assert abs(a.solve.iterations - b.solve.iterations) <= 2
    u, v, w = st.vel.numpy()
    assert rel(np.concatenate([u.ravel(), v.ravel(), w.ravel()]),
               np.concatenate([ost.u.ravel(), ost.v.ravel(), ost.w.ravel()])) <= 1e-8
