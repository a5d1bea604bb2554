"""GPU: the reference's known-answer, property and determinism checks
 replayed through the device path.

Bars: exact where the reference pins bits (maxpy == add(scale), the unit
pressure gradient, wall sealing, run determinism); the reference's own
tolerances elsewhere (spmv_sym vs spmv 1e-14, variant equivalence 1e-9,
DIC <= half the Jacobi iterations, positive lid-driven circulation).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def test_unit_pressure_gradient_shifts_interior_u(cuda):
    """p = x at the cell centres subtracts dt/(rho h) * h = dt from every
    interior u face (tests/test_sim.py:304-312 of the reference)."""
    from paper_2504_03697_b200 import sim

    cfg = cuda.SimConfig(n=4, dt=0.4, t_end=0.4, density=1.0)
    st = cuda.initial_state(cfg)
    p = cuda.ScalarField(cfg.spec)
    c = (np.arange(4) + 0.5) * cfg.h
    p3 = np.broadcast_to(c[:, None, None], (4, 4, 4))
    p.data.copy_(dev(p3.flatten(order="F")))
    sim.apply_pressure_correction(st, p, cfg)
    u = st.vel.numpy()[0]
    assert np.allclose(u[1:-1], -0.4, rtol=1e-14, atol=0.0)
    # a constant pressure leaves the interior untouched (ghost p = 0 only at the walls)
    st2 = cuda.initial_state(cfg)
    st2.vel.u[:] = 1.0
    sim.enforce_boundaries(st2)
    before = st2.vel.numpy()[0][1:-1].copy()
    p.data.fill_(3.0)
    sim.apply_pressure_correction(st2, p, cfg)
    assert np.array_equal(st2.vel.numpy()[0][1:-1], before)


def test_maxpy_equals_add_of_scale_bitwise(cuda):
    """y += a x is bit-identical to add(y, scale(a, x)): no FMA contraction."""
    rng = np.random.default_rng(1234)
    x, y = rng.standard_normal(100_003), rng.standard_normal(100_003)
    for a in (0.1, -3.7, 1e-300, 7.0 / 3.0):
        yd = dev(y)
        cuda.multiply_add_inplace(yd, a, dev(x))
        ref = cuda.add(dev(y), cuda.scale(a, dev(x)))
        assert np.array_equal(host(yd), host(ref))


def test_spmv_sym_matches_spmv_on_random_symmetric(cuda):
    """100 random exact-mirror symmetric matrices: the symmetric-storage SpMV
    equals the full CSR SpMV within 1e-14 (tests/test_acceptance.py:129-143)."""
    rng = np.random.default_rng(1234)
    for _ in range(100):
        n = int(rng.integers(2, 40))
        dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.3)
        dense = np.triu(dense, 1)
        dense = dense + dense.T + np.diag(rng.standard_normal(n) + n)
        rows, cols = np.nonzero(dense)
        ptr = np.concatenate(([0], np.cumsum(np.bincount(rows, minlength=n))))
        a = cuda.CsrMatrix(n, n, ptr, cols, dense[rows, cols])
        s = cuda.to_symmetric(a)
        x = rng.standard_normal(n)
        y1 = np.asarray(cuda.spmv(a, x))
        y2 = np.asarray(cuda.spmv_sym(s, x))
        assert np.allclose(y2, y1, rtol=1e-14, atol=1e-14 * np.abs(y1).max())
        assert np.allclose(y1, dense @ x, rtol=1e-12, atol=1e-12 * np.abs(dense).sum())


def test_dic_needs_at_most_half_the_jacobi_iterations(cuda):
    """On the n=16 cavity's first pressure system (tests/test_acceptance.py:99-126)."""
    from paper_2504_03697_b200 import sim

    cfg = cuda.SimConfig(n=16, dt=0.4, t_end=0.4)
    st = cuda.initial_state(cfg)
    sim.apply_forces(st, cfg)
    sim.enforce_boundaries(st)
    st.vel = sim.solve_advection(st, cfg)
    sim.enforce_boundaries(st)
    b = (-cfg.density / cfg.dt) * host(cuda.divergence(st.vel).data)
    a = cuda.poisson_symmetric(cfg.n, cfg.h)

    def apply_a(x, out=None):
        return cuda.spmv_sym(a, x, out=out)

    _, sd = cuda.pcg(apply_a, b, precond=cuda.dic_from(a), tol=1e-6)
    _, sj = cuda.pcg(apply_a, b, precond=cuda.jacobi_from(a), tol=1e-6)
    assert sd.converged and sj.converged
    assert sj.iterations >= 2 * sd.iterations


def test_vortex_circulation_and_sealed_walls(cuda, tmp_path):
    """The lid-driven run turns with the +x lid: positive circulation around
    the outermost square of the mid-z slice, wall-normal faces exactly zero
    (tests/test_acceptance.py:164-192; n=16 here, the reference's n=24 run
    pattern)."""
    cfg = cuda.SimConfig(n=16, dt=0.4, t_end=2.0, output_dir=str(tmp_path))
    st, rep = cuda.run(cfg)
    snap = cuda.read_snapshot(rep.snapshot_paths[-1])
    n = snap.spec.n
    u3 = snap.u.reshape((n, n, n), order="F")
    v3 = snap.v.reshape((n, n, n), order="F")
    k = n // 2
    circ = (np.sum(u3[:, n - 1, k] - u3[:, 0, k]) + np.sum(v3[0, :, k] - v3[n - 1, :, k])) * snap.spec.h
    assert circ > 0.0
    u, v, w = st.vel.numpy()
    assert max(np.abs(u[0]).max(), np.abs(u[n]).max(), np.abs(v[:, 0]).max(), np.abs(v[:, n]).max(),
               np.abs(w[:, :, 0]).max(), np.abs(w[:, :, n]).max()) == 0.0


def test_run_is_deterministic(cuda):
    """Two runs of the same configuration are bit-identical (fixed reduction
    trees, no atomics in any sum): the device analogue of the reference's
    single-thread determinism pin."""
    cfg = cuda.SimConfig(n=24, h=1.0 / 24, dt=0.05, t_end=0.15, tol=1e-8, variant="optimized",
                         preconditioner="jacobi")
    out = []
    for _ in range(2):
        st, rep = cuda.run(cfg)
        out.append((*st.vel.numpy(), st.p.numpy(), [s.solve.iterations for s in rep.steps]))
    for a, b in zip(out[0][:4], out[1][:4]):
        assert np.array_equal(a, b)
    assert out[0][4] == out[1][4]


def test_variants_agree(cuda):
    """baseline (full CSR order) and optimized (symmetric order) runs agree
    to 1e-9 at a tight tolerance (tests/test_sim.py:381-391)."""
    res = []
    for variant in ("baseline", "optimized"):
        cfg = cuda.SimConfig(n=12, h=1.0 / 12, dt=0.05, t_end=0.15, tol=1e-12, max_iter=5000, variant=variant,
                             preconditioner="jacobi")
        st, _ = cuda.run(cfg)
        res.append(np.concatenate([a.ravel() for a in st.vel.numpy()] + [st.p.numpy()]))
    assert np.linalg.norm(res[0] - res[1]) <= 1e-9 * np.linalg.norm(res[1])
