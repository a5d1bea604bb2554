"""Pin the CPU oracle against fixtures produced by the reference itself.

The oracle (oracle/) is the checker for every GPU parity test, so it must
first be shown to reproduce the reference: bit-for-bit wherever the
reference's operation order is deterministic (single chunk, or the same
chunk bounds), which covers assembly, SpMV, dot, axpy, DIC, advection,
divergence, correction, PCG and whole cavity runs.
"""

import numpy as np
import pytest

import oracle as orc


def test_assembly_matches_reference(golden):
    g = golden("sparse")
    for n in (5, 16):
        h = float(g[f"n{n}_h"])
        a = orc.poisson_csr(n, h)
        s = orc.poisson_sym(n, h)
        assert np.array_equal(a.row_ptr, g[f"n{n}_row_ptr"])
        assert np.array_equal(a.col_idx, g[f"n{n}_col_idx"])
        assert np.array_equal(a.values, g[f"n{n}_values"])
        assert np.array_equal(s.row_ptr, g[f"n{n}_sym_row_ptr"])
        assert np.array_equal(s.col_idx, g[f"n{n}_sym_col_idx"])
        assert np.array_equal(s.values, g[f"n{n}_sym_values"])


def test_kernels_bitwise(golden):
    g = golden("sparse")
    for n in (5, 16):
        h = float(g[f"n{n}_h"])
        a, s, x = orc.poisson_csr(n, h), orc.poisson_sym(n, h), g[f"n{n}_x"]
        y = orc.spmv(a, x)
        assert np.array_equal(y, g[f"n{n}_spmv"])
        assert np.array_equal(orc.spmv(a, x, threads=3), y)
        assert np.array_equal(orc.spmv_sym(s, x), g[f"n{n}_spmv_sym"])
        assert orc.dot(x, y) == float(g[f"n{n}_dot_t1"])
        assert orc.dot(x, y, threads=3) == float(g[f"n{n}_dot_t3"])
        z = y.copy()
        orc.maxpy(z, 0.7391, x)
        assert np.array_equal(z, g[f"n{n}_maxpy"])
        dic = orc.Dic(a)
        assert np.array_equal(dic.modified_diag, g[f"n{n}_dic_diag"])
        assert np.array_equal(dic.apply(x), g[f"n{n}_dic_apply"])
        assert np.array_equal(orc.Dic(s).modified_diag, dic.modified_diag)


@pytest.mark.parametrize("n", [12, 32])
def test_pcg_bitwise(golden, n):
    g = golden("pcg")
    h = 1.0 / n
    b = g[f"n{n}_b"]
    a_sym, a_full = orc.poisson_sym(n, h), orc.poisson_csr(n, h)
    cases = {
        "jacobi_opt": (lambda x, o: orc.spmv_sym(a_sym, x, 1, o), orc.jacobi_from(a_sym), "optimized"),
        "dic_base": (lambda x, o: orc.spmv(a_full, x, 1, o), orc.Dic(a_full), "baseline"),
        "none_opt": (lambda x, o: orc.spmv_sym(a_sym, x, 1, o), None, "optimized"),
    }
    for tag, (op, pre, variant) in cases.items():
        x, st = orc.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, variant=variant)
        assert st.iterations == int(g[f"n{n}_{tag}_it"]), tag
        assert st.final_residual_rel == float(g[f"n{n}_{tag}_res"]), tag
        assert np.array_equal(x, g[f"n{n}_{tag}_x"]), tag
    x, st = orc.pcg(cases["jacobi_opt"][0], b, x0=g[f"n{n}_x0"], precond=orc.jacobi_from(a_sym),
                    tol=1e-8, max_iter=20000)
    assert st.iterations == int(g[f"n{n}_warm_it"])
    assert np.array_equal(x, g[f"n{n}_warm_x"])


@pytest.mark.slow
def test_pcg_config2_iterations(golden):
    """BASELINE config 2 (128^3, tol 1e-8, seed 0) with the reference's 8 chunks."""
    g = golden("pcg")
    n = 128
    a = orc.poisson_sym(n, 1.0 / n)
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    b -= b.mean()
    x, st = orc.pcg(lambda v, o: orc.spmv_sym(a, v, 8, o), b, precond=orc.jacobi_from(a), tol=1e-8,
                    max_iter=20000, variant="optimized", threads=8)
    assert st.iterations == int(g["c2_seed0_it"]) == 446
    assert st.final_residual_rel == float(g["c2_seed0_res"])
    assert np.array_equal(x[::4099], g["c2_seed0_x_sample"])


@pytest.mark.parametrize("n", [6, 16])
def test_advection_divergence_correction_bitwise(golden, n):
    g = golden("advection")
    h, dt = 1.0 / n, float(g[f"n{n}_dt"])
    u, v, w = (g[f"n{n}_in_{c}"] for c in "uvw")
    nu, nv, nw = orc.advect(u, v, w, n, h, dt)
    assert np.array_equal(nu, g[f"n{n}_out_u"])
    assert np.array_equal(nv, g[f"n{n}_out_v"])
    assert np.array_equal(nw, g[f"n{n}_out_w"])
    assert np.array_equal(orc.advect(u, v, w, n, h, dt, threads=4)[2], nw)
    assert np.array_equal(orc.divergence(u, v, w, h), g[f"n{n}_div"])
    s = orc.State(nu.copy(), nv.copy(), nw.copy(), g[f"n{n}_p"].copy())
    div_post = orc.correct(s, orc.Cfg(n=n, h=h, dt=dt))
    assert div_post == float(g[f"n{n}_div_post"])
    for c in "uvw":
        assert np.array_equal(getattr(s, c), g[f"n{n}_corr_{c}"])


CAVITY_RUNS = {
    "c1_opt_jacobi": dict(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000,
                          variant="optimized", preconditioner="jacobi"),
    "c1_base_dic": dict(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000,
                        variant="baseline", preconditioner="dic"),
    "n8_warm": dict(n=8, dt=0.4, t_end=1.2, warm_start=True, variant="optimized",
                    preconditioner="jacobi"),
    "n8_golden": dict(n=8, dt=0.4, t_end=1.2, variant="baseline"),
}


@pytest.mark.parametrize("tag", list(CAVITY_RUNS))
def test_cavity_runs_bitwise(golden, tag):
    g = golden("cavity")
    cfg = orc.Cfg(**CAVITY_RUNS[tag])
    s, results = orc.run(cfg)
    assert [r.solve.iterations for r in results] == g[f"{tag}_its"].tolist()
    assert [r.div_pre for r in results] == g[f"{tag}_div_pre"].tolist()
    assert [r.div_post for r in results] == g[f"{tag}_div_post"].tolist()
    for c in "uvw":
        assert np.array_equal(getattr(s, c), g[f"{tag}_{c}"])
    assert np.array_equal(s.p, g[f"{tag}_p"])


def test_reference_golden_snapshot(golden):
    """The reference's committed n=8 golden CSV (tests/test_acceptance.py:216-226)."""
    g = golden("cavity")
    s, _ = orc.run(orc.Cfg(**CAVITY_RUNS["n8_golden"]))
    cols = orc.snapshot_columns(s, 1.0)
    for c in "xyzuvwp":
        assert np.abs(cols[c] - g[f"ref_csv_{c}"]).max() <= 1e-9, c
        assert np.array_equal(cols[c], g[f"ref_csv_{c}"]), c


def test_known_answers():
    """Hand cases of the reference suite (tests/test_solver.py:27-57)."""
    a = np.array([[4.0, 1.0], [1.0, 3.0]])
    x, st = orc.pcg(lambda v, o: np.dot(a, v, out=o), np.array([1.0, 2.0]), tol=1e-10)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=1e-8)
    x, st = orc.pcg(lambda v, o: np.dot(np.eye(2), v, out=o), np.zeros(2))
    assert st.iterations == 0 and st.converged and not x.any()
    with pytest.raises(orc.Breakdown):
        orc.pcg(lambda v, o: np.dot(-np.eye(4), v, out=o), np.ones(4))


def test_extension_diffusion_known_answers():
    """The extension's restatement (oracle/physics_ext.py): a unit spike spreads
    kdt to its six neighbours and keeps 1 - 6 kdt; a uniform tangential field is
    invariant under mirror ghosts away from the normal walls; the moving lid
    pulls u towards U."""
    from oracle import physics_ext as ext

    n, kdt = 6, 0.1
    u = np.zeros((n + 1, n, n)); v = np.zeros((n, n + 1, n)); w = np.zeros((n, n, n + 1))
    u[3, 2, 2] = 1.0
    nu, nv, nw = ext.diffuse(u, v, w, n, kdt)
    assert nu[3, 2, 2] == 1.0 - 6 * kdt
    for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        assert nu[3 + d[0], 2 + d[1], 2 + d[2]] == kdt
    assert not nv.any() and not nw.any()
    v[:] = 0.7
    v[:, 0] = v[:, n] = 0.0
    _, nv, _ = ext.diffuse(u * 0, v, w, n, kdt)
    assert np.allclose(nv[:, 2:n - 1], 0.7, rtol=0, atol=1e-15)
    nu, _, _ = ext.diffuse(u * 0, v * 0, w, n, kdt, lid_u=1.0, no_slip=True)
    assert np.all(nu[1:n, n - 1, :] == kdt * 2.0)


def test_extension_implicit_diffusion_restatement():
    """Backward-Euler operator of the extension: symmetric (CG-safe), and the
    solve satisfies (I - kdt L) u = u* (+ lid term); for small kdt it agrees
    with the explicit step to O(kdt^2)."""
    from oracle import physics_ext as ext

    n, kdt = 6, 0.3
    rng = np.random.default_rng(2)
    for comp, shape in enumerate(((n + 1, n, n), (n, n + 1, n), (n, n, n + 1))):
        a, b = rng.standard_normal(shape), rng.standard_normal(shape)
        for arr in (a, b):  # wall-normal faces are fixed zeros
            sl = [slice(None)] * 3
            sl[comp] = 0
            arr[tuple(sl)] = 0.0
            sl[comp] = -1
            arr[tuple(sl)] = 0.0
        for lid, ns in ((None, False), (1.0, True)):
            Aa = ext.helmholtz_apply(comp, a, n, kdt, lid, ns)[0]
            Ab = ext.helmholtz_apply(comp, b, n, kdt, lid, ns)[0]
            assert abs(np.sum(b * Aa) - np.sum(a * Ab)) <= 1e-12 * np.abs(np.sum(b * Aa))
    u = 0.1 * rng.standard_normal((n + 1, n, n)); u[0] = u[n] = 0
    v = 0.1 * rng.standard_normal((n, n + 1, n)); v[:, 0] = v[:, n] = 0
    w = 0.1 * rng.standard_normal((n, n, n + 1)); w[:, :, 0] = w[:, :, n] = 0
    iu, iv, iw = ext.diffuse_implicit(u, v, w, n, 1e-3, 1.0, True, tol=1e-13)
    eu, ev, ew = ext.diffuse(u, v, w, n, 1e-3, 1.0, True)
    assert np.abs(iu - eu).max() <= 1e-4 and np.abs(iw - ew).max() <= 1e-4
    r = ext.helmholtz_apply(0, iu, n, 1e-3, 1.0, True)[0]
    want = u.copy(); want[1:n, n - 1, :] += 1e-3 * 2.0
    assert np.abs(r - want).max() <= 1e-11


def test_box_restatement_consistency(golden):
    """The non-cubic extension (shape=(nx,ny,nz)): shape=(n,n,n) reproduces the
    reference-pinned cube exactly; a box operator is symmetric with diagonal
    6/h^2 and the CSR/symmetric forms agree to rounding; a box run projects."""
    g = golden("sparse")
    h = float(g["n5_h"])
    cube = orc.poisson_csr(5, h, (5, 5, 5))
    assert np.array_equal(cube.row_ptr, g["n5_row_ptr"]) and np.array_equal(cube.col_idx, g["n5_col_idx"])
    shape = (7, 4, 6)
    a, s = orc.poisson_csr(0, h, shape), orc.poisson_sym(0, h, shape)
    x = np.random.default_rng(0).standard_normal(7 * 4 * 6)
    dense = np.zeros((a.n_rows, a.n_rows))
    for r in range(a.n_rows):
        dense[r, a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]]] = a.values[a.row_ptr[r]:a.row_ptr[r + 1]]
    assert np.array_equal(dense, dense.T) and np.all(np.diag(dense) == 6.0 / h ** 2)
    assert np.allclose(orc.spmv_sym(s, x), dense @ x, rtol=0, atol=1e-9 / h ** 2)
    # cell (i,j,k) neighbours: i+1 is +1, j+1 is +nx, k+1 is +nx*ny
    r = 1 + 7 * (1 + 4 * 1)
    cols = set(a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]].tolist())
    assert cols == {r, r - 1, r + 1, r - 7, r + 7, r - 28, r + 28}
    cfg = orc.Cfg(n=9, h=1.0 / 9, dt=0.05, t_end=0.1, tol=1e-8, max_iter=5000, preconditioner="jacobi",
                  variant="optimized", shape=(9, 5, 7))
    st, results = orc.run(cfg)
    assert st.u.shape == (10, 5, 7) and st.p.shape == (9 * 5 * 7,)
    for res in results:
        assert res.solve.converged and res.div_post <= 1e-3 * res.div_pre


def test_sample_velocity_matches_reference(golden):
    """src/grid.py:124-142 on reference-sampled random fields (inside, lattice
    nodes, walls, far outside): bit for bit."""
    g = golden("grid")
    for tag in "abc":
        u, v, w, h = g[f"{tag}_u"], g[f"{tag}_v"], g[f"{tag}_w"], float(g[f"{tag}_h"])
        got = np.array([orc.sample_velocity(u, v, w, h, p) for p in g[f"{tag}_pts"]])
        assert np.array_equal(got, g[f"{tag}_samples"]), tag
