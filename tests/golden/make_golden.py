"""Regenerate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by importing ``cavityflow`` (the reference package)
and calling its public API on seeded inputs; nothing here reimplements the
algorithm.  The fixtures pin ``oracle/`` (tests/test_oracle.py) and, on the
GPU, the CUDA path (tests/test_gpu_*.py).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import cavityflow as cf  # noqa: E402
from cavityflow import sim  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(np.asarray(a).nbytes for a in arrays.values()), "bytes raw")


def compliant_state(n, seed, scale):
    cfg = sim.SimConfig(n=n, h=1.0 / n, dt=0.01, t_end=0.0)
    st = sim.initial_state(cfg)
    rng = np.random.default_rng(seed)
    st.vel.u[:] = scale * rng.standard_normal(st.vel.u.shape)
    st.vel.v[:] = scale * rng.standard_normal(st.vel.v.shape)
    st.vel.w[:] = scale * rng.standard_normal(st.vel.w.shape)
    sim.enforce_boundaries(st)
    return st


def sparse_fixtures():
    out = {}
    for n, h in ((5, 0.7), (16, 1.0 / 16)):
        full = sim.poisson_full_csr(n, h)
        sym = sim.poisson_symmetric(n, h)
        x = np.random.default_rng(n).uniform(-1, 1, n ** 3)
        out[f"n{n}_h"] = np.float64(h)
        out[f"n{n}_row_ptr"] = full.row_ptr
        out[f"n{n}_col_idx"] = full.col_idx
        out[f"n{n}_values"] = full.values
        out[f"n{n}_sym_row_ptr"] = sym.row_ptr
        out[f"n{n}_sym_col_idx"] = sym.col_idx
        out[f"n{n}_sym_values"] = sym.values
        out[f"n{n}_x"] = x
        out[f"n{n}_spmv"] = cf.spmv(full, x)
        out[f"n{n}_spmv_sym"] = cf.spmv_sym(sym, x)
        with cf.WorkerPool(3) as pool:
            out[f"n{n}_dot_t3"] = np.float64(cf.dot(x, out[f"n{n}_spmv"], pool))
        out[f"n{n}_dot_t1"] = np.float64(cf.dot(x, out[f"n{n}_spmv"]))
        y = out[f"n{n}_spmv"].copy()
        cf.multiply_add_inplace(y, 0.7391, x)
        out[f"n{n}_maxpy"] = y
        dic = cf.dic_from(full)
        out[f"n{n}_dic_diag"] = dic.modified_diag
        out[f"n{n}_dic_apply"] = dic.apply(x)
    save("sparse.npz", **out)


def pcg_fixtures():
    out = {}
    for n in (12, 32):
        h = 1.0 / n
        a_sym = sim.poisson_symmetric(n, h)
        a_full = sim.poisson_full_csr(n, h)
        b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
        b -= b.mean()
        out[f"n{n}_b"] = b
        for tag, a, pre, variant in (
            ("jacobi_opt", a_sym, cf.jacobi_from(a_sym), "optimized"),
            ("dic_base", a_full, cf.dic_from(a_full), "baseline"),
            ("none_opt", a_sym, None, "optimized"),
        ):
            op = (lambda x, out=None, a=a: cf.spmv_sym(a, x, out=out)) if a is a_sym else \
                (lambda x, out=None, a=a: cf.spmv(a, x, out=out))
            x, st = cf.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, variant=variant)
            out[f"n{n}_{tag}_x"] = x
            out[f"n{n}_{tag}_it"] = np.int64(st.iterations)
            out[f"n{n}_{tag}_res"] = np.float64(st.final_residual_rel)
        # warm start from a perturbed guess
        x0 = np.random.default_rng(1).uniform(-1, 1, n ** 3) * 1e-3
        x, st = cf.pcg(lambda v, out=None: cf.spmv_sym(a_sym, v, out=out), b, x0=x0,
                       precond=cf.jacobi_from(a_sym), tol=1e-8, max_iter=20000, variant="optimized")
        out[f"n{n}_x0"] = x0
        out[f"n{n}_warm_x"] = x
        out[f"n{n}_warm_it"] = np.int64(st.iterations)
    # config 2 (128^3, tol 1e-8): iteration counts and solution checksums only
    n = 128
    a_sym = sim.poisson_symmetric(n, 1.0 / n)
    with cf.WorkerPool(os.cpu_count()) as pool:
        for seed in (0, 1):
            b = np.random.default_rng(seed).uniform(-1, 1, n ** 3)
            b -= b.mean()
            x, st = cf.pcg(lambda v, out=None: cf.spmv_sym(a_sym, v, out=out, pool=pool), b,
                           precond=cf.jacobi_from(a_sym), tol=1e-8, max_iter=20000,
                           variant="optimized", pool=pool)
            out[f"c2_seed{seed}_it"] = np.int64(st.iterations)
            out[f"c2_seed{seed}_res"] = np.float64(st.final_residual_rel)
            out[f"c2_seed{seed}_xnorm"] = np.float64(np.linalg.norm(x))
            out[f"c2_seed{seed}_xsum"] = np.float64(x.sum())
            out[f"c2_seed{seed}_x_sample"] = x[:: 4099].copy()
    save("pcg.npz", **out)


def advection_fixtures():
    out = {}
    for n, dt, scale, seed in ((6, 0.3, 0.4, 11), (16, 0.01, 20.0, 12)):
        st = compliant_state(n, seed, scale)
        cfg = sim.SimConfig(n=n, h=1.0 / n, dt=dt, t_end=0.0)
        new = sim.solve_advection(st, cfg)
        for c, a in zip("uvw", st.vel.components()):
            out[f"n{n}_in_{c}"] = a
        for c, a in zip("uvw", new.components()):
            out[f"n{n}_out_{c}"] = a
        out[f"n{n}_dt"] = np.float64(dt)
        out[f"n{n}_div"] = cf.divergence(st.vel).data
        # pressure correction of the advected field with a seeded pressure
        p = cf.ScalarField(st.vel.spec, np.random.default_rng(seed + 100).standard_normal(n ** 3))
        st2 = sim.SimState(vel=new.copy(), p=p)
        div_post = sim.apply_pressure_correction(st2, p, cfg)
        out[f"n{n}_p"] = p.data
        for c, a in zip("uvw", st2.vel.components()):
            out[f"n{n}_corr_{c}"] = a
        out[f"n{n}_div_post"] = np.float64(div_post)
    save("advection.npz", **out)


def cavity_fixtures():
    out = {}
    runs = {
        # BASELINE config 1 geometry in reference physics (nu = 0, lid accel)
        "c1_opt_jacobi": dict(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000,
                              variant="optimized", preconditioner="jacobi"),
        "c1_base_dic": dict(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000,
                            variant="baseline", preconditioner="dic"),
        "n8_warm": dict(n=8, dt=0.4, t_end=1.2, warm_start=True, variant="optimized",
                        preconditioner="jacobi"),
        # the reference golden-snapshot configuration (tests/data/make_reference.py)
        "n8_golden": dict(n=8, dt=0.4, t_end=1.2, variant="baseline"),
    }
    for tag, kw in runs.items():
        cfg = sim.SimConfig(output_dir=None, **kw)
        state = sim.initial_state(cfg)
        cache = sim.PoissonCache()
        its, res, dpre, dpost = [], [], [], []
        for s in range(cfg.num_steps):
            st = sim.step(state, cfg, cache)
            its.append(st.solve.iterations)
            res.append(st.solve.final_residual_rel)
            dpre.append(st.div_pre)
            dpost.append(st.div_post)
            if s == 0:
                for c, a in zip("uvw", state.vel.components()):
                    out[f"{tag}_step1_{c}"] = a.copy()
                out[f"{tag}_step1_p"] = state.p.data.copy()
        for c, a in zip("uvw", state.vel.components()):
            out[f"{tag}_{c}"] = a
        out[f"{tag}_p"] = state.p.data
        out[f"{tag}_its"] = np.array(its, dtype=np.int64)
        out[f"{tag}_res"] = np.array(res)
        out[f"{tag}_div_pre"] = np.array(dpre)
        out[f"{tag}_div_post"] = np.array(dpost)
    # the reference's own committed golden snapshot, as read by its reader
    snap = cf.read_snapshot("/root/reference/pkg/tests/data/reference_n8_step3.csv")
    for c in "xyzuvwp":
        out[f"ref_csv_{c}"] = snap.column(c)
    save("cavity.npz", **out)


REF_CSV = "/root/reference/pkg/tests/data/reference_n8_step3.csv"


def snapshot_fixtures():
    """Byte-level pins of the snapshot writer (src/snapshots.py:65-108):
    the sha256 of the reference's committed CSV, and the reference writer's
    output (both modes) on a state with values spanning every branch of the
    repr format (exponent forms, integral values, signed zeros, subnormals)."""
    import hashlib
    import tempfile

    from cavityflow import snapshots

    out = {}
    with open(REF_CSV, "rb") as f:
        raw = f.read()
    out["ref_csv_sha256"] = np.frombuffer(hashlib.sha256(raw).digest(), dtype=np.uint8)
    out["ref_csv_len"] = np.int64(len(raw))
    n, h = 6, 0.1
    cfg = sim.SimConfig(n=n, h=h, dt=0.01, t_end=0.0)
    st = sim.initial_state(cfg)
    rng = np.random.default_rng(17)

    def exotic(shape):
        a = rng.standard_normal(shape) * 10.0 ** rng.integers(-20, 24, size=shape)
        flat = a.reshape(-1)
        pick = rng.random(flat.size)
        flat[pick < 0.1] = np.round(flat[pick < 0.1] * 1e-3 * 10.0 ** rng.integers(0, 8))
        flat[(pick >= 0.1) & (pick < 0.13)] = 0.0
        flat[(pick >= 0.13) & (pick < 0.16)] = -0.0
        flat[(pick >= 0.16) & (pick < 0.18)] = 5e-324 * rng.integers(1, 1000)
        flat[(pick >= 0.18) & (pick < 0.2)] = np.array([1e16, 1e15, 1e-4, 1e-5, 0.0001234, 123456789012345678.0,
                                                          9999999999999998.0, 2.0 ** 60, 0.1, 1.0 / 3.0])[
            rng.integers(0, 10, size=int(((pick >= 0.18) & (pick < 0.2)).sum()))]
        return a

    st.vel.u[:] = exotic(st.vel.u.shape)
    st.vel.v[:] = exotic(st.vel.v.shape)
    st.vel.w[:] = exotic(st.vel.w.shape)
    st.p.data[:] = exotic(st.p.data.shape)
    with tempfile.TemporaryDirectory() as d:
        a, b = os.path.join(d, "a.csv"), os.path.join(d, "b.csv")
        snapshots.write_snapshot(st, a)
        snapshots.write_snapshot(st, b, mode="buffered_parallel", threads=3)
        with open(a, "rb") as f:
            sa = f.read()
        with open(b, "rb") as f:
            assert f.read() == sa
    out["exotic_h"] = np.float64(h)
    for c, arr in zip("uvw", st.vel.components()):
        out[f"exotic_{c}"] = arr.copy()
    out["exotic_p"] = st.p.data.copy()
    out["exotic_sha256"] = np.frombuffer(hashlib.sha256(sa).digest(), dtype=np.uint8)
    out["exotic_len"] = np.int64(len(sa))
    save("snapshot.npz", **out)


def profiling_fixtures():
    """The reference's report renderers and writers (src/bench.py:159-324) on
    fixed region records: render_report, save_report, compare_reports,
    render_comparison and write_scaling_csv outputs, as text."""
    import json
    import tempfile

    from cavityflow import bench

    R = bench.RegionStats
    a = [R("cavityflow", None, 1, 12.5, 1.0), R("write_to_file", "cavityflow", 4, 0.75, 0.06),
         R("applyForces", "cavityflow", 3, 0.01, 0.0008), R("solveAdvection", "cavityflow", 3, 1.2, 0.096),
         R("solvePressureCorrection", "cavityflow", 3, 10.0, 0.8), R("pcg", "solvePressureCorrection", 3, 9.5, 0.76),
         R("spmv", "pcg", 300, 4.0, 0.32), R("dot", "pcg", 900, 1.5, 0.12),
         R("applyPressureCorrection", "cavityflow", 3, 0.4, 0.032), R("other_root", None, 2, 0.0, 0.0)]
    b = [R("cavityflow", None, 1, 3.25, 1.0), R("applyForces", "cavityflow", 3, 0.02, 0.006),
         R("solvePressureCorrection", "cavityflow", 3, 2.0, 0.6), R("pcg", "solvePressureCorrection", 3, 1.9, 0.58),
         R("fused_cg", "pcg", 3, 1.8, 0.55), R("write_to_file", "cavityflow", 4, 0.5, 0.15)]
    rows = [(1, "cavityflow", 12.5), (2, "pcg", 0.1 + 0.2), (8, "dot", 1e-7)]
    with tempfile.TemporaryDirectory() as d:
        bench.save_report(a, os.path.join(d, "r.json"))
        with open(os.path.join(d, "r.json"), encoding="utf-8") as f:
            saved = f.read()
        bench.write_scaling_csv(rows, os.path.join(d, "s.csv"))
        with open(os.path.join(d, "s.csv"), encoding="utf-8", newline="") as f:
            scaling = f.read()
    cmp = bench.compare_reports(a, b)
    out = {"a": [vars(r) for r in a], "b": [vars(r) for r in b], "scaling_rows": rows,
           "render_a": bench.render_report(a), "render_b": bench.render_report(b), "saved_a": saved,
           "compare": cmp, "render_compare": bench.render_comparison(cmp), "scaling_csv": scaling}
    path = os.path.join(HERE, "profiling.json")
    with open(path, "w", encoding="utf-8") as f:
        json.dump(out, f, indent=1, ensure_ascii=False)
    print("wrote", path)


def grid_fixtures():
    """sample_velocity (src/grid.py:124-142) on seeded random fields: points
    inside the domain, on lattice nodes, on the walls and far outside (the
    clamp), at a cube with h != 1 and one with h = 1."""
    from cavityflow import grid

    out = {}
    for tag, n, h, seed in (("a", 5, 0.4, 11), ("b", 8, 1.0, 12), ("c", 3, 0.7, 13)):
        spec = grid.GridSpec(n, h)
        f = grid.VelocityField(spec)
        rng = np.random.default_rng(seed)
        f.u[:] = rng.standard_normal(f.u.shape)
        f.v[:] = rng.standard_normal(f.v.shape)
        f.w[:] = rng.standard_normal(f.w.shape)
        L = spec.side_length
        pts = [rng.random(3) * L for _ in range(40)]
        pts += [rng.uniform(-0.5 * L, 1.5 * L, 3) for _ in range(20)]  # partly outside: clamped
        pts += [np.array([i * h, (j + 0.5) * h, (k + 0.5) * h]) for i, j, k in ((0, 0, 0), (n, n - 1, n - 1), (2, 1, 0))]
        pts += [np.array([0.0, 0.0, 0.0]), np.array([L, L, L]), np.array([1e6, -1e6, 0.5 * L])]
        pts = np.array(pts)
        out[f"{tag}_n"], out[f"{tag}_h"] = np.int64(n), np.float64(h)
        out[f"{tag}_u"], out[f"{tag}_v"], out[f"{tag}_w"] = f.u.copy(), f.v.copy(), f.w.copy()
        out[f"{tag}_pts"] = pts
        out[f"{tag}_samples"] = np.array([grid.sample_velocity(f, p) for p in pts])
    save("grid.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"{name}_fixtures"]()
        sys.exit(0)
    profiling_fixtures()
    snapshot_fixtures()
    sparse_fixtures()
    advection_fixtures()
    cavity_fixtures()
    pcg_fixtures()
    grid_fixtures()
