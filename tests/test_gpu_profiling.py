"""GPU: profiler/report parity -- device-timed regions,
z-slab runs reporting the reference's region tree, the scaling sweep (the
emulated multi-slab leg, and the torchrun launcher at one rank)."""

import pytest

pytestmark = pytest.mark.gpu

STEP_REGIONS = ["applyForces", "solveAdvection", "solvePressureCorrection", "pcg", "applyPressureCorrection"]


def test_event_timer_run_report(cuda):
    from paper_2504_03697_b200.profiling import Profiler, render_report

    cfg = cuda.SimConfig(n=32, h=1.0 / 32, dt=0.01, t_end=0.03, variant="optimized", preconditioner="jacobi")
    _, wall = cuda.run(cfg)
    _, ev = cuda.run(cfg, profiler=Profiler(timer="events"))
    names_w = [(r.name, r.parent, r.calls) for r in wall.regions]
    names_e = [(r.name, r.parent, r.calls) for r in ev.regions]
    assert names_w == names_e
    # the fused solve reports the reference's pcg sub-regions (src/solver.py:148-170,
    # PAPER.md Table 1): reference call counts, device loop time split by bytes
    sub = ["spmv", "dot", "multiply_add_inplace", "precondition"]
    assert [n for n, _, _ in names_e[1:]] == STEP_REGIONS[:4] + sub + [STEP_REGIONS[4]]
    by = {r.name: r for r in ev.regions}
    assert by["pcg"].inclusive_seconds > 0 and by["pcg"].inclusive_seconds <= by["cavityflow"].inclusive_seconds
    assert all(by[n].parent == "pcg" for n in sub)
    assert sum(by[n].inclusive_seconds for n in sub) <= by["pcg"].inclusive_seconds * 1.05
    assert by["dot"].calls == 3 * by["spmv"].calls  # converged solves: 1 + 2k + (k - 1) dots for k spmvs
    assert by["multiply_add_inplace"].calls == 3 * by["spmv"].calls - 3  # 3 steps, 2k + (k - 1) each
    assert "└─ applyPressureCorrection" in render_report(ev.regions)


def test_slab_run_regions_and_result(cuda):
    from paper_2504_03697_b200 import distributed

    cfg = cuda.SimConfig(n=32, h=1.0 / 32, dt=0.01, t_end=0.02, tol=1e-10, max_iter=5000, variant="optimized",
                         preconditioner="jacobi")
    st, rep = cuda.run(cfg)
    sim, srep = distributed.run(cfg, slabs=3)
    assert [r.name for r in srep.regions] == ["cavityflow"] + STEP_REGIONS
    assert [s.solve.iterations for s in srep.steps] == pytest.approx([s.solve.iterations for s in rep.steps], abs=2)
    with pytest.raises(ValueError, match="snapshots"):
        distributed.run(cuda.SimConfig(n=32, output_dir="/tmp/x", preconditioner="jacobi"), slabs=2)


def test_scaling_sweep_emulated_and_launcher(cuda, tmp_path):
    from paper_2504_03697_b200 import profiling as pf

    cfg = cuda.SimConfig(n=32, h=1.0 / 32, dt=0.01, t_end=0.02, variant="optimized", preconditioner="jacobi")
    rows = pf.scaling_sweep(cfg, [1, 2, 4], emulate=True)
    assert sorted({g for g, _, _ in rows}) == [1, 2, 4]
    assert {r for g, r, _ in rows if g == 4} == {"cavityflow", *STEP_REGIONS}
    path = tmp_path / "s.csv"
    pf.write_scaling_csv(rows, path)
    assert path.read_text().splitlines()[0] == "threads,region,seconds"
    # the multi-GPU leg's launcher + rank worker, at one rank (this box has one GPU)
    regions = pf._ranks_report(cfg, 1)
    assert [r.name for r in regions] == ["cavityflow"] + STEP_REGIONS
    with pytest.raises(ValueError, match="GPUs requested"):
        pf.scaling_sweep(cfg, [1, 64])
