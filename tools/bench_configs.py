"""Measure BASELINE.json configs 1, 2, 3 and 5 on one B200 (config 4 is bench.py).

    python tools/bench_configs.py [--skip-512] > profiles/r01_configs.json

Device times are CUDA events on the current stream (synchronised around each
timed region); inputs are seeded synthetic data (numpy PCG64), as in
SURVEY.md §8(d).  Physics "reference" = the reference's inviscid model (the
parity baseline); "extension" = BASELINE's viscosity / lid velocity / no-slip.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps=1):
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    out = None
    for _ in range(reps):
        out = fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def cavity(n, dt, steps, tol, ext=False, warm=2):
    kw = dict(n=n, h=1.0 / n, dt=dt, t_end=dt * (steps + warm), tol=tol, max_iter=50000, variant="optimized",
              preconditioner="jacobi")
    if ext:
        kw.update(lid_accel=0.0, viscosity=0.01 if n == 16 else 0.001, lid_velocity=1.0, no_slip=True,
                  initial_pressure=0.0)
    cfg = cf.SimConfig(**kw)
    st = cf.initial_state(cfg)
    cache = cf.PoissonCache()
    for _ in range(warm):
        cf.step(st, cfg, cache)
    its = []

    def run():
        for _ in range(steps):
            its.append(cf.step(st, cfg, cache).solve.iterations)

    ms, _ = timed(run)
    return {"n": n, "dt": dt, "steps": steps, "tol": tol, "physics": "extension" if ext else "reference",
            "ms_per_step": ms / steps, "steps_per_s": steps / (ms / 1e3), "cg_iterations": its,
            "cg_iterations_per_s": sum(its) / (ms / 1e3)}


def poisson(n, seed, tol):
    b = np.random.default_rng(seed).uniform(-1, 1, n ** 3)
    b -= b.mean()
    bd = torch.as_tensor(b, device="cuda")
    op = cf.StencilOperator(n, 1.0 / n, "sym")
    pre = cf.jacobi_from(op)
    cf.pcg(op, bd, precond=pre, tol=tol, max_iter=50000)
    ms, (x, st) = timed(lambda: cf.pcg(op, bd, precond=pre, tol=tol, max_iter=50000))
    loop = op._cg_ws.last_loop_ms
    return {"n": n, "seed": seed, "tol": tol, "iterations": st.iterations, "converged": st.converged,
            "solve_ms": ms, "us_per_iteration": 1e3 * loop / st.iterations,
            "iterations_per_s": st.iterations / (loop / 1e3),
            "note": "128^3 CG working set (4 x 16.8 MB) is L2-resident: per-iteration time, not an HBM fraction"}


def spmv(n, reps=100):
    h = 1.0 / n
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
    y = torch.empty_like(x)
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
    N = n ** 3
    out = {"n": n, "reps": reps, "peak_gbs": peak()}
    for order in ("csr", "sym"):
        op = cf.StencilOperator(n, h, order)
        op(x, out=y)
        ms, _ = timed(lambda: op(x, out=y), reps)
        gbs = 16 * N / (ms / 1e3) / 1e9
        out[f"stencil_{order}_order"] = {"us": 1e3 * ms, "bytes": 16 * N, "gbs": gbs, "frac": gbs / peak()}
    a = cf.poisson_full_csr(n, h)
    cf.spmv(a, x, out=y)
    ms, _ = timed(lambda: cf.spmv(a, x, out=y), reps)
    nbytes = 12 * a.nnz + 4 * (N + 1) + 16 * N
    out["csr_int32"] = {"us": 1e3 * ms, "nnz": a.nnz, "bytes": nbytes, "gbs": nbytes / (ms / 1e3) / 1e9,
                        "frac": nbytes / (ms / 1e3) / 1e9 / peak()}
    del a
    s = cf.poisson_symmetric(n, h)
    cf.spmv_sym(s, x, out=y)
    ms, _ = timed(lambda: cf.spmv_sym(s, x, out=y), reps)
    nb = 8 * N + 12 * len(s.values) + 4 * (N + 1) + 8 * len(s.values) + 4 * (N + 1) + 16 * N
    out["sym_int32"] = {"us": 1e3 * ms, "bytes": nb, "gbs": nb / (ms / 1e3) / 1e9}
    del flush
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-512", action="store_true")
    a = ap.parse_args()
    cf.load_library()
    res = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    res["config1_reference_physics"] = cavity(16, 0.01, 10, 1e-6)
    res["config1_extension_physics"] = cavity(16, 0.01, 10, 1e-6, ext=True)
    res["config2_poisson_128"] = [poisson(128, s, 1e-8) for s in (0, 1, 2)]
    res["config3_spmv_256"] = spmv(256)
    res["config4_extension_physics_256"] = cavity(256, 0.002, 3, 1e-8, ext=True, warm=1)
    if not a.skip_512:
        res["config5_512_reference_physics"] = cavity(512, 0.001, 2, 1e-8, warm=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
