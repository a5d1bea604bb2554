"""Run every hot-path kernel once or a few times at 256^3 so ONE ncu launch
list (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)
covers them all: a reference-physics step (advection, divergence, CG init,
the CG kernels host-driven, correction), an extension-physics step
(diffusion), the config-3 SpMV forms and a DIC-PCG of a few iterations.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/table_step.csv python tools/ncu_table.py 256 step
    (the same with table_cg.csv and "256 cg")
    python tools/kernel_table.py gpurun_out/table_step.csv,gpurun_out/table_cg.csv profiles/r02_kernel_table.json

The CG is capped at a few iterations (max_iter) so the list stays short; the
solve warns about non-convergence, which is expected here.
"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CF_CG_DIRECT", "2")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
part = sys.argv[2] if len(sys.argv) > 2 else "all"  # step | cg | all
h = 1.0 / n
its = 6


def steps(ext):
    kw = dict(lid_accel=0.0, viscosity=0.001, lid_velocity=1.0, no_slip=True, initial_pressure=0.0) if ext else {}
    cfg = cf.SimConfig(n=n, h=h, dt=0.002, t_end=0.002 * 3, tol=1e-8, max_iter=its, variant="optimized",
                       preconditioner="jacobi", **kw)
    st = cf.initial_state(cfg)
    cache = cf.PoissonCache()
    for _ in range(2):
        cf.step(st, cfg, cache)
    torch.cuda.synchronize()


if part in ("step", "all"):
    steps(False)
    steps(True)
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
for order in ("csr", "sym") if part in ("step", "all") else ():
    op = cf.StencilOperator(n, h, order)
    y = op(x)
    op(x, out=y)
if part in ("step", "all"):
    a = cf.poisson_full_csr(n, h)
    y = cf.spmv(a, x)
    cf.spmv(a, x, out=y)
    s = cf.poisson_symmetric(n, h)
    y = cf.spmv_sym(s, x)
    cf.spmv_sym(s, x, out=y)
b = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, n ** 3), device="cuda")
op = cf.StencilOperator(n, h, "sym")
# the CG kernels on a dense random right-hand side: the default single pass,
# then the two-kernel loop (CF_CG_ALGO=two), then DIC (two-kernel + sweeps).
# (The cavity's first steps have mostly-zero CG vectors, which the memory
# system moves with fewer DRAM bytes, so the CG rows come from this part.)
if part == "step":
    torch.cuda.synchronize()
    print("ncu_table done", n, part)
    sys.exit(0)
cf.pcg(op, b, precond=cf.jacobi_from(op), tol=1e-12, max_iter=8)
os.environ["CF_CG_ALGO"] = "two"
op2 = cf.StencilOperator(n, h, "sym")
cf.pcg(op2, b, precond=cf.jacobi_from(op2), tol=1e-12, max_iter=8)
del os.environ["CF_CG_ALGO"]
pre = cf.dic_from(op)
cf.pcg(op, b, precond=pre, tol=1e-8, max_iter=3)
torch.cuda.synchronize()
print("ncu_table done", n)
