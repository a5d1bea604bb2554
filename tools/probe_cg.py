"""Profiling probe (not product): a bounded 256^3 fused CG solve.

    python tools/probe_cg.py [--n 256] [--iters 20] [--order sym]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--order", default="sym")
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
cf.load_library()
op = cf.StencilOperator(a.n, 1.0 / a.n, a.order)
b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, a.n ** 3), device="cuda")
pre = cf.jacobi_from(op)
for _ in range(a.repeat):
    x, st = cf.pcg(op, b, precond=pre, tol=1e-12, max_iter=a.iters)
ws = op._cg_ws
print(f"n={a.n} iters={st.iterations} loop_ms={ws.last_loop_ms:.3f} us/iter={1e3 * ws.last_loop_ms / st.iterations:.1f}")
