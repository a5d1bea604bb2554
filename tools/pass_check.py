"""Single-reduction CG (CF_CG_ALGO default) vs the two-kernel form: iterations,
solution difference, us per iteration at several sizes."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

for n in [int(a) for a in (sys.argv[1:] or ["32", "48", "64", "128", "256"])]:
    b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
    res = {}
    for algo in ("two", "pass"):
        os.environ["CF_CG_ALGO"] = algo
        op = cf.StencilOperator(n, 1.0 / n, "sym")
        pre = cf.jacobi_from(op)
        for _ in range(2):
            x, st = cf.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000)
        ms = op._cg_ws.last_loop_ms
        res[algo] = (x, st.iterations, 1e3 * ms / max(st.iterations, 1))
    x2, i2, t2 = res["two"]
    x1, i1, t1 = res["pass"]
    d = float(torch.linalg.norm(x1 - x2) / torch.linalg.norm(x2))
    print(f"n={n}: two {i2} it {t2:.1f} us/it | pass {i1} it {t1:.1f} us/it | rel x diff {d:.2e}", flush=True)
