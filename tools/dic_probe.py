"""DIC-preconditioned fused CG: iterations and time per iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

for n in [int(a) for a in (sys.argv[1:] or ["64", "128"])]:
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    b -= b.mean()
    bd = torch.as_tensor(b, device="cuda")
    op = cf.StencilOperator(n, 1.0 / n, "sym")
    for name, pre in (("jacobi", cf.jacobi_from(op)), ("dic", cf.dic_from(op))):
        for _ in range(2):
            x, st = cf.pcg(op, bd, precond=pre, tol=1e-8, max_iter=20000)
        ms = op._cg_ws.last_loop_ms
        print(f"n={n} {name}: {st.iterations} it, {ms:.2f} ms, {1e3 * ms / st.iterations:.1f} us/it", flush=True)
