"""TMA-fed single-reduction pass (CF_CG_ALGO=spass) vs the two-kernel CG:
iterations, solution difference, true residual, us per iteration.

    python tools/spass_check.py [n ...]      (nx,ny,nz boxes as 96x80x72)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402


def run(shape, algo, b, tol=1e-8):
    os.environ["CF_CG_ALGO"] = algo
    n = shape[0]
    op = cf.StencilOperator(n, 1.0 / n, "sym", shape=None if len(set(shape)) == 1 else shape)
    pre = cf.jacobi_from(op)
    for _ in range(2):
        x, st = cf.pcg(op, b, precond=pre, tol=tol, max_iter=20000)
    ms = op._cg_ws.last_loop_ms
    res = float(torch.linalg.norm(b - op(x)) / torch.linalg.norm(b))
    return x, st, 1e3 * ms / max(st.iterations, 1), res


for a in sys.argv[1:] or ["64", "128", "256"]:
    shape = tuple(int(v) for v in a.split("x")) if "x" in a else (int(a),) * 3
    cells = shape[0] * shape[1] * shape[2]
    b = np.random.default_rng(0).uniform(-1, 1, cells)
    b -= b.mean()
    b = torch.as_tensor(b, device="cuda")
    x2, s2, t2, e2 = run(shape, "two", b)
    x1, s1, t1, e1 = run(shape, "spass", b)
    d = float(torch.linalg.norm(x1 - x2) / torch.linalg.norm(x2))
    print(f"{a}: two {s2.iterations} it {t2:.1f} us/it true res {e2:.2e} | spass {s1.iterations} it {t1:.1f} us/it "
          f"true res {e1:.2e} rec {s1.final_residual_rel:.2e} | rel x diff {d:.2e}", flush=True)
