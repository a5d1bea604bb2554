"""Debug tool: recurrence vs true residual of the fused CG over grid sizes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_03697_b200 as cf
for n in [int(a) for a in sys.argv[1:]]:
    b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
    for order in ("sym",):
        op = cf.StencilOperator(n, 1.0 / n, order)
        x, st = cf.pcg(op, b, precond=cf.jacobi_from(op), tol=1e-8, max_iter=20000)
        tr = float(torch.linalg.norm(b - op(x)) / torch.linalg.norm(b))
        ws = op._cg_ws
        print(n, order, st.iterations, f"rec={st.final_residual_rel:.3e} true={tr:.3e}", flush=True)
