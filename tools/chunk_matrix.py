"""Debug tool: true vs recurrence residual at 128^3 (run under env overrides)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_03697_b200 as cf
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
op = cf.StencilOperator(n, 1.0 / n, "sym")
out = []
for rep in range(3):
    x, st = cf.pcg(op, b, precond=cf.jacobi_from(op), tol=1e-8, max_iter=20000)
    tr = float(torch.linalg.norm(b - op(x)) / torch.linalg.norm(b))
    out.append(f"{tr/st.final_residual_rel:.3f}")
print(os.environ.get("CF_TMA_CHUNKS_DIR"), os.environ.get("CF_TMA_CHUNKS_UPD"), " ".join(out), flush=True)
