"""Debug tool: compare the first fused-CG iterates with the oracle at one size."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_03697_b200 as cf
import oracle as orc
n = int(sys.argv[1]); order = sys.argv[2] if len(sys.argv) > 2 else "sym"
h = 1.0 / n
b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
a = orc.poisson_sym(n, h)
op = cf.StencilOperator(n, h, order)
for k in [int(a) for a in sys.argv[3].split(",")]:
    x, st = cf.pcg(op, b, precond=cf.jacobi_from(op), tol=1e-30, max_iter=k)
    xo, so = orc.pcg(lambda v, o: orc.spmv_sym(a, v, 8, o), b, precond=orc.jacobi_from(a), tol=1e-30, max_iter=k, threads=8)
    d = np.abs(x - xo).reshape(n, n, n)  # [k][j][i]
    idx = np.argwhere(d > 1e-9 * np.abs(xo).max())
    print(k, "rel", np.linalg.norm(x - xo) / np.linalg.norm(xo), "bad", len(idx), idx[:8].tolist(), flush=True)
# true vs recurrence residual at the end
x, st = cf.pcg(op, b, precond=cf.jacobi_from(op), tol=1e-8, max_iter=20000)
bt = torch.as_tensor(b, device="cuda")
print("final", st.iterations, st.final_residual_rel, float(torch.linalg.norm(bt - op(torch.as_tensor(x, device="cuda"))) / torch.linalg.norm(bt)))
