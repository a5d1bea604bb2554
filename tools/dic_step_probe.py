import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2504_03697_b200 as cf
n = 256
op = cf.StencilOperator(n, 1.0 / n, "csr")
b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
pre = cf.dic_from(op)
x, st = cf.pcg(op, b, precond=pre, tol=1e-12, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 6, variant="baseline")
torch.cuda.synchronize()
print("its", st.iterations, "loop ms", op._cg_ws.last_loop_ms)
