"""One DIC-PCG solve (a few iterations) on one box, kernels launched from the
host (CF_CG_DIRECT) so that ncu sees the sweep kernels: nx ny nz [iterations]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CF_CG_DIRECT", "1")
os.environ.setdefault("CF_NO_SMALL", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

shp = tuple(int(a) for a in sys.argv[1:4])
its = int(sys.argv[4]) if len(sys.argv) > 4 else 3
b = np.random.default_rng(0).uniform(-1, 1, int(np.prod(shp)))
b -= b.mean()
op = cf.StencilOperator(max(shp), 1.0 / max(shp), "sym", shape=shp)
x, st = cf.pcg(op, torch.as_tensor(b, device="cuda"), precond=cf.dic_from(op), tol=1e-30, max_iter=its)
torch.cuda.synchronize()
print(shp, st.iterations, "iterations", op._cg_ws.last_loop_ms, "ms")
