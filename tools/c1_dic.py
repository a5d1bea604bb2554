"""Config 1 (16^3 cavity, 10 steps) with the reference's default DIC / baseline settings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

for pre, var in (("dic", "baseline"), ("dic", "optimized"), ("jacobi", "optimized")):
    cfg = cf.SimConfig(n=16, h=1.0 / 16, dt=0.01, t_end=0.1, tol=1e-6, max_iter=10000, preconditioner=pre,
                       variant=var)
    st = cf.initial_state(cfg)
    cache = cf.PoissonCache()
    cf.step(st, cfg, cache)
    torch.cuda.synchronize()
    t = time.perf_counter()
    its = [cf.step(st, cfg, cache).solve.iterations for _ in range(10)]
    torch.cuda.synchronize()
    print(pre, var, f"{(time.perf_counter() - t) / 10 * 1e3:.3f} ms/step", its, flush=True)
