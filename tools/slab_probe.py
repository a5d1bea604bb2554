"""z-slab CG on one device: us per iteration of the peer-memory form (all
slabs in one launch per phase) and the NCCL form's emulation (per-slab
kernels + sum/scalar kernels), for several slab counts.

    python tools/slab_probe.py [--n 256] [--iters 100]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402
from paper_2504_03697_b200.distributed import PeerSlabCG, SlabCG  # noqa: E402
from paper_2504_03697_b200.parallel import SlabDecomposition  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--slabs", default="1,2,4,8")
a = ap.parse_args()
cf.load_library()
n = a.n
b = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
pl = n * n
for ns in (int(s) for s in a.slabs.split(",")):
    bounds = SlabDecomposition.bounds(n, ns).tolist()
    parts = [b[bounds[k] * pl:bounds[k + 1] * pl] for k in range(ns)]
    for name, cls in (("p2p", PeerSlabCG), ("nccl-emu", SlabCG)):
        solver = cls(n, n, n, 1.0 / n, "sym", bounds=bounds)
        for _ in range(2):
            xs, st = solver.solve(parts, 1e-14, a.iters, "jacobi")
        print(f"n={n} slabs={ns} {name:9s}: {1e3 * solver.last_loop_ms / st.iterations:7.1f} us/iter "
              f"({st.iterations} iterations)", flush=True)
        del solver
