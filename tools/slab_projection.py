"""Per-GPU cost of a strong-scaling point measured on one GPU: the single
pass on one 512 x 512 x (512 / G) slab (the slab CG with one rank: its halo
planes are ghosts, no mailbox exchange) next to the whole 512^3 cube.

    python tools/slab_projection.py [G ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402
from paper_2504_03697_b200.distributed import PeerSlabCG  # noqa: E402

n = 512
for G in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    nzl = n // G
    b = torch.as_tensor(np.random.default_rng(G).uniform(-1, 1, n * n * nzl), device="cuda")
    solver = PeerSlabCG(n, n, nzl, 1.0 / n, "sym", bounds=[0, nzl])
    for _ in range(2):
        xs, st = solver.solve([b], 1e-14, 60, "jacobi")
    us = 1e3 * solver.last_loop_ms / st.iterations
    print(f"G={G}: one {n}x{n}x{nzl} slab, single pass: {us:.1f} us per iteration "
          f"({'single pass' if solver.single_pass else 'two-kernel'})", flush=True)
    del solver
