"""Skewed-warp DIC sweeps against the level schedule after ONE PCG iteration
(x = alpha * M^-1 b): prints where the two differ."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

os.environ["CF_NO_SMALL"] = "1"
shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [(48, 48, 48)]
for shape in shapes:
    n = max(shape)
    b = torch.as_tensor(np.random.default_rng(7).standard_normal(int(np.prod(shape))), device="cuda")
    out = []
    for levels in ("1", None):
        if levels:
            os.environ["CF_DIC_LEVELS"] = levels
        else:
            os.environ.pop("CF_DIC_LEVELS", None)
        op = cf.StencilOperator(n, 1.0 / n, "sym", shape=shape)
        for it in (1, 2):
            x, st = cf.pcg(op, b, precond=cf.dic_from(op), tol=1e-30, max_iter=it)
            out.append(x.cpu().numpy().reshape(shape[2], shape[1], shape[0]))
    for it in (0, 1):
        bad = np.argwhere(out[it] != out[2 + it])
        print(shape, "iterations", it + 1, "mismatches", len(bad), "of", out[0].size)
        if len(bad):
            print("  first (k, j, i):", bad[:8].tolist())
            print("  k range", bad[:, 0].min(), bad[:, 0].max(), "j range", bad[:, 1].min(), bad[:, 1].max(), "i range",
                  bad[:, 2].min(), bad[:, 2].max())
            print("  distinct i%32:", sorted(set((bad[:, 2] % 32).tolist()))[:40])
            print("  distinct j%4:", sorted(set((bad[:, 1] % 4).tolist())))
