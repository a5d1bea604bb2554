"""DIC wavefront pace: DIC-PCG minus Jacobi-PCG time per iteration on boxes of
1..N tiles, so the per-diagonal-step cost of one tile and the per-crossing
lag between tiles can be read apart (tiles are 16 x 8 cell columns over z)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402

shapes = [(16, 8, 256), (16, 8, 1024), (32, 8, 256), (16, 16, 256), (64, 8, 256), (16, 64, 256),
          (256, 8, 256), (16, 256, 256), (128, 128, 128), (256, 256, 256)]
if len(sys.argv) == 4:  # one box from the command line: nx ny nz
    shapes = [tuple(int(a) for a in sys.argv[1:4])]
for shp in shapes[: int(os.environ.get("NSHAPES", len(shapes)))]:
    nx, ny, nz = shp
    b = np.random.default_rng(0).uniform(-1, 1, nx * ny * nz)
    b -= b.mean()
    bd = torch.as_tensor(b, device="cuda")
    op = cf.StencilOperator(max(shp), 1.0 / max(shp), "sym", shape=shp)
    res = {}
    for name, pre in (("jacobi", cf.jacobi_from(op)), ("dic", cf.dic_from(op))):
        for _ in range(2):
            x, st = cf.pcg(op, bd, precond=pre, tol=1e-8, max_iter=300)
        res[name] = (st.iterations, 1e3 * op._cg_ws.last_loop_ms / st.iterations)
    steps = 2 * (nz + 16 + 8 - 2)
    ntx, nty = -(-nx // 16), -(-ny // 8)
    extra = res["dic"][1] - res["jacobi"][1]
    print(f"{shp} tiles {ntx}x{nty}: dic {res['dic'][1]:.1f} us/it, jacobi {res['jacobi'][1]:.1f}; "
          f"sweeps {extra:.1f} us = {1e3 * extra / steps:.0f} ns per own step", flush=True)
