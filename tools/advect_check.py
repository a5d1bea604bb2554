"""TMA-fed advection (default) vs the global-gather kernel (CF_ADVECT=global):
bit-identical output and time per call at n^3 on a random velocity field
scaled to a given CFL number (|v| dt / h).

    python tools/advect_check.py [n] [cfl ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03697_b200 as cf  # noqa: E402
from paper_2504_03697_b200.sim import _advect_into  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfls = [float(a) for a in sys.argv[2:]] or [0.5, 1.0, 2.5]
h, dt = 1.0 / n, 0.002
cfg = cf.SimConfig(n=n, h=h, dt=dt, t_end=dt, tol=1e-8)
spec = cf.GridSpec(n, h)
rng = np.random.default_rng(0)
for cfl in cfls:
    vmax = cfl * h / dt
    src = cf.VelocityField(spec)
    for t in src._phys:
        t.copy_(torch.as_tensor(rng.uniform(-vmax, vmax, tuple(t.shape)), device="cuda"))
    out = {}
    for mode in ("global", "tma"):
        if mode == "global":
            os.environ["CF_ADVECT"] = "global"
        else:
            os.environ.pop("CF_ADVECT", None)
        dst = cf.VelocityField(spec)
        _advect_into(src, dst, cfg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _advect_into(src, dst, cfg)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = ([t.clone() for t in dst._phys], e0.elapsed_time(e1) / 5)
    same = all(torch.equal(a, b) for a, b in zip(out["global"][0], out["tma"][0]))
    nbytes = 48 * (n + 1) * n * n
    print(f"n={n} cfl={cfl}: bitwise {same}; global {out['global'][1]:.3f} ms, tma {out['tma'][1]:.3f} ms "
          f"({nbytes / out['tma'][1] / 1e6:.0f} GB/s on 48 F)", flush=True)
