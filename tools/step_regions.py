"""Region times of 256^3 config-4 steps (wall-clock regions with stream sync).

    python tools/step_regions.py [n] [ext]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03697_b200 as cf  # noqa: E402
from paper_2504_03697_b200.profiling import Profiler, render_report  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ext = len(sys.argv) > 2 and sys.argv[2] == "ext"  # BASELINE's viscosity / lid velocity / no-slip
kw = dict(lid_accel=0.0, viscosity=0.001, lid_velocity=1.0, no_slip=True, initial_pressure=0.0) if ext else {}
cfg = cf.SimConfig(n=n, h=1.0 / n, dt=0.002, t_end=0.002 * 4, tol=1e-8, max_iter=20000, variant="optimized",
                   preconditioner="jacobi", **kw)
st = cf.initial_state(cfg)
cache = cf.PoissonCache()
cf.step(st, cfg, cache)
prof = Profiler()
with prof.region("cavityflow"):
    for _ in range(3):
        s = cf.step(st, cfg, cache, None, prof)
print(render_report(prof.stats()))
print("iterations", s.solve.iterations)
