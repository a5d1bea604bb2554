"""Debug tool: time the standalone stencil apply (config 3, 256^3)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2504_03697_b200 as cf
n = 256
x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n ** 3), device="cuda")
y = torch.empty_like(x)
op = cf.StencilOperator(n, 1.0 / n, os.environ.get("ORDER", "sym"))
for _ in range(3): op(x, out=y)
s = torch.cuda.current_stream(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(100): op(x, out=y)
b.record(s); torch.cuda.synchronize()
us = a.elapsed_time(b) * 10
print(os.environ.get("CF_APPLY", "lean"), os.environ.get("ORDER", "sym"), f"{us:.1f} us  {16 * n**3 / us / 1e3:.0f} GB/s")
