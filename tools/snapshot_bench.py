"""Time the snapshot path: device cell-centring + D2H +
native CSV writer at 128^3 / 256^3, against the reference's formatter rule
restated in the oracle (pure Python repr, single thread) on a 32^3 sample
scaled per row.  Prints one JSON line per size."""

import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03697_b200 as cf  # noqa: E402
import oracle as orc  # noqa: E402


def state(n):
    cfg = cf.SimConfig(n=n, h=1.0 / n, dt=0.002, t_end=0.002)
    st = cf.initial_state(cfg)
    g = torch.Generator(device="cuda").manual_seed(0)
    for comp in st.vel.components():
        comp.copy_(torch.randn(comp.shape, dtype=torch.float64, device="cuda", generator=g))
    st.p.data.copy_(torch.randn(st.p.data.shape, dtype=torch.float64, device="cuda", generator=g))
    return st


def main():
    threads = os.cpu_count() or 1
    d = tempfile.mkdtemp()
    s32 = state(32)
    u, v, w = s32.vel.numpy()
    cols = orc.snapshot_columns(orc.State(u, v, w, s32.p.numpy()), 1.0 / 32)
    t0 = time.perf_counter()
    orc.snapshot_csv(cols)
    py_row = (time.perf_counter() - t0) / 32 ** 3
    for n in (128, 256):
        st = state(n)
        path = os.path.join(d, f"s{n}.csv")
        cf.write_snapshot(st, path, mode="buffered_parallel", threads=threads)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cf.write_snapshot(st, path, mode="buffered_parallel", threads=threads)
        t_par = time.perf_counter() - t0
        t0 = time.perf_counter()
        cf.write_snapshot(st, path, mode="serial")
        t_ser = time.perf_counter() - t0
        size = os.path.getsize(path)
        os.remove(path)
        print(json.dumps({"n": n, "rows": n ** 3, "bytes": size, "native_parallel_s": t_par, "threads": threads,
                          "native_serial_s": t_ser, "python_repr_est_s": py_row * n ** 3,
                          "speedup_vs_python": py_row * n ** 3 / t_par}))


if __name__ == "__main__":
    main()
