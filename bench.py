"""Benchmark of the cavity time-step hot path (BASELINE.json config 4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 256]

One bench "step" is one full time step of the 256^3 lid-driven cavity
(h=1/256, dt=0.002, CG tol 1e-8, Jacobi PCG, optimized variant) in
reference physics, continuing the simulation from rest.
Inputs: the fields, resident in HBM; at 537 MB of velocity+pressure (and
4 x 134 MB of CG vectors) every pass is far larger than the 126 MB L2, so
no flush is needed between iterations.

value   = CG iterations / second over the K timed steps (whole steps, so
          advection/divergence/correction time is included), device-timed
          with CUDA events between barrier+synchronize brackets, max over ranks.
e2e     = the same metric through the public API with the state in pinned
          HOST memory: H2D of the step's inputs (u, v, w; p too with
          warm_start) + step() + D2H of u, v, w, p every step; the velocity's
          D2H and the next step's H2D run chunk-pipelined on two copy streams
          (full-duplex PCIe), the pressure's D2H beside the next step.
roofline: the fused CG iteration (the single TMA-fed pass by default; the
          two-kernel loop with CF_CG_ALGO=two), algorithmic bytes 88*N per
          iteration / measured loop time per iteration,
          against MEASURED_PEAKS.json hbm_gbs; design_frac / dram_frac on the
          bytes the kernels move (40 N single pass) / ncu measured.
cpu_baseline: the oracle port (oracle/, the reference's algorithm in C with
          the reference's WorkerPool chunking) on a bounded sample: 256^3
          Jacobi PCG iterations with the symmetric SpMV, all host threads.
--impl reference: that CPU path alone, as the driver's reference arm.
--gpus N > 1: z-slab decomposition, one slab per GPU, max over ranks.  Run
          outside torchrun, bench.py re-executes itself under
          torch.distributed.run (N ranks, 127.0.0.1).  Default --scaling weak:
          the cavity extruded to 256x256x(256*N), one 256^3 slab per GPU (value
          in 256^3-equivalent CG iterations/s); --scaling strong: the 256^3
          cube split over the GPUs.
sub-records (each its own CUDA-event timed region after the main one):
          config5 (512^3, BASELINE config 5; at N > 1 the cube split over the
          ranks -> strong-scaling points), dic (the reference's default
          baseline/DIC solver at 256^3), config4_as_written (nu=0.001, lid
          velocity 1, no-slip); --no-extra skips them.
roofline.traffic: DRAM bytes per CG iteration from the newest committed ncu
          summary of the same CG form (profiles/ncu_cg_r*.json, "form"; named
          in traffic_source).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG iterations/s and fused-iteration HBM GB/s (% of peak); sim steps/s at 256³"
UNIT = "CG iterations/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU baseline


def cpu_baseline(n: int, iters: int, threads: int):
    """Oracle PCG on a 256^3 Poisson system: CG iterations/s on host cores."""
    import numpy as np

    import oracle as orc

    a = orc.poisson_sym(n, 1.0 / n)
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    pre = orc.jacobi_from(a)
    op = lambda v, o: orc.spmv_sym(a, v, threads, o)  # noqa: E731
    orc.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, variant="optimized", threads=threads, max_count=1)
    t0 = time.perf_counter()
    _, st = orc.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, variant="optimized", threads=threads,
                    max_count=iters)
    dt = time.perf_counter() - t0
    return st.iterations / dt, dt, st.iterations


def run_reference(args, rank):
    if rank != 0:
        return 0
    import numpy as np

    import oracle as orc

    threads = os.cpu_count() or 1
    n = args.grid
    a = orc.poisson_sym(n, 1.0 / n)
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    pre = orc.jacobi_from(a)
    op = lambda v, o: orc.spmv_sym(a, v, threads, o)  # noqa: E731
    per_step = args.ref_iters
    for _ in range(args.warmup):
        orc.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, threads=threads, max_count=per_step)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        _, st = orc.pcg(op, b, precond=pre, tol=1e-8, max_iter=20000, threads=threads, max_count=per_step)
        total += st.iterations
    dt = time.perf_counter() - t0
    value = total / dt
    sample = (f"{n}^3 Poisson Jacobi-PCG (symmetric CSR SpMV, reference chunking), {per_step} iterations "
              f"per step, oracle port in C/OpenMP")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": args.scaling if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cavity-{n}^3 pressure solve (CPU sample)", "n": n, "tol": 1e-8,
                   # CPU cost per iteration is linear in cells, so the n^3 rate is
                   # also the n^3-equivalent rate of the weak-scaling boxes
                   "value_normalisation": "n^3-equivalent CG iterations/s"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


# ---------------------------------------------------------------- our arm


# the CG form a solve ran (solver.FORMS) -> roofline description / bytes per cell it moves
KERNELS = {"single-pass": "fused CG iteration: ONE TMA-fed single-reduction pass (cg_spass_kernel; "
                          "x updated every 2nd pass)",
           "two-kernel": "fused CG iteration (cg_dir_lean2 + cg_update_tma; x updated every 2nd iteration)"}
DESIGN_BYTES = {"single-pass": 40, "two-kernel": 60}


def load_traffic(form=None):
    """Per-iteration DRAM bytes of the fused CG kernels from the newest committed
    ncu summary for this CG form (ncu cannot run inside the timed bench):
    (bytes, source path)."""
    import glob
    found = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_cg_r*.json")))
    for path in reversed(found):
        try:
            with open(path) as f:
                d = json.load(f)
        except Exception:
            continue
        if d.get("form", "two-kernel") == (form or "two-kernel"):
            return d.get("dram_bytes_per_iteration"), os.path.relpath(path, ROOT)
    return None, None


class RoundTrip:
    """The e2e state round trip between steps: the step's outputs go D2H and
    the next step's inputs (the same host copy) go back H2D in ~32 MB chunks
    on two copy streams -- chunk c's D2H beside chunk c-1's H2D (PCIe is full
    duplex), each chunk uploaded only after it landed in host memory -- and the
    output-only arrays (the pressure) go D2H beside the next step.  Every
    step still uploads its inputs from pinned memory and reads its whole
    result back inside the timed region."""

    CH = 4 << 20  # doubles per chunk

    def __init__(self, stream):
        import torch
        self.torch = torch
        self.stream = stream
        self.d2h, self.h2d = torch.cuda.Stream(), torch.cuda.Stream()

    def _chunks(self, ts):
        return [(t.view(-1), a, min(a + self.CH, t.numel())) for t in ts for a in range(0, t.numel(), self.CH)]

    def before_step(self):
        self.stream.wait_stream(self.h2d)

    def after_step(self, dev_in, pin_in, dev_out, pin_out):
        torch = self.torch
        done = torch.cuda.Event()
        done.record(self.stream)
        self.d2h.wait_event(done)
        evs = []
        with torch.cuda.stream(self.d2h):
            for (d_, a, b), (h_, _, _) in zip(self._chunks(dev_in), self._chunks(pin_in)):
                h_[a:b].copy_(d_[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.d2h)
                evs.append(ev)
            for h_, d_ in zip(pin_out, dev_out):
                h_.copy_(d_, non_blocking=True)
        with torch.cuda.stream(self.h2d):
            for ev, (d_, a, b), (h_, _, _) in zip(evs, self._chunks(dev_in), self._chunks(pin_in)):
                self.h2d.wait_event(ev)
                d_[a:b].copy_(h_[a:b], non_blocking=True)

    def finish(self):
        self.stream.wait_stream(self.d2h)
        self.stream.wait_stream(self.h2d)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2504_03697_b200 as cf

    torch.cuda.set_device(local_rank)
    cf.load_library()
    n = args.grid
    cfg = cf.SimConfig(n=n, h=1.0 / n, dt=args.dt, t_end=args.dt * (args.warmup + 2 * args.steps), tol=1e-8,
                       max_iter=20000, variant="optimized", preconditioner="jacobi")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1 or args.force_slabs:
        return run_slabs(args, cfg, rank, world, local_rank, barrier)
    state = cf.initial_state(cfg)
    cache = cf.PoissonCache()
    for _ in range(args.warmup):
        cf.step(state, cfg, cache)

    # ---- device-resident timed region
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its, loop_ms, launches, form = [], 0.0, 0, None
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            s = cf.step(state, cfg, cache)
            its.append(s.solve.iterations)
            ws = cache.operator(cfg)._cg_ws
            loop_ms += ws.last_loop_ms
            # forces, advect, divergence, correct + the solve's own count (init,
            # the while body of two iterations, the x fix-up: cf_cg_last_form)
            launches += 4 + ws.last_launches
            form = ws.last_form
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms, float(sum(its))], device="cuda", dtype=torch.float64)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms_max, total_its = float(mx[0]), float(t[1])
    else:
        ms_max, total_its = ms, float(sum(its))
    value = total_its / (ms_max / 1e3)

    # ---- end to end through the public API with host-resident state: every
    # step uploads its inputs (the velocity field; the pressure is an output
    # of a cold-start step, src/sim.py:379-423) from pinned memory and reads
    # the whole new state (u, v, w, p) back
    phys = [*state.vel._phys, state.p.data]
    pinned = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in phys]
    for h_, d_ in zip(pinned, phys):
        h_.copy_(d_)
    n_in = 3 if not cfg.warm_start else 4
    h2d = sum(t.numel() * t.element_size() for t in phys[:n_in])
    d2h = sum(t.numel() * t.element_size() for t in phys)
    barrier()
    # The round trip between steps is pipelined in ~32 MB chunks over two copy
    # streams: chunk c of the new velocity goes D2H while chunk c-1 goes back
    # H2D (PCIe is full duplex), each chunk uploaded only after it landed in
    # host memory; the pressure (an output only) goes D2H beside the next
    # step.  Every step still uploads its inputs from pinned memory and reads
    # its whole result back inside the timed region.
    rt = RoundTrip(stream)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_its = 0
    e2.record(stream)
    for _ in range(args.steps):
        rt.before_step()  # this step's inputs are on the device
        s = cf.step(state, cfg, cache)
        e2e_its += s.solve.iterations
        phys = [*state.vel._phys, state.p.data]
        rt.after_step(phys[:n_in], pinned[:n_in], phys[n_in:], pinned[n_in:])
    rt.finish()
    e3.record(stream)
    barrier()
    e2e_ms = e2.elapsed_time(e3)
    e2e_value = e2e_its * (world if world > 1 else 1) / (e2e_ms / 1e3)

    if rank != 0:
        return 0
    peak, peak_kind = peaks()
    cells = n ** 3
    alg_bytes = 88 * cells
    iter_s = (loop_ms / 1e3) / max(sum(its), 1)
    achieved = alg_bytes / iter_s / 1e9
    design = DESIGN_BYTES.get(form, 60)
    traffic, traffic_src = load_traffic(form)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"lid-driven cavity {n}^3 (BASELINE config 4), one time step per bench step",
                   "n": n, "h": 1.0 / n, "dt": args.dt, "tol": 1e-8, "preconditioner": "jacobi",
                   "variant": "optimized", "physics": "reference (lid acceleration, inviscid)",
                   "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "sim_steps_per_s": args.steps / (ms_max / 1e3),
        "cg_iterations": its,
        "fused_iter_us": iter_s * 1e6,
        "fused_iter_gbs": achieved,
        "fused_iter_frac": achieved / peak,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": KERNELS.get(form, form),
                     "algorithmic_bytes_per_iteration": alg_bytes, "design_bytes_per_iteration": design * cells,
                     # the same iteration time against the bytes this design moves (40 N for the
                     # single pass, 60 N for the two-kernel loop) and against the DRAM traffic ncu
                     # measured per iteration (frac above uses the reference op sequence's 88 N,
                     # SURVEY.md 8(d), hence > 1)
                     "design_frac": design * cells / iter_s / 1e9 / peak,
                     "dram_frac": (traffic / iter_s / 1e9 / peak) if traffic else None,
                     "peak_kind": peak_kind},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if not args.no_extra:
        del state, cache, pinned, phys
        torch.cuda.empty_cache()
        line.update(extra_records(args))
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, k = cpu_baseline(n, args.cpu_iters, threads)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"{n}^3 Jacobi-PCG, {k} iterations ({dt:.1f} s), oracle port"}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- sub-records


def _timed_steps(step, steps, warmup):
    """Device time (CUDA events, synchronised both sides) of `steps` calls
    after `warmup` untimed ones; returns (ms, [StepStats])."""
    import torch

    for _ in range(warmup):
        step()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    out = [step() for _ in range(steps)]
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def _cavity_record(cfg, steps, warmup, note):
    import torch

    import paper_2504_03697_b200 as cf

    st = cf.initial_state(cfg)
    cache = cf.PoissonCache()
    loop = []

    def step():
        s = cf.step(st, cfg, cache)
        loop.append(cache.operator(cfg)._cg_ws.last_loop_ms)
        return s

    ms, out = _timed_steps(step, steps, warmup)
    its = [s.solve.iterations for s in out]
    loop_ms = sum(loop[-steps:])
    rec = {"workload": note, "n": cfg.n, "dt": cfg.dt, "tol": cfg.tol, "preconditioner": cfg.preconditioner,
           "variant": cfg.variant, "steps_timed": steps, "warmup": warmup, "ms_per_step": ms / steps,
           "sim_steps_per_s": steps / (ms / 1e3), "cg_iterations": its,
           "cg_iterations_per_s": sum(its) / (ms / 1e3),
           "cg_ms_per_iteration": loop_ms / max(sum(its), 1), "converged": all(s.solve.converged for s in out)}
    del st, cache
    torch.cuda.empty_cache()
    return rec


def extra_records(args):
    """Sub-records of the N=1 line (each its own timed region, CUDA events):
    config5 -- BASELINE config 5's 512^3 cavity (h=1/512, dt=0.001, tol 1e-8),
        reference physics, Jacobi: the single-GPU t_1 of the strong-scaling
        curve (N > 1 lines carry the same cube split over the ranks);
    dic -- the reference's DEFAULT solver (baseline variant, DIC preconditioner,
        src/sim.py:65) on the config-4 cavity at 256^3;
    config4_as_written -- config 4's physics as BASELINE states it
        (nu = 0.001, lid velocity 1, no-slip, explicit diffusion)."""
    import paper_2504_03697_b200 as cf

    out = {}
    n = args.grid
    if args.config5_steps > 0:
        cfg5 = cf.SimConfig(n=512, h=1.0 / 512, dt=0.001, t_end=1.0, tol=1e-8, max_iter=50000,
                            variant="optimized", preconditioner="jacobi")
        out["config5"] = _cavity_record(cfg5, args.config5_steps, 1,
                                        "BASELINE config 5: 512^3 cavity, reference physics, 1 GPU")
    base = dict(n=n, h=1.0 / n, dt=args.dt, t_end=1.0, tol=1e-8, max_iter=50000)
    out["dic"] = _cavity_record(cf.SimConfig(variant="baseline", preconditioner="dic", **base), 2, 1,
                                f"{n}^3 cavity (config 4 grid) with the reference's default solver: "
                                "baseline variant, DIC preconditioner")
    out["config4_as_written"] = _cavity_record(
        cf.SimConfig(variant="optimized", preconditioner="jacobi", lid_accel=0.0, viscosity=0.001,
                     lid_velocity=1.0, no_slip=True, initial_pressure=0.0, **base), 2, 1,
        f"BASELINE config 4 as written: {n}^3, nu=0.001, lid velocity 1, no-slip, explicit diffusion")
    return out


def run_slabs(args, cfg, rank, world, local_rank, barrier):
    """N > 1: the cavity z-slab sharded over the ranks, one slab per GPU:
    velocity/pressure halos by NCCL P2P; the CG with its collectives fused
    into the kernels over peer memory (cf_pcg, default) or as NCCL all-reduce
    + r-halo send/recv (cf_dcg, --collective nccl).

    --scaling weak (default): the config-4 cavity extruded in z to
    n x n x (n*N) cells, one n^3 slab per GPU (the per-GPU work of the N=1
    run; BASELINE config 5's weak-scaling form).  value = global CG
    iterations/s x cells / n^3, i.e. n^3-equivalent iterations/s, the N=1
    unit.  --scaling strong: the n^3 cube split over the N GPUs."""
    import dataclasses

    import torch
    import torch.distributed as dist

    from paper_2504_03697_b200.distributed import SlabSim
    from paper_2504_03697_b200.parallel import SlabDecomposition

    n = cfg.n
    weak = args.scaling == "weak"
    nz = n * world if weak else n
    if weak:
        cfg = dataclasses.replace(cfg, shape=(n, n, nz))
    norm = nz / n  # cells / n^3
    dec = SlabDecomposition(n, n, nz, world, rank)
    from paper_2504_03697_b200.distributed import PeerLinkError

    try:
        sim = SlabSim(cfg, [dec.z0, dec.z1], distributed=True, collective=args.collective)
    except PeerLinkError as err:  # all ranks raise alike: the NCCL form on every rank
        print(f"[bench] {err}; using the NCCL collective form", file=sys.stderr)
        args.collective = "nccl"
        sim = SlabSim(cfg, [dec.z0, dec.z1], distributed=True, collective="nccl")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        sim.step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its, loop_ms = [], 0.0
    with ClockSampler(local_rank) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            s = sim.step()
            its.append(s.solve.iterations)
            loop_ms += sim.cg.last_loop_ms
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, loop_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, loop_max = float(t[0]), float(t[1])
    value = norm * sum(its) / (ms_max / 1e3)  # global CG iterations (every rank runs the same ones)
    # e2e: each rank's slab state through pinned host memory every step --
    # upload u, v, w (the cold-start pressure solve's inputs), read u, v, w, p back
    sl = sim.slabs[0]
    phys = [*sl.vel[sl.cur], sl.p]
    pinned = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in phys]
    for h_, d_ in zip(pinned, phys):
        h_.copy_(d_)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e2.record(stream)
    e2e_its = 0
    rt = RoundTrip(stream)
    for _ in range(args.steps):
        rt.before_step()
        s = sim.step()
        e2e_its += s.solve.iterations
        rt.after_step([*sl.vel[sl.cur]], pinned[:3], [sl.p], pinned[3:])
    rt.finish()
    e3.record(stream)
    barrier()
    t2 = torch.tensor([e2.elapsed_time(e3)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = norm * e2e_its / (float(t2[0]) / 1e3)
    bytes_in = sum(x.numel() * x.element_size() for x in phys[:3])
    bytes_out = sum(x.numel() * x.element_size() for x in phys)
    clock_summary = clocks.summary()
    single_pass = bool(getattr(sim.cg, "single_pass", False))
    c5 = None
    if not args.no_extra and args.config5_steps > 0:
        del sim, sl, phys, pinned
        torch.cuda.empty_cache()
        c5 = config5_slabs(args, rank, world, barrier)
    if rank != 0:
        return 0
    peak, peak_kind = peaks()
    cells_rank = n * n * dec.planes
    iter_s = (loop_max / 1e3) / max(sum(its), 1)
    achieved = 88 * cells_rank / iter_s / 1e9
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": (f"lid-driven cavity {n}x{n}x{nz} (BASELINE config 4 extruded in z), one {n}^3 "
                                f"z-slab per GPU" if weak else
                                f"lid-driven cavity {n}^3 (BASELINE config 4), z-slab over {world} GPUs"),
                   "shape": [n, n, nz], "n": n, "h": 1.0 / n,
                   "value_normalisation": ("global CG iterations/s x cells/n^3 (n^3-equivalent iterations/s)"
                                           if weak else "global CG iterations/s"), "dt": args.dt, "tol": 1e-8, "preconditioner": "jacobi",
                   "variant": "optimized", "physics": "reference (lid acceleration, inviscid)",
                   "parallelism": f"zslab{world}", "collective": args.collective, "l2": "inputs larger than L2 (no flush needed)"},
        "sim_steps_per_s": args.steps / (ms_max / 1e3), "cg_iterations": its,
        "fused_iter_us": iter_s * 1e6, "fused_iter_gbs_per_gpu": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None,
                     "kernel": (f"per-GPU z-slab CG iteration: one single-reduction pass (sp_slab_pass; halo planes "
                                f"stored into the neighbours, one mailbox all-reduce; {args.collective})"
                                if single_pass else
                                f"per-GPU z-slab CG iteration (dir + update + all-reduces + r halo; {args.collective})"),
                     "algorithmic_bytes_per_iteration": 88 * cells_rank, "peak_kind": peak_kind},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bytes_in * world,
                "d2h_bytes_per_step": bytes_out * world},
        # step kernels (forces, advect, divergence, correction, halo packing ~10) + the CG's:
        # single pass 2 init + 1 per iteration (+ odd-count early exit) + fix-up; two-kernel 6 per iteration
        "gpu_launches": sum((i + (i & 1) + 3 + 10) if single_pass else (6 * i + 10) for i in its),
        "clocks": clock_summary,
        **({"config5": c5} if c5 else {}),
    }))
    return 0


def config5_slabs(args, rank, world, barrier):
    """BASELINE config 5 (512^3, h=1/512, dt=0.001, tol 1e-8, reference
    physics, Jacobi) as a strong-scaling point: the 512^3 cube split into
    `world` z-slabs.  Against the N=1 line's config5 record (t_1) the driver's
    SCALE runs give E(N) = t_1 / (N t_N).  Device time, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2504_03697_b200 as cf
    from paper_2504_03697_b200.distributed import SlabSim
    from paper_2504_03697_b200.parallel import SlabDecomposition

    cfg = cf.SimConfig(n=512, h=1.0 / 512, dt=0.001, t_end=1.0, tol=1e-8, max_iter=50000,
                       variant="optimized", preconditioner="jacobi")
    dec = SlabDecomposition(512, 512, 512, world, rank)
    sim = SlabSim(cfg, [dec.z0, dec.z1], distributed=True, collective=args.collective)
    sim.step()
    barrier()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    its, loop = [], 0.0
    for _ in range(args.config5_steps):
        its.append(sim.step().solve.iterations)
        loop += sim.cg.last_loop_ms
    b.record(stream)
    barrier()
    t = torch.tensor([a.elapsed_time(b), loop], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, loop_ms = float(t[0]), float(t[1])
    del sim
    torch.cuda.empty_cache()
    return {"workload": f"BASELINE config 5: 512^3 cavity, reference physics, z-slab over {world} GPUs (strong)",
            "n": 512, "dt": 0.001, "tol": 1e-8, "preconditioner": "jacobi", "steps_timed": args.config5_steps,
            "warmup": 1, "ms_per_step": ms / args.config5_steps, "sim_steps_per_s": args.config5_steps / (ms / 1e3),
            "cg_iterations": its, "cg_iterations_per_s": sum(its) / (ms / 1e3),
            "cg_ms_per_iteration": loop_ms / max(sum(its), 1), "collective": args.collective}


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-exec this script under
    torch.distributed.run, one rank per GPU on this node (127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dry_run(args, rank, world) -> int:
    """Plumbing check without a GPU: the rank layout bench.py would use, over
    gloo, with one all-reduce (the timing reduction) across the ranks."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "world": world, "n_gpus": args.gpus, "max_rank_plus_1": float(t[0]),
                          "impl": args.impl}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--dt", type=float, default=0.002)
    ap.add_argument("--cpu-iters", type=int, default=40)
    ap.add_argument("--ref-iters", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config5 / dic / config4_as_written sub-records")
    ap.add_argument("--config5-steps", type=int, default=2, help="timed 512^3 steps of the config5 sub-record")
    ap.add_argument("--collective", choices=("p2p", "nccl"), default="p2p",
                    help="z-slab CG collectives (N > 1): fused peer-memory kernels, or NCCL calls")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="N > 1: one n^3 slab per GPU (weak, default) or the n^3 cube split over the GPUs (strong)")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the z-slab/NCCL path even on one rank (plumbing check)")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank)
    use_pg = world > 1 or args.force_slabs
    if use_pg:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if use_pg:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
