"""Region profiler and report tools (mirror of src/bench.py).

Same region names, nesting rule (identity = the (parent, name) pair),
``RegionStats`` records, JSON report format, comparison table and
scaling-sweep CSV as the reference, so its ``compare_reports`` and viz
scripts consume runs of this package unchanged.

Device timing: the kernels are asynchronous, so a wall-clock region
(``timer="wall"``, the default) synchronises the current CUDA stream at
both ends -- the recorded time is the device work the region enqueued plus
its host time.  ``timer="events"`` instead records a CUDA event pair on the
current stream per region call (no synchronisation inside the run) and
reports device-stream time; regions that do only host work (file output)
read as ~0 there.
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass, replace


class ProfileError(RuntimeError):
    pass


@dataclass
class RegionStats:
    name: str
    parent: str | None
    calls: int
    inclusive_seconds: float
    fraction: float


_FIELDS = ("name", "parent", "calls", "inclusive_seconds", "fraction")


def _sync():
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()
    except Exception:  # pragma: no cover - profiling must never break a run
        pass


class _Region:
    __slots__ = ("_prof", "_name")

    def __init__(self, prof, name):
        self._prof = prof
        self._name = name

    def __enter__(self):
        self._prof.enter(self._name)

    def __exit__(self, exc_type, exc, tb):
        self._prof.exit(self._name)
        return False


class Profiler:
    """Call counts and inclusive time per nested region path (src/bench.py:60-120)."""

    _FOLD_AT = 4096  # pending event pairs before they are resolved

    def __init__(self, sync: bool = True, timer: str = "wall"):
        if timer not in ("wall", "events"):
            raise ValueError(f"timer must be 'wall' or 'events', got {timer!r}")
        self._nodes = {}  # path tuple -> [calls, ns]
        self._path = []
        self._starts = []
        self._sync = sync
        self._events = timer == "events"
        self._pending = []  # (path, start event, end event)

    def enter(self, name: str):
        if self._events:
            import torch

            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._starts.append(ev)
        else:
            if self._sync:
                _sync()
            self._starts.append(time.perf_counter_ns())
        self._path.append(name)

    def exit(self, name: str):
        if not self._path or self._path[-1] != name:
            open_name = self._path[-1] if self._path else None
            raise ProfileError(f"unbalanced region exit: got {name!r} while {open_name!r} is open")
        key = tuple(self._path)
        self._path.pop()
        start = self._starts.pop()
        node = self._nodes.setdefault(key, [0, 0])
        node[0] += 1
        if self._events:
            import torch

            end = torch.cuda.Event(enable_timing=True)
            end.record()
            self._pending.append((key, start, end))
            if len(self._pending) >= self._FOLD_AT:
                self._resolve()
        else:
            if self._sync:
                _sync()
            node[1] += time.perf_counter_ns() - start

    def _resolve(self):
        if not self._pending:
            return
        self._pending[-1][2].synchronize()
        for key, a, b in self._pending:
            self._nodes[key][1] += int(round(a.elapsed_time(b) * 1e6))
        self._pending.clear()

    def region(self, name: str) -> _Region:
        return _Region(self, name)

    def record(self, name: str, calls: int, seconds: float):
        """Add `calls` and `seconds` to the child region `name` of the open
        region without timing it (rows of work done inside one fused kernel)."""
        node = self._nodes.setdefault(tuple(self._path) + (name,), [0, 0])
        node[0] += int(calls)
        node[1] += int(round(seconds * 1e9))

    def reset(self):
        if self._path:
            raise ProfileError(f"cannot reset while region {self._path[-1]!r} is open")
        self._nodes.clear()
        self._pending.clear()

    def stats(self) -> list:
        """Depth-first records, children in first-entry order; fraction is of
        the summed top-level time."""
        if self._path:
            raise ProfileError(f"region {self._path[-1]!r} is still open")
        self._resolve()
        children = {}
        for path in self._nodes:
            children.setdefault(path[:-1], []).append(path)
        total_ns = sum(self._nodes[p][1] for p in children.get((), []))
        out = []
        stack = list(reversed(children.get((), [])))
        while stack:
            path = stack.pop()
            calls, ns = self._nodes[path]
            if total_ns > 0:
                frac = ns / total_ns
            else:
                frac = 1.0 if len(path) == 1 else 0.0
            out.append(RegionStats(path[-1], path[-2] if len(path) > 1 else None, calls, ns * 1e-9, frac))
            stack.extend(reversed(children.get(path, [])))
        return out


class NullProfiler:
    def enter(self, name):
        pass

    def exit(self, name):
        pass

    def region(self, name):
        return _NullRegion()

    def record(self, name, calls, seconds):
        pass

    def stats(self):
        return []


class _NullRegion:
    __slots__ = ()

    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


NULL_PROFILER = NullProfiler()


# ---------------------------------------------------------------- reports


def _tree_labels(stats) -> list:
    """Region names with box-drawing tree prefixes, for the depth-first
    record order ``Profiler.stats`` produces."""
    # rebuild the tree: a record's parent is the nearest open ancestor named ``parent``
    kids = {-1: []}
    open_stack = []  # (index, name)
    for idx, rec in enumerate(stats):
        while open_stack and open_stack[-1][1] != rec.parent:
            open_stack.pop()
        parent_idx = open_stack[-1][0] if open_stack else -1
        kids.setdefault(parent_idx, []).append(idx)
        kids[idx] = []
        open_stack.append((idx, rec.name))
    labels = [""] * len(stats)

    def walk(idx, trunk, depth):
        for pos, child in enumerate(kids[idx]):
            name = stats[child].name
            if depth == 0:  # top-level regions carry no prefix
                labels[child] = name
                walk(child, "", 1)
                continue
            last = pos == len(kids[idx]) - 1
            labels[child] = trunk + ("└─ " if last else "├─ ") + name
            walk(child, trunk + ("   " if last else "│  "), depth + 1)

    walk(-1, "", 0)
    return labels


def render_report(stats) -> str:
    """Hotspot table in tree order (src/bench.py:195-207)."""
    labels = _tree_labels(stats)
    width = max([len("Region")] + [len(s) for s in labels])
    rows = [f"{'Region':<{width}}  {'Calls':>8}  {'Incl. s':>10}  {'Rt. %':>7}"]
    for label, rec in zip(labels, stats):
        rows.append(f"{label:<{width}}  {rec.calls:>8d}  {rec.inclusive_seconds:>10.3f}  {100.0 * rec.fraction:>7.2f}")
    return "\n".join(rows)


def save_report(stats, path) -> None:
    """JSON list of records (src/bench.py:210-223)."""
    with open(path, "w", encoding="utf-8") as f:
        json.dump([{k: getattr(r, k) for k in _FIELDS} for r in stats], f, indent=2)
        f.write("\n")


def load_report(path) -> list:
    """src/bench.py:226-232 (also reads this package's round-1 {"regions": [...]} form)."""
    with open(path, "r", encoding="utf-8") as f:
        data = json.load(f)
    if isinstance(data, dict):
        data = data["regions"]
    return [RegionStats(*(r[k] for k in _FIELDS)) for r in data]


def _pct(new, old):
    return 100.0 * (new - old) / old


def compare_reports(a, b) -> list:
    """Merge two reports by (parent, name) with relative-change columns
    (src/bench.py:235-268): rows in a's order, then b-only regions."""
    ia = {(r.parent, r.name): r for r in a}
    ib = {(r.parent, r.name): r for r in b}
    order = list(ia) + [k for k in ib if k not in ia]
    rows = []
    for parent, name in order:
        ra, rb = ia.get((parent, name)), ib.get((parent, name))
        total = per_call = None
        if ra is not None and rb is not None and ra.inclusive_seconds > 0:
            total = _pct(rb.inclusive_seconds, ra.inclusive_seconds)
            per_call = _pct(rb.inclusive_seconds / rb.calls, ra.inclusive_seconds / ra.calls)
        rows.append({
            "name": name,
            "parent": parent,
            "calls_a": None if ra is None else ra.calls,
            "seconds_a": None if ra is None else ra.inclusive_seconds,
            "calls_b": None if rb is None else rb.calls,
            "seconds_b": None if rb is None else rb.inclusive_seconds,
            "total_change_pct": total,
            "per_call_change_pct": per_call,
        })
    return rows


def render_comparison(rows) -> str:
    """src/bench.py:271-291."""

    def cell(v, spec):
        return "-" if v is None else format(v, spec)

    width = max([len("Region")] + [len(r["name"]) for r in rows])
    out = [f"{'Region':<{width}}  {'Calls A':>8} {'Secs A':>10}  {'Calls B':>8} {'Secs B':>10}"
           f"  {'Ttl %':>8} {'Per-call %':>10}"]
    for r in rows:
        out.append(f"{r['name']:<{width}}  {cell(r['calls_a'], 'd'):>8} {cell(r['seconds_a'], '.3f'):>10}"
                   f"  {cell(r['calls_b'], 'd'):>8} {cell(r['seconds_b'], '.3f'):>10}"
                   f"  {cell(r['total_change_pct'], '+.2f'):>8} {cell(r['per_call_change_pct'], '+.2f'):>10}")
    return "\n".join(out)


# ---------------------------------------------------------------- scaling


def _ranks_report(cfg, gpus: int) -> list:
    """Regions of one z-slab run on ``gpus`` ranks (torchrun, NCCL), rank 0's view."""
    import dataclasses
    import os
    import socket
    import subprocess
    import sys
    import tempfile

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "regions.json")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", "-m", "paper_2504_03697_b200.distributed",
               "--config", json.dumps(dataclasses.asdict(cfg)), "--out", out]
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        subprocess.run(cmd, check=True, env=env, cwd=root)
        return load_report(out)


def scaling_sweep(cfg, gpu_counts, emulate: bool = False) -> list:
    """Run the configured problem once per GPU count (src/bench.py:294-316,
    whose axis is host threads): 1 = the single-domain run, G > 1 = the
    z-slab run on G ranks (one GPU each, launched with torchrun), or with
    ``emulate=True`` G slabs on this one device.  Returns one
    ``(gpus, region, seconds)`` row per region and count; snapshot output is
    disabled during the sweep."""
    import torch

    from . import distributed, sim

    if not gpu_counts:
        raise ValueError("at least one GPU count is required")
    if any(int(g) < 1 for g in gpu_counts):
        raise ValueError(f"GPU counts must be >= 1, got {list(gpu_counts)}")
    if not emulate and max(int(g) for g in gpu_counts) > torch.cuda.device_count():
        raise ValueError(f"{max(gpu_counts)} GPUs requested, {torch.cuda.device_count()} visible "
                         "(emulate=True runs the slabs on one device)")
    # warm-up on a toy problem so the first row is not charged for library/graph setup
    sim.run(replace(cfg, n=8, h=1.0 / 8, shape=None, t_end=cfg.dt, output_dir=None))
    rows = []
    for g in (int(x) for x in gpu_counts):
        sweep_cfg = replace(cfg, output_dir=None)
        if g == 1:
            regions = sim.run(sweep_cfg)[1].regions
        elif emulate:
            regions = distributed.run(sweep_cfg, slabs=g)[1].regions
        else:
            regions = _ranks_report(sweep_cfg, g)
        rows.extend((g, r.name, r.inclusive_seconds) for r in regions)
    return rows


def write_scaling_csv(rows, path) -> None:
    """src/bench.py:319-324 (the count column keeps the reference's name)."""
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f)
        w.writerow(["threads", "region", "seconds"])
        for count, region, seconds in rows:
            w.writerow([count, region, repr(float(seconds))])
