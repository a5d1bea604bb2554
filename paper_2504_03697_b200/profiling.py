"""Region profiler (mirror of src/bench.py:36-152, :195-287).

Same region names, nesting rules, ``RegionStats`` records and report
helpers as the reference, so its reports and comparisons consume runs of
this package unchanged.  The kernels are asynchronous, so a region
synchronises the current CUDA stream when it closes: the recorded time is
the device work the region enqueued, not just the launch cost.
"""

from __future__ import annotations

import json
import time
from dataclasses import asdict, dataclass


class ProfileError(RuntimeError):
    pass


@dataclass
class RegionStats:
    name: str
    parent: str | None
    calls: int
    inclusive_seconds: float
    fraction: float


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
    """Call counts and inclusive time per nested region path."""

    def __init__(self, sync: bool = True):
        self._nodes = {}
        self._path = []
        self._starts = []
        self._sync = sync

    def enter(self, name: str):
        if self._sync:
            _sync()
        self._path.append(name)
        self._starts.append(time.perf_counter_ns())

    def exit(self, name: str):
        if not self._path or self._path[-1] != name:
            open_name = self._path[-1] if self._path else None
            raise ProfileError(f"unbalanced region exit: got {name!r} while {open_name!r} is open")
        if self._sync:
            _sync()
        elapsed = time.perf_counter_ns() - self._starts.pop()
        key = tuple(self._path)
        self._path.pop()
        node = self._nodes.setdefault(key, [0, 0])
        node[0] += 1
        node[1] += elapsed

    def region(self, name: str) -> _Region:
        return _Region(self, name)

    def reset(self):
        if self._path:
            raise ProfileError(f"cannot reset while region {self._path[-1]!r} is open")
        self._nodes.clear()

    def stats(self) -> list:
        if self._path:
            raise ProfileError(f"region {self._path[-1]!r} is still open")
        kids = {}
        for path in self._nodes:
            kids.setdefault(path[:-1], []).append(path)
        root_ns = sum(self._nodes[p][1] for p in kids.get((), []))
        out = []

        def visit(path):
            calls, ns = self._nodes[path]
            frac = ns / root_ns if root_ns > 0 else (1.0 if len(path) == 1 else 0.0)
            out.append(RegionStats(path[-1], path[-2] if len(path) > 1 else None, calls, ns * 1e-9, frac))
            for c in kids.get(path, []):
                visit(c)

        for top in kids.get((), []):
            visit(top)
        return out


class NullProfiler:
    def enter(self, name):
        pass

    def exit(self, name):
        pass

    def region(self, name):
        return _NullRegion()

    def stats(self):
        return []


class _NullRegion:
    __slots__ = ()

    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


NULL_PROFILER = NullProfiler()


def render_report(regions) -> str:
    """Indented hotspot tree (src/bench.py:195-207)."""
    depth = {}
    lines = [f"{'region':40s} {'calls':>8s} {'seconds':>12s} {'share':>8s}"]
    for r in regions:
        d = 0 if r.parent is None else depth.get(r.parent, 0) + 1
        depth[r.name] = d
        lines.append(f"{'  ' * d + r.name:40s} {r.calls:8d} {r.inclusive_seconds:12.6f} {100 * r.fraction:7.2f}%")
    return "\n".join(lines)


def save_report(regions, path) -> None:
    with open(path, "w") as f:
        json.dump({"regions": [asdict(r) for r in regions]}, f, indent=2)


def load_report(path) -> list:
    with open(path) as f:
        return [RegionStats(**r) for r in json.load(f)["regions"]]
