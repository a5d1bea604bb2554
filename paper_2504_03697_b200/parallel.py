"""Parallel backends (mirror of src/parallel.py) and the z-slab decomposition.

``WorkerPool`` keeps the reference's chunked host dispatch
(src/parallel.py:15-56) for code that calls ``run_chunks`` directly; the
device kernels ignore the ``pool`` argument -- the GPU grid *is* the pool.

``SlabDecomposition`` is the multi-GPU layout (SURVEY.md §5.7, §8 e): rank
r of G owns the contiguous z-planes [z0, z1) of the cube (x fastest, so a
slab is one contiguous block of every scalar field), with one halo plane
below/above when a neighbour exists.  It is pure host logic so it is
tested on CPU (gloo) and shared by the NCCL path.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


class WorkerPool:
    """Fixed-size thread pool dispatching contiguous index chunks."""

    def __init__(self, threads: int = 1):
        if threads < 1:
            raise ValueError(f"thread count must be >= 1, got {threads}")
        self.threads = threads
        self._executor = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def chunk_bounds(self, n_items: int) -> np.ndarray:
        chunks = max(1, min(self.threads, n_items)) if n_items > 0 else 1
        return np.linspace(0, n_items, chunks + 1).astype(np.int64)

    def run_chunks(self, fn, n_items: int, *args) -> list:
        b = self.chunk_bounds(n_items)
        spans = [(int(b[i]), int(b[i + 1])) for i in range(len(b) - 1)]
        if self._executor is None or len(spans) <= 1:
            return [fn(*args, lo, hi) for lo, hi in spans]
        futs = [self._executor.submit(fn, *args, lo, hi) for lo, hi in spans]
        return [f.result() for f in futs]

    def close(self):
        if self._executor is not None:
            self._executor.shutdown(wait=True)
            self._executor = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


@dataclass(frozen=True)
class SlabDecomposition:
    """z-slab ownership of an nx*ny*nz grid over `world` ranks."""

    nx: int
    ny: int
    nz: int
    world: int
    rank: int

    def __post_init__(self):
        if not (0 <= self.rank < self.world):
            raise ValueError(f"rank {self.rank} outside world {self.world}")
        if self.nz < self.world:
            raise ValueError(f"{self.nz} planes cannot be split over {self.world} ranks")

    @staticmethod
    def bounds(nz: int, world: int) -> np.ndarray:
        # balanced contiguous split, the WorkerPool rule applied to planes
        return np.linspace(0, nz, world + 1).astype(np.int64)

    @property
    def z0(self) -> int:
        return int(self.bounds(self.nz, self.world)[self.rank])

    @property
    def z1(self) -> int:
        return int(self.bounds(self.nz, self.world)[self.rank + 1])

    @property
    def planes(self) -> int:
        return self.z1 - self.z0

    @property
    def lo_neighbor(self):
        return self.rank - 1 if self.rank > 0 else None

    @property
    def hi_neighbor(self):
        return self.rank + 1 if self.rank < self.world - 1 else None

    @property
    def plane_cells(self) -> int:
        return self.nx * self.ny

    def local_slice(self) -> slice:
        """Flat index range of the owned planes in the global (x-fastest) vector."""
        return slice(self.z0 * self.plane_cells, self.z1 * self.plane_cells)

    def halo_layout(self):
        """(lo_halo, hi_halo, owned offset) of the local buffer
        [lo halo plane][owned planes][hi halo plane]."""
        lo = self.lo_neighbor is not None
        hi = self.hi_neighbor is not None
        return lo, hi, (self.plane_cells if lo else 0)
