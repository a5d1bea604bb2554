"""Multi-GPU z-slab pressure solve (SURVEY.md §5.8, §8 e).

One process per GPU (``torch.distributed`` for the plumbing: rank, world and
the NCCL unique-id broadcast); the solve itself runs in libcfgpu
(``cf_dcg_*``): per CG iteration the two fused kernels on the local slab,
two ``ncclAllReduce`` of the CG partial sums and one ``ncclSend/Recv`` of the
r halo planes, all stream-ordered without host round trips (the host polls
the ``done`` flag once per batch of iterations).

The same solver runs several slabs in ONE process on one device
(``SlabCG(..., bounds=[z0, z1, z2, ...])`` without a communicator): the
decomposition's halo logic then executes on the real kernels and is
parity-tested on a single B200 (tests/test_gpu_dist.py) -- no ranks wait on
each other inside kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .grid import as_device, to_host
from .parallel import SlabDecomposition
from .solver import BreakdownError, SolveStats
from .sparse import StencilOperator


def nccl_unique_id() -> bytes:
    lib = _lib.load_library()
    buf = ctypes.create_string_buffer(128)
    _lib.check(lib.cf_nccl_unique_id(buf), "cf_nccl_unique_id")
    return buf.raw


class SlabCG:
    """CG over the z-slabs [bounds[k], bounds[k+1]) owned by this process."""

    def __init__(self, nx: int, ny: int, nz: int, h: float, order: str = "sym", bounds=None, nranks: int = 1,
                 rank: int = 0, uid: bytes | None = None, lo_rank: int = -1, hi_rank: int = -1):
        lib = _lib.load_library()
        bounds = [0, nz] if bounds is None else [int(b) for b in bounds]
        self.nx, self.ny, self.nz, self.h = nx, ny, nz, float(h)
        self.bounds = bounds
        self.plane = nx * ny
        self.order = _lib.ORDER_CSR if order == "csr" else _lib.ORDER_SYM
        self.inv_diag_value = 1.0 / (6.0 / (self.h * self.h))
        arr = (ctypes.c_int * len(bounds))(*bounds)
        uid_buf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
        hdl = ctypes.c_void_p()
        _lib.check(lib.cf_dcg_create(ctypes.byref(hdl), nx, ny, nz, self.h, self.order, nranks, rank, uid_buf,
                                     len(bounds) - 1, arr, lo_rank, hi_rank, _lib.stream()), "cf_dcg_create")
        self._h = hdl
        self.last_loop_ms = 0.0

    def solve(self, b_slabs, tol: float = 1e-6, max_iter: int = 1000, precond: str | None = "jacobi"):
        """b_slabs: one CUDA tensor per local slab (its owned planes, flat).
        Returns (x_slabs, SolveStats)."""
        lib = _lib.load_library()
        ns = len(self.bounds) - 1
        if len(b_slabs) != ns:
            raise ValueError(f"expected {ns} slabs, got {len(b_slabs)}")
        bs = [as_device(b)[0].contiguous() for b in b_slabs]
        for k, b in enumerate(bs):
            want = self.plane * (self.bounds[k + 1] - self.bounds[k])
            if b.numel() != want:
                raise ValueError(f"slab {k} needs {want} values, got {b.numel()}")
        xs = [torch.empty_like(b) for b in bs]
        bp = (ctypes.c_void_p * ns)(*(b.data_ptr() for b in bs))
        xp = (ctypes.c_void_p * ns)(*(x.data_ptr() for x in xs))
        pk = _lib.PRECOND_JACOBI if precond == "jacobi" else _lib.PRECOND_NONE
        its = ctypes.c_int64()
        res = ctypes.c_double()
        rc = lib.cf_dcg_solve(self._h, bp, xp, float(tol), int(max_iter), pk, ctypes.byref(its), ctypes.byref(res),
                              _lib.stream())
        ms = ctypes.c_float()
        lib.cf_dcg_last_loop_ms(self._h, ctypes.byref(ms))
        self.last_loop_ms = float(ms.value)
        if rc == _lib.CF_BREAKDOWN:
            raise BreakdownError(_lib.last_error())
        _lib.check(rc, "cf_dcg_solve")
        return xs, SolveStats(int(its.value), float(res.value), rc == _lib.CF_OK)

    def __del__(self):
        try:
            if self._h and _lib._lib is not None:
                _lib._lib.cf_dcg_destroy(self._h)
        except Exception:
            pass


def emulated_pcg(op: StencilOperator, b, nslabs: int, tol: float = 1e-6, max_iter: int = 1000,
                 precond: str | None = "jacobi"):
    """Single-device run of the z-slab decomposition (slabs = contiguous views
    of the global x-fastest vector).  Returns (x, SolveStats, SlabCG)."""
    bd, host = as_device(b)
    bd = bd.contiguous()
    n = op.n
    bounds = SlabDecomposition.bounds(n, nslabs).tolist()
    scg = SlabCG(n, n, n, op.h, "csr" if op.order == _lib.ORDER_CSR else "sym", bounds=bounds)
    pl = n * n
    xs, st = scg.solve([bd[bounds[k] * pl:bounds[k + 1] * pl] for k in range(nslabs)], tol, max_iter, precond)
    x = torch.cat(xs)
    return (to_host(x) if host else x), st, scg


def init_slab_cg(n: int, h: float, order: str = "sym", nz: int | None = None) -> tuple:
    """Per-rank z-slab solver over torch.distributed (one GPU per rank).
    Returns (SlabCG, SlabDecomposition)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    nz = n if nz is None else nz
    dec = SlabDecomposition(n, n, nz, world, rank)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    lo = dec.lo_neighbor if dec.lo_neighbor is not None else -1
    hi = dec.hi_neighbor if dec.hi_neighbor is not None else -1
    scg = SlabCG(n, n, nz, h, order, bounds=[dec.z0, dec.z1], nranks=world, rank=rank, uid=obj[0], lo_rank=lo,
                 hi_rank=hi)
    return scg, dec
