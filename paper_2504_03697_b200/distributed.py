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



def _slab_precond(precond) -> int:
    """The z-slab CG runs Jacobi or no preconditioner; DIC does not shard
    (SURVEY.md §8(e)), so it is rejected instead of silently dropped."""
    if precond == "jacobi":
        return _lib.PRECOND_JACOBI
    if precond is None or precond == "none":
        return _lib.PRECOND_NONE
    raise ValueError(f"the z-slab CG supports precond 'jacobi' or None, got {precond!r}")


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
        pk = _slab_precond(precond)
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


class PeerLinkError(RuntimeError):
    """The ranks could not link their CG vectors through CUDA IPC (raised on
    every rank alike, so a caller can fall back to the NCCL form together)."""


class PeerSlabCG:
    """CG over z-slabs with the collectives fused into the kernels over peer
    memory (cf_pcg_*, csrc/cf_p2p.cu): one slab per rank (GPU) linked through
    CUDA IPC handles exchanged over torch.distributed, or -- ``bounds`` with
    several slabs, no process group -- every slab on this device, the
    single-device verification of the same kernels and protocol.
    Same ``solve`` interface as ``SlabCG`` (the NCCL form)."""

    def __init__(self, nx: int, ny: int, nz: int, h: float, order: str = "sym", bounds=None,
                 distributed: bool = False):
        lib = _lib.load_library()
        bounds = [0, nz] if bounds is None else [int(b) for b in bounds]
        self.nx, self.ny, self.nz, self.h = nx, ny, nz, float(h)
        self.bounds = bounds
        self.plane = nx * ny
        self.order = _lib.ORDER_CSR if order == "csr" else _lib.ORDER_SYM
        nslab = len(bounds) - 1
        if distributed:
            import torch.distributed as dist

            nranks, rank = dist.get_world_size(), dist.get_rank()
            if nslab != 1:
                raise ValueError("one slab per rank in a distributed run")
        else:
            nranks, rank = nslab, 0
        arr = (ctypes.c_int * len(bounds))(*bounds)
        hdl = ctypes.c_void_p()
        _lib.check(lib.cf_pcg_create(ctypes.byref(hdl), nx, ny, nz, self.h, self.order, nranks, rank, nslab, arr,
                                     _lib.stream()), "cf_pcg_create")
        self._h = hdl
        self.last_loop_ms = 0.0
        form = ctypes.c_int()
        _lib.check(lib.cf_pcg_form(hdl, ctypes.byref(form)), "cf_pcg_form")
        # the single pass over slabs (one collective per iteration) or the two-kernel form
        self.single_pass = form.value == _lib.CG_FORM_SPASS
        if distributed and nranks > 1:  # publish this rank's IPC handles, open the peers'
            import torch.distributed as dist

            size = lib.cf_pcg_export_size()
            blob = ctypes.create_string_buffer(size)
            _lib.check(lib.cf_pcg_export(self._h, blob, size), "cf_pcg_export")
            blobs = [None] * nranks
            dist.all_gather_object(blobs, blob.raw)
            allb = ctypes.create_string_buffer(b"".join(blobs), size * nranks)
            rc = lib.cf_pcg_import(self._h, allb, nranks)
            why = _lib.last_error() if rc != 0 else ""
            # every rank must agree: a rank that linked would otherwise wait on
            # mailboxes a failed rank never writes
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
            ok = torch.tensor([1 if rc == 0 else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                raise PeerLinkError(f"peer-memory CG linking failed on at least one rank ({why or 'another rank'})")
            dist.barrier()

    def solve(self, b_slabs, tol: float = 1e-6, max_iter: int = 1000, precond: str | None = "jacobi"):
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
        pk = _slab_precond(precond)
        its = ctypes.c_int64()
        res = ctypes.c_double()
        rc = lib.cf_pcg_solve(self._h, bp, xp, float(tol), int(max_iter), pk, ctypes.byref(its), ctypes.byref(res),
                              _lib.stream())
        ms = ctypes.c_float()
        lib.cf_pcg_last_loop_ms(self._h, ctypes.byref(ms))
        self.last_loop_ms = float(ms.value)
        if rc == _lib.CF_BREAKDOWN:
            raise BreakdownError(_lib.last_error())
        _lib.check(rc, "cf_pcg_solve")
        return xs, SolveStats(int(its.value), float(res.value), rc == _lib.CF_OK)

    def __del__(self):
        try:
            if self._h and _lib._lib is not None:
                _lib._lib.cf_pcg_destroy(self._h)
        except Exception:
            pass


def emulated_pcg(op: StencilOperator, b, nslabs: int, tol: float = 1e-6, max_iter: int = 1000,
                 precond: str | None = "jacobi", collective: str = "nccl"):
    """Single-device run of the z-slab decomposition (slabs = contiguous views
    of the global x-fastest vector).  ``collective``: "nccl" (SlabCG, the
    kernels + collective calls form) or "p2p" (PeerSlabCG, collectives fused
    into the kernels).  Returns (x, SolveStats, solver)."""
    bd, host = as_device(b)
    bd = bd.contiguous()
    bounds = SlabDecomposition.bounds(op.nz, nslabs).tolist()
    cls = PeerSlabCG if collective == "p2p" else SlabCG
    scg = cls(op.nx, op.ny, op.nz, op.h, "csr" if op.order == _lib.ORDER_CSR else "sym", bounds=bounds)
    pl = op.nx * op.ny
    xs, st = scg.solve([bd[bounds[k] * pl:bounds[k + 1] * pl] for k in range(nslabs)], tol, max_iter, precond)
    x = torch.cat(xs)
    return (to_host(x) if host else x), st, scg


HALO = 2  # velocity halo planes: the backtrace moves <= 1 cell (CFL <= 1) + the trilinear stencil


class _SlabFields:
    """One slab's device fields: velocity (two buffers) with HALO planes,
    pressure with one halo plane each side, the Poisson RHS."""

    def __init__(self, nx: int, ny: int, z0: int, z1: int, dev):
        from .grid import padded_ld

        self.nx, self.ny, self.z0, self.z1 = nx, ny, z0, z1
        self.nzl = z1 - z0
        self.pl = nx * ny
        self.ld = [padded_ld(nx + 1), padded_ld(nx), padded_ld(nx)]
        self.nb = [ny, ny + 1, ny]
        planes = [self.nzl + 2 * HALO, self.nzl + 2 * HALO, self.nzl + 1 + 2 * HALO]
        self.vel = [[torch.zeros((planes[c], self.nb[c], self.ld[c]), dtype=torch.float64, device=dev)
                     for c in range(3)] for _ in range(2)]
        self.cur = 0
        self.p = torch.zeros((self.nzl + 2) * self.pl, dtype=torch.float64, device=dev)
        self.rhs = torch.zeros(self.nzl * self.pl, dtype=torch.float64, device=dev)

    def planes(self, c: int, buf: int, k0: int, k1: int) -> torch.Tensor:
        """Stored planes for global planes [k0, k1) of component c."""
        kb = self.z0 - HALO
        return self.vel[buf][c][k0 - kb:k1 - kb]

    def p_owned(self) -> torch.Tensor:
        return self.p[self.pl:self.pl * (self.nzl + 1)]

    def ptrs(self, buf: int):
        return tuple(t.data_ptr() for t in self.vel[buf])


class SlabSim:
    """The cavity time step (src/sim.py:452-474) over z-slabs.

    ``bounds`` are the global plane bounds of this process's consecutive slabs
    (several slabs = single-device emulation; one slab per rank under
    torch.distributed with ``distributed=True``).  Reference physics,
    Jacobi/none PCG (DIC does not shard), cold-start pressure solves.
    Halo exchanges: velocity (HALO planes) before advection and after it (for
    the divergence's top w face), pressure (1 plane) before the correction;
    the CG exchanges its own r halos inside cf_dcg.
    """

    def __init__(self, cfg, bounds, distributed: bool = False, collective: str = "p2p"):
        import torch.distributed as dist

        if collective not in ("p2p", "nccl"):
            raise ValueError(f"collective must be 'p2p' or 'nccl', got {collective!r}")
        if cfg.preconditioner != "jacobi":
            raise ValueError("the z-slab solver shards Jacobi-PCG only (DIC's sweeps do not shard)")
        if cfg.warm_start:
            raise ValueError("warm_start is not supported by the z-slab solver")
        if cfg.viscosity > 0.0 and cfg.diffusion != "explicit":
            raise ValueError("the z-slab step runs explicit diffusion only")
        lib = _lib.load_library()
        self.cfg = cfg
        self.nx, self.ny, self.nz = cfg.spec.dims  # the cube, or a box (extension)
        self.bounds = [int(b) for b in bounds]
        self.dist = distributed
        dev = torch.device("cuda", torch.cuda.current_device())
        self.slabs = [_SlabFields(self.nx, self.ny, self.bounds[k], self.bounds[k + 1], dev)
                      for k in range(len(bounds) - 1)]
        for s in self.slabs:
            if s.nzl < HALO + 1:
                raise ValueError(f"slab [{s.z0}, {s.z1}) is thinner than {HALO + 1} planes")
        order = "sym" if cfg.variant == "optimized" else "csr"
        self.collective = collective
        if collective == "p2p":
            self.rank, self.world = (dist.get_rank(), dist.get_world_size()) if distributed else (0, 1)
            self.cg = PeerSlabCG(self.nx, self.ny, self.nz, cfg.h, order, bounds=self.bounds,
                                 distributed=distributed)
        elif distributed:
            self.rank, self.world = dist.get_rank(), dist.get_world_size()
            obj = [nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            lo = self.rank - 1 if self.rank > 0 else -1
            hi = self.rank + 1 if self.rank < self.world - 1 else -1
            self.cg = SlabCG(self.nx, self.ny, self.nz, cfg.h, order, bounds=self.bounds, nranks=self.world,
                             rank=self.rank, uid=obj[0], lo_rank=lo, hi_rank=hi)
        else:
            self.rank, self.world = 0, 1
            self.cg = SlabCG(self.nx, self.ny, self.nz, cfg.h, order, bounds=self.bounds)
        self.step_count = 0
        self._lib = lib

    # ------------------------------------------------------------ state I/O
    def load_global(self, u, v, w, p=None):
        """Scatter reference-layout global arrays (C order [i, j, k]) into the slabs."""
        comps = [np.asarray(u), np.asarray(v), np.asarray(w)]
        for s in self.slabs:
            for c, arr in enumerate(comps):
                k1 = s.z1 + (1 if (c == 2 and s.z1 == self.nz) else 0)
                blk = torch.as_tensor(np.ascontiguousarray(arr[:, :, s.z0:k1].transpose(2, 1, 0)))
                s.planes(c, s.cur, s.z0, k1)[:, :, :arr.shape[0]].copy_(blk)
            if p is not None:
                s.p_owned().copy_(torch.as_tensor(np.asarray(p)[s.z0 * s.pl:s.z1 * s.pl]))

    def gather(self):
        """Global reference-layout (u, v, w, p) of the local slabs (emulation: the whole box)."""
        nx, ny, nz = self.nx, self.ny, self.nz
        out = [np.zeros((nx + 1, ny, nz)), np.zeros((nx, ny + 1, nz)), np.zeros((nx, ny, nz + 1))]
        p = np.zeros(nx * ny * nz)
        for s in self.slabs:
            for c in range(3):
                k1 = s.z1 + (1 if (c == 2 and s.z1 == nz) else 0)
                blk = s.planes(c, s.cur, s.z0, k1)[:, :, :out[c].shape[0]].cpu().numpy()
                out[c][:, :, s.z0:k1] = blk.transpose(2, 1, 0)
            p[s.z0 * s.pl:s.z1 * s.pl] = s.p_owned().cpu().numpy()
        return out[0], out[1], out[2], p

    # ------------------------------------------------------------ halos
    def _exchange_vel(self, buf_attr="cur"):
        """Velocity halo planes from the neighbouring slabs' owned planes."""
        for a, b in zip(self.slabs, self.slabs[1:]):
            ba, bb = getattr(a, buf_attr), getattr(b, buf_attr)
            for c in range(3):
                # a's hi halo <- b's owned [z, z + HALO (+1 for w)]
                top = HALO + (1 if c == 2 else 0)
                a.planes(c, ba, b.z0, b.z0 + top).copy_(b.planes(c, bb, b.z0, b.z0 + top))
                # b's lo halo <- a's owned [z - HALO, z)
                b.planes(c, bb, b.z0 - HALO, b.z0).copy_(a.planes(c, ba, b.z0 - HALO, b.z0))
        if self.dist and self.world > 1:
            self._exchange_vel_ranks(buf_attr)

    def _exchange_vel_ranks(self, buf_attr):
        import torch.distributed as dist

        s = self.slabs[0]
        buf = getattr(s, buf_attr)
        ops = []
        for c in range(3):
            top = HALO + (1 if c == 2 else 0)
            if self.rank > 0:
                ops.append(dist.P2POp(dist.isend, s.planes(c, buf, s.z0, s.z0 + top).contiguous(), self.rank - 1))
                ops.append(dist.P2POp(dist.irecv, s.planes(c, buf, s.z0 - HALO, s.z0), self.rank - 1))
            if self.rank < self.world - 1:
                ops.append(dist.P2POp(dist.isend, s.planes(c, buf, s.z1 - HALO, s.z1).contiguous(), self.rank + 1))
                ops.append(dist.P2POp(dist.irecv, s.planes(c, buf, s.z1, s.z1 + top), self.rank + 1))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def _exchange_p(self):
        pl = self.nx * self.ny
        for a, b in zip(self.slabs, self.slabs[1:]):
            a.p[pl * (a.nzl + 1):pl * (a.nzl + 2)].copy_(b.p[pl:2 * pl])
            b.p[0:pl].copy_(a.p[pl * a.nzl:pl * (a.nzl + 1)])
        if self.dist and self.world > 1:
            import torch.distributed as dist

            s = self.slabs[0]
            ops = []
            if self.rank > 0:
                ops.append(dist.P2POp(dist.isend, s.p[pl:2 * pl], self.rank - 1))
                ops.append(dist.P2POp(dist.irecv, s.p[0:pl], self.rank - 1))
            if self.rank < self.world - 1:
                ops.append(dist.P2POp(dist.isend, s.p[pl * s.nzl:pl * (s.nzl + 1)], self.rank + 1))
                ops.append(dist.P2POp(dist.irecv, s.p[pl * (s.nzl + 1):pl * (s.nzl + 2)], self.rank + 1))
            for r in dist.batch_isend_irecv(ops):
                r.wait()

    def _max(self, vals):
        m = max(vals)
        if self.dist and self.world > 1:
            import torch.distributed as dist

            t = torch.tensor([m], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            m = float(t.item())
        return m

    # ------------------------------------------------------------ the step
    def _forces(self, lib, st, dims):
        cfg = self.cfg
        for s in self.slabs:  # forces + walls (src/sim.py:134-149)
            u, v, w = s.ptrs(s.cur)
            _lib.check(lib.cf_forces_bc_slab(u, v, w, *dims, s.z0, s.z1, HALO, *s.ld, cfg.lid_accel * cfg.dt, 1, st),
                       "forces_bc_slab")

    def _advect(self, lib, st, dims):
        cfg = self.cfg
        self._exchange_vel()
        # the HALO-plane halo covers a backtrace of <= 1 cell in z
        wmax = []
        for s in self.slabs:
            r = ctypes.c_double()
            w = s.vel[s.cur][2]
            _lib.check(lib.cf_max_abs(w.data_ptr(), w.numel(), ctypes.byref(r), st), "max|w|")
            wmax.append(r.value)
        if self._max(wmax) * cfg.dt / cfg.h > HALO - 1:
            raise ValueError("CFL in z exceeds the slab halo (max|w| dt/h > 1)")
        for s in self.slabs:  # advection into the spare buffer (src/sim.py:259-289)
            u, v, w = s.ptrs(s.cur)
            nu, nv, nw = s.ptrs(1 - s.cur)
            _lib.check(lib.cf_advect_slab(u, v, w, nu, nv, nw, *dims, s.z0, s.z1, HALO, *s.ld, cfg.h, cfg.dt, st),
                       "advect_slab")
            s.cur = 1 - s.cur
        self._exchange_vel()  # the divergence (and diffusion) read neighbour planes

    def _diffuse(self, lib, st, dims):
        cfg = self.cfg
        kdt = cfg.viscosity * cfg.dt / (cfg.h * cfg.h)
        lid = cfg.lid_velocity
        for s in self.slabs:
            u, v, w = s.ptrs(s.cur)
            nu, nv, nw = s.ptrs(1 - s.cur)
            _lib.check(lib.cf_diffuse_slab(u, v, w, nu, nv, nw, *dims, s.z0, s.z1, HALO, *s.ld, kdt,
                                           0.0 if lid is None else float(lid), 0 if lid is None else 1,
                                           1 if cfg.no_slip else 0, st), "diffuse_slab")
            s.cur = 1 - s.cur
        self._exchange_vel()

    def _pressure(self, lib, st, dims, prof):
        cfg = self.cfg
        maxb = []
        for s in self.slabs:  # b = -(rho/dt) div (src/sim.py:359-360)
            u, v, w = s.ptrs(s.cur)
            mx = ctypes.c_double()
            _lib.check(lib.cf_divergence_slab(u, v, w, *dims, s.z0, s.z1, HALO, *s.ld, cfg.h, -cfg.density / cfg.dt,
                                              s.rhs.data_ptr(), ctypes.byref(mx), st), "divergence_slab")
            maxb.append(mx.value)
        div_pre = self._max(maxb) * cfg.dt / cfg.density
        with prof.region("pcg"):
            xs, stats = self.cg.solve([s.rhs for s in self.slabs], cfg.tol, cfg.max_iter, "jacobi")
        for s, x in zip(self.slabs, xs):
            s.p_owned().copy_(x)
        self._exchange_p()
        return stats, div_pre

    def _correct(self, lib, st, dims):
        cfg = self.cfg
        coef = cfg.dt / (cfg.density * cfg.h)
        posts = []
        for s in self.slabs:  # correction + div_post + walls (src/sim.py:426-449)
            u, v, w = s.ptrs(s.cur)
            nu, nv, nw = s.ptrs(1 - s.cur)
            out = ctypes.c_double()
            _lib.check(lib.cf_pressure_correct_slab(u, v, w, nu, nv, nw, s.p.data_ptr() + 8 * s.pl, *dims, s.z0, s.z1,
                                                    HALO, *s.ld, cfg.h, coef, ctypes.byref(out), st),
                       "pressure_correct_slab")
            posts.append(out.value)
            s.cur = 1 - s.cur
        return self._max(posts)

    def step(self, profiler=None):
        """Advance one time step; returns StepStats (src/sim.py:452-474).
        ``profiler`` times the reference's step regions (src/sim.py:461-471)."""
        from .profiling import NULL_PROFILER
        from .sim import StepStats

        prof = NULL_PROFILER if profiler is None else profiler
        lib, st = self._lib, _lib.stream()
        dims = (self.nx, self.ny, self.nz)
        with prof.region("applyForces"):
            self._forces(lib, st, dims)
        with prof.region("solveAdvection"):
            self._advect(lib, st, dims)
        if self.cfg.viscosity > 0.0:  # extension: explicit diffusion
            with prof.region("solveDiffusion"):
                self._diffuse(lib, st, dims)
        with prof.region("solvePressureCorrection"):
            stats, div_pre = self._pressure(lib, st, dims, prof)
        with prof.region("applyPressureCorrection"):
            div_post = self._correct(lib, st, dims)
        self.step_count += 1
        return StepStats(solve=stats, div_pre=div_pre, div_post=div_post)


def init_slab_cg(n: int, h: float, order: str = "sym", nz: int | None = None, collective: str = "p2p") -> tuple:
    """Per-rank z-slab solver over torch.distributed (one GPU per rank):
    ``collective`` "p2p" (collectives fused into the kernels, PeerSlabCG) or
    "nccl" (SlabCG).  Returns (solver, SlabDecomposition)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    nz = n if nz is None else nz
    dec = SlabDecomposition(n, n, nz, world, rank)
    if collective == "p2p":
        return PeerSlabCG(n, n, nz, h, order, bounds=[dec.z0, dec.z1], distributed=True), dec
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    lo = dec.lo_neighbor if dec.lo_neighbor is not None else -1
    hi = dec.hi_neighbor if dec.hi_neighbor is not None else -1
    scg = SlabCG(n, n, nz, h, order, bounds=[dec.z0, dec.z1], nranks=world, rank=rank, uid=obj[0], lo_rank=lo,
                 hi_rank=hi)
    return scg, dec


def run(cfg, slabs: int | None = None, distributed: bool = False, collective: str = "p2p"):
    """``sim.run`` (src/sim.py:477-505) over z-slabs: ``distributed=True``
    gives this rank its slab of a torch.distributed job (one GPU per rank);
    otherwise ``slabs`` consecutive slabs are emulated on this device.
    Returns (SlabSim, RunReport) with the reference's region names; no
    snapshot output (gather() the state and write it on one rank)."""
    import time

    from .profiling import Profiler
    from .sim import ROOT_REGION, RunReport

    if cfg.output_dir is not None:
        raise ValueError("z-slab runs write no snapshots: set output_dir=None and gather() the state")
    nx, ny, nz = cfg.spec.dims
    if distributed:
        import torch.distributed as dist

        dec = SlabDecomposition(nx, ny, nz, dist.get_world_size(), dist.get_rank())
        bounds = [dec.z0, dec.z1]
    else:
        bounds = SlabDecomposition.bounds(nz, 1 if slabs is None else int(slabs)).tolist()
    sim = SlabSim(cfg, bounds, distributed=distributed, collective=collective)
    prof = Profiler()
    report = RunReport()
    t0 = time.perf_counter()
    with prof.region(ROOT_REGION):
        for _ in range(cfg.num_steps):
            report.steps.append(sim.step(prof))
    report.regions = prof.stats()
    report.wall_seconds = time.perf_counter() - t0
    return sim, report


def _sweep_worker(argv=None) -> int:
    """One rank of profiling.scaling_sweep's multi-GPU leg (launched by torchrun)."""
    import argparse
    import dataclasses
    import json
    import os

    import torch.distributed as dist

    from .profiling import save_report
    from .sim import SimConfig

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    kw = json.loads(a.config)
    if kw.get("shape") is not None:
        kw["shape"] = tuple(kw["shape"])
    names = {f.name for f in dataclasses.fields(SimConfig)}
    cfg = SimConfig(**{k: v for k, v in kw.items() if k in names})
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        _, report = run(cfg, distributed=True)
        if dist.get_rank() == 0:
            save_report(report.regions, a.out)
        dist.barrier()
    finally:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(_sweep_worker())
