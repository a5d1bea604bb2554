"""CPU (gloo, world_size 2 and 3) checks of the multi-GPU host logic.

The device path (libcfgpu cf_dcg_*) exchanges only the r halo planes per
iteration and recomputes p on the halo planes from them; partial sums are
all-reduced.  Here the same data flow is replayed with numpy on gloo ranks,
using the product's SlabDecomposition for ownership, and checked against the
single-domain oracle PCG: the decomposition is exact up to reduction order.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03697_b200.parallel import SlabDecomposition


def test_slab_bounds_cover_the_grid():
    for nz, world in ((16, 2), (17, 3), (512, 8), (9, 9)):
        b = SlabDecomposition.bounds(nz, world)
        assert b[0] == 0 and b[-1] == nz and np.all(np.diff(b) >= 1)
        decs = [SlabDecomposition(8, 8, nz, world, r) for r in range(world)]
        assert sum(d.planes for d in decs) == nz
        assert decs[0].lo_neighbor is None and decs[-1].hi_neighbor is None
        for a, c in zip(decs, decs[1:]):
            assert a.z1 == c.z0 and a.hi_neighbor == c.rank and c.lo_neighbor == a.rank
        lo, hi, off = decs[0].halo_layout()
        assert lo is False and off == 0 and hi is (world > 1)
    with pytest.raises(ValueError):
        SlabDecomposition(4, 4, 2, 3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _stencil(xh, lo, hi, zlo_exists, zhi_exists, off, diag):
    """7-point operator on the owned planes of xh[(lo)+nzl+(hi), ny, nx] (SYM order)."""
    nzl = xh.shape[0] - lo - hi
    own = xh[lo:lo + nzl]
    out = diag * own
    ny, nx = own.shape[1:]
    xp = np.zeros_like(own); xp[:, :, :-1] = own[:, :, 1:]
    yp = np.zeros_like(own); yp[:, :-1, :] = own[:, 1:, :]
    zp = np.zeros_like(own); zp[:-1] = own[1:]
    if hi:
        zp[-1] = xh[lo + nzl]
    xm = np.zeros_like(own); xm[:, :, 1:] = own[:, :, :-1]
    ym = np.zeros_like(own); ym[:, 1:, :] = own[:, :-1, :]
    zm = np.zeros_like(own); zm[1:] = own[:-1]
    if lo:
        zm[0] = xh[0]
    # existence masks (a missing neighbour's term is dropped, as in the kernels)
    out = out + off * xp * (np.arange(nx) < nx - 1)[None, None, :]
    out = out + off * yp * (np.arange(ny) < ny - 1)[None, :, None]
    zmask_hi = np.ones(nzl, dtype=bool)
    if not zhi_exists:
        zmask_hi[-1] = False
    out = out + off * zp * zmask_hi[:, None, None]
    zmask_lo = np.ones(nzl, dtype=bool)
    if not zlo_exists:
        zmask_lo[0] = False
    out = out + off * zm * zmask_lo[:, None, None]
    out = out + off * ym * (np.arange(ny) > 0)[None, :, None]
    out = out + off * xm * (np.arange(nx) > 0)[None, None, :]
    return out


def _exchange(rh, dec, lo, hi):
    """Owned boundary planes of r into the neighbours' halo planes (send/recv)."""
    reqs = []
    nzl = dec.planes
    bufs = {}
    if dec.lo_neighbor is not None:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(rh[lo])), dec.lo_neighbor))
        bufs["lo"] = torch.empty(rh.shape[1:], dtype=torch.float64)
        reqs.append(dist.irecv(bufs["lo"], dec.lo_neighbor))
    if dec.hi_neighbor is not None:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(rh[lo + nzl - 1])), dec.hi_neighbor))
        bufs["hi"] = torch.empty(rh.shape[1:], dtype=torch.float64)
        reqs.append(dist.irecv(bufs["hi"], dec.hi_neighbor))
    for r in reqs:
        r.wait()
    if "lo" in bufs:
        rh[0] = bufs["lo"].numpy()
    if "hi" in bufs:
        rh[lo + nzl] = bufs["hi"].numpy()


def _allreduce(vals):
    t = torch.tensor(vals, dtype=torch.float64)
    dist.all_reduce(t)
    return t.tolist()


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = 1.0 / n
        off, diag = -1.0 / (h * h), 6.0 / (h * h)
        c = 1.0 / diag
        dec = SlabDecomposition(n, n, n, world, rank)
        lo_halo, hi_halo, _ = dec.halo_layout()
        lo, hi = int(lo_halo), int(hi_halo)
        b = np.random.default_rng(0).uniform(-1, 1, n ** 3).reshape(n, n, n)  # [k][j][i]
        bl = b[dec.z0:dec.z1]
        nzl = dec.planes
        shape = (lo + nzl + hi, n, n)
        rh = np.zeros(shape)
        rh[lo:lo + nzl] = bl
        x = np.zeros_like(bl)
        bb, rz = _allreduce([float((bl * bl).sum()), float((bl * (bl * c)).sum())])
        norm_b = np.sqrt(bb)
        _exchange(rh, dec, lo, hi)
        p_old = np.zeros(shape)
        it, beta = 0, 0.0
        while True:
            # p on owned AND halo planes (halo from the exchanged r)
            p_new = rh * c if it == 0 else rh * c + beta * p_old
            ap = _stencil(p_new, lo, hi, dec.z0 > 0, dec.z1 < n, off, diag)
            own = p_new[lo:lo + nzl]
            (pap,) = _allreduce([float((own * ap).sum())])
            alpha = rz / pap
            x = x + alpha * own
            rn = rh[lo:lo + nzl] + (-alpha) * ap
            rh[lo:lo + nzl] = rn
            it += 1
            rr, rz_new = _allreduce([float((rn * rn).sum()), float((rn * (rn * c)).sum())])
            if np.sqrt(rr) / norm_b <= 1e-8 or it >= 5000:
                break
            beta = rz_new / rz
            rz = rz_new
            _exchange(rh, dec, lo, hi)
            p_old = p_new
        q.put((rank, dec.z0, dec.z1, it, x))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_cg_matches_single_domain(world):
    import oracle as orc

    n = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    x = np.concatenate([r[4] for r in res]).ravel()  # planes in order -> flat x-fastest
    its = {r[3] for r in res}
    assert len(its) == 1  # every rank stopped at the same iteration
    a = orc.poisson_sym(n, 1.0 / n)
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    xo, so = orc.pcg(lambda v, o: orc.spmv_sym(a, v, 1, o), b, precond=orc.jacobi_from(a), tol=1e-8,
                     max_iter=5000)
    assert abs(its.pop() - so.iterations) <= 2
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-10


def test_slab_precond_validation():
    """The z-slab CG accepts only Jacobi or no preconditioner (DIC does not
    shard); anything else is a ValueError, not a silent
    unpreconditioned solve."""
    from paper_2504_03697_b200 import _lib, distributed

    assert distributed._slab_precond("jacobi") == _lib.PRECOND_JACOBI
    assert distributed._slab_precond(None) == _lib.PRECOND_NONE
    assert distributed._slab_precond("none") == _lib.PRECOND_NONE
    for bad in ("dic", "Jacobi", 3):
        with pytest.raises(ValueError, match="z-slab CG"):
            distributed._slab_precond(bad)
