"""GPU: the peer-memory z-slab CG's cross-process linking (cf_pcg_export /
cf_pcg_import over torch.distributed), with two ranks as two processes on the
one GPU of the test box.  No kernel runs -- nothing waits on another process
-- only the CUDA IPC handles are exchanged and opened, and each rank reads,
through the opened pointers, the neighbour plane its boundary r plane would
be stored into: it must hold exactly what the neighbour wrote at that plane
of its own allocation (the hi halo plane of the lower slab, the lo halo plane
of the upper one)."""

import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NX, NY, NZ = 32, 8, 16


def _pattern(rank, planes):
    return (np.arange(planes * NX * NY, dtype=np.float64).reshape(planes, NX * NY) + 1e6 * (rank + 1)).ravel()


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2504_03697_b200 import _lib
        from paper_2504_03697_b200.distributed import PeerSlabCG
        from paper_2504_03697_b200.parallel import SlabDecomposition

        dec = SlabDecomposition(NX, NY, NZ, world, rank)
        cg = PeerSlabCG(NX, NY, NZ, 1.0 / NX, "sym", bounds=[dec.z0, dec.z1], distributed=True)
        lib = _lib.load_library()
        lo, hi = int(rank > 0), int(rank < world - 1)
        planes = dec.z1 - dec.z0 + lo + hi
        mine = _pattern(rank, planes)
        _lib.check(lib.cf_pcg_debug_io(cg._h, 0, 1, mine.ctypes.data, mine.size), "write")
        dist.barrier()
        pl = NX * NY
        got = {}
        for which, peer in ((1, rank - 1), (2, rank + 1)):
            if 0 <= peer < world:
                buf = np.empty(pl)
                _lib.check(lib.cf_pcg_debug_io(cg._h, which, 0, buf.ctypes.data, pl), "read")
                got[which] = buf
        # the single pass's arrays: two halo planes each side, two planes per neighbour
        sp = {}
        if cg.single_pass:
            sp_planes = dec.z1 - dec.z0 + 4
            mine2 = _pattern(rank + 10, sp_planes)
            _lib.check(lib.cf_pcg_debug_io(cg._h, 3, 1, mine2.ctypes.data, mine2.size), "write sp")
        dist.barrier()
        if cg.single_pass:
            for which, peer in ((4, rank - 1), (5, rank + 1)):
                if 0 <= peer < world:
                    buf = np.empty(2 * pl)
                    _lib.check(lib.cf_pcg_debug_io(cg._h, which, 0, buf.ctypes.data, 2 * pl), "read sp")
                    sp[which] = buf
        dist.barrier()
        res = {}
        for which, buf in sp.items():
            peer = rank - 1 if which == 4 else rank + 1
            pdec = SlabDecomposition(NX, NY, NZ, world, peer)
            ref = _pattern(peer + 10, pdec.z1 - pdec.z0 + 4).reshape(-1, pl)
            # lower neighbour: its hi halo planes (array planes nzl + 2, + 3); upper: its planes 0, 1
            lo_plane = (pdec.z1 - pdec.z0) + 2 if which == 4 else 0
            want = ref[lo_plane:lo_plane + 2].ravel()
            res[which] = bool(np.array_equal(buf, want)) or (buf[:3].tolist(), want[:3].tolist())
        for which, buf in got.items():
            peer = rank - 1 if which == 1 else rank + 1
            pdec = SlabDecomposition(NX, NY, NZ, world, peer)
            plo, phi = int(peer > 0), int(peer < world - 1)
            pplanes = pdec.z1 - pdec.z0 + plo + phi
            ref = _pattern(peer, pplanes).reshape(pplanes, pl)
            # lower neighbour: its hi halo plane (after its lo halo + owned planes); upper: its lo halo plane 0
            want = ref[plo + (pdec.z1 - pdec.z0)] if which == 1 else ref[0]
            res[which] = bool(np.array_equal(buf, want)) or (buf[:3].tolist(), want[:3].tolist())
        del cg
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, None, repr(exc)))


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_linking_across_processes(cuda, world):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, res, err in out:
        assert err is None, (rank, err)
        expect = {1} if rank == world - 1 else ({2} if rank == 0 else {1, 2})
        expect |= {w + 3 for w in expect}  # the single pass's arrays (the default form)
        assert set(res) == expect and all(v is True for v in res.values()), (rank, res)
