"""GPU: the snapshot path -- device cell-centring
(cf_snapshot_cells) + one D2H + the native writer -- against the reference's
writer bytes (tests/golden/snapshot.npz, produced by the reference itself)
and the oracle's columns.  Bar: bit-exact columns, byte-identical files."""

import hashlib

import numpy as np
import pytest

import oracle as orc

pytestmark = pytest.mark.gpu


def test_device_cell_centring_bitwise(cuda, golden):
    s = golden("snapshot")
    n, h = s["exotic_p"].shape[0], float(s["exotic_h"])
    n = round(n ** (1 / 3))
    spec = cuda.GridSpec(n, h)
    st = cuda.SimState(vel=cuda.VelocityField(spec, s["exotic_u"], s["exotic_v"], s["exotic_w"]),
                       p=cuda.ScalarField(spec, s["exotic_p"]))
    snap = cuda.snapshot_from_state(st)
    want = orc.snapshot_columns(orc.State(s["exotic_u"], s["exotic_v"], s["exotic_w"], s["exotic_p"]), h)
    for c in "xyzuvwp":
        assert np.array_equal(snap.column(c), want[c], equal_nan=True), c


@pytest.mark.parametrize("mode,threads", [("serial", 1), ("buffered_parallel", 3)])
def test_state_snapshot_bytes_match_reference_writer(cuda, golden, tmp_path, mode, threads):
    s = golden("snapshot")
    n = round(s["exotic_p"].shape[0] ** (1 / 3))
    spec = cuda.GridSpec(n, float(s["exotic_h"]))
    st = cuda.SimState(vel=cuda.VelocityField(spec, s["exotic_u"], s["exotic_v"], s["exotic_w"]),
                       p=cuda.ScalarField(spec, s["exotic_p"]))
    path = tmp_path / "s.csv"
    cuda.write_snapshot(st, str(path), mode=mode, threads=threads)
    assert hashlib.sha256(path.read_bytes()).digest() == s["exotic_sha256"].tobytes()
    # a prebuilt Snapshot writes the same file
    path2 = tmp_path / "s2.csv"
    cuda.write_snapshot(cuda.snapshot_from_state(st), str(path2))
    assert path2.read_bytes() == path.read_bytes()


def test_run_snapshots_roundtrip_and_box(cuda, tmp_path):
    """A run's snapshot files re-read to the device state's columns; a box
    snapshot reads back with shape=."""
    cfg = cuda.SimConfig(n=8, dt=0.4, t_end=0.8, output_dir=str(tmp_path / "r"))
    st, rep = cuda.run(cfg)
    back = cuda.read_snapshot(rep.snapshot_paths[-1])
    now = cuda.snapshot_from_state(st)
    assert cuda.compare_snapshots(back, now, 0.0).passed
    shape = (12, 7, 9)
    bcfg = cuda.SimConfig(n=12, h=1.0 / 12, dt=0.01, t_end=0.02, shape=shape, preconditioner="jacobi",
                          variant="optimized")
    bst = cuda.initial_state(bcfg)
    for _ in range(bcfg.num_steps):
        cuda.step(bst, bcfg)
    path = tmp_path / "box.csv"
    cuda.write_snapshot(bst, str(path))
    snap = cuda.read_snapshot(str(path), shape=shape)
    u, v, w = bst.vel.numpy()
    ost = orc.State(u, v, w, bst.p.numpy())
    nx, ny, nz = shape
    assert np.array_equal(snap.u, (0.5 * (u[:-1] + u[1:])).flatten(order="F"))
    assert np.array_equal(snap.w, (0.5 * (w[:, :, :-1] + w[:, :, 1:])).flatten(order="F"))
    assert np.array_equal(snap.y, np.tile(np.repeat((np.arange(ny) + 0.5) * (1.0 / 12), nx), nz))
    assert np.array_equal(snap.p, ost.p)
    with pytest.raises(ValueError, match="not a cube"):
        cuda.read_snapshot(str(path))
