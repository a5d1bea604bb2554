"""The native snapshot CSV writer on the host: its value
formatter against the reference's rule (repr, integral '.0' dropped;
src/snapshots.py:65-70) and its files against the reference's bytes --
the committed golden CSV (sha256) and the reference writer's output on an
exotic-valued state (tests/golden/snapshot.npz).  Host-only entry points:
no GPU needed.  Bar: byte-identical."""

import ctypes
import hashlib
import struct

import numpy as np
import pytest

import oracle as orc


@pytest.fixture(scope="module")
def lib():
    from paper_2504_03697_b200 import _lib

    return _lib.host_library()


def fmt(lib, v):
    buf = ctypes.create_string_buffer(32)
    n = lib.cf_format_double(float(v), buf, 32)
    return buf.raw[:n].decode()


def test_format_double_matches_repr_rule(lib):
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 63, size=100_000, dtype=np.int64).view(np.float64)
    vals = list(bits[np.isfinite(bits)])
    vals += list(rng.standard_normal(50_000) * 10.0 ** rng.integers(-30, 30, 50_000))
    vals += list(np.round(rng.standard_normal(20_000) * 10.0 ** rng.integers(0, 20, 20_000)))
    edges = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e16, 1e15, 9999999999999998.0, 1e17, 1e-4, 1e-5, 0.00012345,
             1.2345e-5, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 123456789012345678.0,
             2.0 ** 53, 2.0 ** 53 + 2, 1.0 / 3.0, 2.0 / 3.0, 100.0, 1e22, 1e23, 1e-7, 0.3, float("inf"),
             float("-inf"), float("nan")]
    vals += edges + [-e for e in edges]
    bad = [(v, fmt(lib, v), orc.format_value(v)) for v in vals if fmt(lib, v) != orc.format_value(v)]
    assert not bad, bad[:5]


def test_format_double_rejects_small_buffer(lib):
    buf = ctypes.create_string_buffer(8)
    assert lib.cf_format_double(1.0, buf, 8) == -1


def _write_columns(lib, path, cols, threads):
    arrs = [np.ascontiguousarray(cols[c], dtype=np.float64) for c in "xyzuvwp"]
    rc = lib.cf_csv_write_columns(str(path).encode(), *(a.ctypes.data for a in arrs), len(arrs[0]), threads)
    assert rc == 0
    return path.read_bytes()


@pytest.mark.parametrize("threads", [1, 4])
def test_reference_golden_csv_bytes(lib, golden, tmp_path, threads):
    """Re-writing the reference's golden CSV values reproduces its file byte for byte."""
    g, s = golden("cavity"), golden("snapshot")
    cols = {c: g[f"ref_csv_{c}"] for c in "xyzuvwp"}
    data = _write_columns(lib, tmp_path / "g.csv", cols, threads)
    assert len(data) == int(s["ref_csv_len"])
    assert hashlib.sha256(data).digest() == s["ref_csv_sha256"].tobytes()


def test_reference_writer_bytes_exotic_values(lib, golden, tmp_path):
    s = golden("snapshot")
    st = orc.State(s["exotic_u"], s["exotic_v"], s["exotic_w"], s["exotic_p"])
    cols = orc.snapshot_columns(st, float(s["exotic_h"]))
    assert hashlib.sha256(orc.snapshot_csv(cols)).digest() == s["exotic_sha256"].tobytes()  # oracle pinned
    data = _write_columns(lib, tmp_path / "e.csv", cols, 3)
    assert hashlib.sha256(data).digest() == s["exotic_sha256"].tobytes()


def test_multi_block_thread_invariance(lib, tmp_path):
    """Several 32768-row blocks, any thread count: the same bytes as the oracle."""
    rng = np.random.default_rng(5)
    nrows = 70_001
    cols = {c: rng.standard_normal(nrows) * 10.0 ** rng.integers(-8, 8, nrows) for c in "xyzuvwp"}
    want = orc.snapshot_csv(cols)
    for t in (1, 2, 7):
        assert _write_columns(lib, tmp_path / f"m{t}.csv", cols, t) == want


def test_write_errors(lib, tmp_path):
    from paper_2504_03697_b200 import _lib

    x = np.zeros(1)
    rc = lib.cf_csv_write_columns(str(tmp_path / "no" / "such" / "dir.csv").encode(), *([x.ctypes.data] * 7), 1, 1)
    assert rc == _lib.CF_EIO
    with pytest.raises(OSError, match="cannot open"):
        _lib.check(rc, "write")
