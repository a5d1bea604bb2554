"""Profiler / report parity on the host: the renderers
and writers against the reference's own outputs on fixed records
(tests/golden/profiling.json, made by tests/golden/make_golden.py from the
reference), the region bookkeeping, and the sweep's argument checks.
Bar: identical text / bytes."""

import json
import os
import time

import pytest

from paper_2504_03697_b200 import profiling as pf

HERE = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fx():
    with open(os.path.join(HERE, "profiling.json"), encoding="utf-8") as f:
        return json.load(f)


def recs(rows):
    return [pf.RegionStats(**r) for r in rows]


def test_render_report_matches_reference(fx):
    assert pf.render_report(recs(fx["a"])) == fx["render_a"]
    assert pf.render_report(recs(fx["b"])) == fx["render_b"]
    assert pf.render_report([]) == f"{'Region':<6}  {'Calls':>8}  {'Incl. s':>10}  {'Rt. %':>7}"


def test_report_json_roundtrip_matches_reference(fx, tmp_path):
    path = tmp_path / "r.json"
    pf.save_report(recs(fx["a"]), path)
    assert path.read_text(encoding="utf-8") == fx["saved_a"]
    assert pf.load_report(path) == recs(fx["a"])
    # round-1 form of this package still loads
    legacy = tmp_path / "old.json"
    legacy.write_text(json.dumps({"regions": fx["b"]}))
    assert pf.load_report(legacy) == recs(fx["b"])


def test_compare_reports_matches_reference(fx):
    rows = pf.compare_reports(recs(fx["a"]), recs(fx["b"]))
    assert rows == fx["compare"]
    assert pf.render_comparison(rows) == fx["render_compare"]


def test_scaling_csv_matches_reference(fx, tmp_path):
    path = tmp_path / "s.csv"
    pf.write_scaling_csv([tuple(r) for r in fx["scaling_rows"]], path)
    assert path.read_bytes() == fx["scaling_csv"].encode()


def test_profiler_tree_and_errors():
    p = pf.Profiler()
    with p.region("root"):
        for _ in range(3):
            with p.region("a"):
                with p.region("x"):
                    time.sleep(0.001)
            with p.region("b"):
                pass
    with p.region("root2"):
        pass
    st = p.stats()
    assert [(r.name, r.parent, r.calls) for r in st] == [("root", None, 1), ("a", "root", 3), ("x", "a", 3),
                                                        ("b", "root", 3), ("root2", None, 1)]
    assert st[0].inclusive_seconds >= st[1].inclusive_seconds >= st[2].inclusive_seconds >= 0.003
    assert abs(st[0].fraction + st[4].fraction - 1.0) < 1e-12
    p.enter("open")
    with pytest.raises(pf.ProfileError, match="still open"):
        p.stats()
    with pytest.raises(pf.ProfileError, match="unbalanced"):
        p.exit("other")
    with pytest.raises(pf.ProfileError, match="cannot reset"):
        p.reset()
    p.exit("open")
    p.reset()
    assert p.stats() == []
    with pytest.raises(ValueError):
        pf.Profiler(timer="cycles")


def test_scaling_sweep_argument_checks():
    from paper_2504_03697_b200.sim import SimConfig

    cfg = SimConfig(n=8, dt=0.4, t_end=0.4)
    with pytest.raises(ValueError, match="at least one"):
        pf.scaling_sweep(cfg, [])
    with pytest.raises(ValueError, match=">= 1"):
        pf.scaling_sweep(cfg, [1, 0])
