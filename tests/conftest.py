import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(os.path.join(GOLDEN, name + ".npz")) as d:
                cache[name] = {k: d[k] for k in d.files}
        return cache[name]

    return load


@pytest.fixture
def rng():
    # same seed as the reference suite (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def cuda():
    """The CUDA product path; GPU tests fail loudly if it cannot load."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test collected but no CUDA device is visible")
    import paper_2504_03697_b200 as cf

    cf.load_library()
    return cf


_ACHIEVED = []


@pytest.fixture
def achieved(request):
    """Record an achieved parity error (printed in the terminal summary and
    written to gpurun_out/parity_achieved.json, so a drift inside a tolerance
    band is visible run to run)."""

    def rec(what: str, **vals):
        _ACHIEVED.append({"test": request.node.nodeid, "what": what, **vals})

    return rec


def pytest_terminal_summary(terminalreporter):
    if not _ACHIEVED:
        return
    import json

    terminalreporter.write_sep("-", "achieved parity (GPU vs oracle / reference fixtures)")
    for r in _ACHIEVED:
        vals = " ".join(f"{k}={v:.2e}" if isinstance(v, float) else f"{k}={v}" for k, v in r.items()
                        if k not in ("test", "what"))
        terminalreporter.write_line(f"{r['what']}: {vals}")
    out = os.path.join(ROOT, "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_achieved.json"), "w") as f:
            json.dump(_ACHIEVED, f, indent=1)
    except OSError:
        pass
