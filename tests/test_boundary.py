"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/cfgpu.h declares (no CUDA call is made),
and the host-side API mirrors the reference's names and argument checks."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cfgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int)\s*(cf_\w+)\s*\(", text, re.M)))


def test_header_declares_the_reference_seams():
    names = declared_symbols()
    for must in ("cf_dot", "cf_axpy", "cf_csr_spmv", "cf_sym_spmv", "cf_stencil7_apply", "cf_cg_solve",
                 "cf_advect", "cf_divergence", "cf_pressure_correct", "cf_forces_bc", "cf_dic_apply"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2504_03697_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__

        __graft_entry__.build()
    lib = _lib.open_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.EXPORTED)
    assert lib.cf_version() == 1


def test_library_is_sm100a_only():
    """The shipped cubin targets sm_100a (no PTX JIT, no other arch)."""
    import subprocess

    from paper_2504_03697_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\w+", out))
    assert archs == {"sm_100a"}, archs


def test_level_schedule_host_only():
    """cf_level_schedule is host code: the 7-point lower triangle levels are i+j+k."""
    from paper_2504_03697_b200 import _lib
    from paper_2504_03697_b200.sim import poisson_full_csr

    lib = _lib.open_library()
    n = 5
    a = poisson_full_csr(n, 1.0)
    rows = a.row_indices()
    m = a.col_idx < rows
    ptr = np.concatenate(([0], np.cumsum(np.bincount(rows[m], minlength=n ** 3)))).astype(np.int64)
    col = np.ascontiguousarray(a.col_idx[m])
    lv = np.empty(n ** 3, dtype=np.int32)
    nl = np.zeros(1, dtype=np.int32)
    assert lib.cf_level_schedule(n ** 3, ptr.ctypes.data, col.ctypes.data, lv.ctypes.data, nl.ctypes.data) == 0
    idx = np.arange(n ** 3)
    assert np.array_equal(lv, idx % n + (idx // n) % n + idx // (n * n))
    assert nl[0] == 3 * n - 2


def test_config_validation_mirrors_reference():
    from paper_2504_03697_b200.sim import SimConfig

    for bad in (dict(n=1), dict(dt=0.0), dict(t_end=-1.0), dict(preconditioner="ilu"),
                dict(variant="turbo"), dict(threads=0), dict(max_iter=0), dict(tol=0.0)):
        with pytest.raises(ValueError):
            SimConfig(**bad)
    assert SimConfig(n=4, dt=0.4, t_end=6.0).num_steps == 15
    assert SimConfig(n=4, dt=0.1, t_end=1.0).num_steps == 10


def test_csr_validation_mirrors_reference():
    from paper_2504_03697_b200.sparse import CsrMatrix, to_symmetric

    with pytest.raises(ValueError, match="row_ptr"):
        CsrMatrix(2, 2, [1, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="decreases"):
        CsrMatrix(3, 2, [0, 2, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="out of range"):
        CsrMatrix(2, 2, [0, 1, 2], [0, 5], [1.0, 1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        CsrMatrix(2, 3, [0, 2, 2], [1, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="nnz"):
        CsrMatrix(2, 2, [0, 1, 3], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="not symmetric"):
        to_symmetric(CsrMatrix.from_dense([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(ValueError, match="not symmetric"):
        to_symmetric(CsrMatrix.from_dense([[1.0, 2.0], [3.0, 1.0]]))
    with pytest.raises(ValueError, match="square"):
        to_symmetric(CsrMatrix(1, 2, [0, 1], [1], [1.0]))
    s = to_symmetric(CsrMatrix.from_dense([[2.0, -1.0], [-1.0, 2.0]]))
    assert np.array_equal(s.diag, [2.0, 2.0]) and np.array_equal(s.col_idx, [1])


def test_assembly_matches_reference_fixture(golden):
    from paper_2504_03697_b200.sim import poisson_full_csr, poisson_symmetric

    g = golden("sparse")
    for n in (5, 16):
        h = float(g[f"n{n}_h"])
        a, s = poisson_full_csr(n, h), poisson_symmetric(n, h)
        assert np.array_equal(a.row_ptr, g[f"n{n}_row_ptr"])
        assert np.array_equal(a.col_idx, g[f"n{n}_col_idx"])
        assert np.array_equal(a.values, g[f"n{n}_values"])
        assert np.array_equal(s.row_ptr, g[f"n{n}_sym_row_ptr"])
        assert np.array_equal(s.values, g[f"n{n}_sym_values"])


def test_product_path_fails_loudly_without_cuda():
    """No CPU fallback: without a device every compute entry point raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import paper_2504_03697_b200 as cf

    with pytest.raises(RuntimeError, match="CUDA"):
        cf.dot(np.ones(3), np.ones(3))
    with pytest.raises(RuntimeError, match="CUDA"):
        cf.StencilOperator(4, 1.0)(np.ones(64))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2504_03697_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text, f
