"""GPU: the z-slab decomposition of the CG (the multi-GPU data path) run as
several slabs in one process on one device -- the real kernels with halo
planes, halo-p recomputation and per-slab partial sums -- against the
single-domain fused solve and the oracle.

Tolerances: iteration counts within +-2 (only the summation order of the
partial sums changes), solution rel-L2 <= 1e-9 between decomposed and
single-domain solves at tol 1e-10, <= 1e-8 against the oracle at tol 1e-8.
"""

import numpy as np
import pytest
import torch

import oracle as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("order", ["sym", "csr"])
@pytest.mark.parametrize("nslabs", [2, 3, 5])
def test_slabs_match_single_domain(cuda, order, nslabs):
    from paper_2504_03697_b200.distributed import emulated_pcg

    n = 64
    h = 1.0 / n
    b = np.random.default_rng(nslabs).uniform(-1, 1, n ** 3)
    op = cuda.StencilOperator(n, h, order)
    x1, s1 = cuda.pcg(op, b, precond=cuda.jacobi_from(op), tol=1e-10, max_iter=20000)
    xs, ss, _ = emulated_pcg(op, b, nslabs, tol=1e-10, max_iter=20000)
    assert ss.converged
    assert abs(ss.iterations - s1.iterations) <= 2, (ss.iterations, s1.iterations)
    assert rel(xs, x1) <= 1e-9


def test_slabs_match_oracle(cuda):
    from paper_2504_03697_b200.distributed import emulated_pcg

    n = 32
    h = 1.0 / n
    b = np.random.default_rng(0).uniform(-1, 1, n ** 3)
    b -= b.mean()
    a = orc.poisson_sym(n, h)
    xo, so = orc.pcg(lambda v, o: orc.spmv_sym(a, v, 1, o), b, precond=orc.jacobi_from(a), tol=1e-8,
                     max_iter=20000)
    x, st, _ = emulated_pcg(cuda.StencilOperator(n, h, "sym"), b, 4, tol=1e-8, max_iter=20000)
    assert abs(st.iterations - so.iterations) <= 2
    assert rel(x, xo) <= 1e-8


def test_slabs_edge_cases(cuda):
    from paper_2504_03697_b200.distributed import emulated_pcg

    op = cuda.StencilOperator(32, 1.0, "sym")
    x, st, _ = emulated_pcg(op, np.zeros(32 ** 3), 2)
    assert st.iterations == 0 and st.converged and not x.any()
    b = np.random.default_rng(1).standard_normal(32 ** 3)
    x, st, _ = emulated_pcg(op, b, 2, tol=1e-14, max_iter=3)
    assert not st.converged and st.iterations == 3
    xo, so = orc.pcg(lambda v, o: orc.spmv_sym(orc.poisson_sym(32, 1.0), v, 1, o), b,
                     precond=orc.jacobi_from(orc.poisson_sym(32, 1.0)), tol=1e-14, max_iter=3)
    assert rel(x, xo) <= 1e-12


def test_slabs_full_size(cuda):
    """256^3 split in 4 slabs: same iterations as the single-domain solve, true residual at tol."""
    from paper_2504_03697_b200.distributed import emulated_pcg

    n = 256
    h = 1.0 / n
    b = torch.as_tensor(np.random.default_rng(7).uniform(-1, 1, n ** 3), device="cuda")
    op = cuda.StencilOperator(n, h, "sym")
    x1, s1 = cuda.pcg(op, b, precond=cuda.jacobi_from(op), tol=1e-8, max_iter=20000)
    x4, s4, _ = emulated_pcg(op, b, 4, tol=1e-8, max_iter=20000)
    assert abs(s4.iterations - s1.iterations) <= 2
    r = b - op(x4)
    assert float(torch.linalg.norm(r) / torch.linalg.norm(b)) <= 2e-8
    assert float(torch.linalg.norm(x4 - x1) / torch.linalg.norm(x1)) <= 1e-7
