"""pcg_jacobi / CsrMatrix::multiply on a caller matrix through the GPU (C ABI
tg_pcg_jacobi / tg_csr_multiply): the reference's own sparse pins
(proj/tests/test_sparse.cpp) plus a comparison with the unmodified
reference pcg_jacobi on the same matrices (iterations, solution)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2511_20432_b200 as tg

pytestmark = pytest.mark.gpu


def test_identity_solve(gpu_ctx):
    x, it, rel = gpu_ctx.pcg_jacobi(np.eye(3), [3.0, -2.0, 0.5])
    assert x == pytest.approx([3.0, -2.0, 0.5], rel=1e-12)
    assert rel <= 1e-10


def test_2x2_by_hand(gpu_ctx):
    x, _, _ = gpu_ctx.pcg_jacobi([[4.0, 1.0], [1.0, 3.0]], [1.0, 2.0])
    assert x[0] == pytest.approx(1.0 / 11.0, rel=1e-10)
    assert x[1] == pytest.approx(7.0 / 11.0, rel=1e-10)


def random_spd(n, seed):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n))
    return G.T @ G + n * np.eye(n), rng.standard_normal(n)


def test_random_spd_residual_contract(gpu_ctx):
    A, b = random_spd(50, 33)
    x, _, _ = gpu_ctx.pcg_jacobi(A, b, tol=1e-10, max_iter=500)
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) <= 1e-9


def test_iteration_cap_raises(gpu_ctx):
    with pytest.raises(tg.NumericError, match=r"pcg: no convergence in 1 iterations, "
                                              r"relative residual"):
        gpu_ctx.pcg_jacobi([[4.0, 1.0], [1.0, 3.0]], [1.0, 2.0], tol=1e-14, max_iter=1)


def test_zero_rhs_returns_zero(gpu_ctx):
    x, it, rel = gpu_ctx.pcg_jacobi([[2.0, 0.0], [0.0, 2.0]], [0.0, 0.0], x=[5.0, -1.0])
    assert it == 0 and x[0] == 0.0 and x[1] == 0.0


def test_non_spd_errors(gpu_ctx):
    with pytest.raises(tg.NumericError, match="pcg: non-positive diagonal, matrix not SPD"):
        gpu_ctx.pcg_jacobi([[0.0, 1.0], [1.0, 2.0]], [1.0, 1.0])
    with pytest.raises(tg.NumericError, match="pcg: indefinite direction, matrix not SPD"):
        gpu_ctx.pcg_jacobi([[1.0, 3.0], [3.0, 1.0]], [1.0, -1.0])


def test_matches_reference_pcg(gpu_ctx, ref):
    """Same iterates as the unmodified reference on a larger sparse SPD
    system: iteration count within one, solution within 1e-12."""
    n = 2000
    rng = np.random.default_rng(5)
    main = 4.0 + rng.uniform(0, 1, n)
    off = -rng.uniform(0.5, 1.0, n - 1)
    A = sp.diags([off, main, off], [-1, 0, 1], format="csr")
    A.sort_indices()
    b = rng.standard_normal(n)
    x, it, rel = gpu_ctx.pcg_jacobi(A, b, tol=1e-12, max_iter=5000)
    xr, itr, relr = ref.pcg(A.indptr, A.indices, A.data, b, np.zeros(n), tol=1e-12, max_iter=5000)
    assert abs(it - itr) <= 1
    assert np.abs(x - xr).max() <= 1e-12 * np.abs(xr).max()
    assert np.array_equal(gpu_ctx.csr_multiply(A, x), gpu_ctx.csr_multiply(A, x))
    y = gpu_ctx.csr_multiply(A, x)
    assert np.abs(y - A @ x).max() <= 1e-14 * np.abs(A @ x).max()
