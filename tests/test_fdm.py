"""Fast-diagonalization factors (host/fdm.cpp) on CPU: for every direction of
the config-0 Kronecker operator (free grid: the constrained first z layer
dropped), V^T M V = I, V^T K V = diag(lam), and lam equals the generalized
eigenvalues of (K, M) from LAPACK."""
import ctypes as C
import os

import numpy as np
import pytest
import scipy.linalg

import paper_2511_20432_b200 as tg
from conftest import ROOT


def dense(B, first, n):
    w = B.shape[1]
    p = w // 2
    A = np.zeros((n, n))
    for i in range(n):
        for d in range(-p, p + 1):
            if 0 <= i + d < n:
                A[i, i + d] = B[first + i, p + d]
    return A


@pytest.mark.parametrize("name", ["cfg0_parity", "cfg0_oddx"])
def test_fdm_factor_generalized_eigenpairs(name):
    s = tg.Simulation(os.path.join(ROOT, "configs", name + ".cfg"), host_only=True)
    L = tg.lib()
    L.tg_fdm_factor.argtypes = [C.POINTER(C.c_double)] * 2 + [C.c_int] * 4 + [C.POINTER(C.c_double)] * 2
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for d in range(3):
        M, K = (np.ascontiguousarray(a) for a in s.kron_factors(d))
        nb, w = M.shape
        p = w // 2
        first = 1 if d == 2 else 0
        n = nb - first
        V = np.zeros(n * n)
        lam = np.zeros(n)
        assert L.tg_fdm_factor(dp(M), dp(K), nb, p, first, n, dp(V), dp(lam)) == 0
        V = V.reshape(n, n).T  # column-major -> V[:, k] = eigenvector k
        Md, Kd = dense(M, first, n), dense(K, first, n)
        assert np.abs(V.T @ Md @ V - np.eye(n)).max() <= 1e-12
        assert np.abs(V.T @ Kd @ V - np.diag(lam)).max() <= 1e-11 * np.abs(lam).max()
        ref = scipy.linalg.eigh(Kd, Md, eigvals_only=True)
        assert np.allclose(np.sort(lam), ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    s.close()
