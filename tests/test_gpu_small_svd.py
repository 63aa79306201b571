"""The in-house dense factorisations of the Nystrom step against LAPACK (numpy): the cluster
block Jacobi SVD (ngd_svd.cu) on graded matrices like the Nystrom factor's R (singular values
spanning 1 .. 1e-8, with a tail cluster at the shift floor), the Cholesky kernels including the
blocked form above 512 (ngd_chol.cu + DMMA GEMM updates), and cuSOLVER's polar SVD used above 512."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2505_11638_b200 import _lib  # noqa: E402
from paper_2505_11638_b200.gramian import utility_context  # noqa: E402


def graded(n, seed):
    rng = np.random.default_rng(seed)
    s = np.concatenate([np.logspace(0, -8, n // 2), 1e-8 * (1 + 1e-3 * np.arange(n - n // 2))])
    qa, _ = np.linalg.qr(rng.standard_normal((n, n)))
    qb, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (qa * s) @ qb.T
    # even seeds: the triangular factor of a QR (the Nystrom case); odd: a dense matrix
    return np.linalg.qr(a)[1] if seed % 2 == 0 else a


@pytest.mark.parametrize("method,n", [(3, 7), (3, 100), (3, 101), (3, 160), (3, 300), (3, 301), (3, 310),
                                      (4, 7), (4, 100), (4, 101), (4, 160), (4, 300), (4, 301), (4, 310),
                                      (4, 311), (4, 400), (4, 401), (4, 500), (4, 512), (1, 700), (1, 1000)])
def test_jacobi_svd_matches_lapack(method, n):
    a = graded(n, n)
    ctx = utility_context()
    A = torch.as_tensor(np.asfortranarray(a).T.copy(), device="cuda")  # column-major storage
    U = torch.empty((n, n), dtype=torch.float64, device="cuda")
    S = torch.empty(n, dtype=torch.float64, device="cuda")
    sweeps = _lib.ctypes.c_int32()
    ctx.call("ngd_small_svd", _lib.ptr(A), n, _lib.ptr(U), _lib.ptr(S), method, _lib.ctypes.byref(sweeps))
    assert sweeps.value > 0 or method == 1, "Jacobi did not converge"
    print(f"n={n} sweeps={sweeps.value}")
    s_ref = np.linalg.svd(a, compute_uv=False)
    s = S.cpu().numpy()
    # absolute accuracy eps * s1 (backward stability) and relative accuracy on the head
    assert np.max(np.abs(s - s_ref)) <= 50 * n * 2.2e-16 * s_ref[0]
    head = s_ref > 1e-6 * s_ref[0]
    assert np.max(np.abs(s[head] - s_ref[head]) / s_ref[head]) <= 1e-10
    u = U.cpu().numpy().T  # back to row-major (n, n): columns are left singular vectors
    assert np.linalg.norm(u.T @ u - np.eye(n)) <= 1e-12 * n
    # A = U diag(s) V^T  <=>  ||U^T A||_rows == s
    np.testing.assert_allclose(np.linalg.norm(u.T @ a, axis=1), s, rtol=1e-8, atol=1e-13)


@pytest.mark.parametrize("n", [1, 5, 16, 17, 100, 160, 300])
def test_small_cholesky_matches_lapack(n):
    """In-house Cholesky (ngd_chol.cu) via the Nystrom prepare path: Omega <- Omega R^{-1}
    must be orthonormal and R upper with R^T R = Omega0^T Omega0."""
    rng = np.random.default_rng(n)
    p = 4 * n + 3
    om0 = rng.standard_normal((p, n))
    ctx = utility_context()
    Om = torch.as_tensor(om0.T.copy(), device="cuda")  # p x n column-major
    ctx.call("ngd_nystrom_prepare", _lib.ptr(Om), p, n)
    q = Om.cpu().numpy().T
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-13 * max(n, 1)
    r = q.T @ om0
    np.testing.assert_allclose(np.triu(r), r, atol=1e-11)
    np.testing.assert_allclose(np.abs(np.diag(r)), np.abs(np.diag(np.linalg.qr(om0)[1])), rtol=1e-10)


@pytest.mark.parametrize("method", [1, 2, 0])
@pytest.mark.parametrize("n", [1, 5, 31, 32, 33, 100, 160, 300, 512, 513, 700, 1000, 1100])
def test_cholesky_kernels(n, method):
    """ngd_small_cholesky: one-CTA (n <= 160), cluster (n <= 512) and the library's choice (blocked
    with DMMA GEMM updates above 512) agree with LAPACK."""
    if (method == 1 and n > 160) or (method == 2 and n > 512):
        pytest.skip("kernel size limit")
    rng = np.random.default_rng(100 + n)
    g = rng.standard_normal((2 * n + 5, n))
    a = g.T @ g + 1e-3 * np.eye(n)
    ctx = utility_context()
    A = torch.as_tensor(a.T.copy(), device="cuda")  # column-major
    info = _lib.ctypes.c_int32()
    ctx.call("ngd_small_cholesky", _lib.ptr(A), n, method, _lib.ctypes.byref(info))
    assert info.value == 0
    u = np.triu(A.cpu().numpy().T)
    ref = np.linalg.cholesky(a).T
    assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref) * max(1.0, np.linalg.cond(ref))
    np.testing.assert_allclose(u.T @ u, a, rtol=0, atol=1e-12 * np.abs(a).max())


@pytest.mark.parametrize("method", [1, 2, 0])
@pytest.mark.parametrize("n,k", [(40, 0), (40, 17), (300, 250), (300, 31), (300, 32), (1000, 100),
                                 (1000, 700), (1000, 512)])
def test_cholesky_failure_index(n, k, method):
    """Non-positive pivot k: info = k + 1 (LAPACK potrf semantics) for every method."""
    if (method == 1 and n > 160) or (method == 2 and n > 512):
        pytest.skip("kernel size limit")
    d = np.ones(n)
    d[k] = -1.0
    q, _ = np.linalg.qr(np.random.default_rng(n + k).standard_normal((n, n)))
    # block structure keeps the leading k x k minor positive definite and makes pivot k fail
    a = np.diag(d)
    a[:k, :k] = q[:k, :k] @ q[:k, :k].T + np.eye(k)
    ctx = utility_context()
    A = torch.as_tensor(a.T.copy(), device="cuda")
    info = _lib.ctypes.c_int32()
    ctx.call("ngd_small_cholesky", _lib.ptr(A), n, method, _lib.ctypes.byref(info))
    assert info.value == k + 1
