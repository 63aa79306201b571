"""The in-house FP64 DMMA GEMM (ngd_gemm.cu) behind every dense product of the Nystrom sketch and
factorisation, through the C-ABI test hook ngd_gemm: all four operand layouts (TMA K-major and
MN-major boxes), partial tiles, split-K (fixed-order partial sums: bitwise reproducible), odd
leading dimensions (staged copies), alpha / beta, and the sketch's own shapes at C2."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2505_11638_b200 import _lib  # noqa: E402
from paper_2505_11638_b200.gramian import utility_context  # noqa: E402


def colmajor(a, ld=None):
    """numpy (r, c) -> CUDA storage of the column-major matrix with leading dimension ld >= r."""
    r, c = a.shape
    ld = ld or r
    buf = np.zeros((c, ld))
    buf[:, :r] = a.T
    return torch.as_tensor(buf, device="cuda"), ld


def run(ta, tb, M, N, K, alpha=1.0, beta=0.0, lda_pad=0, ldb_pad=0, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((K, M) if ta else (M, K))
    b = rng.standard_normal((N, K) if tb else (K, N))
    c0 = rng.standard_normal((M, N))
    A, lda = colmajor(a, a.shape[0] + lda_pad)
    B, ldb = colmajor(b, b.shape[0] + ldb_pad)
    C, ldc = colmajor(c0)
    ctx = utility_context()
    ctx.call("ngd_gemm", int(ta), int(tb), M, N, K, float(alpha), _lib.ptr(A), lda, _lib.ptr(B), ldb, float(beta),
             _lib.ptr(C), ldc)
    out = C.cpu().numpy()[:, :M].T
    ref = alpha * ((a.T if ta else a) @ (b.T if tb else b)) + beta * c0
    scale = np.abs(alpha) * np.sqrt(K) * 1.0 + np.abs(beta) * np.abs(c0).max()
    return out, ref, scale


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (128, 128, 16), (129, 130, 17), (64, 300, 1000),
                                   (300, 300, 8577), (513, 257, 33)])
def test_layouts_and_shapes(ta, tb, M, N, K):
    out, ref, scale = run(ta, tb, M, N, K, seed=M + N + K)
    assert np.max(np.abs(out - ref)) <= 1e-14 * scale * 8


@pytest.mark.parametrize("ta,tb,lda_pad,ldb_pad", [(1, 0, 1, 0), (0, 0, 3, 1), (0, 1, 0, 2), (1, 1, 5, 3)])
def test_odd_leading_dimensions_and_alpha_beta(ta, tb, lda_pad, ldb_pad):
    out, ref, scale = run(ta, tb, 200, 150, 301, alpha=-0.5, beta=1.5, lda_pad=lda_pad, ldb_pad=ldb_pad)
    assert np.max(np.abs(out - ref)) <= 1e-14 * scale * 8


@pytest.mark.parametrize("M,N,K,ta,tb", [(4608, 300, 8577, 1, 0),  # C2 sketch: S = J_c Omega (split-K)
                                         (8577, 300, 4608, 0, 0),  # C2 sketch: Y = J_c^T S
                                         (300, 300, 8577, 1, 0)])  # tall Gram
def test_sketch_shapes_bitwise_reproducible(M, N, K, ta, tb):
    o1, ref, scale = run(ta, tb, M, N, K, seed=5)
    o2, _, _ = run(ta, tb, M, N, K, seed=5)
    assert np.max(np.abs(o1 - ref)) <= 1e-14 * scale * 8
    assert np.array_equal(o1, o2)
