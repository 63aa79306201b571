"""The FP64-exact GEMM on the INT8 tensor cores (Ozaki scheme II, ngd_ozaki.cu) behind the large
sketches' S = J_c Omega and Y += J_c^T S (gramian.py:55-61):

* integer-valued operands (the modular arithmetic and CRT are exact; the one final rounding of
  C' 2^-(alpha+beta) leaves <= 2 ulp);
* graded / wide-range random operands against an extended-precision product: inside the scheme's
  error bound 2^-52 (max|A_m.| sum|B_.n| + sum|A_m.| max|B_.n|) + 2^-52 |AB| (the same order as an
  FP64 GEMM's own bound, and compared with the in-house DMMA GEMM's error on the same inputs);
* K beyond one exact int32 accumulation (two K-splits), partial tiles, alpha / beta, zero rows,
  non-finite inputs (NaN rows / columns, not silently finite);
* the sketch itself: Y = G Omega on the INT8 engine vs the DMMA engine at the configs' full sizes,
  and vs the CPU oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
ngd = pytest.importorskip("paper_2505_11638_b200")
from paper_2505_11638_b200 import _lib  # noqa: E402
from paper_2505_11638_b200.gramian import utility_context  # noqa: E402


def oz(a, b, alpha=1.0, beta=0.0, c0=None):
    """C = alpha a b + beta c0 via ngd_gemm_ozaki (a: M x K, b: K x N numpy)."""
    M, K = a.shape
    N = b.shape[1]
    A = torch.as_tensor(np.ascontiguousarray(a), device="cuda")  # K-major rows: A[m K + k]
    B = torch.as_tensor(np.ascontiguousarray(b.T), device="cuda")  # B[n K + k]
    C = torch.as_tensor(np.ascontiguousarray((c0 if c0 is not None else np.zeros((M, N))).T), device="cuda")
    utility_context().call("ngd_gemm_ozaki", M, N, K, float(alpha), _lib.ptr(A), K, _lib.ptr(B), K, float(beta),
                           _lib.ptr(C), M)
    return C.cpu().numpy().T


def dmma(a, b):
    M, K = a.shape
    N = b.shape[1]
    A = torch.as_tensor(np.ascontiguousarray(a.T), device="cuda")  # column-major M x K
    B = torch.as_tensor(np.ascontiguousarray(b.T), device="cuda")
    C = torch.zeros((N, M), dtype=torch.float64, device="cuda")
    utility_context().call("ngd_gemm", 0, 0, M, N, K, 1.0, _lib.ptr(A), M, _lib.ptr(B), K, 0.0, _lib.ptr(C), M)
    return C.cpu().numpy().T


def exact_ld(a, b):
    return (a.astype(np.longdouble) @ b.astype(np.longdouble))


def bound(a, b, ref):
    u = 2.0 ** -52
    aa, bb = np.abs(a), np.abs(b)
    return u * (aa.max(axis=1)[:, None] * bb.sum(axis=0)[None, :] + aa.sum(axis=1)[:, None] * bb.max(axis=0)[None, :]) \
        + u * np.abs(ref.astype(np.float64))


@pytest.mark.parametrize("pair", [0, 1])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (5, 7, 3), (128, 256, 128), (129, 257, 129), (300, 100, 1000),
                                   (600, 1030, 700)])
def test_integer_operands_exact_crt(M, N, K, pair):
    """Both INT8 GEMM forms: one CTA per 128 x 256 tile, and CTA pairs (cta_group::2, 256 x 512 items)."""
    rng = np.random.default_rng(M * 7 + N + K)
    a = rng.integers(-(1 << 20), 1 << 20, size=(M, K)).astype(np.float64)
    b = rng.integers(-(1 << 20), 1 << 20, size=(K, N)).astype(np.float64)
    want = (a.astype(object) @ b.astype(object)).astype(np.float64)  # |C| < 2^50: exact in FP64
    with _lib.option("i8_pair", pair):
        got = oz(a, b)
    assert np.all(np.abs(got - want) <= 2.0 ** -51 * np.abs(want))


@pytest.mark.parametrize("M,N,K,spread", [(200, 300, 2000, 0), (257, 129, 4097, 20), (64, 520, 777, 60),
                                          (40, 30, 140000, 8)])
def test_graded_operands_within_bound(M, N, K, spread):
    """Rows / columns graded over 2^spread, entries over a further 2^12 range; K = 140000 takes two
    K-splits (one exact int32 accumulation holds <= 130944 products)."""
    rng = np.random.default_rng(K + spread)
    a = rng.standard_normal((M, K)) * 2.0 ** rng.uniform(-6, 6, (M, K)) * 2.0 ** rng.uniform(0, spread, (M, 1))
    b = rng.standard_normal((K, N)) * 2.0 ** rng.uniform(-6, 6, (K, N)) * 2.0 ** rng.uniform(-spread, 0, (1, N))
    ref = exact_ld(a, b)
    got = oz(a, b)
    err = np.abs(got - ref.astype(np.float64))
    assert np.all(err <= bound(a, b, ref)), float(np.max(err / bound(a, b, ref)))
    if K < 10000:  # same inputs on the FP64 DMMA GEMM: the emulation is at least as accurate, normwise
        e_dmma = np.linalg.norm((dmma(a, b) - ref).astype(np.float64))
        assert np.linalg.norm(err) <= 4.0 * e_dmma + 1e-300


def test_alpha_beta_zero_rows_and_nonfinite():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((150, 333))
    b = rng.standard_normal((333, 70))
    a[7] = 0.0
    b[:, 3] = 0.0
    c0 = rng.standard_normal((150, 70))
    got = oz(a, b, alpha=-0.75, beta=1.25, c0=c0)
    ref = (-0.75 * exact_ld(a, b) + 1.25 * c0).astype(np.float64)
    assert np.max(np.abs(got - ref)) <= 1e-14 * np.abs(ref).max()
    assert np.array_equal(got[7], 1.25 * c0[7]) and np.array_equal(got[:, 3], 1.25 * c0[:, 3])
    a[11, 5] = np.nan
    b[9, 4] = np.inf
    got = oz(a, b)
    assert np.all(np.isnan(got[11])) and np.all(np.isnan(got[:, 4]))
    mask = np.ones_like(got, dtype=bool)
    mask[11] = False
    mask[:, 4] = False
    assert np.all(np.isfinite(got[mask]))


CONFIGS = {
    "c2": ((2, 64, 64, 64, 1), "sin2d", 4096, 512, 300),
    "c3": ((5, 128, 128, 128, 1), "sinsum", 16384, 4096, 500),
    "c4": ((2, 256, 256, 256, 1), "lap", 65536, 0, 512),
    "c5": ((10, 256, 256, 256, 256, 1), "gauss", 131072, 16384, 1000),
}


def make(name):
    widths, kind, nint, nbnd, ell = CONFIGS[name]
    top = ngd.MlpTopology(widths)
    if kind == "sin2d":
        prob = ngd.Poisson2D(top)
    elif kind == "lap":
        prob = ngd.LaplacianStack(top)
    else:
        prob = ngd.PoissonND(top, kind)
    quad = prob.sample_quadrature(nint, nbnd, 0)
    return prob, quad, ngd.init(top, 0).values, ell


@pytest.mark.parametrize("name,pair", [("c2", 0), ("c2", 1), ("c3", 0), ("c3", 1), ("c4", 1), ("c5", 1)])
def test_sketch_engines_agree_full_size(name, pair):
    """Y = G Omega at the config's full size and rank: INT8 (Ozaki) engine vs FP64 DMMA engine."""
    prob, quad, theta, ell = make(name)
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    p = gop.dim
    om = torch.randn(p, ell, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    om = torch.linalg.qr(om)[0] if name != "c5" else om / np.sqrt(p)
    with _lib.option("sketch_gemm", 0):
        y0 = gop.matmat(om)
    with _lib.option("sketch_gemm", 1), _lib.option("i8_pair", pair):
        y1 = gop.matmat(om)
        y2 = gop.matmat(om)
    assert torch.equal(y1, y2)  # deterministic
    rel = (torch.linalg.norm(y1 - y0, dim=0) / torch.linalg.norm(y0, dim=0)).max().item()
    print(f"{name}: max column rel diff INT8 vs DMMA {rel:.3e}")
    assert rel <= 1e-13


@pytest.mark.parametrize("name,ncols", [("c2", 4), ("c3", 4)])
def test_int8_sketch_against_oracle(name, ncols):
    from oracle import ngd_oracle as O

    widths, kind, nint, nbnd, _ = CONFIGS[name]
    prob, quad, theta, _ = make(name)
    oprob = O.PoissonProblem(widths, kind=kind)
    oq = O.Quadrature(quad.interior_points, quad.interior_weights, quad.boundary_points, quad.boundary_weights)
    om = np.linalg.qr(np.random.default_rng(10).standard_normal((len(theta), ncols)), mode="reduced")[0]
    gop = ngd.GramianOperator.from_problem(prob, theta, quad)
    with _lib.option("sketch_gemm", 1):
        got = gop.matmat(om)
    want = O.GramianOracle(oprob, theta, oq).matmat(om)
    for j in range(ncols):
        assert np.linalg.norm(got[:, j] - want[:, j]) <= 1e-10 * np.linalg.norm(want[:, j]), j
