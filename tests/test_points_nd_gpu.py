"""GPU parity of the at-points path for d >= 3: the rank-space coarse-grid +
slab-remainder route of points_nd.cuh against the reference's MergeND recursion
(dnc.py:65-135, 307-410; fixtures tests/golden/nd.npz written by make_golden.py --nd) and against
the oracle's direct sums on larger inputs."""

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb
from conftest import GOLDEN, Golden

pytestmark = pytest.mark.gpu


def rel_err(got, ref, scale=None):
    got, ref = np.asarray(got), np.asarray(ref)
    s = np.abs(ref) if scale is None else np.asarray(scale)
    s = np.maximum(s, np.finfo(float).tiny)
    return float(np.max(np.abs(got - ref) / s)) if ref.size else 0.0


@pytest.fixture(scope="module")
def nd_golden():
    return Golden(GOLDEN / "nd.npz")


@pytest.mark.parametrize("d", [3, 4, 5])
def test_nd_reference_golden(d, nd_golden):
    g, key = nd_golden, f"nd{d}"
    x, w, h = g[key + ".x"], g[key + ".w"], g[key + ".h"]
    s, su = fcb.validate_sample(x, w), fcb.validate_sample(x)
    assert rel_err(fcb.ecdf_dnc(s, scaled=False).values, g[key + ".ecdf_w"],
                   np.maximum(g[key + ".ecdf_w"], 1.0)) <= 1e-12
    # unit weights: counts, bit-exact (also count / N)
    np.testing.assert_array_equal(fcb.ecdf_dnc(su, include_self=True, scaled=False).values,
                                  g[key + ".ecdf_unit_self"])
    np.testing.assert_array_equal(fcb.ecdf_dnc(su).values, g[key + ".ecdf_scaled"])
    bw = fcb.Bandwidth.diag(h)
    assert rel_err(fcb.kde_dnc(s, fcb.laplacian(), bw).values, g[key + ".kde_w"]) <= 1e-9
    assert rel_err(fcb.kde_dnc(su, fcb.laplacian(), bw).values, g[key + ".kde_unit"]) <= 1e-9
    assert rel_err(fcb.kde_dnc(s, fcb.matern32_additive(), bw).values, g[key + ".mat_w"]) <= 1e-9
    if d <= 4:
        tt = fcb.kde_terms_dnc(s, bw, (0, d - 1, 1, 1))
        rows, ref = g[key + ".terms_rows"], g[key + ".terms"]
        scale = np.maximum(np.max(np.abs(ref), axis=0, keepdims=True), 1e-300)
        assert np.max(np.abs(tt.table[rows] - ref) / scale) <= 1e-11


@pytest.mark.parametrize("d,n", [(3, 8192), (3, 8193), (3, 200_000), (4, 60_000), (6, 20_000)])
def test_nd_ecdf_dnc_vs_oracle(d, n, oracle):
    rng = np.random.default_rng(100 * d + n % 97)
    x = rng.standard_normal((n, d))
    w = rng.integers(1, 6, n).astype(float)  # integer weights: exact sums in any order
    q = rng.integers(0, n, 1500)
    got = fcb.ecdf_dnc(fcb.validate_sample(x, w), scaled=False).values
    ref = oracle.ecdf_naive(x, w, x[q], (-1,) * d, scaled=False)
    np.testing.assert_array_equal(got[q], ref)
    got = fcb.ecdf_dnc(fcb.validate_sample(x), include_self=True, scaled=False).values
    ref = oracle.ecdf_naive(x, None, x[q], (-1,) * d, scaled=False) + 1.0
    np.testing.assert_array_equal(got[q], ref)


@pytest.mark.parametrize("case", ["levels300", "skewed_ties", "continuous"])
def test_nd_ecdf_esf_at_points_with_ties(case, oracle):
    """ecdf_at_points / esf_at_points (naive.py:90-114, 210-217 semantics) past the rank-lattice
    budget: mixed deltas, ties, and a dimension with three levels (query buckets of n / 3)."""
    rng = np.random.default_rng(7)
    n = 60_000
    if case == "levels300":
        x = np.floor(rng.random((n, 3)) * 300) / 300
    elif case == "skewed_ties":
        x = rng.standard_normal((n, 3))
        x[:, 0] = rng.integers(0, 3, n)
        x[:, 2] = np.round(x[:, 2], 2)
    else:
        x = rng.standard_normal((n, 4))
    d = x.shape[1]
    w = rng.integers(1, 4, n).astype(float)
    s = fcb.validate_sample(x, w)
    q = rng.integers(0, n, 800)
    for delta in [(1,) * d, (1, -1, 1, -1)[:d], (-1,) * d]:
        got = fcb.ecdf_at_points(s, fcb.DeltaVector(delta), scaled=False).values
        np.testing.assert_array_equal(got[q], oracle.ecdf_naive(x, w, x[q], delta, scaled=False))
    e, f = fcb.ecdf_esf_at_points(fcb.validate_sample(x), fcb.DeltaVector((1,) * d), scaled=False)
    np.testing.assert_array_equal(e.values[q], oracle.ecdf_naive(x, None, x[q], (1,) * d, scaled=False))
    np.testing.assert_array_equal(f.values[q], oracle.esf_naive(x, None, x[q], scaled=False))


@pytest.mark.parametrize("d,n", [(3, 9000), (3, 150_000), (4, 40_000), (5, 16_384)])
def test_nd_kde_dnc_vs_oracle(d, n, oracle):
    rng = np.random.default_rng(d * 1000 + 3)
    x = rng.standard_normal((n, d))
    x[: n // 3] = x[: n // 3] * 0.05 + 1.0  # a dense cluster: most pairs near-field there
    w = rng.standard_normal(n)              # signed weights
    h = rng.uniform(0.15, 0.6, d)
    q = rng.integers(0, n, 600)
    got = fcb.kde_dnc(fcb.validate_sample(x, w), fcb.laplacian(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_naive_laplacian(x, w, x[q], h)
    scale = oracle.kde_naive_laplacian(x, np.abs(w), x[q], h)
    assert rel_err(got[q], ref, scale) <= 1e-9
    # two weight vectors in one pass (density + regression numerator)
    from paper_2005_03246_b200 import points as pts

    y = rng.uniform(-1, 1, n)
    num = pts.kde_numerators(fcb.validate_sample(x), [None, y], fcb.Bandwidth.diag(h))
    num = [np.asarray(v) for v in num]
    ref0 = oracle.kde_naive_laplacian(x, None, x[q], h)
    ref1 = oracle.kde_naive_laplacian(x, y, x[q], h)
    assert rel_err(num[0][q], ref0) <= 1e-9
    assert rel_err(num[1][q], ref1, oracle.kde_naive_laplacian(x, np.abs(y), x[q], h)) <= 1e-9


def test_nd_kde_wide_span(oracle):
    """span / h near the overflow guard (600): exp(+-u) up to e^300 per dimension."""
    rng = np.random.default_rng(11)
    n = 12_000
    x = rng.random((n, 3)) * np.array([590.0, 1.0, 40.0])
    h = np.array([1.0, 0.2, 1.0])
    q = rng.integers(0, n, 400)
    got = fcb.kde_dnc(fcb.validate_sample(x), fcb.laplacian(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_naive_laplacian(x, None, x[q], h)
    assert rel_err(got[q], ref) <= 1e-9


def test_nd_terms_vs_direct(oracle):
    rng = np.random.default_rng(81)
    n, d = 9000, 3
    pts = rng.standard_normal((n, d))
    w = rng.standard_normal(n)
    tt = fcb.kde_terms_dnc(fcb.validate_sample(pts, w), fcb.Bandwidth.diag(np.full(d, 5.0)))
    q = rng.integers(0, n, 60)
    exp_q = np.zeros((60, 8))
    for code in range(8):
        sp = pts * fcb.DeltaVector.from_code(code, d).as_array()
        for a, j in enumerate(q):
            exp_q[a, code] = tt.psi[np.all(sp < sp[j], axis=1), code].sum()
    assert np.max(np.abs(tt.table[q] - exp_q)) <= 1e-11 * np.max(np.abs(exp_q))


@pytest.mark.parametrize("d,n", [(3, 120_000), (4, 30_000)])
def test_nd_kde_dnc_matern32_vs_oracle(d, n, oracle):
    """matern32-additive at the points for d = 3, 4 (dnc.py:659-685): two far-field channels per
    sign code + the table-form near field, against the direct sum on a query subset."""
    rng = np.random.default_rng(900 + d)
    x = rng.standard_normal((n, d))
    x[: n // 4] = x[: n // 4] * 0.03 - 0.5
    w = rng.standard_normal(n)  # signed weights
    h = rng.uniform(0.2, 0.7, d)
    q = rng.integers(0, n, 300)
    got = fcb.kde_dnc(fcb.validate_sample(x, w), fcb.matern32_additive(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_naive_matern32(x, w, x[q], h)
    scale = oracle.kde_naive_matern32(x, np.abs(w), x[q], h)
    assert rel_err(got[q], ref, scale) <= 1e-9


@pytest.mark.slow
def test_nd_large_chunks(oracle):
    """d = 3 at 1.5e6 points: the cost model picks 2048- / 4096-rank chunks (several source
    tiles per chunk, triangular tile ranges); counts bit-exact, KDE to 1e-9, on a query subset."""
    rng = np.random.default_rng(77)
    n, d = 1_500_000, 3
    x = rng.standard_normal((n, d))
    q = rng.integers(0, n, 300)
    got = fcb.ecdf_dnc(fcb.validate_sample(x), scaled=False).values
    np.testing.assert_array_equal(got[q], oracle.ecdf_naive(x, None, x[q], (-1,) * d, scaled=False))
    w = rng.uniform(0.5, 2.0, n)
    h = [0.2, 0.25, 0.3]
    got = fcb.kde_dnc(fcb.validate_sample(x, w), fcb.laplacian(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_naive_laplacian(x, w, x[q], h)
    assert rel_err(got[q], ref) <= 1e-9


def test_nd_route_vs_direct_tiles_random_shapes(monkeypatch):
    """Random shapes, tie patterns, deltas and weights: the rank-space route against the direct
    O(n^2) tiles of the same library (FCG_ND=off), on the device for every query."""
    from paper_2005_03246_b200 import _lib

    rng = np.random.default_rng(2024)
    for trial in range(14):
        d = int(rng.integers(3, 7))
        n = int(rng.integers(8192, 30_000))
        x = rng.standard_normal((n, d))
        mode = trial % 4
        if mode == 1:    # heavy ties in one dimension, light ties in another
            x[:, 0] = rng.integers(0, 5, n)
            x[:, d - 1] = np.round(x[:, d - 1], 1)
        elif mode == 2:  # lattice-valued but too many levels for the rank lattice
            x = np.floor(rng.random((n, d)) * 200) / 200
        elif mode == 3:  # a tight cluster plus outliers
            x[: n // 2] = 1e-3 * x[: n // 2]
        w = rng.integers(1, 9, n).astype(float)
        delta = tuple(int(v) for v in rng.choice([-1, 1], d))
        s = fcb.validate_sample(x, w)
        monkeypatch.delenv("FCG_ND", raising=False)
        _lib.profile_enable(True)
        e1, f1 = fcb.ecdf_esf_at_points(s, fcb.DeltaVector(delta), scaled=False)
        assert "pts_nd_near" in _lib.profile_report()
        monkeypatch.setenv("FCG_ND", "off")
        e0, f0 = fcb.ecdf_esf_at_points(s, fcb.DeltaVector(delta), scaled=False)
        rep = _lib.profile_report()
        _lib.profile_enable(False)
        assert "pts_brute" in rep and "pts_nd_near" not in rep
        np.testing.assert_array_equal(e1.values, e0.values, err_msg=f"trial {trial} d={d} n={n}")
        np.testing.assert_array_equal(f1.values, f0.values, err_msg=f"trial {trial} d={d} n={n}")
        if mode in (0, 3):  # distinct coordinates: the KDE at the points as well
            h = rng.uniform(0.3, 0.9, d)
            monkeypatch.delenv("FCG_ND", raising=False)
            k1 = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag(h)).values
            monkeypatch.setenv("FCG_ND", "off")
            k0 = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag(h)).values
            assert rel_err(k1, k0) <= 1e-10, (trial, d, n)
    monkeypatch.delenv("FCG_ND", raising=False)
