"""GPU parity of the at-points path: ranking, generalized ECDF / ESF at the points with ties
(rank lattice and rank-space dominance routes), ecdf_dnc, kde_dnc, kernel regression."""

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb
from conftest import cfg_golden

pytestmark = pytest.mark.gpu

THREE = [[0.2, 0.7], [0.5, 0.1], [0.9, 0.9]]


def rel_err(got, ref, scale=None):
    got, ref = np.asarray(got), np.asarray(ref)
    s = np.abs(ref) if scale is None else np.asarray(scale)
    s = np.maximum(s, np.finfo(float).tiny)
    return float(np.max(np.abs(got - ref) / s)) if ref.size else 0.0


# ---- ecdf_dnc (dnc.py:531-561; reference tests test_dnc.py:23-72) -----------------------

def test_ecdf_dnc_kats(small_golden):
    s = fcb.validate_sample(THREE)
    np.testing.assert_array_equal(fcb.ecdf_dnc(s).values, small_golden["kat.dnc"])
    np.testing.assert_array_equal(fcb.ecdf_dnc(s, include_self=True).values,
                                  small_golden["kat.dnc_self"])
    s1 = fcb.validate_sample([[0.3, 0.4]])
    assert fcb.ecdf_dnc(s1).values[0] == 0.0
    assert fcb.ecdf_dnc(s1, include_self=True).values[0] == 1.0
    with pytest.raises(fcb.TieError, match="dimension"):
        fcb.ecdf_dnc(fcb.validate_sample([[1.0, 2.0], [1.0, 3.0]]))


def test_ecdf_dnc_golden_bit_exact(small_golden):
    g = small_golden
    for d in (1, 2, 3):
        for seed in range(4):
            key = f"dnc.{d}.{seed}"
            s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
            np.testing.assert_array_equal(fcb.ecdf_dnc(s, scaled=False).values, g[key + ".out"])
            np.testing.assert_array_equal(fcb.ecdf_dnc(s, include_self=True).values,
                                          g[key + ".self"])


@pytest.mark.parametrize("n", [1, 2, 33, 4095, 4097, 20_000, 300_001])
def test_ecdf_dnc_vs_oracle_2d(n, oracle):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 2))
    w = rng.integers(1, 5, n).astype(float)
    got = fcb.ecdf_dnc(fcb.validate_sample(x, w), scaled=False).values
    np.testing.assert_array_equal(got, oracle.ecdf_dnc(x, w, scaled=False))
    got = fcb.ecdf_dnc(fcb.validate_sample(x)).values
    np.testing.assert_array_equal(got, oracle.ecdf_dnc(x, None))


def test_ecdf_dnc_permutation_invariance():
    rng = np.random.default_rng(17)
    pts = rng.standard_normal((2000, 2))
    w = rng.uniform(0.5, 2.0, 2000)
    perm = rng.permutation(2000)
    a = fcb.ecdf_dnc(fcb.validate_sample(pts, w)).values
    b = fcb.ecdf_dnc(fcb.validate_sample(pts[perm], w[perm])).values
    assert rel_err(a[perm], b) <= 1e-12


# ---- generalized ECDF / ESF at the points with ties -------------------------------------

def test_points_with_ties_golden(small_golden):
    g = small_golden
    for d in (1, 2, 3):
        for seed in range(3):
            key = f"pts.{d}.{seed}"
            s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
            for code in range(1 << d):
                dv = fcb.DeltaVector.from_code(code, d)
                got = fcb.ecdf_at_points(s, dv).values
                assert rel_err(got, g[f"{key}.ecdf.{code}"]) <= 1e-12
            assert rel_err(fcb.esf_at_points(s).values, g[key + ".esf"]) <= 1e-12


def test_points_dominance_route_with_ties(oracle):
    """Distinct-level product above the lattice budget forces the rank-space dominance kernel
    with tie-aware thresholds."""
    oracle.set_threads(0)
    rng = np.random.default_rng(42)
    n = 1_500_000
    x = np.floor(rng.random((n, 2)) * 6000) / 6000  # ties in both dims, 3.6e7 level pairs
    y = rng.random(n)
    s = fcb.validate_sample(x, y)
    q = rng.integers(0, n, 1500)
    for delta in [(1, 1), (1, -1), (-1, 1), (-1, -1)]:
        got = fcb.ecdf_at_points(s, fcb.DeltaVector(delta)).values[q]
        ref = oracle.ecdf_naive(x, y, x[q], delta)
        assert rel_err(got, ref) <= 1e-12, delta
    got = fcb.esf_at_points(s).values[q]
    assert rel_err(got, oracle.esf_naive(x, y, x[q])) <= 1e-12
    cnt = fcb.ecdf_at_points(fcb.validate_sample(x), fcb.DeltaVector((1, -1)), scaled=False).values[q]
    np.testing.assert_array_equal(cnt, oracle.ecdf_naive(x, None, x[q], (1, -1), scaled=False))


def test_cfg2_full(oracle, cfg_meta):
    import workloads as wl

    w = wl.cfg2()
    s = fcb.validate_sample(w.points, w.weights)
    ecdf = fcb.ecdf_at_points(s, fcb.DeltaVector(w.delta)).values
    esf = fcb.esf_at_points(s).values
    ref = oracle.ecdf_at_points(w.points, w.weights, w.delta)
    assert rel_err(ecdf, ref) <= 1e-12
    assert rel_err(esf, oracle.esf_at_points(w.points, w.weights)) <= 1e-12
    gold = cfg_golden("cfg2")
    meta = cfg_meta["cfg2"]
    assert meta["input_sha"] == wl.digest(w.points), "config-2 input differs from the golden's"
    assert meta["weights_sha"] == wl.digest(w.weights)
    idx = gold["idx"]
    assert rel_err(ecdf[idx], gold["ecdf"]) <= 1e-12
    assert rel_err(esf[idx], gold["esf"]) <= 1e-12
    assert rel_err(ecdf[idx[:1000]], gold["naive_ecdf"]) <= 1e-12
    assert rel_err(esf[idx[:1000]], gold["naive_esf"]) <= 1e-12
    # unit weights: exact integer counts
    cnt = fcb.ecdf_at_points(fcb.validate_sample(w.points), fcb.DeltaVector(w.delta), scaled=False).values
    np.testing.assert_array_equal(cnt, oracle.ecdf_at_points(w.points, None, w.delta, scaled=False))
    # both outputs from one ranking (fp64 atomics in the lattice scatter: run-to-run rounding)
    e2, s2 = fcb.ecdf_esf_at_points(s, fcb.DeltaVector(w.delta))
    assert rel_err(e2.values, ecdf) <= 1e-14
    assert rel_err(s2.values, esf) <= 1e-14


@pytest.mark.parametrize("case", ["lattice_d3", "dominance_d2", "d1"])
def test_ecdf_esf_at_points_routes(case, oracle):
    """The shared-ranking pair on every route: rank lattice (d = 3, ties), dominance (d = 2
    with too many levels for the lattice budget) and d = 1 (prefix and suffix from one sort)."""
    rng = np.random.default_rng(23)
    if case == "lattice_d3":
        x = np.floor(rng.random((20_000, 3)) * 17) / 17
        delta = (1, -1, 1)
    elif case == "dominance_d2":
        x = np.floor(rng.random((300_000, 2)) * 1e5) / 1e5  # ~1e10 level pairs > budget
        delta = (-1, 1)
    else:
        x = np.floor(rng.random((50_000, 1)) * 999) / 999
        delta = (-1,)
    y = rng.random(x.shape[0])
    s = fcb.validate_sample(x, y)
    e, f = fcb.ecdf_esf_at_points(s, fcb.DeltaVector(delta))
    q = rng.integers(0, x.shape[0], 400)
    assert rel_err(e.values[q], oracle.ecdf_naive(x, y, x[q], delta)) <= 1e-12
    assert rel_err(f.values[q], oracle.esf_naive(x, y, x[q])) <= 1e-12
    assert rel_err(e.values, fcb.ecdf_at_points(s, fcb.DeltaVector(delta)).values) <= 1e-14


# ---- kde_dnc (dnc.py:635-690; reference tests test_dnc.py:163-189) ---------------------

def test_kde_dnc_kats():
    s = fcb.validate_sample([[0.0], [1.0]])
    v = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag([1.0])).values
    np.testing.assert_allclose(v, 0.25 * (1 + np.exp(-1.0)), rtol=1e-15)
    s = fcb.validate_sample([[0.4, -0.2]], [3.0])
    v = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag([0.5, 0.5])).values
    np.testing.assert_allclose(v[0], 3.0 * 0.25 / 0.25, rtol=1e-15)
    with pytest.raises(fcb.ParameterError):
        fcb.kde_dnc(fcb.validate_sample([[0.0], [1.0]]), fcb.uniform(), fcb.Bandwidth.diag([1.0]))
    with pytest.raises(fcb.OverflowGuardError, match="dimension 0"):
        fcb.kde_dnc(fcb.validate_sample([[0.0], [700.0]]), fcb.laplacian(), fcb.Bandwidth.diag([1.0]))
    with pytest.raises(fcb.TieError):
        fcb.kde_dnc(fcb.validate_sample([[0.0, 1.0], [0.0, 2.0]]), fcb.laplacian(),
                    fcb.Bandwidth.diag([1.0, 1.0]))


def test_kde_dnc_golden(small_golden):
    g = small_golden
    for d in (1, 2, 3):
        key = f"kdednc.{d}"
        s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
        got = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag(g[key + ".h"])).values
        assert rel_err(got, g[key + ".out"]) <= 1e-9
        assert np.max(np.abs(got - g[key + ".naive"])) <= 1e-13  # reference bound


def test_kde_dnc_matern32_golden(small_golden):
    """matern32-additive at the points (dnc.py:659-685) vs the reference's own output."""
    g = small_golden
    for d in (1, 2, 3):
        key = f"kdednc.{d}"
        s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
        got = fcb.kde_dnc(s, fcb.matern32_additive(), fcb.Bandwidth.diag(g[key + ".h"])).values
        assert rel_err(got, g[key + ".mat"]) <= 1e-9
        assert np.max(np.abs(got - g[key + ".matnaive"])) <= 1e-13


@pytest.mark.parametrize("n", [7, 5000, 300_001])
def test_kde_dnc_matern32_vs_oracle_signed(n, oracle):
    rng = np.random.default_rng(3000 + n)
    x = rng.standard_normal((n, 2))
    w = rng.standard_normal(n)
    h = [0.25, 0.4]
    got = fcb.kde_dnc(fcb.validate_sample(x, w), fcb.matern32_additive(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_dnc_matern32(x, w, h)
    absk = oracle.kde_dnc_matern32(x, np.abs(w), h)
    assert rel_err(got, ref, absk) <= 1e-9
    x1 = rng.standard_normal((n, 1))  # d = 1: prefix / suffix channels
    got = fcb.kde_dnc(fcb.validate_sample(x1, w), fcb.matern32_additive(), fcb.Bandwidth.diag([0.3])).values
    assert rel_err(got, oracle.kde_dnc_matern32(x1, w, [0.3]),
                   oracle.kde_dnc_matern32(x1, np.abs(w), [0.3])) <= 1e-9


@pytest.mark.parametrize("n", [5, 4096, 9000, 250_000])
def test_kde_dnc_vs_oracle_signed(n, oracle):
    rng = np.random.default_rng(1000 + n)
    x = rng.standard_normal((n, 2))
    w = rng.standard_normal(n)  # signed weights: compare on the |w| KDE scale
    h = [0.3, 0.2]
    s = fcb.validate_sample(x, w)
    got = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_dnc_laplacian(x, w, h)
    absk = oracle.kde_dnc_laplacian(x, np.abs(w), h)
    assert rel_err(got, ref, absk) <= 1e-9


def _check_cfg4(w, golden_name, cfg_meta):
    """kde_numerators / kde_dnc / kernel_regression at the points of a config-4 workload vs the
    reference's own kde_dnc outputs on its seeded subset (dnc.py:635-690): density <= 1e-9
    relative, regression numerator <= 1e-9 on the |y|-KDE scale, Nadaraya-Watson ratio within
    the bound those two imply.  The input digests must match the golden's (no silent skip)."""
    import workloads as wl

    meta = cfg_meta[golden_name]
    assert meta["input_sha"] == wl.digest(w.points), "config-4 input differs from the golden's"
    y = w.extra["y"]
    assert meta["y_sha"] == wl.digest(y), "config-4 response differs from the golden's"
    gold = cfg_golden(golden_name)
    idx = gold["idx"]
    s = fcb.validate_sample(w.points)
    bw = fcb.Bandwidth.diag(w.h)
    num = fcb.kde_numerators(s, [None, y], bw)
    assert rel_err(num[0][idx], gold["density"]) <= 1e-9
    assert rel_err(num[1][idx], gold["regression"], gold["abs_regression"]) <= 1e-9
    dens = fcb.kde_dnc(s, fcb.laplacian(), bw).values
    assert rel_err(dens[idx], gold["density"]) <= 1e-9
    assert rel_err(num[0], dens) <= 1e-12
    nw = fcb.kernel_regression(s, y, fcb.laplacian(), bw).values
    ref_nw = gold["regression"] / gold["density"]
    bound = 2e-9 * gold["abs_regression"] / gold["density"]
    assert np.all(np.abs(nw[idx] - ref_nw) <= bound)
    return num


def test_cfg4_1e6_and_regression(cfg_meta):
    import workloads as wl

    _check_cfg4(wl.cfg4(1_000_000), "cfg4_1e6", cfg_meta)


@pytest.mark.slow
def test_cfg4_full(cfg_meta):
    """BASELINE config 4 at its size (N = 1e7) against the reference's N = 1e7 run."""
    import workloads as wl

    w = wl.cfg4()
    num = _check_cfg4(w, "cfg4", cfg_meta)
    assert np.all(num[0] > 0)


@pytest.mark.slow
def test_cfg4_3e7_two_vectors(oracle):
    """N = 3e7 with two weight vectors: coarse rows (7,325 blocks x 2 channels = 117 KB) exceed
    one shared-memory segment, so the row histogram runs in segments (no N ceiling below the
    device budget).  Checked on a seeded subset of queries against the direct O(N) sum
    (naive.py's Laplacian kernel), density relative and the regression numerator on the
    |y|-weighted scale."""
    import workloads as wl

    oracle.set_threads(0)
    w = wl.cfg4(30_000_000)
    y = w.extra["y"]
    s = fcb.validate_sample(w.points)
    num = fcb.kde_numerators(s, [None, y], fcb.Bandwidth.diag(w.h))
    q = np.random.default_rng(17).integers(0, w.n, 96)
    dens = oracle.kde_naive_laplacian(w.points, None, w.points[q], w.h)
    reg = oracle.kde_naive_laplacian(w.points, y, w.points[q], w.h)
    absreg = oracle.kde_naive_laplacian(w.points, np.abs(y), w.points[q], w.h)
    assert rel_err(num[0][q], dens) <= 1e-9
    assert rel_err(num[1][q], reg, absreg) <= 1e-9


def test_dominance_size_guard():
    """A d = 2 problem whose coarse grid would exceed the device budget is refused up front with
    ParameterError (never the O(N^2) fallback)."""
    from paper_2005_03246_b200 import _lib

    with pytest.raises(fcb.ParameterError, match="coarse grid"):
        _lib.call_ws("fcg_dnc_ecdf", None, 400_000_000, 2, None, 0, 1, None)


def test_d3_brute_paths(oracle):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3000, 3))
    w = rng.uniform(0.5, 2, 3000)
    s = fcb.validate_sample(x, w)
    got = fcb.ecdf_dnc(s, scaled=False).values
    ref = oracle.ecdf_naive(x, w, x, (-1, -1, -1), scaled=False)
    assert rel_err(got, ref) <= 1e-12
    got = fcb.kde_dnc(s, fcb.laplacian(), fcb.Bandwidth.diag([0.4, 0.5, 0.6])).values
    ref = oracle.kde_naive_laplacian(x, w, x, [0.4, 0.5, 0.6])
    assert rel_err(got, ref) <= 1e-9
    xt = np.floor(rng.random((50_000, 3)) * 300) / 300  # 2.7e7 level triples > budget -> brute
    got = fcb.ecdf_at_points(fcb.validate_sample(xt), fcb.DeltaVector((1, -1, 1)), scaled=False).values
    q = rng.integers(0, 50_000, 500)
    np.testing.assert_array_equal(got[q], oracle.ecdf_naive(xt, None, xt[q], (1, -1, 1), scaled=False))


def test_distinct_flags_device():
    import torch

    x = torch.tensor([[1.0, 3.0], [1.0, 4.0], [2.0, -0.0], [5.0, 0.0]], device="cuda")
    assert fcb.validate_sample(x).distinct_by_dim == (False, False)  # -0.0 == +0.0
    x = torch.tensor([[1.0, 3.0], [2.0, 4.0]], device="cuda")
    assert fcb.validate_sample(x).distinct_by_dim == (True, True)


# ---- ranking subsystem (fcg_rank_f64) vs np.argsort(stable) / index_matrix_sorted -------

def _rank_ref(keys):
    k = np.asarray(keys, dtype=np.float64)
    order = np.argsort(k, kind="stable")
    pos = np.empty_like(order)
    pos[order] = np.arange(k.size)
    srt = k[order]
    lower = np.searchsorted(srt, k, side="left")
    upper = np.searchsorted(srt, k, side="right")
    uniq = np.unique(k)
    dense = np.searchsorted(uniq, k, side="left")
    return order, pos, lower, upper, dense, uniq


@pytest.mark.parametrize("case", ["ties1024", "continuous", "signed_zero", "tiny"])
def test_rank_f64_vs_stable_argsort(case, oracle):
    """order == np.argsort(kind="stable") (dnc.py:523-528); dense / dense+1 equal the
    reference's sorted-scan bins with knots = the distinct values (histogram.py:122-133,
    index_matrix_sorted) for delta = +1 / -1; lower / upper are the < / <= counts under ties;
    -0.0 and +0.0 rank equal."""
    rng = np.random.default_rng(7)
    if case == "ties1024":  # config 2's 1024 quantisation levels, N = 1e6
        keys = np.floor(rng.random(1_000_000) * 1024) / 1024
    elif case == "continuous":
        keys = rng.standard_normal(1_000_000) * 1e3
    elif case == "signed_zero":
        keys = rng.choice([-0.0, 0.0, -1.5, 2.0, np.inf, -np.inf, 1e-300, -1e-300], 100_000)
    else:
        keys = np.array([3.0, -1.0, 3.0, 0.0, -0.0, 7.5])
    order, pos, lower, upper, dense = fcb.rank_f64(keys)
    r_order, r_pos, r_lower, r_upper, r_dense, uniq = _rank_ref(keys)
    np.testing.assert_array_equal(order, r_order)
    np.testing.assert_array_equal(pos, r_pos)
    np.testing.assert_array_equal(lower, r_lower)
    np.testing.assert_array_equal(upper, r_upper)
    np.testing.assert_array_equal(dense, r_dense)
    # the reference's own rank oracle: sorted-scan bins with knots = the distinct values
    if case != "signed_zero":  # from_knots needs finite strictly increasing knots
        col = keys.reshape(-1, 1)
        np.testing.assert_array_equal(dense, oracle.index_matrix_sorted(col, [uniq], [1])[0])
        np.testing.assert_array_equal(dense + 1, oracle.index_matrix_sorted(col, [uniq], [-1])[0])
    if case == "signed_zero":
        z = keys == 0.0
        assert np.unique(dense[z]).size == 1 and np.unique(lower[z]).size == 1


def test_rank_f64_device_tensor_and_empty():
    import torch

    k = torch.tensor([2.0, 1.0, 2.0, -3.0], dtype=torch.float64, device="cuda")
    order, pos, lower, upper, dense = fcb.rank_f64(k)
    assert order.is_cuda and order.dtype == torch.int32
    assert order.cpu().tolist() == [3, 1, 0, 2]
    assert upper.cpu().tolist() == [4, 2, 4, 1]
    assert dense.cpu().tolist() == [2, 1, 2, 0]
    outs = fcb.rank_f64(np.empty(0))
    assert all(o.size == 0 for o in outs)


# ---- kde_terms_dnc / rank_tiebreak (dnc.py:502-520, 608-632; reference tests test_dnc.py:95-146)

def _brute_delta_table(points, psi):
    n, d = points.shape
    out = np.zeros((n, 1 << d))
    for code in range(1 << d):
        signs = fcb.DeltaVector.from_code(code, d).as_array()
        sp = points * signs
        for j in range(n):
            out[j, code] = psi[np.all(sp < sp[j], axis=1), code].sum()
    return out


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_kde_terms_matches_brute_force(d):
    rng = np.random.default_rng(50 + d)
    n = 120
    pts = rng.standard_normal((n, d))
    w = rng.uniform(0.5, 2.0, n)
    h = rng.uniform(0.6, 1.4, d)
    monomial = (int(rng.integers(0, d)), int(rng.integers(0, d)), 1, 0)
    tt = fcb.kde_terms_dnc(fcb.validate_sample(pts, w), fcb.Bandwidth.diag(h), monomial)
    l, m, p, q = monomial
    psi = np.empty((n, 1 << d))
    for code in range(1 << d):
        signs = fcb.DeltaVector.from_code(code, d).as_array()
        psi[:, code] = w * pts[:, l] ** p * pts[:, m] ** q * np.exp(pts @ (signs / h))
    np.testing.assert_array_equal(tt.psi, psi)
    expected = _brute_delta_table(pts, psi)
    assert np.max(np.abs(tt.table - expected)) <= 1e-13 * max(1.0, np.max(np.abs(expected)))
    assert tt.delta_for_column(1) == fcb.DeltaVector.from_code(1, d)


def test_kde_terms_fingerprint_and_guards():
    rng = np.random.default_rng(81)
    pts = rng.standard_normal((3000, 3))
    w = rng.standard_normal(3000)  # signed weights: any double-counted pair breaks equality
    tt = fcb.kde_terms_dnc(fcb.validate_sample(pts, w), fcb.Bandwidth.diag(np.full(3, 5.0)))
    q = rng.integers(0, 3000, 50)
    exp_q = np.zeros((50, 8))
    for code in range(8):
        sp = pts * fcb.DeltaVector.from_code(code, 3).as_array()
        for a, j in enumerate(q):
            exp_q[a, code] = tt.psi[np.all(sp < sp[j], axis=1), code].sum()
    assert np.max(np.abs(tt.table[q] - exp_q)) <= 1e-12
    single = fcb.kde_terms_dnc(fcb.validate_sample([[0.3, 0.4]]), fcb.Bandwidth.diag([1.0, 1.0]))
    np.testing.assert_array_equal(single.table, np.zeros((1, 4)))
    with pytest.raises(fcb.ParameterError):
        fcb.kde_terms_dnc(fcb.validate_sample([[0.0], [1.0]]), fcb.Bandwidth.diag([1.0]), (2, 0, 1, 0))
    with pytest.raises(fcb.TieError):
        fcb.kde_terms_dnc(fcb.validate_sample([[0.0, 1.0], [0.0, 2.0]]), fcb.Bandwidth.diag([1.0, 1.0]))


def test_rank_tiebreak_matches_stable_argsort():
    rng = np.random.default_rng(9)
    pts = np.floor(rng.random((5000, 3)) * 17)
    ref = np.empty_like(pts)
    for k in range(3):
        ref[np.argsort(pts[:, k], kind="stable"), k] = np.arange(5000)
    np.testing.assert_array_equal(fcb.rank_tiebreak(pts), ref)
    # ranks restore distinct coordinates: the strict ECDF then counts index-ordered ties
    assert fcb.validate_sample(fcb.rank_tiebreak(pts)).distinct


@pytest.mark.parametrize("case", ["one_top_half", "short_runs", "mixed"])
def test_split_key_ranking_paths(case, oracle):
    """The positions-only ranking sorts the keys' top 32 bits and orders runs of equal top halves
    by the low halves; coordinates that share their top halves by the thousand must fall back to
    the full-key sort.  Checked through ecdf_dnc (bit-exact counts) on d = 2."""
    rng = np.random.default_rng(5)
    n = 60_000
    if case == "one_top_half":   # every coordinate in [1, 1 + 2^-21): one run of n members
        x = 1.0 + rng.permutation(n)[:, None] * 2.0 ** -50 + np.array([[0.0, 2.0 ** -51]])
        x = np.stack([x[:, 0], 1.0 + rng.permutation(n) * 2.0 ** -50], axis=1)
    elif case == "short_runs":   # runs of ~8 members sharing 32 top bits
        base = rng.standard_normal((n // 8, 2)).astype(np.float32).astype(np.float64)
        x = np.repeat(base, 8, axis=0) * (1.0 + rng.permutation(n)[:, None] * 2.0 ** -45)
    else:
        x = rng.standard_normal((n, 2))
        x[: n // 2, 0] = 3.0 + rng.permutation(n // 2) * 2.0 ** -48
    s = fcb.validate_sample(x)
    got = fcb.ecdf_dnc(s, scaled=False).values
    np.testing.assert_array_equal(got, oracle.ecdf_dnc(x, None, scaled=False))


@pytest.mark.parametrize("case", ["diagonal", "anti_diagonal", "cluster"])
def test_level2_correlated_layouts(case, oracle):
    """Rank-correlated inputs put a block's points into one chunk (long runs of the query's own
    chunk in the block solver: the neighbour walk gives way to the searches) and crowd slot /
    rank cells; checked bit-exactly through ecdf_dnc and to 1e-9 through the signed KDE."""
    rng = np.random.default_rng(21)
    n = 70_001
    t = rng.random(n)
    if case == "diagonal":
        x = np.stack([t, t + 1e-7 * rng.standard_normal(n)], axis=1)
    elif case == "anti_diagonal":
        x = np.stack([t, -t + 1e-7 * rng.standard_normal(n)], axis=1)
    else:
        x = rng.standard_normal((n, 2))
        x[: n // 2] = 0.3 + 1e-4 * rng.standard_normal((n // 2, 2))
    w = rng.integers(1, 7, n).astype(float)
    got = fcb.ecdf_dnc(fcb.validate_sample(x, w), scaled=False).values
    np.testing.assert_array_equal(got, oracle.ecdf_dnc(x, w, scaled=False))
    ws = rng.standard_normal(n)
    h = [0.05, 0.07]
    got = fcb.kde_dnc(fcb.validate_sample(x, ws), fcb.laplacian(), fcb.Bandwidth.diag(h)).values
    q = rng.integers(0, n, 400)
    ref = oracle.kde_naive_laplacian(x, ws, x[q], h)
    scale = oracle.kde_naive_laplacian(x, np.abs(ws), x[q], h)
    assert rel_err(got[q], ref, scale) <= 1e-9


def test_level2_direct_vs_masked_passes_random(monkeypatch):
    """The direct level-2 kernels against the per-code masked passes they replaced
    (FCG_LEVEL2=codes) on random sizes (ragged last groups), layouts and weights: counts
    bit-exact, KDE numerators (one and two weight vectors, signed) to 1e-11 of the |w| scale."""
    from paper_2005_03246_b200 import points as pts

    rng = np.random.default_rng(99)
    for trial in range(12):
        n = int(rng.integers(1, 60_000)) if trial else 2049
        x = rng.standard_normal((n, 2))
        if trial % 3 == 1:
            x[: n // 2] = 0.5 + 1e-5 * x[: n // 2]
        elif trial % 3 == 2:
            x[:, 1] = x[:, 0] * (1.0 if trial % 2 else -1.0) + 1e-6 * x[:, 1]
        w = rng.integers(1, 9, n).astype(float)
        y = rng.standard_normal(n)
        h = rng.uniform(0.05, 0.5, 2)
        s = fcb.validate_sample(x, w)
        out = {}
        for mode in ("direct", "codes"):
            if mode == "codes":
                monkeypatch.setenv("FCG_LEVEL2", "codes")
            else:
                monkeypatch.delenv("FCG_LEVEL2", raising=False)
            out[mode] = (fcb.ecdf_dnc(s, scaled=False).values,
                         fcb.kde_dnc(fcb.validate_sample(x, y), fcb.laplacian(),
                                     fcb.Bandwidth.diag(h)).values,
                         [np.asarray(v) for v in pts.kde_numerators(
                             fcb.validate_sample(x), [None, y], fcb.Bandwidth.diag(h))],
                         fcb.kde_dnc(fcb.validate_sample(x, np.abs(y)), fcb.laplacian(),
                                     fcb.Bandwidth.diag(h)).values)
        monkeypatch.delenv("FCG_LEVEL2", raising=False)
        a, b = out["direct"], out["codes"]
        np.testing.assert_array_equal(a[0], b[0], err_msg=f"trial {trial} n={n}")
        scale = np.maximum(b[3], np.finfo(float).tiny)
        assert np.max(np.abs(a[1] - b[1]) / scale) <= 1e-11, (trial, n)
        assert rel_err(a[2][0], b[2][0]) <= 1e-11, (trial, n)
        assert np.max(np.abs(a[2][1] - b[2][1]) / scale) <= 1e-11, (trial, n)
