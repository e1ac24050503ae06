"""Pin the oracle (oracle/, a CPU restatement of the reference) against fixtures produced by the
reference package itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import cfg_golden


def test_local_sums_and_flat_bins(small_golden, oracle):
    g = small_golden
    for seed in g.keys("ls."):
        key = f"ls.{seed}"
        x, w, delta = g[key + ".x"], g[key + ".w"], tuple(g[key + ".delta"])
        knots = g.knots(key)
        np.testing.assert_array_equal(oracle.flat_bin_indices(x, knots, delta), g[key + ".flat"])
        np.testing.assert_array_equal(oracle.local_sums(x, w, knots, delta), g[key + ".out"])


def test_ecdf_fastsum_bit_exact(small_golden, oracle):
    g = small_golden
    n_checked = 0
    for d in range(1, 6):
        for seed in range(6):
            key = f"ecdf.{d}.{seed}"
            x, knots, delta = g[key + ".x"], g.knots(key), tuple(g[key + ".delta"])
            np.testing.assert_array_equal(
                oracle.ecdf_fastsum(x, g[key + ".w"], knots, delta, scaled=False), g[key + ".out"])
            np.testing.assert_array_equal(
                oracle.ecdf_fastsum(x, None, knots, delta, scaled=True), g[key + ".unit"])
            np.testing.assert_array_equal(
                oracle.ecdf_fastsum(x, g[key + ".wf"], knots, delta), g[key + ".outf"])
            np.testing.assert_allclose(oracle.esf_fastsum(x, g[key + ".wf"], knots),
                                       g[key + ".esf"], rtol=0, atol=1e-15)
            n_checked += 1
    assert n_checked == 30


def test_directional_sweep(small_golden, oracle):
    g = small_golden
    for d in range(1, 5):
        t = g[f"sweep.{d}.in"]
        for code in range(1 << d):
            signs = tuple(-1 if (code >> k) & 1 else 1 for k in range(d))
            np.testing.assert_array_equal(oracle.cumsum_directional(t, signs), g[f"sweep.{d}.{code}"])


def test_kde_fastsum_laplacian(small_golden, oracle):
    g = small_golden
    for d in (1, 2, 3):
        key = f"kde.{d}"
        got = oracle.kde_fastsum_laplacian(g[key + ".x"], g[key + ".w"], g.knots(key), g[key + ".h"])
        np.testing.assert_allclose(got, g[key + ".fast"], rtol=1e-13, atol=0)
        naive = oracle.kde_naive_laplacian(g[key + ".x"], g[key + ".w"],
                                           _lattice(g.knots(key)), g[key + ".h"])
        np.testing.assert_allclose(naive, g[key + ".naive"], rtol=1e-14, atol=0)
    got = oracle.kde_fastsum_laplacian(g["kdeknots.x"], g["kdeknots.w"], g.knots("kdeknots"),
                                       [0.25, 0.4])
    np.testing.assert_allclose(got, g["kdeknots.fast"], rtol=1e-13, atol=0)


def _lattice(knots):
    axes = np.meshgrid(*knots, indexing="ij")
    return np.stack([a.reshape(-1) for a in axes], axis=1)


def test_naive(small_golden, oracle):
    g = small_golden
    x, w, q = g["naive.x"], g["naive.w"], g["naive.q"]
    for code in range(4):
        signs = tuple(-1 if (code >> k) & 1 else 1 for k in range(2))
        np.testing.assert_array_equal(oracle.ecdf_naive(x, w, q, signs), g[f"naive.ecdf.{code}"])
    np.testing.assert_array_equal(oracle.esf_naive(x, w, q), g["naive.esf"])
    np.testing.assert_array_equal(oracle.kde_naive_laplacian(x, w, q, [0.4, 0.6]), g["naive.kde"])


def test_dnc(small_golden, oracle):
    g = small_golden
    for d in (1, 2):
        for seed in range(4):
            key = f"dnc.{d}.{seed}"
            x, w = g[key + ".x"], g[key + ".w"]
            np.testing.assert_array_equal(oracle.ecdf_dnc(x, w, scaled=False), g[key + ".out"])
            np.testing.assert_array_equal(oracle.ecdf_dnc(x, w, include_self=True), g[key + ".self"])
    for d in (1, 2):
        key = f"kdednc.{d}"
        got = oracle.kde_dnc_laplacian(g[key + ".x"], g[key + ".w"], g[key + ".h"])
        np.testing.assert_allclose(got, g[key + ".out"], rtol=1e-13, atol=0)
    tab = oracle.run_all_delta(g["kdednc.2.x"], g["kdednc.2.psi"], 1)
    np.testing.assert_allclose(tab, g["kdednc.2.table"], rtol=1e-13, atol=1e-300)
    tab = oracle.run_all_delta(g["finger.x"], g["finger.psi"], 1)
    np.testing.assert_allclose(tab, g["finger.table"], rtol=0, atol=1e-12)


def test_points_with_ties(small_golden, oracle):
    g = small_golden
    for d in (1, 2, 3):
        for seed in range(3):
            key = f"pts.{d}.{seed}"
            x, w = g[key + ".x"], g[key + ".w"]
            for code in range(1 << d):
                signs = tuple(-1 if (code >> k) & 1 else 1 for k in range(d))
                np.testing.assert_allclose(oracle.ecdf_at_points(x, w, signs), g[f"{key}.ecdf.{code}"],
                                           rtol=1e-12, atol=1e-15)
                np.testing.assert_array_equal(oracle.ecdf_naive(x, w, x, signs), g[f"{key}.ecdf.{code}"])
            np.testing.assert_allclose(oracle.esf_at_points(x, w), g[key + ".esf"], rtol=1e-12,
                                       atol=1e-15)


def test_cfg1_full(oracle):
    gold = cfg_golden("cfg1")
    if gold is None:
        pytest.skip("cfg1 golden not generated")
    import workloads as wl

    w = wl.cfg1()
    got = oracle.ecdf_fastsum(w.points, None, w.knots, w.delta, scaled=False)
    np.testing.assert_array_equal(got, gold["counts"].astype(np.float64))


def test_matern32_additive(small_golden, oracle):
    """matern32-additive through the Laplacian terms (fastsum.py:170-181, dnc.py:659-685),
    pinned to the reference's own fast and naive outputs."""
    g = small_golden
    for d in (1, 2, 3):
        key = f"kde.{d}"
        got = oracle.kde_fastsum_matern32(g[key + ".x"], g[key + ".w"], g.knots(key), g[key + ".h"])
        np.testing.assert_allclose(got, g[key + ".mat"], rtol=1e-13, atol=0)
        np.testing.assert_allclose(got, g[key + ".matnaive"], rtol=1e-12, atol=0)
    for d in (1, 2):
        key = f"kdednc.{d}"
        got = oracle.kde_dnc_matern32(g[key + ".x"], g[key + ".w"], g[key + ".h"])
        np.testing.assert_allclose(got, g[key + ".mat"], rtol=1e-13, atol=0)
        np.testing.assert_allclose(got, g[key + ".matnaive"], rtol=1e-12, atol=0)


def test_multilinear_interp(small_golden, oracle):
    g = small_golden
    for d in (1, 2, 3):
        key = f"interp.{d}"
        out, cc = oracle.multilinear_interp(g.knots(key), g[key + ".vals"], g[key + ".q"])
        np.testing.assert_array_equal(out, g[key + ".out"])
        assert cc == int(g[key + ".clamp"])


def test_nd_direct_sums_vs_reference_recursion(oracle):
    """The oracle's direct at-points sums (naive.py:187-248 restated) against the reference's
    MergeND recursion for d = 3..5 (nd.npz, dnc.py:65-135, 307-410, 531-690): pins the checker
    that the d >= 3 device route is compared with on larger inputs."""
    from conftest import GOLDEN, Golden

    g = Golden(GOLDEN / "nd.npz")
    for d in (3, 4, 5):
        key = f"nd{d}"
        x, w, h = g[key + ".x"], g[key + ".w"], g[key + ".h"]
        got = oracle.ecdf_naive(x, w, x, (-1,) * d, scaled=False)
        np.testing.assert_allclose(got, g[key + ".ecdf_w"], rtol=1e-12, atol=1e-9)
        got = oracle.ecdf_naive(x, None, x, (-1,) * d, scaled=False) + 1.0
        np.testing.assert_array_equal(got, g[key + ".ecdf_unit_self"])
        got = oracle.kde_naive_laplacian(x, w, x, h)
        np.testing.assert_allclose(got, g[key + ".kde_w"], rtol=1e-10, atol=0)
        sub = np.arange(0, x.shape[0], 37)
        got = oracle.kde_naive_matern32(x, w, x[sub], h)
        np.testing.assert_allclose(got, g[key + ".mat_w"][sub], rtol=1e-10, atol=0)
