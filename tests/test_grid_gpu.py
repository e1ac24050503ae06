"""GPU parity of the grid path (local sums, directional sweep, grid ECDF / ESF / KDE) against the
golden fixtures produced by the reference and against the pinned oracle."""

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb
from conftest import cfg_golden

pytestmark = pytest.mark.gpu

THREE = [[0.2, 0.7], [0.5, 0.1], [0.9, 0.9]]
REL_F64 = 1e-12   # north_star: weighted fp64 ECDF tolerance
REL_KDE = 1e-9    # north_star: KDE tolerance


def _grid(knots):
    return fcb.RectilinearGrid.from_knots([np.asarray(z, float) for z in knots])


def assert_rel(got, ref, rel):
    got, ref = np.asarray(got), np.asarray(ref)
    assert got.shape == ref.shape
    scale = np.maximum(np.abs(ref), np.finfo(float).tiny)
    err = np.max(np.abs(got - ref) / scale) if ref.size else 0.0
    assert err <= rel, f"max relative error {err:.3e} > {rel:.1e}"


# ---- hand KATs (reference tests test_histogram.py:18-40, test_fastsum.py:52-85) ----------

def test_kat_local_sums(small_golden):
    s = fcb.validate_sample(THREE)
    g = _grid([[0.5], [0.5]])
    np.testing.assert_array_equal(fcb.local_sums_sorted(s, g, fcb.DeltaVector((1, 1))).data,
                                  small_golden["kat.ls_pp"])
    np.testing.assert_array_equal(fcb.local_sums_sorted(s, g, fcb.DeltaVector((-1, 1))).data,
                                  small_golden["kat.ls_mp"])
    t = fcb.local_sums_sorted(s, _grid([[5.0], [0.5]]))
    assert t.data[1].sum() == 0
    np.testing.assert_array_equal(t.data[0], [1.0, 2.0])


def test_kat_ecdf_esf(small_golden):
    s = fcb.validate_sample(THREE)
    g = _grid([[0.5, 0.9], [0.5, 0.9]])
    np.testing.assert_array_equal(fcb.ecdf_fastsum(s, g).values, small_golden["kat.ecdf"])
    np.testing.assert_array_equal(fcb.ecdf_fastsum(s, g, fcb.DeltaVector((-1, -1))).values,
                                  small_golden["kat.ecdf_mm"])
    assert fcb.ecdf_fastsum(s, g, fcb.DeltaVector((-1, -1))).values[0] == 0.0
    np.testing.assert_array_equal(fcb.ecdf_fastsum(s, _grid([[-2, -1], [-2, -1]])).values,
                                  np.zeros(4))
    np.testing.assert_array_equal(fcb.esf_fastsum(s, _grid([[0.4], [0.4]])).values,
                                  small_golden["kat.esf04"])
    assert fcb.esf_fastsum(s, _grid([[2.0], [2.0]])).values[0] == 0.0
    assert fcb.esf_fastsum(s, _grid([[-1.0], [-1.0]])).values[0] == 1.0


def test_uniform_formula_knot_hits():
    # x = 0.5 on knots (0, .5, 1): bin 1 under <=, bin 2 under <; x = -3 -> bin 0
    s = fcb.validate_sample([[0.5], [-3.0]])
    g = _grid([[0.0, 0.5, 1.0]])
    np.testing.assert_array_equal(fcb.local_sums(s, g, fcb.DeltaVector((1,))).data, [1, 1, 0, 0])
    np.testing.assert_array_equal(fcb.local_sums(s, g, fcb.DeltaVector((-1,))).data, [1, 0, 1, 0])


# ---- seeded fixtures ---------------------------------------------------------------------

def test_local_sums_golden_bit_exact(small_golden):
    g = small_golden
    seeds = g.keys("ls.")
    assert len(seeds) == 40
    for seed in seeds:
        key = f"ls.{seed}"
        s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
        grid = _grid(g.knots(key))
        delta = fcb.DeltaVector(tuple(int(v) for v in g[key + ".delta"]))
        np.testing.assert_array_equal(fcb.local_sums(s, grid, delta).data, g[key + ".out"])
        su = fcb.validate_sample(g[key + ".x"])
        cnt = np.bincount(g[key + ".flat"], minlength=int(np.prod([len(z) + 1 for z in g.knots(key)])))
        np.testing.assert_array_equal(fcb.local_sums(su, grid, delta).data.reshape(-1), cnt)


def test_ecdf_fastsum_golden(small_golden):
    g = small_golden
    for d in range(1, 6):
        for seed in range(6):
            key = f"ecdf.{d}.{seed}"
            x, grid = g[key + ".x"], _grid(g.knots(key))
            delta = fcb.DeltaVector(tuple(int(v) for v in g[key + ".delta"]))
            # integer weights: exact
            got = fcb.ecdf_fastsum(fcb.validate_sample(x, g[key + ".w"]), grid, delta, scaled=False)
            np.testing.assert_array_equal(got.values, g[key + ".out"])
            # unit weights: int32 lattice, count / N bitwise
            got = fcb.ecdf_fastsum(fcb.validate_sample(x), grid, delta)
            np.testing.assert_array_equal(got.values, g[key + ".unit"])
            # float weights: tolerance
            sw = fcb.validate_sample(x, g[key + ".wf"])
            assert_rel(fcb.ecdf_fastsum(sw, grid, delta).values, g[key + ".outf"], REL_F64)
            assert_rel(fcb.esf_fastsum(sw, grid).values, g[key + ".esf"], REL_F64)


def test_directional_sweep_golden(small_golden):
    g = small_golden
    for d in range(1, 5):
        t = g[f"sweep.{d}.in"]
        for code in range(1 << d):
            out = fcb.directional_sweep(fcb.LocalSumTensor(t.copy()), fcb.DeltaVector.from_code(code, d))
            assert_rel(out.data, g[f"sweep.{d}.{code}"], 1e-13)
    data = np.arange(6.0).reshape(2, 3)
    t = fcb.LocalSumTensor(data.copy())
    fcb.directional_sweep(t, fcb.DeltaVector((1, 1)))
    np.testing.assert_array_equal(t.data, data)  # input not mutated


def test_kde_fastsum_golden(small_golden):
    g = small_golden
    for d in (1, 2, 3):
        key = f"kde.{d}"
        s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
        grid = _grid(g.knots(key))
        bw = fcb.Bandwidth.diag(g[key + ".h"])
        got = fcb.kde_fastsum(s, grid, fcb.laplacian(), bw).values
        assert_rel(got, g[key + ".fast"], REL_KDE)
        assert np.max(np.abs(got - g[key + ".naive"])) <= 1e-13  # reference bound
        # uniform kernel = signed sum of 2^d ECDFs: zero regions cancel to +-1e-16 in the
        # reference itself, so compare against the field's scale (reference bound: atol 1e-13)
        uni = fcb.kde_fastsum(s, grid, fcb.uniform(), bw).values
        ref = g[key + ".unif"]
        assert np.max(np.abs(uni - ref)) <= 1e-12 * np.max(np.abs(ref))
    s = fcb.validate_sample(g["kdeknots.x"], g["kdeknots.w"])
    got = fcb.kde_fastsum(s, _grid(g.knots("kdeknots")), fcb.laplacian(),
                          fcb.Bandwidth.diag([0.25, 0.4])).values
    assert_rel(got, g["kdeknots.fast"], REL_KDE)


def test_kde_single_point_kats():
    s = fcb.validate_sample([[0.0]])
    v = fcb.kde_fastsum(s, _grid([[-1.0, 1.0]]), fcb.laplacian(), fcb.Bandwidth.diag([1.0])).values
    np.testing.assert_allclose(v, 0.5 * np.exp(-1.0), rtol=1e-15)
    s = fcb.validate_sample([[0.0, 0.0]])
    v = fcb.kde_fastsum(s, _grid([[0.0, 1.0], [0.0, 1.0]]), fcb.laplacian(),
                        fcb.Bandwidth.diag([1.0, 1.0])).values
    assert np.isclose(v[-1], 0.25 * np.exp(-2.0)) and np.isclose(v[0], 0.25)


# ---- errors (reference error contracts) --------------------------------------------------

def test_error_contracts():
    s = fcb.validate_sample([[0.1, 0.2]])
    with pytest.raises(fcb.ParameterError):
        fcb.local_sums_sorted(s, _grid([[0.5]]))
    with pytest.raises(fcb.ParameterError):
        fcb.local_sums_uniform(fcb.validate_sample([[0.5]]), _grid([[0.0, 0.4, 1.0]]))
    rng = np.random.default_rng(3)
    s = fcb.validate_sample(np.column_stack([rng.uniform(0, 1, 50), rng.uniform(0, 700, 50)]))
    g = fcb.build_grid_auto(s, [4, 4])
    with pytest.raises(fcb.OverflowGuardError, match="dimension 1"):
        fcb.kde_fastsum(s, g, fcb.laplacian(), fcb.Bandwidth.diag([1.0, 1.0]))
    with pytest.raises(fcb.ParameterError):
        fcb.kde_fastsum(fcb.validate_sample([[0.0], [1.0]]), _grid([[0.0, 1.0]]), fcb.gaussian(),
                        fcb.Bandwidth.diag([1.0]))
    with pytest.raises(fcb.ParameterError):
        fcb.kde_fastsum(fcb.validate_sample([[0.0, 0.0], [1.0, 1.0]]), _grid([[0, 1], [0, 1]]),
                        fcb.laplacian(), fcb.Bandwidth.full(np.eye(2)))


# ---- random properties vs the oracle -----------------------------------------------------

@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6])
def test_ecdf_vs_oracle_random(d, oracle):
    for seed in range(5):
        rng = np.random.default_rng(7000 + 10 * d + seed)
        n = int(rng.integers(1, 3000))
        x = rng.standard_normal((n, d))
        m = [int(v) for v in rng.integers(1, 40 if d <= 3 else 9, d)]
        knots = [np.sort(rng.uniform(-2.5, 2.5, mk)) for mk in m]
        knots = [np.unique(np.concatenate([z, x[rng.integers(0, n, 2), k]])) for k, z in enumerate(knots)]
        delta = tuple(int(v) for v in rng.choice([-1, 1], d))
        grid = _grid(knots)
        got = fcb.ecdf_fastsum_counts(fcb.validate_sample(x), grid, fcb.DeltaVector(delta))
        ref = oracle.ecdf_fastsum(x, None, knots, delta, scaled=False)
        np.testing.assert_array_equal(got, ref.astype(np.int64))
        got = fcb.esf_fastsum(fcb.validate_sample(x), grid, scaled=False).values
        np.testing.assert_array_equal(got, oracle.esf_fastsum(x, None, knots, scaled=False))


def test_long_axis_chunked_scan(oracle):
    """1-D grid with 200k knots forces the chunked 3-phase scan path."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((300_000, 1))
    knots = [np.linspace(-3, 3, 200_000)]
    w = rng.uniform(0, 1, x.shape[0])
    got = fcb.ecdf_fastsum(fcb.validate_sample(x), _grid(knots), scaled=False).values
    np.testing.assert_array_equal(got, oracle.ecdf_fastsum(x, None, knots, scaled=False))
    got = fcb.ecdf_fastsum(fcb.validate_sample(x, w), _grid(knots)).values
    assert_rel(got, oracle.ecdf_fastsum(x, w, knots), REL_F64)


def test_device_tensor_roundtrip(oracle):
    import torch

    rng = np.random.default_rng(5)
    x = rng.standard_normal((5000, 3))
    knots = [np.linspace(-2, 2, 17)] * 3
    s_dev = fcb.validate_sample(torch.from_numpy(x).cuda())
    res = fcb.ecdf_fastsum(s_dev, _grid(knots), scaled=False)
    assert isinstance(res.values, torch.Tensor) and res.values.is_cuda
    np.testing.assert_array_equal(res.values.cpu().numpy(),
                                  oracle.ecdf_fastsum(x, None, knots, scaled=False))


# ---- full-size configurations ------------------------------------------------------------

def test_cfg1_full_bit_exact(oracle):
    import workloads as wl

    gold = cfg_golden("cfg1")
    w = wl.cfg1()
    s = fcb.validate_sample(w.points)
    grid = _grid(w.knots)
    counts = fcb.ecdf_fastsum_counts(s, grid, fcb.DeltaVector(w.delta))
    ref = oracle.ecdf_fastsum(w.points, None, w.knots, w.delta, scaled=False)
    np.testing.assert_array_equal(counts, ref.astype(np.int64))
    vals = fcb.ecdf_fastsum(s, grid, fcb.DeltaVector(w.delta)).values
    np.testing.assert_array_equal(vals, oracle.ecdf_fastsum(w.points, None, w.knots, w.delta))
    np.testing.assert_array_equal(counts, gold["counts"].astype(np.int64))


@pytest.mark.slow
def test_cfg3_full_bit_exact(oracle, cfg_meta):
    import workloads as wl

    oracle.set_threads(0)
    w = wl.cfg3()
    s = fcb.validate_sample(w.points)
    counts = fcb.ecdf_fastsum_counts(s, _grid(w.knots), fcb.DeltaVector(w.delta))
    meta = cfg_meta["cfg3"]
    assert meta["input_sha"] == wl.digest(w.points), "config-3 input differs from the golden's"
    assert wl.digest(counts) == meta["out_sha_i64"]  # the reference's own output digest
    ref = oracle.ecdf_fastsum(w.points, None, w.knots, w.delta, scaled=False)
    np.testing.assert_array_equal(counts, ref.astype(np.int64))
    # size-independent property: last corner == number of points inside the grid box
    inside = np.all(w.points <= 4.0, axis=1).sum()
    assert counts[-1] == inside


# ---- plane-partitioned pipeline (d >= 3, n >= 2^20) ----------------------------------------

# planes >= 2 x 148 SMs so the partitioned route is taken; (300, 700, 300) needs 9 row blocks
@pytest.mark.parametrize("dims,delta", [((300, 53, 61), (1, -1, 1)), ((40, 9, 150, 77), (-1, 1, 1, -1)),
                                        ((300, 700, 300), (1, 1, -1)), ((12, 10, 5, 7, 9), (1, 1, 1, 1, 1)),
                                        # d = 4 with 16 | columns: the fused axis-1 + axis-0 final
                                        ((37, 11, 24, 40), (1, -1, -1, 1)), ((30, 13, 16, 64), (-1, 1, 1, -1))])
def test_partitioned_ecdf_esf_vs_oracle(dims, delta, oracle):
    oracle.set_threads(0)
    d = len(dims)
    rng = np.random.default_rng(sum(dims))
    n = 1_200_000
    x = rng.standard_normal((n, d))
    knots = [np.sort(rng.uniform(-2.2, 2.2, m)) for m in dims]
    knots = [np.unique(np.concatenate([z[:-2], x[:2, k]])) for k, z in enumerate(knots)]
    grid = _grid(knots)
    got = fcb.ecdf_fastsum_counts(fcb.validate_sample(x), grid, fcb.DeltaVector(delta))
    ref = oracle.ecdf_fastsum(x, None, knots, delta, scaled=False)
    np.testing.assert_array_equal(got, ref.astype(np.int64))
    got = fcb.esf_fastsum(fcb.validate_sample(x), grid).values
    np.testing.assert_array_equal(got, oracle.esf_fastsum(x, None, knots))


@pytest.mark.parametrize("dims", [(300, 53, 61), (30, 13, 16, 64)])
def test_partitioned_ecdf_clustered(dims, oracle):
    """90% of the points in one cell (one bucket holding most keys), the rest spread out."""
    oracle.set_threads(0)
    d = len(dims)
    rng = np.random.default_rng(3 * sum(dims))
    n = 1_200_000
    x = rng.standard_normal((n, d))
    k = int(0.9 * n)
    x[:k] = 0.31 + 1e-5 * rng.random((k, d))
    knots = [np.linspace(-2.2, 2.2, m) for m in dims]
    got = fcb.ecdf_fastsum_counts(fcb.validate_sample(x), _grid(knots), fcb.DeltaVector((1,) * d))
    ref = oracle.ecdf_fastsum(x, None, knots, (1,) * d, scaled=False)
    np.testing.assert_array_equal(got, ref.astype(np.int64))


def test_kde_matern32_golden(small_golden):
    """matern32-additive grid KDE (fastsum.py:170-181) against the reference's own output."""
    g = small_golden
    for d in (1, 2, 3):
        key = f"kde.{d}"
        s = fcb.validate_sample(g[key + ".x"], g[key + ".w"])
        got = fcb.kde_fastsum(s, _grid(g.knots(key)), fcb.matern32_additive(),
                              fcb.Bandwidth.diag(g[key + ".h"])).values
        assert_rel(got, g[key + ".mat"], REL_KDE)
        assert np.max(np.abs(got - g[key + ".matnaive"])) <= 1e-13


@pytest.mark.parametrize("d", [2, 4])
def test_kde_matern32_vs_oracle(d, oracle):
    rng = np.random.default_rng(40 + d)
    n = 30000
    x = rng.standard_normal((n, d))
    w = rng.exponential(1.0, n)
    m = {2: (61, 47), 4: (9, 12, 7, 10)}[d]
    knots = [np.linspace(-2.5, 2.2, k) for k in m]
    knots[0] = np.unique(np.concatenate([knots[0], x[:2, 0]]))  # knot hits
    h = rng.uniform(0.15, 0.5, d)
    got = fcb.kde_fastsum(fcb.validate_sample(x, w), _grid(knots), fcb.matern32_additive(),
                          fcb.Bandwidth.diag(h)).values
    assert_rel(got, oracle.kde_fastsum_matern32(x, w, knots, h), REL_KDE)


@pytest.mark.parametrize("dims", [(320, 17, 40), (20, 16, 33, 21), (300, 40, 128), (300, 40, 64),
                                  (24, 20, 16, 128), (19, 21, 8, 64)])
def test_partitioned_kde_vs_oracle(dims, oracle):
    """Partitioned KDE paths vs the oracle: per-group plane kernel (W = 40, 21), all-groups
    plane kernel for every (E, NG) instance (W = 64, 128 at d = 3 and 4; blocks of <= 8 rows
    take the unrolled walk, taller ones the look-ahead walk) with the fused axis-1 + axis-0
    final (d = 4, 16 | columns)."""
    oracle.set_threads(0)
    d = len(dims)
    rng = np.random.default_rng(7 * sum(dims))
    n = 1_100_000
    x = rng.uniform(-1, 1, (n, d))
    w = rng.exponential(1.0, n)
    knots = [np.linspace(-1.1, 0.9, m) for m in dims]
    knots[0] = np.unique(np.concatenate([knots[0], x[:3, 0]]))  # knot hits
    h = rng.uniform(0.05, 0.3, d)
    got = fcb.kde_fastsum(fcb.validate_sample(x, w), _grid(knots), fcb.laplacian(),
                          fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_fastsum_laplacian(x, w, knots, h)
    assert_rel(got, ref, REL_KDE)


@pytest.mark.parametrize("dims", [(24, 20, 16, 128), (300, 40, 128)])
def test_partitioned_kde_clustered(dims, oracle):
    """Most points in one cell (runs of equal keys far longer than a window, one coarse segment
    holding most of the records, most segments empty) plus a uniform background."""
    oracle.set_threads(0)
    d = len(dims)
    rng = np.random.default_rng(13 * sum(dims))
    n = 1_100_000
    x = rng.uniform(-1, 1, (n, d))
    k = int(0.9 * n)
    x[:k] = 0.0123 + 1e-4 * rng.random((k, d))
    w = rng.exponential(1.0, n)
    knots = [np.linspace(-1.1, 0.9, m) for m in dims]
    h = rng.uniform(0.1, 0.3, d)
    got = fcb.kde_fastsum(fcb.validate_sample(x, w), _grid(knots), fcb.laplacian(),
                          fcb.Bandwidth.diag(h)).values
    assert_rel(got, oracle.kde_fastsum_laplacian(x, w, knots, h), REL_KDE)


def _kde_ex(x, w, knots, h, centre, u_bound):
    import torch
    from paper_2005_03246_b200 import _lib

    grid = _grid(knots)
    xd = _lib.to_device_f64(x)
    wd = _lib.to_device_f64(w)
    kn = _lib.device_knots(grid)
    out = torch.empty(grid.size, dtype=torch.float64, device=xd.device)
    _lib.call_ws("fcg_kde_grid_laplacian_ex", _lib.ptr(xd), x.shape[0], x.shape[1], _lib.ptr(wd),
                 _lib.ptr(kn), _lib.i64_array(grid.shape), _lib.f64_array(h),
                 None if centre is None else _lib.f64_array(centre), float(x.shape[0]), u_bound,
                 None, _lib.ptr(out))
    return out.cpu().numpy()


@pytest.mark.parametrize("dims", [(24, 20, 16, 64), (300, 40, 128), (9, 11)])
def test_kde_auto_centre_matches_explicit(dims):
    """centre == NULL: the hull taken by the binning pass gives the caller-side midrange of
    fastsum.py:118-129 exactly, so the partitioned densities are bit-identical."""
    d = len(dims)
    rng = np.random.default_rng(11 * sum(dims))
    n = 1_100_000
    x = rng.uniform(-1, 1.3, (n, d))
    w = rng.exponential(1.0, n)
    knots = [np.linspace(-1.4, 0.9, m) for m in dims]
    h = rng.uniform(0.05, 0.3, d)
    lo = np.minimum(x.min(0), [z[0] for z in knots])
    hi = np.maximum(x.max(0), [z[-1] for z in knots])
    c = 0.5 * (lo + hi)
    ub = float(np.sum((hi - lo) / (2 * h))) * 1.000001
    got, ref = _kde_ex(x, w, knots, h, None, -1.0), _kde_ex(x, w, knots, h, c, ub)
    if d >= 3:  # the partitioned pipeline is deterministic
        np.testing.assert_array_equal(got, ref)
    else:  # fp64 atomics: run-to-run summation order
        assert_rel(got, ref, 1e-13)


def test_partitioned_kde_raw_records(oracle):
    """sum_k span_k / (2 h_k) > 600 with every span_k / h_k <= 600: the auto-centre plan assumed
    factored records, the run falls back to per-term exponentials on the group kernel."""
    oracle.set_threads(0)
    dims = (24, 20, 16, 64)
    rng = np.random.default_rng(5)
    n = 1_100_000
    x = rng.uniform(-1, 1, (n, 4))
    w = rng.exponential(1.0, n)
    knots = [np.linspace(-1.0, 1.0, m) for m in dims]
    h = np.full(4, 0.006)  # span / h = 333 per axis, bound 667
    got = fcb.kde_fastsum(fcb.validate_sample(x, w), _grid(knots), fcb.laplacian(),
                          fcb.Bandwidth.diag(h)).values
    ref = oracle.kde_fastsum_laplacian(x, w, knots, h)
    assert_rel(got, ref, REL_KDE)


def test_partitioned_kde_overflow_guard():
    rng = np.random.default_rng(6)
    n = 1_100_000
    x = rng.uniform(0, 1, (n, 4))
    x[:, 2] *= 700.0
    knots = [np.linspace(0.0, 1.0, 64)] * 4
    with pytest.raises(fcb.OverflowGuardError, match="dimension 2: span/bandwidth = "):
        fcb.kde_fastsum(fcb.validate_sample(x), _grid(knots), fcb.laplacian(),
                        fcb.Bandwidth.diag([1.0] * 4))


@pytest.mark.slow
def test_cfg5_full(cfg_meta):
    """Config 5 at full size (N = 1e8, 128^4): the ECDF's int64 counts must equal the digest of
    the reference's own output and its seeded subset; the KDE is checked on the reference's
    seeded subset to 1e-9.  The input digests must match the goldens' (no silent skip)."""
    import workloads as wl

    w = wl.cfg5()
    grid = _grid(w.knots)
    meta_a, meta_b = cfg_meta["cfg5a"], cfg_meta["cfg5b"]
    assert meta_a["input_sha"] == wl.digest(w.points), "config-5 points differ from the golden's"
    assert meta_b["input_sha"] == wl.digest(w.points)
    assert meta_b["y_sha"] == wl.digest(w.extra["y"]), "config-5 weights differ from the golden's"
    counts = fcb.ecdf_fastsum_counts(fcb.validate_sample(w.points), grid, fcb.DeltaVector(w.delta))
    # size-independent properties: monotone along the last axis, corner = N (all points inside)
    c4 = counts.reshape(128, 128, 128, 128)
    assert counts[-1] == w.n
    assert np.all(np.diff(c4[::17, ::13, ::11, :], axis=-1) >= 0)
    assert wl.digest(counts) == meta_a["out_sha_i64"]
    gold_a = cfg_golden("cfg5a")
    np.testing.assert_array_equal(counts[gold_a["idx"]], gold_a["vals"].astype(np.int64))
    del counts, c4
    vals = fcb.kde_fastsum(fcb.Sample(w.points, w.extra["y"], None, False), grid, fcb.laplacian(),
                           fcb.Bandwidth.diag(w.h)).values
    gold_b = cfg_golden("cfg5b")
    assert_rel(vals[gold_b["idx"]], gold_b["vals"], REL_KDE)
    assert np.all(vals > 0)


@pytest.mark.parametrize("seed", range(24))
def test_random_grid_configs_vs_oracle(seed, oracle):
    """Seeded sweep over dimension, grid shape (uniform and irregular knots, knot hits), delta,
    weights and sample size: grid ECDF counts bit-exact, weighted ECDF / ESF to 1e-12, the
    Laplacian KDE to 1e-9."""
    oracle.set_threads(0)
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(1, 5))
    n = int(rng.choice([1, 2, 7, 500, 20_000]))
    x = rng.standard_normal((n, d)) * rng.uniform(0.5, 2.0)
    knots = []
    for _ in range(d):
        m = int(rng.integers(1, 40))
        z = np.linspace(-2.5, 2.5, m) if rng.random() < 0.5 else np.sort(rng.uniform(-3, 3, m))
        z = np.unique(np.concatenate([z, x[: int(rng.integers(0, 3)), len(knots)]]))
        knots.append(z)
    delta = tuple(int(v) for v in rng.choice([-1, 1], d))
    grid = _grid(knots)
    got = fcb.ecdf_fastsum_counts(fcb.validate_sample(x), grid, fcb.DeltaVector(delta))
    np.testing.assert_array_equal(got, oracle.ecdf_fastsum(x, None, knots, delta, scaled=False)
                                  .astype(np.int64))
    w = rng.uniform(0.1, 2.0, n)
    s = fcb.validate_sample(x, w)
    assert_rel(fcb.ecdf_fastsum(s, grid, fcb.DeltaVector(delta)).values,
               oracle.ecdf_fastsum(x, w, knots, delta), 1e-12)
    assert_rel(fcb.esf_fastsum(s, grid).values, oracle.esf_fastsum(x, w, knots), 1e-12)
    lo = np.minimum(x.min(0), [z[0] for z in knots])
    hi = np.maximum(x.max(0), [z[-1] for z in knots])
    h = np.maximum((hi - lo) / rng.uniform(5, 40, d), 1e-3)
    assert_rel(fcb.kde_fastsum(s, grid, fcb.laplacian(), fcb.Bandwidth.diag(h)).values,
               oracle.kde_fastsum_laplacian(x, w, knots, h), REL_KDE)


@pytest.mark.parametrize("dims", [(300, 5, 256), (320, 3, 512), (4, 80, 7, 256)])
def test_fused_plane_scan_vs_oracle(dims, oracle):
    """Lattices whose last axis is a multiple of 256 with >= 2 x 148 planes take the fused
    in-plane (axes d-1, d-2) scan: int32 counts (both delta signs on the in-plane axes), fp64
    weighted ESF (suffix sums) and the per-term Laplacian KDE."""
    oracle.set_threads(0)
    d = len(dims)
    rng = np.random.default_rng(77 + sum(dims))
    n = 60_000
    x = rng.standard_normal((n, d))
    w = rng.uniform(0.1, 2.0, n)
    knots = [np.linspace(-2.6, 2.6, m) for m in dims]
    grid = _grid(knots)
    for delta in [(1,) * d, (1,) * (d - 2) + (-1, 1), (1,) * (d - 2) + (1, -1)]:
        got = fcb.ecdf_fastsum_counts(fcb.validate_sample(x), grid, fcb.DeltaVector(delta))
        np.testing.assert_array_equal(got, oracle.ecdf_fastsum(x, None, knots, delta, scaled=False)
                                      .astype(np.int64))
    s = fcb.validate_sample(x, w)
    assert_rel(fcb.esf_fastsum(s, grid).values, oracle.esf_fastsum(x, w, knots), 1e-12)
    h = np.full(d, 0.4)
    assert_rel(fcb.kde_fastsum(s, grid, fcb.laplacian(), fcb.Bandwidth.diag(h)).values,
               oracle.kde_fastsum_laplacian(x, w, knots, h), REL_KDE)


def test_bench_ladder_small(tmp_path):
    """The reference-schema ladder drives the device functions (cli.py:163-196)."""
    from paper_2005_03246_b200 import harness

    rows = harness.bench_ladder("ecdf", ["fastsum", "dnc"], [2], [2000], repeats=2,
                                out=tmp_path / "l.csv")
    assert len(rows) == 4 and all(r[5] > 0 for r in rows)
    rows = harness.bench_ladder("kde", ["fastsum", "dnc"], [2], [500], repeats=1)
    assert len(rows) == 2
    assert (tmp_path / "l.csv").read_text().startswith("task,method,dim,n,repeat,seconds\n")


@pytest.mark.parametrize("m", [(256, 256), (3, 1000), (17, 300), (1000, 5), (1024, 1024), (1, 7)])
def test_small2d_one_launch_vs_oracle(m, oracle):
    """The one-launch small 2-D pipeline (lattices <= 2^20 cells) on every shape class: rows
    longer than 256 (generic row loop), fewer rows than axis-0 chunks, uneven chunks, the 2^20
    boundary; counts, int64 counts, weighted sums, every delta and the ESF."""
    oracle.set_threads(0)
    rng = np.random.default_rng(sum(m))
    n = 40_000
    x = rng.standard_normal((n, 2))
    knots = [np.sort(rng.uniform(-2.5, 2.5, mk)) if mk > 1 else np.array([0.1]) for mk in m]
    knots[0] = np.unique(np.concatenate([knots[0], x[:2, 0]]))  # knot hits
    grid = _grid(knots)
    w = rng.uniform(0.1, 2.0, n)
    for delta in [(1, 1), (-1, 1), (1, -1), (-1, -1)]:
        dv = fcb.DeltaVector(delta)
        ref = oracle.ecdf_fastsum(x, None, knots, delta, scaled=False)
        np.testing.assert_array_equal(fcb.ecdf_fastsum_counts(fcb.validate_sample(x), grid, dv),
                                      ref.astype(np.int64))
        np.testing.assert_array_equal(fcb.ecdf_fastsum(fcb.validate_sample(x), grid, dv).values,
                                      ref / n)  # count / N: the IEEE quotient bit for bit
        assert_rel(fcb.ecdf_fastsum(fcb.validate_sample(x, w), grid, dv).values,
                   oracle.ecdf_fastsum(x, w, knots, delta), REL_F64)
    np.testing.assert_array_equal(fcb.esf_fastsum(fcb.validate_sample(x), grid, scaled=False).values,
                                  oracle.esf_fastsum(x, None, knots, scaled=False))


@pytest.mark.parametrize("nbytes", [8, 8 << 20, (32 << 20) + 8, (100 << 20) + 24, 3 * (32 << 20)])
def test_staged_copies_roundtrip(nbytes):
    """fcg_copy_h2d / fcg_copy_d2h (the numpy path): exact round trips across chunk boundaries
    (32 MB chunks, ring of 4) and for small sizes."""
    import ctypes as C

    import torch
    from paper_2005_03246_b200 import _lib

    n = nbytes // 8
    a = np.random.default_rng(n).standard_normal(n)
    lib = _lib.load_library()
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(lib.fcg_copy_h2d(C.c_void_p(d.data_ptr()), a.ctypes.data_as(C.c_void_p), a.nbytes,
                                _lib.stream_handle()), "fcg_copy_h2d")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d.cpu().numpy(), a)
    d.mul_(2.0)
    out = np.empty_like(a)
    _lib.check(lib.fcg_copy_d2h(out.ctypes.data_as(C.c_void_p), C.c_void_p(d.data_ptr()), a.nbytes,
                                _lib.stream_handle()), "fcg_copy_d2h")
    np.testing.assert_array_equal(out, 2.0 * a)
    # the package paths: numpy in -> device, device -> numpy out
    np.testing.assert_array_equal(_lib.to_host(_lib.to_device_f64(a)), a)
