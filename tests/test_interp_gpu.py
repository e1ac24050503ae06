"""multilinear_interp (interp.py:24-75) on the device: bit-exact against the reference's own
outputs (goldens) and the oracle; the behaviours of the reference's test_interp.py."""

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb

pytestmark = pytest.mark.gpu


def _grid(knots):
    return fcb.RectilinearGrid.from_knots([np.asarray(z, dtype=float) for z in knots])


def _grid_result(knots, fn):
    g = _grid(knots)
    return g, fcb.EvalResult(np.array([fn(z) for z in g.lattice()]), "grid")


def test_interp_golden(small_golden):
    g = small_golden
    for d in (1, 2, 3):
        key = f"interp.{d}"
        grid = _grid(g.knots(key))
        r = fcb.multilinear_interp(grid, fcb.EvalResult(g[key + ".vals"], "grid"), g[key + ".q"])
        np.testing.assert_array_equal(r.values, g[key + ".out"])
        assert r.metadata["clamp_count"] == int(g[key + ".clamp"])
    x = g["interp.ecdf.x"]
    grid = _grid(g.knots("interp.ecdf"))
    vals = fcb.ecdf_fastsum(fcb.validate_sample(x), grid)
    np.testing.assert_array_equal(fcb.multilinear_interp(grid, vals, x).values, g["interp.ecdf.out"])


def test_interp_kats():
    g, vals = _grid_result([[0.0, 1.0]], lambda z: z[0])
    assert fcb.multilinear_interp(g, vals, [[0.5]]).values[0] == 0.5
    out = fcb.multilinear_interp(g, vals, [[-3.0], [0.5], [7.0]])
    np.testing.assert_array_equal(out.values, [0.0, 0.5, 1.0])
    assert out.metadata["clamp_count"] == 2
    rng = np.random.default_rng(2)
    knots = [np.sort(rng.standard_normal(5)), np.sort(rng.standard_normal(4))]
    g = _grid(knots)
    raw = rng.standard_normal(g.size)
    np.testing.assert_array_equal(
        fcb.multilinear_interp(g, fcb.EvalResult(raw, "grid"), g.lattice()).values, raw)
    g, vals = _grid_result([[0.0, 1.0], [0.0, 1.0]], lambda z: 2 * z[0] + 3 * z[1])
    assert np.isclose(fcb.multilinear_interp(g, vals, [[0.25, 0.75]]).values[0], 2.75)
    knots = [np.sort(rng.uniform(-1, 1, 4)) for _ in range(3)]
    g, vals = _grid_result(knots, lambda z: 1.5 * z[0] - 0.5 * z[1] + 2 * z[2])
    q = rng.uniform([k[0] for k in knots], [k[-1] for k in knots], (30, 3))
    np.testing.assert_allclose(fcb.multilinear_interp(g, vals, q).values,
                               1.5 * q[:, 0] - 0.5 * q[:, 1] + 2 * q[:, 2], atol=1e-14)
    knots = np.sort(rng.standard_normal(12))
    g = _grid([knots])
    q = np.sort(rng.uniform(knots[0], knots[-1], 200)).reshape(-1, 1)
    out = fcb.multilinear_interp(g, fcb.EvalResult(np.sort(rng.random(12)), "grid"), q)
    assert np.all(np.diff(out.values) >= 0)


@pytest.mark.parametrize("d", [2, 4])
def test_interp_vs_oracle_large(d, oracle):
    rng = np.random.default_rng(60 + d)
    m = {2: (300, 177), 4: (9, 14, 11, 6)}[d]
    knots = [np.sort(rng.uniform(-2, 2, k)) for k in m]
    if d == 2:
        knots[0] = np.linspace(-2, 2, m[0])  # uniform axis: the mesh-guess path
    vals = rng.standard_normal(int(np.prod(m)))
    q = rng.uniform(-2.2, 2.2, (500_000, d))
    q[:1000, 0] = rng.choice(knots[0], 1000)  # queries on knots
    r = fcb.multilinear_interp(_grid(knots), fcb.EvalResult(vals, "grid"), q)
    ref, cc = oracle.multilinear_interp(knots, vals, q)
    np.testing.assert_array_equal(r.values, ref)
    assert r.metadata["clamp_count"] == cc


def test_interp_device_tensors():
    import torch

    g, vals = _grid_result([[0.0, 1.0, 3.0]], lambda z: z[0] ** 2)
    q = torch.tensor([[0.5], [2.0]], dtype=torch.float64, device="cuda")
    r = fcb.multilinear_interp(g, vals, q)
    assert r.values.is_cuda
    np.testing.assert_array_equal(r.values.cpu().numpy(), [0.5, 5.0])
