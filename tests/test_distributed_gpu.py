"""The slab decomposition (paper_2005_03246_b200.distributed) with the real device engine on
one GPU: the ranks are threads and the collectives host-side rendezvous (tests/thread_dist.py),
so the routing, boundary duplication, per-slab CUDA pipelines (incl. the partitioned / grouped
KDE and its weighted carry planes) and the fix-up kernels all run on the device.  Each rank's
slab must equal the single-GPU result: ECDF counts bit-exactly, the KDE to 1e-9."""

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb
from paper_2005_03246_b200 import distributed as fdist

from thread_dist import ThreadDist

REL_KDE = 1e-9


def _run(world, x, w, knots, h, monkeypatch):
    import torch

    td = ThreadDist(world)
    monkeypatch.setattr(fdist, "_dist", lambda: td)
    grid = fcb.RectilinearGrid.from_knots(knots)
    d = x.shape[1]

    def rank_fn(r):
        torch.cuda.set_device(0)
        sl = slice(r, None, world)
        sw = fcb.validate_sample(x[sl], w[sl])
        su = fcb.validate_sample(x[sl])
        kde = fdist.kde_fastsum_slab(sw, grid, fcb.laplacian(), fcb.Bandwidth.diag(h))
        ecdf = fdist.ecdf_fastsum_slab(su, grid, fcb.DeltaVector((1, -1) + (1,) * (d - 2)),
                                       scaled=False)
        return (kde.metadata["slab"], kde.values.cpu().numpy(), ecdf.values.cpu().numpy())

    return td.run(rank_fn), grid


def _assemble(parts, idx, shape):
    full = np.zeros(shape)
    for p in parts:
        lo, hi = p[0]
        full[:, lo:hi] = p[idx].reshape((shape[0], hi - lo) + tuple(shape[2:]))
    return full


CASES = {
    # d = 2: per-term pipeline with epilogue plane capture
    "d2": dict(n=20000, m=(37, 29), h=(0.3, 0.2)),
    # d = 3 / 4, >= 2^20 points per rank: partitioned grouped KDE (kz = 2 with slab planes)
    "d3": dict(n=3_300_000, m=(320, 12, 64), h=(0.3, 0.2, 0.25)),
    "d4": dict(n=3_300_000, m=(40, 24, 16, 32), h=(0.3, 0.2, 0.5, 0.4)),
}


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", sorted(CASES))
def test_slab_pipeline_on_device_matches_single_gpu(case, world, monkeypatch):
    cfg = CASES[case]
    rng = np.random.default_rng(7 + world)
    d = len(cfg["m"])
    x = rng.uniform(-1, 1, (cfg["n"], d))
    knots = [np.linspace(-0.95, 0.95, m) for m in cfg["m"]]
    x[: cfg["n"] // 7, 1] = rng.choice(knots[1], cfg["n"] // 7)  # points on slab boundaries
    w = rng.exponential(1.0, cfg["n"])
    parts, grid = _run(world, x, w, knots, cfg["h"], monkeypatch)
    shape = grid.shape
    ref = fcb.kde_fastsum(fcb.validate_sample(x, w), grid, fcb.laplacian(),
                          fcb.Bandwidth.diag(cfg["h"])).values
    ref = np.asarray(ref.cpu() if hasattr(ref, "cpu") else ref).reshape(shape)
    got = _assemble(parts, 1, shape)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err < REL_KDE, err
    e_ref = fcb.ecdf_fastsum(fcb.validate_sample(x), grid, fcb.DeltaVector((1, -1) + (1,) * (d - 2)),
                             scaled=False).values
    e_ref = np.asarray(e_ref.cpu() if hasattr(e_ref, "cpu") else e_ref).reshape(shape)
    np.testing.assert_array_equal(_assemble(parts, 2, shape), e_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_points_query_shards_on_device(world, monkeypatch):
    """At-points query sharding with the device kernels: each thread-rank evaluates its chunks
    of the dimension-1 rank order, the SUM gather reproduces the single-GPU numerators, the
    Nadaraya-Watson ratio and the strict-dominance ECDF bit for bit."""
    import torch
    import workloads as wl

    td = ThreadDist(world)
    monkeypatch.setattr(fdist, "_dist", lambda: td)
    w = wl.cfg4(1_000_000)
    y = w.extra["y"]
    bw = fcb.Bandwidth.diag(w.h)
    s = fcb.validate_sample(w.points)
    sy = fcb.validate_sample(w.points, np.abs(y))

    def rank_fn(r):
        torch.cuda.set_device(0)
        num = fdist.kde_numerators_sharded(s, [None, y], bw)
        own = fdist.kde_numerators_sharded(s, [None], bw, gather=False)[0]
        nw = fdist.kernel_regression_sharded(s, y, fcb.laplacian(), bw).values
        ec = fdist.ecdf_dnc_sharded(sy).values
        return num, own, nw, ec

    parts = td.run(rank_fn)
    ref = fcb.kde_numerators(s, [None, y], bw)
    scale = fcb.kde_numerators(s, [None, np.abs(y)], bw)  # |y|-weighted scale for the numerator
    ref_ec = fcb.ecdf_dnc(sy).values
    # the coarse histograms sum in shared-memory atomics (run-to-run order), so repeated calls
    # agree to rounding, not bitwise
    for num, _, nw, ec in parts:
        assert np.max(np.abs(num[0] - ref[0]) / scale[0]) <= 1e-12
        assert np.max(np.abs(num[1] - ref[1]) / scale[1]) <= 1e-12
        assert np.max(np.abs(nw - ref[1] / ref[0]) * ref[0] / scale[1]) <= 1e-11
        assert np.max(np.abs(ec - ref_ec) / ref_ec.max()) <= 1e-12
    owned = np.stack([p[1] != 0 for p in parts])
    assert np.all(owned.sum(axis=0) == 1)
    assert np.max(np.abs(sum(p[1] for p in parts) - ref[0]) / ref[0]) <= 1e-12
