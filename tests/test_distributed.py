"""Multi-process (gloo, CPU) tests of the slab decomposition along axis 1: routing, the
boundary duplicates of the KDE, the carry-plane all-gather and the final fix-ups are exactly
the package's code; local steps run on the oracle (tests/dist_engine.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2005_03246_b200 as fcb
from paper_2005_03246_b200 import distributed as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _data(seed, n, d):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, d))
    knots = [np.linspace(-0.9, 0.9, m) for m in (5, 11, 6, 4)[:d]]
    # put a block of points exactly on axis-1 knots (slab boundaries included)
    x[: n // 5, 1] = rng.choice(knots[1], n // 5)
    w = rng.exponential(1.0, n)
    return x, w, knots


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_engine import OracleEngine

        eng = OracleEngine()
        res = {}
        for d in (2, 3, 4):
            x, w, knots = _data(100 + d, 3000, d)
            grid = fcb.RectilinearGrid.from_knots(knots)
            sl = slice(rank, None, world)                    # this rank's shard of the points
            su = fcb.validate_sample(x[sl])
            sw = fcb.validate_sample(x[sl], w[sl])
            for delta in [(1,) * d, (-1,) + (1,) * (d - 1), (1, -1) + (1,) * (d - 2)]:
                r = fdist.ecdf_fastsum_slab(su, grid, fcb.DeltaVector(delta), scaled=False, engine=eng)
                res[("ecdf", d, delta)] = (r.metadata["slab"], r.values.numpy())
            r = fdist.ecdf_fastsum_slab(sw, grid, fcb.DeltaVector((1,) * d), engine=eng)
            res[("ecdfw", d)] = (r.metadata["slab"], r.values.numpy())
            r = fdist.ecdf_fastsum_slab(su, grid, survival=True, scaled=False, engine=eng)
            res[("esf", d)] = (r.metadata["slab"], r.values.numpy())
            r = fdist.kde_fastsum_slab(sw, grid, fcb.laplacian(),
                                       fcb.Bandwidth.diag([0.3, 0.2, 0.5, 0.4][:d]), engine=eng)
            res[("kde", d)] = (r.metadata["slab"], r.values.numpy())
        out = [None] * world
        dist.all_gather_object(out, res)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _assemble(parts, key, shape):
    m1 = shape[1]
    full = np.zeros(shape)
    for res in parts:
        (lo, hi), vals = res[key]
        full[:, lo:hi] = vals.reshape((shape[0], hi - lo) + tuple(shape[2:]))
    return full.reshape(-1)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_slab_decomposition_matches_single_grid(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for d in (2, 3, 4):
        x, w, knots = _data(100 + d, 3000, d)
        shape = tuple(len(z) for z in knots)
        for delta in [(1,) * d, (-1,) + (1,) * (d - 1), (1, -1) + (1,) * (d - 2)]:
            got = _assemble(parts, ("ecdf", d, delta), shape)
            np.testing.assert_array_equal(got, oracle.ecdf_fastsum(x, None, knots, delta, scaled=False))
        got = _assemble(parts, ("ecdfw", d), shape)
        ref = oracle.ecdf_fastsum(x, w, knots, (1,) * d)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)
        got = _assemble(parts, ("esf", d), shape)
        np.testing.assert_array_equal(got, oracle.esf_fastsum(x, None, knots, scaled=False))
        got = _assemble(parts, ("kde", d), shape)
        ref = oracle.kde_fastsum_laplacian(x, w, knots, [0.3, 0.2, 0.5, 0.4][:d])
        np.testing.assert_allclose(got, ref, rtol=1e-11, atol=0)


def test_slab_bounds():
    assert fdist.slab_bounds(128, 8) == list(range(0, 129, 16))
    b = fdist.slab_bounds(129, 8)
    assert b[0] == 0 and b[-1] == 129 and max(np.diff(b)) - min(np.diff(b)) <= 1
    with pytest.raises(fcb.ParameterError):
        fdist.slab_bounds(3, 4)


# ---- at-points query sharding (replicated ranked data, sharded queries) -------

def _points_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_engine import OracleEngine

        eng = OracleEngine()
        rng = np.random.default_rng(5)
        n = 9000  # a few rank chunks: shards own 0..3 chunks each
        x = rng.standard_normal((n, 2))
        y = np.sin(3 * x[:, 0]) + rng.normal(0, 0.1, n)
        s = fcb.validate_sample(x)
        bw = fcb.Bandwidth.diag([0.3, 0.4])
        res = {
            "num": fdist.kde_numerators_sharded(s, [None, y], bw, engine=eng),
            "own": fdist.kde_numerators_sharded(s, [None], bw, engine=eng, gather=False)[0],
            "nw": fdist.kernel_regression_sharded(s, y, fcb.laplacian(), bw, engine=eng).values,
            "ecdf": fdist.ecdf_dnc_sharded(fcb.validate_sample(x, np.abs(y)), engine=eng).values,
        }
        res = {k: np.asarray(v) for k, v in res.items()}
        out = [None] * world
        dist.all_gather_object(out, res)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_points_query_shards_match_single(world):
    """The sharded at-points calls, gathered, equal the single-process oracle; each point is
    evaluated by exactly one rank (the non-gathered outputs partition the queries)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_points_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    n = 9000
    x = rng.standard_normal((n, 2))
    y = np.sin(3 * x[:, 0]) + rng.normal(0, 0.1, n)
    dens = oracle.kde_dnc_laplacian(x, None, [0.3, 0.4])
    reg = oracle.kde_dnc_laplacian(x, y, [0.3, 0.4])
    for r in range(world):
        np.testing.assert_array_equal(parts[r]["num"][0], dens)
        np.testing.assert_array_equal(parts[r]["num"][1], reg)
        np.testing.assert_array_equal(parts[r]["nw"], reg / dens)
        np.testing.assert_array_equal(parts[r]["ecdf"], oracle.ecdf_dnc(x, np.abs(y)))
    owned = np.stack([parts[r]["own"] != 0 for r in range(world)])
    assert np.all(owned.sum(axis=0) == 1)  # densities are > 0: ownership is a partition
    np.testing.assert_array_equal(sum(parts[r]["own"] for r in range(world)), dens)


def test_query_shard_chunks_partition():
    for n in (1, 2047, 2048, 4095, 4096, 9000, 10_000_000):
        for G in (1, 2, 3, 8):
            spans = [fdist.query_shard_chunks(n, s, G) for s in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == -(-n // fdist.POINTS_CHUNK)
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
