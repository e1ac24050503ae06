"""Multi-GPU grid ECDF / ESF / Laplacian KDE: slab decomposition along axis 1.

One process per GPU (torch.distributed, NCCL).  Every rank starts with its own shard of the
points; the output lattice is split along axis 1 into contiguous slabs, one per rank.

1. Routing: each point goes to the rank owning its axis-1 cell (``fcg_axis_owner``), rows are
   partitioned by owner on the device (``fcg_partition_rows``) and exchanged with one
   ``all_to_all_single`` per array.
2. Local pipeline: the rank runs the ordinary single-GPU pipeline on the sub-grid whose axis-1
   knots are its slab's knots.  Because prefix sums along different axes commute, everything
   except the axis-1 coupling between slabs is exact locally.
3. Carry exchange: the slab-boundary plane of every rank (last axis-1 plane for a forward scan,
   first plane for a reverse one) is all-gathered; rank r adds the sum of the lower ranks'
   planes (forward) or the higher ranks' planes (reverse), broadcast along axis 1
   (``fcg_slab_finish``).  Unit-weight counts stay int64 until the final division by the
   global N, so the result is bit-identical to the single-GPU one.
4. Laplacian KDE: every term's S = local S + carry plane; since the term enters the output as
   zfac * S (linear), all 2^d exchanged carry planes are folded in one pass
   (``fcg_kde_carry_fixup``).  The centre c is the global hull midrange (one all-reduce), so
   all ranks use the same exponential frame.  A point whose delta=+1 bin is a slab's first bin
   is also needed by the slab below (its delta_1 = -1 cell), so it is sent to both.

Output stays sharded: rank r returns values for axis-1 cells [lo_r, hi_r) (lexicographic
within the slab).  ``engine`` exists so the CPU tests can drive the same decomposition with
the oracle; the product path always uses the device engine.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .core import (
    EXP_OVERFLOW_GUARD,
    GRID_ALIGNED,
    POINT_ALIGNED,
    Bandwidth,
    DeltaVector,
    EvalResult,
    OverflowGuardError,
    ParameterError,
    RectilinearGrid,
    Sample,
    as_sample,
)


def slab_bounds(m1: int, world: int) -> list[int]:
    """Contiguous, balanced split of m1 axis-1 cells over `world` ranks (uneven allowed)."""
    if m1 < world:
        raise ParameterError(f"axis 1 has {m1} cells, fewer than {world} ranks")
    base, extra = divmod(m1, world)
    out = [0]
    for r in range(world):
        out.append(out[-1] + base + (1 if r < extra else 0))
    return out


class DeviceEngine:
    """Local steps on the current CUDA device through the C-ABI."""

    def tensor(self, a):
        return _lib.to_device_f64(a)

    def axis_owner(self, x, knots_axis, le, shift, bounds):
        import torch

        n, d = x.shape
        owner = torch.empty(n, dtype=torch.int32, device=x.device)
        kn = _lib.to_device_f64(knots_axis)
        _lib.check(_lib.load_library().fcg_axis_owner(
            _lib.ptr(x), n, d, 1, _lib.ptr(kn), int(kn.numel()), int(le), int(shift),
            _lib.i64_array(bounds), len(bounds) - 1, _lib.ptr(owner), _lib.stream_handle()),
            "fcg_axis_owner")
        return owner

    def partition(self, x, w, owner, G):
        import torch

        n, d = x.shape
        xo = torch.empty_like(x)
        wo = None if w is None else torch.empty_like(w)
        counts = (C.c_int64 * G)()
        _lib.call_ws("fcg_partition_rows", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(owner), G,
                     _lib.ptr(xo), _lib.ptr(wo), counts)
        return xo, wo, [int(c) for c in counts]

    def local_ecdf(self, x, w, grid, delta, survival):
        """Unscaled slab-local values: int64 counts (w None) or fp64 sums."""
        from .fastsum import _ecdf_grid_device

        s = Sample(x, w if w is not None else None, None, w is None)
        return _ecdf_grid_device(s, grid, delta, survival, False, counts=w is None)

    def slab_finish(self, local, carry, A, J, B, div):
        import torch

        out = torch.empty(A * J * B, dtype=torch.float64, device=local.device)
        kind = 0 if local.dtype == torch.int64 else 1
        _lib.check(_lib.load_library().fcg_slab_finish(
            _lib.ptr(local), kind, _lib.ptr(carry), A, J, B, float(div), _lib.ptr(out),
            _lib.stream_handle()), "fcg_slab_finish")
        return out

    def minmax(self, x):
        return _lib.minmax(x)

    def local_kde(self, x, w, grid, h, centre, n_scale, u_bound=-1.0):
        """Slab-local KDE and the 2^d slab-boundary planes of S."""
        import torch

        n, d = x.shape
        m = grid.shape
        plane = int(np.prod(m)) // m[1]
        out = torch.empty(int(np.prod(m)), dtype=torch.float64, device=x.device)
        planes = torch.zeros((1 << d) * plane, dtype=torch.float64, device=x.device)
        kn = _lib.device_knots(grid)
        _lib.call_ws("fcg_kde_grid_laplacian_ex", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(kn),
                     _lib.i64_array(m), _lib.f64_array(h), _lib.f64_array(centre),
                     float(n_scale), float(u_bound), _lib.ptr(planes), _lib.ptr(out))
        return out, planes

    def kde_fixup(self, out, grid, h, centre, carries, n_scale):
        kn = _lib.device_knots(grid)
        _lib.call_ws("fcg_kde_carry_fixup", _lib.ptr(out), grid.dim, _lib.i64_array(grid.shape),
                     _lib.ptr(kn), _lib.f64_array(h), _lib.f64_array(centre), _lib.ptr(carries),
                     float(n_scale))
        return out


    # ---- at-points query shards (d = 2) ----------------------------------------------------
    def kde_points_shard(self, x, wmat, nw, h, centre, shard, nshards):
        import torch

        n = x.shape[0]
        out = torch.empty((nw, n), dtype=torch.float64, device=x.device)
        _lib.call_ws("fcg_kde_points_laplacian_shard", _lib.ptr(x), n, 2, _lib.ptr(wmat), nw,
                     _lib.f64_array(h), _lib.f64_array(centre), int(shard), int(nshards),
                     _lib.ptr(out))
        return out

    def dnc_ecdf_shard(self, x, w, include_self, scaled, shard, nshards):
        import torch

        n = x.shape[0]
        out = torch.empty(n, dtype=torch.float64, device=x.device)
        _lib.call_ws("fcg_dnc_ecdf_shard", _lib.ptr(x), n, 2, _lib.ptr(w), int(include_self),
                     int(scaled), int(shard), int(nshards), _lib.ptr(out))
        return out


def _dist():
    import torch.distributed as dist

    if not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised")
    return dist


def _exchange_rows(x, w, owner, world, engine, group):
    """Partition local rows by owner and all-to-all them; returns the received (x, w)."""
    import torch

    dist = _dist()
    d = x.shape[1]
    xs, ws, counts = engine.partition(x, w, owner, world)
    send = torch.tensor(counts, dtype=torch.int64, device=x.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(v) for v in recv.tolist()]
    live = sum(counts)
    xr = torch.empty((sum(rc), d), dtype=torch.float64, device=x.device)
    dist.all_to_all_single(xr.view(-1), xs[:live].reshape(-1).contiguous(),
                           output_split_sizes=[c * d for c in rc],
                           input_split_sizes=[c * d for c in counts], group=group)
    wr = None
    if w is not None:
        wr = torch.empty(sum(rc), dtype=torch.float64, device=x.device)
        dist.all_to_all_single(wr, ws[:live].contiguous(), output_split_sizes=rc,
                               input_split_sizes=counts, group=group)
    return xr, wr


def _sub_grid(grid, lo, hi):
    knots = [np.asarray(z, dtype=np.float64) for z in grid.knots]
    knots[1] = knots[1][lo:hi]
    return RectilinearGrid.from_knots(knots)


def _gather_planes(plane, world, group):
    import torch

    dist = _dist()
    bufs = [torch.empty_like(plane) for _ in range(world)]
    dist.all_gather(bufs, plane.contiguous(), group=group)
    return bufs


def ecdf_fastsum_slab(sample: Sample, grid: RectilinearGrid, delta: DeltaVector | None = None,
                      scaled: bool = True, survival: bool = False, group=None,
                      engine=None) -> EvalResult:
    """Distributed ecdf_fastsum (survival=False) / esf_fastsum (survival=True); each rank passes
    its shard of the points and receives its axis-1 slab of the grid values."""
    import torch

    sample = as_sample(sample)
    dist = _dist()
    eng = engine or DeviceEngine()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    d = sample.dim
    if d < 2 or grid.dim != d:
        raise ParameterError("slab decomposition needs d >= 2 and a matching grid")
    delta = delta or DeltaVector.ones(d)
    m = grid.shape
    bounds = slab_bounds(m[1], world)
    lo, hi = bounds[rank], bounds[rank + 1]
    x = eng.tensor(sample.points)
    w = None if sample.unit_weights else eng.tensor(sample.weights)
    le = 0 if survival else int(delta.signs[1] < 0)
    shift = 1 if survival else 0
    if world > 1:
        owner = eng.axis_owner(x, grid.knots[1], le, shift, bounds)
        xr, wr = _exchange_rows(x, w, owner, world, eng, group)
    else:  # one slab: every point is already on its owner (dead points are skipped locally)
        xr, wr = x, w
    n_total = torch.tensor([sample.count], dtype=torch.int64, device=x.device)
    dist.all_reduce(n_total, group=group)
    sub = _sub_grid(grid, lo, hi)
    local = eng.local_ecdf(xr, wr, sub, delta, survival)
    A, J = m[0], hi - lo
    B = int(np.prod(m[2:])) if d > 2 else 1
    cube = local.view(A, J, B)
    plane = (cube[:, 0, :] if survival else cube[:, J - 1, :]).contiguous()
    planes = _gather_planes(plane, world, group)
    others = planes[rank + 1:] if survival else planes[:rank]
    # carry = sum of the lower (forward) / higher (survival) ranks' boundary planes, on device
    carry = torch.stack(others).sum(0) if others else None
    out = eng.slab_finish(local, carry, A, J, B, float(n_total.item()) if scaled else 0.0)
    return EvalResult(out, GRID_ALIGNED, {"method": "fastsum-slab", "scaled": scaled,
                                          "slab": (lo, hi), "world": world})


def kde_fastsum_slab(sample: Sample, grid: RectilinearGrid, kernel, bandwidth: Bandwidth,
                     group=None, engine=None) -> EvalResult:
    """Distributed Laplacian kde_fastsum; each rank passes its shard of the points (and their
    weights) and receives its axis-1 slab of the density grid."""
    import torch

    sample = as_sample(sample)
    dist = _dist()
    eng = engine or DeviceEngine()
    if kernel.family != "laplacian":
        raise ParameterError("the slab-decomposed KDE supports the laplacian kernel")
    if not bandwidth.is_diagonal:
        raise ParameterError("kde_fastsum requires a diagonal bandwidth")
    h = np.ascontiguousarray(bandwidth.diagonal, dtype=np.float64)
    d = sample.dim
    if d < 2 or grid.dim != d or h.size != d:
        raise ParameterError("slab decomposition needs d >= 2 and matching grid / bandwidth")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    m = grid.shape
    bounds = slab_bounds(m[1], world)
    lo, hi = bounds[rank], bounds[rank + 1]
    x = eng.tensor(sample.points)
    w = None if sample.unit_weights else eng.tensor(sample.weights)
    # global hull midrange of data and grid + overflow guard (fastsum.py:114-129)
    dmin, dmax = eng.minmax(x)
    mm = torch.tensor(np.concatenate([-dmin, dmax]), dtype=torch.float64, device=x.device)
    dist.all_reduce(mm, op=dist.ReduceOp.MAX, group=group)
    mm = mm.cpu().numpy()
    lo_h = np.minimum(-mm[:d], np.array([float(np.asarray(z)[0]) for z in grid.knots]))
    hi_h = np.maximum(mm[d:], np.array([float(np.asarray(z)[-1]) for z in grid.knots]))
    span = hi_h - lo_h
    for k in range(d):
        if span[k] / h[k] > EXP_OVERFLOW_GUARD:
            raise OverflowGuardError(
                f"dimension {k}: span/bandwidth = {span[k] / h[k]:.1f} exceeds "
                f"{EXP_OVERFLOW_GUARD:.0f}; enlarge the bandwidth or rescale")
    centre = 0.5 * (lo_h + hi_h)
    # route by the delta=+1 cell and, for the delta_1 = -1 terms, by the cell one bin lower:
    # a point in the first bin of slab r > 0 is also needed by slab r - 1.  Those duplicates are
    # a thin layer (about G / M_1 of the points), so they are compacted first and routed alone.
    if world > 1:
        own_a = eng.axis_owner(x, grid.knots[1], 0, 0, bounds)
        own_b = eng.axis_owner(x, grid.knots[1], 0, 1, bounds)
        dup = torch.nonzero((own_b != own_a) & (own_b >= 0)).flatten()
        xa, wa = _exchange_rows(x, w, own_a, world, eng, group)
        xd = x[dup].contiguous()
        wd = None if w is None else w[dup].contiguous()
        xb, wb = _exchange_rows(xd, wd, own_b[dup].contiguous(), world, eng, group)
        xr = torch.cat([xa, xb]) if xb.shape[0] else xa
        wr = None if w is None else (torch.cat([wa, wb]) if wb.shape[0] else wa)
    else:  # one slab: no routing and no slab boundary to duplicate across
        xr, wr = x, w
    n_total = torch.tensor([sample.count], dtype=torch.int64, device=x.device)
    dist.all_reduce(n_total, group=group)
    N = float(n_total.item())
    sub = _sub_grid(grid, lo, hi)
    out, planes = eng.local_kde(xr, wr, sub, h, centre, N, float(np.sum(span / (2.0 * h))) * 1.000001)
    ncodes = 1 << d
    if world == 1:  # no other slab: every carry plane is zero
        return EvalResult(out, GRID_ALIGNED, {"method": "fastsum-slab", "kernel": str(kernel),
                                              "slab": (lo, hi), "world": world})
    gathered = torch.stack(_gather_planes(planes, world, group)).view(world, ncodes, -1)
    # forward codes (delta_1 = +1) add the lower ranks' planes, reverse codes the higher ones';
    # two prefix sums over the rank axis, on device
    fwd = gathered[:rank].sum(0) if rank > 0 else torch.zeros_like(gathered[0])
    rev = gathered[rank + 1:].sum(0) if rank + 1 < world else torch.zeros_like(gathered[0])
    is_rev = torch.tensor([bool((c >> 1) & 1) for c in range(ncodes)], device=planes.device)
    carries = torch.where(is_rev[:, None], rev, fwd).reshape(-1).contiguous()
    out = eng.kde_fixup(out, sub, h, centre, carries, N)
    return EvalResult(out, GRID_ALIGNED, {"method": "fastsum-slab", "kernel": str(kernel),
                                          "slab": (lo, hi), "world": world})


# ------------------------------------------------------------------------------------------
# At-points queries, sharded ("sample-point queries are sharded with the ranked data
# replicated").  Every rank holds the whole sample; the device call ranks and groups all n
# sources (replicated, no communication) and evaluates only the rank's queries: the points
# whose dimension-1 rank falls in a contiguous 1/G slice of the POINTS_CHUNK-point chunks.  Other
# entries come back as exact zeros, so the optional final gather is one SUM all-reduce of the
# owned values (computed by the single-GPU arithmetic).  The hot loop has no collective.

POINTS_CHUNK = 2048  # points per rank chunk of the d = 2 dominance route (csrc/points.cu: S)


def query_shard_chunks(n: int, shard: int, nshards: int,
                       chunk: int = POINTS_CHUNK) -> tuple[int, int]:
    """[c_lo, c_hi): the dimension-1 rank chunks whose points shard `shard` evaluates."""
    P = -(-n // chunk)
    return P * shard // nshards, P * (shard + 1) // nshards


def _shard_group(group):
    dist = _dist()
    return dist, dist.get_rank(group), dist.get_world_size(group)


def _finish_points(out, dist, group, world, gather):
    if gather and world > 1:
        dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def kde_numerators_sharded(sample: Sample, weights_list, bandwidth: Bandwidth, group=None,
                           engine=None, gather: bool = True):
    """kde_numerators (Laplacian, d = 2) with the queries sharded over the ranks of `group`.
    Returns the (nw, n) numerators: all of them when `gather`, else the rank's own entries
    (zeros elsewhere).  Drop-in for points.kde_numerators on every rank."""
    import torch

    from .dnc import _diag_bandwidth, _require_distinct

    sample = as_sample(sample)
    if sample.dim != 2:
        raise ParameterError("query sharding is implemented for d = 2")
    _require_distinct(sample)
    h = _diag_bandwidth(sample, bandwidth)
    if not 1 <= len(weights_list) <= 2:
        raise ParameterError("one or two weight vectors per pass")
    dist, rank, world = _shard_group(group)
    engine = engine or DeviceEngine()
    x = engine.tensor(sample.points)
    n = x.shape[0]
    lo, hi = engine.minmax(x)  # overflow guard and data midrange (dnc.py:598-605, 656)
    span = hi - lo
    for k in range(2):
        if span[k] / h[k] > EXP_OVERFLOW_GUARD:
            raise OverflowGuardError(
                f"dimension {k}: span/bandwidth = {span[k] / h[k]:.1f} exceeds "
                f"{EXP_OVERFLOW_GUARD:.0f}; enlarge the bandwidth or rescale")
    c = 0.5 * (lo + hi)
    ws = [None if w is None else engine.tensor(w) for w in weights_list]
    if any(w is None for w in ws):
        ws = [torch.ones(n, dtype=torch.float64, device=x.device) if w is None else w for w in ws]
    wmat = torch.stack(ws).contiguous()
    out = engine.kde_points_shard(x, wmat, len(ws), h, c, rank, world)
    out = _finish_points(out, dist, group, world, gather)
    return out if sample.on_device else _lib.to_host(out)


def kernel_regression_sharded(sample: Sample, y, kernel, bandwidth: Bandwidth, group=None,
                              engine=None) -> EvalResult:
    """points.kernel_regression with the queries sharded (both numerators in one pass per
    rank, one SUM all-reduce, then the ratio)."""
    if kernel.family != "laplacian":
        raise ParameterError(f"kernel_regression supports the laplacian kernel, got {kernel.family!r}")
    num = kde_numerators_sharded(sample, [y, None], bandwidth, group, engine)
    return EvalResult(num[0] / num[1], POINT_ALIGNED, {"method": "dnc-nadaraya-watson-sharded",
                                                  "kernel": str(kernel)})


def kde_dnc_sharded(sample: Sample, kernel, bandwidth: Bandwidth, group=None,
                    engine=None) -> EvalResult:
    """dnc.kde_dnc (Laplacian, d = 2) with the queries sharded and gathered."""
    if kernel.family != "laplacian":
        raise ParameterError(f"kde_dnc_sharded supports the laplacian kernel, got {kernel.family!r}")
    sample = as_sample(sample)
    w = None if sample.unit_weights else sample.weights
    vals = kde_numerators_sharded(sample, [w], bandwidth, group, engine)[0]
    return EvalResult(vals, POINT_ALIGNED, {"method": "dnc-sharded", "kernel": str(kernel)})


def ecdf_dnc_sharded(sample: Sample, include_self: bool = False, scaled: bool = True,
                     group=None, engine=None, gather: bool = True) -> EvalResult:
    """dnc.ecdf_dnc (d = 2) with the queries sharded over the ranks of `group`."""
    from .dnc import _require_distinct

    sample = as_sample(sample)
    if sample.dim != 2:
        raise ParameterError("query sharding is implemented for d = 2")
    _require_distinct(sample)
    dist, rank, world = _shard_group(group)
    engine = engine or DeviceEngine()
    x = engine.tensor(sample.points)
    w = None if sample.unit_weights else engine.tensor(sample.weights)
    out = engine.dnc_ecdf_shard(x, w, include_self, scaled, rank, world)
    out = _finish_points(out, dist, group, world, gather)
    return EvalResult(out if sample.on_device else _lib.to_host(out), POINT_ALIGNED,
                      {"method": "dnc-sharded", "scaled": scaled, "include_self": include_self})
