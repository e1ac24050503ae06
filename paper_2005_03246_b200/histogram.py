"""Local sums over grid cells — the generalized multivariate histogram of Eq. (4).

Drop-in for the reference's ``fastcdf.histogram`` public functions (histogram.py:191-217).  The
bin rule is the reference's (histogram.py:3-15): in dimension k a point lands in bin
b = #knots < x for delta_k = +1 and b = #knots <= x for delta_k = -1, b in [0, M_k], so a plain
prefix sum reproduces the strict / non-strict inequality exactly.  Binning and scatter-add run
in one fused sm_100a kernel (``fcg_local_sums``); unit-weight samples accumulate exact int32
counts, weighted samples fp64 sums.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import as_sample, DeltaVector, ParameterError, RectilinearGrid, Sample


@dataclass(frozen=True)
class LocalSumTensor:
    """Dense (M_1+1) x ... x (M_d+1) per-cell sums, last dimension contiguous (raw, unscaled)."""

    data: object
    scaled: bool = False

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(int(v) for v in self.data.shape)

    def total(self) -> float:
        return float(self.data.sum())


def _check_dims(sample: Sample, grid: RectilinearGrid, delta: DeltaVector):
    if grid.dim != sample.dim or delta.dim != sample.dim:
        raise ParameterError(
            f"dimension mismatch: sample d={sample.dim}, grid d={grid.dim}, delta d={delta.dim}")


def _local_sums_device(sample: Sample, grid: RectilinearGrid, delta: DeltaVector):
    """Run fcg_local_sums; returns an fp64 CUDA tensor of shape (M_k + 1)_k."""
    import torch

    _check_dims(sample, grid, delta)
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    dims = tuple(m + 1 for m in grid.shape)
    unit = sample.unit_weights
    w = None if unit else _lib.to_device_f64(sample.weights)
    kn = _lib.device_knots(grid)
    lat = torch.empty(dims, dtype=torch.int32 if unit else torch.float64, device=x.device)
    _lib.call_ws("fcg_local_sums", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(kn),
                 _lib.i64_array(grid.shape), _lib.i32_array(delta.signs),
                 _lib.LAT_I32 if unit else _lib.LAT_F64, _lib.ptr(lat))
    return lat.to(torch.float64) if unit else lat


def _wrap(sample: Sample, t):
    return t if sample.on_device else _lib.to_host(t)


def local_sums(sample: Sample, grid: RectilinearGrid,
               delta: DeltaVector | None = None) -> LocalSumTensor:
    """Local sums with the delta bin convention (histogram.py:210-217)."""
    sample = as_sample(sample)
    delta = delta or DeltaVector.ones(sample.dim)
    return LocalSumTensor(_wrap(sample, _local_sums_device(sample, grid, delta)))


def local_sums_sorted(sample: Sample, grid: RectilinearGrid,
                      delta: DeltaVector | None = None) -> LocalSumTensor:
    """Reference name for the sort-based binning (histogram.py:191-197).  The device binner
    is exact for any rectilinear grid, so both entry points share one kernel."""
    return local_sums(sample, grid, delta)


def local_sums_uniform(sample: Sample, grid: RectilinearGrid,
                       delta: DeltaVector | None = None) -> LocalSumTensor:
    """Mesh-division binning (histogram.py:200-207); requires a uniform grid like the
    reference, and returns output identical to :func:`local_sums_sorted`."""
    if not grid.is_uniform:
        raise ParameterError("mesh-division binning requires a uniform grid")
    return local_sums(sample, grid, delta)


def scatter_total(t: LocalSumTensor) -> float:
    return float(np.asarray(t.data).sum()) if not _lib.is_torch(t.data) else float(t.data.sum())
