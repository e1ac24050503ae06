"""Lexicographic fast-sum evaluation on rectilinear grids (Algorithm 1) on sm_100a.

Drop-in for the reference's ``fastcdf.fastsum`` (fastsum.py:60-233): same signatures, the same
EvalResult layout (grid-aligned, lexicographic, last dimension fastest) and the same guards
and exceptions.  Each call is one native pipeline (bin+scatter, one scan pass per axis, the
last pass writing the output) launched on the caller's current CUDA stream.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (
    as_sample,
    EXP_OVERFLOW_GUARD,
    GRID_ALIGNED,
    Bandwidth,
    DeltaVector,
    EvalResult,
    OverflowGuardError,
    ParameterError,
    RectilinearGrid,
    Sample,
)
from .histogram import LocalSumTensor, _check_dims
from .kernels import KernelSpec


@dataclass(frozen=True)
class CumulativeTensor:
    """Directional cumulative form of a local-sum tensor (fastsum.py:36-42)."""

    data: object
    scaled: bool = False


def _out(sample: Sample, t):
    return t if sample.on_device else _lib.to_host(t)


def directional_sweep(tensor: LocalSumTensor, delta: DeltaVector) -> CumulativeTensor:
    """Prefix sums along every axis, suffix sums where delta is -1 (fastsum.py:60-66).
    The input tensor is not modified."""
    import torch

    dims = tuple(int(v) for v in tensor.data.shape)
    if delta.dim != len(dims):
        raise ParameterError("delta dimension does not match tensor rank")
    was_torch = _lib.is_torch(tensor.data)
    lat = _lib.to_device_f64(tensor.data)
    if was_torch and lat.data_ptr() == tensor.data.data_ptr():
        lat = lat.clone()
    _lib.call_ws("fcg_directional_sweep", _lib.ptr(lat), _lib.LAT_F64, len(dims),
                 _lib.i64_array(dims), _lib.i32_array(delta.signs))
    return CumulativeTensor(lat if was_torch else _lib.to_host(lat), tensor.scaled)


def _ecdf_grid_device(sample: Sample, grid: RectilinearGrid, delta: DeltaVector | None,
                      survival: bool, scaled: bool, counts: bool = False):
    import torch

    d = sample.dim
    delta = delta or DeltaVector.ones(d)
    _check_dims(sample, grid, delta)
    x = _lib.to_device_f64(sample.points)
    n = x.shape[0]
    unit = sample.unit_weights
    if counts and not unit:
        raise ParameterError("integer counts need unit weights")
    w = None if unit else _lib.to_device_f64(sample.weights)
    kn = _lib.device_knots(grid)
    out = torch.empty(grid.size, dtype=torch.int64 if counts else torch.float64, device=x.device)
    _lib.call_ws("fcg_ecdf_grid", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(kn),
                 _lib.i64_array(grid.shape), _lib.i32_array(delta.signs), int(survival),
                 int(scaled), 1 if counts else 0, _lib.ptr(out))
    return out


def ecdf_fastsum(sample: Sample, grid: RectilinearGrid, delta: DeltaVector | None = None,
                 scaled: bool = True) -> EvalResult:
    """Generalized ECDF F_N(z, delta; x, y) at every grid node, exactly (fastsum.py:69-92).
    Unit weights give exact integer counts before the single division by N."""
    sample = as_sample(sample)
    t0 = time.perf_counter()
    vals = _ecdf_grid_device(sample, grid, delta, False, scaled)
    return EvalResult(_out(sample, vals), GRID_ALIGNED, {
        "method": "fastsum", "scaled": scaled,
        "runtime_seconds": time.perf_counter() - t0})


def ecdf_fastsum_counts(sample: Sample, grid: RectilinearGrid,
                        delta: DeltaVector | None = None):
    """Unit-weight grid ECDF as exact int64 counts (device tensor or numpy)."""
    sample = as_sample(sample)
    return _out(sample, _ecdf_grid_device(sample, grid, delta, False, False, counts=True))


def esf_fastsum(sample: Sample, grid: RectilinearGrid, scaled: bool = True) -> EvalResult:
    """Empirical survival function sum_i y_i prod_k [x_ik > z_k] on the grid
    (fastsum.py:95-111), computed directly as suffix sums of strictly-above bins."""
    sample = as_sample(sample)
    t0 = time.perf_counter()
    vals = _ecdf_grid_device(sample, grid, None, True, scaled)
    return EvalResult(_out(sample, vals), GRID_ALIGNED, {
        "method": "fastsum-esf", "scaled": scaled,
        "runtime_seconds": time.perf_counter() - t0})


def _exp_guard_and_center(sample: Sample, grid: RectilinearGrid, h: np.ndarray):
    """Hull midrange of data and grid; OverflowGuardError past span/h > 600
    (fastsum.py:114-129).  Also returns sum_k span_k / (2 h_k), the bound on the centred
    exponents that lets the kernels factor each term's weights."""
    dmin, dmax = _lib.minmax(sample.points)
    lo = np.minimum(dmin, np.array([float(np.asarray(z)[0]) for z in grid.knots]))
    hi = np.maximum(dmax, np.array([float(np.asarray(z)[-1]) for z in grid.knots]))
    span = hi - lo
    for k in range(sample.dim):
        if span[k] / h[k] > EXP_OVERFLOW_GUARD:
            raise OverflowGuardError(
                f"dimension {k}: span/bandwidth = {span[k] / h[k]:.1f} exceeds "
                f"{EXP_OVERFLOW_GUARD:.0f}; enlarge the bandwidth or rescale")
    return 0.5 * (lo + hi), float(np.sum(span / (2.0 * h)))


def _kde_laplacian_grid(sample: Sample, grid: RectilinearGrid, h: np.ndarray):
    """Laplacian terms (fastsum.py:139-169).  The library takes the hull midrange and applies
    the overflow guard of fastsum.py:114-129 itself (auto centre), from the binning pass."""
    import torch

    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    kn = _lib.device_knots(grid)
    out = torch.empty(grid.size, dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_kde_grid_laplacian_ex", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(kn),
                 _lib.i64_array(grid.shape), _lib.f64_array(h), None, float(n), -1.0, None,
                 _lib.ptr(out))
    return out


def _kde_matern32_grid(sample: Sample, grid: RectilinearGrid, h: np.ndarray):
    """matern32-additive: the Laplacian terms with d + 1 channels each (fastsum.py:139-181)."""
    import torch

    c, _ = _exp_guard_and_center(sample, grid, h)
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    kn = _lib.device_knots(grid)
    out = torch.empty(grid.size, dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_kde_grid_matern32", _lib.ptr(x), n, d, _lib.ptr(w), _lib.ptr(kn),
                 _lib.i64_array(grid.shape), _lib.f64_array(h), _lib.f64_array(c), _lib.ptr(out))
    return out


def _kde_uniform_grid(sample: Sample, grid: RectilinearGrid, h: np.ndarray):
    """Uniform kernel as 2^d shifted-grid generalized ECDFs with parity signs
    (fastsum.py:185-201, Eq. 15)."""
    import torch

    d, n = sample.dim, sample.count
    total = None
    for code in range(1 << d):
        delta = DeltaVector.from_code(code, d)
        shifted = grid.shifted(delta.as_array() * h)
        term = _ecdf_grid_device(sample, shifted, delta, False, False)
        term = term if delta.parity > 0 else -term
        total = term if total is None else total + term
    return total / (2.0 ** d * n * float(np.prod(h)))


def kde_fastsum(sample: Sample, grid: RectilinearGrid, kernel: KernelSpec,
                bandwidth: Bandwidth) -> EvalResult:
    """Kernel density estimate at every grid node by CDF decomposition (fastsum.py:204-233)."""
    sample = as_sample(sample)
    t0 = time.perf_counter()
    if not bandwidth.is_diagonal:
        raise ParameterError("kde_fastsum requires a diagonal bandwidth")
    h = np.ascontiguousarray(bandwidth.diagonal, dtype=np.float64)
    if h.size != sample.dim or grid.dim != sample.dim:
        raise ParameterError("bandwidth/grid dimension does not match sample")
    fam = kernel.family
    if fam == "laplacian":
        vals = _kde_laplacian_grid(sample, grid, h)
    elif fam == "uniform":
        vals = _kde_uniform_grid(sample, grid, h)
    elif fam == "matern32-additive":
        vals = _kde_matern32_grid(sample, grid, h)
    else:
        raise ParameterError(f"kde_fastsum supports laplacian, uniform and matern32-additive "
                             f"kernels, got {fam!r}")
    return EvalResult(_out(sample, vals), GRID_ALIGNED, {
        "method": "fastsum", "kernel": str(kernel),
        "runtime_seconds": time.perf_counter() - t0})
