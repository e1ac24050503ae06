"""Generalized ECDF / ESF at the sample points with ties allowed, and Nadaraya-Watson kernel
regression — the at-points extensions BASELINE config 2 and config 4 need.

* ``ecdf_at_points(sample, delta)``: F(x_j) = (1/N) sum_i y_i prod_k [x_ik <= x_jk] (delta_k=+1)
  or [x_ik < x_jk] (delta_k=-1), i == j included — exactly Eq. (3) as the reference's
  ``ecdf_naive(sample, sample.points, delta)`` evaluates it (naive.py:90-114, 187-207).
* ``esf_at_points(sample)``: (1/N) sum_i y_i prod_k [x_ik > x_jk] — ``esf_naive`` at the points
  (naive.py:210-217), i.e. F_N(-z, -1; -x, y) of PAPER.md:48-49.
* ``kernel_regression(sample, y, kernel, bandwidth)``: sum_i y_i K_h(x_i - x_j) /
  sum_i K_h(x_i - x_j), both numerators from one device pass of the Laplacian kde_dnc kernel
  (the reference has no dedicated function; its weights double as the response, core.py:53-58,
  PAPER.md:415-419).
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from .core import as_sample, POINT_ALIGNED, Bandwidth, DeltaVector, EvalResult, ParameterError, Sample
from .dnc import _diag_bandwidth, _kde_points, _out, _require_distinct
from .kernels import KernelSpec


def _points_device(sample: Sample, delta: DeltaVector | None, survival: bool, scaled: bool):
    import torch

    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    signs = delta.signs if delta is not None else (1,) * d
    if len(signs) != d:
        raise ParameterError("delta dimension does not match sample")
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    out = torch.empty(n, dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_ecdf_points", _lib.ptr(x), n, d, _lib.ptr(w), _lib.i32_array(signs),
                 int(survival), int(scaled), _lib.ptr(out))
    return out


def ecdf_at_points(sample: Sample, delta: DeltaVector | None = None,
                   scaled: bool = True) -> EvalResult:
    sample = as_sample(sample)
    t0 = time.perf_counter()
    vals = _points_device(sample, delta, False, scaled)
    return EvalResult(_out(sample, vals), POINT_ALIGNED, {
        "method": "rank-dominance", "scaled": scaled,
        "runtime_seconds": time.perf_counter() - t0})


def esf_at_points(sample: Sample, scaled: bool = True) -> EvalResult:
    sample = as_sample(sample)
    t0 = time.perf_counter()
    vals = _points_device(sample, None, True, scaled)
    return EvalResult(_out(sample, vals), POINT_ALIGNED, {
        "method": "rank-dominance-esf", "scaled": scaled,
        "runtime_seconds": time.perf_counter() - t0})


def ecdf_esf_at_points(sample: Sample, delta: DeltaVector | None = None,
                       scaled: bool = True) -> tuple[EvalResult, EvalResult]:
    """``(ecdf_at_points(sample, delta), esf_at_points(sample))`` from one device ranking of
    every dimension (``fcg_ecdf_esf_points``): the two outputs of BASELINE config 2."""
    import torch

    sample = as_sample(sample)
    t0 = time.perf_counter()
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    signs = delta.signs if delta is not None else (1,) * d
    if len(signs) != d:
        raise ParameterError("delta dimension does not match sample")
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    out = torch.empty((2, n), dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_ecdf_esf_points", _lib.ptr(x), n, d, _lib.ptr(w), _lib.i32_array(signs),
                 int(scaled), _lib.ptr(out[0]), _lib.ptr(out[1]))
    meta = {"scaled": scaled, "runtime_seconds": time.perf_counter() - t0}
    return (EvalResult(_out(sample, out[0]), POINT_ALIGNED, {"method": "rank-dominance", **meta}),
            EvalResult(_out(sample, out[1]), POINT_ALIGNED, {"method": "rank-dominance-esf", **meta}))


def kde_numerators(sample: Sample, weights_list, bandwidth: Bandwidth):
    """Laplacian KDE numerators at the points for one or two weight vectors (None = unit) in a
    single device pass; (nw, n) tensor (device sample) or array."""
    sample = as_sample(sample)
    _require_distinct(sample)
    h = _diag_bandwidth(sample, bandwidth)
    if not 1 <= len(weights_list) <= 2:
        raise ParameterError("one or two weight vectors per pass")
    return _out(sample, _kde_points(sample, list(weights_list), h))


def kernel_regression(sample: Sample, y, kernel: KernelSpec, bandwidth: Bandwidth) -> EvalResult:
    """Nadaraya-Watson regression at the sample points with a Laplacian kernel."""
    sample = as_sample(sample)
    t0 = time.perf_counter()
    if kernel.family != "laplacian":
        raise ParameterError(f"kernel_regression supports the laplacian kernel, got {kernel.family!r}")
    num = kde_numerators(sample, [y, None], bandwidth)
    ratio = num[0] / num[1]
    return EvalResult(ratio, POINT_ALIGNED, {
        "method": "dnc-nadaraya-watson", "kernel": str(kernel),
        "runtime_seconds": time.perf_counter() - t0})


def rank_f64(keys):
    """Per-dimension ranking (north_star subsystem 1) of a 1-D key vector on the device:
    (order, pos, lower, upper, dense).  ``order`` is ``np.argsort(keys, kind="stable")``
    (dnc.py:523-528), ``dense`` / ``dense + 1`` are the reference's sorted-scan bins with
    knots = the distinct values for delta = +1 / -1 (histogram.py:122-133), ``lower`` /
    ``upper`` count the keys strictly below / at-or-below each key (the < and <= tie rules).
    Returns numpy arrays for host input, int32 CUDA tensors for device input."""
    outs = _lib.rank_f64(keys)
    if _lib.is_torch(keys) and keys.device.type == "cuda":
        return outs
    return tuple(o.cpu().numpy() for o in outs)
