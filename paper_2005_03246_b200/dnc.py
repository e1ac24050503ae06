"""Dominance sums at the sample points — drop-in for the reference's ``fastcdf.dnc`` public
functions ``ecdf_dnc`` (dnc.py:531-561) and ``kde_dnc`` (dnc.py:635-690).

The reference computes them with an O(N log N) divide-and-conquer recursion; here the same sums
come from the rank-space dominance kernel of ``fcg_dnc_ecdf`` / ``fcg_kde_points_laplacian``
(device radix ranking + a 3-level coarse-grid / shared-memory decomposition, d = 2; sort + scan
for d = 1; a coarse G^d rank grid + per-dimension slab phases for 3 <= d <= 6 in place of the
MergeND recursion dnc.py:65-135, 307-410; direct tiles for tiny inputs and d >= 7).  Semantics, guards and exceptions follow the
reference: distinct coordinates are required (TieError), strict comparisons on raw coordinates,
exponentials on midrange-centred coordinates, the self term w_j added before the shared
1/(2^d N prod h) normalisation.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import (
    as_sample,
    EXP_OVERFLOW_GUARD,
    POINT_ALIGNED,
    Bandwidth,
    DeltaVector,
    EvalResult,
    OverflowGuardError,
    ParameterError,
    Sample,
    TieError,
)
from .kernels import KernelSpec


def _require_distinct(sample: Sample):
    """TieError when a dimension has duplicates (dnc.py:491-499)."""
    if not sample.distinct:
        bad = [k for k, ok in enumerate(sample.distinct_by_dim) if not ok]
        raise TieError(
            f"duplicate coordinates in dimension(s) {bad}; the recursion requires distinct "
            f"values per dimension - jitter the data, deduplicate with merged weights, or use "
            f"rank_tiebreak() for pure ECDF counting")


def _diag_bandwidth(sample: Sample, bandwidth: Bandwidth) -> np.ndarray:
    """dnc.py:588-595."""
    if not bandwidth.is_diagonal:
        raise ParameterError("divide-and-conquer KDE requires a diagonal bandwidth; rotate "
                             "matrix bandwidths first")
    h = np.ascontiguousarray(bandwidth.diagonal, dtype=np.float64)
    if h.size != sample.dim:
        raise ParameterError("bandwidth dimension does not match sample")
    return h


def _span_guard_and_centre(sample: Sample, h: np.ndarray) -> np.ndarray:
    """Overflow guard (dnc.py:598-605) and data midrange (dnc.py:656)."""
    lo, hi = _lib.minmax(sample.points)
    span = hi - lo
    for k in range(sample.dim):
        if span[k] / h[k] > EXP_OVERFLOW_GUARD:
            raise OverflowGuardError(
                f"dimension {k}: span/bandwidth = {span[k] / h[k]:.1f} exceeds "
                f"{EXP_OVERFLOW_GUARD:.0f}; enlarge the bandwidth or rescale")
    return 0.5 * (lo + hi)


def _out(sample: Sample, t):
    return t if sample.on_device else _lib.to_host(t)


def ecdf_dnc(sample: Sample, include_self: bool = False, scaled: bool = True) -> EvalResult:
    """Weight sum over the points strictly below each point in every dimension
    (dnc.py:531-561); + own weight when ``include_self``; / N when ``scaled``."""
    sample = as_sample(sample)
    import torch

    t0 = time.perf_counter()
    _require_distinct(sample)
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    out = torch.empty(n, dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_dnc_ecdf", _lib.ptr(x), n, d, _lib.ptr(w), int(include_self),
                 int(scaled), _lib.ptr(out))
    return EvalResult(_out(sample, out), POINT_ALIGNED, {
        "method": "dnc", "scaled": scaled, "include_self": include_self,
        "runtime_seconds": time.perf_counter() - t0})


def _kde_points(sample: Sample, weights_list, h: np.ndarray):
    """Laplacian KDE numerators at the sample points for up to two weight vectors in one
    pass; returns a (nw, n) device tensor."""
    import torch

    c = _span_guard_and_centre(sample, h)
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    ws = [None if w is None else _lib.to_device_f64(w) for w in weights_list]
    nw = len(ws)
    out = torch.empty((nw, n), dtype=torch.float64, device=x.device)
    if d == 2:  # one pointer per weight vector, NULL = unit: no stacked copy
        _lib.call_ws("fcg_kde_points_laplacian_w2", _lib.ptr(x), n, d, _lib.ptr(ws[0]),
                     _lib.ptr(ws[1] if nw > 1 else None), nw, _lib.f64_array(h),
                     _lib.f64_array(c), _lib.ptr(out))
        return out
    if any(w is None for w in ws):
        ws = [torch.ones(n, dtype=torch.float64, device=x.device) if w is None else w for w in ws]
    wmat = torch.stack(ws).contiguous()
    _lib.call_ws("fcg_kde_points_laplacian", _lib.ptr(x), n, d, _lib.ptr(wmat), nw,
                 _lib.f64_array(h), _lib.f64_array(c), _lib.ptr(out))
    return out


def _kde_points_matern32(sample: Sample, h: np.ndarray):
    import torch

    c = _span_guard_and_centre(sample, h)
    x = _lib.to_device_f64(sample.points)
    n, d = x.shape
    w = None if sample.unit_weights else _lib.to_device_f64(sample.weights)
    out = torch.empty(n, dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_kde_points_matern32", _lib.ptr(x), n, d, _lib.ptr(w), _lib.f64_array(h),
                 _lib.f64_array(c), _lib.ptr(out))
    return out


def kde_dnc(sample: Sample, kernel: KernelSpec, bandwidth: Bandwidth) -> EvalResult:
    """Kernel density estimate at the sample points (dnc.py:635-690): laplacian and
    matern32-additive families."""
    sample = as_sample(sample)
    t0 = time.perf_counter()
    _require_distinct(sample)
    fam = kernel.family
    if fam not in ("laplacian", "matern32-additive"):
        raise ParameterError(f"kde_dnc supports laplacian and matern32-additive kernels, "
                             f"got {fam!r}")
    h = _diag_bandwidth(sample, bandwidth)
    w = None if sample.unit_weights else sample.weights
    if fam == "matern32-additive":
        vals = _kde_points_matern32(sample, h)
    else:
        vals = _kde_points(sample, [w], h)[0]
    return EvalResult(_out(sample, vals), POINT_ALIGNED, {
        "method": "dnc", "kernel": str(kernel),
        "runtime_seconds": time.perf_counter() - t0})


@dataclass(frozen=True)
class DeltaTermTable:
    """Per-point, per-sign-code weighted strict-dominance sums (dnc.py:475-487): column ``b``
    of ``table`` sums ``psi[i, b]`` over the points i strictly dominating j under
    ``DeltaVector.from_code(b, dim)`` (the point itself excluded)."""

    table: object
    psi: object
    dim: int

    def delta_for_column(self, b: int) -> DeltaVector:
        return DeltaVector.from_code(b, self.dim)


def kde_terms_dnc(sample: Sample, bandwidth: Bandwidth,
                  monomial: tuple[int, int, int, int] = (0, 0, 0, 0)) -> DeltaTermTable:
    """All-delta dominance tables for exponential kernel compositions (dnc.py:608-632):
    psi(x_i, delta) = w_i x_{l,i}^p x_{m,i}^q exp(sum_k delta_k x_{k,i} / h_k), formed exactly
    as the reference does (numpy, host inputs) and summed over the dominating points on the
    device (``fcg_dominance_terms``: one rank-space dominance sum per code)."""
    import torch

    sample = as_sample(sample)
    _require_distinct(sample)
    h = _diag_bandwidth(sample, bandwidth)
    _span_guard_and_centre(sample, h)
    l, m, p, q = monomial
    d, n = sample.dim, sample.count
    if not (0 <= l < d and 0 <= m < d) or p < 0 or q < 0:
        raise ParameterError(f"invalid monomial {monomial} for dimension {d}")
    if sample.on_device:
        pts = _lib.to_device_f64(sample.points)
        w = _lib.to_device_f64(sample.weights) if sample.weights is not None else None
        poly = pts[:, l] ** p * pts[:, m] ** q
        psi = torch.empty((n, 1 << d), dtype=torch.float64, device=pts.device)
        for code in range(1 << d):
            signs = torch.tensor(DeltaVector.from_code(code, d).as_array() / h, device=pts.device)
            psi[:, code] = (w if w is not None else 1.0) * poly * torch.exp(pts @ signs)
        psi_d, x = psi, pts
    else:
        pts = np.ascontiguousarray(sample.points, dtype=np.float64)
        w = np.ones(n) if sample.weights is None else np.asarray(sample.weights, dtype=np.float64)
        poly = pts[:, l] ** p * pts[:, m] ** q
        psi = np.empty((n, 1 << d))
        for code in range(1 << d):
            signs = DeltaVector.from_code(code, d).as_array()
            psi[:, code] = w * poly * np.exp(pts @ (signs / h))
        psi_d, x = _lib.to_device_f64(psi), _lib.to_device_f64(pts)
    table = torch.empty((n, 1 << d), dtype=torch.float64, device=x.device)
    _lib.call_ws("fcg_dominance_terms", _lib.ptr(x), n, d, _lib.ptr(psi_d), _lib.ptr(table))
    return DeltaTermTable(table if sample.on_device else _lib.to_host(table), psi, d)


def rank_tiebreak(points):
    """Each dimension's values replaced by their stable sort ranks (dnc.py:502-520): ties
    broken by input index, an infinitesimal index-ordered perturbation for ECDF counting.  The
    ranks come from the device ranking (``fcg_rank_f64``, stable order)."""
    on_dev = _lib.is_torch(points)
    pts = _lib.to_device_f64(points)
    if pts.dim() == 1:
        pts = pts.reshape(-1, 1)
    out = pts.new_empty(pts.shape)
    for k in range(pts.shape[1]):
        _, pos, _, _, _ = _lib.rank_f64(pts[:, k].contiguous())
        out[:, k] = pos.to(out.dtype)
    return out if on_dev else _lib.to_host(out)
