"""Multilinear interpolation from grid-aligned results to arbitrary points — the grid -> points
bridge of the reference (interp.py:24-75), on the device (``fcg_multilinear_interp``).

Same checks, messages and metadata as the reference: ShapeError for point-aligned values, a
value vector of the wrong size or queries of the wrong width; ParameterError for a dimension
with fewer than 2 knots; queries outside the hull are clamped per coordinate and counted in
``metadata["clamp_count"]``.  Results are bit-identical to the reference's numpy evaluation.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .core import GRID_ALIGNED, POINT_ALIGNED, EvalResult, ParameterError, RectilinearGrid, ShapeError


def multilinear_interp(grid: RectilinearGrid, values: EvalResult, queries) -> EvalResult:
    """Interpolate grid-aligned values at query points (interp.py:24-75)."""
    import torch

    t0 = time.perf_counter()
    if values.alignment != GRID_ALIGNED:
        raise ShapeError("multilinear_interp needs grid-aligned values")
    vals = values.values
    size = int(vals.numel()) if _lib.is_torch(vals) else int(np.asarray(vals).size)
    if size != grid.size:
        raise ShapeError(f"value vector has {size} entries, grid has {grid.size} points")
    if any(m < 2 for m in grid.shape):
        raise ParameterError("interpolation needs at least 2 knots per dimension")
    on_device = _lib.is_torch(queries) or _lib.is_torch(vals)
    if _lib.is_torch(queries):
        q = queries if queries.dim() == 2 else queries.reshape(1, -1)
    else:
        q = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    d = grid.dim
    if q.shape[1] != d:
        raise ShapeError(f"queries must be ({'Q'}, {d}), got {tuple(q.shape)}")
    qd = _lib.to_device_f64(q)
    vd = _lib.to_device_f64(vals).reshape(-1)
    nq = int(qd.shape[0])
    out = torch.empty(nq, dtype=torch.float64, device=qd.device)
    cc = C.c_int64(0)
    _lib.call_ws("fcg_multilinear_interp", _lib.ptr(_lib.device_knots(grid)),
                 _lib.i64_array(grid.shape), d, _lib.ptr(vd), _lib.ptr(qd), nq, _lib.ptr(out),
                 C.addressof(cc))
    res = out if on_device else _lib.to_host(out)
    return EvalResult(res, POINT_ALIGNED, {
        "method": "multilinear",
        "clamp_count": int(cc.value),
        "runtime_seconds": time.perf_counter() - t0,
    })
