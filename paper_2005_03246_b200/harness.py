"""Benchmark ladder with the reference's CSV schema (cli.py:163-196, ``fastcdf bench``): the
same grid rule (M ~ N through build_grid_auto, cli.py:50-61), the same jit/warm-up instance
before timing, the same row format ``task,method,dim,n,repeat,seconds`` with %.17g seconds, so
the reference's ladders and plots can be driven by this build.  Methods: ``fastsum`` (grid) and
``dnc`` (at the points); timings include the device synchronisation the numpy result implies.
"""

from __future__ import annotations

import time

import numpy as np

from .core import Bandwidth, build_grid_auto, generate_gaussian_sample

HEADER = "task,method,dim,n,repeat,seconds\n"


def grid_for(sample, n_target: int | None = None):
    """cli.py:50-61 default evaluation budget: M approximately equal to N."""
    n_target = n_target or sample.count
    per_dim = max(2, round(n_target ** (1.0 / sample.dim)))
    return build_grid_auto(sample, [per_dim] * sample.dim)


def _call(task, method, sample, grid, kernel, bw):
    from . import dnc, fastsum

    if task == "ecdf":
        return fastsum.ecdf_fastsum(sample, grid) if method == "fastsum" else dnc.ecdf_dnc(sample)
    if method == "fastsum":
        return fastsum.kde_fastsum(sample, grid, kernel, bw)
    return dnc.kde_dnc(sample, kernel, bw)


def write_rows(rows, path) -> None:
    """The reference's bench CSV (cli.py:189-192)."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(HEADER)
        for task, m, d, n, rep, dt in rows:
            fh.write(f"{task},{m},{d},{n},{rep},{dt:.17g}\n")


def bench_ladder(task: str, methods, dims, sizes, repeats: int = 3, seed: int = 1,
                 kernel=None, bandwidth: float = 0.3, out=None):
    """Time every (method, d, n) of the ladder; returns the rows (and writes them to `out`)."""
    from .kernels import laplacian

    kernel = kernel or laplacian()
    rows = []
    for d in dims:
        bw = Bandwidth.diag([bandwidth] * d)
        warm = generate_gaussian_sample(max(64, 2 ** d), d, seed)
        for m in methods:
            _call(task, m, warm, grid_for(warm), kernel, bw)
        for n in sizes:
            sample = generate_gaussian_sample(n, d, seed)
            grid = grid_for(sample, n)
            for m in methods:
                for rep in range(repeats):
                    t0 = time.perf_counter()
                    _call(task, m, sample, grid, kernel, bw)
                    rows.append((task, m, d, n, rep, time.perf_counter() - t0))
    if out is not None:
        write_rows(rows, out)
    return rows
