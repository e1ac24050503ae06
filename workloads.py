"""Seeded synthetic inputs for the five BASELINE.json configurations.

Shared by bench.py, the tests and tests/golden/make_golden.py.  Everything is generated with
numpy elementwise arithmetic only (no BLAS), so the same seed yields bit-identical inputs on the
build container and on any GPU box running this image.  BASELINE names no public dataset; the
reference paper itself uses synthetic Gaussian inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEEDS = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5}


@dataclass
class Workload:
    name: str
    points: np.ndarray
    weights: np.ndarray | None          # None = unit weights (y == 1)
    knots: list | None = None           # grid configs
    delta: tuple | None = None
    h: np.ndarray | None = None
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.points.shape[0])

    @property
    def d(self) -> int:
        return int(self.points.shape[1])


def gaussian_sample_points(n: int, d: int, seed: int) -> np.ndarray:
    """Reference generator (core.py:311-347) via the package's bit-identical restatement."""
    from paper_2005_03246_b200.core import generate_gaussian_sample

    return generate_gaussian_sample(n, d, seed).points


def cfg1(n: int = 65_536, m: int = 256) -> Workload:
    """2-D grid ECDF: N(0, I_2) from the reference generator, y == 1, delta = (1, 1),
    256 x 256 grid on [-4, 4]^2."""
    x = gaussian_sample_points(n, 2, SEEDS["cfg1"])
    kn = np.linspace(-4.0, 4.0, m)
    return Workload("cfg1", x, None, [kn, kn.copy()], (1, 1))


def cfg2(n: int = 1_000_000, levels: int = 1024) -> Workload:
    """2-D ECDF at the points: Uniform[0,1]^2 quantised to multiples of 1/1024 (ties),
    y ~ U(0,1), delta = (1, -1), plus the ESF."""
    rng = np.random.default_rng(SEEDS["cfg2"])
    x = np.floor(rng.random((n, 2)) * levels) / levels
    y = rng.random(n)
    return Workload("cfg2", x, y, None, (1, -1))


def _cfg3_points(n: int, rng) -> np.ndarray:
    z = rng.standard_normal((n, 3))
    # Cholesky factor of the unit-variance, 0.5-correlation matrix, written out analytically
    # (elementwise only, no BLAS) so every host produces identical bits.
    l10 = 0.5
    l11 = math.sqrt(0.75)
    l20 = 0.5
    l21 = 0.25 / l11
    l22 = math.sqrt(1.0 - l20 * l20 - l21 * l21)
    x = np.empty_like(z)
    x[:, 0] = z[:, 0]
    x[:, 1] = l10 * z[:, 0] + l11 * z[:, 1]
    x[:, 2] = (l20 * z[:, 0] + l21 * z[:, 1]) + l22 * z[:, 2]
    return x


def cfg3(n: int = 10_000_000, m: int = 512) -> Workload:
    """3-D grid ECDF: correlated Gaussian (rho = 0.5), y == 1, delta = (1,1,1), 512^3 grid on
    [-4, 4]^3."""
    rng = np.random.default_rng(SEEDS["cfg3"])
    x = _cfg3_points(n, rng)
    kn = np.linspace(-4.0, 4.0, m)
    return Workload("cfg3", x, None, [kn, kn.copy(), kn.copy()], (1, 1, 1))


def cfg4(n: int = 10_000_000) -> Workload:
    """2-D Laplacian KDE + kernel regression at the points: 4-component Gaussian mixture,
    h = 0.1, w == 1 (density) and y = sin(3 x1) + cos(2 x2) + N(0, 0.1^2) (regression)."""
    rng = np.random.default_rng(SEEDS["cfg4"])
    comp = rng.integers(0, 4, n)
    means = np.array([[-1.5, -1.5], [-1.5, 1.5], [1.5, -1.5], [1.5, 1.5]])
    x = means[comp] + 0.5 * rng.standard_normal((n, 2))
    y = np.sin(3.0 * x[:, 0]) + np.cos(2.0 * x[:, 1]) + 0.1 * rng.standard_normal(n)
    return Workload("cfg4", x, None, None, None, np.array([0.1, 0.1]), {"y": y})


def nd3(n: int = 1_000_000) -> Workload:
    """Not a BASELINE config (SURVEY §8f #3 widening): config 4's problem in three dimensions --
    Laplacian KDE + kernel regression at the points, 8-component Gaussian mixture, h = 0.2."""
    rng = np.random.default_rng(43)
    comp = rng.integers(0, 8, n)
    means = np.array([[a, b, c] for a in (-1.5, 1.5) for b in (-1.5, 1.5) for c in (-1.5, 1.5)])
    x = means[comp] + 0.5 * rng.standard_normal((n, 3))
    y = np.sin(3.0 * x[:, 0]) + np.cos(2.0 * x[:, 1]) + x[:, 2] + 0.1 * rng.standard_normal(n)
    return Workload("nd3", x, None, None, None, np.array([0.2, 0.2, 0.2]), {"y": y})


def cfg5(n: int = 100_000_000, m: int = 128, dtype_chunk: int = 0) -> Workload:
    """4-D grid ECDF (y == 1) + Laplacian KDE (y ~ Exp(1), h = 0.05): Uniform[0,1]^4,
    128^4 grid on [0, 1]^4."""
    rng = np.random.default_rng(SEEDS["cfg5"])
    x = rng.random((n, 4))
    y = rng.exponential(1.0, n)
    kn = np.linspace(0.0, 1.0, m)
    return Workload("cfg5", x, None, [kn, kn.copy(), kn.copy(), kn.copy()], (1, 1, 1, 1),
                    np.full(4, 0.05), {"y": y})


def digest(a: np.ndarray) -> str:
    import hashlib

    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.view(np.uint8).reshape(-1)).hexdigest()
