"""Kernel descriptors consumed by the KDE entry points.

Only the descriptor contract of the reference's ``KernelSpec`` (kernels.py:33-72) is kept: the
hot path reads ``family`` alone.  The CDF-decomposable family evaluated on the GPU is the
Laplacian (Eq. 12); the other reference families are accepted as descriptors so that the
entry points can raise the reference's ParameterError for them (fastsum.py:223-227,
dnc.py:647-651).  Quadrature, normalizers and bandwidth rotation are outside the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import ParameterError

FAMILIES = (
    "laplacian",
    "uniform",
    "beta",
    "polyexp",
    "matern",
    "matern32-additive",
    "matern32-product",
    "fourth-order-laplacian",
    "gaussian",
)


@dataclass(frozen=True)
class KernelSpec:
    family: str
    params: tuple = ()

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ParameterError(f"unknown kernel family {self.family!r}")

    def __str__(self) -> str:
        if not self.params:
            return self.family
        return self.family + ":" + ",".join(str(p) for p in self.params)


def laplacian() -> KernelSpec:
    return KernelSpec("laplacian")


def uniform() -> KernelSpec:
    return KernelSpec("uniform")


def gaussian() -> KernelSpec:
    return KernelSpec("gaussian")


def matern32_additive() -> KernelSpec:
    return KernelSpec("matern32-additive")


def matern32_product() -> KernelSpec:
    return KernelSpec("matern32-product")


def parse_kernel_spec(text: str) -> KernelSpec:
    """Accept the reference's ``family[:params]`` grammar (kernels.py:325-374) head."""
    head, _, tail = text.strip().partition(":")
    fam = head.strip().lower()
    if fam not in FAMILIES:
        raise ParameterError(f"unknown kernel family in spec {text!r}")
    return KernelSpec(fam, tuple(p for p in tail.split(",") if p) if tail else ())
