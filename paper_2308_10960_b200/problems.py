"""Synthetic model problems of BASELINE.json (host setup; not on the hot path).

The reference ships icosphere centroids, random sphere points, an area-weighted
Laplace SLP and a Bessel-based Matern kernel (geometry.cpp, kernels.cpp); the
BASELINE configs name other geometries and kernels, added here behind the same
"entry(i, j)" idea as kernel::KernelEvaluator (kernels.hpp:21-27):

  * Fibonacci sphere with seeded jitter (config 1/3/5)
  * uniform points in the unit cube (config 4)
  * Laplace 1/(4 pi |x-y|), self term 0 (config 1/3)
  * Matern nu=1.5, closed form sigma^2 (1 + sqrt3 d/l) exp(-sqrt3 d/l) (config 4;
    equal to MaternCovariance{1, l, 1.5} up to rounding, kernels.cpp:58-66)
  * random sphere points as in geometry.cpp:22-34

All inputs are seeded (numpy PCG64 unless noted), generated once on the host.
"""
from __future__ import annotations

import math

import numpy as np
import torch


def fibonacci_sphere(n: int, jitter: float = 1e-3, seed: int = 1) -> np.ndarray:
    """z_i = 1 - (2i+1)/n, phi_i = i pi (3 - sqrt5), + U[-jitter, jitter]^3, reprojected"""
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * math.pi * (3.0 - math.sqrt(5.0))
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    p = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)
    if jitter:
        rng = np.random.default_rng(seed)
        p = p + rng.uniform(-jitter, jitter, size=p.shape)
        p /= np.linalg.norm(p, axis=1, keepdims=True)
    return p


def unit_cube(n: int, seed: int = 1) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, size=(n, 3))


def random_sphere(n: int, seed: int = 1) -> np.ndarray:
    """area-preserving cylindrical map (geometry.cpp:22-34), numpy RNG"""
    rng = np.random.default_rng(seed)
    z = 2.0 * rng.uniform(size=n) - 1.0
    phi = 2.0 * math.pi * rng.uniform(size=n)
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def _dist(a: torch.Tensor, b: torch.Tensor, separated: bool) -> torch.Tensor:
    """pairwise distances; `separated` (admissible blocks: the clusters are at least
    diam / eta apart) takes the GEMM form |a|^2 + |b|^2 - 2 a.b, exact to ~1e-15
    relative there and far faster on large blocks; near-field blocks keep the
    difference form (no cancellation for close points)"""
    if separated:
        return torch.cdist(a, b, compute_mode="use_mm_for_euclid_dist")
    return torch.cdist(a, b, compute_mode="donot_use_mm_for_euclid_dist")


class PointKernel:
    """entry(x, y) evaluated on blocks of points (torch, any device, FP64)"""
    name = "kernel"

    def block(self, a: torch.Tensor, b: torch.Tensor, separated: bool = False) -> torch.Tensor:
        """a: [..., m, 3], b: [..., n, 3] -> [..., m, n]"""
        raise NotImplementedError


class Laplace(PointKernel):
    name = "laplace"

    def block(self, a, b, separated=False):
        d = _dist(a, b, separated)
        out = torch.where(d > 0, 1.0 / (4.0 * math.pi * d), torch.zeros_like(d))
        return out


class Matern15(PointKernel):
    name = "matern"

    def __init__(self, length: float = 0.1, sigma2: float = 1.0):
        self.length, self.sigma2 = length, sigma2

    def block(self, a, b, separated=False):
        d = _dist(a, b, separated)
        t = math.sqrt(3.0) * d / self.length
        return self.sigma2 * (1.0 + t) * torch.exp(-t)


class Helmholtz(PointKernel):
    """exp(i kappa |x - y|) / (4 pi |x - y|), self term 0 (BASELINE config 5;
    complex FP64 -- assemble_complex splits it into real / imaginary parts)"""
    name = "helmholtz"
    complex = True

    def __init__(self, kappa: float = 16.0):
        self.kappa = kappa

    def block(self, a, b, separated=False):
        d = _dist(a, b, separated)
        inv = torch.where(d > 0, 1.0 / (4.0 * math.pi * torch.where(d > 0, d, torch.ones_like(d))),
                          torch.zeros_like(d))
        return torch.polar(inv, self.kappa * d)


def config(name: str) -> dict:
    """BASELINE.json configs (index 0..4) as build parameters"""
    name = str(name)
    table = {
        "1": dict(geometry="fibonacci", n=8192, kernel="laplace", eps=1e-6, leaf=64, eta=2.0),
        "3": dict(geometry="fibonacci", n=131072, kernel="laplace", eps=1e-8, leaf=64, eta=2.0),
        "4": dict(geometry="cube", n=524288, kernel="matern", eps=1e-6, leaf=64, eta=2.0),
        "5": dict(geometry="fibonacci", n=262144, kernel="helmholtz", eps=1e-6, leaf=64, eta=2.0, nrhs=16),
    }
    return dict(table[name])


def make_points(geometry: str, n: int, seed: int = 1) -> np.ndarray:
    if geometry == "fibonacci":
        return fibonacci_sphere(n, 1e-3, seed)
    if geometry == "cube":
        return unit_cube(n, seed)
    if geometry == "sphere":
        return random_sphere(n, seed)
    raise ValueError(f"unknown geometry {geometry}")


def make_kernel(name: str) -> PointKernel:
    if name == "laplace":
        return Laplace()
    if name == "matern":
        return Matern15(0.1, 1.0)
    if name == "helmholtz":
        return Helmholtz(16.0)
    raise ValueError(f"unknown kernel {name}")
