"""Structured Dirichlet grids and the finite-difference heat operator.

Mirrors ``heat.py`` of the reference: interior unknowns only, C order with
x fastest.  ``HeatOperator.apply`` / ``diagonal`` run the sm_100a stencil
kernels (csrc/stencil.cu); inputs may be numpy arrays (returned as numpy,
drop-in) or fp64 CUDA tensors (returned on the device).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from ._device import like_input, new_field, ptr, require_field, stream_ptr, to_device


@dataclass(frozen=True)
class Grid:
    """``n`` cells per dimension on [0, length]^dim (heat.py:16-52)."""

    dim: int
    n: int
    length: float = 1.0

    def __post_init__(self):
        if self.dim not in (1, 2, 3):
            raise ValueError(f"dim must be 1, 2, or 3, got {self.dim}")
        if self.n < 2 or self.n & (self.n - 1):
            raise ValueError(f"n must be a power of two >= 2, got {self.n}")

    @property
    def dx(self) -> float:
        return self.length / self.n

    @property
    def shape(self) -> tuple:
        return (self.n - 1,) * self.dim

    @property
    def dof(self) -> int:
        return (self.n - 1) ** self.dim

    def interior_coords(self) -> np.ndarray:
        return self.dx * np.arange(1, self.n)

    def coarsen(self) -> "Grid":
        if self.n < 4:
            raise ValueError(f"grid with n={self.n} cannot be coarsened")
        return Grid(self.dim, self.n // 2, self.length)

    def zeros(self):
        return np.zeros(self.shape)


def initial_condition(grid: Grid, k: int) -> np.ndarray:
    """Product of sine modes sin(k pi x / L) at interior points (heat.py:55-62).
    Host-side synthetic input."""
    axis = np.sin(k * np.pi * grid.interior_coords() / grid.length)
    u = axis
    for _ in range(grid.dim - 1):
        u = np.multiply.outer(u, axis)
    return u


def seeded_field(grid: Grid, seed: int = 1407, modes: int = 16, kmax: int = 32,
                 amp: float = 1e-2) -> np.ndarray:
    """u0 of BASELINE configs 2-4: sin-product base mode plus
    ``modes`` seeded Fourier modes; for each mode, k = rng.integers(1, kmax+1,
    size=dim) then a = rng.uniform(0, amp).  Host-side synthetic input."""
    rng = np.random.default_rng(seed)
    x = grid.interior_coords()
    u = initial_condition(grid, 1)
    for _ in range(modes):
        k = rng.integers(1, kmax + 1, size=grid.dim)
        a = rng.uniform(0, amp)
        term = np.sin(int(k[0]) * np.pi * x / grid.length)
        for d in range(1, grid.dim):
            term = np.multiply.outer(term, np.sin(int(k[d]) * np.pi * x / grid.length))
        u = u + a * term
    return u


@dataclass(frozen=True)
class HeatOperator:
    """nu times the order-2 / order-4 discrete Laplacian (heat.py:95-158)."""

    grid: Grid
    nu: float = 1.0
    order: int = 2

    def __post_init__(self):
        if self.order not in (2, 4):
            raise ValueError(f"stencil order must be 2 or 4, got {self.order}")

    def _args(self):
        g = self.grid
        return g.dim, g.n, float(g.length), float(self.nu), self.order

    def apply_into(self, u, out):
        """out = nu Lap_h u for device tensors (no allocation)."""
        require_field(u, self.grid.dim, "HeatOperator.apply_into(u)")
        require_field(out, self.grid.dim, "HeatOperator.apply_into(out)")
        capi.check(capi.lib().pl_heat_apply(ptr(u), ptr(out), *self._args(), stream_ptr()),
                   "HeatOperator.apply")
        return out

    def apply(self, u):
        if tuple(np.shape(u)) != self.grid.shape:
            raise ValueError(f"expected shape {self.grid.shape}, got {tuple(np.shape(u))}")
        t, host = to_device(u, self.grid.dim)
        out = new_field(self.grid.shape)
        self.apply_into(t, out)
        return like_input(out, host)

    def diagonal(self, as_numpy: bool = True):
        out = new_field(self.grid.shape)
        capi.check(capi.lib().pl_heat_diagonal(ptr(out), *self._args(), 0.0, 0, stream_ptr()),
                   "HeatOperator.diagonal")
        return like_input(out, as_numpy)
