"""Drop-in ``build_render_graph`` / ``build_grid`` (raygauss/association.py mirror).

The association runs on the GPU (K0 camera setup, K1 fp64 PBF preprocess,
depth-ordered emit and tile radix sort); these wrappers export it into the
reference's ``RenderGraph`` / ``CSFGrid`` layouts (association.py:272-298,
353-370) so it can be compared entry for entry with the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

NEAR_LIMIT = 0.01  # association.py:36
MIN_CLAMPED_OPACITY = 0.05  # association.py:39
DEFAULT_TILE_PX = 16  # association.py:41


@dataclass
class CSFGrid:
    """association.py:272-298."""

    n_x: int
    n_y: int
    mirror_edges_x: np.ndarray
    mirror_edges_y: np.ndarray
    pixel_tile: np.ndarray

    @property
    def n_tiles(self) -> int:
        return self.n_x * self.n_y

    def window(self):
        return ((self.mirror_edges_x[0], self.mirror_edges_x[-1]), (self.mirror_edges_y[0], self.mirror_edges_y[-1]))

    def pixels_of_tile(self, tile: int):
        ys, xs = np.nonzero(self.pixel_tile == tile)
        return xs, ys


@dataclass
class RenderGraph:
    """association.py:353-370."""

    grid: CSFGrid
    order: np.ndarray
    entry_tile: np.ndarray
    ranges: np.ndarray
    mu_c: np.ndarray
    depth: np.ndarray
    keep: np.ndarray
    clamped: np.ndarray

    def tile_entries(self, tile: int) -> np.ndarray:
        return self.order[self.ranges[tile]: self.ranges[tile + 1]]

    def tile_sets(self):
        return [set(self.tile_entries(t).tolist()) for t in range(self.grid.n_tiles)]


def export_graph(ctx: _lib.Context, n: int, width: int, height: int) -> RenderGraph:
    lib = ctx._lib
    n_ent = ctypes.c_int64()
    n_x = ctypes.c_int32()
    n_y = ctypes.c_int32()
    _lib.check(lib.geer_graph_info(ctx.ptr, ctypes.byref(n_ent), ctypes.byref(n_x), ctypes.byref(n_y)))
    e, nx, ny = n_ent.value, n_x.value, n_y.value
    order = np.empty(e, dtype=np.int64)
    entry_tile = np.empty(e, dtype=np.int64)
    ranges = np.empty(nx * ny + 1, dtype=np.int64)
    mu_c = np.empty((n, 3), dtype=np.float64)
    depth = np.empty(n, dtype=np.float64)
    keep = np.empty(n, dtype=np.uint8)
    clamped = np.empty(n, dtype=np.uint8)
    pixel_tile = np.empty((height, width), dtype=np.int64)
    ex = np.empty(nx + 1, dtype=np.float64)
    ey = np.empty(ny + 1, dtype=np.float64)
    ptr = lambda a: a.ctypes.data if a.size else None
    _lib.check(lib.geer_graph_export(ctx.ptr, ptr(order), ptr(entry_tile), ptr(ranges), ptr(mu_c), ptr(depth),
                                     ptr(keep), ptr(clamped), ptr(pixel_tile), ex.ctypes.data, ey.ctypes.data))
    grid = CSFGrid(nx, ny, ex, ey, pixel_tile)
    return RenderGraph(grid=grid, order=order, entry_tile=entry_tile, ranges=ranges, mu_c=mu_c, depth=depth,
                       keep=keep.astype(bool), clamped=clamped.astype(bool))


def build_render_graph(scene, camera, lam: float = 3.0, tile_px: int = DEFAULT_TILE_PX,
                       grid: CSFGrid | None = None, *, device: int = 0) -> RenderGraph:
    """association.py:391-476 on the GPU.

    ``grid`` is accepted for signature compatibility; the GPU always rebuilds
    the camera's grid (it is a deterministic function of camera and tile_px).
    """
    from .renderer import build_graph_for

    return build_graph_for(scene, camera, lam, tile_px, device=device)


def build_grid(camera, tile_px: int = DEFAULT_TILE_PX, *, device: int = 0) -> CSFGrid:
    """association.py:301-332 on the GPU (K0)."""
    from .scene import GaussianScene

    return build_render_graph(GaussianScene.empty(1), camera, 3.0, tile_px, device=device).grid
