"""Tiling types (reference: gridwave/tiles.py).

On one B200 the persistent tile engine owns tiling (64x64 tiles, global
tile queue, asynchronous border exchange), so ``recon_tiled``/``edt_tiled``
ignore ``tile_dims`` for scheduling (the result is identical by the
reference's own contract, tiles.py:1-20).  ``partition``/``TileGrid`` keep
the reference's arithmetic for callers and for the multi-GPU slab planner
(``paper_1209_3314_b200.distributed``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import ContractViolation


@dataclass
class Tile:
    id: int
    x0: int
    y0: int
    x1: int
    y1: int
    state: str = "idle"

    @property
    def bounds(self):
        return (self.x0, self.y0, self.x1, self.y1)


@dataclass
class TileGrid:
    width: int
    height: int
    tile_w: int
    tile_h: int
    tiles: list

    @property
    def shape(self):
        """(columns, rows) of the tile lattice."""
        return -(-self.width // self.tile_w), -(-self.height // self.tile_h)

    def tile_at(self, x: int, y: int) -> int:
        return (y // self.tile_h) * self.shape[0] + (x // self.tile_w)


def partition(image, tile_w: int, tile_h: int) -> TileGrid:
    """tiles.py:78-90: raster-ordered ceil(W/tw) x ceil(H/th) cover; edge
    tiles may be smaller."""
    if tile_w < 1 or tile_h < 1:
        raise ContractViolation("tile dimensions must be >= 1")
    W, H = image.width, image.height
    tiles = [Tile(i, x0, y0, min(x0 + tile_w, W), min(y0 + tile_h, H))
             for i, (y0, x0) in enumerate((y, x) for y in range(0, H, tile_h)
                                          for x in range(0, W, tile_w))]
    return TileGrid(W, H, tile_w, tile_h, tiles)


@dataclass
class MicroConfig:
    n_bands: int = 1


@dataclass
class PipelineConfig:
    """tiles.py:365-372.  ``n_workers`` is accepted for compatibility; on
    the device the engine sizes its own persistent grid."""

    n_workers: int = 1
    micro: MicroConfig | None = None
    max_waves: int | None = None
    pool: object = None
    events: list = field(default_factory=list)
    bp_waves: int = 0
