"""Tiling types and the wave pipeline (reference: gridwave/tiles.py).

On one B200 the persistent tile engine owns tiling (32x32 tiles, global
tile queue, asynchronous border exchange), so ``run_pipeline`` -- and with
it ``recon_tiled``/``edt_tiled`` -- ignores ``tile_dims`` for scheduling
(the result is identical by the reference's own contract, tiles.py:1-20).
Across GPUs (an initialised torch.distributed group, one rank per GPU) the
pipeline's waves are the slab waves of ``distributed``: each rank owns a
horizontal slab, border rows travel between neighbours after every wave,
and an all-reduce of the changed-border count ends the loop.
``partition``/``TileGrid`` keep the reference's arithmetic for callers.
"""

from __future__ import annotations

import json
import time
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
class EventRecord:
    """One pipeline task (tiles.py:96-112).  On the device a "TP" task is
    one engine run (all tiles of a wave at once, tile_id -1), a "BP" task
    one border exchange of the slab protocol."""

    task_id: int
    kind: str
    wave: int
    tile_id: int
    worker: int
    start: float
    end: float

    def to_line(self) -> str:
        return json.dumps({"task": self.task_id, "kind": self.kind, "wave": self.wave,
                           "tile": self.tile_id, "worker": self.worker,
                           "start": self.start, "end": self.end})


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


def _dist_world():
    """(group world size, rank) of an initialised torch.distributed group,
    or (1, 0)."""
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover
        return 1, 0
    if not (dist.is_available() and dist.is_initialized()):
        return 1, 0
    return dist.get_world_size(), dist.get_rank()


def run_pipeline(image, rule, initial_seed_fn, tile_dims, cfg: PipelineConfig | None = None):
    """tiles.py:375-431: propagate ``rule`` over ``image`` until no tile
    has work left; returns the mutated image (the object the rule works on).

    The device runs the two rules the package ships:

    * ``recon.ReconRule``: the rule's fixed point -- the unique
      reconstruction of the rule's current J under its mask -- computed by
      the tile engine in place on ``rule.J``.  ``initial_seed_fn`` names the
      active set the reference's waves start from; the engine detects that
      set itself (a full seed scan), which is the same set whenever the
      function returns every active cell, as recon_tiled's does
      (recon.py:316-322).
    * ``edt.DistanceRule``: two-phase rounds from the seeds
      ``initial_seed_fn()`` returns, in place on ``rule.vr``
      (``edt_propagate``; tiles.py:305-331 advances one round per wave,
      which is the same canonical schedule).

    ``cfg.max_waves`` caps the waves (ContractViolation), ``cfg.bp_waves``
    reports them, ``cfg.events`` receives one record per task.  One device
    needs a single wave; under a torch.distributed group a ReconRule runs as
    slab waves across the ranks.
    """
    from .edt import DistanceRule, edt_propagate
    from .recon import ReconRule, reconstruct

    cfg = cfg or PipelineConfig()
    partition(image, *tile_dims)  # the reference's tile-dimension contract
    cfg.bp_waves = 0
    if cfg.max_waves is not None and cfg.max_waves < 1:
        raise ContractViolation(f"no stability within {cfg.max_waves} waves")
    world, rank = _dist_world()
    t0 = time.perf_counter()
    if isinstance(rule, ReconRule):
        kind = getattr(rule, "elem_kind", None) or getattr(image, "elem_kind", None)
        conn = rule.se.connectivity
        if world > 1:
            from .distributed import recon_slabs
            out, st = recon_slabs(rule.J, rule.I, conn, max_waves=cfg.max_waves)
            waves = st.waves
        else:
            out = reconstruct(rule.J, rule.I, conn, kind=kind)
            waves = 1
        if hasattr(rule.J, "copy_"):
            rule.J.copy_(out)
        else:
            rule.J[...] = out
    elif isinstance(rule, DistanceRule):
        from .edt import VoronoiMap
        seeds = initial_seed_fn()
        vmap = VoronoiMap(rule.width, rule.height, rule.vr)
        edt_propagate(vmap, seeds if seeds is not None else [], rule.se)
        waves = 1
    else:
        raise ContractViolation(
            f"{type(rule).__name__}: the B200 pipeline runs ReconRule and DistanceRule "
            "(per-cell Python hooks cannot drive the device engines)")
    t1 = time.perf_counter()
    cfg.bp_waves = waves
    for w in range(waves):
        cfg.events.append(EventRecord(2 * w, "TP", w, -1, rank, t0, t1))
        cfg.events.append(EventRecord(2 * w + 1, "BP", w, -1, rank, t1, t1))
    return image
