"""Engine / queue configuration types (reference: engine.py:46-69,
wqueue.py:48-73).

The reference schedules propagation on CPU workers with a round-based
hierarchical queue; here every operator runs on the B200 engines, so these
dataclasses are accepted for drop-in compatibility and mapped onto device
knobs:

* ``EngineConfig.n_workers`` / ``QueueConfig.strategy`` / ``tq/bq
  capacities`` do not change results (unique fixed point for
  reconstruction; canonical round schedule for the EDT) and are ignored by
  the device engines;
* ``QueueConfig.gbq_capacity`` bounds the device block queue (smaller
  values force the overflow -> rescan -> re-execute path, the reference's
  fault-injection knob, test_acceptance.py:218-231);
* ``EngineConfig.max_rounds`` caps the rounds of one execution (EngineError,
  engine.py:311-317): EDT rounds, and for reconstruction the device engine's
  tile activations per tile (its counterpart of a round: each activation
  runs one tile to its local fixed point);
* ``EngineConfig.stats`` receives the device counters.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .errors import ContractViolation

DEFAULT_TQ_CAPACITY = 32
DEFAULT_BQ_CAPACITY = 1024
MIN_GBQ_CAPACITY = 1024
GBQ_HEADROOM = 1.1

BACKENDS = ("auto", "b200", "compiled", "threads", "serial")


class QueueStrategy(Enum):
    NAIVE = "naive"
    PREFIX_SUM = "prefix"
    PER_WORKER = "perworker"


@dataclass
class QueueConfig:
    strategy: QueueStrategy = QueueStrategy.PER_WORKER
    tq_capacity: int = DEFAULT_TQ_CAPACITY
    bq_capacity: int = DEFAULT_BQ_CAPACITY
    gbq_capacity: int | None = None


def auto_gbq_capacity(n_initial: int) -> int:
    """wqueue.py:72-73: max(1.1 * seeds + 1, 1024)."""
    return max(int(GBQ_HEADROOM * n_initial) + 1, MIN_GBQ_CAPACITY)


@dataclass
class RunStats:
    """Counters (engine.py:46-59) plus the device engine's own."""

    rounds: int = 0
    executions: int = 0
    overflow_count: int = 0
    queued_total: int = 0
    tiles_processed: int = 0
    tile_reruns: int = 0
    seeds: int = 0

    def reset(self):
        for k in self.__dataclass_fields__:
            setattr(self, k, 0)

    def add(self, d: dict):
        for k in ("rounds", "executions", "overflow_count", "queued_total",
                  "tiles_processed", "tile_reruns", "seeds"):
            setattr(self, k, getattr(self, k) + int(d.get(k, 0)))


@dataclass
class EngineConfig:
    n_workers: int = 1
    queue: QueueConfig = field(default_factory=QueueConfig)
    backend: str = "auto"
    max_rounds: int | None = None
    stats: RunStats = field(default_factory=RunStats)

    def validate(self):
        if self.n_workers < 1:
            raise ContractViolation("n_workers must be >= 1")
        if self.backend not in BACKENDS:
            raise ContractViolation(f"unknown backend {self.backend!r}")
        if self.queue.gbq_capacity is not None and self.queue.gbq_capacity < 1:
            raise ContractViolation("gbq_capacity must be >= 1")


class PropagationRule:
    """The reference's rule plugin interface (engine.py:72-178), kept so
    callers can name, subclass and pass rules exactly as with gridwave.

    A rule binds state arrays and defines, on packed flat indices, when a
    cell p improves its neighbour q (``condition``), the value it offers
    (``propose``) and whether a value beats the held one (``improves``);
    synchronous rules also take offers from round-start snapshots
    (``gather`` / ``condition_from`` / ``propose_from``).

    The B200 engines implement the two rules the package ships --
    ``recon.ReconRule`` (K.193-303) and ``edt.DistanceRule`` (K.309-433) --
    as fused kernels; ``tiles.run_pipeline`` dispatches on those types.
    Per-item Python hooks are far too fine-grained to drive a GPU (SURVEY
    8(b)), so a custom subclass raises ``ContractViolation`` there instead of
    silently running on the CPU.  The hooks below are the rule's semantics,
    usable for inspection and small host-side checks.
    """

    #: history-sensitive rules (two-phase rounds): offers use round-start values
    synchronous = False

    def __init__(self, width: int, height: int, se, bounds=None):
        self.width = width
        self.height = height
        self.se = se
        self.bounds = bounds if bounds is not None else (0, 0, width, height)

    def read(self, q: int):
        raise NotImplementedError

    def write(self, q: int, value) -> None:
        raise NotImplementedError

    def condition(self, p: int, q: int) -> bool:
        raise NotImplementedError

    def propose(self, p: int, q: int):
        raise NotImplementedError

    def improves(self, q: int, old, new) -> bool:
        raise NotImplementedError

    def gather(self, items):
        return [self.read(int(p)) for p in items]

    def condition_from(self, v, p: int, q: int) -> bool:
        raise NotImplementedError

    def propose_from(self, v, p: int, q: int):
        raise NotImplementedError

    def rebound(self, bounds) -> "PropagationRule":
        raise NotImplementedError

    def iter_neighbors(self, p: int):
        """In-window neighbours of p in the structuring element's raster order."""
        x0, y0, x1, y1 = self.bounds
        w = self.width
        px, py = p % w, p // w
        for dx, dy in self.se.offsets:
            nx, ny = px + dx, py + dy
            if x0 <= nx < x1 and y0 <= ny < y1:
                yield ny * w + nx

    def seed_scan(self) -> list:
        """Cells that could propagate now, raster order (the restart set)."""
        x0, y0, x1, y1 = self.bounds
        out = []
        for y in range(y0, y1):
            for x in range(x0, x1):
                p = y * self.width + x
                if any(self.condition(p, q) for q in self.iter_neighbors(p)):
                    out.append(p)
        return out

    # the reference's optional compiled hooks: the device engines replace them
    def kernel_wavefront(self, seeds):
        return None

    def kernel_round_block(self, items, start, stride, payload=None):
        return None

    def kernel_seed_scan(self):
        return None

    def has_round_kernel(self) -> bool:
        return False
