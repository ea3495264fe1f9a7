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
* ``EngineConfig.max_rounds`` caps EDT rounds (EngineError, engine.py:311-317);
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
