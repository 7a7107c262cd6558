"""Run results with the reference's metric schema (runtime.py:105-127, 183-187).

On the B200 path a "rank" is a GPU (count_space_surrogate) or a logical
worker of the device task queue (count_dynamic); the counters keep the
reference's meaning so results are comparable field by field.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

WORD_BYTES = 8  # wire cost model, runtime.py:32


@dataclass
class RankMetrics:
    rank: int
    nranks: int
    triangles: int = 0
    data_msgs_sent: int = 0
    bytes_sent: int = 0
    requests_sent: int = 0
    completion_msgs_sent: int = 0
    tasks_executed: int = 0
    idle_poll_cycles: int = 0
    busy_time: float = 0.0
    idle_time: float = 0.0
    partition_bytes: int = 0
    data_msgs_to: np.ndarray = None
    requests_to: np.ndarray = None
    task_log: list = field(default_factory=list)
    # B200 extension (not in the reference): bytes this rank actually moved
    # through its collectives (the counters above keep the reference's
    # per-message wire model, runtime.py:139-149).
    wire_bytes: int = 0

    def __post_init__(self):
        if self.data_msgs_to is None:
            self.data_msgs_to = np.zeros(self.nranks, dtype=np.int64)
        if self.requests_to is None:
            self.requests_to = np.zeros(self.nranks, dtype=np.int64)


@dataclass
class RunResult:
    results: list
    metrics: list
    wall: float  # seconds (device time of the counting phase)
