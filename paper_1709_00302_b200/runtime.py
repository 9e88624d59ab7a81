"""Execution-group compatibility shim (ref runtime.py).

The reference runs each phase on a sequential group T_S and a parallel
group T_P of Python threads (ref runtime.py:142-180, 191-244). On the B200
those groups are the library's `panel` and `main` CUDA streams inside one
context, so an `ExecGroups` object only carries the *choice*: ts_count == 0
means no overlap (the reference degenerates to one pool, runtime.py:214-222),
which maps to look-ahead depth 0. It is accepted wherever the reference
accepts `groups` so call sites stay unchanged.
"""
from __future__ import annotations

import threading


class EventTrace:
    """Task records (task_id, group, start, end) like the reference's
    EventTrace (ref runtime.py:76-104). On the GPU the records come from CUDA
    events around each task: group "seq" = panel stream, "par" = main stream,
    start/end in microseconds of device time since the reduction began."""

    def __init__(self):
        self._lock = threading.Lock()
        self.records = []

    def append(self, task_id, group, start, end):
        with self._lock:
            self.records.append((task_id, group, start, end))

    def of_group(self, group):
        return [r for r in self.records if r[1] == group]

    def find(self, prefix):
        return [r for r in self.records if r[0].startswith(prefix)]

    def dump(self, path):
        with open(path, "w") as f:
            for task_id, group, start, end in self.records:
                f.write(f"{task_id}\t{group}\t{start}\t{end}\n")


class ExecGroups:
    def __init__(self, total_workers: int = 1, ts_count: int = 1):
        if total_workers < 1:
            raise ValueError("total_workers >= 1")
        if not (0 <= ts_count <= total_workers):
            raise ValueError("0 <= ts_count <= total_workers")
        self.total = int(total_workers)
        self.ts_count = int(ts_count)
        self.tp_count = self.total - self.ts_count
        self.trace = EventTrace()

    @property
    def overlap(self) -> bool:
        return self.ts_count > 0

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


class WriteOverlapError(ValueError):
    """Declared write ranges of the two groups of one phase intersect
    (ref runtime.py:34-35). The GPU schedules are disjoint by construction."""
