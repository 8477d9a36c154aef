"""Native engine queue for the topology-aware scheduler (C ABI `tsv_topo_*`, csrc/tsv_sched.cpp).

`runtime.form_batch_topo` mirrors the reference's batch formation
(pkg/src/teola_sim/runtime.py:208-261) over the Python task objects and rebuilds its buckets
from every queued task on every call; `_dispatch` then filters the whole queue
(runtime.py:608). With thousands of queued stage tasks — the embedding and LLM engines of a
workflow with tens of queries in flight — that was most of the real-time runtime's host time
(scripts/host_profile.py). `TopoQueue` keeps the queue in native memory: a task's static fields
and request loads are pushed once, `form` returns the same BatchPlan the mirror forms (the 300
reference snapshots and the reference's full traces are checked through both), `commit`
consumes a dispatched batch and drops drained tasks in O(entries)."""

from __future__ import annotations

import ctypes
import itertools
from array import array

from . import _native as nat
from .errors import ConfigParse

PHASE_CODES = {"general": 0, "prefill": 1, "decode": 2}
PHASE_NAMES = {v: k for k, v in PHASE_CODES.items()}


class TopoQueue:
    def __init__(self, eps: float = 1e-9):
        self._lib = nat.load()
        h = ctypes.c_void_p()
        nat.check(self._lib.tsv_topo_create(float(eps), ctypes.byref(h)))
        self._h = h
        self._tasks: dict[int, object] = {}
        self._ids = itertools.count(1)
        self._cap = 0
        self._grow(64)
        self._n = ctypes.c_int64()
        self._load = ctypes.c_double()
        self._phase = ctypes.c_int()

    def _grow(self, cap: int) -> None:
        self._cap = cap
        self._handles = (ctypes.c_int64 * cap)()
        self._counts = (ctypes.c_int64 * cap)()

    def __len__(self) -> int:
        return len(self._tasks)

    def tasks(self) -> list:
        return list(self._tasks.values())

    def push(self, task) -> None:
        """Queue a NodeTask (fields as in runtime.NodeTask; read once)."""
        h = next(self._ids)
        loads = array("d", task.loads)
        ptr = loads.buffer_info()[0] if len(loads) else None
        phase = PHASE_CODES.get(task.phase)
        if phase is None:
            raise ConfigParse(f"unknown phase {task.phase!r}")
        nat.check(self._lib.tsv_topo_push(
            self._h, h, task.ctx.query_id.encode(), task.node.node_id.encode(), int(task.depth),
            phase, float(task.arrival_ms), ptr, len(loads), int(task.next_request)))
        task._topo_handle = h
        self._tasks[h] = task

    def form(self, max_slots: float):
        """One batch under `max_slots` (runtime.form_batch_topo's decisions)."""
        from .runtime import BatchPlan

        while True:
            rc = self._lib.tsv_topo_form(self._h, float(max_slots), self._cap, self._handles,
                                         self._counts, ctypes.byref(self._n),
                                         ctypes.byref(self._load), ctypes.byref(self._phase))
            if rc == 0:
                break
            if self._n.value > self._cap:
                self._grow(max(self._n.value, 2 * self._cap))
                continue
            nat.check(rc)
        plan = BatchPlan()
        n = self._n.value
        if n == 0:
            return plan
        tasks = self._tasks
        hs, cs = self._handles, self._counts
        plan.entries = [(tasks[hs[i]], cs[i]) for i in range(n)]
        plan.load = self._load.value
        plan.phase = PHASE_NAMES[self._phase.value]
        return plan

    def commit(self, entries) -> None:
        """A dispatched batch's entries [(task, n)] (after their next_request advanced)."""
        m = len(entries)
        if m > self._cap:
            self._grow(m)
        hs, cs = self._handles, self._counts
        for i, (task, n) in enumerate(entries):
            hs[i] = task._topo_handle
            cs[i] = n
        nat.check(self._lib.tsv_topo_commit(self._h, hs, cs, m))
        for task, _ in entries:
            if task.pending() <= 0:
                self._tasks.pop(task._topo_handle, None)

    def close(self) -> None:
        if self._h is not None and self._h.value:
            self._lib.tsv_topo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
