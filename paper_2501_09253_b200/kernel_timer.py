"""Per-entry-point CUDA-event timing of library calls (measurement only: bench.py, tools).

`KernelTimer(names, flush_bytes)` installed as `_lib.TIMER` brackets every call of the
named C entry points with CUDA events on the current stream.  With `flush_bytes` > 0 it
first READS a buffer that large (bigger than the 126 MB L2; a read leaves no dirty lines to
write back inside the timed launch) so each timed launch starts cold, the way the kernel's
inputs arrive in a real step once the previous stage's output no longer fits L2; the flush is
outside the event pair.
"""

from __future__ import annotations

from collections import defaultdict

import torch

from . import _lib


class KernelTimer:
    def __init__(self, names, flush_bytes: int = 0):
        self.names = set(names)
        self.events = defaultdict(list)
        self._open = {}
        self._flush = (torch.ones(flush_bytes // 4, dtype=torch.float32, device="cuda")
                       if flush_bytes else None)
        self._sink = None

    def wants(self, name: str) -> bool:
        return name in self.names

    def before(self, name: str) -> None:
        if self._flush is not None:
            self._sink = self._flush.sum()
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self._open[name] = e

    def after(self, name: str) -> None:
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events[name].append((self._open.pop(name), e))

    def times_ms(self) -> dict:
        torch.cuda.synchronize()
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.events.items()}

    def __enter__(self):
        self._prev = _lib.TIMER
        _lib.TIMER = self
        return self

    def __exit__(self, *exc):
        _lib.TIMER = self._prev
