"""Cold-cache timing helper for the benchmarks.

`L2Flusher.flush()` evicts the 126 MB L2 of a B200 before a timed step: it
writes a 256 MiB buffer (the flush the benchmark contract asks for) and then
reads a second 256 MiB buffer, so that the L2 is left full of CLEAN lines.
Without the read, the next timed kernel would pay for ~126 MB of dirty
write-backs that are not part of its own traffic (measured: a 100 MB stream
drops from 4.3 to 3.9 TB/s effective).  Neither step is inside a timed region.
"""

from __future__ import annotations


class L2Flusher:
    def __init__(self, device, mib=256):
        import torch
        self._w = torch.empty(mib << 20, dtype=torch.uint8, device=device)
        self._r = torch.zeros((mib << 20) // 8, dtype=torch.float64, device=device)

    def flush(self):
        self._w.zero_()
        self._r.sum()
