"""Phase tracing: NVTX ranges always; synchronised host timers when
SPHC_TRACE=1 (adds syncs, so never on in a timed run)."""

import os
import time
from collections import defaultdict
from contextlib import contextmanager

import torch

ENABLED = os.environ.get("SPHC_TRACE") == "1"
TIMES = defaultdict(float)
COUNTS = defaultdict(int)


@contextmanager
def phase(name):
    if not ENABLED:
        yield
        return
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(name)
    t0 = time.perf_counter()
    try:
        yield
    finally:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        TIMES[name] += time.perf_counter() - t0
        COUNTS[name] += 1


def report(reset=True):
    rows = sorted(TIMES.items(), key=lambda kv: -kv[1])
    out = "\n".join(f"{k:40s} {v * 1e3:10.2f} ms  x{COUNTS[k]}" for k, v in rows)
    if reset:
        TIMES.clear()
        COUNTS.clear()
    return out
