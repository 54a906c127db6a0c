"""Operation histogram of a workload (host-side counters, no device cost).

Counts, per (op, level), how many times the *reference* algorithm would run
the op: a key switch over a batch of B components counts B, a cached
bootstrap diagonal used in a transform counts as one encode (the reference
re-encodes it on every call, bootstrap.py:219-236).  bench.py uses the
histogram to weight the CPU oracle's per-op timings into a modelled
reference step time.
"""

import contextlib
from collections import Counter

_enabled = [False]
_counts = Counter()


def enable(on=True):
    _enabled[0] = on
    if on:
        _counts.clear()


def enabled():
    return _enabled[0]


def count(op, level, n=1):
    if _enabled[0]:
        _counts[(op, int(level))] += int(n)


def snapshot():
    return {f"{op}@{lvl}": n for (op, lvl), n in sorted(_counts.items())}


@contextlib.contextmanager
def paused():
    """Suspend counting (the caller counts the reference's ops itself)."""
    prev = _enabled[0]
    _enabled[0] = False
    try:
        yield
    finally:
        _enabled[0] = prev
