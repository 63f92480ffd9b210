"""``threads=`` plumbing (reference ``pkg/src/nwave/parallel.py:20-25``).

The reference sets a process-global numba pool.  Here one host thread
drives one device stream, so the request is validated and the effective
count is always 1.
"""

from __future__ import annotations


def thread_cap() -> int:
    return 1


def resolve_threads(requested: int | None = 0) -> int:
    if requested is not None and int(requested) < 0:
        raise ValueError(f"threads must be >= 0, got {requested}")
    return 1
